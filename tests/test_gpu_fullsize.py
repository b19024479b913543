"""BASELINE.json configs[4] at full size (synthetic n = 40, 965M nodes, CFR+,
f64) in the launch configuration bench.py times.  The oracle cannot run this
size, so the checks are:
  * the flattened sizes equal the closed-form counts of the generator;
  * the streaming path (k_bwd_stream, bench's configuration) and the tile
    kernels (k_bwd, FLAG_NO_STREAM: a separately written backward kernel) reach
    bit-identical state after T iterations -- the exact accumulation (reading
    Q8) makes the result independent of how members are grouped and summed;
  * sampled outputs against the oracle: after one iteration, the regrets R^1
    of randomly drawn deepest-level infosets (Eq 6/7), their S_den = pi_bar
    (Eq 5 / Eq 10), their sigma^2 = RM(R^1) (Eq 9), and the expected value of
    sigma_bar^1 = sigma^1 (the uniform profile: a plain sum over all 917M
    terminals of pi(z) u(z)) equal oracle/sampled.py (the definitions, pinned
    against the full oracle in test_oracle_pins.py) within the north-star
    tolerance (1e-10 relative, f64);
  * properties that hold at any size: sigma and sigma_bar are distributions per
    infoset, CFR+ regrets are non-negative."""
import gc

import numpy as np
import pytest

import gamegen
from gamegen.synthetic_tree import synthetic_counts
import paper_2408_14778_b200 as pb
from oracle.sampled import first_iteration_pibar, first_iteration_regrets, qbase, regret_matching, uniform_ev

pytestmark = pytest.mark.gpu

T = 3


def _run(game, flags, iters=T, variant="cfr+"):
    s = pb.Solver(game, variant=variant, precision=64, flags=flags)
    s.run(iters)
    out = dict(kernels=s.level_kernels(), avg=s.average_strategy(), cur=s.current_strategy(),
               ev=s.expected_values(), **s.state())
    del s
    gc.collect()
    return out


def test_full_size_stream_vs_tile_and_invariants(cuda):
    desc = gamegen.synthetic(n_types=40, seed=0)
    game = pb.Game(desc)
    cnt = synthetic_counts(40)
    assert game.V == cnt["V"] and game.H == cnt["H"] and game.Q == cnt["Q"]

    q = qbase(desc)
    dec = np.flatnonzero(desc.player > 0)
    rng = np.random.default_rng(2408)
    hs = np.unique(desc.infoset[rng.choice(dec[-len(dec) // 10:], 8, replace=False)])
    pib = first_iteration_pibar(desc, hs)
    ev_u, mag = uniform_ev(desc)
    for variant, plus in (("cfr+", True), ("cfr", False)):   # CFR: signed regrets
        one = _run(game, 0, 1, variant)
        assert "k_bwd_stream" in one["kernels"], one["kernels"]
        ref = first_iteration_regrets(desc, hs, plus=plus)
        for h in hs:
            got = one["regret"][q[h]:q[h + 1]]
            tol = 1e-10 * np.abs(ref[h]).max()
            assert np.abs(ref[h]).max() > 0
            assert np.all(np.abs(got - ref[h]) <= tol), (variant, h, got, ref[h])
            assert abs(one["sden"][h] - pib[h]) <= 1e-10 * pib[h], (h, one["sden"][h], pib[h])
            want = regret_matching(ref[h])
            assert np.all(np.abs(one["cur"][q[h]:q[h + 1]] - want) <= 1e-10 * want.max()), (h, want)
        if not plus:
            assert any((ref[h] < 0).any() for h in hs)
        # EV of sigma_bar^1 = sigma^1: rounding of the device's Eq 1 tree sums is
        # bounded by (depth + 1) * 2^-53 * sum_z pi(z)|u(z)| (depth 11)
        assert np.all(np.abs(one["ev"] - ev_u) <= 12 * 2.0 ** -53 * mag), (one["ev"], ev_u, mag)
        assert np.all(np.abs(one["ev"] - ev_u) <= 1e-10 * np.abs(ev_u)), (one["ev"], ev_u)
        del one
    del desc, dec
    gc.collect()

    a = _run(game, 0)
    assert "k_bwd_stream" in a["kernels"], a["kernels"]
    b = _run(game, pb.FLAG_NO_STREAM)
    assert "k_bwd_stream" not in b["kernels"]
    for k in ("regret", "snum", "sden", "avg", "cur", "ev"):
        assert np.array_equal(a[k], b[k]), k

    q = game.qbase()
    for k in ("avg", "cur"):
        sums = np.add.reduceat(a[k], q[:-1])
        assert np.all(np.abs(sums - 1.0) <= 1e-12), (k, np.abs(sums - 1.0).max())
        assert np.all(a[k] >= 0.0)
    assert np.all(a["regret"] >= 0.0)
