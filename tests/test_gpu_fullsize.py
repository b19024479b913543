"""BASELINE.json configs[4] at full size (synthetic n = 40, 965M nodes, CFR+,
f64) in the launch configuration bench.py times.  The oracle cannot run this
size, so the checks are:
  * the flattened sizes equal the closed-form counts of the generator;
  * the streaming path (k_bwd_stream, bench's configuration) and the tile
    kernels (k_bwd, FLAG_NO_STREAM: a separately written backward kernel) reach
    bit-identical state after T iterations -- the exact accumulation (reading
    Q8) makes the result independent of how members are grouped and summed;
  * properties that hold at any size: sigma and sigma_bar are distributions per
    infoset, CFR+ regrets are non-negative, the game is zero-sum so the two
    expected values cancel."""
import gc

import numpy as np
import pytest

import gamegen
from gamegen.synthetic_tree import synthetic_counts
import paper_2408_14778_b200 as pb

pytestmark = pytest.mark.gpu

T = 3


def _run(game, flags):
    s = pb.Solver(game, variant="cfr+", precision=64, flags=flags)
    s.run(T)
    out = dict(kernels=s.level_kernels(), avg=s.average_strategy(), cur=s.current_strategy(),
               ev=s.expected_values(), **s.state())
    del s
    gc.collect()
    return out


def test_full_size_stream_vs_tile_and_invariants(cuda):
    desc = gamegen.synthetic(n_types=40, seed=0)
    game = pb.Game(desc)
    del desc
    cnt = synthetic_counts(40)
    assert game.V == cnt["V"] and game.H == cnt["H"] and game.Q == cnt["Q"]

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
    ev = a["ev"]
    assert abs(ev[0] + ev[1]) <= 1e-9 * max(1.0, abs(ev[0])), ev
