"""Subtree mode (k_sub + k_sub_update, kernels/subtree.cuh; SURVEY.md §8(f) f2,
PAPER.md P:401 / P:403): the levels below a cut run in one launch, each subtree's
reach / values / terminal utilities in shared memory, infoset sums added as exact
int64 slices with atomics.  Every result must be bit-identical to the CPU oracle
(the same IEEE operations; integer sums do not depend on the subtrees' order)."""
import numpy as np
import pytest

import gamegen
import oracle
import paper_2408_14778_b200 as pb
from tests.parity import assert_same, run_pair

pytestmark = pytest.mark.gpu

F = pb.FLAG_FORCE_SUBTREE


def sub_levels(s):
    k = s.level_kernels()
    assert "k_sub" in k, k
    return k


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("name", ["kuhn", "kuhn3", "leduc", "goofspiel"])
def test_subtree_real_games(cuda, name, variant, precision):
    out, s, o = run_pair(gamegen.by_name(name), variant, precision, 200, flags=F)
    sub_levels(s)


@pytest.mark.parametrize("precision", [64, 32])
def test_subtree_liars_dice(cuda, precision):
    out, s, o = run_pair(gamegen.liars_dice(), 1, precision, 100 if precision == 64 else 50, flags=F)
    sub_levels(s)


@pytest.mark.parametrize("variant", [2, 3, 4])
@pytest.mark.parametrize("name", ["leduc", "goofspiel"])
def test_subtree_variants(cuda, name, variant):
    out, s, o = run_pair(gamegen.by_name(name), variant, 64, 40, flags=F)
    sub_levels(s)


@pytest.mark.parametrize("seed", range(12))
def test_subtree_random_games(cuda, seed):
    # 2-4 players, chance nodes, general-sum payoffs (value columns Pc > 1) for odd seeds
    desc = gamegen.random_game(seed, num_players=2 + seed % 3, max_nodes=6000)
    out, s, o = run_pair(desc, seed % 5, 64, 25, flags=F)
    if any(k == "k_sub" for k in s.level_kernels()):
        return
    pytest.skip("random game not eligible for the subtree kernel (deferred infosets)")


def test_subtree_default_on_and_flags(cuda):
    """Default flags pick k_sub for a mid-size game k_tiny does not take; a flag that
    selects another kernel family, or CFR_FLAG_NO_SUBTREE, keeps the level kernels."""
    g = pb.Game(gamegen.liars_dice())
    assert "k_sub" in pb.Solver(g, variant="cfr+", precision=64).level_kernels()
    for fl in (pb.FLAG_NO_SUBTREE, pb.FLAG_NO_STREAM, pb.FLAG_FORCE_STREAM):
        assert "k_sub" not in pb.Solver(g, variant="cfr+", precision=64, flags=fl).level_kernels()


def test_subtree_same_bits_as_level_kernels(cuda):
    """Subtree mode and the per-level kernels give the same bits (Goofspiel, CFR+)."""
    desc = gamegen.goofspiel()
    g = pb.Game(desc)
    a = pb.Solver(g, variant="cfr+", precision=64, flags=F).run(300)
    b = pb.Solver(g, variant="cfr+", precision=64, flags=pb.FLAG_NO_SUBTREE).run(300)
    assert "k_sub" in a.level_kernels() and "k_sub" not in b.level_kernels()
    sa, sb = a.state(), b.state()
    for k in ("regret", "snum", "sden"):
        assert np.array_equal(sa[k], sb[k]), k
    assert np.array_equal(a.average_strategy(), b.average_strategy())


def test_subtree_synthetic_and_battleship(cuda):
    """A bench-shaped tree (40-way chance types, 20 actions) and a Battleship board."""
    out, s, o = run_pair(gamegen.synthetic(n_types=2, seed=3), 1, 64, 3, flags=F, checks=("state",))
    sub_levels(s)
    from gamegen.battleship import battleship
    out, s, o = run_pair(battleship(2, 2, (1,), 2), 0, 64, 30, flags=F)
    sub_levels(s)


def test_subtree_resume_and_tracked(cuda):
    """set_state (checkpoint / resume) and the in-graph exploitability curve run
    through the subtree mode as well."""
    desc = gamegen.goofspiel()
    g = pb.Game(desc)
    full = pb.Solver(g, variant="cfr+", precision=64, flags=F).run(60)
    half = pb.Solver(g, variant="cfr+", precision=64, flags=F).run(30)
    st = half.state()
    res = pb.Solver(g, variant="cfr+", precision=64, flags=F)
    res.set_state(30, st["regret"], st["snum"], st["sden"])
    res.run(30)
    assert np.array_equal(res.state()["regret"], full.state()["regret"])
    assert np.array_equal(res.average_strategy(), full.average_strategy())
    tr = pb.Solver(g, variant="cfr+", precision=64, flags=F).run_tracked(40, 20)
    o = oracle.Oracle(desc, precision=64).run(40, 1)
    assert_same("NashConv at T=40", [tr["nash_conv"][-1]], [o.exploitability()["nash_conv"]], 64)


@pytest.mark.parametrize("variant", [0, 1, 4])
@pytest.mark.parametrize("name", ["leduc", "goofspiel", "liars_dice"])
def test_subtree_longer_runs(cuda, name, variant):
    """Longer runs (the chaotic trajectory magnifies any difference), alternating
    updates included: one pass per player per iteration."""
    T = 300 if name == "liars_dice" else 1000
    out, s, o = run_pair(gamegen.by_name(name), variant, 64, T, flags=F, checks=("state",))
    n = s.launches_per_iteration()
    ref = pb.Solver(pb.Game(gamegen.by_name(name)), variant=1, precision=64, flags=F).launches_per_iteration()
    assert n == (2 * ref if variant == 4 else ref)


@pytest.mark.parametrize("staged", ["0", "1"])
@pytest.mark.parametrize("name,precision", [("leduc", 64), ("goofspiel", 64), ("liars_dice", 32),
                                            ("battleship3", 64)])
def test_subtree_table_layouts(cuda, name, precision, staged, monkeypatch):
    """Both k_sub layouts: tables and edge probabilities staged in shared memory,
    or read from global memory in each level step (CFR_SUB_STAGED forces one)."""
    from gamegen.battleship import paper_battleship
    desc = paper_battleship(name) if name.startswith("battleship") else gamegen.by_name(name)
    monkeypatch.setenv("CFR_SUB_STAGED", staged)
    out, s, o = run_pair(desc, 1, precision, 40, flags=F)
    sub_levels(s)


@pytest.mark.parametrize("precision", [64, 32])
def test_subtree_with_deferred_infosets(cuda, precision):
    """Goofspiel-6 (2.0 M nodes; infosets of up to 230 members, split across tiles and
    so deferred on the level path): below the cut every infoset is accumulated
    globally anyway, so the subtree mode takes them (k_deferred is not launched)."""
    desc = gamegen.goofspiel(6)
    out, s, o = run_pair(desc, 1, precision, 6, flags=F, checks=("state",))
    sub_levels(s)


@pytest.mark.parametrize("trunk", ["1", "0"])
@pytest.mark.parametrize("name,variant", [("leduc", 0), ("leduc", 4), ("liars_dice", 1)])
def test_subtree_chance_trunk(cuda, name, variant, trunk, monkeypatch):
    """A chance-only trunk (Leduc's and liar's dice's deals) folded into the subtree
    launches: k_sub computes each root's reach along its chance path and
    k_sub_update's last CTA the trunk values and the iteration count -- two launches
    per pass; CFR_SUB_TRUNK=0 keeps the trunk's level kernels.  Both match the
    oracle."""
    monkeypatch.setenv("CFR_SUB_TRUNK", trunk)
    T = 40 if name == "liars_dice" else 300
    out, s, o = run_pair(gamegen.by_name(name), variant, 64, T, flags=F)
    passes = 2 if variant == 4 else 1
    if trunk == "1":
        assert s.launches_per_iteration() == 2 * passes
    else:
        assert s.launches_per_iteration() > 2 * passes


def test_chance_trunk_tracked_and_profile(cuda):
    """Leduc through the folded chance trunk: the in-graph exploitability curve and
    the per-launch profile run on it, and the curve matches the oracle."""
    desc = gamegen.leduc()
    g = pb.Game(desc)
    s = pb.Solver(g, variant="cfr+", precision=64)
    assert s.launches_per_iteration() == 2
    tr = s.run_tracked(40, 20)
    o = oracle.Oracle(desc, precision=64).run(40, 1)
    assert list(tr["T"]) == [20, 40]
    assert_same("NashConv at T=40", [tr["nash_conv"][-1]], [o.exploitability()["nash_conv"]], 64)
    p = s.profile(3)
    assert p["bwd_ms"] > 0
    assert s.iteration == 43
