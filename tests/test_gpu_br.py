"""Device best response / exploitability for general games (reading Q17) and the
in-graph exploitability curve (Fig 3), against the oracle.

Infosets that span depths, tiles or ranks are "deferred": their best-response
sums are accumulated exactly across the whole pass and decided after it, and the
pass repeats until every decision below is final (cfr_solver_br_passes).  Every
comparison is IEEE equality with the oracle (tests/parity.py)."""
import numpy as np
import pytest

import gamegen
import oracle
import paper_2408_14778_b200 as pb
from tests.parity import assert_same, run_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", list(range(12)))
def test_depth_spanning_infosets_best_response(cuda, seed):
    """Random perfect-recall games whose infosets pool nodes of several depths:
    state, EV, BR and NashConv bit-identical to the oracle (never unsupported)."""
    desc = gamegen.random_game(seed, num_players=2 + seed % 3, span_depths=True, max_depth=7)
    g = pb.Game(desc)
    assert not g.info["depth_homogeneous"]
    for variant in (0, 1):
        for precision in (64, 32):
            out, s, o = run_pair(desc, variant, precision, 15)
            assert s.br_passes() == g.D + 1


@pytest.mark.parametrize("seed", [0, 3])
def test_best_response_of_arbitrary_profiles(cuda, seed):
    """BR after T = 1, 2, 3 (three different sigma_bar profiles) on a depth-spanning
    game, each compared with the oracle's recursive best response."""
    desc = gamegen.random_game(seed, num_players=2, span_depths=True, max_depth=7)
    o = oracle.Oracle(desc)
    s = pb.Solver(pb.Game(desc), variant="cfr", precision=64)
    for _ in range(3):
        o.run(1, 0)
        s.run(1)
        se, oe = s.exploitability(), o.exploitability()
        assert_same("BR", se["br"], oe["br"], 64)
        assert_same("NashConv", [se["nash_conv"]], [oe["nash_conv"]], 64)


@pytest.mark.parametrize("name,variant,T,every", [("kuhn", 0, 200, 20), ("leduc", 1, 100, 10),
                                                   ("goofspiel", 1, 60, 15), ("random_span", 0, 40, 8)])
def test_tracked_exploitability_curve(cuda, name, variant, T, every):
    """cfr_solver_run_tracked: one in-graph evaluation every `every` iterations.
    Each row equals (bitwise) the oracle's EV / BR / NashConv at that T, and the
    solver ends in the same state as an untracked run."""
    desc = (gamegen.random_game(5, num_players=3, span_depths=True, max_depth=7) if name == "random_span"
            else gamegen.by_name(name))
    g = pb.Game(desc)
    s = pb.Solver(g, variant=variant, precision=64)
    curve = s.run_tracked(T, every)
    assert s.iteration == T
    assert list(curve["T"]) == list(range(every, T + 1, every))
    o = oracle.Oracle(desc)
    done = 0
    for k, t in enumerate(curve["T"]):
        o.run(int(t) - done, variant)
        done = int(t)
        oe = o.exploitability()
        assert_same(f"EV@{t}", curve["ev"][k], oe["ev"], 64)
        assert_same(f"BR@{t}", curve["br"][k], oe["br"], 64)
        assert_same(f"NashConv@{t}", [curve["nash_conv"][k]], [oe["nash_conv"]], 64)
    ref = pb.Solver(g, variant=variant, precision=64).run(T)
    assert np.array_equal(ref.average_strategy(), s.average_strategy())
    if name in ("kuhn", "leduc"):   # Fig 3: exploitability of sigma_bar falls
        assert curve["nash_conv"][-1] < curve["nash_conv"][0]


def test_tracked_streaming_and_sharded_shapes(cuda):
    """The tracked evaluation on the bench's kernel configuration (streaming levels)
    and an iteration count that is not a multiple of `every`."""
    desc = gamegen.synthetic(n_types=3, seed=4)
    s = pb.Solver(pb.Game(desc), variant="cfr+", precision=64, flags=pb.FLAG_FORCE_STREAM)
    curve = s.run_tracked(7, 3)
    assert list(curve["T"]) == [3, 6] and s.iteration == 7
    o = oracle.Oracle(desc).run(3, 1)
    assert_same("NashConv@3", [curve["nash_conv"][0]], [o.exploitability()["nash_conv"]], 64)
