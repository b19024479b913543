"""GPU parity of the discounted variants (reading Q18): linear CFR (2) and
DCFR(3/2, 0, 2) (3) against the oracle, every kernel family (tile, pipelined,
streaming, deferred, sharded)."""
import pytest

import gamegen
import paper_2408_14778_b200 as pb
from tests.parity import run_pair

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("variant", [2, 3])
@pytest.mark.parametrize("name", ["kuhn", "kuhn3", "leduc", "goofspiel"])
def test_discounted_real_games(cuda, name, variant, precision):
    run_pair(gamegen.by_name(name), variant, precision, 30)


@pytest.mark.parametrize("variant", [2, 3])
def test_discounted_matrix_game_and_random(cuda, variant):
    run_pair(gamegen.matrix_game([[0.0, -1.0, 2.0], [1.0, 0.0, -1.0], [-1.0, 1.0, 0.0]]), variant, 64, 200)
    for seed in range(6):
        run_pair(gamegen.random_game(seed, num_players=2 + seed % 3), variant, 64, 15)


@pytest.mark.parametrize("variant", [2, 3])
def test_discounted_streaming_kernel(cuda, variant):
    desc = gamegen.synthetic(n_types=3, seed=4)
    out, s, o = run_pair(desc, variant, 64, 4, flags=pb.FLAG_FORCE_STREAM, checks=("state",))
    assert "k_bwd_stream" in s.level_kernels()
    c = s.counters()
    assert c["live_infosets"] == c["infosets"]   # discounting: every infoset is updated


def test_discounted_liars_dice(cuda):
    run_pair(gamegen.liars_dice(), 3, 64, 5)


# ---- CFR+ with alternating updates (variant 4, reading Q19)
@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("name", ["kuhn", "kuhn3", "leduc", "goofspiel"])
def test_alternating_real_games(cuda, name, precision):
    run_pair(gamegen.by_name(name), 4, precision, 25)


def test_alternating_random_and_streaming(cuda):
    for seed in range(6):
        run_pair(gamegen.random_game(seed, num_players=2 + seed % 3), 4, 64, 12)
    out, s, o = run_pair(gamegen.synthetic(n_types=3, seed=2), 4, 64, 3, flags=pb.FLAG_FORCE_STREAM,
                         checks=("state",))
    assert "k_bwd_stream" in s.level_kernels()
    ref = pb.Solver(pb.Game(gamegen.kuhn(2)), variant="cfr+", precision=64, flags=pb.FLAG_NO_TINY)
    alt = pb.Solver(pb.Game(gamegen.kuhn(2)), variant="cfr+alt", precision=64, flags=pb.FLAG_NO_TINY)
    assert alt.launches_per_iteration() == 2 * ref.launches_per_iteration()
