"""GPU parity of the streaming (TMA bulk-copy) backward kernel k_bwd_stream
against the CPU oracle.  FLAG_FORCE_STREAM routes every eligible level through
it however small, so the small games the oracle finishes in seconds exercise the
same kernel the synthetic bench times."""
import pytest

import gamegen
import paper_2408_14778_b200 as pb
from tests.parity import run_pair

pytestmark = pytest.mark.gpu


def _stream_levels(solver):
    return [L for L, k in enumerate(solver.level_kernels()) if k == "k_bwd_stream"]


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("n_types,seed", [(2, 0), (3, 1), (5, 2)])
def test_stream_synthetic(cuda, n_types, seed, variant, precision):
    desc = gamegen.synthetic(n_types=n_types, seed=seed)
    out, s, o = run_pair(desc, variant, precision, 3, flags=pb.FLAG_FORCE_STREAM, checks=("state",))
    assert len(_stream_levels(s)) >= 4, s.level_kernels()


@pytest.mark.parametrize("name", ["goofspiel", "liars_dice", "kuhn", "leduc"])
def test_stream_real_games(cuda, name):
    desc = gamegen.by_name(name)
    T = 5 if name == "liars_dice" else 20
    for variant in (0, 1):
        out, s, o = run_pair(desc, variant, 64, T, flags=pb.FLAG_FORCE_STREAM)


def test_stream_vs_tile_kernels_same_bits(cuda):
    """The streaming kernel and the tile kernels give identical state (n_types = 6)."""
    import numpy as np
    desc = gamegen.synthetic(n_types=6, seed=3)
    g = pb.Game(desc)
    a = pb.Solver(g, variant="cfr+", precision=64, flags=pb.FLAG_FORCE_STREAM)
    b = pb.Solver(g, variant="cfr+", precision=64, flags=pb.FLAG_NO_STREAM)
    assert _stream_levels(a) and not _stream_levels(b)
    a.run(4)
    b.run(4)
    sa, sb = a.state(), b.state()
    for k in ("regret", "snum", "sden"):
        assert np.array_equal(sa[k], sb[k]), k
    assert np.array_equal(a.current_strategy(), b.current_strategy())


@pytest.mark.parametrize("precision", [64, 32])
def test_fused_forward_same_bits_as_separate_forward(cuda, precision):
    """The deepest level's forward pass fused into its streaming backward kernel
    gives the same state as the separate k_fwd launch (and the oracle)."""
    import numpy as np
    desc = gamegen.synthetic(n_types=4, seed=9)
    g = pb.Game(desc)
    a = pb.Solver(g, variant="cfr+", precision=precision, flags=pb.FLAG_FORCE_STREAM | pb.FLAG_FUSED_FORWARD)
    b = pb.Solver(g, variant="cfr+", precision=precision, flags=pb.FLAG_FORCE_STREAM)
    assert a.launches_per_iteration() == b.launches_per_iteration() - 1
    a.run(5)
    b.run(5)
    sa, sb = a.state(), b.state()
    for k in ("regret", "snum", "sden"):
        assert np.array_equal(sa[k], sb[k]), k
    run_pair(desc, 1, precision, 5, flags=pb.FLAG_FORCE_STREAM | pb.FLAG_FUSED_FORWARD, checks=("state",))


@pytest.mark.parametrize("precision", [64, 32])
def test_stream_general_sum_and_multiplayer(cuda, precision):
    """Value columns Pc > 1 (general-sum / 3-4 players) through the streaming kernel."""
    for desc in (gamegen.kuhn(3), gamegen.signal_game()):
        out, s, o = run_pair(desc, 1, precision, 12, flags=pb.FLAG_FORCE_STREAM)
    hit = 0
    for seed in range(12):
        desc = gamegen.random_game(seed, num_players=2 + seed % 3)
        out, s, o = run_pair(desc, seed % 5, precision, 8, flags=pb.FLAG_FORCE_STREAM)
        hit += "k_bwd_stream" in s.level_kernels()
    assert hit > 0


def test_stream_degenerate_games(cuda):
    """Tiny / degenerate trees under the forced streaming path: a single decision, a
    chance-only game, one-infoset matrix game."""
    for desc in (gamegen.single_decision(), gamegen.chance_pm1(2),
                 gamegen.matrix_game([[1.0, -1.0], [-1.0, 1.0]])):
        for variant in range(5):
            run_pair(desc, variant, 64, 6, flags=pb.FLAG_FORCE_STREAM)


@pytest.mark.parametrize("name", ["goofspiel", "liars_dice", "leduc"])
def test_stream_f32_unaligned_windows(cuda, name):
    """f32 through the streaming kernel: compact reach rows are 8 bytes, so tiles
    starting at an odd member need the TMA window offsets (child rows of odd
    length likewise)."""
    desc = gamegen.by_name(name)
    T = 4 if name == "liars_dice" else 12
    for variant in (1, 3):
        out, s, o = run_pair(desc, variant, 32, T, flags=pb.FLAG_FORCE_STREAM)
