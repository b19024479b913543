"""GPU parity: the CUDA path (via the C ABI) against the CPU oracle, element by
element, on seeded synthetic inputs (DESIGN.md §3 recipe)."""
import numpy as np
import pytest

import gamegen
from tests.parity import run_pair

pytestmark = pytest.mark.gpu

SMALL = ["kuhn", "kuhn3", "leduc", "goofspiel"]


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("name", SMALL)
def test_real_games_T1_T10(cuda, name, variant, precision):
    desc = gamegen.by_name(name)
    out, s, o = run_pair(desc, variant, precision, 1)
    # continue the same solvers to T = 10 (parity holds along the trajectory)
    o.run(9, variant)
    s.run(9)
    from tests.parity import assert_same
    assert_same("sigma@10", s.current_strategy(), o.current_strategy(), precision)
    assert_same("avg@10", s.average_strategy(), o.average_strategy(), precision)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("precision", [64, 32])
def test_tiny_fixtures(cuda, variant, precision):
    for desc in (gamegen.single_decision(), gamegen.chance_pm1(2), gamegen.chance_pm1(1), gamegen.signal_game()):
        run_pair(desc, variant, precision, 5)


@pytest.mark.parametrize("seed", list(range(20)))
def test_random_games(cuda, seed):
    desc = gamegen.random_game(seed, num_players=2 + seed % 3)
    for variant in (0, 1):
        for precision in (64, 32):
            run_pair(desc, variant, precision, 20)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_node_order_and_infoset_labels_do_not_matter(cuda, seed):
    base = gamegen.leduc()
    desc = base.shuffled(seed).relabel_infosets(seed + 7)
    run_pair(desc, seed % 2, 64, 10)


def test_kuhn_1000_vanilla_f64(cuda):
    """BASELINE.json configs[0]: 1000 vanilla CFR iterations on Kuhn, fp64."""
    desc = gamegen.kuhn(2)
    out, s, o = run_pair(desc, 0, 64, 1000)
    ev = s.expected_values()
    assert abs(ev[0] + 1.0 / 18.0) <= 1e-4
    assert abs(ev[0] + 1.0 / 18.0) <= s.exploitability()["nash_conv"]


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("variant", [0, 1])
def test_leduc_1000(cuda, variant, precision):
    """BASELINE.json configs[1] (Leduc, CFR and CFR+, fp64 and fp32), T = 1000."""
    run_pair(gamegen.leduc(), variant, precision, 1000)


def test_liars_dice_cfr_plus(cuda):
    """BASELINE.json configs[2]: liar's dice 1x6, CFR+ on 1 B200 (T = 20 here)."""
    run_pair(gamegen.liars_dice(), 1, 64, 20)


def test_synthetic_small(cuda):
    """configs[4] shape at a size the oracle finishes in seconds (n_types = 2)."""
    desc = gamegen.synthetic(n_types=2)
    run_pair(desc, 1, 64, 2, checks=("state",))
    desc = gamegen.synthetic(n_types=2, seed=5)
    run_pair(desc, 0, 32, 2, checks=("state",))


def test_removed_persistent_flag_is_rejected(cuda):
    """CFR_FLAG_PERSISTENT selected the cooperative single-launch kernel, removed
    (slower than the graph): creation fails loudly."""
    import paper_2408_14778_b200 as pb
    with pytest.raises(pb.NativeError) as ei:
        pb.Solver(pb.Game(gamegen.kuhn()), variant="cfr", precision=64, flags=pb.FLAG_PERSISTENT)
    assert ei.value.name == "CFR_ERR_UNSUPPORTED"


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_tiny_shared_memory_kernel_matches_per_level_launches(cuda, variant, precision):
    """k_tiny (one CTA, all state in shared memory, T iterations per launch) and the
    per-level kernel graph give the same bits (and the oracle's: run_pair)."""
    import paper_2408_14778_b200 as pb
    games = [gamegen.kuhn(2), gamegen.kuhn(3), gamegen.matrix_game([[0, -1, 2], [1, 0, -1], [-1, 1, 0]]),
             gamegen.signal_game(), gamegen.random_game(3, num_players=2)]
    games.append(gamegen.leduc())   # f32: all in shared memory; f64: node values in global memory
    used = 0
    for desc in games:
        g = pb.Game(desc)
        a = pb.Solver(g, variant=variant, precision=precision)
        b = pb.Solver(g, variant=variant, precision=precision, flags=pb.FLAG_NO_TINY)
        used += a.launches_per_iteration() == 1
        a.run(17)
        b.run(17)
        sa, sb = a.state(), b.state()
        for k in ("regret", "snum", "sden"):
            assert np.array_equal(sa[k], sb[k]), (desc.name, k)
        assert np.array_equal(a.current_strategy(), b.current_strategy())
        assert np.array_equal(a.expected_values(), b.expected_values())
    assert used >= 4
    run_pair(gamegen.kuhn(2), variant, precision, 40)
    run_pair(gamegen.leduc(), variant, precision, 15)


@pytest.mark.parametrize("precision", [64, 32])
def test_int64_index_kernels(cuda, precision):
    """The 64-bit-index instantiations (used automatically for >= 2^31 nodes / pairs)
    on small games: tile, streaming and tiny paths, against the oracle."""
    import paper_2408_14778_b200 as pb
    F = pb.FLAG_INDEX64
    run_pair(gamegen.leduc(), 1, precision, 10, flags=F)
    run_pair(gamegen.goofspiel(), 3, precision, 6, flags=F | pb.FLAG_FORCE_STREAM)
    run_pair(gamegen.synthetic(n_types=2, seed=7), 1, precision, 2, flags=F | pb.FLAG_FORCE_STREAM, checks=("state",))
    for seed in range(4):
        run_pair(gamegen.random_game(seed, num_players=2 + seed % 3), 4, precision, 6, flags=F)
