"""The paper's Experiment 2 games (Table 5 / Table 7): Battleship,
general-sum (two value columns on the device), through every kernel family and the
level-sharded path, bit-identical to the oracle (tests/parity.py)."""
import pytest

import paper_2408_14778_b200 as pb
from gamegen.battleship import paper_battleship
from tests.parity import run_pair
from tests.test_gpu_sharded import run_world
import oracle
from tests.parity import assert_same

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["battleship0", "battleship1", "battleship2", "battleship3"])
@pytest.mark.parametrize("variant,precision", [(0, 64), (1, 64), (0, 32), (1, 32)])
def test_small_battleships(cuda, name, variant, precision):
    """Battleship-0..3 (2.6k-34k nodes): default kernels (k_tiny where the state fits
    one CTA, else the per-level graph), T = 50."""
    run_pair(paper_battleship(name), variant, precision, 50)


@pytest.mark.parametrize("variant,precision", [(0, 64), (1, 32)])
def test_battleship_streaming_levels(cuda, variant, precision):
    """Battleship-5 (427k nodes) with every eligible level on k_bwd_stream (two value
    columns: the vectorized two-column value pass and row-byte-sized tiles)."""
    out, s, _ = run_pair(paper_battleship("battleship5"), variant, precision, 6, flags=pb.FLAG_FORCE_STREAM)
    assert "k_bwd_stream" in s.level_kernels()


def test_battleship_tile_kernels(cuda):
    """Battleship-4 (general-sum, ships [1;2], 3 shots) on the tile kernels only."""
    run_pair(paper_battleship("battleship4"), 0, 64, 8, flags=pb.FLAG_NO_TINY | pb.FLAG_NO_STREAM)


@pytest.mark.parametrize("world", [2, 4])
def test_battleship_sharded(cuda, world):
    """Battleship-3 level-sharded over 2 / 4 ranks (exact exchanges in one process)."""
    desc = paper_battleship("battleship3")
    T = 10
    o = oracle.Oracle(desc).run(T, 0)
    r = run_world(desc, 0, 64, T, world)
    os_ = o.state()
    assert_same("average strategy", r["avg"], os_["avg"], 64)
    assert_same("regret", r["regret"], os_["regret"], 64)
    for ev in r["ev"]:
        assert_same("EV(avg)", ev, o.expected_values(), 64)
    oe = o.exploitability()
    for b in r["br"]:
        assert_same("BR", b, oe["br"], 64)
