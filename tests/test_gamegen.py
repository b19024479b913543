"""Input generators: determinism, validity and the fast C emitter of the synthetic."""
import numpy as np
import pytest

import gamegen


FIELDS = ("parent", "player", "infoset", "action", "chance_prob", "utility")


@pytest.mark.parametrize("n,c", [(2, gamegen.DEFAULT_C), (3, (2, 3, 1)), (4, (3, 2))])
def test_synthetic_c_emitter_equals_numpy(n, c):
    a = gamegen.synthetic(n_types=n, c=c, seed=11)
    b = gamegen.synthetic_numpy(n_types=n, c=c, seed=11)
    for f in FIELDS:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_synthetic_shape_like_battleship():
    c = gamegen.synthetic_counts(40)
    assert abs(c["T"] / c["V"] - 0.95) < 0.001          # 95 % terminals
    assert c["decision"] == 48257600 and c["H"] / c["V"] < 0.002


def test_generators_deterministic():
    for name in ("kuhn", "leduc", "random:5"):
        a, b = gamegen.by_name(name), gamegen.by_name(name)
        for f in FIELDS:
            assert np.array_equal(getattr(a, f), getattr(b, f))


def test_random_games_perfect_recall_and_valid():
    import oracle
    for seed in range(30):
        d = gamegen.random_game(seed, num_players=1 + seed % 4)
        oracle.Oracle(d)   # validates structure
        # perfect recall: all members of an infoset share the owner's (infoset, action) history
        par = d.parent
        hist = {}
        for v in np.nonzero(d.player >= 1)[0]:
            pl = d.player[v]
            seq = []
            u = v
            while par[u] >= 0:
                p = par[u]
                if d.player[p] == pl:
                    seq.append((int(d.infoset[p]), int(d.action[u])))
                u = p
            key = int(d.infoset[v])
            assert hist.setdefault(key, tuple(seq)) == tuple(seq)


def test_zero_sum_fixtures():
    for name in ("kuhn", "leduc", "liars_dice", "goofspiel"):
        d = gamegen.by_name(name)
        t = d.player < 0
        assert np.array_equal(d.utility[t, 1], -d.utility[t, 0])


@pytest.mark.parametrize("name", ["battleship0", "battleship1", "battleship2", "battleship3", "battleship4",
                                  "battleship5", "battleship6", "battleship7", "battleship8", "battleship11"])
def test_battleship_table7_counts(name):
    """PAPER.md Table 7: nodes, terminals and infosets of the
    Experiment 2 battleship games, exactly (generator rules: DESIGN.md Q20)."""
    from gamegen.battleship import PAPER_CONFIGS, paper_battleship

    want = PAPER_CONFIGS[name][1]
    d = paper_battleship(name)
    assert (d.num_nodes, int((d.player == -1).sum()), d.num_infosets) == want[:3]
    assert d.utility.shape == (d.num_nodes, 2)
    # sanity of the general-sum payoffs (ship values 1, loss multiplier 2)
    term = d.player == -1
    assert set(np.unique(d.utility[term, 0])) <= {1.0, 0.0, -2.0, -1.0, 2.0, -4.0, -3.0, -5.0, -6.0, 3.0}
