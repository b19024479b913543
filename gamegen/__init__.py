"""Seeded, synthetic game-tree generators (test/bench INPUTS only).

This package is shared by the oracle (``oracle/``) and the CUDA product path
(``paper_2408_14778_b200``).  It holds NONE of the method's arithmetic: it only
emits the extensive-form game of PAPER.md Def. 2.1 as flat arrays in
the C-ABI layout of ``include/cfr_b200.h``:

    parent[V]      int64   f_parents; -1 at the root v0
    player[V]      int32   -1 terminal, 0 chance (nature i0), 1..P rational player
    infoset[V]     int64   f_h at player decision nodes, dense 0..H+-1; -1 elsewhere
    action[V]      int32   f_a: incoming action index 0..|A(h)|-1; -1 at the root
    chance_prob[V] float64 sigma_0 of the edge INTO v when parent(v) is a chance node
    utility[V, P]  float64 u(t, i+) at terminals (0 elsewhere)

Node order is arbitrary (the library canonicalises); generators emit DFS order
and ``GameDesc.shuffled`` produces a random permutation for order-independence
tests.  Rules follow SURVEY.md Appendix C (they reproduce PAPER.md Table 7,
P:659-673).
"""
from .desc import GameDesc, Builder
from .games import (kuhn, leduc, liars_dice, goofspiel, random_game, chance_pm1, single_decision, signal_game,
                    matrix_game)
from .synthetic_tree import synthetic, synthetic_numpy, synthetic_counts, DEFAULT_C

__all__ = [
    "GameDesc", "Builder", "kuhn", "leduc", "liars_dice", "goofspiel", "random_game",
    "chance_pm1", "single_decision", "signal_game", "matrix_game", "synthetic", "synthetic_numpy", "synthetic_counts", "DEFAULT_C",
    "by_name",
]


def by_name(name: str) -> GameDesc:
    """Named fixtures used by tests and bench (`kuhn`, `kuhn3`, `leduc`, `liars_dice`,
    `goofspiel`, `random:<seed>`, `synthetic:<scale>`)."""
    if name in ("kuhn", "kuhn2"):
        return kuhn(2)
    if name == "kuhn3":
        return kuhn(3)
    if name == "leduc":
        return leduc()
    if name == "liars_dice":
        return liars_dice()
    if name == "goofspiel":
        return goofspiel()
    if name.startswith("random:"):
        return random_game(int(name.split(":", 1)[1]))
    if name.startswith("synthetic"):
        parts = name.split(":")
        n = int(parts[1]) if len(parts) > 1 else 40
        return synthetic(n_types=n)
    raise KeyError(name)
