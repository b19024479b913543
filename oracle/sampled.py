"""Sampled oracle for trees too large for the full oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may import this module.  It shares no code with the CUDA product.

`first_iteration_regrets` evaluates, for a few chosen infosets, the regret after
the first iteration from the uniform strategy sigma^1 (Eq 8), straight from
the definitions, walking only those infosets' members and their ancestors:

    r(h, a) = sum_{v in h} pi_check_{-i}(v) * (u_i(v.a) - u_i(v))      (Eq 6/7)
    u_i(v)  = sum_b sigma^1(h, b) u_i(v.b),  sigma^1(h, b) = 1 / |A(h)|    (Eq 1)
    pi_check_{-i}(v) = product over the edges above v of the chance probability
                       (chance node) or sigma^1 (node of a player other than i)  (Eq 2)

and returns R^1 = r (vanilla CFR) or max(r, 0) (CFR+, Eq 9 / reading Q3).  Only
infosets whose members' children are all terminal are accepted (the deepest
decision level of the synthetic tree), so u_i(v.a) is a stored payoff.

Node layout (gamegen.GameDesc): player 0 = chance, 1..P = players, -1 = terminal;
chance_prob[c] is the probability of the edge into c; the parent array must be
sorted (canonical BFS order), so the children of v are one searchsorted range.

Pinned by tests/test_oracle_pins.py against the full oracle (oracle.Oracle) on
every qualifying infoset of small trees.
"""
from __future__ import annotations

import numpy as np


def _children(parent: np.ndarray, v: int) -> np.ndarray:
    lo = int(np.searchsorted(parent, v, side="left"))
    hi = int(np.searchsorted(parent, v, side="right"))
    return np.arange(lo, hi, dtype=np.int64)


def qbase(desc) -> np.ndarray:
    """q offsets per infoset (caller numbering, actions in order): |A(h)| summed."""
    par = desc.parent
    dec = np.flatnonzero(desc.player > 0)
    cnt = np.searchsorted(par, dec, side="right") - np.searchsorted(par, dec, side="left")
    n = np.zeros(int(desc.infoset[dec].max()) + 1, dtype=np.int64)
    n[desc.infoset[dec]] = cnt
    return np.concatenate([[0], np.cumsum(n)])


def first_iteration_regrets(desc, infosets, plus: bool) -> dict:
    """{h: R^1(h, .)} for the given infosets (see module docstring)."""
    par, ply, inf, act = desc.parent, desc.player, desc.infoset, desc.action
    if not np.all(par[1:-1] <= par[2:]):
        raise ValueError("parent array must be sorted (canonical BFS order)")
    out = {}
    for h in infosets:
        members = np.flatnonzero(inf == h)
        i = int(ply[members[0]])
        r = None
        for v in members:
            ch = _children(par, int(v))
            ch = ch[np.argsort(act[ch], kind="stable")]
            if not np.all(ply[ch] == -1):
                raise ValueError(f"infoset {h}: children are not all terminal")
            n = len(ch)
            ua = desc.utility[ch, i - 1].astype(np.float64)
            uv = float(np.sum(ua / n))
            # pi_check_{-i}(v): walk to the root
            w, pi = int(v), 1.0
            while par[w] >= 0:
                p = int(par[w])
                if ply[p] == 0:
                    pi *= float(desc.chance_prob[w])
                elif ply[p] != i:
                    pi /= len(_children(par, p))
                w = p
            term = pi * (ua - uv)
            r = term if r is None else r + term
        out[int(h)] = np.maximum(r, 0.0) if plus else r
    return out
