"""Synthetic battleship-shaped tree, emitted directly in
canonical level order with numpy.

Chance deals private types t1 then t2 (uniform over n); then a public alternating
tree, P1 first: every public decision node has b children, of which the first c[k]
(public depth k) are decision nodes; public depth len(c) children are all terminal.
Infoset = (own type, public node).  u1 = 2*(splitmix64(seed ^ (deal<<32 | pub_id))>>11)
*2^-53 - 1, u2 = -u1.  With n=40, b=20, c=[4,3,4,3,4,3,4,3]: V = 965,153,641,
916,896,000 terminals, H+ = 1,206,440 (shaped like PAPER.md Table 7's Battleship-11
row: 95 % terminals, ~0.1 % infosets per node).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .desc import GameDesc

DEFAULT_C = (4, 3, 4, 3, 4, 3, 4, 3)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x += np.uint64(0x9E3779B97F4A7C15)
        z = x
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _public_shape(b: int, c: tuple):
    """Per public depth k: number of all nodes n_all[k] and decision nodes n_dec[k]."""
    n_dec = [1]
    n_all = [1]
    for ck in c:
        n_all.append(n_dec[-1] * b)
        n_dec.append(n_dec[-1] * ck)
    # the last public depth's decisions have b terminal children
    n_all.append(n_dec[-1] * b)
    n_dec.append(0)
    return n_all, n_dec


def synthetic_counts(n_types: int = 40, b: int = 20, c: tuple = DEFAULT_C) -> dict:
    n_all, n_dec = _public_shape(b, tuple(c))
    deals = n_types * n_types
    pub_nodes = sum(n_all)
    pub_dec = sum(n_dec)
    V = 1 + n_types + deals * pub_nodes
    T = deals * (pub_nodes - pub_dec)
    h1 = n_types * sum(n_dec[k] for k in range(0, len(n_dec), 2))
    h2 = n_types * sum(n_dec[k] for k in range(1, len(n_dec), 2))
    return dict(V=V, T=T, H=h1 + h2, H1=h1, H2=h2, Q=(h1 + h2) * b, decision=deals * pub_dec,
                D=2 + len(c) + 1, levels=[1, n_types] + [deals * x for x in n_all])


_HERE = os.path.dirname(os.path.abspath(__file__))
_CSRC = os.path.join(_HERE, "synthetic_gen.c")
_CLIB = os.path.join(_HERE, "libsynthetic_gen.so")
_clib = None


def _load_c():
    """gcc -O2 -fopenmp build of synthetic_gen.c (multi-threaded emitter)."""
    global _clib
    if _clib is None:
        if not os.path.exists(_CLIB) or os.path.getmtime(_CLIB) < os.path.getmtime(_CSRC):
            tmp = _CLIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _CSRC])
            os.replace(tmp, _CLIB)
        L = ctypes.CDLL(_CLIB)
        P = ctypes.c_void_p
        L.synthetic_fill.argtypes = [ctypes.c_int64, ctypes.c_int64, P, ctypes.c_int64, ctypes.c_uint64,
                                     P, P, P, P, P, P]
        L.synthetic_fill.restype = ctypes.c_int
        _clib = L
    return _clib


def synthetic(n_types: int = 40, b: int = 20, c: tuple = DEFAULT_C, seed: int = 0, fast: bool = True) -> GameDesc:
    """The synthetic tree; `fast` uses the OpenMP C emitter (same arrays)."""
    if fast:
        return _synthetic_c(n_types, b, tuple(c), seed)
    return synthetic_numpy(n_types, b, c, seed)


def _synthetic_c(n_types, b, c, seed):
    cnt = synthetic_counts(n_types, b, c)
    V = cnt["V"]
    parent = np.empty(V, dtype=np.int64)
    player = np.empty(V, dtype=np.int32)
    infoset = np.empty(V, dtype=np.int64)
    action = np.empty(V, dtype=np.int32)
    chance = np.empty(V, dtype=np.float64)
    util = np.empty((V, 2), dtype=np.float64)
    ca = np.asarray(c, dtype=np.int64)
    p = lambda a: ctypes.c_void_p(a.ctypes.data)
    rc = _load_c().synthetic_fill(n_types, b, p(ca), len(c), seed, p(parent), p(player), p(infoset), p(action),
                                  p(chance), p(util))
    if rc != 0:
        raise ValueError("synthetic_fill failed")
    return GameDesc(f"synthetic_n{n_types}", 2, parent, player, infoset, action, chance, util,
                    dict(zero_sum=True, canonical=True, n_types=n_types, b=b, c=c, seed=seed, H=cnt["H"]))


def synthetic_numpy(n_types: int = 40, b: int = 20, c: tuple = DEFAULT_C, seed: int = 0) -> GameDesc:
    c = tuple(c)
    n_all, n_dec = _public_shape(b, c)
    n = n_types
    deals = n * n
    K = len(n_all)                       # public depths 0..K-1
    level_sizes = [1, n] + [deals * x for x in n_all]
    level_off = np.cumsum([0] + level_sizes)
    V = int(level_off[-1])
    pub_off = np.cumsum([0] + n_all)     # public-tree BFS id offsets
    # infoset numbering: P1 infosets first (public depths 0,2,...), then P2
    h_off = {}
    acc = 0
    for par in (0, 1):
        for k in range(K):
            if k % 2 == par and n_dec[k] > 0:
                h_off[k] = acc
                acc += n * n_dec[k]
    H = acc

    parent = np.empty(V, dtype=np.int64)
    player = np.empty(V, dtype=np.int32)
    infoset = np.full(V, -1, dtype=np.int64)
    action = np.empty(V, dtype=np.int32)
    chance = np.zeros(V, dtype=np.float64)
    util = np.zeros((V, 2), dtype=np.float64)

    # level 0 / 1 (chance)
    parent[0] = -1
    action[0] = -1
    player[0] = 0
    s1 = slice(level_off[1], level_off[2])
    parent[s1] = 0
    action[s1] = np.arange(n)
    player[s1] = 0
    chance[s1] = 1.0 / n
    for k in range(K):
        lo, hi = int(level_off[2 + k]), int(level_off[3 + k])
        m = n_all[k]
        idx = np.arange(hi - lo, dtype=np.int64)
        deal = idx // m
        j = idx % m                          # position among all public nodes at depth k
        if k == 0:
            parent[lo:hi] = level_off[1] + deal // n
            action[lo:hi] = (deal % n).astype(np.int32)
            chance[lo:hi] = 1.0 / n
            is_dec = np.ones(hi - lo, dtype=bool)
            dec_idx = np.zeros(hi - lo, dtype=np.int64)
        else:
            pd = j // b                      # parent's decision index at depth k-1
            a = j % b
            if k - 1 == 0:
                ppos = np.zeros_like(pd)
            else:
                ck2 = c[k - 2]
                ppos = (pd // ck2) * b + (pd % ck2)
            parent[lo:hi] = level_off[1 + k] + deal * n_all[k - 1] + ppos
            action[lo:hi] = a.astype(np.int32)
            if k < K - 1:
                is_dec = a < c[k - 1]
                dec_idx = pd * c[k - 1] + a
            else:
                is_dec = np.zeros(hi - lo, dtype=bool)
                dec_idx = np.zeros(hi - lo, dtype=np.int64)
        pl = 1 + (k % 2)
        player[lo:hi] = np.where(is_dec, pl, -1)
        if is_dec.any():
            own = (deal // n) if pl == 1 else (deal % n)
            inf = h_off[k] + own * n_dec[k] + dec_idx
            infoset[lo:hi] = np.where(is_dec, inf, -1)
        term = ~is_dec
        if term.any():
            pub_id = (pub_off[k] + j).astype(np.uint64)
            key = (np.uint64(seed) ^ ((deal.astype(np.uint64) << np.uint64(32)) | pub_id))
            z = _splitmix64(key) >> np.uint64(11)
            u1 = 2.0 * (z.astype(np.float64) * (2.0 ** -53)) - 1.0
            util[lo:hi, 0] = np.where(term, u1, 0.0)
            util[lo:hi, 1] = np.where(term, -u1, 0.0)
    return GameDesc(f"synthetic_n{n}", 2, parent, player, infoset, action, chance, util,
                    dict(zero_sum=True, canonical=True, n_types=n, b=b, c=c, seed=seed, H=H))
