"""Battleship (PAPER.md Experiment 2; Table 5, Table 7 rows
P:676-698): OpenSpiel's battleship with (board width, board height, ship sizes,
shots per player) and ship values 1, emitted by the C++ generator
``battleship_gen.cpp`` (rules in its header; reading Q20)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .desc import GameDesc

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "battleship_gen.cpp")
_LIB = os.path.join(_HERE, "libbattleship_gen.so")
_lib = None

# PAPER.md Table 5 / Table 7: name -> (W, H, ship sizes, shots),
# and Table 7's (nodes, terminals, infosets, actions)
PAPER_CONFIGS = {
    "battleship0": ((2, 2, (1,), 2), (2581, 1936, 210, 8)),
    "battleship1": ((2, 2, (1, 2), 2), (21877, 16384, 1970, 10)),
    "battleship2": ((2, 2, (1,), 3), (23317, 17488, 2514, 8)),
    "battleship3": ((2, 3, (1,), 2), (33739, 28116, 1118, 12)),
    "battleship4": ((2, 2, (1, 2), 3), (324981, 243712, 46962, 10)),
    "battleship5": ((3, 3, (1,), 2), (426556, 379161, 5915, 18)),
    "battleship6": ((2, 3, (1,), 3), (843739, 703116, 33518, 12)),
    "battleship7": ((3, 4, (1,), 2), (2529949, 2319120, 19154, 24)),
    "battleship8": ((4, 4, (1,), 2), (14811409, 13885696, 61698, 32)),
    "battleship9": ((2, 3, (1,), 4), (21093739, 17578116, 1005518, 12)),
    "battleship10": ((3, 3, (1, 2), 2), (52081183, 46294416, 204980, 24)),
    "battleship11": ((4, 5, (1,), 2), (57920421, 55024400, 152402, 40)),
}


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-o", tmp, _SRC])
            os.replace(tmp, _LIB)
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.battleship_generate.restype = P
        L.battleship_generate.argtypes = [ctypes.c_int, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.battleship_num_nodes.restype = ctypes.c_int64
        L.battleship_num_nodes.argtypes = [P]
        L.battleship_num_infosets.restype = ctypes.c_int64
        L.battleship_num_infosets.argtypes = [P]
        L.battleship_copy.argtypes = [P, P, P, P, P, P]
        L.battleship_free.argtypes = [P]
        _lib = L
    return _lib


def battleship(width: int = 2, height: int = 2, ship_sizes=(1,), shots: int = 2,
               loss_multiplier: float = 2.0) -> GameDesc:
    L = _load()
    sz = np.ascontiguousarray(ship_sizes, dtype=np.int32)
    h = L.battleship_generate(int(width), int(height), ctypes.c_void_p(sz.ctypes.data), len(sz), int(shots),
                              float(loss_multiplier))
    if not h:
        raise ValueError("bad battleship parameters")
    try:
        V = L.battleship_num_nodes(h)
        parent = np.empty(V, dtype=np.int64)
        player = np.empty(V, dtype=np.int32)
        infoset = np.empty(V, dtype=np.int64)
        action = np.empty(V, dtype=np.int32)
        util = np.empty((V, 2), dtype=np.float64)
        L.battleship_copy(h, *(ctypes.c_void_p(a.ctypes.data) for a in (parent, player, infoset, action, util)))
    finally:
        L.battleship_free(h)
    name = f"battleship_{width}x{height}_{'-'.join(map(str, ship_sizes))}_{shots}"
    return GameDesc(name, 2, parent, player, infoset, action, np.zeros(V), util,
                    dict(width=width, height=height, ship_sizes=tuple(ship_sizes), shots=shots,
                         loss_multiplier=loss_multiplier))


def paper_battleship(name: str) -> GameDesc:
    (W, H, sizes, shots), _ = PAPER_CONFIGS[name]
    return battleship(W, H, sizes, shots)
