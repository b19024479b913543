"""CPU oracle for arXiv 2408.14778 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The CUDA product
(``paper_2408_14778_b200``) never imports it and shares no code with it.

The arithmetic lives in ``cfr_oracle.cpp`` (plain recursive CFR/CFR+, see its
header for the equation-by-equation citations).  This module is ctypes
marshalling only, plus on-demand compilation with ``g++ -O2 -ffp-contract=off``.

Parity status: every function is pinned (see DESIGN.md §3 and tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cfr_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CXXFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++; IEEE RNE, no FMA contraction -- reading Q9)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CXXFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            c = ctypes
            P = c.c_void_p
            L.oracle_create.restype = P
            L.oracle_create.argtypes = [c.c_int64, c.c_int32, P, P, P, P, P, P, c.c_int32]
            L.oracle_destroy.argtypes = [P]
            L.oracle_last_error.restype = c.c_char_p
            L.oracle_dims.argtypes = [P, P]
            L.oracle_qbase.argtypes = [P, P]
            L.oracle_run.argtypes = [P, c.c_int32, c.c_int64]
            L.oracle_run.restype = c.c_int
            L.oracle_state.argtypes = [P, P, P, P, P, P, P]
            L.oracle_expected_values.argtypes = [P, c.c_int32, P, P]
            L.oracle_best_response.argtypes = [P, c.c_int32, P, c.c_int32, P, P]
            L.oracle_best_response.restype = c.c_int
            L.oracle_exploitability.argtypes = [P, c.c_int32, P, P, P, P, P]
            L.oracle_exploitability.restype = c.c_int
            L.oracle_slice_sum.argtypes = [P, c.c_int64, c.c_int32, P, P]
            _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


class OracleError(RuntimeError):
    pass


AVERAGE, CURRENT, GIVEN = 0, 1, 2


class Oracle:
    """Recursive CFR (variant 0) / CFR+ (variant 1) on one game, f64 or f32."""

    def __init__(self, desc, precision: int = 64):
        L = _load()
        self._L = L
        self.desc = desc
        self.precision = precision
        self._keep = [np.ascontiguousarray(desc.parent, dtype=np.int64),
                      np.ascontiguousarray(desc.player, dtype=np.int32),
                      np.ascontiguousarray(desc.infoset, dtype=np.int64),
                      np.ascontiguousarray(desc.action, dtype=np.int32),
                      np.ascontiguousarray(desc.chance_prob, dtype=np.float64),
                      np.ascontiguousarray(desc.utility, dtype=np.float64)]
        k = self._keep
        self._h = L.oracle_create(desc.num_nodes, desc.num_players, *(_ptr(x) for x in k), precision)
        if not self._h:
            raise OracleError(L.oracle_last_error().decode())
        dims = np.zeros(6, dtype=np.int64)
        L.oracle_dims(self._h, _ptr(dims))
        self.V, self.P, self.H, self.Q, self.E, self.root = (int(x) for x in dims)
        self.qbase = np.zeros(self.H + 1, dtype=np.int64)
        L.oracle_qbase(self._h, _ptr(self.qbase))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.oracle_destroy(h)
            self._h = None

    def run(self, iterations: int, variant: int = 0) -> "Oracle":
        if self._L.oracle_run(self._h, int(variant), int(iterations)) != 0:
            raise OracleError(self._L.oracle_last_error().decode())
        return self

    def state(self) -> dict:
        Q, H = self.Q, self.H
        out = {k: np.zeros(Q) for k in ("sigma", "regret", "snum", "avg")}
        out["sden"] = np.zeros(H)
        t = np.zeros(1, dtype=np.int64)
        self._L.oracle_state(self._h, _ptr(out["sigma"]), _ptr(out["regret"]), _ptr(out["snum"]),
                             _ptr(out["sden"]), _ptr(out["avg"]), _ptr(t))
        out["t"] = int(t[0])
        return out

    def average_strategy(self) -> np.ndarray:
        return self.state()["avg"]

    def current_strategy(self) -> np.ndarray:
        return self.state()["sigma"]

    def _which(self, strategy):
        if strategy is None or (isinstance(strategy, str) and strategy == "average"):
            return AVERAGE, None
        if isinstance(strategy, str) and strategy == "current":
            return CURRENT, None
        s = np.ascontiguousarray(strategy, dtype=np.float64)
        assert s.shape == (self.Q,)
        return GIVEN, s

    def expected_values(self, strategy=None) -> np.ndarray:
        w, s = self._which(strategy)
        out = np.zeros(self.P)
        self._L.oracle_expected_values(self._h, w, _ptr(s), _ptr(out))
        return out

    def best_response(self, player: int, strategy=None):
        w, s = self._which(strategy)
        val = np.zeros(1)
        acts = np.zeros(self.H, dtype=np.int32)
        if self._L.oracle_best_response(self._h, w, _ptr(s), int(player), _ptr(val), _ptr(acts)) != 0:
            raise OracleError(self._L.oracle_last_error().decode())
        return float(val[0]), acts

    def exploitability(self, strategy=None) -> dict:
        w, s = self._which(strategy)
        nc = np.zeros(1)
        ex = np.zeros(1)
        br = np.zeros(self.P)
        ev = np.zeros(self.P)
        if self._L.oracle_exploitability(self._h, w, _ptr(s), _ptr(nc), _ptr(ex), _ptr(br), _ptr(ev)) != 0:
            raise OracleError(self._L.oracle_last_error().decode())
        return dict(nash_conv=float(nc[0]), exploitability=float(ex[0]), br=br, ev=ev)


def slice_sum(x, E: int):
    """Exact 3x40-bit slice accumulation of x: (acc3, decoded)."""
    L = _load()
    x = np.ascontiguousarray(x, dtype=np.float64)
    acc = np.zeros(3, dtype=np.int64)
    dec = np.zeros(1)
    L.oracle_slice_sum(_ptr(x), x.shape[0], int(E), _ptr(acc), _ptr(dec))
    return acc, float(dec[0])
