"""Build + ctypes loading of libcfr_b200.so (the C ABI in include/cfr_b200.h).

Argument marshalling only: every step of the CFR iteration runs in the CUDA
kernels of csrc/solver.cu.  There is no CPU fallback: if the shared library is
missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
_CSRC = os.path.join(_HERE, "csrc")
LIB_PATH = os.path.join(_HERE, "libcfr_b200.so")
SOURCES = [os.path.join(_CSRC, f) for f in ("solver.cu", "flatten.cpp", "shard.cpp", "store.cpp", "cabi.cpp")]
HEADERS = [os.path.join(_CSRC, "game.hpp"), os.path.join(os.path.dirname(_HERE), "include", "cfr_b200.h")] + [
    os.path.join(_CSRC, "kernels", f) for f in sorted(os.listdir(os.path.join(_CSRC, "kernels"))) if f.endswith(".cuh")]

_NCCL = os.path.join(os.path.dirname(os.path.dirname(os.__file__)), "site-packages", "nvidia", "nccl")
if not os.path.isdir(_NCCL):
    import sysconfig
    _NCCL = os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    # IEEE arithmetic contract (reading Q9): no FMA contraction,
    # correctly rounded division/sqrt, no flush-to-zero, never --use_fast_math.
    "--fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off,-fopenmp",
    "-shared", "-lgomp",
    # NCCL (the torch-bundled 2.28 build) for the multi-GPU exchanges
    "-I" + os.path.join(_NCCL, "include"), "-L" + os.path.join(_NCCL, "lib"), "-l:libnccl.so.2",
    "-Xlinker", "-rpath=" + os.path.join(_NCCL, "lib"),
]

_lock = threading.Lock()
_lib = None


def _nvcc() -> str:
    for p in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.sep not in p or os.path.exists(p):
            return p
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, variant: str | None = None, defines=()) -> str:
    """nvcc -gencode arch=compute_100a,code=sm_100a ... -> libcfr_b200.so (in-tree).
    `variant` + `defines` build an experiment copy libcfr_b200.<variant>.so."""
    out = LIB_PATH if not variant else os.path.join(_HERE, f"libcfr_b200.{variant}.so")
    if not variant and not force and not needs_build():
        return LIB_PATH
    tmp = out + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, *SOURCES]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


class NativeError(RuntimeError):
    def __init__(self, status: int, name: str, msg: str):
        super().__init__(f"{name}: {msg}")
        self.status = status
        self.name = name


class GameDescC(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int64), ("num_players", ctypes.c_int32),
                ("parent", ctypes.c_void_p), ("player", ctypes.c_void_p), ("infoset", ctypes.c_void_p),
                ("action", ctypes.c_void_p), ("chance_prob", ctypes.c_void_p), ("utility", ctypes.c_void_p)]


class GameInfoC(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int64), ("num_terminals", ctypes.c_int64),
                ("num_decision", ctypes.c_int64), ("num_chance", ctypes.c_int64),
                ("num_infosets", ctypes.c_int64), ("num_pairs", ctypes.c_int64),
                ("num_players", ctypes.c_int32), ("depth", ctypes.c_int32),
                ("max_infoset_nodes", ctypes.c_int64), ("depth_homogeneous", ctypes.c_int32),
                ("zero_sum_2p", ctypes.c_int32)]


class SolverConfigC(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class DistC(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world_size", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p)]


# every symbol declared in include/cfr_b200.h: name -> (restype, argtypes)
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
SIGNATURES = {
    "cfr_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "cfr_last_error": (ctypes.c_char_p, []),
    "cfr_game_create": (ctypes.c_int, [_P, _P]),
    "cfr_game_destroy": (None, [_P]),
    "cfr_game_info": (ctypes.c_int, [_P, _P]),
    "cfr_game_qbase": (ctypes.c_int, [_P, _P]),
    "cfr_game_canonical": (ctypes.c_int, [_P, _P, _P]),
    "cfr_solver_workspace_bytes": (ctypes.c_int, [_P, _P, _P, _P]),
    "cfr_solver_create": (ctypes.c_int, [_P, _P, _P, ctypes.c_size_t, _P, _P, _P]),
    "cfr_solver_destroy": (None, [_P]),
    "cfr_solver_run": (ctypes.c_int, [_P, _I64]),
    "cfr_solver_enqueue": (ctypes.c_int, [_P, _I64]),
    "cfr_solver_sync": (ctypes.c_int, [_P]),
    "cfr_solver_iteration": (ctypes.c_int, [_P, _P]),
    "cfr_solver_average_strategy": (ctypes.c_int, [_P, _P]),
    "cfr_solver_current_strategy": (ctypes.c_int, [_P, _P]),
    "cfr_solver_get_state": (ctypes.c_int, [_P, _P, _P, _P]),
    "cfr_solver_set_state": (ctypes.c_int, [_P, ctypes.c_int64, _P, _P, _P]),
    "cfr_solver_expected_values": (ctypes.c_int, [_P, _I32, _P]),
    "cfr_solver_exploitability": (ctypes.c_int, [_P, _P, _P, _P]),
    "cfr_solver_launches_per_iteration": (ctypes.c_int, [_P, _P]),
    "cfr_solver_profile": (ctypes.c_int, [_P, _I64, _P]),
    "cfr_solver_model_bytes": (ctypes.c_int, [_P, _P]),
    "cfr_solver_level_kernels": (ctypes.c_int, [_P, _P, _I32, _P]),
    "cfr_solver_counters": (ctypes.c_int, [_P, _P, _I32, _P]),
    "cfr_solver_level_profile": (ctypes.c_int, [_P, _P, _I32, _P]),
    "cfr_nccl_unique_id": (ctypes.c_int, [_P]),
    "cfr_solver_phase": (ctypes.c_int, [_P, _I32, _P]),
    "cfr_solver_br_phase": (ctypes.c_int, [_P, _I32, _I32, _P]),
    "cfr_solver_br_passes": (ctypes.c_int, [_P, _P]),
    "cfr_solver_run_tracked": (ctypes.c_int, [_P, _I64, _I64, _P, _P]),
    "cfr_solver_exchange_size": (ctypes.c_int, [_P, _I32, _P]),
    "cfr_solver_exchange": (ctypes.c_int, [_P, _I32, _I32, _P, ctypes.c_size_t]),
    "cfr_solver_shard_info": (ctypes.c_int, [_P, _P]),
    "cfr_game_shard_info": (ctypes.c_int, [_P, _I32, _I32, _P]),
    "cfr_game_save_shards": (ctypes.c_int, [_P, _I32, ctypes.c_char_p]),
    "cfr_game_load_shard": (ctypes.c_int, [ctypes.c_char_p, _I32, _I32, _P]),
}


def load():
    """Load (building first if needed) the native library.  Raises on failure."""
    global _lib
    with _lock:
        if _lib is None:
            path = LIB_PATH
            alt = os.environ.get("CFR_B200_LIB_VARIANT")   # A/B kernel experiments: libcfr_b200.<variant>.so
            if alt:
                path = os.path.join(_HERE, f"libcfr_b200.{alt}.so")
            elif needs_build():
                build()
            L = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def check(status: int):
    if status != 0:
        L = load()
        raise NativeError(status, L.cfr_status_string(status).decode(), L.cfr_last_error().decode())
