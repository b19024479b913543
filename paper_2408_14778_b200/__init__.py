"""paper_2408_14778_b200 -- B200-native CFR / CFR+ (arXiv 2408.14778) behind a C ABI.

Thin Python binding of ``include/cfr_b200.h`` (ctypes).  PyTorch supplies the
device workspace (one uint8 tensor) and the CUDA stream; every step of the
iteration runs in the sm_100a kernels of ``csrc/solver.cu``.  There is no CPU
fallback: without the native library or a CUDA device the solver raises.

    game = Game(desc)                   # desc: gamegen.GameDesc-like arrays
    s = Solver(game, variant="cfr+", precision=64)
    s.run(1000)
    s.average_strategy(); s.expected_values(); s.exploitability()
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from ._native import NativeError, build, load

__all__ = ["Game", "Solver", "NativeError", "build", "load", "CFR", "CFR_PLUS", "nccl_unique_id"]


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 creates it; broadcast it to the others)."""
    L = load()
    buf = ctypes.create_string_buffer(128)
    _native.check(L.cfr_nccl_unique_id(buf))
    return buf.raw

CFR, CFR_PLUS, CFR_LINEAR, CFR_DISCOUNTED, CFR_PLUS_ALT = 0, 1, 2, 3, 4
# cfr_solver_config.flags (include/cfr_b200.h)
FLAG_NO_GRAPH = 1
FLAG_PERSISTENT = 2
FLAG_NO_PIPELINE = 4
FLAG_NO_PDL = 8
FLAG_NO_STREAM = 16
FLAG_FORCE_STREAM = 32
FLAG_FUSED_FORWARD = 64
FLAG_NO_TINY = 128
FLAG_INDEX64 = 256
FLAG_NO_SUBTREE = 512
FLAG_FORCE_SUBTREE = 1024


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


class Game:
    """cfr_game_create over the Def. 2.1 arrays (any node order)."""

    def __init__(self, desc=None, _handle=None):
        L = load()
        self._L = L
        if _handle is not None:
            self._h = _handle
            self._info()
            return
        self.num_players = int(desc.num_players)
        self._arrays = [np.ascontiguousarray(desc.parent, dtype=np.int64),
                        np.ascontiguousarray(desc.player, dtype=np.int32),
                        np.ascontiguousarray(desc.infoset, dtype=np.int64),
                        np.ascontiguousarray(desc.action, dtype=np.int32),
                        np.ascontiguousarray(desc.chance_prob, dtype=np.float64),
                        np.ascontiguousarray(desc.utility, dtype=np.float64)]
        a = self._arrays
        d = _native.GameDescC(a[0].shape[0], self.num_players, *(x.ctypes.data for x in a))
        h = ctypes.c_void_p()
        _native.check(L.cfr_game_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        self._arrays = None   # the library copied what it needs
        self._info()

    def _info(self):
        L = self._L
        info = _native.GameInfoC()
        _native.check(L.cfr_game_info(self._h, ctypes.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in info._fields_}
        self.V = self.info["num_nodes"]
        self.H = self.info["num_infosets"]
        self.Q = self.info["num_pairs"]
        self.D = self.info["depth"]
        self.num_players = self.info["num_players"]

    @classmethod
    def load_shard(cls, prefix: str, rank: int, world: int) -> "Game":
        """Load this rank's view written by save_shards (multi-GPU on one host)."""
        L = load()
        h = ctypes.c_void_p()
        _native.check(L.cfr_game_load_shard(prefix.encode(), int(rank), int(world), ctypes.byref(h)))
        return cls(_handle=h)

    def save_shards(self, world: int, prefix: str):
        _native.check(self._L.cfr_game_save_shards(self._h, int(world), prefix.encode()))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.cfr_game_destroy(h)
            self._h = None

    def qbase(self) -> np.ndarray:
        q = np.zeros(self.H + 1, dtype=np.int64)
        _native.check(self._L.cfr_game_qbase(self._h, _ptr(q)))
        return q

    SHARD_KEYS = ("cut", "n_cut", "owned_nodes", "local_nodes", "local_decision", "deferred", "deferred_pairs",
                  "world", "owned_cut", "reported")

    def shard_info(self, rank: int, world: int) -> dict:
        """Host-side level-sharding plan for (rank, world)."""
        out = np.zeros(10, dtype=np.int64)
        _native.check(self._L.cfr_game_shard_info(self._h, int(rank), int(world), _ptr(out)))
        return {k: int(v) for k, v in zip(self.SHARD_KEYS, out)}

    def canonical(self):
        c = np.zeros(self.V, dtype=np.int64)
        lp = np.zeros(self.D + 2, dtype=np.int64)
        _native.check(self._L.cfr_game_canonical(self._h, _ptr(c), _ptr(lp)))
        return c, lp


class Solver:
    """cfr_solver_* over a torch-allocated device workspace and a torch stream."""

    def __init__(self, game: Game, variant="cfr", precision: int = 64, device="cuda", stream=None,
                 flags: int = 0, rank: int = 0, world_size: int = 1, nccl_id: bytes | None = None):
        """world_size > 1: level-sharded solver for `rank`.  With
        `nccl_id` (128 bytes from nccl_unique_id(), broadcast by the caller) the
        exchanges run over NCCL inside the graph; without it the caller drives
        phase() / exchange_get() / exchange_put() ("external" mode)."""
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2408_14778_b200.Solver needs a CUDA device (no CPU fallback)")
        L = load()
        self._L = L
        self.game = game
        v = {"cfr": CFR, "vanilla": CFR, "cfr+": CFR_PLUS, "cfrplus": CFR_PLUS, "lcfr": CFR_LINEAR,
             "linear": CFR_LINEAR, "dcfr": CFR_DISCOUNTED, "discounted": CFR_DISCOUNTED,
             "cfr+alt": CFR_PLUS_ALT, "alternating": CFR_PLUS_ALT}.get(variant, variant)
        self.cfg = _native.SolverConfigC(int(v), int(precision), int(flags), 0)
        self.precision = int(precision)
        self.rank, self.world_size = int(rank), int(world_size)
        self._nid = None
        dist = None
        if self.world_size > 1:
            if nccl_id is not None:
                self._nid = ctypes.create_string_buffer(bytes(nccl_id), 128)
            dist = _native.DistC(self.rank, self.world_size,
                                 ctypes.cast(self._nid, ctypes.c_void_p) if self._nid is not None else None)
        self._dist = dist
        dptr = ctypes.byref(dist) if dist is not None else None
        nbytes = ctypes.c_size_t()
        _native.check(L.cfr_solver_workspace_bytes(game._h, ctypes.byref(self.cfg), dptr, ctypes.byref(nbytes)))
        self.workspace_bytes = int(nbytes.value)
        dev = torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        with torch.cuda.device(dev):
            self.stream = stream if stream is not None else torch.cuda.Stream(dev)
            # The workspace comes from torch's caching allocator on the current
            # stream; every kernel runs on self.stream.  Order the two: the solver
            # stream waits for pending work on the allocating stream (a reused
            # block may still be in use there), and the block is recorded as used
            # by the solver stream so the allocator never hands it out while
            # solver kernels may still write it.
            self.workspace = torch.empty(self.workspace_bytes + 256, dtype=torch.uint8, device=dev)
            self.stream.wait_stream(torch.cuda.current_stream(dev))
            self.workspace.record_stream(self.stream)
        base = self.workspace.data_ptr()
        aligned = (base + 255) & ~255
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _native.check(L.cfr_solver_create(game._h, ctypes.byref(self.cfg), ctypes.c_void_p(aligned),
                                              self.workspace_bytes, ctypes.c_void_p(self.stream.cuda_stream),
                                              dptr, ctypes.byref(h)))
        self._h = h
        self.Q, self.H, self.P = game.Q, game.H, game.num_players

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.cfr_solver_destroy(h)   # synchronises the solver stream first
            self._h = None

    # -- iteration
    def run(self, iterations: int) -> "Solver":
        _native.check(self._L.cfr_solver_run(self._h, int(iterations)))
        return self

    def enqueue(self, iterations: int) -> "Solver":
        _native.check(self._L.cfr_solver_enqueue(self._h, int(iterations)))
        return self

    def sync(self) -> "Solver":
        _native.check(self._L.cfr_solver_sync(self._h))
        return self

    @property
    def iteration(self) -> int:
        t = ctypes.c_int64()
        _native.check(self._L.cfr_solver_iteration(self._h, ctypes.byref(t)))
        return int(t.value)

    # -- readbacks (caller (h, a) order)
    def _out_buf(self, out):
        if out is None:
            return np.empty(self.Q)
        if out.dtype != np.float64 or out.shape != (self.Q,) or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a C-contiguous float64 array of shape ({self.Q},)")
        return out

    def average_strategy(self, out: np.ndarray | None = None) -> np.ndarray:
        """sigma_bar in caller (h, a) order; `out` (float64[Q], C-contiguous) is reused if given."""
        out = self._out_buf(out)
        _native.check(self._L.cfr_solver_average_strategy(self._h, _ptr(out)))
        return out

    def current_strategy(self, out: np.ndarray | None = None) -> np.ndarray:
        out = self._out_buf(out)
        _native.check(self._L.cfr_solver_current_strategy(self._h, _ptr(out)))
        return out

    def state(self) -> dict:
        r, sn, sd = np.zeros(self.Q), np.zeros(self.Q), np.zeros(self.H)
        _native.check(self._L.cfr_solver_get_state(self._h, _ptr(r), _ptr(sn), _ptr(sd)))
        return dict(regret=r, snum=sn, sden=sd)

    def set_state(self, T: int, regret, snum, sden) -> "Solver":
        """Resume from a checkpoint: T iterations done and the state() arrays
        (include/cfr_b200.h cfr_solver_set_state)."""
        r = np.ascontiguousarray(regret, dtype=np.float64)
        sn = np.ascontiguousarray(snum, dtype=np.float64)
        sd = np.ascontiguousarray(sden, dtype=np.float64)
        if r.shape != (self.Q,) or sn.shape != (self.Q,) or sd.shape != (self.H,):
            raise ValueError(f"state shapes must be ({self.Q},), ({self.Q},), ({self.H},)")
        _native.check(self._L.cfr_solver_set_state(self._h, int(T), _ptr(r), _ptr(sn), _ptr(sd)))
        return self

    def expected_values(self, which: str = "average") -> np.ndarray:
        if which not in ("average", "current"):
            raise ValueError(f"which must be 'average' or 'current', not {which!r}")
        out = np.zeros(self.P)
        w = 0 if which == "average" else 1
        _native.check(self._L.cfr_solver_expected_values(self._h, w, _ptr(out)))
        return out

    def exploitability(self) -> dict:
        nc, ex = ctypes.c_double(), ctypes.c_double()
        br = np.zeros(self.P)
        _native.check(self._L.cfr_solver_exploitability(self._h, ctypes.byref(nc), ctypes.byref(ex), _ptr(br)))
        return dict(nash_conv=nc.value, exploitability=ex.value, br=br)

    def run_tracked(self, iterations: int, every: int) -> dict:
        """PAPER.md Fig 3 curve: run `iterations` iterations and evaluate NashConv of
        sigma_bar on the device every `every` of them (one CUDA graph per
        evaluation, no host sync in between).  Returns arrays T, nash_conv, ev [.., P],
        br [.., P]."""
        rows_cap = max(1, int(iterations) // int(every))
        out = np.zeros((rows_cap, 2 + 2 * self.P))
        rows = ctypes.c_int64()
        _native.check(self._L.cfr_solver_run_tracked(self._h, int(iterations), int(every), _ptr(out),
                                                     ctypes.byref(rows)))
        out = out[:rows.value]
        return dict(T=out[:, 0].astype(np.int64), nash_conv=out[:, 1], ev=out[:, 2:2 + self.P],
                    br=out[:, 2 + self.P:])

    def br_passes(self) -> int:
        n = ctypes.c_int32()
        _native.check(self._L.cfr_solver_br_passes(self._h, ctypes.byref(n)))
        return int(n.value)

    # -- instrumentation
    def launches_per_iteration(self) -> int:
        n = ctypes.c_int64()
        _native.check(self._L.cfr_solver_launches_per_iteration(self._h, ctypes.byref(n)))
        return int(n.value)

    def profile(self, iterations: int) -> dict:
        out = np.zeros(5)
        _native.check(self._L.cfr_solver_profile(self._h, int(iterations), _ptr(out)))
        return dict(fwd_ms=out[0], bwd_ms=out[1], deferred_ms=out[2], dominant_ms=out[3], dominant_level=int(out[4]))

    # -- multi-GPU (external mode drives the phases; see include/cfr_b200.h)
    PHASE_LOWER, PHASE_UPPER, PHASE_UPDATE, PHASE_EV_LOWER, PHASE_EV_UPPER = 0, 1, 2, 3, 4
    BR_SETUP, BR_LOWER, BR_UPPER, BR_DECIDE = 0, 1, 2, 3
    XCHG_CUT, XCHG_ACC = 0, 1

    def phase(self, ph: int):
        out = np.zeros(self.P)
        _native.check(self._L.cfr_solver_phase(self._h, int(ph), _ptr(out)))
        return out

    def br_phase(self, ph: int, player: int = 1):
        out = np.zeros(self.P)
        _native.check(self._L.cfr_solver_br_phase(self._h, int(ph), int(player), _ptr(out)))
        return out

    def exchange_get(self, which: int) -> np.ndarray:
        n = ctypes.c_size_t()
        _native.check(self._L.cfr_solver_exchange_size(self._h, int(which), ctypes.byref(n)))
        dt = np.int64 if which == self.XCHG_ACC else (np.float64 if self.precision == 64 else np.float32)
        buf = np.zeros(n.value // np.dtype(dt).itemsize, dtype=dt)
        _native.check(self._L.cfr_solver_exchange(self._h, int(which), 0, _ptr(buf), n.value))
        return buf

    def exchange_put(self, which: int, buf: np.ndarray):
        buf = np.ascontiguousarray(buf)
        _native.check(self._L.cfr_solver_exchange(self._h, int(which), 1, _ptr(buf), buf.nbytes))

    def shard_info(self) -> dict:
        out = np.zeros(8, dtype=np.int64)
        _native.check(self._L.cfr_solver_shard_info(self._h, _ptr(out)))
        keys = ("cut", "n_cut", "owned_nodes", "local_nodes", "local_decision", "deferred", "deferred_pairs", "world")
        return {k: int(v) for k, v in zip(keys, out)}

    KERNEL_NAMES = {0: None, 1: "k_bwd", 2: "k_bwd_fast", 3: "k_bwd_stream", 4: "k_sub"}

    def level_kernels(self) -> list:
        """Backward kernel of each parent level (include/cfr_b200.h cfr_solver_level_kernels)."""
        D = max(1, self.game.D)
        out = np.zeros(D, dtype=np.int32)
        nl = ctypes.c_int32()
        _native.check(self._L.cfr_solver_level_kernels(self._h, _ptr(out), D, ctypes.byref(nl)))
        return [self.KERNEL_NAMES[int(x)] for x in out[:min(nl.value, D)]]

    def counters(self) -> dict:
        """Cumulative streaming-level work counters (include/cfr_b200.h cfr_solver_counters),
        summed over levels, plus the per-level table."""
        D = max(1, self.game.D)
        out = np.zeros(4 * D, dtype=np.int64)
        nl = ctypes.c_int32()
        _native.check(self._L.cfr_solver_counters(self._h, _ptr(out), D, ctypes.byref(nl)))
        per = out[:4 * min(nl.value, D)].reshape(-1, 4)
        tot = per.sum(0)
        return dict(live_infosets=int(tot[0]), live_pairs=int(tot[1]), infosets=int(tot[2]), pairs=int(tot[3]),
                    per_level=per.tolist())

    def level_profile(self) -> list:
        """Per level of the last profile(): forward / backward ms and model bytes."""
        D = max(1, self.game.D)
        out = np.zeros(4 * D)
        nl = ctypes.c_int32()
        _native.check(self._L.cfr_solver_level_profile(self._h, _ptr(out), D, ctypes.byref(nl)))
        per = out[:4 * min(nl.value, D)].reshape(-1, 4)
        kern = self.level_kernels()
        return [dict(level=L, fwd_ms=float(r[0]), bwd_ms=float(r[1]), fwd_bytes=float(r[2]), bwd_bytes=float(r[3]),
                     bwd_kernel=kern[L] if L < len(kern) else None) for L, r in enumerate(per)]

    def model_bytes(self) -> dict:
        out = np.zeros(5)
        _native.check(self._L.cfr_solver_model_bytes(self._h, _ptr(out)))
        return dict(total=out[0], fwd=out[1], bwd=out[2], update=out[3], dominant=out[4])
