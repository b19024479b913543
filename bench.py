#!/usr/bin/env python
"""Benchmark of one CFR+ iteration on the B200 -- bench contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A "step" is one full CFR iteration (all §8(a) rows: forward reach pass, backward
value pass, exact per-infoset aggregation, fused regret / average-strategy update
and regret matching) over the workload, default = BASELINE.json configs[4]: the
synthetic battleship-shaped tree (965,153,641 nodes, 1,206,440 infosets), f64,
CFR+.  Inputs are resident in HBM; the working set (~13 GB per iteration) is far
larger than the 126 MB L2, so no flush is needed between iterations.

Rank 0 prints ONE JSON line.  `value` = iterations/s (whole job), `ms_per_step`
from CUDA events on the solver's stream, max over ranks.  The `reference` arm
times the CPU oracle (test infrastructure) on a bounded sample of the same
workload and reports the same metric extrapolated by node count (the oracle's
cost is linear in V).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gamegen  # noqa: E402

METRIC = "CFR iterations/sec (node-updates/sec = V x it/s; achieved HBM GB/s vs peak)"
UNIT = "it/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n-types", type=int, default=40, help="synthetic size (40 = configs[4], ~1e9 nodes)")
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32])
    ap.add_argument("--variant", default="cfr+", choices=["cfr", "cfr+"])
    ap.add_argument("--no-games", action="store_true", help="skip the per-game (Kuhn/Leduc/...) lines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--no-variants", action="store_true", help="skip the configs[4] variant / precision lines")
    ap.add_argument("--variant-steps", type=int, default=50)
    ap.add_argument("--cpu-sample-types", type=int, default=4)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(n_types: int, precision: int):
    """dram__bytes_read+write per launch of the dominant kernel, from the committed
    ncu --set full summary (profiles/ncu_dominant.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_dominant.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        key = f"n{n_types}_f{precision}"
        return d.get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(n_types: int, variant: int, precision: int, seconds: float, V_full: int):
    """The oracle (as it stands) on a bounded sample of the workload, 1 core."""
    import oracle

    d = gamegen.synthetic(n_types=n_types)
    o = oracle.Oracle(d, precision=precision)
    del d
    with pinned_core() as pc:
        t0 = time.perf_counter()
        it = 0
        while True:
            o.run(1, variant)
            it += 1
            if time.perf_counter() - t0 >= seconds:
                break
        dt = time.perf_counter() - t0
    node_s = o.V * it / dt
    return {
        "value": node_s / V_full,
        "unit": UNIT,
        "cores": 1,
        "kind": "oracle",
        "pinned_core": pc.core,
        "node_updates_per_s": node_s,
        "sample": (f"synthetic n_types={n_types} ({o.V:,} nodes = {100.0 * o.V / V_full:.2f}% of the "
                   f"workload), {it} oracle iteration(s) in {dt:.1f} s; value = node-updates/s / V_workload "
                   f"(extrapolated by node count)"),
    }


# BASELINE.json configs[0-3] (+ Goofspiel-6, a paper-scale second real game) as
# secondary lines: (name, variant, precision, GPU iterations timed, oracle
# iterations timed).  The oracle (test infrastructure, as it stands, 1 pinned core)
# runs beside each line on this box's host.
GAME_LINES = (
    ("kuhn", "cfr", 64, 1000, 1000),          # configs[0]
    ("leduc", "cfr", 64, 10000, 2000),        # configs[1]
    ("leduc", "cfr", 32, 10000, 2000),
    ("leduc", "cfr+", 64, 10000, 2000),
    ("leduc", "cfr+", 32, 10000, 2000),
    ("liars_dice", "cfr+", 64, 1000, 100),    # configs[2]
    ("liars_dice", "cfr+", 32, 1000, 100),
    ("goofspiel", "cfr+", 64, 2000, 500),     # configs[3]
    ("goofspiel", "cfr+", 32, 2000, 500),
    ("goofspiel6", "cfr+", 64, 300, 10),
    ("battleship7", "cfr", 64, 300, 10),      # PAPER.md Experiment 2
    ("battleship7", "cfr", 32, 300, 10),
    ("battleship11", "cfr", 64, 100, 2),      # the paper's largest game
    ("battleship11", "cfr", 32, 100, 2),
)
# PAPER.md Table 2, vanilla CFR, RTX 4090 + CuPy, mean ms per iteration
PAPER_MS = {("kuhn", 64): 3.319, ("kuhn", 32): 3.362, ("leduc", 64): 6.269, ("leduc", 32): 6.178,
            ("liars_dice", 64): 10.766, ("liars_dice", 32): 8.443,
            # Table 5, 10 iterations
            ("battleship7", 64): 38.554, ("battleship7", 32): 20.437,
            ("battleship11", 64): 856.541, ("battleship11", 32): 446.369}


def shard_dir(V: int) -> str:
    """Directory for the per-rank shard files (≈ 15.5 bytes per node in total):
    $CFR_SHARD_DIR, else the first of /dev/shm, /tmp with room for them."""
    if os.environ.get("CFR_SHARD_DIR"):
        return os.environ["CFR_SHARD_DIR"]
    need = int(16 * V * 1.2)
    for d in ("/dev/shm", "/tmp"):
        try:
            st = os.statvfs(d)
            if st.f_bavail * st.f_frsize >= need:
                return d
        except OSError:
            continue
    return "/tmp"


# PAPER.md Table 9: seconds to serialize the game into the paper's sparse
# matrices (context for our generate + flatten + create)
PAPER_SETUP_S = {"kuhn": 0.010, "leduc": 1.051, "liars_dice": 34.264, "battleship7": 254.096,
                 "battleship11": 5470.082}


def host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model,
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None}


class pinned_core:
    """Run the oracle on one host core (restores the affinity afterwards)."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = min(self.old)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.old)


def game_desc(name: str):
    if name.startswith("battleship"):
        from gamegen.battleship import paper_battleship

        return paper_battleship(name)
    return gamegen.goofspiel(6) if name == "goofspiel6" else gamegen.by_name(name)


def per_game(pb, torch, with_oracle: bool):
    """Secondary lines of the metric: it/s and node-updates/s per BASELINE config
    (latency-bound, L2-resident games: no HBM fraction), the oracle beside each."""
    out = []
    for name, variant, prec, iters, oiters in GAME_LINES:
        t0 = time.perf_counter()
        d = game_desc(name)
        t1 = time.perf_counter()
        g = pb.Game(d)
        t2 = time.perf_counter()
        s = pb.Solver(g, variant=variant, precision=prec)
        t3 = time.perf_counter()
        s.run(5)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream)
        s.enqueue(iters)
        e1.record(s.stream)
        s.sync()
        ms = e0.elapsed_time(e1) / iters
        e = {"game": name, "variant": variant, "dtype": f"f{prec}", "iterations": iters,
             "it_per_s": round(1e3 / ms, 1), "node_updates_per_s": float(f"{g.V * 1e3 / ms:.4g}"), "V": g.V,
             "launches_per_iter": s.launches_per_iteration(), "kernels": sorted({k for k in s.level_kernels() if k})
             if s.launches_per_iteration() > 1 else ["k_tiny"],
             "setup_s": {"generate": round(t1 - t0, 3), "flatten": round(t2 - t1, 3), "solver_create": round(t3 - t2, 3)}}
        if name in PAPER_SETUP_S:
            e["setup_s"]["paper"] = PAPER_SETUP_S[name]
        del s
        if "k_sub" in e["kernels"]:
            # the same game on the per-level kernels (CFR_FLAG_NO_SUBTREE): what the
            # subtree mode buys on this line
            s = pb.Solver(g, variant=variant, precision=prec, flags=pb.FLAG_NO_SUBTREE)
            s.run(5)
            e0.record(s.stream)
            s.enqueue(iters)
            e1.record(s.stream)
            s.sync()
            ms_l = e0.elapsed_time(e1) / iters
            e["level_path"] = {"it_per_s": round(1e3 / ms_l, 1), "launches_per_iter": s.launches_per_iteration(),
                               "kernels": sorted({k for k in s.level_kernels() if k})
                               if s.launches_per_iteration() > 1 else ["k_tiny"]}
            e["subtree_speedup"] = round(ms_l / ms, 2)
            del s
        if with_oracle:
            import oracle

            o = oracle.Oracle(d, precision=prec)
            with pinned_core() as pc:
                t0 = time.perf_counter()
                o.run(oiters, 1 if variant == "cfr+" else 0)
                dt = time.perf_counter() - t0
            e["oracle"] = {"it_per_s": round(oiters / dt, 1), "node_updates_per_s": float(f"{g.V * oiters / dt:.4g}"),
                           "iterations": oiters, "cores": 1, "pinned_core": pc.core}
            e["gpu_over_oracle"] = round(e["it_per_s"] / e["oracle"]["it_per_s"], 2)
            del o
        pm = PAPER_MS.get((name, prec))
        if pm is not None:
            e["paper_context"] = {"it_per_s": round(1e3 / pm, 2), "variant": "cfr",
                                  "hardware": "RTX 4090 + CuPy (PAPER.md Table 2 P:426 / Table 5 P:570)",
                                  "ratio": round(e["it_per_s"] * pm / 1e3, 1)}
        out.append(e)
        del g
    return out


def synthetic_variants(pb, torch, game, dev, lines, steps: int):
    """configs[4] under the other variant / precision combinations (each its own
    solver on the same flattened game; CUDA events around `steps` graph replays)."""
    out = []
    for variant, prec in lines:
        s = pb.Solver(game, variant=variant, precision=prec, device=dev)
        s.run(3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream)
        s.enqueue(steps)
        e1.record(s.stream)
        s.sync()
        ms = e0.elapsed_time(e1) / steps
        prof = s.profile(3)
        mb = s.model_bytes()
        out.append({"variant": variant, "dtype": f"f{prec}", "steps": steps, "it_per_s": round(1e3 / ms, 2),
                    "ms_per_step": round(ms, 4), "node_updates_per_s": float(f"{game.V * 1e3 / ms:.4g}"),
                    "dominant_ms": round(prof["dominant_ms"], 4),
                    "dominant_GBps": round(mb["dominant"] / (prof["dominant_ms"] * 1e-3) / 1e9, 1),
                    "whole_step_model_GBps": round(mb["total"] / (ms * 1e-3) / 1e9, 1)})
        del s
        torch.cuda.empty_cache()
    return out


PAPER_CONTEXT = {
    "max_speedup_vs_openspiel_python": 401.2, "max_speedup_vs_openspiel_cpp": 203.6,
    "games": "tic_tac_toe f32 (P:487); Battleship-7 f32 (P:632)",
    "largest_game_node_updates_per_s": 1.30e8,
    "largest_game": "Battleship-11, 57.9M nodes, f32, 446.4 ms/it (P:602)",
    "hardware": "NVIDIA RTX 4090 (CuPy/cuSPARSE) vs AMD Ryzen 9 3900X (PAPER.md P:345)",
    "note": "context only: another machine, vanilla CFR, OpenSpiel baselines (P:7)",
}


def config_of(args, V=None, D=None, H=None, Q=None):
    """The `config` object: identical for both arms (same workload)."""
    w = f"synthetic_n{args.n_types}"
    if V is None:
        c = gamegen.synthetic_counts(args.n_types)
        V, D, H, Q = c["V"], c["D"], c["H"], c["Q"]
    return {"workload": f"{w}: {V:,} nodes, D={D}, {H:,} infosets, {Q:,} (h,a) pairs (BASELINE.json configs[4])",
            "variant": args.variant, "precision": f"f{args.precision}"}


def run_reference(args):
    """The oracle (as it stands, one pinned host core) on a bounded sample of the
    workload: each step = one oracle iteration over the n = cpu_sample_types
    synthetic; `value` is extrapolated to the full workload by node count (the
    oracle's cost per iteration is linear in V)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    variant = 1 if args.variant == "cfr+" else 0
    V_full = gamegen.synthetic_counts(args.n_types)["V"]
    import oracle

    d = gamegen.synthetic(n_types=args.cpu_sample_types)
    o = oracle.Oracle(d, precision=args.precision)
    del d
    with pinned_core() as pc:
        for _ in range(args.warmup):
            o.run(1, variant)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            o.run(1, variant)
        dt = time.perf_counter() - t0
    node_s = o.V * args.steps / dt
    value = node_s / V_full
    sample = (f"synthetic n_types={args.cpu_sample_types} ({o.V:,} nodes = {100.0 * o.V / V_full:.2f}% of the "
              f"workload), {args.steps} oracle iterations in {dt:.1f} s on 1 pinned core; value = node-updates/s / V_workload")
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup,
        # the measured time of one sample step (what the timed region holds); the
        # full-workload time per iteration is 1e3 / value (extrapolated)
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": f"f{args.precision}", "data": "synthetic",
        "config": config_of(args),
        "extrapolated": {"from_nodes": o.V, "to_nodes": V_full, "factor": V_full / o.V,
                         "full_workload_ms_per_iteration": 1e3 / value,
                         "note": "value = sample node-updates/s / V_workload (oracle cost linear in V)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "node_updates_per_s": node_s,
        "host": host_info(),
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2408_14778_b200 as pb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # a collective that never completes must fail the run, not hang it: the
        # library's NCCL communicator has no timeout of its own
        def _watchdog():
            time.sleep(float(os.environ.get("CFR_BENCH_TIMEOUT_S", "1500")))
            print(f"[rank {rank}] bench watchdog: no completion, aborting", file=sys.stderr, flush=True)
            os._exit(3)
        threading.Thread(target=_watchdog, daemon=True).start()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
    variant = 1 if args.variant == "cfr+" else 0

    # ---- setup (not timed): generate, flatten, upload.  N > 1:
    # rank 0 flattens once and writes one shard file per rank; every rank loads
    # only its own view; the two per-iteration exchanges run over NCCL.
    t0 = time.time()
    t_gen = t_flat = 0.0
    if world == 1:
        desc = gamegen.synthetic(n_types=args.n_types, seed=0)
        t_gen = time.time() - t0
        t0 = time.time()
        game = pb.Game(desc)
        t_flat = time.time() - t0
        del desc
        nid = None
    else:
        # rank 0 picks the directory (free space) and tells the others
        pbox = [os.path.join(shard_dir(gamegen.synthetic_counts(args.n_types)["V"]), f"cfr_synth_n{args.n_types}")
                if rank == 0 else None]
        dist.broadcast_object_list(pbox, src=0)
        prefix = pbox[0]
        files = [f"{prefix}.r{r}of{world}.cfrshard" for r in range(world)]
        if rank == 0 and not all(os.path.exists(f) for f in files):
            desc = gamegen.synthetic(n_types=args.n_types, seed=0)
            t_gen = time.time() - t0
            t0 = time.time()
            full = pb.Game(desc)
            del desc
            full.save_shards(world, prefix)
            del full
            t_flat = time.time() - t0
        dist.barrier()
        t0 = time.time()
        game = pb.Game.load_shard(prefix, rank, world)
        t_flat += time.time() - t0
        box = [pb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        nid = box[0]
    t0 = time.time()
    solver = pb.Solver(game, variant=args.variant, precision=args.precision, device=dev,
                       rank=rank, world_size=world, nccl_id=nid)
    t_up = time.time() - t0
    st = solver.stream

    # ---- warm-up, then the timed region (CUDA events on the solver stream)
    solver.run(args.warmup)
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    solver.enqueue(args.steps)
    e1.record(st)
    solver.sync()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    launches = solver.launches_per_iteration()
    shard_cut = solver.shard_info()["cut"] if world > 1 else None

    # ---- roofline of the dominant kernel (live CUDA events, un-graphed launches)
    prof = solver.profile(5)
    mb = solver.model_bytes()
    peak, peak_src = peaks()
    dom_ms = prof["dominant_ms"]
    achieved = mb["dominant"] / (dom_ms * 1e-3) / 1e9 if dom_ms > 0 else None
    kernels = solver.level_kernels()
    dom = prof["dominant_level"]
    cnt = solver.counters()["per_level"]
    live = None
    if 0 <= dom < len(cnt) and cnt[dom][2] > 0:
        live = round(cnt[dom][0] / cnt[dom][2], 4)
    levels = []
    for r in solver.level_profile():
        e = {"level": r["level"], "bwd_kernel": r["bwd_kernel"], "bwd_ms": round(r["bwd_ms"], 4),
             "fwd_ms": round(r["fwd_ms"], 4)}
        if r["bwd_ms"] > 0 and r["bwd_bytes"] > 0:
            e["bwd_GBps"] = round(r["bwd_bytes"] / (r["bwd_ms"] * 1e-3) / 1e9, 1)
        if r["fwd_ms"] > 0 and r["fwd_bytes"] > 0:
            e["fwd_GBps"] = round(r["fwd_bytes"] / (r["fwd_ms"] * 1e-3) / 1e9, 1)
        levels.append(e)
    roofline = {
        "bound": "hbm", "kernel": f"{kernels[dom]} (parent level {dom})",
        "live_infoset_fraction": live,
        "achieved": round(achieved, 1) if achieved else None, "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4) if achieved else None,
        "traffic": ncu_traffic(args.n_types, args.precision),
        "algorithmic_bytes_per_launch": mb["dominant"], "launch_ms": dom_ms, "peak_source": peak_src,
        "step_share": round(dom_ms / (prof["fwd_ms"] + prof["bwd_ms"] + prof["deferred_ms"]), 4),
        "whole_step_model_GBps": round(mb["total"] / (ms * 1e-3) / 1e9, 1),
        "levels": levels,
    }

    # ---- end to end through the public API with host buffers.  The host result
    # buffer is allocated (and the library's pinned staging warmed) before the
    # timed region, like any caller reusing its buffers.
    Q = solver.Q
    host_avg = np.empty(Q)
    solver.average_strategy(out=host_avg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        solver.run(1)                       # enqueue + sync + 16-byte status D2H
    avg = solver.average_strategy(out=host_avg)   # sigma_bar D2H into the host buffer
    e2e_dt = time.perf_counter() - t0
    w = args.precision // 8
    e2e = {"value": args.e2e_steps / e2e_dt, "unit": UNIT, "h2d_bytes_per_step": 0,
           "d2h_bytes_per_step": int(16 + Q * w / args.e2e_steps),
           "note": "per step: cfr_solver_run(1) (status read back); sigma_bar read back once per window"}
    assert np.isfinite(avg).all()

    # ---- configs[4] under the other variants / precisions (the headline solver
    # is released first: each solver holds the full device state)
    del solver
    torch.cuda.empty_cache()
    variants = None
    if rank == 0 and world == 1 and not args.no_variants:
        others = [(v, p) for v in ("cfr+", "cfr") for p in (64, 32) if (v, p) != (args.variant, args.precision)]
        variants = synthetic_variants(pb, torch, game, dev, others, args.variant_steps)

    games = None
    if rank == 0 and world == 1 and not args.no_games:
        games = per_game(pb, torch, with_oracle=not args.no_cpu)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.cpu_sample_types, variant, args.precision, args.cpu_seconds, game.V)

    if rank == 0:
        value = 1e3 / ms   # whole-job iterations/s (one iteration = the full tree, sharded over the ranks)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": f"f{args.precision}", "data": "synthetic",
            "config": config_of(args, game.V, game.D, game.H, game.Q),
            "parallelism": "single GPU" if world == 1 else
            f"level-sharded x{world} (cut depth {shard_cut}, NCCL exchanges)",
            "l2": "no flush: per-iteration working set ~12 GB >> 126 MB L2",
            "setup_s": {"generate": round(t_gen, 1), "flatten": round(t_flat, 1), "upload": round(t_up, 1),
                        "note": "one-time setup (PAPER.md P:397, Table 9), outside the timed region"},
            "node_updates_per_s": float(f"{game.V * value:.4g}"),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches * args.steps),
            "launches_per_step": launches,
            "clocks": clk,
            "synthetic_variants": variants,
            "per_game": games,
            "host": host_info(),
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        if rank == 0 and not os.environ.get("CFR_SHARD_DIR"):
            for f in files:   # the shard files are scratch (≈ 15 GB for configs[4])
                try:
                    os.remove(f)
                except OSError:
                    pass
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
