"""PAPER.md Fig 3: exploitability (NashConv / P) of the average
strategy vs iterations, computed on the device inside the iteration graph
(cfr_solver_run_tracked), for Kuhn, Leduc, Goofspiel and liar's dice under CFR and
CFR+ -- written to profiles/r02_fig3_curves.json.  Timing of the tracked run is
reported beside the untracked it/s."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gamegen
import paper_2408_14778_b200 as pb

RUNS = [("kuhn", "cfr", 10000, 100), ("kuhn", "cfr+", 10000, 100), ("leduc", "cfr", 10000, 100),
        ("leduc", "cfr+", 10000, 100), ("goofspiel", "cfr+", 2000, 50), ("liars_dice", "cfr+", 1000, 50)]
out = []
for name, variant, T, every in RUNS:
    g = pb.Game(gamegen.by_name(name))
    s = pb.Solver(g, variant=variant, precision=64)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c = s.run_tracked(T, every)
    dt = time.perf_counter() - t0
    P = g.num_players
    expl = (c["nash_conv"] / P).tolist()
    row = {"game": name, "variant": variant, "iterations": T, "every": every, "T": c["T"].tolist(),
           "exploitability": expl, "ev_player1": c["ev"][:, 0].tolist(), "tracked_wall_s": round(dt, 3),
           "final_exploitability": expl[-1], "final_ev": c["ev"][-1].tolist()}
    out.append(row)
    print(f"{name:10s} {variant:5s} T={T}: exploitability {expl[0]:.3e} (T={every}) -> {expl[-1]:.3e}; "
          f"EV1 {c['ev'][-1][0]:+.6f}; {dt:.2f} s with {T // every} in-graph evaluations", flush=True)
os.makedirs("profiles", exist_ok=True)
json.dump(out, open("gpurun_out/r02_fig3_curves.json", "w"))
