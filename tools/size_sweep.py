"""Node-updates/s vs tree size (Fig 1's runtime-vs-size view):
the four real games, Goofspiel-6 and the synthetic at growing n_types, CFR+ f64,
one JSON line per game (CUDA events over graph replays / single launches)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gamegen
import paper_2408_14778_b200 as pb


def measure(name, desc, iters):
    g = pb.Game(desc)
    s = pb.Solver(g, variant="cfr+", precision=64)
    s.run(5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream)
    s.enqueue(iters)
    e1.record(s.stream)
    s.sync()
    ms = e0.elapsed_time(e1) / iters
    s.profile(3)                      # live-infoset counts for the byte model
    mb = s.model_bytes()["total"]
    row = {"game": name, "V": g.V, "it_per_s": round(1e3 / ms, 2), "node_updates_per_s": float(f"{g.V * 1e3 / ms:.4g}"),
           "model_GBps": round(mb / (ms * 1e-3) / 1e9, 1), "launches_per_iter": s.launches_per_iteration()}
    print(json.dumps(row), flush=True)
    del s, g


for name, iters in (("kuhn", 5000), ("leduc", 2000), ("goofspiel", 1000), ("liars_dice", 500)):
    measure(name, gamegen.by_name(name), iters)
measure("goofspiel6", gamegen.goofspiel(6), 300)
for n in (4, 8, 16, 24, 32, 40):
    t0 = time.time()
    d = gamegen.synthetic(n_types=n)
    measure(f"synthetic_n{n}", d, 50 if n >= 24 else 200)
    del d
