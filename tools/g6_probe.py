"""Goofspiel-6 (2.0M nodes): it/s per precision / variant and the kernel per level."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gamegen, paper_2408_14778_b200 as pb
t0 = time.time()
d = gamegen.goofspiel(6)
g = pb.Game(d)
print(f"goofspiel6 V={g.V} D={g.D} H={g.H} build {time.time() - t0:.1f}s", flush=True)
for prec in (64, 32):
    s = pb.Solver(g, variant="cfr+", precision=prec)
    s.run(5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream); s.enqueue(200); e1.record(s.stream); s.sync()
    ms = e0.elapsed_time(e1) / 200
    print(f"f{prec}: {1e3 / ms:.1f} it/s ({ms * 1e3:.1f} us/it) launches {s.launches_per_iteration()} "
          f"kernels {s.level_kernels()}", flush=True)
    s.profile(3)
    for r in s.level_profile():
        print("  ", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()})
