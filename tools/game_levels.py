"""Per-level forward / backward time, kernel and model bytes of one game (not the
bench): python tools/game_levels.py battleship11 [cfr|cfr+] [64|32]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gamegen
import paper_2408_14778_b200 as pb
from gamegen.battleship import paper_battleship

name = sys.argv[1]
variant = sys.argv[2] if len(sys.argv) > 2 else "cfr"
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 64
d = paper_battleship(name) if name.startswith("battleship") else gamegen.by_name(name)
g = pb.Game(d)
print(name, g.info, flush=True)
for flags in (0, pb.FLAG_FORCE_STREAM):
    s = pb.Solver(g, variant=variant, precision=prec, flags=flags)
    s.run(3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream); s.enqueue(50); e1.record(s.stream); s.sync()
    ms = e0.elapsed_time(e1) / 50
    prof = s.profile(3)
    mb = s.model_bytes()
    print(f"flags={flags}: {ms:.4f} ms/it ({1e3 / ms:.1f} it/s), model {mb['total'] / 1e9:.3f} GB -> "
          f"{mb['total'] / ms / 1e6:.0f} GB/s; launches {s.launches_per_iteration()}", flush=True)
    for r in s.level_profile():
        print(f"   L{r['level']:2d} {str(r['bwd_kernel']):13s} fwd {r['fwd_ms']:.4f} ms bwd {r['bwd_ms']:.4f} ms "
              f"bytes fwd {r['fwd_bytes'] / 1e6:8.2f} MB bwd {r['bwd_bytes'] / 1e6:8.2f} MB", flush=True)
    del s
