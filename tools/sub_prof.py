"""Per-launch split of one subtree-mode iteration (cfr_solver_level_profile):
python tools/sub_prof.py game ..."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gamegen, paper_2408_14778_b200 as pb

for name in sys.argv[1:]:
    g = pb.Game(gamegen.by_name(name))
    for fl, lab in ((0, "default"), (pb.FLAG_NO_SUBTREE, "levels")):
        s = pb.Solver(g, variant="cfr+", precision=64, flags=fl)
        s.run(20)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream); s.enqueue(500); e1.record(s.stream); s.sync()
        us = e0.elapsed_time(e1) * 1e3 / 500
        p = s.profile(20)
        lv = s.level_profile()
        print(f"{name} {lab}: {us:.1f} us/it graph; profile fwd {p['fwd_ms']*1e3:.1f} bwd {p['bwd_ms']*1e3:.1f} us; "
              f"kernels {s.level_kernels()}", flush=True)
        print("   per level (fwd us, bwd us):", [(x['level'], round(x['fwd_ms'] * 1e3, 1), round(x['bwd_ms'] * 1e3, 1)) for x in lv], flush=True)
