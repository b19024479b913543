"""A/B of solver flags on the synthetic (not the bench): python tools/ab_flags.py N PREC FLAGS,FLAGS,..."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gamegen, paper_2408_14778_b200 as pb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 64
flag_list = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0"])]
variant = sys.argv[4] if len(sys.argv) > 4 else "cfr+"
d = gamegen.synthetic(n_types=n)
g = pb.Game(d); del d
for flags in flag_list:
    s = pb.Solver(g, variant=variant, precision=prec, flags=flags)
    s.run(5)
    st = s.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 30
    e0.record(st); s.enqueue(iters); e1.record(st); s.sync()
    ms = e0.elapsed_time(e1) / iters
    prof = s.profile(3)
    mb = s.model_bytes()
    lv = s.level_profile()
    print(f"n={n} f{prec} {variant} flags={flags}: {ms:.4f} ms/it ({1e3/ms:.1f} it/s) dominant L{prof['dominant_level']} "
          f"{prof['dominant_ms']:.4f} ms -> {mb['dominant']/prof['dominant_ms']/1e6:.0f} GB/s; "
          f"fwd {prof['fwd_ms']:.4f} bwd {prof['bwd_ms']:.4f} model {mb['total']/1e9:.2f} GB", flush=True)
    print("   levels:", [(x['level'], round(x['fwd_ms'], 4), round(x['bwd_ms'], 4)) for x in lv], flush=True)
    del s
    torch.cuda.empty_cache()
