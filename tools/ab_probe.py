"""A/B of backward-kernel variants on the synthetic (not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gamegen, paper_2408_14778_b200 as pb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
precs = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["64"])]
d = gamegen.synthetic(n_types=n)
g = pb.Game(d); del d
for prec in precs:
    for flags in (0, 4):
        s = pb.Solver(g, variant="cfr+", precision=prec, flags=flags)
        s.run(3)
        st = s.stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 20
        e0.record(st); s.enqueue(iters); e1.record(st); s.sync()
        ms = e0.elapsed_time(e1) / iters
        prof = s.profile(3)
        mb = s.model_bytes()
        print(f"n={n} f{prec} flags={flags}: {ms:.3f} ms/it ({1e3/ms:.1f} it/s) dominant L{prof['dominant_level']} "
              f"{prof['dominant_ms']:.3f} ms -> {mb['dominant']/prof['dominant_ms']/1e6:.0f} GB/s; "
              f"fwd {prof['fwd_ms']:.3f} bwd {prof['bwd_ms']:.3f}", flush=True)
        del s
        torch.cuda.empty_cache()
