"""Quick throughput probe (not the bench): it/s per game via CUDA events."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import gamegen, paper_2408_14778_b200 as pb

def probe(name, desc, variant, prec, iters):
    t0 = time.time(); g = pb.Game(desc); t1 = time.time()
    s = pb.Solver(g, variant=variant, precision=prec); t2 = time.time()
    s.run(3)
    st = s.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.enqueue(iters); e1.record(st); s.sync()
    ms = e0.elapsed_time(e1) / iters
    prof = s.profile(3)
    mb = s.model_bytes()
    print(f"{name:12s} {variant:5s} f{prec}: V={g.V} {ms*1e3:9.1f} us/it  {1e3/ms:10.1f} it/s  "
          f"{g.V*1e3/ms:.3e} node/s  launches={s.launches_per_iteration()} flatten={t1-t0:.1f}s create={t2-t1:.1f}s "
          f"prof={ {k: round(v,4) for k,v in prof.items()} } modelGB={mb['total']/1e9:.3f} -> {mb['total']/ms/1e6:.1f} GB/s",
          flush=True)

for name in ["kuhn", "leduc", "goofspiel", "liars_dice"]:
    d = gamegen.by_name(name)
    for v in ("cfr", "cfr+"):
        probe(name, d, v, 64, 200)
    probe(name, d, "cfr+", 32, 200)
for n in (8, 16):
    d = gamegen.synthetic(n_types=n)
    probe(f"synth{n}", d, "cfr+", 64, 10)
    probe(f"synth{n}", d, "cfr+", 32, 10)
