"""A/B of solver-creation environment knobs on the n = 40 synthetic (not the bench):
python tools/ab_env.py PREC FLAGS 'NAME=VAL,NAME2=VAL|-' ... (- = no knob); each config
runs REPS times interleaved; prints ms/it and the dominant level's time."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gamegen, paper_2408_14778_b200 as pb

prec, flags = int(sys.argv[1]), int(sys.argv[2])
cfgs = sys.argv[3:]
reps = int(os.environ.get("AB_REPS", "3"))
n = int(os.environ.get("SWEEP_N", "40"))
variant = os.environ.get("AB_VARIANT", "cfr+")
d = gamegen.synthetic(n_types=n)
g = pb.Game(d); del d
known = set()
for c in cfgs:
    if c != "-":
        known |= {kv.split("=")[0] for kv in c.split(",")}
res = {c: [] for c in cfgs}
for r in range(reps):
    for c in cfgs:
        for k in known: os.environ.pop(k, None)
        if c != "-":
            for kv in c.split(","):
                k, v = kv.split("=")
                os.environ[k] = v
        s = pb.Solver(g, variant=variant, precision=prec, flags=flags)
        s.run(5)
        st = s.stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 40
        e0.record(st); s.enqueue(iters); e1.record(st); s.sync()
        ms = e0.elapsed_time(e1) / iters
        prof = s.profile(3)
        mb = s.model_bytes()
        res[c].append((ms, prof['dominant_ms']))
        print(f"f{prec} {variant} [{c}] rep {r}: {ms:.4f} ms/it ({1e3/ms:.1f} it/s) L{prof['dominant_level']} "
              f"{prof['dominant_ms']:.4f} ms -> {mb['dominant']/prof['dominant_ms']/1e6:.0f} GB/s "
              f"(frac {mb['dominant']/prof['dominant_ms']/1e6/6454.3:.3f})", flush=True)
        lv = s.level_profile()
        print("   levels:", [(x['level'], round(x['fwd_ms'], 4), round(x['bwd_ms'], 4)) for x in lv[5:]], flush=True)
        del s
        torch.cuda.empty_cache()
for c in cfgs:
    v = sorted(res[c])
    print(f"SUMMARY f{prec} {variant} [{c}]: best {v[0][0]:.4f} ms/it median {v[len(v)//2][0]:.4f}; dominant best {min(x[1] for x in v):.4f} ms")
