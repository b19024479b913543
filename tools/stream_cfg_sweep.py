"""Sweep k_bwd_stream launch configurations on the n = 40 synthetic (not the bench):
python tools/stream_cfg_sweep.py PREC 'STAGES:TILE:FLAGS[:DEBUG]' ...  (TILE 0 = default;
DEBUG = timing-knob bits, effective only in a -DCFR_STREAM_EXPERIMENTS build)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gamegen, paper_2408_14778_b200 as pb

prec = int(sys.argv[1])
n = int(os.environ.get("SWEEP_N", "40"))
d = gamegen.synthetic(n_types=n)
g = pb.Game(d); del d
for cfg in sys.argv[2:]:
    s_, t, flags, *rest = cfg.split(":")
    os.environ["CFR_STREAM_DEBUG"] = rest[0] if rest else "0"
    os.environ["CFR_STREAM_STAGES"] = s_
    if t != "0": os.environ["CFR_STREAM_TILE"] = t
    else: os.environ.pop("CFR_STREAM_TILE", None)
    s = pb.Solver(g, variant="cfr+", precision=prec, flags=int(flags))
    s.run(5)
    st = s.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 30
    e0.record(st); s.enqueue(iters); e1.record(st); s.sync()
    ms = e0.elapsed_time(e1) / iters
    prof = s.profile(3)
    mb = s.model_bytes()
    lv = s.level_profile()
    print(f"f{prec} cfg={cfg}: {ms:.4f} ms/it ({1e3/ms:.1f} it/s) dominant L{prof['dominant_level']} "
          f"{prof['dominant_ms']:.4f} ms -> {mb['dominant']/prof['dominant_ms']/1e6:.0f} GB/s; "
          f"fwd {prof['fwd_ms']:.4f} bwd {prof['bwd_ms']:.4f} model {mb['total']/1e9:.2f} GB", flush=True)
    print("   levels:", [(x['level'], round(x['fwd_ms'], 4), round(x['bwd_ms'], 4)) for x in lv[5:]], flush=True)
    del s
    torch.cuda.empty_cache()
