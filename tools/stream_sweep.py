"""Sweep the streaming kernel's tile size / ring depth on the n=40 synthetic:
per configuration, mean ms per iteration (CUDA events, graph replay) and the
dominant backward level's time.  Env CFR_STREAM_TILE / CFR_STREAM_STAGES are read
at solver creation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gamegen
import paper_2408_14778_b200 as pb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
prec = int(os.environ.get("SWEEP_PRECISION", "64"))
configs = [tuple(int(x) for x in c.split(",")) for c in sys.argv[2:]] or [(240, 2, 0)]
configs = [c if len(c) == 3 else (c[0], c[1], 0) for c in configs]
d = gamegen.synthetic(n_types=n)
g = pb.Game(d)
del d
for tile, stages, dbg in configs:
    os.environ["CFR_STREAM_TILE"] = str(tile)
    os.environ["CFR_STREAM_STAGES"] = str(stages)
    os.environ["CFR_STREAM_DEBUG"] = str(dbg)
    s = pb.Solver(g, variant="cfr+", precision=prec)
    s.run(5) if dbg == 0 else s.enqueue(5)
    st = s.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.enqueue(30)
    e1.record(st)
    if dbg == 0:
        s.sync()
    else:
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    try:
        prof = s.profile(3)
    except pb.NativeError:
        prof = {"dominant_level": -1, "dominant_ms": 0, "bwd_ms": 0, "fwd_ms": 0}
    try:
        cnt = s.counters()
        live = f"live {cnt['live_infosets'] / max(1, cnt['infosets']):.3f}"
    except Exception:
        live = ""
    print(f"{live} tile={tile:4d} stages={stages} debug={dbg}: {ms:.3f} ms/it ({1e3 / ms:.1f} it/s)  dominant L{prof['dominant_level']} "
          f"{prof['dominant_ms']:.3f} ms  bwd {prof['bwd_ms']:.3f} fwd {prof['fwd_ms']:.3f}  kernels {s.level_kernels()}",
          flush=True)
    del s
    torch.cuda.empty_cache()
