"""it/s of the four real games: persistent (default) vs per-level graph launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gamegen, paper_2408_14778_b200 as pb
for name, iters in (("kuhn", 5000), ("leduc", 2000), ("goofspiel", 1000), ("liars_dice", 300)):
    d = gamegen.by_name(name)
    g = pb.Game(d)
    for flags, tag in ((0, "default"), (pb.FLAG_NO_TINY, "graph")):
        for prec in (64, 32):
            s = pb.Solver(g, variant="cfr+", precision=prec, flags=flags)
            s.run(5)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s.stream); s.enqueue(iters); e1.record(s.stream); s.sync()
            ms = e0.elapsed_time(e1) / iters
            print(f"{name:11s} f{prec} {tag:10s}: {1e3 / ms:10.1f} it/s ({ms * 1e3:8.2f} us/it)", flush=True)
            del s
