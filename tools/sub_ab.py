"""A/B of the subtree mode (k_sub) against the per-level kernels on the per-game
configurations: python tools/sub_ab.py [game ...]; prints us/it for default flags,
CFR_FLAG_FORCE_SUBTREE (k_sub even where k_tiny fits) and CFR_FLAG_NO_SUBTREE."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gamegen, paper_2408_14778_b200 as pb
from gamegen.battleship import paper_battleship

games = sys.argv[1:] or ["kuhn", "leduc", "liars_dice", "goofspiel", "goofspiel6", "battleship7", "battleship9"]


def desc_of(name):
    if name.startswith("battleship"):
        return paper_battleship(name)
    return gamegen.goofspiel(6) if name == "goofspiel6" else gamegen.by_name(name)


for name in games:
    d = desc_of(name)
    g = pb.Game(d)
    for prec in (64, 32):
        for variant in ("cfr", "cfr+"):
            res = []
            for lab, fl in (("default", 0), ("force_sub", pb.FLAG_FORCE_SUBTREE), ("no_sub", pb.FLAG_NO_SUBTREE)):
                s = pb.Solver(g, variant=variant, precision=prec, flags=fl)
                ks = sorted(set(k for k in s.level_kernels() if k))
                s.run(20)
                iters = 400 if g.V < 1e6 else 100
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                best = 1e9
                for _ in range(3):
                    e0.record(s.stream); s.enqueue(iters); e1.record(s.stream); s.sync()
                    best = min(best, e0.elapsed_time(e1) * 1e3 / iters)
                res.append(f"{lab} {best:8.1f} us/it {ks} launches={s.launches_per_iteration()}")
                del s
            print(f"{name} (V={g.V}) f{prec} {variant}: " + " | ".join(res), flush=True)
    del g
    torch.cuda.empty_cache()
