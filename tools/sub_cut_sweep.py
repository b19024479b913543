"""Subtree-mode cut sweep: python tools/sub_cut_sweep.py game ...; for each cut
level (CFR_SUB_CUT) that fits, us/it of CFR+ f64 / f32 under CFR_FLAG_FORCE_SUBTREE."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gamegen, paper_2408_14778_b200 as pb
from gamegen.battleship import paper_battleship


def desc_of(name):
    if name.startswith("battleship"):
        return paper_battleship(name)
    return gamegen.goofspiel(6) if name == "goofspiel6" else gamegen.by_name(name)


for name in sys.argv[1:]:
    g = pb.Game(desc_of(name))
    for prec in (64, 32):
        row = []
        for c in ["auto"] + list(range(1, min(g.D, 8))):
            if c == "auto":
                os.environ.pop("CFR_SUB_CUT", None)
            else:
                os.environ["CFR_SUB_CUT"] = str(c)
            s = pb.Solver(g, variant="cfr+", precision=prec, flags=pb.FLAG_FORCE_SUBTREE)
            ks = s.level_kernels()
            if "k_sub" not in ks:
                continue
            cut = ks.index("k_sub")
            s.run(20)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e9
            for _ in range(3):
                e0.record(s.stream); s.enqueue(300); e1.record(s.stream); s.sync()
                best = min(best, e0.elapsed_time(e1) * 1e3 / 300)
            row.append(f"{c}->cut {cut}: {best:.1f}")
            del s
        os.environ.pop("CFR_SUB_CUT", None)
        print(f"{name} f{prec} cfr+ (us/it): " + " | ".join(row), flush=True)
