"""Short target for ncu: liar's dice CFR+ f64 through the subtree mode (default)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gamegen, paper_2408_14778_b200 as pb
g = pb.Game(gamegen.by_name(sys.argv[1] if len(sys.argv) > 1 else "liars_dice"))
s = pb.Solver(g, variant="cfr+", precision=64)
s.run(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
print("done", g.V, s.iteration, s.level_kernels())
