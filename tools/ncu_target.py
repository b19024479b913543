"""Short target for ncu: build the synthetic and run a few iterations (graph replay)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gamegen, paper_2408_14778_b200 as pb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 64
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
d = gamegen.synthetic(n_types=n)
g = pb.Game(d); del d
s = pb.Solver(g, variant="cfr+", precision=prec)
s.run(iters)
print("done", g.V, s.iteration)
