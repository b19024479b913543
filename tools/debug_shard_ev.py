import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, gamegen, oracle, paper_2408_14778_b200 as pb
desc = gamegen.leduc()
g = pb.Game(desc)
s1 = pb.Solver(g, "cfr+", 64)
s1.run(3)
print("single EV", s1.expected_values())
ss = [pb.Solver(g, "cfr+", 64, rank=r, world_size=2) for r in range(2)]
def allreduce(which):
    bufs = [s.exchange_get(which) for s in ss]
    tot = bufs[0] + bufs[1]
    for s in ss: s.exchange_put(which, tot)
    return bufs, tot
for _ in range(3):
    for s in ss: s.phase(0)
    allreduce(0)
    for s in ss: s.phase(1)
    allreduce(1)
    for s in ss: s.phase(2)
for s in ss: s.phase(3)
bufs, tot = allreduce(0)
print("cut bufs", bufs, tot)
for s in ss: print("ev upper", s.phase(4))
# CFR-mode cut values for comparison
for s in ss: s.phase(0)
bufs, tot = allreduce(0)
print("cfr cut", bufs)
