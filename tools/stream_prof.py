"""Per-phase cycle split of k_bwd_stream (built with -DCFR_STREAM_PROFILE as the
'sprof' library variant): cycles per consumer warp per tile, summed over the
iteration's streaming levels.  python tools/stream_prof.py [n_types | battleshipK] [variant] [precision]"""
import ctypes
import os
import sys

os.environ["CFR_B200_LIB_VARIANT"] = "sprof"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import gamegen
import paper_2408_14778_b200 as pb
from paper_2408_14778_b200 import _native

arg = sys.argv[1] if len(sys.argv) > 1 else "40"
variant = sys.argv[2] if len(sys.argv) > 2 else "cfr+"
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 64
if arg.startswith("battleship"):
    from gamegen.battleship import paper_battleship
    d = paper_battleship(arg)
else:
    d = gamegen.synthetic(n_types=int(arg))
g = pb.Game(d)
del d
s = pb.Solver(g, variant=variant, precision=prec)
s.run(4)
L = _native.load()
f = L.cfr_debug_stream_profile
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(80, dtype=np.uint64)
f(buf.ctypes.data, 1)
s.run(1)
f(buf.ctypes.data, 1)
tiles = int(buf[64])
names = ["loop", "wait_full", "A_values", "A_store_reach", "A_compact", "A_barrier", "B+C", "end_barrier"]
per = buf[:64].reshape(8, 8).astype(np.float64) / tiles
print(f"tiles {tiles}; cycles per tile, per consumer warp (rows) and mark (columns):")
print("warp " + " ".join(f"{n:>13s}" for n in names))
for w in range(8):
    print(f"{w:4d} " + " ".join(f"{x:13.1f}" for x in per[w]))
print("mean " + " ".join(f"{x:13.1f}" for x in per.mean(0)))
