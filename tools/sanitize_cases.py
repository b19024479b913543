"""Small runs for compute-sanitizer (memcheck / racecheck / synccheck):
Kuhn and Leduc (k_tiny, the subtree mode and the per-level kernels), Goofspiel and a
3-player general-sum random game through the subtree mode (k_sub), the synthetic n = 2 through
the forced streaming kernel (compact and fused forward, f64 / f32), device best
response, and one in-process world-2 sharded iteration.  Each case checks its
result against the oracle so a sanitizer-perturbed run cannot pass silently."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import gamegen
import oracle
import paper_2408_14778_b200 as pb

FAST = os.environ.get("SAN_FAST") == "1"


def check(desc, variant, prec, flags, T, br=True):
    s = pb.Solver(pb.Game(desc), variant=variant, precision=prec, flags=flags)
    s.run(T)
    o = oracle.Oracle(desc, precision=prec).run(T, 1 if variant == "cfr+" else 0)
    assert np.array_equal(s.current_strategy(), o.state()["sigma"]), desc.name
    if br:
        assert s.exploitability()["nash_conv"] == o.exploitability()["nash_conv"], desc.name
    print(f"ok {desc.name} {variant} f{prec} flags={flags} T={T} kernels={sorted({k for k in s.level_kernels() if k})}",
          flush=True)


check(gamegen.kuhn(), "cfr", 64, 0, 20)
check(gamegen.leduc(), "cfr+", 64, 0, 5)
check(gamegen.leduc(), "cfr+", 32, pb.FLAG_NO_TINY, 3)
# subtree mode (k_sub + k_sub_update: shared-memory subtrees, global int64 atomics)
check(gamegen.goofspiel(), "cfr", 64, 0, 2, br=not FAST)
check(gamegen.random_game(5, num_players=3, max_nodes=3000), "cfr", 64, pb.FLAG_FORCE_SUBTREE, 3, br=not FAST)
check(gamegen.leduc(), "cfr+", 32, pb.FLAG_FORCE_SUBTREE, 3, br=False)
syn = gamegen.synthetic(n_types=2, seed=1)
check(syn, "cfr+", 64, pb.FLAG_FORCE_STREAM, 2, br=not FAST)
check(syn, "cfr", 32, pb.FLAG_FORCE_STREAM | pb.FLAG_FUSED_FORWARD, 2, br=False)
if not FAST:
    check(gamegen.random_game(3, num_players=2, span_depths=True, max_depth=7), "cfr", 64, pb.FLAG_NO_TINY, 4)
    # one world-2 sharded iteration in external mode (tests/test_gpu_sharded.py drives it fully)
    from tests.test_gpu_sharded import run_world  # noqa: E402
    d = gamegen.goofspiel()
    out = run_world(d, pb.CFR_PLUS, 64, 2, 2, br=False)
    o = oracle.Oracle(d, precision=64).run(2, 1)
    assert np.array_equal(out["cur"], o.state()["sigma"])
    print("ok goofspiel sharded world 2", flush=True)
    # rank-spanning levels on the streaming kernel (deferred mode), world 2
    d = gamegen.synthetic(n_types=4, c=(3, 2, 3, 2), seed=2)
    out = run_world(d, pb.CFR_PLUS, 64, 2, 2, br=False, flags=pb.FLAG_FORCE_STREAM)
    o = oracle.Oracle(d, precision=64).run(2, 1)
    assert np.array_equal(out["cur"], o.state()["sigma"])
    print("ok synthetic sharded world 2 (deferred streaming levels)", flush=True)
    # checkpoint / resume
    g = pb.Game(gamegen.leduc())
    a = pb.Solver(g, variant="cfr+", precision=64).run(5)
    st = a.state()
    b = pb.Solver(g, variant="cfr+", precision=64)
    b.set_state(5, st["regret"], st["snum"], st["sden"]).run(2)
    print("ok resume", flush=True)
# release every solver and the caching allocator's blocks so memcheck's leak check
# reports only real leaks
import gc  # noqa: E402

import torch  # noqa: E402

gc.collect()
torch.cuda.synchronize()
torch.cuda.empty_cache()
print("all sanitizer cases done", flush=True)
