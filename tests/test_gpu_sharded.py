"""Level-sharded multi-GPU path on ONE GPU: `world` solver ranks in
one process, the two per-iteration exchanges done here with exact host sums
(the NCCL mode performs the same sums with ncclAllReduce inside the graph).
Results must be bit-identical to the oracle for every world size."""
import numpy as np
import pytest

import gamegen
import oracle
import paper_2408_14778_b200 as pb
from tests.parity import assert_same

pytestmark = pytest.mark.gpu


def run_world(desc, variant, precision, T, world, shard_prefix=None, br=True, flags=0):
    g = pb.Game(desc)
    games = [g] * world
    if shard_prefix is not None:      # ranks load their own view from shard files
        g.save_shards(world, shard_prefix)
        games = [pb.Game.load_shard(shard_prefix, r, world) for r in range(world)]
    ss = [pb.Solver(games[r], variant=int(variant), precision=precision, rank=r, world_size=world, flags=flags)
          for r in range(world)]

    def allreduce(which):
        bufs = [s.exchange_get(which) for s in ss]
        tot = bufs[0].copy()
        for b in bufs[1:]:
            tot = tot + b          # int64 (exact) or values with one nonzero contribution (exact)
        for s in ss:
            s.exchange_put(which, tot)

    for _ in range(T):
        for s in ss:
            s.phase(pb.Solver.PHASE_LOWER)
        allreduce(pb.Solver.XCHG_CUT)
        for s in ss:
            s.phase(pb.Solver.PHASE_UPPER)
        allreduce(pb.Solver.XCHG_ACC)
        for s in ss:
            s.phase(pb.Solver.PHASE_UPDATE)
    for s in ss:
        assert s.iteration == T
    # readbacks: every rank returns the infosets it reports, zeros elsewhere
    avg = sum(s.average_strategy() for s in ss)
    cur = sum(s.current_strategy() for s in ss)
    st = [s.state() for s in ss]
    reg = sum(x["regret"] for x in st)
    sden = sum(x["sden"] for x in st)
    # EV under sigma_bar through the sharded values pass
    for s in ss:
        s.phase(pb.Solver.PHASE_EV_LOWER)
    allreduce(pb.Solver.XCHG_CUT)
    evs = [s.phase(pb.Solver.PHASE_EV_UPPER) for s in ss]
    out = dict(avg=avg, cur=cur, regret=reg, sden=sden, ev=evs, info=[s.shard_info() for s in ss],
               kernels=[s.level_kernels() for s in ss])
    if br:
        out["br"] = world_best_response(ss, allreduce)
    return out


def world_best_response(ss, allreduce):
    """Best response to sigma_bar of every player through the sharded BR passes
    (include/cfr_b200.h CFR_BR_*): per pass lower -> cut sum -> upper -> int64 sum
    of the deferred infosets' exact BR sums -> decide.  Returns [rank][player]."""
    P = ss[0].P
    for s in ss:
        s.br_phase(pb.Solver.BR_SETUP)
    passes = ss[0].br_passes()
    assert all(s.br_passes() == passes for s in ss)
    res = [[0.0] * P for _ in ss]
    for i in range(1, P + 1):
        for _ in range(passes):
            for s in ss:
                s.br_phase(pb.Solver.BR_LOWER, i)
            allreduce(pb.Solver.XCHG_CUT)
            for s in ss:
                s.br_phase(pb.Solver.BR_UPPER, i)
            allreduce(pb.Solver.XCHG_ACC)
            outs = [s.br_phase(pb.Solver.BR_DECIDE, i) for s in ss]
        for r, o in enumerate(outs):
            res[r][i - 1] = o[i - 1]
    return res


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("name,variant,precision,T", [("leduc", 1, 64, 30), ("leduc", 0, 32, 30),
                                                       ("goofspiel", 1, 64, 10), ("kuhn3", 0, 64, 20),
                                                       ("leduc", 3, 64, 20), ("goofspiel", 2, 32, 8)])
def test_sharded_bit_identical_to_oracle(cuda, name, variant, precision, T, world):
    desc = gamegen.by_name(name)
    o = oracle.Oracle(desc, precision=precision).run(T, variant)
    r = run_world(desc, variant, precision, T, world)
    os_ = o.state()
    assert_same("average strategy", r["avg"], os_["avg"], precision)
    assert_same("current strategy", r["cur"], os_["sigma"], precision)
    assert_same("regret", r["regret"], os_["regret"], precision)
    assert_same("S_den", r["sden"], os_["sden"], precision)
    for ev in r["ev"]:
        assert_same("EV(avg)", ev, o.expected_values(), precision)
    oe = o.exploitability()
    for b in r["br"]:   # every rank holds the same best-response values
        assert_same("BR", b, oe["br"], precision)
    if name != "kuhn3":
        assert r["info"][0]["cut"] >= 1


def test_sharded_liars_dice_and_random(cuda):
    desc = gamegen.liars_dice()
    o = oracle.Oracle(desc).run(3, 1)
    r = run_world(desc, 1, 64, 3, 4)
    assert_same("average strategy", r["avg"], o.state()["avg"], 64)
    for seed in range(6):
        d = gamegen.random_game(seed, num_players=2 + seed % 2, max_depth=7, max_nodes=6000)
        o = oracle.Oracle(d).run(8, seed % 2)
        r = run_world(d, seed % 2, 64, 8, 2 + seed % 3)
        assert_same("avg", r["avg"], o.state()["avg"], 64)
        for b in r["br"]:
            assert_same("BR", b, o.exploitability()["br"], 64)
        assert_same("regret", r["regret"], o.state()["regret"], 64)


def test_sharded_from_shard_files(cuda, tmp_path):
    desc = gamegen.goofspiel()
    o = oracle.Oracle(desc).run(6, 1)
    r = run_world(desc, 1, 64, 6, 3, shard_prefix=str(tmp_path / "g"))
    assert_same("average strategy", r["avg"], o.state()["avg"], 64)
    for ev in r["ev"]:
        assert_same("EV(avg)", ev, o.expected_values(), 64)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("variant,precision", [(1, 64), (0, 32), (2, 64)])
def test_sharded_synthetic_streaming_deferred_levels(cuda, world, variant, precision):
    """The synthetic tree sharded by player 1's type: player 2's infosets span the
    ranks, so player 2's levels run k_bwd_stream in deferred mode (exact partial
    sums into the exchange block, updated after the all-reduce) -- bit-identical
    to the oracle, like the fused levels."""
    desc = gamegen.synthetic(n_types=2 * world, c=(3, 2, 3, 2), seed=2)   # cut at player 1's type
    T = 4
    o = oracle.Oracle(desc, precision=precision).run(T, variant)
    r = run_world(desc, variant, precision, T, world, br=False, flags=pb.FLAG_FORCE_STREAM)
    os_ = o.state()
    assert_same("average strategy", r["avg"], os_["avg"], precision)
    assert_same("current strategy", r["cur"], os_["sigma"], precision)
    assert_same("regret", r["regret"], os_["regret"], precision)
    assert_same("S_den", r["sden"], os_["sden"], precision)
    for ev in r["ev"]:
        assert_same("EV(avg)", ev, o.expected_values(), precision)
    info = r["info"][0]
    assert info["deferred"] > 0
    # player 2's deepest decision level (depth D - 2) streams although its infosets span ranks
    for ks in r["kernels"]:
        assert ks.count("k_bwd_stream") >= 2, ks
