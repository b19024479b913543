"""N > 1 host-side logic on CPU with torch.distributed gloo, world_size 2:
the level-sharding plan is consistent across ranks (same cut, same deferred
exchange layout, owned node / cut / reported-infoset sets partition the game),
the NCCL-id bootstrap bytes broadcast intact, and the exact int64 slice sums that
the second exchange all-reduces combine to the single-process bits."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import gamegen
        import oracle
        import paper_2408_14778_b200 as pb

        out = {}
        for name in ("leduc", "goofspiel", "liars_dice"):
            g = pb.Game(gamegen.by_name(name))
            info = g.shard_info(rank, world)
            infos = [None] * world
            dist.all_gather_object(infos, info)
            out[name] = (infos, g.V, g.H, g.info)
        # bootstrap id (opaque 128 bytes) broadcast from rank 0
        blob = [os.urandom(128) if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, blob[0])
        out["ids_equal"] = all(x == ids[0] for x in ids) and len(ids[0]) == 128
        # exchange 2 semantics: per-rank exact partial sums, int64 sum-allreduce
        rng = np.random.default_rng(7)
        terms = rng.uniform(-1, 1, size=4000) * rng.choice([1, 1e-6, 1e-13], size=4000)
        part = terms[rank::world]
        acc, _ = oracle.slice_sum(part, 2)
        t = torch.tensor(acc, dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        full, full_dec = oracle.slice_sum(terms, 2)
        out["exact"] = np.array_equal(t.numpy(), full)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("world", [2])
def test_sharding_plan_and_exchange_semantics_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, err = q.get(timeout=600)
        assert err is None, err
        res[rank] = out
    for p in ps:
        p.join(timeout=60)
    out = res[0]
    assert out["ids_equal"] and out["exact"] and res[1]["exact"]
    for name, (infos, V, H, ginfo) in out.items() if False else [(k, v) for k, v in out.items() if k not in ("ids_equal", "exact")]:
        assert len({i["cut"] for i in infos}) == 1, name
        assert len({i["deferred"] for i in infos}) == 1 and len({i["deferred_pairs"] for i in infos}) == 1
        cut = infos[0]["cut"]
        assert cut >= 1, name
        assert sum(i["owned_cut"] for i in infos) == infos[0]["n_cut"]
        assert sum(i["reported"] for i in infos) == H
        below = sum(i["owned_nodes"] for i in infos)
        # every node below the cut is owned by exactly one rank
        trunk_nodes = infos[0]["local_nodes"] - infos[0]["owned_nodes"]
        assert below + trunk_nodes == V
        assert all(i["local_nodes"] - i["owned_nodes"] == trunk_nodes for i in infos)
