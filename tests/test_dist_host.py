"""Host-side logic of the rank group on CPU (gloo, world_size 2): partition
ranges, the window-handle exchange, the pair-space shares, and the
ascending-partition reduction order that makes a multi-rank PCG bitwise
equal to the single-process run. No GPU needed."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, parts, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2008_00409_b200 import weft
        out = {}
        b, e = weft.rank_partitions(parts, world, rank)
        out["parts"] = (b, e)
        # handle exchange: opaque 64-byte blobs, rank order
        mine = bytes([rank + 1]) * weft.IPC_HANDLE_BYTES
        out["handles"] = weft.exchange_handles(mine, world)
        # row window of this rank for p vertices
        p = 1001
        pb = weft.make_partitions(p, parts)
        out["rows"] = (pb[b][0], pb[e - 1][1])
        # pair-space shares of the replicated broad phase
        out["share"] = weft.rank_share(123457, world, rank)
        # ordered all-reduce: each rank contributes its partitions' partials,
        # every rank sums all partitions in ascending order
        rng = np.random.default_rng(3)
        partials = rng.standard_normal(parts) * 10.0 ** rng.integers(-8, 8, parts)
        mine_p = np.zeros(parts)
        mine_p[b:e] = partials[b:e]
        allp = [None] * world
        dist.all_gather_object(allp, mine_p)
        slots = sum(allp)  # disjoint supports: exact
        tot = 0.0
        for d in range(parts):
            tot = tot + slots[d]
        out["sum"] = tot
        single = 0.0
        for d in range(parts):
            single = single + partials[d]
        out["single"] = single
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_rank_group_host_logic(parts):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, parts, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2008_00409_b200 import weft
    span = parts // world
    assert [res[r]["parts"] for r in range(world)] == [(r * span, (r + 1) * span) for r in range(world)]
    for r in range(world):
        assert res[r]["handles"] == [bytes([q + 1]) * weft.IPC_HANDLE_BYTES for q in range(world)]
    # row windows tile [0, p) in rank order
    assert res[0]["rows"][0] == 0 and res[world - 1]["rows"][1] == 1001
    assert all(res[r]["rows"][1] == res[r + 1]["rows"][0] for r in range(world - 1))
    # shares are exactly split_workload's ranges
    assert [res[r]["share"] for r in range(world)] == weft.split_workload(123457, world)
    # bitwise: multi-rank ordered reduction == single-process ascending sum
    assert all(res[r]["sum"] == res[r]["single"] for r in range(world))


def test_rank_partitions_errors():
    from paper_2008_00409_b200 import weft
    with pytest.raises(weft.TopologyError):
        weft.rank_partitions(4, 3, 0)
    with pytest.raises(weft.TopologyError):
        weft.rank_partitions(4, 2, 2)
    assert weft.rank_partitions(8, 4, 3) == (6, 8)
