"""N>1 host-side logic on CPU: world_size-2 gloo ranks shard the KV batch, plan their own
GPU node's routes through the C-ABI and exchange peer-segment handles, as bench.py does
over NCCL on a B200 box."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2604_00368_b200 as sp
    from paper_2604_00368_b200 import fabrics, sharding
    first, last = sharding.kv_shard(4096, rank, world)
    e = sp.Engine(fabrics.kv_offload(rank, sm_rails=1), None, device=rank)
    e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, f"g{rank}", [sp.BufferDesc(0, 1 << 20, 0x1000)]))
    e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, f"g{rank}", [sp.BufferDesc(0, 1 << 20, 0x2000)]))
    stream, backend = e.plan_candidates("hbm", "host")
    handle = bytes([rank]) * sp.IPC_HANDLE_BYTES  # stands in for a handle exported by spray_ipc_export
    shards = [None] * world
    dist.all_gather_object(shards, (first, last, stream.tolist(), backend, handle))
    peer = sharding.flow_peer(rank, world)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max-over-ranks timing reduction
    q.put((rank, shards, peer, float(t.item())))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_sharding_and_handle_exchange():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in ps:
        p.join(timeout=30)
        assert p.exitcode == 0
    res.sort()
    shards = res[0][1]
    assert shards == res[1][1]
    covered = []
    for first, last, stream, backend, handle in shards:
        covered.extend(range(first, last))
        assert backend == "cuda" and stream[0] == 1 and stream[1] == 1
    assert sorted(covered) == list(range(4096))
    assert [r[2] for r in res] == [1, 0]
    assert all(r[3] == 2.0 for r in res)
    assert shards[1][4] == bytes([1]) * sp_handle_bytes()


def sp_handle_bytes():
    import paper_2604_00368_b200 as sp
    return sp.IPC_HANDLE_BYTES
