"""One process per GPU (the deployment shape of bench.py at N > 1): peer HBM shared through
spray_ipc_export / spray_ipc_open, exchanged over torch.distributed (gloo). The exported
tensors are deliberately sub-allocated by PyTorch's caching allocator (non-zero offset
inside their cudaMalloc block): the handle must carry the offset. Rank 0 moves bytes into
rank 1's tensor with its engine; a dataflow-gated chain forwards them on when >= 3 GPUs."""
import json
import multiprocessing as mp
import os
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2604_00368_b200 as sp
    from paper_2604_00368_b200 import fabrics
    try:
        pad = torch.zeros(4096 + 512 * rank, dtype=torch.uint8, device=f"cuda:{rank}")  # noqa: F841
        small = torch.zeros(64 << 10, dtype=torch.uint8, device=f"cuda:{rank}")  # noqa: F841
        buf = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{rank}")  # inside a pooled block
        e = sp.Engine(fabrics.peer_fabric([rank, (rank + 1) % world]), json.dumps({"b200": {"chunk_bytes": 65536}}), rank)
        e.start()
        cb = e.chunk_bytes()
        flags = torch.zeros(n // cb, dtype=torch.int32, device=f"cuda:{rank}")
        if rank == 0:
            sp.fill_splitmix(0, buf.data_ptr(), n, 77)
        hs = [None] * world
        dist.all_gather_object(hs, (sp.ipc_export(rank, buf.data_ptr()), sp.ipc_export(rank, flags.data_ptr())))
        opened = []
        e.register_segment(sp.SegmentDescriptor(f"w{rank}", sp.Medium.DEVICE, f"g{rank}",
                                                [sp.BufferDesc(0, n, buf.data_ptr())]))
        prep = None
        if rank + 1 < world:
            pb, pf = sp.ipc_open(rank, hs[rank + 1][0]), sp.ipc_open(rank, hs[rank + 1][1])
            opened += [pb, pf]
            e.register_segment(sp.SegmentDescriptor(f"w{rank + 1}", sp.Medium.DEVICE, f"g{rank + 1}",
                                                    [sp.BufferDesc(0, n, pb)]))
            if world > 2:
                e.gate_segment(f"w{rank + 1}", sp.Engine.GATE_PRODUCE, pf)
                if rank > 0:
                    e.gate_segment(f"w{rank}", sp.Engine.GATE_CONSUME, flags.data_ptr())
            prep = e.prepare_transfers([sp.TransferRequest(f"w{rank}", 0, f"w{rank + 1}", 0, n)])
        dist.barrier()
        state = "COMPLETE"
        if prep:
            b = e.allocate_batch()
            prep.run(b)
            state = e.batch_status(b).state.name
            e.free_batch(b)
        torch.cuda.synchronize()
        dist.barrier()
        ck = [None] * world
        dist.all_gather_object(ck, sp.checksum(rank, buf.data_ptr(), n))
        for p in opened:
            sp.ipc_close(p)
        e.stop()
        q.put((rank, state, ck))
    except Exception as ex:  # reported to the parent
        q.put((rank, f"error: {type(ex).__name__}: {ex}", None))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_ipc_peer_segments_one_process_per_gpu():
    world = min(3, _ngpu())
    n = 64 << 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(60)
    for rank, state, ck in res:
        assert state == "COMPLETE", (rank, state)
    ck = res[0][2]
    assert all(c == ck[0] for c in ck), ck
