"""One process per GPU (the deployment shape of bench.py at N > 1): peer HBM shared through
spray_ipc_export / spray_ipc_open, exchanged over torch.distributed (gloo). The exported
tensors are deliberately sub-allocated by PyTorch's caching allocator (non-zero offset
inside their cudaMalloc block): the handle must carry the offset. Rank 0 moves bytes into
rank 1's tensor with its engine; with 3 ranks a dataflow-gated chain forwards them on
(rank 1 consumes granule by granule while rank 0 is still producing).

Two placements: "per_gpu" (one process per GPU, 2 or 3 GPUs) and "one_gpu" (three
processes time-sharing GPU 0: the same IPC export/open of sub-allocated tensors, the same
cross-process gated chain; CUDA IPC only forbids opening a handle in the exporting process,
not on the same device)."""
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


def _worker(rank, world, port, n, q, one_gpu=False):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dev = 0 if one_gpu else rank
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2604_00368_b200 as sp
    from paper_2604_00368_b200 import fabrics
    try:
        cuda = f"cuda:{dev}"
        pad = torch.zeros(4096 + 512 * rank, dtype=torch.uint8, device=cuda)  # noqa: F841
        small = torch.zeros(64 << 10, dtype=torch.uint8, device=cuda)  # noqa: F841
        buf = torch.zeros(n, dtype=torch.uint8, device=cuda)  # inside a pooled block
        e = sp.Engine(fabrics.peer_fabric([rank, (rank + 1) % world]), json.dumps({"b200": {"chunk_bytes": 65536}}), dev)
        e.start()
        cb = e.chunk_bytes()
        flags = torch.zeros(n // cb, dtype=torch.int32, device=cuda)
        if rank == 0:
            sp.fill_splitmix(dev, buf.data_ptr(), n, 77)
        hs = [None] * world
        dist.all_gather_object(hs, (sp.ipc_export(dev, buf.data_ptr()), sp.ipc_export(dev, flags.data_ptr())))
        opened = []
        e.register_segment(sp.SegmentDescriptor(f"w{rank}", sp.Medium.DEVICE, f"g{rank}",
                                                [sp.BufferDesc(0, n, buf.data_ptr())]))
        prep = None
        if rank + 1 < world:
            pb, pf = sp.ipc_open(dev, hs[rank + 1][0]), sp.ipc_open(dev, hs[rank + 1][1])
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
        dist.all_gather_object(ck, sp.checksum(dev, buf.data_ptr(), n))
        for p in opened:
            sp.ipc_close(p)
        e.stop()
        q.put((rank, state, ck))
    except Exception as ex:  # reported to the parent
        q.put((rank, f"error: {type(ex).__name__}: {ex}", None))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("placement", ["one_gpu", "per_gpu"])
def test_ipc_peer_segments_one_process_per_gpu(placement):
    if _ngpu() < 1:
        pytest.skip("needs a GPU")
    if placement == "per_gpu" and _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    one = placement == "one_gpu"
    world = 3 if one else min(3, _ngpu())
    n = 64 << 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, q, one)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(60)
    for rank, state, ck in res:
        assert state == "COMPLETE", (rank, state)
    ck = res[0][2]
    assert all(c == ck[0] for c in ck), ck
