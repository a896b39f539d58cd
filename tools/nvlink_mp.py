"""C2 and the C4 chain across processes: one process per GPU (torchrun), peer HBM shared
through CUDA IPC handles (spray_ipc_export / spray_ipc_open) exchanged over
torch.distributed. No data-path collective: NCCL/gloo carry only handles, barriers and
the max-over-ranks timing.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/nvlink_mp.py c2
  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/nvlink_mp.py chain
"""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "c2"
    size = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 30
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    gpus = list(range(world))
    e = sp.Engine(fabrics.peer_fabric(gpus), json.dumps({"resilience": {"degradation_ratio": 1e9}}), rank)
    e.start()
    cb = e.chunk_bytes()
    buf = torch.zeros(size, dtype=torch.uint8, device=f"cuda:{rank}")
    flags = torch.zeros(size // cb, dtype=torch.int32, device=f"cuda:{rank}")
    if rank == 0:
        sp.fill_splitmix(0, buf.data_ptr(), size, 2026)
    handles = [None] * world
    dist.all_gather_object(handles, (sp.ipc_export(rank, buf.data_ptr()), sp.ipc_export(rank, flags.data_ptr())))
    opened = []

    def peer(j):
        pb, pf = sp.ipc_open(rank, handles[j][0]), sp.ipc_open(rank, handles[j][1])
        opened.extend([pb, pf])
        return pb, pf

    e.register_segment(sp.SegmentDescriptor(f"w{rank}", sp.Medium.DEVICE, f"g{rank}", [sp.BufferDesc(0, size, buf.data_ptr())]))
    role = None
    if mode == "c2":
        if rank == 0:
            pb, _ = peer(1)
            e.register_segment(sp.SegmentDescriptor("w1", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, size, pb)]))
            role = sp.TransferRequest("w0", 0, "w1", 0, size)
    else:  # chain: rank k forwards w_k -> w_{k+1} granule by granule
        if rank + 1 < world:
            pb, pf = peer(rank + 1)
            e.register_segment(sp.SegmentDescriptor(f"w{rank + 1}", sp.Medium.DEVICE, f"g{rank + 1}",
                                                    [sp.BufferDesc(0, size, pb)]))
            e.gate_segment(f"w{rank + 1}", sp.Engine.GATE_PRODUCE, pf)
            if rank > 0:
                e.gate_segment(f"w{rank}", sp.Engine.GATE_CONSUME, flags.data_ptr())
            role = sp.TransferRequest(f"w{rank}", 0, f"w{rank + 1}", 0, size)
    prep = e.prepare_transfers([role]) if role else None
    times = []
    for rep in range(4):
        if rank > 0:
            buf.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        ms = 0.0
        if prep:
            b = e.allocate_batch()
            ms = prep.run(b)
            assert e.batch_status(b).state == sp.BatchState.COMPLETE
            e.free_batch(b)
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rep:
            times.append(float(t.item()))
    dist.barrier()
    ck = torch.tensor([float(sp.checksum(rank, buf.data_ptr(), size) % (1 << 52))], dtype=torch.float64)
    cks = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(cks, ck)
    if rank == 0:
        last = world - 1 if mode == "chain" else 1
        ok = all(float(cks[j].item()) == float(cks[0].item()) for j in range(1, last + 1))
        best = min(times)
        receivers = (world - 1) if mode == "chain" else 1
        print(json.dumps({"mode": f"{mode}-multiprocess", "ranks": world, "bytes": size, "max_over_ranks_ms": round(best, 3),
                          "delivered_gbs": round(receivers * size / (best * 1e-3) / 1e9, 2), "bit_exact": ok}),
              flush=True)
    for p in opened:
        sp.ipc_close(p)
    e.stop()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
