"""Debug probe: small KV offload batches through the ring, with counters."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

topo = fabrics.kv_offload(0, sm_rails=1)
k = sp.Engine(topo, None, 0)
k.start()
blk = 64 << 10
for nb, hostdst in ((4, True), (4, False), (64, True), (4096, True)):
    pool = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
    sp.fill_splitmix(0, pool.data_ptr(), blk * nb, 7)
    if hostdst:
        other = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
        k.register_segment(sp.SegmentDescriptor(f"o{nb}{hostdst}", sp.Medium.HOST, "g0",
                                                [sp.BufferDesc(0, blk * nb, other.data_ptr())]))
    else:
        other = torch.zeros(blk * nb, dtype=torch.uint8, device="cuda:0")
        k.register_segment(sp.SegmentDescriptor(f"o{nb}{hostdst}", sp.Medium.DEVICE, "g0",
                                                [sp.BufferDesc(0, blk * nb, other.data_ptr())]))
    k.register_segment(sp.SegmentDescriptor(f"p{nb}{hostdst}", sp.Medium.DEVICE, "g0",
                                            [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
    reqs = [sp.TransferRequest(f"p{nb}{hostdst}", i * blk, f"o{nb}{hostdst}", i * blk, blk) for i in range(nb)]
    b = k.allocate_batch()
    t0 = time.perf_counter()
    k.submit_transfers(b, reqs)
    st = k.await_batch(b, 3_000_000_000)
    t1 = time.perf_counter()
    print(nb, hostdst, st, f"{(t1-t0)*1e3:.2f} ms", k.counters(), k.rail_stats(0).bytes_ok, flush=True)
    if st.state != sp.BatchState.COMPLETE:
        import ctypes as C
        from paper_2604_00368_b200 import _lib as L
        for rep in range(3):
            w = (C.c_uint64 * 16)()
            L.lib.spray_engine_debug(k._h, w, 16)
            print("debug", list(w), flush=True)
            time.sleep(0.5)
        break
    eq = torch.equal(pool.cpu(), other.cpu())
    print("equal", eq, flush=True)
    k.free_batch(b)
print("done", flush=True)
os._exit(0)
