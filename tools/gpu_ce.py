"""Debug probe for the copy-engine rail path."""
import ctypes as C
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import _lib as L, fabrics  # noqa: E402

topo = fabrics.kv_offload(0, sm_rails=1, ce_rails=1)
e = sp.Engine(topo, json.dumps({"resilience": {"degradation_ratio": 1e9}}), 0)
e.start()
blk, nb = 1 << 20, 64
pool = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, pool.data_ptr(), blk * nb, 21)
host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, "g0", [sp.BufferDesc(0, blk * nb, host.data_ptr())]))
b = e.allocate_batch()
e.submit_transfers(b, [sp.TransferRequest("hbm", i * blk, "host", i * blk, blk) for i in range(nb)])
st = e.await_batch(b, 3_000_000_000)
print(st, flush=True)
w = (C.c_uint64 * 40)()
L.lib.spray_engine_debug(e._h, w, 40)
print(list(w), flush=True)
for r in range(e.rail_count()):
    print(e.rail_stats(r), flush=True)
os._exit(0)
