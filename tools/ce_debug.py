"""Debug: two CE rails, one 64 MiB intent (1024 slices): decisions and per-rail bytes."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

topo = fabrics.kv_offload(0, sm_rails=0, ce_rails=2)
e = sp.Engine(topo, json.dumps({"resilience": {"degradation_ratio": 1e9}}), 0)
e.start()
e.trace_enable(1 << 16)
blk, nb = 256 << 10, 256
pool = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, pool.data_ptr(), blk * nb, 22)
host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, "g0", [sp.BufferDesc(0, blk * nb, host.data_ptr())]))
print("cands", e.plan_candidates("hbm", "host"), flush=True)
b = e.allocate_batch()
e.submit_transfer(b, sp.TransferRequest("hbm", 0, "host", 0, blk * nb))
print(e.await_batch(b, 30_000_000_000), flush=True)
ev, dec = e.trace_fetch(1 << 16)
print("decisions", len(dec), "locals", np.unique(dec["local"], return_counts=True), flush=True)
print("stats", [(e.rail_id(r), e.rail_stats(r).bytes_ok, e.rail_stats(r).bytes_failed, e.rail_stats(r).health) for r in range(e.rail_count())], flush=True)
print("heal", e.heal_stats(), flush=True)
comp = ev[ev["kind"] == 2]
for r in (0, 1):
    c = comp[comp["rail"] == r]
    st = (c["flags"] >> 8) & 0xFF
    print("rail", r, "completions", len(c), "status counts", np.unique(st, return_counts=True),
          "t_ns first", c["t_ns"][:5].tolist(), flush=True)
os._exit(0)
