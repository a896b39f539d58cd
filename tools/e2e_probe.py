"""Where the e2e time of the KV batch goes: host submit (make_intent + ring publish) vs
await, against the device-resident (prepared) run of the same batch."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

blk, nb, g = 64 << 10, 4096, 32
e = sp.Engine(fabrics.kv_offload(0), json.dumps({"resilience": {"degradation_ratio": 1e9}}), 0)
e.start()
hbm = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
hbm2 = torch.zeros(blk * nb, dtype=torch.uint8, device="cuda:0")
host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
host2 = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
for sid, med, t in (("h", sp.Medium.DEVICE, hbm), ("h2", sp.Medium.DEVICE, hbm2),
                    ("p", sp.Medium.HOST, host), ("p2", sp.Medium.HOST, host2)):
    e.register_segment(sp.SegmentDescriptor(sid, med, "g0", [sp.BufferDesc(0, blk * nb, t.data_ptr())]))
rng = np.random.default_rng(1)
po, pn = rng.permutation(nb), rng.permutation(nb)
off = [sp.TransferRequest("h", i * blk, "p", int(po[i]) * blk, blk) for i in range(nb)]
on = [sp.TransferRequest("p2", int(pn[i]) * blk, "h2", i * blk, blk) for i in range(nb)]
reqs = [r for k in range(0, nb, g) for r in off[k:k + g] + on[k:k + g]]
creqs = sp.Requests(reqs)
p = e.prepare_transfers(reqs)
for _ in range(3):
    b = e.allocate_batch()
    ms = p.run(b)
    e.free_batch(b)
print(f"prepared: {ms:.3f} ms", flush=True)
for _ in range(5):
    b = e.allocate_batch()
    t0 = time.perf_counter()
    e.submit_transfers(b, creqs)
    t1 = time.perf_counter()
    st = e.await_batch(b)
    t2 = time.perf_counter()
    e.free_batch(b)
    print(f"e2e: submit {1e3 * (t1 - t0):.3f} ms, await {1e3 * (t2 - t1):.3f} ms, total {1e3 * (t2 - t0):.3f} ms "
          f"({len(reqs) * blk / (t2 - t0) / 1e9:.1f} GB/s) {st.state.name}", flush=True)
os._exit(0)
