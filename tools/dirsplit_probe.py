"""Experiment: does giving each PCIe direction its own worker CTAs help? Two engines on
one GPU (offload engine, reload engine, grid G each) run their halves of the KV batch
concurrently, vs one engine running the interleaved batch."""
import json
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

blk, nb = 64 << 10, 4096
G = int(sys.argv[1]) if len(sys.argv) > 1 else 25
hbm = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
hbm2 = torch.zeros(blk * nb, dtype=torch.uint8, device="cuda:0")
host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
host2 = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
rng = np.random.default_rng(1)
po, pn = rng.permutation(nb), rng.permutation(nb)
engines, preps = [], []
for name in ("off", "on"):
    e = sp.Engine(fabrics.kv_offload(0), json.dumps({"resilience": {"degradation_ratio": 1e9}, "b200": {"grid": G}}), 0)
    e.start()
    for sid, med, t in (("h", sp.Medium.DEVICE, hbm), ("h2", sp.Medium.DEVICE, hbm2),
                        ("p", sp.Medium.HOST, host), ("p2", sp.Medium.HOST, host2)):
        e.register_segment(sp.SegmentDescriptor(sid, med, "g0", [sp.BufferDesc(0, blk * nb, t.data_ptr())]))
    if name == "off":
        reqs = [sp.TransferRequest("h", i * blk, "p", int(po[i]) * blk, blk) for i in range(nb)]
    else:
        reqs = [sp.TransferRequest("p2", int(pn[i]) * blk, "h2", i * blk, blk) for i in range(nb)]
    engines.append(e)
    preps.append(e.prepare_transfers(reqs))
for rep in range(4):
    res = [None, None]
    bs = [e.allocate_batch() for e in engines]

    def run(k):
        res[k] = preps[k].run(bs[k])
    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    for e, b in zip(engines, bs):
        e.free_batch(b)
    print(f"grid {G} x 2 engines: offload {res[0]:.3f} ms, reload {res[1]:.3f} ms, "
          f"both {2 * nb * blk / (max(res) * 1e-3) / 1e9:.1f} GB/s (wall {2 * nb * blk / wall / 1e9:.1f})", flush=True)
os._exit(0)
