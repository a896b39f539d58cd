"""Batch latency through the public C-ABI timed in C++ (spray_batch_latency): a single 4 KiB
intent (HBM -> HBM and HBM -> pinned host) and the 64 x 64 KiB KV batch (32 offloads + 32
reloads, random block tables). P50/P90/P99 per bench.cpp:213-215 (exact_percentile)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402


def pct(a, q):
    a = np.sort(np.asarray(a, dtype=np.float64))
    k = max(0, min(len(a) - 1, int(np.ceil(q * len(a))) - 1))
    return float(a[k])


def summary(ns):
    us = np.asarray(ns, dtype=np.float64) / 1e3
    return {"p50_us": round(pct(us, 0.5), 2), "p90_us": round(pct(us, 0.9), 2), "p99_us": round(pct(us, 0.99), 2),
            "mean_us": round(float(us.mean()), 2), "n": len(us)}


out = {}
dev = 0
nb, blk = 4096, 64 << 10
b200 = {"chunk_bytes": 65536, **json.loads(os.environ.get("LAT_B200", "{}"))}  # LAT_B200: extra engine knobs
cfg = json.dumps({"resilience": {"degradation_ratio": 1e9}, "b200": b200})
e = sp.Engine(fabrics.kv_offload(dev, sm_rails=1), cfg, dev)
e.start()
hbm = torch.empty(nb * blk, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, hbm.data_ptr(), nb * blk, 3)
hbm2 = torch.zeros(nb * blk, dtype=torch.uint8, device="cuda:0")
host = torch.zeros(nb * blk, dtype=torch.uint8, pin_memory=True)
host2 = torch.zeros(nb * blk, dtype=torch.uint8, pin_memory=True)
for sid, med, t in (("hbm", sp.Medium.DEVICE, hbm), ("hbm2", sp.Medium.DEVICE, hbm2),
                    ("host", sp.Medium.HOST, host), ("host2", sp.Medium.HOST, host2)):
    e.register_segment(sp.SegmentDescriptor(sid, med, "g0", [sp.BufferDesc(0, nb * blk, t.data_ptr())]))
rng = np.random.default_rng(1)
p1, p2 = rng.permutation(nb), rng.permutation(nb)
d2d = [sp.TransferRequest("hbm", int(p1[i]) * blk, "hbm2", i * blk, 4096) for i in range(256)]
d2h = [sp.TransferRequest("hbm", int(p1[i]) * blk, "host", i * blk, 4096) for i in range(256)]
off = [sp.TransferRequest("hbm", i * blk, "host", int(p1[i]) * blk, blk) for i in range(nb)]
on = [sp.TransferRequest("host2", int(p2[i]) * blk, "hbm2", i * blk, blk) for i in range(nb)]
kv = [r for g in range(0, nb, 32) for r in off[g:g + 32] + on[g:g + 32]]
kv_rf = [r for g in range(0, nb, 32) for r in on[g:g + 32] + off[g:g + 32]]  # the reloads first in each batch
cases = [("intent_4k_hbm2hbm", d2d, 1), ("intent_4k_hbm2host", d2h, 1), ("kv_64x64k", kv, 64)]
if os.environ.get("LAT_KV_REVERSED"):
    cases.append(("kv_64x64k_reloads_first", kv_rf, 64))
for name, reqs, per in cases:
    e.batch_latency_ns(reqs, per, 50)  # warm
    out[name] = summary(e.batch_latency_ns(reqs, per, 1000))
    print(name, json.dumps(out[name]), flush=True)
e.stop()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/latency_c.json", "w"), indent=1)
os._exit(0)
