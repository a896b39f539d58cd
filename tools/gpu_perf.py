"""Perf probe: the bench KV batch (offload + reload, prepared path) with per-warp scheduler
cycle counters, plus single-direction variants."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import _lib as L, fabrics  # noqa: E402

NAMES = ["host_tail", "sub_tail", "sub_head", "state", "now", "disp", "term", "failed", "retried", "trace_n",
         "stream", "loops", "serial", "obs", "fb", "n_comp", "n_dec", "apply", "decide", "ctl", "ingress", "complete",
         "egress", "egress_blocks", "ingress_blocks", "entries", "pub_busy", "rx_busy", "n_fences", "p1", "p2", "p3", "x15"]


def dbg(k):
    w = (C.c_uint64 * 48)()
    L.lib.spray_engine_debug(k._h, w, 48)
    return dict(zip(NAMES, list(w)))


chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": chunk}}
if grid:
    cfg["b200"]["grid"] = grid
print(f"chunk={chunk} grid={grid or 'default'}", flush=True)
k = sp.Engine(fabrics.kv_offload(0, sm_rails=1), json.dumps(cfg), 0)
k.start()
blk, nb = 64 << 10, 4096
pool = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, pool.data_ptr(), blk * nb, 7)
pool2 = torch.zeros(blk * nb, dtype=torch.uint8, device="cuda:0")
host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
host2 = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
for sid, med, t in (("hbm", sp.Medium.DEVICE, pool), ("hbm2", sp.Medium.DEVICE, pool2),
                    ("host", sp.Medium.HOST, host), ("host2", sp.Medium.HOST, host2)):
    k.register_segment(sp.SegmentDescriptor(sid, med, "g0", [sp.BufferDesc(0, blk * nb, t.data_ptr())]))
perm = np.random.default_rng(3).permutation(nb)
off = [sp.TransferRequest("hbm", i * blk, "host", int(perm[i]) * blk, blk) for i in range(nb)]
on = [sp.TransferRequest("host2", int(perm[i]) * blk, "hbm2", i * blk, blk) for i in range(nb)]
d2d = [sp.TransferRequest("hbm", i * blk, "hbm2", int(perm[i]) * blk, blk) for i in range(nb)]
mixed = [r for g in range(0, nb, 32) for r in off[g:g + 32] + on[g:g + 32]]
for name, reqs in (("offload", off), ("reload", on), ("both", off + on), ("mixed32", mixed), ("hbm2hbm", d2d)):
    p = k.prepare_transfers(reqs)
    for it in range(3):
        b = k.allocate_batch()
        ms = p.run(b)
        st = k.batch_status(b)
        k.free_batch(b)
    d = dbg(k)  # counters of the last launch (they restart per launch)
    gbs = len(reqs) * blk / (ms * 1e-3) / 1e9
    keys = ("loops", "entries", "serial", "obs", "fb", "n_comp", "apply", "decide", "ctl", "ingress", "complete", "egress", "pub_busy", "rx_busy", "n_fences", "p1", "p2", "p3")
    ghz = 1.9e9
    print(f"{name:8s} {st.state.name} {gbs:7.2f} GB/s {ms:7.3f} ms  " +
          " ".join(f"{kk}={d[kk] / ghz * 1e3:.2f}ms" if kk not in ("loops", "n_comp", "entries", "n_fences") else f"{kk}={d[kk]}"
                   for kk in keys), flush=True)
os._exit(0)
