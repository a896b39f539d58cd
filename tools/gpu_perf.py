"""Perf probe: KV offload batches (ring + prepared paths) with scheduler phase timers."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import _lib as L, fabrics  # noqa: E402

NAMES = ["host_tail", "sub_tail", "sub_head", "state", "now", "disp", "term", "failed", "retried", "trace_n",
         "stream", "loops", "comp_ns", "sub_ns", "ctl_ns", "n_comp", "n_dec", "x0", "x1", "x2", "x3", "x4", "x5", "x6", "x7"]


def dbg(k):
    w = (C.c_uint64 * 32)()
    L.lib.spray_engine_debug(k._h, w, 32)
    return dict(zip(NAMES, list(w)))


cfg = {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": int(sys.argv[1]) if len(sys.argv) > 1 else 65536}}
topo = fabrics.kv_offload(0, sm_rails=1)
k = sp.Engine(topo, json.dumps(cfg), 0)
k.start()
blk, nb = 64 << 10, 4096
pool = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, pool.data_ptr(), blk * nb, 7)
host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
pool2 = torch.zeros(blk * nb, dtype=torch.uint8, device="cuda:0")
k.register_segment(sp.SegmentDescriptor("kv/hbm", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
k.register_segment(sp.SegmentDescriptor("kv/hbm2", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, blk * nb, pool2.data_ptr())]))
k.register_segment(sp.SegmentDescriptor("kv/host", sp.Medium.HOST, "g0", [sp.BufferDesc(0, blk * nb, host.data_ptr())]))
perm = np.random.default_rng(3).permutation(nb)
for dst in ("kv/host", "kv/hbm2"):
    reqs = [sp.TransferRequest("kv/hbm", i * blk, dst, int(perm[i]) * blk, blk) for i in range(nb)]
    for it in range(3):
        d0 = dbg(k)
        b = k.allocate_batch()
        t0 = time.perf_counter()
        k.submit_transfers(b, reqs)
        st = k.await_batch(b, 5_000_000_000)
        t1 = time.perf_counter()
        d1 = dbg(k)
        delta = {n: d1[n] - d0[n] for n in ("comp_ns", "sub_ns", "ctl_ns", "n_comp", "x0", "x1", "x2", "x3", "x4", "x5")}
        print(dst, "ring", it, st.state.name, f"{blk*nb/(t1-t0)/1e9:.2f} GB/s", f"{(t1-t0)*1e3:.2f} ms", delta, flush=True)
        if st.state != sp.BatchState.COMPLETE:
            print(dbg(k))
            os._exit(1)
        k.free_batch(b)
    p = k.prepare_transfers(reqs)
    for it in range(3):
        d0 = dbg(k)
        b = k.allocate_batch()
        ms = p.run(b)
        d1 = dbg(k)
        delta = {n: d1[n] - d0[n] for n in ("comp_ns", "sub_ns", "ctl_ns", "n_comp", "x0", "x1", "x2", "x3", "x4", "x5")}
        st = k.batch_status(b)
        print(dst, "prepared", it, st.state.name, f"{blk*nb/(ms*1e-3)/1e9:.2f} GB/s", f"{ms:.3f} ms", delta, flush=True)
        k.free_batch(b)
print("rail", k.rail_stats(0), flush=True)
os._exit(0)
