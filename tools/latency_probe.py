"""Batch latency vs batch size on one GPU: submit -> await through the public API, one
batch in flight, persistent kernel already running. Splits the fixed cost from the
bandwidth term. Usage: python tools/latency_probe.py [--fabric kv|hbm]"""
import argparse
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fabric", default="kv", choices=["kv", "hbm"])
    ap.add_argument("--reps", type=int, default=300)
    ap.add_argument("--chunk-kib", type=int, default=64)
    a = ap.parse_args()
    dev = 0
    cfg = {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": a.chunk_kib << 10}}
    if a.fabric == "kv":
        e = sp.Engine(fabrics.kv_offload(dev), json.dumps(cfg), dev)
    else:
        e = sp.Engine(fabrics.two_node(1, 3.2e12, backend="cuda"), json.dumps(cfg), dev)
    e.start()
    n = 64 << 20
    hbm = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    sp.fill_splitmix(dev, hbm.data_ptr(), n, 3)
    if a.fabric == "kv":
        host = torch.zeros(n, dtype=torch.uint8, pin_memory=True)
        e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, n, hbm.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("d", sp.Medium.HOST, "g0", [sp.BufferDesc(0, n, host.data_ptr())]))
    else:
        dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
        e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, hbm.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    out = {"fabric": a.fabric, "chunk_kib": a.chunk_kib}
    for nint, blk in ((1, 4096), (1, 65536), (8, 65536), (64, 65536), (1, 4 << 20), (256, 65536)):
        reqs = sp.Requests([sp.TransferRequest("s", i * blk, "d", i * blk, blk) for i in range(nint)])
        lat, sub = [], []
        for k in range(a.reps + 20):
            t0 = time.perf_counter()
            b = e.allocate_batch()
            e.submit_transfers(b, reqs)
            t1 = time.perf_counter()
            st = e.await_batch(b)
            t2 = time.perf_counter()
            assert st.state == sp.BatchState.COMPLETE
            e.free_batch(b)
            if k >= 20:
                lat.append((t2 - t0) * 1e6)
                sub.append((t1 - t0) * 1e6)
        lat.sort()
        out[f"{nint}x{blk >> 10}KiB"] = {"p50_us": round(statistics.median(lat), 1),
                                         "p90_us": round(lat[int(0.9 * len(lat)) - 1], 1),
                                         "submit_us": round(statistics.median(sub), 1)}
    # one prepared (drain-mode) launch per shape: the scheduler's timeline of that batch
    import ctypes as C
    from paper_2604_00368_b200 import _lib as L
    tls = {}
    for nint, blk in ((1, 65536), (64, 65536), (1, 4 << 20)):
        p = e.prepare_transfers([sp.TransferRequest("s", i * blk, "d", i * blk, blk) for i in range(nint)])
        ms = []
        for _ in range(5):
            b = e.allocate_batch()
            ms.append(p.run(b))
            e.free_batch(b)
        w = (C.c_uint64 * 48)()
        L.lib.spray_engine_debug(e._h, w, 48)
        tl = list(w)[37:44]
        tls[f"{nint}x{blk >> 10}KiB"] = {"kernel_us": round(min(ms) * 1e3, 1), **dict(zip(
            ["first_stamp", "first_decide", "last_decide", "first_apply", "last_apply", "exit"],
            [round((x - tl[0]) / 1e3, 1) if x else None for x in tl[1:]]))}
        p.free()
    out["prepared_timeline_us"] = tls
    e.stop()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
