"""Where a staged-ring lap spends its time: run StagedRoute with both engines traced and
print per-slice service times (dispatch -> completion, device clock) of the producer's
ring writes and the consumer's ring reads (the latter include the gate wait), plus the
gaps between consecutive decisions and completions. Usage:
python tools/staged_trace.py [--mib 256] [--depth 4]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402
from paper_2604_00368_b200.trace import EV_COMPLETE, EV_DECIDE  # noqa: E402


def pct(x):
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        return {}
    return {"n": int(x.size), "p10_us": round(float(np.percentile(x, 10)) / 1e3, 1),
            "p50_us": round(float(np.percentile(x, 50)) / 1e3, 1), "p90_us": round(float(np.percentile(x, 90)) / 1e3, 1),
            "max_us": round(float(x.max()) / 1e3, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--depth", type=int, default=4)
    o = ap.parse_args()
    cfg = json.dumps({"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536, "gate_timeout_ms": 20000}})
    a = sp.Engine(fabrics.kv_offload(0), cfg, 0)
    b = sp.Engine(fabrics.kv_offload(0), cfg, 0)
    a.start()
    b.start()
    n = o.mib << 20
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    sp.fill_splitmix(0, src.data_ptr(), n, 5)
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    a.register_segment(sp.SegmentDescriptor("src", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, n, src.data_ptr())]))
    b.register_segment(sp.SegmentDescriptor("dst", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, n, dst.data_ptr())]))
    route = sp.StagedRoute(a, b, "g0", "g0", chunk_bytes=4 << 20, depth=o.depth)
    assert route.transfer("src", 0, "dst", 0, n) == sp.BatchState.COMPLETE  # warm
    a.trace_enable(1 << 16)
    b.trace_enable(1 << 16)
    route.stats = {"wait_s": 0.0, "submit_s": 0.0, "pieces": 0}
    assert route.transfer("src", 0, "dst", 0, n) == sp.BatchState.COMPLETE
    ok = torch.equal(src, dst)
    out = {"bytes": n, "pool": route.ring_bytes, "bit_exact": ok, "host": route.stats}
    for name, e in (("producer", a), ("consumer", b)):
        ev, _ = e.trace_fetch(1 << 16)
        comp = ev[ev["kind"] == EV_COMPLETE]
        dec = ev[ev["kind"] == EV_DECIDE]
        out[name] = {"service": pct(comp["t_ns"]), "decides": int(dec.size), "completes": int(comp.size)}
        if dec.size and comp.size:
            t0 = int(dec["now_ns"].min())
            out[name]["span_ms"] = round((int(comp["now_ns"].max()) - t0) / 1e6, 3)
            out[name]["completion_gap"] = pct(np.diff(np.sort(comp["now_ns"].astype(np.int64))))
            out[name]["decide_gap"] = pct(np.diff(np.sort(dec["now_ns"].astype(np.int64))))
    a.stop()
    b.stop()
    route.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
