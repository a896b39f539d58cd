"""Throughput of the staged route the engine synthesizes toward a GPU without peer access
(engine.cpp:465-610 of the reference): GPU 0's engine is told GPU 1
has no peer access (b200.no_peer), so it declares a host-staged relay rail: hop 1 stores each
chunk into the bounded pinned pool (2048 x 32 KiB = 64 MiB), a forwarder on GPU 1 drains it
into GPU 1's HBM, completions return through the host ring. Sizes: 64 MiB (one pass of the
pool) and 1 GiB (16 laps). Bytes checked after every size.
Usage: python tools/staged_synth_bench.py [--reps 5]  (needs 2 GPUs)"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--mib", type=int, nargs="*", default=[64, 256, 1024])
args = ap.parse_args()
assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
cfg = {"resilience": {"degradation_ratio": 1e9}, "b200": {"no_peer": [1], **json.loads(os.environ.get("ST_B200", "{}"))}}
e = sp.Engine(fabrics.peer_fabric([0, 1], sm_rails=1), json.dumps(cfg), 0)
e.start()
out = {"what": "GPU0 HBM -> pinned host pool (64 MiB) -> GPU1 HBM, engine-synthesized staged rail, b200.no_peer=[1]",
       "rails": [e.rail_id(r) for r in range(e.rail_count())]}
big = 1 << 30
src = torch.empty(big, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, src.data_ptr(), big, 51)
dst = torch.zeros(big, dtype=torch.uint8, device="cuda:1")
e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, big, src.data_ptr())]))
e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, big, dst.data_ptr())]))
for n in [m << 20 for m in args.mib]:
    best = None
    for _ in range(args.reps):
        b = e.allocate_batch()
        t0 = time.perf_counter()
        e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
        st = e.await_batch(b, 120_000_000_000)
        dt = time.perf_counter() - t0
        e.free_batch(b)
        assert st.state == sp.BatchState.COMPLETE, st
        best = dt if best is None else min(best, dt)
    exact = sp.checksum(1, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
    out[f"{n >> 20}MiB"] = {"gbs": round(n / best / 1e9, 2), "ms": round(best * 1e3, 3), "bit_exact": bool(exact)}
    print(json.dumps({f"{n >> 20}MiB": out[f"{n >> 20}MiB"]}), flush=True)
out["bytes_by_rail"] = {e.rail_id(r): e.rail_stats(r).bytes_ok for r in range(e.rail_count())}
if json.loads(os.environ.get("ST_B200", "{}")).get("diag"):
    import ctypes as C
    from paper_2604_00368_b200 import _lib as L
    w = (C.c_uint64 * 62)()
    L.lib.spray_engine_debug(e._h, w, 62)
    d = list(w)[45:61]
    out["diag"] = {"hostrx_staged_reads": d[0], "hostrx_read_cycles_avg": d[1] / max(1, d[0]), "hostrx_read_cycles_max": d[2],
                   "fwd_tickets": d[4], "fwd_wait_ns_avg": d[5] / max(1, d[4]), "fwd_wait_ns_max": d[7],
                   "fwd_copy_ns_avg": d[6] / max(1, d[4]), "hop1_chunks": d[8], "hop1_copy_fence_ns_avg": d[9] / max(1, d[8]),
                   "hop1_wait_ns_avg": d[10] / max(1, d[8])}
    print(json.dumps(out["diag"]), flush=True)
e.stop()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/staged_synth.json", "w"), indent=1)
print(json.dumps(out), flush=True)
os._exit(0)
