"""Where a single 4 KiB intent's latency goes: the engine runs with b200.diag, each round is
one batch (allocate / submit / await / free, timed in C++), and after each round the
per-stage timeline words (Control::lat, engine ns of each stage's last pass) are read.
Reported as stage-to-stage deltas (median over rounds)."""
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

STAGES = ["hostrx_fetch", "ingress_block", "state_decide", "egress_post", "publish_stamp", "complete_gather",
          "state_apply", "publish_done"]
# usage: latency_stages.py [4k|kv]; LAT_B200='{"worker_fence": "gpu"}' adds engine knobs
mode = sys.argv[1] if len(sys.argv) > 1 else "4k"
b200 = {"diag": True, **json.loads(os.environ.get("LAT_B200", "{}"))}
cfg = json.dumps({"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536, **b200}})
if mode == "kv":  # 32 offloads HBM -> host + 32 reloads host -> HBM, 64 KiB each (latency_c.py's batch)
    nb, blk = 1024, 64 << 10
    e = sp.Engine(fabrics.kv_offload(0, sm_rails=1), cfg, 0)
    e.start()
    bufs = {"hbm": torch.empty(nb * blk, dtype=torch.uint8, device="cuda:0"),
            "hbm2": torch.zeros(nb * blk, dtype=torch.uint8, device="cuda:0"),
            "host": torch.zeros(nb * blk, dtype=torch.uint8, pin_memory=True),
            "host2": torch.zeros(nb * blk, dtype=torch.uint8, pin_memory=True)}
    for sid, t in bufs.items():
        e.register_segment(sp.SegmentDescriptor(sid, sp.Medium.DEVICE if sid.startswith("hbm") else sp.Medium.HOST,
                                                "g0", [sp.BufferDesc(0, nb * blk, t.data_ptr())]))
    rng = np.random.default_rng(1)
    p1, p2 = rng.permutation(nb), rng.permutation(nb)
    reqs = [r for g in range(0, nb, 32)
            for r in [sp.TransferRequest("hbm", i * blk, "host", int(p1[i]) * blk, blk) for i in range(g, g + 32)] +
            [sp.TransferRequest("host2", int(p2[i]) * blk, "hbm2", i * blk, blk) for i in range(g, g + 32)]]
    per = 64
else:
    n = 1 << 20
    e = sp.Engine(fabrics.two_node(1, 1e9, backend="cuda"), cfg, 0)
    e.start()
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    reqs = [sp.TransferRequest("s", 4096 * i, "d", 4096 * i, 4096) for i in range(64)]
    per = 1
e.batch_latency_ns(reqs, per, 50)
deltas, tot = [], []
w = (C.c_uint64 * 102)()
for k in range(200):
    t = e.batch_latency_ns(reqs, per, 1)[0]
    L.lib.spray_engine_debug(e._h, w, 102)
    lat = list(w)[62:70]
    lw = list(w)[70:75]
    # stamp -> worker pickup -> copied -> fenced -> counted -> COMPLETE sees the word
    ls = list(w)[94:102]
    deltas.append([lat[i + 1] - lat[i] for i in range(7)] +
                  [lw[0] - lat[4], lw[1] - lw[0], lw[2] - lw[1], lw[3] - lw[2], lw[4] - lw[3]] +
                  [ls[0] - lat[1], ls[1] - ls[0], ls[2] - ls[1], lat[2] - ls[2], ls[4] - lat[5], ls[5] - ls[4], lat[6] - ls[5],
                   ls[3] - ls[5], ls[6] - ls[3], ls[7] - ls[6], lat[6] - ls[7]])
    tot.append(t)
d = np.median(np.array(deltas, dtype=np.int64), axis=0)
SSTAGES = ["ingress_block->state_sees_block", "sees_block->slots_reserved", "slots->set_loaded", "set->decided",
           "complete_gather->state_sees_entry", "sees_entry->feedback_done", "feedback_done->applied",
           "  apply: fb_done->prologue_done", "  apply: prologue->lead_done", "  apply: lead->slots_freed", "  apply: freed->end"]
WSTAGES = ["stamp->worker_pickup", "pickup->copied", "copied->fenced", "fenced->counted", "counted->complete_sees"]
out = {"mode": mode, "b200": b200, "round_us_median": round(float(np.median(tot)) / 1e3, 2),
       "device_span_us": round(float(np.median([sum(x[:7]) for x in deltas])) / 1e3, 2),
       "stage_deltas_us": {f"{STAGES[i]}->{STAGES[i + 1]}": round(float(d[i]) / 1e3, 2) for i in range(7)},
       "worker_deltas_us": {WSTAGES[i]: round(float(d[7 + i]) / 1e3, 2) for i in range(5)},
       "state_deltas_us": {SSTAGES[i]: round(float(d[12 + i]) / 1e3, 2) for i in range(11)}}
tot_a = np.array(tot)
if mode == "kv":  # rounds split at the median: where the slow ones lose their time
    arr = np.array(deltas, dtype=np.int64)
    med = np.median(tot_a)
    for name, sel in (("fast_rounds", tot_a <= med), ("slow_rounds", tot_a > med)):
        if sel.any():
            dd = np.median(arr[sel], axis=0)
            out[name] = {"n": int(sel.sum()), "round_us": round(float(np.median(tot_a[sel])) / 1e3, 2),
                         "stage_deltas_us": {f"{STAGES[i]}->{STAGES[i + 1]}": round(float(dd[i]) / 1e3, 2) for i in range(7)},
                         "worker_deltas_us": {WSTAGES[i]: round(float(dd[7 + i]) / 1e3, 2) for i in range(5)}}
    out["round_us_hist"] = np.histogram(tot_a / 1e3, bins=8)[0].tolist()
    out["round_us_edges"] = [round(float(x), 1) for x in np.histogram(tot_a / 1e3, bins=8)[1]]
print(json.dumps(out, indent=1), flush=True)
os._exit(0)
