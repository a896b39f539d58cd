"""Small-slice regime probe: 4096 x 64 KiB HBM->HBM (scattered block table) through the engine
with 1, 2 and 4 rails per node, prepared intents, drain-mode launch timed by CUDA events.
Prints GB/s and the STATE warp's cycle split per launch (spray_engine_debug words)."""
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
         "egress", "egress_blocks", "ingress_blocks", "entries", "pub_busy", "rx_busy", "n_fences", "p1", "p2", "fb_busy",
         "scans"]


def dbg(k):
    w = (C.c_uint64 * 94)()
    L.lib.spray_engine_debug(k._h, w, 94)
    d = dict(zip(NAMES, list(w)))
    d["dy"] = list(w)[78:86]
    d["dz"] = list(w)[86:94]
    return d


blk = int(os.environ.get("BLK_KIB", "64")) << 10
nb = int(os.environ.get("NB", "4096"))
out = {}
src = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, src.data_ptr(), blk * nb, 7)
dst = torch.zeros(blk * nb, dtype=torch.uint8, device="cuda:0")
perm = np.random.default_rng(3).permutation(nb)
for rails in (1, 2, 4):
    for chunk in (65536,):
        cfg = {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": chunk}}
        k = sp.Engine(fabrics.two_node(rails, 1.6e12 / rails, backend="cuda"), json.dumps(cfg), 0)
        k.start()
        k.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, blk * nb, src.data_ptr())]))
        k.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, blk * nb, dst.data_ptr())]))
        p = k.prepare_transfers([sp.TransferRequest("s", i * blk, "d", int(perm[i]) * blk, blk) for i in range(nb)])
        ms = []
        for it in range(6):
            b = k.allocate_batch()
            ms.append(p.run(b))
            assert k.batch_status(b).state == sp.BatchState.COMPLETE
            k.free_batch(b)
        d = dbg(k)
        best = min(ms[2:])
        gbs = nb * blk / (best * 1e-3) / 1e9
        ghz = 1.9e9
        keys = ("apply", "decide", "ctl", "serial", "obs", "fb", "complete", "egress", "ingress", "pub_busy", "p1", "p2", "fb_busy")
        row = {"rails": rails, "chunk": chunk, "gbs": round(gbs, 1), "ms": round(best, 4),
               "slices_per_s_M": round(nb / (best * 1e-3) / 1e6, 2), "entries": d["entries"], "loops": d["loops"]}
        row.update({kk + "_ms": round(d[kk] / ghz * 1e3, 3) for kk in keys})
        dy = d["dy"]  # table, broadcast, lane-0 loop cycles; its decisions, blocks; hand-back; warp-path decisions
        row["dec_split"] = {"table_cyc_per_blk": round(dy[0] / max(1, dy[4] or 1), 1),
                            "bcast_cyc_per_blk": round(dy[1] / max(1, dy[4]), 1),
                            "loop_cyc_per_dec": round(dy[2] / max(1, dy[3]), 1),
                            "handback_cyc_per_blk": round(dy[5] / max(1, dy[4]), 1),
                            "scalar_blocks": dy[4], "scalar_decisions": dy[3], "warp_decisions": dy[6]}
        dz = d["dz"]
        row["dec_extra_cyc_per_blk"] = {"cand_eval_slots_dq": round(dz[3] / max(1, dy[4] or 1), 1),
                                        "tail_records": round(dz[4] / max(1, dy[4] or 1), 1),
                                        "slot_reserve_load_set": round(dz[5] / max(1, dy[4] or 1), 1)}
        row["fb_split"] = {"chain_cyc_per_completion": round(dz[0] / max(1, dz[1]), 1), "completions": dz[1],
                           "entries": dz[2], "busy_cyc_per_completion": round(d["fb_busy"] / max(1, dz[1]), 1)}
        print(json.dumps(row), flush=True)
        out[f"r{rails}_c{chunk}"] = row
        assert torch.equal(dst.view(nb, blk)[torch.as_tensor(perm)], src.view(nb, blk))
        p.free()
        k.stop()
        del k
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/smallslice.json", "w"), indent=1)
os._exit(0)
