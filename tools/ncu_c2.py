"""Profiling driver for the NVLink copy path: C2 (1 GiB GPU0 -> GPU1 over the direct SM
peer-store rail, 4096 x 256 KiB slices, 32 KiB granules), prepared path, `--runs` drain-mode
launches so ncu can capture one after warm-up:

  ncu --set full --clock-control none --import-source on --replay-mode application \
      -k regex:spray_engine_kernel --launch-skip 3 -c 1 -o gpurun_out/c2 \
      python tools/ncu_c2.py --runs 5
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=5)
ap.add_argument("--size", type=int, default=1 << 30)
args = ap.parse_args()
n = args.size
src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
dst = torch.zeros(n, dtype=torch.uint8, device="cuda:1")
sp.fill_splitmix(0, src.data_ptr(), n, 5)
e = sp.Engine(fabrics.peer_fabric([0, 1]), json.dumps({"resilience": {"degradation_ratio": 1e9}}), 0)
e.start()
e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, n, src.data_ptr())]))
e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, n, dst.data_ptr())]))
p = e.prepare_transfers([sp.TransferRequest("s", 0, "d", 0, n)])
ms = []
for _ in range(args.runs):
    b = e.allocate_batch()
    ms.append(p.run(b))
    assert e.batch_status(b).state == sp.BatchState.COMPLETE
    e.free_batch(b)
assert sp.checksum(1, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
print(json.dumps({"kernel_ms": [round(x, 3) for x in ms], "gbs": round(n / (min(ms) * 1e-3) / 1e9, 2)}))
e.stop()
