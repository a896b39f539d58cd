"""Profiling driver: the small-slice regime (4096 x 64 KiB HBM->HBM, one slice per intent)
over `--rails` rails, prepared path, `--runs` launches, so ncu can capture one
spray_engine_kernel launch after warm-up (source-level stalls of the STATE warp):

  ncu --set full --clock-control none --import-source on --replay-mode application \\
      -k regex:spray_engine_kernel --launch-skip 3 -c 1 -o gpurun_out/small \\
      python tools/ncu_small.py --runs 4 --rails 2
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=4)
ap.add_argument("--rails", type=int, default=2)
args = ap.parse_args()
blk, nb = 64 << 10, 4096
src = torch.empty(nb * blk, dtype=torch.uint8, device="cuda:0")
dst = torch.zeros(nb * blk, dtype=torch.uint8, device="cuda:0")
e = sp.Engine(fabrics.two_node(args.rails, 1.6e12 / args.rails, backend="cuda"),
              json.dumps({"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536}}), 0)
e.start()
e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, nb * blk, src.data_ptr())]))
e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, nb * blk, dst.data_ptr())]))
perm = np.random.default_rng(3).permutation(nb)
p = e.prepare_transfers([sp.TransferRequest("s", i * blk, "d", int(perm[i]) * blk, blk) for i in range(nb)])
for _ in range(args.runs):
    b = e.allocate_batch()
    ms = p.run(b)
    assert e.batch_status(b).state == sp.BatchState.COMPLETE
    e.free_batch(b)
print(json.dumps({"last_ms": ms}), flush=True)
os._exit(0)
