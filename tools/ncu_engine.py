"""Profiling driver: runs the bench's KV batch (offload and reload interleaved in groups of
32 intents, prepared path) `--runs` times, so ncu can capture one spray_engine_kernel
launch after warm-up:

  ncu --set full --clock-control none --import-source on --replay-mode application \
      -k regex:spray_engine_kernel --launch-skip 3 -c 1 -o gpurun_out/engine \
      python tools/ncu_engine.py --runs 4
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
ap.add_argument("--blocks", type=int, default=4096)
args = ap.parse_args()

blk, nb = 64 << 10, args.blocks
b200 = {"chunk_bytes": 65536}
b200.update(json.loads(os.environ.get("SPRAY_BENCH_B200", "{}")))
e = sp.Engine(fabrics.kv_offload(0), json.dumps({"resilience": {"degradation_ratio": 1e9}, "b200": b200}), 0)
e.start()
hbm = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
hbm2 = torch.zeros(blk * nb, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, hbm.data_ptr(), blk * nb, 7)
hb, hb2 = sp.NumaHostBuffer(0, blk * nb), sp.NumaHostBuffer(0, blk * nb)  # as the bench: NUMA-local pools
host, host2 = hb.tensor(), hb2.tensor()
for sid, med, t in (("hbm", sp.Medium.DEVICE, hbm), ("hbm2", sp.Medium.DEVICE, hbm2),
                    ("host", sp.Medium.HOST, host), ("host2", sp.Medium.HOST, host2)):
    e.register_segment(sp.SegmentDescriptor(sid, med, "g0", [sp.BufferDesc(0, blk * nb, t.data_ptr())]))
perm = np.random.default_rng(3).permutation(nb)
off = [sp.TransferRequest("hbm", i * blk, "host", int(perm[i]) * blk, blk) for i in range(nb)]
on = [sp.TransferRequest("host2", int(perm[i]) * blk, "hbm2", i * blk, blk) for i in range(nb)]
reqs = [r for g in range(0, nb, 32) for r in off[g:g + 32] + on[g:g + 32]]
p = e.prepare_transfers(reqs)
for i in range(args.runs):
    b = e.allocate_batch()
    ms = p.run(b)
    st = e.batch_status(b)
    e.free_batch(b)
    print(f"run {i}: {st.state.name} {len(reqs) * blk / (ms * 1e-3) / 1e9:.2f} GB/s {ms:.3f} ms", flush=True)
os._exit(0)
