"""Real-contention congestion experiment (>= 2 GPUs, one process): GPU 0 offloads a KV batch
(4096 x 64 KiB, HBM -> pinned host, random block table) while a background copy-engine flow
the engine does not control saturates GPU 0's own PCIe root in the same direction (repeated
256 MiB cudaMemcpyAsync D2H on a separate stream). The engine's rails: g0.pcie0 (SM stores
over GPU 0's root) and g0.rl1 (2-hop: NVLink into GPU 1's HBM, GPU 1's SMs store over GPU 1's
root). Compared under the same background load:
  telemetry  the engine's cost-model spray (it sees the congested rail slow down)
  rr         the engine with the state-blind round-robin policy (Policy::kRoundRobin)
  striping   state-blind round-robin cudaMemcpyAsync striping of the same blocks on GPU 0
             (4 streams, one call per block: the baseline the north star names)
and without background load for reference. Bytes checked after every run."""
import json
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
nb, blk = 4096, 64 << 10
pool = torch.empty(nb * blk, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, pool.data_ptr(), nb * blk, 9)
hb = sp.NumaHostBuffer(0, nb * blk)
host = hb.tensor()
perm = np.random.default_rng(4).permutation(nb)
ref = pool.view(nb, blk).cpu()


class Background:
    """A copy-engine D2H flow on GPU 0 the engine does not control."""

    def __init__(self):
        self.src = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
        self.dst = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
        self.stream = torch.cuda.Stream(device=0)
        self.run = False
        self.bytes = 0

    def __enter__(self):
        self.run = True
        self.t = threading.Thread(target=self.loop, daemon=True)
        self.t.start()
        time.sleep(0.05)
        return self

    def loop(self):
        with torch.cuda.stream(self.stream):
            while self.run:
                for _ in range(4):
                    self.dst.copy_(self.src, non_blocking=True)
                    self.bytes += self.src.numel()
                self.stream.synchronize()

    def __exit__(self, *a):
        self.run = False
        self.t.join()


def check():
    return bool(torch.equal(host.view(nb, blk)[torch.as_tensor(perm)], ref))


def engine_run(policy, reps=4):
    cfg = {"resilience": {"degradation_ratio": 1e9}, "scheduler": {"policy": policy}, "b200": {"chunk_bytes": 65536}}
    e = sp.Engine(fabrics.kv_offload(0, sm_rails=1, relay_via=[1]), json.dumps(cfg), 0)
    e.start()
    e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, nb * blk, pool.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, "g0", [sp.BufferDesc(0, nb * blk, hb.ptr)]))
    reqs = sp.Requests([sp.TransferRequest("hbm", i * blk, "host", int(perm[i]) * blk, blk) for i in range(nb)])
    ts = []
    for k in range(reps + 1):
        host.zero_()
        t0 = time.perf_counter()
        b = e.allocate_batch()
        e.submit_transfers(b, reqs)
        st = e.await_batch(b, 60_000_000_000)
        dt = time.perf_counter() - t0
        assert st.state == sp.BatchState.COMPLETE, st
        e.free_batch(b)
        assert check(), f"{policy}: bytes differ"
        if k:
            ts.append(dt)
    share = {s.rail_id: s.bytes_ok for s in (e.rail_stats(r) for r in range(e.rail_count()))}
    tot = sum(share.values()) or 1
    e.stop()
    return {"gbs": round(nb * blk / (sum(ts) / len(ts)) / 1e9, 2),
            "bytes_share": {k: round(v / tot, 3) for k, v in share.items()}}


def striping(reps=4):
    src = [pool.data_ptr() + i * blk for i in range(nb)]
    dst = [hb.ptr + int(perm[i]) * blk for i in range(nb)]
    ms = []
    for k in range(reps + 1):
        host.zero_()
        m = sp.rr_copy(0, src, dst, [blk] * nb, 4)
        assert check(), "striping: bytes differ"
        if k:
            ms.append(m)
    return {"gbs": round(nb * blk / (sum(ms) / len(ms) * 1e-3) / 1e9, 2)}


out = {"workload": f"{nb} x {blk >> 10} KiB offload GPU0 HBM -> pinned host (NUMA node {hb.node}), random block table",
       "rails": "g0.pcie0 (SM stores, GPU 0 root) + g0.rl1 (relay: NVLink -> GPU 1 HBM -> GPU 1 root)",
       "background": "256 MiB cudaMemcpyAsync D2H loop on GPU 0 (separate stream), not controlled by the engine"}
out["idle"] = {"telemetry": engine_run("telemetry"), "rr": engine_run("rr"), "striping": striping()}
with Background() as bg:
    t0 = time.perf_counter()
    b0 = bg.bytes
    cong = {"telemetry": engine_run("telemetry"), "rr": engine_run("rr"), "striping": striping()}
    cong["background_gbs"] = round((bg.bytes - b0) / (time.perf_counter() - t0) / 1e9, 2)
out["congested"] = cong
out["telemetry_over_striping"] = round(cong["telemetry"]["gbs"] / cong["striping"]["gbs"], 3)
out["telemetry_over_rr"] = round(cong["telemetry"]["gbs"] / cong["rr"]["gbs"], 3)
print(json.dumps(out, indent=1), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/congestion_real.json", "w"), indent=1)
os._exit(0)
