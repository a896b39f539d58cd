"""Quick end-to-end probe of the CUDA path on one B200 (development aid)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics, trace  # noqa: E402
from oracle.oracle import COracle, ResConfig, SchedConfig  # noqa: E402

out = {}
co = COracle()
# 1. device replay vs golden
z = np.load("tests/golden/replay.npz")
cases = sorted({k.split("__")[0] for k in z.files})
ok = 0
for c in cases:
    sc = SchedConfig.from_buffer_copy(z[c + "__sc"].tobytes())
    rc = ResConfig.from_buffer_copy(z[c + "__rc"].tobytes())
    from paper_2604_00368_b200 import _lib as L
    sc2 = L.SchedConfig.from_buffer_copy(bytes(sc))
    rc2 = L.ResConfig.from_buffer_copy(bytes(rc))
    dec, bad = trace.replay_device(0, sc2, rc2, z[c + "__bw"], z[c + "__tier"], z[c + "__rank"], z[c + "__stream"],
                                   z[c + "__events"])
    same = dec.tobytes() == z[c + "__decisions"].tobytes()
    ok += same
    if not same:
        g = z[c + "__decisions"]
        k = next((i for i in range(min(len(g), len(dec))) if g[i].tobytes() != dec[i].tobytes()), None)
        print("replay mismatch", c, len(dec), len(g), "first diff", k, dec[k] if k is not None else None,
              g[k] if k is not None else None, flush=True)
out["replay_ok"] = f"{ok}/{len(cases)}"
print(out, flush=True)

# 2. engine: 64 MiB HBM -> HBM over 2 rails (config 1 plan on device)
topo = fabrics.two_node(2, 1e9, backend="cuda")
e = sp.Engine(topo, json.dumps({"backends": ["cuda"]}), 0)
e.start()
e.trace_enable(1 << 16)
n = 64 << 20
src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, src.data_ptr(), n, 1 ^ 0x517CC1B727220A95)
torch.cuda.synchronize()
e.register_segment(sp.SegmentDescriptor("bench/src", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
e.register_segment(sp.SegmentDescriptor("bench/dst", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
b = e.allocate_batch()
t0 = time.perf_counter()
e.submit_transfer(b, sp.TransferRequest("bench/src", 0, "bench/dst", 0, n))
st = e.await_batch(b, 20_000_000_000)
t1 = time.perf_counter()
out["c1_status"] = str(st)
out["c1_ms"] = (t1 - t0) * 1e3
out["c1_equal"] = bool(torch.equal(src, dst))
ev, dec = e.trace_fetch(1 << 16)
out["c1_decisions"] = int(len(dec))
out["c1_rails"] = np.bincount(dec["local"]).tolist() if len(dec) else []
z1 = np.load("tests/golden/c1.npz")
g = z1["decisions"]
out["c1_plan_identical"] = bool(len(dec) == len(g) and np.array_equal(dec["local"], g["local"]) and
                                np.array_equal(dec["remote"], g["remote"]))
out["c1_checksum_ok"] = sp.checksum(0, dst.data_ptr(), n) == int(z1["dst_checksum"])
print(out, flush=True)
e.free_batch(b)

# 3. KV offload: 4096 x 64 KiB HBM -> pinned host, random block table
topo = fabrics.kv_offload(0, sm_rails=1)
k = sp.Engine(topo, None, 0)
k.start()
blk, nb = 64 << 10, 4096
pool = torch.empty(blk * nb, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, pool.data_ptr(), blk * nb, 7)
host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
k.register_segment(sp.SegmentDescriptor("kv/hbm", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
k.register_segment(sp.SegmentDescriptor("kv/host", sp.Medium.HOST, "g0", [sp.BufferDesc(0, blk * nb, host.data_ptr())]))
perm = np.random.default_rng(3).permutation(nb)
reqs = [sp.TransferRequest("kv/hbm", i * blk, "kv/host", int(perm[i]) * blk, blk) for i in range(nb)]
for it in range(3):
    b = k.allocate_batch()
    t0 = time.perf_counter()
    k.submit_transfers(b, reqs)
    st = k.await_batch(b, 20_000_000_000)
    t1 = time.perf_counter()
    k.free_batch(b)
    out[f"kv_e2e_gbs_{it}"] = blk * nb / (t1 - t0) / 1e9
p = k.prepare_transfers(reqs)
for it in range(3):
    b = k.allocate_batch()
    ms = p.run(b)
    st = k.batch_status(b)
    k.free_batch(b)
    out[f"kv_dev_gbs_{it}"] = blk * nb / (ms * 1e-3) / 1e9
    out[f"kv_dev_state_{it}"] = str(st.state)
hv = host.numpy().reshape(nb, blk)
pv = pool.cpu().numpy().reshape(nb, blk)
out["kv_equal"] = bool(np.array_equal(hv[perm], pv))
out["kv_rail"] = str(k.rail_stats(0))[:200]
print(json.dumps(out, indent=1), flush=True)
k.stop()
e.stop()
