"""Debug: relay rail via the engine's own GPU (1-GPU placement). Runs one small relay-only
batch with a short await, prints the engine's debug words and the relay state, and exits
hard (os._exit) so a stuck forwarder cannot hang the caller."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import _lib as L, fabrics  # noqa: E402

via = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sm = int(sys.argv[2]) if len(sys.argv) > 2 else 0
grid = int(sys.argv[3]) if len(sys.argv) > 3 else 0
topo = fabrics.peer_fabric([0, 1], sm_rails=sm, relay_via=[via], relay_affinity="direct")
print(json.dumps(json.loads(topo)["rails"]), flush=True)
cfg = {"resilience": {"degradation_ratio": 1e9, "slice_timeout_ms": 500}, "b200": {"diag": True}}
if grid:
    cfg["b200"]["grid"] = grid
e = sp.Engine(topo, json.dumps(cfg), 0)
e.start()
n = 8 << 20
src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, src.data_ptr(), n, 5)
dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, n, src.data_ptr())]))
e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, n, dst.data_ptr())]))
b = e.allocate_batch()
e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
st = e.await_batch(b, 10_000_000_000)
w = (C.c_uint64 * 64)()
L.lib.spray_engine_debug(e._h, w, 64)
print("state", st, "debug", list(w), flush=True)
print("relay tail/head/seq0/stamp0/exit_gen", list(w)[45:50], 
      "seq[0:4]", list(w)[53:57], "stamp[0:4]", [hex(x) for x in list(w)[57:61]], "launch_gen", w[61], flush=True)
print("bytes ok", [(e.rail_id(r), e.rail_stats(r).bytes_ok) for r in range(e.rail_count())], flush=True)
if st.state == sp.BatchState.COMPLETE:
    print("exact", sp.checksum(0, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n), flush=True)
os._exit(0)
