"""Debug: direct SM rail DOWN mid-transfer with a relay alternate via the engine's own GPU
(tests/test_gpu_relay.py::test_direct_rail_down_reroutes_over_relay[same_gpu]); prints the
engine state while the batch is in flight."""
import ctypes as C
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import _lib as L, fabrics  # noqa: E402

n = int(os.environ.get("NBYTES", str(1 << 30)))
T0 = time.time()


def mark(*a):
    print(f"[{time.time() - T0:7.3f}s]", *a, flush=True)


mark("start", n)
e = sp.Engine(fabrics.peer_fabric([0, 1], sm_rails=1, relay_via=[0]),
              json.dumps({"resilience": {"degradation_ratio": 1e9}, "b200": {"diag": True}}), 0)
e.start()
mark("engine started")
src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
sp.fill_splitmix(0, src.data_ptr(), n, 34)
dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, n, src.data_ptr())]))
e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, n, dst.data_ptr())]))
mark("buffers ready")
b0 = e.allocate_batch()
e.submit_transfer(b0, sp.TransferRequest("s", 0, "d", 0, 1 << 20))
mark("warm submitted")
w0 = (C.c_uint64 * 72)()
for _ in range(5):
    st0 = e.await_batch(b0, 2_000_000_000)
    L.lib.spray_engine_debug(e._h, w0, 72)
    mark("warm", st0, "words", list(w0)[:20], "relay", list(w0)[45:47])
    if st0.state != sp.BatchState.IN_FLIGHT:
        break
b = e.allocate_batch()
e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
now = e.now_ns()
e.inject_fault("g0.nvl0", sp.FaultEffect.DOWN, now + 300_000, now + 60_000_000_000)
w = (C.c_uint64 * 72)()
for k in range(8):
    st = e.await_batch(b, 1_000_000_000)
    L.lib.spray_engine_debug(e._h, w, 72)
    ww = list(w)
    print(k, st.state.name, st.remaining, "counters", e.counters(), "heal", e.heal_stats(),
          "rails", [(e.rail_id(r), e.rail_stats(r).bytes_ok, e.rail_stats(r).bytes_failed, e.rail_stats(r).health.name,
                     e.rail_stats(r).queue_depth) for r in range(e.rail_count())],
          "relay tail/head", ww[45:47], "seq", ww[53:57], flush=True)
    if st.state != sp.BatchState.IN_FLIGHT:
        break
if st.state == sp.BatchState.COMPLETE:
    print("exact", sp.checksum(0, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n), flush=True)
os._exit(0)
