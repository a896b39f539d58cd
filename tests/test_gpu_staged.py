"""Staged routes synthesized by the engine (orchestrator.cpp:120-234,
engine.cpp:465-610): when the destination GPU has no peer access (b200.no_peer here, so the
test runs on any box), the engine declares a host-staged relay rail: hop 1 stores each chunk
into a bounded pinned-host pool (2048 x 32 KiB = 64 MiB, the reference's staging pool),
a forwarder on the destination GPU drains it into its HBM, and the chunk's completion comes
back through a ticket-indexed host ring (no peer access to the engine's counters needed).

Placements: "same_gpu" (1 GPU: the destination node is backed by GPU 0, the forwarder runs
beside the engine) and "peer" (>= 2 GPUs: the destination is GPU 1's HBM, drained by GPU 1)."""
import json
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

pytestmark = pytest.mark.gpu


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.fixture(params=["same_gpu", "peer"])
def dgpu(request):
    if request.param == "same_gpu":
        return 0
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    return 1


def make(dgpu, cfg=None):
    base = {"resilience": {"degradation_ratio": 1e9}, "b200": {"no_peer": [1]}}
    for k, v in (cfg or {}).items():
        base.setdefault(k, {}).update(v)
    topo = json.loads(fabrics.peer_fabric([0, 1], sm_rails=1))
    if dgpu == 0:  # the destination node's memory is GPU 0's: its forwarder must run there
        for node, g in (("g0", 0), ("g1", 1)):
            topo["rails"].append({"id": f"{node}.st1", "node": node, "bandwidth_bytes_per_sec": 55e9,
                                  "affinity": "direct", "backend": "cuda", "executor": "relay", "via": 0,
                                  "gpu": g, "staging": "host"})
    e = sp.Engine(json.dumps(topo), json.dumps(base), 0)
    e.start()
    return e


def segs(e, src, dst):
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, src.numel(), src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, dst.numel(), dst.data_ptr())]))


def bytes_by_rail(e):
    return {e.rail_id(r): e.rail_stats(r).bytes_ok for r in range(e.rail_count())}


def test_staged_route_elephant_through_bounded_pool_bit_exact(dgpu):
    """1 GiB through the 64 MiB host pool (16 laps of every staging slot), bit-exact; every
    byte crossed the synthesized staged rail."""
    e = make(dgpu)
    n = 1 << 30
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    sp.fill_splitmix(0, src.data_ptr(), n, 41)
    dst = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dgpu}")
    segs(e, src, dst)
    b = e.allocate_batch()
    t0 = time.perf_counter()
    e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
    st = e.await_batch(b, 120_000_000_000)
    dt = time.perf_counter() - t0
    assert st.state == sp.BatchState.COMPLETE, st
    assert sp.checksum(dgpu, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
    by = bytes_by_rail(e)
    assert by["g0.st1"] == n and by.get("g0.nvl0", 0) == 0
    print(f"staged 1 GiB: {n / dt / 1e9:.1f} GB/s")
    e.stop()


def test_staged_route_random_intents_bit_exact(dgpu):
    """Unaligned offsets and lengths (sub-chunk heads and tails), one batch."""
    e = make(dgpu)
    n = 96 << 20
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    sp.fill_splitmix(0, src.data_ptr(), n, 42)
    dst = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dgpu}")
    segs(e, src, dst)
    rng = np.random.default_rng(6)
    reqs, cover = [], torch.zeros(n, dtype=torch.bool)
    for _ in range(64):
        off = int(rng.integers(0, n - 1))
        ln = int(rng.integers(1, min(3 << 20, n - off) + 1))
        reqs.append(sp.TransferRequest("s", off, "d", off, ln))
        cover[off:off + ln] = True
    b = e.allocate_batch()
    e.submit_transfers(b, reqs)
    assert e.await_batch(b, 60_000_000_000).state == sp.BatchState.COMPLETE
    s_, d_ = src.cpu(), dst.cpu()
    assert torch.equal(d_[cover], s_[cover])
    assert not d_[~cover].any()
    e.stop()


def test_staged_route_across_kernel_relaunches(dgpu):
    """The engine exits when idle and relaunches; staged tickets, the host ring and the
    forwarder restart with each launch generation."""
    e = make(dgpu, {"b200": {"idle_exit_ms": 1}})
    n = 16 << 20
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    sp.fill_splitmix(0, src.data_ptr(), n, 43)
    dst = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dgpu}")
    segs(e, src, dst)
    for k in range(5):
        dst.zero_()
        torch.cuda.synchronize(dgpu)
        b = e.allocate_batch()
        e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
        assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
        e.free_batch(b)
        assert sp.checksum(dgpu, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
        time.sleep(0.01)
    e.stop()
