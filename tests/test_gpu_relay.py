"""2-hop relay rails (executor "relay"): hop 1 by this engine's copy workers into a staging
slot in the relay GPU's HBM, hop 2 by a forwarder kernel on the relay GPU, which does the
chunk's completion accounting in the engine's counters. Bytes must be bit-exact whatever
the mix of rails, across kernel relaunches, and when the direct rail fails mid-transfer
(the relay is then the alternate path).

Each test runs in two placements:
  * "same_gpu" (1 GPU): source, destination and relay GPU are all GPU 0 (the destination
    segment sits on topology node g1, backed by GPU 0's HBM). Hop 1 stores into the staging
    slots, the forwarder kernel runs beside the engine kernel on the same GPU (the engine
    leaves 16 SMs to it), and every ticket, stamp, slot-recycling and forwarder-exit path
    runs exactly as across GPUs; only the links are local HBM instead of NVLink.
  * "peer" (>= 2 GPUs): destination on GPU 1; the relay GPU is GPU 2 with >= 3 GPUs, else
    the destination GPU itself (hop 2 is then a local HBM copy there)."""
import json

import pytest

torch = pytest.importorskip("torch")

import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

pytestmark = pytest.mark.gpu


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.fixture(params=["same_gpu", "peer"])
def place(request):
    """(destination GPU, relay GPU) for the placement."""
    if request.param == "same_gpu":
        return 0, 0
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    return 1, (2 if ngpu() >= 3 else 1)


def buf(dev, n, seed=None):
    t = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dev}")
    if seed is not None:
        sp.fill_splitmix(dev, t.data_ptr(), n, seed)
    return t


def engine(topo, cfg=None, dev=0):
    base = {"resilience": {"degradation_ratio": 1e9}}
    base.update(cfg or {})
    e = sp.Engine(topo, json.dumps(base), dev)
    e.start()
    return e


def seg(e, sid, g, t):
    """Source segments live on topology node g0, destinations on g1 (whatever GPU backs them)."""
    node = "g0" if sid.startswith("s") else "g1"
    e.register_segment(sp.SegmentDescriptor(sid, sp.Medium.DEVICE, node, [sp.BufferDesc(0, t.numel(), t.data_ptr())]))


def bytes_by_rail(e):
    return {e.rail_id(r): e.rail_stats(r).bytes_ok for r in range(e.rail_count())}


def test_relay_only_random_transfers_bit_exact(place):
    """Every slice crosses the relay GPU: random offsets and lengths (unaligned heads and
    tails, sub-chunk and multi-chunk slices), one batch."""
    dg, v = place
    e = engine(fabrics.peer_fabric([0, 1], sm_rails=0, relay_via=[v], relay_affinity="direct"))
    n = 64 << 20
    src, dst = buf(0, n, 31), buf(dg, n)
    seg(e, "s", 0, src)
    seg(e, "d", dg, dst)
    g = torch.Generator().manual_seed(5)
    reqs, cover = [], torch.zeros(n, dtype=torch.bool)
    for _ in range(48):
        off = int(torch.randint(0, n - 1, (1,), generator=g))
        ln = int(torch.randint(1, min(3 << 20, n - off) + 1, (1,), generator=g))
        reqs.append(sp.TransferRequest("s", off, "d", off, ln))
        cover[off:off + ln] = True
    b = e.allocate_batch()
    e.submit_transfers(b, reqs)
    assert e.await_batch(b, 60_000_000_000).state == sp.BatchState.COMPLETE
    s_, d_ = src.cpu(), dst.cpu()
    assert torch.equal(d_[cover], s_[cover])
    assert not d_[~cover].any()
    assert bytes_by_rail(e)[f"g0.rl{v}"] > 0
    e.stop()


def test_direct_and_relay_sprayed_together_bit_exact(place):
    """A tier-1 SM rail and a tier-1 relay rail share one elephant flow: the scheduler
    sprays slices over both and the delivered bytes are exact."""
    dg, v = place
    e = engine(fabrics.peer_fabric([0, 1], sm_rails=1, relay_via=[v], relay_affinity="direct"))
    n = 256 << 20
    src, dst = buf(0, n, 32), buf(dg, n)
    seg(e, "s", 0, src)
    seg(e, "d", dg, dst)
    for _ in range(3):
        b = e.allocate_batch()
        e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
        assert e.await_batch(b, 60_000_000_000).state == sp.BatchState.COMPLETE
        e.free_batch(b)
    assert sp.checksum(dg, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
    by = bytes_by_rail(e)
    assert by["g0.nvl0"] > 0 and by[f"g0.rl{v}"] > 0
    e.stop()


def test_relay_across_kernel_relaunches(place):
    """The persistent kernel exits when idle and relaunches on the next submit; relay
    tickets restart and the forwarder follows each launch generation."""
    dg, v = place
    e = engine(fabrics.peer_fabric([0, 1], sm_rails=0, relay_via=[v], relay_affinity="direct"),
               {"b200": {"idle_exit_ms": 1}})
    n = 16 << 20
    src = buf(0, n, 33)
    import time
    for k in range(6):
        dst = buf(dg, n)
        seg(e, f"d{k}", dg, dst)
        if k == 0:
            seg(e, "s", 0, src)
        b = e.allocate_batch()
        e.submit_transfer(b, sp.TransferRequest("s", 0, f"d{k}", 0, n))
        assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
        e.free_batch(b)
        assert sp.checksum(dg, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
        time.sleep(0.01)  # past the idle exit: the next submit relaunches
    e.stop()


def test_direct_rail_down_reroutes_over_relay(place):
    """C5 with a relay alternate: the direct SM rail goes DOWN mid-transfer; its slices
    fail, the rail is excluded and the retries cross the relay GPU. Zero lost bytes, heal
    well under 50 ms."""
    dg, v = place
    e = engine(fabrics.peer_fabric([0, 1], sm_rails=1, relay_via=[v]))
    n = 1 << 30
    src, dst = buf(0, n, 34), buf(dg, n)
    seg(e, "s", 0, src)
    seg(e, "d", dg, dst)
    b0 = e.allocate_batch()
    e.submit_transfer(b0, sp.TransferRequest("s", 0, "d", 0, 1 << 20))
    e.await_batch(b0)
    b = e.allocate_batch()
    e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
    now = e.now_ns()
    e.inject_fault("g0.nvl0", sp.FaultEffect.DOWN, now + 300_000, now + 60_000_000_000)
    st = e.await_batch(b, 60_000_000_000)
    assert st.state == sp.BatchState.COMPLETE
    assert sp.checksum(dg, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
    h = e.heal_stats()
    assert h["failed_attempts"] >= 3 and h["retried_ok"] > 0
    heal_ms = (h["first_reroute_ok_ns"] - h["fault_start_ns"]) / 1e6
    assert 0 < heal_ms < 50.0, h
    assert bytes_by_rail(e)[f"g0.rl{v}"] > 0
    e.stop()
