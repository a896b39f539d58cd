"""Timeouts, lost completions, jitter and posting windows on the device (SURVEY.md §8 a12,
a14, a16).

* DROP_COMPLETION (sim_backend.cpp:118-121, 139): the bytes land but the completion is lost;
  the device deadline scan (worker_timeout_phase, engine.cpp:996-1022) times the attempt
  out, handle_failure retries it elsewhere, the batch completes bit-exact
  (test_engine.cpp:236-256; acceptance criterion 9, acceptance.cpp:470-538).
* JITTER (sim_backend.cpp:52-63): uniform added delay per unit; bytes exact, plans replay.
* Posting windows + post-time re-decide (engine.cpp:855-971): a DOWN rail fails at most a
  window of attempts; the slices queued behind it are released and decided again, and the
  RELEASE / DECIDE events replay identically through the oracle and the device replay.
* Exactly-once accounting under stress: more CE orders than the proxy ring holds, and more
  than 16 failed batches whose slots are reused while their slices are still in flight.
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import _lib, fabrics, trace  # noqa: E402
from oracle.oracle import RefOracle, ref_available, res_config, sched_config  # noqa: E402

DEV = 0
EV_COMPLETE, EV_RELEASE, EV_DECIDE = 2, 4, 1


def dev_buf(n, fill_seed=None):
    t = torch.zeros(max(n, 1), dtype=torch.uint8, device=f"cuda:{DEV}")
    if fill_seed is not None:
        sp.fill_splitmix(DEV, t.data_ptr(), n, fill_seed)
    return t


def make_engine(topo, cfg=None):
    e = sp.Engine(topo, json.dumps(cfg or {}), DEV)
    e.start()
    return e


def segs(e, src, dst, n, src_node="a", dst_node="b"):
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, src_node, [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, dst_node, [sp.BufferDesc(0, n, dst.data_ptr())]))


def warm(e):
    """One small batch so the kernel (and the engine clock) is live."""
    b = e.allocate_batch()
    e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, 4096))
    assert e.await_batch(b, 20_000_000_000).state == sp.BatchState.COMPLETE
    e.free_batch(b)


def rails_of(topo):
    doc = json.loads(topo)
    ids = [r["id"] for r in doc["rails"]]
    order = sorted(range(len(ids)), key=lambda i: ids[i])
    rank = [0] * len(ids)
    for k, i in enumerate(order):
        rank[i] = k
    aff = {"direct": 1, "same_socket": 2, "cross_socket": 3}
    return ([float(r["bandwidth_bytes_per_sec"]) for r in doc["rails"]],
            [aff[r["affinity"]] for r in doc["rails"]], rank)


def replay_live(co, e, topo, sc, rc):
    """The engine's live trace through the C oracle, the device replay and (when built)
    the unmodified reference library: identical decisions, no health mismatch."""
    ev, dec = e.trace_fetch(1 << 20)
    cand = e.trace_candidates()
    bw, tier, rank = rails_of(topo)
    ref = co.replay(sc, rc, bw, tier, rank, cand, ev)
    assert ref["decisions"].tobytes() == dec.tobytes()
    assert ref["expect_failures"] == 0
    ddec, bad = trace.replay_device(DEV, _lib.SchedConfig.from_buffer_copy(bytes(sc)),
                                    _lib.ResConfig.from_buffer_copy(bytes(rc)), bw, tier, rank, cand, ev)
    assert ddec.tobytes() == dec.tobytes() and bad == 0
    if ref_available():
        r = RefOracle().replay(topo, sc, rc, cand, ev, len(bw))
        assert r["decisions"].tobytes() == dec.tobytes()
    return ev, dec


def quiescent(e):
    c = e.counters()
    assert c["bytes_dispatched"] == c["bytes_terminated"], c


# ------------------------------------------------------------------ lost completions
def test_dropped_completions_recover_via_timeout_driven_retry(co):
    """test_engine.cpp:236-256: a.r0 drops every completion for 100 s. Its attempts land
    their bytes but report nothing; each times out (20 ms here), counts as a failure
    (three exclude the rail), and the retry lands on a.r1. Complete, bit-exact, no failed
    batch, bytes_failed > 0, quiescent; the live trace (with TIMEOUT completions) replays
    identically through the oracle, the device replay and the reference."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    cfg = {"resilience": {"degradation_ratio": 1e9, "slice_timeout_ms": 20}}
    e = make_engine(topo, cfg)
    e.trace_enable(1 << 16)
    n = 1 << 20
    src, dst = dev_buf(n, 61), dev_buf(n)
    segs(e, src, dst, n)
    warm(e)
    e.inject_fault("a.r0", sp.FaultEffect.DROP_COMPLETION, 0, 100_000_000_000)
    b = e.allocate_batch()
    e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
    st = e.await_batch(b, 30_000_000_000)
    assert st.state == sp.BatchState.COMPLETE
    assert torch.equal(src, dst)
    assert e.counters()["batches_failed"] == 0
    failed = sum(e.rail_stats(r).bytes_failed for r in range(e.rail_count()))
    assert failed > 0
    assert e.rail_stats(0).health != sp.Health.HEALTHY  # three timeouts excluded a.r0
    quiescent(e)
    ev, _ = replay_live(co, e, topo, sched_config(), res_config(degradation_ratio=1e9))
    comp = ev[ev["kind"] == EV_COMPLETE]
    assert ((comp["flags"] >> 8) & 0xFF == 2).sum() >= 3  # SPRAY_SLICE_TIMEOUT
    e.stop()


def test_criterion9_drop_completion_random_schedules():
    """acceptance.cpp:470-538 (criterion 9): random fabrics of 2-4 rails per node, 1..rails
    DROP_COMPLETION faults on random rails and random windows, a random-length transfer;
    every round completes byte-exact (timeouts + idempotent retries)."""
    rng = np.random.default_rng(99)
    for rnd in range(10):
        rails = 2 + int(rng.integers(0, 3))
        topo = fabrics.two_node(rails, 1e9, backend="cuda")
        e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9, "slice_timeout_ms": 10,
                                              "probe_interval_ms": 20}})
        ln = 1 + int(rng.integers(0, 4 << 20))
        src, dst = dev_buf(ln, 1000 + rnd), dev_buf(ln)
        segs(e, src, dst, ln)
        if ln >= 4096:
            warm(e)
        now = e.now_ns()
        used = set()
        for _ in range(1 + int(rng.integers(0, rails))):
            rail = ("a.r" if rng.integers(0, 2) else "b.r") + str(int(rng.integers(0, rails)))
            if rail in used:
                continue
            used.add(rail)
            start = now + int(rng.integers(0, 5_000_000))
            e.inject_fault(rail, sp.FaultEffect.DROP_COMPLETION, start,
                           start + 100_000_000 + int(rng.integers(0, 2_000_000_000)))
        dst.zero_()
        torch.cuda.synchronize()
        b = e.allocate_batch()
        e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, ln))
        st = e.await_batch(b, 300_000_000_000)
        assert st.state == sp.BatchState.COMPLETE, f"round {rnd} failed"
        assert torch.equal(src[:ln], dst[:ln]), f"round {rnd} bytes differ"
        quiescent(e)
        e.stop()


def test_dropped_completions_on_copy_engine_rail_time_out():
    """The CE proxy honours DROP_COMPLETION too: the host copy lands, the completion is
    never posted, the device deadline scan retries it on the SM rail."""
    topo = fabrics.kv_offload(DEV, sm_rails=1, ce_rails=1)
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9, "slice_timeout_ms": 20}})
    blk, nb = 1 << 20, 32
    pool = dev_buf(blk * nb, fill_seed=71)
    host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
    e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, f"g{DEV}", [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, f"g{DEV}", [sp.BufferDesc(0, blk * nb, host.data_ptr())]))
    e.inject_fault(f"g{DEV}.ce0", sp.FaultEffect.DROP_COMPLETION, 0, 1 << 62)
    b = e.allocate_batch()
    e.submit_transfers(b, [sp.TransferRequest("hbm", i * blk, "host", i * blk, blk) for i in range(nb)])
    assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
    assert torch.equal(pool.cpu(), host)
    ids = {e.rail_id(r): r for r in range(e.rail_count())}
    assert e.rail_stats(ids[f"g{DEV}.ce0"]).bytes_failed > 0
    quiescent(e)
    e.stop()


# ------------------------------------------------------------------ jitter
def test_jitter_fault_bit_exact_and_trace_replays(co):
    """JITTER on a.r0 (uniform added delay up to 300 us per unit): slower completions feed
    the cost model (beta1 rises, the spray shifts to a.r1); bytes exact and the live plan
    replays identically."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536}})
    e.trace_enable(1 << 18)
    n = 64 << 20
    src, dst = dev_buf(n, 81), dev_buf(n)
    segs(e, src, dst, n)
    warm(e)
    e.inject_fault("a.r0", sp.FaultEffect.JITTER, 0, 1 << 62, jitter_us=300.0)
    rng = np.random.default_rng(5)
    ranges = []
    for _ in range(4):
        b = e.allocate_batch()
        reqs = []
        for _ in range(6):
            ln = int(rng.integers(64 << 10, 4 << 20))
            off = int(rng.integers(0, n - ln))
            reqs.append(sp.TransferRequest("s", off, "d", off, ln))
            ranges.append((off, ln))
        e.submit_transfers(b, reqs)
        assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
        e.free_batch(b)
    torch.cuda.synchronize()
    for off, ln in ranges:
        assert torch.equal(src[off:off + ln], dst[off:off + ln])
    assert e.rail_stats(0).beta1 > e.rail_stats(1).beta1
    quiescent(e)
    replay_live(co, e, topo, sched_config(), res_config(degradation_ratio=1e9))
    e.stop()


def test_jitter_entry_validation():
    topo = fabrics.two_node(1, 1e9, backend="cuda")
    e = make_engine(topo)
    with pytest.raises(sp.ConfigError):
        e.inject_fault("a.r0", sp.FaultEffect.JITTER, 0, 10, jitter_us=-1.0)
    with pytest.raises(sp.ConfigError):
        e.inject_fault("a.r0", sp.FaultEffect.DEGRADE, 0, 10, factor=1.5)
    with pytest.raises(sp.ConfigError):
        e.inject_fault("a.r0", sp.FaultEffect.DROP_COMPLETION, 10, 10)
    e.stop()


# ------------------------------------------------------------------ posting windows
@pytest.mark.parametrize("policy", ["telemetry", "rr"])
def test_down_fault_fails_at_most_a_window_and_redecides_the_queue(co, policy):
    """engine.cpp:884-948 + 896-916: with a 64-unit posting window per rail, a rail that
    goes DOWN under a 256 MiB flow fails at most its window (plus the attempts posted
    while the first failures travel back) instead of every queued slice; the rest of its
    queue is released and decided again on the healthy rail. Bit-exact; RELEASE events in
    the live trace; it replays identically."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    win = 64
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9},
                           "scheduler": {"policy": policy},
                           "b200": {"chunk_bytes": 65536, "post_window": win}})
    e.trace_enable(1 << 18)
    n = 256 << 20
    src, dst = dev_buf(n, 91), dev_buf(n)
    segs(e, src, dst, n)
    warm(e)
    b = e.allocate_batch()
    e.submit_transfers(b, [sp.TransferRequest("s", k * (n // 8), "d", k * (n // 8), n // 8) for k in range(8)])
    now = e.now_ns()
    e.inject_fault("a.r0", sp.FaultEffect.DOWN, now + 200_000, now + 60_000_000_000)
    st = e.await_batch(b, 60_000_000_000)
    assert st.state == sp.BatchState.COMPLETE
    assert torch.equal(src, dst)
    h = e.heal_stats()
    window_slices = win  # 32 MiB transfers decompose into 512 x 64 KiB slices: one unit each
    assert 3 <= h["failed_attempts"] <= 2 * window_slices + 32, (h, window_slices)
    ev, _ = replay_live(co, e, topo, sched_config(policy={"telemetry": 0, "rr": 1}[policy]),
                        res_config(degradation_ratio=1e9))
    assert (ev["kind"] == EV_RELEASE).sum() > 0  # queued slices were released and re-decided
    quiescent(e)
    e.stop()


def test_window_bounds_units_in_flight_without_changing_bytes():
    """Tiny windows (1 unit) still deliver everything: the queue drains one unit at a time
    per rail as completions retire."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}, "b200": {"post_window": 1}})
    n = 32 << 20
    src, dst = dev_buf(n, 93), dev_buf(n)
    segs(e, src, dst, n)
    b = e.allocate_batch()
    e.submit_transfers(b, [sp.TransferRequest("s", k << 20, "d", k << 20, 1 << 20) for k in range(32)])
    assert e.await_batch(b, 60_000_000_000).state == sp.BatchState.COMPLETE
    assert torch.equal(src, dst)
    quiescent(e)
    e.stop()


# ------------------------------------------------------------------ exactly-once under stress
def test_more_ce_orders_than_the_proxy_ring():
    """8192 scattered 64 KiB blocks on one copy-engine rail (the proxy ring holds
    4096 orders): the CE window (2048) keeps EGRESS from overrunning the proxy."""
    topo = fabrics.kv_offload(DEV, sm_rails=0, ce_rails=1)
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    blk, nb = 64 << 10, 8192
    pool = dev_buf(blk * nb, fill_seed=73)
    host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
    e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, f"g{DEV}", [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, f"g{DEV}", [sp.BufferDesc(0, blk * nb, host.data_ptr())]))
    perm = np.random.default_rng(3).permutation(nb)
    b = e.allocate_batch()
    e.submit_transfers(b, [sp.TransferRequest("hbm", int(i) * blk, "host", int(p) * blk, blk) for i, p in enumerate(perm)])
    assert e.await_batch(b, 120_000_000_000).state == sp.BatchState.COMPLETE
    h = host.view(nb, blk)
    p = pool.cpu().view(nb, blk)
    assert torch.equal(h[torch.as_tensor(perm)], p)
    quiescent(e)
    e.stop()


def test_many_failed_batches_with_reused_slots():
    """more than 16 batches fail (AllRoutesExhausted, max_attempts 1) and are freed
    while their other slices are still in flight, in 4 reused batch slots; the batches
    that follow in the same slots must count only their own slices (no early COMPLETE,
    no stuck IN_FLIGHT) and deliver exact bytes."""
    topo = fabrics.two_node(1, 1e9, backend="cuda")
    # a failure threshold no run reaches: the rail is never excluded, so every batch fails fast
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9, "max_attempts": 1,
                                          "failure_threshold": 1000000},
                           "b200": {"batch_slots": 4}})
    n = 64 << 20
    src, dst = dev_buf(n, 95), dev_buf(n)
    segs(e, src, dst, n)
    warm(e)
    now = e.now_ns()
    e.inject_fault("a.r0", sp.FaultEffect.DOWN, now, now + 400_000_000)
    failed = 0
    for k in range(24):
        b = e.allocate_batch()
        e.submit_transfers(b, [sp.TransferRequest("s", j << 20, "d", j << 20, 1 << 20) for j in range(16)])
        st = e.await_batch(b, 20_000_000_000)
        failed += st.state == sp.BatchState.FAILED
        e.free_batch(b)  # freed while its other slices may still be in flight
    assert failed > 16
    e.clear_faults()
    for k in range(8):
        dst.zero_()
        torch.cuda.synchronize()
        b = e.allocate_batch()
        e.submit_transfers(b, [sp.TransferRequest("s", j << 22, "d", j << 22, 4 << 20) for j in range(16)])
        st = e.await_batch(b, 60_000_000_000)
        assert st.state == sp.BatchState.COMPLETE, (k, st)
        assert torch.equal(src, dst), k
        e.free_batch(b)
    e.stop()
