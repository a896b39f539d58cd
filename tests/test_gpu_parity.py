"""Parity of the CUDA path (libspray_b200.so on a B200) with the oracle and the reference.

* Device decision function (replay kernel) vs reference-recorded decisions: bit-exact.
* Live engine traces replayed through the C oracle and the device replay: identical plans.
* Config 1 (64 MiB over 2 rails): plan identical to the reference's, delivered bytes equal
  to the reference engine's delivered bytes (checksum).
* Delivered bytes bit-exact for random intents, KV batches, faults and retries.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import _lib, fabrics, trace  # noqa: E402
from oracle.oracle import COracle, ResConfig, SchedConfig, res_config, sched_config  # noqa: E402

DEV = 0


def _cfg_c(sc):
    return _lib.SchedConfig.from_buffer_copy(bytes(sc))


def _rcfg_c(rc):
    return _lib.ResConfig.from_buffer_copy(bytes(rc))


@pytest.fixture(scope="module")
def co():
    return COracle()


def dev_buf(n, fill_seed=None):
    t = torch.zeros(max(n, 1), dtype=torch.uint8, device=f"cuda:{DEV}")
    if fill_seed is not None:
        sp.fill_splitmix(DEV, t.data_ptr(), n, fill_seed)
    return t


# ------------------------------------------------------------------ device decision function
def test_device_replay_matches_reference_goldens(golden_dir):
    z = np.load(os.path.join(golden_dir, "replay.npz"))
    cases = sorted({k.split("__")[0] for k in z.files})
    for c in cases:
        sc = _cfg_c(SchedConfig.from_buffer_copy(z[c + "__sc"].tobytes()))
        rc = _rcfg_c(ResConfig.from_buffer_copy(z[c + "__rc"].tobytes()))
        dec, bad = trace.replay_device(DEV, sc, rc, z[c + "__bw"], z[c + "__tier"], z[c + "__rank"],
                                       z[c + "__stream"], z[c + "__events"])
        assert dec.tobytes() == z[c + "__decisions"].tobytes(), c
        assert bad == 0


def test_fill_and_checksum_match_oracle(co):
    for n in (1, 7, 8, 4099, 1 << 20, (1 << 20) + 3):
        t = dev_buf(n, fill_seed=1234)
        host = t.cpu().numpy()[:n]
        assert np.array_equal(host, co.fill(n, 1234))
        assert sp.checksum(DEV, t.data_ptr(), n) == co.checksum(host)


# ------------------------------------------------------------------ engine helpers
def make_engine(topo, cfg=None):
    e = sp.Engine(topo, json.dumps(cfg or {}), DEV)
    e.start()
    return e


def replay_live(co, e, sc, rc, bw, tier, rank):
    ev, dec = e.trace_fetch(1 << 20)
    cand = e.trace_candidates()
    ref = co.replay(sc, rc, bw, tier, rank, cand, ev)
    assert ref["decisions"].tobytes() == dec.tobytes()
    assert ref["expect_failures"] == 0
    ddec, bad = trace.replay_device(DEV, _cfg_c(sc), _rcfg_c(rc), bw, tier, rank, cand, ev)
    assert ddec.tobytes() == dec.tobytes() and bad == 0
    return ev, dec


def rails_of(topo):
    doc = json.loads(topo)
    ids = [r["id"] for r in doc["rails"]]
    order = sorted(range(len(ids)), key=lambda i: ids[i])
    rank = [0] * len(ids)
    for k, i in enumerate(order):
        rank[i] = k
    aff = {"direct": 1, "same_socket": 2, "cross_socket": 3}
    return ([float(r["bandwidth_bytes_per_sec"]) for r in doc["rails"]], [aff[r["affinity"]] for r in doc["rails"]],
            rank)


# ------------------------------------------------------------------ config 1
def test_config1_plan_and_bytes_match_reference(co, golden_dir):
    z = np.load(os.path.join(golden_dir, "c1.npz"))
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"backends": ["cuda"]})
    e.trace_enable(1 << 16)
    n = 64 << 20
    src = dev_buf(n, fill_seed=1 ^ 0x517CC1B727220A95)  # bench.cpp:99 payload, seed 1
    dst = dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("bench/src", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("bench/dst", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    b = e.allocate_batch()
    e.submit_transfer(b, sp.TransferRequest("bench/src", 0, "bench/dst", 0, n))
    st = e.await_batch(b, 30_000_000_000)
    assert st.state == sp.BatchState.COMPLETE and st.remaining == 0
    assert sp.checksum(DEV, dst.data_ptr(), n) == int(z["dst_checksum"])
    ev, dec = e.trace_fetch(1 << 16)
    g = z["decisions"]
    assert np.array_equal(dec["local"], g["local"]) and np.array_equal(dec["remote"], g["remote"])
    assert dec.tobytes() == g.tobytes()
    c = e.counters()
    assert c["bytes_dispatched"] == c["bytes_terminated"] == n
    e.stop()


# ------------------------------------------------------------------ live trace parity
@pytest.mark.parametrize("policy", ["telemetry", "rr", "hash"])
def test_live_trace_replays_identically(co, policy):
    bws = [4e9, 2e9, 1e9, 1e9]
    topo = fabrics.two_node(4, bws, backend="cuda", affinities=["direct", "direct", "same_socket", "direct"])
    sc = sched_config(policy={"telemetry": 0, "rr": 1, "hash": 2}[policy])
    e = make_engine(topo, {"scheduler": {"policy": policy}, "resilience": {"degradation_ratio": 1e9},
                           "b200": {"chunk_bytes": 65536}})
    e.trace_enable(1 << 18)
    n = 96 << 20
    src = dev_buf(n, fill_seed=5)
    dst = dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    rng = np.random.default_rng(17)
    for _ in range(6):
        b = e.allocate_batch()
        reqs = []
        for _ in range(int(rng.integers(1, 12))):
            ln = int(rng.integers(1, 8 << 20))
            off = int(rng.integers(0, n - ln))
            reqs.append(sp.TransferRequest("s", off, "d", off, ln, sp.Direction(int(rng.integers(0, 2)))))
        e.submit_transfers(b, reqs)
        st = e.await_batch(b, 30_000_000_000)
        assert st.state == sp.BatchState.COMPLETE
        e.free_batch(b)
    torch.cuda.synchronize()
    bw, tier, rank = rails_of(topo)
    ev, dec = replay_live(co, e, sc, res_config(degradation_ratio=1e9), bw, tier, rank)
    assert len(dec) > 50 and (ev["kind"] == 2).sum() == len(dec)
    e.stop()


@pytest.mark.parametrize("policy", ["telemetry", "rr", "hash"])
def test_live_trace_many_candidates_and_uniform_blocks_replay_identically(co, policy):
    """The decision paths by candidate count: 2 and 3 rails (the lane-0 scalar loop over
    per-block score tables) and 8 rails (the warp loop), each fed both uniform 32-slice
    blocks (one-slice intents of one length) and ragged multi-slice intents."""
    for n_rails in (2, 3, 8):
        bws = [float(4e9 / (1 + (i % 3))) for i in range(n_rails)]
        topo = fabrics.two_node(n_rails, bws, backend="cuda")
        sc = sched_config(policy={"telemetry": 0, "rr": 1, "hash": 2}[policy])
        e = make_engine(topo, {"scheduler": {"policy": policy}, "resilience": {"degradation_ratio": 1e9},
                               "b200": {"chunk_bytes": 65536}})
        e.trace_enable(1 << 18)
        n = 64 << 20
        src = dev_buf(n, fill_seed=7 + n_rails)
        dst = dev_buf(n)
        e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
        rng = np.random.default_rng(23 + n_rails)
        for k in range(4):
            b = e.allocate_batch()
            if k % 2 == 0:  # uniform: 256 one-slice intents of 64 KiB at random offsets
                reqs = [sp.TransferRequest("s", int(o) * 65536, "d", int(o) * 65536, 65536)
                        for o in rng.permutation(n // 65536)[:256]]
            else:
                reqs = []
                for _ in range(8):
                    ln = int(rng.integers(1, 6 << 20))
                    off = int(rng.integers(0, n - ln))
                    reqs.append(sp.TransferRequest("s", off, "d", off, ln))
            e.submit_transfers(b, reqs)
            assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
            e.free_batch(b)
        torch.cuda.synchronize()
        bw, tier, rank = rails_of(topo)
        ev, dec = replay_live(co, e, sc, res_config(degradation_ratio=1e9), bw, tier, rank)
        assert len(dec) > 500 and (ev["kind"] == 2).sum() == len(dec)
        e.stop()


def test_live_trace_with_degradation_exclusions_replays_identically(co):
    """Tight degradation settings so rails are excluded by observe() on OK completions
    (the completion fast path's lane-parallel classification) and reintegrated by probes;
    the live trace must still replay to the same decisions and health expectations."""
    topo = fabrics.two_node(2, [2e9, 1e9], backend="cuda")
    rc_kw = dict(degradation_ratio=1.02, degradation_events=2, degradation_min_t_obs_s=0.0,
                 probe_interval_ns=200_000, probe_successes_needed=1)
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1.02, "degradation_events": 2,
                                          "degradation_min_t_obs_ms": 0.0, "probe_interval_ms": 0.2,
                                          "probe_successes": 1},
                           "b200": {"chunk_bytes": 65536}})
    e.trace_enable(1 << 18)
    n = 64 << 20
    src = dev_buf(n, fill_seed=11)
    dst = dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    rng = np.random.default_rng(23)
    ranges = []
    for _ in range(8):
        b = e.allocate_batch()
        reqs = []
        for _ in range(int(rng.integers(2, 10))):
            ln = int(rng.integers(64 << 10, 6 << 20))
            off = int(rng.integers(0, n - ln))
            reqs.append(sp.TransferRequest("s", off, "d", off, ln))
            ranges.append((off, ln))
        e.submit_transfers(b, reqs)
        assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
        e.free_batch(b)
    torch.cuda.synchronize()
    for off, ln in ranges:
        assert torch.equal(src[off:off + ln], dst[off:off + ln])
    bw, tier, rank = rails_of(topo)
    ev, dec = replay_live(co, e, sched_config(), res_config(**rc_kw), bw, tier, rank)
    assert (ev["kind"] == 8).sum() > 0  # SPRAY_EV_EXPECT_HEALTH: exclusions happened
    e.stop()


def test_large_submit_races_device_completion():
    """One submit call whose first published groups complete on the device before the
    host has built the rest: the batch must not be taken for complete mid-call."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    n = 16 << 20
    s, d = dev_buf(n, 3), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, s.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, d.data_ptr())]))
    reqs = sp.Requests([sp.TransferRequest("s", i * 4096, "d", i * 4096, 4096) for i in range(n // 4096)])
    for _ in range(10):
        b = e.allocate_batch()
        e.submit_transfers(b, reqs)
        assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
        e.free_batch(b)
    assert torch.equal(s, d)
    e.stop()


def test_device_decompose_matches_oracle_at_edges(co):
    """SliceScheduler::decompose (scheduler.cpp:94-106) as the INGRESS warp runs it, at the
    edges: single bytes, one short of / exactly / one past the minimum slice and its
    double, the 4096-slice cap (1 GiB -> 256 KiB slices) and a ragged size past the cap.
    Every DECIDE in the live trace carries the slice's length and absolute source offset."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    e.trace_enable(1 << 16)
    n = (1 << 30) + (1 << 20)
    src, dst = dev_buf(n, 19), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    lens = [1, 4095, 65535, 65536, 65537, 131071, 131072, 131073, (64 << 20) + 3, 1 << 30, (1 << 30) + 12345]
    offs = [7, 100, 0, 65536, 3, 1 << 20, 0, 11, 5 << 20, 0, 999]
    b = e.allocate_batch()
    for ln, off in zip(lens, offs):
        e.submit_transfer(b, sp.TransferRequest("s", off, "d", off, ln))
    assert e.await_batch(b, 60_000_000_000).state == sp.BatchState.COMPLETE
    ev, dec = e.trace_fetch(1 << 16)
    d = ev[ev["kind"] == 1]
    k = 0
    for ln, off in zip(lens, offs):
        o, l = co.decompose(ln)
        got = d[k:k + len(o)]
        assert np.array_equal(got["len"], l), ln
        assert np.array_equal(got["offset"] - off, o), ln
        k += len(o)
    assert k == len(d)
    for ln, off in zip(lens, offs):
        assert torch.equal(src[off:off + ln], dst[off:off + ln]), ln
    e.stop()


def test_many_tiny_transfers_in_one_batch_bit_exact():
    """20000 intents of 1..512 bytes at random (unaligned) offsets in one submit call."""
    topo = fabrics.two_node(3, [3e9, 2e9, 1e9], backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    n = 32 << 20
    src, dst = dev_buf(n, 23), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    rng = np.random.default_rng(99)
    cells = rng.permutation(n // 1024)[:20000]  # disjoint 1 KiB cells
    lens = rng.integers(1, 513, size=len(cells))
    offs = cells * 1024 + rng.integers(0, 512, size=len(cells))
    b = e.allocate_batch()
    e.submit_transfers(b, [sp.TransferRequest("s", int(o), "d", int(o), int(l)) for o, l in zip(offs, lens)])
    assert e.await_batch(b, 60_000_000_000).state == sp.BatchState.COMPLETE
    mask = torch.zeros(n, dtype=torch.bool)
    for o, l in zip(offs, lens):
        mask[int(o):int(o) + int(l)] = True
    s_, d_ = src.cpu(), dst.cpu()
    assert torch.equal(s_[mask], d_[mask]) and int((d_[~mask] != 0).sum()) == 0
    e.stop()


# ------------------------------------------------------------------ bytes
def test_random_transfers_bit_exact():
    """Acceptance criterion 1 analogue: randomized lengths (1 B .. 32 MiB) and offsets,
    both directions, HBM->HBM and HBM<->pinned host; delivered bytes memcmp-equal."""
    topo = fabrics.two_node(3, [2e9, 1e9, 1e9], backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    n = 64 << 20
    src = dev_buf(n, fill_seed=9)
    dst = dev_buf(n)
    hsrc = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    hsrc.copy_(src.cpu())
    hdst = torch.zeros(n, dtype=torch.uint8, pin_memory=True)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("hs", sp.Medium.HOST, "a", [sp.BufferDesc(0, n, hsrc.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("hd", sp.Medium.HOST, "b", [sp.BufferDesc(0, n, hdst.data_ptr())]))
    rng = np.random.default_rng(20260809)
    for k in range(60):
        bits = int(rng.integers(0, 26))
        ln = (1 << bits) | (int(rng.integers(0, 1 << bits)) if bits else 0)
        ln = min(ln, n)
        so = int(rng.integers(0, n - ln + 1))
        do = int(rng.integers(0, n - ln + 1))
        s_id, d_id = [("s", "d"), ("s", "hd"), ("hs", "d"), ("hs", "hd")][k % 4]
        b = e.allocate_batch()
        e.submit_transfer(b, sp.TransferRequest(s_id, so, d_id, do, ln, sp.Direction(k % 2)))
        st = e.await_batch(b, 30_000_000_000)
        assert st.state == sp.BatchState.COMPLETE, (k, ln)
        S = src if s_id == "s" else hsrc
        D = dst if d_id == "d" else hdst
        assert torch.equal(S[so:so + ln].cpu(), D[do:do + ln].cpu()), (k, ln, so, do)
        e.free_batch(b)
    c = e.counters()
    assert c["bytes_dispatched"] == c["bytes_terminated"]
    e.stop()


def test_kv_batch_block_table_bit_exact():
    """Config 3 shape: 4096 x 64 KiB HBM -> pinned host through a random block table,
    then host -> HBM back into a second pool."""
    topo = fabrics.kv_offload(DEV, sm_rails=1)
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    blk, nb = 64 << 10, 4096
    pool = dev_buf(blk * nb, fill_seed=7)
    pool2 = dev_buf(blk * nb)
    host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
    e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, f"g{DEV}", [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("hbm2", sp.Medium.DEVICE, f"g{DEV}", [sp.BufferDesc(0, blk * nb, pool2.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, f"g{DEV}", [sp.BufferDesc(0, blk * nb, host.data_ptr())]))
    perm = np.random.default_rng(3).permutation(nb)
    b = e.allocate_batch()
    e.submit_transfers(b, [sp.TransferRequest("hbm", i * blk, "host", int(perm[i]) * blk, blk) for i in range(nb)])
    assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
    e.free_batch(b)
    hv = host.numpy().reshape(nb, blk)
    assert np.array_equal(hv[perm], pool.cpu().numpy().reshape(nb, blk))
    p = e.prepare_transfers([sp.TransferRequest("host", int(perm[i]) * blk, "hbm2", i * blk, blk) for i in range(nb)])
    b = e.allocate_batch()
    ms = p.run(b)
    assert ms > 0 and e.batch_status(b).state == sp.BatchState.COMPLETE
    assert torch.equal(pool, pool2)
    e.free_batch(b)
    e.stop()


# ------------------------------------------------------------------ batch API semantics
def test_batch_api_semantics():
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo)
    n = 1 << 20
    s, d = dev_buf(n, 1), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, s.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, d.data_ptr())]))
    b = e.allocate_batch()
    assert e.batch_status(b).state == sp.BatchState.COMPLETE  # empty batch is complete
    with pytest.raises(sp.InvalidRangeError):
        e.submit_transfer(b, sp.TransferRequest("s", n - 10, "d", 0, 20))
    with pytest.raises(sp.InvalidRangeError):
        e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, 0))
    with pytest.raises(sp.EngineError, match="unknown segment"):
        e.submit_transfer(b, sp.TransferRequest("nope", 0, "d", 0, 10))
    with pytest.raises(sp.EngineError, match="unknown batch"):
        e.submit_transfer(999999, sp.TransferRequest("s", 0, "d", 0, 10))
    e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
    assert e.await_batch(b, 10_000_000_000).state == sp.BatchState.COMPLETE
    with pytest.raises(sp.EngineError, match="already complete"):
        e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, 10))
    e.free_batch(b)
    assert torch.equal(s, d)
    e.stop()


@pytest.mark.parametrize("bad_at", [None, 1500, 2047])
def test_large_submission_staged_through_hbm(bad_at):
    """submit_transfers with >= 1024 requests goes to the device as bulk intent arrays
    (1024 per copy, rotating HBM areas): bytes, ids and batch accounting as one by one,
    across several submissions that reuse the areas; an invalid request raises after the
    requests before it were submitted, exactly as the ring path does."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"b200": {"chunk_bytes": 65536}})
    blk, nb = 16 << 10, 3000
    n = blk * nb
    s, d = dev_buf(n, 31), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, s.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, d.data_ptr())]))
    perm = np.random.default_rng(5).permutation(nb)
    for rep in range(3):  # 3 x 3 pieces: every staging area is reused
        d.zero_()
        torch.cuda.synchronize()
        reqs = [sp.TransferRequest("s", i * blk, "d", int(perm[i]) * blk, blk) for i in range(nb)]
        if bad_at is not None:
            reqs[bad_at] = sp.TransferRequest("s", n - 10, "d", 0, 20)  # out of range
        b = e.allocate_batch()
        if bad_at is None:
            e.submit_transfers(b, reqs)
            upto = nb
        else:
            with pytest.raises(sp.InvalidRangeError):
                e.submit_transfers(b, reqs)
            upto = bad_at
        st = e.await_batch(b, 30_000_000_000)
        assert st.state == sp.BatchState.COMPLETE and st.remaining == 0
        e.free_batch(b)
        src_v, dst_v = s.view(nb, blk), d.view(nb, blk)
        idx = torch.as_tensor(perm[:upto])
        assert torch.equal(dst_v[idx], src_v[:upto])
        if upto < nb:
            assert not dst_v[torch.as_tensor(perm[upto:])].any()
    e.stop()


# ------------------------------------------------------------------ self-healing
@pytest.mark.parametrize("policy", ["telemetry", "rr", "hash"])
def test_down_fault_reroutes_with_zero_lost_bytes(co, policy):
    """Disable one of two rails mid-transfer: its in-flight slices fail (partial prefix
    writes), three consecutive failures exclude it (resilience.cpp:71-83), retries land
    on the healthy rail (engine.cpp:405-454); the batch completes bit-exact and the
    live trace still replays identically, under every policy."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536},
                           "scheduler": {"policy": policy}})
    e.trace_enable(1 << 18)
    n = 256 << 20
    src, dst = dev_buf(n, 11), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    # warm the kernel so the engine clock is live, then fail a.r0 from "now" on
    b0 = e.allocate_batch()
    e.submit_transfer(b0, sp.TransferRequest("s", 0, "d", 0, 1 << 20))
    e.await_batch(b0)
    now = e.now_ns()
    e.inject_fault("a.r0", sp.FaultEffect.DOWN, now, now + 60_000_000_000)
    b = e.allocate_batch()
    for k in range(8):
        e.submit_transfer(b, sp.TransferRequest("s", k * (n // 8), "d", k * (n // 8), n // 8))
    st = e.await_batch(b, 60_000_000_000)
    assert st.state == sp.BatchState.COMPLETE
    assert torch.equal(src, dst)
    h = e.heal_stats()
    assert h["failed_attempts"] >= 3 and h["retried_ok"] > 0
    assert e.rail_stats(0).health != sp.Health.HEALTHY
    heal_ms = (h["first_reroute_ok_ns"] - h["fault_start_ns"]) / 1e6
    assert 0 < heal_ms < 50.0
    bw, tier, rank = rails_of(topo)
    replay_live(co, e, sched_config(policy={"telemetry": 0, "rr": 1, "hash": 2}[policy]),
                res_config(degradation_ratio=1e9), bw, tier, rank)
    e.stop()


@pytest.mark.parametrize("delay_us", [0, 150, 600])
def test_fault_starting_mid_transfer_is_bit_exact(delay_us):
    """A DOWN fault that begins while chunks of the rail are in flight (the scheduled-
    fault path: 16 KiB steps, stop at the fault's start, partial prefix write): every
    affected attempt must be reported FAILED and re-sprayed; no holes in delivered bytes."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    n = 512 << 20
    src, dst = dev_buf(n, 13 + delay_us), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    b0 = e.allocate_batch()
    e.submit_transfer(b0, sp.TransferRequest("s", 0, "d", 0, 1 << 20))
    e.await_batch(b0)
    b = e.allocate_batch()
    e.submit_transfers(b, [sp.TransferRequest("s", k * (n // 16), "d", k * (n // 16), n // 16) for k in range(16)])
    now = e.now_ns()
    e.inject_fault("a.r0", sp.FaultEffect.DOWN, now + delay_us * 1000, now + 60_000_000_000)
    st = e.await_batch(b, 60_000_000_000)
    assert st.state == sp.BatchState.COMPLETE
    assert torch.equal(src, dst)
    c = e.counters()
    assert c["bytes_dispatched"] == c["bytes_terminated"]
    e.stop()


def test_dataflow_gate_forwarding_chain_bit_exact():
    """Two engines form a 2-hop relay on one GPU: engine A copies src -> mid and produces
    mid's granules; engine B copies mid -> dst and consumes them granule by granule while
    A is still writing. Repeated runs reuse the same counters; bytes stay exact."""
    topo = fabrics.two_node(1, 1e9, backend="cuda")
    cfg = {"resilience": {"degradation_ratio": 1e9},
           "b200": {"grid": 64, "gate_timeout_ms": 20000, "chunk_bytes": 65536}}  # 64 KiB slices = granules
    a, b = make_engine(topo, cfg), make_engine(topo, cfg)
    n = 64 << 20
    src, mid, dst = dev_buf(n, 41), dev_buf(n), dev_buf(n)
    for e in (a, b):
        e.register_segment(sp.SegmentDescriptor("src", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("mid", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, mid.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("dst", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    cb = a.chunk_bytes()
    flags = torch.zeros(n // cb, dtype=torch.int32, device=f"cuda:{DEV}")
    a.gate_segment("mid", sp.Engine.GATE_PRODUCE, flags.data_ptr())
    b.gate_segment("mid", sp.Engine.GATE_CONSUME, flags.data_ptr())
    with pytest.raises(sp.InvalidRangeError):
        bx = b.allocate_batch()
        b.submit_transfer(bx, sp.TransferRequest("mid", 100, "dst", 0, cb))
    for run in range(3):
        mid.zero_()
        dst.zero_()
        torch.cuda.synchronize()
        bb = b.allocate_batch()
        b.submit_transfer(bb, sp.TransferRequest("mid", 0, "dst", 0, n))  # waits on the gate
        ba = a.allocate_batch()
        a.submit_transfer(ba, sp.TransferRequest("src", 0, "mid", 0, n))
        assert a.await_batch(ba, 60_000_000_000).state == sp.BatchState.COMPLETE
        assert b.await_batch(bb, 60_000_000_000).state == sp.BatchState.COMPLETE
        a.free_batch(ba)
        b.free_batch(bb)
        assert torch.equal(src, dst), run
        assert int(flags.min()) == run + 1 and int(flags.max()) == run + 1
    a.stop()
    b.stop()


def test_staged_route_through_host_memory_bit_exact():
    """Staged multi-hop route (engine.cpp:465-610 analog): HBM ->
    pinned host staging -> HBM, pipelined by granule between two engines. The gate
    counters live in mapped host memory, so the route needs no peer access."""
    topo = fabrics.kv_offload(DEV)
    cfg = {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536, "gate_timeout_ms": 20000}}
    a, b = make_engine(topo, cfg), make_engine(topo, cfg)
    n = 128 << 20
    src, dst = dev_buf(n, 57), dev_buf(n)
    stage = torch.zeros(n, dtype=torch.uint8, pin_memory=True)
    cb = a.chunk_bytes()
    flags_p = sp.host_alloc(4 * (n // cb))
    C.memset(flags_p, 0, 4 * (n // cb))
    node = f"g{DEV}"
    for e in (a, b):
        e.register_segment(sp.SegmentDescriptor("src", sp.Medium.DEVICE, node, [sp.BufferDesc(0, n, src.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("stage", sp.Medium.HOST, node, [sp.BufferDesc(0, n, stage.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("dst", sp.Medium.DEVICE, node, [sp.BufferDesc(0, n, dst.data_ptr())]))
    a.gate_segment("stage", sp.Engine.GATE_PRODUCE, flags_p)
    b.gate_segment("stage", sp.Engine.GATE_CONSUME, flags_p)
    flags = np.ctypeslib.as_array((C.c_uint32 * (n // cb)).from_address(flags_p))
    for run in range(2):
        dst.zero_()
        torch.cuda.synchronize()
        bb = b.allocate_batch()
        b.submit_transfer(bb, sp.TransferRequest("stage", 0, "dst", 0, n))
        ba = a.allocate_batch()
        a.submit_transfer(ba, sp.TransferRequest("src", 0, "stage", 0, n))
        assert a.await_batch(ba, 60_000_000_000).state == sp.BatchState.COMPLETE
        assert b.await_batch(bb, 60_000_000_000).state == sp.BatchState.COMPLETE
        a.free_batch(ba)
        b.free_batch(bb)
        assert torch.equal(src, dst), run
        assert int(flags.min()) == run + 1 and int(flags.max()) == run + 1
    a.stop()
    b.stop()
    sp.host_free(flags_p)


def test_staged_ring_route_bounded_pool_bit_exact():
    """Staged route through a BOUNDED staging pool (reference staged_* pipeline,
    engine.cpp:465-527; 4 MiB chunks x ring depth 4, engine.hpp:56-58): 192 MiB moves
    HBM -> 16 MiB pinned-host ring -> HBM, 12 laps, in two transfers that continue the
    ring's lap count. Every byte arrives; every granule's credit equals its laps; a
    transfer larger than the ring and a misaligned offset are rejected like the reference's
    InvalidRangeError."""
    topo = fabrics.kv_offload(DEV)
    cfg = {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536, "gate_timeout_ms": 20000}}
    a, b = make_engine(topo, cfg), make_engine(topo, cfg)
    n = 96 << 20
    src, dst = dev_buf(n, 91), dev_buf(n)
    node = f"g{DEV}"
    for e in (a, b):
        e.register_segment(sp.SegmentDescriptor("src", sp.Medium.DEVICE, node, [sp.BufferDesc(0, n, src.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("dst", sp.Medium.DEVICE, node, [sp.BufferDesc(0, n, dst.data_ptr())]))
    route = sp.StagedRoute(a, b, node, node, chunk_bytes=4 << 20, depth=4)
    assert route.ring_bytes == 16 << 20
    granules = route.ring_bytes // a.chunk_bytes()
    ctl = np.ctypeslib.as_array((C.c_uint32 * (2 * granules)).from_address(route._ctl))
    for run in range(2):
        dst.zero_()
        torch.cuda.synchronize()
        assert route.transfer("src", 0, "dst", 0, n) == sp.BatchState.COMPLETE
        assert torch.equal(src, dst), run
        laps = (run + 1) * n // route.ring_bytes
        assert int(ctl[:granules].min()) == laps and int(ctl[:granules].max()) == laps  # flags
        assert int(ctl[granules:].min()) == laps and int(ctl[granules:].max()) == laps  # credits
    ba = a.allocate_batch()
    with pytest.raises(sp.InvalidRangeError):
        a.submit_transfer(ba, sp.TransferRequest("src", 0, route.seg_id, route.cursor, route.ring_bytes + (64 << 10)))
    with pytest.raises(sp.InvalidRangeError):
        a.submit_transfer(ba, sp.TransferRequest("src", 4096, route.seg_id, route.cursor, 1 << 20))
    a.free_batch(ba)
    a.stop()
    b.stop()
    route.close()


def test_telemetry_csv_windows_account_every_byte():
    """TelemetrySnapshot::to_csv columns (telemetry.cpp:123-158) from the device window
    cells: per-window bytes sum to the delivered bytes, per rail; percentiles ordered."""
    topo = fabrics.two_node(2, [2e9, 1e9], backend="cuda")
    e = make_engine(topo, {"stats_window_ms": 1, "resilience": {"degradation_ratio": 1e9}})
    n = 96 << 20
    src, dst = dev_buf(n, 3), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    for k in range(4):
        b = e.allocate_batch()
        e.submit_transfer(b, sp.TransferRequest("s", k * (n // 4), "d", k * (n // 4), n // 4))
        assert e.await_batch(b).state == sp.BatchState.COMPLETE
        e.free_batch(b)
    csv = e.telemetry_csv().strip().splitlines()
    assert csv[0] == ("window_start_ms,rail_id,bytes_ok,bytes_failed,queue_depth_bytes,p50_us,p99_us,"
                      "health_state,throughput_gbps")
    rows = [r.split(",") for r in csv[1:]]
    assert len(rows) > 0 and len(rows) % 4 == 0  # every window has one row per rail
    by_rail = {}
    for r in rows:
        by_rail[r[1]] = by_rail.get(r[1], 0) + int(r[2])
        assert int(r[3]) == 0 and r[7] in ("healthy", "excluded", "probing")
        assert float(r[6]) >= float(r[5]) >= 0.0
    for i in range(e.rail_count()):
        assert by_rail.get(e.rail_id(i), 0) == e.rail_stats(i).bytes_ok
    assert sum(by_rail.values()) == n
    e.stop()


def test_all_rails_down_stall_then_complete_after_probing(co):
    """test_engine.cpp:258-272: every rail down for 100 ms; slices park, the prober
    (1 s cadence, 2 OK probes) reintegrates the rails, the batch completes bit-exact with
    zero failed batches; the live trace (with DUE_PROBES / PROBE_DONE) replays identically."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    e.trace_enable(1 << 16)
    n = 1 << 20
    src, dst = dev_buf(n, 4), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    b0 = e.allocate_batch()
    e.submit_transfer(b0, sp.TransferRequest("s", 0, "d", 0, 4096))
    e.await_batch(b0)
    now = e.now_ns()
    for r in ("a.r0", "a.r1", "b.r0", "b.r1"):
        e.inject_fault(r, sp.FaultEffect.DOWN, 0, now + 100_000_000)
    b = e.allocate_batch()
    e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
    st = e.await_batch(b, 20_000_000_000)
    assert st.state == sp.BatchState.COMPLETE
    assert torch.equal(src, dst)
    assert e.counters()["batches_failed"] == 0
    assert all(e.rail_stats(r).health == sp.Health.HEALTHY for r in range(4))
    bw, tier, rank = rails_of(topo)
    ev, _ = replay_live(co, e, sched_config(), res_config(degradation_ratio=1e9), bw, tier, rank)
    assert (ev["kind"] == 9).sum() >= 1 and (ev["kind"] == 10).sum() >= 2
    e.stop()


def test_attempts_exhausted_fails_batch_with_all_routes_exhausted():
    topo = fabrics.two_node(1, 1e9, backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9, "max_attempts": 1}})
    n = 4 << 20
    src, dst = dev_buf(n, 3), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    e.inject_fault("a.r0", sp.FaultEffect.DOWN, 0, 1 << 62)
    b = e.allocate_batch()
    e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
    st = e.await_batch(b, 20_000_000_000)
    assert st.state == sp.BatchState.FAILED and st.failure_reason == "AllRoutesExhausted"
    e.free_batch(b)
    e.stop()


def test_backend_substitution_after_exhausted_attempts(co):
    """substitute_or_fail / advance_past_backend / reissue (engine.cpp:676-761,
    orchestrator.cpp:20-33): the plan holds two routes, backend "cuda" (active, better
    tier) and backend "memory". Every rail of the active route is DOWN for the whole run;
    each slice exhausts its attempts there, moves to the next route, is decided there with
    the model and completes. Bit-exact, no failed batch, and the live trace (with the
    decisions on the second route's candidate set) replays identically."""
    doc = json.loads(fabrics.two_node(2, 1e9, backend="cuda"))
    for n_ in ("a", "b"):
        doc["rails"].append({"id": f"{n_}.m0", "node": n_, "bandwidth_bytes_per_sec": 5e8,
                             "affinity": "same_socket", "backend": "memory"})
    topo = json.dumps(doc)
    e = make_engine(topo, {"backends": ["cuda", "memory"],
                           "resilience": {"degradation_ratio": 1e9, "max_attempts": 2, "failure_threshold": 1000}})
    e.trace_enable(1 << 16)
    n = 8 << 20
    src, dst = dev_buf(n, 12), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    for r in ("a.r0", "a.r1"):
        e.inject_fault(r, sp.FaultEffect.DOWN, 0, 1 << 62)
    b = e.allocate_batch()
    e.submit_transfer(b, sp.TransferRequest("s", 0, "d", 0, n))
    st = e.await_batch(b, 30_000_000_000)
    assert st.state == sp.BatchState.COMPLETE, st
    assert sp.checksum(DEV, dst.data_ptr(), n) == sp.checksum(DEV, src.data_ptr(), n)
    assert e.counters()["batches_failed"] == 0
    by = {e.rail_id(r): e.rail_stats(r).bytes_ok for r in range(e.rail_count())}
    assert by["a.m0"] == n and by["a.r0"] == 0 and by["a.r1"] == 0
    assert int(e.trace_candidates()[0]) >= 2  # both routes of the plan are candidate sets
    bw, tier, rank = rails_of(topo)
    ev, dec = replay_live(co, e, sched_config(), res_config(degradation_ratio=1e9, max_attempts=2,
                                                             failure_threshold=1000), bw, tier, rank)
    assert (ev["kind"] == 1).sum() == len(dec) > 0
    e.free_batch(b)
    e.stop()


# ------------------------------------------------------------------ copy-engine rails
def test_copy_engine_rail_bit_exact():
    topo = fabrics.kv_offload(DEV, sm_rails=1, ce_rails=1)
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    blk, nb = 1 << 20, 64
    pool = dev_buf(blk * nb, fill_seed=21)
    host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
    e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, f"g{DEV}", [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, f"g{DEV}", [sp.BufferDesc(0, blk * nb, host.data_ptr())]))
    b = e.allocate_batch()
    e.submit_transfers(b, [sp.TransferRequest("hbm", i * blk, "host", i * blk, blk) for i in range(nb)])
    assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
    assert torch.equal(pool.cpu(), host)
    ids = {e.rail_id(r): e.rail_stats(r).bytes_ok for r in range(e.rail_count())}
    assert ids[f"g{DEV}.ce0"] > 0 and ids[f"g{DEV}.pcie0"] > 0
    e.stop()


@pytest.mark.parametrize("layout", ["contiguous", "strided", "scattered"])
def test_copy_engine_runs_coalesced_bit_exact(layout):
    """The CE proxy merges consecutive orders into one copy: contiguous runs into a 1D
    copy, constant-pitch runs into one 2D copy (rows = slices), anything else per order.
    Two CE rails on separate proxy streams take alternate slices (strided), or one rail
    takes a block table (scattered); bytes are exact in every layout."""
    # strided: two CE rails (ce_index 0 and 1: two proxy streams) alternate slices, so each
    # proxy sees a pitch-2 run
    topo = fabrics.kv_offload(DEV, sm_rails=0, ce_rails=2 if layout == "strided" else 1)
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}})
    blk, nb = 256 << 10, 256
    pool = dev_buf(blk * nb, fill_seed=22)
    host = torch.zeros(blk * nb, dtype=torch.uint8, pin_memory=True)
    e.register_segment(sp.SegmentDescriptor("hbm", sp.Medium.DEVICE, f"g{DEV}", [sp.BufferDesc(0, blk * nb, pool.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("host", sp.Medium.HOST, f"g{DEV}", [sp.BufferDesc(0, blk * nb, host.data_ptr())]))
    perm = np.random.default_rng(3).permutation(nb) if layout == "scattered" else np.arange(nb)
    b = e.allocate_batch()
    if layout == "scattered":
        e.submit_transfers(b, [sp.TransferRequest("hbm", i * blk, "host", int(perm[i]) * blk, blk) for i in range(nb)])
    else:  # one 64 MiB intent: 1024 slices of 64 KiB in order
        e.submit_transfer(b, sp.TransferRequest("hbm", 0, "host", 0, blk * nb))
    assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
    got = host.view(nb, blk)[torch.from_numpy(perm)]
    assert torch.equal(pool.cpu().view(nb, blk), got)
    by = {e.rail_id(r): e.rail_stats(r).bytes_ok for r in range(e.rail_count())}
    assert all(v > 0 for v in by.values()), by
    e.stop()


# ------------------------------------------------------------------ plugin boundary
def test_transport_backend_plugin():
    be = sp.CudaBackend(DEV)
    be.start()
    caps = be.capabilities()
    assert caps.id == b"cuda" and caps.cross_node and caps.same_node
    n = 8 << 20
    src, dst = dev_buf(n, 31), dev_buf(n)
    blob = be.attach_segment_metadata(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    assert blob == b"cuda:s"
    be.attach_segment_metadata(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    assert be.attach_segment_metadata(sp.SegmentDescriptor("f", sp.Medium.FILE, "a", [])) is None
    reqs = [sp.SliceWorkRequest(i, 1, "s", i * 65536, "d", i * 65536, 65536, local_rail=i % 2) for i in range(128)]
    r = be.post_slices(reqs)
    assert 0 < r.accepted <= 64 and not r.fatal  # in-flight window: the suffix is backpressure
    done = []
    posted = r.accepted
    import time
    t0 = time.time()
    while len(done) < 128 and time.time() - t0 < 30:
        done += be.poll_completions(32)
        if posted < 128:
            posted += be.post_slices(reqs[posted:]).accepted
    assert sorted(c.slice for c in done) == list(range(128))
    assert all(c.status == 0 and c.bytes == 65536 for c in done)
    assert torch.equal(src[:128 * 65536], dst[:128 * 65536])
    be.latch_fatal()
    assert be.fatal() and be.post_slices(reqs[:1]).fatal
    be.stop()
    be.close()


# ------------------------------------------------------------------ global load board
def test_load_board_steers_and_replays_identically(co):
    """GlobalLoadBoard (scheduler.cpp:63-79, 108-114; engine.cpp:1090-1093): another
    instance's slot reports rail a.r0 heavily loaded, so with diffusion_weight 0.5 this
    engine sprays onto a.r1. The engine publishes its own slot; its live trace (BOARD
    events included) replays identically through the C oracle and the device replay."""
    topo = fabrics.two_node(2, 1e9, backend="cuda")
    e = make_engine(topo, {"resilience": {"degradation_ratio": 1e9}, "scheduler": {"diffusion_weight": 0.5},
                           "b200": {"chunk_bytes": 65536}})
    nslot = 2
    board = torch.zeros(sp.board_bytes(nslot), dtype=torch.uint8, pin_memory=True)
    words = board.view(torch.int64).view(nslot, -1)  # [heartbeat, pad, queued[64]] per slot
    words[1, 0] = (1 << 62)           # the other instance's heartbeat: never stale
    words[1, 2 + 0] = 1 << 34         # ... and its queue on rail a.r0 (index 0)
    e.attach_board(board.data_ptr(), nslot, 0, 1_000_000)
    e.trace_enable(1 << 18)
    n = 64 << 20
    src, dst = dev_buf(n, 41), dev_buf(n)
    e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, n, src.data_ptr())]))
    e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, n, dst.data_ptr())]))
    import time
    for k in range(4):
        b = e.allocate_batch()
        e.submit_transfers(b, [sp.TransferRequest("s", i * (n // 8), "d", i * (n // 8), n // 8) for i in range(8)])
        assert e.await_batch(b, 30_000_000_000).state == sp.BatchState.COMPLETE
        e.free_batch(b)
        time.sleep(0.003)  # the board refreshes every 1 ms
    assert torch.equal(src, dst)
    by = {e.rail_id(r): e.rail_stats(r).bytes_ok for r in range(e.rail_count())}
    assert by["a.r1"] > 0.9 * (by["a.r0"] + by["a.r1"]), by
    assert int(words[0, 0]) != 0  # this engine published its slot
    bw, tier, rank = rails_of(topo)
    ev, _ = replay_live(co, e, sched_config(omega=0.5), res_config(degradation_ratio=1e9), bw, tier, rank)
    from oracle.oracle import EV_BOARD
    boards = ev[ev["kind"] == EV_BOARD]
    assert len(boards) >= 2 and (boards["len"][boards["rail"] == 0] >= (1 << 34)).all()
    e.stop()
