"""NVLink configurations of SURVEY.md §8(d) on one box, one process, all GPUs visible.

  c2        1 GiB GPU0 -> GPU1 sprayed over the direct SM peer-store rail and k copy-engine
            rails (4096 x 256 KiB slices), vs state-blind round-robin striping of the same
            slices over cudaMemcpyAsync streams and vs one cudaMemcpyPeer of the whole GiB.
  elephant  the 8-GPU variant: 8 disjoint 1 GiB flows i -> (i+1) mod N, one engine per GPU.
  c4        broadcast S bytes GPU0 -> every other GPU (naive fan-out through GPU0's engine).
  c5        c2 traffic; the direct SM rail goes DOWN mid-transfer: heal time and bytes
            (alternate: a copy-engine rail, or the relay rails of --relay-via).
  congest   c2 over several rails with one DEGRADEd (injected congestion): telemetry vs
            round-robin policy.
  --relay-via K [..]  add 2-hop relay rails through GPU K (tier 2, or --relay-affinity direct)

Prints one JSON object per mode. Delivered bytes are checked with the device checksum.
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00368_b200 as sp  # noqa: E402
from paper_2604_00368_b200 import fabrics  # noqa: E402

GiB = 1 << 30


def buf(dev, n, seed=None):
    t = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev}")
    if seed is not None:
        sp.fill_splitmix(dev, t.data_ptr(), n, seed)
    else:
        t.zero_()
    return t


CE_GBS = 770.0  # declared bandwidth of copy-engine rails (--ce-gbs)


RELAY = {"via": [], "affinity": "same_socket"}  # --relay-via / --relay-affinity


def engine(dev, gpus, sm_rails, ce_rails, extra_cfg=None):
    cfg = {"resilience": {"degradation_ratio": 1e9}}
    if RELAY.get("chunk"):
        cfg["b200"] = {"chunk_bytes": RELAY["chunk"]}
    if RELAY.get("max_slices"):
        cfg["scheduler"] = {"max_slices_per_transfer": RELAY["max_slices"]}
    cfg.update(extra_cfg or {})
    if os.environ.get("NV_B200"):  # extra engine knobs, e.g. NV_B200='{"copy": "ldg"}'
        cfg["b200"] = {**cfg.get("b200", {}), **json.loads(os.environ["NV_B200"])}
    e = sp.Engine(fabrics.peer_fabric(gpus, sm_rails=sm_rails, ce_rails=ce_rails, bw_ce=CE_GBS * 1e9,
                                      relay_via=RELAY["via"], relay_affinity=RELAY["affinity"]),
                  json.dumps(cfg), dev)
    e.start()
    return e


def reg(e, sid, dev, t):
    e.register_segment(sp.SegmentDescriptor(sid, sp.Medium.DEVICE, f"g{dev}", [sp.BufferDesc(0, t.numel(), t.data_ptr())]))


def timed_prepared(e, reqs, reps):
    p = e.prepare_transfers(reqs)
    ms = []
    for i in range(reps + 2):
        b = e.allocate_batch()
        t = p.run(b)
        st = e.batch_status(b)
        assert st.state == sp.BatchState.COMPLETE, st
        e.free_batch(b)
        if i >= 2:
            ms.append(t)
    return min(ms), sum(ms) / len(ms)


def c2(args):
    n = args.size
    src, dst = buf(0, n, 77), buf(1, n)
    out = {"mode": "c2", "bytes": n, "slices": 4096, "sm_rails": args.sm_rails, "ce_rails": args.ce_rails,
           "pull": bool(args.pull)}
    # --pull: the engine (and so the copying SMs) sits on the destination GPU, which loads
    # from peer HBM and stores locally
    e = engine(1 if args.pull else 0, [0, 1], args.sm_rails, args.ce_rails)
    reg(e, "src", 0, src)
    reg(e, "dst", 1, dst)
    req = [sp.TransferRequest("src", 0, "dst", 0, n)]
    best, mean = timed_prepared(e, req, args.reps)
    out["engine_gbs"] = round(n / (best * 1e-3) / 1e9, 2)
    out["engine_gbs_mean"] = round(n / (mean * 1e-3) / 1e9, 2)
    if args.prof:  # scheduler-warp cycle counters of the last launch (tools/gpu_perf.py names)
        import ctypes as C
        from paper_2604_00368_b200 import _lib as L
        w = (C.c_uint64 * 48)()
        L.lib.spray_engine_debug(e._h, w, 48)
        names = ["host_tail", "sub_tail", "sub_head", "state", "now", "disp", "term", "failed", "retried", "trace_n",
                 "stream", "loops", "serial", "obs", "fb", "n_comp", "n_dec", "apply", "decide", "ctl", "ingress",
                 "complete", "egress", "egress_blocks", "ingress_blocks", "entries", "pub_busy", "rx_busy",
                 "n_fences", "p1", "p2", "p3"]
        d = dict(zip(names, list(w)))
        out["prof_ms"] = {k: round(d[k] / 1.965e6, 3) for k in ("serial", "obs", "fb", "p1", "p2", "p3", "apply",
                                                               "decide", "ctl", "ingress", "complete", "egress",
                                                               "pub_busy")}
        out["prof_counts"] = {k: d[k] for k in ("loops", "entries", "n_comp", "n_dec", "n_fences")}
        tl = list(w)[37:44]  # launch timeline (engine ns), relative to the scheduler's start
        out["timeline_us"] = dict(zip(["first_stamp", "first_decide", "last_decide", "first_apply", "last_apply",
                                       "exit"], [round((x - tl[0]) / 1e3, 1) if x else None for x in tl[1:]]))
    assert sp.checksum(1, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
    # e2e through the public API
    t0 = time.perf_counter()
    for _ in range(args.reps):
        b = e.allocate_batch()
        e.submit_transfer(b, req[0])
        assert e.await_batch(b).state == sp.BatchState.COMPLETE
        e.free_batch(b)
    out["e2e_gbs"] = round(args.reps * n / (time.perf_counter() - t0) / 1e9, 2)
    stats = [e.rail_stats(r) for r in range(e.rail_count())]
    out["bytes_by_rail"] = {s.rail_id: s.bytes_ok for s in stats if s.bytes_ok}
    e.stop()
    dst.zero_()
    # state-blind round-robin striping of the same 4096 slices (cudaMemcpyAsync, peer)
    sl = n // 4096
    srcs = [src.data_ptr() + i * sl for i in range(4096)]
    dsts = [dst.data_ptr() + i * sl for i in range(4096)]
    sp.rr_copy(0, srcs, dsts, [sl] * 4096, 4)
    rr = min(sp.rr_copy(0, srcs, dsts, [sl] * 4096, 4) for _ in range(args.reps))
    out["rr_striping_gbs"] = round(n / (rr * 1e-3) / 1e9, 2)
    assert sp.checksum(1, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
    # one copy-engine peer copy of the whole buffer
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.device(0):
        dst.copy_(src)
        times = []
        for _ in range(args.reps):
            evs[0].record()
            dst.copy_(src)
            evs[1].record()
            evs[1].synchronize()
            times.append(evs[0].elapsed_time(evs[1]))
    out["memcpy_peer_gbs"] = round(n / (min(times) * 1e-3) / 1e9, 2)
    # raw SM peer stores without any scheduling: the plugin backend's group copy kernel
    # (one launch, 64 x 16 MiB slices, 128 KiB chunks over 4 CTAs per SM)
    be = sp.CudaBackend(0)
    be.start()
    be.attach_segment_metadata(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "g0", [sp.BufferDesc(0, n, src.data_ptr())]))
    be.attach_segment_metadata(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "g1", [sp.BufferDesc(0, n, dst.data_ptr())]))
    k = 64
    reqs = [sp.SliceWorkRequest(i, 1, "s", i * (n // k), "d", i * (n // k), n // k) for i in range(k)]
    best_raw = 1e9
    for _ in range(args.reps + 1):
        torch.cuda.synchronize(0)
        t0 = time.perf_counter()
        assert be.post_slices(reqs).accepted == k
        got = 0
        while got < k:
            got += len(be.poll_completions(k))
        best_raw = min(best_raw, time.perf_counter() - t0)
    be.stop()
    out["raw_sm_peer_gbs"] = round(n / best_raw / 1e9, 2)
    return out


def elephant(args):
    g = torch.cuda.device_count()
    n = args.size
    srcs = [buf(i, n, 100 + i) for i in range(g)]
    dsts = [buf(i, n) for i in range(g)]
    engines, preps = [], []
    for i in range(g):
        j = (i + 1) % g
        e = engine(i, list(range(g)), args.sm_rails, args.ce_rails)
        reg(e, f"src{i}", i, srcs[i])
        reg(e, f"dst{j}", j, dsts[j])
        engines.append(e)
        preps.append(e.prepare_transfers([sp.TransferRequest(f"src{i}", 0, f"dst{j}", 0, n)]))
    # concurrent: launch every engine's prepared batch, then wait for all
    for rep in range(2):
        t0 = time.perf_counter()
        batches = [e.allocate_batch() for e in engines]
        import threading
        res = [None] * g

        def run(k):
            res[k] = preps[k].run(batches[k])
        th = [threading.Thread(target=run, args=(k,)) for k in range(g)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.perf_counter() - t0
        for e, b in zip(engines, batches):
            assert e.batch_status(b).state == sp.BatchState.COMPLETE
            e.free_batch(b)
    for i in range(g):
        j = (i + 1) % g
        assert sp.checksum(j, dsts[j].data_ptr(), n) == sp.checksum(i, srcs[i].data_ptr(), n)
    for e in engines:
        e.stop()
    return {"mode": "elephant", "gpus": g, "bytes_per_flow": n, "per_flow_kernel_ms": [round(x, 3) for x in res],
            "aggregate_gbs_by_slowest": round(g * n / (max(res) * 1e-3) / 1e9, 2),
            "aggregate_gbs_wall": round(g * n / wall / 1e9, 2)}


def c4(args):
    g = torch.cuda.device_count()
    n = args.size
    src = buf(0, n, 5)
    dsts = {j: buf(j, n) for j in range(1, g)}
    e = engine(0, list(range(g)), args.sm_rails, args.ce_rails)
    reg(e, "w", 0, src)
    for j, t in dsts.items():
        reg(e, f"w{j}", j, t)
    reqs = [sp.TransferRequest("w", 0, f"w{j}", 0, n) for j in dsts]
    best, mean = timed_prepared(e, reqs, args.reps)
    for j, t in dsts.items():
        assert sp.checksum(j, t.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
    e.stop()
    return {"mode": "c4-fanout", "gpus": g, "bytes": n, "delivered": (g - 1) * n,
            "ms": round(best, 3), "delivered_gbs": round((g - 1) * n / (best * 1e-3) / 1e9, 2)}


def c4chain(args):
    """Pipelined relay chain GPU0 -> GPU1 -> ... -> GPU(g-1): engine k forwards granule i of
    its copy as soon as it has arrived (dataflow gates), so every receiver's ingress is
    busy at once instead of GPU0's egress carrying g-1 copies."""
    import threading
    g = torch.cuda.device_count()
    n = args.size
    ws = [buf(0, n, 5)] + [buf(j, n) for j in range(1, g)]
    engines, preps = [], []
    flags = {}
    for k in range(g - 1):
        e = engine(k, list(range(g)), args.sm_rails, 0)
        cb = e.chunk_bytes()
        reg(e, f"w{k}", k, ws[k])
        reg(e, f"w{k + 1}", k + 1, ws[k + 1])
        if k + 1 not in flags:
            flags[k + 1] = torch.zeros((n + cb - 1) // cb, dtype=torch.int32, device=f"cuda:{k + 1}")
        e.gate_segment(f"w{k + 1}", sp.Engine.GATE_PRODUCE, flags[k + 1].data_ptr())
        if k > 0:
            e.gate_segment(f"w{k}", sp.Engine.GATE_CONSUME, flags[k].data_ptr())
        engines.append(e)
        preps.append(e.prepare_transfers([sp.TransferRequest(f"w{k}", 0, f"w{k + 1}", 0, n)]))
    walls, kms = [], []
    for rep in range(args.reps + 1):
        for t in ws[1:]:
            t.zero_()
        for d in range(g):
            torch.cuda.synchronize(d)
        batches = [e.allocate_batch() for e in engines]
        res = [None] * len(engines)

        def run(k):
            res[k] = preps[k].run(batches[k])
        th = [threading.Thread(target=run, args=(k,)) for k in range(len(engines))]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.perf_counter() - t0
        for e, b in zip(engines, batches):
            assert e.batch_status(b).state == sp.BatchState.COMPLETE
            e.free_batch(b)
        if rep:
            walls.append(wall)
            kms.append(max(res))
    ref = sp.checksum(0, ws[0].data_ptr(), n)
    for j in range(1, g):
        assert sp.checksum(j, ws[j].data_ptr(), n) == ref, j
    for e in engines:
        e.stop()
    best = min(kms)
    return {"mode": "c4-chain", "gpus": g, "bytes": n, "delivered": (g - 1) * n, "slowest_engine_ms": round(best, 3),
            "wall_ms": round(min(walls) * 1e3, 3),
            "delivered_gbs": round((g - 1) * n / (best * 1e-3) / 1e9, 2),
            "per_receiver_gbs": round(n / (best * 1e-3) / 1e9, 2)}


def c5(args):
    n = args.size
    src, dst = buf(0, n, 91), buf(1, n)
    e = engine(0, [0, 1], 1, 0 if RELAY["via"] else max(1, args.ce_rails))
    reg(e, "src", 0, src)
    reg(e, "dst", 1, dst)
    b = e.allocate_batch()
    e.submit_transfer(b, sp.TransferRequest("src", 0, "dst", 0, n))
    time.sleep(args.fault_after_ms * 1e-3)
    now = e.now_ns()
    e.inject_fault("g0.nvl0", sp.FaultEffect.DOWN, now, now + 10**12, 0.0)
    st = e.await_batch(b, 60_000_000_000)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    same = sp.checksum(1, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
    ok = st.state == sp.BatchState.COMPLETE and same
    if not same:
        d, s_ = dst.view(-1, 1 << 18).cpu(), src.view(-1, 1 << 18).cpu()
        bad = [i for i in range(d.shape[0]) if not torch.equal(d[i], s_[i])]
        detail = []
        # which source 4 KiB page does each bad destination page hold?
        sp_pages = src.view(-1, 4096).cpu()
        keys = {}
        h = sp_pages[:, :16].contiguous().view(-1, 16).numpy()
        for pi in range(h.shape[0]):
            keys[h[pi].tobytes()] = pi
        for i in bad[:4]:
            dpg = d[i].view(-1, 4096)[:, :16].contiguous().numpy()
            detail.append({"slice": i, "holds_src_pages": [keys.get(dpg[q].tobytes(), -1) for q in (0, 1, 31, 32, 63)],
                           "expected_first_page": i * 64})
        # the first bad page: where does each of its 16-byte words come from?
        i0 = bad[0]
        eqp = (d[i0] == s_[i0]).view(-1, 4096).all(dim=1)
        pg = int((~eqp).nonzero()[0])
        words = d[i0].view(-1, 4096)[pg].view(-1, 16).numpy()
        exp_words = s_[i0].view(-1, 4096)[pg].view(-1, 16).numpy()
        srcw = src.cpu().view(-1, 16).numpy()
        idx = {srcw[w].tobytes(): w for w in range(0, srcw.shape[0])}
        base_w = (i0 * (1 << 18) + pg * 4096) // 16
        where = [idx.get(words[w].tobytes(), -1) - base_w if idx.get(words[w].tobytes(), -1) >= 0 else None
                 for w in range(words.shape[0])]
        detail.append({"page": pg, "word_ok": [bool((words[w] == exp_words[w]).all()) for w in range(0, 256, 8)],
                       "word_src_delta": where[:48]})
        for i in bad[:4]:
            eq = (d[i] == s_[i]).view(-1, 4096).all(dim=1)  # per 4 KiB page
            zero = (d[i] == 0).view(-1, 4096).all(dim=1)
            detail.append({"slice": i, "pages_ok": int(eq.sum()), "pages_zero": int(zero.sum()),
                           "first_bad_page": int((~eq).nonzero()[0]) if (~eq).any() else -1})
        print(json.dumps({"state": st.state.name, "remaining": st.remaining, "bad_slices": len(bad), "first": bad[:8],
                          "detail": detail}), flush=True)
    heal = e.heal_stats()
    stats = {s.rail_id: (s.bytes_ok, s.bytes_failed, s.health.name) for s in (e.rail_stats(r) for r in range(e.rail_count()))}
    e.stop()
    return {"mode": "c5", "bytes": n, "complete_and_bit_exact": bool(ok), "heal": heal, "rails": stats}


def congest(args):
    """Injected congestion on C2: the flow sprays over the direct SM rail(s) and any
    --relay-via rails (tier 1); rail --congest-rail is DEGRADEd to --factor of its
    bandwidth for the whole run (sim_backend.cpp:83-93 semantics on the real fabric).
    Telemetry spraying vs the state-blind round-robin policy (a25), same rails."""
    n = args.size
    src, dst = buf(0, n, 61), buf(1, n)
    out = {"mode": "congest", "bytes": n, "congested": args.congest_rail, "factor": args.factor}
    for pol in ("telemetry", "rr"):
        e = engine(0, [0, 1], args.sm_rails, args.ce_rails, {"scheduler": {"policy": pol}})
        reg(e, "src", 0, src)
        reg(e, "dst", 1, dst)
        now = e.now_ns()
        e.inject_fault(args.congest_rail, sp.FaultEffect.DEGRADE, now, now + 10 ** 13, args.factor)
        best, mean = timed_prepared(e, [sp.TransferRequest("src", 0, "dst", 0, n)], args.reps)
        assert sp.checksum(1, dst.data_ptr(), n) == sp.checksum(0, src.data_ptr(), n)
        stats = [e.rail_stats(r) for r in range(e.rail_count())]
        tot = sum(x.bytes_ok for x in stats) or 1
        out[pol] = {"gbs": round(n / (mean * 1e-3) / 1e9, 2),
                    "share": {x.rail_id: round(x.bytes_ok / tot, 3) for x in stats if x.bytes_ok}}
        e.stop()
        dst.zero_()
    out["telemetry_over_rr"] = round(out["telemetry"]["gbs"] / out["rr"]["gbs"], 3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["c2", "elephant", "c4", "c4chain", "c5", "congest"])
    ap.add_argument("--size", type=int, default=GiB)
    ap.add_argument("--sm-rails", type=int, default=1)
    ap.add_argument("--ce-rails", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--fault-after-ms", type=float, default=0.3)
    ap.add_argument("--prof", action="store_true", help="c2: print scheduler-warp cycle counters")
    ap.add_argument("--ce-gbs", type=float, default=770.0, help="declared bandwidth of each copy-engine rail")
    ap.add_argument("--relay-via", type=int, nargs="*", default=[], help="2-hop relay rails through these GPUs")
    ap.add_argument("--relay-affinity", default="same_socket", help="relay rail tier (direct = tier 1)")
    ap.add_argument("--chunk-kib", type=int, default=0, help="b200.chunk_bytes (SM work granule), KiB")
    ap.add_argument("--congest-rail", default="g0.nvl0", help="congest: the DEGRADEd rail")
    ap.add_argument("--max-slices", type=int, default=0, help="scheduler.max_slices_per_transfer (diagnostic)")
    ap.add_argument("--pull", action="store_true", help="c2: run the engine on the destination GPU (peer loads)")
    ap.add_argument("--factor", type=float, default=0.25, help="congest: bandwidth factor of the DEGRADEd rail")
    args = ap.parse_args()
    RELAY["via"], RELAY["affinity"] = args.relay_via, args.relay_affinity
    RELAY["chunk"] = args.chunk_kib << 10 if args.chunk_kib else 0
    RELAY["max_slices"] = args.max_slices
    global CE_GBS
    CE_GBS = args.ce_gbs
    out = {"c2": c2, "elephant": elephant, "c4": c4, "c4chain": c4chain, "c5": c5, "congest": congest}[args.mode](args)
    print(json.dumps(out), flush=True)
    os._exit(0)


if __name__ == "__main__":
    main()
