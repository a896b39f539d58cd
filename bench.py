#!/usr/bin/env python
"""bench.py — the B200 slice-spraying data plane on its headline single-GPU workload.

Workload (BASELINE.json configs[2], the largest single-GPU configuration): a HiCache-style
KV batch per GPU — 4096 x 64 KiB offloads (HBM -> pinned host) plus 4096 x 64 KiB reloads
(pinned host -> HBM), both through seeded random block tables, as ONE batch of 8192
transfer intents. A "step" is one such batch (512 MiB delivered). At N GPUs every rank
runs its own batch over its own PCIe root (weak scaling, no data-path collective).

  value    device-resident intents (prepared once in HBM), engine kernel launched in
           drain mode and timed with CUDA events on its stream: GB/s delivered.
  e2e      the public C-ABI path from host arrays: submit_transfers (8192 intents; the
           engine stages them to HBM as bulk arrays, 1024 per copy-engine copy, inside the
           timed region) + await_batch, wall clock.
  roofline the engine kernel against PCIe Gen5 x16 full duplex.
  cpu_baseline  the reference's own CPU engine (oracle/_ref, unmodified reference sources)
           on this host: memory backend, real clock, same block batch, one direction.

`--impl reference` times that reference CPU path alone with all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PCIE_NOMINAL_GBS = 64.0  # per direction, PCIe Gen5 x16


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--blocks", type=int, default=4096)
    p.add_argument("--block-kib", type=int, default=64)
    p.add_argument("--group", type=int, default=32, help="offload/reload intents alternate in runs of this size")
    p.add_argument("--sm-rails", type=int, default=1, help="SM copy rails on the GPU's PCIe root (KV batch)")
    p.add_argument("--ce-rails", type=int, default=0, help="copy-engine rails sprayed beside the SM rail")
    p.add_argument("--ce-gbs", type=float, default=15.0, help="declared bandwidth of each copy-engine rail")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--lat-batches", type=int, default=200, help="small batches timed for the batch-latency percentiles")
    p.add_argument("--lat-intents", type=int, default=64, help="intents per latency batch (half offload, half reload)")
    p.add_argument("--no-congestion", action="store_true")
    p.add_argument("--no-small", action="store_true", help="skip the small-slice HBM->HBM sub-line")
    p.add_argument("--no-nvlink", action="store_true", help="N>1: skip the NVLink phase (elephant, broadcast chain, fault)")
    p.add_argument("--nvl-bytes", type=int, default=1 << 30, help="N>1: bytes per elephant flow (C2 shape)")
    p.add_argument("--bcast-bytes", type=int, default=16 << 30, help="N>1: broadcast size (C4 shape)")
    p.add_argument("--nvl-mode", default="push", choices=["pull", "push"],
                   help="N>1: which end's engine moves elephant flows and chain hops")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


# ------------------------------------------------------------------ reference CPU path
def reference_kv(blocks, block, seconds_budget, threads):
    """The reference Engine (oracle/_ref: unmodified /root/reference sources) moving the
    KV batch host->host with `threads` rails/workers. Returns (GB/s, iters, cores, kind)."""
    from oracle.oracle import RefOracle, ref_available
    if not ref_available():
        return None
    ref = RefOracle()
    t, ok = ref.cpu_kv_batch(threads, threads, block, blocks, 1234, 1)  # one sample to size the run
    iters = max(1, min(50, int(seconds_budget / max(t, 1e-3))))
    best, ok2 = ref.cpu_kv_batch(threads, threads, block, blocks, 1234, iters)
    if not (ok and ok2):
        raise RuntimeError("reference CPU path delivered wrong bytes")
    return blocks * block / best / 1e9, iters, threads


def best_reference_threads(ref, block, blocks):
    """The reference engine serialises every worker on one mutex (engine.hpp:263), so more
    threads can be slower: give it the best rails/workers count this host offers, chosen
    by a short calibration on a quarter batch."""
    best, best_t = 1, None
    t = 1
    while t <= min(os.cpu_count() or 1, 16):
        dt, ok = ref.cpu_kv_batch(t, t, block, max(64, blocks // 4), 99, 1)
        if ok and (best_t is None or dt < best_t):
            best, best_t = t, dt
        t *= 2
    return best


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    block = args.block_kib << 10
    from oracle.oracle import RefOracle, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libspray_ref.so not built"}))
        return
    ref = RefOracle()
    threads = best_reference_threads(ref, block, args.blocks)
    for _ in range(args.warmup):
        ref.cpu_kv_batch(threads, threads, block, args.blocks, 1234, 1)
    times = []
    for _ in range(args.steps):
        t, ok = ref.cpu_kv_batch(threads, threads, block, args.blocks, 1234, 1)
        if not ok:
            raise RuntimeError("reference delivered wrong bytes")
        times.append(t)
    total = sum(times)
    gbs = args.steps * args.blocks * block / total / 1e9
    line = {
        "impl": "reference", "metric": "sprayed transfer GB/s (KV batch, HBM<->pinned host)", "value": round(gbs, 3),
        "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"kv_batch {args.blocks}x{args.block_kib}KiB, reference CPU engine "
                               f"(memory backend, real clock, {threads} rails/workers: the best of 1..nproc), "
                               "host->host"},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "nproc": os.cpu_count(),
                         "kind": "reference",
                         "sample": f"{args.steps} batches of {args.blocks}x{args.block_kib} KiB"},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = f"/tmp/spray_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=open(self.path + ".err", "w"))
            # the timed region starts only once the sampler is producing rows
            t0 = time.time()
            while time.time() - t0 < 5.0 and self.proc.poll() is None:
                if os.path.exists(self.path) and os.path.getsize(self.path) > 0:
                    break
                time.sleep(0.02)
            self.mark = os.path.getsize(self.path) if os.path.exists(self.path) else 0
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        try:
            text = open(self.path).read()
            rows = [r.split(",") for r in text[getattr(self, "mark", 0):].strip().splitlines() if r.strip()]
            if not rows:  # the region was shorter than one sampling period: keep the last pre-region row
                rows = [r.split(",") for r in text.strip().splitlines()[-1:] if r.strip()]
        except Exception:
            return None
        if not rows:
            err = open(self.path + ".err").read().strip() if os.path.exists(self.path + ".err") else ""
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "error": err[:200]}
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 3 + i and r[3 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}



# ------------------------------------------------------------------ batch latency
def pct(xs, q):
    """exact_percentile (bench.cpp): the value at rank ceil(q*n) of the sorted sample."""
    ys = sorted(xs)
    if not ys:
        return None
    k = max(0, min(len(ys) - 1, int(-(-q * len(ys) // 1)) - 1))
    return ys[k]


def batch_latency(sp, eng, reqs, n_batches, per_batch):
    """P50/P90/P99 batch latency (bench.cpp:156-157, 213-215: submit -> batch terminal) of
    small KV batches (per_batch intents, offloads and reloads interleaved) through the
    public API, one batch in flight, as a HiCache prefetch/offload request sees it."""
    groups = [sp.Requests(reqs[i:i + per_batch]) for i in range(0, len(reqs) - per_batch + 1, per_batch)]
    lat = []
    for k in range(n_batches + 10):
        g = groups[k % len(groups)]
        t0 = time.perf_counter()
        b = eng.allocate_batch()
        eng.submit_transfers(b, g)
        st = eng.await_batch(b)
        if st.state != sp.BatchState.COMPLETE:
            raise RuntimeError(f"latency batch not complete: {st}")
        eng.free_batch(b)
        if k >= 10:
            lat.append((time.perf_counter() - t0) * 1e6)
    return {"intents_per_batch": per_batch, "bytes_per_batch": sum(r.length for r in reqs[:per_batch]),
            "batches": len(lat), "p50_us": round(pct(lat, 0.5), 1), "p90_us": round(pct(lat, 0.9), 1),
            "p99_us": round(pct(lat, 0.99), 1), "mean_us": round(sum(lat) / len(lat), 1)}


def batch_latency_c(sp, eng, reqs, per_batch, n_batches=1000):
    """The same percentiles with the rounds timed in C++ (spray_batch_latency: allocate /
    submit_transfers / await / free through the C-ABI, as a C++ application calls them)."""
    eng.batch_latency_ns(reqs, per_batch, 50)  # warm
    us = [x / 1e3 for x in eng.batch_latency_ns(reqs, per_batch, n_batches).tolist()]
    return {"intents_per_batch": per_batch, "bytes_per_batch": sum(r.length for r in reqs[:per_batch]),
            "batches": len(us), "p50_us": round(pct(us, 0.5), 2), "p90_us": round(pct(us, 0.9), 2),
            "p99_us": round(pct(us, 0.99), 2), "mean_us": round(sum(us) / len(us), 2)}


def small_slices(sp, fabrics, dev, hbm, hbm2, nb, blk, perm, hbm_peak_gbs, reps=4):
    """The scheduler-bound regime: nb x blk HBM -> HBM through a random block table (one
    slice per intent), 1 and 2 rails, prepared intents, drain-mode launch timed by CUDA
    events. Roofline: the HBM copy roofline (delivered bytes = half the HBM traffic)."""
    out = {"workload": f"{nb} x {blk >> 10} KiB HBM->HBM, random block table, one slice per intent",
           "roofline_gbs": round(hbm_peak_gbs / 2, 1),
           "roofline_source": "MEASURED_PEAKS.json hbm_gbs / 2 (a copy reads and writes each byte)"}
    for rails in (1, 2):
        cfg = {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536}}
        e = sp.Engine(fabrics.two_node(rails, 1.6e12 / rails, backend="cuda"), json.dumps(cfg), dev)
        e.start()
        e.register_segment(sp.SegmentDescriptor("s", sp.Medium.DEVICE, "a", [sp.BufferDesc(0, nb * blk, hbm.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("d", sp.Medium.DEVICE, "b", [sp.BufferDesc(0, nb * blk, hbm2.data_ptr())]))
        prep = e.prepare_transfers([sp.TransferRequest("s", i * blk, "d", int(perm[i]) * blk, blk) for i in range(nb)])
        ms = []
        for k in range(reps + 2):
            b = e.allocate_batch()
            t = prep.run(b)
            if e.batch_status(b).state != sp.BatchState.COMPLETE:
                raise RuntimeError("small-slice batch not complete")
            e.free_batch(b)
            if k >= 2:
                ms.append(t)
        best = min(ms)
        gbs = nb * blk / (statistics.mean(ms) * 1e-3) / 1e9
        out[f"rails_{rails}"] = {"gbs": round(gbs, 2), "best_gbs": round(nb * blk / (best * 1e-3) / 1e9, 2),
                                 "slices_per_s_M": round(nb / (statistics.mean(ms) * 1e-3) / 1e6, 3),
                                 "frac": round(gbs / (hbm_peak_gbs / 2), 4)}
        prep.free()
        e.stop()
    return out


# ------------------------------------------------------------------ injected congestion
def congestion(sp, fabrics, dev, hbm, host, nb, blk, perm, reps=4):
    """Telemetry spraying vs state-blind round robin (Policy::kRoundRobin, a25) on the same
    two SM rails of this GPU's PCIe root when one rail is congested: a DEGRADE fault
    (sim_backend.cpp:83-93 semantics on the real fabric: FIFO service at factor x B)
    throttles g.pcie1 to 10% for the whole run. Workload: the offload half of the KV batch.
    The cost model only (degradation exclusion off), so the difference is the scheduler's."""
    out = {"kind": "software throttle: a DEGRADE fault (FIFO service at 10% of B on g.pcie1) inside the "
                   "engine's own copy workers, not real contention (see congestion_real at N > 1)",
           "workload": f"{nb} x {blk >> 10} KiB offload HBM->pinned host per batch",
           "fabric": "2 SM rails on one PCIe root, g.pcie1 DEGRADE factor 0.1",
           "exclusion": "off (degradation_ratio 1e9): cost-model steering only"}
    for pol in ("telemetry", "round_robin"):
        cfg = {"resilience": {"degradation_ratio": 1e9}, "scheduler": {"policy": pol},
               "b200": {"chunk_bytes": 65536}}
        e = sp.Engine(fabrics.kv_offload(dev, sm_rails=2), json.dumps(cfg), dev)
        e.start()
        node = f"g{dev}"
        e.register_segment(sp.SegmentDescriptor("c/hbm", sp.Medium.DEVICE, node, [sp.BufferDesc(0, nb * blk, hbm.data_ptr())]))
        e.register_segment(sp.SegmentDescriptor("c/host", sp.Medium.HOST, node, [sp.BufferDesc(0, nb * blk, host.data_ptr())]))
        now = e.now_ns()
        e.inject_fault(f"g{dev}.pcie1", sp.FaultEffect.DEGRADE, now, now + 10 ** 13, 0.1)
        prep = e.prepare_transfers([sp.TransferRequest("c/hbm", i * blk, "c/host", int(perm[i]) * blk, blk)
                                    for i in range(nb)])
        ms = []
        for k in range(reps + 2):
            b = e.allocate_batch()
            t = prep.run(b)
            if e.batch_status(b).state != sp.BatchState.COMPLETE:
                raise RuntimeError("congestion batch not complete")
            e.free_batch(b)
            if k >= 2:
                ms.append(t)
        share = {s.rail_id: s.bytes_ok for s in (e.rail_stats(r) for r in range(e.rail_count())) if s.bytes_ok}
        tot = sum(share.values()) or 1
        out[pol] = {"gbs": round(nb * blk / (statistics.mean(ms) * 1e-3) / 1e9, 3),
                    "ms_per_batch": round(statistics.mean(ms), 3),
                    "bytes_share": {k: round(v / tot, 4) for k, v in share.items()}}
        prep.free()
        e.stop()
    out["telemetry_over_rr"] = round(out["telemetry"]["gbs"] / out["round_robin"]["gbs"], 3)
    return out


# ------------------------------------------------------------------ NVLink phase (N > 1)
def nvlink_phase(sp, fabrics, args, rank, world, dev):
    """The NVLink configurations at N GPUs, one process per GPU, peer HBM shared through CUDA
    IPC handles (exchanged over torch.distributed: handles, barriers and max-over-ranks
    timing only; no data-path collective). Every time is the engine kernel's CUDA-event
    time on its own stream, max over ranks.
      elephant  C2 x N: N disjoint flows rank r -> r+1 (mod N), nvl_bytes each, 4096 slices
      bcast     C4: bcast_bytes from rank 0 to every other rank as a pipelined chain
                0 -> 1 -> ... -> N-1 (dataflow gates), vs rank 0 fanning out alone
      fault     C5: rank 0's flow loses its direct SM rail mid-transfer (DOWN) while every
                other flow keeps running (background load); alternate = copy-engine rail
    Delivered bytes are checked by device checksums against the senders'."""
    import torch
    import torch.distributed as dist
    GBs = lambda b, ms: round(b / (ms * 1e-3) / 1e9, 2)  # noqa: E731
    out = {"ranks": world}
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    opened = {}

    def gather(obj):
        objs = [None] * world
        dist.all_gather_object(objs, obj)
        return objs

    def maxr(x):
        t = torch.tensor([float(x)], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allok(x):
        t = torch.tensor([0.0 if x else 1.0], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item()) == 0.0

    def open_peer(h):  # one mapping per exported allocation
        if h not in opened:
            opened[h] = sp.ipc_open(dev, h)
        return opened[h]

    def seg(e, sid, g, n, ptr):
        e.register_segment(sp.SegmentDescriptor(sid, sp.Medium.DEVICE, f"g{g}", [sp.BufferDesc(0, n, ptr)]))

    # ---- elephant flows. push (default): the sender's engine moves each flow (peer
    # stores); pull: the receiver's (peer loads, storing locally). A lone flow pulls faster
    # (peer loads reach the copy-engine ceiling, ~786 GB/s, where peer stores stop at ~709:
    # tools/peer_pull.cu), but in the ring, where every GPU sends and receives at once,
    # push measured 636 GB/s per flow against 572 for pull (4 x B200).
    pull = args.nvl_mode == "pull"
    n = args.nvl_bytes
    src = torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev}")
    sp.fill_splitmix(dev, src.data_ptr(), n, 500 + rank)
    dst = torch.zeros(n, dtype=torch.uint8, device=f"cuda:{dev}")
    hs = gather((sp.ipc_export(dev, src.data_ptr()), sp.ipc_export(dev, dst.data_ptr())))
    pdst = open_peer(hs[nxt][1])
    cfg = json.dumps({"resilience": {"degradation_ratio": 1e9}})
    ecfg = json.dumps({"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536 if pull else 32768}})
    if pull:
        e = sp.Engine(fabrics.peer_fabric(sorted({prv, rank})), ecfg, dev)
        e.start()
        seg(e, f"src{prv}", prv, n, open_peer(hs[prv][0]))
        seg(e, f"dst{rank}", rank, n, dst.data_ptr())
        flow = sp.TransferRequest(f"src{prv}", 0, f"dst{rank}", 0, n)
    else:
        e = sp.Engine(fabrics.peer_fabric(sorted({rank, nxt})), ecfg, dev)
        e.start()
        seg(e, f"src{rank}", rank, n, src.data_ptr())
        seg(e, f"dst{nxt}", nxt, n, pdst)
        flow = sp.TransferRequest(f"src{rank}", 0, f"dst{nxt}", 0, n)
    prep = e.prepare_transfers([flow])
    times = []
    for k in range(args.warmup + max(3, args.steps)):
        torch.cuda.synchronize(dev)
        dist.barrier()
        b = e.allocate_batch()
        ms = prep.run(b)
        ok = e.batch_status(b).state == sp.BatchState.COMPLETE
        e.free_batch(b)
        ms = maxr(ms if ok else 1e9)
        if k >= args.warmup:
            times.append(ms)
    torch.cuda.synchronize(dev)
    dist.barrier()
    sums = gather(sp.checksum(dev, src.data_ptr(), n))
    exact = allok(sp.checksum(dev, dst.data_ptr(), n) == sums[prv])
    mean = statistics.mean(times)
    out["elephant"] = {"flows": f"{world} x (r -> r+1 mod {world})", "bytes_per_flow": n, "slices_per_flow": 4096,
                       "rails": ("1 SM rail per GPU, driven by the receiver (peer loads), 64 KiB granules" if pull
                                 else "1 SM rail per GPU, driven by the sender (peer stores), 32 KiB granules"),
                       "ms_max_over_ranks": round(mean, 4),
                       "aggregate_gbs": GBs(world * n, mean), "per_flow_gbs": GBs(n, mean),
                       "best_aggregate_gbs": GBs(world * n, min(times)),
                       "roofline": {"peak_gbs": 900.0 * world, "unit": "GB/s",
                                    "frac": round(world * n / (mean * 1e-3) / 1e9 / (900.0 * world), 4),
                                    "peak_source": "nominal NVLink 5, 900 GB/s per direction per GPU",
                                    "measured_ceiling_gbs_per_flow": {"sm_peer_loads": 786, "copy_engine": 782,
                                                                      "sm_peer_stores": 709}},
                       "bit_exact": exact}
    prep.free()
    e.stop()

    # ---- broadcast: pipelined chain vs fan-out from rank 0
    nb_ = args.bcast_bytes
    w = torch.empty(nb_, dtype=torch.uint8, device=f"cuda:{dev}")
    if rank == 0:
        sp.fill_splitmix(dev, w.data_ptr(), nb_, 4242)
    else:
        w.zero_()
    cb = 65536  # the gate granule: b200.chunk_bytes of the chain engines, one flag per granule
    chain_cfg = json.dumps({"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": cb}})
    flags = torch.zeros(nb_ // cb, dtype=torch.int32, device=f"cuda:{dev}")
    hs = gather((sp.ipc_export(dev, w.data_ptr()), sp.ipc_export(dev, flags.data_ptr())))
    ec, pc = None, None
    if pull and rank > 0:
        # rank k pulls w_{k-1} -> w_k: it waits granule by granule for rank k-1 to have
        # delivered w_{k-1} (CONSUME, counters in this GPU's HBM, written by rank k-1) and
        # signals rank k+1 (PRODUCE into rank k+1's counters)
        pw = open_peer(hs[rank - 1][0])
        ec = sp.Engine(fabrics.peer_fabric(sorted({rank - 1, rank})), chain_cfg, dev)
        ec.start()
        seg(ec, f"w{rank - 1}", rank - 1, nb_, pw)
        seg(ec, f"w{rank}", rank, nb_, w.data_ptr())
        if rank > 1:
            ec.gate_segment(f"w{rank - 1}", sp.Engine.GATE_CONSUME, flags.data_ptr())
        if rank + 1 < world:
            ec.gate_segment(f"w{rank}", sp.Engine.GATE_PRODUCE, open_peer(hs[rank + 1][1]))
        pc = ec.prepare_transfers([sp.TransferRequest(f"w{rank - 1}", 0, f"w{rank}", 0, nb_)])
    elif not pull and rank + 1 < world:
        # rank k pushes w_k -> w_{k+1} and signals rank k+1 (PRODUCE into its counters)
        pw, pf = open_peer(hs[rank + 1][0]), open_peer(hs[rank + 1][1])
        ec = sp.Engine(fabrics.peer_fabric(sorted({rank, rank + 1})), chain_cfg, dev)
        ec.start()
        seg(ec, f"w{rank}", rank, nb_, w.data_ptr())
        seg(ec, f"w{rank + 1}", rank + 1, nb_, pw)
        ec.gate_segment(f"w{rank + 1}", sp.Engine.GATE_PRODUCE, pf)
        if rank > 0:
            ec.gate_segment(f"w{rank}", sp.Engine.GATE_CONSUME, flags.data_ptr())
        pc = ec.prepare_transfers([sp.TransferRequest(f"w{rank}", 0, f"w{rank + 1}", 0, nb_)])
    ctimes = []
    for k in range(3):
        if rank > 0:
            w.zero_()
        torch.cuda.synchronize(dev)
        dist.barrier()
        ms = 0.0
        if pc:
            b = ec.allocate_batch()
            ms = pc.run(b)
            st = ec.batch_status(b)
            if st.state != sp.BatchState.COMPLETE:
                print(f"rank {rank}: chain batch {st} counters {ec.counters()} heal {ec.heal_stats()}",
                      file=sys.stderr, flush=True)
                ms = 1e9
            ec.free_batch(b)
        ms = maxr(ms)
        if k:
            ctimes.append(ms)
    torch.cuda.synchronize(dev)
    dist.barrier()
    ref = gather(sp.checksum(dev, w.data_ptr(), nb_) if rank == 0 else None)[0]
    exact = allok(sp.checksum(dev, w.data_ptr(), nb_) == ref)
    if ec:
        pc.free()
        ec.stop()
    # fan-out: rank 0 alone writes into every peer
    ftime = None
    w.zero_() if rank > 0 else None
    torch.cuda.synchronize(dev)
    dist.barrier()
    if rank == 0:
        peers = [open_peer(hs[j][0]) for j in range(1, world)]
        ef = sp.Engine(fabrics.peer_fabric(list(range(world))), chain_cfg, dev)
        ef.start()
        seg(ef, "w0", 0, nb_, w.data_ptr())
        for j, p in enumerate(peers, start=1):
            seg(ef, f"w{j}", j, nb_, p)
        pf_ = ef.prepare_transfers([sp.TransferRequest("w0", 0, f"w{j}", 0, nb_) for j in range(1, world)])
        b = ef.allocate_batch()
        ftime = pf_.run(b)
        if ef.batch_status(b).state != sp.BatchState.COMPLETE:
            ftime = None
        ef.free_batch(b)
        pf_.free()
        ef.stop()
    torch.cuda.synchronize(dev)
    dist.barrier()
    fexact = allok(sp.checksum(dev, w.data_ptr(), nb_) == ref)
    cm = statistics.mean(ctimes)
    out["bcast"] = {"bytes": nb_, "receivers": world - 1, "dtype": "bf16 bit patterns moved as bytes",
                    "chain": ("each hop pulled by the receiving GPU's engine" if pull else
                              "each hop pushed by the forwarding GPU's engine") + ", 64 KiB gated granules",
                    "chain_ms": round(cm, 3), "chain_delivered_gbs": GBs((world - 1) * nb_, cm),
                    "chain_per_receiver_gbs": GBs(nb_, cm), "chain_bit_exact": exact,
                    "fanout_ms": round(ftime, 3) if ftime else None,
                    "fanout_delivered_gbs": GBs((world - 1) * nb_, ftime) if ftime else None,
                    "fanout_bit_exact": fexact,
                    "ideal_pipelined_ms": round(nb_ / 900e9 * 1e3, 3),
                    "ideal_fanout_ms": round((world - 1) * nb_ / 900e9 * 1e3, 3)}
    del w, flags
    torch.cuda.empty_cache()

    # ---- fault under load: rank 0's direct rail DOWN mid-transfer; others keep flowing
    dst.zero_()
    torch.cuda.synchronize(dev)
    dist.barrier()
    ce_gbs = 60e9  # the copy-engine rail's declared bandwidth (per-slice host issue bound)
    # link-down handling only (failure_threshold exclusion + re-spray); the cost model's
    # degradation exclusion stays off as in the other phases
    ef = sp.Engine(fabrics.peer_fabric(sorted({rank, nxt}), sm_rails=1, ce_rails=1 if rank == 0 else 0, bw_ce=ce_gbs),
                   cfg, dev)
    ef.start()
    seg(ef, f"src{rank}", rank, n, src.data_ptr())
    seg(ef, f"dst{nxt}", nxt, n, pdst)
    req = sp.TransferRequest(f"src{rank}", 0, f"dst{nxt}", 0, n)
    heal, state = None, None
    dist.barrier()
    if rank == 0:
        b = ef.allocate_batch()
        ef.submit_transfer(b, req)
        time.sleep(0.3e-3)
        now = ef.now_ns()
        ef.inject_fault(f"g{rank}.nvl0", sp.FaultEffect.DOWN, now, now + 10 ** 13, 0.0)
        st = ef.await_batch(b, 60_000_000_000)
        state = st.state.name
        ef.free_batch(b)
        heal = ef.heal_stats()
        rails = {s.rail_id: {"bytes_ok": s.bytes_ok, "bytes_failed": s.bytes_failed, "health": s.health.name}
                 for s in (ef.rail_stats(r) for r in range(ef.rail_count()))}
    else:
        for _ in range(4):  # background flows
            b = ef.allocate_batch()
            ef.submit_transfer(b, req)
            ef.await_batch(b, 60_000_000_000)
            ef.free_batch(b)
    torch.cuda.synchronize(dev)
    dist.barrier()
    exact = allok(sp.checksum(dev, dst.data_ptr(), n) == sums[prv])
    ef.stop()
    if rank == 0:
        hm = None
        if heal and heal["first_reroute_ok_ns"] and heal["fault_start_ns"]:
            hm = round((heal["first_reroute_ok_ns"] - heal["fault_start_ns"]) / 1e6, 3)
        out["fault"] = {"what": f"g0.nvl0 DOWN 0.3 ms into a {n >> 20} MiB flow 0 -> 1 while the other "
                                f"{world - 1} flow(s) run; alternate = copy-engine rail g0.ce0",
                        "state": state, "heal_ms": hm, "failed_attempts": heal["failed_attempts"],
                        "retried_ok": heal["retried_ok"], "rails": rails, "all_flows_bit_exact": exact,
                        "target_ms": 50}
    for p in opened.values():
        sp.ipc_close(p)
    return out


# ------------------------------------------------------------------ B200 arm
def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2604_00368_b200 as sp
    from paper_2604_00368_b200 import fabrics

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = local
    blk = args.block_kib << 10
    nb = args.blocks
    pool_bytes = blk * nb

    cfg = {"resilience": {"degradation_ratio": 1e9}, "b200": {"chunk_bytes": 65536}}
    cfg["b200"].update(json.loads(os.environ.get("SPRAY_BENCH_B200", "{}")))  # experiments: engine knobs
    eng = sp.Engine(fabrics.kv_offload(dev, sm_rails=args.sm_rails, ce_rails=args.ce_rails, bw_ce=args.ce_gbs * 1e9),
                    json.dumps(cfg), dev)
    eng.start()
    node = f"g{dev}"
    hbm = torch.empty(pool_bytes, dtype=torch.uint8, device=f"cuda:{dev}")
    hbm2 = torch.zeros(pool_bytes, dtype=torch.uint8, device=f"cuda:{dev}")
    sp.fill_splitmix(dev, hbm.data_ptr(), pool_bytes, 1000 + rank)
    # the pinned-host staging pools of this GPU's PCIe root, on the root's NUMA node
    hbuf, hbuf2 = sp.NumaHostBuffer(dev, pool_bytes), sp.NumaHostBuffer(dev, pool_bytes)
    host, host2 = hbuf.tensor(), hbuf2.tensor()
    host2.copy_(hbm.cpu())
    for sid, med, t in (("kv/hbm", sp.Medium.DEVICE, hbm), ("kv/hbm2", sp.Medium.DEVICE, hbm2),
                        ("kv/host", sp.Medium.HOST, host), ("kv/host2", sp.Medium.HOST, host2)):
        eng.register_segment(sp.SegmentDescriptor(sid, med, node, [sp.BufferDesc(0, pool_bytes, t.data_ptr())]))
    rng = np.random.default_rng(7 + rank)
    p_off, p_on = rng.permutation(nb), rng.permutation(nb)
    off = [sp.TransferRequest("kv/hbm", i * blk, "kv/host", int(p_off[i]) * blk, blk) for i in range(nb)]
    on = [sp.TransferRequest("kv/host2", int(p_on[i]) * blk, "kv/hbm2", i * blk, blk) for i in range(nb)]
    g = args.group
    reqs = [r for k in range(0, nb, g) for r in off[k:k + g] + on[k:k + g]]  # swap-out and swap-in interleaved
    step_bytes = 2 * pool_bytes

    # ---- value: device-resident intents, drain-mode launch timed with CUDA events
    prep = eng.prepare_transfers(reqs)
    for _ in range(args.warmup):
        b = eng.allocate_batch()
        prep.run(b)
        assert eng.batch_status(b).state == sp.BatchState.COMPLETE
        eng.free_batch(b)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    kernel_ms = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            b = eng.allocate_batch()
            kernel_ms.append(prep.run(b))
            st = eng.batch_status(b)
            if st.state != sp.BatchState.COMPLETE:
                raise RuntimeError(f"batch not complete: {st}")
            eng.free_batch(b)
    torch.cuda.synchronize()
    total_ms = sum(kernel_ms)
    # bytes check once (outside timing): offload placed by the block table, reload exact
    ok = bool(np.array_equal(host.numpy().reshape(nb, blk)[p_off], hbm.cpu().numpy().reshape(nb, blk)))
    ok = ok and bool(torch.equal(hbm2.cpu().reshape(nb, blk), host2.reshape(nb, blk)[torch.from_numpy(p_on)]))
    if not ok:
        raise RuntimeError("delivered bytes differ")

    # ---- e2e: public API from host arrays, wall clock. The request descriptors are a C
    # array (spray_transfer_request[]) marshalled once, as a C++/cgo caller holds them.
    creqs = sp.Requests(reqs)
    for _ in range(max(1, args.warmup // 2)):
        b = eng.allocate_batch()
        eng.submit_transfers(b, creqs)
        eng.await_batch(b)
        eng.free_batch(b)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step_t = []
    for _ in range(args.steps):
        ts = time.perf_counter()
        b = eng.allocate_batch()
        eng.submit_transfers(b, creqs)
        st = eng.await_batch(b)
        if st.state != sp.BatchState.COMPLETE:
            raise RuntimeError(f"e2e batch not complete: {st}")
        eng.free_batch(b)
        step_t.append((time.perf_counter() - ts) * 1e3)
    # the step ends when await_batch has read COMPLETE from the mapped counters (published
    # after the delivered bytes were fenced); a device-wide synchronize here would instead
    # wait out the persistent kernel's idle-exit timer
    e2e_ms = (time.perf_counter() - t0) * 1e3
    if os.environ.get("SPRAY_BENCH_DEBUG"):
        print("e2e step ms:", [round(x, 3) for x in step_t], file=sys.stderr, flush=True)

    e2e_step_ms = step_t
    lat = batch_latency(sp, eng, reqs, args.lat_batches, args.lat_intents) if args.lat_batches else None
    lat_c = None
    if args.lat_batches:
        one = [sp.TransferRequest("kv/hbm", int(p_off[i]) * blk, "kv/host", i * blk, 4096) for i in range(256)]
        lat_c = {"intent_4k_hbm_to_host": batch_latency_c(sp, eng, one, 1),
                 "kv_batch": batch_latency_c(sp, eng, reqs, args.lat_intents)}

    # ---- state-blind baseline: round-robin cudaMemcpyAsync striping of the same blocks
    # (one call per block from C++, the same interleaved order, 4 streams)
    hb0, hs0, h20, hb20 = hbm.data_ptr(), host.data_ptr(), host2.data_ptr(), hbm2.data_ptr()
    rr_src, rr_dst = [], []
    for k in range(0, nb, g):
        for i in range(k, min(nb, k + g)):
            rr_src.append(hb0 + i * blk)
            rr_dst.append(hs0 + int(p_off[i]) * blk)
        for i in range(k, min(nb, k + g)):
            rr_src.append(h20 + int(p_on[i]) * blk)
            rr_dst.append(hb20 + i * blk)
    rr_len = [blk] * len(rr_src)
    sp.rr_copy(dev, rr_src, rr_dst, rr_len, 4)
    rr_steps = max(1, min(5, args.steps))
    rr_ms = sum(sp.rr_copy(dev, rr_src, rr_dst, rr_len, 4) for _ in range(rr_steps)) / rr_steps

    # ---- max over ranks
    vals = torch.tensor([total_ms, e2e_ms, rr_ms], dtype=torch.float64, device=f"cuda:{dev}")
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    total_ms, e2e_ms, rr_ms = vals.tolist()
    eng.stop()

    small = None
    if rank == 0 and not args.no_small:
        try:
            peak = 6544.7
            try:
                peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
            except Exception:
                pass
            small = small_slices(sp, fabrics, dev, hbm, hbm2, nb, blk, p_off, peak)
        except Exception as ex:  # reported, never fatal
            small = {"error": str(ex)[:300]}
    cong = None
    if rank == 0 and not args.no_congestion:
        try:
            cong = congestion(sp, fabrics, dev, hbm, host, nb, blk, p_off)
        except Exception as ex:  # reported, never fatal
            cong = {"error": str(ex)[:300]}
    nvl = None
    if world > 1 and not args.no_nvlink:
        try:
            del hbm2, host2
            nvl = nvlink_phase(sp, fabrics, args, rank, world, dev)
        except Exception as ex:  # reported, never fatal
            nvl = {"error": f"{type(ex).__name__}: {str(ex)[:300]}"}

    if rank == 0:
        value = world * args.steps * step_bytes / (total_ms * 1e-3) / 1e9
        e2e = world * args.steps * step_bytes / (e2e_ms * 1e-3) / 1e9
        per_launch_gbs = step_bytes / (total_ms / args.steps * 1e-3) / 1e9
        # denominator: the host link's measured full-duplex ceiling on this pool (copy
        # engines, tools/pcie_peak.cu); MEASURED_PEAKS.json and the profiling guide carry no
        # PCIe figure. Nominal Gen5 x16 (2 x 64 GB/s) and the SM load/store ceiling for context.
        peak, peak_src, link = 2 * PCIE_NOMINAL_GBS, "nominal PCIe Gen5 x16, 2 x 64 GB/s", {}
        try:
            link = json.load(open(os.path.join(ROOT, "profiles", "pcie_peak_r01.json")))
            peak = float(link["ce_both_gbs"])
            peak_src = ("measured: copy-engine full-duplex HBM<->pinned host on this pool "
                        "(tools/pcie_peak.cu -> profiles/pcie_peak_r01.json)")
        except Exception:
            pass
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_engine_kernel_r02c.json")
        if not os.path.exists(prof):
            prof = os.path.join(ROOT, "profiles", "ncu_engine_kernel_final_r01.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        line = {
            "metric": "sprayed transfer GB/s (KV batch, HBM<->pinned host)",
            "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"kv_batch: {nb} x {args.block_kib} KiB offload HBM->pinned host + {nb} x "
                                   f"{args.block_kib} KiB reload pinned host->HBM per GPU, random block tables, "
                                   f"one batch of {2 * nb} intents per step, offloads and reloads alternating in "
                                   f"runs of {args.group}",
                       "fabric": f"{args.sm_rails} SM PCIe rail(s) + {args.ce_rails} copy-engine rail(s) per GPU (kv_offload)",
                       "bytes_per_step_per_gpu": step_bytes,
                       "host_pools": f"pinned + device-mapped, NUMA node {hbuf.node} of GPU {dev}'s PCIe root "
                                     f"(spray_host_alloc_numa; -1 = host reports no node, first-touch placement)",
                       "l2": "inputs (2 x 256 MiB pools) larger than the 126 MB L2",
                       "parallelism": f"weak x{world} (one batch per GPU, no data-path collective)"},
            "e2e": {"value": round(e2e, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": pool_bytes + 64 * 2 * nb, "d2h_bytes_per_step": pool_bytes + 16},
            "roofline": {"bound": "pcie", "achieved": round(per_launch_gbs, 3), "peak": peak, "unit": "GB/s",
                         "frac": round(per_launch_gbs / peak, 4), "traffic": traffic,
                         "traffic_unit": "DRAM bytes per launch (ncu, " + os.path.relpath(prof, ROOT) + "); the "
                                         "host-link bytes per launch there equal the algorithmic 512 MiB",
                         "peak_source": peak_src, "nominal_gbs": 2 * PCIE_NOMINAL_GBS,
                         "sm_copy_ceiling_gbs": link.get("sm_both_lsu_gbs", 80.35),
                         "kernel": "spray_engine_kernel (drain-mode launch per step)"},
            "rr_baseline": {"value": round(world * step_bytes / (rr_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                            "what": "state-blind round-robin striping: one cudaMemcpyAsync per block from C++ "
                                    "(spray_rr_copy), 4 streams, same blocks and order"},
            "batch_latency": {"kv_batch_8192_intents": {"p50_ms": round(pct(e2e_step_ms, 0.5), 3),
                                                        "p90_ms": round(pct(e2e_step_ms, 0.9), 3),
                                                        "steps": len(e2e_step_ms)},
                              "small_batches": lat,
                              "small_batches_cpp": lat_c,
                              "how": "submit -> batch terminal through the public C-ABI, one batch in flight; "
                                     "exact_percentile as bench.cpp:213-215"},
            "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
        }
        if small is not None:
            line["small_slices"] = small
        if cong is not None:
            line["congestion"] = cong
        if nvl is not None:
            line["nvlink"] = nvl
        if world == 1 and not args.no_cpu_baseline:
            try:
                r = reference_kv(nb, blk, 10.0, 2)
                if r:
                    gbs, iters, cores = r
                    line["cpu_baseline"] = {"value": round(gbs, 3), "unit": "GB/s", "cores": cores,
                                            "nproc": os.cpu_count(), "kind": "reference",
                                            "sample": f"best of {iters} batches of {nb} x {args.block_kib} KiB "
                                                      "host->host through the reference Engine (memory backend, "
                                                      "real clock, 2 rails / 2 workers)"}
            except Exception as ex:  # reported, never fatal
                line["cpu_baseline"] = {"value": None, "error": str(ex)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
