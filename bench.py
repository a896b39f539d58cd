#!/usr/bin/env python
"""bench.py — the B200 slice-spraying data plane on its headline single-GPU workload.

Workload (BASELINE.json configs[2], the largest single-GPU configuration): a HiCache-style
KV batch per GPU — 4096 x 64 KiB offloads (HBM -> pinned host) plus 4096 x 64 KiB reloads
(pinned host -> HBM), both through seeded random block tables, as ONE batch of 8192
transfer intents. A "step" is one such batch (512 MiB delivered). At N GPUs every rank
runs its own batch over its own PCIe root (weak scaling, no data-path collective).

  value    device-resident intents (prepared once in HBM), engine kernel launched in
           drain mode and timed with CUDA events on its stream: GB/s delivered.
  e2e      the public C-ABI path from host arrays: submit_transfers (8192 intents through
           the mapped submission ring) + await_batch, wall clock, CUDA-synchronised.
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
    p.add_argument("--ce-rails", type=int, default=0, help="copy-engine rails sprayed beside the SM rail")
    p.add_argument("--ce-gbs", type=float, default=15.0, help="declared bandwidth of each copy-engine rail")
    p.add_argument("--no-cpu-baseline", action="store_true")
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
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
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
    eng = sp.Engine(fabrics.kv_offload(dev, sm_rails=1, ce_rails=args.ce_rails, bw_ce=args.ce_gbs * 1e9),
                    json.dumps(cfg), dev)
    eng.start()
    node = f"g{dev}"
    hbm = torch.empty(pool_bytes, dtype=torch.uint8, device=f"cuda:{dev}")
    hbm2 = torch.zeros(pool_bytes, dtype=torch.uint8, device=f"cuda:{dev}")
    sp.fill_splitmix(dev, hbm.data_ptr(), pool_bytes, 1000 + rank)
    host = torch.zeros(pool_bytes, dtype=torch.uint8, pin_memory=True)
    host2 = torch.empty(pool_bytes, dtype=torch.uint8, pin_memory=True)
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
        prof = os.path.join(ROOT, "profiles", "ncu_engine_kernel.json")
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
                       "fabric": f"1 SM PCIe rail + {args.ce_rails} copy-engine rails per GPU (kv_offload)", "bytes_per_step_per_gpu": step_bytes,
                       "l2": "inputs (2 x 256 MiB pools) larger than the 126 MB L2",
                       "parallelism": f"weak x{world} (one batch per GPU, no data-path collective)"},
            "e2e": {"value": round(e2e, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": pool_bytes + 64 * 2 * nb, "d2h_bytes_per_step": pool_bytes + 16},
            "roofline": {"bound": "pcie", "achieved": round(per_launch_gbs, 3), "peak": peak, "unit": "GB/s",
                         "frac": round(per_launch_gbs / peak, 4), "traffic": traffic,
                         "traffic_unit": "DRAM bytes per launch (ncu, profiles/ncu_engine_kernel.json); the "
                                         "host-link bytes per launch there equal the algorithmic 512 MiB",
                         "peak_source": peak_src, "nominal_gbs": 2 * PCIE_NOMINAL_GBS,
                         "sm_copy_ceiling_gbs": link.get("sm_both_lsu_gbs", 80.35),
                         "kernel": "spray_engine_kernel (drain-mode launch per step)"},
            "rr_baseline": {"value": round(world * step_bytes / (rr_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                            "what": "state-blind round-robin striping: one cudaMemcpyAsync per block from C++ "
                                    "(spray_rr_copy), 4 streams, same blocks and order"},
            "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                r = reference_kv(nb, blk, 10.0, 2)
                if r:
                    gbs, iters, cores = r
                    line["cpu_baseline"] = {"value": round(gbs, 3), "unit": "GB/s", "cores": cores,
                                            "kind": "reference",
                                            "sample": f"best of {iters} batches of {nb} x {args.block_kib} KiB "
                                                      "host->host through the reference Engine (memory backend, "
                                                      "real clock, 2 rails / 2 workers)"}
            except Exception as ex:  # reported, never fatal
                line["cpu_baseline"] = {"value": None, "error": str(ex)}
        print(json.dumps(line), flush=True)
    eng.stop()
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
