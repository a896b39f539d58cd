"""Generate tests/golden/ fixtures FROM THE REFERENCE ITSELF (oracle/_ref).

Run in the container that has /root/reference (after `make -f oracle/Makefile`):
    python tests/golden/make_golden.py
Every fixture stores the inputs and the reference library's outputs; the CPU tests
check the C oracle against them and the GPU tests check the CUDA path against the
oracle and the fixtures.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.oracle import (EVENT_DTYPE, EV_DECIDE, COracle, CState, RefOracle, caps,  # noqa: E402
                           res_config, sched_config)
import spraygen  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def decompose_fixture(ref):
    rng = np.random.default_rng(11)
    totals = [1 << 20, 10 * 1024, 1 << 30, 64 << 20, 16 << 30, 65536, 65535, 65537, 1, 4096 * 65536 + 1]
    totals += [int(x) for x in rng.integers(1, 1 << 34, 200)]
    cfgs = [(65536, 4096), (4096, 7), (1 << 20, 4096), (65536, 1)]
    rows = []
    for mn, mx in cfgs:
        for t in totals:
            off, ln = ref.decompose(t, mn, mx)
            rows.append([t, mn, mx, len(off), int(ln[0]), int(ln[-1]), int(off[-1])])
    np.save(os.path.join(OUT, "decompose.npy"), np.array(rows, np.uint64))


def cands_for(ref, topo, caps_list, direction=1, src=("a", 0, ""), dst=("b", 0, ""), sc=None):
    sc = sc or sched_config()
    stream, backend, nroutes = ref.candidates(topo, caps_list, src, dst, direction, sc)
    return stream


def replay_fixtures(ref, co):
    rng = np.random.default_rng(2026)
    cases = {}
    for case in range(24):
        topo = spraygen.random_doc(rng)
        policy = [0, 0, 0, 1, 2][case % 5]
        tol = [0.05, 1e-9, 0.5][case % 3]
        pens = [(1.0, 3.0, 0.0), (1.0, 3.0, 9.0), (1.0, 0.0, 0.0), (1.0, 1.0, 1.0)][case % 4]
        sc = sched_config(policy=policy, tolerance=tol, penalties=pens,
                          reset_interval_ns=[30_000_000_000, 5_000_000][case % 2])
        rc = res_config()
        bw, tier, rank, ids = ref.rails(topo)
        sim_caps = caps("sim", **spraygen.SIM_CAPS)
        try:
            s_w = cands_for(ref, topo, [sim_caps], 1, sc=sc)
            s_r = cands_for(ref, topo, [sim_caps], 0, sc=sc)
        except RuntimeError:
            continue  # NoRoute under this penalty set
        stream = spraygen.stream_concat([s_w, s_r])
        st = CState(co, sc, rc, bw, tier, rank, stream)
        events = spraygen.random_trace(rng, st, 2, len(bw), bw, 1500)
        out = ref.replay(topo, sc, rc, stream, events, len(bw))
        cases[f"case{case}"] = dict(topo=topo, sc=bytes(sc), rc=bytes(rc), stream=stream, events=events,
                                   decisions=out["decisions"], queued=out["queued"], beta=out["beta"],
                                   health=out["health"], expect_failures=out["expect_failures"],
                                   bw=bw, tier=tier, rank=rank)
    # GlobalLoadBoard cases (scheduler.cpp:63-79, 108-114): omega > 0 with BOARD events;
    # a separate generator so the cases above stay as they were
    rng = np.random.default_rng(2027)
    for case in range(24, 32):
        topo = spraygen.random_doc(rng)
        policy = [0, 0, 1, 2][case % 4]
        omega = [0.25, 0.5, 0.9, 1.0][case % 4]
        sc = sched_config(policy=policy, tolerance=[0.05, 1e-9][case % 2], omega=omega)
        rc = res_config()
        bw, tier, rank, ids = ref.rails(topo)
        sim_caps = caps("sim", **spraygen.SIM_CAPS)
        try:
            s_w = cands_for(ref, topo, [sim_caps], 1, sc=sc)
            s_r = cands_for(ref, topo, [sim_caps], 0, sc=sc)
        except RuntimeError:
            continue
        stream = spraygen.stream_concat([s_w, s_r])
        st = CState(co, sc, rc, bw, tier, rank, stream)
        events = spraygen.random_trace(rng, st, 2, len(bw), bw, 1500, board=True)
        out = ref.replay(topo, sc, rc, stream, events, len(bw))
        cases[f"case{case}"] = dict(topo=topo, sc=bytes(sc), rc=bytes(rc), stream=stream, events=events,
                                   decisions=out["decisions"], queued=out["queued"], beta=out["beta"],
                                   health=out["health"], expect_failures=out["expect_failures"],
                                   bw=bw, tier=tier, rank=rank)
    np.savez_compressed(os.path.join(OUT, "replay.npz"),
                        **{f"{k}__{f}": (np.frombuffer(v, np.uint8) if isinstance(v, bytes)
                                         else np.array(v)) for k, d in cases.items() for f, v in d.items()})


def c1_fixture(ref):
    """Config 1: 64 MiB host->host over 2 simulated rails per node (uniform, 1e9 B/s)."""
    topo = spraygen.two_node_doc(2, 1e9, backend="sim")
    sc = sched_config()
    stream = cands_for(ref, topo, [caps("sim", **spraygen.SIM_CAPS)], 1, sc=sc)
    off, ln = ref.decompose(64 << 20)
    ev = np.zeros(len(off), EVENT_DTYPE)
    ev["kind"] = EV_DECIDE
    ev["rail"] = 0
    ev["len"] = ln
    ev["offset"] = off
    out = ref.replay(topo, sc, res_config(), stream, ev, 4)
    dst, ok = ref.engine_sim_transfer(topo, 64 << 20, 1, 4)
    co = COracle()
    np.savez_compressed(os.path.join(OUT, "c1.npz"), topo=np.frombuffer(topo.encode(), np.uint8),
                        stream=stream, decisions=out["decisions"], dst_checksum=np.uint64(co.checksum(dst)),
                        rail_bytes_ok=ok)


def orchestrator_fixture(ref):
    """Candidate ordering (orchestrator.cpp:39-81) on several fabrics, both directions."""
    docs = {"uniform8": open("/root/reference/proj/fabrics/uniform8.json").read(),
            "skewed8": open("/root/reference/proj/fabrics/skewed8.json").read(),
            "tiered": open("/root/reference/proj/fabrics/tiered.json").read()}
    rows = {}
    for name, topo in docs.items():
        for direction in (0, 1):
            for cname, cps in (("sim", [caps("sim", **spraygen.SIM_CAPS)]),
                               ("mem", [caps("memory", **spraygen.MEMORY_CAPS)])):
                try:
                    s = cands_for(ref, topo, cps, direction)
                except RuntimeError as e:
                    s = np.array([-1], np.int32)
                rows[f"{name}__{direction}__{cname}"] = s
    np.savez_compressed(os.path.join(OUT, "orchestrator.npz"),
                        **{k.replace("__", "_X_"): v for k, v in rows.items()},
                        **{f"doc_{k}": np.frombuffer(v.encode(), np.uint8) for k, v in docs.items()})


def sim_fixture(ref):
    """sim_backend service arithmetic KATs (test_backends.cpp:95-120) via the reference."""
    topo = json.dumps({"nodes": [{"id": "a"}, {"id": "b"}],
                       "rails": [{"id": "a.r0", "node": "a", "bandwidth_bytes_per_sec": float(1 << 30),
                                  "affinity": "direct", "sim": {"latency_us": 10}},
                                 {"id": "b.r0", "node": "b", "bandwidth_bytes_per_sec": float(1 << 30),
                                  "affinity": "direct", "sim": {"latency_us": 10}}]})
    rows = []
    for ln in (1 << 20, 4096, 65536, 262144, 4 << 20, 12345):
        for deg in (1.0, 0.25, 0.5):
            rows.append([ln, int(deg * 1000), ref.sim_one(topo, ln, deg)])
    np.save(os.path.join(OUT, "sim.npy"), np.array(rows, np.uint64))


if __name__ == "__main__":
    ref = RefOracle()
    co = COracle()
    decompose_fixture(ref)
    replay_fixtures(ref, co)
    c1_fixture(ref)
    orchestrator_fixture(ref)
    sim_fixture(ref)
    print("golden fixtures written to", OUT)
