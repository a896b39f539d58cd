"""Deterministic fabrics and telemetry traces for the parity tests (test infrastructure).

Topology documents use the reference's JSON format (proj/src/fabric.cpp:157-210);
traces use the event format of include/spray_b200.h. Everything here is seeded, so
tests regenerate exactly the inputs tests/golden/make_golden.py recorded.
"""
from __future__ import annotations

import json

import numpy as np

from oracle.oracle import (EV_BOARD, EV_CHARGE, EV_COMPLETE, EV_DECIDE, EV_DUE_PROBES, EV_EXPECT, EV_HEALTH,
                           EV_PROBE_DONE, EV_RELEASE, EV_RESET, EV_RESET_RAIL, EVENT_DTYPE, EVF_CANCELLED,
                           EVF_MODEL, NO_RAIL)

SIM_CAPS = dict(pairs="all", cross=True, same=False)          # sim_backend.cpp:9-25
MEMORY_CAPS = dict(pairs="all", cross=True, same=True)        # memory_backend.cpp:8-19


def two_node_doc(rails_per_node, bw=1e9, affinities=None, backend="sim", devices=True):
    """Nodes a and b with `rails_per_node` rails each (ids a.rK / b.rK)."""
    nodes = []
    for n in ("a", "b"):
        devs = [{"id": f"{n}.mem", "kind": "host_memory"}]
        if devices:
            devs.append({"id": f"{n}.dev", "kind": "device_memory"})
        nodes.append({"id": n, "devices": devs})
    rails = []
    for n in ("a", "b"):
        for i in range(rails_per_node):
            b = bw[i] if isinstance(bw, (list, tuple)) else bw
            aff = affinities[i] if affinities else "direct"
            rails.append({"id": f"{n}.r{i}", "node": n, "bandwidth_bytes_per_sec": float(b),
                          "affinity": aff, "backend": backend})
    return json.dumps({"nodes": nodes, "rails": rails})


def random_doc(rng: np.random.Generator, backend="sim"):
    """Random 2-node fabric in the spirit of acceptance.cpp:64-86, with tier-3 rails too."""
    k = int(rng.integers(1, 9))
    bws = [float(0.5e9 + rng.integers(0, 3500) * 1e6) for _ in range(k)]
    affs = []
    for i in range(k):
        r = rng.integers(0, 6)
        affs.append("direct" if i == 0 or r < 3 else ("same_socket" if r < 5 else "cross_socket"))
    return two_node_doc(k, bws, affs, backend)


def random_trace(rng: np.random.Generator, cstate, n_sets: int, n_rails: int, bw, n_events: int,
                 health_changes=True, resets=True, board=False):
    """Realistic event stream: decisions, completions of earlier decisions (OK, FAILED,
    with/without feedback), retries as CHARGE, health flips, periodic resets, and (board)
    load-board refreshes: one BOARD event per rail carrying a global queue that is this
    instance's queue plus other instances' load. `cstate` (oracle.CState) is stepped
    alongside so completions release what was charged."""
    events = []
    outstanding = []   # (local, remote, len, predicted, x, model)
    probes = []        # rails with a probe in flight
    now = 0
    for _ in range(n_events):
        now += int(rng.integers(1_000, 200_000))
        if board and rng.random() < 0.04:
            _, queued, _, _, _ = cstate.step(np.zeros(0, EVENT_DTYPE))
            for r in range(n_rails):
                other = int(rng.choice([0, 0, int(rng.integers(0, 1 << 24)), int(rng.integers(0, 1 << 30))]))
                b = np.zeros(1, EVENT_DTYPE)
                b["kind"] = EV_BOARD
                b["rail"] = r
                b["len"] = max(0, int(queued[r])) + other
                b["now_ns"] = now
                cstate.step(b)
                events.append(b[0])
        u = rng.random()
        e = np.zeros(1, EVENT_DTYPE)
        if u < 0.45 or not outstanding:
            e["kind"] = EV_DECIDE
            e["rail"] = int(rng.integers(0, n_sets))
            e["len"] = int(rng.choice([65536, 262144, 4 << 20, int(rng.integers(1, 1 << 22))]))
            e["offset"] = int(rng.integers(0, 1 << 40))
            dec, *_ = cstate.step(e)
            d = dec[0]
            if d["ok"]:
                outstanding.append((int(d["local"]), int(d["remote"]), int(e["len"][0]),
                                    float(d["predicted_s"]), float(d["x_norm"]), True))
        elif u < 0.85:
            k = int(rng.integers(0, len(outstanding)))
            local, remote, ln, pred, x, model = outstanding.pop(k)
            status = 0 if rng.random() < 0.9 else int(rng.integers(1, 3))
            slow = 1.0 if rng.random() < 0.8 else float(rng.choice([3.0, 6.0, 12.0]))
            t_ns = max(1, int((ln / bw[local]) * 1e9 * slow * (0.5 + rng.random())))
            e["kind"] = EV_COMPLETE
            e["rail"] = local
            e["remote"] = remote
            flags = (EVF_MODEL if model else 0) | (EVF_CANCELLED if rng.random() < 0.03 else 0)
            e["flags"] = flags | (status << 8)
            e["len"] = ln
            e["t_ns"] = t_ns
            e["now_ns"] = now
            e["predicted"] = pred
            e["x_norm"] = x
            cstate.step(e)
            if status != 0 and rng.random() < 0.7:
                # engine retry (dispatch_retry): bypasses the model but charges L
                r = int(rng.integers(0, n_rails))
                c = np.zeros(1, EVENT_DTYPE)
                c["kind"] = EV_CHARGE
                c["rail"] = r
                c["len"] = ln
                cstate.step(c)
                events.append(e[0])
                e = c
                outstanding.append((r, NO_RAIL, ln, 0.0, 0.0, False))
        elif u < 0.88 and health_changes:
            e["kind"] = EV_HEALTH
            e["rail"] = int(rng.integers(0, n_rails))
            e["flags"] = int(rng.choice([0, 0, 1]))
            cstate.step(e)
        elif u < 0.90 and health_changes:
            # prober: due_probes(now) moves due excluded rails to PROBING; each gets a
            # probe slice (charged) whose completion runs observe_probe
            before = cstate.step(np.zeros(0, EVENT_DTYPE))[3].copy()
            e["kind"] = EV_DUE_PROBES
            e["t_ns"] = now + int(rng.integers(0, 3)) * 1_000_000_000
            _, _, _, health, _ = cstate.step(e)
            events.append(e[0])
            for r in np.nonzero((health == 2) & (before == 1))[0]:
                c = np.zeros(1, EVENT_DTYPE)
                c["kind"] = EV_CHARGE
                c["rail"] = int(r)
                c["len"] = 4096
                cstate.step(c)
                events.append(c[0])
                probes.append(int(r))
            continue
        elif u < 0.91 and probes:
            r = probes.pop(int(rng.integers(0, len(probes))))
            e["kind"] = EV_PROBE_DONE
            e["rail"] = r
            e["len"] = 4096
            e["flags"] = (0 if rng.random() < 0.7 else 1) << 8
            e["now_ns"] = now
            cstate.step(e)
        elif u < 0.93 and resets:
            e["kind"] = EV_RESET
            e["t_ns"] = now * int(rng.integers(1, 400))
            cstate.step(e)
        elif u < 0.95 and resets:
            e["kind"] = EV_RESET_RAIL
            e["rail"] = int(rng.integers(0, n_rails))
            e["t_ns"] = now
            cstate.step(e)
        else:
            # reroute at post time (engine.cpp:896-916): release then decide again
            k = int(rng.integers(0, len(outstanding)))
            local, remote, ln, pred, x, model = outstanding.pop(k)
            e["kind"] = EV_RELEASE
            e["rail"] = local
            e["len"] = ln
            cstate.step(e)
        events.append(e[0])
    # final health assertions, recorded from the generator's own state
    _, _, _, health, _ = cstate.step(np.zeros(0, EVENT_DTYPE))
    for r in range(n_rails):
        x = np.zeros(1, EVENT_DTYPE)
        x["kind"] = EV_EXPECT
        x["rail"] = r
        x["flags"] = int(health[r])
        events.append(x[0])
    return np.array(events, dtype=EVENT_DTYPE)


def stream_concat(streams):
    """Concatenate single-set candidate streams into one multi-set stream."""
    out = [len(streams)]
    for s in streams:
        s = list(s)
        assert s[0] == 1
        out.extend(s[1:])
    return np.array(out, np.int32)
