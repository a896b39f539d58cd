"""Trace records (include/spray_b200.h spray_trace_event / spray_decision) and the device
replay entry: the live scheduler's decision function run over a recorded trace."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .engine import _check

EVENT_DTYPE = np.dtype([
    ("kind", "<u4"), ("rail", "<u4"), ("remote", "<u4"), ("flags", "<u4"),
    ("len", "<u8"), ("offset", "<u8"), ("t_ns", "<u8"), ("now_ns", "<u8"),
    ("predicted", "<f8"), ("x_norm", "<f8")])
DECISION_DTYPE = np.dtype([
    ("local", "<u4"), ("remote", "<u4"), ("tier", "<i4"), ("ok", "<u4"),
    ("predicted_s", "<f8"), ("x_norm", "<f8")])

EV_DECIDE, EV_COMPLETE, EV_CHARGE, EV_RELEASE, EV_HEALTH, EV_RESET, EV_RESET_RAIL, EV_EXPECT = range(1, 9)


def sched_config(**kw) -> L.SchedConfig:
    c = L.SchedConfig()
    L.lib.spray_sched_config_default(C.byref(c))
    for k, v in kw.items():
        if k == "penalties":
            for i in range(3):
                c.penalty[i] = v[i] if v[i] is not None else 0.0
        else:
            setattr(c, k, v)
    return c


def res_config(**kw) -> L.ResConfig:
    r = L.ResConfig()
    L.lib.spray_resilience_config_default(C.byref(r))
    for k, v in kw.items():
        setattr(r, k, v)
    return r


def replay_device(device: int, sc: L.SchedConfig, rc: L.ResConfig, bandwidth, base_tier, id_rank,
                  cand_stream, events):
    """Decisions of the device decision function (the code the live engine runs) for a
    trace; returns (decisions, expect_failures)."""
    events = np.ascontiguousarray(events, EVENT_DTYPE)
    bw = np.ascontiguousarray(bandwidth, np.float64)
    tier = np.ascontiguousarray(base_tier, np.int32)
    rank = np.ascontiguousarray(id_rank, np.uint32)
    cand = np.ascontiguousarray(cand_stream, np.int32)
    cap = max(1, int((events["kind"] == EV_DECIDE).sum()))
    dec = np.zeros(cap, DECISION_DTYPE)
    nd = C.c_size_t()
    bad = C.c_uint64()
    _check(L.lib.spray_replay_device(device, C.byref(sc), C.byref(rc), len(bw), bw.ctypes.data,
                                     tier.ctypes.data, rank.ctypes.data, cand.ctypes.data, cand.size,
                                     events.ctypes.data, events.size, dec.ctypes.data, cap, C.byref(nd),
                                     C.byref(bad)))
    return dec[: nd.value], bad.value
