"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

* ``C``   : oracle/_build/libspray_oracle.so, the plain-C restatement (spray_oracle.c).
* ``REF`` : oracle/_ref/libspray_ref.so, the UNMODIFIED reference library plus
            ref_harness.cpp (present when it was built in the container that has
            /root/reference; it travels to GPU boxes as a prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this.
The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

EVENT_DTYPE = np.dtype([
    ("kind", "<u4"), ("rail", "<u4"), ("remote", "<u4"), ("flags", "<u4"),
    ("len", "<u8"), ("offset", "<u8"), ("t_ns", "<u8"), ("now_ns", "<u8"),
    ("predicted", "<f8"), ("x_norm", "<f8")])
DECISION_DTYPE = np.dtype([
    ("local", "<u4"), ("remote", "<u4"), ("tier", "<i4"), ("ok", "<u4"),
    ("predicted_s", "<f8"), ("x_norm", "<f8")])
assert EVENT_DTYPE.itemsize == 64 and DECISION_DTYPE.itemsize == 32

EV_DECIDE, EV_COMPLETE, EV_CHARGE, EV_RELEASE, EV_HEALTH, EV_RESET, EV_RESET_RAIL, EV_EXPECT = range(1, 9)
EV_DUE_PROBES, EV_PROBE_DONE, EV_BOARD = 9, 10, 11
EVF_MODEL, EVF_CANCELLED = 1, 2
NO_RAIL = 0xFFFFFFFF


class SchedConfig(C.Structure):
    _fields_ = [("min_slice_size", C.c_uint64), ("max_slices_per_transfer", C.c_uint32),
                ("policy", C.c_int32), ("tolerance", C.c_double), ("penalty", C.c_double * 3),
                ("ewma_alpha", C.c_double), ("reset_interval_ns", C.c_uint64),
                ("beta0_init_s", C.c_double), ("beta1_init", C.c_double),
                ("feedback_clamp", C.c_double), ("diffusion_weight", C.c_double)]


class ResConfig(C.Structure):
    _fields_ = [("failure_threshold", C.c_int32), ("degradation_events", C.c_int32),
                ("degradation_ratio", C.c_double), ("degradation_min_t_obs_s", C.c_double),
                ("probe_successes_needed", C.c_int32), ("probe_backoff_cap", C.c_int32),
                ("probe_bytes", C.c_uint64), ("probe_interval_ns", C.c_uint64),
                ("probe_backoff_mult", C.c_double), ("max_attempts", C.c_uint32),
                ("pad_", C.c_uint32), ("slice_timeout_ns", C.c_uint64)]


class BackendCaps(C.Structure):
    _fields_ = [("id", C.c_char * 32), ("media_pairs_mask", C.c_uint32),
                ("supports_read", C.c_uint8), ("supports_write", C.c_uint8),
                ("cross_node", C.c_uint8), ("same_node", C.c_uint8),
                ("max_post_size", C.c_uint64), ("batched_posting", C.c_uint8),
                ("pad_", C.c_uint8 * 7)]


def sched_config(policy=0, tolerance=0.05, penalties=(1.0, 3.0, 0.0), alpha=0.2,
                 reset_interval_ns=30_000_000_000, min_slice=65536, max_slices=4096,
                 beta0=0.0, beta1=1.0, clamp=5.0, omega=0.0) -> SchedConfig:
    """Defaults of spray::SchedulerConfig (scheduler.hpp:44-58)."""
    c = SchedConfig()
    c.min_slice_size, c.max_slices_per_transfer, c.policy = min_slice, max_slices, policy
    c.tolerance = tolerance
    for i in range(3):
        c.penalty[i] = penalties[i] if penalties[i] is not None else 0.0
    c.ewma_alpha, c.reset_interval_ns = alpha, reset_interval_ns
    c.beta0_init_s, c.beta1_init, c.feedback_clamp = beta0, beta1, clamp
    c.diffusion_weight = omega
    return c


def res_config(**kw) -> ResConfig:
    """Defaults of spray::ResilienceConfig (resilience.hpp:17-28)."""
    r = ResConfig()
    r.failure_threshold, r.degradation_events = 3, 8
    r.degradation_ratio, r.degradation_min_t_obs_s = 4.0, 1e-3
    r.probe_successes_needed, r.probe_backoff_cap = 2, 3
    r.probe_bytes, r.probe_interval_ns = 4096, 1_000_000_000
    r.probe_backoff_mult, r.max_attempts = 1.0, 4
    r.slice_timeout_ns = 500_000_000
    for k, v in kw.items():
        setattr(r, k, v)
    return r


def caps(id_: str, pairs="all", read=True, write=True, cross=True, same=True) -> BackendCaps:
    b = BackendCaps()
    b.id = id_.encode()
    if pairs == "all":
        mask = 0
        for s in (0, 1):
            for d in (0, 1):
                mask |= 1 << (s * 3 + d)
    else:
        mask = 0
        for s, d in pairs:
            mask |= 1 << (s * 3 + d)
    b.media_pairs_mask = mask
    b.supports_read, b.supports_write, b.cross_node, b.same_node = read, write, cross, same
    b.max_post_size = 1 << 30
    b.batched_posting = 1
    return b


def _ptr(a, t=C.c_void_p):
    return a.ctypes.data_as(t)


def build_c() -> str:
    """Compile the C restatement if needed (gcc exists on every box of this image)."""
    so = os.path.join(HERE, "_build", "libspray_oracle.so")
    src = os.path.join(HERE, "spray_oracle.c")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(so), exist_ok=True)
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", so, src])
    return so


class COracle:
    def __init__(self):
        self.lib = C.CDLL(build_c())
        L = self.lib
        L.so_decompose.restype = C.c_uint64
        L.so_decompose.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint64]
        L.so_replay_flat.restype = C.c_int
        L.so_checksum.restype = C.c_uint64
        L.so_checksum.argtypes = [C.c_void_p, C.c_uint64]
        L.so_fill_pattern.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.so_hist_bucket.argtypes = [C.c_uint64]
        L.so_sim_done_ns.restype = C.c_uint64
        L.so_sim_done_ns.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                     C.c_double, C.c_double]
        L.so_sim_partial_bytes.restype = C.c_uint64
        L.so_sim_partial_bytes.argtypes = [C.c_uint64] * 4
        L.so_sched_config_validate.argtypes = [C.POINTER(SchedConfig)]

    def decompose(self, total, min_slice=65536, max_slices=4096):
        n = self.lib.so_decompose(total, min_slice, max_slices, None, None, 0)
        off = np.zeros(n, np.uint64)
        ln = np.zeros(n, np.uint64)
        self.lib.so_decompose(total, min_slice, max_slices, _ptr(off), _ptr(ln), n)
        return off, ln

    def replay(self, sc, rc, bw, tier, id_rank, cand_stream, events):
        return _replay_common(self.lib.so_replay_flat, None, sc, rc, bw, tier, id_rank, cand_stream, events)

    def fill(self, n, seed) -> np.ndarray:
        a = np.zeros(n, np.uint8)
        self.lib.so_fill_pattern(_ptr(a), n, seed)
        return a

    def checksum(self, a: np.ndarray) -> int:
        a = np.ascontiguousarray(a).view(np.uint8)
        return int(self.lib.so_checksum(_ptr(a), a.nbytes))


def _replay_common(fn, topo, sc, rc, bw, tier, id_rank, cand_stream, events):
    events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    cand = np.ascontiguousarray(cand_stream, dtype=np.int32)
    n_rails = len(bw)
    ndec_cap = int((events["kind"] == EV_DECIDE).sum())
    dec = np.zeros(max(ndec_cap, 1), DECISION_DTYPE)
    nd = C.c_size_t()
    bad = C.c_uint64()
    queued = np.zeros(n_rails, np.int64)
    beta = np.zeros(2 * n_rails, np.float64)
    health = np.zeros(n_rails, np.int32)
    if topo is None:
        bw = np.ascontiguousarray(bw, np.float64)
        tier = np.ascontiguousarray(tier, np.int32)
        id_rank = np.ascontiguousarray(id_rank, np.uint32)
        rcode = fn(C.byref(sc), C.byref(rc), C.c_uint32(n_rails), _ptr(bw), _ptr(tier), _ptr(id_rank),
                   _ptr(cand), C.c_size_t(cand.size), _ptr(events), C.c_size_t(events.size),
                   _ptr(dec), C.c_size_t(dec.size), C.byref(nd), C.byref(bad),
                   _ptr(queued), _ptr(beta), _ptr(health))
    else:
        rcode = fn(topo.encode(), C.byref(sc), C.byref(rc), _ptr(cand), C.c_size_t(cand.size),
                   _ptr(events), C.c_size_t(events.size), _ptr(dec), C.c_size_t(dec.size),
                   C.byref(nd), C.byref(bad), _ptr(queued), _ptr(beta), _ptr(health))
    if rcode != 0:
        raise RuntimeError(f"replay failed rc={rcode}")
    return {"decisions": dec[: nd.value], "expect_failures": bad.value, "queued": queued,
            "beta": beta.reshape(-1, 2), "health": health}


REF_SO = os.path.join(HERE, "_ref", "libspray_ref.so")


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefOracle:
    """The reference library itself (oracle/_ref)."""

    def __init__(self):
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        self.lib = C.CDLL(REF_SO)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_cpu_kv_batch.restype = C.c_double
        L.ref_cpu_kv_batch.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64,
                                       C.c_int, C.POINTER(C.c_uint64)]

    def err(self):
        return self.lib.ref_last_error().decode()

    def decompose(self, total, min_slice=65536, max_slices=4096):
        n = C.c_uint64()
        self.lib.ref_decompose(C.c_uint64(total), C.c_uint64(min_slice), C.c_uint32(max_slices),
                               None, None, C.c_uint64(0), C.byref(n))
        off = np.zeros(n.value, np.uint64)
        ln = np.zeros(n.value, np.uint64)
        self.lib.ref_decompose(C.c_uint64(total), C.c_uint64(min_slice), C.c_uint32(max_slices),
                               _ptr(off), _ptr(ln), C.c_uint64(n.value), C.byref(n))
        return off, ln

    def rails(self, topo: str):
        cap = 1024
        bw = np.zeros(cap, np.float64)
        tier = np.zeros(cap, np.int32)
        rank = np.zeros(cap, np.uint32)
        n = C.c_uint32()
        ids = C.create_string_buffer(1 << 16)
        rc = self.lib.ref_rails(topo.encode(), _ptr(bw), _ptr(tier), _ptr(rank), C.c_uint32(cap),
                                C.byref(n), ids, C.c_size_t(1 << 16))
        if rc != 0:
            raise RuntimeError(self.err())
        k = n.value
        return bw[:k].copy(), tier[:k].copy(), rank[:k].copy(), ids.value.decode().split("\n")[:k]

    def candidates(self, topo, caps_list, src, dst, direction, sc):
        """src/dst = (node, medium, device). Returns (stream, backend, n_routes) or raises."""
        arr = (BackendCaps * len(caps_list))(*caps_list)
        cap = 1 << 16
        stream = np.zeros(cap, np.int32)
        ln = C.c_size_t()
        be = C.create_string_buffer(64)
        nr = C.c_uint32()
        rc = self.lib.ref_build_candidates(
            topo.encode(), arr, C.c_uint32(len(caps_list)), src[0].encode(), C.c_int(src[1]),
            (src[2] or "").encode(), dst[0].encode(), C.c_int(dst[1]), (dst[2] or "").encode(),
            C.c_int(direction), C.byref(sc), _ptr(stream), C.c_size_t(cap), C.byref(ln), be,
            C.c_size_t(64), C.byref(nr))
        if rc != 0:
            raise RuntimeError(f"rc={rc}: {self.err()}")
        return stream[: ln.value].copy(), be.value.decode(), nr.value

    def replay(self, topo, sc, rc, cand_stream, events, n_rails):
        return _replay_common(self.lib.ref_replay, topo, sc, rc, [0.0] * n_rails, None, None,
                              cand_stream, events)

    def sim_one(self, topo, length, degrade=1.0):
        out = C.c_uint64()
        rc = self.lib.ref_sim_one(topo.encode(), C.c_uint64(length), C.c_double(degrade), C.byref(out))
        if rc != 0:
            raise RuntimeError(self.err())
        return out.value

    def engine_sim_transfer(self, topo, nbytes, seed, n_rails):
        dst = np.zeros(nbytes, np.uint8)
        ok = np.zeros(n_rails, np.uint64)
        rc = self.lib.ref_engine_sim_transfer(topo.encode(), C.c_uint64(nbytes), C.c_uint64(seed),
                                              _ptr(dst), _ptr(ok), C.c_uint32(n_rails))
        if rc != 0:
            raise RuntimeError(self.err())
        return dst, ok

    def cpu_kv_batch(self, rails, workers, block, n_blocks, seed, iters):
        ok = C.c_uint64()
        t = self.lib.ref_cpu_kv_batch(rails, workers, block, n_blocks, seed, iters, C.byref(ok))
        if t < 0:
            raise RuntimeError(self.err())
        return t, bool(ok.value)


class CState:
    """Incremental C-oracle scheduler state (so_state_*), for trace generators."""

    def __init__(self, oracle: COracle, sc, rc, bw, tier, id_rank, cand_stream):
        L = oracle.lib
        L.so_state_new.restype = C.c_void_p
        L.so_state_free.argtypes = [C.c_void_p]
        self.L = L
        self.n_rails = len(bw)
        self._keep = [np.ascontiguousarray(bw, np.float64), np.ascontiguousarray(tier, np.int32),
                      np.ascontiguousarray(id_rank, np.uint32), np.ascontiguousarray(cand_stream, np.int32)]
        bw_, tier_, rank_, cand_ = self._keep
        self.sc, self.rc = sc, rc
        self.h = L.so_state_new(C.byref(sc), C.byref(rc), C.c_uint32(self.n_rails), _ptr(bw_),
                                _ptr(tier_), _ptr(rank_), _ptr(cand_), C.c_size_t(cand_.size))
        if not self.h:
            raise RuntimeError("so_state_new failed")

    def step(self, events):
        events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        n = int((events["kind"] == EV_DECIDE).sum())
        dec = np.zeros(max(n, 1), DECISION_DTYPE)
        nd = C.c_size_t()
        bad = C.c_uint64()
        queued = np.zeros(self.n_rails, np.int64)
        beta = np.zeros(2 * self.n_rails)
        health = np.zeros(self.n_rails, np.int32)
        rc = self.L.so_state_step(C.c_void_p(self.h), _ptr(events), C.c_size_t(events.size), _ptr(dec),
                                  C.c_size_t(dec.size), C.byref(nd), C.byref(bad), _ptr(queued),
                                  _ptr(beta), _ptr(health))
        if rc != 0:
            raise RuntimeError("so_state_step failed")
        return dec[: nd.value], queued, beta.reshape(-1, 2), health, bad.value

    def __del__(self):
        if getattr(self, "h", None):
            self.L.so_state_free(C.c_void_p(self.h))
            self.h = None
