"""Host-side mirror of the reference interface for the slice-spraying path.

Same names, argument meaning and error behaviour as proj/include/spray/engine.hpp:90-131
(Engine), proj/include/spray/backend.hpp:49-72 (TransportBackend) and
proj/include/spray/common.hpp:31-41 (error classes). Every call goes through the C-ABI
of libspray_b200.so; nothing here moves bytes or makes scheduling decisions.
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L

lib = L.lib


# ------------------------------------------------------------------ errors (common.hpp:31-41)
class SprayError(RuntimeError):
    pass


class ConfigError(SprayError):
    pass


class EngineError(SprayError):
    pass


class InvalidRangeError(EngineError):
    pass


class NoRouteError(EngineError):
    pass


class CudaError(SprayError):
    pass


class BackendFatal(EngineError):
    pass


class CapabilityError(EngineError):
    pass


_ERRS = {-1: ConfigError, -2: EngineError, -3: InvalidRangeError, -4: NoRouteError, -5: CudaError,
         -6: BackendFatal, -7: CapabilityError}


def _check(rc: int):
    if rc != 0:
        msg = lib.spray_last_error().decode(errors="replace")
        raise _ERRS.get(rc, SprayError)(msg)


# ------------------------------------------------------------------ enums / records
class Direction(enum.IntEnum):
    READ = 0
    WRITE = 1


class Medium(enum.IntEnum):
    HOST = 0
    DEVICE = 1
    FILE = 2


class BatchState(enum.IntEnum):
    IN_FLIGHT = 0
    COMPLETE = 1
    FAILED = 2


class Health(enum.IntEnum):
    HEALTHY = 0
    EXCLUDED = 1
    PROBING = 2


class FaultEffect(enum.IntEnum):
    DOWN = 0
    DEGRADE = 1
    JITTER = 2
    DROP_COMPLETION = 3


@dataclass
class BufferDesc:
    offset: int
    length: int
    data: int  # device pointer (DEVICE) or pinned host pointer (HOST)


@dataclass
class SegmentDescriptor:
    id: str
    medium: Medium
    node: str
    buffers: List[BufferDesc]
    device: str = ""


@dataclass
class TransferRequest:
    src_segment: str
    src_offset: int
    dst_segment: str
    dst_offset: int
    length: int
    direction: Direction = Direction.WRITE


@dataclass
class BatchStatus:
    state: BatchState
    remaining: int
    failure_reason: str = ""


@dataclass
class RailStats:
    rail_id: str
    bytes_posted: int
    bytes_ok: int
    bytes_failed: int
    queue_depth: int
    beta0: float
    beta1: float
    health: Health
    latency_hist: List[int] = field(default_factory=list)


def _seg_c(d: SegmentDescriptor):
    bufs = (L.BufferDescC * len(d.buffers))(*[L.BufferDescC(b.offset, b.length, b.data) for b in d.buffers])
    s = L.SegmentDescC(d.id.encode(), int(d.medium), d.node.encode(), bufs, len(d.buffers),
                       (d.device or "").encode())
    return s, bufs


def _req_c(r: TransferRequest):
    return L.TransferRequestC(r.src_segment.encode(), r.src_offset, r.dst_segment.encode(), r.dst_offset,
                              r.length, int(r.direction))


def _reqs_c(reqs: Sequence[TransferRequest]):
    keep = []
    arr = (L.TransferRequestC * len(reqs))()
    for i, r in enumerate(reqs):
        s, d = r.src_segment.encode(), r.dst_segment.encode()
        keep += [s, d]
        arr[i] = L.TransferRequestC(s, r.src_offset, d, r.dst_offset, r.length, int(r.direction))
    return arr, keep


class Requests:
    """A request list marshalled once into the C-ABI's spray_transfer_request array, for
    callers that resubmit the same block table (the C-ABI call then takes host arrays
    directly, as a C++ or cgo caller would)."""

    def __init__(self, reqs: Sequence[TransferRequest]):
        self.arr, self._keep = _reqs_c(reqs)
        self.n = len(reqs)

    def __len__(self):
        return self.n


def _status(st: L.BatchStatusC) -> BatchStatus:
    return BatchStatus(BatchState(st.state), int(st.remaining), st.failure_reason.decode())


# ------------------------------------------------------------------ Engine
class Engine:
    """spray::Engine (engine.hpp:90-131) on one B200. `topology` is the reference JSON
    topology document; `config` the engine config document (unknown keys rejected)."""

    def __init__(self, topology: str, config: Optional[str] = None, device: int = 0):
        h = C.c_void_p()
        _check(lib.spray_engine_create(config.encode() if config else None, topology.encode(), device,
                                       C.byref(h)))
        self._h = h
        self.device = device
        self._keep = []

    def close(self):
        if getattr(self, "_h", None):
            lib.spray_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        self.start()
        return self

    def __exit__(self, *exc):
        self.stop()
        self.close()

    def start(self):
        _check(lib.spray_engine_start(self._h))

    def stop(self):
        _check(lib.spray_engine_stop(self._h))

    def register_segment(self, desc: SegmentDescriptor):
        s, bufs = _seg_c(desc)
        _check(lib.spray_register_segment(self._h, C.byref(s)))

    def allocate_batch(self) -> int:
        b = C.c_uint64()
        _check(lib.spray_allocate_batch(self._h, C.byref(b)))
        return b.value

    def submit_transfer(self, batch: int, req: TransferRequest) -> int:
        r = _req_c(req)
        t = C.c_uint64()
        _check(lib.spray_submit_transfer(self._h, batch, C.byref(r), C.byref(t)))
        return t.value

    def submit_transfers(self, batch: int, reqs) -> List[int]:
        """`reqs`: a sequence of TransferRequest, or a prebuilt Requests array."""
        if isinstance(reqs, Requests):
            arr = reqs.arr
        else:
            arr, keep = _reqs_c(reqs)
        n = len(reqs)
        ids = (C.c_uint64 * max(1, n))()
        done = C.c_size_t()
        _check(lib.spray_submit_transfers(self._h, batch, arr, n, ids, C.byref(done)))
        return list(ids[: done.value])

    def batch_status(self, batch: int) -> BatchStatus:
        st = L.BatchStatusC()
        _check(lib.spray_batch_status(self._h, batch, C.byref(st)))
        return _status(st)

    def await_batch(self, batch: int, limit_ns: int = 120_000_000_000) -> BatchStatus:
        st = L.BatchStatusC()
        _check(lib.spray_await_batch(self._h, batch, limit_ns, C.byref(st)))
        return _status(st)

    def free_batch(self, batch: int):
        _check(lib.spray_free_batch(self._h, batch))

    # ---- device-resident submission
    def batch_latency_ns(self, reqs, per_batch: int, n_batches: int) -> np.ndarray:
        """Per-batch submit -> terminal latency (ns) of n_batches rounds of allocate / submit
        (per_batch requests) / await / free, timed in C++ (spray_batch_latency)."""
        r = reqs if isinstance(reqs, Requests) else Requests(reqs)
        out = np.zeros(n_batches, dtype=np.uint64)
        _check(lib.spray_batch_latency(self._h, r.arr, len(r), per_batch, n_batches,
                                       out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    def prepare_transfers(self, reqs: Sequence[TransferRequest]) -> "Prepared":
        arr, keep = _reqs_c(reqs)
        p = C.c_void_p()
        _check(lib.spray_prepare_transfers(self._h, arr, len(reqs), C.byref(p)))
        return Prepared(self, p)

    # ---- introspection
    def rail_count(self) -> int:
        n = C.c_uint32()
        _check(lib.spray_rail_count(self._h, C.byref(n)))
        return n.value

    def rail_id(self, r: int) -> str:
        buf = C.create_string_buffer(256)
        _check(lib.spray_rail_id(self._h, r, buf, 256))
        return buf.value.decode()

    def rail_stats(self, r: int) -> RailStats:
        s = L.RailStatsC()
        _check(lib.spray_rail_stats_get(self._h, r, C.byref(s)))
        return RailStats(self.rail_id(r), s.bytes_posted, s.bytes_ok, s.bytes_failed, s.queue_depth, s.beta0,
                         s.beta1, Health(s.health), list(s.latency_hist))

    def counters(self):
        d, t, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib.spray_engine_counters(self._h, C.byref(d), C.byref(t), C.byref(f)))
        return {"bytes_dispatched": d.value, "bytes_terminated": t.value, "batches_failed": f.value}

    def inject_fault(self, rail_id: str, effect: FaultEffect, start_ns: int, end_ns: int, factor: float = 1.0,
                     jitter_us: float = 0.0):
        """One FaultEntry (backend.hpp:79-86): DOWN, DEGRADE (factor), JITTER (jitter_us) or
        DROP_COMPLETION on `rail_id` over [start_ns, end_ns) of the engine clock."""
        fe = L.FaultEntryC(rail_id.encode(), int(effect), int(start_ns), int(end_ns), float(factor), float(jitter_us))
        _check(lib.spray_inject_fault_entry(self._h, C.byref(fe)))

    def clear_faults(self):
        _check(lib.spray_clear_faults(self._h))

    def now_ns(self) -> int:
        return int(lib.spray_engine_now_ns(self._h))

    # ---- dataflow gates (forwarding / relays / broadcast chains)
    GATE_CONSUME, GATE_PRODUCE = 1, 2

    def attach_board(self, board_ptr: int, n_slots: int, slot: int, period_ns: int = 10_000_000):
        """GlobalLoadBoard (scheduler.hpp:66-90): publish this engine's per-rail queued bytes
        into `slot` of a zeroed host board of board_bytes(n_slots) bytes every period and
        blend the fresh entries in with scheduler.diffusion_weight."""
        _check(lib.spray_engine_attach_board(self._h, board_ptr, n_slots, slot, period_ns))

    def gate_segment(self, segment_id: str, role: int, flags_ptr: int):
        """Gate a registered single-buffer segment: `flags_ptr` points at one zeroed uint32
        counter per chunk_bytes() granule, shared by the producing and consuming engines."""
        _check(lib.spray_gate_segment(self._h, segment_id.encode(), int(role), flags_ptr))

    def gate_ring(self, segment_id: str, role: int, flags_ptr: int, credits_ptr: int, logical_bytes: int):
        """Ring gate (the staged route's bounded staging pool, engine.hpp:56-58): the
        segment's single buffer is a ring that intents address through a logical window of
        `logical_bytes` (lap = offset // ring). `flags_ptr` / `credits_ptr`: one zeroed uint32
        per granule each, shared by both engines. See spray_gate_ring in include/spray_b200.h."""
        _check(lib.spray_gate_ring(self._h, segment_id.encode(), int(role), flags_ptr, credits_ptr,
                                   int(logical_bytes)))

    def telemetry_csv(self) -> str:
        """TelemetrySnapshot::to_csv columns from the device telemetry windows."""
        n = C.c_size_t()
        _check(lib.spray_telemetry_csv(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib.spray_telemetry_csv(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def chunk_bytes(self) -> int:
        v = C.c_uint64()
        _check(lib.spray_engine_chunk_bytes(self._h, C.byref(v)))
        return v.value

    def heal_stats(self):
        a, b, c, d = (C.c_uint64() for _ in range(4))
        _check(lib.spray_heal_stats(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return {"fault_start_ns": a.value, "first_reroute_ok_ns": b.value, "failed_attempts": c.value,
                "retried_ok": d.value}

    # ---- trace (slice-plan parity)
    def trace_enable(self, capacity: int = 1 << 20):
        _check(lib.spray_trace_enable(self._h, capacity))

    def trace_fetch(self, cap: int = 1 << 20):
        from .trace import EVENT_DTYPE, DECISION_DTYPE
        ev = np.zeros(cap, EVENT_DTYPE)
        dec = np.zeros(cap, DECISION_DTYPE)
        n, nd = C.c_size_t(), C.c_size_t()
        _check(lib.spray_trace_fetch(self._h, ev.ctypes.data, cap, C.byref(n), dec.ctypes.data, cap,
                                     C.byref(nd)))
        if n.value > cap or nd.value > cap:
            raise EngineError(f"trace overflow: {n.value} events / {nd.value} decisions > capacity {cap}")
        return ev[: n.value].copy(), dec[: nd.value].copy()

    def trace_candidates(self) -> np.ndarray:
        n = C.c_size_t()
        _check(lib.spray_trace_candidates(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, np.int32)
        _check(lib.spray_trace_candidates(self._h, out.ctypes.data, n.value, C.byref(n)))
        return out

    def plan_candidates(self, src: str, dst: str, direction: Direction = Direction.WRITE):
        n = C.c_size_t()
        b = C.create_string_buffer(64)
        _check(lib.spray_plan_candidates(self._h, src.encode(), dst.encode(), int(direction), None, 0,
                                         C.byref(n), b, 64))
        out = np.zeros(n.value, np.int32)
        _check(lib.spray_plan_candidates(self._h, src.encode(), dst.encode(), int(direction), out.ctypes.data,
                                         n.value, C.byref(n), b, 64))
        return out, b.value.decode()


class Prepared:
    """Intents planned once and staged in HBM; run() submits them into a batch and times
    the drain-mode engine launch with CUDA events on the engine stream."""

    def __init__(self, eng: Engine, h):
        self.eng, self._h = eng, h

    def run(self, batch: int) -> float:
        ms = C.c_float()
        _check(lib.spray_run_prepared(self.eng._h, batch, self._h, C.byref(ms)))
        return ms.value

    def free(self):
        if self._h:
            lib.spray_prepared_free(self._h)
            self._h = None

    def __del__(self):
        self.free()


# ------------------------------------------------------------------ TransportBackend (plugin mode)
@dataclass
class SliceWorkRequest:  # backend.hpp:15-27
    slice: int
    batch: int
    src_segment: str
    src_offset: int
    dst_segment: str
    dst_offset: int
    length: int
    direction: Direction = Direction.WRITE
    local_rail: int = 0
    remote_rail: int = 0xFFFFFFFF
    attempt: int = 0


@dataclass
class CompletionEvent:  # backend.hpp:33-40
    slice: int
    batch: int
    status: int
    rail: int
    t_obs: int
    bytes: int


@dataclass
class PostResult:  # backend.hpp:44-47
    accepted: int
    fatal: bool = False


def hash128(s: str):
    """common.hpp:111-120 two-lane FNV-1a."""
    def fnv(data: bytes, h: int) -> int:
        for b in data:
            h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
        return h
    d = s.encode()
    return fnv(d, 0xCBF29CE484222325), fnv(d, 0x84222325CBF29CE4)


class CudaBackend:
    """TransportBackend over CUDA (the insertion point the reference's load_backends,
    engine.cpp:116-140, would bind as "cuda")."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib.spray_backend_open(device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.spray_backend_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def start(self):
        _check(lib.spray_backend_start(self._h))

    def stop(self):
        _check(lib.spray_backend_stop(self._h))

    def capabilities(self) -> L.BackendCaps:
        c = L.BackendCaps()
        _check(lib.spray_backend_capabilities(self._h, C.byref(c)))
        return c

    def attach_segment_metadata(self, desc: SegmentDescriptor) -> Optional[bytes]:
        s, bufs = _seg_c(desc)
        blob = C.create_string_buffer(256)
        n = C.c_size_t()
        rc = lib.spray_backend_attach_segment(self._h, C.byref(s), blob, 256, C.byref(n))
        if rc == -7:
            return None
        _check(rc)
        return blob.raw[: n.value]

    def post_slices(self, reqs: Sequence[SliceWorkRequest]) -> PostResult:
        arr = (L.SliceWR * len(reqs))()
        for i, r in enumerate(reqs):
            slo, shi = hash128(r.src_segment)
            dlo, dhi = hash128(r.dst_segment)
            arr[i] = L.SliceWR(r.slice, r.batch, slo, shi, r.src_offset, dlo, dhi, r.dst_offset, r.length,
                               int(r.direction), r.local_rail, r.remote_rail, r.attempt)
        acc = C.c_size_t()
        rc = lib.spray_backend_post(self._h, arr, len(reqs), C.byref(acc))
        if rc == -6:
            return PostResult(0, True)
        _check(rc)
        return PostResult(acc.value, False)

    def poll_completions(self, max_events: int = 32) -> List[CompletionEvent]:
        arr = (L.CQE * max_events)()
        n = C.c_size_t()
        _check(lib.spray_backend_poll(self._h, arr, max_events, C.byref(n)))
        return [CompletionEvent(c.slice, c.batch, c.status, c.rail, c.t_obs_ns, c.bytes) for c in arr[: n.value]]

    def fatal(self) -> bool:
        return bool(lib.spray_backend_fatal(self._h))

    def latch_fatal(self):
        lib.spray_backend_latch_fatal(self._h)


# ------------------------------------------------------------------ utilities
def fill_splitmix(device: int, ptr: int, n: int, seed: int):
    """Device fill with the reference payload generator (bench.cpp:59-67)."""
    _check(lib.spray_fill_splitmix(device, ptr, n, seed))


def checksum(device: int, ptr: int, n: int) -> int:
    out = C.c_uint64()
    _check(lib.spray_checksum(device, ptr, n, C.byref(out)))
    return out.value


def rr_copy(device: int, src, dst, lens, streams: int = 4) -> float:
    """State-blind baseline: one cudaMemcpyAsync per range, round-robin over `streams`
    streams (spray_rr_copy). Returns wall milliseconds."""
    import numpy as np
    s = np.ascontiguousarray(src, dtype=np.uint64)
    d = np.ascontiguousarray(dst, dtype=np.uint64)
    n = np.ascontiguousarray(lens, dtype=np.uint64)
    ms = C.c_double()
    U = C.POINTER(C.c_uint64)
    _check(lib.spray_rr_copy(device, s.ctypes.data_as(U), d.ctypes.data_as(U), n.ctypes.data_as(U), len(n), streams,
                             C.byref(ms)))
    return ms.value


def host_alloc(n: int) -> int:
    p = C.c_void_p()
    _check(lib.spray_host_alloc(n, C.byref(p)))
    return p.value


def host_free(p: int):
    _check(lib.spray_host_free(p))


def device_numa_node(device: int) -> int:
    """NUMA node of the GPU's PCIe root (-1 when unknown)."""
    n = C.c_int32()
    _check(lib.spray_device_numa_node(device, C.byref(n)))
    return n.value


class NumaHostBuffer:
    """Pinned, device-mapped host memory on the GPU's own NUMA node (spray_host_alloc_numa):
    the pinned-host staging pool of one PCIe root. `.ptr`, `.node`, and a zero-copy uint8
    `torch` / `numpy` view of the first n bytes."""

    def __init__(self, device: int, n: int):
        p = C.c_void_p()
        node = C.c_int32()
        _check(lib.spray_host_alloc_numa(device, n, C.byref(p), C.byref(node)))
        self.ptr, self.n, self.node = p.value, n, node.value

    def numpy(self):
        return np.ctypeslib.as_array((C.c_uint8 * self.n).from_address(self.ptr))

    def tensor(self):
        import torch
        return torch.from_numpy(self.numpy())

    def free(self):
        if self.ptr:
            _check(lib.spray_host_free_numa(self.ptr))
            self.ptr = 0


def board_bytes(n_slots: int) -> int:
    """Size of a load board with n_slots engine instances (spray_board_bytes)."""
    return int(lib.spray_board_bytes(n_slots))


IPC_HANDLE_BYTES = 72  # SPRAY_IPC_HANDLE_BYTES: CUDA IPC handle + offset inside the allocation


def ipc_export(device: int, ptr: int) -> bytes:
    buf = (C.c_uint8 * IPC_HANDLE_BYTES)()
    _check(lib.spray_ipc_export(device, ptr, buf))
    return bytes(buf)


def ipc_open(device: int, handle: bytes) -> int:
    buf = (C.c_uint8 * IPC_HANDLE_BYTES).from_buffer_copy(handle)
    p = C.c_void_p()
    _check(lib.spray_ipc_open(device, buf, C.byref(p)))
    return p.value


def ipc_close(ptr: int):
    _check(lib.spray_ipc_close(ptr))


class StagedRoute:
    """Staged multi-hop route through a bounded pinned-host staging ring (SURVEY.md §8(f)
    rank 1; reference `build_staged_exec` / `staged_try_start_chunks`, engine.cpp:465-527,
    with `staging_chunk_bytes` 4 MiB and `staging_ring_depth` 4, engine.hpp:56-58).

    The producer engine moves src -> ring and the consumer engine ring -> dst; a ring gate
    (spray_gate_ring) pipelines them granule by granule on the device, so at most
    `depth` chunks of the transfer occupy the pool and the host only writes intents. The
    two engines may sit on different GPUs without peer access: the ring, its flags and
    its credits live in mapped pinned host memory. Register while both engines are idle.
    """

    def __init__(self, producer: "Engine", consumer: "Engine", producer_node: str, consumer_node: str,
                 chunk_bytes: int = 4 << 20, depth: int = 4, seg_id: str = "staged/ring",
                 max_laps: int = 1 << 24):
        cb = producer.chunk_bytes()
        if consumer.chunk_bytes() != cb:
            raise ConfigError("staged route: both engines need the same b200.chunk_bytes")
        if chunk_bytes % cb or depth < 1:
            raise ConfigError("staged route: chunk_bytes must be a multiple of b200.chunk_bytes, depth >= 1")
        self.producer, self.consumer = producer, consumer
        self.seg_id, self.chunk, self.granule = seg_id, chunk_bytes, cb
        self.ring_bytes = chunk_bytes * depth
        granules = self.ring_bytes // cb
        self._ring = host_alloc(self.ring_bytes)
        self._ctl = host_alloc(8 * granules)  # flags then credits, one uint32 per granule each
        C.memset(self._ctl, 0, 8 * granules)
        flags, credits = self._ctl, self._ctl + 4 * granules
        self._credits = np.ctypeslib.as_array((C.c_uint32 * granules).from_address(credits))
        for eng, node in ((producer, producer_node), (consumer, consumer_node)):
            eng.register_segment(SegmentDescriptor(seg_id, Medium.HOST, node,
                                                   [BufferDesc(0, self.ring_bytes, self._ring)]))
        logical = self.ring_bytes * max_laps
        producer.gate_ring(seg_id, Engine.GATE_PRODUCE, flags, credits, logical)
        consumer.gate_ring(seg_id, Engine.GATE_CONSUME, flags, credits, logical)
        self.logical_bytes = logical
        self.cursor = 0  # next logical ring offset (monotonic: the lap is cursor // ring_bytes)
        self.stats = {"wait_s": 0.0, "submit_s": 0.0, "pieces": 0}  # host time of transfer()

    def transfer(self, src_segment: str, src_offset: int, dst_segment: str, dst_offset: int, length: int,
                 timeout_s: float = 60.0) -> BatchState:
        """Move src[src_offset:+length] -> dst[dst_offset:+length] through the ring as
        `chunk_bytes` pieces (the reference's staged chunks): one consumer intent and one
        producer intent per piece. Offsets must be multiples of b200.chunk_bytes. Blocks
        until both ends finish; returns COMPLETE or FAILED.

        Like `staged_try_start_chunks` (engine.cpp:506-527), at most `depth` pieces are
        ahead of the consumer: a piece that reuses a ring slot is queued only once the
        consumer's credits show the slot's previous lap drained (the credits sit in host
        memory, so this poll costs no PCIe traffic). Neither engine's device pipeline then
        holds work that waits on the other side. Pieces go into the engines' batches; a
        batch that drained between two pieces is replaced by a fresh one (a completed
        batch takes no more intents, engine.cpp:239-253)."""
        if length <= 0:
            raise InvalidRangeError("zero-length transfer")
        if self.cursor + length > self.logical_bytes:
            raise InvalidRangeError("staged route: logical ring window exhausted")
        batches = {self.producer: [], self.consumer: []}

        def put(eng, req):
            for _ in range(2):
                if not batches[eng]:
                    batches[eng].append(eng.allocate_batch())
                try:
                    eng.submit_transfer(batches[eng][-1], req)
                    return
                except EngineError as e:
                    if "already complete" not in str(e):
                        raise
                    batches[eng].append(eng.allocate_batch())
            raise EngineError("staged route: could not queue a piece")

        pos = 0
        deadline = time.monotonic() + timeout_s
        while pos < length:
            n = min(self.chunk, length - pos)
            c = self.cursor
            lap, g0 = divmod(c, self.ring_bytes)
            g0 //= self.granule
            ng = -(-n // self.granule)
            t0 = time.perf_counter()
            while lap and int(self._credits[g0:g0 + ng].min()) < lap:
                if time.monotonic() > deadline:
                    raise EngineError("staged route: the consumer did not drain the ring in time")
                time.sleep(10e-6)
            t1 = time.perf_counter()
            put(self.consumer, TransferRequest(self.seg_id, c, dst_segment, dst_offset + pos, n))
            put(self.producer, TransferRequest(src_segment, src_offset + pos, self.seg_id, c, n))
            self.stats["wait_s"] += t1 - t0
            self.stats["submit_s"] += time.perf_counter() - t1
            self.stats["pieces"] += 1
            self.cursor += ng * self.granule
            pos += n
        state = BatchState.COMPLETE
        rem_ns = max(1, int((deadline - time.monotonic()) * 1e9))
        for eng in (self.producer, self.consumer):
            for b in batches[eng]:
                st = eng.await_batch(b, rem_ns)
                if st.state != BatchState.COMPLETE:
                    state = BatchState.FAILED
                eng.free_batch(b)
        return state

    def close(self):
        """Free the ring once both engines are stopped."""
        if self._ring:
            host_free(self._ring)
            host_free(self._ctl)
            self._ring = self._ctl = 0
