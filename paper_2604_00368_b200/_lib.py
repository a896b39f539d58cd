"""ctypes binding of libspray_b200.so (include/spray_b200.h). Loads the in-tree build and
fails loudly when it is missing: there is no CPU fallback for any entry point."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libspray_b200.so")

if not os.path.exists(SO_PATH):
    raise ImportError(f"{SO_PATH} is not built: run `python -m paper_2604_00368_b200.build` "
                      "(the B200 data plane has no CPU fallback)")

lib = C.CDLL(SO_PATH)


class SchedConfig(C.Structure):
    _fields_ = [("min_slice_size", C.c_uint64), ("max_slices_per_transfer", C.c_uint32),
                ("policy", C.c_int32), ("tolerance", C.c_double), ("penalty", C.c_double * 3),
                ("ewma_alpha", C.c_double), ("reset_interval_ns", C.c_uint64),
                ("beta0_init_s", C.c_double), ("beta1_init", C.c_double), ("feedback_clamp", C.c_double),
                ("diffusion_weight", C.c_double)]


class ResConfig(C.Structure):
    _fields_ = [("failure_threshold", C.c_int32), ("degradation_events", C.c_int32),
                ("degradation_ratio", C.c_double), ("degradation_min_t_obs_s", C.c_double),
                ("probe_successes_needed", C.c_int32), ("probe_backoff_cap", C.c_int32),
                ("probe_bytes", C.c_uint64), ("probe_interval_ns", C.c_uint64),
                ("probe_backoff_mult", C.c_double), ("max_attempts", C.c_uint32),
                ("pad_", C.c_uint32), ("slice_timeout_ns", C.c_uint64)]


class BufferDescC(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("length", C.c_uint64), ("data", C.c_void_p)]


class SegmentDescC(C.Structure):
    _fields_ = [("id", C.c_char_p), ("medium", C.c_int32), ("node", C.c_char_p),
                ("buffers", C.POINTER(BufferDescC)), ("n_buffers", C.c_uint32), ("device", C.c_char_p)]


class TransferRequestC(C.Structure):
    _fields_ = [("src_segment", C.c_char_p), ("src_offset", C.c_uint64), ("dst_segment", C.c_char_p),
                ("dst_offset", C.c_uint64), ("length", C.c_uint64), ("direction", C.c_int32)]


class FaultEntryC(C.Structure):  # spray_fault_entry (FaultEntry, backend.hpp:79-86)
    _fields_ = [("rail_id", C.c_char_p), ("effect", C.c_int32), ("start_ns", C.c_uint64), ("end_ns", C.c_uint64),
                ("factor", C.c_double), ("jitter_us", C.c_double)]


class BatchStatusC(C.Structure):
    _fields_ = [("state", C.c_int32), ("remaining", C.c_uint64), ("failure_reason", C.c_char * 64)]


class RailStatsC(C.Structure):
    _fields_ = [("bytes_posted", C.c_uint64), ("bytes_ok", C.c_uint64), ("bytes_failed", C.c_uint64),
                ("queue_depth", C.c_int64), ("beta0", C.c_double), ("beta1", C.c_double),
                ("health", C.c_int32), ("latency_hist", C.c_uint32 * 48)]


class SliceWR(C.Structure):
    _fields_ = [("slice", C.c_uint64), ("batch", C.c_uint64), ("src_seg_lo", C.c_uint64),
                ("src_seg_hi", C.c_uint64), ("src_offset", C.c_uint64), ("dst_seg_lo", C.c_uint64),
                ("dst_seg_hi", C.c_uint64), ("dst_offset", C.c_uint64), ("length", C.c_uint64),
                ("direction", C.c_int32), ("local_rail", C.c_uint32), ("remote_rail", C.c_uint32),
                ("attempt", C.c_uint32)]


class CQE(C.Structure):
    _fields_ = [("slice", C.c_uint64), ("batch", C.c_uint64), ("status", C.c_int32), ("rail", C.c_uint32),
                ("t_obs_ns", C.c_uint64), ("bytes", C.c_uint64)]


class BackendCaps(C.Structure):
    _fields_ = [("id", C.c_char * 32), ("media_pairs_mask", C.c_uint32), ("supports_read", C.c_uint8),
                ("supports_write", C.c_uint8), ("cross_node", C.c_uint8), ("same_node", C.c_uint8),
                ("max_post_size", C.c_uint64), ("batched_posting", C.c_uint8), ("pad_", C.c_uint8 * 7)]


assert C.sizeof(SliceWR) == 88 and C.sizeof(CQE) == 40

P = C.c_void_p
VP = C.POINTER(C.c_void_p)
U64P = C.POINTER(C.c_uint64)
SZP = C.POINTER(C.c_size_t)

_SIGS = {
    "spray_last_error": (C.c_char_p, []),
    "spray_abi_version": (C.c_uint32, []),
    "spray_sched_config_default": (None, [C.POINTER(SchedConfig)]),
    "spray_resilience_config_default": (None, [C.POINTER(ResConfig)]),
    "spray_engine_create": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, VP]),
    "spray_engine_destroy": (None, [P]),
    "spray_engine_start": (C.c_int, [P]),
    "spray_engine_stop": (C.c_int, [P]),
    "spray_register_segment": (C.c_int, [P, C.POINTER(SegmentDescC)]),
    "spray_allocate_batch": (C.c_int, [P, U64P]),
    "spray_submit_transfer": (C.c_int, [P, C.c_uint64, C.POINTER(TransferRequestC), U64P]),
    "spray_submit_transfers": (C.c_int, [P, C.c_uint64, C.POINTER(TransferRequestC), C.c_size_t, U64P, SZP]),
    "spray_batch_status": (C.c_int, [P, C.c_uint64, C.POINTER(BatchStatusC)]),
    "spray_await_batch": (C.c_int, [P, C.c_uint64, C.c_uint64, C.POINTER(BatchStatusC)]),
    "spray_free_batch": (C.c_int, [P, C.c_uint64]),
    "spray_batch_latency": (C.c_int, [P, C.POINTER(TransferRequestC), C.c_size_t, C.c_size_t, C.c_size_t, U64P]),
    "spray_rail_count": (C.c_int, [P, C.POINTER(C.c_uint32)]),
    "spray_rail_id": (C.c_int, [P, C.c_uint32, C.c_char_p, C.c_size_t]),
    "spray_rail_stats_get": (C.c_int, [P, C.c_uint32, C.POINTER(RailStatsC)]),
    "spray_engine_counters": (C.c_int, [P, U64P, U64P, U64P]),
    "spray_inject_fault": (C.c_int, [P, C.c_char_p, C.c_int32, C.c_uint64, C.c_uint64, C.c_double]),
    "spray_inject_fault_entry": (C.c_int, [P, C.POINTER(FaultEntryC)]),
    "spray_clear_faults": (C.c_int, [P]),
    "spray_engine_now_ns": (C.c_uint64, [P]),
    "spray_heal_stats": (C.c_int, [P, U64P, U64P, U64P, U64P]),
    "spray_gate_segment": (C.c_int, [P, C.c_char_p, C.c_int, P]),
    "spray_gate_ring": (C.c_int, [P, C.c_char_p, C.c_int, P, P, C.c_uint64]),
    "spray_engine_chunk_bytes": (C.c_int, [P, U64P]),
    "spray_board_bytes": (C.c_size_t, [C.c_uint32]),
    "spray_engine_attach_board": (C.c_int, [P, P, C.c_uint32, C.c_uint32, C.c_uint64]),
    "spray_telemetry_csv": (C.c_int, [P, C.c_char_p, C.c_size_t, SZP]),
    "spray_engine_debug": (C.c_int, [P, U64P, C.c_size_t]),
    "spray_trace_enable": (C.c_int, [P, C.c_size_t]),
    "spray_trace_fetch": (C.c_int, [P, P, C.c_size_t, SZP, P, C.c_size_t, SZP]),
    "spray_trace_candidates": (C.c_int, [P, P, C.c_size_t, SZP]),
    "spray_plan_candidates": (C.c_int, [P, C.c_char_p, C.c_char_p, C.c_int32, P, C.c_size_t, SZP,
                                        C.c_char_p, C.c_size_t]),
    "spray_prepare_transfers": (C.c_int, [P, C.POINTER(TransferRequestC), C.c_size_t, VP]),
    "spray_run_prepared": (C.c_int, [P, C.c_uint64, P, C.POINTER(C.c_float)]),
    "spray_prepared_free": (None, [P]),
    "spray_replay_device": (C.c_int, [C.c_int, C.POINTER(SchedConfig), C.POINTER(ResConfig), C.c_uint32,
                                      P, P, P, P, C.c_size_t, P, C.c_size_t, P, C.c_size_t, SZP, U64P]),
    "spray_fill_splitmix": (C.c_int, [C.c_int, P, C.c_uint64, C.c_uint64]),
    "spray_checksum": (C.c_int, [C.c_int, P, C.c_uint64, U64P]),
    "spray_host_alloc": (C.c_int, [C.c_uint64, VP]),
    "spray_host_free": (C.c_int, [P]),
    "spray_device_numa_node": (C.c_int, [C.c_int, C.POINTER(C.c_int32)]),
    "spray_host_alloc_numa": (C.c_int, [C.c_int, C.c_uint64, VP, C.POINTER(C.c_int32)]),
    "spray_host_free_numa": (C.c_int, [P]),
    "spray_rr_copy": (C.c_int, [C.c_int, U64P, U64P, U64P, C.c_size_t, C.c_int, C.POINTER(C.c_double)]),
    "spray_ipc_export": (C.c_int, [C.c_int, P, P]),
    "spray_ipc_open": (C.c_int, [C.c_int, P, VP]),
    "spray_ipc_close": (C.c_int, [P]),
    "spray_backend_open": (C.c_int, [C.c_int, VP]),
    "spray_backend_close": (None, [P]),
    "spray_backend_start": (C.c_int, [P]),
    "spray_backend_stop": (C.c_int, [P]),
    "spray_backend_capabilities": (C.c_int, [P, C.POINTER(BackendCaps)]),
    "spray_backend_attach_segment": (C.c_int, [P, C.POINTER(SegmentDescC), P, C.c_size_t, SZP]),
    "spray_backend_post": (C.c_int, [P, C.POINTER(SliceWR), C.c_size_t, SZP]),
    "spray_backend_poll": (C.c_int, [P, C.POINTER(CQE), C.c_size_t, SZP]),
    "spray_backend_fatal": (C.c_int, [P]),
    "spray_backend_latch_fatal": (C.c_int, [P]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)
