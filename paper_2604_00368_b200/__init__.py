"""B200-native slice-spraying data plane (TENT, arXiv 2604.00368) behind the reference's
declarative transfer-intent API and fabric plugin boundary.

The product is libspray_b200.so (C++ host + sm_100a CUDA); this package is its Python
binding. Importing it without the built library raises ImportError: there is no CPU path.
"""
from .engine import (BatchState, BatchStatus, BufferDesc, CapabilityError, CompletionEvent,  # noqa: F401
                     ConfigError, CudaBackend, CudaError, Direction, Engine, EngineError, FaultEffect, Health,
                     InvalidRangeError, Medium, NoRouteError, PostResult, Prepared, RailStats, Requests,
                     SegmentDescriptor,
                     SliceWorkRequest, StagedRoute, TransferRequest, checksum, fill_splitmix, hash128, host_alloc, host_free, rr_copy,
                     IPC_HANDLE_BYTES, NumaHostBuffer, board_bytes, device_numa_node, ipc_close, ipc_export,
                     ipc_open)
from . import fabrics  # noqa: F401

__all__ = ["Engine", "CudaBackend", "TransferRequest", "SegmentDescriptor", "BufferDesc", "Direction", "Medium",
           "BatchState", "BatchStatus", "ConfigError", "EngineError", "InvalidRangeError", "NoRouteError",
           "fabrics"]
