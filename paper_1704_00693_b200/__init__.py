"""B200-native lazy stencil-chain executor (arXiv 1704.00693 hot path).

The reference's Runtime front door (par_loop / flush / fetch_reduction / get /
put) over device-resident fp64 fields, a run-time skewed-tile planner and
sm_100a CUDA executors. See DESIGN.md.
"""
from . import kernels
from .runtime import (AccessError, AccessMode, ArgSpec, CudaError, ExecMode, InvalidArgument, KernelHandle,
                      PlanError, Range, ReduceOp, Runtime, RuntimeConfig, SizerError, TcgError, auto_tile_size,
                      body_known, comm_unique_id, device_info, load_library, parse_report, parse_schedule, LIB_PATH)

__all__ = ["kernels", "AccessError", "AccessMode", "ArgSpec", "CudaError", "ExecMode", "InvalidArgument",
           "KernelHandle", "PlanError", "Range", "ReduceOp", "Runtime", "RuntimeConfig", "SizerError", "TcgError",
           "auto_tile_size", "body_known", "comm_unique_id", "device_info", "load_library", "parse_report", "parse_schedule", "LIB_PATH"]
