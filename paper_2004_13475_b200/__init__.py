"""B200-native λ(ω) block-space thread map for the embedded Sierpinski gasket.

A drop-in for the reference's dispatch engine (arXiv 2004.13475 artifact,
/root/reference/proj): the same workloads (single write, reduction, cellular
automaton) launched either over the bounding box or over the compact λ(ω)
orthotope, computed by hand-written sm_100a kernels behind the C ABI in
include/nbb_gpu.h. See DESIGN.md.
"""
from .nbb import (CaResult, CaRule, CompactGrid, CudaError, DispatchConfig, DomainError, FractalSpec, Grid,
                  IntraBlockStrategy, InvalidArgument, KernelFamily, LambdaBackend, MapMode,
                  NbbError, OutOfRange, ReductionResult, ResourceError, SingleWriteResult,
                  WorkReport, backend_from_string, compact_load, compact_store, device_count,
                  lambda_coords, lambda_inverse, read_compact, write_compact,
                  launch_block_count, mode_from_string, plan_report, random_member_grid,
                  random_member_values, release, run_ca, run_reduction, run_single_write,
                  strategy_from_string, to_string, work_quotient)

__all__ = [
    "CaResult", "CaRule", "CompactGrid", "CudaError", "DispatchConfig", "DomainError", "FractalSpec", "Grid",
    "IntraBlockStrategy", "InvalidArgument", "KernelFamily", "LambdaBackend", "MapMode",
    "NbbError", "OutOfRange", "ReductionResult", "ResourceError", "SingleWriteResult",
    "WorkReport", "backend_from_string", "compact_load", "compact_store", "device_count",
    "lambda_coords", "lambda_inverse", "read_compact", "write_compact", "launch_block_count",
    "mode_from_string", "plan_report", "random_member_grid", "random_member_values", "release",
    "run_ca", "run_reduction", "run_single_write", "strategy_from_string", "to_string",
    "work_quotient",
]
