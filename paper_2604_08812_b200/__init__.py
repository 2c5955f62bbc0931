"""B200-native greedy D-optimal sensor selection (arXiv 2604.08812 hot path).

Product = libdsel.so (sm_100a CUDA + NCCL) behind the C ABI include/dsel.h.
This package is the thin host mirror of the reference selection interface.
"""
from ._abi import LIB_PATH, lib  # noqa: F401  (raises ImportError if the library is missing)
from .selector import (CorruptFile, DselError, Engine, IoError, GpuOptions, IndexOutOfRange,  # noqa: F401
                       LtiProblem,
                       InfeasibleRound, InvalidConfig, ParallelRunReport, SelectionState,
                       SelectionTrace, TraceRow, WorkerFailure, gpu_greedy_select,
                       alloc_count, batched_logdet, fold_records, measure_fp64_peak, nccl_unique_id, synthetic_v)

__all__ = ["Engine", "LtiProblem", "GpuOptions", "gpu_greedy_select", "synthetic_v", "nccl_unique_id", "fold_records", "alloc_count", "batched_logdet", "measure_fp64_peak",
           "DselError", "IoError", "CorruptFile", "InvalidConfig", "IndexOutOfRange", "InfeasibleRound", "WorkerFailure",
           "SelectionState", "SelectionTrace", "ParallelRunReport", "TraceRow", "LIB_PATH"]
