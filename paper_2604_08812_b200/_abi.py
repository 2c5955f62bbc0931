"""ctypes mirror of include/dsel.h (the C ABI of libdsel.so).

The product path is libdsel.so: if it is missing this module raises at import
time -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libdsel.so")

DSEL_OK = 0
STATUS_NAMES = {0: "DSEL_OK", 1: "DSEL_E_INVALID", 2: "DSEL_E_RANGE", 3: "DSEL_E_INFEASIBLE",
                4: "DSEL_E_CUDA", 5: "DSEL_E_NCCL", 6: "DSEL_E_OOM", 7: "DSEL_E_IO",
                8: "DSEL_E_STATE", 9: "DSEL_E_CORRUPT"}

# every entry point declared in include/dsel.h (tests check the exports)
EXPORTS = ["dsel_abi_version", "dsel_fold_records", "dsel_nccl_unique_id", "dsel_create", "dsel_destroy",
           "dsel_last_error", "dsel_sync", "dsel_connect", "dsel_abort", "dsel_device_bytes", "dsel_get_plan", "dsel_alloc_count", "dsel_measure_fp64_peak", "dsel_batched_logdet", "dsel_load_block_row",
           "dsel_load_block_col", "dsel_load_k", "dsel_attach_host_k", "dsel_attach_host_rows", "dsel_load_kbf", "dsel_attach_kbf", "dsel_read_block_row", "dsel_synthetic_v",
           "dsel_gen_synthetic", "dsel_gen_synthetic_device", "dsel_lti_from_config", "dsel_lti_free",
           "dsel_assemble_lti", "dsel_step", "dsel_step_forced", "dsel_run", "dsel_peek_gains",
           "dsel_get_trace", "dsel_reset", "dsel_get_stats", "dsel_export_factor",
           "dsel_export_factor_row"]


class DselConfig(C.Structure):
    _fields_ = [("n_sensors", C.c_int), ("n_steps", C.c_int), ("budget", C.c_int),
                ("n_candidates", C.c_int), ("candidates", C.POINTER(C.c_int)),
                ("device", C.c_int), ("world_size", C.c_int), ("rank", C.c_int),
                ("nccl_id", C.c_void_p), ("storage", C.c_int), ("keep_pristine", C.c_int),
                ("export_factor", C.c_int), ("near_tie_tau", C.c_double),
                ("full_square", C.c_int), ("algorithm", C.c_int),
                ("panel_layout", C.c_int), ("hbm_budget", C.c_uint64),
                ("defer_connect", C.c_int)]


class DselPlan(C.Structure):
    _fields_ = [("storage", C.c_int), ("algorithm", C.c_int), ("symmetric", C.c_int),
                ("packed", C.c_int), ("device_bytes", C.c_uint64), ("planned_bytes", C.c_uint64),
                ("budget_bytes", C.c_uint64), ("host_store_bytes", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class DselStepInfo(C.Structure):
    _fields_ = [("k", C.c_int), ("chosen_index", C.c_int), ("gain", C.c_double),
                ("objective", C.c_double), ("runner_up", C.c_int),
                ("runner_up_gain", C.c_double), ("near_tie", C.c_int),
                ("n_evaluated", C.c_int), ("n_infeasible", C.c_int),
                ("bytes_exchanged", C.c_uint64), ("ms_gain", C.c_double),
                ("ms_exchange", C.c_double), ("ms_panel", C.c_double),
                ("ms_update", C.c_double), ("ms_round", C.c_double),
                ("update_flops", C.c_double), ("ms_io", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class DselArgRec(C.Structure):
    _fields_ = [("g1", C.c_double), ("g2", C.c_double), ("s1", C.c_int), ("s2", C.c_int),
                ("n_eval", C.c_int), ("n_inf", C.c_int)]


class DselLti(C.Structure):
    _fields_ = [("n_params", C.c_int), ("n_sensors", C.c_int), ("n_steps", C.c_int),
                ("noise_sigma", C.c_double), ("impulse", C.c_void_p), ("spatial", C.c_void_p),
                ("mask", C.c_void_p), ("cost_weights", C.c_void_p)]


class DselStats(C.Structure):
    _fields_ = [("rounds", C.c_int), ("kernel_launches", C.c_uint64), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("nccl_bytes", C.c_uint64),
                ("time_to_k_ms", C.c_double), ("update_ms", C.c_double),
                ("update_flops", C.c_double), ("io_ms", C.c_double),
                ("io_exposed_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (the selection path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, ip, dp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double)
    L.dsel_abi_version.restype = C.c_int
    L.dsel_nccl_unique_id.argtypes = [vp]
    L.dsel_create.argtypes = [C.POINTER(DselConfig), C.POINTER(vp)]
    L.dsel_destroy.argtypes = [vp]
    L.dsel_destroy.restype = None
    L.dsel_last_error.argtypes = [vp]
    L.dsel_last_error.restype = C.c_char_p
    L.dsel_sync.argtypes = [vp]
    L.dsel_connect.argtypes = [vp]
    L.dsel_abort.argtypes = [vp]
    L.dsel_device_bytes.argtypes = [vp]
    L.dsel_device_bytes.restype = C.c_uint64
    L.dsel_get_plan.argtypes = [vp, C.POINTER(DselPlan)]
    L.dsel_alloc_count.argtypes = []
    L.dsel_alloc_count.restype = C.c_uint64
    L.dsel_measure_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double)]
    L.dsel_batched_logdet.argtypes = [C.c_int, vp, C.c_int, C.c_int64, C.c_int, vp, vp]
    L.dsel_load_block_row.argtypes = [vp, C.c_int, vp]
    L.dsel_load_block_col.argtypes = [vp, C.c_int, vp]
    L.dsel_load_k.argtypes = [vp, vp]
    L.dsel_attach_host_k.argtypes = [vp, vp]
    L.dsel_gen_synthetic_device.argtypes = [vp, C.c_int, C.c_double, C.c_uint64]
    L.dsel_attach_host_rows.argtypes = [vp, vp]
    L.dsel_lti_from_config.argtypes = [C.c_char_p, C.POINTER(DselLti), C.POINTER(vp)]
    L.dsel_lti_free.argtypes = [vp]
    L.dsel_lti_free.restype = None
    L.dsel_assemble_lti.argtypes = [vp, C.POINTER(DselLti), vp]
    L.dsel_load_kbf.argtypes = [vp, C.c_char_p, C.c_int, C.c_int]
    L.dsel_attach_kbf.argtypes = [vp, C.c_char_p, C.c_int]
    L.dsel_read_block_row.argtypes = [vp, C.c_int, vp]
    L.dsel_synthetic_v.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, vp, C.c_int]
    L.dsel_gen_synthetic.argtypes = [vp, vp, C.c_int, C.c_double]
    L.dsel_step.argtypes = [vp, C.POINTER(DselStepInfo)]
    L.dsel_step_forced.argtypes = [vp, C.c_int, C.POINTER(DselStepInfo)]
    L.dsel_run.argtypes = [vp, ip]
    L.dsel_peek_gains.argtypes = [vp, vp]
    L.dsel_get_trace.argtypes = [vp, C.POINTER(DselStepInfo), C.c_int]
    L.dsel_get_trace.restype = C.c_int
    L.dsel_reset.argtypes = [vp]
    L.dsel_export_factor.argtypes = [vp, vp, C.c_int64]
    L.dsel_export_factor_row.argtypes = [vp, C.c_int, vp, C.c_int64]
    L.dsel_get_stats.argtypes = [vp, C.POINTER(DselStats)]
    L.dsel_fold_records.argtypes = [C.POINTER(DselArgRec), C.c_int, C.POINTER(DselArgRec)]
    L.dsel_fold_records.restype = None
    for name in EXPORTS:
        if name not in ("dsel_destroy", "dsel_last_error", "dsel_device_bytes", "dsel_fold_records",
                        "dsel_alloc_count",
                        "dsel_lti_free",
                        "dsel_get_trace", "dsel_abi_version"):
            getattr(L, name).restype = C.c_int
    return L


lib = _load()
