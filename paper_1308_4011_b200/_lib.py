"""Loader for the in-tree libmmgpu.so. Fails loudly: there is no fallback."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from . import abi

import os

# MMGPU_LIB: an alternative build of the same library (A/B experiments); default in-tree
_LIB_PATH = Path(os.environ.get("MMGPU_LIB") or (Path(__file__).resolve().parent / "libmmgpu.so"))
_lib = None


class MMError(RuntimeError):
    """A non-OK mm_status. `.status` holds the code."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"{abi.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class MMRangeError(MMError, IndexError):
    """MM_E_RANGE — the reference throws std::out_of_range here."""


class MMArgError(MMError, ValueError):
    """MM_E_ARG — the reference throws std::invalid_argument here."""


def _exc_for(status: int):
    return {abi.MM_E_RANGE: MMRangeError, abi.MM_E_ARG: MMArgError}.get(status, MMError)


_SIGS = {
    "mm_abi_version": (C.c_int, []),
    "mm_device_count": (C.c_int, []),
    "mm_last_error": (C.c_char_p, [C.c_void_p]),
    "mm_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "mm_ctx_destroy": (None, [C.c_void_p]),
    "mm_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "mm_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "mm_ctx_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "mm_kernel_stats": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_kernel_stat), C.c_int, C.POINTER(C.c_int)]),
    "mm_reset_kernel_stats": (C.c_int, [C.c_void_p]),
    "mm_upload": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_system)]),
    "mm_system_bytes": (C.c_uint64, [C.POINTER(abi.mm_system)]),
    "mm_compute_metrics": (C.c_int, [C.c_void_p]),
    "mm_class_metrics": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mm_class_metrics_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "mm_fan_metrics": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "mm_similarities": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "mm_suggest_similarity": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_double, C.c_uint32, C.c_void_p,
                                        C.c_uint64, C.c_void_p]),
    "mm_estimate_workload": (C.c_int, [C.c_void_p, C.c_void_p]),
    "mm_lcom_normalized": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_double)]),
    "mm_lcom_ck": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64)]),
    "mm_cbo": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32)]),
    "mm_compute_thresholds": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_overrides), C.POINTER(abi.mm_thresholds)]),
    "mm_report_thresholds": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                       C.c_uint64, C.POINTER(abi.mm_overrides), C.POINTER(abi.mm_thresholds)]),
    "mm_sequential_mean": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int)]),
    "mm_what_if": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(abi.mm_whatif)]),
    "mm_set_gates": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "mm_sweep": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_sweep_params), C.POINTER(C.c_uint64)]),
    "mm_run": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_sweep_params)]),
    "mm_collect_timings": (C.c_int, [C.c_void_p]),
    "mm_sweep_device_result": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]),
    "mm_sweep_device_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "mm_ctx_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "mm_group_create": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)]),
    "mm_group_destroy": (None, [C.c_void_p]),
    "mm_group_last_error": (C.c_char_p, [C.c_void_p]),
    "mm_group_size": (C.c_int, [C.c_void_p]),
    "mm_group_uses_nccl": (C.c_int, [C.c_void_p]),
    "mm_group_ctx": (C.c_void_p, [C.c_void_p, C.c_int]),
    "mm_group_upload": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_system)]),
    "mm_group_shard": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "mm_group_set_gates": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "mm_group_run": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_sweep_params), C.POINTER(C.c_uint64)]),
    "mm_group_synchronize": (C.c_int, [C.c_void_p]),
    "mm_group_counts": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]),
    "mm_group_device_result": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]),
    "mm_group_copy_suggestions": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "mm_sweep_stats_get": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_sweep_stats)]),
    "mm_copy_suggestions": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "mm_suggest": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_sweep_params), C.c_void_p, C.c_uint64,
                             C.POINTER(C.c_uint64)]),
    "mm_pinned_alloc": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "mm_pinned_free": (None, [C.c_void_p]),
    "mm_plan_shards": (C.c_int, [C.POINTER(abi.mm_system), C.c_uint32, C.POINTER(C.c_uint32)]),
    "mm_generate": (C.c_int, [C.POINTER(abi.mm_gen_config), C.POINTER(C.c_void_p)]),
    "mm_host_system_view": (C.POINTER(abi.mm_system), [C.c_void_p]),
    "mm_host_system_free": (None, [C.c_void_p]),
}

EXPORTED = tuple(_SIGS)

# include/mmfacts.h (facts ingest, host-only)
_FACTS_SIGS = {
    "mm_facts_parse": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "mm_facts_load": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "mm_facts_free": (None, [C.c_void_p]),
    "mm_facts_status": (C.c_int, [C.c_void_p]),
    "mm_facts_error": (C.c_char_p, [C.c_void_p]),
    "mm_facts_system": (C.c_int, [C.c_void_p, C.POINTER(abi.mm_system)]),
    "mm_facts_violation_count": (C.c_uint32, [C.c_void_p]),
    "mm_facts_violation": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_int), C.POINTER(C.c_char_p)]),
    "mm_facts_warning_count": (C.c_uint32, [C.c_void_p]),
    "mm_facts_warning": (C.c_char_p, [C.c_void_p, C.c_uint32]),
    "mm_facts_class_name": (C.c_void_p, [C.c_void_p, C.c_uint32, C.POINTER(C.c_size_t)]),
    "mm_facts_method_name": (C.c_void_p, [C.c_void_p, C.c_uint32, C.POINTER(C.c_size_t)]),
    "mm_facts_attribute_name": (C.c_void_p, [C.c_void_p, C.c_uint32, C.POINTER(C.c_size_t)]),
    "mm_facts_to_json": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
}

FACTS_EXPORTED = tuple(_FACTS_SIGS)


def lib_path() -> Path:
    return _LIB_PATH


def lib() -> C.CDLL:
    """The loaded libmmgpu.so. Raises if it has not been built — never falls back."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(
                f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(this engine has no CPU fallback)")
        l = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in {**_SIGS, **_FACTS_SIGS}.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def check(status: int, ctx, what: str) -> None:
    if status != abi.MM_OK:
        msg = lib().mm_last_error(ctx).decode() if ctx else what
        raise _exc_for(status)(status, f"{what}: {msg}")
