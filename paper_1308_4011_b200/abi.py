"""ctypes mirror of include/mmgpu.h (structs, status codes, criterion bits)."""
from __future__ import annotations

import ctypes as C

import numpy as np

MM_OK = 0
MM_E_RANGE = 1
MM_E_ARG = 2
MM_E_CUDA = 3
MM_E_OOM = 4
MM_E_STATE = 5
MM_E_UNSUPPORTED = 6
MM_E_CAPACITY = 7
MM_E_PARSE = 8
MM_E_VALIDATION = 9
MM_E_IO = 10
MM_E_NCCL = 11

STATUS_NAMES = {
    0: "MM_OK", 1: "MM_E_RANGE", 2: "MM_E_ARG", 3: "MM_E_CUDA", 4: "MM_E_OOM",
    5: "MM_E_STATE", 6: "MM_E_UNSUPPORTED", 7: "MM_E_CAPACITY", 8: "MM_E_PARSE", 9: "MM_E_VALIDATION", 10: "MM_E_IO",
    11: "MM_E_NCCL",
}

MM_CRIT_SIMILARITY = 1 << 0
MM_CRIT_COHESION = 1 << 1
MM_CRIT_COUPLING = 1 << 2
MM_COMBINE_UNION = 0
MM_COMBINE_INTERSECTION = 1
MM_THR_EXPLICIT = 0
MM_THR_DEVICE_MEANS = 1
MM_SWEEP_EXACT_RANGE = 1

U32P = C.POINTER(C.c_uint32)


class mm_system(C.Structure):
    _fields_ = [
        ("n_classes", C.c_uint32), ("n_methods", C.c_uint32), ("n_attributes", C.c_uint32),
        ("reserved", C.c_uint32),
        ("method_owner", U32P), ("attribute_owner", U32P),
        ("class_method_off", U32P), ("class_methods", U32P),
        ("class_attr_off", U32P), ("class_attrs", U32P),
        ("call_off", U32P), ("call_tgt", U32P),
        ("acc_off", U32P), ("acc_tgt", U32P),
    ]


class mm_similarity(C.Structure):
    """SimilarityEntry, metrics.hpp:31-37."""
    _fields_ = [("first", C.c_uint32), ("second", C.c_uint32), ("value", C.c_double)]


SIMILARITY_DTYPE = np.dtype([("first", np.uint32), ("second", np.uint32), ("value", np.float64)])


class mm_workload(C.Structure):
    """WorkloadEstimate, metrics.hpp:195-207."""
    _fields_ = [(f, C.c_uint64) for f in ("m", "c", "k_m", "k_a", "n_fan", "n_sim", "n_lcom", "n_cbo", "n_total")]


class mm_whatif(C.Structure):
    _fields_ = [
        ("lcom_origin_before", C.c_double), ("lcom_origin_after", C.c_double),
        ("lcom_dest_before", C.c_double), ("lcom_dest_after", C.c_double),
        ("cbo_origin_before", C.c_uint32), ("cbo_origin_after", C.c_uint32),
        ("cbo_dest_before", C.c_uint32), ("cbo_dest_after", C.c_uint32),
        ("origin_degenerate_after", C.c_uint8), ("dest_degenerate_after", C.c_uint8),
        ("pad", C.c_uint8 * 6),
    ]


class mm_suggestion(C.Structure):
    _fields_ = [
        ("lcom_origin_before", C.c_double), ("lcom_origin_after", C.c_double),
        ("lcom_dest_before", C.c_double), ("lcom_dest_after", C.c_double),
        ("method", C.c_uint32), ("origin", C.c_uint32), ("destination", C.c_uint32),
        ("cbo_origin_before", C.c_uint32), ("cbo_origin_after", C.c_uint32),
        ("cbo_dest_before", C.c_uint32), ("cbo_dest_after", C.c_uint32),
        ("criteria", C.c_uint8), ("origin_degenerate_after", C.c_uint8),
        ("dest_degenerate_after", C.c_uint8), ("pad", C.c_uint8),
    ]


class mm_overrides(C.Structure):
    _fields_ = [
        ("has_similarity", C.c_uint8), ("has_lcom", C.c_uint8), ("has_cbo", C.c_uint8), ("pad", C.c_uint8),
        ("similarity", C.c_double), ("lcom", C.c_double), ("cbo", C.c_double),
    ]


class mm_thresholds(C.Structure):
    _fields_ = [
        ("similarity", C.c_double), ("lcom", C.c_double), ("cbo", C.c_double),
        ("explicit_mode", C.c_uint8), ("pad", C.c_uint8 * 7),
    ]


class mm_sweep_params(C.Structure):
    _fields_ = [
        ("criteria", C.c_uint32), ("combine", C.c_uint32), ("all_candidates", C.c_uint32),
        ("top_k", C.c_uint32), ("thr_lcom", C.c_double), ("thr_cbo", C.c_double),
        ("class_begin", C.c_uint32), ("class_end", C.c_uint32),
        ("threshold_source", C.c_uint32), ("flags", C.c_uint32),
    ]


class mm_sweep_stats(C.Structure):
    _fields_ = [("candidates", C.c_uint64), ("gated_whatifs", C.c_uint64),
                ("suggestions", C.c_uint64), ("methods", C.c_uint64)]


class mm_kernel_stat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_uint64), ("total_ms", C.c_double)]


class mm_gen_config(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("n_classes", C.c_uint32), ("n_methods", C.c_uint32),
        ("n_attributes", C.c_uint32), ("k_max_calls", C.c_uint32), ("k_max_accesses", C.c_uint32),
        ("pad", C.c_uint32), ("intra_class_bias", C.c_double), ("zipf_s", C.c_double),
    ]


assert C.sizeof(mm_suggestion) == 64
assert C.sizeof(mm_whatif) == 56

# numpy view of mm_suggestion records (same layout)
SUGGESTION_DTYPE = np.dtype([
    ("lcom_origin_before", "<f8"), ("lcom_origin_after", "<f8"),
    ("lcom_dest_before", "<f8"), ("lcom_dest_after", "<f8"),
    ("method", "<u4"), ("origin", "<u4"), ("destination", "<u4"),
    ("cbo_origin_before", "<u4"), ("cbo_origin_after", "<u4"),
    ("cbo_dest_before", "<u4"), ("cbo_dest_after", "<u4"),
    ("criteria", "u1"), ("origin_degenerate_after", "u1"), ("dest_degenerate_after", "u1"), ("pad", "u1"),
])
assert SUGGESTION_DTYPE.itemsize == 64

WHATIF_FIELDS = [
    "lcom_origin_before", "lcom_origin_after", "lcom_dest_before", "lcom_dest_after",
    "cbo_origin_before", "cbo_origin_after", "cbo_dest_before", "cbo_dest_after",
    "origin_degenerate_after", "dest_degenerate_after",
]
