"""Python mirror of the reference's metric + suggestion API over libmmgpu.so.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/modmetrics/{metrics,parallel,suggest}.hpp:

=====================================  ==========================================
reference (C++)                        here
=====================================  ==========================================
parallel_class_metrics (parallel:149)  Engine.parallel_class_metrics / module fn
parallel_lcom_ck (parallel:164)        Engine.parallel_lcom_ck / module fn
lcom_normalized / lcom_ck / cbo        Engine.lcom_normalized / .lcom_ck_of / .cbo
compute_thresholds (suggest:46)        Engine.compute_thresholds
what_if_move (suggest:87)              Engine.what_if_move / module fn
suggest_by_cohesion / _coupling        Engine.suggest_by_cohesion / _coupling
suggest_all (suggest:303)              Engine.suggest_all / module fn
=====================================  ==========================================

std::out_of_range -> MMRangeError (an IndexError); std::invalid_argument ->
MMArgError (a ValueError). Everything computes on the GPU; a missing library
or device raises (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np

from . import abi
from ._lib import MMArgError, MMError, check, lib
from .system import System


class Criterion(enum.IntEnum):  # suggest.hpp:17
    Similarity = 0
    Cohesion = 1
    Coupling = 2


class Combine(enum.IntEnum):  # suggest.hpp:296
    Union = 0
    Intersection = 1


@dataclass(frozen=True)
class Thresholds:  # suggest.hpp:35-41
    similarity: float = 0.0
    lcom: float = 0.0
    cbo: float = 0.0
    explicit_mode: bool = False


@dataclass(frozen=True)
class ThresholdOverrides:  # suggest.hpp:28-32
    similarity: Optional[float] = None
    lcom: Optional[float] = None
    cbo: Optional[float] = None


@dataclass(frozen=True)
class ClassMetrics:  # parallel.hpp:139-144
    lcom: np.ndarray
    cbo: np.ndarray


def criteria_mask(criteria: Iterable) -> int:
    m = 0
    for c in criteria:
        m |= 1 << int(c)
    return m


def criteria_of_mask(mask: int) -> list:
    return [c for c in Criterion if mask & (1 << int(c))]


class PinnedBuffer:
    """A reusable page-locked host buffer (mm_pinned_alloc), viewed as numpy."""

    def __init__(self):
        self.ptr = C.c_void_p()
        self.nbytes = 0

    def view(self, dtype, count: int) -> np.ndarray:
        need = max(1, np.dtype(dtype).itemsize * count)
        if need > self.nbytes:
            self.free()
            cap = max(need, 2 * self.nbytes)
            check(lib().mm_pinned_alloc(cap, C.byref(self.ptr)), None, "mm_pinned_alloc")
            self.nbytes = cap
        buf = (C.c_char * self.nbytes).from_address(self.ptr.value)
        return np.frombuffer(buf, dtype=dtype, count=count)

    def free(self):
        if self.ptr:
            lib().mm_pinned_free(self.ptr)
            self.ptr = C.c_void_p()
            self.nbytes = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Engine:
    """One GPU context (`mm_ctx`) holding one uploaded system."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self._pinned = {}
        self._ctx = C.c_void_p()
        check(lib().mm_ctx_create(device, C.byref(self._ctx)), None, f"mm_ctx_create(device={device})")
        if stream is not None:
            self.set_stream(stream)
        self.system: Optional[System] = None

    # ---- context ------------------------------------------------------
    def close(self) -> None:
        for b in getattr(self, "_pinned", {}).values():
            b.free()
        if self._ctx:
            lib().mm_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, what: str) -> None:
        check(st, self._ctx, what)

    def set_stream(self, stream_handle: Optional[int]) -> None:
        self._check(lib().mm_ctx_set_stream(self._ctx, C.c_void_p(stream_handle or 0)), "mm_ctx_set_stream")

    def synchronize(self) -> None:
        self._check(lib().mm_ctx_synchronize(self._ctx), "mm_ctx_synchronize")

    def set_profiling(self, on: bool) -> None:
        self._check(lib().mm_ctx_set_profiling(self._ctx, int(on)), "mm_ctx_set_profiling")

    def kernel_stats(self) -> dict:
        n = C.c_int()
        lib().mm_kernel_stats(self._ctx, None, 0, C.byref(n))
        arr = (abi.mm_kernel_stat * max(1, n.value))()
        self._check(lib().mm_kernel_stats(self._ctx, arr, n.value, C.byref(n)), "mm_kernel_stats")
        return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms)) for i in range(n.value)}

    def reset_kernel_stats(self) -> None:
        self._check(lib().mm_reset_kernel_stats(self._ctx), "mm_reset_kernel_stats")

    # ---- model --------------------------------------------------------
    def upload(self, system: System, owner_tables: bool = True) -> "Engine":
        """H2D of the system. owner_tables=False leaves method_owner /
        attribute_owner out of the copy: the device derives them from the
        membership lists (equal for any model that passes validate())."""
        s = system.as_c()
        if not owner_tables:
            s.method_owner = abi.U32P()
            s.attribute_owner = abi.U32P()
        self._check(lib().mm_upload(self._ctx, C.byref(s)), "mm_upload")
        self.system = system
        return self

    # ---- metric pass --------------------------------------------------
    def compute_metrics(self) -> None:
        self._check(lib().mm_compute_metrics(self._ctx), "mm_compute_metrics")

    def _staging(self, name: str, dtype, count: int) -> np.ndarray:
        b = self._pinned.get(name)
        if b is None:
            b = self._pinned[name] = PinnedBuffer()
        return b.view(dtype, count)

    def class_metrics_all(self, copy: bool = True):
        """(lcom f64[c], lcom_ck u64[c], cbo u32[c]) — full_report's class fields.
        D2H lands in reusable pinned buffers; copy=False returns views of them
        (valid until the next call)."""
        n = self.system.n_classes
        lcom = self._staging("lcom", np.float64, n)
        ck = self._staging("ck", np.uint64, n)
        cbo = self._staging("cbo", np.uint32, n)
        self._check(lib().mm_class_metrics(self._ctx, lcom.ctypes.data, ck.ctypes.data, cbo.ctypes.data),
                    "mm_class_metrics")
        if copy:
            return lcom.copy(), ck.copy(), cbo.copy()
        return lcom, ck, cbo

    def fan_metrics(self):
        """(fan_in u32[m], fan_out u32[m]) — MetricsReport's fan fields
        (metrics.hpp:79-93, parallel_fan_metrics parallel.hpp:186)."""
        m = self.system.n_methods
        fi, fo = np.empty(m, np.uint32), np.empty(m, np.uint32)
        self._check(lib().mm_fan_metrics(self._ctx, fi.ctypes.data, fo.ctypes.data), "mm_fan_metrics")
        return fi, fo

    def similarities(self) -> np.ndarray:
        """all_similarities (metrics.hpp:67-77): every pair with a nonzero
        Jaccard similarity, ordered by (first, second), as SIMILARITY_DTYPE."""
        n = C.c_uint64()
        self._check(lib().mm_similarities(self._ctx, None, 0, C.byref(n)), "mm_similarities")
        out = np.zeros(n.value, dtype=abi.SIMILARITY_DTYPE)
        if n.value:
            self._check(lib().mm_similarities(self._ctx, out.ctypes.data, n.value, C.byref(n)), "mm_similarities")
        return out

    def full_report(self) -> dict:
        """full_report (metrics.hpp:249-264), every field from the device:
        fan_in, fan_out, similarity, lcom, lcom_ck, cbo, workload."""
        fi, fo = self.fan_metrics()
        lcom, ck, cbo = self.class_metrics_all()
        return {"fan_in": fi, "fan_out": fo, "similarity": self.similarities(), "lcom": lcom, "lcom_ck": ck,
                "cbo": cbo, "workload": self.estimate_workload()}

    def estimate_workload(self) -> dict:
        """WorkloadEstimate (metrics.hpp:195-233): k_m / k_a by a device max-reduce."""
        w = abi.mm_workload()
        self._check(lib().mm_estimate_workload(self._ctx, C.byref(w)), "mm_estimate_workload")
        return {f: getattr(w, f) for f, _ in abi.mm_workload._fields_}

    def class_metrics_async(self):
        """Enqueue the D2H of (lcom, lcom_ck, cbo) into the pinned staging
        buffers behind the work already launched; it overlaps what is launched
        next. The returned views hold the results after synchronize()."""
        n = self.system.n_classes
        lcom = self._staging("lcom", np.float64, n)
        ck = self._staging("ck", np.uint64, n)
        cbo = self._staging("cbo", np.uint32, n)
        self._check(lib().mm_class_metrics_async(self._ctx, lcom.ctypes.data, ck.ctypes.data, cbo.ctypes.data),
                    "mm_class_metrics_async")
        return lcom, ck, cbo

    def parallel_class_metrics(self, n_workers: int = 1) -> ClassMetrics:
        if n_workers == 0:
            raise MMArgError(abi.MM_E_ARG, "plan_partition: zero workers")  # parallel.hpp:29
        lcom, _, cbo = self.class_metrics_all()
        return ClassMetrics(lcom, cbo)

    def parallel_lcom_ck(self, n_workers: int = 1) -> np.ndarray:
        if n_workers == 0:
            raise MMArgError(abi.MM_E_ARG, "plan_partition: zero workers")
        return self.class_metrics_all()[1]

    def lcom_normalized(self, cls: int) -> float:
        v = C.c_double()
        self._check(lib().mm_lcom_normalized(self._ctx, cls, C.byref(v)), "lcom_normalized")
        return v.value

    def lcom_ck_of(self, cls: int) -> int:
        v = C.c_uint64()
        self._check(lib().mm_lcom_ck(self._ctx, cls, C.byref(v)), "lcom_ck")
        return v.value

    def cbo(self, cls: int) -> int:
        v = C.c_uint32()
        self._check(lib().mm_cbo(self._ctx, cls, C.byref(v)), "cbo")
        return v.value

    # ---- thresholds ---------------------------------------------------
    def compute_thresholds(self, overrides: Optional[ThresholdOverrides] = None) -> Thresholds:
        """compute_thresholds(full_report(...), overrides): the means of this
        engine's lcom / cbo and of its similarity table (built when absent)."""
        ov = abi.mm_overrides()
        if overrides is not None:
            for name in ("similarity", "lcom", "cbo"):
                v = getattr(overrides, name)
                if v is not None:
                    setattr(ov, "has_" + name, 1)
                    setattr(ov, name, float(v))
        t = abi.mm_thresholds()
        self._check(lib().mm_compute_thresholds(self._ctx, C.byref(ov), C.byref(t)), "compute_thresholds")
        return Thresholds(t.similarity, t.lcom, t.cbo, bool(t.explicit_mode))

    def report_thresholds(self, lcom, cbo, similarity=None,
                          overrides: Optional[ThresholdOverrides] = None) -> Thresholds:
        """compute_thresholds(report, overrides) (suggest.hpp:46-61) on a caller's
        report vectors: every mean on the device, bit-identical to the
        reference's sequential double sums. `similarity` = the report's
        similarity values (or a SIMILARITY_DTYPE table)."""
        l = np.ascontiguousarray(lcom, dtype=np.float64)
        c = np.ascontiguousarray(cbo, dtype=np.uint32)
        if similarity is None:
            sv = np.zeros(0, np.float64)
        elif getattr(similarity, "dtype", None) is not None and similarity.dtype.names:
            sv = np.ascontiguousarray(similarity["value"], dtype=np.float64)
        else:
            sv = np.ascontiguousarray(similarity, dtype=np.float64)
        ov = abi.mm_overrides()
        if overrides is not None:
            for name in ("similarity", "lcom", "cbo"):
                v = getattr(overrides, name)
                if v is not None:
                    setattr(ov, "has_" + name, 1)
                    setattr(ov, name, float(v))
        t = abi.mm_thresholds()
        self._check(lib().mm_report_thresholds(self._ctx, l.ctypes.data, len(l), c.ctypes.data, len(c),
                                               sv.ctypes.data, len(sv), C.byref(ov), C.byref(t)),
                    "compute_thresholds")
        return Thresholds(t.similarity, t.lcom, t.cbo, bool(t.explicit_mode))

    def sequential_mean(self, values) -> tuple:
        """(mean, fast_path) of values with the reference's sequential double-sum semantics."""
        v = np.ascontiguousarray(values, dtype=np.float64)
        out, fast = C.c_double(), C.c_int()
        self._check(lib().mm_sequential_mean(self._ctx, v.ctypes.data, len(v), C.byref(out), C.byref(fast)),
                    "mm_sequential_mean")
        return out.value, bool(fast.value)

    # ---- what-if ------------------------------------------------------
    def what_if_move(self, method: int, origin: int, destination: int) -> dict:
        w = abi.mm_whatif()
        self._check(lib().mm_what_if(self._ctx, method, origin, destination, C.byref(w)), "what_if_move")
        return {f: (bool(getattr(w, f)) if f.endswith("degenerate_after") else getattr(w, f))
                for f in abi.WHATIF_FIELDS}

    # ---- sweep --------------------------------------------------------
    @staticmethod
    def _params(criteria, combine, thresholds, all_candidates, top_k, class_range) -> abi.mm_sweep_params:
        p = abi.mm_sweep_params(criteria=criteria_mask(criteria), combine=int(combine),
                                all_candidates=int(bool(all_candidates)), top_k=int(top_k))
        if thresholds is None:
            p.threshold_source = abi.MM_THR_DEVICE_MEANS
        else:
            p.threshold_source = abi.MM_THR_EXPLICIT
            p.thr_lcom = float(thresholds.lcom)
            p.thr_cbo = float(thresholds.cbo)
        if class_range is not None:
            p.class_begin, p.class_end = int(class_range[0]), int(class_range[1])
        return p

    def sweep(self, criteria=(Criterion.Cohesion, Criterion.Coupling), combine=Combine.Union,
              thresholds: Optional[Thresholds] = None, all_candidates: bool = False, top_k: int = 1,
              class_range: Optional[tuple] = None, want_count: bool = True) -> Optional[int]:
        """Device-resident sweep. thresholds=None uses the device-computed means."""
        p = self._params(criteria, combine, thresholds, all_candidates, top_k, class_range)
        n = C.c_uint64()
        self._check(lib().mm_sweep(self._ctx, C.byref(p), C.byref(n) if want_count else None), "mm_sweep")
        return n.value if want_count else None

    def set_gates(self, lcom=None, cbo=None) -> None:
        """Gate on the caller's report vectors (None, None: the device metrics)."""
        if lcom is None and cbo is None:
            self._check(lib().mm_set_gates(self._ctx, None, None), "mm_set_gates")
            return
        self._gl = np.ascontiguousarray(lcom, dtype=np.float64)
        self._gc = np.ascontiguousarray(cbo, dtype=np.uint32)
        self._check(lib().mm_set_gates(self._ctx, self._gl.ctypes.data, self._gc.ctypes.data), "mm_set_gates")

    def run(self, criteria=(Criterion.Cohesion, Criterion.Coupling), combine=Combine.Union,
            thresholds: Optional[Thresholds] = None, all_candidates: bool = False, top_k: int = 1,
            class_range: Optional[tuple] = None) -> None:
        """One full step (metric pass + sweep), replayed from a CUDA graph; no host sync."""
        p = self._params(criteria, combine, thresholds, all_candidates, top_k, class_range)
        self._check(lib().mm_run(self._ctx, C.byref(p)), "mm_run")

    def collect_timings(self) -> None:
        self._check(lib().mm_collect_timings(self._ctx), "mm_collect_timings")

    def sweep_stats(self) -> dict:
        s = abi.mm_sweep_stats()
        self._check(lib().mm_sweep_stats_get(self._ctx, C.byref(s)), "mm_sweep_stats_get")
        return {"candidates": s.candidates, "gated_whatifs": s.gated_whatifs, "suggestions": s.suggestions,
                "methods": s.methods}

    def device_result(self):
        """(device pointer, count) of the last sweep's mm_suggestion records."""
        ptr = C.c_void_p()
        n = C.c_uint64()
        self._check(lib().mm_sweep_device_result(self._ctx, C.byref(ptr), C.byref(n)), "mm_sweep_device_result")
        return ptr.value, n.value

    def suggestions(self, copy: bool = True) -> np.ndarray:
        """The last sweep's ordered records (D2H into a reusable pinned buffer;
        copy=False returns a view of it, valid until the next call)."""
        # one round trip when the staging buffer already fits the list (the
        # previous sweep's count), else size query + copy
        n = C.c_uint64()
        cap = getattr(self, "_sugg_cap", 0)
        if cap:
            buf = self._staging("sugg", abi.SUGGESTION_DTYPE, cap)
            st = lib().mm_copy_suggestions(self._ctx, buf.ctypes.data, cap, C.byref(n))
            if st == abi.MM_OK:
                self._sugg_cap = max(int(n.value), 1)
                out = buf[: n.value]
                return out.copy() if copy else out
            if st != abi.MM_E_CAPACITY:
                self._check(st, "mm_copy_suggestions")
        st = lib().mm_copy_suggestions(self._ctx, None, 0, C.byref(n))
        if st not in (abi.MM_OK, abi.MM_E_CAPACITY):
            self._check(st, "mm_copy_suggestions")
        out = self._staging("sugg", abi.SUGGESTION_DTYPE, n.value)
        if n.value:
            self._check(lib().mm_copy_suggestions(self._ctx, out.ctypes.data, n.value, C.byref(n)),
                        "mm_copy_suggestions")
        self._sugg_cap = max(int(n.value), 1)
        return out.copy() if copy else out

    def suggest_all(self, thresholds: Thresholds, criteria: Sequence = (Criterion.Cohesion, Criterion.Coupling),
                    combine: Combine = Combine.Union, all_candidates: bool = False, top_k: int = 1,
                    class_range: Optional[tuple] = None, copy: bool = True) -> np.ndarray:
        """suggest_all (suggest.hpp:303): ordered by (origin, method, destination)."""
        crit = set(Criterion(c) for c in criteria)
        if Criterion.Similarity not in crit:
            self.sweep(criteria, combine, thresholds, all_candidates, top_k, class_range, want_count=False)
            return self.suggestions(copy=copy)
        if top_k != 1 or class_range is not None:
            raise MMError(abi.MM_E_UNSUPPORTED, "suggest_all: top-k / class ranges with the similarity criterion")
        # the sweep for the other criteria, the similarity criterion on its own,
        # merged by (method, destination) as suggest.hpp:315-341 does
        parts = [self.suggest_by_similarity(thresholds.similarity, all_candidates)]
        rest = crit - {Criterion.Similarity}
        if rest:
            parts.append(self.suggest_all(thresholds, sorted(rest), combine, all_candidates))
        recs = np.concatenate(parts) if len(parts) > 1 else parts[0]
        if not len(recs):
            return recs
        order = np.lexsort((recs["destination"], recs["method"]))
        recs = recs[order]
        key = recs["method"].astype(np.uint64) << np.uint64(32) | recs["destination"].astype(np.uint64)
        first = np.ones(len(recs), dtype=bool)
        first[1:] = key[1:] != key[:-1]
        groups = np.cumsum(first) - 1
        tags = np.zeros(int(groups[-1]) + 1, dtype=np.uint8)
        np.bitwise_or.at(tags, groups, recs["criteria"])
        out = recs[first].copy()
        out["criteria"] = tags
        if combine == Combine.Intersection:
            out = out[out["criteria"] == criteria_mask(crit)]
        return out[np.lexsort((out["destination"], out["method"], out["origin"]))]

    def suggest_by_similarity(self, thr: float, all_candidates: bool = False, table: np.ndarray = None) -> np.ndarray:
        """suggest_by_similarity (suggest.hpp:200-232), ordered by method then
        destination; `table` = the caller's report.similarity (default: the
        device table, as all_similarities)."""
        ptr, n_tab = None, 0
        if table is not None:
            table = np.ascontiguousarray(table, dtype=abi.SIMILARITY_DTYPE)
            ptr, n_tab = table.ctypes.data, len(table)
        n = C.c_uint64()
        st = lib().mm_suggest_similarity(self._ctx, ptr, n_tab, float(thr), int(all_candidates), None, 0, C.byref(n))
        if st not in (abi.MM_OK, abi.MM_E_CAPACITY):
            self._check(st, "mm_suggest_similarity")
        out = np.zeros(n.value, dtype=abi.SUGGESTION_DTYPE)
        if n.value:
            self._check(lib().mm_suggest_similarity(self._ctx, ptr, n_tab, float(thr), int(all_candidates),
                                                    out.ctypes.data, n.value, C.byref(n)), "mm_suggest_similarity")
        return out

    def suggest_by_cohesion(self, thresholds: Thresholds, all_candidates: bool = False) -> np.ndarray:
        """suggest_by_cohesion (suggest.hpp:239) — as a set; ordered (origin, method, dest)."""
        return self.suggest_all(thresholds, [Criterion.Cohesion], Combine.Union, all_candidates)

    def suggest_by_coupling(self, thresholds: Thresholds, all_candidates: bool = False) -> np.ndarray:
        return self.suggest_all(thresholds, [Criterion.Coupling], Combine.Union, all_candidates)


class Group:
    """Several GPUs in one process (`mm_group`, include/mmgpu.h): the
    reference's n_workers mapped to GPUs. Metric pass replicated, sweep on
    cost-balanced class-range shards, exact-count NCCL exchange into every
    GPU's assembled list (= suggest_all's ordered list)."""

    def __init__(self, devices: Optional[Sequence[int]] = None, n: Optional[int] = None):
        # mm_group dlopens libnccl.so.2 and reuses one already in the process:
        # load torch's first when torch is present, so both share one NCCL
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        if devices is None:
            devices = list(range(n if n is not None else 1))
        arr = (C.c_int * max(1, len(devices)))(*devices)
        self._g = C.c_void_p()
        st = lib().mm_group_create(arr, len(devices), C.byref(self._g))
        if st:
            check(st, None, f"mm_group_create(devices={list(devices)})")
        self.n = len(devices)
        self.system: Optional[System] = None

    def close(self) -> None:
        if self._g:
            lib().mm_group_destroy(self._g)
            self._g = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, what: str) -> None:
        if st:
            from ._lib import _exc_for
            raise _exc_for(st)(st, f"{what}: {lib().mm_group_last_error(self._g).decode(errors='replace')}")

    @property
    def uses_nccl(self) -> bool:
        return bool(lib().mm_group_uses_nccl(self._g))

    def upload(self, system: System) -> "Group":
        self._s = system.as_c()
        self._check(lib().mm_group_upload(self._g, C.byref(self._s)), "mm_group_upload")
        self.system = system
        return self

    def shards(self) -> list:
        out = []
        for i in range(self.n):
            b, e = C.c_uint32(), C.c_uint32()
            self._check(lib().mm_group_shard(self._g, i, C.byref(b), C.byref(e)), "mm_group_shard")
            out.append((b.value, e.value))
        return out

    def run(self, criteria=(Criterion.Cohesion, Criterion.Coupling), combine=Combine.Union,
            thresholds: Optional[Thresholds] = None, all_candidates: bool = False, top_k: int = 1,
            want_count: bool = True) -> Optional[int]:
        p = Engine._params(criteria, combine, thresholds, all_candidates, top_k, None)
        n = C.c_uint64()
        self._check(lib().mm_group_run(self._g, C.byref(p), C.byref(n) if want_count else None), "mm_group_run")
        return n.value if want_count else None

    def counts(self) -> list:
        c = np.zeros(self.n, np.uint64)
        t = C.c_uint64()
        self._check(lib().mm_group_counts(self._g, c.ctypes.data, C.byref(t)), "mm_group_counts")
        return [int(x) for x in c]

    def suggestions(self) -> np.ndarray:
        n = C.c_uint64()
        st = lib().mm_group_copy_suggestions(self._g, None, 0, C.byref(n))
        if st not in (abi.MM_OK, abi.MM_E_CAPACITY):
            self._check(st, "mm_group_copy_suggestions")
        out = np.zeros(n.value, dtype=abi.SUGGESTION_DTYPE)
        if n.value:
            self._check(lib().mm_group_copy_suggestions(self._g, out.ctypes.data, n.value, C.byref(n)),
                        "mm_group_copy_suggestions")
        return out

    def synchronize(self) -> None:
        self._check(lib().mm_group_synchronize(self._g), "mm_group_synchronize")


# ---- free functions with the reference's call shapes ---------------------

def plan_shards(system: System, n_shards: int) -> np.ndarray:
    """Cost-balanced contiguous class ranges (bounds, len n_shards + 1)."""
    b = np.zeros(n_shards + 1, dtype=np.uint32)
    s = system.as_c()
    check(lib().mm_plan_shards(C.byref(s), n_shards, b.ctypes.data_as(abi.U32P)), None, "mm_plan_shards")
    return b


def parallel_class_metrics(system: System, n_workers: int = 1, device: int = 0) -> ClassMetrics:
    with Engine(device) as e:
        return e.upload(system).parallel_class_metrics(n_workers)


def parallel_lcom_ck(system: System, n_workers: int = 1, device: int = 0) -> np.ndarray:
    with Engine(device) as e:
        return e.upload(system).parallel_lcom_ck(n_workers)


def what_if_move(method: int, origin: int, destination: int, system: System, device: int = 0) -> dict:
    with Engine(device) as e:
        return e.upload(system).what_if_move(method, origin, destination)


def all_similarities(system: System, device: int = 0) -> np.ndarray:
    """all_similarities (metrics.hpp:67-77) as SIMILARITY_DTYPE records."""
    with Engine(device) as e:
        return e.upload(system).similarities()


def full_report(system: System, device: int = 0) -> dict:
    """full_report (metrics.hpp:249-264), every field from the device."""
    with Engine(device) as e:
        return e.upload(system).full_report()


def suggest_all(system: System, thresholds: Thresholds, criteria: Sequence, combine: Combine = Combine.Union,
                all_candidates: bool = False, device: int = 0) -> np.ndarray:
    with Engine(device) as e:
        return e.upload(system).suggest_all(thresholds, criteria, combine, all_candidates)
