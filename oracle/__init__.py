"""ctypes bindings to the CPU oracle (liboracle.so) and the compiled reference (_ref/libmmref.so).

TEST INFRASTRUCTURE ONLY. Importable solely from tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline / --impl reference leg — as the checker or the
timed CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import importlib.util
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def _load_abi():
    """The ctypes mirror of include/mmgpu.h (plain struct layouts), loaded by
    path: the oracle never imports the product package, so bench.py's
    reference arm loads no product library."""
    name = "_mm_abi_for_oracle"
    if name not in sys.modules:
        spec = importlib.util.spec_from_file_location(name, HERE.parent / "paper_1308_4011_b200" / "abi.py")
        mod = importlib.util.module_from_spec(spec)
        sys.modules[name] = mod
        spec.loader.exec_module(mod)
    return sys.modules[name]


abi = _load_abi()
_FIELDS = ("method_owner", "attribute_owner", "class_method_off", "class_methods", "class_attr_off",
           "class_attrs", "call_off", "call_tgt", "acc_off", "acc_tgt")


class CsrSystem:
    """A system in the mm_system CSR layout (the same fields as the product's
    System, which the oracle functions also accept: any object with these
    arrays and n_classes / n_methods / n_attributes)."""

    def __init__(self, n_classes, n_methods, n_attributes, **arrays):
        self.n_classes, self.n_methods, self.n_attributes = n_classes, n_methods, n_attributes
        for f in _FIELDS:
            setattr(self, f, np.ascontiguousarray(arrays[f], dtype=np.uint32))

    @classmethod
    def from_view(cls, v):
        nc, nm, na = v.n_classes, v.n_methods, v.n_attributes

        def take(ptr, n):
            return np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n else np.zeros(0, np.uint32)

        co, ao = take(v.call_off, nm + 1), take(v.acc_off, nm + 1)
        return cls(nc, nm, na, method_owner=take(v.method_owner, nm), attribute_owner=take(v.attribute_owner, na),
                   class_method_off=take(v.class_method_off, nc + 1), class_methods=take(v.class_methods, nm),
                   class_attr_off=take(v.class_attr_off, nc + 1), class_attrs=take(v.class_attrs, na),
                   call_off=co, call_tgt=take(v.call_tgt, int(co[-1])), acc_off=ao,
                   acc_tgt=take(v.acc_tgt, int(ao[-1])))

    @property
    def n_calls(self):
        return int(self.call_off[-1])

    @property
    def n_accesses(self):
        return int(self.acc_off[-1])

    def equals(self, other) -> bool:
        return (self.n_classes, self.n_methods, self.n_attributes) == (
            other.n_classes, other.n_methods, other.n_attributes) and all(
            np.array_equal(getattr(self, f), getattr(other, f)) for f in _FIELDS)


def _csys(sys_):
    """(keep-alive, address) of an mm_system over sys_'s arrays."""
    s = abi.mm_system(n_classes=sys_.n_classes, n_methods=sys_.n_methods, n_attributes=sys_.n_attributes)
    for f in _FIELDS:
        setattr(s, f, np.ascontiguousarray(getattr(sys_, f), np.uint32).ctypes.data_as(abi.U32P))
    return s, C.addressof(s)
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libmmref.so"
_or = None
_ref = None


def oracle_lib():
    global _or
    if _or is None:
        l = C.CDLL(str(ORACLE_SO))
        S = C.c_void_p
        l.or_class_metrics.argtypes = [S, C.c_void_p, C.c_void_p, C.c_void_p]
        l.or_fan_metrics.argtypes = [S, C.c_void_p, C.c_void_p]
        l.or_similarities.argtypes = [S, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        l.or_thresholds.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                    C.POINTER(abi.mm_overrides), C.POINTER(abi.mm_thresholds)]
        l.or_what_if.argtypes = [S, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(abi.mm_whatif)]
        l.or_suggest.argtypes = [S, C.c_void_p, C.c_void_p, C.POINTER(abi.mm_sweep_params), C.c_void_p,
                                 C.c_uint64, C.POINTER(C.c_uint64)]
        _or = l
    return _or


def ref_available() -> bool:
    return REF_SO.exists()


def ref_lib():
    global _ref
    if _ref is None:
        l = C.CDLL(str(REF_SO))
        S = C.c_void_p
        l.ref_model_create.argtypes = [S]
        l.ref_model_create.restype = C.c_void_p
        l.ref_model_free.argtypes = [C.c_void_p]
        l.ref_validate.argtypes = [C.c_void_p]
        l.ref_generate.argtypes = [C.POINTER(abi.mm_gen_config)]
        l.ref_generate.restype = C.c_void_p
        l.ref_model_view.argtypes = [C.c_void_p]
        l.ref_model_view.restype = C.POINTER(abi.mm_system)
        l.ref_class_metrics.argtypes = [C.c_void_p, C.c_uint, C.c_void_p, C.c_void_p, C.c_void_p]
        l.ref_fan_metrics.argtypes = [C.c_void_p, C.c_uint, C.c_void_p, C.c_void_p]
        l.ref_similarities.argtypes = [C.c_void_p, C.c_uint, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        l.ref_suggest_full.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(abi.mm_sweep_params),
                                       C.c_double, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        l.ref_single_metric.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.POINTER(C.c_double),
                                        C.POINTER(C.c_uint64)]
        l.ref_thresholds.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                     C.POINTER(abi.mm_overrides), C.POINTER(abi.mm_thresholds)]
        l.ref_what_if.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(abi.mm_whatif)]
        l.ref_suggest.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(abi.mm_sweep_params), C.c_void_p,
                                  C.c_uint64, C.POINTER(C.c_uint64)]
        l.ref_suggest_by.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p,
                                     C.POINTER(abi.mm_sweep_params), C.c_void_p, C.c_uint64,
                                     C.POINTER(C.c_uint64)]
        l.ref_sweep_sample.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_uint32,
                                       C.c_uint32, C.c_uint, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        l.ref_sweep.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(abi.mm_sweep_params), C.c_void_p,
                                C.c_uint64, C.c_uint, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        l.ref_sweep_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        l.ref_candidates.argtypes = [C.c_void_p]
        l.ref_candidates.restype = C.c_uint64
        _ref = l
    return _ref


def _overrides(ov):
    o = abi.mm_overrides()
    if ov:
        for k, v in ov.items():
            if v is not None:
                setattr(o, "has_" + k, 1)
                setattr(o, k, float(v))
    return o


def _params(criteria_mask, combine=0, all_candidates=False, top_k=1, thr_lcom=0.0, thr_cbo=0.0,
            class_range=None):
    p = abi.mm_sweep_params(criteria=criteria_mask, combine=combine, all_candidates=int(all_candidates),
                            top_k=top_k, thr_lcom=thr_lcom, thr_cbo=thr_cbo)
    if class_range:
        p.class_begin, p.class_end = class_range
    return p


# ---- oracle (C restatement) ----------------------------------------------

def fan_metrics(sys_):
    s, sp = _csys(sys_)
    fi, fo = np.empty(sys_.n_methods, np.uint32), np.empty(sys_.n_methods, np.uint32)
    oracle_lib().or_fan_metrics(sp, fi.ctypes.data, fo.ctypes.data)
    return fi, fo


def similarities(sys_):
    s, sp = _csys(sys_)
    n = C.c_uint64()
    oracle_lib().or_similarities(sp, None, 0, C.byref(n))
    out = np.zeros(n.value, dtype=abi.SIMILARITY_DTYPE)
    if n.value:
        oracle_lib().or_similarities(sp, out.ctypes.data, n.value, C.byref(n))
    return out


def class_metrics(sys_):
    s, sp = _csys(sys_)
    n = sys_.n_classes
    lcom, ck, cbo = np.empty(n, np.float64), np.empty(n, np.uint64), np.empty(n, np.uint32)
    oracle_lib().or_class_metrics(sp, lcom.ctypes.data, ck.ctypes.data, cbo.ctypes.data)
    return lcom, ck, cbo


def thresholds(lcom, cbo, similarity=None, overrides=None):
    lcom = np.ascontiguousarray(lcom, np.float64)
    cbo = np.ascontiguousarray(cbo, np.uint32)
    sim = np.ascontiguousarray(similarity if similarity is not None else [], np.float64)
    t = abi.mm_thresholds()
    o = _overrides(overrides)
    oracle_lib().or_thresholds(lcom.ctypes.data, cbo.ctypes.data, len(lcom), sim.ctypes.data, len(sim),
                               C.byref(o), C.byref(t))
    return t


def what_if(sys_, u, o, d):
    s, sp = _csys(sys_)
    w = abi.mm_whatif()
    st = oracle_lib().or_what_if(sp, u, o, d, C.byref(w))
    return st, w


def suggest(sys_, lcom_gate, cbo_gate, criteria_mask, combine=0, all_candidates=False, top_k=1,
            thr_lcom=0.0, thr_cbo=0.0, class_range=None):
    s, sp = _csys(sys_)
    lg = np.ascontiguousarray(lcom_gate, np.float64)
    cg = np.ascontiguousarray(cbo_gate, np.uint32)
    p = _params(criteria_mask, combine, all_candidates, top_k, thr_lcom, thr_cbo, class_range)
    n = C.c_uint64()
    st = oracle_lib().or_suggest(sp, lg.ctypes.data, cg.ctypes.data, C.byref(p), None, 0, C.byref(n))
    out = np.zeros(n.value, dtype=abi.SUGGESTION_DTYPE)
    if n.value:
        st = oracle_lib().or_suggest(sp, lg.ctypes.data, cg.ctypes.data, C.byref(p), out.ctypes.data,
                                     n.value, C.byref(n))
    if st:
        raise RuntimeError(f"or_suggest status {st}")
    return out


# ---- the reference itself (compiled headers) -----------------------------

class RefModel:
    def __init__(self, sys_=None, handle=None):
        self._keep = sys_
        if handle is None:
            cs, sp = _csys(sys_)
        self.h = handle if handle is not None else ref_lib().ref_model_create(sp)
        view = ref_lib().ref_model_view(self.h).contents if handle is not None else None
        self.n_classes = view.n_classes if view is not None else sys_.n_classes
        self.n_methods = view.n_methods if view is not None else sys_.n_methods

    def close(self):
        if self.h:
            ref_lib().ref_model_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def validate(self) -> int:
        return ref_lib().ref_validate(self.h)

    def similarities(self, n_workers=0):
        n = C.c_uint64()
        st = ref_lib().ref_similarities(self.h, n_workers, None, 0, C.byref(n))
        if st:
            raise RuntimeError(f"ref_similarities status {st}")
        out = np.zeros(n.value, dtype=abi.SIMILARITY_DTYPE)
        if n.value:
            st = ref_lib().ref_similarities(self.h, n_workers, out.ctypes.data, n.value, C.byref(n))
        if st:
            raise RuntimeError(f"ref_similarities status {st}")
        return out

    def suggest_full(self, lcom_gate, cbo_gate, criteria_mask, combine=0, all_candidates=False, thr_sim=0.0,
                     thr_lcom=0.0, thr_cbo=0.0):
        """suggest_all with every criterion, the report's similarity = all_similarities."""
        lg = np.ascontiguousarray(lcom_gate, np.float64)
        cg = np.ascontiguousarray(cbo_gate, np.uint32)
        p = _params(criteria_mask, combine, all_candidates, 1, thr_lcom, thr_cbo, None)
        n = C.c_uint64()
        st = ref_lib().ref_suggest_full(self.h, lg.ctypes.data, cg.ctypes.data, C.byref(p), thr_sim, None, 0,
                                        C.byref(n))
        out = np.zeros(n.value, dtype=abi.SUGGESTION_DTYPE)
        if n.value:
            st = ref_lib().ref_suggest_full(self.h, lg.ctypes.data, cg.ctypes.data, C.byref(p), thr_sim,
                                            out.ctypes.data, n.value, C.byref(n))
        if st:
            raise RuntimeError(f"ref_suggest_full status {st}")
        return out

    def fan_metrics(self, n_workers=0):
        m = self.n_methods
        fi, fo = np.empty(m, np.uint32), np.empty(m, np.uint32)
        st = ref_lib().ref_fan_metrics(self.h, n_workers, fi.ctypes.data, fo.ctypes.data)
        if st:
            raise RuntimeError(f"ref_fan_metrics status {st}")
        return fi, fo

    def class_metrics(self, n_workers=0):
        n = self.n_classes
        lcom, ck, cbo = np.empty(n, np.float64), np.empty(n, np.uint64), np.empty(n, np.uint32)
        st = ref_lib().ref_class_metrics(self.h, n_workers, lcom.ctypes.data, ck.ctypes.data, cbo.ctypes.data)
        if st:
            raise RuntimeError(f"ref_class_metrics status {st}")
        return lcom, ck, cbo

    def what_if(self, u, o, d):
        w = abi.mm_whatif()
        st = ref_lib().ref_what_if(self.h, u, o, d, C.byref(w))
        return st, w

    def suggest(self, lcom_gate, cbo_gate, criteria_mask, combine=0, all_candidates=False, thr_lcom=0.0,
                thr_cbo=0.0, by=None):
        lg = np.ascontiguousarray(lcom_gate, np.float64)
        cg = np.ascontiguousarray(cbo_gate, np.uint32)
        p = _params(criteria_mask, combine, all_candidates, 1, thr_lcom, thr_cbo)
        n = C.c_uint64()
        L = ref_lib()

        def call(out, cap):
            if by is None:
                return L.ref_suggest(self.h, lg.ctypes.data, cg.ctypes.data, C.byref(p), out, cap, C.byref(n))
            return L.ref_suggest_by(self.h, by, lg.ctypes.data, cg.ctypes.data, C.byref(p), out, cap, C.byref(n))

        st = call(None, 0)
        if st not in (0, abi.MM_E_CAPACITY):
            return st, None
        out = np.zeros(n.value, dtype=abi.SUGGESTION_DTYPE)
        if n.value:
            st = call(out.ctypes.data, n.value)
        return st, out

    def sweep(self, lcom_gate, cbo_gate, criteria_mask, thr_lcom, thr_cbo, combine=0, all_candidates=False,
              methods=None, n_workers=1, dynamic=True):
        """suggest_all's cohesion/coupling list restricted to `methods` (None =
        all), evaluated by the reference's own per-method code on n_workers
        threads (ref_sweep in ref_shim.cpp). Returns (records, candidates)."""
        lg = np.ascontiguousarray(lcom_gate, np.float64)
        cg = np.ascontiguousarray(cbo_gate, np.uint32)
        p = _params(criteria_mask, combine, all_candidates, 1, thr_lcom, thr_cbo)
        ml = None if methods is None else np.ascontiguousarray(methods, np.uint32)
        nr, nc = C.c_uint64(), C.c_uint64()
        st = ref_lib().ref_sweep(self.h, lg.ctypes.data, cg.ctypes.data, C.byref(p),
                                 None if ml is None else ml.ctypes.data, 0 if ml is None else len(ml), n_workers,
                                 int(dynamic), C.byref(nr), C.byref(nc))
        if st:
            raise RuntimeError(f"ref_sweep status {st}")
        out = np.zeros(nr.value, dtype=abi.SUGGESTION_DTYPE)
        if nr.value:
            st = ref_lib().ref_sweep_copy(self.h, out.ctypes.data, nr.value)
            if st:
                raise RuntimeError(f"ref_sweep_copy status {st}")
        return out, nc.value

    def candidates(self) -> int:
        return int(ref_lib().ref_candidates(self.h))

    def sweep_sample(self, lcom_gate, cbo_gate, thr_lcom, thr_cbo, class_begin, class_end, n_workers):
        lg = np.ascontiguousarray(lcom_gate, np.float64)
        cg = np.ascontiguousarray(cbo_gate, np.uint32)
        ns, nc = C.c_uint64(), C.c_uint64()
        st = ref_lib().ref_sweep_sample(self.h, lg.ctypes.data, cg.ctypes.data, thr_lcom, thr_cbo, class_begin,
                                        class_end, n_workers, C.byref(ns), C.byref(nc))
        if st:
            raise RuntimeError(f"ref_sweep_sample status {st}")
        return ns.value, nc.value


def ref_generate(**cfg) -> CsrSystem:
    """The reference's generate() (generate.hpp:94); zipf_s > 0: config C3's
    skewed ownership with the reference's dependency draws (ref_shim.cpp)."""
    c = abi.mm_gen_config(**cfg)
    h = ref_lib().ref_generate(C.byref(c))
    try:
        return CsrSystem.from_view(ref_lib().ref_model_view(h).contents)
    finally:
        ref_lib().ref_model_free(h)


def ref_generate_model(**cfg) -> "RefModel":
    """generate() straight into a reference model handle (no CSR round trip)."""
    c = abi.mm_gen_config(**cfg)
    return RefModel(handle=ref_lib().ref_generate(C.byref(c)))


def ref_thresholds(lcom, cbo, similarity=None, overrides=None):
    lcom = np.ascontiguousarray(lcom, np.float64)
    cbo = np.ascontiguousarray(cbo, np.uint32)
    sim = np.ascontiguousarray(similarity if similarity is not None else [], np.float64)
    t = abi.mm_thresholds()
    o = _overrides(overrides)
    ref_lib().ref_thresholds(lcom.ctypes.data, cbo.ctypes.data, len(lcom), sim.ctypes.data, len(sim), C.byref(o),
                             C.byref(t))
    return t
