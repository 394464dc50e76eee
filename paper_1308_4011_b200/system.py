"""Host-side system snapshots: SystemModel + DependencyTable in CSR form.

`System` mirrors the reference's input types (model.hpp:19-53) as flat u32
numpy arrays — exactly the layout the C ABI (`mm_system`, include/mmgpu.h)
uploads. Constructors:

* `System.build(classes, calls, accesses)` — fixtures::build_system
  (tests/support/fixtures.hpp:22-69): explicit memberships, lists sorted and
  deduplicated.
* `System.from_facts(obj)` — the facts JSON schema (facts.hpp:91-256 semantics:
  self-calls dropped, dependency lists sorted+deduplicated, ids dense).
* `System.generate(...)` — the reference generator (generate.hpp:94), native
  via libmmgpu's `mm_generate`; `zipf_s > 0` gives the skewed C3 variant.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np

from . import abi

_FIELDS = ("method_owner", "attribute_owner", "class_method_off", "class_methods", "class_attr_off",
           "class_attrs", "call_off", "call_tgt", "acc_off", "acc_tgt")


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _csr(rows: Sequence[Sequence[int]]):
    off = np.zeros(len(rows) + 1, dtype=np.uint32)
    if rows:
        off[1:] = np.cumsum([len(r) for r in rows])
    flat = np.fromiter((v for r in rows for v in r), dtype=np.uint32, count=int(off[-1]))
    return off, flat


@dataclass
class System:
    n_classes: int
    n_methods: int
    n_attributes: int
    method_owner: np.ndarray
    attribute_owner: np.ndarray
    class_method_off: np.ndarray
    class_methods: np.ndarray
    class_attr_off: np.ndarray
    class_attrs: np.ndarray
    call_off: np.ndarray
    call_tgt: np.ndarray
    acc_off: np.ndarray
    acc_tgt: np.ndarray

    # ---- constructors -------------------------------------------------
    @classmethod
    def build(cls, classes: Sequence[tuple], calls: Sequence[Sequence[int]] = (),
              accesses: Sequence[Sequence[int]] = ()) -> "System":
        """classes = [(attribute_ids, method_ids), ...] (fixtures.hpp:22-69)."""
        n_m = sum(len(m) for _, m in classes)
        n_a = sum(len(a) for a, _ in classes)
        mo = np.zeros(n_m, dtype=np.uint32)
        ao = np.zeros(n_a, dtype=np.uint32)
        mem_m, mem_a = [], []
        for ci, (attrs, methods) in enumerate(classes):
            a_sorted = sorted(attrs)
            m_sorted = sorted(methods)
            mem_a.append(a_sorted)
            mem_m.append(m_sorted)
            for p in m_sorted:
                mo[p] = ci
            for a in a_sorted:
                ao[a] = ci
        calls = [sorted(set(r)) for r in list(calls) + [[]] * (n_m - len(calls))]
        accesses = [sorted(set(r)) for r in list(accesses) + [[]] * (n_m - len(accesses))]
        cmo, cm = _csr(mem_m)
        cao, ca = _csr(mem_a)
        co, ct = _csr(calls)
        ao_, at = _csr(accesses)
        return cls(len(classes), n_m, n_a, mo, ao, cmo, cm, cao, ca, co, ct, ao_, at)

    @classmethod
    def from_facts(cls, obj) -> "System":
        """Facts JSON (facts.hpp schema): dict, JSON text/bytes or a path. Parsed
        natively (mmfacts.h) with the reference's parse_facts semantics; errors
        raise facts.FactsParseError / FactsValidationError (ValueError) or
        FactsIoError."""
        from .facts import load_facts, parse_facts
        if isinstance(obj, dict):
            return parse_facts(json.dumps(obj)).system
        if isinstance(obj, Path) or (isinstance(obj, str) and not obj.lstrip().startswith(("{", "[")) and Path(obj).exists()):
            return load_facts(obj).system
        return parse_facts(obj).system

    @classmethod
    def generate(cls, seed: int, n_classes: int, n_methods: int, n_attributes: int,
                 k_max_calls: int = 4, k_max_accesses: int = 4, intra_class_bias: float = 0.5,
                 zipf_s: float = 0.0) -> "System":
        from ._lib import lib, check
        cfg = abi.mm_gen_config(seed=seed, n_classes=n_classes, n_methods=n_methods,
                                n_attributes=n_attributes, k_max_calls=k_max_calls,
                                k_max_accesses=k_max_accesses, intra_class_bias=intra_class_bias,
                                zipf_s=zipf_s)
        h = C.c_void_p()
        check(lib().mm_generate(C.byref(cfg), C.byref(h)), None, "mm_generate")
        try:
            return cls.from_view(lib().mm_host_system_view(h).contents)
        finally:
            lib().mm_host_system_free(h)

    @classmethod
    def from_view(cls, v: abi.mm_system) -> "System":
        nc, nm, na = v.n_classes, v.n_methods, v.n_attributes

        def take(ptr, n):
            if n == 0:
                return np.zeros(0, dtype=np.uint32)
            return np.ctypeslib.as_array(ptr, shape=(n,)).copy()

        call_off = take(v.call_off, nm + 1)
        acc_off = take(v.acc_off, nm + 1)
        return cls(nc, nm, na,
                   take(v.method_owner, nm), take(v.attribute_owner, na),
                   take(v.class_method_off, nc + 1), take(v.class_methods, nm),
                   take(v.class_attr_off, nc + 1), take(v.class_attrs, na),
                   call_off, take(v.call_tgt, int(call_off[-1])),
                   acc_off, take(v.acc_tgt, int(acc_off[-1])))

    # ---- views --------------------------------------------------------
    def __post_init__(self):
        for f in _FIELDS:
            setattr(self, f, _u32(getattr(self, f)))

    def as_c(self) -> abi.mm_system:
        """mm_system pointing into this object's arrays (keep `self` alive)."""
        s = abi.mm_system(n_classes=self.n_classes, n_methods=self.n_methods, n_attributes=self.n_attributes)
        for f in _FIELDS:
            setattr(s, f, getattr(self, f).ctypes.data_as(abi.U32P))
        return s

    @property
    def n_calls(self) -> int:
        return int(self.call_off[-1])

    @property
    def n_accesses(self) -> int:
        return int(self.acc_off[-1])

    def members(self, c: int) -> np.ndarray:
        return self.class_methods[self.class_method_off[c]:self.class_method_off[c + 1]]

    def attrs(self, c: int) -> np.ndarray:
        return self.class_attrs[self.class_attr_off[c]:self.class_attr_off[c + 1]]

    def calls(self, p: int) -> np.ndarray:
        return self.call_tgt[self.call_off[p]:self.call_off[p + 1]]

    def accesses(self, p: int) -> np.ndarray:
        return self.acc_tgt[self.acc_off[p]:self.acc_off[p + 1]]

    def used_classes(self) -> np.ndarray:
        """|used_classes(u)| per method (suggest.hpp:152-159), vectorised."""
        own = self.method_owner
        rows_c = np.repeat(np.arange(self.n_methods, dtype=np.int64), np.diff(self.call_off))
        rows_a = np.repeat(np.arange(self.n_methods, dtype=np.int64), np.diff(self.acc_off))
        rows = np.concatenate([rows_c, rows_a])
        owners = np.concatenate([self.method_owner[self.call_tgt], self.attribute_owner[self.acc_tgt]]).astype(np.int64)
        keep = owners != own[rows]
        key = np.unique(rows[keep] * (self.n_classes + 1) + owners[keep])
        return np.bincount(key // (self.n_classes + 1), minlength=self.n_methods)

    def n_candidates(self) -> int:
        """N_cand = Σ_u |used_classes(u)|."""
        return int(self.used_classes().sum())

    def nbytes(self) -> int:
        return sum(getattr(self, f).nbytes for f in _FIELDS)

    def equals(self, other: "System") -> bool:
        return (self.n_classes, self.n_methods, self.n_attributes) == (
            other.n_classes, other.n_methods, other.n_attributes) and all(
            np.array_equal(getattr(self, f), getattr(other, f)) for f in _FIELDS)

    def digest(self) -> str:
        import hashlib
        h = hashlib.sha256()
        h.update(np.array([self.n_classes, self.n_methods, self.n_attributes], dtype=np.uint64).tobytes())
        for f in _FIELDS:
            h.update(getattr(self, f).tobytes())
        return h.hexdigest()
