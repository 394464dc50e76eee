"""Facts ingest straight to the engine's CSR (include/mmfacts.h).

Python mirror of the reference's `parse_facts` / `load_facts` / `facts_to_json`
(/root/reference/proj/include/modmetrics/facts.hpp:91-320): same accepted
documents, same model, same warnings, same error classes and messages
(`FactsParseError` <-> ParseError, `FactsValidationError` <-> ValidationError
with `.violations`, `FactsIoError` <-> IoError). The parse runs natively in
libmmgpu.so (one streaming pass, no DOM) and hands back a `System` that
`Engine.upload` takes as-is.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Tuple, Union

from . import abi
from ._lib import MMError, lib
from .system import System

# modmetrics::ViolationKind (model.hpp:72-85)
VIOLATION_KINDS = (
    "NonDenseClassIds", "DuplicateMethodMembership", "DuplicateAttributeMembership", "UnownedMethod",
    "UnownedAttribute", "OwnerMismatch", "DependencyTableSize", "DanglingCallTarget", "DanglingAccessTarget",
    "SelfCall", "UnsortedDependencySet", "UnsupportedSchemaVersion",
)


class FactsParseError(MMError, ValueError):
    """modmetrics::ParseError (facts.hpp:22-24)."""


class FactsValidationError(MMError, ValueError):
    """modmetrics::ValidationError (facts.hpp:28-37); `.violations` = [(kind, message)]."""

    def __init__(self, status: int, msg: str, violations: List[Tuple[str, str]]):
        super().__init__(status, msg)
        self.violations = violations


class FactsIoError(MMError, OSError):
    """modmetrics::IoError (facts.hpp:39-41)."""


class FactsNumberOverflow(MMError, OverflowError):
    """nlohmann::json::out_of_range 406: a float token overflowing a double (escapes parse_facts)."""


@dataclass
class Facts:
    """LoadResult (facts.hpp:43-47) with the model as CSR; names read on demand."""
    system: System
    warnings: List[str] = field(default_factory=list)
    _h: C.c_void_p = None

    def __del__(self):
        if self._h:
            lib().mm_facts_free(self._h)
            self._h = None

    def _name(self, fn, i: int) -> str:
        n = C.c_size_t()
        p = fn(self._h, i, C.byref(n))
        if p is None:
            raise IndexError(i)
        return C.string_at(p, n.value).decode("utf-8")

    def class_name(self, c: int) -> str:
        return self._name(lib().mm_facts_class_name, c)

    def method_name(self, p: int) -> str:
        return self._name(lib().mm_facts_method_name, p)

    def attribute_name(self, a: int) -> str:
        return self._name(lib().mm_facts_attribute_name, a)

    def to_json(self) -> bytes:
        """facts_to_json (facts.hpp:270-320): canonical bytes, trailing newline."""
        n = C.c_size_t()
        lib().mm_facts_to_json(self._h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value)
        st = lib().mm_facts_to_json(self._h, buf, n.value, C.byref(n))
        if st != abi.MM_OK:
            raise MMError(st, "mm_facts_to_json")
        return buf.raw[: n.value]


def _finish(st: int, h: C.c_void_p) -> Facts:
    l = lib()
    if st != abi.MM_OK:
        try:
            msg = l.mm_facts_error(h).decode("utf-8", "replace") if h else "invalid argument"
            if st == abi.MM_E_PARSE:
                raise FactsParseError(st, msg)
            if st == abi.MM_E_IO:
                raise FactsIoError(st, msg)
            if st == abi.MM_E_RANGE:
                raise FactsNumberOverflow(st, "[json.exception.out_of_range.406] " + msg)
            if st == abi.MM_E_VALIDATION:
                vs = []
                for i in range(l.mm_facts_violation_count(h)):
                    kind, m = C.c_int(), C.c_char_p()
                    l.mm_facts_violation(h, i, C.byref(kind), C.byref(m))
                    vs.append((VIOLATION_KINDS[kind.value], m.value.decode("utf-8", "replace")))
                raise FactsValidationError(st, msg, vs)
            if st == abi.MM_E_OOM:
                raise MemoryError(msg)
            raise MMError(st, msg)
        finally:
            if h:
                l.mm_facts_free(h)
    view = abi.mm_system()
    l.mm_facts_system(h, C.byref(view))
    warnings = [l.mm_facts_warning(h, i).decode("utf-8") for i in range(l.mm_facts_warning_count(h))]
    return Facts(System.from_view(view), warnings, h)


def parse_facts(text: Union[str, bytes]) -> Facts:
    """parse_facts (facts.hpp:91)."""
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    st = lib().mm_facts_parse(data, len(data), C.byref(h))
    return _finish(st, h)


def load_facts(path: Union[str, Path]) -> Facts:
    """load_facts (facts.hpp:258)."""
    h = C.c_void_p()
    st = lib().mm_facts_load(str(path).encode(), C.byref(h))
    return _finish(st, h)
