"""Facts ingest (include/mmfacts.h, paper_1308_4011_b200.facts) against the
reference's parse_facts / load_facts / facts_to_json (facts.hpp:91-320).

* golden outcomes: tests/golden/facts/outcomes.json holds the reference's own
  outcome (exception type, what(), violations, warnings, canonical bytes) for
  86 documents — test_facts.cpp's cases, shape/violation/syntax errors at
  every level; made by `oracle/_ref/facts_parity --golden` (the reference
  compiled in place);
* generated systems round-trip through the canonical text into the same CSR;
* the C++ harness (reference vs drop-in in one binary, plus a 20k-document
  mutation fuzz) when oracle/_ref was built here;
* on a GPU: a parsed system uploads straight to the engine and gives the same
  metrics as the generator's CSR.
All host-only except the last."""
import json
import resource
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1308_4011_b200 import (Engine, FactsIoError, FactsNumberOverflow, FactsParseError, FactsValidationError,
                                  System, load_facts, parse_facts)
from paper_1308_4011_b200._lib import FACTS_EXPORTED, lib
from paper_1308_4011_b200.facts import VIOLATION_KINDS

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden" / "facts" / "outcomes.json"
HARNESS = ROOT / "oracle" / "_ref" / "facts_parity"

_TYPE = {FactsParseError: "ParseError", FactsValidationError: "ValidationError", FactsIoError: "IoError",
         FactsNumberOverflow: "json::out_of_range"}


def _outcome(doc: bytes):
    try:
        f = parse_facts(doc)
    except (FactsParseError, FactsValidationError, FactsIoError, FactsNumberOverflow) as e:
        vs = [(VIOLATION_KINDS.index(k), m) for k, m in getattr(e, "violations", [])]
        return _TYPE[type(e)], str(e).split(": ", 1)[1], vs, [], b""
    return "none", "", [], f.warnings, f.to_json()


def test_mmfacts_symbols_exported():
    import re
    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "mmfacts.h").read_text(), flags=re.S)
    names = sorted(set(re.findall(r"\b(mm_facts_[a-z_]+)\s*\(", text)))
    assert len(names) == 14
    l = lib()
    for n in names:
        assert hasattr(l, n), n
    assert set(names) == set(FACTS_EXPORTED)


def _golden():
    return json.loads(GOLDEN.read_text())


@pytest.mark.parametrize("i", range(len(_golden())))
def test_golden_outcome(i):
    g = _golden()[i]
    doc = bytes.fromhex(g["doc"])
    typ, what, vs, warnings, canon = _outcome(doc)
    assert typ == g["type"], (doc, what)
    if typ != "none":
        assert what == bytes.fromhex(g["what"]).decode("utf-8")
    assert vs == [(k, bytes.fromhex(m).decode("utf-8")) for k, m in g["violations"]]
    assert warnings == [bytes.fromhex(w).decode("utf-8") for w in g["warnings"]]
    assert canon == bytes.fromhex(g["canonical"])


def test_reference_examples():
    """test_facts.cpp:26-37, :119-138 restated."""
    f = parse_facts('{"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [{"id": 0, "name": "x"}],'
                    ' "methods": [{"id": 0, "name": "f", "calls": [1, 1, 0], "accesses": [0, 0]},'
                    ' {"id": 1, "name": "g", "calls": [], "accesses": []}]}]}')
    s = f.system
    assert (s.n_classes, s.n_methods, s.n_attributes) == (1, 2, 1)
    assert f.class_name(0) == "A" and f.method_name(0) == "f" and f.attribute_name(0) == "x"
    assert list(s.calls(0)) == [1] and list(s.accesses(0)) == [0]
    assert f.warnings == ["method 0 calls itself; self-call dropped"]
    with pytest.raises(FactsParseError, match="line 3, column"):
        parse_facts('{\n  "schema_version": "1",\n  !\n}')
    with pytest.raises(FactsValidationError) as e:
        parse_facts('{"schema_version": "2", "classes": []}')
    assert e.value.violations == [("UnsupportedSchemaVersion", 'schema_version must be "1", got "2"')]
    assert isinstance(e.value, ValueError)


def test_load_facts_io(tmp_path):
    with pytest.raises(FactsIoError, match="cannot open /nonexistent/x.json"):
        load_facts("/nonexistent/x.json")
    p = tmp_path / "f.json"
    p.write_text('{"classes": [], "schema_version": "1"}')
    f = load_facts(p)
    assert f.system.n_classes == 0 and f.to_json() == b'{"classes":[],"schema_version":"1"}\n'
    # a directory opens and reads as nothing under std::ifstream, and so does an
    # empty file: the reference then fails to parse "" (checked against it by hand)
    empty = tmp_path / "empty.json"
    empty.write_bytes(b"")
    for q in (tmp_path, empty):
        with pytest.raises(FactsParseError, match=r"facts: JSON parse error at line 1, column 1$"):
            load_facts(q)


def _canonical(s: System) -> str:
    """facts_to_json's layout (keys sorted, compact) built from a System."""
    classes = []
    for c in range(s.n_classes):
        classes.append({
            "attributes": [{"id": int(a), "name": f"a{a}"} for a in s.attrs(c)],
            "id": c,
            "methods": [{"accesses": [int(x) for x in s.accesses(p)], "calls": [int(x) for x in s.calls(p)],
                         "id": int(p), "name": f"m{p}"} for p in s.members(c)],
            "name": f"C{c}",
        })
    return json.dumps({"classes": classes, "schema_version": "1"}, separators=(",", ":"), sort_keys=True) + "\n"


@pytest.mark.parametrize("cfg", [(1, 1000, 10000, 20000, 4, 4, 0.5), (42, 5, 30, 12, 3, 3, 0.6),
                                 (7, 300, 4000, 900, 6, 9, 0.9)])
def test_generated_roundtrip(cfg):
    s = System.generate(*cfg)
    text = _canonical(s)
    f = parse_facts(text)
    assert f.system.equals(s)
    assert f.to_json() == text.encode()
    assert f.method_name(int(s.members(0)[0])) == f"m{int(s.members(0)[0])}"
    # key order and whitespace do not matter; System.from_facts goes the same way
    obj = json.loads(text)
    assert System.from_facts(json.dumps(obj, indent=2)[::1]).equals(s)
    assert System.from_facts(obj).equals(s)


def test_number_overflow_is_not_a_parse_error():
    with pytest.raises(FactsNumberOverflow, match=r"\[json.exception.out_of_range.406\] number overflow parsing '1e400'"):
        parse_facts('{"a": 1e400}')
    with pytest.raises(FactsParseError):  # unexpected token first
        parse_facts('{"a" 1e400}')


def _limit_memory():
    resource.setrlimit(resource.RLIMIT_AS, (8 << 30, 8 << 30))


@pytest.mark.skipif(not HARNESS.exists(), reason="oracle/_ref/facts_parity not built (needs /root/reference)")
def test_cpp_harness_reference_vs_dropin():
    # the reference grows its id tables to max id + 1 (facts.hpp:146-149); the
    # address-space limit turns the fuzz's absurd ids into bad_alloc on both sides
    res = subprocess.run([str(HARNESS), "20000"], capture_output=True, text=True, timeout=600,
                         preexec_fn=_limit_memory)
    assert res.returncode == 0, res.stdout[-3000:]
    assert "PASS" in res.stdout


@pytest.mark.skipif(not HARNESS.exists(), reason="oracle/_ref/facts_parity not built (needs /root/reference)")
def test_cpp_harness_parallel_reader():
    # every document through the speculative parallel reader (chunks guessed,
    # verified by the sequential walk), against the reference
    import os
    env = dict(os.environ, MMGPU_FACTS_PAR_MIN="1", MMGPU_FACTS_THREADS="5")
    res = subprocess.run([str(HARNESS), "10000"], capture_output=True, text=True, timeout=600,
                         preexec_fn=_limit_memory, env=env)
    assert res.returncode == 0, res.stdout[-3000:]
    assert "PASS" in res.stdout


@pytest.mark.parametrize("threads", ["2", "7"])
def test_parallel_reader_equals_sequential(monkeypatch, threads):
    s = System.generate(3, 400, 6000, 3000, 5, 7, 0.3)
    text = _canonical(s)
    spaced = text.replace(",", ", ").replace("{", "{\n ")
    monkeypatch.setenv("MMGPU_FACTS_PAR_MIN", "1")
    monkeypatch.setenv("MMGPU_FACTS_THREADS", threads)
    for doc in (text, spaced):
        f = parse_facts(doc)
        assert f.system.equals(s) and f.to_json() == text.encode()


@pytest.mark.gpu
def test_parsed_system_uploads():
    s = System.generate(1, 1000, 10000, 20000, 4, 4, 0.5)
    f = parse_facts(_canonical(s))
    a, b = Engine(0), Engine(0)
    a.upload(f.system)
    b.upload(s)
    a.compute_metrics()
    b.compute_metrics()
    for x, y in zip(a.class_metrics_all(), b.class_metrics_all()):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))


@pytest.mark.parametrize("bad_at", [40000, 1, 399999])
def test_large_document_non_object_class(bad_at):
    # ≥ 8 MB takes the parallel reader + optimistic parallel walk: the id
    # tables are presized only up to the first non-object class, so that walk
    # must not run (it once wrote past the tables: ADVICE r1 facts.cpp:877).
    # The reference stops at that element with a ParseError.
    n = 400000
    parts = [f'{{"attributes":[{{"id":{c},"name":"a{c}"}}],"id":{c},'
             f'"methods":[{{"accesses":[{c}],"calls":[],"id":{c},"name":"m{c}"}}],"name":"C{c}"}}'
             for c in range(n)]
    parts[bad_at] = "null"
    doc = '{"classes":[' + ",".join(parts) + '],"schema_version":"1"}\n'
    assert len(doc) > 8 << 20
    with pytest.raises(FactsParseError, match=rf"classes\[{bad_at}\]: expected an object$"):
        parse_facts(doc)
    # a well-formed document of the same size parses (parallel walk taken)
    parts[bad_at] = (f'{{"attributes":[{{"id":{bad_at},"name":"a"}}],"id":{bad_at},'
                     f'"methods":[{{"accesses":[],"calls":[],"id":{bad_at},"name":"m"}}],"name":"C"}}')
    f = parse_facts('{"classes":[' + ",".join(parts) + '],"schema_version":"1"}\n')
    assert f.system.n_classes == n and f.system.n_methods == n
