import json
import struct
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


def unhex(h: str) -> float:
    return struct.unpack("<d", bytes.fromhex(h))[0]


def golden_names():
    return sorted(p.stem for p in GOLDEN.glob("*.json"))


def load_golden(name: str) -> dict:
    return json.loads((GOLDEN / f"{name}.json").read_text())


def golden_system(case: dict):
    from paper_1308_4011_b200 import System
    spec = case["system"]
    if "generate" in spec:
        s = System.generate(**spec["generate"])
    else:
        b = spec["build"]
        s = System.build([tuple(c) for c in b["classes"]], b["calls"], b["accesses"])
    assert s.digest() == case["digest"], "fixture system drifted"
    return s


def golden_records(recs) -> np.ndarray:
    from paper_1308_4011_b200 import SUGGESTION_DTYPE
    out = np.zeros(len(recs), dtype=SUGGESTION_DTYPE)
    for i, r in enumerate(recs):
        for k, v in r.items():
            out[i][k] = unhex(v) if k.startswith("lcom") else v
    return out


def records_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """Bitwise equality of two mm_suggestion arrays (pad bytes ignored)."""
    if len(a) != len(b):
        return False
    fields = [f for f in a.dtype.names if f != "pad"]
    return all(a[f].tobytes() == b[f].tobytes() for f in fields)


def first_diff(a: np.ndarray, b: np.ndarray) -> str:
    n = min(len(a), len(b))
    for i in range(n):
        if not records_equal(a[i:i + 1], b[i:i + 1]):
            return f"len {len(a)} vs {len(b)}; first diff at {i}: {a[i]} vs {b[i]}"
    return f"len {len(a)} vs {len(b)}"


@pytest.fixture(scope="session")
def gpu_engine():
    from paper_1308_4011_b200 import Engine
    e = Engine(0)
    yield e
    e.close()
