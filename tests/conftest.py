import gzip
import json
import pathlib
import sys

import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = REPO / "tests" / "golden"



def pytest_terminal_summary(terminalreporter):
    """Numeric parity margins (max-abs error vs the test's tolerance) of the GPU tests that ran."""
    try:
        from mvtest import MARGINS
    except Exception:
        return
    if not MARGINS:
        return
    terminalreporter.section("parity margins (max-abs error / tolerance)")
    worst = max(MARGINS, key=lambda m: m[1] / m[2])
    for name, err, tol in MARGINS:
        terminalreporter.write_line(f"{err:.3e} / {tol:.0e}  ({err / tol:5.1%})  {name}")
    terminalreporter.write_line(f"worst: {worst[0]} at {worst[1] / worst[2]:.1%} of its tolerance")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through the C-ABI library")


def load_jsonl(name):
    with gzip.open(GOLDEN / name, "rt") as f:
        return [json.loads(line) for line in f if line.strip()]


@pytest.fixture(scope="session")
def dag_golden():
    return load_jsonl("dag.jsonl.gz")


@pytest.fixture(scope="session")
def toy_golden():
    return {r["name"]: r for r in load_jsonl("toy.jsonl.gz")}


def kv_logs():
    return sorted(p.name for p in GOLDEN.glob("kv_*.jsonl.gz"))


def fnv1a(data: bytes) -> str:
    h = 1469598103934665603
    for b in data:
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
