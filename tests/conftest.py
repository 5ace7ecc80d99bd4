"""Shared fixtures.  `-m "not gpu"` runs on a CPU-only box (oracle vs golden
vectors, host logic, compiler vs oracle through a numpy emulation of the
device program format, C-ABI symbol table, gloo sharding); `-m gpu` are the
parity tests proper and go through the C-ABI of libptsbe_b200.so."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_cases.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as fp:
        return json.load(fp)


@pytest.fixture(scope="session")
def golden_cases(golden):
    return {c["name"]: c for c in golden["cases"]}


def case_objects(case):
    """(Circuit, sizes, [ErrorSet]) of one golden case."""
    from paper_2604_08467_b200.circuits import circuit_from_json
    from paper_2604_08467_b200.engine import ErrorSet

    c = circuit_from_json(case["circuit"])
    es = [ErrorSet(id=k["id"], realized=tuple(k["realized"]), m=k["m"]) for k in case["errorsets"]]
    return c, tuple(case["sizes"]), es


@pytest.fixture(scope="session")
def have_gpu():
    from paper_2604_08467_b200 import _capi

    return _capi.device_count() > 0


@pytest.fixture(autouse=True)
def _gpu_guard(request):
    if request.node.get_closest_marker("gpu"):
        from paper_2604_08467_b200 import _capi

        if _capi.device_count() < 1:
            pytest.skip("no CUDA device")


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
