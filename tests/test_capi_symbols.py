"""The C-ABI library loads on a CPU-only box, exports every symbol that
include/ptsbe_b200.h declares, and refuses to compute without a device."""

import os
import re

import numpy as np
import pytest

from paper_2604_08467_b200 import _capi
from paper_2604_08467_b200.errors import DeviceError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "ptsbe_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ptsbe_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_are_exported():
    lib = _capi.load()
    names = _declared()
    assert len(names) >= 19
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_capi.EXPORTS) == names


def test_version_and_device_count():
    lib = _capi.load()
    assert b"sm_100a" in lib.ptsbe_version()
    assert _capi.device_count() >= 0


def test_no_cpu_fallback():
    if _capi.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(DeviceError):
        _capi.histogram_merge(np.zeros((1, 1), np.uint64), np.ones(1, np.uint64))
    with pytest.raises(DeviceError):
        _capi.sample_stage(1, 1, 0, np.ones((1, 2)), [1], [0], [0])
    from paper_2604_08467_b200.tensor import Index, Tensor, contract_pair

    with pytest.raises(DeviceError):
        contract_pair(Tensor([Index(0, 2)], [1, 0]), Tensor([Index(0, 2)], [1, 0]))
    # the widened rows (non-proportional sampler, run_ptsbe in both modes) have no CPU path either
    from paper_2604_08467_b200 import workloads
    from paper_2604_08467_b200.engine import (BatchPlan, CircuitNetwork, ErrorSet, RunConfig, run_ptsbe,
                                              sample_nonproportional)

    c, sizes = workloads.ghz(4, p=0.1)
    k = ErrorSet(0, tuple("I" * len(g.targets) for g in c.gates), 1)
    with pytest.raises(DeviceError):
        sample_nonproportional(CircuitNetwork.from_circuit(c), k, BatchPlan(sizes), np.random.default_rng(0))
    for mode in ("ptsbe-proportional", "ptsbe-nonproportional"):
        with pytest.raises(DeviceError):
            run_ptsbe(c, RunConfig(n=4, g=len(c.gates), mode=mode, batch_sizes=sizes, error_sets=2, total_shots=4,
                                   hypersamples=2))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_08467_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
