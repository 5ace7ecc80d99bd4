"""Production paths for large E*m that no twin reaches at default settings: the error sets of a
call are processed in chunks (bounded slot arrays / hoist records, csrc/capi.cu run_batch) and
their outputs joined.  PTSBE_CHUNK_SHOTS forces many small chunks; results must equal the
single-chunk run (merged and per-error-set output, one- and two-word keys, proportional and
non-proportional), as the reference's per-set API has no size limit (engine.py:493-524).  Plus
the C-ABI input guards: out-of-range Kraus indices, ragged arrays, batches outliving their plan."""

import os

import numpy as np
import pytest

from paper_2604_08467_b200 import workloads
from paper_2604_08467_b200.engine import (
    BatchPlan, CircuitNetwork, DevicePipeline, SamplerContext, VariantTables,
)
from paper_2604_08467_b200.errors import DeviceError

pytestmark = pytest.mark.gpu


def _pipe(c, sizes, shots, chunk_shots=None, dtype="complex128", **plan_kw):
    tpl = CircuitNetwork.from_circuit(c)
    old = os.environ.get("PTSBE_CHUNK_SHOTS")
    if chunk_shots is not None:
        os.environ["PTSBE_CHUNK_SHOTS"] = str(chunk_shots)
    try:
        return DevicePipeline(tpl, BatchPlan(sizes, **plan_kw), VariantTables.from_channels(tpl),
                              SamplerContext(hypersamples=4, dtype=dtype), shots_per_set=float(shots))
    finally:
        if chunk_shots is not None:
            if old is None:
                del os.environ["PTSBE_CHUNK_SHOTS"]
            else:
                os.environ["PTSBE_CHUNK_SHOTS"] = old


def _cases():
    c1, _ = workloads.hea(10, 3, gamma=0.05, p=0.08, seed=3)      # one-word keys
    c2, _ = workloads.random40(70, 260, seed=7)                   # 70 qubits: two-word keys
    return [("hea10", c1, (4, 3, 3)), ("random70", c2, (10, 8, 8, 8, 8, 8, 8, 6, 6))]


@pytest.mark.parametrize("which", [0, 1])
def test_multi_chunk_outputs_equal_single_chunk(which):
    name, c, sizes = _cases()[which]
    sets, shots, seed = 23, 60, 5
    rows = workloads.presample_matrix(c, sets, np.random.default_rng(8))
    sh = np.full(sets, shots, np.uint32)
    sh[::5] = 7
    ids = (np.arange(sets, dtype=np.uint32) * 3 + 11)
    one, many = _pipe(c, sizes, shots), _pipe(c, sizes, shots, chunk_shots=150)
    try:
        for merged in (True, False):
            k1, e1, c1, s1 = one.device_plan.sample(rows, sh, ids, seed, merged=merged)
            k2, e2, c2, s2 = many.device_plan.sample(rows, sh, ids, seed, merged=merged)
            assert int(s1.n_chunks) == 1 and int(s2.n_chunks) > 3, (name, int(s2.n_chunks))
            np.testing.assert_array_equal(k1, k2)
            np.testing.assert_array_equal(c1, c2)
            if not merged:
                np.testing.assert_array_equal(e1, e2)
                assert int(c2.sum()) == int(sh.sum()) or int(s2.flagged_sets) > 0
                assert np.all(np.diff(e2.astype(np.int64)) >= 0)  # records grouped by error set, in order
            assert [int(s1.stage_events[j]) for j in range(len(sizes))] == \
                   [int(s2.stage_events[j]) for j in range(len(sizes))]
    finally:
        one.close()
        many.close()


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_packed_records_equal_the_wide_histogram(dtype):
    """ptsbe_sample_packed: the merged histogram as (key, count) rows of two u32 -- the same records as
    ptsbe_sample(merged), single- and multi-chunk; refused for plans of more than 32 measured qubits."""
    name, c, sizes = _cases()[0]
    sets, shots, seed = 23, 60, 5
    rows = workloads.presample_matrix(c, sets, np.random.default_rng(8))
    sh = np.full(sets, shots, np.uint32)
    sh[::5] = 7
    ids = (np.arange(sets, dtype=np.uint32) * 3 + 11)
    one, many = _pipe(c, sizes, shots, dtype=dtype), _pipe(c, sizes, shots, chunk_shots=150, dtype=dtype)
    try:
        k, _, cnt, s0 = one.device_plan.sample(rows, sh, ids, seed, merged=True)
        for pipe in (one, many):
            rec, st = pipe.device_plan.sample_packed(rows, sh, ids, seed)
            assert rec.dtype == np.uint32 and rec.shape == (k.shape[0], 2)
            np.testing.assert_array_equal(rec[:, 0].astype(np.uint64) << np.uint64(32), k[:, 0])
            np.testing.assert_array_equal(rec[:, 1].astype(np.uint64), cnt)
            assert int(st.d2h_bytes) == 8 * rec.shape[0] and int(s0.d2h_bytes) == 16 * rec.shape[0]
            assert int(st.n_records) == rec.shape[0]
    finally:
        one.close()
        many.close()
    _, c2, sizes2 = _cases()[1]
    wide = _pipe(c2, sizes2, 4)
    try:
        rows2 = workloads.presample_matrix(c2, 2, np.random.default_rng(1))
        with pytest.raises(ValueError, match="32 measured qubits"):
            wide.device_plan.sample_packed(rows2, np.full(2, 4, np.uint32), None, 1)
    finally:
        wide.close()


@pytest.mark.parametrize("final_mode", ["exhaustive", "direct"])
def test_nonproportional_multi_chunk_equals_single_chunk(final_mode):
    c, _ = workloads.hea(10, 3, gamma=0.05, p=0.08, seed=3)
    sizes, sets = (4, 3, 3), 17
    rows = workloads.presample_matrix(c, sets, np.random.default_rng(9))
    ids = np.arange(100, 100 + sets, dtype=np.uint32)
    kw = dict(nonfinal_shots=3, final_mode=final_mode, threshold=1e-3, direct_count=5)
    one, many = _pipe(c, sizes, 3, **kw), _pipe(c, sizes, 3, chunk_shots=200, **kw)
    try:
        a = one.device_plan.sample_nonproportional(rows, ids, 21, 3, final_mode, 1e-3, 5)
        b = many.device_plan.sample_nonproportional(rows, ids, 21, 3, final_mode, 1e-3, 5)
        assert int(a[4].n_chunks) == 1 and int(b[4].n_chunks) > 1
        for x, y in zip(a[:3], b[:3]):
            np.testing.assert_array_equal(x, y)
        if final_mode == "exhaustive":
            np.testing.assert_array_equal(a[3], b[3])
    finally:
        one.close()
        many.close()


def test_capi_rejects_bad_inputs_and_outlived_batches():
    c, _ = workloads.hea(6, 2, gamma=0.05, p=0.05, seed=1)
    g = len(c.gates)
    pipe = _pipe(c, (3, 3), 10)
    dp = pipe.device_plan
    rows = np.zeros((4, g), np.uint8)
    sh = np.full(4, 10, np.uint32)
    with pytest.raises(ValueError):
        dp.sample(rows[:, :-1], sh, None, 1)                    # wrong number of sites
    with pytest.raises(ValueError):
        dp.sample(rows, sh[:3], None, 1)                        # ragged shots
    with pytest.raises(ValueError):
        dp.sample(rows, sh, np.arange(5, dtype=np.uint32), 1)   # ragged ids
    bad = rows.copy()
    bad[2, 1] = 200                                             # no such variant at this site
    with pytest.raises(ValueError, match="out of range"):
        dp.sample(bad, sh, None, 1)
    with pytest.raises(ValueError, match="out of range"):
        dp.marginals(1, bad, np.zeros((4, dp.words), np.uint64))
    bt = dp.upload(rows, sh)
    n, _ = bt.run(3)
    assert n > 0
    pipe.close()                                                # closes the batch with the plan
    with pytest.raises(DeviceError):
        bt.run(3)
    bt.close()                                                  # harmless afterwards
    del bt
