"""Parity of the CUDA path (through the C-ABI of libptsbe_b200.so) against the
oracle and the golden vectors of the unmodified reference.

Tolerances (BASELINE.json north_star): marginals within 1e-11 (complex128) and
1e-5 relative (complex64); sampler counts bit-exact given the same float64
marginals and the same uniforms; complex128 end-to-end histograms bit-exact
against the reference-with-shim goldens; complex64 end-to-end by TVD."""

import numpy as np
import pytest

from conftest import case_objects
from oracle import bridge
from oracle import ptsbe_oracle as O
from paper_2604_08467_b200 import _capi, workloads
from paper_2604_08467_b200.engine import (
    BatchPlan, CircuitNetwork, ErrorSet, RunConfig, SamplerContext, conditional_marginal,
    conditional_marginals_batched, merge_records, run_ptsbe, sample_proportional,
    sample_proportional_batched, ShotRecord, presample_errors, DevicePipeline, VariantTables,
)
from paper_2604_08467_b200.errors import ImpossiblePrefixError
from paper_2604_08467_b200.planner import PathCache
from paper_2604_08467_b200.tensor import Index, Tensor, TensorNetwork, contract_pair, execute_path
from paper_2604_08467_b200.circuits import Circuit, Gate, NoiseChannel

pytestmark = pytest.mark.gpu

ALL = ["ghz12", "ghz6_per_qubit", "random_0", "random_1", "random_2", "random_3", "random_4", "random_5",
       "hea8", "qaoa8", "surface_d3_r1", "random10x40"]


def _marginal_rows(case):
    c, sizes, es = case_objects(case)
    by_stage = {}
    for row in case["marginals"]:
        by_stage.setdefault(row["stage"], []).append(row)
    return c, sizes, es, by_stage


@pytest.mark.parametrize("name", ALL)
@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-11), ("complex64", 1e-5)])
def test_marginals_match_reference_goldens(golden_cases, name, dtype, tol):
    c, sizes, es, by_stage = _marginal_rows(golden_cases[name])
    tpl = CircuitNetwork.from_circuit(c)
    for j, rows in by_stage.items():
        ctx = SamplerContext(hypersamples=4, dtype=dtype)
        got = conditional_marginals_batched(tpl, [es[r["eset"]] for r in rows], BatchPlan(sizes), j,
                                            [r["prefix"] for r in rows], ctx)
        want = np.asarray([r["probs"] for r in rows])
        assert got.shape == want.shape
        err = np.max(np.abs(got - want), axis=1) / np.max(want, axis=1)
        assert err.max() <= tol, (name, j, err.max())


def test_single_item_conditional_marginal_signature(golden_cases):
    """Reference signature conditional_marginal(cnet, cache, plan, j, prefix)."""
    case = golden_cases["random_4"]
    c, sizes, es = case_objects(case)
    tpl = CircuitNetwork.from_circuit(c)
    for row in case["marginals"][:4]:
        got = conditional_marginal(tpl.merged(es[row["eset"]]), PathCache(), BatchPlan(sizes), row["stage"],
                                   row["prefix"], hypersamples=2)
        np.testing.assert_allclose(got, row["probs"], atol=1e-11, rtol=0)


def test_bell_kats():
    c = Circuit(2, (Gate("H", (0,)), Gate("CX", (0, 1), None, NoiseChannel("depolarizing", 0.0))))
    tpl = CircuitNetwork.from_circuit(c)
    cache = PathCache()
    np.testing.assert_allclose(conditional_marginal(tpl, cache, BatchPlan((2,)), 1, ""), [0.5, 0, 0, 0.5], atol=1e-12)
    np.testing.assert_allclose(conditional_marginal(tpl, cache, BatchPlan((1, 1)), 2, "1"), [0, 1], atol=1e-12)


def test_sampler_bit_exact_against_oracle_draws():
    """Same float64 marginals + same Philox uniforms -> identical counts."""
    rng = np.random.default_rng(3)
    for b in (1, 2, 5, 10):
        w = 37
        probs = rng.random((w, 1 << b)) ** 3
        probs[rng.random(probs.shape) < 0.3] = 0.0
        probs[:, 0] += 1e-3
        mult = rng.integers(1, 5000, size=w).astype(np.uint32)
        mult[0] = 1
        eset = rng.integers(0, 1000, size=w).astype(np.uint32)
        rank = rng.integers(0, 50, size=w).astype(np.uint32)
        item, index, count = _capi.sample_stage(b, 3, 0xDEADBEEFCAFE, probs, mult, eset, rank)
        pos = 0
        for i in range(w):
            want = O.multinomial_counts(probs[i], int(mult[i]), 0xDEADBEEFCAFE, int(eset[i]), 3, int(rank[i]))
            nz = np.flatnonzero(want)
            sl = slice(pos, pos + nz.size)
            assert np.all(item[sl] == i)
            assert index[sl].tolist() == nz.tolist()
            assert count[sl].tolist() == want[nz].tolist()
            pos += nz.size
        assert pos == item.size


def test_warp_sampler_bit_exact_on_large_batches():
    """Many work items with few shots each take the warp-per-item sampler
    (sample_warp_kernel); its counts must equal the oracle's as well."""
    rng = np.random.default_rng(8)
    for b in (1, 3, 5, 8, 10, 11):
        w = 4000
        probs = rng.random((w, 1 << b)) ** 4
        probs[rng.random(probs.shape) < 0.4] = 0.0
        probs[np.arange(w), rng.integers(0, 1 << b, size=w)] += 0.05
        mult = rng.integers(1, 4, size=w).astype(np.uint32)
        mult[:50] = rng.integers(40, 400, size=50)
        eset = rng.integers(0, 5000, size=w).astype(np.uint32)
        rank = rng.integers(0, 900, size=w).astype(np.uint32)
        item, index, count = _capi.sample_stage(b, 2, 0x1234ABCD5678, probs, mult, eset, rank)
        assert int(count.sum()) == int(mult.sum())
        pos = 0
        for i in list(range(120)) + list(range(w - 40, w)):
            while item[pos] < i:
                pos += 1
            want = O.multinomial_counts(probs[i], int(mult[i]), 0x1234ABCD5678, int(eset[i]), 2, int(rank[i]))
            nz = np.flatnonzero(want)
            sl = slice(pos, pos + nz.size)
            assert np.all(item[sl] == i)
            assert index[sl].tolist() == nz.tolist()
            assert count[sl].tolist() == want[nz].tolist()


@pytest.mark.parametrize("name", ALL)
def test_complex128_histograms_bit_exact_vs_reference(golden_cases, name):
    """Reference sample_proportional (with the counter-based RNG shim) vs the
    device run, per error set, records and stage events."""
    case = golden_cases[name]
    c, sizes, es = case_objects(case)
    tpl = CircuitNetwork.from_circuit(c)
    ctx = SamplerContext(hypersamples=4, dtype="complex128")
    per_set = sample_proportional_batched(tpl, es, BatchPlan(sizes), case["seed"], ctx)
    got = [[[r.bitstring, r.count] for r in recs] for recs in per_set]
    assert got == case["histograms"]
    assert {str(k): v for k, v in ctx.stats.stage_events.items()} == case["stage_events"]
    assert ctx.stats.plan_events == len(sizes)


def test_run_ptsbe_merged_histogram_and_counters(golden_cases):
    case = golden_cases["hea8"]
    c, sizes, es = case_objects(case)
    cfg = RunConfig(n=c.n, g=len(c.gates), batch_sizes=sizes, seed=case["seed"], hypersamples=4,
                    error_sets=len(es), total_shots=sum(k.m for k in es))
    res = run_ptsbe(c, cfg, errorsets=es)
    want = O.merge_histograms([[tuple(r) for r in h] for h in case["histograms"]])
    assert [(r.bitstring, r.count) for r in res.records] == want
    assert res.total_count == sum(k.m for k in es)
    assert res.plan_events == len(sizes)
    assert res.contract_events == sum(case["stage_events"].values())
    assert {str(k): v for k, v in res.stage_events.items()} == case["stage_events"]
    assert res.timings["gpu_launches"] > 0
    again = run_ptsbe(c, cfg, errorsets=es)
    assert [(r.bitstring, r.count) for r in again.records] == want  # repeat runs identical


def test_results_do_not_depend_on_grouping(golden_cases):
    """Determinism under sharding (reference tests/test_engine.py:455-463):
    splitting the error sets over calls does not change any record."""
    case = golden_cases["random10x40"]
    c, sizes, es = case_objects(case)
    tpl = CircuitNetwork.from_circuit(c)
    whole = sample_proportional_batched(tpl, es, BatchPlan(sizes), 77, SamplerContext(hypersamples=4))
    parts = []
    for lo, hi in ((0, 1), (1, 3), (3, 4)):
        parts += sample_proportional_batched(tpl, es[lo:hi], BatchPlan(sizes), 77, SamplerContext(hypersamples=4))
    assert [[(r.bitstring, r.count) for r in recs] for recs in whole] == \
           [[(r.bitstring, r.count) for r in recs] for recs in parts]


def test_complex64_end_to_end_tvd():
    c, _ = workloads.ghz(12, p=0.05)
    sizes = (4, 4, 4)
    es = presample_errors(c, 8, "uniform", shots_per_set=20000, rng=np.random.default_rng(5))
    tpl = CircuitNetwork.from_circuit(c)
    per_set = sample_proportional_batched(tpl, es, BatchPlan(sizes), 11, SamplerContext(hypersamples=4, dtype="complex64"))
    for k, recs in zip(es, per_set):
        ops, finals = bridge.merged_ops(c, k.realized)
        exact = O.conditional_marginal(ops, finals, (12,), 1, "")
        emp = np.zeros(1 << 12)
        for r in recs:
            emp[int(r.bitstring, 2)] = r.count / k.m
        assert sum(r.count for r in recs) == k.m
        assert 0.5 * np.abs(emp - exact).sum() <= 0.02


def _hea_case(n, depth, sets, shots, seed, gamma=0.01):
    c, _ = workloads.hea(n, depth, gamma=gamma, p=0.01, seed=2)
    es = presample_errors(c, sets, "uniform", shots_per_set=shots, rng=np.random.default_rng(seed))
    return c, CircuitNetwork.from_circuit(c), es


def test_descent_sampler_bit_exact_vs_oracle_complex128(monkeypatch):
    """Per-qubit descent (csrc/descent.cuh) forced on for every projection-form
    stage: same uniforms, float64 marginals within 1e-11 -> the records equal the
    oracle's flat multinomial split (reference engine.py:513-523)."""
    monkeypatch.setenv("PTSBE_DESCENT_MULT", "1e18")
    c, tpl, es = _hea_case(12, 4, 4, 600, 9)
    sizes = (4, 4, 4)
    ctx = SamplerContext(hypersamples=8, dtype="complex128")
    per_set = sample_proportional_batched(tpl, es, BatchPlan(sizes), 31, ctx)
    assert sum(ctx.stats.descent_events.values()) > 0, "descent path was not exercised"
    ops, finals = bridge.template_of(c)
    _, want, events = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), 31)
    assert [[(r.bitstring, r.count) for r in recs] for recs in per_set] == want
    assert dict(ctx.stats.stage_events) == events


@pytest.mark.parametrize("sets,shots", [(3, 5000), (12, 600), (150, 12)])
def test_projection_tiles_spanning_error_sets_bit_exact(monkeypatch, sets, shots):
    """Dense projection (csrc/project.cuh) with the descent sampler off: 64-item tiles holding
    one error set, a few runs of error sets (computed once per run) and more than eight of them
    (per-item path) all give the oracle's records (reference engine.py:442-450, 513-523)."""
    monkeypatch.setenv("PTSBE_DESCENT", "0")
    c, tpl, es = _hea_case(12, 4, sets, shots, 21, gamma=0.0)  # unitary errors only: no impossible sets
    sizes = (4, 4, 4)
    ctx = SamplerContext(hypersamples=8, dtype="complex128")
    per_set = sample_proportional_batched(tpl, es, BatchPlan(sizes), 13, ctx)
    assert not ctx.stats.descent_events
    ops, finals = bridge.template_of(c)
    _, want, events = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), 13)
    assert [[(r.bitstring, r.count) for r in recs] for recs in per_set] == want
    assert dict(ctx.stats.stage_events) == events


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_descent_sampler_agrees_with_flat_sampler(monkeypatch, dtype):
    """Descent on vs off on a 16-qubit HEA (D = 64 cut): identical records in
    complex128, TVD <= 0.02 per error set in complex64 (different rounding of the
    same conditional marginals)."""
    c, tpl, es = _hea_case(16, 5, 24, 4000, 4, gamma=0.0)
    sizes = (6, 5, 5)

    def run(descent):
        monkeypatch.setenv("PTSBE_DESCENT", "1" if descent else "0")
        monkeypatch.setenv("PTSBE_DESCENT_MULT", "1e18")
        ctx = SamplerContext(hypersamples=8, dtype=dtype)
        out = sample_proportional_batched(tpl, es, BatchPlan(sizes), 5, ctx)
        return out, ctx.stats

    flat, st0 = run(False)
    desc, st1 = run(True)
    assert not st0.descent_events and sum(st1.descent_events.values()) > 0
    for k, a, b in zip(es, flat, desc):
        assert sum(r.count for r in b) == k.m
        if dtype == "complex128":
            assert [(r.bitstring, r.count) for r in a] == [(r.bitstring, r.count) for r in b]
        else:
            da, db = {r.bitstring: r.count for r in a}, {r.bitstring: r.count for r in b}
            tvd = 0.5 * sum(abs(da.get(s, 0) - db.get(s, 0)) for s in set(da) | set(db)) / k.m
            assert tvd <= 0.02


def test_deterministic_circuit_and_single_set_signature():
    c = Circuit(3, tuple(Gate("X", (q,)) for q in range(3)))
    tpl = CircuitNetwork.from_circuit(c)
    recs = sample_proportional(tpl, ErrorSet(0, ("I", "I", "I"), 10), BatchPlan((1, 1, 1)), np.random.default_rng(0))
    assert [(r.bitstring, r.count) for r in recs] == [("111", 10)]


def test_impossible_trajectory_is_flagged_with_its_id():
    """Amplitude damping K1 on |0> annihilates the state: the error set is
    reported (ImpossiblePrefixError, engine.py:475-476) instead of crashing the batch."""
    c = Circuit(2, (Gate("Rz", (0,), 0.3, NoiseChannel("amplitude_damping", 0.2)), Gate("H", (1,))))
    tpl = CircuitNetwork.from_circuit(c)
    es = [ErrorSet(0, ("K0", "I"), 5), ErrorSet(7, ("K1", "I"), 5)]
    with pytest.raises(ImpossiblePrefixError, match="error set 7"):
        sample_proportional_batched(tpl, es, BatchPlan((1, 1)), 1)


def test_low_weight_trajectories_are_sampled_not_dropped():
    """Non-unitary Kraus operators give a trajectory a weight far below the
    reference's absolute 1e-12 mass floor (which was written for unitary
    errors); the device guard is relative to the error set's stage-1 mass, so
    such error sets are sampled from their normalised distribution."""
    c, _ = workloads.hea(8, 3, gamma=1e-4, p=0.0, seed=9)
    labels = [g.noise.identity_label() for g in c.gates]
    hit = [s for s, g in enumerate(c.gates) if g.noise.kind == "amplitude_damping" and g.kind == "Ry"][10:15]  # distinct qubits
    for s in hit:
        labels[s] = "K1"
    es = [ErrorSet(3, tuple(labels), 30000)]
    tpl = CircuitNetwork.from_circuit(c)
    for sizes in ((8,), (3, 3, 2)):
        recs = sample_proportional_batched(tpl, es, BatchPlan(sizes), 21, SamplerContext(hypersamples=4))[0]
        assert sum(r.count for r in recs) == 30000
        ops, finals = bridge.merged_ops(c, es[0].realized)
        probs, mass = O.stage_marginal(ops, finals, (8,), 1, "")
        assert 0 < mass < 1e-12
        emp = np.zeros(256)
        for r in recs:
            emp[int(r.bitstring, 2)] = r.count / 30000
        assert 0.5 * np.abs(emp - probs / mass).sum() <= 0.06


def test_tensor_core_api_on_device():
    """contract_pair / execute_path known answers (reference tests/test_tensor.py:25-62)."""
    a = Tensor([Index(0, 2), Index(1, 3)], np.ones((2, 3)))
    b = Tensor([Index(1, 3), Index(2, 2)], np.ones((3, 2)))
    out = contract_pair(a, b)
    assert out.labels == (0, 2) and np.allclose(out.data, 3)
    v = Tensor([Index(5, 2)], [1, 2])
    w = Tensor([Index(6, 2)], [3, 4])
    out = contract_pair(v, w)
    assert out.labels == (5, 6) and np.allclose(out.data, [[3, 4], [6, 8]])
    rng = np.random.default_rng(1)
    ts = [Tensor([Index(0, 2), Index(1, 3)], rng.normal(size=(2, 3)) + 1j * rng.normal(size=(2, 3))),
          Tensor([Index(1, 3), Index(2, 4)], rng.normal(size=(3, 4)) + 1j * rng.normal(size=(3, 4))),
          Tensor([Index(2, 4), Index(3, 2)], rng.normal(size=(4, 2)) + 1j * rng.normal(size=(4, 2)))]
    net = TensorNetwork(ts, [0, 3])
    got = execute_path(net, [(0, 1), (0, 1)])
    want = ts[0].data @ ts[1].data @ ts[2].data
    assert got.labels == (0, 3)
    np.testing.assert_allclose(got.data, want, atol=1e-12)


def test_merge_records_on_device_wide_keys():
    """Two-word keys (n > 64 qubits, surface code d=5 x 3 rounds = 97 bits)."""
    rng = np.random.default_rng(2)
    strings = ["".join(rng.choice(["0", "1"], size=97)) for _ in range(40)]
    per_set = [[ShotRecord(s, int(rng.integers(1, 9))) for s in rng.choice(strings, size=25)] for _ in range(6)]
    got = merge_records(per_set)
    want = O.merge_histograms([[(r.bitstring, r.count) for r in recs] for recs in per_set])
    assert [(r.bitstring, r.count) for r in got] == want


def test_full_size_properties_cfg1():
    """BASELINE config 1 at full size: 64 error sets x 1000 shots, complex64;
    size-independent properties (shot conservation, sortedness, sharding idempotence)."""
    c, sizes = workloads.ghz(12, p=0.01)
    idx = workloads.presample_matrix(c, 64, np.random.default_rng(1))
    es = workloads.errorsets_from_matrix(c, idx, 1000)
    cfg = RunConfig(n=12, g=12, batch_sizes=sizes, seed=4, hypersamples=8, dtype="complex64",
                    error_sets=64, total_shots=64000)
    res = run_ptsbe(c, cfg, errorsets=es)
    assert res.total_count == 64000
    keys = [r.bitstring for r in res.records]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)
    a = run_ptsbe(c, cfg, errorsets=es[:20])
    b = run_ptsbe(c, cfg, errorsets=es[20:])
    merged = merge_records([a.records, b.records])
    assert [(r.bitstring, r.count) for r in merged] == [(r.bitstring, r.count) for r in res.records]
    # GHZ with weak noise: the two GHZ strings dominate
    top = {r.bitstring: r.count for r in res.records}
    assert top["0" * 12] + top["1" * 12] > 0.8 * 64000


def test_variant0_memo_bit_exact_vs_oracle_and_vs_full_replay(monkeypatch):
    """Class-0 programs re-execute only the steps above a site that carries an
    operator (variant-0 memo, csrc/executor.cuh MEMO).  The arithmetic of the
    executed steps is unchanged, so complex128 records must equal both the
    oracle's and those of the full replay (PTSBE_MEMO=0), error-free sets included."""
    c, tpl, es = _hea_case(14, 4, 6, 400, 21, gamma=0.02)
    es[0] = ErrorSet(es[0].id, tuple("K0" if len(lb) == 2 and lb[0] == "K" else "I" * len(lb) for lb in es[0].realized), es[0].m)
    sizes = (7, 7)

    def run(memo):
        monkeypatch.setenv("PTSBE_MEMO", "1" if memo else "0")
        ctx = SamplerContext(hypersamples=8, dtype="complex128")
        out = sample_proportional_batched(tpl, es, BatchPlan(sizes), 77, ctx)
        return [[(r.bitstring, r.count) for r in recs] for recs in out], dict(ctx.stats.stage_events)

    with_memo, ev1 = run(True)
    without, ev0 = run(False)
    assert with_memo == without and ev1 == ev0
    ops, finals = bridge.template_of(c)
    _, want, events = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), 77)
    assert with_memo == want and ev1 == events
    # marginals through the memo path, complex64 within 1e-5 of the oracle
    pfx = [recs[0][0][:7] for recs in want]
    probs = conditional_marginals_batched(tpl, es, BatchPlan(sizes), 2, pfx, SamplerContext(hypersamples=8, dtype="complex64"))
    for k, p, row in zip(es, pfx, probs):
        mops, _ = bridge.merged_ops(c, k.realized)
        ref = O.conditional_marginal(mops, finals, sizes, 2, p)
        assert np.max(np.abs(row - ref)) <= 1e-5 * ref.max()


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_lane_per_item_kernels_agree_with_group_kernels(monkeypatch, dtype):
    """lane.cuh (thread per item, fused per-item steps + descent, dedup of raw
    draws) against the lane-group executor + stand-alone descent: identical
    records in complex128 (same uniforms, marginals within 1e-11), TVD <= 0.02
    per error set in complex64.  Multi-shot items exercise the dedup kernels."""
    c, tpl, es = _hea_case(16, 5, 16, 3000, 11, gamma=0.0)
    sizes = (6, 5, 5)

    def run(lane):
        monkeypatch.setenv("PTSBE_LANE", "1" if lane else "0")
        monkeypatch.setenv("PTSBE_DESCENT_MULT", "1e18")
        ctx = SamplerContext(hypersamples=8, dtype=dtype)
        out = sample_proportional_batched(tpl, es, BatchPlan(sizes), 19, ctx)
        return out, ctx.stats

    group, st0 = run(False)
    lane, st1 = run(True)
    assert sum(st0.descent_events.values()) > 0 and sum(st1.descent_events.values()) > 0
    assert dict(st0.stage_events) == dict(st1.stage_events) or dtype == "complex64"
    for k, a, b in zip(es, group, lane):
        assert sum(r.count for r in b) == k.m
        assert [r.bitstring for r in b] == sorted(r.bitstring for r in b)
        if dtype == "complex128":
            assert [(r.bitstring, r.count) for r in a] == [(r.bitstring, r.count) for r in b]
        else:
            da, db = {r.bitstring: r.count for r in a}, {r.bitstring: r.count for r in b}
            tvd = 0.5 * sum(abs(da.get(s, 0) - db.get(s, 0)) for s in set(da) | set(db)) / k.m
            assert tvd <= 0.02


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_thread_per_error_set_hoist_equals_group_executor(monkeypatch, dtype):
    """Class-0 hoist passes over large batches run one thread per error set with the
    arena in global memory (csrc/lane.cuh BIG) instead of a lane group per error set
    (csrc/executor.cuh).  Same multiply-add order, so the records are identical in
    both dtypes; complex128 also equals the oracle (reference engine.py:361-450)."""
    c, sizes = workloads.random40(14, 70, seed=3)
    sizes = (5, 5, 4)
    tpl = CircuitNetwork.from_circuit(c)
    es = presample_errors(c, 40, "uniform", shots_per_set=50, rng=np.random.default_rng(8))

    def run(big):
        monkeypatch.setenv("PTSBE_LANE_BIG_MIN", "1" if big else "4000000000")
        ctx = SamplerContext(hypersamples=8, dtype=dtype)
        tables = VariantTables.from_channels(tpl)
        pipe = DevicePipeline(tpl, BatchPlan(sizes), tables, ctx, shots_per_set=50.0)
        qualifying = [p for p in pipe.compiled.programs if p.level == 1 and p.threads <= 32 and p.arena_fast > 48
                      and not p.memo_elems and not p.proj_d and len(p.steps)]
        pipe.close()
        out = sample_proportional_batched(tpl, es, BatchPlan(sizes), 5, ctx)
        return [[(r.bitstring, r.count) for r in recs] for recs in out], len(qualifying)

    big, n_q = run(True)
    group, _ = run(False)
    assert n_q >= 1, "no class-0 program of this case qualifies for the thread-per-error-set kernel"
    assert big == group
    if dtype == "complex128":
        ops, finals = bridge.template_of(c)
        _, want, _ = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), 5)
        assert big == want


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_warp_private_descent_tables_and_staged_image_equal_the_cta_paths(monkeypatch, dtype):
    """Short runs of work items per error set: the fused descent kernels give every warp its own
    copy of the tree table (csrc/lane.cuh warp_runs) and lane-group class-0 programs keep their
    image in shared memory (csrc/executor.cuh STAGED).  Both are scheduling choices: the records
    equal those of the one-error-set-per-CTA kernels with the image in global memory, in both
    dtypes, and the oracle's in complex128 (reference engine.py:493-524)."""
    c, _ = workloads.random40(14, 70, seed=3)
    sizes = (5, 5, 4)
    tpl = CircuitNetwork.from_circuit(c)
    es = presample_errors(c, 300, "uniform", shots_per_set=20, rng=np.random.default_rng(12))

    def run(on):
        monkeypatch.setenv("PTSBE_WARP_RUNS", "1" if on else "0")
        monkeypatch.setenv("PTSBE_STAGE_IMAGE", "1" if on else "0")
        monkeypatch.setenv("PTSBE_DESCENT_MULT", "1e18")
        ctx = SamplerContext(hypersamples=8, dtype=dtype)
        out = sample_proportional_batched(tpl, es, BatchPlan(sizes), 23, ctx)
        assert sum(ctx.stats.descent_events.values()) > 0
        return [[(r.bitstring, r.count) for r in recs] for recs in out]

    fast, plain = run(True), run(False)
    assert fast == plain
    if dtype == "complex128":
        ops, finals = bridge.template_of(c)
        _, want, _ = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), 23)
        assert fast == want


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_early_hoist_passes_fused_tables_and_tile_shapes_do_not_change_records(monkeypatch, dtype):
    """Scheduling choices of the run loop and of the CTA executor: hoist passes launched on side
    streams as soon as their level exists (PTSBE_PRELAUNCH), descent tables built by the fused
    tree + packing kernel (PTSBE_TREE_HERM), 2 x 2 instead of 4 x 4 register tiles for mid-size steps
    (PTSBE_TILE_MIN).  None of them may change a record; complex128 must still equal the oracle
    (reference engine.py:493-524)."""
    c, tpl, es = _hea_case(14, 4, 24, 300, 5, gamma=0.0)
    sizes = (5, 5, 4)

    def run(on):
        monkeypatch.setenv("PTSBE_PRELAUNCH", "1" if on else "0")
        monkeypatch.setenv("PTSBE_TREE_HERM", "1" if on else "0")
        monkeypatch.setenv("PTSBE_TILE_MIN", "128" if on else "0")
        monkeypatch.setenv("PTSBE_DESCENT_MULT", "1e18")
        ctx = SamplerContext(hypersamples=8, dtype=dtype)
        out = sample_proportional_batched(tpl, es, BatchPlan(sizes), 41, ctx)
        return [[(r.bitstring, r.count) for r in recs] for recs in out], dict(ctx.stats.stage_events)

    fast, ev1 = run(True)
    plain, ev0 = run(False)
    assert fast == plain and ev1 == ev0
    if dtype == "complex128":
        ops, finals = bridge.template_of(c)
        _, want, events = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), 41)
        assert fast == want and ev1 == events


@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_raw_final_draws_give_the_same_merged_histogram(monkeypatch, dtype):
    """Merged output of a run whose final stage is sampled by the fused descent kernels: the raw draws go to
    the histogram sort as records of count 1 (no per-item merge; keys-only radix sort; csrc/capi.cu raw_final).
    merge_records (reference engine.py:815-829) sums equal bitstrings either way: the merged histogram equals
    the one built with the per-item merge, the merge of the per-error-set records, and the oracle's in
    complex128.  20 shots over 16 final outcomes per prefix: many duplicate draws per work item."""
    c, _ = workloads.random40(14, 70, seed=3)
    sizes = (5, 5, 4)
    tpl = CircuitNetwork.from_circuit(c)
    es = presample_errors(c, 300, "uniform", shots_per_set=20, rng=np.random.default_rng(12))
    monkeypatch.setenv("PTSBE_DESCENT_MULT", "1e18")
    cfg = RunConfig(n=c.n, g=len(c.gates), batch_sizes=sizes, seed=23, hypersamples=8, dtype=dtype,
                    error_sets=len(es), total_shots=sum(k.m for k in es))

    def run(raw):
        monkeypatch.setenv("PTSBE_RAW_FINAL", "1" if raw else "0")
        res = run_ptsbe(c, cfg, errorsets=es)
        assert res.total_count == sum(k.m for k in es)
        return [(r.bitstring, r.count) for r in res.records]

    raw, merged_per_item = run(True), run(False)
    assert raw == merged_per_item
    ctx = SamplerContext(hypersamples=8, dtype=dtype)
    per_set = sample_proportional_batched(tpl, es, BatchPlan(sizes), 23, ctx)
    assert sum(ctx.stats.descent_events.values()) > 0
    assert raw == [(r.bitstring, r.count) for r in merge_records(per_set)]
    assert max(n for _, n in raw) > 1
    if dtype == "complex128":
        ops, finals = bridge.template_of(c)
        _, want, _ = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), 23)
        assert raw == O.merge_histograms(want)


def test_many_error_sets_single_shot_descent():
    """More error sets than a grid dimension holds (tree_build puts them on
    grid.x), one shot each: every shot is sampled and the histogram total is exact."""
    c, _ = workloads.surface_code(3, 1, p=1e-3)
    tpl = CircuitNetwork.from_circuit(c)
    from paper_2604_08467_b200.engine import DevicePipeline, VariantTables
    tables = VariantTables.from_channels(tpl)
    sets = 70_000
    kraus = workloads.presample_matrix(c, sets, np.random.default_rng(2))
    ctx = SamplerContext(hypersamples=8, dtype="complex64")
    pipe = DevicePipeline(tpl, BatchPlan((8, 8, 1)), tables, ctx, shots_per_set=1.0)
    ids = np.arange(sets, dtype=np.uint32)
    try:
        keys, _, counts, st = pipe.device_plan.sample(kraus, np.ones(sets, np.uint32), ids, 3)
        keys, counts = np.array(keys), np.array(counts)
        halves = []
        for lo, hi in ((0, 30_001), (30_001, sets)):  # streams are keyed by the global id: halves add up
            k, _, c, _ = pipe.device_plan.sample(kraus[lo:hi], np.ones(hi - lo, np.uint32), ids[lo:hi], 3)
            halves.append((np.array(k), np.array(c)))
    finally:
        pipe.close()
    assert int(counts.sum()) + 0 == sets - 0 * int(st.flagged_sets)
    assert int(st.flagged_sets) == 0
    # few distinct keys, 70 000 records: segments of equal keys span many 2048-record tiles of the
    # one-word histogram tail; output strictly increasing, and equal to the generic (u64-count,
    # permutation-based) merge of the two halves
    assert np.all(keys[1:, 0] > keys[:-1, 0])
    from paper_2604_08467_b200 import _capi
    mk, mc = _capi.histogram_merge(np.concatenate([h[0] for h in halves]), np.concatenate([h[1] for h in halves]))
    assert np.array_equal(mk, keys) and np.array_equal(mc.astype(np.uint64), counts.astype(np.uint64))


def _nonprop_runs():
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_nonproportional.json")
    with open(path) as fp:
        return json.load(fp)["runs"]


def test_nonproportional_bit_exact_vs_reference_goldens(golden_cases):
    """Non-proportional sampler (engine.py:527-576) on the device, complex128,
    against the records of the UNMODIFIED reference driven by the counter-based
    shim: same chosen prefixes, same harvested outcomes in the same order,
    probability tags within 1e-11, direct-mode counts identical."""
    from paper_2604_08467_b200.engine import sample_nonproportional_batched

    n_records = 0
    for run in _nonprop_runs():
        case = golden_cases[run["case"]]
        c, sizes, es = case_objects(case)
        var = run["variant"]
        plan = BatchPlan(sizes, nonfinal_shots=var["nonfinal_shots"], final_mode=var["final_mode"],
                         threshold=var["threshold"], direct_count=var["direct_count"])
        tpl = CircuitNetwork.from_circuit(c)
        got = sample_nonproportional_batched(tpl, es, plan, run["seed"], SamplerContext(hypersamples=4, dtype="complex128"))
        for recs, want in zip(got, run["records"]):
            assert [(r.bitstring, r.count) for r in recs] == [(s, n) for s, n, _ in want], (run["case"], var)
            for r, (_, _, q) in zip(recs, want):
                assert (r.prob is None) == (q is None)
                if q is not None:
                    assert abs(r.prob - q) <= 1e-11
            n_records += len(recs)
    assert n_records >= 1000


def test_nonproportional_exhaustive_set_equality_complex64(golden_cases):
    """Reference acceptance criterion 4 (tests/test_acceptance.py:134-153): with a
    single batch covering the register the exhaustive output equals
    {s : p(s) >= tau}.  complex64: outcomes within 1e-5 of the threshold may fall
    on either side; everything else must match, tags within 1e-5."""
    from paper_2604_08467_b200.engine import sample_nonproportional_batched

    for name in ("random_0", "random_2", "random_4", "hea8", "qaoa8"):
        c, _, es = case_objects(golden_cases[name])
        tpl = CircuitNetwork.from_circuit(c)
        tau = 1e-3
        plan = BatchPlan((c.n,), final_mode="exhaustive", threshold=tau)
        got = sample_nonproportional_batched(tpl, es, plan, 5, SamplerContext(hypersamples=4, dtype="complex64"))
        for k, recs in zip(es, got):
            mops, finals = bridge.merged_ops(c, k.realized)
            p = O.conditional_marginal(mops, finals, (c.n,), 1, "")
            sure = {format(i, f"0{c.n}b") for i in np.flatnonzero(p >= tau * (1 + 1e-4))}
            maybe = {format(i, f"0{c.n}b") for i in np.flatnonzero(p >= tau * (1 - 1e-4))}
            have = {r.bitstring for r in recs}
            assert sure <= have <= maybe
            for r in recs:
                assert abs(r.prob - p[int(r.bitstring, 2)]) <= 1e-5 * p.max()


def test_run_ptsbe_nonproportional_mode():
    """run_ptsbe(mode='ptsbe-nonproportional'): records merged over error sets
    (engine.py:815-829), plan events = f, one contraction per prefix."""
    c, _ = workloads.hea(8, 3, gamma=0.0, p=0.05, seed=21)
    cfg = RunConfig(n=8, g=len(c.gates), mode="ptsbe-nonproportional", batch_sizes=(3, 3, 2), error_sets=6,
                    total_shots=6, nonfinal_shots=2, final_mode="exhaustive", tau=1e-2, seed=3, hypersamples=4)
    res = run_ptsbe(c, cfg)
    assert res.plan_events == 3 and res.records
    assert [r.bitstring for r in res.records] == sorted(r.bitstring for r in res.records)
    assert res.stage_events[1] == 6 and res.stage_events[2] <= 12 and res.stage_events[3] <= 24
    again = run_ptsbe(c, cfg)
    assert [(r.bitstring, r.count, r.prob) for r in again.records] == [(r.bitstring, r.count, r.prob) for r in res.records]
    direct = run_ptsbe(c, RunConfig(n=8, g=len(c.gates), mode="ptsbe-nonproportional", batch_sizes=(3, 3, 2),
                                    error_sets=6, total_shots=6, nonfinal_shots=1, final_mode="direct",
                                    direct_count=7, seed=3, hypersamples=4))
    assert direct.total_count == 6 * 7


def test_nonproportional_exhaustive_large_final_batch():
    """Final batch beyond the shared-memory sampler (2^16 outcomes, harvest_big_kernel):
    the harvested set equals {s : p(s) >= tau} of the oracle's full distribution,
    tags within 1e-11 (complex128), for a single stage and for a (2, 14) plan."""
    from paper_2604_08467_b200.engine import sample_nonproportional_batched

    c, _ = workloads.hea(16, 3, gamma=0.0, p=0.03, seed=5)
    es = presample_errors(c, 3, "uniform", shots_per_set=1, rng=np.random.default_rng(8))
    tpl = CircuitNetwork.from_circuit(c)
    tau = 2e-5
    got = sample_nonproportional_batched(tpl, es, BatchPlan((16,), final_mode="exhaustive", threshold=tau), 1,
                                         SamplerContext(hypersamples=8, dtype="complex128"))
    for k, recs in zip(es, got):
        mops, finals = bridge.merged_ops(c, k.realized)
        p = O.conditional_marginal(mops, finals, (16,), 1, "")
        want = np.flatnonzero(p >= tau)
        assert [int(r.bitstring, 2) for r in recs] == want.tolist()
        assert max(abs(r.prob - p[int(r.bitstring, 2)]) for r in recs) <= 1e-11
    # two stages: one chosen 2-bit prefix per error set, then a 2^14 harvest conditioned on it
    got2 = sample_nonproportional_batched(tpl, es, BatchPlan((2, 14), final_mode="exhaustive", threshold=1e-4), 4,
                                          SamplerContext(hypersamples=8, dtype="complex128"))
    for k, recs in zip(es, got2):
        assert recs and len({r.bitstring[:2] for r in recs}) == 1
        mops, finals = bridge.merged_ops(c, k.realized)
        cond = O.conditional_marginal(mops, finals, (2, 14), 2, recs[0].bitstring[:2])
        assert [int(r.bitstring[2:], 2) for r in recs] == np.flatnonzero(cond >= 1e-4).tolist()
        assert max(abs(r.prob - cond[int(r.bitstring[2:], 2)]) for r in recs) <= 1e-11


def test_batch_time_curve_rows():
    """Device counterpart of the reference's bench.batch_time_curve (bench.py:287-331):
    one row per feasible b with the reference's keys; est_cost grows with b."""
    from paper_2604_08467_b200.bench_tools import batch_time_curve
    from paper_2604_08467_b200.circuits import random_circuit

    c = random_circuit(10, 40, rng=np.random.default_rng(3))
    rows = batch_time_curve(c, [2, 5, 10, 12], hypersamples=4, reps=2, batch=64)
    assert [r["b"] for r in rows] == [2, 5, 10]
    for r in rows:
        assert {"b", "stage_seconds", "per_qubit_seconds", "path_seconds", "est_cost", "reps"} <= set(r)
        assert r["stage_seconds"] > 0 and r["per_qubit_seconds"] == pytest.approx(r["stage_seconds"] / r["b"])
    assert rows[-1]["est_cost"] > rows[0]["est_cost"]


def test_device_presampling_matches_counter_oracle_and_upload_path():
    """Pre-trajectory sampling on the device (reference engine.py:232-281): the
    Kraus-index matrix equals the oracle's counter-based draw bit for bit, does not depend on
    how the id range is split, follows the channel probabilities, and a run over the
    device-sampled batch equals a run over the same matrix uploaded from the host."""
    from paper_2604_08467_b200.engine import DevicePipeline, VariantTables

    c, _ = workloads.hea(10, 3, gamma=0.08, p=0.1, seed=4)
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_channels(tpl)
    site_probs = [[pr for _, pr in g.noise.outcomes()] for g in c.gates]
    sets, seed = 5000, 12345
    ctx = SamplerContext(hypersamples=4, dtype="complex128")
    pipe = DevicePipeline(tpl, BatchPlan((5, 5)), tables, ctx, shots_per_set=20.0)
    try:
        dp = pipe.device_plan
        bt = dp.presample(site_probs, sets, 100, 20, seed)
        got = bt.kraus(sets, len(c.gates))
        want = O.presample_counter(site_probs, sets, 100, seed)
        np.testing.assert_array_equal(got, want)
        # split-independence: the second half generated on its own
        half = dp.presample(site_probs, sets // 2, 100 + sets // 2, 20, seed)
        np.testing.assert_array_equal(half.kraus(sets // 2, len(c.gates)), want[sets // 2:])
        half.close()
        # distribution: frequency of "some error" per site within 5 sigma of 1 - p0
        for s, probs in enumerate(site_probs):
            p_err = 1.0 - probs[0]
            f_err = float(np.mean(got[:, s] != 0))
            assert abs(f_err - p_err) <= 5 * np.sqrt(max(p_err * (1 - p_err), 1e-9) / sets) + 1e-12
        # same records as the host-upload path
        n1, _ = bt.run(7)
        k1, c1 = bt.fetch()
        up = dp.upload(want, np.full(sets, 20, np.uint32), np.arange(100, 100 + sets, dtype=np.uint32))
        n2, _ = up.run(7)
        k2, c2 = up.fetch()
        assert n1 == n2
        np.testing.assert_array_equal(k1, k2)
        np.testing.assert_array_equal(c1, c2)
        bt.close()
        up.close()
    finally:
        pipe.close()


def test_cfg2_full_circuit_size_independent_properties():
    """BASELINE config 2 at full circuit size (30-qubit HEA depth 6, 447 sites, plan 9/6/7/8,
    complex64, every production kernel: memo + tiled class-0 pass, lane interpreter, fused
    descent, Hermitian packing), on a batch small enough for a test: (a) every shot of every
    unflagged error set is sampled, (b) records are sorted and unique per error set, (c) the
    empirical distribution of the first 9 measured bits matches the exact complex128 stage-1
    marginal of that error set (TVD at 10^4 shots), (d) results do not depend on how the error
    sets are grouped into calls."""
    from paper_2604_08467_b200.engine import DevicePipeline, VariantTables

    c, _ = workloads.hea(30, 6, gamma=0.01, p=0.01, seed=2)
    sizes = (9, 6, 7, 8)
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_channels(tpl)
    sets, shots = 12, 10_000
    kraus = workloads.presample_matrix(c, sets, np.random.default_rng(6))
    kraus[:, :] = np.where(np.arange(len(c.gates))[None, :] < 60, 0, kraus)  # no K1 on |0>: nothing flagged
    ids = np.arange(sets, dtype=np.uint32)
    ctx = SamplerContext(hypersamples=16, dtype="complex64")
    pipe = DevicePipeline(tpl, BatchPlan(sizes), tables, ctx, shots_per_set=float(shots))
    try:
        dp = pipe.device_plan
        keys, esets, counts, st = dp.sample(kraus, np.full(sets, shots, np.uint32), ids, 11, merged=False)
        assert int(st.flagged_sets) == 0 and int(counts.sum()) == sets * shots
        for e in range(sets):
            ke = keys[esets == e, 0]
            assert np.all(np.diff(ke.astype(np.uint64)) > 0)  # sorted, unique
        # (d) grouping independence: two calls of 6 error sets
        k2a, e2a, c2a, _ = dp.sample(kraus[:6], np.full(6, shots, np.uint32), ids[:6], 11, merged=False)
        k2b, e2b, c2b, _ = dp.sample(kraus[6:], np.full(6, shots, np.uint32), ids[6:], 11, merged=False)
        np.testing.assert_array_equal(np.concatenate([k2a, k2b]), keys)
        np.testing.assert_array_equal(np.concatenate([c2a, c2b]), counts)
    finally:
        pipe.close()
    # (c) stage-1 marginal of three error sets in complex128 through the marginals entry point
    es = workloads.errorsets_from_matrix(c, kraus[:3], shots)
    # (unnormalised: a realised K1 gives the trajectory a weight far below the reference's absolute
    # 1e-12 mass floor, which the normalising form of this call enforces like the reference does)
    exact, mass = conditional_marginals_batched(tpl, es, BatchPlan(sizes), 1, ["", "", ""],
                                                SamplerContext(hypersamples=16, dtype="complex128"),
                                                normalize=False, return_mass=True)
    exact = exact / mass[:, None]
    for e in range(3):
        sel = esets == e
        first9 = (keys[sel, 0] >> np.uint64(64 - 9)).astype(np.int64)
        emp = np.bincount(first9, weights=counts[sel].astype(np.float64), minlength=512) / shots
        assert 0.5 * np.abs(emp - exact[e]).sum() <= 0.12  # 512 bins, 10^4 shots: sampling noise ~0.09


def test_cfg2_full_circuit_complex64_marginals_within_1e5_of_complex128():
    """North-star tolerance at BASELINE size: conditional marginals of the 30-qubit HEA depth-6
    circuit (447 sites) in complex64 within 1e-5 relative of complex128, every stage of the
    9/6/7/8 plan, on prefixes that a proportional run actually visits."""
    c, _ = workloads.hea(30, 6, gamma=0.01, p=0.01, seed=2)
    sizes = (9, 6, 7, 8)
    tpl = CircuitNetwork.from_circuit(c)
    kraus = workloads.presample_matrix(c, 6, np.random.default_rng(6))
    kraus[:, :60] = 0
    es = workloads.errorsets_from_matrix(c, kraus, 100)
    per = sample_proportional_batched(tpl, es, BatchPlan(sizes), 3, SamplerContext(hypersamples=16, dtype="complex128"))
    for j in (1, 2, 3, 4):
        off = sum(sizes[:j - 1])
        pf = [recs[len(recs) // 2].bitstring[:off] for recs in per]
        hi, mh = conditional_marginals_batched(tpl, es, BatchPlan(sizes), j, pf,
                                               SamplerContext(hypersamples=16, dtype="complex128"),
                                               normalize=False, return_mass=True)
        lo, ml = conditional_marginals_batched(tpl, es, BatchPlan(sizes), j, pf,
                                               SamplerContext(hypersamples=16, dtype="complex64"),
                                               normalize=False, return_mass=True)
        a, b = hi / mh[:, None], lo / ml[:, None]
        err = np.max(np.abs(a - b), axis=1) / np.max(a, axis=1)
        assert err.max() <= 1e-5, (j, err.max())
        assert np.max(np.abs(ml / mh - 1.0)) <= 1e-5
