"""Host-side mirror of the reference API: known answers of the reference's own
tests (/root/reference/pkg/tests/test_engine.py:53-61, 103-106, 139-145;
test_circuits.py) and rng call-order compatibility pinned by golden vectors
generated from the unmodified reference."""

import io
import json

import numpy as np
import pytest

import paper_2604_08467_b200 as P
from conftest import case_objects
from paper_2604_08467_b200 import workloads
from paper_2604_08467_b200.circuits import (
    TWO_QUBIT_PAULIS, circuit_from_json, circuit_to_json, gate_matrix, pauli_matrix,
)
from paper_2604_08467_b200.engine import (
    BatchPlan, CircuitNetwork, ErrorSet, RunConfig, RunResult, ShotRecord, VariantTables, merge_errors,
    pack_prefixes, presample_errors, unpack_keys, marginal_network,
)
from paper_2604_08467_b200.errors import NetworkStructureError
from paper_2604_08467_b200.planner import ContractionPath, PathCache, find_path_optimal, merges_to_steps, path_cost
from paper_2604_08467_b200.tensor import Index, Tensor, TensorNetwork, network_signature

REFERENCE_EXPORTS = [
    "BatchPlan", "Circuit", "CircuitNetwork", "ContractionPath", "EngineStats", "ErrorSet", "Gate", "Index",
    "NetworkSignature", "NoiseChannel", "PathCache", "RunConfig", "RunResult", "SamplerContext", "ShotRecord",
    "Tensor", "TensorNetwork", "build_network", "cache_lookup_or_plan", "conditional_marginal", "contract_pair",
    "execute_path", "find_path_greedy", "find_path_optimal", "gate_matrix", "insert_errors", "marginal_network",
    "merge_errors", "merge_records", "network_signature", "path_cost", "presample_errors", "random_circuit",
    "run_mode", "run_ptsbe", "sample_baseline", "sample_nonproportional", "sample_proportional",
    "sample_unoptimized_ptsbe", "spawn_rng",
]


def test_reference_names_are_exported():
    for name in REFERENCE_EXPORTS:
        assert hasattr(P, name), name


def test_batch_plan_partitions():
    assert BatchPlan.fixed(50, 24).sizes == (24, 24, 2)
    assert BatchPlan.with_final(50, 10, 28).sizes == (10, 10, 2, 28)
    assert BatchPlan.with_final(12, 10, 28).sizes == (12,)
    p = BatchPlan((4, 4, 4))
    assert (p.f, p.n, p.offset(3), list(p.stage_qubits(2))) == (3, 12, 8, [4, 5, 6, 7])
    with pytest.raises(ValueError):
        BatchPlan((4, 0))


def test_presample_remainder_spreading():
    c = P.random_circuit(4, 10, rng=np.random.default_rng(0))
    sets = presample_errors(c, 4, "proportional", 10, rng=np.random.default_rng(1))
    assert [k.m for k in sets] == [3, 3, 2, 2]
    with pytest.raises(ValueError):
        presample_errors(c, 4, "proportional", 3)


def test_rng_call_order_matches_reference(golden):
    """random_circuit and presample_errors consume the generator exactly like
    the reference, so a seed means the same inputs in both packages."""
    for row in golden["producers"]:
        mine = P.random_circuit(row["n"], row["g"], rng=np.random.default_rng(row["seed"]))
        assert json.loads(circuit_to_json(mine)) == json.loads(row["circuit"])
        sets = presample_errors(mine, 4, "proportional", 10, rng=np.random.default_rng(row["presample_seed"]))
        assert [list(k.realized) for k in sets] == row["realized"]
        assert [k.m for k in sets] == row["alloc"]


def test_gate_conventions():
    cx = gate_matrix(P.Gate("CX", (0, 1), None, P.NoiseChannel("depolarizing", 0.0)))
    assert np.allclose(cx, np.eye(4)[[0, 1, 3, 2]])
    for kind, angle in (("H", None), ("T", None), ("Rx", 0.7), ("Ry", 1.1), ("Rz", 2.3), ("S", None)):
        u = gate_matrix(P.Gate(kind, (0,), angle))
        assert np.allclose(u @ u.conj().T, np.eye(2))
    u = gate_matrix(P.Gate("RZZ", (0, 3), 0.4, P.NoiseChannel("depolarizing", 0.0)))
    assert np.allclose(u @ u.conj().T, np.eye(4)) and np.allclose(u, np.diag(np.diag(u)))
    assert np.allclose(pauli_matrix("XZ"), np.kron(pauli_matrix("X"), pauli_matrix("Z")))
    assert len(TWO_QUBIT_PAULIS) == 15
    ad = P.NoiseChannel("amplitude_damping", 0.3)
    k0, k1 = ad.operator("K0"), ad.operator("K1")
    assert np.allclose(k0.conj().T @ k0 + k1.conj().T @ k1, np.eye(2))


def test_merge_errors_keeps_structure_and_is_noop_on_identity(golden_cases):
    for name in ("random_0", "random_4", "hea8"):
        c, sizes, es = case_objects(golden_cases[name])
        tpl = CircuitNetwork.from_circuit(c)
        sig = network_signature(tpl.net)
        for k in es:
            assert network_signature(tpl.merged(k).net) == sig
        ident = ErrorSet(0, tuple(g.noise.identity_label() for g in c.gates if g.noise.kind != "amplitude_damping"), 1)
        if len(ident.realized) == len(c.gates):
            same = merge_errors(tpl.net, ident)
            assert all(np.array_equal(a.data, b.data) for a, b in zip(same.operands, tpl.net.operands))
    with pytest.raises(NetworkStructureError):
        merge_errors(tpl.net, ErrorSet(0, ("I",) * 500, 1))


def test_variant_tables_encode_upv():
    c, _ = workloads.ghz(4, p=0.1)
    tpl = CircuitNetwork.from_circuit(c)
    es = [ErrorSet(0, ("I", "II", "XZ", "II"), 1), ErrorSet(1, ("Y", "II", "II", "ZZ"), 1)]
    t = VariantTables.from_errorsets(tpl, es)
    idx = t.encode(es)
    assert idx.dtype == np.uint8 and idx.shape == (2, 4)
    for r, k in enumerate(es):
        merged = tpl.merged(k).net
        for s in range(4):
            assert np.allclose(t.data[s][idx[r, s]], merged.operands[4 + s].data.reshape(-1))
    full = VariantTables.from_channels(tpl)
    assert [d.shape[0] for d in full.data] == [4, 16, 16, 16]


def test_stage_network_operand_count():
    c, _ = workloads.ghz(12)
    tpl = CircuitNetwork.from_circuit(c)
    plan = BatchPlan((4, 4, 4))
    assert [len(marginal_network(tpl, plan, j, "0" * plan.offset(j)).net) for j in (1, 2, 3)] == [52, 60, 68]


def test_key_packing_round_trip():
    rng = np.random.default_rng(0)
    for n in (1, 12, 64, 65, 97, 130):
        strings = ["".join(rng.choice(["0", "1"], size=n)) for _ in range(9)]
        keys = pack_prefixes(strings, n)
        assert keys.shape == (9, max(1, (n + 63) // 64))
        assert unpack_keys(keys, n) == strings
    order = sorted(range(9), key=lambda i: strings[i])
    tup = [tuple(int(v) for v in row) for row in keys]
    assert sorted(range(9), key=lambda i: tup[i]) == order  # numeric key order == string order


def test_path_json_and_cache_round_trip(golden_cases):
    c, sizes, _ = case_objects(golden_cases["random_1"])
    net = marginal_network(CircuitNetwork.from_circuit(c), BatchPlan(sizes), 1, "").net
    path = P.find_path_greedy(net, hypersamples=2, rng=np.random.default_rng(0))
    assert ContractionPath.from_json(path.to_json()) == path
    cache = PathCache()
    got, hit = P.cache_lookup_or_plan(cache, net, stage=1, hypersamples=2, rng=np.random.default_rng(0))
    assert not hit and cache.misses == 1
    buf = io.StringIO()
    cache.save(buf)
    buf.seek(0)
    warm = PathCache.load(buf)
    again, hit = P.cache_lookup_or_plan(warm, net, stage=1)
    assert hit and again == got
    _, miss = P.cache_lookup_or_plan(warm, net, stage=2, hypersamples=1, rng=np.random.default_rng(0))
    assert not miss


def test_optimal_planner_bounds_greedy():
    rng = np.random.default_rng(4)
    ts = [Tensor([Index(0, 2), Index(1, 8)], rng.normal(size=(2, 8))),
          Tensor([Index(1, 8), Index(2, 3)], rng.normal(size=(8, 3))),
          Tensor([Index(2, 3), Index(3, 9)], rng.normal(size=(3, 9))),
          Tensor([Index(3, 9), Index(4, 2)], rng.normal(size=(9, 2)))]
    net = TensorNetwork(ts, [0, 4])
    best = find_path_optimal(net)
    greedy = P.find_path_greedy(net, hypersamples=16, rng=np.random.default_rng(0))
    assert path_cost(net, best) == pytest.approx(best.est_cost)
    assert best.est_cost <= greedy.est_cost + 1e-9
    assert greedy.est_cost == pytest.approx(best.est_cost)  # matrix chain: greedy finds the optimum


def test_merges_to_steps_convention():
    # stable ids 0..3: merge (1,3) then (0,2) then (0,1) -> slots shift down after deletions
    assert merges_to_steps(4, [(1, 3), (0, 2), (0, 1)]) == ((1, 3), (0, 2), (0, 1))
    assert merges_to_steps(4, [(2, 3), (0, 1), (0, 2)]) == ((2, 3), (0, 1), (0, 1))


def test_run_config_and_result_round_trip():
    cfg = RunConfig(n=6, g=10, batch_sizes=(3, 3), dtype="complex64")
    assert RunConfig.from_dict(cfg.to_dict()) == cfg
    with pytest.raises(ValueError):
        RunConfig(n=6, g=10, batch_sizes=(3, 2))
    with pytest.raises(ValueError):
        RunConfig(n=6, g=10, mode="nope")
    res = RunResult(mode="ptsbe-proportional", records=[ShotRecord("01", 3)], unique_shots=1, total_count=3,
                    timings={"loop_s": 0.1}, plan_events=2, contract_events=5, stage_events={1: 2, 2: 3},
                    stage_seconds={1: 0.0, 2: 0.0}, config=cfg.to_dict(), seed=0, shot_allocations=[3])
    assert RunResult.from_json(res.to_json()) == res


def test_out_of_scope_modes_say_so():
    with pytest.raises(NotImplementedError):
        P.sample_baseline()
    with pytest.raises(NotImplementedError):
        P.run_mode(P.random_circuit(3, 4, rng=np.random.default_rng(0)), RunConfig(n=3, g=4, mode="baseline"))


def test_workload_shapes():
    c, sizes = workloads.ghz()
    assert (c.n, len(c.gates), sizes) == (12, 12, (4, 4, 4))
    c, sizes = workloads.hea()
    assert c.n == 30 and sizes == (10, 10, 10) and len(c.gates) == 6 * 60 + 3 * 15 + 3 * 14
    c, sizes = workloads.surface_code()
    assert c.n == 97 and sum(sizes) == 97
    c, sizes = workloads.qaoa()
    assert c.n == 50 and len(c.gates) == 50 + 2 * (75 + 50)
    c, sizes = workloads.random40()
    assert c.n == 40 and len(c.gates) == 400
    idx = workloads.presample_matrix(c, 1000, np.random.default_rng(0))
    assert idx.shape == (1000, 400) and idx.max() <= 15
    es = workloads.errorsets_from_matrix(c, idx[:3], 7)
    assert es[2].m == 7 and len(es[0].realized) == 400
