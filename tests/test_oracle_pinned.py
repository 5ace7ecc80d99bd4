"""Pins oracle/ptsbe_oracle.py to the reference: golden vectors generated from
the UNMODIFIED reference (oracle/make_golden.py) and the closed-form known
answers of the reference's own tests (tests/test_engine.py:53-61, 103-106,
163-173, 283-289 of /root/reference/pkg)."""

import math

import numpy as np
import pytest

from conftest import case_objects
from oracle import bridge
from oracle import ptsbe_oracle as O

H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / math.sqrt(2)
X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
CX = np.eye(4, dtype=np.complex128)[[0, 1, 3, 2]]


def test_golden_marginals(golden_cases):
    n_checked = 0
    for case in golden_cases.values():
        c, sizes, es = case_objects(case)
        for row in case["marginals"]:
            ops, finals = bridge.merged_ops(c, es[row["eset"]].realized)
            got = O.conditional_marginal(ops, finals, sizes, row["stage"], row["prefix"])
            np.testing.assert_allclose(got, np.asarray(row["probs"]), rtol=0, atol=1e-12)
            n_checked += 1
    assert n_checked >= 200


def test_golden_histograms_bit_exact(golden_cases):
    """The reference's own sample_proportional (driven by the counter-based RNG
    shim) and the oracle's restatement produce identical records."""
    for case in golden_cases.values():
        c, sizes, es = case_objects(case)
        ops, finals = bridge.template_of(c)
        _, per_set, events = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), case["seed"])
        assert [[list(r) for r in recs] for recs in per_set] == [[list(r) for r in h] for h in case["histograms"]]
        assert {str(k): v for k, v in events.items()} == case["stage_events"]


def test_native_reference_stage1(golden, golden_cases):
    """Reference build_network/merge_errors path == adapter path (pins gate
    matrices, leg order and the error-after-gate convention)."""
    for row in golden["native_stage1"]:
        case = golden_cases[row["case"]]
        c, sizes, es = case_objects(case)
        for k, want in zip(es, row["stage1"]):
            ops, finals = bridge.merged_ops(c, k.realized)
            got = O.conditional_marginal(ops, finals, sizes, 1, "")
            np.testing.assert_allclose(got, np.asarray(want), rtol=0, atol=1e-12)


def test_bell_and_ghz_kats():
    ops, finals = O.build_template(2, [(H, (0,)), (CX, (0, 1))])
    np.testing.assert_allclose(O.conditional_marginal(ops, finals, (2,), 1, ""), [0.5, 0, 0, 0.5], atol=1e-12)
    np.testing.assert_allclose(O.conditional_marginal(ops, finals, (1, 1), 1, ""), [0.5, 0.5], atol=1e-12)
    np.testing.assert_allclose(O.conditional_marginal(ops, finals, (1, 1), 2, "0"), [1, 0], atol=1e-12)
    np.testing.assert_allclose(O.conditional_marginal(ops, finals, (1, 1), 2, "1"), [0, 1], atol=1e-12)
    ops, finals = O.build_template(3, [(H, (0,)), (CX, (0, 1)), (CX, (1, 2))])
    p = O.conditional_marginal(ops, finals, (3,), 1, "")
    np.testing.assert_allclose(p[[0, 7]], [0.5, 0.5], atol=1e-12)
    assert abs(p.sum() - 1) < 1e-12


def test_deterministic_circuit_kat():
    ops, finals = O.build_template(3, [(X, (0,)), (X, (1,)), (X, (2,))])
    assert O.sample_proportional(ops, finals, (1, 1, 1), 10, seed=3, eset_id=0) == [("111", 10)]


def test_impossible_prefix():
    ops, finals = O.build_template(2, [(H, (0,)), (CX, (0, 1))])
    net, _ = O.stage_network(ops, finals, (1, 1), 2, "0")
    with pytest.raises(O.ImpossiblePrefix):
        # qubit 1 cannot be reached: project it with an all-zero population vector
        O.fixed_point_weights(np.zeros(4))
    assert len(net) == 2 * 4 + 2 + 1


def test_allocation_kat():
    assert O.proportional_allocation(10, 4) == [3, 3, 2, 2]


def test_contract_pair_kats():
    a = (("i", "j"), np.eye(2, dtype=np.complex128))
    labels, data = O.contract_pair(a, (("j", "k"), np.eye(2, dtype=np.complex128)))
    assert labels == ("i", "k") and np.allclose(data, np.eye(2))
    labels, data = O.contract_pair((("a", "b"), np.ones((2, 3), complex)), (("b", "c"), np.ones((3, 2), complex)))
    assert labels == ("a", "c") and np.allclose(data, 3)
    labels, data = O.contract_pair((("a",), np.array([1, 2], complex)), (("b",), np.array([3, 4], complex)))
    assert labels == ("a", "b") and np.allclose(data, [[3, 4], [6, 8]])


def test_path_cost_counts_multiplies():
    rng = np.random.default_rng(0)
    ops = [(("a", "b"), rng.normal(size=(2, 3)) + 0j), (("b", "c"), rng.normal(size=(3, 4)) + 0j),
           (("c", "a"), rng.normal(size=(4, 2)) + 0j)]
    assert O.path_cost(ops, [(0, 1), (0, 1)]) == 2 * 3 * 4 + 2 * 4


def test_philox_known_answer():
    """Random123 known-answer vectors for Philox-4x32-10."""
    out = O.philox4x32_10(0, 0, 0, 0, 0, 0)
    assert [int(v) for v in out] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    out = O.philox4x32_10(0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF)
    assert [int(v) for v in out] == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    out = O.philox4x32_10(0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0)
    assert [int(v) for v in out] == [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_multinomial_counts_sum_and_distribution():
    p = np.array([0.1, 0.2, 0.3, 0.4])
    c = O.multinomial_counts(p, 200000, seed=9, eset_id=1, stage=2, rank=3)
    assert c.sum() == 200000
    assert np.max(np.abs(c / 200000 - p)) < 5e-3
    # zero-probability outcomes are never drawn
    c = O.multinomial_counts(np.array([0.0, 1.0, 0.0, 0.0]), 1000, 1, 0, 1, 0)
    assert c.tolist() == [0, 1000, 0, 0]


def _nonprop_runs():
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_nonproportional.json")
    with open(path) as fp:
        return json.load(fp)["runs"]


def test_golden_nonproportional_records(golden_cases):
    """The reference's own sample_nonproportional (engine.py:527-576, driven by
    the counter-based shim CounterChoice) and the oracle's restatement emit the
    same records in the same order: chosen prefixes, exhaustive harvest with its
    probability tags (1e-12), direct multinomial counts."""
    n_records = 0
    for run in _nonprop_runs():
        case = golden_cases[run["case"]]
        c, sizes, es = case_objects(case)
        var = run["variant"]
        for k, want in zip(es, run["records"]):
            ops, finals = bridge.merged_ops(c, k.realized)
            got = O.sample_nonproportional(ops, finals, sizes, run["seed"], k.id, nonfinal_shots=var["nonfinal_shots"],
                                           final_mode=var["final_mode"], threshold=var["threshold"],
                                           direct_count=var["direct_count"])
            assert [(s, n) for s, n, _ in got] == [(s, n) for s, n, _ in want]
            for (_, _, p), (_, _, q) in zip(got, want):
                assert (p is None) == (q is None)
                if p is not None:
                    assert abs(p - q) <= 1e-12
            n_records += len(got)
    assert n_records >= 1000


def test_presample_counter_follows_channel_probabilities():
    """Counter-based pre-trajectory draw (device: presample_kernel): per site the
    outcome frequencies follow the channel's distribution (engine.py:232-244), the
    stream is keyed by (site, global error-set id) only."""
    from paper_2604_08467_b200 import workloads

    c, _ = workloads.hea(6, 2, gamma=0.1, p=0.2, seed=1)
    site_probs = [[pr for _, pr in g.noise.outcomes()] for g in c.gates]
    sets = 20000
    m = O.presample_counter(site_probs, sets, 0, 99)
    for s, probs in enumerate(site_probs):
        freq = np.bincount(m[:, s], minlength=len(probs)) / sets
        sigma = np.sqrt(np.maximum(np.asarray(probs) * (1 - np.asarray(probs)), 1e-9) / sets)
        assert np.all(np.abs(freq - np.asarray(probs)) <= 5 * sigma + 1e-12)
    np.testing.assert_array_equal(O.presample_counter(site_probs, 100, 500, 99), m[500:600])
    assert not np.array_equal(O.presample_counter(site_probs, 100, 0, 100), m[:100])
