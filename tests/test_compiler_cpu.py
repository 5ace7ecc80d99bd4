"""Plan compiler vs oracle, on the CPU: the flat device programs (gather
tables, arena placement, hoist passes, Kraus/prefix selectors, folded output
permutation) are interpreted by tests/emulator.py and must reproduce the
golden marginals of the unmodified reference."""

import numpy as np
import pytest

import emulator
from conftest import case_objects
from paper_2604_08467_b200 import compiler
from paper_2604_08467_b200.engine import (
    BatchPlan, CircuitNetwork, DevicePipeline, SamplerContext, VariantTables, marginal_network,
)
from paper_2604_08467_b200.planner import PathCache, find_path_greedy, path_cost
from paper_2604_08467_b200.tensor import network_signature


def _pipeline(case, dtype="complex128", hypersamples=4):
    c, sizes, es = case_objects(case)
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_errorsets(tpl, es)
    ctx = SamplerContext(hypersamples=hypersamples, planner_seed=5, dtype=dtype)
    pipe = DevicePipeline(tpl, BatchPlan(sizes), tables, ctx, shots_per_set=100.0, upload=False)
    return pipe, tables, es


@pytest.mark.parametrize("name", ["ghz12", "ghz6_per_qubit", "random_0", "random_4", "hea8", "qaoa8",
                                  "surface_d3_r1", "random10x40"])
def test_compiled_programs_reproduce_golden_marginals(golden_cases, name):
    case = golden_cases[name]
    pipe, tables, es = _pipeline(case)
    idx = tables.encode(es)
    for row in case["marginals"]:
        j = row["stage"]
        bits = [int(ch) for ch in row["prefix"]] + [0] * (pipe.plan.n - len(row["prefix"]))
        rec = emulator.run_stage(pipe.programs_of(j), pipe.compiled.pool, idx[row["eset"]], bits)
        probs = np.clip(rec.real, 0, None)
        assert np.max(np.abs(rec.imag)) < 1e-12
        np.testing.assert_allclose(probs / probs.sum(), np.asarray(row["probs"]), rtol=0, atol=1e-11)


def test_complex64_pool_within_tolerance(golden_cases):
    case = golden_cases["hea8"]
    pipe, tables, es = _pipeline(case, dtype="complex64")
    assert pipe.compiled.pool.dtype == np.complex64
    idx = tables.encode(es)
    for row in case["marginals"][:12]:
        bits = [int(ch) for ch in row["prefix"]] + [0] * (pipe.plan.n - len(row["prefix"]))
        rec = emulator.run_stage(pipe.programs_of(row["stage"]), pipe.compiled.pool, idx[row["eset"]], bits,
                                 dtype=np.complex64)
        probs = np.clip(rec.real, 0, None)
        want = np.asarray(row["probs"])
        assert np.max(np.abs(probs / probs.sum() - want)) <= 1e-5 * want.max()


def test_hoisting_moves_work_out_of_the_marginal_pass(golden_cases):
    """Error-independent unified path: in stage j >= 2 part of the tree depends
    on the error set only (pass 0) and is not recomputed per prefix."""
    pipe, _, _ = _pipeline(golden_cases["random10x40"], hypersamples=16)
    for j in range(2, pipe.plan.f + 1):
        flops = pipe.stage_flops[j]
        assert len(flops) == j
        assert flops[0] > 0
        assert flops[-1] < sum(flops)
    # one plan event per stage, paths shared by every error set (engine.py:864-879)
    assert pipe.ctx.stats.plan_events == pipe.plan.f


def test_one_stored_path_per_stage_and_cache_reuse(golden_cases):
    case = golden_cases["ghz12"]
    c, sizes, es = case_objects(case)
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_errorsets(tpl, es)
    cache = PathCache()
    ctx = SamplerContext(cache=cache, hypersamples=2)
    DevicePipeline(tpl, BatchPlan(sizes), tables, ctx, upload=False)
    assert ctx.stats.plan_events == 3 and len(cache) == 3
    ctx2 = SamplerContext(cache=cache, hypersamples=2)
    DevicePipeline(tpl, BatchPlan(sizes), tables, ctx2, upload=False)
    assert ctx2.stats.plan_events == 0 and cache.hits == 3


def test_signature_is_prefix_and_error_independent(golden_cases):
    c, sizes, es = case_objects(golden_cases["random_4"])
    tpl = CircuitNetwork.from_circuit(c)
    plan = BatchPlan(sizes)
    a = network_signature(marginal_network(tpl, plan, 2, "000").net)
    b = network_signature(marginal_network(tpl.merged(es[0]), plan, 2, "101").net)
    assert a == b


def test_planner_path_is_valid_and_cost_matches(golden_cases):
    c, sizes, _ = case_objects(golden_cases["random10x40"])
    tpl = CircuitNetwork.from_circuit(c)
    net = marginal_network(tpl, BatchPlan(sizes), 2, "0000").net
    one = find_path_greedy(net, hypersamples=1, rng=np.random.default_rng(0))
    many = find_path_greedy(net, hypersamples=32, rng=np.random.default_rng(0))
    assert len(one.steps) == len(net.operands) - 1
    assert path_cost(net, one) == pytest.approx(one.est_cost)
    assert path_cost(net, many) == pytest.approx(many.est_cost)
    assert many.est_cost <= one.est_cost * 1.0000001
    again = find_path_greedy(net, hypersamples=32, rng=np.random.default_rng(0))
    assert again.steps == many.steps


def test_arena_buffers_never_overlap_live_values(golden_cases):
    """Liveness placement: an output buffer must not alias an operand that is
    still to be read (checked structurally on every step)."""
    pipe, _, _ = _pipeline(golden_cases["surface_d3_r1"])
    for pr in pipe.compiled.programs:
        live = {}
        for st in pr.steps:
            ak, ar, bk, br, ok, orf, out_n = (int(v) for v in st[:7])
            if ok == 0:
                for off, n in live.items():
                    reads = [(k, r) for k, r in ((ak, ar), (bk, br)) if k == 0]
                    if any(r == off for _, r in reads):
                        continue
                    assert orf + out_n <= off or off + n <= orf, "output overlaps a live intermediate"
                live[orf] = out_n
            for k, r in ((ak, ar), (bk, br)):
                if k == 0:
                    live.pop(r, None)


def test_bra_subtrees_are_conjugate_twins_not_recomputed(golden_cases):
    """The bra half of the per-item network is the conjugate of the ket half
    (reference engine.py:393 builds it with np.conj): the compiler reads the ket
    results with a conjugation flag instead of contracting the bra half again."""
    pipe, tables, es = _pipeline(golden_cases["hea8"], hypersamples=16)
    flagged = sum(int(np.count_nonzero(pr.steps[:, 11] & 3)) for pr in pipe.compiled.programs if len(pr.steps))
    assert flagged >= 1
    # and the emulated programs still reproduce the reference marginals (checked per case above)
    j = pipe.plan.f
    top = pipe.programs_of(j)[-1]
    assert top.proj_d >= 1 and top.result_kind == 3


def test_variant0_memo_skips_clean_steps_and_keeps_values():
    """Class-0 programs carry a variant-0 memo: steps whose inputs see no error
    are not re-executed per error set.  Emulated with and without the memo the
    records must be identical, and most steps must be skipped at low noise."""
    import dataclasses

    from paper_2604_08467_b200 import workloads

    c, _ = workloads.hea(14, 4, gamma=0.02, p=0.02, seed=7)
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_channels(tpl)
    ctx = SamplerContext(hypersamples=8, planner_seed=3, dtype="complex128")
    pipe = DevicePipeline(tpl, BatchPlan((7, 7)), tables, ctx, shots_per_set=1000.0, upload=False)
    rows = workloads.presample_matrix(c, 12, np.random.default_rng(5))
    rows[0] = 0  # an error-free set: only the always-run steps execute
    memo_programs = 0
    for j in (1, 2):
        progs = pipe.programs_of(j)
        memo_programs += sum(1 for pr in progs if pr.memo_elems)
        plain = [dataclasses.replace(pr, memo_elems=0) for pr in progs]
        for r, row in enumerate(rows):
            bits = [(r >> k) & 1 for k in range(14)]
            stats = {}
            got = emulator.run_stage(progs, pipe.compiled.pool, row, bits, stats=stats)
            want = emulator.run_stage(plain, pipe.compiled.pool, row, bits)
            np.testing.assert_array_equal(got, want)
            if stats:
                assert stats["executed"] < stats["total"]
                if r == 0:
                    assert stats["executed"] <= 0.25 * stats["total"]
    assert memo_programs >= 1


def test_unitary_light_cone_drops_sites_and_keeps_marginals(golden_cases):
    """Sites that act only on traced qubits behind the measured light cone cancel
    against their conjugates (Pauli channels: every realised operator is
    unitary).  Early stages of a unitary-noise circuit lose most of their
    operands; the emulated marginals still equal the reference goldens, and a
    non-unitary channel (amplitude damping) blocks the cancellation."""
    from paper_2604_08467_b200 import workloads
    from paper_2604_08467_b200.engine import _light_cone, stage_operands

    case = golden_cases["random10x40"]
    c, sizes, es = case_objects(case)
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_errorsets(tpl, es)
    plan = BatchPlan(sizes)
    n_kets = len(tpl.net.operands) - tables.n_sites
    dropped = [len(_light_cone(tpl, tables, n_kets, plan.stage_qubits(j).stop)[0]) for j in range(1, plan.f + 1)]
    assert dropped[0] > 0 and dropped[-1] == 0 and dropped == sorted(dropped, reverse=True)
    full, _, _ = stage_operands(tpl, plan, 1, tables, split=True, lightcone=False)
    cone, _, _ = stage_operands(tpl, plan, 1, tables, split=True, lightcone=True)
    assert len(cone) < len(full)
    # values: the golden-marginal test above runs with the light cone on (DevicePipeline default);
    # here: amplitude damping sites are never dropped
    ch, _ = workloads.hea(6, 2, gamma=0.05, p=0.0, seed=1)
    tpl2 = CircuitNetwork.from_circuit(ch)
    tab2 = VariantTables.from_channels(tpl2)
    nk2 = len(tpl2.net.operands) - tab2.n_sites
    gone, _ = _light_cone(tpl2, tab2, nk2, 2)
    kinds = {type(ch.gates[s].noise).__name__ + ":" + ch.gates[s].noise.kind for s in gone}
    assert all("amplitude" not in k for k in kinds)


def test_separable_form_tables_match_the_gather_tables():
    """Large steps carry a GEMM form (aOff, bOff, oA, oB); it must address the
    same operand and output elements as the lo/hi gather tables."""
    from paper_2604_08467_b200 import workloads

    c, _ = workloads.hea(14, 4, gamma=0.02, p=0.02, seed=7)
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_channels(tpl)
    ctx = SamplerContext(hypersamples=8, planner_seed=3, dtype="complex128")
    pipe = DevicePipeline(tpl, BatchPlan((7, 7)), tables, ctx, shots_per_set=1000.0, upload=False)
    checked = 0
    for pr in pipe.compiled.programs:
        t = pr.tables.astype(np.int64)
        for st in pr.steps:
            out_n, kn, lo_n, hi_n, tab = (int(st[k]) for k in (6, 7, 8, 9, 10))
            g_off, m, n = int(st[16]), int(st[17]), int(st[18])
            if not m:
                continue
            assert m * n == out_n
            loA, loB = t[tab: tab + lo_n], t[tab + lo_n: tab + 2 * lo_n]
            hiA = t[tab + 2 * lo_n: tab + 2 * lo_n + hi_n]
            hiB = t[tab + 2 * lo_n + hi_n: tab + 2 * lo_n + 2 * hi_n]
            a_plain = (hiA[:, None] + loA[None, :]).reshape(-1)
            b_plain = (hiB[:, None] + loB[None, :]).reshape(-1)
            aOff, bOff = t[g_off: g_off + m], t[g_off + m: g_off + m + n]
            oA, oB = t[g_off + m + n: g_off + 2 * m + n], t[g_off + 2 * m + n: g_off + 2 * m + 2 * n]
            out = (oA[:, None] + oB[None, :]).reshape(-1)
            assert sorted(out.tolist()) == list(range(out_n))
            a_gemm = np.repeat(aOff, n)
            b_gemm = np.tile(bOff, m)
            np.testing.assert_array_equal(a_plain[out], a_gemm)
            np.testing.assert_array_equal(b_plain[out], b_gemm)
            checked += 1
    assert checked >= 1


@pytest.mark.parametrize("layout,fold", [("0", "0"), ("1", "0"), ("2", "2"), ("1", "2")])
@pytest.mark.parametrize("name", ["random10x40", "hea8", "surface_d3_r1"])
def test_record_layout_and_hoist_folding_do_not_change_values(monkeypatch, golden_cases, name, layout, fold):
    """The compiler may store a record in any label order (consumer layout 0 / 1 / 2) and may evaluate
    a prefix class with the per-item class instead of in a hoist pass of its own (fold): the programs
    must still reproduce the reference's golden marginals (reference engine.py:361-450)."""
    monkeypatch.setenv("PTSBE_RECORD_LAYOUT", layout)
    monkeypatch.setenv("PTSBE_FOLD", fold)
    case = golden_cases[name]
    pipe, tables, es = _pipeline(case, hypersamples=8)
    idx = tables.encode(es)
    for row in case["marginals"]:
        j = row["stage"]
        bits = [int(ch) for ch in row["prefix"]] + [0] * (pipe.plan.n - len(row["prefix"]))
        rec = emulator.run_stage(pipe.programs_of(j), pipe.compiled.pool, idx[row["eset"]], bits)
        probs = np.clip(rec.real, 0, None)
        np.testing.assert_allclose(probs / probs.sum(), np.asarray(row["probs"]), rtol=0, atol=1e-11)


def test_depth_first_step_order_is_topological_and_shrinks_arenas(golden_cases):
    """compile_stage replays the steps of a pass depth first (larger live footprint first): same nodes,
    same values, a smaller or equal arena than in stored-path order."""
    case = golden_cases["random10x40"]
    c, sizes, es = case_objects(case)
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_errorsets(tpl, es)
    from paper_2604_08467_b200.engine import stage_operands
    from paper_2604_08467_b200.planner import plan_stage
    from paper_2604_08467_b200.compiler import SEL_PREFIX, Pool, compile_stage
    plan = BatchPlan(sizes)
    total = {"dfs": 0, "path": 0}
    for j in range(1, plan.f + 1):
        ops, opens, mirror = stage_operands(tpl, plan, j, tables, split=True)
        path = plan_stage([o.labels for o in ops], [o.dims for o in ops], [o.cls for o in ops],
                          [o.sel_kind == SEL_PREFIX for o in ops], opens, [1.0] + [100.0] * (j - 1), 26.0, 26.0,
                          op_mirror=mirror, hypersamples=4, rng=np.random.default_rng(3))
        progs = {}
        for order in ("dfs", "path"):
            progs[order], _ = compile_stage(ops, path.steps, opens, j, Pool(), 16, mirror=mirror, step_order=order)
            total[order] += sum(p.arena_fast + p.arena_spill for p in progs[order])
        for a, b in zip(progs["dfs"], progs["path"]):
            assert len(a.steps) == len(b.steps) and a.flops == b.flops and a.out_elems == b.out_elems
            # every operand of a step is a leaf, a record or the output of an EARLIER step of the program
            produced = set()
            for st in a.steps:
                for kind, ref in ((int(st[0]), int(st[1])), (int(st[2]), int(st[3]))):
                    if kind == 0:
                        assert any(lo <= ref < hi for lo, hi in produced), "arena operand read before it is written"
                if int(st[4]) == 0:
                    produced.add((int(st[5]), int(st[5]) + int(st[6])))
    assert total["dfs"] <= total["path"]
