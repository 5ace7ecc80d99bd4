"""GPU-mode harness (paper_2604_08467_b200/bench_tools.py) against the reference's bench module
(/root/reference/pkg/src/ptsbe/bench.py): metric KATs, seeds, CSV format, sweep row structure."""

import io
import json
import os

import numpy as np
import pytest

from paper_2604_08467_b200 import bench_tools as B
from paper_2604_08467_b200.engine import RunConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_metric_kats():
    assert B.throughput(100, 4.0) == 25.0
    with pytest.raises(ValueError):
        B.throughput(1, 0.0)
    with pytest.raises(ValueError):
        B.throughput(-1, 1.0)
    assert B.speedup(10.0, 4.0) == 2.5
    with pytest.raises(ValueError):
        B.speedup(1.0, 0.0)
    gm, gsd = B.geo_stats([1.0, 4.0])
    assert gm == pytest.approx(2.0) and gsd == pytest.approx(2.0)
    assert B.geo_stats([5.0]) == (pytest.approx(5.0), pytest.approx(1.0))
    with pytest.raises(ValueError):
        B.geo_stats([])
    with pytest.raises(ValueError):
        B.geo_stats([1.0, 0.0])


def test_circuit_seeds_are_the_references():
    # values printed by the unmodified reference's bench.circuit_instance_seed
    assert B.circuit_instance_seed(7, 5, 14, 0) == 2946264899232920356
    assert B.circuit_instance_seed(7, 5, 14, 3) == 6329219505679610253
    assert B.circuit_instance_seed(123, 16, 80, 1) == 8767528430280540777
    cfg = RunConfig(n=5, g=14)
    c1, s1 = B.instance_circuit(cfg, 7, 0)
    c2, s2 = B.instance_circuit(RunConfig(n=5, g=14, mode="ptsbe-nonproportional"), 7, 0)
    assert s1 == s2 and c1 == c2  # never depends on the mode


def test_csv_columns_and_lossless_round_trip():
    assert B.CSV_COLUMNS[:30] == [
        "row_type", "mode", "n", "g", "instance", "circuit_seed", "run_seed", "batch_sizes", "final_mode", "tau",
        "nonfinal_shots", "hypersamples", "error_sets", "total_shots", "unique_shots", "path_time_s", "loop_time_s",
        "contract_time_s", "throughput", "speedup", "plan_events", "contract_events", "failed", "failed_fraction",
        "geo_mean_throughput", "gsd_throughput", "geo_mean_speedup", "gsd_speedup", "flagged", "error"]
    x = 0.1 + 0.2
    rows = [{"row_type": "instance", "mode": "ptsbe-proportional", "n": 5, "throughput": repr(x), "failed": False,
             "device_loop_s": repr(1e-3 / 3), "not_a_column": 1},
            {"row_type": "summary", "geo_mean_throughput": repr(x), "flagged": False}]
    buf = io.StringIO()
    B.write_csv(rows, buf)
    buf.seek(0)
    back = B.read_csv(buf)
    assert len(back) == 2 and "not_a_column" not in back[0]
    assert float(back[0]["throughput"]) == x and float(back[0]["device_loop_s"]) == 1e-3 / 3
    assert float(back[1]["geo_mean_throughput"]) == x


@pytest.mark.gpu
def test_sweep_rows_shared_circuits_and_failure_rows():
    tpl = RunConfig(n=6, g=20, error_sets=3, total_shots=60, nonfinal_batch=3, final_batch=3, hypersamples=4,
                    seed=5, final_mode="direct", direct_count=4, timeout_s=None)
    modes = ["ptsbe-proportional", "ptsbe-nonproportional", "baseline"]
    rows = B.sweep(tpl, [6, 7], [20], modes, circuits_per_point=2)
    assert len(rows) == 2 * len(modes) * (2 + 1)
    inst = [r for r in rows if r["row_type"] == "instance"]
    summ = [r for r in rows if r["row_type"] == "summary"]
    assert len(summ) == 2 * len(modes)
    for n in (6, 7):
        seeds = {m: [r["circuit_seed"] for r in inst if r["mode"] == m and r["n"] == n] for m in modes}
        assert seeds[modes[0]] == seeds[modes[1]] == seeds[modes[2]]  # shared circuit instances
    good = [r for r in inst if r["mode"] != "baseline"]
    assert all(not r["failed"] and float(r["throughput"]) > 0 and r["plan_events"] >= 1 for r in good)
    assert all(r["unique_shots"] >= 1 and float(r["device_loop_s"]) > 0 for r in good)
    base = [r for r in inst if r["mode"] == "baseline"]
    assert all(r["failed"] and "NotImplementedError" in r["error"] for r in base)
    for s in summ:
        if s["mode"] == "baseline":
            assert s["flagged"] and float(s["failed_fraction"]) == 1.0
        else:
            assert not s["flagged"] and float(s["geo_mean_throughput"]) > 0 and float(s["gsd_throughput"]) >= 1.0
    buf = io.StringIO()
    B.write_csv(rows, buf)
    buf.seek(0)
    assert len(B.read_csv(buf)) == len(rows)


@pytest.mark.gpu
def test_device_presampling_matches_reference_label_frequencies():
    """the device's pre-trajectory sampler against the UNMODIFIED reference's
    presample_errors (engine.py:232-281) -- label frequencies per gate site over 6000 error sets,
    two-sample chi-square (the streams differ: PCG64 there, counter-based Philox here)."""
    from paper_2604_08467_b200.circuits import circuit_from_json
    from paper_2604_08467_b200.engine import (BatchPlan, CircuitNetwork, DevicePipeline, SamplerContext,
                                              VariantTables)

    doc = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_presample_freq.json")))
    for case in doc["cases"]:
        c = circuit_from_json(case["circuit"])
        e = case["error_sets"]
        tpl = CircuitNetwork.from_circuit(c)
        half = c.n // 2
        pipe = DevicePipeline(tpl, BatchPlan((half, c.n - half)), VariantTables.from_channels(tpl),
                              SamplerContext(hypersamples=2), shots_per_set=1.0)
        try:
            site_probs = [[pr for _, pr in g.noise.outcomes()] for g in c.gates]
            labels = [[lb for lb, _ in g.noise.outcomes()] for g in c.gates]
            bt = pipe.device_plan.presample(site_probs, e, 0, 1, 2468 + case["seed"])
            got = bt.kraus(e, len(c.gates))
            bt.close()
        finally:
            pipe.close()
        chi2, dof = 0.0, 0
        for s, tally in enumerate(case["site_counts"]):
            mine = np.bincount(got[:, s], minlength=len(labels[s])).astype(float)
            ref = np.asarray([tally.get(lb, 0) for lb in labels[s]], dtype=float)
            assert ref.sum() == e and mine.sum() == e
            # pool rare labels (two-qubit depolarizing: 15 labels at p / 15 each) so every cell expects >= 5
            order = np.argsort(-(mine + ref))
            cells, acc_m, acc_r = [], 0.0, 0.0
            for k in order:
                acc_m += mine[k]
                acc_r += ref[k]
                if acc_m + acc_r >= 20:
                    cells.append((acc_m, acc_r))
                    acc_m = acc_r = 0.0
            if acc_m + acc_r > 0 and cells:
                cells[-1] = (cells[-1][0] + acc_m, cells[-1][1] + acc_r)
            if len(cells) < 2:
                continue
            for a, b in cells:
                chi2 += (a - b) ** 2 / (a + b)
            dof += len(cells) - 1
        assert dof > 20
        # chi-square with dof degrees of freedom: mean dof, sd sqrt(2 dof); 5 sigma
        assert chi2 <= dof + 5.0 * np.sqrt(2.0 * dof), (case["seed"], chi2, dof)
