"""Harness on top of the device path: the reference's bench module
(/root/reference/pkg/src/ptsbe/bench.py) restated for the GPU modes, so that `sweep`, the CSV
format and `batch_time_curve` drive this package unchanged.

  throughput / speedup / geo_stats      bench.py:40-64 (unique bitstrings per loop second,
                                        geometric mean and geometric standard deviation)
  circuit_instance_seed / instance_circuit   bench.py:71-89: circuits depend on (root seed, n, g,
                                        instance) only, every mode of a sweep point sees the same ones
  run_instance / sweep / CSV_COLUMNS    bench.py:92-284: instance rows + one summary row per
                                        (point, mode); failures are recorded, not raised, and a
                                        summary is flagged above 20 % failures
  write_csv / read_csv                  bench.py:334-342, lossless (floats are stored by repr)
  batch_time_curve                      bench.py:287-331 (the paper's batch-size study,
                                        PAPER.md:208-214) with device timing

The reference's column list is kept as is and in order (a CSV written here loads in the reference's
reader); GPU columns are appended after it.  `loop_time_s` is the host wall time of the batched device
call (H2D + kernels + D2H), `device_loop_s` the CUDA-event time of the kernels alone.  The comparison
modes ("baseline", "unoptimized-ptsbe") are the reference's deliberately slow CPU strawmen and are
out of scope here: a sweep that names them gets failed rows saying so (and therefore no speed-up
column), exactly like any other per-instance failure.

`batch_time_curve`: for each batch size b the first-stage marginal of a
`BatchPlan.fixed(n, b)` plan is planned once (excluded from timing) and the
stage contraction is timed.  On the device a "contraction" is one work item of
a batched launch, so the figure reported is the CUDA-event time of the
stage-1 executor pass divided by the number of error sets in the batch (row
keys are the reference's, plus `batch` and `device`)."""

from __future__ import annotations

import csv
import time
from dataclasses import replace
from typing import Iterable, Optional, Sequence

import numpy as np

from .circuits import Circuit, random_circuit
from .engine import (BatchPlan, CircuitNetwork, DevicePipeline, RunConfig, RunResult, SamplerContext, VariantTables,
                     run_mode, spawn_rng)
from .errors import SimulationError
from .workloads import presample_matrix

FAILURE_FLAG_FRACTION = 0.2

REFERENCE_COLUMNS = [
    "row_type", "mode", "n", "g", "instance", "circuit_seed", "run_seed", "batch_sizes", "final_mode", "tau",
    "nonfinal_shots", "hypersamples", "error_sets", "total_shots", "unique_shots", "path_time_s", "loop_time_s",
    "contract_time_s", "throughput", "speedup", "plan_events", "contract_events", "failed", "failed_fraction",
    "geo_mean_throughput", "gsd_throughput", "geo_mean_speedup", "gsd_speedup", "flagged", "error",
]
DEVICE_COLUMNS = ["dtype", "device", "device_loop_s", "h2d_s", "d2h_s", "gpu_launches", "shots_per_s"]
CSV_COLUMNS = REFERENCE_COLUMNS + DEVICE_COLUMNS


def throughput(unique_shots: int, loop_seconds: float) -> float:
    if not loop_seconds > 0.0:
        raise ValueError(f"cannot compute throughput over {loop_seconds} s of loop time")
    if unique_shots < 0:
        raise ValueError("unique shot count cannot be negative")
    return unique_shots / loop_seconds


def speedup(fast: float, slow: float) -> float:
    if not slow > 0.0:
        raise ValueError("reference throughput must be positive")
    return fast / slow


def geo_stats(values: Sequence[float]) -> tuple:
    v = np.asarray(list(values), dtype=float)
    if v.size == 0:
        raise ValueError("geo_stats needs at least one value")
    if (v <= 0.0).any():
        raise ValueError("geo_stats requires strictly positive values")
    lg = np.log(v)
    return float(np.exp(lg.mean())), float(np.exp(lg.std()))


def result_throughput(result: RunResult) -> float:
    return throughput(result.unique_shots, result.loop_seconds)


def circuit_instance_seed(root_seed: int, n: int, g: int, instance: int) -> int:
    """Same stream as the reference (spawn key (10, n, g, instance)), so a CSV row's circuit_seed
    regenerates the same circuit in either package."""
    return int(spawn_rng(root_seed, 10, n, g, instance).integers(2**63))


def instance_circuit(config: RunConfig, root_seed: int, instance: int) -> tuple:
    seed = circuit_instance_seed(root_seed, config.n, config.g, instance)
    c = random_circuit(config.n, config.g, two_qubit_fraction=config.two_qubit_fraction, p_range=config.p_range,
                       rng=np.random.default_rng(seed))
    return c, seed


def _echo(config: RunConfig) -> dict:
    plan = BatchPlan.fixed(config.n, config.baseline_batch) if config.mode == "baseline" else config.plan()
    return {
        "mode": config.mode, "n": config.n, "g": config.g, "batch_sizes": ",".join(map(str, plan.sizes)),
        "final_mode": config.final_mode, "tau": repr(config.tau), "nonfinal_shots": config.nonfinal_shots,
        "hypersamples": config.baseline_hypersamples if config.mode == "baseline" else config.hypersamples,
        "error_sets": config.error_sets, "total_shots": config.total_shots,
        "dtype": config.dtype, "device": config.device,
    }


def run_instance(c: Circuit, config: RunConfig, instance: int, circuit_seed: int) -> dict:
    """One run as an instance row.  Simulation failures (resource guards, flagged error sets) and
    modes outside the device path end up in the row's `failed` / `error` fields."""
    row = dict(row_type="instance", instance=instance, circuit_seed=circuit_seed, run_seed=config.seed,
               failed=False, error="", **_echo(config))
    try:
        res = run_mode(c, config)
    except (SimulationError, NotImplementedError) as exc:
        row["failed"], row["error"] = True, f"{type(exc).__name__}: {exc}"
        return row
    t = res.timings
    row.update(unique_shots=res.unique_shots, path_time_s=repr(t["path_s"]), loop_time_s=repr(res.loop_seconds),
               contract_time_s=repr(t["contract_s"]), throughput=repr(result_throughput(res)),
               plan_events=res.plan_events, contract_events=res.contract_events,
               device_loop_s=repr(t.get("device_loop_s", 0.0)), h2d_s=repr(t.get("h2d_s", 0.0)),
               d2h_s=repr(t.get("d2h_s", 0.0)), gpu_launches=t.get("gpu_launches", 0),
               shots_per_s=repr(res.total_count / res.loop_seconds))
    return row


def _summary_row(rows: list) -> dict:
    good = [r for r in rows if not r["failed"]]
    frac = 1.0 - len(good) / len(rows)
    first = rows[0]
    out = {k: first[k] for k in ("mode", "n", "g", "batch_sizes", "final_mode", "tau", "hypersamples", "error_sets",
                                 "total_shots", "dtype", "device")}
    out.update(row_type="summary", failed_fraction=repr(frac), flagged=frac > FAILURE_FLAG_FRACTION)
    if good:
        gm, gsd = geo_stats([float(r["throughput"]) for r in good])
        out.update(geo_mean_throughput=repr(gm), gsd_throughput=repr(gsd))
        ratios = [float(r["speedup"]) for r in good if r.get("speedup")]
        if ratios:
            gm, gsd = geo_stats(ratios)
            out.update(geo_mean_speedup=repr(gm), gsd_speedup=repr(gsd))
    return out


def _sweep_point(template: RunConfig, n: int, g: int, modes, per_point: int, circuits) -> list:
    sizes = template.batch_sizes if (template.batch_sizes and sum(template.batch_sizes) == n) else None
    cfg0 = replace(template, n=n, g=g, batch_sizes=sizes)
    inst = []
    for i in range(per_point):
        c, cs = (circuits[i], template.seed) if circuits is not None else instance_circuit(cfg0, template.seed, i)
        inst.append((i, c, cs))
    table = {}
    for mode in modes:
        table[mode] = [run_instance(c, replace(cfg0, mode=mode,
                                               seed=int(spawn_rng(template.seed, 11, n, g, i).integers(2**31))), i, cs)
                       for i, c, cs in inst]
    base = {r["instance"]: float(r["throughput"]) for r in table.get("baseline", ()) if not r["failed"]}
    out = []
    for mode in modes:
        for r in table[mode]:
            if mode != "baseline" and not r["failed"] and base.get(r["instance"]):
                r["speedup"] = repr(speedup(float(r["throughput"]), base[r["instance"]]))
        out += table[mode] + [_summary_row(table[mode])]
    return out


def sweep(template: RunConfig, ns: Sequence[int], gs: Sequence[int], modes: Sequence[str], circuits_per_point: int = 10,
          circuits: Optional[Sequence[Circuit]] = None, point_workers: int = 1) -> list:
    """Grid sweep over (n, g) points x modes on shared circuit instances (bench.py:215-254).  One device serves
    every run, so points run one after the other whatever `point_workers` says (the argument is kept for
    signature compatibility; concurrent points would only share the GPU)."""
    if circuits is not None and (len(ns) != 1 or len(gs) != 1):
        raise ValueError("explicit circuits require a single (n, g) point")
    rows = []
    for n in ns:
        for g in gs:
            rows += _sweep_point(template, n, g, modes, circuits_per_point, circuits)
    return rows


def write_csv(rows: Iterable[dict], fp) -> None:
    w = csv.DictWriter(fp, fieldnames=CSV_COLUMNS, extrasaction="ignore")
    w.writeheader()
    for r in rows:
        w.writerow(r)


def read_csv(fp) -> list:
    return [dict(r) for r in csv.DictReader(fp)]


def batch_time_curve(c: Circuit, b_values: Sequence[int], hypersamples: int = 100, seed: int = 0, reps: int = 3,
                     max_intermediate: int = 2**26, batch: int = 1024, dtype: str = "complex128",
                     device: int = 0) -> list:
    rows = []
    template = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_channels(template)
    kraus = presample_matrix(c, batch, np.random.default_rng([seed, 77]))
    shots = np.ones(batch, dtype=np.uint32)
    for b in b_values:
        if b > c.n or b > 14:  # the flat sampler serves stage batches of at most 14 qubits
            continue
        plan = BatchPlan.fixed(c.n, b)
        ctx = SamplerContext(hypersamples=hypersamples, planner_seed=seed, max_intermediate=max_intermediate,
                             dtype=dtype, device=device)
        t0 = time.perf_counter()
        pipe = DevicePipeline(template, plan, tables, ctx, shots_per_set=1.0)  # all stages: the run goes through them
        path_s = time.perf_counter() - t0
        try:
            resident = pipe.device_plan.upload(kraus, shots, np.arange(batch, dtype=np.uint32))
            times = []
            for r in range(reps + 1):  # first pass builds the variant-0 memo and warms the workspaces
                _, st = resident.run(seed + r)
                if r:
                    times.append(float(st.marg_ms[0]) * 1e-3 / batch)
            resident.close()
        finally:
            pipe.close()
        best = min(times)
        rows.append({"b": b, "stage_seconds": best, "per_qubit_seconds": best / b, "path_seconds": path_s,
                     "est_cost": float(sum(pipe.stage_flops[1])), "reps": reps, "batch": batch, "device": device})
    return rows
