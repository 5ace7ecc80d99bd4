"""Runs the vendored, UNMODIFIED reference (oracle/_ref/ptsbe, see
oracle/vendor_ref.py) on a bounded sample of a bench workload -- TEST
INFRASTRUCTURE ONLY (bench.py's cpu_baseline / --impl reference leg and the
parity tests).

What is executed is the reference's own proportional pipeline, exactly as its
`run_ptsbe` arranges it (engine.py:832-929): one path per stage planned by ITS
planner on the error-free template (`cache_lookup_or_plan`, engine.py:867-879;
excluded from loop time as the reference excludes it, bench.py:5-8), then its
`sample_proportional` (engine.py:493-524) per error set against the shared
`PathCache`.  `run_ptsbe` itself cannot be called for the BASELINE workloads
because its `Circuit` model rejects their gate set; the
network enters through `ref_adapter.kraus_network` (a `CircuitNetwork` subclass
overriding `.merged`, which is all the sampler touches).  The `rng` argument
is the counter-based shim (`oracle.ptsbe_oracle.CounterMultinomial`), so the
histograms are comparable bit for bit with the device's.  Error sets are
sharded over PROCESSES (the reference's thread lanes slow it down, SURVEY
section 0 finding 5).  Nothing from libptsbe_b200.so is loaded here.
"""

from __future__ import annotations

import io
import os
import time

import numpy as np

from . import ref_adapter, vendor_ref


def _site_tables(c):
    from paper_2604_08467_b200.circuits import is_identity_label

    return [{lb: g.noise.operator(lb) for lb, _ in g.noise.outcomes() if not is_identity_label(lb) or lb == "K0"}
            for g in c.gates]


def reference_network(c):
    """The circuit as the reference's engine sees it (template CircuitNetwork)."""
    from paper_2604_08467_b200.circuits import gate_matrix

    ref = vendor_ref.load()
    return ref_adapter.kraus_network(ref, c.n, [(gate_matrix(g), g.targets) for g in c.gates], _site_tables(c))


def plan_paths(c, sizes, hypersamples: int, seed: int) -> tuple:
    """(PathCache JSON, planning seconds): the warm-up loop of run_ptsbe (engine.py:867-879)."""
    vendor_ref.load()
    from ptsbe.engine import BatchPlan, marginal_network, spawn_rng
    from ptsbe.planner import PathCache, cache_lookup_or_plan

    net = reference_network(c)
    plan = BatchPlan(sizes=tuple(sizes))
    cache = PathCache()
    t0 = time.perf_counter()
    for j in range(1, plan.f + 1):
        mnet = marginal_network(net, plan, j, "0" * plan.offset(j))
        cache_lookup_or_plan(cache, mnet.net, stage=j, hypersamples=hypersamples, rng=spawn_rng(seed, 3, j))
    plan_s = time.perf_counter() - t0
    buf = io.StringIO()
    cache.save(buf)
    return buf.getvalue(), plan_s


def _worker(job):
    os.environ["OMP_NUM_THREADS"] = "1"
    c, sizes, rows, ids, shots, seed, cache_json, hypersamples = job
    vendor_ref.load()
    from ptsbe.engine import BatchPlan, ErrorSet, SamplerContext, sample_proportional
    from ptsbe.errors import SimulationError
    from ptsbe.planner import PathCache

    from paper_2604_08467_b200 import workloads

    from .ptsbe_oracle import CounterMultinomial

    net = reference_network(c)
    plan = BatchPlan(sizes=tuple(sizes))
    cache = PathCache.load(io.StringIO(cache_json))
    es = workloads.errorsets_from_matrix(c, rows, shots)
    out, events, done, plan_events = [], {}, 0, 0
    t0 = time.perf_counter()
    for k, gid in zip(es, ids):
        ctx = SamplerContext(cache=cache, hypersamples=hypersamples, planner_seed=seed, max_intermediate=2**26)
        try:
            recs = sample_proportional(net, ErrorSet(id=int(gid), realized=tuple(k.realized), m=k.m), plan,
                                       CounterMultinomial(seed, int(gid)), ctx)
            out.append([(r.bitstring, int(r.count)) for r in recs])
        except SimulationError as exc:  # ImpossiblePrefixError / NumericalError: the set is reported, not sampled
            out.append(type(exc).__name__)
        done += k.m
        plan_events += ctx.stats.plan_events
        for j, v in ctx.stats.stage_events.items():
            events[j] = events.get(j, 0) + v
    return done, time.perf_counter() - t0, out, events, plan_events


def run_sample(c, sizes, rows, ids, shots, seed: int, procs: int, hypersamples: int = 100, cache_json=None) -> dict:
    """Reference proportional sampling of error sets `rows` (Kraus-index matrix, global ids `ids`),
    `shots` per set, over `procs` processes.  Returns shots/s over the loop wall time (planning
    excluded), the per-set histograms in id order, the stage events and the planning time."""
    import multiprocessing as mp

    plan_s = 0.0
    if cache_json is None:
        cache_json, plan_s = plan_paths(c, sizes, hypersamples, seed)
    n = rows.shape[0]
    procs = max(1, min(procs, n))
    ids = np.asarray(ids)
    jobs = []
    for r in range(procs):
        sl = slice(r * n // procs, (r + 1) * n // procs)
        jobs.append((c, tuple(sizes), rows[sl], ids[sl], shots, seed, cache_json, hypersamples))
    t0 = time.perf_counter()
    if procs == 1:
        res = [_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_worker, jobs)
    wall = time.perf_counter() - t0
    events: dict = {}
    for r in res:
        for j, v in r[3].items():
            events[j] = events.get(j, 0) + v
    return {
        "shots_per_s": sum(r[0] for r in res) / wall, "wall_s": wall, "procs": procs, "plan_s": plan_s,
        "records": [h for r in res for h in r[2]], "stage_events": events,
        "replans_in_loop": sum(r[4] for r in res), "cache_json": cache_json,
    }
