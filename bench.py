#!/usr/bin/env python
"""Throughput of the PTSBE proportional hot path (BASELINE.json metric:
shots/sec, device-timed, max over ranks) on synthetic circuits of the named
shapes.

  python bench.py --gpus N --steps K --warmup W            # this repo's CUDA path
  python bench.py --impl reference --gpus N --steps K ...  # the reference algorithm on the host cores

A step = one pass of the hot path (stored-path contraction + non-degenerate
sampling + local histogram) over one batch of pre-sampled error sets.  Weak
scaling: every GPU gets `--sets` error sets; with N > 1 each step ends with
the NCCL exchange of the per-rank histograms by key range (all_to_all) and the
merge of every rank's slice.  Planning/compilation is
excluded from the timed region, as the reference excludes path planning from
its loop time (reference bench.py:5-8, engine.py:895-901).

`value`    inputs resident in HBM (ptsbe_batch_run), device-timed.
`e2e`      ptsbe_sample() with HOST buffers: pinned Kraus-index matrix and shot
           counts copied H2D, histogram copied D2H, inside the timed region.
`roofline` the dominant kernel (stored-path executor, marginal pass of the
           busiest stage): algorithmic bytes and flops per launch over the
           CUDA-event time of those launches.
`cpu_baseline` / `--impl reference`: oracle/ptsbe_oracle.py (numpy port of the
           reference algorithm; the reference itself is pure Python and cannot
           travel to the GPU box) on a bounded sample of the same workload,
           one process per host core.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "shots/sec (device-timed, max over ranks)"


# --------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------

def build_workload(name: str, args):
    from paper_2604_08467_b200 import workloads

    if name == "cfg2":
        c, _ = workloads.hea(30, 6, gamma=0.01, p=0.01, seed=2)
        sizes = (9, 6, 7, 8)  # BatchPlan is an input of the method (reference engine.py:76-142); best of a sweep
        dflt = dict(sets=4096, shots=10_000, dtype="complex64",
                    label="cfg2: 30-qubit HEA depth 6, amplitude damping 0.01 + 2q depolarizing 0.01")
    elif name == "cfg1":
        c, sizes = workloads.ghz(12, p=0.01)
        dflt = dict(sets=64, shots=1000, dtype="complex64", label="cfg1: 12-qubit GHZ, depolarizing 0.01")
    elif name == "cfg3":
        c, sizes = workloads.surface_code(5, 3, p=1e-3, order="ancilla_first")
        dflt = dict(sets=100_000, shots=1, dtype="complex64", label="cfg3: surface code d=5, 3 rounds, p=1e-3")
    elif name == "cfg4":
        c, sizes = workloads.qaoa(50, 2, p=1e-3, seed=4)
        dflt = dict(sets=10_000, shots=10_000, dtype="complex128", label="cfg4: 50-qubit QAOA p=2, 3-regular")
    elif name == "cfg3r1":
        # largest member of the cfg3 family that exact dense contraction reaches: the d = 5 lattice, one round
        # (49 qubits, ancilla blocks first); DESIGN.md section 6b has the width study of 2 and 3 rounds
        c, sizes = workloads.surface_code(5, 1, p=1e-3, order="ancilla_first")
        dflt = dict(sets=100_000, shots=1, dtype="complex64", label="cfg3 at one round: surface code d=5, 1 round, p=1e-3 (49 qubits)")
    elif name == "cfg3s":
        # the full-size cfg3 / cfg4 networks exceed the 2^26-entry intermediate ceiling (the reference's own
        # execute_path raises ResourceLimitError for them too); these are the largest twins that plan
        c, sizes = workloads.surface_code(3, 1, p=1e-3)
        dflt = dict(sets=100_000, shots=1, dtype="complex64", label="cfg3 twin: surface code d=3, 1 round, p=1e-3 (17 qubits)")
    elif name == "cfg4s":
        c, _ = workloads.qaoa(12, 2, p=1e-3, seed=4)
        sizes = (5, 5, 2)
        dflt = dict(sets=2_000, shots=10_000, dtype="complex128", label="cfg4 twin: 12-qubit QAOA p=2, 3-regular")
    elif name == "harvest24":
        # data-harvesting showcase for --mode nonproportional: 24-qubit HEA depth 4, final batch of 20 qubits
        c, _ = workloads.hea(24, 4, gamma=0.0, p=0.01, seed=3)
        sizes = (4, 20)
        dflt = dict(sets=64, shots=1, dtype="complex64", label="24-qubit HEA depth 4, 2q depolarizing 0.01, final batch 20 qubits")
    elif name == "cfg5":
        c, _ = workloads.random40(40, 400, seed=5)
        sizes = (10, 6, 6, 6, 6, 6)  # best of a sweep; 6-qubit stages keep the descent tree in shared memory
        dflt = dict(sets=100_000, shots=100, dtype="complex64", label="cfg5: random_circuit(40, 400)")
    else:
        raise SystemExit(f"unknown workload {name!r}")
    if args.plan:
        sizes = tuple(int(v) for v in args.plan.split(","))
        if sum(sizes) != c.n:
            raise SystemExit(f"--plan must sum to {c.n}")
    sets = args.sets or dflt["sets"]
    shots = args.shots or dflt["shots"]
    dtype = args.dtype or dflt["dtype"]
    return c, sizes, sets, shots, dtype, dflt["label"]


def error_matrix(c, sets: int, first_id: int, seed: int) -> np.ndarray:
    """Kraus-index rows of global error sets [first_id, first_id + sets): the
    stream is keyed by the block of 4096 ids, so any rank layout sees the same
    error set under the same global id."""
    from paper_2604_08467_b200 import workloads

    blk = 4096
    out = np.empty((sets, len(c.gates)), dtype=np.uint8)
    b0, b1 = first_id // blk, (first_id + sets - 1) // blk
    for b in range(b0, b1 + 1):
        rows = workloads.presample_matrix(c, blk, np.random.default_rng([seed, b]))
        lo, hi = max(first_id, b * blk), min(first_id + sets, (b + 1) * blk)
        out[lo - first_id: hi - first_id] = rows[lo - b * blk: hi - b * blk]
    return out


# --------------------------------------------------------------------------
# CPU legs (oracle port of the reference algorithm, process-parallel over error sets)
# --------------------------------------------------------------------------

def _cpu_worker(job):
    """Oracle port (numpy restatement) over a slice of error sets; relative=True applies the
    device's documented relative vanishing-mass floor (oracle.sample_proportional docstring)."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import bridge
    from oracle import ptsbe_oracle as O
    from paper_2604_08467_b200 import workloads

    c, sizes, rows, ids, shots, seed, paths, relative = job
    ops, finals = bridge.template_of(c)
    es = workloads.errorsets_from_matrix(c, rows, shots)
    t0 = time.perf_counter()
    done, recs = 0, []
    for k, gid in zip(es, ids):
        merged = O.merge_errors(ops, bridge.realized_operators(c, k.realized))
        try:
            recs.append(O.sample_proportional(merged, finals, sizes, k.m, seed, int(gid), paths,
                                              relative_floor=relative))
        except O.OracleError as exc:
            recs.append(type(exc).__name__)
        done += k.m
    return done, time.perf_counter() - t0, recs


def oracle_leg(c, sizes, seed: int, rows, ids, shots: int, procs: int, relative: bool = False):
    """The oracle port on the given error sets, one process per core (paths: the oracle's own
    greedy, planned once on the template, excluded from the wall time)."""
    import multiprocessing as mp

    from oracle import bridge
    from oracle import ptsbe_oracle as O

    ops, finals = bridge.template_of(c)
    paths = O.stage_paths(ops, finals, sizes)
    n = rows.shape[0]
    procs = max(1, min(procs, n))
    jobs = []
    for r in range(procs):
        sl = slice(r * n // procs, (r + 1) * n // procs)
        jobs.append((c, sizes, rows[sl], np.asarray(ids)[sl], shots, seed, paths, relative))
    t0 = time.perf_counter()
    if procs == 1:
        res = [_cpu_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    return {"shots_per_s": sum(r[0] for r in res) / wall, "wall_s": wall, "procs": procs,
            "records": [h for r in res for h in r[2]], "plan_s": 0.0}


def cpu_leg(c, sizes, seed: int, sets: int, shots: int, procs: int, hypersamples: int = 100, cache_json=None):
    """Times the reference on `sets` error sets x `shots` shots of the workload (global ids
    0..sets-1 of the bench's error-set stream), error sets sharded over processes, planning excluded
    (reference bench.py:5-8).  kind "reference": the vendored UNMODIFIED reference package
    (oracle/_ref, see oracle/ref_runner.py) -- its planner, its sample_proportional; kind "port":
    the numpy oracle, only when oracle/_ref is absent."""
    from oracle import vendor_ref

    rows = error_matrix(c, sets, 0, seed)
    ids = np.arange(sets, dtype=np.uint32)
    if vendor_ref.available():
        from oracle import ref_runner

        out = ref_runner.run_sample(c, sizes, rows, ids, shots, seed, procs, hypersamples=hypersamples,
                                    cache_json=cache_json)
        out["kind"] = "reference"
    else:
        out = oracle_leg(c, sizes, seed, rows, ids, shots, procs)
        out["kind"] = "port"
    out.update(rows=rows, ids=ids, shots=shots)
    return out


def parity_check(c, sizes, seed: int, cpu: dict, procs: int, device: int, hypersamples: int):
    """Device (complex128, through the C-ABI, per-error-set records) against the CPU leg's
    histograms of the SAME error sets, ids, shots and seed: records must be identical.  Error sets
    the reference refuses (its ABSOLUTE 1e-12 mass floor fires on the trajectory weight of
    amplitude-damping jumps -- a channel its own circuit model does not have) are compared with the
    oracle under the device's relative floor instead, and counted separately."""
    from paper_2604_08467_b200.engine import (BatchPlan, CircuitNetwork, DevicePipeline, SamplerContext,
                                              VariantTables, unpack_keys)

    rows, ids, shots = cpu["rows"], cpu["ids"], cpu["shots"]
    n = rows.shape[0]
    want = list(cpu["records"])
    refused = [e for e in range(n) if isinstance(want[e], str)]
    if refused:
        alt = oracle_leg(c, sizes, seed, rows[refused], ids[refused], shots, procs, relative=True)
        for e, rec in zip(refused, alt["records"]):
            want[e] = rec
    tpl = CircuitNetwork.from_circuit(c)
    ctx = SamplerContext(hypersamples=hypersamples, planner_seed=seed, dtype="complex128", device=device)
    pipe = DevicePipeline(tpl, BatchPlan(sizes), VariantTables.from_channels(tpl), ctx, shots_per_set=float(shots),
                          calibrate=True)
    try:
        keys, esets, counts, st = pipe.device_plan.sample(rows, np.full(n, shots, np.uint32), ids, seed, merged=False)
    finally:
        pipe.close()
    strings = unpack_keys(keys, sum(sizes))
    got = [[] for _ in range(n)]
    for s_, e_, n_ in zip(strings, esets.tolist(), counts.tolist()):
        got[e_].append((s_, int(n_)))
    bad = [e for e in range(n) if isinstance(want[e], str) or got[e] != [tuple(r) for r in want[e]]]
    return {"checked_sets": n, "equal": not bad, "mismatched_sets": bad[:8], "dtype": "complex128",
            "records_compared": int(sum(len(g) for g in got)), "shots_per_set": int(shots),
            "against": cpu["kind"], "reference_refused_sets": len(refused),
            "note": ("per-error-set records of the device vs the CPU leg on identical error sets, ids, seed; "
                     "sets refused by the reference's absolute mass floor are checked against the oracle "
                     "with the relative floor") if refused else
                    "per-error-set records of the device vs the CPU leg on identical error sets, ids, seed"}


def cpu_sample_size(name: str):
    """(error sets, shots per set) of the bounded CPU sample: about 10-30 s of
    host work for the whole pool."""
    return {"cfg1": (64, 1000), "cfg2": (None, 48), "cfg3": (None, 1), "cfg4": (None, 8),
            "cfg5": (None, 40), "cfg3r1": (None, 1), "cfg3s": (64, 1), "cfg4s": (None, 50), "harvest24": (None, 1)}[name]


# --------------------------------------------------------------------------
# clocks
# --------------------------------------------------------------------------

class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.rows, self.proc = [], None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "20", "-i", str(index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), line.strip()))

    def stop(self, t0: float, t1: float) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for t, line in self.rows:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7 or not (t0 <= t <= t1):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# main
# --------------------------------------------------------------------------

def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        doc = json.load(open(path))
        return float(doc["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _cpu_summary(cpu: dict, sets: int, shots: int) -> dict:
    what = ("unmodified reference package (oracle/_ref): its planner (100 hypersamples) and sample_proportional, "
            "counter-based rng shim" if cpu["kind"] == "reference" else "numpy oracle port (oracle/_ref not vendored)")
    return {"value": cpu["shots_per_s"], "unit": "shots/s", "cores": cpu["procs"], "kind": cpu["kind"],
            "sample": f"{sets} error sets x {shots} shots of the same circuit/plan, {cpu['wall_s']:.1f} s wall "
                      f"(planning {cpu['plan_s']:.1f} s excluded); {what}"}


def reference_arm(args):
    """The reference's own CPU implementation of the path on the host cores (one process per core),
    on a bounded sample of the arm's workload; cfg1 runs at its full size (64 x 1000)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    c, sizes, sets, shots, dtype, label = build_workload(args.workload, args)
    cores = os.cpu_count() or 1
    s_sets, s_shots = cpu_sample_size(args.workload)
    s_sets = s_sets or cores
    if args.cpu_sets:
        s_sets = args.cpu_sets
    if args.cpu_shots:
        s_shots = args.cpu_shots
    elif args.steps > 5 and not (s_sets == sets and s_shots == shots):
        # a step is a bounded sample (~18 s for cfg2 at the default size): keep K steps within a few minutes
        s_shots = max(4, s_shots * 5 // args.steps)
    cache_json = None
    for _ in range(min(args.warmup, 1)):
        w = cpu_leg(c, sizes, args.seed, min(s_sets, cores), max(1, s_shots // 4), cores)
        cache_json = w.get("cache_json")
    vals, walls, last = [], [], None
    for _ in range(args.steps):
        last = cpu_leg(c, sizes, args.seed, s_sets, s_shots, cores, cache_json=cache_json)
        cache_json = last.get("cache_json", cache_json)
        vals.append(last["shots_per_s"])
        walls.append(last["wall_s"])
    value = float(np.mean(vals))
    last = dict(last, shots_per_s=value)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "shots/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(walls)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (f64)",
        "data": "synthetic",
        "config": {"workload": label, "plan": list(sizes), "error_sets": s_sets, "shots_per_set": s_shots,
                   "full_size": f"{sets} error sets x {shots} shots per GPU",
                   "same_size_as_gpu_arm": bool(s_sets == sets and s_shots == shots)},
        "cpu_baseline": _cpu_summary(last, s_sets, s_shots),
        "e2e": {"value": value, "unit": "shots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def _np_cpu_worker(job):
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import bridge
    from oracle import ptsbe_oracle as O
    from paper_2604_08467_b200 import workloads

    c, sizes, rows, ids, seed, nonfinal, tau, paths = job
    ops, finals = bridge.template_of(c)
    es = workloads.errorsets_from_matrix(c, rows, 1)
    n = 0
    for k, gid in zip(es, ids):
        merged = O.merge_errors(ops, bridge.realized_operators(c, k.realized))
        try:
            n += len(O.sample_nonproportional(merged, finals, sizes, seed, int(gid), nonfinal_shots=nonfinal,
                                              final_mode="exhaustive", threshold=tau, paths=paths))
        except O.ImpossiblePrefix:
            pass
    return n


def nonproportional_bench(args):
    """Data-harvesting mode (non-proportional NBS, exhaustive final stage): records per second through the
    host-buffer C-ABI call ptsbe_sample_nonproportional (H2D of the Kraus-index matrix and D2H of the records
    inside the timed region), next to the oracle port on the host cores.  Throughput is counted the way the
    reference counts it for this mode: harvested bitstrings / loop seconds (reference bench.py:40-46)."""
    import multiprocessing as mp

    from paper_2604_08467_b200 import _capi
    from paper_2604_08467_b200.engine import (BatchPlan, CircuitNetwork, DevicePipeline, SamplerContext,
                                              VariantTables, marginal_network)
    from paper_2604_08467_b200.planner import find_path_greedy

    c, sizes, sets, _, dtype, label = build_workload(args.workload, args)
    cores = os.cpu_count() or 1
    # CPU leg first (before CUDA is touched): a bounded sample of the same workload
    cpu = None
    if not args.no_cpu:
        tpl, bp = CircuitNetwork.from_circuit(c), BatchPlan(sizes)
        paths = [list(find_path_greedy(marginal_network(tpl, bp, j, "0" * bp.offset(j)).net, hypersamples=100,
                                       rng=np.random.default_rng([args.seed, j])).steps) for j in range(1, bp.f + 1)]
        n_cpu = args.cpu_sets or 8 * cores
        rows = error_matrix(c, n_cpu, 0, args.seed)
        jobs = [(c, sizes, rows[r::cores], np.arange(n_cpu)[r::cores], args.seed, args.nonfinal_shots, args.tau, paths)
                for r in range(min(cores, n_cpu))]
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(len(jobs)) as pool:
            got = sum(pool.map(_np_cpu_worker, jobs))
        wall = time.perf_counter() - t0
        cpu = {"value": got / wall, "unit": "bitstrings/s", "cores": len(jobs), "kind": "port",
               "sample": f"{n_cpu} error sets of the same circuit/plan, {wall:.1f} s wall"}
    if _capi.device_count() < 1:
        raise SystemExit("bench.py needs a CUDA device: libptsbe_b200 has no CPU fallback")
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_channels(tpl)
    ctx = SamplerContext(hypersamples=args.hypersamples, planner_seed=args.seed, dtype=dtype)
    plan = BatchPlan(sizes, nonfinal_shots=args.nonfinal_shots, final_mode="exhaustive", threshold=args.tau)
    pipe = DevicePipeline(tpl, plan, tables, ctx, shots_per_set=float(args.nonfinal_shots))
    dp = pipe.device_plan
    kraus = error_matrix(c, sets, 0, args.seed)
    ids = np.arange(sets, dtype=np.uint32)
    for w in range(max(args.warmup, 1)):
        dp.sample_nonproportional(kraus, ids, args.seed - 1 - w, args.nonfinal_shots, "exhaustive", args.tau, 1)
    t0 = time.perf_counter()
    n_rec, dev_ms, launches = 0, 0.0, 0
    for i in range(args.steps):
        keys, _, counts, probs, st = dp.sample_nonproportional(kraus, ids, args.seed + i, args.nonfinal_shots,
                                                               "exhaustive", args.tau, 1)
        n_rec += int(counts.size)
        dev_ms += float(st.loop_ms)
        launches += int(st.gpu_launches)
    wall = time.perf_counter() - t0
    f = len(sizes)
    print(json.dumps({
        "metric": "harvested bitstrings/sec (non-proportional NBS, exhaustive final stage)", "mode": "nonproportional",
        "value": n_rec / (dev_ms * 1e-3), "unit": "bitstrings/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c64 (f32 FMA)" if dtype == "complex64" else "c128 (f64 FMA)", "data": "synthetic",
        "config": {"workload": label, "plan": list(sizes), "error_sets_per_gpu": sets,
                   "nonfinal_shots": args.nonfinal_shots, "tau": args.tau},
        "e2e": {"value": n_rec / wall, "unit": "bitstrings/s", "h2d_bytes_per_step": int(kraus.nbytes + ids.nbytes),
                "d2h_bytes_per_step": int((n_rec // args.steps) * (8 * dp.words + 8 + 8 + 4))},
        "gpu_launches": launches, "records_per_step": n_rec // args.steps,
        "stage_events": [int(st.stage_events[j]) for j in range(f)], "flagged_work_items": int(st.flagged_sets),
        "cpu_baseline": cpu,
    }))
    pipe.close()


def histogram_checksum(keys: np.ndarray, counts: np.ndarray) -> np.ndarray:
    """Three u64 words, each a sum modulo 2^64 over the records (so slices of a histogram held by
    different ranks add up): record count, total count, sum of mix(key) * count."""
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    if counts.size == 0:
        return np.zeros(3, dtype=np.uint64)
    keys = np.ascontiguousarray(keys, dtype=np.uint64).reshape(len(counts), -1)
    with np.errstate(over="ignore"):
        mix = np.zeros(len(counts), dtype=np.uint64)
        for w in range(keys.shape[1]):
            mix = (mix ^ keys[:, w]) * np.uint64(0x9E3779B97F4A7C15)
            mix ^= mix >> np.uint64(29)
        return np.asarray([len(counts), counts.sum(dtype=np.uint64), (mix * counts).sum(dtype=np.uint64)], dtype=np.uint64)


def dry_run(args, rank: int, world: int, backend: str, sets: int, shots: int):
    """Launcher / rank plumbing without a device: every rank fabricates the histogram of its error-set
    block (key = global id, count = shots), the ranks run the same key-range exchange and reductions
    as the real bench, rank 0 prints the JSON line.  Used by the CPU tests of `--gpus N`."""
    import torch
    import torch.distributed as dist

    from paper_2604_08467_b200.partition import exchange_histograms_by_key_range, shard_bounds

    if world > 1:
        dist.init_process_group("gloo" if backend != "gloo" else backend)
    if args.scaling == "strong":
        lo, hi = shard_bounds(np.full(sets, shots, dtype=np.int64), world)[rank]
    else:
        lo, hi = rank * sets, (rank + 1) * sets
    keys = (torch.arange(lo, hi, dtype=torch.int64) << 58).reshape(-1, 1)  # spread over the key ranges
    counts = torch.full((hi - lo,), shots, dtype=torch.int64)
    if world > 1:
        keys, counts = exchange_histograms_by_key_range(keys, counts)
    ck = histogram_checksum(keys.numpy().view(np.uint64), counts.numpy().view(np.uint64))
    t = torch.tensor([int(v) for v in ck.view(np.int64)], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "shots/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "scaling": args.scaling, "dry_run": True,
                          "error_sets_total": int(t[0]), "shots_total": int(t[1]),
                          "histogram_checksum": [int(v) & (2**64 - 1) for v in t.tolist()]}))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "cfg3r1", "cfg3s", "cfg4s", "harvest24"])
    ap.add_argument("--sets", type=int, default=0, help="error sets PER GPU")
    ap.add_argument("--shots", type=int, default=0, help="shots per error set")
    ap.add_argument("--plan", default="", help="comma-separated batch sizes")
    ap.add_argument("--dtype", default="", choices=["", "complex64", "complex128"])
    ap.add_argument("--hypersamples", type=int, default=64)
    ap.add_argument("--seed", type=int, default=20260408)
    ap.add_argument("--cpu-sets", type=int, default=0)
    ap.add_argument("--cpu-shots", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-wide", action="store_true", help="time the u64 form of the host-buffer call even where the u32 form applies")
    ap.add_argument("--device-presample", action="store_true",
                    help="draw the error sets on the device (ptsbe_batch_presample) for the device-timed leg")
    ap.add_argument("--mode", default="proportional", choices=["proportional", "nonproportional"],
                    help="nonproportional: data-harvesting mode (reference engine.py:527-576), SURVEY 8f #1")
    ap.add_argument("--nonfinal-shots", type=int, default=1)
    ap.add_argument("--tau", type=float, default=1e-4)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: --sets error sets PER GPU; strong: --sets error sets in total, block-partitioned "
                         "over the ranks by shots (partition.shard_bounds)")
    ap.add_argument("--no-parity", action="store_true", help="skip the device-vs-CPU-leg record comparison")
    ap.add_argument("--no-c128", action="store_true", help="skip the complex128 figure printed beside a complex64 run")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / rank plumbing only: synthetic per-rank histograms, no device work (CPU tests)")
    args = ap.parse_args()

    # ---- launcher: `python bench.py --gpus N` starts its own N ranks (one per GPU) ----
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200" and args.mode == "proportional":
        import socket

        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if args.impl == "b200" and args.mode == "proportional" and int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={os.environ.get('WORLD_SIZE', '1')} but --gpus {args.gpus}; "
                         "launch one rank per GPU (torchrun --nproc-per-node N) or let --gpus N start them")

    if args.mode == "nonproportional":
        return nonproportional_bench(args)
    if args.impl == "reference":
        return reference_arm(args)

    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    c, sizes, sets, shots, dtype, label = build_workload(args.workload, args)
    # PTSBE_BENCH_BACKEND=gloo: rendezvous and the final exchange over host memory, ranks may share a
    # GPU (CPU tests of the launcher; a 1-GPU box exercising the N-rank path).  Default: NCCL, one GPU each.
    backend = os.environ.get("PTSBE_BENCH_BACKEND", "nccl")
    if args.dry_run:
        return dry_run(args, rank, world, backend, sets, shots)

    # ---- cpu_baseline leg first (rank 0, N = 1 only), before CUDA is touched ----
    cpu, cpu_raw = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        s_sets, s_shots = cpu_sample_size(args.workload)
        s_sets = args.cpu_sets or s_sets or cores
        s_shots = args.cpu_shots or s_shots
        cpu_raw = cpu_leg(c, sizes, args.seed, s_sets, s_shots, cores)
        cpu = _cpu_summary(cpu_raw, s_sets, s_shots)

    import torch
    import torch.distributed as dist

    from paper_2604_08467_b200 import _capi
    from paper_2604_08467_b200.engine import BatchPlan, CircuitNetwork, DevicePipeline, SamplerContext, VariantTables
    from paper_2604_08467_b200.partition import exchange_histograms_by_key_range, merge_on_device, shard_bounds, _merge_for

    n_dev = _capi.device_count()
    if n_dev < 1:
        raise SystemExit("bench.py needs a CUDA device: libptsbe_b200 has no CPU fallback")
    if backend == "nccl" and world > n_dev:
        raise SystemExit(f"bench.py: {world} ranks but {n_dev} CUDA device(s); NCCL needs one GPU per rank")
    dev = local_rank % n_dev
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            dist.init_process_group(backend)
    where = f"cuda:{dev}" if backend == "nccl" else "cpu"

    # ---- inputs: global error-set ids; weak = `sets` per GPU, strong = `sets` in total, block-partitioned ----
    if args.scaling == "strong":
        lo, hi = shard_bounds(np.full(sets, shots, dtype=np.int64), world)[rank]
        first, sets_local = lo, hi - lo
        if sets_local < 1:
            raise SystemExit(f"strong scaling: rank {rank} got no error sets ({sets} sets over {world} ranks)")
    else:
        first, sets_local = rank * sets, sets
    sets_global = sets if args.scaling == "strong" else sets * world
    kraus = error_matrix(c, sets_local, first, args.seed)
    shots_arr = np.full(sets_local, shots, dtype=np.uint32)
    ids = np.arange(first, first + sets_local, dtype=np.uint32)
    total_shots_local = int(shots_arr.sum())

    # ---- plan once (excluded from timing); identical on every rank (global shots per set) ----
    t0 = time.perf_counter()
    tpl = CircuitNetwork.from_circuit(c)
    tables = VariantTables.from_channels(tpl)
    ctx = SamplerContext(hypersamples=args.hypersamples, planner_seed=args.seed, dtype=dtype, device=dev)
    pipe = DevicePipeline(tpl, BatchPlan(sizes), tables, ctx, shots_per_set=float(shots), calibrate=True)
    plan_s = time.perf_counter() - t0
    dp = pipe.device_plan
    if args.device_presample:
        # error sets [first, first + sets) drawn on the device from the channel probabilities
        site_probs = [[pr for _, pr in g.noise.outcomes()] for g in c.gates]
        batch = dp.presample(site_probs, sets_local, first, shots, args.seed)
        kraus = batch.kraus(sets_local, len(c.gates))  # the host-buffer leg below replays the same error sets
    else:
        batch = dp.upload(kraus, shots_arr, ids)
    merge_fn = _merge_for(where, dev)

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def step(i):
        """One pass over the batch; returns (device ms of this rank, stats)."""
        n_rec, st = batch.run(args.seed + i)
        ms = float(st.loop_ms)
        if world > 1:
            k, cnt = batch.histogram_dev()
            kt = torch.as_tensor(k, device=f"cuda:{dev}").view(torch.int64) if n_rec else \
                torch.zeros((0, dp.words), dtype=torch.int64, device=f"cuda:{dev}")
            ct = torch.as_tensor(cnt, device=f"cuda:{dev}").view(torch.int64) if n_rec else \
                torch.zeros(0, dtype=torch.int64, device=f"cuda:{dev}")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0 = time.perf_counter()
            e0.record()
            if where == "cpu":
                kt, ct = kt.cpu(), ct.cpu()
            # final exchange: every rank receives and merges only its key range of the global histogram
            ks, cs = exchange_histograms_by_key_range(kt, ct, merge=merge_fn)
            e1.record()
            torch.cuda.synchronize()
            # NCCL: device time of the exchange + merge on torch's stream; gloo test mode: host wall clock
            ms += e0.elapsed_time(e1) if where != "cpu" else 1e3 * (time.perf_counter() - w0)
            last_slice[0] = (ks, cs)
        return ms, st

    last_slice = [None]

    for i in range(args.warmup):
        step(-1 - i)
    sync_all()
    sampler = ClockSampler(dev) if rank == 0 else None
    time.sleep(0.15 if sampler else 0.0)
    wall0 = time.perf_counter()
    dev_ms, stats = 0.0, []
    for i in range(args.steps):
        ms, st = step(i)
        dev_ms += ms
        stats.append(st)
    sync_all()
    wall1 = time.perf_counter()
    clocks = sampler.stop(wall0, wall1) if sampler else None

    # shots actually sampled in the last step (histogram total); error sets whose trajectory has zero
    # weight (e.g. amplitude-damping K1 on |0>) are flagged by the device and contribute none
    last_keys, last_counts = batch.fetch()
    sampled_local = int(last_counts.sum())
    # order-independent checksum of the GLOBAL histogram: equal for any world size in strong scaling
    if world > 1 and last_slice[0] is not None:
        ck_keys = last_slice[0][0].cpu().numpy().view(np.uint64)
        ck_counts = last_slice[0][1].cpu().numpy().view(np.uint64)
    else:
        ck_keys, ck_counts = last_keys, last_counts
    checksum_local = histogram_checksum(ck_keys, ck_counts)
    del last_counts, last_keys, ck_keys, ck_counts
    # the resident batch hands its workspaces back to the plan before the host-buffer leg creates its
    # own batch (at E = 10^6 the two would not fit side by side)
    batch.close()
    flagged_local = int(stats[-1].flagged_sets)
    if sampled_local != total_shots_local and flagged_local == 0:
        raise SystemExit(f"histogram holds {sampled_local} shots, expected {total_shots_local}, and nothing was flagged")
    t = torch.tensor([dev_ms, (wall1 - wall0) * 1e3], dtype=torch.float64, device=where)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms_max, wall_ms_max = float(t[0]), float(t[1])
    cnt = torch.tensor([sampled_local, flagged_local] + [int(v) for v in checksum_local.view(np.int64)],
                       dtype=torch.int64, device=where)
    if world > 1:
        dist.all_reduce(cnt)  # int64 sums wrap: the checksum words are sums modulo 2^64
    total_shots = int(cnt[0])
    flagged_total = int(cnt[1])
    checksum = [int(v) & (2**64 - 1) for v in cnt[2:].tolist()]
    value = total_shots * args.steps / (dev_ms_max * 1e-3)

    # ---- e2e through the host-buffer C-ABI call (pinned inputs) ----
    e2e = None
    if not args.no_e2e:
        pin_k = torch.empty(kraus.shape, dtype=torch.uint8, pin_memory=True)
        pin_s = torch.empty(sets_local, dtype=torch.int32, pin_memory=True)
        pin_i = torch.empty(sets_local, dtype=torch.int32, pin_memory=True)
        pin_k.numpy()[:] = kraus
        pin_s.numpy().view(np.uint32)[:] = shots_arr
        pin_i.numpy().view(np.uint32)[:] = ids
        e_steps = max(1, min(args.steps, 3))
        # warm-up: the library hands histograms out in page-locked host buffers that it recycles when
        # the caller drops them; the timed loop holds one result while the next call runs, so two
        # buffer sets must exist before timing starts (pinning 600 MB costs more than a whole step)
        held = None
        for w in range(max(2, min(args.warmup, 3))):
            held = dp.sample(pin_k.numpy(), pin_s.numpy().view(np.uint32), pin_i.numpy().view(np.uint32),
                             args.seed - 1 - w)
        keys = counts = None
        del held
        # one GPU, at most 32 measured qubits: the (key, count) rows come back as two u32 (ptsbe_sample_packed,
        # the call run_ptsbe makes for such plans); the sharded exchange works on the u64 form
        packed = world == 1 and c.n <= 32 and total_shots_local < 2**32 and not args.e2e_wide
        if packed:
            for w in range(2):
                held = dp.sample_packed(pin_k.numpy(), pin_s.numpy().view(np.uint32), pin_i.numpy().view(np.uint32),
                                        args.seed - 10 - w)
            del held
        sync_all()
        w0 = time.perf_counter()
        h2d = d2h = 0
        for i in range(e_steps):
            if packed:
                keys, st = dp.sample_packed(pin_k.numpy(), pin_s.numpy().view(np.uint32),
                                            pin_i.numpy().view(np.uint32), args.seed + i)
            else:
                keys, _, counts, st = dp.sample(pin_k.numpy(), pin_s.numpy().view(np.uint32),
                                                pin_i.numpy().view(np.uint32), args.seed + i)
            h2d, d2h = int(st.h2d_bytes), int(st.d2h_bytes)
            e_parts = {"loop_ms": float(st.loop_ms), "h2d_ms": float(st.h2d_ms), "d2h_ms": float(st.d2h_ms)}
            if world > 1:
                kt = torch.from_numpy(keys.view(np.int64)).to(where)
                ct = torch.from_numpy(counts.view(np.int64)).to(where)
                kk, cc = exchange_histograms_by_key_range(kt, ct, merge=merge_fn)
                cc.cpu()
        sync_all()
        te = torch.tensor([(time.perf_counter() - w0)], dtype=torch.float64, device=where)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": total_shots * e_steps / float(te[0]), "unit": "shots/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e_steps,
               "last_step_device_ms": e_parts, "wall_ms_per_step": 1e3 * float(te[0]) / e_steps,
               "call": "ptsbe_sample_packed (records [R][2] u32)" if packed else "ptsbe_sample (keys u64, counts u64)",
               "timing": "host wall clock around the call, streams drained on both sides"}

    # ---- parity: the CPU leg's histograms against the device on the same error sets (N = 1) ----
    parity = None
    if cpu_raw is not None and not args.no_parity:
        parity = parity_check(c, sizes, args.seed, cpu_raw, os.cpu_count() or 1, dev, args.hypersamples)

    # ---- the same workload in complex128 (the reference's arithmetic), printed beside a complex64 run ----
    c128_leg = None
    if dtype == "complex64" and world == 1 and not args.no_c128:
        ctx2 = SamplerContext(hypersamples=args.hypersamples, planner_seed=args.seed, dtype="complex128", device=dev)
        pipe2 = DevicePipeline(tpl, BatchPlan(sizes), tables, ctx2, shots_per_set=float(shots), calibrate=True)
        b2 = pipe2.device_plan.upload(kraus, shots_arr, ids)
        b2.run(args.seed - 1)
        ms2, k2 = 0.0, min(args.steps, 2)
        for i in range(k2):
            _, st2 = b2.run(args.seed + i)
            ms2 += float(st2.loop_ms)
        c128_leg = {"value": total_shots_local * k2 / (ms2 * 1e-3), "unit": "shots/s", "ms_per_step": ms2 / k2,
                    "steps": k2, "dtype": "c128 (f64 FMA)", "note": "same error sets, plan and seeds; device-timed"}
        b2.close()
        pipe2.close()

    if rank == 0:
        f = len(sizes)
        st = stats[-1]
        elem = 8 if dtype == "complex64" else 16
        real = elem // 2
        marg = [sum(float(s.marg_ms[j]) for s in stats) for j in range(f)]
        hoist = [sum(float(s.hoist_ms[j]) for s in stats) for j in range(f)]
        samp = [sum(float(s.sampler_ms[j]) for s in stats) for j in range(f)]
        comp = [sum(float(s.compact_ms[j]) for s in stats) for j in range(f)]
        hist_ms = sum(float(s.histogram_ms) for s in stats)
        projm = [sum(float(s.project_ms[j]) for s in stats) for j in range(f)]
        desc = [sum(float(s.descent_ms[j]) for s in stats) for j in range(f)]
        words = dp.words
        # candidates for "the dominant kernel": per stage, the per-item executor pass and the dense projection
        cands = []
        for j in range(f):
            pr = pipe.programs_of(j + 1)[-1]
            n_items = sum(int(s.stage_events[j]) for s in stats)
            launches_j = sum(int(s.marg_launches[j]) for s in stats)
            d_items = sum(int(s.descent_items[j]) for s in stats)
            if pr.proj_d and d_items and marg[j] == 0.0:
                # fused descent kernels (csrc/lane.cuh, lane_x.cuh): per-item steps (thread per item) + per-qubit
                # descent (4 lanes or 1 lane per draw); v never leaves the SM.  HBM traffic of one work item: its
                # list entry (eset, parent, mult, slot_off, rank, id, prefix words), one (index, count)
                # pair per draw, nnz; plus, amortised, every record of an earlier pass and every tree
                # column once per launch.
                b_j = sizes[j]
                progs_j = pipe.programs_of(j + 1)
                shots_j = total_shots_local * args.steps
                rec_bytes = sum(float(sum(int(s.stage_events[p]) for s in stats)) * progs_j[p].out_elems * elem
                                for p in range(1, j))  # pass 0 records: read through the tree only
                tree_bytes = float(sets * args.steps) * pr.proj_d * elem * (1 << b_j)
                per_item = 24 + 8 * words + 4 + 8.0 * shots_j / max(d_items, 1) + (rec_bytes + tree_bytes) / max(d_items, 1)
                flops_item = 8.0 * pr.flops * (1.0 + shots_j / max(d_items, 1)) + 4.0 * pr.proj_d * (b_j + 1) * shots_j / max(d_items, 1)
                # Hermitian cuts with 4 or 8 complex entries in complex64 are served by lane_descent_x_kernel
                # (csrc/lane_x.cuh: one lane per draw), everything else by lane_descent_kernel (4 lanes per draw)
                herm_x = dtype == "complex64" and pr.proj_d in (16, 64)
                kname = "lane_descent_x_kernel" if herm_x else "lane_descent_kernel"
                cands.append((desc[j], f"{kname} (per-item steps + per-qubit descent fused, D={pr.proj_d}, b={b_j}), stage {j + 1}, "
                                       "incl. the per-error-set tree tables and the dedup of raw draws",
                              d_items, launches_j, per_item, flops_item, kname))
            elif pr.proj_d and d_items:
                # per-item steps, vector written as one row per item
                cands.append((marg[j], f"exec_kernel (per-item steps -> v[{pr.proj_d}]), stage {j + 1}", n_items, launches_j,
                              pr.ext_read_elems * elem + 8 + 8 * words + pr.proj_d * elem, 8.0 * pr.flops))
                # descent: v read, list entry (eset, mult, slot_off, rank, id), one (index, count) per child,
                # tree columns re-read once per 512-item tile; (b + 1) dot products of D terms per draw
                b_j = sizes[j]
                shots_j = total_shots_local * args.steps
                cands.append((desc[j], f"descent_kernel (per-qubit descent, D={pr.proj_d}, b={b_j}), stage {j + 1}",
                              d_items, launches_j,
                              pr.proj_d * elem + 20 + 8 + pr.proj_d * elem * (1 << b_j) / 512.0,
                              4.0 * pr.proj_d * (b_j + 1) * shots_j / max(d_items, 1)))
            elif pr.proj_d:
                # per-item steps: records read + list entry + Kraus row amortised + vector written
                cands.append((marg[j], f"exec_kernel (per-item steps -> v[{pr.proj_d}]), stage {j + 1}", n_items, launches_j,
                              pr.ext_read_elems * elem + 8 + 8 * words + pr.proj_d * elem, 8.0 * pr.flops))
                # projection: v read, population vector written, M read once per error set and launch
                m_bytes = pr.proj_d * pr.out_elems * elem * (sets * args.steps + launches_j) / max(n_items, 1)
                cands.append((projm[j], f"project_kernel (P = Re(v.M), D={pr.proj_d}, N={pr.out_elems}), stage {j + 1}",
                              n_items, launches_j, pr.proj_d * elem + pr.out_elems * real + m_bytes,
                              4.0 * pr.proj_d * pr.out_elems))
            else:
                # from 3072 error sets on, a stage-1 pass of a lane-sized program runs one thread per error set
                # (exec_lane_kernel<R, 1>, capi.cu lane_big_min), below that the CTA / lane-group kernels
                mname = "exec_lane_kernel (one thread per error set)" if (j == 0 and sets >= 3072 and pr.threads <= 32) \
                    else "exec_kernel"
                cands.append((marg[j], f"{mname} (marginal pass; its span also holds the concurrent up-front passes "
                                       f"of later stages), stage {j + 1}", n_items, launches_j,
                              pr.ext_read_elems * elem + 8 + 8 * words + pr.out_elems * real + 16, 8.0 * pr.flops))
        top = max(cands, key=lambda x: x[0])
        top_ms, top_name, items, launches, item_bytes, item_flops = top[:6]
        # DRAM bytes per work item measured by ncu --set full for this kernel, read from profiles/ncu_traffic.json
        ncu_item_traffic, traffic_src = None, None
        lsu_view = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if len(top) > 6 and os.path.exists(tpath):
            ent = json.load(open(tpath)).get(top[6], {}).get(f"{args.workload}:{dtype}")
            if ent:
                ncu_item_traffic, traffic_src = float(ent["dram_bytes_per_item"]), ent["source"]
                if "lsu_wavefronts_pct_of_peak" in ent:
                    lsu_view = {"frac": float(ent["lsu_wavefronts_pct_of_peak"]) / 100.0, "source": ent["lsu_source"]}
        hbm_peak, peak_src = peaks()
        t_s = top_ms * 1e-3
        achieved = items * item_bytes / t_s / 1e9 if t_s > 0 else 0.0
        fp32_peak, fp64_peak = _capi.measure_fma_peak(dev)
        fma_peak = fp32_peak if dtype == "complex64" else fp64_peak
        tflops = items * item_flops / t_s / 1e12 if t_s > 0 else 0.0
        timed_ms = sum(float(s.loop_ms) for s in stats)
        out = {
            "metric": METRIC, "value": value, "unit": "shots/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None,
            "dtype": "c64 (f32 FMA)" if dtype == "complex64" else "c128 (f64 FMA)", "data": "synthetic",
            "config": {"workload": label, "plan": list(sizes),
                       "error_sets_per_gpu": sets if args.scaling == "weak" else None,
                       "error_sets_total": sets_global, "shots_per_set": shots, "backend": backend if world > 1 else None,
                       "gates": len(c.gates), "hypersamples": args.hypersamples, "plan_s": round(plan_s, 3),
                       "stage_samplers": ["descent" if k else "flat" for k in pipe.stage_samplers.tolist()],
                       "error_sets_from": "device pre-sampling" if args.device_presample else "host matrix",
                       "l2": "per-step working set (work lists, hoisted records, population vectors) exceeds the 126 MB L2"
                             if total_shots_local * 8 > 126e6 else "working set below L2 size (small workload)",
                       "parallelism": f"error sets sharded over {world} GPU(s), {args.scaling} scaling; no traffic while sampling, "
                                      "final NCCL exchange of the histogram by key range (all_to_all) + per-rank merge"},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": int(sum(int(s.gpu_launches) for s in stats)),
            "wall_ms_per_step": wall_ms_max / args.steps,
            "unique_bitstrings": int(st.n_records),
            "sampled_shots_per_step": total_shots, "requested_shots_per_step": sets_global * shots,
            "histogram_checksum": checksum,
            "flagged_work_items": flagged_total,
            "stage_events": [int(st.stage_events[j]) for j in range(f)],
            "kernel_ms_per_step": {
                "exec_marginal": [m / args.steps for m in marg], "project": [m / args.steps for m in projm], "exec_hoist": [h / args.steps for h in hoist],
                "descent": [x / args.steps for x in desc],
                "sampler": [s / args.steps for s in samp], "compaction": [x / args.steps for x in comp],
                "histogram": hist_ms / args.steps, "stage_total": [sum(float(s.stage_ms[j]) for s in stats) / args.steps for j in range(f)],
            },
            "programs": [[{"steps": int(len(pr.steps)), "macs": float(pr.flops), "arena": int(pr.arena_fast),
                           "lanes": int(pr.threads), "proj_d": int(pr.proj_d), "record": int(pr.out_elems)}
                          for pr in pipe.programs_of(j + 1)] for j in range(f)],
            "roofline": {
                "kernel": top_name + (" <float>" if dtype == "complex64" else " <double>"),
                "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak,
                "traffic": (ncu_item_traffic * items / max(launches, 1)) if ncu_item_traffic else None,
                "traffic_source": traffic_src,
                "peak_source": peak_src,
                "bytes_per_item": item_bytes, "items_per_launch": items / max(launches, 1),
                "launch_ms": top_ms / max(launches, 1), "share_of_step": top_ms / max(timed_ms, 1e-9),
                "fma": {"achieved_tflops": tflops, "peak_tflops": fma_peak, "frac": tflops / fma_peak if fma_peak else None,
                        "flops_per_item": item_flops, "peak_source": "ptsbe_measure_fma_peak (independent FMA chains, this run)"},
                # the unit the kernel actually saturates, from the committed ncu capture (not measured in this run)
                "lsu_pipe": lsu_view,
            },
            "cpu_baseline": cpu,
            "parity": parity,
            "c128": c128_leg,
        }
        print(json.dumps(out))
    pipe.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
