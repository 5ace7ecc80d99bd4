"""Randomised check (GPU) of the merged-output path: run_ptsbe's merged histogram (raw draws of a final descent
stage sorted keys-only, packed u32 records where the plan measures at most 32 qubits) against the merge of the
per-error-set records of the same device run and, in complex128, against the oracle.
Usage: python tools/fuzz_merged.py [cases] [seed]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bridge
from oracle import ptsbe_oracle as O
from paper_2604_08467_b200 import workloads
from paper_2604_08467_b200.circuits import random_circuit
from paper_2604_08467_b200.engine import (BatchPlan, CircuitNetwork, RunConfig, SamplerContext, merge_records,
                                          presample_errors, run_ptsbe, sample_proportional_batched)

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for t in range(cases):
    if t % 2 == 0:
        n = int(rng.integers(4, 13)); c = random_circuit(n, int(rng.integers(n, 5 * n)), rng=rng)
    else:
        n = int(rng.integers(5, 13)); c, _ = workloads.hea(n, int(rng.integers(2, 5)), gamma=float(rng.choice([0.0, 0.05])),
                                                          p=0.05, seed=int(rng.integers(1 << 30)))
    sizes, left = [], c.n
    while left:
        b = int(rng.integers(1, min(left, 6) + 1)); sizes.append(b); left -= b
    sizes = tuple(sizes)
    sets = int(rng.integers(1, 40)); shots = int(rng.choice([1, 3, 20, 300]))
    es = presample_errors(c, sets, "uniform", shots_per_set=shots, rng=rng)
    seed = int(rng.integers(1 << 40))
    dtype = str(rng.choice(["complex128", "complex64"]))
    os.environ["PTSBE_DESCENT_MULT"] = str(rng.choice(["1e18", "4"]))
    cfg = RunConfig(n=c.n, g=len(c.gates), batch_sizes=sizes, seed=seed, hypersamples=4, dtype=dtype,
                    error_sets=len(es), total_shots=sum(k.m for k in es))
    try:
        got = [(r.bitstring, r.count) for r in run_ptsbe(c, cfg, errorsets=es).records]
        per_set = sample_proportional_batched(CircuitNetwork.from_circuit(c), es, BatchPlan(sizes), seed,
                                              SamplerContext(hypersamples=4, dtype=dtype))
        want = [(r.bitstring, r.count) for r in merge_records(per_set)]
        ok = got == want
        if ok and dtype == "complex128":
            ops, finals = bridge.template_of(c)
            _, ora, _ = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), seed)
            ok = got == O.merge_histograms(ora)
    except Exception as exc:  # flagged error sets raise the same exception on both paths: skip the case
        print(f"case {t}: {type(exc).__name__}: {exc}")
        continue
    if not ok:
        bad += 1
        print(f"case {t} MISMATCH n={c.n} sizes={sizes} sets={sets} shots={shots} dtype={dtype} seed={seed}")
print(f"{cases} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
