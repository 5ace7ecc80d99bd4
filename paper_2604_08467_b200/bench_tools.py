"""Harness helpers on top of the device path.

`batch_time_curve` is the device counterpart of the reference's
`bench.batch_time_curve` (bench.py:287-331: the paper's batch-size study,
PAPER.md:208-214): for each batch size b the first-stage marginal of a
`BatchPlan.fixed(n, b)` plan is planned once (excluded from timing) and the
stage contraction is timed.  On the device a "contraction" is one work item of
a batched launch, so the figure reported is the CUDA-event time of the
stage-1 executor pass divided by the number of error sets in the batch (row
keys are the reference's, plus `batch` and `device`)."""

from __future__ import annotations

import time
from typing import Sequence

import numpy as np

from .circuits import Circuit
from .engine import BatchPlan, CircuitNetwork, DevicePipeline, SamplerContext, VariantTables
from .workloads import presample_matrix


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
