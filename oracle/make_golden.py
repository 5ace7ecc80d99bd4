"""Generates tests/golden/*.json from the UNMODIFIED reference -- TEST
INFRASTRUCTURE ONLY.  Run in the build container (needs /root/reference):

    python -m oracle.make_golden

What is pinned (the reference stores no golden vectors,
so they are produced by running it here):
  * conditional marginals per (error set, stage, prefix) from the reference's
    `conditional_marginal` (engine.py:453-477), float64, printed with repr so
    the JSON round trip is exact;
  * histograms from the reference's own `sample_proportional`
    (engine.py:493-524) driven by the counter-based RNG shim
    (oracle.ptsbe_oracle.CounterMultinomial) -- i.e. the reference's loop,
    prefix ordering and normalisation with our uniform draws;
  * the reference's `random_circuit` / `presample_errors` outputs for fixed
    seeds (rng call-order compatibility of the host-side input producers).
Circuits that the reference's circuit model rejects (Ry/Rz/RZZ, non-adjacent
pairs, amplitude damping) enter its engine through oracle.ref_adapter.kraus_network.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import ref_adapter  # noqa: E402
from oracle.ptsbe_oracle import CounterMultinomial  # noqa: E402
from paper_2604_08467_b200 import workloads  # noqa: E402
from paper_2604_08467_b200.circuits import (  # noqa: E402
    Circuit, Gate, NoiseChannel, circuit_from_json, circuit_to_json, gate_matrix, is_identity_label,
)
from paper_2604_08467_b200.engine import ErrorSet, presample_errors  # noqa: E402


def site_tables(c: Circuit):
    return [
        {lb: g.noise.operator(lb) for lb, _ in g.noise.outcomes() if not is_identity_label(lb) or lb == "K0"}
        for g in c.gates
    ]


def reference_case(ref, name, c: Circuit, sizes, errorsets, seed, max_prefixes=3):
    from ptsbe.engine import BatchPlan, ErrorSet as RefErrorSet, SamplerContext, conditional_marginal, sample_proportional
    from ptsbe.planner import PathCache

    tables = site_tables(c)
    net = ref_adapter.kraus_network(ref, c.n, [(gate_matrix(g), g.targets) for g in c.gates], tables)
    plan = BatchPlan(sizes=tuple(sizes))
    cache = PathCache()
    hists, margs = [], []
    events: dict = {}
    for pos, k in enumerate(errorsets):
        rk = RefErrorSet(id=k.id, realized=tuple(k.realized), m=k.m)
        ctx = SamplerContext(cache=cache, hypersamples=4, planner_seed=7)
        shim = CounterMultinomial(seed, k.id)
        recs = sample_proportional(net, rk, plan, shim, ctx)
        hists.append([[r.bitstring, int(r.count)] for r in recs])
        for j, v in ctx.stats.stage_events.items():
            events[str(j)] = events.get(str(j), 0) + v
        merged = net.merged(rk)
        for j in range(1, plan.f + 1):
            off = plan.offset(j)
            seen = sorted({r.bitstring[:off] for r in recs})[:max_prefixes]
            for prefix in seen:
                probs = conditional_marginal(merged, cache, plan, j, prefix, hypersamples=4, planner_seed=7)
                margs.append({"eset": pos, "stage": j, "prefix": prefix, "probs": [float(x) for x in probs]})
    return {
        "name": name,
        "circuit": circuit_to_json(c),
        "sizes": list(sizes),
        "errorsets": [{"id": k.id, "realized": list(k.realized), "m": k.m} for k in errorsets],
        "seed": seed,
        "histograms": hists,
        "stage_events": events,
        "marginals": margs,
    }


def native_reference_check(ref, c: Circuit, sizes, errorsets):
    """For circuits the reference's own model accepts: its build_network /
    merge_errors path must agree with the adapter path (pins gate matrices,
    leg order and the error-after-gate convention)."""
    from ptsbe.circuits import circuit_from_json as ref_from_json
    from ptsbe.engine import BatchPlan, CircuitNetwork, ErrorSet as RefErrorSet, conditional_marginal
    from ptsbe.planner import PathCache

    rc = ref_from_json(circuit_to_json(c))
    tpl = CircuitNetwork.from_circuit(rc)
    plan = BatchPlan(sizes=tuple(sizes))
    out = []
    for k in errorsets:
        merged = tpl.merged(RefErrorSet(id=k.id, realized=tuple(k.realized), m=k.m))
        out.append([float(x) for x in conditional_marginal(merged, PathCache(), plan, 1, "", hypersamples=4)])
    return out


def main():
    ref = ref_adapter.load_reference()
    from ptsbe.circuits import circuit_to_json as ref_to_json, random_circuit as ref_random
    from ptsbe.engine import presample_errors as ref_presample

    cases = []
    # ---- cfg1 twin: GHZ-12, (4,4,4), 6 error sets x 1000 shots -------------------------
    c, sizes = workloads.ghz(12, p=0.05)
    es = presample_errors(c, 6, "uniform", shots_per_set=1000, rng=np.random.default_rng(11))
    cases.append(reference_case(ref, "ghz12", c, sizes, es, seed=101))
    # per-qubit plan on a smaller GHZ (12 stages would be slow on the CPU reference)
    c, _ = workloads.ghz(6, p=0.1)
    es = presample_errors(c, 4, "uniform", shots_per_set=200, rng=np.random.default_rng(12))
    cases.append(reference_case(ref, "ghz6_per_qubit", c, (1,) * 6, es, seed=102))
    # ---- reference random circuits (its own generator and channel kinds) -------------
    native = []
    for seed in range(6):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(3, 8))
        g = int(rng.integers(4, 3 * n))
        rc = ref_random(n, g, rng=rng)
        cmine = circuit_from_json(ref_to_json(rc))
        es = presample_errors(cmine, 3, "uniform", shots_per_set=500, rng=np.random.default_rng(100 + seed))
        half = max(1, n // 2)
        sizes = (half, n - half)
        cases.append(reference_case(ref, f"random_{seed}", cmine, sizes, es, seed=200 + seed))
        native.append({"case": f"random_{seed}", "stage1": native_reference_check(ref, cmine, sizes, es)})
    # ---- cfg2 twin: HEA 8 qubits depth 3, amplitude damping + depolarizing ------------
    c, _ = workloads.hea(8, 3, gamma=0.05, p=0.05, seed=21)
    es = presample_errors(c, 5, "uniform", shots_per_set=400, rng=np.random.default_rng(22))
    cases.append(reference_case(ref, "hea8", c, (3, 3, 2), es, seed=301))
    # ---- cfg4 twin: QAOA 8 qubits p=2 on a 3-regular graph (non-adjacent RZZ) ---------
    c, _ = workloads.qaoa(8, 2, p=0.05, seed=31)
    es = presample_errors(c, 4, "uniform", shots_per_set=300, rng=np.random.default_rng(32))
    cases.append(reference_case(ref, "qaoa8", c, (4, 4), es, seed=401))
    # ---- cfg3 twin: surface code d=2-ish is not defined; use d=3, 1 round (n=17) ------
    c, _ = workloads.surface_code(3, 1, p=0.02)
    es = presample_errors(c, 3, "uniform", shots_per_set=50, rng=np.random.default_rng(42))
    cases.append(reference_case(ref, "surface_d3_r1", c, (6, 6, 5), es, seed=501, max_prefixes=2))
    # ---- cfg5 twin: reference random_circuit(10, 40) ---------------------------------
    rc = ref_random(10, 40, 0.2, (0.02, 0.2), np.random.default_rng(5))
    cmine = circuit_from_json(ref_to_json(rc))
    es = presample_errors(cmine, 4, "uniform", shots_per_set=100, rng=np.random.default_rng(52))
    cases.append(reference_case(ref, "random10x40", cmine, (4, 3, 3), es, seed=601))

    # ---- input producers: rng call-order compatibility ----------------------------------
    producers = []
    for seed in range(4):
        rc = ref_random(5, 14, rng=np.random.default_rng(seed))
        sets = ref_presample(rc, 4, "proportional", 10, rng=np.random.default_rng(50 + seed))
        producers.append({
            "seed": seed, "n": 5, "g": 14, "circuit": ref_to_json(rc),
            "presample_seed": 50 + seed,
            "realized": [list(k.realized) for k in sets], "alloc": [k.m for k in sets],
        })

    out_dir = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "reference_cases.json"), "w") as fp:
        json.dump({"generator": "oracle/make_golden.py", "reference": "/root/reference/pkg (unmodified)",
                   "numpy": np.__version__, "cases": cases, "native_stage1": native,
                   "producers": producers}, fp)
    size = os.path.getsize(os.path.join(out_dir, "reference_cases.json"))
    print(f"wrote {len(cases)} cases, {sum(len(c['marginals']) for c in cases)} marginals, {size} bytes")


if __name__ == "__main__":
    main()
