"""Generates tests/golden/reference_nonproportional.json from the UNMODIFIED
reference -- TEST INFRASTRUCTURE ONLY.  Run in the build container:

    python -m oracle.make_golden_nonprop

Pins the non-proportional sampler (reference engine.py:527-576): the
reference's own `sample_nonproportional` is driven by the counter-based shim
oracle.ptsbe_oracle.CounterChoice (its `rng` is duck-typed: `.choice` at
engine.py:555 and `.multinomial` at engine.py:569 are the only calls), on the
circuits of tests/golden/reference_cases.json, for
(nonfinal_shots, final_mode) in {(1, exhaustive), (3, exhaustive), (2, direct)}.
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref_adapter  # noqa: E402
from oracle.make_golden import site_tables  # noqa: E402
from oracle.ptsbe_oracle import CounterChoice  # noqa: E402
from paper_2604_08467_b200.circuits import circuit_from_json, gate_matrix  # noqa: E402

VARIANTS = [
    {"nonfinal_shots": 1, "final_mode": "exhaustive", "threshold": 1e-3, "direct_count": 1},
    {"nonfinal_shots": 3, "final_mode": "exhaustive", "threshold": 1e-2, "direct_count": 1},
    {"nonfinal_shots": 2, "final_mode": "direct", "threshold": 1e-6, "direct_count": 5},
]
CASES = ["ghz12", "random_0", "random_2", "random_4", "hea8", "qaoa8", "surface_d3_r1", "random10x40"]


def main():
    ref = ref_adapter.load_reference()
    from ptsbe.engine import BatchPlan, ErrorSet as RefErrorSet, SamplerContext, sample_nonproportional
    from ptsbe.planner import PathCache

    with open(os.path.join(ROOT, "tests", "golden", "reference_cases.json")) as fp:
        base = {c["name"]: c for c in json.load(fp)["cases"]}
    out = []
    for name in CASES:
        case = base[name]
        c = circuit_from_json(case["circuit"])
        net = ref_adapter.kraus_network(ref, c.n, [(gate_matrix(g), g.targets) for g in c.gates], site_tables(c))
        cache = PathCache()
        for v, var in enumerate(VARIANTS):
            plan = BatchPlan(sizes=tuple(case["sizes"]), nonfinal_shots=var["nonfinal_shots"],
                             final_mode=var["final_mode"], threshold=var["threshold"], direct_count=var["direct_count"])
            seed = 9000 + 10 * len(out) + v
            per_set = []
            for k in case["errorsets"]:
                rk = RefErrorSet(id=k["id"], realized=tuple(k["realized"]), m=k["m"])
                ctx = SamplerContext(cache=cache, hypersamples=4, planner_seed=7)
                recs = sample_nonproportional(net, rk, plan, CounterChoice(seed, k["id"], case["sizes"]), ctx)
                per_set.append([[r.bitstring, int(r.count), None if r.prob is None else float(r.prob)] for r in recs])
            out.append({"case": name, "variant": var, "seed": seed, "records": per_set})
    path = os.path.join(ROOT, "tests", "golden", "reference_nonproportional.json")
    with open(path, "w") as fp:
        json.dump({"generator": "oracle/make_golden_nonprop.py", "reference": "/root/reference/pkg (unmodified)",
                   "runs": out}, fp)
    print(f"wrote {len(out)} runs, {sum(len(r) for run in out for r in run['records'])} records, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
