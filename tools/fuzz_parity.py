"""Randomised parity campaign (GPU): random circuits / noise / batch plans, device complex128
records against the oracle (bit-exact under shared uniforms), proportional and non-proportional.
Usage: python tools/fuzz_parity.py [cases] [seed]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bridge
from oracle import ptsbe_oracle as O
from paper_2604_08467_b200 import workloads
from paper_2604_08467_b200.circuits import random_circuit
from paper_2604_08467_b200.engine import (BatchPlan, CircuitNetwork, SamplerContext, presample_errors,
                                          sample_nonproportional_batched, sample_proportional_batched)

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
only = int(sys.argv[3]) if len(sys.argv) > 3 else None  # replay one case of a campaign
bad = 0
for t in range(cases):
    kind = t % 3
    gamma = 0.0
    if kind == 0:
        n = int(rng.integers(4, 11)); c = random_circuit(n, int(rng.integers(n, 5 * n)), rng=rng)
    elif kind == 1:
        gamma = float(rng.choice([0.0, 0.05]))
        n = int(rng.integers(5, 13)); c, _ = workloads.hea(n, int(rng.integers(2, 5)), gamma=gamma, p=0.05, seed=int(rng.integers(1 << 30)))
    else:
        n = 2 * int(rng.integers(3, 6)); c, _ = workloads.qaoa(n, 2, p=0.05, seed=int(rng.integers(1 << 30)))
    # random batch plan
    sizes, left = [], c.n
    while left:
        b = int(rng.integers(1, min(left, 6) + 1)); sizes.append(b); left -= b
    sizes = tuple(sizes)
    sets = int(rng.integers(1, 6)); shots = int(rng.choice([1, 3, 50, 700]))
    es = presample_errors(c, sets, "uniform", shots_per_set=shots, rng=rng)
    tpl = CircuitNetwork.from_circuit(c)
    seed = int(rng.integers(1 << 40))
    nf, mode = int(rng.integers(1, 4)), str(rng.choice(["exhaustive", "direct"]))
    if only is not None and t != only:
        continue
    ops, finals = bridge.template_of(c)
    try:
        _, want, events = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es), seed)
    except O.ImpossiblePrefix:
        continue
    for lane in ("1", "0"):
        os.environ["PTSBE_LANE"] = lane
        os.environ["PTSBE_DESCENT_MULT"] = "1e18" if t % 2 else "4"
        ctx = SamplerContext(hypersamples=4, dtype="complex128")
        got = sample_proportional_batched(tpl, es, BatchPlan(sizes), seed, ctx)
        got = [[(r.bitstring, r.count) for r in recs] for recs in got]
        if got != want or dict(ctx.stats.stage_events) != events:
            bad += 1
            print("MISMATCH proportional", t, kind, c.n, sizes, sets, shots, "lane", lane, flush=True)
    # non-proportional
    plan = BatchPlan(sizes, nonfinal_shots=nf, final_mode=mode, threshold=1e-3, direct_count=4)
    from paper_2604_08467_b200.errors import ImpossiblePrefixError
    try:
        got = sample_nonproportional_batched(tpl, es, plan, seed, SamplerContext(hypersamples=4, dtype="complex128"))
        dev_raised = False
    except ImpossiblePrefixError:
        got, dev_raised = [[] for _ in es], True
    ref_raised = False
    refs = []
    for k in es:
        mops, _ = bridge.merged_ops(c, k.realized)
        try:
            refs.append(O.sample_nonproportional(mops, finals, sizes, seed, k.id, nonfinal_shots=nf, final_mode=mode,
                                                 threshold=1e-3, direct_count=4))
        except O.ImpossiblePrefix:
            ref_raised = True
            refs.append([])
    if dev_raised or ref_raised:
        # a chosen low-probability child can push the joint mass under the reference's 1e-12 floor
        # (engine.py:475-476): both sides must then report the impossible prefix
        if ref_raised and not dev_raised and gamma > 0.0:
            # documented deviation: the device's vanishing-mass floor is relative to the trajectory weight
            # (non-unitary Kraus operators), the reference's is absolute
            pass
        elif dev_raised != ref_raised:
            # show how many outcomes of each stage-1 / stage-2 population are "positive" only by rounding
            for k in es:
                mops, _ = bridge.merged_ops(c, k.realized)
                p1 = O.conditional_marginal(mops, finals, sizes, 1, "")
                print("  error set", k.id, "stage-1 populations: positive", int((p1 > 0).sum()),
                      "above 1e-12", int((p1 > 1e-12).sum()), "min positive", float(p1[p1 > 0].min()))
            bad += 1
            print("MISMATCH nonproportional error behaviour", t, kind, c.n, sizes, nf, mode, dev_raised, ref_raised, flush=True)
    else:
        for recs, ref in zip(got, refs):
            # outcomes within 1e-9 of the threshold may fall on either side
            a = [(r.bitstring, r.count) for r in recs]
            b = [(s, n_) for s, n_, _ in ref]
            if a != b:
                near = {s for s, _, p in ref if p is not None and abs(p - 1e-3) < 1e-9}
                if {x for x in a if x[0] not in near} != {x for x in b if x[0] not in near}:
                    bad += 1
                    print("MISMATCH nonproportional", t, kind, c.n, sizes, nf, mode, flush=True)
    if t % 10 == 9:
        print(f"{t + 1} cases, {bad} mismatches", flush=True)
print("done:", cases, "cases,", bad, "mismatches")
sys.exit(1 if bad else 0)
