"""Generates tests/golden/reference_presample_freq.json from the UNMODIFIED reference -- TEST
INFRASTRUCTURE ONLY (needs /root/reference):  python -m oracle.make_golden_presample

Pins the device-side pre-trajectory sampler to the reference's own
`presample_errors` / `draw_realization` (engine.py:232-281): per gate site, how often each
realized label came out over E error sets drawn by the reference's PCG64 stream.  The device
draws from its counter-based stream, so the comparison is a two-sample chi-square test of the
label frequencies (tests/test_gpu_parity.py), not bit equality."""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import ref_adapter  # noqa: E402


def main():
    ref_adapter.load_reference()
    from ptsbe.circuits import circuit_to_json, random_circuit
    from ptsbe.engine import presample_errors

    cases = []
    for seed, (n, g, e) in enumerate([(6, 30, 6000), (9, 45, 6000)]):
        rc = random_circuit(n, g, 0.3, (0.05, 0.25), np.random.default_rng(900 + seed))
        sets = presample_errors(rc, e, "proportional", e, rng=np.random.default_rng(950 + seed))
        counts = []
        for s in range(g):
            tally: dict = {}
            for k in sets:
                tally[k.realized[s]] = tally.get(k.realized[s], 0) + 1
            counts.append(tally)
        cases.append({"seed": seed, "n": n, "g": g, "error_sets": e, "circuit": circuit_to_json(rc), "site_counts": counts})
    out = os.path.join(ROOT, "tests", "golden", "reference_presample_freq.json")
    with open(out, "w") as fp:
        json.dump({"generator": "oracle/make_golden_presample.py", "reference": "/root/reference/pkg (unmodified)",
                   "numpy": np.__version__, "cases": cases}, fp)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
