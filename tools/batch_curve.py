"""Batch-size study on the device (paper Fig. 6 analogue; reference acceptance criterion 7,
tests/test_acceptance.py:230-261): stage-1 contraction time vs batch size b for random_circuit(16, 80)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_08467_b200.bench_tools import batch_time_curve
from paper_2604_08467_b200.circuits import random_circuit

c = random_circuit(16, 80, rng=np.random.default_rng(7))
for dtype in ("complex128", "complex64"):
    rows = batch_time_curve(c, [2, 4, 6, 8, 10, 12, 14], hypersamples=32, seed=1, reps=3, batch=2048, dtype=dtype)
    for r in rows:
        print(json.dumps({"dtype": dtype, **{k: (round(v, 9) if isinstance(v, float) else v) for k, v in r.items()}}))
