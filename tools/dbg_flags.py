"""Debug aid: which guard (vanishing mass / negative diagonal) flags work items of a
workload, per dtype and batch plan.  Usage: python tools/dbg_flags.py [cfg5|cfg2] [sets]"""
import numpy as np, sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_08467_b200 import workloads, _capi
from paper_2604_08467_b200.engine import *
which = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
sets = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
if which == "cfg5":
    c, _ = workloads.random40(40, 400, seed=5)
    shots, plans = 100, ((10, 10, 10, 10), (10, 6, 6, 6, 6, 6))
else:
    c, _ = workloads.hea()
    shots, plans = 10000, ((10, 7, 7, 6),)
tpl = CircuitNetwork.from_circuit(c)
tables = VariantTables.from_channels(tpl)
kraus = workloads.presample_matrix(c, sets, np.random.default_rng(3))
for dtype in ("complex64", "complex128"):
    for sizes in plans:
        ctx = SamplerContext(hypersamples=64, planner_seed=1, dtype=dtype)
        pipe = DevicePipeline(tpl, BatchPlan(sizes), tables, ctx, shots_per_set=float(shots))
        keys, _, counts, st = pipe.device_plan.sample(kraus, np.full(sets, shots, np.uint32), np.arange(sets, dtype=np.uint32), 5, merged=True)
        f = len(sizes)
        print(dtype, sizes, "events", [int(st.stage_events[j]) for j in range(f)], "records", int(st.n_records), "total", int(counts.sum()),
              "flagged", int(st.flagged_sets), "kind", int(st.first_flag_kind), "stage", int(st.first_flag_stage), "id", int(st.first_flagged_id), flush=True)
        pipe.close()
