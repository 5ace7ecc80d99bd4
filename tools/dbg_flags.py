import numpy as np, sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_08467_b200 import workloads, _capi
from paper_2604_08467_b200.engine import *
c, _ = workloads.hea()
tpl = CircuitNetwork.from_circuit(c)
tables = VariantTables.from_channels(tpl)
kraus = workloads.presample_matrix(c, 8, np.random.default_rng(3))
for dtype in ("complex64", "complex128"):
    for sizes in ((10,10,10), (10,10,5,5), (10,5,5,5,5)):
        ctx = SamplerContext(hypersamples=64, planner_seed=1, dtype=dtype)
        pipe = DevicePipeline(tpl, BatchPlan(sizes), tables, ctx, shots_per_set=1e4)
        keys, _, counts, st = pipe.device_plan.sample(kraus, np.full(8, 10000, np.uint32), np.arange(8, dtype=np.uint32), 5, merged=True)
        f = len(sizes)
        print(dtype, sizes, "events", [int(st.stage_events[j]) for j in range(f)], "records", int(st.n_records), "total", int(counts.sum()),
              "flagged", int(st.flagged_sets), "kind", int(st.first_flag_kind), "stage", int(st.first_flag_stage), "id", int(st.first_flagged_id))
        pipe.close()
