"""Sharded runs on the device: `run_ptsbe_sharded` with 2 and 3 ranks (gloo
rendezvous, the ranks share GPU 0 -- the test box has one GPU; with NCCL every
rank owns a GPU and the same code moves device buffers) must return exactly
the records of the single-process `run_ptsbe`, in complex64 as well as
complex128: every rank builds tables, light cone, paths and the per-stage
sampler choice from the full error-set list, and RNG streams are keyed by the
global error-set id (determinism under sharding, reference
tests/test_engine.py:455-463)."""

import json
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _job(mode, dtype):
    from paper_2604_08467_b200 import workloads
    from paper_2604_08467_b200.engine import RunConfig, presample_errors

    c, _ = workloads.hea(12, 3, gamma=0.03, p=0.05, seed=9)
    shots = [40, 900, 7, 300, 1200, 55, 2, 640, 81, 350, 19]
    es = presample_errors(c, len(shots), "uniform", shots_per_set=shots, rng=np.random.default_rng(4))
    # ids are global and need not be positions
    es = [type(k)(id=100 + 3 * k.id, realized=k.realized, m=k.m) for k in es]
    cfg = RunConfig(n=12, g=len(c.gates), mode=mode, batch_sizes=(5, 4, 3), seed=17, hypersamples=8, dtype=dtype,
                    nonfinal_shots=2, final_mode="exhaustive", tau=1e-3, timeout_s=None)
    return c, cfg, es


def _worker(rank, world, port, mode, dtype, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_08467_b200.partition import run_ptsbe_sharded

    c, cfg, es = _job(mode, dtype)
    res = run_ptsbe_sharded(c, cfg, es)
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fp:
        json.dump({"records": [[r.bitstring, r.count, r.prob] for r in res.records],
                   "stage_events": {str(k): v for k, v in res.stage_events.items()},
                   "contract_events": res.contract_events, "total": res.total_count}, fp)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,dtype,world", [
    ("ptsbe-proportional", "complex64", 2),
    ("ptsbe-proportional", "complex128", 3),
    ("ptsbe-nonproportional", "complex128", 2),
])
def test_sharded_run_equals_single_process(tmp_path, mode, dtype, world):
    from paper_2604_08467_b200.engine import run_ptsbe

    c, cfg, es = _job(mode, dtype)
    one = run_ptsbe(c, cfg, errorsets=es)
    want = [[r.bitstring, r.count, r.prob] for r in one.records]
    mp.spawn(_worker, args=(world, _free_port(), mode, dtype, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        doc = json.load(open(tmp_path / f"rank{r}.json"))
        assert doc["records"] == want, (mode, dtype, r)
        assert doc["total"] == one.total_count
        assert {int(k): v for k, v in doc["stage_events"].items()} == one.stage_events
        assert doc["contract_events"] == one.contract_events
