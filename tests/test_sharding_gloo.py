"""Multi-GPU host logic on CPU: world_size-2 gloo processes shard the error
sets, each rank samples its shard (here with the oracle standing in for the
device run -- the partitioner/gather code under test is the product's), the
histograms are gathered and merged; the result must equal the single-process
histogram (determinism under sharding, reference tests/test_engine.py:455-463)."""

import json
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case_json, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import case_objects
    from oracle import bridge
    from oracle import ptsbe_oracle as O
    from paper_2604_08467_b200.engine import pack_prefixes, unpack_keys
    from paper_2604_08467_b200.partition import gather_histograms, shard_bounds

    case = json.loads(case_json)
    c, sizes, es = case_objects(case)
    lo, hi = shard_bounds([k.m for k in es], world)[rank]
    ops, finals = bridge.template_of(c)
    if hi > lo:
        hist, _, _ = O.run_proportional(ops, finals, sizes, bridge.oracle_errorsets(c, es[lo:hi]), case["seed"])
    else:
        hist = []
    keys = torch.from_numpy(pack_prefixes([s for s, _ in hist], c.n).view(np.int64))
    counts = torch.tensor([v for _, v in hist], dtype=torch.int64)

    def merge(k, cnt):  # stand-in for ptsbe_histogram_merge_dev on a CPU-only box
        rows = O.merge_histograms([list(zip(unpack_keys(k.numpy().view(np.uint64), c.n), cnt.tolist()))])
        return (torch.from_numpy(pack_prefixes([s for s, _ in rows], c.n).view(np.int64)),
                torch.tensor([v for _, v in rows], dtype=torch.int64))

    k, cnt = gather_histograms(keys, counts, merge=merge)
    got = list(zip(unpack_keys(k.numpy().view(np.uint64), c.n), cnt.tolist()))
    # key-range exchange: every rank ends with a disjoint, merged slice of the same histogram
    from paper_2604_08467_b200.partition import exchange_histograms_by_key_range
    ks, cs = exchange_histograms_by_key_range(keys, counts, merge=merge)
    mine = list(zip(unpack_keys(ks.numpy().view(np.uint64), c.n), cs.tolist()))
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fp:
        json.dump({"hist": got, "shard": [lo, hi], "slice": mine}, fp)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("hea8", 2), ("random10x40", 2), ("random_2", 4)])
def test_sharded_histogram_equals_single_process(golden_cases, tmp_path, name, world):
    from oracle import ptsbe_oracle as O

    case = golden_cases[name]
    want = O.merge_histograms([[tuple(r) for r in h] for h in case["histograms"]])
    mp.spawn(_worker, args=(world, _free_port(), json.dumps(case), str(tmp_path)), nprocs=world, join=True)
    shards, slices = [], []
    for r in range(world):
        doc = json.load(open(tmp_path / f"rank{r}.json"))
        assert [tuple(x) for x in doc["hist"]] == want
        shards.append(tuple(doc["shard"]))
        slices += [tuple(x) for x in doc["slice"]]
    assert slices == want  # slices in rank order = the merged histogram, sorted by key
    assert shards[0][0] == 0 and shards[-1][1] == len(case["errorsets"])
    assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))


def test_shard_bounds_properties():
    from paper_2604_08467_b200.partition import shard_bounds

    rng = np.random.default_rng(0)
    for _ in range(50):
        e = int(rng.integers(1, 200))
        w = int(rng.integers(1, 9))
        shots = rng.integers(1, 1000, size=e)
        b = shard_bounds(shots, w)
        assert len(b) == w and b[0][0] == 0 and b[-1][1] == e
        assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
        if e >= w:
            assert all(hi > lo for lo, hi in b)
            loads = [shots[lo:hi].sum() for lo, hi in b]
            assert max(loads) <= shots.sum() / w + shots.max() + 1
    assert shard_bounds([5] * 8, 8) == [(i, i + 1) for i in range(8)]
