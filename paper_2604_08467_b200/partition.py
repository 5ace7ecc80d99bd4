"""Error-set partitioner (north-star subsystem 4): one process per GPU, error
sets split into contiguous blocks, NO traffic while sampling, one gather of
the per-rank histograms at the end.

The reference has no distributed layer; what it pins is the determinism
contract under sharding -- results are independent of how error sets are
spread over lanes (/root/reference/pkg/tests/test_engine.py:455-463, per
error-set RNG streams keyed by k.id, engine.py:889).  The device sampler keys
its Philox streams by (seed, GLOBAL error-set id, stage, prefix rank), so the
merged histogram is bit-identical for any world size.

`merge_records` across ranks (engine.py:815-829) = all_gather of lengths,
padded all_gather of (key words, count) rows, sort + reduce-by-key on the
device (`ptsbe_histogram_merge_dev`).  torch.distributed is plumbing only.
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np


def shard_bounds(shots: Sequence[int], world_size: int) -> list:
    """Contiguous [lo, hi) blocks of error sets per rank, balanced by
    cumulative shots (the cheap proxy for sum_j U_ij); every rank gets at
    least one error set while there are enough of them."""
    shots = np.asarray(shots, dtype=np.int64)
    e = int(shots.size)
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    if e <= world_size:
        return [(min(r, e), min(r + 1, e)) for r in range(world_size)]
    cum = np.cumsum(shots)
    total = int(cum[-1])
    cuts = [0]
    for r in range(1, world_size):
        target = total * r / world_size
        k = int(np.searchsorted(cum, target, side="left")) + 1
        k = max(k, cuts[-1] + 1)          # non-empty shard
        k = min(k, e - (world_size - r))  # leave one for every later rank
        k = max(k, cuts[-1])              # fewer error sets than ranks
        cuts.append(min(max(k, 0), e))
    cuts.append(e)
    return [(cuts[r], cuts[r + 1]) for r in range(world_size)]


def gather_histograms(keys, counts, *, group=None, merge: Optional[Callable] = None):
    """All ranks contribute (keys [R_r, words] u64-as-int64, counts [R_r]) torch
    tensors living on the backend's device (cuda for nccl, cpu for gloo);
    every rank returns the concatenation of all ranks' rows, merged by
    `merge(keys, counts) -> (keys, counts)` when given.  Two collectives:
    lengths, then padded rows -- nothing else crosses NVLink."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    words = keys.shape[1]
    n_local = torch.tensor([keys.shape[0]], dtype=torch.int64, device=keys.device)
    lens = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(lens, n_local, group=group)
    lens = [int(v.item()) for v in lens]
    cap = max(max(lens), 1)
    rows = torch.zeros((cap, words + 1), dtype=torch.int64, device=keys.device)
    if keys.shape[0]:
        rows[: keys.shape[0], :words] = keys
        rows[: keys.shape[0], words] = counts
    out = [torch.empty_like(rows) for _ in range(world)]
    dist.all_gather(out, rows, group=group)
    cat = torch.cat([o[:n] for o, n in zip(out, lens)], dim=0)
    k, c = cat[:, :words].contiguous(), cat[:, words].contiguous()
    if merge is not None:
        k, c = merge(k, c)
    return k, c


def exchange_histograms_by_key_range(keys, counts, *, group=None, merge: Optional[Callable] = None):
    """Final exchange for LARGE histograms: instead of every rank receiving and merging
    everything (`gather_histograms`), the key space is cut into `world` equal ranges of the
    first key word and rank r receives, from every rank, only the records whose key falls into
    range r (one all_to_all of the split sizes, one all_to_all of the rows), then merges its
    slice.  The global histogram is the concatenation of the ranks' slices in rank order, each
    sorted by key; merge work and memory per rank are 1 / world of the gathered form.

    `keys` [R_r, words] (u64 bit patterns as int64) must be sorted by key, as every merged
    per-rank histogram is.  Returns this rank's (keys, counts) slice."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    words = keys.shape[1]
    n = keys.shape[0]
    # destination rank = floor(key0 / 2^64 * world), on the top 32 bits of the first word
    if n:
        top = torch.bitwise_and(torch.bitwise_right_shift(keys[:, 0], 32), 0xFFFFFFFF)
        dest = torch.bitwise_right_shift(top * world, 32)
        send = torch.bincount(dest, minlength=world).to(torch.int64)
    else:
        send = torch.zeros(world, dtype=torch.int64, device=keys.device)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    send_l, recv_l = [int(v) for v in send.tolist()], [int(v) for v in recv.tolist()]
    rows = torch.empty((n, words + 1), dtype=torch.int64, device=keys.device)
    if n:
        rows[:, :words] = keys
        rows[:, words] = counts
    got = torch.empty((sum(recv_l), words + 1), dtype=torch.int64, device=keys.device)
    # sorted input: the records for rank r are one contiguous block, blocks in rank order
    dist.all_to_all_single(got, rows, output_split_sizes=recv_l, input_split_sizes=send_l, group=group)
    k, c = got[:, :words].contiguous(), got[:, words].contiguous()
    if merge is not None and k.shape[0]:
        k, c = merge(k, c)
    return k, c


def merge_on_device(keys, counts, device: int):
    """Sort + reduce-by-key of gathered rows with the library's device kernels.
    Inputs/outputs are int64 cuda tensors holding u64 bit patterns."""
    import torch

    from . import _capi

    torch.cuda.synchronize(device)
    n, words = int(keys.shape[0]), int(keys.shape[1])
    ok, oc = _capi.histogram_merge_dev(keys.data_ptr(), counts.data_ptr(), n, words, device)
    m = ok.shape[0]
    if m == 0:
        return keys[:0], counts[:0]
    k = torch.as_tensor(ok, device=f"cuda:{device}").view(torch.int64).clone()
    c = torch.as_tensor(oc, device=f"cuda:{device}").view(torch.int64).clone()
    ok.free()
    oc.free()
    return k, c


def run_ptsbe_sharded(c, config, errorsets, *, group=None, cache=None):
    """`run_ptsbe` with the error sets block-partitioned over the ranks of the
    (already initialised) process group; every rank returns the same merged
    `RunResult.records`.  Counters (`contract_events`, `stage_events`) are
    summed over ranks; `timings["device_loop_s"]` is the max over ranks."""
    import torch
    import torch.distributed as dist

    from . import engine

    if config.mode != "ptsbe-proportional":
        raise NotImplementedError("the sharded run gathers count histograms; the non-proportional mode "
                                  "(records with probability tags) runs per rank and is merged with merge_records")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    device = config.device
    lo, hi = shard_bounds([k.m for k in errorsets], world)[rank]
    plan = config.plan()
    if hi > lo:
        local = engine.run_ptsbe(c, config, cache=cache, errorsets=errorsets[lo:hi], _keep_packed=True)
    else:  # more ranks than error sets: this rank only takes part in the gather
        words = max(1, (plan.n + 63) // 64)
        local = engine.RunResult(
            mode=config.mode, records=[], unique_shots=0, total_count=0,
            timings={"generate_s": 0.0, "plan_s": 0.0, "loop_s": 0.0, "aggregate_s": 0.0, "path_s": 0.0,
                     "contract_s": 0.0, "device_loop_s": 0.0, "h2d_s": 0.0, "d2h_s": 0.0, "gpu_launches": 0},
            plan_events=0, contract_events=0, stage_events={}, stage_seconds={}, config=config.to_dict(),
            seed=config.seed, shot_allocations=[], packed_keys=np.zeros((0, words), np.uint64),
            packed_counts=np.zeros(0, np.uint64))
    keys = torch.from_numpy(local.packed_keys.view(np.int64)).to(f"cuda:{device}")
    counts = torch.from_numpy(local.packed_counts.view(np.int64)).to(f"cuda:{device}")
    k, cnt = gather_histograms(keys, counts, group=group, merge=lambda a, b: merge_on_device(a, b, device))
    records = [engine.ShotRecord(bitstring=s, count=int(v)) for s, v in
               zip(engine.unpack_keys(k.cpu().numpy().view(np.uint64), plan.n), cnt.cpu().tolist())]
    # counters: sum over ranks; device time: max over ranks
    f = plan.f
    vec = torch.tensor([local.contract_events] + [local.stage_events.get(j, 0) for j in range(1, f + 1)],
                       dtype=torch.int64, device=f"cuda:{device}")
    dist.all_reduce(vec, group=group)
    tmax = torch.tensor([local.timings["device_loop_s"]], dtype=torch.float64, device=f"cuda:{device}")
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX, group=group)
    local.records = records
    local.unique_shots = len(records)
    local.total_count = sum(r.count for r in records)
    local.contract_events = int(vec[0].item())
    local.stage_events = {j: int(vec[j].item()) for j in range(1, f + 1)}
    local.timings["device_loop_s"] = float(tmax.item())
    local.shot_allocations = [int(k.m) for k in errorsets]
    return local
