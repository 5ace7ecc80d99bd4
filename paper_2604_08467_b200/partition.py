"""Error-set partitioner (north-star subsystem 4): one process per GPU, error
sets split into contiguous blocks, NO traffic while sampling, one gather of
the per-rank histograms at the end.

The reference has no distributed layer; what it pins is the determinism
contract under sharding -- results are independent of how error sets are
spread over lanes (/root/reference/pkg/tests/test_engine.py:455-463, per
error-set RNG streams keyed by k.id, engine.py:889).  The device sampler keys
its Philox streams by (seed, GLOBAL error-set id, stage, prefix rank), and
`run_ptsbe_sharded` builds everything that shapes the arithmetic (variant
tables, light cone, planner weights, stored paths, per-stage sampler choice)
from the full error-set list on every rank, so the merged histogram does not
depend on the world size (GPU test: tests/test_gpu_sharded.py).

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


def _collective_device(group, device: int) -> str:
    """Where tensors must live for the group's backend: NCCL moves device memory over
    NVLink, gloo (CPU tests; several ranks sharing one GPU) moves host memory."""
    import torch.distributed as dist

    return f"cuda:{device}" if dist.get_backend(group) == "nccl" else "cpu"


def _merge_for(where: str, device: int):
    """reduce-by-key of gathered rows on the GPU: device pointers for cuda tensors, the
    host-buffer entry point (H2D + D2H inside) for cpu tensors."""
    if where != "cpu":
        return lambda a, b: merge_on_device(a, b, device)

    def merge_host(k, c):
        import torch

        from . import _capi

        ok, oc = _capi.histogram_merge(k.numpy().view(np.uint64), c.numpy().view(np.uint64), device)
        return (torch.from_numpy(np.ascontiguousarray(ok).view(np.int64)),
                torch.from_numpy(np.ascontiguousarray(oc).view(np.int64)))

    return merge_host


def run_ptsbe_sharded(c, config, errorsets, *, group=None, cache=None):
    """`run_ptsbe` with the error sets block-partitioned over the ranks of the
    (already initialised) process group; every rank returns the same merged
    `RunResult.records`.  Counters (`contract_events`, `stage_events`) are
    summed over ranks; `timings["device_loop_s"]` is the max over ranks.

    Determinism under sharding (reference tests/test_engine.py:455-463): every
    rank builds the variant tables, the light cone, the planner weights, the
    stored paths and the per-stage sampler choice from the FULL error-set list
    and the global mean shot count -- exactly what a single-process run builds --
    and only the error sets it samples differ.  The RNG streams are keyed by the
    global error-set id, so the merged histogram does not depend on the world
    size.  The per-rank histogram never leaves the device before the exchange
    (`ptsbe_batch_histogram_dev`); a failing error set is reported on every rank
    (the ranks agree on the failure before anyone raises, so none is left
    waiting in a collective)."""
    import time

    import torch
    import torch.distributed as dist

    from . import engine
    from .errors import STATUS_TO_ERROR, SimulationError

    if config.mode not in ("ptsbe-proportional", "ptsbe-nonproportional"):
        raise ValueError(f"run_ptsbe_sharded handles optimized modes only, got {config.mode!r}")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    device = config.device
    where = _collective_device(group, device)
    plan = config.plan()
    if plan.n != c.n:
        raise ValueError(f"plan covers {plan.n} qubits, circuit has {c.n}")
    errorsets = list(errorsets)
    lo, hi = shard_bounds([k.m for k in errorsets], world)[rank]
    f = plan.f

    def agree_on_failure(exc):
        """(kind, error-set id) of the failure with the smallest id over all ranks, or None."""
        code = 0
        eid = 2**62
        if exc is not None:
            code = next((k for k, v in STATUS_TO_ERROR.items() if isinstance(exc, v) and type(exc) is v), 1)
            eid = getattr(exc, "eset_id", 2**62 - 1)
        t = torch.tensor([eid, code], dtype=torch.int64, device=where)
        rows = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(rows, t, group=group)
        bad = sorted((int(r[0]), int(r[1])) for r in rows if int(r[1]))
        return bad[0] if bad else None

    if config.mode == "ptsbe-nonproportional":
        # records carry probability tags: per-rank merged records travel as objects, then merge_records
        # (engine.py:815-829; counts summed, a tag survives only if all contributors agree)
        err, local = None, None
        try:
            if hi > lo:
                local = engine.run_ptsbe(c, config, cache=cache, errorsets=errorsets, _shard=(lo, hi))
        except SimulationError as exc:
            err = exc
        bad = agree_on_failure(err)
        if bad is not None:
            raise err if err is not None else SimulationError(f"error set {bad[0]}: failed on another rank")
        parts = [None] * world
        dist.all_gather_object(parts, None if local is None else
                               (local.records, local.contract_events, local.stage_events,
                                local.timings["device_loop_s"]), group=group)
        parts = [p for p in parts if p is not None]
        records = engine.merge_records([p[0] for p in parts])
        stage_events = {j: sum(p[2].get(j, 0) for p in parts) for j in range(1, f + 1)}
        return engine.RunResult(
            mode=config.mode, records=records, unique_shots=len(records),
            total_count=sum(r.count for r in records),
            timings=dict(local.timings, device_loop_s=max(p[3] for p in parts)) if local is not None
            else {"device_loop_s": max(p[3] for p in parts)},
            plan_events=local.plan_events if local is not None else 0,
            contract_events=sum(p[1] for p in parts), stage_events=stage_events,
            stage_seconds=local.stage_seconds if local is not None else {}, config=config.to_dict(),
            seed=config.seed, shot_allocations=[int(k.m) for k in errorsets])

    ctx = engine.SamplerContext(
        cache=cache if cache is not None else engine.PathCache(), hypersamples=config.hypersamples,
        planner_seed=config.seed, max_intermediate=config.max_intermediate,
        deadline=(time.perf_counter() + config.timeout_s) if config.timeout_s else None,
        dtype=config.dtype, device=device)
    t0 = time.perf_counter()
    template = engine.CircuitNetwork.from_circuit(c)
    tables = engine.VariantTables.from_errorsets(template, errorsets)
    shots_all = np.asarray([k.m for k in errorsets], dtype=np.uint32)
    if shots_all.min() < 1:
        raise ValueError("proportional sampling needs m >= 1")
    pipe = engine.DevicePipeline(template, plan, tables, ctx, shots_per_set=float(shots_all.mean()), calibrate=True)
    plan_s = time.perf_counter() - t0
    words = max(1, (plan.n + 63) // 64)
    batch, st, err = None, None, None
    try:
        t0 = time.perf_counter()
        if hi > lo:
            mine = errorsets[lo:hi]
            batch = pipe.device_plan.upload(tables.encode(mine), shots_all[lo:hi],
                                            np.asarray([k.id for k in mine], dtype=np.uint32))
            n_rec, st = batch.run(config.seed)
            try:
                engine._raise_flagged(st)
            except SimulationError as exc:
                exc.eset_id = int(st.first_flagged_id)
                err = exc
        bad = agree_on_failure(err)
        if bad is not None:
            exc_cls = STATUS_TO_ERROR.get(bad[1], SimulationError)
            raise err if (err is not None and int(st.first_flagged_id) == bad[0]) else \
                exc_cls(f"error set {bad[0]}: flagged on another rank")
        if batch is not None and n_rec:
            dk, dc = batch.histogram_dev()
            keys = torch.as_tensor(dk, device=f"cuda:{device}").view(torch.int64)
            counts = torch.as_tensor(dc, device=f"cuda:{device}").view(torch.int64)
            if where == "cpu":
                keys, counts = keys.cpu(), counts.cpu()
        else:
            keys = torch.zeros((0, words), dtype=torch.int64, device=where)
            counts = torch.zeros(0, dtype=torch.int64, device=where)
        k, cnt = gather_histograms(keys, counts, group=group, merge=_merge_for(where, device))
        loop_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        records = [engine.ShotRecord(bitstring=s, count=int(v)) for s, v in
                   zip(engine.unpack_keys(k.cpu().numpy().view(np.uint64), plan.n), cnt.cpu().tolist())]
        aggregate_s = time.perf_counter() - t0
        # counters: sum over ranks; device time: max over ranks
        ev = [int(st.stage_events[j]) if st is not None else 0 for j in range(f)]
        vec = torch.tensor([sum(ev)] + ev, dtype=torch.int64, device=where)
        dist.all_reduce(vec, group=group)
        tmax = torch.tensor([st.loop_ms * 1e-3 if st is not None else 0.0], dtype=torch.float64, device=where)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX, group=group)
    finally:
        if batch is not None:
            batch.close()
        pipe.close()
    if st is not None:
        engine._account(ctx.stats, st, f)
    return engine.RunResult(
        mode=config.mode, records=records, unique_shots=len(records),
        total_count=sum(r.count for r in records),
        timings={"generate_s": 0.0, "plan_s": plan_s, "loop_s": loop_s, "aggregate_s": aggregate_s,
                 "path_s": ctx.stats.path_seconds, "contract_s": ctx.stats.contract_seconds,
                 "device_loop_s": float(tmax.item()),
                 "h2d_s": (st.h2d_ms * 1e-3) if st is not None else 0.0, "d2h_s": 0.0,
                 "gpu_launches": int(st.gpu_launches) if st is not None else 0},
        plan_events=ctx.stats.plan_events, contract_events=int(vec[0].item()),
        stage_events={j: int(vec[j].item()) for j in range(1, f + 1)},
        stage_seconds=dict(sorted(ctx.stats.stage_seconds.items())),
        config=config.to_dict(), seed=config.seed, shot_allocations=[int(k.m) for k in errorsets])
