"""Path planner front end and the signature-keyed path cache.

Public surface of the reference planner (planner.py:34-442): `ContractionPath`
(JSON wire-compatible), `path_cost`, `find_path_greedy`, `find_path_optimal`,
`PathCache` (same JSON persistence format, planner.py:372-413) and
`cache_lookup_or_plan`.  The search itself runs in native code
(`csrc/planner.cpp`, entry point `ptsbe_plan_greedy`); it is seeded
deterministically from the caller's `rng` but does not reproduce the
reference's descent order -- paths are interchangeable (same step convention,
validated by structural replay), not identical.

Batch-aware extension: `op_class` / `class_weight` make the search minimise
sum(step flops x number of distinct instances of the step's result in the
batch) instead of plain flops, which is what the hoisting executor pays.
"""

from __future__ import annotations

import json
import math
import threading
from dataclasses import dataclass
from typing import Hashable, Optional, Sequence

import numpy as np

from .errors import CapacityError, NetworkStructureError, PathCacheError
from .tensor import NetworkSignature, TensorNetwork, network_signature, replay_shapes


@dataclass(frozen=True)
class ContractionPath:
    """Slot-pair schedule: step (i, j), i < j, contracts slots i and j into
    slot i and deletes slot j (planner.py:34-54)."""

    steps: tuple
    est_cost: float

    def to_json(self) -> str:
        return json.dumps({"steps": [list(s) for s in self.steps], "est_cost": self.est_cost})

    @classmethod
    def from_json(cls, text: str) -> "ContractionPath":
        doc = json.loads(text)
        return cls(tuple((int(i), int(j)) for i, j in doc["steps"]), float(doc["est_cost"]))


def path_cost(net: TensorNetwork, path) -> float:
    """Sum over steps of prod(dims of the union of both operands' labels)
    (planner.py:61-103)."""
    from .errors import IncompletePathError

    steps = getattr(path, "steps", path)
    cost, _, slots = replay_shapes(net, steps)
    if len(slots) != 1:
        raise IncompletePathError(f"path left {len(slots)} operands, expected 1")
    if set(slots[0]) != set(net.open_indices):
        raise NetworkStructureError("replayed path does not produce the open indices")
    return cost


def merges_to_steps(n: int, merges) -> tuple:
    """Stable-id merges (result keeps the smaller id) -> slot steps under the
    replace-lower / shift-down convention (planner.py:106-118).  Uses a Fenwick
    tree so 1000-operand paths convert in O(n log n)."""
    tree = [0] * (n + 1)

    def add(i, v):
        i += 1
        while i <= n:
            tree[i] += v
            i += i & -i

    def before(i):  # number of alive ids < i
        s = 0
        while i > 0:
            s += tree[i]
            i -= i & -i
        return s

    for k in range(n):
        add(k, 1)
    out = []
    for x, y in merges:
        x, y = int(x), int(y)
        if x > y:
            x, y = y, x
        out.append((before(x), before(y)))
        add(y, -1)
    return tuple(out)


def find_path_greedy(
    net: TensorNetwork,
    hypersamples: int = 100,
    rng: Optional[np.random.Generator] = None,
    *,
    op_class: Optional[Sequence[int]] = None,
    class_weight: Optional[Sequence[float]] = None,
    size_cap_log2: float = 0.0,
    class_cap_log2: Optional[Sequence[float]] = None,
) -> ContractionPath:
    """Best of `hypersamples` randomized greedy descents (planner.py:212-251).
    `est_cost` is the reference flop estimate of the chosen path."""
    from . import _capi

    if hypersamples < 1:
        raise ValueError("hypersamples must be >= 1")
    n = len(net.operands)
    if n == 0:
        raise NetworkStructureError("network has no operands")
    if n == 1:
        return ContractionPath(steps=(), est_cost=0.0)
    if rng is None:
        rng = np.random.default_rng()
    seed = int(rng.integers(0, 2**63 - 1))
    merges, _, flops = _capi.plan_greedy(
        [t.labels for t in net.operands],
        [[ix.dim for ix in t.indices] for t in net.operands],
        op_class=op_class,
        class_weight=class_weight,
        hypersamples=hypersamples,
        seed=seed,
        size_cap_log2=size_cap_log2,
        class_cap_log2=class_cap_log2,
    )
    return ContractionPath(steps=merges_to_steps(n, merges), est_cost=float(flops))


def _min_cut_source_side(n: int, edges, sources, sinks) -> tuple:
    """Dinic max-flow on an undirected capacity graph; returns (cut value, set
    of nodes on the source side of the min cut closest to the sources)."""
    from collections import deque

    src, dst = n, n + 1
    graph = [[] for _ in range(n + 2)]

    def add(u, v, c_uv, c_vu):
        graph[u].append([v, c_uv, len(graph[v])])
        graph[v].append([u, c_vu, len(graph[u]) - 1])

    inf = 1 << 40
    for u, v, c in edges:
        add(u, v, c, c)
    for x in sources:
        add(src, x, inf, 0)
    for x in sinks:
        add(x, dst, inf, 0)
    flow = 0
    while True:
        level = [-1] * (n + 2)
        level[src] = 0
        dq = deque([src])
        while dq:
            u = dq.popleft()
            for v, c, _ in graph[u]:
                if c > 0 and level[v] < 0:
                    level[v] = level[u] + 1
                    dq.append(v)
        if level[dst] < 0:
            break
        it = [0] * (n + 2)
        while True:  # iterative DFS for one augmenting path in the level graph
            stack, found = [src], False
            while stack:
                u = stack[-1]
                if u == dst:
                    found = True
                    break
                adv = False
                while it[u] < len(graph[u]):
                    v, c, _ = graph[u][it[u]]
                    if c > 0 and level[v] == level[u] + 1:
                        stack.append(v)
                        adv = True
                        break
                    it[u] += 1
                if not adv:
                    stack.pop()
                    if stack:
                        it[stack[-1]] += 1
            if not found:
                break
            push = inf
            for u in stack[:-1]:
                push = min(push, graph[u][it[u]][1])
            for u in stack[:-1]:
                e = graph[u][it[u]]
                e[1] -= push
                graph[e[0]][e[2]][1] += push
            flow += push
            if flow >= inf:
                return flow, set()
    seen = {src}
    dq = deque([src])
    while dq:
        u = dq.popleft()
        for v, c, _ in graph[u]:
            if c > 0 and v not in seen:
                seen.add(v)
                dq.append(v)
    return flow, {u for u in seen if u < n}


def plan_stage(op_labels, op_dims, op_class, op_is_prefix, open_labels, class_weight,
               item_cap_log2: float, record_cap_log2: float, hypersamples: int = 100,
               rng: Optional[np.random.Generator] = None,
               op_mirror: Optional[Sequence[int]] = None) -> ContractionPath:
    """Path for one stage network of the batched executor (north-star
    subsystem 1: found once on the template, stored, replayed for every error
    set and prefix).  Two candidates, the cheaper batch-weighted cost wins:

    generic   class-weighted randomized greedy over the whole network
              (csrc/planner.cpp);
    cut       the operands are split by a minimum cut between the prefix
              projectors (everything that varies per work item) and the open
              batch legs.  The far side holds no projector, so it contracts
              ONCE PER ERROR SET into a record M[cut legs, open legs]; the near
              side contracts per work item into a vector v[cut legs]; the root
              step P = v . M is a dense matrix product over all items of an
              error set, which the executor runs as a GEMM (csrc/project.cuh).

    With `op_mirror` (ket <-> bra twin of every operand) the near side is
    searched on its ket half only when the two halves are disconnected: the
    bra half is contracted in the mirrored order, which lets the compiler
    recognise every bra subtree as the conjugate of a ket subtree and skip it.

    Returns the path in the reference's slot-step convention (planner.py:34-54)
    over the given operand order; est_cost is the plain flop estimate."""
    from . import _capi

    n = len(op_labels)
    if n == 1:
        return ContractionPath(steps=(), est_cost=0.0)
    if rng is None:
        rng = np.random.default_rng()
    seed = int(rng.integers(0, 2**63 - 1))
    n_cls = len(class_weight)
    caps = [record_cap_log2] * (n_cls - 1) + [item_cap_log2]
    if n_cls == 1:
        caps = [record_cap_log2]
    unit = [1 if u else 0 for u in op_is_prefix]
    merges, wcost, flops = _capi.plan_greedy(op_labels, op_dims, op_class=op_class, class_weight=class_weight,
                                             hypersamples=hypersamples, seed=seed, class_cap_log2=caps,
                                             op_unit=unit)
    best = (wcost, merges, flops)
    sources = [k for k in range(n) if op_is_prefix[k]]
    opens = set(open_labels)
    sinks = [k for k in range(n) if any(lb in opens for lb in op_labels[k])]
    if sources and sinks and n_cls > 1:
        owner: dict = {}
        for k in range(n):
            for lb, d in zip(op_labels[k], op_dims[k]):
                owner.setdefault(lb, []).append((k, d))
        # capacities in units of 1/64 bit so non-power-of-two bonds keep their order
        edges = [(v[0][0], v[1][0], max(1, int(round(64 * math.log2(v[0][1])))))
                 for v in owner.values() if len(v) == 2 and v[0][1] > 1]
        cut, near = _min_cut_source_side(n, edges, sources, sinks)
        log2_n = sum(math.log2(d) for k in range(n) for lb, d in zip(op_labels[k], op_dims[k]) if lb in opens)
        far = [k for k in range(n) if k not in near]
        if near and far and cut / 64.0 + log2_n <= record_cap_log2 and cut / 64.0 <= item_cap_log2:
            gv = sorted(near)

            def sub(ids, cw, cc, hs=hypersamples):
                if len(ids) == 1:
                    return [], 0.0, 0.0
                m, wc, fl = _capi.plan_greedy([op_labels[k] for k in ids], [op_dims[k] for k in ids],
                                              op_class=[op_class[k] for k in ids], class_weight=cw,
                                              hypersamples=hs, seed=seed + 1, class_cap_log2=cc,
                                              op_unit=[unit[k] for k in ids])
                return [(ids[int(a)], ids[int(b)]) for a, b in m], wc, fl

            # ket / bra halves of the near side: disconnected and mirror images of each other?
            half = None
            if op_mirror is not None and all(op_mirror[k] >= 0 and op_mirror[k] in near for k in gv):
                ket = [k for k in gv if k < op_mirror[k]]
                ket_set = set(ket)
                ket_labels = {lb for k in ket for lb in op_labels[k]}
                bra_labels = {lb for k in gv if k not in ket_set for lb in op_labels[k]}
                order_ok = all(op_mirror[a] < op_mirror[b] for a, b in zip(ket, ket[1:]))
                if len(ket) * 2 == len(gv) and not (ket_labels & bra_labels) and order_ok:
                    half = ket
            search = half if half is not None else gv
            # near side: the hoisted classes are searched under several record caps.  Hoisted
            # merges are nearly free in the batch-weighted cost, so an uncapped greedy keeps
            # merging them into blobs that the per-item steps then have to slice; a small cap
            # stops at "site tensor" size.  Every candidate is judged by the same weighted cost.
            mv, wv, fv = None, math.inf, 0.0
            for rec_cap in (4.0, 5.0, 6.0, 7.0, 8.0, 10.0, 13.0, record_cap_log2):
                cc = [min(rec_cap, record_cap_log2)] * (n_cls - 1) + [item_cap_log2]
                # the near side is small (a few hundred operands) and decides the per-item cost:
                # it gets many more descents than the rest
                m_, w_, f_ = sub(search, class_weight, cc, hs=NEAR_SIDE_DESCENTS * hypersamples)
                if w_ < wv:
                    mv, wv, fv = m_, w_, f_
            if half is not None:
                # mirrored merges for the bra half (its subtrees are conjugate twins: free), then
                # the outer product of the two halves
                mv = list(mv) + [(op_mirror[a], op_mirror[b]) for a, b in mv] + \
                    [(min(half[0], op_mirror[half[0]]), max(half[0], op_mirror[half[0]]))]
                wv += (2.0 ** (cut / 64.0) + kStepOverheadMacs) * class_weight[-1]
                fv = 2 * fv + 2.0 ** (cut / 64.0)
            mm, wm, fm = sub(far, class_weight, [record_cap_log2] * n_cls)
            root = 2.0 ** (cut / 64.0 + log2_n)
            total = wv + wm + root * class_weight[-1]
            if total < best[0]:
                joined = list(mv) + list(mm) + [(min(gv[0], far[0]), max(gv[0], far[0]))]
                best = (total, np.asarray(joined, dtype=np.int64).reshape(-1, 2), fv + fm + root)
    return ContractionPath(steps=merges_to_steps(n, best[1]), est_cost=float(best[2]))


MAX_OPTIMAL_OPERANDS = 14
kStepOverheadMacs = 400.0  # same constant as csrc/planner.cpp
NEAR_SIDE_DESCENTS = 8    # multiplier on hypersamples for the near-side search


def find_path_optimal(net: TensorNetwork) -> ContractionPath:
    """Minimum-flop path by DP over operand subsets, <= 14 operands
    (planner.py:257-340).  Verification oracle only; host code."""
    n = len(net.operands)
    if n == 0:
        raise NetworkStructureError("network has no operands")
    if n > MAX_OPTIMAL_OPERANDS:
        raise CapacityError(f"optimal planner capped at {MAX_OPTIMAL_OPERANDS} operands, got {n}")
    if n == 1:
        return ContractionPath(steps=(), est_cost=0.0)
    # label -> (dim, occupancy mask)
    occ: dict[int, int] = {}
    dim: dict[int, int] = {}
    for k, t in enumerate(net.operands):
        for ix in t.indices:
            occ[ix.label] = occ.get(ix.label, 0) | (1 << k)
            dim[ix.label] = ix.dim
    labels = list(occ)
    full = (1 << n) - 1

    def union_size(m1: int, m2: int) -> float:
        s = 1.0
        for lb in labels:
            i1, i2 = occ[lb] & m1, occ[lb] & m2
            if (i1 and i1 & (i1 - 1) == 0) or (i2 and i2 & (i2 - 1) == 0):
                s *= dim[lb]
        return s

    best = {1 << k: (0.0, None) for k in range(n)}
    by_pop = sorted(range(1, full + 1), key=lambda m: bin(m).count("1"))
    for mask in by_pop:
        if mask & (mask - 1) == 0:
            continue
        low = mask & -mask
        top_cost, top_split = math.inf, None
        sub = (mask - 1) & mask
        while sub:
            if sub & low:
                rest = mask ^ sub
                c = best[sub][0] + best[rest][0] + union_size(sub, rest)
                if c < top_cost:
                    top_cost, top_split = c, (sub, rest)
            sub = (sub - 1) & mask
        best[mask] = (top_cost, top_split)
    merges = []

    def emit(mask: int) -> int:
        if mask & (mask - 1) == 0:
            return mask.bit_length() - 1
        s1, s2 = best[mask][1]
        a, b = emit(s1), emit(s2)
        merges.append((min(a, b), max(a, b)))
        return min(a, b)

    emit(full)
    return ContractionPath(steps=merges_to_steps(n, merges), est_cost=best[full][0])


class PathCache:
    """(NetworkSignature, stage descriptor) -> ContractionPath.  Readers are
    lock-free, writers take a lock, planning the same key twice is idempotent
    (planner.py:343-413).  The JSON format is the reference's, so a cache file
    written by either package warms the other."""

    def __init__(self):
        self._store: dict = {}
        self._lock = threading.Lock()
        self.hits = 0
        self.misses = 0

    def __len__(self):
        return len(self._store)

    def get(self, sig: NetworkSignature, stage: Hashable):
        return self._store.get((sig, stage))

    def put(self, sig: NetworkSignature, stage: Hashable, path: ContractionPath) -> None:
        with self._lock:
            self._store[(sig, stage)] = path

    def clear(self) -> None:
        with self._lock:
            self._store.clear()
            self.hits = self.misses = 0

    def save(self, fp) -> None:
        rows = []
        for (sig, stage), path in self._store.items():
            rows.append(
                {
                    "signature": {
                        "num_operands": sig.num_operands,
                        "shapes": [list(s) for s in sig.shapes],
                        "bonds": [[list(p) for p in b] for b in sig.bonds],
                        "open_legs": [list(o) for o in sig.open_legs],
                    },
                    "stage": stage,
                    "steps": [list(s) for s in path.steps],
                    "est_cost": path.est_cost,
                }
            )
        json.dump({"entries": rows}, fp)

    @classmethod
    def load(cls, fp) -> "PathCache":
        cache = cls()
        for row in json.load(fp)["entries"]:
            s = row["signature"]
            sig = NetworkSignature(
                num_operands=int(s["num_operands"]),
                shapes=tuple(tuple(int(d) for d in shape) for shape in s["shapes"]),
                bonds=tuple(tuple(tuple(int(v) for v in p) for p in b) for b in s["bonds"]),
                open_legs=tuple(tuple(int(v) for v in o) for o in s["open_legs"]),
            )
            stage = row["stage"]
            if isinstance(stage, list):
                stage = tuple(stage)
            cache.put(
                sig,
                stage,
                ContractionPath(tuple((int(i), int(j)) for i, j in row["steps"]), float(row["est_cost"])),
            )
        return cache


def cache_lookup_or_plan(
    cache: PathCache,
    net: TensorNetwork,
    stage: Hashable,
    hypersamples: int = 100,
    rng: Optional[np.random.Generator] = None,
    **plan_kw,
) -> tuple:
    """(path, hit).  A hit is validated by structural replay; a stored path
    that does not replay means the cache is corrupt (planner.py:416-442)."""
    sig = network_signature(net)
    path = cache.get(sig, stage)
    if path is not None:
        try:
            path_cost(net, path)
        except NetworkStructureError as exc:
            raise PathCacheError(f"cached path for stage {stage!r} does not replay: {exc}") from exc
        cache.hits += 1
        return path, True
    path = find_path_greedy(net, hypersamples=hypersamples, rng=rng, **plan_kw)
    cache.put(sig, stage, path)
    cache.misses += 1
    return path, False
