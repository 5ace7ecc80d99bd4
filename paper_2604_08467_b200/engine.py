"""Trajectory engine of the drop-in host API, running on the B200 path.

Same public names, argument meaning and error behaviour as the reference
engine for the proportional PTSBE path
(/root/reference/pkg/src/ptsbe/engine.py:57-524, 664-929); the arithmetic is
done by libptsbe_b200.so:

  merge_errors (UPV, engine.py:284-313)      -> per-site variant tables, gathered on device
  marginal_network (engine.py:361-407)       -> static operand table built once per stage
  _contract_marginal (engine.py:417-450)     -> exec_kernel + fused epilogue
  sample_proportional (engine.py:493-524)    -> sample_kernel + order-preserving compaction
  merge_records (engine.py:815-829)          -> device sort + reduce-by-key
  run_ptsbe fan-out (engine.py:885-906)      -> one batched run over all error sets

New, batch-granular entry points:
`conditional_marginals_batched` and `sample_proportional_batched`.

Out of scope (SURVEY.md sections 2 and 8f): the non-proportional sampler and the
deliberately slow comparison modes.  Their names are exported for import
compatibility and raise NotImplementedError when called.
"""

from __future__ import annotations

import json
import os
import math
import time
from dataclasses import dataclass, field
from typing import NamedTuple, Optional, Sequence

import numpy as np

from . import compiler
from .circuits import (
    PAULI_KINDS,
    TWO_QUBIT_PAULIS,
    Circuit,
    build_network,
    final_qubit_labels,
    gate_matrix,
    is_identity_label,
    pauli_matrix,
)
from .compiler import SEL_CONST, SEL_KRAUS, SEL_PREFIX, CompiledPlan, Operand, Pool
from .errors import (
    STATUS_TO_ERROR,
    ImpossiblePrefixError,
    NetworkStructureError,
    NumericalError,
    ResourceLimitError,
    SimulationError,
)
from .planner import PathCache, cache_lookup_or_plan, plan_stage
from .tensor import DEFAULT_INTERMEDIATE_CEILING, Index, NetworkSignature, Tensor, TensorNetwork

NEGATIVE_DIAG_TOLERANCE = -1e-12
VANISHING_MASS = 1e-12

_BASIS = np.eye(2, dtype=np.complex128)
_COPY3 = np.zeros((2, 2, 2), dtype=np.complex128)
_COPY3[0, 0, 0] = _COPY3[1, 1, 1] = 1.0

_KEY_PRESAMPLE, _KEY_SAMPLER, _KEY_BASELINE, _KEY_PLANNER = 0, 1, 2, 3


def spawn_rng(seed: int, *key: int) -> np.random.Generator:
    """Independent generator per key path (engine.py:57-59)."""
    return np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=key))


@dataclass(frozen=True)
class ErrorSet:
    """One pre-sampled realization: operator label per gate site plus its shot
    allocation (engine.py:62-73)."""

    id: int
    realized: tuple
    m: int

    def __post_init__(self):
        if self.m < 0:
            raise ValueError("shot allocation must be non-negative")


@dataclass(frozen=True)
class BatchPlan:
    """Ordered qubit batches for staged sampling (engine.py:76-142).  The
    non-proportional knobs are carried for API compatibility only."""

    sizes: tuple
    nonfinal_shots: int = 1
    final_mode: str = "exhaustive"
    direct_count: int = 1
    threshold: float = 1e-6

    def __post_init__(self):
        object.__setattr__(self, "sizes", tuple(int(b) for b in self.sizes))
        if not self.sizes or min(self.sizes) < 1:
            raise ValueError(f"batch sizes must be positive, got {self.sizes}")
        if self.final_mode not in ("direct", "exhaustive"):
            raise ValueError(f"unknown final mode {self.final_mode!r}")
        if self.direct_count < 1:
            raise ValueError("direct count must be >= 1")
        if self.threshold <= 0.0:
            raise ValueError("exhaustive threshold must be positive")
        if self.nonfinal_shots < 1:
            raise ValueError("nonfinal_shots must be >= 1")

    @property
    def f(self) -> int:
        return len(self.sizes)

    @property
    def n(self) -> int:
        return sum(self.sizes)

    def offset(self, j: int) -> int:
        return sum(self.sizes[: j - 1])

    def stage_qubits(self, j: int) -> range:
        lo = self.offset(j)
        return range(lo, lo + self.sizes[j - 1])

    def stage_of_qubit(self, q: int) -> int:
        acc = 0
        for j, b in enumerate(self.sizes, start=1):
            acc += b
            if q < acc:
                return j
        raise ValueError(f"qubit {q} outside the plan")

    @classmethod
    def fixed(cls, n: int, b: int, **kw) -> "BatchPlan":
        if b < 1:
            raise ValueError("batch size must be >= 1")
        f = max(1, math.ceil(n / b))
        return cls(sizes=tuple([b] * (f - 1) + [n - b * (f - 1)]), **kw)

    @classmethod
    def with_final(cls, n: int, nonfinal: int = 10, final: int = 28, **kw) -> "BatchPlan":
        last = min(final, n)
        k, r = divmod(n - last, nonfinal)
        return cls(sizes=tuple([nonfinal] * k + ([r] if r else []) + [last]), **kw)


@dataclass
class ShotRecord:
    bitstring: str
    count: int
    prob: Optional[float] = None


@dataclass
class EngineStats:
    """Plan/contraction counters and times per stage (engine.py:155-181).
    On this path `contract_seconds` / `stage_seconds` are device times."""

    plan_events: int = 0
    contract_events: int = 0
    path_seconds: float = 0.0
    contract_seconds: float = 0.0
    stage_events: dict = field(default_factory=dict)
    stage_seconds: dict = field(default_factory=dict)
    # device-only: work items of a stage sampled by per-qubit descent (csrc/descent.cuh)
    descent_events: dict = field(default_factory=dict)

    def record_contraction(self, stage: int, seconds: float, events: int = 1) -> None:
        self.contract_events += events
        self.contract_seconds += seconds
        self.stage_events[stage] = self.stage_events.get(stage, 0) + events
        self.stage_seconds[stage] = self.stage_seconds.get(stage, 0.0) + seconds

    def merge(self, other: "EngineStats") -> None:
        self.plan_events += other.plan_events
        self.contract_events += other.contract_events
        self.path_seconds += other.path_seconds
        self.contract_seconds += other.contract_seconds
        for k, v in other.stage_events.items():
            self.stage_events[k] = self.stage_events.get(k, 0) + v
        for k, v in other.stage_seconds.items():
            self.stage_seconds[k] = self.stage_seconds.get(k, 0.0) + v
        for k, v in other.descent_events.items():
            self.descent_events[k] = self.descent_events.get(k, 0) + v


@dataclass
class SamplerContext:
    """Cache, counters, planner settings and guards of one run
    (engine.py:184-209) plus the device knobs."""

    cache: PathCache = field(default_factory=PathCache)
    stats: EngineStats = field(default_factory=EngineStats)
    hypersamples: int = 100
    planner_seed: int = 0
    max_intermediate: int = DEFAULT_INTERMEDIATE_CEILING
    deadline: Optional[float] = None
    dtype: str = "complex128"
    device: int = 0

    def check_deadline(self) -> None:
        if self.deadline is not None and time.perf_counter() > self.deadline:
            raise ResourceLimitError("wall-clock deadline exceeded")

    def fork(self) -> "SamplerContext":
        return SamplerContext(
            cache=self.cache, stats=EngineStats(), hypersamples=self.hypersamples,
            planner_seed=self.planner_seed, max_intermediate=self.max_intermediate,
            deadline=self.deadline, dtype=self.dtype, device=self.device,
        )


@dataclass(frozen=True)
class CircuitNetwork:
    """Uncontracted network + per-qubit final labels (engine.py:212-229).
    `channels` (one NoiseChannel or None per gate site) lets non-Pauli
    operator labels such as "K1" be resolved; Pauli labels need nothing."""

    net: TensorNetwork
    final_labels: tuple
    channels: Optional[tuple] = None

    @classmethod
    def from_circuit(cls, c: Circuit) -> "CircuitNetwork":
        return cls(net=build_network(c), final_labels=final_qubit_labels(c),
                   channels=tuple(g.noise for g in c.gates))

    @property
    def n(self) -> int:
        return len(self.final_labels)

    def operator(self, site: int, label: str) -> np.ndarray:
        if self.channels is not None and self.channels[site] is not None:
            return self.channels[site].operator(label)
        return pauli_matrix(label)

    def merged(self, k: ErrorSet) -> "CircuitNetwork":
        return CircuitNetwork(net=merge_errors(self.net, k, self), final_labels=self.final_labels)


def draw_realization(c: Circuit, rng: np.random.Generator) -> tuple:
    """One realized label per gate site.  The rng call order for the
    reference's channel kinds is the reference's (engine.py:232-244), so a
    seed produces the same realization in both packages."""
    out = []
    for g in c.gates:
        ch = g.noise
        if rng.random() < ch.p:
            if ch.kind == "depolarizing":
                out.append(TWO_QUBIT_PAULIS[int(rng.integers(15))])
            elif ch.kind == "depolarizing1":
                out.append(PAULI_KINDS[int(rng.integers(3))])
            elif ch.kind == "amplitude_damping":
                out.append("K1")
            else:
                out.append(ch.kind)
        else:
            out.append(ch.identity_label())
    return tuple(out)


def _allocate(e: int, rule: str, total_shots: int, shots_per_set) -> list:
    if e < 1:
        raise ValueError("need at least one error set")
    if rule == "proportional":
        if total_shots < e:
            raise ValueError("proportional rule needs total_shots >= number of sets")
        base, rem = divmod(total_shots, e)
        return [base + 1 if i < rem else base for i in range(e)]
    if rule == "uniform":
        if shots_per_set is None:
            raise ValueError("uniform rule needs shots_per_set")
        if isinstance(shots_per_set, (int, np.integer)):
            return [int(shots_per_set)] * e
        alloc = [int(v) for v in shots_per_set]
        if len(alloc) != e:
            raise ValueError("shots_per_set length must equal number of sets")
        return alloc
    raise ValueError(f"unknown allocation rule {rule!r}")


def presample_errors(c: Circuit, e: int, rule: str = "proportional", total_shots: int = 0,
                     rng: Optional[np.random.Generator] = None, shots_per_set=None) -> list:
    """Draw `e` realizations and allot shots (engine.py:247-281)."""
    alloc = _allocate(e, rule, total_shots, shots_per_set)
    if rng is None:
        rng = np.random.default_rng()
    return [ErrorSet(id=i, realized=draw_realization(c, rng), m=alloc[i]) for i in range(e)]


def merge_errors(template: TensorNetwork, k: ErrorSet, owner: Optional[CircuitNetwork] = None) -> TensorNetwork:
    """UPV on the host carriers: error operator left-multiplied into its gate
    tensor, structure untouched (engine.py:284-313).  The device path never
    calls this per error set -- it gathers from variant tables -- but the
    single-network API (`CircuitNetwork.merged`) keeps the reference meaning."""
    g = len(k.realized)
    n = len(template.operands) - g
    if n < 1:
        raise NetworkStructureError(
            f"realization has {g} sites but network has {len(template.operands)} operands"
        )
    ops = list(template.operands)
    for site, label in enumerate(k.realized):
        if is_identity_label(label):
            continue
        old = ops[n + site]
        op = owner.operator(site, label) if owner is not None else pauli_matrix(label)
        arity = int(round(math.log2(op.shape[0])))
        if old.data.ndim != 2 * arity:
            raise NetworkStructureError(
                f"site {site}: {arity}-qubit error on {old.data.ndim // 2}-qubit gate"
            )
        side = 1 << arity
        ops[n + site] = Tensor(old.indices, (op @ old.data.reshape(side, side)).reshape(old.data.shape))
    return TensorNetwork(ops, template.open_indices)


class MarginalNetwork(NamedTuple):
    net: TensorNetwork
    open_labels: tuple


def _stage_layout(cnet: CircuitNetwork, plan: BatchPlan, j: int):
    """Label bookkeeping of the stage-j sandwich (engine.py:373-406): returns
    (bra label map, list of (qubit, ket leg, bra leg) for prefix qubits, list of
    (qubit, ket leg, bra leg, open leg) for batch qubits)."""
    n = cnet.n
    if not 1 <= j <= plan.f:
        raise ValueError(f"stage {j} outside 1..{plan.f}")
    offset = plan.offset(j)
    batch = plan.stage_qubits(j)
    fresh = 1 + max((ix.label for t in cnet.net.operands for ix in t.indices), default=0)
    bra = {}
    for t in cnet.net.operands:
        for ix in t.indices:
            if ix.label not in bra:
                bra[ix.label] = fresh
                fresh += 1
    for q in range(batch.stop, n):  # traced qubits: bra leg joins the ket leg
        bra[cnet.final_labels[q]] = cnet.final_labels[q]
    fixed = [(q, cnet.final_labels[q], bra[cnet.final_labels[q]]) for q in range(offset)]
    opened = []
    for q in batch:
        opened.append((q, cnet.final_labels[q], bra[cnet.final_labels[q]], fresh))
        fresh += 1
    return bra, fixed, opened


def marginal_network(cnet: CircuitNetwork, plan: BatchPlan, j: int, prefix: str) -> MarginalNetwork:
    """Host carrier of the stage-j sandwich for one prefix, operand order as in
    the reference (engine.py:361-407) so signatures -- and therefore cached
    paths -- are interchangeable between the two packages."""
    bra, fixed, opened = _stage_layout(cnet, plan, j)
    if len(prefix) != len(fixed):
        raise ValueError(f"stage {j} expects a {len(fixed)}-bit prefix, got {len(prefix)}")
    ops = list(cnet.net.operands)
    ops.extend(t.conj().relabeled(bra) for t in cnet.net.operands)
    for q, ket_leg, bra_leg in fixed:
        vec = _BASIS[1] if prefix[q] == "1" else _BASIS[0]
        ops.append(Tensor([Index(ket_leg, 2)], vec))
        ops.append(Tensor([Index(bra_leg, 2)], vec))
    for _, ket_leg, bra_leg, open_leg in opened:
        ops.append(Tensor([Index(ket_leg, 2), Index(bra_leg, 2), Index(open_leg, 2)], _COPY3))
    opens = tuple(o[3] for o in opened)
    return MarginalNetwork(net=TensorNetwork(ops, opens), open_labels=opens)


# ---------------------------------------------------------------------------
# device pipeline
# ---------------------------------------------------------------------------

class VariantTables:
    """Per gate site: the distinct realized labels of a batch of error sets and
    the merged tensors `operator @ gate` (UPV, engine.py:300-312).  Error sets
    become rows of a uint8 index matrix."""

    def __init__(self, cnet: CircuitNetwork, n_sites: int, labels_per_site: Sequence[Sequence[str]]):
        self.n_sites = n_sites
        self.labels = [list(lbs) for lbs in labels_per_site]
        self.index = [{lb: k for k, lb in enumerate(lbs)} for lbs in self.labels]
        n_kets = len(cnet.net.operands) - n_sites
        self.data = []
        for site, lbs in enumerate(self.labels):
            base = cnet.net.operands[n_kets + site]
            side = int(round(math.sqrt(base.data.size)))
            rows = []
            for lb in lbs:
                if is_identity_label(lb):
                    rows.append(base.data.reshape(-1))
                    continue
                op = cnet.operator(site, lb)
                if op.shape[0] != side:
                    arity = int(round(math.log2(op.shape[0])))
                    raise NetworkStructureError(
                        f"site {site}: {arity}-qubit error on {base.data.ndim // 2}-qubit gate"
                    )
                rows.append((op @ base.data.reshape(side, side)).reshape(-1))
            if len(rows) > 255:
                raise ValueError(f"site {site}: more than 255 distinct operators")
            self.data.append(np.asarray(rows, dtype=np.complex128))

    @classmethod
    def from_errorsets(cls, cnet: CircuitNetwork, errorsets: Sequence[ErrorSet]) -> "VariantTables":
        if not errorsets:
            raise ValueError("need at least one error set")
        g = len(errorsets[0].realized)
        if len(cnet.net.operands) - g < 1:
            raise NetworkStructureError(
                f"realization has {g} sites but network has {len(cnet.net.operands)} operands"
            )
        seen = [dict() for _ in range(g)]
        for k in errorsets:
            if len(k.realized) != g:
                raise NetworkStructureError("realization length does not match gate count")
            for site, lb in enumerate(k.realized):
                seen[site].setdefault(lb, None)
        return cls(cnet, g, [list(d) for d in seen])

    @classmethod
    def from_channels(cls, cnet: CircuitNetwork) -> "VariantTables":
        """Full tables from the circuit's channels (index = position in
        `NoiseChannel.outcomes()`)."""
        if cnet.channels is None:
            raise ValueError("network carries no channels")
        return cls(cnet, len(cnet.channels), [[lb for lb, _ in ch.outcomes()] for ch in cnet.channels])

    @classmethod
    def none(cls, cnet: CircuitNetwork) -> "VariantTables":
        return cls(cnet, 0, [])

    def encode(self, errorsets: Sequence[ErrorSet]) -> np.ndarray:
        out = np.zeros((len(errorsets), max(self.n_sites, 0)), dtype=np.uint8)
        for r, k in enumerate(errorsets):
            for site, lb in enumerate(k.realized):
                out[r, site] = self.index[site][lb]
        return out


def _schmidt_split(data: np.ndarray, tol: float = 1e-12):
    """Operator-Schmidt split of the variants of one two-qubit site.  `data` is
    [variants, 16] over legs (out_c, out_t, in_c, in_t).  Returns
    (A [variants, 4r] over (out_c, in_c, k), B [variants, 4r] over (k, out_t, in_t), r)
    with r the largest Schmidt rank over the variants, or None when r == 4
    (nothing to gain).  Controlled gates and RZZ have r = 2, and a Pauli (or
    any product) error folded in by UPV does not raise it."""
    nv = data.shape[0]
    parts, rank = [], 1
    for v in range(nv):
        m = data[v].reshape(2, 2, 2, 2).transpose(0, 2, 1, 3).reshape(4, 4)
        u, sv, vh = np.linalg.svd(m)
        r = int(np.sum(sv > tol * max(sv[0], 1e-300)))
        rank = max(rank, r)
        parts.append((u, sv, vh))
    if rank >= 4:
        return None
    a = np.zeros((nv, 4 * rank), dtype=np.complex128)
    b = np.zeros((nv, 4 * rank), dtype=np.complex128)
    for v, (u, sv, vh) in enumerate(parts):
        root = np.sqrt(sv[:rank])
        a[v] = (u[:, :rank] * root[None, :]).reshape(-1)        # (oc, ic, k)
        b[v] = (root[:, None] * vh[:rank, :]).reshape(-1)       # (k, ot, it)
    return a, b, rank


def _light_cone(cnet: CircuitNetwork, tables: "VariantTables", n_kets: int, first_traced: int):
    """Backward sweep over the gate sites.  Returns (dropped sites, {traced qubit: label at which
    its bra leg joins its ket leg}).  A qubit is active once something kept acts on it; measured and
    projected qubits (q < first_traced) are active from the end of the circuit."""
    ops = cnet.net.operands
    end = {q: lb for q, lb in enumerate(cnet.final_labels)}      # current end label of every wire
    owner = {lb: q for q, lb in end.items()}
    active = set(range(first_traced))
    joins = {}
    dropped = set()
    for site in reversed(range(tables.n_sites)):
        t = ops[n_kets + site]
        k = len(t.labels) // 2
        outs, ins = t.labels[:k], t.labels[k:]
        qs = [owner[lb] for lb in outs]
        side = 1 << k
        data = tables.data[site].reshape(-1, side, side)
        unitary = all(np.allclose(v.conj().T @ v, np.eye(side), atol=1e-12) for v in data)
        if unitary and not any(q in active for q in qs):
            dropped.add(site)
        else:
            for q, lb in zip(qs, outs):
                if q not in active:
                    active.add(q)
                    joins[q] = lb        # traced wire enters the light cone here
        for q, lo, li in zip(qs, outs, ins):
            del owner[lo]
            owner[li] = q
            end[q] = li
    for q in range(first_traced, cnet.n):
        if q not in active:
            joins[q] = end[q]            # nothing kept on this wire: <0|0> at the ket label
    return dropped, joins


def stage_operands(cnet: CircuitNetwork, plan: BatchPlan, j: int, tables: VariantTables,
                   split: bool = False, lightcone: bool = True):
    """Static operand table of the stage-j sandwich.  With split=False the
    operand order is that of `marginal_network` (reference engine.py:392-406).
    With split=True every two-qubit site whose variants all have operator-
    Schmidt rank < 4 becomes two rank-3 operands joined by a bond of that rank
    (both selected by the site's Kraus index): same values, but the network
    exposes the true entanglement cut of controlled gates, which is what the
    cut-based planner (planner.plan_stage) needs.  Returns (operands, open
    label order, mirror) where mirror[k] is the operand that is the conjugate
    (bra / ket) copy of operand k, -1 for the copy tensors."""
    bra, fixed, opened = _stage_layout(cnet, plan, j)
    n_kets = len(cnet.net.operands) - tables.n_sites
    dropped: set = set()
    if lightcone and tables.n_sites:
        # Unitary light cone: a site that acts only on traced qubits, after everything that reaches a
        # measured qubit, meets its own conjugate in the sandwich and (P U)^dagger (P U) = 1 for every
        # realised operator P of a unitary channel -- in every error set, so the structure stays
        # error-independent.  Both copies are dropped and the bra leg joins the ket leg at the
        # boundary of the light cone instead of at the end of the circuit.
        first_traced = plan.stage_qubits(j).stop
        dropped, joins = _light_cone(cnet, tables, n_kets, first_traced)
        nxt = 1 + max(list(bra.values()) + [o[3] for o in opened] + [lb for t in cnet.net.operands for lb in t.labels])
        for q in range(first_traced, cnet.n):  # undo the identification at the final labels ...
            bra[cnet.final_labels[q]] = nxt
            nxt += 1
        for lb in joins.values():              # ... and join where the wire enters the light cone
            bra[lb] = lb
    fresh = 1 + max([lb for t in cnet.net.operands for lb in t.labels] + list(bra.values())
                    + [o[3] for o in opened])
    halves = {}
    if split:
        for site in range(tables.n_sites):
            t = cnet.net.operands[n_kets + site]
            if len(t.labels) == 4 and site not in dropped:
                res = _schmidt_split(tables.data[site])
                if res is not None:
                    halves[site] = res + (fresh, fresh + 1)
                    fresh += 2
    ops = []
    for conj in (False, True):
        for slot, t in enumerate(cnet.net.operands):
            labels = tuple(bra.get(lb, lb) for lb in t.labels) if conj else t.labels
            dims = tuple(ix.dim for ix in t.indices)
            site = slot - n_kets
            if site in dropped:
                continue
            if site >= 0 and site in halves:
                a, b, r, k_ket, k_bra = halves[site]
                kind = SEL_KRAUS if a.shape[0] > 1 else SEL_CONST
                kl = k_bra if conj else k_ket
                oc, ot, ic, it = labels
                ops.append(Operand((oc, ic, kl), (2, 2, r), np.conj(a) if conj else a, kind, site, 0))
                ops.append(Operand((kl, ot, it), (r, 2, 2), np.conj(b) if conj else b, kind, site, 0))
                continue
            if site >= 0:
                data, kind, arg = tables.data[site], SEL_KRAUS, site
                if data.shape[0] == 1:
                    kind = SEL_CONST
            else:
                data, kind, arg = t.data.reshape(1, -1), SEL_CONST, 0
            ops.append(Operand(labels, dims, np.conj(data) if conj else data, kind, arg, 0))
    half = len(ops) // 2
    mirror = [k + half for k in range(half)] + [k for k in range(half)]
    for q, ket_leg, bra_leg in fixed:
        s = plan.stage_of_qubit(q)
        ops.append(Operand((ket_leg,), (2,), _BASIS, SEL_PREFIX, q, s))
        ops.append(Operand((bra_leg,), (2,), _BASIS, SEL_PREFIX, q, s))
        mirror += [len(ops) - 1, len(ops) - 2]
    for _, ket_leg, bra_leg, open_leg in opened:
        ops.append(Operand((ket_leg, bra_leg, open_leg), (2, 2, 2), _COPY3.reshape(1, -1)))
        mirror.append(-1)
    return ops, tuple(o[3] for o in opened), mirror


RECORD_CAP_LOG2 = 18.0  # entries of one hoisted record (per error set / per earlier-stage prefix)


def _ops_signature(ops, opens) -> NetworkSignature:
    """Value-independent fingerprint of a stage operand table, same fields as
    the reference's network signature (tensor.py:155-187), so stored paths go
    through the same PathCache and its JSON format."""
    where: dict = {}
    for slot, o in enumerate(ops):
        for axis, lb in enumerate(o.labels):
            where.setdefault(lb, []).append((slot, axis))
    bonds = sorted(tuple(sorted(p)) for p in where.values() if len(p) == 2)
    open_legs = sorted(p[0] for p in where.values() if len(p) == 1)
    return NetworkSignature(num_operands=len(ops), shapes=tuple(tuple(o.dims) for o in ops),
                            bonds=tuple(bonds), open_legs=tuple(open_legs))


def _size_cap_log2(dtype: str) -> float:
    return 13.0 if dtype == "complex64" else 12.0


def _fold_from(weights: Sequence[float]) -> Optional[int]:
    """First prefix-dependent class that is NOT worth a hoist pass of its own: a class with at
    least half as many distinct instances as the stage has work items (late stages of a spread-out
    distribution, where nearly every shot is its own prefix) saves no arithmetic by being hoisted
    and costs a launch plus a record round trip; compiler.compile_stage evaluates it with the
    per-item class instead.  PTSBE_FOLD: 0 (default) = never, 1 = only the class just below the
    per-item one, 2 = every qualifying class.  Off by default: with the kernels of this round the
    folded programs run slower than hoist pass + fused kernel (DESIGN.md section 7 has the A/B).  Decided from the plan-level weights only, so every
    rank and every chunk of a run compiles the same programs."""
    mode = int(os.environ.get("PTSBE_FOLD", "0"))
    top = len(weights) - 1
    if mode <= 0 or top < 2:
        return None
    c = top
    while c - 1 >= 1 and weights[c - 1] >= 0.5 * weights[top] and (mode >= 2 or c == top):
        c -= 1
    return c if c < top else None


class DevicePipeline:
    """Plans (once), compiles and owns the device plan of one
    (circuit structure, batch plan, variant tables) triple."""

    def __init__(self, cnet: CircuitNetwork, plan: BatchPlan, tables: VariantTables,
                 ctx: SamplerContext, stages: Optional[Sequence[int]] = None,
                 shots_per_set: float = 1.0, upload: bool = True, calibrate: bool = False):
        from . import _capi

        if plan.n != cnet.n:
            raise ValueError(f"plan covers {plan.n} qubits, circuit has {cnet.n}")
        self.cnet, self.plan, self.tables, self.ctx = cnet, plan, tables, ctx
        elem = 8 if ctx.dtype == "complex64" else 16
        pool = Pool()
        programs = []
        self.paths = {}
        self.stage_flops = {}
        want = set(range(1, plan.f + 1)) if stages is None else set(stages)
        for j in range(1, plan.f + 1):
            if j not in want:
                programs += [_empty_program(p + 1, 1 << plan.sizes[j - 1] if p == j - 1 else 0) for p in range(j)]
                continue
            ops, opens, mirror = stage_operands(cnet, plan, j, tables, split=True)
            # distinct instances of a class-k result: unique prefixes entering stage k+1
            weights = [float(min(shots_per_set, 2.0 ** min(plan.offset(k + 1), 60))) for k in range(j)]
            sig = _ops_signature(ops, opens)
            key = ("b200", j, round(math.log2(max(shots_per_set, 1.0))))
            t0 = time.perf_counter()
            path = ctx.cache.get(sig, key)
            if path is not None:
                ctx.cache.hits += 1
            else:
                path = plan_stage(
                    [o.labels for o in ops], [o.dims for o in ops], [o.cls for o in ops],
                    [o.sel_kind == SEL_PREFIX for o in ops], opens, weights, op_mirror=mirror,
                    item_cap_log2=_size_cap_log2(ctx.dtype), record_cap_log2=RECORD_CAP_LOG2,
                    hypersamples=ctx.hypersamples, rng=spawn_rng(ctx.planner_seed, _KEY_PLANNER, j))
                ctx.cache.put(sig, key, path)
                ctx.cache.misses += 1
                ctx.stats.plan_events += 1
                ctx.stats.path_seconds += time.perf_counter() - t0
            self.paths[j] = path
            progs, _ = compiler.compile_stage(ops, path.steps, opens, j, pool, elem,
                                              ceiling=ctx.max_intermediate, mirror=mirror,
                                              fold_from=_fold_from(weights),
                                              consumer_layout=int(os.environ.get("PTSBE_RECORD_LAYOUT", "2")))
            self.stage_flops[j] = [p.flops for p in progs]
            programs += progs
        self.compiled = CompiledPlan(
            dtype=ctx.dtype, n_qubits=plan.n, n_sites=tables.n_sites, sizes=plan.sizes,
            pool=pool.finish(ctx.dtype), programs=programs, max_intermediate=ctx.max_intermediate,
            site_variants=np.asarray([min(d.shape[0], 255) for d in tables.data], dtype=np.uint8),
        )
        # upload=False: compile only (plan inspection; CPU-side tests of the compiler)
        self.device_plan = _capi.DevicePlan(self.compiled, ctx.device) if upload else None
        self.stage_samplers = None
        if calibrate and self.device_plan is not None and stages is None:
            self.calibrate_samplers(shots_per_set)

    def calibrate_samplers(self, shots_per_set: float) -> None:
        """Pilot run that fixes the sampler of every stage for the life of the plan.  The device
        has two samplers for the categorical draws of engine.py:519 -- flat inverse CDF over the 2^b
        populations, per-qubit descent -- and the better one depends on the shots a work item
        carries.  Choosing per chunk from the chunk's own work list would make complex64 results
        depend on how error sets are grouped into calls, chunks and ranks; instead ONE error set
        (the error-free circuit, the job's mean shots, fixed seed, flat sampler) is run here and
        stage j gets the descent iff shots / unique prefixes entering it is at most DESCENT_MULT.
        Same circuit + plan + shots => same choice on every rank and in every call."""
        import os

        m = int(min(max(round(shots_per_set), 1), 1 << 17))
        f = self.plan.f
        dp = self.device_plan
        dp.set_stage_samplers(np.zeros(f, np.int32))
        _, _, _, st = dp.sample(np.zeros((1, self.tables.n_sites), np.uint8), np.asarray([m], np.uint32),
                                np.zeros(1, np.uint32), 0x5EED, merged=True)
        mult = float(os.environ.get("PTSBE_DESCENT_MULT") or 4.0)
        kinds = np.zeros(f, np.int32)
        for j in range(1, f):
            u = int(st.stage_events[j])
            kinds[j] = 1 if (u and m <= mult * u) else 0
        dp.set_stage_samplers(kinds)
        self.stage_samplers = kinds

    def close(self):
        if self.device_plan is not None:
            self.device_plan.close()

    def programs_of(self, j: int):
        base = j * (j - 1) // 2
        return self.compiled.programs[base: base + j]


def _empty_program(level: int, out_elems: int) -> compiler.Program:
    return compiler.Program(
        leaves=np.zeros((0, compiler.LEAF_WORDS), np.uint32), steps=np.zeros((0, compiler.STEP_WORDS), np.uint32),
        tables=np.zeros(0, np.uint32), arena_fast=0, arena_spill=0, out_elems=out_elems, threads=32, level=level,
    )


def pack_prefixes(prefixes: Sequence[str], n_qubits: int) -> np.ndarray:
    """Bitstrings -> [W, words] u64; qubit q sits at word q//64, bit 63-(q%64)."""
    words = max(1, (n_qubits + 63) // 64)
    out = np.zeros((len(prefixes), words), dtype=np.uint64)
    for r, s in enumerate(prefixes):
        for q, ch in enumerate(s):
            if ch == "1":
                out[r, q >> 6] |= np.uint64(1) << np.uint64(63 - (q & 63))
            elif ch != "0":
                raise ValueError(f"prefix {s!r} is not a bitstring")
    return out


def unpack_keys(keys: np.ndarray, n_qubits: int) -> list:
    """[R, words] u64 -> list of n-character bitstrings (qubit 0 leftmost)."""
    if keys.shape[0] == 0:
        return []
    be = np.ascontiguousarray(keys.astype(">u8"))
    bits = np.unpackbits(be.view(np.uint8).reshape(keys.shape[0], -1), axis=1)[:, :n_qubits]
    chars = (bits + ord("0")).astype(np.uint8)
    return [row.tobytes().decode("ascii") for row in chars]


def conditional_marginals_batched(
    template: CircuitNetwork,
    errorsets: Sequence[ErrorSet],
    plan: BatchPlan,
    j: int,
    prefixes: Sequence[str],
    ctx: Optional[SamplerContext] = None,
    *,
    normalize: bool = True,
    return_mass: bool = False,
):
    """Conditional distributions of stage j for W work items
    (error set w, prefix w) in one batched device call.  Row w equals the
    reference's `conditional_marginal(template.merged(errorsets[w]), ...,
    j, prefixes[w])` (engine.py:453-477) up to the dtype's tolerance."""
    if ctx is None:
        ctx = SamplerContext()
    if len(errorsets) != len(prefixes):
        raise ValueError("one prefix per error set expected")
    if not 1 <= j <= plan.f:
        raise ValueError(f"stage {j} outside 1..{plan.f}")
    for s in prefixes:
        if len(s) != plan.offset(j):
            raise ValueError(f"stage {j} expects a {plan.offset(j)}-bit prefix, got {len(s)}")
    ctx.check_deadline()
    tables = VariantTables.from_errorsets(template, errorsets)
    pipe = DevicePipeline(template, plan, tables, ctx, stages=[j])
    try:
        probs, mass, mn = pipe.device_plan.marginals(j, tables.encode(errorsets), pack_prefixes(prefixes, plan.n))
    finally:
        pipe.close()
    ctx.stats.record_contraction(j, 0.0, events=len(prefixes))
    _guard(mn, mass, ctx.dtype, [f"error set {k.id}: " for k in errorsets], prefixes, check_mass=normalize)
    if normalize:
        probs = probs / mass[:, None]
    return (probs, mass) if return_mass else probs


def _guard(mn, mass, dtype, who, prefixes, check_mass=True):
    """Numerical guards of engine.py:445-450 and 475-476.  complex64 cannot
    resolve -1e-12, so its negative tolerance scales with the mass."""
    rel = 1e-4 if dtype == "complex64" else 0.0
    for w in range(len(mass)):
        if mn[w] < NEGATIVE_DIAG_TOLERANCE - rel * mass[w]:
            raise NumericalError(f"{who[w]}marginal diagonal entry {mn[w]} below {NEGATIVE_DIAG_TOLERANCE}")
        if check_mass and mass[w] < VANISHING_MASS:
            raise ImpossiblePrefixError(f"{who[w]}prefix {prefixes[w]!r} has vanishing mass {mass[w]}")


def _contract_marginal(mnet: MarginalNetwork, ctx: SamplerContext, j: int, path=None):
    """(clamped unnormalised population vector, mass) of one stage network on
    the device (engine.py:417-450)."""
    from . import _capi

    ctx.check_deadline()
    net = mnet.net
    if path is None:
        t0 = time.perf_counter()
        path, hit = cache_lookup_or_plan(ctx.cache, net, stage=j, hypersamples=ctx.hypersamples,
                                         rng=spawn_rng(ctx.planner_seed, _KEY_PLANNER, j))
        if not hit:
            ctx.stats.plan_events += 1
            ctx.stats.path_seconds += time.perf_counter() - t0
    ops = [Operand(t.labels, tuple(ix.dim for ix in t.indices), t.data.reshape(1, -1)) for t in net.operands]
    pool = Pool()
    steps = getattr(path, "steps", path)
    progs, _ = compiler.compile_stage(ops, steps, mnet.open_labels, 1, pool, 16 if ctx.dtype != "complex64" else 8,
                                      ceiling=ctx.max_intermediate)
    out_elems = progs[0].out_elems
    nbits = out_elems.bit_length() - 1
    if nbits < 1 or (1 << nbits) != out_elems:
        raise NetworkStructureError("a marginal network must leave 2^b (b >= 1) open entries")
    compiled = CompiledPlan(dtype=ctx.dtype, n_qubits=nbits, n_sites=0, sizes=(nbits,), pool=pool.finish(ctx.dtype),
                            programs=progs, max_intermediate=ctx.max_intermediate)
    dp = _capi.DevicePlan(compiled, ctx.device)
    t0 = time.perf_counter()
    try:
        probs, mass, mn = dp.marginals(1, np.zeros((1, 0), np.uint8), np.zeros((1, dp.words), np.uint64))
    finally:
        dp.close()
    ctx.stats.record_contraction(j, time.perf_counter() - t0)
    _guard(mn, mass, ctx.dtype, [""], [""], check_mass=False)
    return probs[0], float(mass[0])


def conditional_marginal(cnet: CircuitNetwork, cache: PathCache, plan: BatchPlan, j: int, prefix: str, *,
                         hypersamples: int = 100, planner_seed: int = 0, stats: Optional[EngineStats] = None,
                         max_intermediate: int = DEFAULT_INTERMEDIATE_CEILING, dtype: str = "complex128") -> np.ndarray:
    """Normalised conditional distribution over the 2^{b_j} outcomes of stage j
    given `prefix` (engine.py:453-477), one work item on the device."""
    ctx = SamplerContext(cache=cache, stats=stats if stats is not None else EngineStats(),
                         hypersamples=hypersamples, planner_seed=planner_seed,
                         max_intermediate=max_intermediate, dtype=dtype)
    probs, mass = _contract_marginal(marginal_network(cnet, plan, j, prefix), ctx, j)
    if mass < VANISHING_MASS:
        raise ImpossiblePrefixError(f"prefix {prefix!r} has vanishing mass {mass}")
    return probs / mass


def _bits(idx: int, width: int) -> str:
    return format(idx, f"0{width}b")


def _raise_flagged(stats, errorsets_by_id=None):
    if not stats.flagged_sets:
        return
    exc = STATUS_TO_ERROR.get(int(stats.first_flag_kind), SimulationError)
    what = ("marginal diagonal entry below tolerance" if exc is NumericalError
            else "prefix has vanishing mass")
    raise exc(f"error set {int(stats.first_flagged_id)}: stage {int(stats.first_flag_stage)}: {what} "
              f"({int(stats.flagged_sets)} work item(s) flagged)")


def sample_proportional_batched(
    template: CircuitNetwork,
    errorsets: Sequence[ErrorSet],
    plan: BatchPlan,
    seed: int,
    ctx: Optional[SamplerContext] = None,
) -> list:
    """Born-rule sampling of every error set's shots in one batched device run.
    Returns one sorted `list[ShotRecord]` per error set -- what the reference's
    `sample_proportional` (engine.py:493-524) returns for each of them.  The
    RNG stream of a work item is Philox(seed; error-set id, stage, prefix rank),
    so results do not depend on how error sets are grouped into calls."""
    if ctx is None:
        ctx = SamplerContext()
    for k in errorsets:
        if k.m < 1:
            raise ValueError("proportional sampling needs m >= 1")
    ctx.check_deadline()
    tables = VariantTables.from_errorsets(template, errorsets)
    shots = np.asarray([k.m for k in errorsets], dtype=np.uint32)
    pipe = DevicePipeline(template, plan, tables, ctx, shots_per_set=float(shots.mean()), calibrate=True)
    try:
        keys, esets, counts, st = pipe.device_plan.sample(
            tables.encode(errorsets), shots, np.asarray([k.id for k in errorsets], dtype=np.uint32),
            seed, merged=False)
    finally:
        pipe.close()
    _account(ctx.stats, st, plan.f)
    _raise_flagged(st)
    strings = unpack_keys(keys, plan.n)
    out = [[] for _ in errorsets]
    for s, e, c in zip(strings, esets.tolist(), counts.tolist()):
        out[e].append(ShotRecord(bitstring=s, count=int(c)))
    return out


def sample_nonproportional_batched(
    template: CircuitNetwork,
    errorsets: Sequence[ErrorSet],
    plan: BatchPlan,
    seed: int,
    ctx: Optional[SamplerContext] = None,
) -> list:
    """Data-harvesting sampling of every error set in one batched device run
    (reference `sample_nonproportional`, engine.py:527-576): each non-final stage
    branches every prefix into up to `plan.nonfinal_shots` distinct children
    (weighted draw without replacement), the final stage emits every outcome
    whose conditional probability reaches `plan.threshold` (tagged with it) or a
    multinomial split of `plan.direct_count` shots.  One list of ShotRecord per
    error set, in the reference's order (sorted by bitstring)."""
    if ctx is None:
        ctx = SamplerContext()
    ctx.check_deadline()
    tables = VariantTables.from_errorsets(template, errorsets)
    pipe = DevicePipeline(template, plan, tables, ctx, shots_per_set=float(max(plan.nonfinal_shots, 1)))
    try:
        keys, esets, counts, probs, st = pipe.device_plan.sample_nonproportional(
            tables.encode(errorsets), np.asarray([k.id for k in errorsets], dtype=np.uint32), seed,
            plan.nonfinal_shots, plan.final_mode, plan.threshold, plan.direct_count)
    finally:
        pipe.close()
    _account(ctx.stats, st, plan.f)
    _raise_flagged(st)
    strings = unpack_keys(keys, plan.n)
    out = [[] for _ in errorsets]
    tags = probs.tolist() if probs is not None else [None] * len(strings)
    for s, e, c, p in zip(strings, esets.tolist(), counts.tolist(), tags):
        out[e].append(ShotRecord(bitstring=s, count=int(c), prob=p))
    return out


def sample_nonproportional(template: CircuitNetwork, k: ErrorSet, plan: BatchPlan, rng,
                           ctx: Optional[SamplerContext] = None) -> list:
    """Single-error-set form of the reference signature (engine.py:527-533).
    `rng` only seeds the device's counter-based streams."""
    seed = int(rng.integers(0, 2**63 - 1)) if hasattr(rng, "integers") else int(rng)
    return sample_nonproportional_batched(template, [k], plan, seed, ctx)[0]


def _account(stats: EngineStats, st, f: int) -> None:
    for j in range(1, f + 1):
        stats.record_contraction(j, st.stage_ms[j - 1] * 1e-3, events=int(st.stage_events[j - 1]))
        if st.descent_items[j - 1]:
            stats.descent_events[j] = stats.descent_events.get(j, 0) + int(st.descent_items[j - 1])


def sample_proportional(template: CircuitNetwork, k: ErrorSet, plan: BatchPlan, rng,
                        ctx: Optional[SamplerContext] = None) -> list:
    """Single-error-set form of the reference signature (engine.py:493-499).
    `rng` only seeds the device's counter-based streams (one 63-bit draw); a
    NumPy generator cannot be replayed on the device."""
    if k.m < 1:
        raise ValueError("proportional sampling needs m >= 1")
    seed = int(rng.integers(0, 2**63 - 1)) if hasattr(rng, "integers") else int(rng)
    return sample_proportional_batched(template, [k], plan, seed, ctx)[0]


def merge_records(per_set: Sequence[Sequence[ShotRecord]]) -> list:
    """Counts summed per bitstring on the device (sort + reduce-by-key); the
    `prob` tag survives only if all contributors agree (engine.py:815-829)."""
    from . import _capi

    rows = [r for recs in per_set for r in recs]
    if not rows:
        return []
    width = len(rows[0].bitstring)
    keys, counts = _capi.histogram_merge(pack_prefixes([r.bitstring for r in rows], width),
                                         np.asarray([r.count for r in rows], dtype=np.uint64))
    tags: dict = {}
    for r in rows:
        if r.bitstring not in tags:
            tags[r.bitstring] = r.prob
        elif tags[r.bitstring] != r.prob:
            tags[r.bitstring] = None
    return [ShotRecord(bitstring=s, count=int(c), prob=tags[s])
            for s, c in zip(unpack_keys(keys, width), counts.tolist())]


MODES = ("ptsbe-proportional", "ptsbe-nonproportional", "unoptimized-ptsbe", "baseline")


@dataclass
class RunConfig:
    """Run description, echoed into results (engine.py:667-747).  `dtype` and
    `device` are the only additions; defaults keep reference numerics."""

    n: int
    g: int
    mode: str = "ptsbe-proportional"
    two_qubit_fraction: float = 0.2
    p_range: tuple = (0.02, 0.2)
    error_sets: int = 4
    total_shots: int = 64
    batch_sizes: Optional[tuple] = None
    nonfinal_batch: int = 10
    final_batch: int = 28
    nonfinal_shots: int = 1
    final_mode: str = "exhaustive"
    tau: float = 1e-6
    direct_count: int = 1
    hypersamples: int = 100
    baseline_batch: int = 24
    baseline_hypersamples: int = 1
    seed: int = 0
    workers: int = 1
    max_intermediate: int = DEFAULT_INTERMEDIATE_CEILING
    timeout_s: Optional[float] = 120.0
    dtype: str = "complex128"
    device: int = 0

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.dtype not in ("complex64", "complex128"):
            raise ValueError(f"dtype must be complex64 or complex128, got {self.dtype!r}")
        if self.batch_sizes is not None:
            self.batch_sizes = tuple(int(b) for b in self.batch_sizes)
            if sum(self.batch_sizes) != self.n:
                raise ValueError(f"batch sizes {self.batch_sizes} must sum to n={self.n}")

    def plan(self) -> BatchPlan:
        kw = dict(nonfinal_shots=self.nonfinal_shots, final_mode=self.final_mode,
                  direct_count=self.direct_count, threshold=self.tau)
        if self.batch_sizes is not None:
            return BatchPlan(sizes=self.batch_sizes, **kw)
        return BatchPlan.with_final(self.n, self.nonfinal_batch, self.final_batch, **kw)

    def to_dict(self) -> dict:
        doc = {k: getattr(self, k) for k in (
            "n", "g", "mode", "two_qubit_fraction", "p_range", "error_sets", "total_shots",
            "batch_sizes", "nonfinal_batch", "final_batch", "nonfinal_shots", "final_mode", "tau",
            "direct_count", "hypersamples", "baseline_batch", "baseline_hypersamples", "seed",
            "workers", "max_intermediate", "timeout_s", "dtype", "device")}
        doc["p_range"] = list(self.p_range)
        doc["batch_sizes"] = list(self.batch_sizes) if self.batch_sizes else None
        return doc

    @classmethod
    def from_dict(cls, doc: dict) -> "RunConfig":
        doc = dict(doc)
        for key in ("p_range", "batch_sizes"):
            if doc.get(key) is not None:
                doc[key] = tuple(doc[key])
        return cls(**doc)


@dataclass
class RunResult:
    """Aggregated records + instrumentation (engine.py:750-812)."""

    mode: str
    records: list
    unique_shots: int
    total_count: int
    timings: dict
    plan_events: int
    contract_events: int
    stage_events: dict
    stage_seconds: dict
    config: dict
    seed: int
    shot_allocations: list
    # packed device-format histogram ([R, words] u64 keys, [R] u64 counts); kept only
    # for the multi-GPU gather (partition.py), never serialised
    packed_keys: Optional[np.ndarray] = field(default=None, repr=False, compare=False)
    packed_counts: Optional[np.ndarray] = field(default=None, repr=False, compare=False)

    @property
    def loop_seconds(self) -> float:
        return self.timings["loop_s"]

    def to_json(self) -> str:
        return json.dumps({
            "mode": self.mode,
            "records": [{"bitstring": r.bitstring, "count": r.count, "prob": r.prob} for r in self.records],
            "unique_shots": self.unique_shots,
            "total_count": self.total_count,
            "timings": self.timings,
            "plan_events": self.plan_events,
            "contract_events": self.contract_events,
            "stage_events": {str(k): v for k, v in self.stage_events.items()},
            "stage_seconds": {str(k): v for k, v in self.stage_seconds.items()},
            "config": self.config,
            "seed": self.seed,
            "shot_allocations": self.shot_allocations,
        })

    @classmethod
    def from_json(cls, text: str) -> "RunResult":
        doc = json.loads(text)
        return cls(
            mode=doc["mode"],
            records=[ShotRecord(r["bitstring"], r["count"], r.get("prob")) for r in doc["records"]],
            unique_shots=doc["unique_shots"], total_count=doc["total_count"], timings=doc["timings"],
            plan_events=doc["plan_events"], contract_events=doc["contract_events"],
            stage_events={int(k): v for k, v in doc["stage_events"].items()},
            stage_seconds={int(k): v for k, v in doc["stage_seconds"].items()},
            config=doc["config"], seed=doc["seed"], shot_allocations=doc["shot_allocations"],
        )


def run_ptsbe(c: Circuit, config: RunConfig, cache: Optional[PathCache] = None,
              errorsets: Optional[Sequence[ErrorSet]] = None, _keep_packed: bool = False,
              _shard: Optional[tuple] = None) -> RunResult:
    """Optimised proportional pipeline on the device (engine.py:832-929):
    pre-sample error sets on the host (same rng stream as the reference), plan
    one path per stage on the error-free template (plan events = f, or 0 with a
    warm cache), then ONE batched device run over all error sets, histogram
    merged on the device.  `errorsets` overrides the pre-sampling (the
    north-star API: pre-sampled error sets in, histogram out).

    `_shard=(lo, hi)` (partition.run_ptsbe_sharded): everything that shapes the
    arithmetic -- variant tables, light cone, planner weights, stored paths,
    sampler choice per stage -- is built from the FULL error-set list, exactly
    as in a single-process run; only error sets [lo, hi) are sampled here."""
    if config.mode not in ("ptsbe-proportional", "ptsbe-nonproportional"):
        raise ValueError(f"run_ptsbe handles optimized modes only, got {config.mode!r}")
    nonprop = config.mode == "ptsbe-nonproportional"
    plan = config.plan()
    if plan.n != c.n:
        raise ValueError(f"plan covers {plan.n} qubits, circuit has {c.n}")
    ctx = SamplerContext(
        cache=cache if cache is not None else PathCache(), hypersamples=config.hypersamples,
        planner_seed=config.seed, max_intermediate=config.max_intermediate,
        deadline=(time.perf_counter() + config.timeout_s) if config.timeout_s else None,
        dtype=config.dtype, device=config.device,
    )
    t0 = time.perf_counter()
    template = CircuitNetwork.from_circuit(c)
    if errorsets is None:
        errorsets = presample_errors(c, config.error_sets, rule="proportional",
                                     total_shots=config.total_shots,
                                     rng=spawn_rng(config.seed, _KEY_PRESAMPLE))
    generate_s = time.perf_counter() - t0

    t0 = time.perf_counter()
    tables = VariantTables.from_errorsets(template, errorsets)
    shots = np.asarray([k.m for k in errorsets], dtype=np.uint32)
    if not nonprop and shots.min() < 1:
        raise ValueError("proportional sampling needs m >= 1")
    pipe = DevicePipeline(template, plan, tables, ctx,
                          shots_per_set=float(plan.nonfinal_shots) if nonprop else float(shots.mean()),
                          calibrate=not nonprop)
    plan_s = time.perf_counter() - t0
    all_sets = errorsets
    if _shard is not None:
        errorsets = list(errorsets[_shard[0]:_shard[1]])
        shots = shots[_shard[0]:_shard[1]]
    try:
        ctx.check_deadline()
        kraus_idx = tables.encode(errorsets)
        ids = np.asarray([k.id for k in errorsets], dtype=np.uint32)
        t0 = time.perf_counter()
        if nonprop:
            keys, esets, counts, probs, st = pipe.device_plan.sample_nonproportional(
                kraus_idx, ids, config.seed, plan.nonfinal_shots, plan.final_mode, plan.threshold, plan.direct_count)
        elif plan.n <= 32 and int(np.asarray(shots, dtype=np.uint64).sum()) < 2**32:
            # (key, count) rows as two u32: half the bytes on the PCIe link, same records
            rec, st = pipe.device_plan.sample_packed(kraus_idx, shots, ids, config.seed)
            keys, counts = rec[:, :1].astype(np.uint64) << np.uint64(32), rec[:, 1]
        else:
            keys, _, counts, st = pipe.device_plan.sample(kraus_idx, shots, ids, config.seed, merged=True)
        loop_s = time.perf_counter() - t0
    finally:
        pipe.close()
    _account(ctx.stats, st, plan.f)
    _raise_flagged(st)
    t0 = time.perf_counter()
    if nonprop:
        # per-error-set records -> merge_records (engine.py:815-829): counts summed per bitstring, the
        # probability tag survives only if every contributor agrees
        per_set = [[] for _ in errorsets]
        tags = probs.tolist() if probs is not None else [None] * int(counts.size)
        for s_, e_, n_, p_ in zip(unpack_keys(keys, plan.n), esets.tolist(), counts.tolist(), tags):
            per_set[e_].append(ShotRecord(bitstring=s_, count=int(n_), prob=p_))
        records = merge_records(per_set)
    else:
        records = [ShotRecord(bitstring=s, count=int(n)) for s, n in zip(unpack_keys(keys, plan.n), counts.tolist())]
    aggregate_s = time.perf_counter() - t0
    return RunResult(
        mode=config.mode, records=records, unique_shots=len(records),
        total_count=sum(r.count for r in records),
        timings={
            "generate_s": generate_s, "plan_s": plan_s, "loop_s": loop_s, "aggregate_s": aggregate_s,
            "path_s": ctx.stats.path_seconds, "contract_s": ctx.stats.contract_seconds,
            "device_loop_s": st.loop_ms * 1e-3, "h2d_s": st.h2d_ms * 1e-3, "d2h_s": st.d2h_ms * 1e-3,
            "gpu_launches": int(st.gpu_launches),
        },
        plan_events=ctx.stats.plan_events, contract_events=ctx.stats.contract_events,
        stage_events=dict(sorted(ctx.stats.stage_events.items())),
        stage_seconds=dict(sorted(ctx.stats.stage_seconds.items())),
        config=config.to_dict(), seed=config.seed, shot_allocations=[int(k.m) for k in errorsets],
        packed_keys=keys if (_keep_packed and not nonprop) else None,
        packed_counts=counts if (_keep_packed and not nonprop) else None,
    )


def run_mode(c: Circuit, config: RunConfig, cache: Optional[PathCache] = None) -> RunResult:
    """Dispatch by mode (engine.py:932-941).  Only the proportional PTSBE mode
    runs on the device; the comparison modes stay with the CPU reference."""
    if config.mode in ("ptsbe-proportional", "ptsbe-nonproportional"):
        return run_ptsbe(c, config, cache=cache)
    raise NotImplementedError(
        f"mode {config.mode!r} is a CPU comparison mode of the reference and is out of scope here"
    )


def _out_of_scope(name: str):
    def stub(*_a, **_k):
        raise NotImplementedError(f"{name} is outside the B200 hot path (SURVEY.md sections 2, 8f); "
                                  "use the CPU reference for it")
    stub.__name__ = name
    return stub


insert_errors = _out_of_scope("insert_errors")
sample_baseline = _out_of_scope("sample_baseline")
sample_unoptimized_ptsbe = _out_of_scope("sample_unoptimized_ptsbe")
