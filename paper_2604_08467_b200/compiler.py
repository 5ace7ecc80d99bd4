"""Stage-program compiler: (stage network structure, stored path) -> flat device
programs for `csrc/executor.cuh`.

What the reference does per contraction at run time -- rebuild the sandwich
network (engine.py:361-407), conjugate every operand (tensor.py:87-88), look
the path up and validate it (planner.py:416-442), dispatch one np.tensordot
per step (tensor.py:236-259) and transpose the result (engine.py:442) -- is
done here ONCE per (circuit structure, batch plan): every step gets
precomputed gather tables, every intermediate gets an arena offset from a
liveness analysis, the bra half is stored pre-conjugated in the operand pool
and the output permutation is folded into the last step.

Error-independent hoisting (north-star subsystem 1): every node of the
contraction tree is tagged with the newest thing its value depends on --
class 0: the error set only; class s: also prefix bits measured in stage s.
Nodes of class p are evaluated in "pass p", once per unique prefix entering
stage p+1, and handed to later passes as records in HBM.  Only the nodes
whose class is j-1 are recomputed for every stage-j work item.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .errors import CapacityError, IncompletePathError, NetworkStructureError, ResourceLimitError

SEL_CONST, SEL_KRAUS, SEL_PREFIX = 0, 1, 2
STEP_WORDS, LEAF_WORDS = 20, 4
GEMM_MIN_MACS = 2048       # steps at least this large also get their separable (GEMM) form
MEMO_NONE = 0xFFFF         # "operand is not produced by a step of this program"
MEMO_MIN_STEPS = 48        # class-0 programs at least this long get a variant-0 memo
LO_TABLE_MAX = 1024          # entries in the per-lane (low) gather table of a step
SMEM_BYTES = 52 * 1024       # shared-memory arena of a CTA-per-item program: 4 CTAs per SM stay resident
SMALL_ARENA_BYTES = 6 * 1024   # up to here the lane count is chosen by issued instructions alone
BIG_ARENA_LANES = 32  # measured on cfg5 (8: 155.8, 16: 150.4, 32: 148.4 ms per step)
WARP_ARENA_BYTES = 16 * 1024  # beyond this a warp-per-item mapping starves occupancy (8 warps x 16 KB = 2 CTAs per SM)


@dataclass
class Operand:
    """One leaf of a stage network.  `data` is [variants, size] complex128,
    row-major over `labels`; the variant is chosen per work item by the Kraus
    index of gate site `sel_arg` (SEL_KRAUS) or by prefix bit `sel_arg`
    (SEL_PREFIX)."""

    labels: tuple
    dims: tuple
    data: np.ndarray
    sel_kind: int = SEL_CONST
    sel_arg: int = 0
    cls: int = 0


class Pool:
    """Operand value pool shared by all programs of a plan; identical blocks
    (kets, basis vectors, copy tensors) are stored once."""

    def __init__(self):
        self.blocks: list[np.ndarray] = []
        self.size = 0
        self._seen: dict[bytes, int] = {}

    def add(self, block: np.ndarray) -> int:
        flat = np.ascontiguousarray(block, dtype=np.complex128).reshape(-1)
        key = flat.tobytes()
        at = self._seen.get(key)
        if at is None:
            at = self.size
            self._seen[key] = at
            self.blocks.append(flat)
            self.size += flat.size
        return at

    def finish(self, dtype: str) -> np.ndarray:
        allv = np.concatenate(self.blocks) if self.blocks else np.zeros(0, np.complex128)
        return allv.astype(np.complex64 if dtype == "complex64" else np.complex128)


@dataclass
class Program:
    leaves: np.ndarray
    steps: np.ndarray
    tables: np.ndarray
    arena_fast: int
    arena_spill: int
    out_elems: int
    threads: int
    level: int
    result_kind: int = 0
    result_ref: int = 0
    flops: float = 0.0          # complex multiply-adds of one execution of this pass
    peak_elems: int = 0
    max_out: int = 0
    ext_read_elems: int = 0     # elements of earlier passes' records one execution reads (HBM/L2)
    leaf_read_elems: int = 0    # elements of operand-pool leaves one execution reads (L1/L2 resident)
    proj_d: int = 0             # > 0: projection form, the steps produce a vector v[proj_d] and the
                                # stage result is Re(v . M), M[proj_d, out_elems] at result_ref in pass 0's record
    # variant-0 memo (class-0 programs): the value of every step under "no error anywhere" is
    # computed once per plan; a work item re-executes only the steps above a site whose Kraus
    # index is non-zero (memo_idx[memo_ptr[s]:memo_ptr[s+1]] = steps depending on site s; row
    # n_sites = steps that always run: record outputs and the result)
    memo_elems: int = 0
    memo_ptr: Optional[np.ndarray] = None
    memo_idx: Optional[np.ndarray] = None


class _Arena:
    """First-fit allocator over element offsets, used for liveness-based
    placement of intermediates."""

    def __init__(self):
        self.free: list[list[int]] = []  # sorted [start, end)
        self.top = 0

    def alloc(self, n: int, cap: Optional[int] = None) -> Optional[int]:
        """Offset of a free run of n elements; None (state untouched) when the
        run would end beyond `cap`."""
        for k, (s, e) in enumerate(self.free):
            if e - s >= n:
                if e - s == n:
                    del self.free[k]
                else:
                    self.free[k][0] = s + n
                return s
        # grow; a trailing free block that touches the top is extended
        tail = bool(self.free) and self.free[-1][1] == self.top
        s = self.free[-1][0] if tail else self.top
        if cap is not None and s + n > cap:
            return None
        if tail:
            del self.free[-1]
        self.top = s + n
        return s

    def release(self, s: int, n: int) -> None:
        self.free.append([s, s + n])
        self.free.sort()
        merged = []
        for blk in self.free:
            if merged and merged[-1][1] == blk[0]:
                merged[-1][1] = blk[1]
            else:
                merged.append(blk)
        self.free = merged


def _offsets(dims: Sequence[int], strides: Sequence[int]) -> np.ndarray:
    """Row-major enumeration of a multi-index -> linear offset with the given
    strides (0 stride = label absent from that operand)."""
    out = np.zeros(1, dtype=np.int64)
    for d, s in zip(dims, strides):
        out = (out[:, None] + (np.arange(d, dtype=np.int64) * s)[None, :]).reshape(-1)
    return out


def _row_major_strides(dims: Sequence[int]) -> list[int]:
    st = [1] * len(dims)
    for k in range(len(dims) - 2, -1, -1):
        st[k] = st[k + 1] * dims[k + 1]
    return st


@dataclass
class _Node:
    labels: tuple
    dims: tuple
    cls: int
    a: int = -1
    b: int = -1
    parent: int = -1
    pass_: int = 0
    size: int = 1


def build_tree(operands: Sequence[Operand], steps, ceiling: Optional[int] = None):
    """Replay slot steps into a binary tree.  Result legs: a's survivors then
    b's (tensor.py:193-195).  Raises like the reference's execute_path."""
    nodes = [
        _Node(tuple(o.labels), tuple(o.dims), o.cls, size=int(np.prod(o.dims, dtype=np.int64)) if o.dims else 1)
        for o in operands
    ]
    slots = list(range(len(operands)))
    flops = 0.0
    for step in steps:
        i, j = int(step[0]), int(step[1])
        if i > j:
            i, j = j, i
        if i == j or i < 0 or j >= len(slots):
            raise NetworkStructureError(f"invalid step {tuple(step)} with {len(slots)} slots")
        na, nb = nodes[slots[i]], nodes[slots[j]]
        bd = dict(zip(nb.labels, nb.dims))
        shared = set()
        for lb, d in zip(na.labels, na.dims):
            if lb in bd:
                if bd[lb] != d:
                    raise NetworkStructureError(f"shared label {lb} has dims {d} vs {bd[lb]}")
                shared.add(lb)
        labels = [lb for lb in na.labels if lb not in shared] + [lb for lb in nb.labels if lb not in shared]
        dims = [d for lb, d in zip(na.labels, na.dims) if lb not in shared] + [
            d for lb, d in zip(nb.labels, nb.dims) if lb not in shared
        ]
        size = int(np.prod(dims, dtype=object)) if dims else 1
        if ceiling is not None and size > ceiling:
            raise ResourceLimitError(f"intermediate of {size} entries exceeds ceiling {ceiling}")
        k = 1
        for lb, d in zip(na.labels, na.dims):
            if lb in shared:
                k *= d
        flops += float(size) * k
        nid = len(nodes)
        nodes.append(_Node(tuple(labels), tuple(dims), max(na.cls, nb.cls), slots[i], slots[j], size=size))
        na.parent = nb.parent = nid
        slots[i] = nid
        del slots[j]
    if len(slots) != 1:
        raise IncompletePathError(f"path left {len(slots)} operands, expected 1")
    return nodes, slots[0], flops


def compile_stage(
    operands: Sequence[Operand],
    steps,
    open_order: Optional[Sequence[int]],
    n_passes: int,
    pool: Pool,
    elem_bytes: int,
    ceiling: Optional[int] = None,
    mirror: Optional[Sequence[int]] = None,
    fold_from: Optional[int] = None,
    consumer_layout: int = 0,
    step_order: str = "dfs",
) -> tuple[list[Program], tuple]:
    """Compile one stage network + stored path into `n_passes` programs.
    Returns (programs, result label order).

    `fold_from` (optional, >= 1): classes fold_from .. n_passes - 2 are not hoisted; their nodes are
    evaluated by the marginal pass together with the per-item class (the caller asks for this when
    those classes have about as many distinct instances as there are work items, so a hoist pass
    would save no arithmetic and cost a launch plus a record round trip through HBM).  The
    programs of the folded passes are empty.

    `step_order`: "dfs" (default) replays the steps of a pass depth first, the child with the larger
    live footprint first (Sethi-Ullman), instead of in stored-path order ("path").  Every node is
    still the contraction of the same two children, so every value is bit-identical; what changes is
    how long intermediates stay alive, i.e. the arena a work item needs (shared memory per item for
    the group kernels, cache footprint for the thread-per-error-set kernel).

    `consumer_layout`: order in which a record (a tensor handed to a later pass) is stored, chosen
    from the step of the latest pass that reads it (see "record layout" below).  0: as the path
    produced it; 1: [slicing bits][contracted][surviving] -- the block one work item reads is
    contiguous, which suits kernels that serve an item with a group of lanes; 2 (the engine's
    default): [contracted][surviving][slicing bits] -- element (k, c) of the blocks of ALL prefixes
    is contiguous, so the 32 work items a warp of a lane-per-item kernel serves, which differ in
    the slicing bits only, touch a few cache lines per load instead of up to 32.  Measured on cfg2
    (DESIGN.md section 7): 40.8 ms per step with 0, 50.1 with 1, 37.6 with 2.

    `mirror[k]` (optional) names the operand whose value is the complex
    conjugate of operand k under a relabelling (the bra copy of a ket operand,
    engine.py:393 of the reference).  A subtree built only from mirror
    operands of an already computed subtree, in the same shape, is its
    conjugate: it is not computed at all, its consumers read the original
    with a conjugation flag (step word 11: bit 0 = conj A, bit 1 = conj B)."""
    nodes, root, _ = build_tree(operands, steps, ceiling)
    n_leaves = len(operands)
    top = n_passes - 1
    rootn = nodes[root]
    if open_order is None:
        open_order = rootn.labels
    if sorted(open_order) != sorted(rootn.labels):
        raise NetworkStructureError(
            f"result labels {sorted(rootn.labels)} != open indices {sorted(open_order)}"
        )
    for nd in nodes:
        nd.pass_ = min(nd.cls, top)
        if fold_from is not None and fold_from >= 1 and nd.pass_ >= fold_from:
            nd.pass_ = top
    if root >= n_leaves:
        rootn.pass_ = top  # the finished record is always produced by the marginal pass

    # projection form: root = (per-item vector v) x (error-set record M[v legs, open legs]).
    # The root step is not interpreted per item; it runs as one dense product over all
    # items that share M (csrc/project.cuh).  M is stored as [v's leg order, open order].
    proj = None
    if top >= 1 and root >= n_leaves:
        for v, m in ((rootn.a, rootn.b), (rootn.b, rootn.a)):
            nv, nm = nodes[v], nodes[m]
            if (v >= n_leaves and m >= n_leaves and nm.cls == 0 and nv.pass_ == top
                    and set(nv.labels) <= set(nm.labels)
                    and set(nm.labels) - set(nv.labels) == set(open_order)):
                proj = (v, m)
                break

    # conjugate subtrees --------------------------------------------------------
    virt: dict[int, int] = {}          # virtual node -> the computed node it is the conjugate of
    if mirror is not None:
        node_mirror: dict[int, int] = {k: int(m) for k, m in enumerate(mirror) if m is not None and m >= 0}
        by_children: dict[tuple, int] = {}
        for nid in range(n_leaves, len(nodes)):
            nd = nodes[nid]
            ma, mb = node_mirror.get(nd.a), node_mirror.get(nd.b)
            twin = by_children.get((ma, mb)) if (ma is not None and mb is not None) else None
            if (twin is not None and twin != nid and twin not in virt and nid != root
                    and nodes[twin].cls == nd.cls and nodes[twin].dims == nd.dims
                    and (proj is None or nid not in proj)):
                virt[nid] = twin
                node_mirror[nid] = twin
                node_mirror[twin] = nid
            else:
                by_children[(nd.a, nd.b)] = nid

    def real_of(nid: int) -> int:
        return virt.get(nid, nid)

    # slice views --------------------------------------------------------------
    # Contracting a prefix-bit basis vector e_x over its only label selects the slice
    # T[.., x, ..] of the other operand.  Such a node is never materialised: it is a VIEW of
    # T's storage (T's strides minus that label, base offset + bit(q) * stride), and its
    # consumers gather straight from T.  Exceptions (materialised by a gather step): views
    # that must live in a record -- consumed by a later pass than the one holding T's buffer,
    # the projection vector, the root.
    def selector_of(nid: int):
        """(selector leaf, other child) when node nid is a slice, else None."""
        nd = nodes[nid]
        for x, other in ((nd.a, nd.b), (nd.b, nd.a)):
            if (x < n_leaves and operands[x].sel_kind == SEL_PREFIX and len(nodes[x].labels) == 1
                    and nodes[x].labels[0] in nodes[other].labels):
                return x, other
        return None

    view: dict[int, tuple] = {}  # view node -> (child it slices, label, qubit)

    def storage_of(nid: int):
        """(materialised node or leaf, conj?, [(qubit, label)...]) behind a node."""
        conj, terms = False, []
        while True:
            if nid in virt:
                nid = virt[nid]
                conj = not conj
                continue
            if nid in view:
                child, lb, q = view[nid]
                terms.append((q, lb))
                nid = child
                continue
            return nid, conj, terms

    for nid in range(n_leaves, len(nodes)):
        if nid in virt or nid == root or (proj is not None and nid in proj):
            continue
        sel = selector_of(nid)
        if sel is None:
            continue
        base, _, _ = storage_of(sel[1])
        # the buffer behind the view must be readable where the view is consumed: a leaf, or a
        # node of the same pass as the view's own pass, or of an earlier pass (then it is a record)
        if base >= n_leaves and nodes[base].pass_ > nodes[nid].pass_:
            continue
        view[nid] = (sel[1], nodes[sel[0]].labels[0], operands[sel[0]].sel_arg)

    # consumers of a materialised node: every computed step that reads its storage, directly,
    # through a conjugate twin or through slice views
    consumers: dict[int, list[int]] = {}
    for nid in range(n_leaves, len(nodes)):
        if nid in virt or nid in view:
            continue
        nd = nodes[nid]
        for ch in (nd.a, nd.b):
            consumers.setdefault(storage_of(ch)[0], []).append(nid)

    # storage decisions ------------------------------------------------------
    # frontier = computed node consumed by a later pass -> lives in its pass's record
    rec_off: dict[int, int] = {}
    rec_size = [0] * n_passes
    for nid in range(n_leaves, len(nodes)):
        nd = nodes[nid]
        if nid in virt or nid in view:
            continue
        if any(nodes[c].pass_ > nd.pass_ for c in consumers.get(nid, ())):
            rec_off[nid] = rec_size[nd.pass_]
            rec_size[nd.pass_] += (nd.size + 3) & ~3  # 4-element granules keep vector loads aligned
    if proj is not None:
        rec_off[proj[0]] = 0  # v is the output record of the marginal pass
        rec_size[top] = nodes[proj[0]].size

    # record layout ------------------------------------------------------------
    # A record is read by tens of millions of per-item steps and written once per instance of its
    # own class, so it is stored in the order its consumer of the latest pass reads it: labels that
    # the consumer slices away with prefix bits first, then the contracted labels, then the
    # surviving ones in the consumer's output order.  The operand of one work item (e.g. the 8 x 8
    # transfer matrix selected by the bits of the previous stage) is then ONE contiguous block with
    # the output index fastest, instead of a gather over the whole record.  Only the label order
    # of the stored tensor changes; every table below is derived from label -> stride maps.
    for R in (list(rec_off) if consumer_layout else ()):
        if R == root or (proj is not None and R in proj):
            continue
        later = [c for c in consumers.get(R, ()) if nodes[c].pass_ > nodes[R].pass_]
        if not later:
            continue
        nd = nodes[max(later, key=lambda c: (nodes[c].pass_, c))]
        for ch, other in ((nd.a, nd.b), (nd.b, nd.a)):
            x = ch
            while x in view and x not in virt:
                x = view[x][0]
            if x != R or x in virt:
                continue
            op_labels = nodes[ch].labels
            others = set(nodes[other].labels)
            shared = [lb for lb in op_labels if lb in others]
            surv = [lb for lb in nd.labels if lb in op_labels and lb not in others]
            surv += [lb for lb in op_labels if lb not in others and lb not in surv]
            sliced = [lb for lb in nodes[R].labels if lb not in op_labels]
            # 1: the per-item block contiguous (lane groups read it as rows); 2: the slicing bits fastest, so
            # the 32 items a warp of a lane-per-item kernel serves find element (k, c) of their 32 different
            # blocks within a few cache lines
            order = sliced + shared + surv if consumer_layout == 1 else shared + surv + sliced
            if sorted(map(str, order)) == sorted(map(str, nodes[R].labels)) and len(set(order)) == len(order):
                _relabel(nodes, virt, view, R, tuple(order))
            break

    programs: list[Program] = []
    result_kind, result_ref = 0, 0
    for p in range(n_passes):
        mine = [nid for nid in range(n_leaves, len(nodes)) if nodes[nid].pass_ == p and nid not in virt and nid not in view]
        if proj is not None and p == top:
            mine = [nid for nid in mine if nid != root]
        if step_order == "dfs":
            mine = _depth_first(nodes, mine, rec_off, lambda x: storage_of(x)[0])
        # sizing of the on-chip arena: try everything on chip, spill the big buffers otherwise
        max_out = max([nodes[nid].size for nid in mine], default=1)
        peak = _place(nodes, mine, rec_off, lambda x: storage_of(x)[0], fast_cap=None)[1]
        if max_out <= 1024 and peak * elem_bytes <= WARP_ARENA_BYTES:
            # sub-warp groups: GS lanes per item, 32 / GS items per warp in lockstep.  Pick the
            # group size with the fewest issued warp-instructions per item (rough model of
            # csrc/executor.cuh: per step ~80, per output ~10, per multiply-add ~8).
            def per_item(gs):
                total = 0.0
                for nid in mine:
                    nd = nodes[nid]
                    kn = 1
                    la = set(nodes[nd.a].labels)
                    for lb, d in zip(nodes[nd.b].labels, nodes[nd.b].dims):
                        if lb in la:
                            kn *= d
                    total += 80 + -(-nd.size // gs) * (10 + 8 * kn)
                return total * gs / 32.0
            threads = min((8, 16, 32), key=per_item)
            if peak * elem_bytes > SMALL_ARENA_BYTES:
                # big arenas leave room for few groups per SM: latency per step, not issued
                # instructions, decides -- spread the item over more lanes
                threads = int(os.environ.get("PTSBE_BIG_GS", BIG_ARENA_LANES))
            fast_cap = peak
        else:
            # CTA per item.  Large steps run as 4 x 4 register tiles (separable form), so 256
            # threads cover 4096 outputs per sweep and two CTAs fit the register file of an SM
            threads = 64
            while threads < 256 and threads * 4 < max_out:
                threads *= 2
            fast_cap = min(peak, SMEM_BYTES // elem_bytes)
        where, peak_fast, peak_spill = _place(nodes, mine, rec_off, lambda x: storage_of(x)[0], fast_cap=fast_cap)

        step_rows, tables = [], []
        tab_off = 0
        flops = 0.0
        step_index: dict[int, int] = {}   # node -> index of the step of this program that computes it
        memo_off: dict[int, int] = {}
        memo_top = 0
        step_sites: list[int] = []        # per step: bitset of the gate sites its value depends on
        always_steps: list[int] = []
        n_sites = 1 + max([o.sel_arg for o in operands if o.sel_kind == SEL_KRAUS], default=-1)
        prog_leaves: list[list[int]] = []
        prog_leaf_index: dict[int, int] = {}
        ext_reads: dict[int, int] = {}

        def ref_of(nid: int, sliced: int = 0):
            """(kind, ref) of a MATERIALISED node or leaf."""
            if nid < n_leaves:
                at = prog_leaf_index.get(nid)
                if at is None:
                    o = operands[nid]
                    blk = np.asarray(o.data, dtype=np.complex128).reshape(o.data.shape[0], -1)
                    size = blk.shape[1]
                    at = len(prog_leaves)
                    prog_leaf_index[nid] = at
                    prog_leaves.append([pool.add(blk), size, o.sel_kind, o.sel_arg])
                return 1, at
            if nid in rec_off:
                # lives in a record: of an earlier pass, or of this very pass (a node that also
                # feeds a later pass; the group wrote it before the barrier that precedes this step)
                if nodes[nid].pass_ != p:
                    ext_reads[nid] = max(ext_reads.get(nid, 0), nodes[nid].size >> sliced)
                elif p == top:
                    raise AssertionError("the projection vector is consumed by the projection kernel only")
                return 2 + nodes[nid].pass_, rec_off[nid]
            return 0, where[nid]

        def layout(nid: int):
            """(materialised base, conj?, strides aligned with nodes[nid].labels,
            [(qubit, stride)] dynamic offset terms) of an operand."""
            if nid in virt:
                b, cj, st, tm = layout(virt[nid])
                return b, not cj, st, tm
            if nid in view:
                child, lb, q = view[nid]
                b, cj, st, tm = layout(child)
                pos = nodes[child].labels.index(lb)
                return b, cj, st[:pos] + st[pos + 1:], tm + [(q, st[pos])]
            return nid, False, _row_major_strides(nodes[nid].dims), []

        for nid in mine:
            nd = nodes[nid]
            ca, cb = nd.a, nd.b
            # a slice that has to be materialised (it feeds a record): the basis vector becomes
            # operand B and the step is flagged (bit 2), the executor gathers instead of multiplying
            select = False
            sel = selector_of(nid)
            if sel is not None:
                ca, cb = sel[1], sel[0]
                select = True
            na, nb = nodes[ca], nodes[cb]
            base_a, conj_a, st_a, terms_a = layout(ca)
            base_b, conj_b, st_b, terms_b = layout(cb)
            a_kind, a_ref = ref_of(base_a, len(terms_a))
            b_kind, b_ref = ref_of(base_b, len(terms_b))
            dyn = bool(terms_a or terms_b)
            conj_flags = (1 if conj_a else 0) | (2 if conj_b else 0) | (4 if select else 0) | (8 if dyn else 0)
            if nid in rec_off:
                o_kind, o_ref = 1, rec_off[nid]
            else:
                o_kind, o_ref = 0, where[nid]
            out_labels = list(open_order) if nid == root else list(nd.labels)
            if proj is not None and nid == proj[1]:
                out_labels = list(nodes[proj[0]].labels) + list(open_order)
            dim_of = dict(zip(na.labels, na.dims))
            dim_of.update(zip(nb.labels, nb.dims))
            sa = dict(zip(na.labels, st_a))
            sb = dict(zip(nb.labels, st_b))
            shared = [lb for lb in na.labels if lb in sb]
            odims = [dim_of[lb] for lb in out_labels]
            # split the output index into a high part and a <= LO_TABLE_MAX low part
            cut, lo_n = len(out_labels), 1
            while cut > 0 and lo_n * odims[cut - 1] <= LO_TABLE_MAX:
                cut -= 1
                lo_n *= odims[cut]
            hi_lab, lo_lab = out_labels[:cut], out_labels[cut:]
            hi_n = int(np.prod([dim_of[lb] for lb in hi_lab], dtype=np.int64)) if hi_lab else 1
            lo_a = _offsets([dim_of[lb] for lb in lo_lab], [sa.get(lb, 0) for lb in lo_lab])
            lo_b = _offsets([dim_of[lb] for lb in lo_lab], [sb.get(lb, 0) for lb in lo_lab])
            hi_a = _offsets([dim_of[lb] for lb in hi_lab], [sa.get(lb, 0) for lb in hi_lab])
            hi_b = _offsets([dim_of[lb] for lb in hi_lab], [sb.get(lb, 0) for lb in hi_lab])
            k_a = _offsets([dim_of[lb] for lb in shared], [sa[lb] for lb in shared])
            k_b = _offsets([dim_of[lb] for lb in shared], [sb[lb] for lb in shared])
            k_n = k_a.size
            parts = [lo_a, lo_b, hi_a, hi_b, k_a, k_b]
            if dyn:  # [nA, (qubit, stride) * nA, nB, (qubit, stride) * nB]
                dyn_words = [len(terms_a)] + [w for t in terms_a for w in t] + \
                            [len(terms_b)] + [w for t in terms_b for w in t]
                parts.append(np.asarray(dyn_words, dtype=np.int64))
            # separable form of the same step: every output label survives from exactly one
            # operand, so out[oA[a] + oB[b]] = sum_k A[aOff[a] + kA[k]] * B[bOff[b] + kB[k]] with
            # a / b enumerating A's / B's surviving labels -- a GEMM the CTA executor runs with
            # register tiles (csrc/executor.cuh, tiled_step)
            gemm_off = gemm_m = gemm_n = 0
            if not select and float(nd.size) * k_n >= GEMM_MIN_MACS:
                ost = dict(zip(out_labels, _row_major_strides(odims)))
                lab_a = [lb for lb in out_labels if lb in sa]
                lab_b = [lb for lb in out_labels if lb not in sa]
                if all(lb in sb for lb in lab_b) and not any(lb in sb for lb in lab_a):
                    a_off = _offsets([dim_of[lb] for lb in lab_a], [sa[lb] for lb in lab_a])
                    b_off = _offsets([dim_of[lb] for lb in lab_b], [sb[lb] for lb in lab_b])
                    o_a = _offsets([dim_of[lb] for lb in lab_a], [ost[lb] for lb in lab_a])
                    o_b = _offsets([dim_of[lb] for lb in lab_b], [ost[lb] for lb in lab_b])
                    gemm_m, gemm_n = a_off.size, b_off.size
                    gemm_off = tab_off + int(sum(part.size for part in parts))
                    parts += [a_off, b_off, o_a, o_b]
            words = np.concatenate(parts).astype(np.uint32)
            tables.append(words)
            # memo words: where the operands' variant-0 values live and which steps produce them
            deps = 0
            memo_words = []
            for base in (base_a, base_b):
                if base in step_index:
                    memo_words.append((memo_off[base], step_index[base]))
                    deps |= step_sites[step_index[base]]
                else:
                    memo_words.append((0, MEMO_NONE))
                    if base < n_leaves and operands[base].sel_kind == SEL_KRAUS:
                        deps |= 1 << operands[base].sel_arg
            is_always = o_kind == 1 or nid == root
            if is_always:
                conj_flags |= 16
                always_steps.append(len(step_rows))
            # operand offsets that do not depend on the output index (a fully contracted operand, e.g.
            # the vector of a vector-matrix step): the lane interpreter loads it once per step
            if not select and not lo_a.any() and not hi_a.any():
                conj_flags |= 32
            if not select and not lo_b.any() and not hi_b.any():
                conj_flags |= 64
            step_index[nid] = len(step_rows)
            memo_off[nid] = memo_top
            step_sites.append(deps)
            step_rows.append(
                [a_kind, a_ref, b_kind, b_ref, o_kind, o_ref, nd.size, k_n, lo_n, hi_n, tab_off, conj_flags,
                 memo_words[0][0], memo_words[1][0], memo_words[0][1] | (memo_words[1][1] << 16), memo_top,
                 gemm_off, gemm_m, gemm_n, 0]
            )
            memo_top += (nd.size + 3) & ~3
            tab_off += words.size
            flops += float(nd.size) if select else float(nd.size) * k_n
            if nid == root:
                result_kind, result_ref = (2 + p, o_ref) if o_kind == 1 else (0, o_ref)
        if p == top and proj is not None:
            result_kind, result_ref = 3, rec_off[proj[1]]
        if p == top and root < n_leaves:
            # single-operand network: the "result" is the leaf itself
            result_kind, result_ref = ref_of(root)
            if tuple(open_order) != tuple(rootn.labels):
                raise CapacityError("single-operand network with permuted open legs")
        memo_elems, memo_ptr, memo_idx = 0, None, None
        uses_prefix = any(row[11] & (4 | 8) for row in step_rows) or any(lf[2] == SEL_PREFIX for lf in prog_leaves)
        if (p == 0 and threads > 32 and MEMO_MIN_STEPS <= len(step_rows) < MEMO_NONE and n_sites > 0
                and not uses_prefix):
            rows_per_site: list[list[int]] = [[] for _ in range(n_sites + 1)]
            for k, deps in enumerate(step_sites):
                while deps:
                    low = deps & -deps
                    rows_per_site[low.bit_length() - 1].append(k)
                    deps ^= low
            rows_per_site[n_sites] = always_steps
            memo_ptr = np.zeros(n_sites + 2, dtype=np.uint32)
            memo_ptr[1:] = np.cumsum([len(r) for r in rows_per_site])
            memo_idx = np.asarray([k for r in rows_per_site for k in r], dtype=np.uint32)
            memo_elems = memo_top
        programs.append(
            Program(
                memo_elems=int(memo_elems), memo_ptr=memo_ptr, memo_idx=memo_idx,
                leaves=np.asarray(prog_leaves, dtype=np.uint32).reshape(-1, LEAF_WORDS),
                steps=np.asarray(step_rows, dtype=np.uint32).reshape(-1, STEP_WORDS),
                tables=np.concatenate(tables).astype(np.uint32) if tables else np.zeros(0, np.uint32),
                arena_fast=int(peak_fast),
                arena_spill=int(peak_spill),
                out_elems=int(rec_size[p]) if p < top else int(rootn.size),
                threads=threads,
                level=p + 1,
                result_kind=result_kind if p == top else 0,
                result_ref=result_ref if p == top else 0,
                flops=flops,
                peak_elems=int(peak_fast + peak_spill),
                max_out=int(max_out),
                ext_read_elems=int(sum(ext_reads.values())),
                leaf_read_elems=int(sum(lf[1] for lf in prog_leaves)),
                proj_d=int(nodes[proj[0]].size) if (proj is not None and p == top) else 0,
            )
        )
    return programs, tuple(open_order)


def _relabel(nodes, virt, view, nid, new_labels):
    """Store node `nid` with its labels in the order `new_labels`.  Nodes whose label order is tied
    to it position by position follow: slice views of it (child order minus the sliced label) and
    conjugate twins (mirror labels in the same positions)."""
    old = nodes[nid].labels
    if tuple(new_labels) == tuple(old):
        return
    perm = [old.index(lb) for lb in new_labels]
    dims = nodes[nid].dims
    nodes[nid].labels = tuple(new_labels)
    nodes[nid].dims = tuple(dims[k] for k in perm)
    for v, twin in virt.items():
        if twin == nid:
            _relabel(nodes, virt, view, v, tuple(nodes[v].labels[k] for k in perm))
    for w, (child, lb, _) in view.items():
        if child == nid:
            _relabel(nodes, virt, view, w, tuple(x for x in new_labels if x != lb))


def _depth_first(nodes, mine, rec_off, real_of):
    """Topological order of the nodes of one pass that keeps few intermediates alive: post-order
    over the pass's forest, at every node the operand whose evaluation needs the larger arena first
    (its result then waits alone while the smaller sibling is evaluated).  Record outputs do not
    occupy the arena.  Nodes with several consumers (conjugate twins make the tree a DAG) are
    evaluated at their first use."""
    mine_set = set(mine)

    def deps(nid):
        out = []
        for ch in (nodes[nid].a, nodes[nid].b):
            ch = real_of(ch)
            if ch in mine_set and ch not in out:
                out.append(ch)
        return out

    # need[n]: arena elements the evaluation of n's subtree peaks at; hold[n]: what stays afterwards
    need: dict[int, int] = {}
    order_of: dict[int, list] = {}
    for nid in mine:  # stored-path order is topological
        ds = deps(nid)
        hold = 0 if nid in rec_off else nodes[nid].size
        held = lambda d: 0 if d in rec_off else nodes[d].size
        # evaluating children in order c1, c2: peak = max(need[c1], held(c1) + need[c2], held(c1) + held(c2) + hold)
        ds.sort(key=lambda d: need[d] - held(d), reverse=True)
        peak, carried = 0, 0
        for d in ds:
            peak = max(peak, carried + need[d])
            carried += held(d)
        need[nid] = max(peak, carried + hold)
        order_of[nid] = ds
    consumed = set()
    for nid in mine:
        consumed.update(order_of[nid])
    out: list[int] = []
    seen: set[int] = set()
    for r in mine:
        if r in consumed:
            continue
        stack = [(r, 0)]
        while stack:
            nid, k = stack.pop()
            if nid in seen:
                continue
            ds = order_of[nid]
            if k < len(ds):
                stack.append((nid, k + 1))
                if ds[k] not in seen:
                    stack.append((ds[k], 0))
            else:
                seen.add(nid)
                out.append(nid)
    assert len(out) == len(mine), "depth-first order lost nodes"
    return out


def _place(nodes, mine, rec_off, real_of, fast_cap):
    """Liveness-based placement of the intermediates of one pass.  Buffers go to
    the fast (shared-memory) arena while they fit under `fast_cap`, otherwise to
    the spill arena whose offsets start at fast_cap.  A buffer is released after
    its last consumer inside the pass (a node can feed its parent and, through a
    conjugate twin, the twin's parent).  Returns (offset per node, fast peak,
    spill peak)."""
    fast, spill = _Arena(), _Arena()
    where: dict[int, int] = {}
    in_spill: set[int] = set()
    mine_set = set(mine)
    uses: dict[int, int] = {}
    for nid in mine:
        for ch in (nodes[nid].a, nodes[nid].b):
            ch = real_of(ch)
            uses[ch] = uses.get(ch, 0) + 1
    for nid in mine:
        nd = nodes[nid]
        if nid not in rec_off:
            off = fast.alloc(nd.size, fast_cap)
            if off is None:
                off = spill.alloc(nd.size)
                in_spill.add(nid)
            where[nid] = off
        for ch in (nd.a, nd.b):
            ch = real_of(ch)
            uses[ch] -= 1
            if uses[ch] == 0 and ch in where and ch in mine_set:
                (spill if ch in in_spill else fast).release(where[ch], nodes[ch].size)
    if fast_cap is None:
        return where, fast.top, 0
    for nid in in_spill:
        where[nid] += fast_cap
    return where, (fast_cap if in_spill else fast.top), spill.top


# ---------------------------------------------------------------------------
# constant networks: execute_path / contract_pair on the device
# ---------------------------------------------------------------------------

@dataclass
class ConstantProgram:
    program: Program
    pool: np.ndarray
    out_shape: tuple


def compile_constant_network(net, steps):
    from .tensor import Index

    ops = [
        Operand(labels=t.labels, dims=tuple(ix.dim for ix in t.indices), data=t.data.reshape(1, -1))
        for t in net.operands
    ]
    pool = Pool()
    progs, order = compile_stage(ops, steps, None, 1, pool, 16)
    dims = {}
    for t in net.operands:
        for ix in t.indices:
            dims[ix.label] = ix.dim
    out_indices = [Index(lb, dims[lb]) for lb in order]
    return ConstantProgram(progs[0], pool.finish("complex128"), tuple(ix.dim for ix in out_indices)), out_indices


def compile_pair(a, b):
    from .tensor import TensorNetwork

    class _Loose:  # contract_pair accepts any two tensors; no open/closed bookkeeping needed
        operands = (a, b)

    return compile_constant_network(_Loose, [(0, 1)])


# ---------------------------------------------------------------------------
# ctypes view of a compiled plan
# ---------------------------------------------------------------------------

class ProgramDesc(ctypes.Structure):
    _fields_ = [
        ("n_leaves", ctypes.c_uint32),
        ("n_steps", ctypes.c_uint32),
        ("n_table_words", ctypes.c_uint32),
        ("arena_fast_elems", ctypes.c_uint32),
        ("arena_spill_elems", ctypes.c_uint32),
        ("out_elems", ctypes.c_uint32),
        ("threads_per_item", ctypes.c_uint32),
        ("level", ctypes.c_uint32),
        ("result_kind", ctypes.c_uint32),
        ("result_ref", ctypes.c_uint32),
        ("proj_d", ctypes.c_uint32),
        ("memo_elems", ctypes.c_uint32),
        ("leaves", ctypes.c_void_p),
        ("steps", ctypes.c_void_p),
        ("tables", ctypes.c_void_p),
        ("memo_ptr", ctypes.c_void_p),
        ("memo_idx", ctypes.c_void_p),
        ("n_memo_idx", ctypes.c_uint32),
        ("n_memo_sites", ctypes.c_uint32),
    ]


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_uint32),
        ("n_qubits", ctypes.c_uint32),
        ("n_sites", ctypes.c_uint32),
        ("n_stages", ctypes.c_uint32),
        ("stage_sizes", ctypes.c_void_p),
        ("pool", ctypes.c_void_p),
        ("pool_elems", ctypes.c_uint64),
        ("programs", ctypes.c_void_p),
        ("max_intermediate", ctypes.c_uint64),
        ("site_variants", ctypes.c_void_p),
    ]


@dataclass
class CompiledPlan:
    """Everything `ptsbe_plan_create` needs, kept alive on the Python side."""

    dtype: str
    n_qubits: int
    n_sites: int
    sizes: tuple
    pool: np.ndarray
    programs: list  # stage-major flat list of Program
    max_intermediate: int
    site_variants: Optional[np.ndarray] = None  # [n_sites] u8: variants per gate site (index validation)
    _keep: list = field(default_factory=list)

    def descriptor(self) -> PlanDesc:
        arr = (ProgramDesc * len(self.programs))()
        keep = []
        for k, pr in enumerate(self.programs):
            lv = np.ascontiguousarray(pr.leaves, dtype=np.uint32)
            st = np.ascontiguousarray(pr.steps, dtype=np.uint32)
            tb = np.ascontiguousarray(pr.tables, dtype=np.uint32)
            keep += [lv, st, tb]
            mp = mi = None
            if pr.memo_elems:
                mp = np.ascontiguousarray(pr.memo_ptr, dtype=np.uint32)
                mi = np.ascontiguousarray(pr.memo_idx, dtype=np.uint32)
                keep += [mp, mi]
            arr[k] = ProgramDesc(
                lv.shape[0], st.shape[0], tb.size, pr.arena_fast, pr.arena_spill, pr.out_elems,
                pr.threads, pr.level, pr.result_kind, pr.result_ref, pr.proj_d, pr.memo_elems,
                lv.ctypes.data, st.ctypes.data, tb.ctypes.data,
                mp.ctypes.data if mp is not None else None, mi.ctypes.data if mi is not None else None,
                mi.size if mi is not None else 0, (mp.size - 2) if mp is not None else 0,
            )
        sizes = np.asarray(self.sizes, dtype=np.uint32)
        pool = np.ascontiguousarray(self.pool)
        keep += [arr, sizes, pool]
        sv = None
        if self.site_variants is not None and self.n_sites:
            sv = np.ascontiguousarray(self.site_variants, dtype=np.uint8)
            if sv.size != self.n_sites:
                raise ValueError("site_variants must have one entry per gate site")
            keep.append(sv)
        self._keep = keep
        return PlanDesc(
            0 if self.dtype == "complex64" else 1,
            self.n_qubits,
            self.n_sites,
            len(self.sizes),
            sizes.ctypes.data,
            pool.ctypes.data,
            pool.size,
            ctypes.addressof(arr),
            self.max_intermediate,
            sv.ctypes.data if sv is not None else None,
        )
