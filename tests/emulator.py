"""numpy interpreter of the device program format (include/ptsbe_b200.h,
csrc/executor.cuh) -- TEST INFRASTRUCTURE ONLY.  Lets the CPU suite check the
plan compiler's tables, arena placement and hoist passes against the oracle
without a GPU.  One work item at a time; like `ptsbe_marginals`, the item is
its own ancestor at every level."""

import numpy as np


def run_stage(programs, pool, kraus_row, prefix_bits, dtype=np.complex128, stats=None):
    """programs: the j pass programs of stage j.  Returns the complex result
    record of the marginal pass (length out_elems).  Programs that carry a
    variant-0 memo are run the way the device runs them: the memo is built
    with an all-zero Kraus row, then only the steps above a non-zero site (and
    the always-run steps) are executed, clean operands being read from the
    memo.  `stats` (dict) receives the number of executed / total steps."""
    pool = np.asarray(pool).astype(dtype)
    records = {}
    result = None
    for p, pr in enumerate(programs):
        memo = None
        if pr.memo_elems:
            memo = _build_memo(pr, pool, dtype)
        arena = np.zeros(pr.arena_fast + pr.arena_spill + 1, dtype=dtype)
        rec = np.zeros(max(pr.out_elems, pr.proj_d, 1), dtype=dtype)
        records[p] = rec  # a pass may read back what it already wrote to its own record

        def resolve(kind, ref):
            if kind == 0:
                return arena, ref
            if kind == 1:
                off, size, sk, sa = (int(v) for v in pr.leaves[ref])
                v = 0
                if sk == 1:
                    v = int(kraus_row[sa])
                elif sk == 2:
                    v = int(prefix_bits[sa])
                return pool, off + v * size
            return records[kind - 2], ref

        dirty = run = None
        if memo is not None:
            n_sites = pr.memo_ptr.size - 2
            dirty = np.zeros(len(pr.steps), dtype=bool)
            for site in range(n_sites):
                if int(kraus_row[site]) != 0:
                    dirty[pr.memo_idx[pr.memo_ptr[site]: pr.memo_ptr[site + 1]]] = True
            run = dirty.copy()
            run[pr.memo_idx[pr.memo_ptr[n_sites]: pr.memo_ptr[n_sites + 1]]] = True
            if stats is not None:
                stats["executed"] = stats.get("executed", 0) + int(run.sum())
                stats["total"] = stats.get("total", 0) + len(pr.steps)
        for k, st in enumerate(pr.steps):
            ak, ar, bk, br, ok, orf, out_n, kn, lo_n, hi_n, tab, flags = (int(v) for v in st[:12])
            if memo is not None and not run[k]:
                continue
            if memo is not None and not dirty[k]:
                # always-run step with clean inputs: its value is the memo's
                val = memo[int(st[15]): int(st[15]) + out_n]
                if ok == 0:
                    arena[orf: orf + out_n] = val
                else:
                    rec[orf: orf + out_n] = val
                continue
            t = pr.tables
            loA = t[tab: tab + lo_n].astype(np.int64)
            loB = t[tab + lo_n: tab + 2 * lo_n].astype(np.int64)
            hiA = t[tab + 2 * lo_n: tab + 2 * lo_n + hi_n].astype(np.int64)
            hiB = t[tab + 2 * lo_n + hi_n: tab + 2 * lo_n + 2 * hi_n].astype(np.int64)
            kA = t[tab + 2 * lo_n + 2 * hi_n: tab + 2 * lo_n + 2 * hi_n + kn].astype(np.int64)
            kB = t[tab + 2 * lo_n + 2 * hi_n + kn: tab + 2 * lo_n + 2 * hi_n + 2 * kn].astype(np.int64)
            assert out_n == lo_n * hi_n
            A, a_base = resolve(ak, ar)
            B, b_base = resolve(bk, br)
            if memo is not None:
                pa, pb = int(st[14]) & 0xFFFF, int(st[14]) >> 16
                if pa != 0xFFFF and not dirty[pa]:
                    A, a_base = memo, int(st[12])
                if pb != 0xFFFF and not dirty[pb]:
                    B, b_base = memo, int(st[13])
            if flags & 8:  # slice views: base offsets depend on measured bits
                at = tab + 2 * lo_n + 2 * hi_n + 2 * kn
                na = int(t[at])
                for i in range(na):
                    a_base += int(prefix_bits[int(t[at + 1 + 2 * i])]) * int(t[at + 2 + 2 * i])
                at += 1 + 2 * na
                nb_ = int(t[at])
                for i in range(nb_):
                    b_base += int(prefix_bits[int(t[at + 1 + 2 * i])]) * int(t[at + 2 + 2 * i])
            ia = a_base + (hiA[:, None] + loA[None, :]).reshape(-1)[:, None] + kA[None, :]
            ib = b_base + (hiB[:, None] + loB[None, :]).reshape(-1)[:, None] + kB[None, :]
            va, vb = A[ia], B[ib]
            if flags & 1:
                va = np.conj(va)
            if flags & 2:
                vb = np.conj(vb)
            val = np.sum(va * vb, axis=1)
            if ok == 0:
                assert orf + out_n <= pr.arena_fast + pr.arena_spill
                arena[orf: orf + out_n] = val
            else:
                rec[orf: orf + out_n] = val
        records[p] = rec
        if p == len(programs) - 1:
            if pr.result_kind == 3:  # projection form: result = v . M, M in pass 0's record
                d, n = pr.proj_d, pr.out_elems
                m = records[0][pr.result_ref: pr.result_ref + d * n].reshape(d, n)
                result = rec[:d] @ m
            else:
                src, base = resolve(pr.result_kind, pr.result_ref)
                result = np.array(src[base: base + pr.out_elems])
    return result


def _build_memo(pr, pool, dtype):
    """Variant-0 values of every step of a class-0 program (device: EXEC_MEMO_BUILD)."""
    memo = np.zeros(pr.memo_elems + 1, dtype=dtype)
    for st in pr.steps:
        ak, ar, bk, br, ok, orf, out_n, kn, lo_n, hi_n, tab, flags = (int(v) for v in st[:12])
        assert not flags & (4 | 8), "memo programs have no prefix-dependent steps"
        t = pr.tables
        loA = t[tab: tab + lo_n].astype(np.int64)
        loB = t[tab + lo_n: tab + 2 * lo_n].astype(np.int64)
        hiA = t[tab + 2 * lo_n: tab + 2 * lo_n + hi_n].astype(np.int64)
        hiB = t[tab + 2 * lo_n + hi_n: tab + 2 * lo_n + 2 * hi_n].astype(np.int64)
        kA = t[tab + 2 * lo_n + 2 * hi_n: tab + 2 * lo_n + 2 * hi_n + kn].astype(np.int64)
        kB = t[tab + 2 * lo_n + 2 * hi_n + kn: tab + 2 * lo_n + 2 * hi_n + 2 * kn].astype(np.int64)
        ops = []
        for kind, ref, prod, moff in ((ak, ar, int(st[14]) & 0xFFFF, int(st[12])), (bk, br, int(st[14]) >> 16, int(st[13]))):
            if prod != 0xFFFF:
                ops.append((memo, moff))
            else:
                assert kind == 1, "a memo program reads only leaves and its own steps"
                off, size, sk, sa = (int(v) for v in pr.leaves[ref])
                assert sk != 2
                ops.append((pool, off))  # variant 0
        (A, a_base), (B, b_base) = ops
        ia = a_base + (hiA[:, None] + loA[None, :]).reshape(-1)[:, None] + kA[None, :]
        ib = b_base + (hiB[:, None] + loB[None, :]).reshape(-1)[:, None] + kB[None, :]
        va, vb = A[ia], B[ib]
        if flags & 1:
            va = np.conj(va)
        if flags & 2:
            vb = np.conj(vb)
        memo[int(st[15]): int(st[15]) + out_n] = np.sum(va * vb, axis=1)
    return memo
