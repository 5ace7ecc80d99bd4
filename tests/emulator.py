"""numpy interpreter of the device program format (include/ptsbe_b200.h,
csrc/executor.cuh) -- TEST INFRASTRUCTURE ONLY.  Lets the CPU suite check the
plan compiler's tables, arena placement and hoist passes against the oracle
without a GPU.  One work item at a time; like `ptsbe_marginals`, the item is
its own ancestor at every level."""

import numpy as np


def run_stage(programs, pool, kraus_row, prefix_bits, dtype=np.complex128):
    """programs: the j pass programs of stage j.  Returns the complex result
    record of the marginal pass (length out_elems)."""
    pool = np.asarray(pool).astype(dtype)
    records = {}
    result = None
    for p, pr in enumerate(programs):
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

        for st in pr.steps:
            ak, ar, bk, br, ok, orf, out_n, kn, lo_n, hi_n, tab, flags = (int(v) for v in st)
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
