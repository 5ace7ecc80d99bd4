"""Correctness and timing probe of the tensor-core projection kernel (csrc/project_tc.cuh) against
numpy float64 and the FP32 FMA kernel (csrc/project.cuh):  python tools/probe_project_tc.py [D N items sets]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_08467_b200 import _capi

def case(D, N, items, sets, reps, seed=0):
    rng = np.random.default_rng(seed)
    v = (rng.standard_normal((items, D)) + 1j * rng.standard_normal((items, D))).astype(np.complex64)
    m = (rng.standard_normal((sets, D, N)) + 1j * rng.standard_normal((sets, D, N))).astype(np.complex64)
    eset = np.sort(rng.integers(0, sets, size=items)).astype(np.uint32)
    want = np.empty((items, N))
    for e in range(sets):
        sel = eset == e
        if sel.any():
            want[sel] = (v[sel].astype(np.complex128) @ m[e].astype(np.complex128)).real
    scale = np.abs(want).max(axis=1, keepdims=True)
    res = {}
    for name, tc in (("fma", False), ("tc", True)):
        got, km, pm = _capi.project_probe(v, m, eset, tc, reps=reps)
        err = float(np.max(np.abs(got - want) / scale))
        res[name] = (err, km, pm)
    flops = 2.0 * items * 2 * D * N
    print(f"D={D} N={N} items={items} sets={sets}: "
          f"fma err {res['fma'][0]:.2e} {res['fma'][1]:.3f} ms ({flops / res['fma'][1] / 1e9:.1f} TFLOP/s) | "
          f"tc err {res['tc'][0]:.2e} {res['tc'][1]:.3f} ms ({flops / res['tc'][1] / 1e9:.1f} TFLOP/s useful, prep {res['tc'][2]:.3f} ms) "
          f"speed-up {res['fma'][1] / res['tc'][1]:.2f}x", flush=True)
    return res

if __name__ == "__main__":
    if len(sys.argv) > 4:
        D, N, items, sets = (int(x) for x in sys.argv[1:5])
        case(D, N, items, sets, reps=5)
    else:
        case(64, 64, 300, 2, reps=1)
        case(64, 64, 5000, 7, reps=1)
        case(16, 32, 1000, 3, reps=1)
        case(40, 128, 3000, 5, reps=1)
        case(64, 256, 4000, 3, reps=1)
        for N in (64, 128, 256):
            case(64, N, 1 << 20, 2048, reps=5)
