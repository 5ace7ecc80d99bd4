"""ctypes binding of libptsbe_b200.so (include/ptsbe_b200.h).

This is the whole Python<->CUDA boundary: plain pointers and sizes, no torch
types.  The library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_2604_08467_b200/csrc`).  There is no CPU fallback: if the
library is missing or no CUDA device is present, compute calls raise
`DeviceError`.
"""

from __future__ import annotations

import ctypes
import os
import weakref
from typing import Optional

import numpy as np

from .compiler import CompiledPlan, ConstantProgram, PlanDesc
from .errors import STATUS_TO_ERROR, DeviceError

LIB_NAME = "libptsbe_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
MAX_STAGES = 64

EXPORTS = (
    "ptsbe_last_error", "ptsbe_device_count", "ptsbe_version", "ptsbe_plan_create",
    "ptsbe_plan_destroy", "ptsbe_marginals", "ptsbe_execute_raw", "ptsbe_sample_stage",
    "ptsbe_sample", "ptsbe_batch_upload", "ptsbe_batch_run", "ptsbe_batch_fetch",
    "ptsbe_batch_destroy", "ptsbe_histogram_merge", "ptsbe_plan_greedy", "ptsbe_free",
    "ptsbe_batch_histogram_dev", "ptsbe_histogram_merge_dev", "ptsbe_free_dev",
    "ptsbe_measure_fma_peak", "ptsbe_sample_nonproportional", "ptsbe_batch_presample", "ptsbe_batch_kraus",
    "ptsbe_plan_set_stage_samplers", "ptsbe_project_probe", "ptsbe_sample_packed",
)


class RunStats(ctypes.Structure):
    _fields_ = [
        ("stage_events", ctypes.c_uint64 * MAX_STAGES),
        ("stage_ms", ctypes.c_float * MAX_STAGES),
        ("gpu_launches", ctypes.c_uint64),
        ("total_shots", ctypes.c_uint64),
        ("n_records", ctypes.c_uint64),
        ("loop_ms", ctypes.c_float),
        ("h2d_ms", ctypes.c_float),
        ("d2h_ms", ctypes.c_float),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
        ("n_chunks", ctypes.c_uint32),
        ("flagged_sets", ctypes.c_uint32),
        ("first_flagged_id", ctypes.c_int64),
        ("first_flag_kind", ctypes.c_uint32),
        ("first_flag_stage", ctypes.c_uint32),
        ("hoist_ms", ctypes.c_float * MAX_STAGES),
        ("marg_ms", ctypes.c_float * MAX_STAGES),
        ("project_ms", ctypes.c_float * MAX_STAGES),
        ("sampler_ms", ctypes.c_float * MAX_STAGES),
        ("compact_ms", ctypes.c_float * MAX_STAGES),
        ("histogram_ms", ctypes.c_float),
        ("marg_launches", ctypes.c_uint32 * MAX_STAGES),
        ("descent_ms", ctypes.c_float * MAX_STAGES),
        ("descent_items", ctypes.c_uint64 * MAX_STAGES),
    ]


_lib = None


def load() -> ctypes.CDLL:
    """dlopen the in-tree library; loud failure when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - depends on the box
        raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
    P, U64, U32, I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
    lib.ptsbe_last_error.restype = ctypes.c_char_p
    lib.ptsbe_version.restype = ctypes.c_char_p
    lib.ptsbe_device_count.restype = I
    lib.ptsbe_plan_create.argtypes = [ctypes.POINTER(PlanDesc), I, ctypes.POINTER(P)]
    lib.ptsbe_plan_destroy.argtypes = [P]
    lib.ptsbe_plan_destroy.restype = None
    lib.ptsbe_plan_set_stage_samplers.argtypes = [P, P, U32]
    lib.ptsbe_marginals.argtypes = [P, U32, P, P, U64, P, P, P]
    lib.ptsbe_execute_raw.argtypes = [P, P]
    lib.ptsbe_sample_stage.argtypes = [U32, U32, U64, U64, P, P, P, P,
                                       ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P),
                                       ctypes.POINTER(U64), I]
    lib.ptsbe_sample.argtypes = [P, P, P, P, U64, U64, I, ctypes.POINTER(P), ctypes.POINTER(P),
                                 ctypes.POINTER(P), ctypes.POINTER(U64), ctypes.POINTER(RunStats)]
    lib.ptsbe_sample_packed.argtypes = [P, P, P, P, U64, U64, ctypes.POINTER(P), ctypes.POINTER(U64),
                                        ctypes.POINTER(RunStats)]
    lib.ptsbe_sample_nonproportional.argtypes = [P, P, P, U64, U64, U32, U32, ctypes.c_double, U32,
                                                 ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P),
                                                 ctypes.POINTER(P), ctypes.POINTER(U64), ctypes.POINTER(RunStats)]
    lib.ptsbe_batch_upload.argtypes = [P, P, P, P, U64, ctypes.POINTER(P)]
    lib.ptsbe_batch_presample.argtypes = [P, P, P, U64, U32, U32, U64, ctypes.POINTER(P)]
    lib.ptsbe_batch_kraus.argtypes = [P, P]
    lib.ptsbe_batch_run.argtypes = [P, U64, ctypes.POINTER(U64), ctypes.POINTER(RunStats)]
    lib.ptsbe_batch_fetch.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(U64)]
    lib.ptsbe_batch_destroy.argtypes = [P]
    lib.ptsbe_batch_destroy.restype = None
    lib.ptsbe_histogram_merge.argtypes = [P, P, U64, U32, ctypes.POINTER(P), ctypes.POINTER(P),
                                          ctypes.POINTER(U64), I]
    lib.ptsbe_plan_greedy.argtypes = [U32, P, P, P, P, P, P, P, U32, U32, U64, ctypes.c_double, P,
                                      ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    lib.ptsbe_free.argtypes = [P]
    lib.ptsbe_free.restype = None
    lib.ptsbe_batch_histogram_dev.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(U64)]
    lib.ptsbe_histogram_merge_dev.argtypes = [P, P, U64, U32, I, ctypes.POINTER(P), ctypes.POINTER(P),
                                              ctypes.POINTER(U64)]
    lib.ptsbe_free_dev.argtypes = [P]
    lib.ptsbe_free_dev.restype = None
    lib.ptsbe_measure_fma_peak.argtypes = [I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    lib.ptsbe_project_probe.argtypes = [I, U32, U32, U64, U32, P, P, P, I, P, I,
                                        ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
    _lib = lib
    return lib


def device_count() -> int:
    return int(load().ptsbe_device_count())


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().ptsbe_last_error().decode("utf-8", "replace")
    raise STATUS_TO_ERROR.get(rc, DeviceError)(msg)


def _release_owned(self):
    addr = ctypes.addressof(self)
    if addr and _lib is not None:
        _lib.ptsbe_free(ctypes.c_void_p(addr))


def _owned_buffer(addr: int, nbytes: int):
    """ctypes view of one library-allocated host array that calls ptsbe_free()
    when its last numpy view goes away (large histograms are page-locked
    buffers the library recycles, so they are wrapped, not copied)."""
    cls = type("_LibBuffer", (ctypes.c_char * nbytes,), {"__del__": _release_owned})
    return cls.from_address(addr)


_COPY_BELOW = 1 << 20


def _take(ptr: ctypes.c_void_p, count: int, dtype) -> np.ndarray:
    """Library-allocated array -> numpy: small arrays are copied and released,
    large ones are wrapped zero-copy and released with their last view."""
    lib = load()
    if not ptr.value:
        return np.zeros(0, dtype=dtype)
    n = int(count)
    nbytes = n * np.dtype(dtype).itemsize
    if nbytes < _COPY_BELOW:
        buf = (ctypes.c_char * nbytes).from_address(ptr.value)
        out = np.frombuffer(buf, dtype=dtype, count=n).copy()
        lib.ptsbe_free(ptr)
        return out
    return np.frombuffer(_owned_buffer(ptr.value, nbytes), dtype=dtype, count=n)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


class DeviceArray:
    """A u64 device buffer owned by the library (or borrowed from a batch),
    exported through `__cuda_array_interface__` so torch can wrap it without a
    copy: `torch.as_tensor(arr, device="cuda")`."""

    def __init__(self, ptr: int, shape: tuple, owner=None, owned: bool = False):
        self.ptr, self.shape, self._owner, self._owned = int(ptr or 0), tuple(shape), owner, owned

    @property
    def __cuda_array_interface__(self):
        return {"shape": self.shape, "typestr": "<u8", "data": (self.ptr, False), "version": 2}

    def free(self):
        if self._owned and self.ptr:
            load().ptsbe_free_dev(self.ptr)
        self.ptr, self._owned = 0, False

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class ResidentBatch:
    """Error sets uploaded once; each `run` leaves its histogram in HBM."""

    def __init__(self, plan: "DevicePlan", kraus_idx, shots, eset_ids):
        self.plan = plan
        self._h = ctypes.c_void_p()
        plan._batches.add(self)  # the C batch holds a raw plan pointer: the plan closes us before it dies
        if kraus_idx is None:  # filled in by DevicePlan.presample
            return
        kraus_idx, shots, ids = plan._check_inputs(kraus_idx, shots, eset_ids)
        check(load().ptsbe_batch_upload(plan._h, _ptr(kraus_idx), _ptr(shots), _ptr(ids),
                                        shots.size, ctypes.byref(self._h)))

    def _live(self):
        if not self._h:
            raise DeviceError("this resident batch was closed (with its plan)")
        return self._h

    def run(self, seed: int) -> tuple[int, RunStats]:
        st = RunStats()
        n = ctypes.c_uint64()
        check(load().ptsbe_batch_run(self._live(), seed & (2**64 - 1), ctypes.byref(n), ctypes.byref(st)))
        return int(n.value), st

    def kraus(self, n_sets: int, g: int) -> np.ndarray:
        """Kraus-index matrix [n_sets, g] of this batch (device-side pre-sampling: what was drawn)."""
        out = np.empty((n_sets, g), dtype=np.uint8)
        check(load().ptsbe_batch_kraus(self._live(), _ptr(out)))
        return out

    def fetch(self) -> tuple[np.ndarray, np.ndarray]:
        k, c, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
        check(load().ptsbe_batch_fetch(self._live(), ctypes.byref(k), ctypes.byref(c), ctypes.byref(n)))
        w = self.plan.words
        return _take(k, n.value * w, np.uint64).reshape(-1, w), _take(c, n.value, np.uint64)

    def histogram_dev(self) -> tuple["DeviceArray", "DeviceArray"]:
        """Histogram of the last run as borrowed device buffers (keys [R, words],
        counts [R]); valid until the next run or close()."""
        k, c, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
        check(load().ptsbe_batch_histogram_dev(self._live(), ctypes.byref(k), ctypes.byref(c), ctypes.byref(n)))
        return (DeviceArray(k.value, (n.value, self.plan.words), owner=self),
                DeviceArray(c.value, (n.value,), owner=self))

    def close(self):
        if self._h:
            load().ptsbe_batch_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DevicePlan:
    """Owner of a `ptsbe_plan*`."""

    def __init__(self, compiled: CompiledPlan, device: int = 0):
        lib = load()
        self.compiled = compiled
        self.words = max(1, (compiled.n_qubits + 63) // 64)
        self.n_sites = compiled.n_sites
        self._h = ctypes.c_void_p()
        self._batches = weakref.WeakSet()
        desc = compiled.descriptor()
        check(lib.ptsbe_plan_create(ctypes.byref(desc), device, ctypes.byref(self._h)))

    def close(self):
        if self._h:
            # batches first: ptsbe_batch_destroy dereferences its plan (stream, workspace cache, mutex)
            for bt in list(self._batches):
                bt.close()
            load().ptsbe_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stage_samplers(self, kinds) -> None:
        """Fix the sampler of every stage: 0 flat, 1 per-qubit descent, -1 per-chunk choice."""
        kinds = np.ascontiguousarray(kinds, dtype=np.int32)
        check(load().ptsbe_plan_set_stage_samplers(self._h, _ptr(kinds), kinds.size))

    def _check_inputs(self, kraus_idx, shots, eset_ids):
        """Shapes and dtypes of the flat arrays the C ABI copies from (it trusts its sizes)."""
        if not self._h:
            raise DeviceError("this device plan was closed")
        kraus_idx = np.ascontiguousarray(kraus_idx, dtype=np.uint8)
        if kraus_idx.ndim != 2 or kraus_idx.shape[1] != self.n_sites:
            raise ValueError(f"kraus_idx must be [n_sets, {self.n_sites}] (one column per gate site), "
                             f"got {kraus_idx.shape}")
        n_sets = kraus_idx.shape[0]
        if shots is not None:
            shots = np.ascontiguousarray(shots, dtype=np.uint32)
            if shots.shape != (n_sets,):
                raise ValueError(f"shots must have one entry per error set ({n_sets}), got shape {shots.shape}")
        ids = None
        if eset_ids is not None:
            ids = np.ascontiguousarray(eset_ids, dtype=np.uint32)
            if ids.shape != (n_sets,):
                raise ValueError(f"eset_ids must have one entry per error set ({n_sets}), got shape {ids.shape}")
        return kraus_idx, shots, ids

    def marginals(self, stage: int, kraus_idx: np.ndarray, prefixes: np.ndarray):
        """(probs [W, 2^b] float64 unnormalised+clamped, mass [W], min [W])."""
        kraus_idx, _, _ = self._check_inputs(kraus_idx, None, None)
        w = kraus_idx.shape[0]
        prefixes = np.ascontiguousarray(prefixes, dtype=np.uint64)
        if prefixes.size != w * self.words:
            raise ValueError(f"prefixes must be [{w}, {self.words}] u64, got {prefixes.shape}")
        prefixes = prefixes.reshape(w, self.words)
        nb = 1 << self.compiled.sizes[stage - 1]
        probs = np.empty((w, nb), dtype=np.float64)
        mass = np.empty(w, dtype=np.float64)
        mn = np.empty(w, dtype=np.float64)
        check(load().ptsbe_marginals(self._h, stage, _ptr(kraus_idx), _ptr(prefixes), w,
                                     _ptr(probs), _ptr(mass), _ptr(mn)))
        return probs, mass, mn

    def execute_raw(self, out: np.ndarray) -> None:
        check(load().ptsbe_execute_raw(self._h, _ptr(out)))

    def sample(self, kraus_idx, shots, eset_ids, seed: int, merged: bool = True):
        """Host-buffer entry point: returns (keys [R, words] u64, eset [R] or None,
        counts [R] u64, RunStats)."""
        kraus_idx, shots, ids = self._check_inputs(kraus_idx, shots, eset_ids)
        k, e, c, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
        st = RunStats()
        check(load().ptsbe_sample(self._h, _ptr(kraus_idx), _ptr(shots), _ptr(ids), shots.size,
                                  seed & (2**64 - 1), 1 if merged else 0, ctypes.byref(k),
                                  ctypes.byref(e), ctypes.byref(c), ctypes.byref(n), ctypes.byref(st)))
        keys = _take(k, n.value * self.words, np.uint64).reshape(-1, self.words)
        counts = _take(c, n.value, np.uint64)
        esets = None if merged else _take(e, n.value, np.uint32)
        return keys, esets, counts, st

    def sample_packed(self, kraus_idx, shots, eset_ids, seed: int):
        """`sample(merged=True)` with the histogram as one [R, 2] uint32 array of (key, count) rows
        (ptsbe_sample_packed: at most 32 measured qubits, fewer than 2^32 shots per call): half the
        device-to-host bytes; key = high half of `sample`'s key word (qubit q at bit 31 - q).
        Returns (records, RunStats)."""
        kraus_idx, shots, ids = self._check_inputs(kraus_idx, shots, eset_ids)
        r, n = ctypes.c_void_p(), ctypes.c_uint64()
        st = RunStats()
        check(load().ptsbe_sample_packed(self._h, _ptr(kraus_idx), _ptr(shots), _ptr(ids), shots.size,
                                         seed & (2**64 - 1), ctypes.byref(r), ctypes.byref(n), ctypes.byref(st)))
        return _take(r, n.value * 2, np.uint32).reshape(-1, 2), st

    def sample_nonproportional(self, kraus_idx, eset_ids, seed: int, nonfinal_shots: int, final_mode: str,
                               threshold: float, direct_count: int):
        """Non-proportional sampling (engine.py:527-576) of every error set in one device run:
        returns (keys [R, words] u64, eset position [R], counts [R], probs [R] or None, RunStats)."""
        kraus_idx, _, ids = self._check_inputs(kraus_idx, None, eset_ids)
        if final_mode not in ("exhaustive", "direct"):
            raise ValueError(f"final_mode must be 'exhaustive' or 'direct', got {final_mode!r}")
        k, e, c, pr, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
        st = RunStats()
        check(load().ptsbe_sample_nonproportional(
            self._h, _ptr(kraus_idx), _ptr(ids), kraus_idx.shape[0], seed & (2**64 - 1), int(nonfinal_shots),
            0 if final_mode == "exhaustive" else 1, float(threshold), int(direct_count),
            ctypes.byref(k), ctypes.byref(e), ctypes.byref(c), ctypes.byref(pr), ctypes.byref(n), ctypes.byref(st)))
        keys = _take(k, n.value * self.words, np.uint64).reshape(-1, self.words)
        esets = _take(e, n.value, np.uint32)
        counts = _take(c, n.value, np.uint64)
        probs = _take(pr, n.value, np.float64)
        return keys, esets, counts, (probs if final_mode == "exhaustive" else None), st

    def presample(self, site_probs, n_sets: int, first_id: int, shots_per_set: int, seed: int) -> ResidentBatch:
        """Resident batch whose error sets [first_id, first_id + n_sets) are drawn on the device from
        the per-site outcome probabilities `site_probs` (list of sequences, outcome 0 = no error)."""
        off = np.zeros(len(site_probs) + 1, dtype=np.uint32)
        off[1:] = np.cumsum([len(p) for p in site_probs])
        cdf = np.concatenate([np.cumsum(np.asarray(p, dtype=np.float64)) for p in site_probs]) if len(site_probs) \
            else np.zeros(0, np.float64)
        bt = ResidentBatch(self, None, None, None)
        check(load().ptsbe_batch_presample(self._h, _ptr(np.ascontiguousarray(cdf)), _ptr(off), int(n_sets),
                                           int(first_id), int(shots_per_set), seed & (2**64 - 1), ctypes.byref(bt._h)))
        return bt

    def upload(self, kraus_idx, shots, eset_ids=None) -> ResidentBatch:
        return ResidentBatch(self, kraus_idx, shots, eset_ids)


def run_constant_program(cp: ConstantProgram) -> np.ndarray:
    """Execute a constant one-item program (tensor.execute_path on the device)."""
    compiled = CompiledPlan(dtype="complex128", n_qubits=1, n_sites=0, sizes=(1,), pool=cp.pool,
                            programs=[cp.program], max_intermediate=0)
    plan = DevicePlan(compiled)
    try:
        out = np.empty(max(cp.program.out_elems, 1), dtype=np.complex128)
        plan.execute_raw(out)
    finally:
        plan.close()
    return out[: cp.program.out_elems].reshape(cp.out_shape)


def sample_stage(b: int, stage: int, seed: int, probs, mult, eset_id, rank, device: int = 0):
    """Sampler-only probe (ptsbe_sample_stage): children as (item, index, count)."""
    probs = np.ascontiguousarray(probs, dtype=np.float64).reshape(-1, 1 << b)
    w = probs.shape[0]
    mult = np.ascontiguousarray(mult, dtype=np.uint32)
    eset_id = np.ascontiguousarray(eset_id, dtype=np.uint32)
    rank = np.ascontiguousarray(rank, dtype=np.uint32)
    ci, cx, cc, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
    check(load().ptsbe_sample_stage(b, stage, seed & (2**64 - 1), w, _ptr(probs), _ptr(mult),
                                    _ptr(eset_id), _ptr(rank), ctypes.byref(ci), ctypes.byref(cx),
                                    ctypes.byref(cc), ctypes.byref(n), device))
    return _take(ci, n.value, np.uint32), _take(cx, n.value, np.uint32), _take(cc, n.value, np.uint32)


def histogram_merge(keys, counts, device: int = 0):
    """Device sort + reduce-by-key of (key, count) records (merge_records)."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    if keys.ndim == 1:
        keys = keys.reshape(-1, 1)
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    ok, oc, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
    check(load().ptsbe_histogram_merge(_ptr(keys), _ptr(counts), counts.size, keys.shape[1],
                                       ctypes.byref(ok), ctypes.byref(oc), ctypes.byref(n), device))
    w = keys.shape[1]
    return _take(ok, n.value * w, np.uint64).reshape(-1, w), _take(oc, n.value, np.uint64)


def histogram_merge_dev(keys_ptr: int, counts_ptr: int, n: int, words: int, device: int = 0):
    """Device-pointer form of `histogram_merge`: returns owned DeviceArrays."""
    ok, oc, m = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
    check(load().ptsbe_histogram_merge_dev(keys_ptr, counts_ptr, n, words, device, ctypes.byref(ok),
                                           ctypes.byref(oc), ctypes.byref(m)))
    return (DeviceArray(ok.value, (m.value, words), owned=True), DeviceArray(oc.value, (m.value,), owned=True))


def project_probe(v: np.ndarray, m: np.ndarray, eset: np.ndarray, use_tc: bool, reps: int = 1, device: int = 0):
    """Dense projection step on raw complex64 arrays (ptsbe_project_probe): v [items, D], m [sets, D, N],
    eset [items] sorted rows into m.  Returns (P [items, N] float32, kernel ms per launch, B-image prep ms)."""
    v = np.ascontiguousarray(v, dtype=np.complex64)
    m = np.ascontiguousarray(m, dtype=np.complex64)
    eset = np.ascontiguousarray(eset, dtype=np.uint32)
    n, d = v.shape
    sets, d2, nn = m.shape
    if d2 != d or eset.shape != (n,) or (n and int(eset.max()) >= sets):
        raise ValueError("inconsistent shapes for the projection probe")
    out = np.empty((n, nn), dtype=np.float32)
    km, pm = ctypes.c_float(), ctypes.c_float()
    check(load().ptsbe_project_probe(device, d, nn, n, sets, _ptr(eset), _ptr(v), _ptr(m), 1 if use_tc else 0,
                                     _ptr(out), int(reps), ctypes.byref(km), ctypes.byref(pm)))
    return out, float(km.value), float(pm.value)


def measure_fma_peak(device: int = 0) -> tuple:
    """(fp32, fp64) sustained non-tensor FMA TFLOP/s of the device."""
    a, b = ctypes.c_double(), ctypes.c_double()
    check(load().ptsbe_measure_fma_peak(device, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def plan_greedy(op_labels, op_dims, op_class=None, class_weight=None, hypersamples=100,
                seed=0, size_cap_log2=0.0, class_cap_log2=None, op_unit=None):
    """Host planner core (csrc/planner.cpp).  Returns (merges [(x, y)...] over
    stable operand ids, weighted cost, reference flop estimate)."""
    n = len(op_labels)
    ptr = np.zeros(n + 1, dtype=np.uint32)
    for k, lb in enumerate(op_labels):
        ptr[k + 1] = ptr[k] + len(lb)
    labels = np.asarray([l for lb in op_labels for l in lb], dtype=np.int64)
    dims = np.asarray([d for ds in op_dims for d in ds], dtype=np.uint32)
    cls = None if op_class is None else np.ascontiguousarray(op_class, dtype=np.uint32)
    cw = None if class_weight is None else np.ascontiguousarray(class_weight, dtype=np.float64)
    cc = None if class_cap_log2 is None else np.ascontiguousarray(class_cap_log2, dtype=np.float64)
    if cc is not None and (cw is None or cc.size != cw.size):
        raise ValueError("class_cap_log2 needs class_weight of the same length")
    un = None if op_unit is None else np.ascontiguousarray(op_unit, dtype=np.uint8)
    merges = np.zeros(2 * max(n - 1, 1), dtype=np.uint32)
    cost, flops = ctypes.c_double(), ctypes.c_double()
    check(load().ptsbe_plan_greedy(n, _ptr(ptr), _ptr(labels), _ptr(dims), _ptr(cls), _ptr(cw), _ptr(cc), _ptr(un),
                                   0 if cw is None else cw.size, hypersamples, seed & (2**64 - 1),
                                   float(size_cap_log2), _ptr(merges), ctypes.byref(cost),
                                   ctypes.byref(flops)))
    return merges[: 2 * (n - 1)].reshape(-1, 2), cost.value, flops.value
