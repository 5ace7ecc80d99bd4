"""Synthetic workloads of BASELINE.json's five configs.

Each builder returns (Circuit, BatchPlan sizes) for the full-size config and
accepts smaller parameters for parity tests (n <= 20 twins that the statevector
oracle can check).  Error sets are drawn by `presample_matrix`: a vectorised
pre-trajectory sampler that yields the uint8 Kraus-index matrix the device
consumes (index = position in `NoiseChannel.outcomes()`); at E = 10^5..10^6 the
per-site Python loop of `presample_errors` would dominate the run.
"""

from __future__ import annotations

import math

import numpy as np

from .circuits import Circuit, Gate, NoiseChannel
from .engine import ErrorSet


def ghz(n: int = 12, p: float = 0.01) -> tuple:
    """cfg1: H(0), CX(q, q+1); single-qubit depolarizing p on the H site,
    two-qubit depolarizing p on the CX sites (the reference's channel kinds, so
    the unmodified CPU reference runs it)."""
    gates = [Gate("H", (0,), None, NoiseChannel("depolarizing1", p))]
    gates += [Gate("CX", (q, q + 1), None, NoiseChannel("depolarizing", p)) for q in range(n - 1)]
    return Circuit(n, tuple(gates)), _even(n, 4)


def hea(n: int = 30, depth: int = 6, gamma: float = 0.01, p: float = 0.01, seed: int = 2) -> tuple:
    """cfg2: hardware-efficient ansatz.  Per layer Ry, Rz on every qubit with
    angles ~ U[0, 2pi), then a brick ladder of CX on (q, q+1), q = layer (mod 2);
    amplitude damping gamma on the rotation sites, two-qubit depolarizing p on
    the CX sites."""
    rng = np.random.default_rng(seed)
    gates = []
    for layer in range(depth):
        for q in range(n):
            gates.append(Gate("Ry", (q,), float(rng.uniform(0, 2 * math.pi)), NoiseChannel("amplitude_damping", gamma)))
            gates.append(Gate("Rz", (q,), float(rng.uniform(0, 2 * math.pi)), NoiseChannel("amplitude_damping", gamma)))
        for q in range(layer % 2, n - 1, 2):
            gates.append(Gate("CX", (q, q + 1), None, NoiseChannel("depolarizing", p)))
    return Circuit(n, tuple(gates)), _even(n, 10)


def surface_code(d: int = 5, rounds: int = 3, p: float = 1e-3, order: str = "data_first", batch: int = 8) -> tuple:
    """cfg3: rotated surface code memory-Z experiment, circuit-level noise,
    deferred measurement with a fresh ancilla per stabiliser per round:
    n = d^2 + rounds * (d^2 - 1) qubits.  X-type ancillas: H, 4 (or 2) CX
    ancilla->data, H; Z-type: CX data->ancilla.  Two-qubit depolarizing p after
    every CX, single-qubit depolarizing p after every H.

    order="data_first" (the golden twins): data qubits 0..d^2-1, then ancillas
    round by round, batches of `batch` qubits.  order="ancilla_first" (SURVEY
    8d: per-round ancilla blocks, data last): round-1 ancillas, round-2
    ancillas, ..., data; batches never straddle a round, so the unitary light
    cone of the stages of round r stops at round r."""
    data = {(r, c): r * d + c for r in range(d) for c in range(d)}
    stabs = []  # (type, [data qubits])
    for r in range(-1, d):
        for c in range(-1, d):
            cells = [(r + dr, c + dc) for dr in (0, 1) for dc in (0, 1)]
            members = [data[x] for x in cells if x in data]
            kind = "X" if (r + c) % 2 == 0 else "Z"
            if len(members) == 4:
                stabs.append((kind, members))
            elif len(members) == 2:
                # boundary stabilisers of the rotated code: X on top/bottom, Z on left/right
                on_row_edge = r in (-1, d - 1)
                if (kind == "X" and on_row_edge) or (kind == "Z" and not on_row_edge):
                    stabs.append((kind, members))
    assert len(stabs) == d * d - 1, len(stabs)
    n = d * d + rounds * len(stabs)
    gates = []
    nxt = d * d
    for _ in range(rounds):
        for kind, members in stabs:
            anc = nxt
            nxt += 1
            if kind == "X":
                gates.append(Gate("H", (anc,), None, NoiseChannel("depolarizing1", p)))
                for q in members:
                    gates.append(Gate("CX", (anc, q), None, NoiseChannel("depolarizing", p)))
                gates.append(Gate("H", (anc,), None, NoiseChannel("depolarizing1", p)))
            else:
                for q in members:
                    gates.append(Gate("CX", (q, anc), None, NoiseChannel("depolarizing", p)))
    if order == "data_first":
        return Circuit(n, tuple(gates)), _even(n, batch)
    if order != "ancilla_first":
        raise ValueError(f"unknown qubit order {order!r}")
    n_data, n_anc = d * d, len(stabs)
    pos = {q: rounds * n_anc + q for q in range(n_data)}
    pos.update({n_data + k: k for k in range(rounds * n_anc)})
    gates = [Gate(g.kind, tuple(pos[q] for q in g.targets), g.angle, g.noise) for g in gates]
    sizes = []
    for block in [n_anc] * rounds + [n_data]:
        sizes += list(_even(block, batch))
    return Circuit(n, tuple(gates)), tuple(sizes)


def qaoa(n: int = 50, layers: int = 2, p: float = 1e-3, seed: int = 4) -> tuple:
    """cfg4: QAOA MaxCut on a random 3-regular graph (pairing model, multi-edges
    and loops rejected): H on every qubit, per layer RZZ(gamma_l) on every edge
    then Rx(beta_l) on every qubit; two-qubit depolarizing p on the RZZ sites."""
    rng = np.random.default_rng(seed)
    edges = _three_regular(n, rng)
    quiet = NoiseChannel("X", 0.0)
    gates = [Gate("H", (q,), None, quiet) for q in range(n)]
    for _ in range(layers):
        gam, beta = float(rng.uniform(0, math.pi)), float(rng.uniform(0, math.pi))
        for a, b in edges:
            gates.append(Gate("RZZ", (a, b), gam, NoiseChannel("depolarizing", p)))
        for q in range(n):
            gates.append(Gate("Rx", (q,), beta, quiet))
    return Circuit(n, tuple(gates)), _even(n, 10)


def random40(n: int = 40, g: int = 400, seed: int = 5) -> tuple:
    """cfg5: the reference's own random_circuit(40, 400) (depth ~ g/n = 10)."""
    from .circuits import random_circuit

    return random_circuit(n, g, 0.2, (0.02, 0.2), np.random.default_rng(seed)), _even(n, 10)


def _even(n: int, b: int) -> tuple:
    f = max(1, math.ceil(n / b))
    return tuple([b] * (f - 1) + [n - b * (f - 1)])


def _three_regular(n: int, rng) -> list:
    if n % 2 or n < 4:
        raise ValueError("3-regular graph needs an even number of >= 4 vertices")
    while True:
        stubs = np.repeat(np.arange(n), 3)
        rng.shuffle(stubs)
        pairs = stubs.reshape(-1, 2)
        if np.any(pairs[:, 0] == pairs[:, 1]):
            continue
        edges = {tuple(sorted(map(int, e))) for e in pairs}
        if len(edges) == pairs.shape[0]:
            return sorted(edges)


def presample_matrix(c: Circuit, e: int, rng: np.random.Generator) -> np.ndarray:
    """uint8 [e, g]: Kraus index of every site for e pre-sampled error sets
    (0 = no error).  Same distribution as `draw_realization`
    (reference engine.py:232-244), different (vectorised) rng call order."""
    g = len(c.gates)
    out = np.zeros((e, g), dtype=np.uint8)
    for s, gate in enumerate(c.gates):
        probs = np.asarray([pr for _, pr in gate.noise.outcomes()])
        if probs[0] >= 1.0:
            continue
        fired = rng.random(e) < (1.0 - probs[0])
        k = int(fired.sum())
        if k and probs.size > 2:
            out[fired, s] = 1 + rng.integers(probs.size - 1, size=k)
        elif k:
            out[fired, s] = 1
    return out


def errorsets_from_matrix(c: Circuit, idx: np.ndarray, shots) -> list:
    """ErrorSet objects (labels) for an index matrix -- for the reference-style API."""
    labels = [[lb for lb, _ in g.noise.outcomes()] for g in c.gates]
    shots = np.broadcast_to(np.asarray(shots), (idx.shape[0],))
    return [
        ErrorSet(id=i, realized=tuple(labels[s][int(v)] for s, v in enumerate(row)), m=int(shots[i]))
        for i, row in enumerate(idx)
    ]
