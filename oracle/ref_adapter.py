"""Drives the UNMODIFIED reference (imported from /root/reference, read-only)
for pinning the oracle and generating tests/golden -- TEST INFRASTRUCTURE ONLY,
usable only in the build container (the GPU box has no /root/reference).

Two shims, both verified against the reference's duck typing
(SURVEY.md section 0 findings 3-4):
  * KrausNetwork: a CircuitNetwork whose .merged(k) folds arbitrary Kraus
    operators (amplitude damping, ...) into arbitrarily wired gate tensors --
    only .n, .net, .final_labels and .merged are used by the reference's
    sampler (engine.py:373-407, 511);
  * oracle.ptsbe_oracle.CounterMultinomial as the `rng` of sample_proportional
    (engine.py:519 is its only use in proportional mode).
"""

from __future__ import annotations

import os
import sys
from dataclasses import dataclass

import numpy as np

REFERENCE_SRC = "/root/reference/pkg/src"


def available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "ptsbe"))


def load_reference():
    """Import the reference package without writing bytecode into its tree."""
    if not available():
        raise RuntimeError("reference sources are not present on this machine")
    sys.dont_write_bytecode = True
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import ptsbe  # noqa: F401

    return ptsbe


def kraus_network(ref, n: int, gates, site_ops):
    """gates: (unitary, targets); site_ops: per site dict label -> operator
    matrix.  Returns an object accepted by the reference's sample_proportional
    and conditional_marginal."""
    from ptsbe.engine import CircuitNetwork
    from ptsbe.tensor import Index, Tensor, TensorNetwork

    head = list(range(n))
    fresh = n
    ops = [Tensor([Index(q, 2)], np.array([1.0, 0.0], dtype=np.complex128)) for q in range(n)]
    for u, targets in gates:
        k = len(targets)
        ins = [head[q] for q in targets]
        outs = list(range(fresh, fresh + k))
        fresh += k
        for q, lb in zip(targets, outs):
            head[q] = lb
        ops.append(Tensor([Index(lb, 2) for lb in outs + ins],
                          np.asarray(u, dtype=np.complex128).reshape((2,) * (2 * k))))
    base = TensorNetwork(ops, head)

    @dataclass(frozen=True)
    class KrausNetwork(CircuitNetwork):
        def merged(self, k):
            operands = list(self.net.operands)
            for site, label in enumerate(k.realized):
                op = site_ops[site].get(label)
                if op is None:
                    continue
                slot = n + site
                old = operands[slot]
                side = op.shape[0]
                operands[slot] = Tensor(old.indices, (op @ old.data.reshape(side, side)).reshape(old.data.shape))
            return CircuitNetwork(net=TensorNetwork(operands, self.net.open_indices),
                                  final_labels=self.final_labels)

    return KrausNetwork(net=base, final_labels=tuple(head))
