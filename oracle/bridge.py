"""Adapters between the product's host objects and the oracle's plain data --
TEST INFRASTRUCTURE ONLY (used by tests/, smoke() and bench.py's CPU legs).

The oracle works on (labels, ndarray) operands; the product's `Circuit`
supplies gate matrices and channel operators.  Nothing here computes a
contraction: it only reshapes inputs so both sides see identical numbers.
"""

from __future__ import annotations

import numpy as np

from paper_2604_08467_b200.circuits import Circuit, gate_matrix, is_identity_label

from . import ptsbe_oracle as O


def template_of(c: Circuit) -> tuple:
    """(operands, final labels) of the error-free template for the oracle."""
    return O.build_template(c.n, [(gate_matrix(g), g.targets) for g in c.gates])


def realized_operators(c: Circuit, realized) -> list:
    """Error-operator matrix per gate site (None = identity) for one error set."""
    out = []
    for g, label in zip(c.gates, realized):
        out.append(None if is_identity_label(label) else g.noise.operator(label))
    return out


def oracle_errorsets(c: Circuit, errorsets) -> list:
    return [(k.id, realized_operators(c, k.realized), k.m) for k in errorsets]


def merged_ops(c: Circuit, realized) -> tuple:
    ops, finals = template_of(c)
    return O.merge_errors(ops, realized_operators(c, realized)), finals


def histogram_of(records) -> list:
    return [(r.bitstring, int(r.count)) for r in records]
