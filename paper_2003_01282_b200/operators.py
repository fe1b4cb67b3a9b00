"""Graph operators on the GPU — mirror of the reference plugin API
(``/root/reference/pkg/src/spectrace/operators.py:31-102``).

``make_operator(g, kind)`` returns a ``LinearOperator(dim, apply, kind, interval)``
exactly like the reference, except that ``apply`` runs the sm_100a SpMM
(bit-identical to the reference closure per column) and the operator carries
its ``DeviceGraph`` so the SLQ engine can run the whole recurrence on device.
Operators that are not graph operators (arbitrary Python closures) are not
accelerated: the SLQ entry points reject them (no CPU fallback).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Callable

import numpy as np

from . import _lib
from .device import DeviceGraph, device_graph
from .graphs import Graph, as_graph

__all__ = ["OperatorKind", "LinearOperator", "degrees", "make_operator", "trace", "trace_squared"]

_KIND_CODE = {"laplacian": _lib.LAPLACIAN, "normalized_laplacian": _lib.NORMALIZED_LAPLACIAN, "density": _lib.DENSITY}


class OperatorKind(Enum):
    LAPLACIAN = "laplacian"
    NORMALIZED_LAPLACIAN = "normalized_laplacian"
    DENSITY = "density"


@dataclass(frozen=True)
class LinearOperator:
    """Symmetric operator: dimension, matvec closure, kind and spectrum interval (operators.py:37-49)."""

    dim: int
    apply: Callable
    kind: OperatorKind | None
    interval: tuple[float, float]
    device_graph: DeviceGraph | None = field(default=None, repr=False, compare=False)


def degrees(g: Graph, device=None) -> np.ndarray:
    """Weighted degree vector d = A.1, computed on the GPU (operators.py:58-62)."""
    g = as_graph(g)
    if g.n == 0:
        return np.zeros(0)
    d, _ = device_graph(g, device).degrees()
    return d.cpu().numpy()


def make_operator(g: Graph, kind: OperatorKind, device=None) -> LinearOperator:
    """Implicit operator of the requested kind on the GPU (operators.py:65-102).

    Raises ValueError for the density matrix of an edgeless graph, like the reference.
    """
    kind = OperatorKind(getattr(kind, "value", kind))   # the reference's own OperatorKind members too
    g = as_graph(g)
    dg = device_graph(g, device)
    interval = dg.interval(kind.value)    # raises ValueError for density without edges

    def apply(x):
        return dg.apply(kind.value, x)

    return LinearOperator(dim=g.n, apply=apply, kind=kind, interval=interval, device_graph=dg)


def trace(g: Graph, kind: OperatorKind) -> float:
    """Exact operator trace from the device-prepared degree statistics (operators.py:105-117)."""
    kind = OperatorKind(getattr(kind, "value", kind))
    g = as_graph(g)
    info = device_graph(g).info
    if kind is OperatorKind.LAPLACIAN:
        return float(info.trace_l)
    if kind is OperatorKind.NORMALIZED_LAPLACIAN:
        return float(info.n - info.isolated)
    if g.m == 0:
        raise ValueError("density matrix undefined for a graph without edges")
    return 1.0


def trace_squared(g: Graph, kind: OperatorKind) -> float:
    """Exact tr(M^2) in one edge pass on the device (operators.py:119-141): L: sum d^2 + sum w^2;
    normalized Laplacian: #non-isolated + sum_e w^2 / (d_r d_c); density: tr(L^2) / tr(L)^2.
    Fixed-order device sums (the reference uses numpy's pairwise sum): equal to rounding."""
    import ctypes

    kind = OperatorKind(getattr(kind, "value", kind))
    g = as_graph(g)
    if kind is OperatorKind.DENSITY and g.m == 0:
        raise ValueError("density matrix undefined for a graph without edges")
    out = ctypes.c_double()
    _lib.check(_lib.load().slq_trace_squared(device_graph(g).handle, _KIND_CODE[kind.value], ctypes.byref(out)))
    return float(out.value)
