"""Lanczos tridiagonalisation and Gauss rules on the GPU — mirror of
``/root/reference/pkg/src/spectrace/lanczos.py:40-163``.

``lanczos_tridiagonalize(op, q0, s)`` runs the device recurrence (CGS reorth
on by default for s <= 100, breakdown at 1e-12 * interval_hi) from a caller
given unit start vector; ``quadrature_rule`` runs the batched device
tridiagonal eigensolver.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device as _device

__all__ = ["Tridiagonal", "QuadratureRule", "lanczos_tridiagonalize", "quadrature_rule"]


@dataclass(frozen=True)
class Tridiagonal:
    alpha: np.ndarray
    beta: np.ndarray
    steps: int

    def to_dense(self) -> np.ndarray:
        t = np.diag(self.alpha)
        if self.beta.size:
            t += np.diag(self.beta, 1) + np.diag(self.beta, -1)
        return t


@dataclass(frozen=True)
class QuadratureRule:
    """Gauss rule: ascending nodes, nonnegative weights summing to 1 (lanczos.py:58-67)."""

    nodes: np.ndarray
    weights: np.ndarray

    def integrate(self, values: np.ndarray) -> float:
        return float(np.dot(self.weights, values))


def _require_graph_operator(op):
    dg = getattr(op, "device_graph", None)
    if dg is None:
        raise TypeError("only graph operators from paper_2003_01282_b200.make_operator run on the GPU engine "
                        "(arbitrary Python closures are not accelerated and there is no CPU fallback)")
    return dg


def lanczos_tridiagonalize(op, q0, s: int, reorth: bool | None = None, *, return_basis: bool = False,
                           dtype: str = "f64"):
    """Up to s Lanczos steps from the unit start vector q0 (lanczos.py:79-145).

    Returns the Tridiagonal, plus the (steps x dim) basis of Lanczos vectors when ``return_basis``
    is set (exported from the device recurrence)."""
    import torch

    if s < 1:
        raise ValueError(f"step budget must be >= 1, got {s}")
    dg = _require_graph_operator(op)
    n = op.dim
    q0 = np.asarray(q0, dtype=np.float64)
    if q0.shape != (n,):
        raise ValueError(f"start vector has shape {q0.shape}, expected ({n},)")
    if abs(np.linalg.norm(q0) - 1.0) > 1e-12:
        raise ValueError("start vector must have unit norm")
    start = torch.as_tensor(q0.reshape(n, 1), device=dg.device)
    code = -1 if reorth is None else int(bool(reorth))
    if return_basis:
        q, alpha, beta, st = dg.lanczos_basis(op.kind.value, 0, 0, 1, s, reorth=code, dtype=dtype, start=start)
    else:
        alpha, beta, st = dg.tridiagonals(op.kind.value, 0, 0, 1, s, reorth=code, dtype=dtype, start=start)
    k = int(st[0])
    tri = Tridiagonal(alpha=alpha[0, :k].cpu().numpy(), beta=beta[0, :k - 1].cpu().numpy(), steps=k)
    if return_basis:
        return tri, q[:k, :, 0].cpu().numpy()
    return tri


def quadrature_rule(tri: Tridiagonal) -> QuadratureRule:
    """Gauss rule of a tridiagonal via the device eigensolver (lanczos.py:148-163)."""
    import torch

    k = int(tri.steps)
    dev = torch.device("cuda", torch.cuda.current_device())
    alpha = torch.zeros((1, k), dtype=torch.float64, device=dev)
    beta = torch.zeros((1, k), dtype=torch.float64, device=dev)
    alpha[0, :k] = torch.as_tensor(np.asarray(tri.alpha, dtype=np.float64))
    if k > 1:
        beta[0, :k - 1] = torch.as_tensor(np.asarray(tri.beta, dtype=np.float64))
    steps = torch.tensor([k], dtype=torch.int32, device=dev)
    rules = _device.gauss_rules(alpha, beta, steps, (-np.inf, np.inf), n=k)
    return QuadratureRule(nodes=rules.nodes[0].cpu().numpy(), weights=rules.weights[0].cpu().numpy())
