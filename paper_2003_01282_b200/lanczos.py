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

__all__ = ["Tridiagonal", "QuadratureRule", "lanczos_tridiagonalize", "quadrature_rule", "extremal_eigenvalues",
           "dense_spectrum", "DENSE_SPECTRUM_CAP"]

DENSE_SPECTRUM_CAP = 20_000   # lanczos.py:34

_BREAKDOWN_REL_TOL = 1e-12   # lanczos.py:36


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


def _select_extreme(pools, k: int, largest: bool):
    """k extreme values of the merged pools, or None if fewer than k (lanczos.py:165-171)."""
    if not pools:
        return None
    merged = np.sort(np.concatenate(pools))
    if merged.size < k:
        return None
    return merged[-k:] if largest else merged[:k]


def _device_ritz(alpha, beta, lengths):
    """Ritz values (ascending) of the leading `L` x `L` blocks of one tridiagonal, for every L in
    `lengths`, from ONE batched device eigensolve (slq_gauss_rules; lanczos.py:174-177 uses
    eigvalsh_tridiagonal)."""
    import torch

    lengths = [int(x) for x in lengths]
    if not lengths:
        return []
    dev = alpha.device
    width = max(lengths)
    a = torch.zeros((len(lengths), width), dtype=torch.float64, device=dev)
    b = torch.zeros_like(a)
    for r, L in enumerate(lengths):
        a[r, :L] = alpha[:L]
        if L > 1:
            b[r, :L - 1] = beta[:L - 1]
    st = torch.tensor(lengths, dtype=torch.int32, device=dev)
    rules = _device.gauss_rules(a, b, st, (-np.inf, np.inf), n=1)
    nodes = rules.nodes.cpu().numpy()
    return [nodes[r, :L].copy() for r, L in enumerate(lengths)]


def extremal_eigenvalues(op, k: int, end: str, *, tol: float = 1e-8, max_steps: int | None = None,
                         check_every: int = 10, dtype: str = "f64") -> np.ndarray:
    """k eigenvalues from one end of the spectrum, ascending (lanczos.py:180-297).

    The reference expands one fully reorthogonalised Lanczos run from a seeded Gaussian start vector
    (``SeedSequence(0x5EC7, spawn_key=(n, k))``) until the k selected Ritz values move by less than
    ``tol`` between checks every ``check_every`` steps; a breakdown makes that run's Ritz values
    exact eigenvalues and restarts from a fresh start vector deflated against everything retained.
    Here the recurrence runs on the device (``slq_lanczos_start``, reorth forced on, step budgets
    doubling from 4 * check_every so an early convergence costs little); the convergence checks of
    every prefix the reference would test come from one batched device eigensolve of the prefix
    tridiagonals, so the stopping step and the returned Ritz values follow the reference's rule.
    After a breakdown the start vector of the next sweep is deflated on the device against every
    retained basis vector (two CGS passes); that sweep's recurrence reorthogonalises against its
    own basis only (the retained subspace is invariant, so they agree in exact arithmetic).
    Raises ``ConvergenceError`` (with the best estimates) when ``max_steps`` is exhausted."""
    import torch

    from .errors import ConvergenceError

    if end not in ("smallest", "largest"):
        raise ValueError(f"end must be 'smallest' or 'largest', got {end!r}")
    dg = _require_graph_operator(op)
    n = op.dim
    if not 1 <= k <= n:
        raise ValueError(f"k must lie in [1, {n}], got {k}")
    if max_steps is None:
        max_steps = 10 * k + 100
    largest = end == "largest"
    rng = np.random.default_rng(np.random.SeedSequence(entropy=0x5EC7, spawn_key=(n, k)))
    kind = op.kind.value
    retained = []          # device bases [n, m_j] of the swept invariant subspaces
    n_basis = 0
    exact_pools: list = []
    prev = None
    partial = None
    steps = 0
    while steps < max_steps and n_basis < n:
        q = torch.as_tensor(rng.standard_normal(n), device=dg.device)
        for _ in range(2 if retained else 0):     # _reorthogonalize against everything retained
            for bmat in retained:
                q = q - bmat @ (bmat.T @ q)
        norm = float(torch.linalg.norm(q))
        if norm < 1e-8:
            break
        q = (q / norm).reshape(n, 1).contiguous()
        remaining = min(max_steps - steps, n - n_basis)
        budget = min(remaining, max(4 * check_every, k + check_every))
        prev_at_start = prev
        while True:
            prev = prev_at_start   # a longer run re-tests every prefix (identical prefixes)
            alpha, beta, st = dg.tridiagonals(kind, 0, 0, 1, budget, reorth=1, dtype=dtype, start=q)
            R = int(st[0])
            broke = R < budget or n_basis + R >= n   # breakdown, or the basis spans the space
            last = broke or budget >= remaining
            # the reference checks after step L (L % check_every == 0, L >= k) only while its run goes on
            checks = [L for L in range(check_every, R, check_every) if L >= k]
            ritz = _device_ritz(alpha[0], beta[0], checks + [R])
            for vals in ritz[:-1]:
                sel = _select_extreme(exact_pools + [vals], k, largest)
                if sel is not None:
                    if prev is not None and np.all(np.abs(sel - prev) < tol):
                        return np.sort(sel)
                    prev = sel
            if last:
                break
            budget = min(remaining, 2 * budget)
        steps += R
        n_basis += R
        run_vals = ritz[-1]
        if not broke:
            partial = run_vals
            break
        exact_pools.append(run_vals)
        qb, _, _, _ = dg.lanczos_basis(kind, 0, 0, 1, R, reorth=1, dtype=dtype, start=q)   # the swept subspace
        retained.append(qb[:R, :, 0].T.contiguous())
        sel = _select_extreme(exact_pools, k, largest)
        if sel is not None:
            if n_basis >= n:
                return np.sort(sel)
            if prev is not None and np.all(np.abs(sel - prev) < tol):
                return np.sort(sel)
            prev = sel
    pools = exact_pools + ([partial] if partial is not None else [])
    merged = np.sort(np.concatenate(pools)) if pools else np.empty(0)
    best = merged[-min(k, merged.size):] if largest else merged[: min(k, merged.size)]
    raise ConvergenceError(f"extremal eigenvalues did not stabilize within {max_steps} steps",
                           best_estimates=np.sort(best))


def dense_spectrum(g, kind, *, cap: int = DENSE_SPECTRUM_CAP) -> np.ndarray:
    """All eigenvalues of the densified operator, ascending (lanczos.py:300-328): the exact reference
    the approximations are compared with.  The dense matrix is the device operator applied to the
    identity (bit-exact columns of the reference's operator) and its spectrum comes from
    ``torch.linalg.eigvalsh`` (cuSOLVER) -- a library call on a path off the SLQ engine; refuses
    graphs above ``cap`` vertices like the reference."""
    import torch

    from .graphs import as_graph
    from .operators import OperatorKind, make_operator

    g = as_graph(g)
    if g.n > cap:
        raise ValueError(f"dense spectrum refused: n={g.n} exceeds cap {cap}")
    kind = OperatorKind(getattr(kind, "value", kind))
    op = make_operator(g, kind)          # ValueError for the density of an edgeless graph
    dg = op.device_graph
    if g.n == 0:
        return np.zeros(0)
    eye = torch.eye(g.n, dtype=torch.float64, device=dg.device)
    mat = dg.apply(kind.value, eye)
    mat = 0.5 * (mat + mat.T)            # exactly symmetric already up to the row-sum rounding
    return torch.linalg.eigvalsh(mat).cpu().numpy()
