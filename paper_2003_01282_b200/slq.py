"""Stochastic Lanczos quadrature on the GPU — mirror of
``/root/reference/pkg/src/spectrace/slq.py:28-168``.

The seam replaced is ``_collect_rules`` (slq.py:80-86) plus the grid loop
(slq.py:168): all probes of a chunk run the recurrence together on the
device, the batched eigensolver builds every rule at once, and the quadrature
kernel evaluates the integrand over the whole t grid.  Known integrands
(heat, wave, x ln x) are evaluated on the device; an arbitrary Python ``f``
is applied to the (tiny) node/weight arrays on the host, exactly as the
reference's ``_apply_rule`` does, after the device has produced the rules.

``threads`` is accepted and ignored (the reference guarantees results never
depend on it).  Results never depend on chunking or GPU count.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _lib
from .device import DeviceRules

__all__ = ["SlqConfig", "SlqEstimate", "slq_trace", "slq_trace_grid", "slq_rules", "Integrand",
           "heat_family", "wave_re_family", "wave_im_family", "xlogx"]

_DISTRIBUTIONS = ("rademacher", "gaussian")


@dataclass(frozen=True)
class SlqConfig:
    """n_v probes, s Lanczos steps, probe law, seed (slq.py:28-45)."""

    n_v: int = 100
    s: int = 10
    distribution: str = "rademacher"
    seed: int = 0

    def __post_init__(self):
        if self.n_v < 1:
            raise ValueError(f"n_v must be >= 1, got {self.n_v}")
        if self.s < 1:
            raise ValueError(f"s must be >= 1, got {self.s}")
        if self.distribution not in _DISTRIBUTIONS:
            raise ValueError(f"distribution must be one of {_DISTRIBUTIONS}, got {self.distribution!r}")


@dataclass(frozen=True)
class SlqEstimate:
    """value = dim * mean(per_vector); std_error = std(dim*pv, ddof=1)/sqrt(n_v) (slq.py:48-60)."""

    value: float
    per_vector: np.ndarray
    std_error: float


@dataclass(frozen=True)
class Integrand:
    """A device-evaluated integrand: code in {heat, wave_re, wave_im, xlogx, identity}, optional t.

    Calling it on host nodes gives the same function, so it is also a plain ``f``."""

    code: int
    t: float | None = None

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        if self.code == _lib.FN_HEAT:
            return np.exp(-self.t * x)
        if self.code == _lib.FN_WAVE_RE:
            return np.cos(self.t * x)
        if self.code == _lib.FN_WAVE_IM:
            return -np.sin(self.t * x)
        if self.code == _lib.FN_XLOGX:
            out = np.zeros_like(x)
            pos = x > 0
            out[pos] = x[pos] * np.log(x[pos])
            return out
        return x


def heat_family(t: float) -> Integrand:
    return Integrand(_lib.FN_HEAT, float(t))


def wave_re_family(t: float) -> Integrand:
    return Integrand(_lib.FN_WAVE_RE, float(t))


def wave_im_family(t: float) -> Integrand:
    return Integrand(_lib.FN_WAVE_IM, float(t))


xlogx = Integrand(_lib.FN_XLOGX)
identity = Integrand(_lib.FN_IDENTITY)


def _graph_of(op):
    dg = getattr(op, "device_graph", None)
    if dg is None:
        raise TypeError("slq_trace needs a graph operator from paper_2003_01282_b200.make_operator; "
                        "arbitrary Python operators are not accelerated (no CPU fallback)")
    return dg


def slq_rules(op, cfg: SlqConfig, *, dtype: str = "f64", reorth: bool | None = None,
              shard: bool = False) -> DeviceRules:
    """Per-probe Gauss rules for probes 0..n_v-1 on the device (slq.py:69-86).

    ``shard=True`` splits the probes over the ranks of the initialised
    torch.distributed group and all-gathers the rules (dist.py)."""
    dg = _graph_of(op)
    code = -1 if reorth is None else int(bool(reorth))
    if cfg.distribution == "gaussian":
        if shard:
            raise NotImplementedError("sharded Gaussian probes: shard Rademacher probes or run one rank")
        return _gaussian_rules(dg, op, cfg, code, dtype)
    if shard:
        from .dist import sharded_rules

        return sharded_rules(dg, op.kind.value, cfg, dtype=dtype, reorth=code)
    return dg.rules(op.kind.value, cfg.seed, 0, cfg.n_v, cfg.s, reorth=code, dtype=dtype)


_GAUSS_BLOCK = 64   # probes per uploaded start block


def gaussian_start_block(n: int, seed: int, begin: int, count: int) -> np.ndarray:
    """Unit Gaussian start vectors [n, count] of probes begin..begin+count-1, drawn exactly as the
    reference (slq.py:63-73: ``default_rng(SeedSequence(seed, spawn_key=(i,))).standard_normal(n)``
    normalised by ``np.linalg.norm``).  numpy's ziggurat runs on the host; the Lanczos recurrence,
    rules and quadrature stay on the device (the start block is uploaded once per 64 probes)."""
    out = np.empty((n, count))
    for c in range(count):
        rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(begin + c,)))
        v = rng.standard_normal(n)
        out[:, c] = v / np.linalg.norm(v)
    return out


def _gaussian_rules(dg, op, cfg: SlqConfig, reorth: int, dtype: str) -> DeviceRules:
    import torch

    from .device import gauss_rules

    s = min(cfg.s, dg.n)
    alphas, betas, steps = [], [], []
    for b in range(0, cfg.n_v, _GAUSS_BLOCK):
        c = min(_GAUSS_BLOCK, cfg.n_v - b)
        q0 = torch.as_tensor(gaussian_start_block(dg.n, cfg.seed, b, c), device=dg.device)
        a, bt, st = dg.tridiagonals(op.kind.value, 0, 0, c, s, reorth=reorth, dtype=dtype, start=q0)
        alphas.append(a)
        betas.append(bt)
        steps.append(st)
    return gauss_rules(torch.cat(alphas), torch.cat(betas), torch.cat(steps), op.interval, dg.n)


def _estimate_host(per_vector: np.ndarray, n: int) -> SlqEstimate:
    n_v = per_vector.size
    value = n * (float(per_vector.sum()) / n_v)
    std = float(np.std(n * per_vector, ddof=1)) / math.sqrt(n_v) if n_v > 1 else 0.0
    return SlqEstimate(value=value, per_vector=per_vector, std_error=std)


def _host_rules(rules: DeviceRules):
    nodes = rules.nodes.cpu().numpy()
    weights = rules.weights.cpu().numpy()
    steps = rules.steps.cpu().numpy()
    return [(nodes[p, :steps[p]], weights[p, :steps[p]]) for p in range(rules.count)]


def _apply_host(rule, f) -> float:
    nodes, weights = rule
    values = np.asarray(f(nodes), dtype=np.float64)
    if not np.all(np.isfinite(values)):
        raise ValueError(f"f returned a non-finite value at quadrature nodes {nodes!r}")
    return float(np.dot(weights, values))


def _finish(rules: DeviceRules, fs: Sequence, n: int, control_variate=None) -> list[SlqEstimate]:
    """Apply each f of ``fs`` to every rule; device path when all are Integrands of one code."""
    if control_variate is None and fs and all(isinstance(f, Integrand) for f in fs) \
            and len({f.code for f in fs}) == 1:
        code = fs[0].code
        ts = None if fs[0].t is None else np.array([f.t for f in fs], dtype=np.float64)
        pv = rules.quadrature(ts, code)
        val, std = rules.estimate(pv)
        rules.check()
        pv_h, val_h, std_h = pv.cpu().numpy(), val.cpu().numpy(), std.cpu().numpy()
        return [SlqEstimate(float(val_h[k]), pv_h[k], float(std_h[k])) for k in range(len(fs))]
    rules.check()
    host = _host_rules(rules)
    out = []
    for f in fs:
        if control_variate is None:
            out.append(_estimate_host(np.array([_apply_host(r, f) for r in host]), n))
            continue
        (c0, c1, c2), exact = control_variate

        def residual(x, f=f):
            return f(x) - (c0 + c1 * x + c2 * x * x)

        base = _estimate_host(np.array([_apply_host(r, residual) for r in host]), n)
        out.append(SlqEstimate(base.value + exact, base.per_vector, base.std_error))
    return out


def slq_trace(op, f: Callable, cfg: SlqConfig, *, threads: int = 1,
              control_variate: tuple[Sequence[float], float] | None = None, dtype: str = "f64",
              shard: bool = False) -> SlqEstimate:
    """Estimate tr f(op) with cfg.n_v probes of cfg.s Lanczos steps (slq.py:108-129)."""
    del threads
    rules = slq_rules(op, cfg, dtype=dtype, shard=shard)
    return _finish(rules, [f], op.dim, control_variate)[0]


def slq_trace_grid(op, f_family: Callable, grid: Sequence[float], cfg: SlqConfig, *, threads: int = 1,
                   dtype: str = "f64", shard: bool = False) -> list[SlqEstimate]:
    """slq_trace at every grid point, sharing the rules (slq.py:153-168)."""
    del threads
    rules = slq_rules(op, cfg, dtype=dtype, shard=shard)
    return _finish(rules, [f_family(t) for t in grid], op.dim)
