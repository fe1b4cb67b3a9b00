"""Spectral graph descriptors on the GPU — mirror of the SLQ entry points of
``/root/reference/pkg/src/spectrace/descriptors.py`` (TimeGrid :53-79,
netlsd_slq :124-149, vnge_slq :227-243, distances/JSON :308-387), plus the
wave trace (new) and the north-star adapters taking a
scipy.sparse adjacency, timescales, lanczos_steps and nvectors.

Heat and wave share ONE Lanczos run on the normalized Laplacian; VNGE is a
second run on the density matrix P = L / tr L.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import IO

import numpy as np

from . import _lib
from .graphs import Graph, as_graph, graph_from_scipy
from .operators import OperatorKind, make_operator
from .slq import SlqConfig, slq_rules

__all__ = ["TimeGrid", "HeatTraceDescriptor", "WaveTraceDescriptor", "EntropyValue", "netlsd_slq",
           "netlsd_taylor", "netlsd_linear", "netlsd_exact", "vnge_taylor", "vnge_finger", "vnge_exact",
           "netlsd_wave_slq", "netlsd_heat_wave_slq", "vnge_slq", "netlsd_slq_sparse", "vnge_slq_sparse",
           "descriptor_distance", "relative_error", "descriptor_to_json", "descriptor_from_json"]


@dataclass(frozen=True)
class TimeGrid:
    """Logarithmic heat-kernel times with pinned endpoints (descriptors.py:53-79)."""

    t_min: float = 1e-2
    t_max: float = 1e2
    count: int = 256
    values: np.ndarray = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        if self.count < 1:
            raise ValueError(f"count must be >= 1, got {self.count}")
        if self.count == 1:
            if not 0 < self.t_min == self.t_max:
                raise ValueError("a single-point grid needs 0 < t_min == t_max")
            values = np.array([self.t_min])
        else:
            if not 0 < self.t_min < self.t_max:
                raise ValueError(f"need 0 < t_min < t_max, got t_min={self.t_min}, t_max={self.t_max}")
            values = np.geomspace(self.t_min, self.t_max, self.count)
            values[0] = self.t_min
            values[-1] = self.t_max
        values.flags.writeable = False
        object.__setattr__(self, "values", values)


@dataclass(frozen=True)
class HeatTraceDescriptor:
    grid: TimeGrid
    values: np.ndarray
    method: str
    params: dict
    graph_hash: str
    std_errors: np.ndarray | None = None


@dataclass(frozen=True)
class WaveTraceDescriptor:
    """Wave trace w_t = sum_k exp(-i t lambda_k) on the normalized Laplacian (complex128 values)."""

    grid: TimeGrid
    values: np.ndarray
    method: str
    params: dict
    graph_hash: str
    std_errors: np.ndarray | None = None   # complex: std of real part + 1j * std of imaginary part


@dataclass(frozen=True)
class EntropyValue:
    value: float
    method: str
    params: dict
    graph_hash: str
    std_error: float | None = None


def _params(cfg: SlqConfig) -> dict:
    return {"n_v": cfg.n_v, "s": cfg.s, "distribution": cfg.distribution, "seed": cfg.seed}


def _integrate_host(rules, t, codes, host_work=None):
    """Device quadrature + aggregate for every integrand, ONE device->host copy, then the status check.
    ``host_work()`` (the descriptor's graph hash) runs on the host while the device computes."""
    import torch

    vals, stds = rules.integrate(t, codes)
    packed = torch.cat([vals.reshape(-1), stds.reshape(-1), rules.status.to(torch.float64)])
    extra = host_work() if host_work is not None else None   # overlaps the queued device work
    packed = packed.cpu().numpy()
    _lib.check_status(int(packed[-1]))
    k = vals.numel()
    shape = tuple(vals.shape)
    return packed[:k].reshape(shape), packed[k:2 * k].reshape(shape), extra


def _hash(g: Graph, with_hash: bool) -> str:
    return g.content_hash() if with_hash else ""


def netlsd_heat_wave_slq(g: Graph, grid: TimeGrid | None = None, cfg: SlqConfig | None = None, *,
                         threads: int = 1, dtype: str = "f64", wave: bool = True, shard: bool = False,
                         with_hash: bool = True):
    """Heat (and wave) traces from one device Lanczos run on the normalized Laplacian."""
    del threads
    import torch

    g = as_graph(g)
    grid = grid or TimeGrid()
    cfg = cfg or SlqConfig()
    # the timescales go up first, while the stream is idle: a pageable upload queued behind the
    # Lanczos run would block the host until the device finishes (no overlap with the graph hash)
    t = torch.tensor(np.array(grid.values, dtype=np.float64), device=_lib.require_cuda().cuda.current_device())
    op = make_operator(g, OperatorKind.NORMALIZED_LAPLACIAN)
    rules = slq_rules(op, cfg, dtype=dtype, shard=shard)
    codes = [_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM] if wave else [_lib.FN_HEAT]
    vals, stds, gh = _integrate_host(rules, t, codes, lambda: _hash(g, with_hash))
    heat = HeatTraceDescriptor(grid=grid, values=vals[0], method="slq", params=_params(cfg), graph_hash=gh,
                               std_errors=stds[0])
    if not wave:
        return heat, None
    wav = WaveTraceDescriptor(grid=grid, values=vals[1] + 1j * vals[2], method="slq", params=_params(cfg),
                              graph_hash=gh, std_errors=stds[1] + 1j * stds[2])
    return heat, wav


def netlsd_slq(g: Graph, grid: TimeGrid | None = None, cfg: SlqConfig | None = None, *, threads: int = 1,
               dtype: str = "f64", shard: bool = False) -> HeatTraceDescriptor:
    """Heat trace by SLQ on the GPU (descriptors.py:124-149)."""
    return netlsd_heat_wave_slq(g, grid, cfg, threads=threads, dtype=dtype, wave=False, shard=shard)[0]


def netlsd_wave_slq(g: Graph, grid: TimeGrid | None = None, cfg: SlqConfig | None = None, *, threads: int = 1,
                    dtype: str = "f64", shard: bool = False) -> WaveTraceDescriptor:
    """Wave trace sum_k exp(-i t lambda_k) by SLQ (new)."""
    return netlsd_heat_wave_slq(g, grid, cfg, threads=threads, dtype=dtype, wave=True, shard=shard)[1]


def vnge_slq(g: Graph, cfg: SlqConfig | None = None, *, threads: int = 1, dtype: str = "f64",
             shard: bool = False, with_hash: bool = True) -> EntropyValue:
    """Von Neumann entropy -tr(P ln P) by SLQ on the GPU (descriptors.py:227-243)."""
    del threads
    g = as_graph(g)
    cfg = cfg or SlqConfig()
    op = make_operator(g, OperatorKind.DENSITY)
    rules = slq_rules(op, cfg, dtype=dtype, shard=shard)
    val, std, gh = _integrate_host(rules, None, [_lib.FN_XLOGX], lambda: _hash(g, with_hash))
    return EntropyValue(value=-float(val[0, 0]), method="slq", params=_params(cfg), graph_hash=gh,
                        std_error=float(std[0, 0]))


# ------------------------------------------------------------------ trace-identity and spectral baselines
def _heat_trace(eigenvalues: np.ndarray, grid: TimeGrid) -> np.ndarray:
    lam = np.maximum(eigenvalues, 0.0)
    return np.exp(-np.outer(grid.values, lam)).sum(axis=1)


def netlsd_taylor(g, grid: TimeGrid | None = None) -> HeatTraceDescriptor:
    """Second-order heat-trace expansion n - t tr + (t^2/2) tr^2 from the device trace identities
    (descriptors.py:152-165; tr and tr^2 of the normalized Laplacian in one edge pass)."""
    from .operators import trace, trace_squared

    g = as_graph(g)
    grid = grid or TimeGrid()
    tr1 = trace(g, OperatorKind.NORMALIZED_LAPLACIAN)
    tr2 = trace_squared(g, OperatorKind.NORMALIZED_LAPLACIAN)
    t = grid.values
    return HeatTraceDescriptor(grid=grid, values=g.n - t * tr1 + 0.5 * t * t * tr2, method="taylor", params={},
                               graph_hash=g.content_hash())


def netlsd_exact(g, grid: TimeGrid | None = None, *, cap: int | None = None) -> HeatTraceDescriptor:
    """Heat trace from the full normalized-Laplacian spectrum (descriptors.py:108-121)."""
    from .lanczos import DENSE_SPECTRUM_CAP, dense_spectrum

    g = as_graph(g)
    grid = grid or TimeGrid()
    eigs = dense_spectrum(g, OperatorKind.NORMALIZED_LAPLACIAN, cap=cap or DENSE_SPECTRUM_CAP)
    return HeatTraceDescriptor(grid=grid, values=_heat_trace(eigs, grid), method="exact", params={},
                               graph_hash=g.content_hash())


def netlsd_linear(g, grid: TimeGrid | None = None, k: int = 300, *, cap: int | None = None) -> HeatTraceDescriptor:
    """Heat trace from k exact eigenvalues at each end (device Lanczos, ``extremal_eigenvalues``) with a
    linearly interpolated interior; the dense route when 2k >= n (descriptors.py:168-199)."""
    from .lanczos import extremal_eigenvalues

    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    g = as_graph(g)
    grid = grid or TimeGrid()
    if 2 * k >= g.n:
        exact = netlsd_exact(g, grid, cap=cap)
        return HeatTraceDescriptor(grid=grid, values=exact.values, method="linear",
                                   params={"k": k, "fallback": "exact"}, graph_hash=g.content_hash())
    op = make_operator(g, OperatorKind.NORMALIZED_LAPLACIAN)
    low = extremal_eigenvalues(op, k, "smallest")
    high = extremal_eigenvalues(op, k, "largest")
    interior_count = g.n - 2 * k
    step = (high[0] - low[-1]) / (interior_count + 1)
    interior = low[-1] + step * np.arange(1, interior_count + 1)
    eigs = np.concatenate([low, interior, high])
    return HeatTraceDescriptor(grid=grid, values=_heat_trace(eigs, grid), method="linear", params={"k": k},
                               graph_hash=g.content_hash())


def _entropy_from_spectrum(eigs: np.ndarray) -> float:
    lam = np.clip(eigs, 0.0, 1.0)
    pos = lam > 0
    return float(-np.sum(lam[pos] * np.log(lam[pos])))


def vnge_exact(g, *, cap: int | None = None) -> EntropyValue:
    """Entropy from the full density-matrix spectrum (descriptors.py:208-216)."""
    from .lanczos import DENSE_SPECTRUM_CAP, dense_spectrum

    g = as_graph(g)
    eigs = dense_spectrum(g, OperatorKind.DENSITY, cap=cap or DENSE_SPECTRUM_CAP)
    return EntropyValue(value=_entropy_from_spectrum(eigs), method="exact", params={}, graph_hash=g.content_hash())


def _taylor_quadratic(g) -> float:
    from .operators import trace, trace_squared

    tr_l = trace(g, OperatorKind.LAPLACIAN)
    tr_l2 = trace_squared(g, OperatorKind.LAPLACIAN)
    return 1.0 - tr_l2 / (tr_l * tr_l)


def vnge_taylor(g, variant: str = "corrected") -> EntropyValue:
    """Quadratic entropy expansion from the device trace identities (descriptors.py:252-275):
    ``corrected`` Q = 1 - tr(L^2)/tr(L)^2; ``printed`` 1 - (tr(L) + 2 tr(L^2))/tr(L)^2 verbatim."""
    from .operators import trace, trace_squared

    if variant not in ("corrected", "printed"):
        raise ValueError(f"variant must be 'corrected' or 'printed', got {variant!r}")
    g = as_graph(g)
    if g.m == 0:
        raise ValueError("entropy undefined for a graph without edges")
    if variant == "corrected":
        value = _taylor_quadratic(g)
    else:
        tr_l = trace(g, OperatorKind.LAPLACIAN)
        tr_l2 = trace_squared(g, OperatorKind.LAPLACIAN)
        value = 1.0 - (tr_l + 2.0 * tr_l2) / (tr_l * tr_l)
    return EntropyValue(value=value, method="taylor", params={"variant": variant}, graph_hash=g.content_hash())


def vnge_finger(g, variant: str = "hat") -> EntropyValue:
    """-Q ln(scale) (descriptors.py:278-305): ``hat`` takes the largest density eigenvalue from the
    device Lanczos run of ``extremal_eigenvalues``; ``bar`` the bound 2 max_deg / tr(L)."""
    from .lanczos import extremal_eigenvalues
    from .operators import trace

    if variant not in ("hat", "bar"):
        raise ValueError(f"variant must be 'hat' or 'bar', got {variant!r}")
    g = as_graph(g)
    if g.m == 0:
        raise ValueError("entropy undefined for a graph without edges")
    q = _taylor_quadratic(g)
    if variant == "hat":
        op = make_operator(g, OperatorKind.DENSITY)
        scale = float(extremal_eigenvalues(op, 1, "largest")[-1])
    else:
        from .device import device_graph

        scale = 2.0 * float(device_graph(g).info.max_degree) / trace(g, OperatorKind.LAPLACIAN)
    if scale <= 0:
        raise ValueError(f"nonpositive spectral scale {scale} for log")
    return EntropyValue(value=-q * np.log(scale), method="finger", params={"variant": variant},
                        graph_hash=g.content_hash())


def _grid_from_timescales(timescales) -> TimeGrid:
    t = np.asarray(timescales, dtype=np.float64)
    grid = TimeGrid(float(t[0]), float(t[-1]), int(t.size)) if t.size > 1 else TimeGrid(float(t[0]), float(t[0]), 1)
    if not np.array_equal(grid.values, t):
        # arbitrary (non-geometric) timescales: carry them verbatim
        object.__setattr__(grid, "values", t.copy())
        grid.values.flags.writeable = False
    return grid


def netlsd_slq_sparse(adjacency, timescales=None, lanczos_steps: int = 10, nvectors: int = 100, seed: int = 0,
                      *, wave: bool = False, dtype: str = "f64"):
    """North-star adapter: scipy.sparse adjacency + timescale grid + lanczos_steps + nvectors."""
    g = graph_from_scipy(adjacency)
    grid = TimeGrid() if timescales is None else _grid_from_timescales(timescales)
    cfg = SlqConfig(n_v=nvectors, s=lanczos_steps, seed=seed)
    heat, wav = netlsd_heat_wave_slq(g, grid, cfg, dtype=dtype, wave=wave)
    return (heat, wav) if wave else heat


def vnge_slq_sparse(adjacency, lanczos_steps: int = 10, nvectors: int = 100, seed: int = 0, *, dtype: str = "f64"):
    g = graph_from_scipy(adjacency)
    return vnge_slq(g, SlqConfig(n_v=nvectors, s=lanczos_steps, seed=seed), dtype=dtype)


def descriptor_distance(a, b) -> float:
    """Euclidean distance between traces, |a-b| between entropies (descriptors.py:308-321)."""
    if isinstance(a, (HeatTraceDescriptor, WaveTraceDescriptor)) and type(a) is type(b):
        if not np.array_equal(a.grid.values, b.grid.values):
            raise ValueError("heat-trace descriptors have mismatched time grids")
        return float(np.linalg.norm(a.values - b.values))
    if isinstance(a, EntropyValue) and isinstance(b, EntropyValue):
        return abs(a.value - b.value)
    raise ValueError(f"cannot compare descriptors of different types: {type(a).__name__} vs {type(b).__name__}")


def relative_error(approx, reference) -> float:
    """Relative l2 error (descriptors.py:324-335)."""
    ref_norm = float(np.linalg.norm(reference.values)) if not isinstance(reference, EntropyValue) \
        else abs(reference.value)
    if ref_norm == 0:
        raise ValueError("reference descriptor has zero norm")
    return descriptor_distance(approx, reference) / ref_norm


def descriptor_to_json(desc, stream: IO[str] | None = None) -> str:
    """Self-describing JSON {kind, method, params, grid?, values | value, seed?, graph_hash}
    (descriptors.py:338-361); the wave trace stores [re, im] pairs."""
    obj: dict = {"method": desc.method, "params": dict(desc.params)}
    if isinstance(desc, (HeatTraceDescriptor, WaveTraceDescriptor)):
        obj["kind"] = "netlsd" if isinstance(desc, HeatTraceDescriptor) else "netlsd_wave"
        obj["grid"] = {"t_min": desc.grid.t_min, "t_max": desc.grid.t_max, "count": desc.grid.count}
        if isinstance(desc, HeatTraceDescriptor):
            obj["values"] = [float(v) for v in desc.values]
        else:
            obj["values"] = [[float(v.real), float(v.imag)] for v in desc.values]
    else:
        obj["kind"] = "vnge"
        obj["value"] = float(desc.value)
    if "seed" in desc.params:
        obj["seed"] = desc.params["seed"]
    obj["graph_hash"] = desc.graph_hash
    text = json.dumps(obj, sort_keys=True, indent=2) + "\n"
    if stream is not None:
        stream.write(text)
    return text


def descriptor_from_json(text: str):
    obj = json.loads(text)
    if obj["kind"] in ("netlsd", "netlsd_wave"):
        grid = TimeGrid(t_min=obj["grid"]["t_min"], t_max=obj["grid"]["t_max"], count=obj["grid"]["count"])
        if obj["kind"] == "netlsd":
            return HeatTraceDescriptor(grid=grid, values=np.asarray(obj["values"], dtype=np.float64),
                                       method=obj["method"], params=obj["params"], graph_hash=obj["graph_hash"])
        v = np.asarray(obj["values"], dtype=np.float64)
        return WaveTraceDescriptor(grid=grid, values=v[:, 0] + 1j * v[:, 1], method=obj["method"],
                                   params=obj["params"], graph_hash=obj["graph_hash"])
    if obj["kind"] == "vnge":
        return EntropyValue(value=float(obj["value"]), method=obj["method"], params=obj["params"],
                            graph_hash=obj["graph_hash"])
    raise ValueError(f"unknown descriptor kind {obj.get('kind')!r}")
