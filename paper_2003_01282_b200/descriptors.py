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
