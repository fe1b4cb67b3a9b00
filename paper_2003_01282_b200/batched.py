"""Batched block-diagonal path for large collections of small graphs (BASELINE C3).

The graphs are stacked into one block-diagonal CSR (``graphs.block_diagonal``); the device runs
one CTA per graph (``slq_lanczos_batched``) and a per-graph quadrature (``slq_integrate_batched``).
Each graph's signature equals ``netlsd_slq(graph, grid, cfg)`` / ``vnge_slq(graph, cfg)`` on that
graph alone (reference ``descriptors.py:124-149, 227-243``): probes are prefixes of the same
seeded streams and every per-graph reduction runs in a fixed order.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .descriptors import EntropyValue, HeatTraceDescriptor, TimeGrid, _params
from .device import DeviceGraph
from .graphs import Graph, block_diagonal
from .slq import SlqConfig

__all__ = ["BatchedGraphs", "netlsd_slq_batch", "vnge_slq_batch"]

_MAX_PROBES = 64


class BatchedGraphs:
    """A block-diagonal stack of graphs resident on one GPU."""

    def __init__(self, graphs: list[Graph] | None = None, *, stacked: Graph | None = None,
                 vertex_offsets=None, device=None):
        import torch

        _lib.require_cuda()
        if graphs is not None:
            stacked, vertex_offsets = block_diagonal(graphs)
        if stacked is None or vertex_offsets is None:
            raise ValueError("give either graphs or (stacked, vertex_offsets)")
        self.graphs = graphs
        self.stacked = stacked
        self.voff = np.asarray(vertex_offsets, dtype=np.int64)
        self.count = int(self.voff.size - 1)
        self.dg = DeviceGraph(stacked, device, fold=None)   # the batched kernels use the stacked CSR itself
        self.voff_d = torch.tensor(self.voff, device=self.dg.device)

    @property
    def sizes(self) -> np.ndarray:
        return np.diff(self.voff)

    def rules(self, kind: str, cfg: SlqConfig, dtype: str = "f64"):
        import torch

        if cfg.distribution != "rademacher":
            raise NotImplementedError("gaussian probes are not on the device path")
        if not 1 <= cfg.n_v <= _MAX_PROBES:
            raise ValueError(f"the batched path takes 1 <= n_v <= {_MAX_PROBES}")
        dev = self.dg.device
        G, c, s = self.count, cfg.n_v, cfg.s
        nodes = torch.zeros((G, c, s), dtype=torch.float64, device=dev)
        weights = torch.zeros_like(nodes)
        steps = torch.zeros((G, c), dtype=torch.int32, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        code = {"normalized_laplacian": _lib.NORMALIZED_LAPLACIAN, "density": _lib.DENSITY}[kind]
        with torch.cuda.device(dev):
            _lib.check(_lib.load().slq_lanczos_batched_seeded(
                self.dg.handle, _lib.ptr(self.voff_d), G, code, _lib.seed_arg(cfg.seed), c, s,
                _lib.F64 if dtype == "f64" else _lib.F32, _lib.ptr(nodes), _lib.ptr(weights), _lib.ptr(steps),
                _lib.ptr(status), _lib.stream_handle(dev)))
        return nodes, weights, steps, status

    def integrate(self, rules, t, fn: int):
        """values/std_errors [G, T] on the device (status accumulates in rules[3])."""
        import torch

        nodes, weights, steps, status = rules
        dev = nodes.device
        tt = None if t is None else torch.tensor(np.asarray(t, dtype=np.float64), device=dev)
        T = 1 if tt is None else int(tt.numel())
        vals = torch.empty((self.count, T), dtype=torch.float64, device=dev)
        stds = torch.empty_like(vals)
        with torch.cuda.device(dev):
            _lib.check(_lib.load().slq_integrate_batched(
                _lib.ptr(nodes), _lib.ptr(weights), _lib.ptr(steps), self.count, int(nodes.shape[1]),
                int(nodes.shape[2]), _lib.ptr(self.voff_d), _lib.ptr(tt), T, fn, _lib.ptr(vals), _lib.ptr(stds),
                _lib.ptr(status), _lib.stream_handle(dev)))
        return vals, stds


def _host(vals, stds, status):
    import torch

    packed = torch.cat([vals.reshape(-1), stds.reshape(-1), status.to(torch.float64)]).cpu().numpy()
    _lib.check_status(int(packed[-1]))
    k = vals.numel()
    return packed[:k].reshape(vals.shape), packed[k:2 * k].reshape(vals.shape)


def netlsd_slq_batch(graphs, grid: TimeGrid | None = None, cfg: SlqConfig | None = None, *, dtype: str = "f64",
                     descriptors: bool = False, with_hash: bool = False):
    """Per-graph heat traces of a list of graphs (or a ``BatchedGraphs``): values, std_errors [G, T],
    or a list of ``HeatTraceDescriptor`` with ``descriptors=True``."""
    grid = grid or TimeGrid()
    cfg = cfg or SlqConfig()
    batch = graphs if isinstance(graphs, BatchedGraphs) else BatchedGraphs(graphs)
    rules = batch.rules("normalized_laplacian", cfg, dtype)
    vals, stds = _host(*batch.integrate(rules, grid.values, _lib.FN_HEAT), rules[3])
    if not descriptors:
        return vals, stds
    gs = batch.graphs or [None] * batch.count
    return [HeatTraceDescriptor(grid=grid, values=vals[k], method="slq", params=_params(cfg),
                                graph_hash=(gs[k].content_hash() if (with_hash and gs[k] is not None) else ""),
                                std_errors=stds[k]) for k in range(batch.count)]


def vnge_slq_batch(graphs, cfg: SlqConfig | None = None, *, dtype: str = "f64", descriptors: bool = False):
    """Per-graph von Neumann entropies (-tr P ln P) of a list of graphs."""
    cfg = cfg or SlqConfig()
    batch = graphs if isinstance(graphs, BatchedGraphs) else BatchedGraphs(graphs)
    off = batch.stacked.row_offsets
    if np.any(off[batch.voff[1:]] == off[batch.voff[:-1]]):
        raise ValueError("density matrix undefined for a graph without edges")
    rules = batch.rules("density", cfg, dtype)
    vals, stds = _host(*batch.integrate(rules, None, _lib.FN_XLOGX), rules[3])
    if not descriptors:
        return -vals[:, 0], stds[:, 0]
    return [EntropyValue(value=-float(vals[k, 0]), method="slq", params=_params(cfg), graph_hash="",
                         std_error=float(stds[k, 0])) for k in range(batch.count)]
