"""Device-resident graphs and per-probe rules (thin wrappers over the C ABI).

PyTorch is only the container for device buffers and the stream handle; all
arithmetic happens in libslq_b200.so.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graphs import Graph, as_graph

KIND_CODES = {"laplacian": _lib.LAPLACIAN, "normalized_laplacian": _lib.NORMALIZED_LAPLACIAN,
              "density": _lib.DENSITY}


# Isolated-vertex fold (slq_graph_fold_isolated): graphs with at least this fraction of unreferenced
# empty rows (and at least FOLD_MIN_N vertices) run the Lanczos recurrence on the folded graph.
FOLD_MIN_FRACTION = 1.0 / 64
FOLD_MIN_N = 256
FLAT_MIN_NNZ = 1 << 24   # csrc/graph.cu kFlatMinNnz: graphs the flat SpMM (and so the degree order) applies to


def worth_folding(row_offsets, n: int, nnz: int, min_fraction: float = FOLD_MIN_FRACTION) -> bool:
    """Host-side pre-check of the isolated-vertex fold: at least FOLD_MIN_N vertices, some edges, and
    empty rows (an upper bound of the foldable vertices) making up >= min_fraction of them."""
    if n < FOLD_MIN_N or nnz <= 0:
        return False
    if nnz >= FLAT_MIN_NNZ:
        return True    # large graphs: the fold's degree order feeds the flat SpMM (the library decides)
    off = np.asarray(row_offsets)
    empty = int(off.size - 1 - np.count_nonzero(off[1:] != off[:-1]))
    return empty >= 1 and empty >= min_fraction * n


class DeviceGraph:
    """Prepared CSR on one GPU: int32 columns, implicit unit weights, degrees, dinv, tiles."""

    folded = 0   # vertices folded into the trailing row of the isolated-vertex fold (0: none)

    def __init__(self, g: Graph, device=None, *, from_device: bool = False,
                 fold: float | None = FOLD_MIN_FRACTION):
        torch = _lib.require_cuda()
        g = as_graph(g)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.graph = g
        self.n = int(g.n)
        self.nnz = int(g.nnz)
        self.handle = ctypes.c_void_p()
        lib = _lib.load()
        with torch.cuda.device(self.device):
            stream = _lib.stream_handle(self.device)
            w = None if g.is_unweighted() else np.ascontiguousarray(g.weights, dtype=np.float64)
            if from_device:
                off = torch.as_tensor(np.asarray(g.row_offsets, dtype=np.int64), device=self.device)
                cols = torch.as_tensor(np.asarray(g.col_indices, dtype=np.int64), device=self.device)
                wt = None if w is None else torch.as_tensor(w, device=self.device)
                rc = lib.slq_graph_create(self.n, g.nnz, _lib.ptr(off), _lib.ptr(cols), _lib.ptr(wt), stream,
                                          ctypes.byref(self.handle))
            else:
                off = np.ascontiguousarray(g.row_offsets, dtype=np.int64)
                cols = np.ascontiguousarray(g.col_indices, dtype=np.int64)
                rc = lib.slq_graph_create_host(self.n, g.nnz, off.ctypes.data, cols.ctypes.data,
                                               None if w is None else w.ctypes.data, stream,
                                               ctypes.byref(self.handle))
        _lib.check(rc)
        self._info = None
        # empty rows counted on the host first: graphs below the threshold never synchronise here
        if fold is not None and worth_folding(g.row_offsets, self.n, g.nnz, fold):
            self.fold_isolated(fold)

    def fold_isolated(self, min_fraction: float = FOLD_MIN_FRACTION) -> int:
        """Build (or with ``min_fraction < 0`` drop) the isolated-vertex fold; returns the number of
        folded vertices (0: not folded).  Synchronises the graph's stream."""
        m = ctypes.c_int64()
        with _lib.require_cuda().cuda.device(self.device):
            _lib.check(_lib.load().slq_graph_fold_isolated(self.handle, float(min_fraction), ctypes.byref(m)))
        self.folded = int(m.value)
        return self.folded

    @classmethod
    def rmat(cls, scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
             seed: int = 0, device=None, fold: float | None = FOLD_MIN_FRACTION) -> "DeviceGraph":
        """An R-MAT graph generated and converted to canonical CSR on the device (no host copy of the
        edges: the C5 workload's 4e9 directed edges never leave HBM).  ``graph`` is None."""
        torch = _lib.require_cuda()
        self = cls.__new__(cls)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.graph = None
        self.handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().slq_graph_create_rmat(int(scale), int(edge_factor), float(a), float(b), float(c),
                                                         int(seed), _lib.stream_handle(self.device),
                                                         ctypes.byref(self.handle)))
        self._info = None
        self.n = int(self.info.n)
        self.nnz = int(self.info.nnz)
        if fold is not None and self.n >= FOLD_MIN_N:
            self.fold_isolated(fold)
        return self

    @classmethod
    def from_csr32(cls, n: int, row_offsets, col_indices, weights=None, device=None,
                   fold: float | None = FOLD_MIN_FRACTION) -> "DeviceGraph":
        """Device graph from a compact CSR: int64 offsets [n+1] and int32 columns [nnz] (numpy arrays,
        pinned host tensors or device tensors), optional float64 weights (None = implicit 1.0) --
        the scale-27 workload's "int32 indices" format, uploaded without an int64 copy.  ``graph``
        is None (no host ``Graph``; descriptors carry an empty hash)."""
        torch = _lib.require_cuda()
        self = cls.__new__(cls)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.graph = None
        self.handle = ctypes.c_void_p()

        def arr(x, dt):
            if isinstance(x, torch.Tensor):
                if x.dtype != dt:
                    raise TypeError(f"expected {dt}, got {x.dtype}")
                return x.contiguous()
            return np.ascontiguousarray(x, dtype={torch.int64: np.int64, torch.int32: np.int32,
                                                  torch.float64: np.float64}[dt])

        off = arr(row_offsets, torch.int64)
        cols = arr(col_indices, torch.int32)
        w = None if weights is None else arr(weights, torch.float64)
        nnz = int(cols.shape[0])
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().slq_graph_create_i32(int(n), nnz, _lib.ptr(off), _lib.ptr(cols), _lib.ptr(w),
                                                        _lib.stream_handle(self.device), ctypes.byref(self.handle)))
        self._info = None
        self.n = int(n)
        self.nnz = nnz
        if fold is not None and self.n >= FOLD_MIN_N:
            self.fold_isolated(fold)
        return self

    @classmethod
    def from_edges(cls, n: int, u, v, w=None, device=None, fold: float | None = FOLD_MIN_FRACTION) -> "DeviceGraph":
        """Canonical CSR built on the device from an edge list (numpy arrays or torch tensors, host
        or device): the semantics of ``graphs.csr_from_edges`` (self-loops dropped, both directions,
        duplicates collapse to the maximum weight, sorted).  ``graph`` is None."""
        torch = _lib.require_cuda()
        self = cls.__new__(cls)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.graph = None
        self.handle = ctypes.c_void_p()

        def arr(x, dt):
            if isinstance(x, torch.Tensor):
                return x.to(dt).contiguous()
            return torch.as_tensor(np.ascontiguousarray(x), dtype=dt)

        ut, vt = arr(u, torch.int64), arr(v, torch.int64)
        wt = None if w is None else arr(w, torch.float64)
        if ut.numel() != vt.numel() or (wt is not None and wt.numel() != ut.numel()):
            raise ValueError("u, v (and w) must have the same length")
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().slq_graph_create_edges(int(n), int(ut.numel()), _lib.ptr(ut), _lib.ptr(vt),
                                                          _lib.ptr(wt), _lib.stream_handle(self.device),
                                                          ctypes.byref(self.handle)))
        self._info = None
        self.n = int(self.info.n)
        self.nnz = int(self.info.nnz)
        if fold is not None and self.n >= FOLD_MIN_N:
            self.fold_isolated(fold)
        return self

    def weights(self):
        """Stored edge weights [nnz] (float64) copied from the device, or None for implicit 1.0."""
        import torch

        if not self.nnz:
            return None
        w = torch.empty(self.nnz, dtype=torch.float64, device=self.device)
        has = ctypes.c_int32()
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().slq_graph_weights(self.handle, _lib.ptr(w), ctypes.byref(has),
                                                      _lib.stream_handle(self.device)))
        return w.cpu().numpy() if has.value else None

    def csr(self):
        """(row_offsets int64 [n+1], col_indices int32 [nnz]) copied from the device (small graphs)."""
        import torch

        off = torch.empty(self.n + 1, dtype=torch.int64, device=self.device)
        cols = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().slq_graph_csr(self.handle, _lib.ptr(off), _lib.ptr(cols),
                                                  _lib.stream_handle(self.device)))
        return off.cpu().numpy(), cols[:self.nnz].cpu().numpy()

    @property
    def info(self):
        """Graph scalars (tr L, max degree, ...); the first access synchronises the stream."""
        if self._info is None:
            info = _lib.GraphInfo()
            _lib.check(_lib.load().slq_graph_info(self.handle, ctypes.byref(info)))
            self._info = info
        return self._info

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.load().slq_graph_destroy(h)
            except Exception:
                pass
            self.handle = ctypes.c_void_p()

    def second_passes(self) -> int:
        """Probe-steps of this graph that ran the conditional second CGS pass (lanczos.py:75-76) since
        it was created: a device counter (diagnostics; synchronises the graph's stream)."""
        v = ctypes.c_int64()
        with _lib.require_cuda().cuda.device(self.device):
            _lib.check(_lib.load().slq_graph_second_passes(self.handle, ctypes.byref(v)))
        return int(v.value)

    def lanczos_row_lengths(self, count: int):
        """(first `count` row lengths, row count) of the graph the recurrence runs on (the fold, in
        descending-degree order, when the graph is folded).  Diagnostics."""
        out = np.zeros(int(count), dtype=np.int64)
        rows = ctypes.c_int64()
        with _lib.require_cuda().cuda.device(self.device):
            _lib.check(_lib.load().slq_graph_lanczos_rows(self.handle, out.ctypes.data, int(count), ctypes.byref(rows)))
        return out, int(rows.value)

    # -- operator set-up -----------------------------------------------------------
    def interval(self, kind: str) -> tuple[float, float]:
        lo, hi = ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.load().slq_operator_interval(self.handle, KIND_CODES[kind], ctypes.byref(lo), ctypes.byref(hi)))
        return float(lo.value), float(hi.value)

    def degrees(self):
        import torch

        d = torch.empty(self.n, dtype=torch.float64, device=self.device)
        dinv = torch.empty(self.n, dtype=torch.float64, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().slq_graph_degrees(self.handle, _lib.ptr(d), _lib.ptr(dinv),
                                                      _lib.stream_handle(self.device)))
        return d, dinv

    def apply(self, kind: str, x):
        """Y = Op(X) for a [n] or [n, k] float64 block (torch CUDA tensor or numpy array)."""
        import torch

        host = isinstance(x, np.ndarray)
        xt = torch.as_tensor(np.asarray(x, dtype=np.float64), device=self.device) if host else x
        if xt.dtype != torch.float64:
            raise TypeError("operator apply takes float64 vectors")
        one = xt.dim() == 1
        xt = xt.reshape(self.n, -1).contiguous()
        y = torch.empty_like(xt)
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().slq_operator_apply(self.handle, KIND_CODES[kind], _lib.ptr(xt), _lib.ptr(y),
                                                       xt.shape[1], xt.shape[1], _lib.stream_handle(self.device)))
        if one:
            y = y.reshape(-1)
        return y.cpu().numpy() if host else y

    # -- Lanczos + rules -----------------------------------------------------------
    def tridiagonals(self, kind: str, seed: int, probe_begin: int, count: int, steps: int, *,
                     reorth: int = -1, dtype: str = "f64", start=None):
        """alpha/beta [count, s'] and steps [count] on the device."""
        import torch

        s = min(int(steps), self.n)
        alpha = torch.zeros((count, s), dtype=torch.float64, device=self.device)
        beta = torch.zeros((count, s), dtype=torch.float64, device=self.device)
        st = torch.zeros(count, dtype=torch.int32, device=self.device)
        code = _lib.F64 if dtype in ("f64", "float64", np.float64) else _lib.F32
        lib = _lib.load()
        with torch.cuda.device(self.device):
            stream = _lib.stream_handle(self.device)
            if start is None:
                rc = lib.slq_lanczos_seeded(self.handle, KIND_CODES[kind], _lib.seed_arg(seed), int(probe_begin),
                                            int(count), int(steps), int(reorth), code, _lib.ptr(alpha), _lib.ptr(beta),
                                            _lib.ptr(st), stream)
            else:
                q0 = start.contiguous()
                rc = lib.slq_lanczos_start(self.handle, KIND_CODES[kind], _lib.ptr(q0), q0.shape[1], int(count),
                                           int(steps), int(reorth), code, _lib.ptr(alpha), _lib.ptr(beta),
                                           _lib.ptr(st), stream)
        _lib.check(rc)
        return alpha, beta, st

    def lanczos_basis(self, kind: str, seed: int, probe_begin: int, count: int, steps: int, *, reorth: int = -1,
                      dtype: str = "f64", start=None):
        """Debug export (``return_basis=True``, lanczos.py:85,143-144): Q [s', n, count] float64 with
        Q[k, :, j] the k-th Lanczos vector of probe probe_begin+j (or of start vector j of ``start``
        [n, count]), plus alpha, beta [count, s'] and steps [count].  Runs on the unfolded graph."""
        import torch

        s = min(int(steps), self.n)
        if start is not None:
            count = int(start.shape[1])
        q = torch.zeros((s, self.n, count), dtype=torch.float64, device=self.device)
        alpha = torch.zeros((count, s), dtype=torch.float64, device=self.device)
        beta = torch.zeros((count, s), dtype=torch.float64, device=self.device)
        st = torch.zeros(count, dtype=torch.int32, device=self.device)
        code = _lib.F64 if dtype in ("f64", "float64", np.float64) else _lib.F32
        lib = _lib.load()
        with torch.cuda.device(self.device):
            stream = _lib.stream_handle(self.device)
            if start is None:
                rc = lib.slq_lanczos_basis(self.handle, KIND_CODES[kind], int(seed), int(probe_begin), int(count),
                                           int(steps), int(reorth), code, _lib.ptr(q), _lib.ptr(alpha),
                                           _lib.ptr(beta), _lib.ptr(st), stream)
            else:
                q0 = start.contiguous()
                rc = lib.slq_lanczos_start_basis(self.handle, KIND_CODES[kind], _lib.ptr(q0), q0.shape[1], count,
                                                 int(steps), int(reorth), code, _lib.ptr(q), _lib.ptr(alpha),
                                                 _lib.ptr(beta), _lib.ptr(st), stream)
        _lib.check(rc)
        return q, alpha, beta, st

    def rules(self, kind: str, seed: int, probe_begin: int, count: int, steps: int, *, reorth: int = -1,
              dtype: str = "f64", status=None) -> "DeviceRules":
        """Gauss rules of probes [probe_begin, +count), asynchronously (errors land in ``status``)."""
        import torch

        s = min(int(steps), self.n)
        nodes = torch.zeros((count, s), dtype=torch.float64, device=self.device)
        weights = torch.zeros_like(nodes)
        st = torch.zeros(count, dtype=torch.int32, device=self.device)
        if status is None:
            status = torch.zeros(1, dtype=torch.int32, device=self.device)
        if KIND_CODES[kind] == _lib.DENSITY and self.nnz == 0:
            raise ValueError("density matrix undefined for a graph without edges")
        code = _lib.F64 if dtype in ("f64", "float64", np.float64) else _lib.F32
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().slq_rules_seeded(self.handle, KIND_CODES[kind], _lib.seed_arg(seed), int(probe_begin),
                                                    int(count), int(steps), int(reorth), code, _lib.ptr(nodes),
                                                    _lib.ptr(weights), _lib.ptr(st), _lib.ptr(status),
                                                    _lib.stream_handle(self.device)))
        return DeviceRules(nodes, weights, st, self.n, status=status)


    def rules_pair(self, seed: int, probe_begin: int, count: int, steps: int, *, reorth: int = -1, dtype: str = "f32",
                   status=None):
        """Normalized-Laplacian and density-matrix rules of the same probes in one call
        (``slq_rules_pair_seeded``): with 9..16 fp32 probes on a large folded graph both Lanczos runs
        share every gathered row.  Returns ``(rules_nl, rules_density, paired)``; per-probe results
        are bitwise those of two ``rules`` calls."""
        import ctypes

        import torch

        if self.nnz == 0:
            raise ValueError("density matrix undefined for a graph without edges")
        s = min(int(steps), self.n)
        out = [torch.zeros((count, s), dtype=torch.float64, device=self.device) for _ in range(4)]
        st = [torch.zeros(count, dtype=torch.int32, device=self.device) for _ in range(2)]
        if status is None:
            status = torch.zeros(1, dtype=torch.int32, device=self.device)
        code = _lib.F64 if dtype in ("f64", "float64", np.float64) else _lib.F32
        paired = ctypes.c_int32(0)
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().slq_rules_pair_seeded(
                self.handle, _lib.seed_arg(seed), int(probe_begin), int(count), int(steps), int(reorth), code,
                _lib.ptr(out[0]), _lib.ptr(out[1]), _lib.ptr(st[0]), _lib.ptr(out[2]), _lib.ptr(out[3]), _lib.ptr(st[1]),
                _lib.ptr(status), ctypes.addressof(paired), _lib.stream_handle(self.device)))
        return (DeviceRules(out[0], out[1], st[0], self.n, status=status),
                DeviceRules(out[2], out[3], st[1], self.n, status=status), bool(paired.value))


@dataclass
class DeviceRules:
    nodes: object      # torch [count, s] float64 (clamped, ascending, zero padded)
    weights: object    # torch [count, s]
    steps: object      # torch [count] int32
    n: int
    alpha: object = None
    beta: object = None
    status: object = None    # device int32[1]: OR of the asynchronous error bits

    def check(self) -> None:
        if self.status is not None:
            _lib.check_status(int(self.status.item()))

    def integrate(self, t, fns):
        """values [nfn, T] and std_errors [nfn, T] on the device (no host synchronisation)."""
        import torch

        dev = self.nodes.device
        if self.status is None:
            self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        if t is None:
            tt, T = None, 1
        else:
            tt = t.to(device=dev, dtype=torch.float64).contiguous() if isinstance(t, torch.Tensor) \
                else torch.tensor(np.asarray(t, dtype=np.float64), device=dev)
            T = int(tt.numel())
        vals = torch.empty((len(fns), T), dtype=torch.float64, device=dev)
        stds = torch.empty_like(vals)
        with torch.cuda.device(dev):
            _lib.check(_lib.load().slq_integrate(_lib.ptr(self.nodes), _lib.ptr(self.weights), _lib.ptr(self.steps),
                                                  self.count, int(self.nodes.shape[1]), _lib.ptr(tt), T,
                                                  _lib.int_array(fns), len(fns), float(self.n), _lib.ptr(vals),
                                                  _lib.ptr(stds), None, _lib.ptr(self.status),
                                                  _lib.stream_handle(dev)))
        return vals, stds

    @property
    def count(self) -> int:
        return int(self.nodes.shape[0])

    def quadrature(self, t, fn: int):
        """per_vector [T, count] on the device."""
        import torch

        dev = self.nodes.device
        if t is None:
            tt = None
        elif isinstance(t, torch.Tensor):
            tt = t.to(device=dev, dtype=torch.float64).contiguous()
        else:
            tt = torch.tensor(np.asarray(t, dtype=np.float64), device=dev)
        T = 1 if tt is None else int(tt.numel())
        pv = torch.empty((T, self.count), dtype=torch.float64, device=dev)
        with torch.cuda.device(dev):
            _lib.check(_lib.load().slq_quadrature(_lib.ptr(self.nodes), _lib.ptr(self.weights), _lib.ptr(self.steps),
                                                   self.count, int(self.nodes.shape[1]), _lib.ptr(tt), T, fn,
                                                   _lib.ptr(pv), _lib.stream_handle(dev)))
        return pv

    def estimate(self, pv):
        """(value [T], std_error [T]) on the device."""
        import torch

        dev = pv.device
        T = int(pv.shape[0])
        val = torch.empty(T, dtype=torch.float64, device=dev)
        std = torch.empty(T, dtype=torch.float64, device=dev)
        with torch.cuda.device(dev):
            _lib.check(_lib.load().slq_estimate(_lib.ptr(pv), T, int(pv.shape[1]), float(self.n), _lib.ptr(val),
                                                 _lib.ptr(std), _lib.stream_handle(dev)))
        return val, std


def gauss_rules(alpha, beta, steps, interval, n: int) -> DeviceRules:
    import torch

    count, width = alpha.shape
    nodes = torch.zeros_like(alpha)
    weights = torch.zeros_like(alpha)
    info = torch.zeros(count, dtype=torch.int32, device=alpha.device)
    if count:
        with torch.cuda.device(alpha.device):
            rc = _lib.load().slq_gauss_rules(_lib.ptr(alpha), _lib.ptr(beta), _lib.ptr(steps), count, width,
                                             float(interval[0]), float(interval[1]), _lib.ptr(nodes),
                                             _lib.ptr(weights), _lib.ptr(info), _lib.stream_handle(alpha.device))
        if rc == _lib.SLQ_ERR_EIGEN:
            bad = int(torch.nonzero(info).flatten()[0])
            k = int(steps[bad])
            _lib.check(rc, alpha=alpha[bad, :k].cpu().numpy(), beta=beta[bad, :k - 1].cpu().numpy())
        _lib.check(rc)
    return DeviceRules(nodes, weights, steps, n, alpha, beta)


def device_graph(g: Graph, device=None) -> DeviceGraph:
    """Cached DeviceGraph for a Graph (Graph arrays are read-only, so the cache stays valid)."""
    import torch

    g = as_graph(g)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = str(dev)
    cache = g._device_cache
    dg = cache.get(key)
    if dg is None:
        dg = DeviceGraph(g, dev)
        cache[key] = dg
    return dg


def device_probes(n: int, seed: int, probe_begin: int, count: int, device=None):
    """Rademacher probes [n, count] (+-1.0, float64) of the seeded streams, generated on the device."""
    torch = _lib.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = torch.empty((n, count), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().slq_probes_seeded(_lib.seed_arg(seed), int(probe_begin), int(count), int(n),
                                                 _lib.ptr(out), int(count), _lib.stream_handle(dev)))
    return out


class CapturedSignature:
    """A whole signature — probes, Lanczos, Gauss rules, quadrature over the grid and the probe
    aggregate — captured once as a CUDA graph and replayed with one launch.  For latency-bound
    workloads (small graphs, many repeated signatures) the replay removes the host submission and
    inter-kernel gaps of the ~40 launches of an eager signature; results are bitwise those of the
    eager path.  ``replay()`` returns the captured output tensors (values, std_errors), overwritten by
    every replay; ``check()`` maps the device status word to the reference exceptions."""

    def __init__(self, dg: "DeviceGraph", kind: str, seed: int, count: int, steps: int, t, fns, *,
                 dtype: str = "f64"):
        torch = _lib.require_cuda()
        self.device = dg.device
        with torch.cuda.device(self.device):
            self._t = None if t is None else torch.tensor(np.array(t, dtype=np.float64), device=self.device)

            def run():
                rules = dg.rules(kind, seed, 0, count, steps, dtype=dtype)
                vals, stds = rules.integrate(self._t, fns)
                return rules, vals, stds

            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):
                run()   # warm-up: kernel attributes, the stream-ordered pool, cached sizes
            torch.cuda.current_stream(self.device).wait_stream(side)
            torch.cuda.synchronize(self.device)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
                self.rules, self.values, self.std_errors = run()

    def replay(self):
        self.graph.replay()
        return self.values, self.std_errors

    def check(self) -> None:
        self.rules.check()
