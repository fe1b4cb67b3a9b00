"""Graph container and canonical CSR assembly (host side).

Mirrors the reference's ``Graph`` (``/root/reference/pkg/src/spectrace/graphs.py:34-88``):
an immutable undirected simple graph in CSR form with int64 row offsets,
int64 column indices sorted within each row, float64 weights and the
undirected edge count ``m``.  The canonical layout rules follow
``graphs.py:110-132`` (both directions stored, rows and columns ascending,
no self-loops, duplicates collapsed to the maximum weight).

This is the host-side input container; the device copy (int32 columns,
implicit unit weights when possible) is built by ``device.DeviceGraph``.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

__all__ = ["Graph", "as_graph", "csr_from_edges", "graph_from_scipy", "block_diagonal", "unique_sorted"]


def unique_sorted(keys: np.ndarray) -> np.ndarray:
    """Sorted distinct values (sort + neighbour mask; much faster than np.unique on large int64)."""
    keys = np.sort(np.asarray(keys), kind="stable")
    if keys.size == 0:
        return keys
    keep = np.empty(keys.size, dtype=bool)
    keep[0] = True
    np.not_equal(keys[1:], keys[:-1], out=keep[1:])
    return keys[keep]


@dataclass(frozen=True, eq=False)
class Graph:
    """Undirected weighted graph in CSR form (reference ``graphs.py:34-60``)."""

    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    weights: np.ndarray
    m: int
    _hash: list = field(default_factory=list, init=False, repr=False, compare=False)
    _device_cache: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        for arr in (self.row_offsets, self.col_indices, self.weights):
            arr.flags.writeable = False

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[self.n]) if self.n else 0

    def __eq__(self, other) -> bool:
        if not isinstance(other, Graph):
            return NotImplemented
        return (self.n == other.n and self.m == other.m
                and np.array_equal(self.row_offsets, other.row_offsets)
                and np.array_equal(self.col_indices, other.col_indices)
                and np.array_equal(self.weights, other.weights))

    __hash__ = object.__hash__

    def is_unweighted(self) -> bool:
        return bool(np.all(self.weights == 1.0))

    def content_hash(self) -> str:
        """SHA-256 over int64 n ‖ offsets ‖ cols ‖ weights (reference ``graphs.py:81-88``).

        The arrays are read-only, so the digest is computed once and cached.
        """
        if not self._hash:
            h = hashlib.sha256()
            h.update(np.int64(self.n).tobytes())
            # buffer views, no byte copies (hashlib reads contiguous arrays in place)
            h.update(memoryview(np.ascontiguousarray(self.row_offsets, dtype=np.int64)).cast("B"))
            h.update(memoryview(np.ascontiguousarray(self.col_indices, dtype=np.int64)).cast("B"))
            h.update(memoryview(np.ascontiguousarray(self.weights, dtype=np.float64)).cast("B"))
            self._hash.append(h.hexdigest())
        return self._hash[0]


_FOREIGN: dict = {}   # id(foreign graph) -> (weakref, Graph view): one device copy per caller object


def as_graph(g) -> "Graph":
    """This package's ``Graph`` for any CSR graph object with the reference's fields.

    The drop-in accepts the reference's own ``spectrace.Graph`` (``graphs.py:34-88``: n,
    row_offsets, col_indices, weights, m) and any object carrying the same attributes.  The arrays
    are viewed, not copied, and the view is cached per caller object (keyed by identity, dropped
    when the caller's graph is garbage collected) so its device copy and content hash are built
    once, as for a native ``Graph``."""
    if isinstance(g, Graph):
        return g
    for attr in ("n", "row_offsets", "col_indices", "weights", "m"):
        if not hasattr(g, attr):
            raise TypeError(f"expected a CSR graph with n, row_offsets, col_indices, weights, m; got {type(g).__name__}")
    import weakref

    key = id(g)
    hit = _FOREIGN.get(key)
    if hit is not None and hit[0]() is g:
        return hit[1]
    view = Graph(int(g.n), np.asarray(g.row_offsets), np.asarray(g.col_indices), np.asarray(g.weights), int(g.m))
    try:
        ref = weakref.ref(g, lambda _r, key=key: _FOREIGN.pop(key, None))
    except TypeError:     # not weak-referenceable: no cache
        return view
    _FOREIGN[key] = (ref, view)
    return view


def csr_from_edges(n: int, u, v, w=None) -> Graph:
    """Canonical Graph from an edge list (any direction, duplicates, self-loops allowed).

    Self-loops are dropped, each edge is stored in both directions, duplicates
    collapse to the maximum weight, rows and columns are sorted ascending.
    """
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    if u.size and (min(u.min(), v.min()) < 0 or max(u.max(), v.max()) >= n):
        raise ValueError("edge endpoint out of range")
    lo = np.minimum(u, v)
    hi = np.maximum(u, v)
    key = lo * n + hi
    if w is None:
        key = unique_sorted(key)
        wt = np.ones(key.size)
    else:
        wt_in = np.asarray(w, dtype=np.float64)[keep]
        order = np.lexsort((wt_in, key))
        key, wt_in = key[order], wt_in[order]
        last = np.ones(key.size, dtype=bool)
        last[:-1] = key[1:] != key[:-1]
        key, wt = key[last], wt_in[last]
    m = int(key.size)
    a, b = key // n, key % n
    # both directions, ordered by (row, col) through one int64 key sort
    both = np.concatenate([key, b * n + a])
    if w is None:
        both.sort(kind="stable")
        ws = np.ones(both.size)
    else:
        order = np.argsort(both, kind="stable")
        both = both[order]
        ws = np.concatenate([wt, wt])[order]
    rows, cols = both // n, both % n
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=offsets[1:])
    return Graph(n=n, row_offsets=offsets, col_indices=cols.astype(np.int64),
                 weights=ws.astype(np.float64), m=m)


def graph_from_scipy(adjacency) -> Graph:
    """Adapter for the north-star signature: a symmetric scipy.sparse adjacency.

    The matrix is canonicalised exactly like an edge list (self-loops dropped,
    symmetrised, max weight on duplicates).
    """
    import scipy.sparse as sp

    coo = sp.coo_matrix(adjacency)
    if coo.shape[0] != coo.shape[1]:
        raise ValueError(f"adjacency must be square, got {coo.shape}")
    data = np.asarray(coo.data, dtype=np.float64)
    nz = data != 0
    return csr_from_edges(coo.shape[0], coo.row[nz], coo.col[nz], data[nz])


def block_diagonal(graphs: list[Graph]) -> tuple[Graph, np.ndarray]:
    """Stack graphs into one block-diagonal Graph; returns (graph, vertex offsets)."""
    sizes = np.array([g.n for g in graphs], dtype=np.int64)
    voff = np.zeros(len(graphs) + 1, dtype=np.int64)
    np.cumsum(sizes, out=voff[1:])
    nnzs = np.array([g.nnz for g in graphs], dtype=np.int64)
    eoff = np.zeros(len(graphs) + 1, dtype=np.int64)
    np.cumsum(nnzs, out=eoff[1:])
    n = int(voff[-1])
    offsets = np.empty(n + 1, dtype=np.int64)
    cols = np.empty(int(eoff[-1]), dtype=np.int64)
    ws = np.empty(int(eoff[-1]), dtype=np.float64)
    for k, g in enumerate(graphs):
        offsets[voff[k]:voff[k + 1]] = g.row_offsets[:-1] + eoff[k]
        cols[eoff[k]:eoff[k + 1]] = g.col_indices + voff[k]
        ws[eoff[k]:eoff[k + 1]] = g.weights
    offsets[n] = eoff[-1]
    return Graph(n=n, row_offsets=offsets, col_indices=cols, weights=ws,
                 m=int(sum(g.m for g in graphs))), voff
