"""Host-side logic that needs no GPU: canonical CSR, graph hash, TimeGrid, SlqConfig, JSON, adapters."""
import numpy as np
import pytest
import scipy.sparse as sp

import golden
from oracle import slq_oracle as O
from paper_2003_01282_b200 import synth
from paper_2003_01282_b200.descriptors import (EntropyValue, HeatTraceDescriptor, TimeGrid, WaveTraceDescriptor,
                                               descriptor_from_json, descriptor_to_json, relative_error)
from paper_2003_01282_b200.graphs import block_diagonal, csr_from_edges, graph_from_scipy
from paper_2003_01282_b200.slq import SlqConfig


def test_csr_canonical_layout_matches_reference_graphs():
    z = golden.load("small.npz")
    for name in [str(x) for x in z["names"]]:
        g = golden.graph(z, f"{name}/")
        # rebuild from the edge list in random order with duplicates and both directions
        rows = np.repeat(np.arange(g.n), np.diff(g.row_offsets))
        u, v, w = rows, g.col_indices, g.weights
        perm = np.random.default_rng(0).permutation(u.size)
        g2 = csr_from_edges(g.n, u[perm], v[perm], None if g.is_unweighted() else w[perm])
        assert g2 == g, name


def test_duplicates_collapse_to_max_weight_and_self_loops_drop():
    g = csr_from_edges(3, [0, 1, 0, 2, 2], [1, 0, 1, 2, 1], [1.0, 3.0, 2.0, 9.0, 0.5])
    assert g.m == 2
    assert np.array_equal(g.row_offsets, [0, 1, 3, 4])
    assert np.array_equal(g.col_indices, [1, 0, 2, 1])
    assert np.array_equal(g.weights, [3.0, 3.0, 0.5, 0.5])


def test_content_hash_matches_reference_graph_hash():
    z = golden.load("small.npz")
    for name in [str(x) for x in z["names"]]:
        g = golden.graph(z, f"{name}/")
        assert g.content_hash() == str(z[f"{name}/desc/graph_hash"]), name


def test_graph_from_scipy_adapter():
    g = synth.barabasi_albert(200, 2, seed=1)
    a = sp.csr_matrix((g.weights, g.col_indices, g.row_offsets), shape=(g.n, g.n))
    assert graph_from_scipy(a) == g
    assert graph_from_scipy(sp.triu(a)) == g   # one triangle is enough: symmetrised


def test_block_diagonal():
    gs = synth.er_batch(5, seed=3)
    big, voff = block_diagonal(gs)
    assert big.n == sum(g.n for g in gs) and big.m == sum(g.m for g in gs)
    for k, g in enumerate(gs):
        lo, hi = voff[k], voff[k + 1]
        sub = big.row_offsets[lo:hi + 1] - big.row_offsets[lo]
        assert np.array_equal(sub, g.row_offsets)


def test_timegrid_matches_reference_definition():
    tg = TimeGrid(1e-2, 1e2, 250)
    assert np.array_equal(tg.values, O.time_grid(1e-2, 1e2, 250))
    assert tg.values[0] == 1e-2 and tg.values[-1] == 1e2
    with pytest.raises(ValueError):
        TimeGrid(1.0, 0.5, 10)
    with pytest.raises(ValueError):
        TimeGrid(count=0)
    assert np.array_equal(TimeGrid(0.5, 0.5, 1).values, [0.5])


def test_slqconfig_validation():
    assert SlqConfig() == SlqConfig(100, 10, "rademacher", 0)
    for bad in (dict(n_v=0), dict(s=0), dict(distribution="uniform")):
        with pytest.raises(ValueError):
            SlqConfig(**bad)


def test_descriptor_json_roundtrip():
    grid = TimeGrid(1e-2, 1e2, 8)
    params = {"n_v": 4, "s": 3, "distribution": "rademacher", "seed": 7}
    h = HeatTraceDescriptor(grid, np.linspace(1, 2, 8), "slq", params, "abc")
    w = WaveTraceDescriptor(grid, np.linspace(1, 2, 8) + 1j * np.linspace(0, 1, 8), "slq", params, "abc")
    e = EntropyValue(1.25, "slq", params, "abc")
    for d in (h, w, e):
        back = descriptor_from_json(descriptor_to_json(d))
        assert type(back) is type(d)
        if isinstance(d, EntropyValue):
            assert back.value == d.value
        else:
            assert np.array_equal(back.values, d.values)
            assert relative_error(back, d) == 0.0
        assert back.params == params and back.graph_hash == "abc"


def test_generators_shapes():
    g = synth.barabasi_albert(1000, 3, seed=0)
    assert g.n == 1000 and g.m == 2991
    s = synth.sbm(20_000, 10, 1e-3, 1e-5, seed=0)
    assert abs(s.m - (10 * 2000 * 1999 / 2 * 1e-3 + (20000 * 19999 / 2 - 10 * 2000 * 1999 / 2) * 1e-5)) < 500
    r = synth.rmat(10, 16, seed=0)
    rows = np.repeat(np.arange(r.n), np.diff(r.row_offsets))
    assert np.all(rows != r.col_indices)           # no self-loops
    assert r.nnz % 2 == 0 and r.m == r.nnz // 2    # symmetric


def test_rmat_device_reference_is_canonical():
    g = synth.rmat_device_reference(10, 8, seed=3)
    off, cols = g.row_offsets, g.col_indices
    assert g.n == 1024 and off[-1] == g.nnz and g.nnz % 2 == 0
    for r in range(0, g.n, 97):
        row = cols[off[r]:off[r + 1]]
        assert np.all(np.diff(row) > 0) and not np.any(row == r)


def test_fold_precheck_counts_empty_rows():
    from paper_2003_01282_b200.device import FOLD_MIN_N, worth_folding
    from paper_2003_01282_b200.graphs import csr_from_edges

    n = 4 * FOLD_MIN_N
    dense = csr_from_edges(n, np.arange(n - 1), np.arange(1, n))            # a path: no empty row
    assert not worth_folding(dense.row_offsets, n, dense.nnz)
    sparse = csr_from_edges(n, np.arange(0, n // 2 - 1), np.arange(1, n // 2))   # half the vertices isolated
    assert worth_folding(sparse.row_offsets, n, sparse.nnz)
    assert not worth_folding(sparse.row_offsets, n, sparse.nnz, min_fraction=0.75)
    small = csr_from_edges(10, [0], [1])                                     # below FOLD_MIN_N
    assert not worth_folding(small.row_offsets, 10, small.nnz)
    empty = csr_from_edges(n, [], [])                                        # no edges: nothing to fold
    assert not worth_folding(empty.row_offsets, n, empty.nnz)
    # large graphs always go to the library (it relabels them by degree for the flat SpMM)
    assert worth_folding(dense.row_offsets, n, 1 << 24)


# ---------------------------------------------------------------- reference objects and the plugin seam
class _ForeignGraph:
    """Duck-typed stand-in for the reference's frozen Graph dataclass (graphs.py:34-60)."""

    def __init__(self, g):
        self.n, self.m = g.n, g.m
        self.row_offsets, self.col_indices, self.weights = g.row_offsets, g.col_indices, g.weights


def test_as_graph_views_and_caches_foreign_graphs():
    from paper_2003_01282_b200.graphs import as_graph

    g = golden.graph(golden.load("c1_ba1000.npz"))
    assert as_graph(g) is g
    fg = _ForeignGraph(g)
    v = as_graph(fg)
    assert v == g and v.content_hash() == g.content_hash()
    assert as_graph(fg) is v                       # one view (and one device copy) per caller object
    assert np.shares_memory(v.col_indices, g.col_indices)
    with pytest.raises(TypeError):
        as_graph(object())


def _reference_package():
    import os
    import sys

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if os.path.isdir(path) and path not in sys.path:
        sys.path.insert(0, path)
    return pytest.importorskip("spectrace")


def test_plugin_install_patches_and_restores_the_seam():
    st = _reference_package()
    from paper_2003_01282_b200 import plugin

    orig_collect, orig_make = st.slq._collect_rules, st.operators.make_operator
    orig_desc_make = st.descriptors.make_operator
    h = plugin.install(st)
    assert st.slq._collect_rules is not orig_collect
    assert st.operators.make_operator is not orig_make and st.descriptors.make_operator is not orig_desc_make
    h.uninstall()
    assert st.slq._collect_rules is orig_collect
    assert st.operators.make_operator is orig_make and st.descriptors.make_operator is orig_desc_make


def test_ctypes_stub_loads_and_patches_without_torch():
    import os
    import sys

    st = _reference_package()
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration"))
    import spectrace_gpu

    orig_collect = st.slq._collect_rules
    uninstall = spectrace_gpu.install(st)
    assert st.slq._collect_rules is not orig_collect
    uninstall()
    assert st.slq._collect_rules is orig_collect
    assert spectrace_gpu.launch_count() >= 0
