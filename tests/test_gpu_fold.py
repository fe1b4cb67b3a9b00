"""Isolated-vertex fold (csrc/graph.cu `graph_fold`, slq_graph_fold_isolated).

Vertices with an empty row that no row references give 0 under every operator kind
(operators.py:76-99), so in the Lanczos recurrence (lanczos.py:122-138) their entries are the probe
sign times one per-probe scalar.  The fold runs the recurrence on the graph without them plus one
trailing row carrying sqrt(m) times that scalar.  Dot products then agree with the unfolded run to
rounding; these tests pin that (tridiagonals, rules, descriptors vs the oracle) and the fold's
bookkeeping (which vertices fold, chunk independence, dropping the fold).
"""
import numpy as np
import pytest
import torch

import golden
from oracle import slq_oracle as O
from paper_2003_01282_b200 import _lib
from paper_2003_01282_b200.device import DeviceGraph
from paper_2003_01282_b200.descriptors import TimeGrid
from paper_2003_01282_b200.graphs import csr_from_edges

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-9
FP32_TOL = 1e-4
GRID = TimeGrid(1e-2, 1e2, 250)
KINDS = ["laplacian", "normalized_laplacian", "density"]


def graph_with_isolated(n, m, iso_frac, seed, weighted=False):
    """Random graph on n vertices whose edges avoid a random iso_frac of them (always including the
    first and the last vertex, so the fold's remap is exercised at both ends)."""
    rng = np.random.default_rng(seed)
    iso = rng.random(n) < iso_frac
    iso[0] = iso[-1] = True
    live = np.flatnonzero(~iso)
    u = live[rng.integers(0, live.size, m)]
    v = live[rng.integers(0, live.size, m)]
    w = rng.uniform(0.5, 2.0, m) if weighted else None
    return csr_from_edges(n, u, v, w)


def empty_rows(g):
    return int(np.count_nonzero(np.diff(np.asarray(g.row_offsets)) == 0))


@pytest.fixture(scope="module")
def rmat12():
    return golden.graph(golden.load("rmat12.npz"))


def test_fold_counts_unreferenced_empty_rows(cuda_device, rmat12):
    dg = DeviceGraph(rmat12, cuda_device)
    assert dg.folded == empty_rows(rmat12) > 0
    assert DeviceGraph(rmat12, cuda_device, fold=None).folded == 0
    # below the threshold nothing folds; a negative fraction drops the fold
    assert DeviceGraph(rmat12, cuda_device, fold=None).fold_isolated(0.5) == 0
    assert dg.fold_isolated(-1.0) == 0 and dg.folded == 0


def test_fold_skips_empty_rows_that_are_referenced(cuda_device):
    import ctypes

    # a non-symmetric CSR through the C ABI: row 1 is empty but row 0 references column 1, so only
    # row 3 may fold
    off = torch.tensor([0, 2, 2, 3, 3], dtype=torch.int64, device=cuda_device)
    cols = torch.tensor([1, 2, 0], dtype=torch.int64, device=cuda_device)
    lib = _lib.load()
    h = ctypes.c_void_p()
    _lib.check(lib.slq_graph_create(4, 3, _lib.ptr(off), _lib.ptr(cols), None, _lib.stream_handle(), ctypes.byref(h)))
    try:
        m = ctypes.c_int64()
        _lib.check(lib.slq_graph_fold_isolated(h, 0.0, ctypes.byref(m)))
        assert m.value == 1
    finally:
        lib.slq_graph_destroy(h)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("weighted", [False, True])
def test_fold_tridiagonals_match_unfolded_fp64(cuda_device, kind, weighted):
    g = graph_with_isolated(6000, 20000, 0.4, seed=3, weighted=weighted)
    folded = DeviceGraph(g, cuda_device)
    plain = DeviceGraph(g, cuda_device, fold=None)
    assert folded.folded == empty_rows(g) > 2000 and plain.folded == 0
    a1, b1, s1 = folded.tridiagonals(kind, 5, 0, 40, 15)
    a2, b2, s2 = plain.tridiagonals(kind, 5, 0, 40, 15)
    assert torch.equal(s1, s2)
    a1, b1, a2, b2 = (x.cpu().numpy() for x in (a1, b1, a2, b2))
    scale = np.abs(a2).max()
    assert np.abs(a1 - a2).max() <= 1e-12 * scale
    assert np.abs(b1 - b2).max() <= 1e-12 * scale


@pytest.mark.parametrize("dtype,tol", [("f64", FP64_TOL), ("f32", FP32_TOL)])
def test_fold_descriptors_match_oracle(cuda_device, rmat12, dtype, tol):
    dg = DeviceGraph(rmat12, cuda_device)
    assert dg.folded > 0
    nl = dg.rules("normalized_laplacian", 0, 0, 16, 15, dtype=dtype)
    vals, _ = nl.integrate(np.array(GRID.values), [_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM])
    vals = vals.cpu().numpy()
    nl.check()
    ref_h, _ = O.heat_trace(rmat12, GRID.values, 16, 15, 0)
    (ref_re, _), (ref_im, _) = O.wave_trace(rmat12, GRID.values, 16, 15, 0)
    assert golden.rel_l2(vals[0], ref_h) <= tol
    assert golden.rel_l2(vals[1] + 1j * vals[2], ref_re + 1j * ref_im) <= tol
    p = dg.rules("density", 0, 0, 16, 15, dtype=dtype)
    v, _ = p.integrate(None, [_lib.FN_XLOGX])
    ref_v, _ = O.vnge(rmat12, 16, 15, 0)
    assert abs(-float(v.cpu().numpy()[0, 0]) - ref_v) <= tol * abs(ref_v)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fold_rules_chunk_and_range_independent(cuda_device, dtype):
    g = graph_with_isolated(3000, 9000, 0.3, seed=11)
    dg = DeviceGraph(g, cuda_device)
    assert dg.folded > 0
    whole = dg.rules("normalized_laplacian", 2, 0, 24, 12, dtype=dtype)
    parts = [dg.rules("normalized_laplacian", 2, b, 8, 12, dtype=dtype) for b in (0, 8, 16)]
    assert torch.equal(whole.nodes, torch.cat([p.nodes for p in parts]))
    assert torch.equal(whole.weights, torch.cat([p.weights for p in parts]))


def test_fold_dropped_reproduces_unfolded_bitwise(cuda_device):
    g = graph_with_isolated(2000, 6000, 0.5, seed=1)
    dg = DeviceGraph(g, cuda_device)
    assert dg.folded > 0
    dg.fold_isolated(-1.0)
    a1, b1, _ = dg.tridiagonals("density", 0, 0, 10, 10)
    a2, b2, _ = DeviceGraph(g, cuda_device, fold=None).tridiagonals("density", 0, 0, 10, 10)
    assert torch.equal(a1, a2) and torch.equal(b1, b2)


def test_fold_device_rmat_matches_host_graph(cuda_device):
    from paper_2003_01282_b200 import synth

    dg = DeviceGraph.rmat(13, 16, seed=3, device=cuda_device)
    g = synth.rmat_device_reference(13, 16, seed=3)
    host = DeviceGraph(g, cuda_device)
    assert dg.folded == host.folded == empty_rows(g) > 0
    a1, b1, s1 = dg.tridiagonals("normalized_laplacian", 0, 0, 16, 15, dtype="f32")
    a2, b2, s2 = host.tridiagonals("normalized_laplacian", 0, 0, 16, 15, dtype="f32")
    assert torch.equal(a1, a2) and torch.equal(b1, b2) and torch.equal(s1, s2)
    ref_h, _ = O.heat_trace(g, GRID.values, 16, 15, 0)
    vals, _ = dg.rules("normalized_laplacian", 0, 0, 16, 15, dtype="f32").integrate(np.array(GRID.values),
                                                                                   [_lib.FN_HEAT])
    assert golden.rel_l2(vals.cpu().numpy()[0], ref_h) <= FP32_TOL


@pytest.mark.parametrize("kind", KINDS)
def test_fold_nearly_all_isolated(cuda_device, kind):
    # one edge among 1000 vertices: the folded recurrence runs on 3 rows (the edge's endpoints and
    # the trailing row) and must break down at the same step as the unfolded one
    g = csr_from_edges(1000, [3], [998])
    folded = DeviceGraph(g, cuda_device)
    plain = DeviceGraph(g, cuda_device, fold=None)
    assert folded.folded == 998
    a1, b1, s1 = folded.tridiagonals(kind, 0, 0, 20, 15)
    a2, b2, s2 = plain.tridiagonals(kind, 0, 0, 20, 15)
    assert torch.equal(s1, s2)
    assert np.allclose(a1.cpu().numpy(), a2.cpu().numpy(), rtol=0, atol=1e-13)
    assert np.allclose(b1.cpu().numpy(), b2.cpu().numpy(), rtol=0, atol=1e-13)
    r1 = folded.rules(kind, 0, 0, 20, 15)
    r2 = plain.rules(kind, 0, 0, 20, 15)
    assert np.allclose(r1.nodes.cpu().numpy(), r2.nodes.cpu().numpy(), rtol=0, atol=1e-12)
    assert np.allclose(r1.weights.cpu().numpy(), r2.weights.cpu().numpy(), rtol=0, atol=1e-12)


def test_large_graph_without_isolated_vertices_is_degree_ordered(cuda_device):
    """Large unit-weight graphs get the fold's degree order even with NO isolated vertex (m = 0: the
    trailing row stays zero), because the flat SpMM (csrc/spmm_flat.cu) needs it.  The relabelled run
    (flat SpMM, prescaled gathers) matches the unfolded run (warp-per-row SpMM) and the CPU oracle."""
    rng = np.random.default_rng(11)
    n = 1 << 19
    ring = np.arange(n, dtype=np.int64)
    u = np.concatenate([ring, rng.integers(0, n, 17 * n)])
    v = np.concatenate([(ring + 1) % n, rng.integers(0, n, 17 * n)])
    g = csr_from_edges(n, u, v)
    assert g.nnz >= 1 << 24 and int(np.min(np.diff(np.asarray(g.row_offsets)))) >= 2
    dg = DeviceGraph(g, cuda_device)
    assert dg.folded == 0                       # nothing folded away ...
    lens, rows = dg.lanczos_row_lengths(64)
    assert rows == n + 1                        # ... but the recurrence runs on the relabelled graph
    assert np.all(np.diff(lens) <= 0) and lens[0] == int(np.max(np.diff(np.asarray(g.row_offsets))))
    plain = DeviceGraph(g, cuda_device, fold=None)
    t = np.array(GRID.values)
    for kind, fn in (("normalized_laplacian", _lib.FN_HEAT), ("density", _lib.FN_XLOGX)):
        a = dg.rules(kind, 0, 0, 8, 12, dtype="f32")
        b = plain.rules(kind, 0, 0, 8, 12, dtype="f32")
        a.check()
        b.check()
        va, _ = a.integrate(t if fn == _lib.FN_HEAT else None, [fn])
        vb, _ = b.integrate(t if fn == _lib.FN_HEAT else None, [fn])
        assert golden.rel_l2(va.cpu().numpy(), vb.cpu().numpy()) <= 1e-5
        if fn == _lib.FN_HEAT:
            ref, _ = O.heat_trace(g, GRID.values, 8, 12, 0, threads=8)
            assert golden.rel_l2(va[0].cpu().numpy(), ref) <= FP32_TOL
