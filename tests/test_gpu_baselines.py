"""Trace-identity and spectral baselines on the GPU against golden values
produced by the real reference (``tests/golden/make_golden_baselines.py``):

* ``netlsd_taylor``, ``vnge_taylor`` (corrected / printed), ``vnge_finger`` bar: closed forms of the
  device trace identities -- within 1e-12 relative (fixed-order device sums vs numpy pairwise sums);
* ``extremal_eigenvalues`` (device Lanczos, reorth forced, convergence checks on every prefix from
  one batched device eigensolve), ``vnge_finger`` hat and ``netlsd_linear``: the reference stops when
  the selected Ritz values move by < 1e-8 between checks, so results agree to that tolerance;
  non-converging cases raise ``ConvergenceError`` with the same best estimates;
* ``netlsd_exact`` / ``vnge_exact``: dense spectrum of the device operator (cuSOLVER eigvalsh) vs
  LAPACK -- within 1e-10.
"""
import numpy as np
import pytest

import golden
from paper_2003_01282_b200.descriptors import (TimeGrid, netlsd_exact, netlsd_linear, netlsd_taylor, vnge_exact,
                                               vnge_finger, vnge_taylor)
from paper_2003_01282_b200.errors import ConvergenceError
from paper_2003_01282_b200.graphs import Graph
from paper_2003_01282_b200.lanczos import extremal_eigenvalues
from paper_2003_01282_b200.operators import OperatorKind, make_operator

pytestmark = pytest.mark.gpu

Z = golden.load("baselines.npz")
NAMES = ["ba", "sbm", "rmat", "wtd"]
GRID = TimeGrid(1e-2, 1e2, 250)


def graph(name) -> Graph:
    p = name + "/"
    return Graph(n=int(Z[p + "n"]), row_offsets=np.array(Z[p + "offsets"], dtype=np.int64),
                 col_indices=np.array(Z[p + "cols"], dtype=np.int64),
                 weights=np.array(Z[p + "weights"], dtype=np.float64), m=int(Z[p + "m"]))


def test_grid_matches_fixture():
    assert np.array_equal(GRID.values, Z["t"])


@pytest.mark.parametrize("name", NAMES)
def test_trace_identity_baselines(cuda_device, name):
    g = graph(name)
    p = name + "/"
    assert golden.rel_l2(netlsd_taylor(g, GRID).values, Z[p + "taylor"]) <= 1e-12
    for variant in ("corrected", "printed"):
        ref = float(Z[p + f"vnge_taylor_{variant}"])
        assert abs(vnge_taylor(g, variant).value - ref) <= 1e-12 * abs(ref)
    ref = float(Z[p + "vnge_finger_bar"])
    assert abs(vnge_finger(g, "bar").value - ref) <= 1e-12 * abs(ref)


@pytest.mark.parametrize("name", NAMES)
def test_finger_hat_uses_device_extremal_eigenvalue(cuda_device, name):
    g = graph(name)
    ref = float(Z[name + "/vnge_finger_hat"])
    assert abs(vnge_finger(g, "hat").value - ref) <= 1e-6 * abs(ref)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("key,kind,k,end", [("nl_smallest6", OperatorKind.NORMALIZED_LAPLACIAN, 6, "smallest"),
                                            ("nl_largest6", OperatorKind.NORMALIZED_LAPLACIAN, 6, "largest"),
                                            ("p_largest1", OperatorKind.DENSITY, 1, "largest"),
                                            ("p_largest4", OperatorKind.DENSITY, 4, "largest")])
def test_extremal_eigenvalues_match_reference(cuda_device, name, key, kind, k, end):
    g = graph(name)
    op = make_operator(g, kind)
    p = name + "/"
    hi = op.interval[1]
    if p + key in Z:
        got = extremal_eigenvalues(op, k, end)
        assert got.shape == (k,)
        assert np.all(np.diff(got) >= 0)
        assert np.max(np.abs(got - Z[p + key])) <= 2e-8 * hi
    else:   # the reference exhausts its step cap here: so must we, with the same best estimates
        with pytest.raises(ConvergenceError) as exc:
            extremal_eigenvalues(op, k, end)
        best = exc.value.best_estimates
        ref = Z[p + key + "_nonconverged"]
        assert best.shape == ref.shape
        assert np.max(np.abs(best - ref)) <= 1e-9 * hi


@pytest.mark.parametrize("name", ["ba", "rmat", "wtd"])
def test_netlsd_linear_matches_reference(cuda_device, name):
    g = graph(name)
    got = netlsd_linear(g, GRID, k=40)
    assert golden.rel_l2(got.values, Z[name + "/linear40"]) <= 1e-7
    assert got.method == "linear" and got.params == {"k": 40}


@pytest.mark.parametrize("name", NAMES)
def test_exact_dense_baselines(cuda_device, name):
    g = graph(name)
    p = name + "/"
    assert golden.rel_l2(netlsd_exact(g, GRID).values, Z[p + "exact"]) <= 1e-10
    ref = float(Z[p + "vnge_exact"])
    assert abs(vnge_exact(g).value - ref) <= 1e-10 * abs(ref)


def test_baseline_argument_errors(cuda_device):
    g = graph("ba")
    with pytest.raises(ValueError):
        vnge_taylor(g, "bogus")
    with pytest.raises(ValueError):
        vnge_finger(g, "bogus")
    with pytest.raises(ValueError):
        netlsd_linear(g, GRID, k=0)
    with pytest.raises(ValueError):
        extremal_eigenvalues(make_operator(g, OperatorKind.DENSITY), 0, "largest")
    with pytest.raises(ValueError):
        extremal_eigenvalues(make_operator(g, OperatorKind.DENSITY), 1, "middle")
    empty = Graph(n=5, row_offsets=np.zeros(6, dtype=np.int64), col_indices=np.zeros(0, dtype=np.int64),
                  weights=np.zeros(0), m=0)
    with pytest.raises(ValueError):
        vnge_taylor(empty)
    with pytest.raises(ValueError):
        vnge_finger(empty, "bar")
