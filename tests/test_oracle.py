"""Pin the oracle against golden fixtures produced by the real reference (CPU only).

The oracle (oracle/) is the checker for the CUDA path; before trusting it we
show that it reproduces the reference's own outputs: the probe stream
(slq.py:63-72), operator applies (operators.py:65-102), per-probe Lanczos
tridiagonals and Gauss rules (lanczos.py:79-163) and the descriptors
(descriptors.py:124-149, 227-243; wave per SURVEY D3).
"""
import numpy as np
import pytest

import golden
from oracle import pcg64, slq_oracle as O

KIND = {"L": O.LAPLACIAN, "NL": O.NORMALIZED_LAPLACIAN, "P": O.DENSITY}


def test_probe_stream_restatement_matches_reference():
    z = golden.load("probes.npz")
    k = 0
    while f"probe{k}_case" in z:
        seed, i, n = (int(x) for x in z[f"probe{k}_case"])
        st = z[f"probe{k}_state"]
        state, inc = pcg64.pcg64_initial_state(seed, i)
        assert state == (int(st[0]) << 64) | int(st[1])
        assert inc == (int(st[2]) << 64) | int(st[3])
        assert np.array_equal(np.array(pcg64.rademacher(seed, i, n)), z[f"probe{k}_v"].astype(np.float64))
        assert np.array_equal(O.draw_probes(n, seed, [i])[:, 0] * np.sqrt(n) > 0, z[f"probe{k}_v"] > 0)
        k += 1
    assert k >= 6


def test_probe_prefix_property():
    # graph-of-size-n probes are prefixes of longer streams
    a = pcg64.rademacher(5, 2, 301)
    b = pcg64.rademacher(5, 2, 64)
    assert a[:64] == b


@pytest.fixture(scope="module")
def small():
    return golden.load("small.npz")


def _names(z):
    return [str(x) for x in z["names"]]


def test_operator_apply_matches_reference(small):
    for name in _names(small):
        g = golden.graph(small, f"{name}/")
        x = small[f"{name}/x"]
        for kname, kind in KIND.items():
            key = f"{name}/apply_{kname}"
            if key not in small:
                continue
            op = O.make_block_operator(g, kind)
            got = op.apply(x)
            # scipy csr_matvecs == csr_matvec per column: bit-exact
            assert np.array_equal(got, small[key]), (name, kname)


def test_density_requires_edges():
    z = golden.load("small.npz")
    g = golden.graph(z, "empty7/")
    with pytest.raises(ValueError, match="without edges"):
        O.make_block_operator(g, O.DENSITY)


def _check_rules(rules, z, prefix, hi):
    steps = z[f"{prefix}/steps"]
    assert np.array_equal(rules.steps, steps), prefix
    for p in range(steps.size):
        k = int(steps[p])
        a_ref, b_ref = z[f"{prefix}/alpha"][p, :k], z[f"{prefix}/beta"][p, :k - 1]
        assert np.allclose(rules.alpha[p, :k], a_ref, rtol=1e-12, atol=1e-14 * hi), prefix
        assert np.allclose(rules.beta[p, :k - 1], b_ref, rtol=1e-12, atol=1e-14 * hi), prefix
        assert np.max(np.abs(rules.nodes[p, :k] - z[f"{prefix}/nodes"][p, :k]), initial=0) <= 1e-12 * hi, prefix
        assert np.allclose(rules.weights[p, :k], z[f"{prefix}/weights"][p, :k], rtol=1e-9, atol=1e-13), prefix


def test_per_probe_rules_match_reference(small):
    for name in _names(small):
        g = golden.graph(small, f"{name}/")
        for kname, kind in KIND.items():
            for s in (4, 10):
                prefix = f"{name}/{kname}_s{s}"
                if f"{prefix}/steps" not in small:
                    continue
                op = O.make_block_operator(g, kind)
                rules = O.slq_rules(op, 8, s, seed=3)
                _check_rules(rules, small, prefix, op.interval[1])


def test_small_descriptors_match_reference(small):
    t = O.time_grid(1e-2, 1e2, 250)
    for name in _names(small):
        g = golden.graph(small, f"{name}/")
        heat, std = O.heat_trace(g, t, 8, 10, 3)
        assert golden.rel_l2(heat, small[f"{name}/desc/heat"]) <= 1e-12, name
        assert np.allclose(std, small[f"{name}/desc/heat_std"], rtol=1e-8, atol=1e-12), name
        (re, _), (im, _) = O.wave_trace(g, t, 8, 10, 3)
        assert golden.rel_l2(re + 1j * im, small[f"{name}/desc/wave_re"] + 1j * small[f"{name}/desc/wave_im"]) <= 1e-12
        if f"{name}/desc/vnge" in small:
            v, _ = O.vnge(g, 8, 10, 3)
            ref = float(small[f"{name}/desc/vnge"])
            assert abs(v - ref) <= 1e-12 * max(1.0, abs(ref)), name


def test_empty_graph_heat_is_exactly_n(small):
    g = golden.graph(small, "empty7/")
    heat, _ = O.heat_trace(g, O.time_grid(1e-2, 1e2, 16), 12, 4, 1)
    assert np.all(heat == 7.0)


@pytest.mark.parametrize("fname", ["c1_ba1000.npz", "sbm5k.npz", "rmat12.npz"])
def test_medium_graphs_match_reference(fname):
    z = golden.load(fname)
    g = golden.graph(z)
    n_v = z["NL/steps"].size
    s = z["NL/alpha"].shape[1]
    t = O.time_grid(1e-2, 1e2, 250)
    op = O.make_block_operator(g, O.NORMALIZED_LAPLACIAN)
    rules = O.slq_rules(op, n_v, s, 0)
    _check_rules(rules, z, "NL", 2.0)
    heat, _ = O.heat_from_rules(rules, g.n, t)
    assert golden.rel_l2(heat, z["heat"]) <= 1e-12
    (re, _), (im, _) = O.wave_from_rules(rules, g.n, t)
    assert golden.rel_l2(re + 1j * im, z["wave_re"] + 1j * z["wave_im"]) <= 1e-11
    opp = O.make_block_operator(g, O.DENSITY)
    rp = O.slq_rules(opp, n_v, s, 0)
    v, _ = O.vnge_from_rules(rp, g.n)
    assert abs(v - float(z["vnge"])) <= 1e-12 * abs(float(z["vnge"]))


def test_er_batch_sample_matches_reference():
    z = golden.load("erbatch40.npz")
    t = O.time_grid(1e-2, 1e2, 250)
    for k in range(int(z["count"])):
        g = golden.graph(z, f"{k}/")
        heat, _ = O.heat_trace(g, t, 20, 10, 0)
        assert golden.rel_l2(heat, z[f"{k}/heat"]) <= 1e-12, k


def _fold(g):
    """CPU restatement of the isolated-vertex fold (csrc/graph.cu graph_fold): unreferenced empty
    rows leave the graph, one trailing empty row is appended, columns relabelled monotonically."""
    from paper_2003_01282_b200.graphs import Graph

    off = np.asarray(g.row_offsets)
    cols = np.asarray(g.col_indices)
    keep = np.diff(off) > 0
    keep[cols] = True
    newid = np.cumsum(keep) - keep
    nprime = int(keep.sum())
    off_f = np.append(off[:-1][keep], [g.nnz, g.nnz]).astype(np.int64)
    folded = Graph(n=nprime + 1, row_offsets=off_f, col_indices=newid[cols].astype(np.int64),
                   weights=np.array(g.weights, dtype=np.float64), m=g.m)
    return folded, keep, g.n - nprime


@pytest.mark.parametrize("kind", ["L", "NL", "P"])
@pytest.mark.parametrize("weighted", [False, True])
def test_isolated_vertex_fold_identity(kind, weighted):
    # The fold's claim: Lanczos on the folded graph from the folded start vector
    # [z_kept, sqrt(m)] / sqrt(n) gives the tridiagonals of the unfolded run up to rounding.
    from paper_2003_01282_b200.graphs import csr_from_edges

    rng = np.random.default_rng(7)
    n = 400
    live = np.flatnonzero(rng.random(n) < 0.55)
    u, v = live[rng.integers(0, live.size, 900)], live[rng.integers(0, live.size, 900)]
    g = csr_from_edges(n, u, v, rng.uniform(0.5, 2.0, 900) if weighted else None)
    gf, keep, m = _fold(g)
    assert m > 100 and gf.n == n - m + 1
    q0 = O.draw_probes(n, 3, range(6))
    q0f = np.vstack([q0[keep], np.sqrt(m) * np.abs(q0[~keep][:1])])   # |z| = 1/sqrt(n) on every row
    t1 = O.lanczos_block(O.make_block_operator(g, KIND[kind]), q0, 12)
    t2 = O.lanczos_block(O.make_block_operator(gf, KIND[kind]), q0f, 12)
    assert np.array_equal(t1.steps, t2.steps)
    scale = np.abs(t1.alpha).max()
    assert np.max(np.abs(t1.alpha - t2.alpha)) <= 1e-12 * scale
    assert np.max(np.abs(t1.beta - t2.beta)) <= 1e-12 * scale
