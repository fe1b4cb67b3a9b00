"""GPU parity ladder: the CUDA path through the C ABI vs the golden
fixtures made by the real reference and vs the oracle.

Tolerances (north star): fp64 descriptors within 1e-9 relative (rel-l2, the
reference's relative_error); fp32 vector storage within 1e-4.  Integer/bit work
(probes, degrees, the operator apply) is bit-exact.
"""
import numpy as np
import pytest
import torch

import golden
from oracle import pcg64, slq_oracle as O
from paper_2003_01282_b200 import _lib
from paper_2003_01282_b200.descriptors import (TimeGrid, netlsd_heat_wave_slq, netlsd_slq, vnge_slq)
from paper_2003_01282_b200.device import DeviceGraph
from paper_2003_01282_b200.graphs import csr_from_edges
from paper_2003_01282_b200.slq import SlqConfig

pytestmark = pytest.mark.gpu

KIND = {"L": "laplacian", "NL": "normalized_laplacian", "P": "density"}
FP64_TOL = 1e-9
FP32_TOL = 1e-4
GRID = TimeGrid(1e-2, 1e2, 250)


@pytest.fixture(scope="module")
def small():
    return golden.load("small.npz")


def names(z):
    return [str(x) for x in z["names"]]


def test_library_runs_on_device(cuda_device):
    before = _lib.launch_count()
    g = csr_from_edges(3, [0, 1], [1, 2])
    DeviceGraph(g, cuda_device).apply("normalized_laplacian", np.eye(3))
    assert _lib.launch_count() > before


# 1. probes: device bits == reference stream (slq.py:63-72)
@pytest.mark.parametrize("seed,begin,count,n", [(0, 0, 5, 1), (0, 0, 33, 2), (3, 7, 40, 129), (123, 90, 10, 1001),
                                                (2**40 + 3, 17, 3, 4097)])
def test_probes_bit_exact(cuda_device, seed, begin, count, n):
    out = torch.zeros((n, count), dtype=torch.float64, device=cuda_device)
    _lib.check(_lib.load().slq_probes(seed, begin, count, n, out.data_ptr(), count, _lib.stream_handle()))
    got = out.cpu().numpy()
    for j in range(count):
        i = begin + j
        if n <= 300:
            ref = np.array(pcg64.rademacher(seed, i, n))
        else:
            rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(i,)))
            ref = rng.integers(0, 2, size=n).astype(np.float64) * 2.0 - 1.0
        assert np.array_equal(got[:, j], ref), (seed, i, n)


def test_probes_golden(cuda_device):
    z = golden.load("probes.npz")
    k = 0
    while f"probe{k}_case" in z:
        seed, i, n = (int(x) for x in z[f"probe{k}_case"])
        out = torch.zeros((n, 1), dtype=torch.float64, device=cuda_device)
        _lib.check(_lib.load().slq_probes(seed, i, 1, n, out.data_ptr(), 1, _lib.stream_handle()))
        assert np.array_equal(out[:, 0].cpu().numpy(), z[f"probe{k}_v"].astype(np.float64))
        k += 1


# 2. degrees / dinv / trL exact (operators.py:58-62, 84-86, 93)
def test_degrees_exact(cuda_device, small):
    for name in names(small):
        g = golden.graph(small, f"{name}/")
        if g.n == 0:
            continue
        dg = DeviceGraph(g, cuda_device)
        d, dinv = dg.degrees()
        ref_d = O.degrees(g)
        assert np.array_equal(d.cpu().numpy(), ref_d), name
        pos = ref_d > 0
        ref_dinv = np.zeros(g.n)
        ref_dinv[pos] = 1.0 / np.sqrt(ref_d[pos])
        assert np.array_equal(dinv.cpu().numpy(), ref_dinv), name
        # unweighted: integer degrees, exact; weighted: numpy's pairwise order differs by <= 1 ulp
        if g.is_unweighted():
            assert dg.info.trace_l == float(ref_d.sum())
        else:
            assert abs(dg.info.trace_l - float(ref_d.sum())) <= 4e-16 * float(ref_d.sum())
        assert dg.info.isolated == int((ref_d == 0).sum())


# 3. operator apply: bit-identical to the reference closure (golden apply_* arrays)
def test_operator_apply_bit_exact(cuda_device, small):
    for name in names(small):
        g = golden.graph(small, f"{name}/")
        dg = DeviceGraph(g, cuda_device)
        x = small[f"{name}/x"]
        for kname, kind in KIND.items():
            key = f"{name}/apply_{kname}"
            if key not in small:
                with pytest.raises(ValueError, match="without edges"):
                    dg.apply(kind, x)
                continue
            got = dg.apply(kind, x)
            if kname == "P" and not g.is_unweighted():
                # scale = 1/tr L: numpy sums weighted degrees pairwise, the device in a fixed tree;
                # tr L may differ in the last bit, so P differs by <= 1 ulp of scale
                assert np.allclose(got, small[key], rtol=4.5e-16, atol=0), (name, kname)
            else:
                assert np.array_equal(got, small[key]), (name, kname, np.max(np.abs(got - small[key])))


def test_operator_apply_many_columns_bit_exact(cuda_device):
    z = golden.load("rmat12.npz")
    g = golden.graph(z)
    x = np.random.default_rng(0).standard_normal((g.n, 70))
    for kind, okind in (("normalized_laplacian", O.NORMALIZED_LAPLACIAN), ("density", O.DENSITY),
                        ("laplacian", O.LAPLACIAN)):
        got = DeviceGraph(g, cuda_device).apply(kind, x)
        ref = O.make_block_operator(g, okind).apply(x)
        short = np.diff(g.row_offsets) <= 1024      # longer rows are summed in segments
        assert np.array_equal(got[short], ref[short]), kind
        assert np.allclose(got[~short], ref[~short], rtol=1e-13, atol=1e-15 * np.abs(ref).max()), kind


# 4./5. per-probe tridiagonals and rules vs the reference
def check_rules(dg, kind, z, prefix, n_v, s, seed, hi):
    alpha, beta, st = dg.tridiagonals(kind, seed, 0, n_v, s)
    rules = dg.rules(kind, seed, 0, n_v, s)
    steps = z[f"{prefix}/steps"]
    assert np.array_equal(st.cpu().numpy(), steps), prefix
    a, b = alpha.cpu().numpy(), beta.cpu().numpy()
    nodes, weights = rules.nodes.cpu().numpy(), rules.weights.cpu().numpy()
    for p in range(n_v):
        k = int(steps[p])
        assert np.allclose(a[p, :k], z[f"{prefix}/alpha"][p, :k], rtol=1e-11, atol=1e-13 * hi), (prefix, p)
        assert np.allclose(b[p, :k - 1], z[f"{prefix}/beta"][p, :k - 1], rtol=1e-11, atol=1e-13 * hi), (prefix, p)
        assert np.max(np.abs(nodes[p, :k] - z[f"{prefix}/nodes"][p, :k]), initial=0) <= 1e-11 * hi, (prefix, p)
        assert np.allclose(weights[p, :k], z[f"{prefix}/weights"][p, :k], rtol=1e-8, atol=1e-12), (prefix, p)


def test_small_graph_rules_match_reference(cuda_device, small):
    for name in names(small):
        g = golden.graph(small, f"{name}/")
        dg = DeviceGraph(g, cuda_device)
        for kname, kind in KIND.items():
            for s in (4, 10):
                prefix = f"{name}/{kname}_s{s}"
                if f"{prefix}/steps" not in small:
                    continue
                hi = float(small[f"{prefix}/interval"][1])
                check_rules(dg, kind, small, prefix, 8, s, 3, hi)


@pytest.mark.parametrize("fname", ["c1_ba1000.npz", "sbm5k.npz", "rmat12.npz"])
def test_medium_graph_rules_match_reference(cuda_device, fname):
    z = golden.load(fname)
    g = golden.graph(z)
    dg = DeviceGraph(g, cuda_device)
    n_v, s = z["NL/alpha"].shape
    check_rules(dg, "normalized_laplacian", z, "NL", n_v, s, 0, 2.0)
    check_rules(dg, "density", z, "P", n_v, s, 0, 1.0)


# 6. descriptors vs the reference (rel-l2, the reference's relative_error)
def test_small_graph_descriptors(cuda_device, small):
    for name in names(small):
        g = golden.graph(small, f"{name}/")
        cfg = SlqConfig(n_v=8, s=10, seed=3)
        heat, wave = netlsd_heat_wave_slq(g, GRID, cfg)
        assert golden.rel_l2(heat.values, small[f"{name}/desc/heat"]) <= FP64_TOL, name
        assert np.allclose(heat.std_errors, small[f"{name}/desc/heat_std"], rtol=1e-7, atol=1e-10), name
        ref_w = small[f"{name}/desc/wave_re"] + 1j * small[f"{name}/desc/wave_im"]
        assert golden.rel_l2(wave.values, ref_w) <= FP64_TOL, name
        assert heat.graph_hash == str(small[f"{name}/desc/graph_hash"])
        if f"{name}/desc/vnge" in small:
            v = vnge_slq(g, cfg)
            ref = float(small[f"{name}/desc/vnge"])
            assert abs(v.value - ref) <= FP64_TOL * max(abs(ref), 1e-300) or abs(v.value - ref) <= 1e-13, name
        else:
            with pytest.raises(ValueError, match="without edges"):
                vnge_slq(g, cfg)


@pytest.mark.parametrize("fname", ["c1_ba1000.npz", "sbm5k.npz", "rmat12.npz"])
def test_medium_graph_descriptors(cuda_device, fname):
    z = golden.load(fname)
    g = golden.graph(z)
    n_v, s = z["NL/alpha"].shape
    cfg = SlqConfig(n_v=n_v, s=s, seed=0)
    heat, wave = netlsd_heat_wave_slq(g, GRID, cfg)
    assert golden.rel_l2(heat.values, z["heat"]) <= FP64_TOL
    assert golden.max_rel(heat.values, z["heat"]) <= FP64_TOL
    assert golden.rel_l2(wave.values, z["wave_re"] + 1j * z["wave_im"]) <= FP64_TOL
    v = vnge_slq(g, cfg)
    assert abs(v.value - float(z["vnge"])) <= FP64_TOL * abs(float(z["vnge"]))
    # fp32 vector storage (fp64 reductions): 1e-4
    h32, w32 = netlsd_heat_wave_slq(g, GRID, cfg, dtype="f32")
    assert golden.rel_l2(h32.values, z["heat"]) <= FP32_TOL
    assert golden.rel_l2(w32.values, z["wave_re"] + 1j * z["wave_im"]) <= FP32_TOL
    v32 = vnge_slq(g, cfg, dtype="f32")
    assert abs(v32.value - float(z["vnge"])) <= FP32_TOL * abs(float(z["vnge"]))


def test_er_batch_sample_descriptors(cuda_device):
    z = golden.load("erbatch40.npz")
    cfg = SlqConfig(n_v=20, s=10, seed=0)
    for k in range(int(z["count"])):
        g = golden.graph(z, f"{k}/")
        h = netlsd_slq(g, GRID, cfg)
        assert golden.rel_l2(h.values, z[f"{k}/heat"]) <= FP64_TOL, k


# determinism: per-probe rules independent of chunk width / probe range (reference prefix property)
def test_rules_independent_of_chunking(cuda_device):
    z = golden.load("sbm5k.npz")
    dg = DeviceGraph(golden.graph(z), cuda_device)
    a_full, b_full, s_full = dg.tridiagonals("normalized_laplacian", 0, 0, 70, 15)
    a1, b1, s1 = dg.tridiagonals("normalized_laplacian", 0, 0, 33, 15)
    a2, b2, s2 = dg.tridiagonals("normalized_laplacian", 0, 33, 37, 15)
    assert torch.equal(a_full, torch.cat([a1, a2]))
    assert torch.equal(b_full, torch.cat([b1, b2]))
    assert torch.equal(s_full, torch.cat([s1, s2]))
    a3, _, _ = dg.tridiagonals("normalized_laplacian", 0, 0, 70, 15)
    assert torch.equal(a_full, a3)
    # narrow chunks (<= 32 columns: 12-row-slot step kernel, half-warp SpMM for <= 16) agree
    # bitwise among themselves and with the wide class to rounding
    n32, nb32, ns32 = dg.tridiagonals("normalized_laplacian", 0, 0, 32, 15)
    for begin, count in ((0, 16), (16, 9), (31, 1)):
        a4, b4, s4 = dg.tridiagonals("normalized_laplacian", 0, begin, count, 15)
        assert torch.equal(a4, n32[begin:begin + count]) and torch.equal(b4, nb32[begin:begin + count])
        assert torch.equal(s4, ns32[begin:begin + count])
    assert torch.equal(ns32, s_full[:32])
    assert torch.allclose(n32, a_full[:32], rtol=1e-13, atol=1e-14)
    for kind in ("normalized_laplacian", "density"):
        f_full, _, _ = dg.tridiagonals(kind, 0, 0, 32, 15, dtype="f32")
        f_narrow, _, _ = dg.tridiagonals(kind, 0, 24, 8, 15, dtype="f32")
        assert torch.equal(f_narrow, f_full[24:32]), kind
        f_wide, _, _ = dg.tridiagonals(kind, 0, 0, 40, 15, dtype="f32")
        assert torch.allclose(f_wide[:32], f_full, rtol=1e-5, atol=1e-6), kind


# edge cases the reference tests
def test_empty_graph_heat_is_exactly_n(cuda_device):
    g = csr_from_edges(7, [], [])
    h = netlsd_slq(g, TimeGrid(1e-2, 1e2, 16), SlqConfig(n_v=12, s=4, seed=1))
    assert np.all(h.values == 7.0)


def test_single_vertex_and_steps_beyond_n(cuda_device):
    g = csr_from_edges(1, [], [])
    h = netlsd_slq(g, TimeGrid(1e-2, 1e2, 8), SlqConfig(n_v=3, s=10, seed=0))
    assert np.all(h.values == 1.0)
    g2 = csr_from_edges(3, [0, 1], [1, 2])
    h2 = netlsd_slq(g2, GRID, SlqConfig(n_v=5, s=10, seed=0))
    ref, _ = O.heat_trace(g2, GRID.values, 5, 10, 0)
    assert golden.rel_l2(h2.values, ref) <= FP64_TOL


def test_k2_vnge_is_zero(cuda_device):
    v = vnge_slq(csr_from_edges(2, [0], [1]), SlqConfig(n_v=8, s=5, seed=2))
    assert abs(v.value) <= 1e-10


def test_nonfinite_f_raises(cuda_device):
    from paper_2003_01282_b200.operators import OperatorKind, make_operator
    from paper_2003_01282_b200.slq import slq_trace

    op = make_operator(csr_from_edges(3, [0, 1], [1, 2]), OperatorKind.NORMALIZED_LAPLACIAN)
    with pytest.raises(ValueError, match="non-finite"):
        slq_trace(op, lambda x: np.full_like(x, np.nan), SlqConfig(n_v=4, s=4, seed=0))


def test_weighted_graph_matches_oracle(cuda_device):
    rng = np.random.default_rng(9)
    n = 300
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(iu.size) < 0.05
    g = csr_from_edges(n, iu[keep], ju[keep], rng.uniform(0.5, 1.5, int(keep.sum())))
    cfg = SlqConfig(n_v=40, s=12, seed=4)
    heat, wave = netlsd_heat_wave_slq(g, GRID, cfg)
    ref, _ = O.heat_trace(g, GRID.values, 40, 12, 4)
    assert golden.rel_l2(heat.values, ref) <= FP64_TOL
    v = vnge_slq(g, cfg)
    ref_v, _ = O.vnge(g, 40, 12, 4)
    assert abs(v.value - ref_v) <= FP64_TOL * abs(ref_v)


def test_lanczos_from_start_vector_matches_oracle(cuda_device):
    from paper_2003_01282_b200.lanczos import lanczos_tridiagonalize, quadrature_rule
    from paper_2003_01282_b200.operators import OperatorKind, make_operator

    z = golden.load("c1_ba1000.npz")
    g = golden.graph(z)
    op = make_operator(g, OperatorKind.NORMALIZED_LAPLACIAN)
    q0 = O.draw_probes(g.n, 0, [0])[:, 0]
    tri = lanczos_tridiagonalize(op, q0, 10)
    assert tri.steps == int(z["NL/steps"][0])
    assert np.allclose(tri.alpha, z["NL/alpha"][0], rtol=1e-12)
    rule = quadrature_rule(tri)
    assert np.allclose(rule.weights, z["NL/weights"][0], rtol=1e-8, atol=1e-13)
    with pytest.raises(ValueError, match="unit norm"):
        lanczos_tridiagonalize(op, 2 * q0, 10)


# full-size configs through size-independent properties + oracle on a probe subset
def test_c2_sbm100k_heat_wave_vs_oracle(cuda_device):
    from paper_2003_01282_b200 import synth

    g = synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0)
    cfg = SlqConfig(n_v=100, s=15, seed=0)
    heat, wave = netlsd_heat_wave_slq(g, GRID, cfg)
    # oracle on the first 12 probes; prefix property makes this a per-probe check
    op = O.make_block_operator(g, O.NORMALIZED_LAPLACIAN)
    rules = O.slq_rules(op, 12, 15, 0, threads=4)
    dg = DeviceGraph(g, cuda_device)
    dr = dg.rules("normalized_laplacian", 0, 0, 12, 15)
    assert np.max(np.abs(dr.nodes.cpu().numpy() - rules.nodes)) <= 1e-11 * 2.0
    assert np.allclose(dr.weights.cpu().numpy(), rules.weights, rtol=1e-8, atol=1e-12)
    h12, _ = O.heat_from_rules(rules, g.n, GRID.values)
    got12 = netlsd_slq(g, GRID, SlqConfig(n_v=12, s=15, seed=0))
    assert golden.rel_l2(got12.values, h12) <= FP64_TOL
    # t -> 0 limit: every rule integrates 1, so h_t -> n (a size-independent check)
    assert abs(heat.values[0] - g.n) / g.n < 0.03
    assert np.all(np.isfinite(wave.values))


def test_long_runs_use_fallback_kernels_and_match_oracle(cuda_device):
    # s = 24 > 17: CGS blocks beyond 16 basis vectors take the non-staged kernels
    z = golden.load("sbm5k.npz")
    g = golden.graph(z)
    ref, _ = O.heat_trace(g, GRID.values, 6, 24, 0)
    h = netlsd_slq(g, GRID, SlqConfig(n_v=6, s=24, seed=0))
    assert golden.rel_l2(h.values, ref) <= FP64_TOL
    ref_v, _ = O.vnge(g, 6, 24, 0)
    assert abs(vnge_slq(g, SlqConfig(n_v=6, s=24, seed=0)).value - ref_v) <= FP64_TOL * abs(ref_v)


def test_flat_kernels_match_staged(cuda_device, tmp_path):
    # the non-staged streaming kernels (SLQ_STAGED=0) give the same rules within fp64 rounding
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); import numpy as np, golden; "
            "from paper_2003_01282_b200.device import DeviceGraph; "
            "g = golden.graph(golden.load('rmat12.npz')); r = DeviceGraph(g).rules('density', 0, 0, 16, 15); "
            f"np.save({str(tmp_path / 'flat_nodes.npy')!r}, r.nodes.cpu().numpy())")
    env = dict(__import__('os').environ, SLQ_STAGED="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env,
                   cwd=__import__('os').path.dirname(__import__('os').path.dirname(__file__)))
    flat = np.load(tmp_path / "flat_nodes.npy")
    g = golden.graph(golden.load("rmat12.npz"))
    staged = DeviceGraph(g, cuda_device).rules("density", 0, 0, 16, 15).nodes.cpu().numpy()
    assert np.max(np.abs(flat - staged)) <= 1e-14


def _hub_graph():
    rng = np.random.default_rng(21)
    n = 6000
    u = [np.zeros(4500, dtype=np.int64), np.full(1500, 7, dtype=np.int64)]
    v = [rng.choice(np.arange(1, n), 4500, replace=False), rng.choice(np.arange(8, n), 1500, replace=False)]
    iu = rng.integers(0, n, 30000)
    iv = rng.integers(0, n, 30000)
    return csr_from_edges(n, np.concatenate(u + [iu]), np.concatenate(v + [iv]))


def test_long_rows_split_into_segments(cuda_device):
    # rows with > 1024 nonzeros are summed in 1024-nonzero segments (R-MAT hubs); short rows stay
    # bit-exact, long rows agree to rounding
    g = _hub_graph()
    deg = np.diff(g.row_offsets)
    assert deg.max() > 4096 and (deg > 1024).sum() >= 2
    x = np.random.default_rng(5).standard_normal((g.n, 37))
    dg = DeviceGraph(g, cuda_device)
    for kind, okind in (("normalized_laplacian", O.NORMALIZED_LAPLACIAN), ("density", O.DENSITY)):
        got = dg.apply(kind, x)
        ref = O.make_block_operator(g, okind).apply(x)
        short = deg <= 1024
        assert np.array_equal(got[short], ref[short]), kind
        assert np.allclose(got[~short], ref[~short], rtol=1e-13, atol=1e-15 * np.abs(ref).max()), kind
    cfg = SlqConfig(n_v=24, s=15, seed=2)
    heat, wave = netlsd_heat_wave_slq(g, GRID, cfg)
    rh, _ = O.heat_trace(g, GRID.values, 24, 15, 2)
    assert golden.rel_l2(heat.values, rh) <= FP64_TOL
    v = vnge_slq(g, cfg)
    rv, _ = O.vnge(g, 24, 15, 2)
    assert abs(v.value - rv) <= FP64_TOL * abs(rv)
    # long rows under every SpMM mapping: half-warp (<= 16 probes), full warp, 2/4 probes per lane
    for n_v, dtype, tol in ((12, "f64", FP64_TOL), (12, "f32", FP32_TOL), (70, "f64", FP64_TOL),
                            (100, "f32", FP32_TOL)):
        c = SlqConfig(n_v=n_v, s=15, seed=2)
        h = netlsd_slq(g, GRID, c, dtype=dtype)
        ref, _ = O.heat_trace(g, GRID.values, n_v, 15, 2)
        assert golden.rel_l2(h.values, ref) <= tol, (n_v, dtype)


# batched block-diagonal path (C3)
def test_batched_er_sample_matches_reference(cuda_device):
    from paper_2003_01282_b200.batched import netlsd_slq_batch

    z = golden.load("erbatch40.npz")
    graphs = [golden.graph(z, f"{k}/") for k in range(int(z["count"]))]
    cfg = SlqConfig(n_v=20, s=10, seed=0)
    vals, stds = netlsd_slq_batch(graphs, GRID, cfg)
    vals32, _ = netlsd_slq_batch(graphs, GRID, cfg, dtype="f32")
    for k in range(len(graphs)):
        ref = z[f"{k}/heat"]
        assert golden.rel_l2(vals[k], ref) <= FP64_TOL, k
        assert np.allclose(stds[k], z[f"{k}/heat_std"], rtol=1e-6, atol=1e-10), k
        assert golden.rel_l2(vals32[k], ref) <= FP32_TOL, k


def test_batched_matches_single_graph_path_and_vnge(cuda_device):
    from paper_2003_01282_b200 import synth
    from paper_2003_01282_b200.batched import netlsd_slq_batch, vnge_slq_batch

    graphs = synth.er_batch(30, seed=7) + [csr_from_edges(5, [0, 1, 2, 3], [1, 2, 3, 4]),
                                          csr_from_edges(3, [0, 1], [1, 2])]   # n < s: steps clamp
    cfg = SlqConfig(n_v=16, s=12, seed=4)
    vals, _ = netlsd_slq_batch(graphs, GRID, cfg)
    ents, _ = vnge_slq_batch(graphs, cfg)
    for k, g in enumerate(graphs):
        single = netlsd_slq(g, GRID, cfg).values
        assert golden.rel_l2(vals[k], single) <= 1e-12, k
        rv, _ = O.vnge(g, 16, 12, 4)
        assert abs(ents[k] - rv) <= FP64_TOL * max(abs(rv), 1e-12), k
    with pytest.raises(ValueError, match="without edges"):
        vnge_slq_batch(graphs + [csr_from_edges(4, [], [])], cfg)


# device R-MAT generator + CSR build (C4/C5 workloads) vs its host restatement and the oracle
@pytest.mark.parametrize("scale,ef,seed", [(8, 4, 1), (12, 16, 0), (15, 16, 7)])
def test_device_rmat_csr_matches_host_restatement(cuda_device, scale, ef, seed):
    from paper_2003_01282_b200 import synth

    dg = DeviceGraph.rmat(scale, ef, seed=seed, device=cuda_device)
    ref = synth.rmat_device_reference(scale, ef, seed=seed)
    off, cols = dg.csr()
    assert dg.n == ref.n and dg.nnz == ref.nnz
    assert np.array_equal(off, ref.row_offsets)
    assert np.array_equal(cols.astype(np.int64), ref.col_indices)


def test_device_rmat_descriptors_match_oracle(cuda_device):
    from paper_2003_01282_b200 import synth

    dg = DeviceGraph.rmat(12, 16, seed=2, device=cuda_device)
    g = synth.rmat_device_reference(12, 16, seed=2)
    host = DeviceGraph(g, cuda_device)
    a1, b1, s1 = dg.tridiagonals("normalized_laplacian", 0, 0, 24, 15)
    a2, b2, s2 = host.tridiagonals("normalized_laplacian", 0, 0, 24, 15)
    assert torch.equal(a1, a2) and torch.equal(b1, b2) and torch.equal(s1, s2)
    rules = dg.rules("normalized_laplacian", 0, 0, 8, 15)
    vals, _ = rules.integrate(np.array(GRID.values), [_lib.FN_HEAT])
    ref, _ = O.heat_trace(g, GRID.values, 8, 15, 0)
    assert golden.rel_l2(vals.cpu().numpy()[0], ref) <= FP64_TOL
    p = dg.rules("density", 0, 0, 8, 15)
    v, _ = p.integrate(None, [_lib.FN_XLOGX])
    ref_v, _ = O.vnge(g, 8, 15, 0)
    assert abs(-float(v.cpu().numpy()[0, 0]) - ref_v) <= FP64_TOL * abs(ref_v)


# device edge list -> canonical CSR (graphs.py:110-132 semantics) vs the host builder
@pytest.mark.parametrize("n,m,weighted,seed", [(50, 400, False, 0), (50, 400, True, 1), (1000, 20000, True, 2),
                                               (7, 0, False, 3), (3000, 5, False, 4)])
def test_device_edge_list_builder_matches_host(cuda_device, n, m, weighted, seed):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    u[: m // 10] = v[: m // 10]                       # self-loops
    if m > 20:
        u[-5:], v[-5:] = v[:5], u[:5]                 # reversed duplicates
    w = rng.choice([0.5, 1.0, 2.0, 3.5], size=m) if weighted else None
    ref = csr_from_edges(n, u, v, w)
    dg = DeviceGraph.from_edges(n, u, v, w, device=cuda_device)
    off, cols = dg.csr()
    assert dg.n == ref.n and dg.nnz == ref.nnz
    assert np.array_equal(off, ref.row_offsets)
    assert np.array_equal(cols.astype(np.int64), ref.col_indices)
    got_w = dg.weights()
    if weighted:
        assert np.array_equal(got_w, ref.weights)
    else:
        assert got_w is None
    if ref.nnz:
        host = DeviceGraph(ref, cuda_device)
        a1, _, s1 = dg.tridiagonals("normalized_laplacian", 0, 0, 8, 10)
        a2, _, s2 = host.tridiagonals("normalized_laplacian", 0, 0, 8, 10)
        assert torch.equal(a1, a2) and torch.equal(s1, s2)


def test_device_edge_list_builder_rejects_out_of_range(cuda_device):
    with pytest.raises(ValueError, match="out of range"):
        DeviceGraph.from_edges(5, np.array([0, 1]), np.array([1, 5]), device=cuda_device)


# Gaussian probes (slq.py:63-73): drawn on the host with numpy's ziggurat, Lanczos on the device
@pytest.mark.parametrize("fname", ["c1_ba1000.npz", "rmat12.npz"])
def test_gaussian_probes_match_oracle(cuda_device, fname):
    g = golden.graph(golden.load(fname))
    cfg = SlqConfig(n_v=70, s=10, seed=5, distribution="gaussian")   # 2 start blocks (64 + 6)
    q0 = np.empty((g.n, cfg.n_v))
    for i in range(cfg.n_v):   # restated from the reference's _draw_probe / _probe_rule
        v = np.random.default_rng(np.random.SeedSequence(entropy=cfg.seed, spawn_key=(i,))).standard_normal(g.n)
        q0[:, i] = v / np.linalg.norm(v)
    for kind, okind in (("heat", O.NORMALIZED_LAPLACIAN), ("vnge", O.DENSITY)):
        op = O.make_block_operator(g, okind)
        ref_rules = O.gauss_rules(O.lanczos_block(op, q0, cfg.s), op.interval)
        if kind == "heat":
            ref, _ = O.heat_from_rules(ref_rules, g.n, np.array(GRID.values))
            got = netlsd_slq(g, GRID, cfg).values
            assert golden.rel_l2(got, ref) <= FP64_TOL
        else:
            ref, _ = O.vnge_from_rules(ref_rules, g.n)
            got = vnge_slq(g, cfg).value
            assert abs(got - ref) <= FP64_TOL * abs(ref)


# trace identities (operators.py:105-141): tr M from degrees, tr M^2 from one edge pass
@pytest.mark.parametrize("fname", ["c1_ba1000.npz", "rmat12.npz"])
def test_trace_identities_match_reference_definitions(cuda_device, fname):
    from paper_2003_01282_b200.operators import OperatorKind, trace, trace_squared

    g = golden.graph(golden.load(fname))
    deg = O.degrees(g)
    w = np.asarray(g.weights, dtype=np.float64)
    src = np.repeat(np.arange(g.n), np.diff(g.row_offsets))
    ref_l2 = float(np.sum(deg * deg) + np.sum(w * w))
    ref_nl2 = float(np.count_nonzero(deg > 0)) + float(np.sum(w * w / (deg[src] * deg[g.col_indices])))
    trl = float(deg.sum())
    assert trace(g, OperatorKind.LAPLACIAN) == trl
    assert trace(g, OperatorKind.NORMALIZED_LAPLACIAN) == float(np.count_nonzero(deg > 0))
    assert abs(trace_squared(g, OperatorKind.LAPLACIAN) - ref_l2) <= 1e-13 * ref_l2
    assert abs(trace_squared(g, OperatorKind.NORMALIZED_LAPLACIAN) - ref_nl2) <= 1e-13 * ref_nl2
    assert abs(trace_squared(g, OperatorKind.DENSITY) - ref_l2 / trl ** 2) <= 1e-13 * ref_l2 / trl ** 2
    # dense check of the identity on the oracle operator
    n = g.n
    if n <= 1500:
        L = O.make_block_operator(g, O.NORMALIZED_LAPLACIAN).apply(np.eye(n))
        assert abs(np.sum(L * L) - ref_nl2) <= 1e-10 * ref_nl2


@pytest.mark.parametrize("count", [24, 32])
def test_spmm_half2_mapping_bitwise_equals_full_warp(cuda_device, tmp_path, count):
    # fp32 chunks of 17..32 probes: the HALF2 mapping (two probes per lane, a half-warp per gathered
    # row) sums every row in the same two chains as the full-warp mapping (SLQ_SPMM_HALF2=0), so the
    # rules are bitwise equal; the hub graph adds long-row segments
    import os
    import subprocess
    import sys

    out = tmp_path / "nodes.npy"
    code = ("import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); import numpy as np, golden; "
            "from test_gpu_parity import _hub_graph; "
            "from paper_2003_01282_b200.device import DeviceGraph; "
            f"r = DeviceGraph(_hub_graph()).rules('normalized_laplacian', 3, 0, {count}, 12, dtype='f32'); "
            f"np.save('{out}', np.stack([r.nodes.cpu().numpy(), r.weights.cpu().numpy()]))")
    env = dict(os.environ, SLQ_SPMM_HALF2="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env,
                   cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    full = np.load(out)
    r = DeviceGraph(_hub_graph(), cuda_device).rules("normalized_laplacian", 3, 0, count, 12, dtype="f32")
    assert np.array_equal(np.stack([r.nodes.cpu().numpy(), r.weights.cpu().numpy()]), full)


def _weighted_hub_graph():
    g = _hub_graph()
    rng = np.random.default_rng(8)
    off, cols = np.asarray(g.row_offsets), np.asarray(g.col_indices)
    rows = np.repeat(np.arange(g.n), np.diff(off))
    keep = rows < cols                       # one weight per undirected edge
    return csr_from_edges(g.n, rows[keep], cols[keep], rng.uniform(0.25, 4.0, int(keep.sum())))


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("dtype,tol", [("f64", FP64_TOL), ("f32", FP32_TOL)])
def test_prescaled_gathers_match_oracle(cuda_device, tmp_path, dtype, tol, weighted):
    # narrow-class normalized-Laplacian runs on large graphs gather dinv (.) u written by the step
    # kernel instead of u times a dinv[col] gather; forced on a small graph here (SLQ_PRESCALE_MIN_N=0):
    # heat within the north-star tolerance of the oracle, and within rounding of the unscaled gathers
    import os
    import subprocess
    import sys

    out = tmp_path / "heat.npy"
    code = ("import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); import numpy as np, golden; "
            "from test_gpu_parity import _hub_graph, _weighted_hub_graph, GRID; from paper_2003_01282_b200 import _lib; "
            "from paper_2003_01282_b200.device import DeviceGraph; "
            f"g = {'_weighted_hub_graph' if weighted else '_hub_graph'}(); "
            f"r = DeviceGraph(g).rules('normalized_laplacian', 0, 0, 24, 15, dtype='{dtype}'); "
            "v, _ = r.integrate(np.array(GRID.values), [_lib.FN_HEAT]); "
            f"np.save('{out}', v.cpu().numpy()[0])")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, SLQ_PRESCALE_MIN_N="0"), cwd=root)
    pre = np.load(out)
    g = _weighted_hub_graph() if weighted else _hub_graph()
    r = DeviceGraph(g, cuda_device).rules("normalized_laplacian", 0, 0, 24, 15, dtype=dtype)
    plain, _ = r.integrate(np.array(GRID.values), [_lib.FN_HEAT])
    plain = plain.cpu().numpy()[0]
    ref, _ = O.heat_trace(g, GRID.values, 24, 15, 0)
    assert golden.rel_l2(pre, ref) <= tol
    assert golden.rel_l2(pre, plain) <= (1e-12 if dtype == "f64" else 1e-5)
    assert not np.array_equal(pre, plain) or dtype == "f64"   # the prescaled path actually ran (fp32 rounding differs)


@pytest.mark.parametrize("count,dtype", [(100, "f64"), (50, "f64"), (128, "f64")])
def test_spmm_vec2_mapping_bitwise_equals_scalar(cuda_device, tmp_path, count, dtype):
    # wide chunks: the VEC2 mapping (probe pairs per lane, one vector load per pair) sums every probe
    # in the same sequential chain as the scalar mapping (SLQ_SPMM_VEC2=0): rules bitwise equal
    import os
    import subprocess
    import sys

    out = tmp_path / "nodes.npy"
    code = ("import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); import numpy as np, golden; "
            "from test_gpu_parity import _hub_graph; "
            "from paper_2003_01282_b200.device import DeviceGraph; "
            f"r = DeviceGraph(_hub_graph()).rules('normalized_laplacian', 1, 0, {count}, 12, dtype='{dtype}'); "
            f"np.save('{out}', np.stack([r.nodes.cpu().numpy(), r.weights.cpu().numpy()]))")
    env = dict(os.environ, SLQ_SPMM_VEC2="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env,
                   cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    scalar = np.load(out)
    r = DeviceGraph(_hub_graph(), cuda_device).rules("normalized_laplacian", 1, 0, count, 12, dtype=dtype)
    assert np.array_equal(np.stack([r.nodes.cpu().numpy(), r.weights.cpu().numpy()]), scalar)


@pytest.mark.parametrize("kind,fns", [("normalized_laplacian", [_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM]),
                                      ("density", [_lib.FN_XLOGX])])
@pytest.mark.parametrize("n", [1000, 100])   # n <= 128 takes the one-CTA small-graph kernel inside the capture
def test_captured_signature_replays_eager_results(cuda_device, kind, fns, n):
    from paper_2003_01282_b200 import synth
    from paper_2003_01282_b200.device import CapturedSignature

    g = synth.barabasi_albert(n, 3, seed=0)
    dg = DeviceGraph(g, cuda_device)
    t = None if kind == "density" else np.array(GRID.values)
    eager = dg.rules(kind, 0, 0, 10, 10)
    ev, es = eager.integrate(t, fns)
    cap = CapturedSignature(dg, kind, 0, 10, 10, t, fns)
    for _ in range(3):
        v, s = cap.replay()
        torch.cuda.synchronize()
        cap.check()
        assert torch.equal(v, ev) and torch.equal(s, es)
    if kind == "density":
        ref, _ = O.vnge(g, 10, 10, 0)
        assert abs(-float(v[0, 0]) - ref) <= FP64_TOL * abs(ref)
    else:
        ref, _ = O.heat_trace(g, GRID.values, 10, 10, 0)
        assert golden.rel_l2(v[0].cpu().numpy(), ref) <= FP64_TOL


# analytic pins of the reference's own test strategy (tests/test_slq.py, tests/test_lanczos.py)
def test_heat_at_t0_is_n(cuda_device):
    # h(0) = n * mean_i sum_k tau_ik^2 = n (weights of every rule sum to 1; tests/test_slq.py:169-177)
    from paper_2003_01282_b200 import synth

    g = synth.barabasi_albert(500, 3, seed=2)
    dg = DeviceGraph(g, cuda_device)
    r = dg.rules("normalized_laplacian", 0, 0, 12, 10)
    v, _ = r.integrate(np.array([0.0, 1e-2]), [_lib.FN_HEAT])
    assert abs(float(v[0, 0]) - g.n) <= 1e-12 * g.n


@pytest.mark.parametrize("kind", ["laplacian", "normalized_laplacian", "density"])
def test_gauss_rule_exact_for_linear_f(cuda_device, kind):
    # per-probe quadratic-form exactness (tests/test_slq.py:47-59, Gauss exactness tests/test_lanczos.py:154-172):
    # sum_k tau_k^2 theta_k = q0^T M q0 with q0 = z / sqrt(n), z the probe re-derived from SeedSequence
    from paper_2003_01282_b200 import synth

    g = synth.barabasi_albert(800, 4, seed=5)
    dg = DeviceGraph(g, cuda_device)
    r = dg.rules(kind, 7, 0, 16, 10)
    pv = r.quadrature(None, _lib.FN_IDENTITY).cpu().numpy()[0]      # per_vector [count]
    op = O.make_block_operator(g, {"laplacian": O.LAPLACIAN, "normalized_laplacian": O.NORMALIZED_LAPLACIAN,
                                   "density": O.DENSITY}[kind])
    q0 = O.draw_probes(g.n, 7, range(16))
    exact = np.einsum("nc,nc->c", q0, op.apply(q0))
    assert np.max(np.abs(pv - exact) / np.abs(exact)) <= 1e-12


def test_trace_estimate_unbiased_over_seeds(cuda_device):
    # E[z^T L z] = tr L for Rademacher z (tests/test_slq.py:88-101): 200 seeds x 4 probes of the
    # identity integrand on the normalized Laplacian average to n - #isolated within 4 standard errors
    from paper_2003_01282_b200 import synth

    g = synth.barabasi_albert(300, 2, seed=9)
    dg = DeviceGraph(g, cuda_device)
    ests = []
    for seed in range(200):
        r = dg.rules("normalized_laplacian", seed, 0, 4, 6)
        v, _ = r.integrate(None, [_lib.FN_IDENTITY])
        ests.append(float(v[0, 0]))
    ests = np.array(ests)
    tr = g.n - int(np.count_nonzero(np.diff(np.asarray(g.row_offsets)) == 0))
    assert abs(ests.mean() - tr) <= 4 * ests.std(ddof=1) / np.sqrt(len(ests))


# the reference's Lanczos-basis tests (tests/test_lanczos.py:41-48, 76-99) on the device basis export
@pytest.mark.parametrize("kind", ["laplacian", "normalized_laplacian", "density"])
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_lanczos_basis_orthonormal_and_tridiagonalizes(cuda_device, kind, dtype, tol):
    from paper_2003_01282_b200 import synth

    g = synth.barabasi_albert(600, 3, seed=4)
    dg = DeviceGraph(g, cuda_device)
    q, alpha, beta, st = dg.lanczos_basis(kind, 3, 0, 8, 12, dtype=dtype)
    q, alpha, beta, st = (x.cpu().numpy() for x in (q, alpha, beta, st))
    okind = {"laplacian": O.LAPLACIAN, "normalized_laplacian": O.NORMALIZED_LAPLACIAN, "density": O.DENSITY}[kind]
    op = O.make_block_operator(g, okind)
    hi = op.interval[1]
    # q_0 is the probe / sqrt(n), bit for bit
    assert np.array_equal(q[0], O.draw_probes(g.n, 3, range(8)))
    for j in range(8):
        m = int(st[j])
        Q = q[:m, :, j].T                                   # n x m
        assert np.max(np.abs(Q.T @ Q - np.eye(m))) <= tol                      # orthonormality
        T = np.diag(alpha[j, :m]) + np.diag(beta[j, :m - 1], 1) + np.diag(beta[j, :m - 1], -1)
        assert np.max(np.abs(Q.T @ op.apply(Q) - T)) <= tol * hi             # Q^T M Q = T
    # the tridiagonals are the ones slq_lanczos returns
    a2, b2, s2 = dg.tridiagonals(kind, 3, 0, 8, 12, dtype=dtype)
    assert np.array_equal(a2.cpu().numpy(), alpha) and np.array_equal(s2.cpu().numpy(), st)
