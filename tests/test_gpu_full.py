"""Parity at BASELINE.json's full configuration sizes, on the GPU.

* C2 (SBM n=100,000, 100 probes x 15 steps, heat + wave, fp64 and fp32) and C4
  (R-MAT scale 20, 100 x 15, fp64 heat + VNGE -- the configuration where VNGE is
  reorthogonalisation-sensitive) against the oracle on ALL probes:
  rel-l2 <= 1e-9 in fp64, <= 1e-4 in fp32 (north_star tolerances).
* A folded R-MAT-23 with prescaled normalized-Laplacian gathers (the C5 code
  path at a size the oracle can still run) against the oracle on a probe prefix.
* C5 (R-MAT scale 27, 4.2e9 nonzeros > 2^31, 128 probes x 15 steps, fp32; no
  CPU oracle can hold it) through size-independent properties: alpha_0 = z^T L z / n
  through the bit-exact operator apply, fp32 vs fp64 storage, folded vs unfolded,
  a probe prefix bitwise equal to the prefix run, weights summing to 1.

These are the slow tests (about 5 minutes together on one B200 + 16 host cores).
"""
import numpy as np
import pytest
import torch

import golden
from oracle import slq_oracle as O
from paper_2003_01282_b200 import _lib, synth
from paper_2003_01282_b200.descriptors import TimeGrid, netlsd_heat_wave_slq, vnge_slq
from paper_2003_01282_b200.device import DeviceGraph, device_probes
from paper_2003_01282_b200.graphs import Graph
from paper_2003_01282_b200.slq import SlqConfig

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-9
FP32_TOL = 1e-4
GRID = TimeGrid(1e-2, 1e2, 250)
THREADS = O.default_threads()


@pytest.fixture(scope="module")
def c2_graph():
    return synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0)


@pytest.fixture(scope="module")
def c2_oracle(c2_graph):
    op = O.make_block_operator(c2_graph, O.NORMALIZED_LAPLACIAN)
    rules = O.slq_rules(op, 100, 15, 0, threads=THREADS)
    heat = O.heat_from_rules(rules, c2_graph.n, GRID.values)
    re, im = O.wave_from_rules(rules, c2_graph.n, GRID.values)
    return rules, heat, re, im


@pytest.mark.parametrize("dtype,tol", [("f64", FP64_TOL), ("f32", FP32_TOL)])
def test_c2_full_heat_and_wave_vs_oracle(cuda_device, c2_graph, c2_oracle, dtype, tol):
    rules, (h_ref, h_std), (re_ref, re_std), (im_ref, im_std) = c2_oracle
    heat, wave = netlsd_heat_wave_slq(c2_graph, GRID, SlqConfig(n_v=100, s=15, seed=0), dtype=dtype)
    assert golden.rel_l2(heat.values, h_ref) <= tol
    assert golden.rel_l2(wave.values, re_ref + 1j * im_ref) <= tol
    assert golden.rel_l2(heat.std_errors, h_std) <= (1e-7 if dtype == "f64" else 1e-3)
    if dtype == "f64":
        dr = DeviceGraph(c2_graph, cuda_device).rules("normalized_laplacian", 0, 0, 100, 15)
        assert np.array_equal(dr.steps.cpu().numpy(), rules.steps)
        assert np.max(np.abs(dr.nodes.cpu().numpy() - rules.nodes)) <= 2e-11
        assert np.allclose(dr.weights.cpu().numpy(), rules.weights, rtol=1e-8, atol=1e-13)


@pytest.fixture(scope="module")
def c4_graph():
    return synth.rmat(20, 16, seed=0)


def test_c4_full_heat_and_vnge_vs_oracle(cuda_device, c4_graph):
    g = c4_graph
    assert g.n == 1 << 20 and g.nnz > 30_000_000
    cfg = SlqConfig(n_v=100, s=15, seed=0)
    heat, _ = netlsd_heat_wave_slq(g, GRID, cfg, wave=False, with_hash=False)
    ent = vnge_slq(g, cfg, with_hash=False)
    h_ref, _ = O.heat_trace(g, GRID.values, 100, 15, 0, threads=THREADS)
    v_ref, v_std = O.vnge(g, 100, 15, 0, threads=THREADS)
    assert golden.rel_l2(heat.values, h_ref) <= FP64_TOL
    # VNGE is the reorthogonalisation-sensitive quantity (7.5e-8 without reorth)
    assert abs(ent.value - v_ref) <= FP64_TOL * abs(v_ref)
    assert abs(ent.std_error - v_std) <= 1e-7 * abs(v_std)


def _device_graph_to_host(dg) -> Graph:
    off, cols = dg.csr()
    return Graph(n=dg.n, row_offsets=off.astype(np.int64), col_indices=cols.astype(np.int64),
                 weights=np.ones(cols.size), m=cols.size // 2)


@pytest.fixture(scope="module")
def rmat23(cuda_device):
    dg = DeviceGraph.rmat(23, 16, seed=0, device=cuda_device)
    g = _device_graph_to_host(dg)
    k = 8
    op = O.make_block_operator(g, O.NORMALIZED_LAPLACIAN)
    h_ref, _ = O.heat_from_rules(O.slq_rules(op, k, 15, 0, threads=min(THREADS, k)), g.n, GRID.values)
    opp = O.make_block_operator(g, O.DENSITY)
    vn_ref, _ = O.vnge_from_rules(O.slq_rules(opp, k, 15, 0, threads=min(THREADS, k)), g.n)
    return dg, k, h_ref, vn_ref


@pytest.mark.parametrize("dtype,tol", [("f32", FP32_TOL), ("f64", FP64_TOL)])
def test_folded_prescaled_rmat23_vs_oracle(cuda_device, rmat23, dtype, tol):
    # the C5 code path (isolated-vertex fold + narrow step class + prescaled gathers, which switch on
    # at >= 2^22 folded rows) at a size the oracle can still run: 8-probe prefix, heat and VNGE
    dg, k, h_ref, vn_ref = rmat23
    info = dg.info
    assert dg.folded > 0 and info.n - info.isolated + 1 >= 1 << 22
    r_nl = dg.rules("normalized_laplacian", 0, 0, k, 15, dtype=dtype)
    v_nl, _ = r_nl.integrate(GRID.values, [_lib.FN_HEAT])
    r_p = dg.rules("density", 0, 0, k, 15, dtype=dtype)
    v_p, _ = r_p.integrate(None, [_lib.FN_XLOGX])
    r_nl.check()
    r_p.check()
    assert golden.rel_l2(v_nl[0].cpu().numpy(), h_ref) <= tol
    assert abs(-float(v_p[0, 0]) - vn_ref) <= tol * abs(vn_ref)


def test_c5_rmat27_full_size_properties(cuda_device):
    dev = cuda_device
    dg = DeviceGraph.rmat(27, 16, 0.57, 0.19, 0.19, seed=0, device=dev, fold=None)
    assert dg.n == 1 << 27
    assert dg.nnz > 2 ** 31                      # int64 offsets and nonzero indices
    folded = dg.fold_isolated()
    assert folded > 0.4 * dg.n
    t = torch.tensor(np.array(GRID.values), device=dev)
    rules = dg.rules("normalized_laplacian", 0, 0, 128, 15, dtype="f32")
    vals, _ = rules.integrate(t, [_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM])
    rules.check()
    st = rules.steps.cpu().numpy()
    assert np.all(st == 15)
    w = rules.weights.cpu().numpy()
    nodes = rules.nodes.cpu().numpy()
    assert np.max(np.abs(w.sum(axis=1) - 1.0)) <= 1e-12
    assert np.all((nodes >= 0.0) & (nodes <= 2.0))
    v = vals.cpu().numpy()
    assert np.all(np.isfinite(v))
    assert abs(v[0, 0] - dg.n) / dg.n < 0.02   # h(t -> 0) -> n: every rule integrates 1
    # a probe prefix is bitwise the prefix run (chunk independence: 4 chunks of 32 vs one of 8)
    pre = dg.rules("normalized_laplacian", 0, 0, 8, 15, dtype="f32")
    assert torch.equal(pre.nodes, rules.nodes[:8]) and torch.equal(pre.weights, rules.weights[:8])
    nl_16_32 = (rules.nodes[16:32].clone(), rules.weights[16:32].clone())
    del rules, pre
    # alpha_0 = z^T L z / n through the exact (bit-exact fp64) operator apply
    a, _, _ = dg.tridiagonals("normalized_laplacian", 0, 0, 4, 2, dtype="f32")
    z = device_probes(dg.n, 0, 0, 4, dev)
    y = dg.apply("normalized_laplacian", z)
    a0 = (z * y).sum(0) / dg.n
    assert float(torch.max(torch.abs(a[:, 0] - a0) / torch.abs(a0))) <= 1e-8
    del y, z
    # fp32 vs fp64 vector storage on a 4-probe prefix: the north_star fp32 bar
    r64 = dg.rules("normalized_laplacian", 0, 0, 4, 15, dtype="f64")
    r32 = dg.rules("normalized_laplacian", 0, 0, 4, 15, dtype="f32")
    h64, _ = r64.integrate(t, [_lib.FN_HEAT])
    h32, _ = r32.integrate(t, [_lib.FN_HEAT])
    assert float(torch.linalg.norm(h32 - h64) / torch.linalg.norm(h64)) <= FP32_TOL
    # folded vs unfolded recurrence on the same prefix
    dg.fold_isolated(-1.0)
    r_un = dg.rules("normalized_laplacian", 0, 0, 4, 15, dtype="f32")
    h_un, _ = r_un.integrate(t, [_lib.FN_HEAT])
    assert float(torch.linalg.norm(h32 - h_un) / torch.linalg.norm(h_un)) <= FP32_TOL
    # VNGE on the density operator
    dg.fold_isolated()
    rp = dg.rules("density", 0, 0, 128, 15, dtype="f32")
    vp, _ = rp.integrate(None, [_lib.FN_XLOGX])
    rp.check()
    assert 0.0 < -float(vp[0, 0]) < np.log(dg.n - dg.info.isolated)
    # the operator-pair block (a rank's share on 8 GPUs: probes 16..31 of both operators in one
    # 32-column block) is bitwise the full runs' rules of those probes
    pair_nl, pair_p, paired = dg.rules_pair(0, 16, 16, 15)
    pair_nl.check()
    assert paired
    assert torch.equal(pair_nl.nodes, nl_16_32[0]) and torch.equal(pair_nl.weights, nl_16_32[1])
    assert torch.equal(pair_p.nodes, rp.nodes[16:32]) and torch.equal(pair_p.weights, rp.weights[16:32])
