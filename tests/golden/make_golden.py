"""Generate golden fixtures by running the REAL reference (``spectrace``) in this container.

Usage (from the repo root, where /root/reference exists):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  The GPU box has no /root/reference; the tests
there read only these committed fixtures.  Graphs are stored inside the
fixtures (CSR arrays) so the fixtures do not depend on generator changes.

Every value is produced through the reference's public API:
``netlsd_slq`` / ``vnge_slq`` (descriptors.py:124-149, 227-243),
``slq_trace_grid`` for the wave trace, and per probe
``lanczos_tridiagonalize`` + ``quadrature_rule`` on the exact q0 the reference
draws (slq.py:69-77).  ``operators.make_operator(...).apply`` outputs pin the
SpMM (bit-exact target).
"""
from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import spectrace as st  # noqa: E402
from spectrace.operators import OperatorKind  # noqa: E402

from paper_2003_01282_b200 import synth  # noqa: E402
from paper_2003_01282_b200.graphs import csr_from_edges  # noqa: E402

KINDS = {"L": OperatorKind.LAPLACIAN, "NL": OperatorKind.NORMALIZED_LAPLACIAN, "P": OperatorKind.DENSITY}


def ref_graph(g):
    return st.Graph(n=g.n, row_offsets=np.array(g.row_offsets, dtype=np.int64),
                    col_indices=np.array(g.col_indices, dtype=np.int64),
                    weights=np.array(g.weights, dtype=np.float64), m=g.m)


def graph_arrays(prefix, g):
    return {f"{prefix}n": np.int64(g.n), f"{prefix}m": np.int64(g.m),
            f"{prefix}offsets": np.asarray(g.row_offsets, np.int64),
            f"{prefix}cols": np.asarray(g.col_indices, np.int32 if g.n < 2**31 else np.int64),
            f"{prefix}weights": np.asarray(g.weights, np.float64)}


def probe_rules(rg, kind, n_v, s, seed):
    """Per-probe tridiagonal + rule exactly as slq._probe_rule does it."""
    op = st.make_operator(rg, kind)
    width = min(s, rg.n)
    alpha = np.zeros((n_v, width))
    beta = np.zeros((n_v, max(width - 1, 0)))
    nodes = np.zeros((n_v, width))
    weights = np.zeros((n_v, width))
    steps = np.zeros(n_v, np.int64)
    for i in range(n_v):
        rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(i,)))
        v = rng.integers(0, 2, size=rg.n).astype(np.float64) * 2.0 - 1.0
        q0 = v / np.linalg.norm(v)
        tri = st.lanczos_tridiagonalize(op, q0, width)
        rule = st.quadrature_rule(tri)
        k = tri.steps
        steps[i] = k
        alpha[i, :k] = tri.alpha
        beta[i, :k - 1] = tri.beta
        nodes[i, :k] = np.clip(rule.nodes, *op.interval)
        weights[i, :k] = rule.weights
    return dict(alpha=alpha, beta=beta, nodes=nodes, weights=weights, steps=steps,
                interval=np.array(op.interval))


def descriptors(rg, grid, cfg, wave=True, vnge=True):
    out = {}
    h = st.netlsd_slq(rg, grid, cfg)
    out["heat"] = h.values
    out["heat_std"] = h.std_errors
    out["graph_hash"] = np.array(h.graph_hash)
    if wave:
        op = st.make_operator(rg, OperatorKind.NORMALIZED_LAPLACIAN)
        re = st.slq_trace_grid(op, lambda t: (lambda x: np.cos(t * x)), grid.values, cfg)
        im = st.slq_trace_grid(op, lambda t: (lambda x: -np.sin(t * x)), grid.values, cfg)
        out["wave_re"] = np.array([e.value for e in re])
        out["wave_im"] = np.array([e.value for e in im])
        out["wave_re_std"] = np.array([e.std_error for e in re])
        out["wave_im_std"] = np.array([e.std_error for e in im])
    if vnge and rg.m > 0:
        v = st.vnge_slq(rg, cfg)
        out["vnge"] = np.float64(v.value)
        out["vnge_std"] = np.float64(v.std_error)
    return out


def small_graphs():
    rng = np.random.default_rng(2024)
    gs = {
        "k2": csr_from_edges(2, [0], [1]),
        "k3": csr_from_edges(3, [0, 0, 1], [1, 2, 2]),
        "p3": csr_from_edges(3, [0, 1], [1, 2]),
        "star3": csr_from_edges(4, [0, 0, 0], [1, 2, 3]),
        "k5": csr_from_edges(5, *zip(*[(i, j) for i in range(5) for j in range(i + 1, 5)])),
        "disjoint4": csr_from_edges(8, [0, 2, 4, 6], [1, 3, 5, 7]),
        "isolated": csr_from_edges(40, [0, 1, 2, 5, 9], [1, 2, 3, 20, 30]),
        "empty7": csr_from_edges(7, [], []),
        "path33": csr_from_edges(33, np.arange(32), np.arange(1, 33)),
    }
    # weighted random graphs (exercise explicit weights), n odd and not a multiple of 32
    for n in (31, 45, 77):
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(iu.size) < 0.2
        w = rng.uniform(0.5, 1.5, size=int(keep.sum()))
        gs[f"wrand{n}"] = csr_from_edges(n, iu[keep], ju[keep], w)
    gs["ba200"] = synth.barabasi_albert(200, 2, seed=5)
    gs["er150"] = synth.erdos_renyi(150, 0.1, np.random.default_rng(3))
    return gs


def main():
    grid = st.TimeGrid(1e-2, 1e2, 250)
    out = {}

    # 1. probe stream pins (slq.py:63-72)
    probe_cases = [(0, 0, 1), (0, 1, 2), (0, 3, 33), (7, 5, 100), (123, 99, 257), (2**40 + 3, 17, 1000)]
    for k, (seed, i, n) in enumerate(probe_cases):
        rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(i,)))
        out[f"probe{k}_case"] = np.array([seed, i, n], dtype=np.uint64)
        out[f"probe{k}_v"] = (rng.integers(0, 2, size=n).astype(np.float64) * 2.0 - 1.0).astype(np.int8)
        st_ = np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=(i,))).state["state"]
        out[f"probe{k}_state"] = np.array([st_["state"] >> 64, st_["state"] & (2**64 - 1),
                                           st_["inc"] >> 64, st_["inc"] & (2**64 - 1)], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "probes.npz"), **out)

    # 2. small graphs: per-probe rules for every operator kind + operator apply pins
    out = {}
    rng = np.random.default_rng(11)
    names = []
    for name, g in small_graphs().items():
        names.append(name)
        rg = ref_graph(g)
        out.update(graph_arrays(f"{name}/", g))
        x = rng.standard_normal((g.n, 3))
        out[f"{name}/x"] = x
        for kname, kind in KINDS.items():
            if kind is OperatorKind.DENSITY and g.m == 0:
                continue
            op = st.make_operator(rg, kind)
            out[f"{name}/apply_{kname}"] = np.stack([op.apply(x[:, j]) for j in range(3)], axis=1)
            for s in (4, 10):
                r = probe_rules(rg, kind, 8, s, seed=3)
                for key, val in r.items():
                    out[f"{name}/{kname}_s{s}/{key}"] = val
        cfg = st.SlqConfig(n_v=8, s=10, seed=3)
        for key, val in descriptors(rg, grid, cfg).items():
            out[f"{name}/desc/{key}"] = val
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)

    # 3. C1 BA n=1000 m=3, n_v=10, s=10, heat + wave + VNGE (BASELINE configs[0])
    g = synth.barabasi_albert(1000, 3, seed=0)
    rg = ref_graph(g)
    cfg = st.SlqConfig(n_v=10, s=10, seed=0)
    out = graph_arrays("", g)
    out.update(descriptors(rg, grid, cfg))
    for kname in ("NL", "P"):
        for key, val in probe_rules(rg, KINDS[kname], 10, 10, 0).items():
            out[f"{kname}/{key}"] = val
    np.savez_compressed(os.path.join(HERE, "c1_ba1000.npz"), **out)

    # 4. medium graphs: SBM (C2 shape, scaled down) and R-MAT (C4 shape, scale 12), s=15
    for fname, g in (("sbm5k.npz", synth.sbm(5000, 10, 1e-2, 1e-4, seed=1)),
                     ("rmat12.npz", synth.rmat(12, 16, seed=2))):
        rg = ref_graph(g)
        cfg = st.SlqConfig(n_v=16, s=15, seed=0)
        out = graph_arrays("", g)
        out.update(descriptors(rg, grid, cfg))
        for kname in ("NL", "P"):
            for key, val in probe_rules(rg, KINDS[kname], 16, 15, 0).items():
                out[f"{kname}/{key}"] = val
        np.savez_compressed(os.path.join(HERE, fname), **out)

    # 5. C3 sample: 40 ER graphs (per-graph heat, n_v=20, s=10)
    graphs = synth.er_batch(40, seed=0)
    out = {"count": np.int64(len(graphs))}
    cfg = st.SlqConfig(n_v=20, s=10, seed=0)
    for k, g in enumerate(graphs):
        out.update(graph_arrays(f"{k}/", g))
        h = st.netlsd_slq(ref_graph(g), grid, cfg)
        out[f"{k}/heat"] = h.values
        out[f"{k}/heat_std"] = h.std_errors
    np.savez_compressed(os.path.join(HERE, "erbatch40.npz"), **out)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
