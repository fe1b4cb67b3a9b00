"""Flat SpMM (csrc/spmm_flat.cu): the cp.async-staged quad kernel that runs the fp32 17..32-probe
gathers of large degree-ordered graphs (the C5 path; replaces `csr_matvec` + the operator
elementwise work of operators.py:76-99 inside the Lanczos recurrence, lanczos.py:122-138).

It must reproduce the warp-per-row kernel bit for bit (same two-chain row sums, same epilogue), for
every operator kind, chunk widths with padded rows (19, 24 probes), the first step (probe bitmask,
[bits | dinv] records), long-row segments, and on graphs that are NOT degree ordered (forced on:
ragged quads, empty rows).  The kernel choice is made from the environment when the library loads, so
each arm runs in its own process.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import golden
from oracle import slq_oracle as O
from paper_2003_01282_b200.descriptors import TimeGrid

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GRID = TimeGrid(1e-2, 1e2, 250)

CHILD = r"""
import sys, json, hashlib
import numpy as np, torch
sys.path.insert(0, %r)
from paper_2003_01282_b200 import _lib, synth
from paper_2003_01282_b200.device import DeviceGraph
mode, out_path = sys.argv[1], sys.argv[2]
dev = torch.device('cuda', 0)
if mode == 'rmat':
    dg = DeviceGraph.rmat(15, 16, seed=0, device=dev)          # folded, degree ordered, long rows
elif mode == 'iso':
    # unfolded, not degree ordered, a third of the rows EMPTY (ragged quads, rows of length 0)
    from paper_2003_01282_b200.graphs import csr_from_edges
    rng = np.random.default_rng(7)
    n, m = 4001, 20000
    live = np.flatnonzero(rng.random(n) > 0.33)
    dg = DeviceGraph(csr_from_edges(n, live[rng.integers(0, live.size, m)], live[rng.integers(0, live.size, m)]),
                     dev, fold=None)
else:
    dg = DeviceGraph(synth.barabasi_albert(3000, 3, seed=1), dev, fold=None)   # not degree ordered
res = {}
for kind in ('normalized_laplacian', 'density', 'laplacian'):
    for nv, dt in ((32, 'f32'), (24, 'f32'), (19, 'f32'), (16, 'f32'), (12, 'f32'), (8, 'f32'), (5, 'f32'),
                   (32, 'f64'), (19, 'f64'), (16, 'f64'), (11, 'f64'), (8, 'f64'), (3, 'f64')):
        a, b, s = dg.tridiagonals(kind, 0, 0, nv, 12, dtype=dt)
        blob = a.cpu().numpy().tobytes() + b.cpu().numpy().tobytes() + s.cpu().numpy().tobytes()
        res[kind + '/' + str(nv) + '/' + dt] = hashlib.sha256(blob).hexdigest()
vals, _ = dg.rules('normalized_laplacian', 0, 0, 32, 12, dtype='f32').integrate(
    np.logspace(-2, 2, 250), [_lib.FN_HEAT])
np.save(out_path, vals.cpu().numpy()[0])
print(json.dumps(res))
""" % ROOT


def _run(mode, flat, out_path):
    env = dict(os.environ, SLQ_SPMM_FLAT=flat, SLQ_PRESCALE_MIN_N="0")
    r = subprocess.run([sys.executable, "-c", CHILD, mode, str(out_path)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("mode", ["rmat", "ba", "iso"])
def test_flat_spmm_bitwise_equals_warp_per_row(cuda_device, tmp_path, mode):
    old = _run(mode, "0", tmp_path / "old.npy")
    new = _run(mode, "1", tmp_path / "new.npy")
    assert old.keys() == new.keys() and len(old) == 39
    assert [k for k in old if old[k] != new[k]] == []
    assert np.array_equal(np.load(tmp_path / "old.npy"), np.load(tmp_path / "new.npy"))


def test_flat_spmm_heat_matches_oracle(cuda_device, tmp_path):
    """The forced-flat fp32 run of a host graph against the CPU oracle (1e-4, BASELINE north_star)."""
    from paper_2003_01282_b200 import synth

    _run("ba", "1", tmp_path / "new.npy")
    g = synth.barabasi_albert(3000, 3, seed=1)
    ref, _ = O.heat_trace(g, np.logspace(-2, 2, 250), 32, 12, 0)
    assert golden.rel_l2(np.load(tmp_path / "new.npy"), ref) <= 1e-4


PAIR_CHILD = r"""
import sys, json, torch
sys.path.insert(0, %r)
from paper_2003_01282_b200.device import DeviceGraph
dg = DeviceGraph.rmat(15, 16, seed=0, device=torch.device('cuda', 0))
res = []
for count, p0 in ((16, 0), (16, 40), (12, 3), (10, 0), (20, 0), (4, 0)):
    a, b, paired = dg.rules_pair(0, p0, count, 12)
    a.check()
    ra = dg.rules('normalized_laplacian', 0, p0, count, 12, dtype='f32')
    rb = dg.rules('density', 0, p0, count, 12, dtype='f32')
    eq = all(torch.equal(x, y) for x, y in ((a.nodes, ra.nodes), (a.weights, ra.weights), (a.steps, ra.steps),
                                            (b.nodes, rb.nodes), (b.weights, rb.weights), (b.steps, rb.steps)))
    res.append([count, p0, bool(paired), bool(eq)])
print(json.dumps(res))
""" % ROOT


def test_operator_pair_block_bitwise_equals_separate_runs(cuda_device):
    """slq_rules_pair_seeded: the normalized-Laplacian and density Lanczos runs of the same probes in
    one 32-column block (one gather per nonzero for both) give, per probe, the bits of two separate
    slq_rules_seeded calls; probe counts outside 9..16 take the separate runs."""
    env = dict(os.environ, SLQ_SPMM_FLAT="1", SLQ_PRESCALE_MIN_N="0")
    r = subprocess.run([sys.executable, "-c", PAIR_CHILD], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(eq for *_, eq in res), res
    assert [paired for _, _, paired, _ in res] == [True, True, True, True, False, False], res


def test_operator_pair_falls_back_on_small_graphs(cuda_device):
    """Without the flat SpMM (a small host graph, default environment) the pair entry runs the two
    operators apart: same results as ``rules``, ``paired`` False."""
    import torch

    from paper_2003_01282_b200 import synth
    from paper_2003_01282_b200.device import DeviceGraph

    dg = DeviceGraph(synth.barabasi_albert(1000, 3, seed=0), cuda_device)
    a, b, paired = dg.rules_pair(0, 0, 16, 10)
    assert not paired
    ra = dg.rules("normalized_laplacian", 0, 0, 16, 10, dtype="f32")
    rb = dg.rules("density", 0, 0, 16, 10, dtype="f32")
    assert torch.equal(a.nodes, ra.nodes) and torch.equal(a.weights, ra.weights)
    assert torch.equal(b.nodes, rb.nodes) and torch.equal(b.weights, rb.weights)


def test_captured_signature_on_the_flat_path(cuda_device):
    """A whole signature captured as a CUDA graph (device.CapturedSignature) on a graph that takes the
    flat SpMM by default (R-MAT-20: >= 2^24 nonzeros, degree-ordered fold): the cp.async kernels, their
    shared-memory opt-in and the L2 window attribute are capturable; replays equal the eager run."""
    import torch

    from paper_2003_01282_b200 import _lib
    from paper_2003_01282_b200.device import CapturedSignature, DeviceGraph

    dg = DeviceGraph.rmat(20, 16, seed=0, device=cuda_device)
    assert dg.nnz >= 1 << 24
    t = np.geomspace(1e-2, 1e2, 64)
    for kind, fns, tt, nv, dt in (("normalized_laplacian", [_lib.FN_HEAT], t, 32, "f32"),
                                  ("density", [_lib.FN_XLOGX], None, 16, "f32"),
                                  ("normalized_laplacian", [_lib.FN_HEAT], t, 16, "f64")):
        cap = CapturedSignature(dg, kind, 0, nv, 12, tt, fns, dtype=dt)
        first = cap.replay()[0].clone()
        cap.check()
        second = cap.replay()[0].clone()
        eager, _ = dg.rules(kind, 0, 0, nv, 12, dtype=dt).integrate(tt, fns)
        assert torch.equal(first, eager) and torch.equal(first, second)


FUZZ_CHILD = r"""
import sys, json, hashlib
import numpy as np, torch
sys.path.insert(0, %r)
from paper_2003_01282_b200.device import DeviceGraph
from paper_2003_01282_b200.graphs import csr_from_edges
dev = torch.device('cuda', 0)
rng = np.random.default_rng(20260321)
res = []
for case in range(24):
    n = int(rng.integers(200, 6000))
    m = int(rng.integers(n // 2, 12 * n))
    live = np.flatnonzero(rng.random(n) > rng.choice([0.0, 0.2, 0.6]))
    if live.size < 2:
        live = np.arange(n)
    hub = live[: max(1, live.size // 50)]
    u = np.where(rng.random(m) < 0.3, hub[rng.integers(0, hub.size, m)], live[rng.integers(0, live.size, m)])
    v = live[rng.integers(0, live.size, m)]
    g = csr_from_edges(n, u, v)
    fold = None if case %% 3 == 0 else 0.0
    dg = DeviceGraph(g, dev, fold=fold)
    kind = ('normalized_laplacian', 'density', 'laplacian')[case %% 3]
    dt = 'f64' if case %% 4 == 3 else 'f32'
    nv = int(rng.integers(1, 33))
    steps = int(rng.integers(3, 16))
    a, b, s = dg.tridiagonals(kind, int(rng.integers(0, 1000)), int(rng.integers(0, 50)), nv, steps, dtype=dt)
    blob = a.cpu().numpy().tobytes() + b.cpu().numpy().tobytes() + s.cpu().numpy().tobytes()
    res.append([n, int(g.nnz), kind, dt, nv, steps, hashlib.sha256(blob).hexdigest()[:16]])
print(json.dumps(res))
""" % ROOT


def test_flat_spmm_fuzz_bitwise(cuda_device):
    """24 random graphs (hubs, up to 60%% empty rows, folded or not), operator kinds, fp32 and fp64,
    1..32 probes, 3..15 steps, random seeds and probe offsets: the flat SpMM forced on gives the bits
    of the warp-per-row kernel."""
    out = {}
    for flat in ("0", "1"):
        env = dict(os.environ, SLQ_SPMM_FLAT=flat, SLQ_PRESCALE_MIN_N="0")
        r = subprocess.run([sys.executable, "-c", FUZZ_CHILD], env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        out[flat] = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(out["0"]) == 24
    assert [c for c, d in zip(out["0"], out["1"]) if c != d] == []
