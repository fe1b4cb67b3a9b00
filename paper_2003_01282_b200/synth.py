"""Seeded synthetic graphs with the shapes BASELINE.json names (host side).

The reference ships only ``erdos_renyi`` (``graphs.py:223-270``); the
benchmark families below are new harness code.  Every
generator emits the canonical CSR of ``graphs.csr_from_edges``.  The paper's
datasets are not available offline: these seeded graphs stand in for them.

* ``barabasi_albert(n, m, seed)``     C1: preferential attachment, star seed graph of m+1 nodes
* ``sbm(n, blocks, p_in, p_out, seed)`` C2: Binomial pair counts per block / across blocks
* ``er_batch(count, seed)``           C3: n ~ U{20..200}, p ~ U[0.05, 0.3], one default_rng stream
* ``rmat(scale, edge_factor, a, b, c, seed)`` C4/C5: recursive quadrant choice, symmetrised
"""
from __future__ import annotations

import numpy as np

from .graphs import Graph, block_diagonal, csr_from_edges, unique_sorted

__all__ = ["barabasi_albert", "sbm", "erdos_renyi", "er_batch", "rmat", "rmat_device_reference"]


def barabasi_albert(n: int, m: int, seed: int = 0) -> Graph:
    """Preferential attachment: each new vertex links to m distinct targets drawn
    with probability proportional to degree (star on m+1 vertices to start)."""
    if not 1 <= m < n:
        raise ValueError(f"need 1 <= m < n, got m={m}, n={n}")
    rng = np.random.default_rng(seed)
    us = [0] * m
    vs = list(range(1, m + 1))
    # vertex ids repeated once per incident edge end: sampling from it is
    # degree-proportional
    pool = np.empty(2 * m * n, dtype=np.int64)
    pool[:m] = 0
    pool[m:2 * m] = np.arange(1, m + 1)
    size = 2 * m
    for src in range(m + 1, n):
        chosen: set[int] = set()
        while len(chosen) < m:
            chosen.add(int(pool[rng.integers(0, size)]))
        tg = np.fromiter(chosen, dtype=np.int64, count=m)
        us.extend([src] * m)
        vs.extend(tg.tolist())
        pool[size:size + m] = tg
        pool[size + m:size + 2 * m] = src
        size += 2 * m
    return csr_from_edges(n, np.array(us), np.array(vs))


def sbm(n: int = 100_000, blocks: int = 10, p_in: float = 1e-3, p_out: float = 1e-5,
        seed: int = 0) -> Graph:
    """Planted partition with equal blocks; pair counts drawn as Binomials and
    pairs sampled uniformly (duplicates collapse)."""
    rng = np.random.default_rng(seed)
    bs = n // blocks
    us, vs = [], []
    for b in range(blocks):
        pairs = bs * (bs - 1) // 2
        k = rng.binomial(pairs, p_in)
        u = rng.integers(0, bs, size=k)
        v = rng.integers(0, bs - 1, size=k)
        v = v + (v >= u)
        us.append(u + b * bs)
        vs.append(v + b * bs)
    cross = (n * (n - 1) // 2) - blocks * (bs * (bs - 1) // 2)
    k = rng.binomial(cross, p_out)
    u = rng.integers(0, n, size=2 * k + 16)
    v = rng.integers(0, n, size=2 * k + 16)
    ok = (u // bs) != (v // bs)
    us.append(u[ok][:k])
    vs.append(v[ok][:k])
    return csr_from_edges(n, np.concatenate(us), np.concatenate(vs))


def erdos_renyi(n: int, p: float, rng: np.random.Generator) -> Graph:
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(iu.size) < p
    return csr_from_edges(n, iu[keep], ju[keep])


def er_batch(count: int = 10_000, seed: int = 0, n_range=(20, 200), p_range=(0.05, 0.3)) -> list[Graph]:
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(n_range[0], n_range[1] + 1))
        p = float(rng.uniform(*p_range))
        out.append(erdos_renyi(n, p, rng))
    return out


def er_batch_stacked(count: int = 10_000, seed: int = 0):
    graphs = er_batch(count, seed)
    g, voff = block_diagonal(graphs)
    return g, voff, graphs


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = x + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def rmat_device_reference(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
                          seed: int = 0) -> Graph:
    """Host restatement of the device R-MAT generator (csrc/rmat.cu, ``DeviceGraph.rmat``): the same
    counter-based uniforms u(seed, sample, level) = splitmix64(splitmix64(seed ^ K) ^ (64 sample + level))
    >> 11 / 2^53 and the same quadrant rule as ``rmat``; used to check the device build edge for edge."""
    n = 1 << scale
    total = edge_factor * n
    with np.errstate(over="ignore"):
        base = _splitmix64(np.array([np.uint64(seed) ^ np.uint64(0xD1B54A32D192ED03)], dtype=np.uint64))[0]
        j = np.arange(total, dtype=np.uint64)
        u = np.zeros(total, dtype=np.int64)
        v = np.zeros(total, dtype=np.int64)
        ab, abc = a + b, a + b + c
        for level in range(scale):
            h = _splitmix64(base ^ (j * np.uint64(64) + np.uint64(level)))
            r = (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
            bit = np.int64(1) << (scale - 1 - level)
            u |= np.where(r >= ab, bit, 0)
            v |= np.where(((r >= a) & (r < ab)) | (r >= abc), bit, 0)
    keep = u != v
    u, v = u[keep], v[keep]
    key = unique_sorted(np.minimum(u, v) * n + np.maximum(u, v))
    return csr_from_edges(n, key // n, key % n)


def rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
         seed: int = 0, chunk: int = 1 << 24) -> Graph:
    """R-MAT: edge_factor * 2^scale samples; per level one uniform draw picks the
    quadrant with probabilities (a, b, c, d=1-a-b-c); symmetrised, deduplicated,
    self-loops removed, no vertex permutation."""
    n = 1 << scale
    total = edge_factor * n
    rng = np.random.default_rng(seed)
    keys = []
    ab, abc = a + b, a + b + c
    for start in range(0, total, chunk):
        k = min(chunk, total - start)
        u = np.zeros(k, dtype=np.int64)
        v = np.zeros(k, dtype=np.int64)
        for level in range(scale):
            r = rng.random(k)
            bit = np.int64(1) << (scale - 1 - level)
            down = r >= ab                       # quadrants c or d: row bit set
            right = ((r >= a) & (r < ab)) | (r >= abc)   # quadrants b or d: col bit set
            u |= np.where(down, bit, 0)
            v |= np.where(right, bit, 0)
        keep = u != v
        u, v = u[keep], v[keep]
        keys.append(unique_sorted(np.minimum(u, v) * n + np.maximum(u, v)))
    key = unique_sorted(np.concatenate(keys))
    return csr_from_edges(n, key // n, key % n)
