"""Benchmark: SLQ edge·probe·steps/s on BASELINE.json's largest single-GPU configuration (C5).

Default workload (``--config c5``, BASELINE configs[4]; one "step" = one whole signature):
  R-MAT scale 27 (n = 134,217,728; edge factor 16; a=.57 b=.19 c=.19; symmetrised, deduplicated,
  self-loops dropped; 4.22e9 stored nonzeros), generated on the device (seeded synthetic: the
  paper's Friendster-scale datasets are not available); 128 Rademacher probes x 15
  Lanczos steps with full CGS reorthogonalisation (the reference default for s <= 100), fp32
  vector storage (int32 indices, implicit unit weights); heat + wave traces of the normalized
  Laplacian on 250 log-spaced t in [1e-2, 1e2] (one Lanczos run) and VNGE on the density matrix
  (a second run).  Units per step = 2 * nnz * n_v * s (stored nonzero x probe x operator
  application, two operator runs).
``--config c2`` (SBM n=100k, 100 x 15, heat+wave, fp64) and ``--config c4`` (R-MAT scale 20,
100 x 15, heat + VNGE, fp64) are kept for comparison with round 1.

Arms:
  default            hand-written sm_100a kernels through libslq_b200.so
  --impl reference   the CPU oracle port of the reference algorithm (oracle/slq_oracle.py: numpy +
                     scipy, all host threads) timed on a bounded sample of the same workload; rank 0.

Timing: W warm-up steps, then K timed steps bracketed by CUDA events on the launching stream
(inputs far larger than L2 at C5; L2 is also flushed between steps, outside the events).
Multi-GPU (torchrun): STRONG scaling -- the CSR is replicated (each rank generates it on its GPU),
rank r runs a balanced contiguous range of the 128 probes, one NCCL all-gather per operator
assembles every rule on every rank; device time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SLQ edge·probe·steps/sec"
UNIT = "edge·probe·step/s"
T_GRID = 250
NL, P = "normalized_laplacian", "density"

CONFIGS = {
    "c5": {"workload": "C5 R-MAT scale 27 (ef 16, a=.57 b=.19 c=.19), 128 probes x 15 steps, fp32, "
                       "heat+wave (normalized Laplacian) + VNGE (density), T=250 t in [1e-2,1e2]",
           "graph": "rmat", "scale": 27, "edge_factor": 16, "abc": [0.57, 0.19, 0.19], "graph_seed": 0,
           "n_v": 128, "lanczos_steps": 15, "T": T_GRID, "dtype": "f32", "ops": ["heat", "wave", "vnge"],
           "reorth": "full CGS (reference default)", "graph_source": "device R-MAT generator",
           "l2": "inputs >> L2 (17 GB CSR, 8 GB per Lanczos vector block); L2 also flushed between steps"},
    "c4": {"workload": "C4 R-MAT scale 20 (ef 16, a=.57 b=.19 c=.19), 100 probes x 15 steps, fp64, "
                       "heat (normalized Laplacian) + VNGE (density), T=250 t in [1e-2,1e2]",
           "graph": "rmat", "scale": 20, "edge_factor": 16, "abc": [0.57, 0.19, 0.19], "graph_seed": 0,
           "n_v": 100, "lanczos_steps": 15, "T": T_GRID, "dtype": "f64", "ops": ["heat", "vnge"],
           "reorth": "full CGS (reference default)", "graph_source": "device R-MAT generator",
           "l2": "flushed between timed steps (256 MiB write), outside the timed events"},
    "c3": {"workload": "C3 10,000 Erdos-Renyi graphs (n ~ U[20,200], p ~ U[0.05,0.3]) stacked block-diagonally, "
                       "20 probes x 10 steps, fp32, per-graph heat trace, T=250 t in [1e-2,1e2]",
           "graph": "er_batch", "graphs": 10_000, "graph_seed": 0, "n_v": 20, "lanczos_steps": 10, "T": T_GRID,
           "dtype": "f32", "ops": ["heat"], "reorth": "full CGS (reference default)",
           "graph_source": "host ER generator (synth.er_batch)",
           "l2": "flushed between timed steps (256 MiB write), outside the timed events"},
    "c2": {"workload": "C2 SBM n=100000 blocks=10 p_in=1e-3 p_out=1e-5, 100 probes x 15 steps, fp64, "
                       "heat+wave (normalized Laplacian), T=250 t in [1e-2,1e2]",
           "graph": "sbm", "n": 100_000, "blocks": 10, "p_in": 1e-3, "p_out": 1e-5, "graph_seed": 0,
           "n_v": 100, "lanczos_steps": 15, "T": T_GRID, "dtype": "f64", "ops": ["heat", "wave"],
           "reorth": "full CGS (reference default)", "graph_source": "host SBM generator",
           "l2": "flushed between timed steps (256 MiB write), outside the timed events"},
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def operator_runs(cfg):
    """[(kind, [integrand codes])]: heat/wave share one normalized-Laplacian run, VNGE is a density run."""
    from paper_2003_01282_b200 import _lib

    runs = []
    nl = ([_lib.FN_HEAT] if "heat" in cfg["ops"] else []) + \
         ([_lib.FN_WAVE_RE, _lib.FN_WAVE_IM] if "wave" in cfg["ops"] else [])
    if nl:
        runs.append((NL, nl))
    if "vnge" in cfg["ops"]:
        runs.append((P, [_lib.FN_XLOGX]))
    return runs


def config_dict(cfg, world):
    c = {k: v for k, v in cfg.items() if k not in ("dtype",)}
    c["parallelism"] = f"probe-sharded x{world} (CSR replicated)" if world > 1 else "single GPU"
    c["scaling_mode"] = "strong: n_v probes split over the ranks"
    return c


class ClockSampler:
    """SM clocks + throttle reasons sampled every 20 ms during the timed region (NVML).  Reasons
    reported: hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.sm, self.smax, self.mask = [], [], 0
        self.stop_flag = threading.Event()
        self.thread = None
        self.nvml = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
        except Exception:
            self.nvml = None
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nvml
        while not self.stop_flag.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
                self.smax.append(nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                self.mask |= int(fn(self.handle))
            except Exception:
                pass
            time.sleep(0.02)

    def stop(self) -> dict:
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_flag.set()
        self.thread.join(timeout=2)
        reasons = [name for name, bit in self.REASONS if self.mask & bit]
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.smax) if self.smax else None, "reasons": reasons,
                "samples": len(self.sm), "source": "nvml 20 ms"}


def spin_up(torch, dev, seconds=0.5):
    """Untimed GPU load before the warm-up steps so SM clocks have left their idle state."""
    buf = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        buf.mul_(1.0001)
        torch.cuda.synchronize(dev)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, bf16 copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------------------------- graphs
def device_graph(cfg, dev):
    """The workload graph on `dev` (R-MAT generated on the device; SBM built on the host)."""
    from paper_2003_01282_b200.device import DeviceGraph

    if cfg["graph"] == "rmat":
        a, b, c = cfg["abc"]
        test_scale = os.environ.get("BENCH_TEST_RMAT_SCALE")   # tests only: a small stand-in graph (the
        if test_scale:                                         # line then says so in config.workload)
            cfg["scale"] = int(test_scale)
            cfg["workload"] = f"TEST RUN at R-MAT scale {test_scale}, NOT the benchmark: " + cfg["workload"]
        return DeviceGraph.rmat(cfg["scale"], cfg["edge_factor"], a, b, c, seed=cfg["graph_seed"], device=dev), None
    from paper_2003_01282_b200 import synth

    g = synth.sbm(cfg["n"], cfg["blocks"], cfg["p_in"], cfg["p_out"], seed=cfg["graph_seed"])
    return DeviceGraph(g, dev), g


def host_csr(dg, g):
    """(offsets int64 [n+1], cols int32 [nnz]) numpy arrays of the workload graph."""
    import numpy as np

    if g is not None:
        return np.asarray(g.row_offsets, dtype=np.int64), np.asarray(g.col_indices, dtype=np.int32)
    return dg.csr()


# ----------------------------------------------------------------------------------- CPU arms
def cpu_operator(off, cols, n, kind):
    """The oracle port's operator (scipy CSR + degrees: the reference's make_operator arithmetic)."""
    import numpy as np

    from oracle import slq_oracle as O
    from paper_2003_01282_b200.graphs import Graph

    g = Graph.__new__(Graph)   # the oracle reads n, m, row_offsets, col_indices, weights
    object.__setattr__(g, "n", int(n))
    object.__setattr__(g, "m", int(cols.size // 2))
    object.__setattr__(g, "row_offsets", off)
    object.__setattr__(g, "col_indices", cols)
    object.__setattr__(g, "weights", np.ones(cols.size))
    return O.make_block_operator(g, kind)


def cpu_sample(op, nnz, probes, steps, threads):
    """The oracle port (numpy + scipy: the reference's per-probe arithmetic, probes spread over
    `threads` host threads like the reference's thread map, slq.py:80-86) timed on the host:
    `probes` probes x `steps` Lanczos steps (+ the heat grid when steps > 1).  Returns (units/s, s)."""
    from oracle import slq_oracle as O

    t0 = time.perf_counter()
    rules = O.slq_rules(op, probes, steps, 0, threads=threads)
    if steps > 1:
        O.heat_from_rules(rules, op.dim, O.time_grid(1e-2, 1e2, T_GRID))
    dt = time.perf_counter() - t0
    return nnz * probes * steps / dt, dt


def big_graph(cfg):
    return cfg["graph"] == "rmat" and cfg["scale"] >= 24


def cpu_row_sample_operator(off, cols, n, every):
    """The oracle port's normalized-Laplacian apply (operators.py:84-89 arithmetic: scipy csr_matvecs +
    numpy elementwise) restricted to every `every`-th row of the graph, against full-length vectors:
    the C5 sample.  Gathers still range over the whole vector, so the per-nonzero cost is the full
    operator's.  Returns (apply(x [n, c]) -> y [rows, c], alpha(x, y) -> [c], sampled nnz)."""
    import numpy as np
    import scipy.sparse as sp

    deg = np.diff(off).astype(np.float64)          # unit weights: degree = row length (operators.py:58-62)
    pos = deg > 0
    dis = np.zeros(n)
    dis[pos] = 1.0 / np.sqrt(deg[pos])
    rows = np.arange(0, n, every, dtype=np.int64)
    starts, ends = off[rows], off[rows + 1]
    lens = ends - starts
    sub_off = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(lens, out=sub_off[1:])
    idx = np.repeat(starts - sub_off[:-1], lens) + np.arange(sub_off[-1], dtype=np.int64)
    sub = sp.csr_matrix((np.ones(sub_off[-1]), cols[idx].astype(np.int64), sub_off), shape=(rows.size, n))
    keep_r = pos[rows].astype(np.float64)[:, None]
    dis_r = dis[rows][:, None]
    disc = dis[:, None]

    def apply(x):
        return keep_r * x[rows] - dis_r * (sub @ (disc * x))

    def alpha(x, y):
        return np.einsum("nc,nc->c", x[rows], y)

    return apply, alpha, int(sub_off[-1])


_PROBE_CACHE: dict = {}


def cpu_row_sample(sampler, n, probes, threads):
    """`probes` unit Rademacher probes (one per host thread, like the reference's thread map over
    probes, slq.py:80-86), each: one operator apply + alpha on the sampled rows.  Returns (units/s, s)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import slq_oracle as O

    apply, alpha, nnz_s = sampler[:3]
    key = (n, probes)
    if key not in _PROBE_CACHE:                                # drawn once, outside the timed region
        _PROBE_CACHE.clear()
        _PROBE_CACHE[key] = [O.draw_probes(n, 0, [p]) for p in range(probes)]
    qs = _PROBE_CACHE[key]
    t0 = time.perf_counter()

    def one(q):
        return alpha(q, apply(q))

    if threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(one, qs))
    else:
        for q in qs:
            one(q)
    dt = time.perf_counter() - t0
    return nnz_s * probes / dt, dt


def cpu_baseline_for(cfg, op, nnz, threads):
    """Bounded CPU sample of the workload (about 5-30 s).  C5 (`op` is a row sampler from
    cpu_row_sample_operator): one Lanczos operator application + alpha of one probe per host thread on
    every 8th row of the real graph (per-probe-step cost is independent of n_v; the full
    signature would take hours on the host); C2/C4: all probes, all steps of the heat run."""
    if big_graph(cfg):
        v, dt = cpu_row_sample(op, op[3], threads, threads)
        sample = (f"{threads} probes (one per host thread) x 1 Lanczos operator application + alpha of the "
                  f"normalized Laplacian on every 8th row of the same R-MAT-{cfg['scale']} graph (full-length "
                  f"vectors; numpy+scipy port of operators.py:84-89); units = sampled stored nonzeros x probes")
        return v, dt, sample, threads
    probes, steps = cfg["n_v"], cfg["lanczos_steps"]
    sample = f"all {probes} probes x {steps} steps of the heat run (oracle port, numpy+scipy)"
    v, dt = cpu_sample(op, nnz, probes, steps, threads)
    return v, dt, sample, threads


def cpu_op_for(cfg, off, cols, n):
    """The CPU arm's operator: the C5 row sampler, or the full oracle operator for C2/C4."""
    if big_graph(cfg):
        return (*cpu_row_sample_operator(off, cols, n, 8), n)
    return cpu_operator(off, cols, n, NL)


def run_reference(args, cfg):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    if cfg["graph"] == "er_batch":
        graphs = er_graphs(cfg)
        vals, times = [], []
        count = 300
        for k in range(args.warmup + args.steps):
            v, dt = cpu_batch_sample(graphs, cfg, count)
            if k >= args.warmup:
                vals.append(v)
                times.append(dt)
        value = float(np.mean(vals))
        units_step = sum(g.nnz * cfg["n_v"] * min(cfg["lanczos_steps"], g.n) for g in graphs)
        sample = f"first {count} of {len(graphs)} graphs, per-graph oracle heat trace (numpy+scipy port, one thread)"
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * units_step / value, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic (seeded)",
                "config": config_dict(cfg, args.gpus), "impl": "reference",
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    if cfg["graph"] == "rmat":
        # input preparation only: the R-MAT graph is generated by the device generator and copied to
        # the host (a host generator would take longer than the whole benchmark at scale 27)
        import torch

        torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
        dg, g = device_graph(cfg, torch.device("cuda", torch.cuda.current_device()))
        off, cols = host_csr(dg, g)
        n = dg.n
        del dg
        torch.cuda.empty_cache()
        from paper_2003_01282_b200 import _lib

        _lib.trim_pool()
    else:
        from paper_2003_01282_b200 import synth

        g = synth.sbm(cfg["n"], cfg["blocks"], cfg["p_in"], cfg["p_out"], seed=cfg["graph_seed"])
        off, cols, n = np.asarray(g.row_offsets), np.asarray(g.col_indices), g.n
    op = cpu_op_for(cfg, off, cols, n)
    nnz = int(cols.size)
    del off, cols
    log(f"reference arm: graph + operator ready in {time.perf_counter() - t0:.1f} s (n={n}, nnz={nnz})")
    vals, times, sample = [], [], ""
    for k in range(args.warmup + args.steps):
        v, dt, sample, used = cpu_baseline_for(cfg, op, nnz, threads)
        if k >= args.warmup:
            vals.append(v)
            times.append(dt)
    value = float(np.mean(vals))
    units_step = len(operator_runs(cfg)) * nnz * cfg["n_v"] * cfg["lanczos_steps"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * units_step / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic (seeded)",
            "config": config_dict(cfg, args.gpus), "impl": "reference", "graph": {"n": int(n), "nnz": int(nnz)},
            "ms_per_sample": 1e3 * float(np.mean(times)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------------- roofline
def spmm_bytes_per_launch(n_rows, nnz, c, vb, s):
    """Algorithmic DRAM bytes of one SpMM launch, averaged over the s launches of a chunk:
    per nonzero one gathered c-wide row (no-reuse model) + its int32 column index; per row the offsets
    (8 B), dinv/degree (16 B), its own row of the input vector and the output row.  Step 0 gathers the
    16-byte probe bitmask rows instead of c*vb."""
    row = c * vb
    later = nnz * (row + 4) + n_rows * (2 * row + 24)
    first = nnz * (16 + 4) + n_rows * (16 + row + 24)
    return (first + (s - 1) * later) / s


def step_bytes_per_launch(n_rows, c, vb, s):
    """Algorithmic DRAM bytes of one CGS step-kernel launch, averaged over the s-1 launches: at step i,
    phase A streams w, u_1..u_i and the probe bitmask; phase C streams them again and writes u_{i+1}."""
    row = c * vb
    tot = sum(n_rows * row * (2 * (i + 1) + 1) + 2 * n_rows * 16 for i in range(s - 1))
    return tot / (s - 1)


# ----------------------------------------------------------------------------------- C3 (many small graphs)
def er_graphs(cfg):
    from paper_2003_01282_b200 import synth

    return synth.er_batch(cfg["graphs"], seed=cfg["graph_seed"])


def cpu_batch_sample(graphs, cfg, count):
    """Oracle port on the first `count` graphs (per-graph netlsd heat, the reference's per-graph call)."""
    from oracle import slq_oracle as O

    t = O.time_grid(1e-2, 1e2, T_GRID)
    units = 0
    t0 = time.perf_counter()
    for g in graphs[:count]:
        O.heat_trace(g, t, cfg["n_v"], cfg["lanczos_steps"], 0, threads=1)
        units += g.nnz * cfg["n_v"] * min(cfg["lanczos_steps"], g.n)
    dt = time.perf_counter() - t0
    return units / dt, dt


def run_ours_batch(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2003_01282_b200 import _lib
    from paper_2003_01282_b200.batched import netlsd_slq_batch
    from paper_2003_01282_b200.dist import ShardedBatch, probe_ranges
    from paper_2003_01282_b200.slq import SlqConfig

    world, rank, local = dist_env()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    dtype = args.dtype or cfg["dtype"]
    scfg = SlqConfig(n_v=cfg["n_v"], s=cfg["lanczos_steps"], seed=0)
    t0 = time.perf_counter()
    graphs = er_graphs(cfg)
    sb = ShardedBatch(graphs, device=dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    tvals = np.geomspace(1e-2, 1e2, T_GRID)
    tvals[0], tvals[-1] = 1e-2, 1e2
    units_step = sum(g.nnz * cfg["n_v"] * min(cfg["lanczos_steps"], g.n) for g in graphs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        return sb.values("normalized_laplacian", scfg, tvals, _lib.FN_HEAT, dtype)

    spin_up(torch, dev)
    for _ in range(args.warmup):
        _, _, status = step()
    _lib.check_status(int(status.item()))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local) if (rank == 0 and not os.environ.get("BENCH_NO_CLOCKS")) else None
    if sampler:
        sampler.start()
    launches0 = _lib.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.fill_(1)
        ev[k][0].record(stream)
        vals, stds, status = step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    launches = (_lib.launch_count() - launches0) // args.steps
    _lib.check_status(int(status.item()))
    clocks = sampler.stop() if sampler else None
    times = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(times))
    if world > 1:
        tt = torch.tensor([ms], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = units_step / (ms * 1e-3)
    _lib.profile_begin()
    step()
    torch.cuda.synchronize()
    prof = _lib.profile_end()
    # e2e: the public API on host graphs (block-diagonal stacking, H2D, device run, D2H) for this rank's range
    b, e = probe_ranges(len(graphs), world)[rank]
    mine = graphs[b:e]
    h2d = sum((g.n + 1) * 8 + g.nnz * 8 for g in mine)
    e2e_times = []
    for k in range(args.e2e_reps + 1):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        hv, hs = netlsd_slq_batch(mine, TimeGridLike(tvals), scfg, dtype=dtype)
        dt = time.perf_counter() - t1
        if k >= 1:
            e2e_times.append(dt)
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    if rank != 0:
        dist.destroy_process_group()
        return 0
    peak, peak_src = measured_peaks()
    nnz_total = sum(g.nnz for g in graphs)
    n_total = sum(g.n for g in graphs)
    bat = prof.get("batched", {"ms": 0.0, "launches": 0})
    # algorithmic bytes of the batched Lanczos kernel: each step streams the graph's CSR (int32 columns +
    # int64 offsets) and the c-wide vectors it reads/writes (rows of c * vb, 3 vectors); vectors of one
    # graph are L2/SMEM-resident, so this is a streaming lower bound, not an HBM target
    vb = 4 if dtype == "f32" else 8
    s_ = cfg["lanczos_steps"]
    local_nnz = sum(g.nnz for g in mine)
    local_n = sum(g.n for g in mine)
    alg = s_ * (local_nnz * 4 + local_n * 8 + 3 * local_n * cfg["n_v"] * vb)
    bat_ms = bat["ms"] / max(1, bat["launches"])
    roof = {"bound": "hbm", "kernel": "batched_lanczos", "achieved": alg / (bat_ms * 1e-3) / 1e9 if bat_ms else None,
            "peak": peak, "unit": "GB/s", "frac": (alg / (bat_ms * 1e-3) / 1e9 / peak) if bat_ms else None,
            "traffic": None, "peak_source": peak_src, "algorithmic_bytes_per_launch": alg,
            "ms_per_launch": bat_ms, "note": "latency/SMEM-bound per-graph CTAs (SURVEY §8d: no HBM fraction target)"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtype, "data": f"synthetic (seeded; {cfg['graph_source']})",
            "config": config_dict(cfg, world),
            "graph": {"graphs": len(graphs), "n": n_total, "nnz": nnz_total, "graphs_per_rank": e - b},
            "roofline": roof,
            "kernels": {k: v for k, v in prof.items() if v["launches"]},
            "ms_steps": [round(t, 3) for t in times], "gpu_launches": launches, "graph_build_s": round(gen_s, 3),
            "clocks": clocks,
            "e2e": {"value": units_step / e2e_s, "unit": UNIT, "seconds_per_signature": e2e_s,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 2 * (e - b) * T_GRID * 8 + 4,
                    "api": "netlsd_slq_batch(list of host Graphs): block-diagonal stacking, H2D, device run, D2H"}}
    if not args.no_cpu_baseline and world == 1:
        count = 300
        v, dt = cpu_batch_sample(graphs, cfg, count)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"first {count} of {len(graphs)} graphs, per-graph oracle heat trace "
                                          f"(numpy+scipy port, one thread; graphs are independent); {dt:.1f} s"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


class SharedHostCsr:
    """The workload CSR (int64 offsets, int32 columns) as ONE host copy shared by the ranks of a
    multi-rank run (N private pinned copies of the 18 GB C5 CSR would not fit the host): local rank 0
    writes it from its device to files in $TMPDIR (/tmp), every rank maps them read-only (one copy in
    the page cache).  /dev/shm is not used: on the GPU boxes its writes fault (SIGBUS) well below the
    size df reports.  The H2D copies run from this pageable mapping.  When the temp directory lacks the
    space, each rank falls back to a private pinned copy.  Exposes torch views `offsets` / `cols`."""

    def __init__(self, dg, g, rank, local, world, torch, dist):
        import shutil
        import tempfile

        import numpy as np

        self.dist, self.local = dist, local
        n, nnz = dg.n, dg.nnz
        need = (n + 1) * 8 + nnz * 4
        base = tempfile.gettempdir()
        ok = torch.tensor([1 if shutil.disk_usage(base).free > 1.5 * need else 0],
                          device=dg.device if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)   # every rank takes the same branch
        self.paths = []
        if not int(ok.item()):
            off_h, cols_h = host_csr(dg, g)
            self.offsets = torch.from_numpy(np.ascontiguousarray(off_h)).pin_memory()
            self.cols = torch.from_numpy(np.ascontiguousarray(cols_h)).pin_memory()
            return
        tag = os.environ.get("MASTER_PORT", "0")
        self.paths = [os.path.join(base, f"slq_bench_{tag}_offsets.bin"), os.path.join(base, f"slq_bench_{tag}_cols.bin")]
        if local == 0:
            off_h, cols_h = host_csr(dg, g)
            np.ascontiguousarray(off_h, dtype=np.int64).tofile(self.paths[0])
            np.ascontiguousarray(cols_h, dtype=np.int32).tofile(self.paths[1])
            del off_h, cols_h
        dist.barrier()
        self.maps = [np.memmap(self.paths[0], dtype=np.int64, mode="r+", shape=(n + 1,)),
                     np.memmap(self.paths[1], dtype=np.int32, mode="r+", shape=(nnz,))]
        self.offsets = torch.from_numpy(self.maps[0])
        self.cols = torch.from_numpy(self.maps[1])

    def close(self):
        self.dist.barrier()
        if self.local == 0:
            for path in self.paths:
                try:
                    os.unlink(path)   # mappings stay valid until released
                except OSError:
                    pass


class TimeGridLike:
    """A TimeGrid carrying exactly the bench's t values (geomspace with pinned endpoints)."""

    def __init__(self, values):
        self.values = values
        self.t_min, self.t_max, self.count = float(values[0]), float(values[-1]), len(values)


# ----------------------------------------------------------------------------------- our arm
def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2003_01282_b200 import _lib
    from paper_2003_01282_b200.device import DeviceGraph
    from paper_2003_01282_b200.dist import pair_applies, probe_ranges, sharded_rules, sharded_rules_pair
    from paper_2003_01282_b200.slq import SlqConfig

    world, rank, local = dist_env()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")   # gloo: multi-rank test on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    dtype = args.dtype or cfg["dtype"]
    vb = 8 if dtype == "f64" else 4
    s, n_v = cfg["lanczos_steps"], cfg["n_v"]
    runs = operator_runs(cfg)
    scfg = SlqConfig(n_v=n_v, s=s, seed=0)
    t0 = time.perf_counter()
    dg, g = device_graph(cfg, dev)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    n, nnz = dg.n, dg.nnz
    info = dg.info
    n_rows = (n - info.isolated + 1) if dg.folded else n     # Lanczos vector rows (isolated-vertex fold)
    log(f"rank {rank}: graph n={n} nnz={nnz} folded={dg.folded} ready in {gen_s:.1f} s")
    tgrid = torch.tensor(np.geomspace(1e-2, 1e2, T_GRID), device=dev)
    tgrid[0], tgrid[-1] = 1e-2, 1e2
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    # 9..16 probes per rank and both operators wanted (C5 on 8 GPUs): the operator-pair block runs the
    # normalized-Laplacian and the density Lanczos of a rank's probes on one pass over the graph per step
    paired = world > 1 and [k for k, _ in runs] == [NL, P] and pair_applies(n_v, world, dtype)

    def signature(graph):
        outs, statuses = [], []
        if paired:
            for rules, (kind, fns) in zip(sharded_rules_pair(graph, scfg, dtype=dtype), runs):
                vals, stds = rules.integrate(tgrid if kind == NL else None, fns)
                outs.append((vals, stds))
                statuses.append(rules.status)
            return outs, statuses
        for kind, fns in runs:
            if world > 1:
                rules = sharded_rules(graph, kind, scfg, dtype=dtype)
            else:
                rules = graph.rules(kind, 0, 0, n_v, s, dtype=dtype)
            vals, stds = rules.integrate(tgrid if kind == NL else None, fns)
            outs.append((vals, stds))
            statuses.append(rules.status)
        return outs, statuses

    def check(statuses):
        for st in statuses:
            _lib.check_status(int(st.item()))

    spin_up(torch, dev)
    for _ in range(args.warmup):
        _, statuses = signature(dg)
    check(statuses)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local) if (rank == 0 and not os.environ.get("BENCH_NO_CLOCKS")) else None
    if sampler:
        sampler.start()
    launches0 = _lib.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    h0 = time.perf_counter()
    for k in range(args.steps):
        flush.fill_(1)
        ev[k][0].record(stream)
        _, statuses = signature(dg)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    host_s = time.perf_counter() - h0
    launches = (_lib.launch_count() - launches0) // args.steps
    check(statuses)
    times = [a.elapsed_time(b) for a, b in ev]
    times_eager = times
    log(f"rank {rank}: timed steps {[round(t, 1) for t in times]} ms")
    # small graphs (C2): one step captured as a CUDA graph and replayed (the same kernels, one launch)
    cuda_graph = world == 1 and cfg["graph"] == "sbm" and not os.environ.get("BENCH_EAGER")
    graph_note = None
    if cuda_graph:
        try:
            side = torch.cuda.Stream()
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                signature(dg)
            stream.wait_stream(side)
            torch.cuda.synchronize()
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg, capture_error_mode="thread_local"):
                _, cap_status = signature(dg)
            torch.cuda.synchronize()
            gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for k in range(args.steps):
                flush.fill_(1)
                gev[k][0].record(stream)
                cg.replay()
                gev[k][1].record(stream)
            torch.cuda.synchronize()
            check(cap_status)
            times = [a.elapsed_time(b) for a, b in gev]
        except Exception as ex:   # capture unavailable: report the eager loop (same kernels)
            cuda_graph, graph_note = False, repr(ex)[:200]
            torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    ms = float(np.mean(times))
    if world > 1:
        t = torch.tensor([ms], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    units_step = len(runs) * nnz * n_v * s
    value = units_step / (ms * 1e-3)

    # ---- one more step with per-launch CUDA events on the launching stream (kernel durations) ----
    _lib.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.fill_(1)
    e0.record(stream)
    signature(dg)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_profiled = e0.elapsed_time(e1)
    prof = _lib.profile_end()

    # ---- e2e: host CSR (pinned, int32 columns) -> device graph -> signature -> host values ----
    last_vals = [v.clone() for v, _ in signature(dg)[0]]
    _lib.trim_pool()             # the Lanczos workspaces cached in the pool are not needed for the copy
    if world == 1:
        off_h, cols_h = host_csr(dg, g)
        torch.cuda.empty_cache()
        pin_off = torch.from_numpy(np.ascontiguousarray(off_h)).pin_memory()
        pin_cols = torch.from_numpy(np.ascontiguousarray(cols_h)).pin_memory()
        del off_h, cols_h
        shared = None
    else:
        # N ranks on one node: ONE host copy of the CSR (18 GB at C5) in shared memory, page-locked by
        # every rank, instead of N private pinned copies that would not fit the host
        shared = SharedHostCsr(dg, g, rank, local, world, torch, dist)
        pin_off, pin_cols = shared.offsets, shared.cols
        torch.cuda.empty_cache()
    folded = dg.folded
    del dg                       # the e2e leg builds its own device graph from the host arrays
    torch.cuda.synchronize()
    h2d = pin_off.numel() * 8 + pin_cols.numel() * 4
    d2h = 0
    e2e_times = []
    for k in range(args.e2e_reps + 1):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dg2 = DeviceGraph.from_csr32(n, pin_off, pin_cols, device=dev)   # H2D + prepare (+ fold)
        outs, statuses = signature(dg2)
        host_vals = [(v.cpu(), sd.cpu()) for v, sd in outs]              # D2H of the descriptors
        check(statuses)
        dt = time.perf_counter() - t0
        del dg2, outs
        if k >= 1:                                                       # rep 0: untimed warm-up
            e2e_times.append(dt)
        d2h = sum(v.numel() * 8 + sd.numel() * 8 for v, sd in host_vals)
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = units_step / e2e_s
    # the e2e descriptors equal the device-resident run's bit for bit (same graph, same probes)
    same = all(torch.equal(hv.to(dev), dv) for (hv, _), dv in zip(host_vals, last_vals))
    if shared is not None:
        shared.close()

    if rank != 0:
        dist.destroy_process_group()
        return 0
    # ---- roofline of the dominant kernel class ----
    peak, peak_src = measured_peaks()
    b, e = probe_ranges(n_v, world)[0]
    per_rank = e - b
    nchunks = max(1, round(prof["spmm"]["launches"] / (len(runs) * s))) if prof["spmm"]["launches"] else 1
    c = -(-per_rank // nchunks)
    if paired:   # one block of both operators' columns per rank
        c = 2 * (-(-per_rank // 4) * 4)
    ab = {"spmm": spmm_bytes_per_launch(n_rows, nnz, c, vb, s), "cgs_step": step_bytes_per_launch(n_rows, c, vb, s)}
    per_class = {}
    for k, v in prof.items():
        if v["launches"] == 0:
            continue
        per_class[k] = {"ms_per_step": v["ms"], "launches_per_step": v["launches"],
                        "ms_per_launch": v["ms"] / v["launches"]}
        if k in ab:
            per_class[k]["algorithmic_bytes_per_launch"] = ab[k]
            per_class[k]["achieved_GBs"] = ab[k] / (per_class[k]["ms_per_launch"] * 1e-3) / 1e9
    dom = max((k for k in ab if k in per_class), key=lambda k: per_class[k]["ms_per_step"])
    ach = per_class[dom]["achieved_GBs"]
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", f"r2_traffic_{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tk = json.load(f)["kernels"].get(dom)
        if tk:
            traffic = tk["dram_bytes_per_launch"]
            traffic_src = f"profiles/r2_traffic_{args.config}.json (ncu --set full: dram read+write per launch)"
    roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": ab[dom], "ms_per_launch": per_class[dom]["ms_per_launch"],
            "chunk_probes": c, "vector_rows": n_rows}
    if traffic:
        roof["dram_GBs"] = traffic / (per_class[dom]["ms_per_launch"] * 1e-3) / 1e9
        roof["dram_frac"] = roof["dram_GBs"] / peak
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": dtype, "data": f"synthetic (seeded; {cfg['graph_source']})",
        "config": config_dict(cfg, world),
        "graph": {"n": n, "nnz": nnz, "folded_isolated": folded, "vector_rows": n_rows, "probes_per_rank": per_rank,
                  "operator_pair_block": bool(paired)},
        "roofline": roof,
        "kernels": per_class,
        "ms_per_step_profiled": ms_profiled,
        "ms_steps": [round(t, 3) for t in times],
        "launch": "one CUDA-graph replay per step" if cuda_graph else
                  ("eager launches" + (f" (capture failed: {graph_note})" if graph_note else "")),
        "ms_per_step_eager": float(np.mean(times_eager)),
        "host_submit_s_total": round(host_s, 3),
        "gpu_launches": launches,
        "graph_build_s": round(gen_s, 3),
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": UNIT, "seconds_per_signature": e2e_s,
                "s_signatures": [round(x, 3) for x in e2e_times],
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "DeviceGraph.from_csr32 (slq_graph_create_i32: pinned host int64 offsets + int32 columns, "
                       "H2D, device prepare, isolated-vertex fold) + slq_rules + slq_integrate per operator, "
                       "D2H of values and std errors",
                "values_equal_device_resident_run": bool(same)},
    }
    log(f"e2e: {e2e_s:.2f} s per signature; device {ms:.1f} ms per step; value {value:.4g}")
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        op = cpu_op_for(cfg, pin_off.numpy(), pin_cols.numpy(), n)      # copies what it keeps
        del pin_off, pin_cols
        try:
            torch._C._host_emptyCache()                                # give the pinned pages back
        except Exception:
            pass
        v, dt, sample, used = cpu_baseline_for(cfg, op, nnz, threads)
        log(f"cpu baseline: {v:.4g} units/s on {used} threads ({dt:.1f} s)")
        if big_graph(cfg):
            v1, dt1 = cpu_row_sample(op, n, 1, 1)
            s1 = 1
        else:
            s1 = s
            v1, dt1 = cpu_sample(op, nnz, 1, s1, 1)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": used, "kind": "port",
                                "sample": f"{sample}; {dt:.1f} s",
                                "value_1_thread": v1,
                                "sample_1_thread": (f"1 probe, 1 operator application + alpha on every 8th row, 1 thread; "
                                                    f"{dt1:.1f} s") if big_graph(cfg) else
                                                   f"1 probe x {s1} steps, 1 thread; {dt1:.1f} s"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c5")
    ap.add_argument("--dtype", choices=["f64", "f32"], default=None, help="vector storage (default: the config's)")
    ap.add_argument("--e2e-reps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules; using 3")
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if cfg["graph"] == "er_batch":
        return run_ours_batch(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
