"""Benchmark: SLQ edge·probe·steps/s on BASELINE.json configs[1] (C2).

Workload (one "step" = one full signature computation over the graph):
  SBM n=100,000, 10 equal blocks, p_in=1e-3, p_out=1e-5 (seeded synthetic), normalized Laplacian,
  n_v=100 Rademacher probes x s=15 Lanczos steps (full CGS reorth, the reference default),
  heat + wave traces on 250 log-spaced t in [1e-2, 1e2], fp64 (``--dtype f32`` for fp32 storage).
  Units per step = nnz * n_v * s (one stored nonzero x one probe x one operator application).

Arms:
  default            hand-written sm_100a kernels through libslq_b200.so
  --impl reference   the CPU oracle port of the reference algorithm (oracle/slq_oracle.py, numpy +
                     scipy, all host threads) on the same config; rank 0 only.

Timing: W warm-up steps, then K timed steps, each bracketed by CUDA events on the launching stream;
L2 is flushed (256 MiB write) between timed steps, outside the events.  Multi-GPU: one process per
GPU (torchrun), weak scaling: rank r runs probes [100r, 100r+100) and the rules are all-gathered
over NCCL; device time = max over ranks.
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

WORKLOAD = {"workload": "C2 SBM n=100000 blocks=10 p_in=1e-3 p_out=1e-5, normalized Laplacian, "
                        "heat+wave T=250 t in [1e-2,1e2]",
            "graph": "sbm", "n": 100_000, "blocks": 10, "p_in": 1e-3, "p_out": 1e-5, "graph_seed": 0,
            "n_v_per_gpu": 100, "lanczos_steps": 15, "T": 250, "reorth": "full CGS (reference default)",
            "l2": "flushed between timed steps (256 MiB write), outside the timed events"}
METRIC = "SLQ edge·probe·steps/sec"
UNIT = "edge·probe·step/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clocks + throttle reasons sampled every 20 ms during the timed region (NVML; nvidia-smi
    fallback).  Reasons reported: hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap."""

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


def build_graph():
    from paper_2003_01282_b200 import synth

    return synth.sbm(WORKLOAD["n"], WORKLOAD["blocks"], WORKLOAD["p_in"], WORKLOAD["p_out"],
                     seed=WORKLOAD["graph_seed"])


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, bf16 copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_baseline(g, n_v, s, grid, threads, max_probes=None):
    """Oracle port of the reference algorithm timed on the host cores (bounded sample)."""
    from oracle import slq_oracle as O

    probes = n_v if max_probes is None else min(n_v, max_probes)
    t0 = time.perf_counter()
    op = O.make_block_operator(g, O.NORMALIZED_LAPLACIAN)
    rules = O.slq_rules(op, probes, s, 0, threads=threads)
    O.heat_from_rules(rules, g.n, grid)
    O.wave_from_rules(rules, g.n, grid)
    dt = time.perf_counter() - t0
    units = g.nnz * probes * s
    return units / dt, dt, probes


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np

    from oracle import slq_oracle as O

    g = build_graph()
    s, n_v = WORKLOAD["lanczos_steps"], WORKLOAD["n_v_per_gpu"]
    grid = O.time_grid(1e-2, 1e2, WORKLOAD["T"])
    threads = os.cpu_count() or 1
    vals, times = [], []
    for k in range(args.warmup + args.steps):
        v, dt, probes = cpu_baseline(g, n_v, s, grid, threads, max_probes=args.ref_probes)
        if k >= args.warmup:
            vals.append(v)
            times.append(dt)
    value = float(np.mean(vals))
    sample = f"first {probes} of {n_v} probes of the C2 workload (per-probe cost is independent of n_v), oracle port"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SBM)",
            "config": dict(WORKLOAD, parallelism="cpu threads"), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def algorithmic_bytes(g, c, s, vb):
    """Per-class algorithmic DRAM bytes of one Lanczos run on one chunk of c probes."""
    n, nnz = g.n, g.nnz
    row = c * vb
    spmm = s * (nnz * (row + 4) + n * (2 * row + 24))
    # CGS step kernel, step i: phase A streams w, u_1..u_i and the probe bitmask (u_0, 16 B/row);
    # phase C streams them again and writes u_{i+1}
    step = sum(n * row * (2 * (i + 1) + 1) + 2 * n * 16 for i in range(s - 1))
    return {"spmm": spmm, "cgs_step": step}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2003_01282_b200 import _lib
    from paper_2003_01282_b200.descriptors import TimeGrid, netlsd_heat_wave_slq
    from paper_2003_01282_b200.device import DeviceGraph
    from paper_2003_01282_b200.dist import gather_rules_arrays
    from paper_2003_01282_b200.graphs import Graph
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
    g = build_graph()
    s, n_v = WORKLOAD["lanczos_steps"], WORKLOAD["n_v_per_gpu"]
    total_probes = n_v * world
    grid = TimeGrid(1e-2, 1e2, WORKLOAD["T"])
    dtype = args.dtype
    vb = 8 if dtype == "f64" else 4
    tgrid = torch.tensor(np.array(grid.values), device=dev)
    off_d = torch.tensor(np.array(g.row_offsets), device=dev)
    cols_d = torch.tensor(np.array(g.col_indices), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    fns = [_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM]

    def step():
        # device-resident input: prepare + probes + Lanczos + rules + quadrature + aggregate (no host sync)
        import ctypes

        dg = DeviceGraph.__new__(DeviceGraph)
        dg.device, dg.graph, dg.n, dg._info = dev, g, g.n, None
        dg.handle = ctypes.c_void_p()
        _lib.check(_lib.load().slq_graph_create(g.n, g.nnz, off_d.data_ptr(), cols_d.data_ptr(), None,
                                                torch.cuda.current_stream().cuda_stream, ctypes.byref(dg.handle)))
        rules = dg.rules("normalized_laplacian", 0, rank * n_v, n_v, s, dtype=dtype)
        if world > 1:
            nodes, weights, steps = gather_rules_arrays(rules.nodes, rules.weights, rules.steps, total_probes)
            rules = type(rules)(nodes, weights, steps, g.n, status=rules.status)
        out = rules.integrate(tgrid, fns)
        del dg
        return out, rules.status

    spin_up(torch, dev)
    for _ in range(args.warmup):
        _, status = step()
    _lib.check_status(int(status.item()))   # the device reported no error on the warm-up steps
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local) if (rank == 0 and not os.environ.get("BENCH_NO_CLOCKS")) else None
    if sampler:
        sampler.start()
    launches0 = _lib.launch_count()
    # Enqueue all K steps without a host sync in between (the host runs ahead of the GPU, so host
    # jitter on a shared machine cannot starve it); each step is bracketed by its own events and
    # the L2 flush sits between steps, outside the events.
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    h0 = time.perf_counter()
    for k in range(args.steps):
        flush.fill_(1)
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    host_ms = 1e3 * (time.perf_counter() - h0)
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in ev]
    launches = (_lib.launch_count() - launches0) // args.steps
    times_eager = times
    # One step captured as a CUDA graph (graph preparation, probes, Lanczos, rules, quadrature and
    # aggregate: the same kernels, launched by one graph launch) and replayed K times; single rank only
    # (the multi-rank step has a host all-gather).  BENCH_EAGER=1 reports the eager loop instead.
    cuda_graph = world == 1 and not os.environ.get("BENCH_EAGER")
    graph_note = None

    def graph_times():
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            step()
        stream.wait_stream(side)
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, capture_error_mode="thread_local"):
            _, cap_status = step()
        torch.cuda.synchronize()
        cg.replay()
        torch.cuda.synchronize()
        _lib.check_status(int(cap_status.item()))
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for k in range(args.steps):
            flush.fill_(1)
            gev[k][0].record(stream)
            cg.replay()
            gev[k][1].record(stream)
        torch.cuda.synchronize()
        _lib.check_status(int(cap_status.item()))
        return [a.elapsed_time(b) for a, b in gev]

    if cuda_graph:
        try:
            times = graph_times()
        except Exception as ex:   # capture unavailable: report the eager loop (same kernels)
            cuda_graph, graph_note = False, repr(ex)[:200]
            times = times_eager
            torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    ms = float(np.mean(times))
    # same K steps again with per-launch CUDA events (kernel durations for the roofline)
    _lib.profile_begin()
    pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.fill_(1)
        pev[k][0].record(stream)
        step()
        pev[k][1].record(stream)
    torch.cuda.synchronize()
    ptimes = [a.elapsed_time(b) for a, b in pev]
    prof = _lib.profile_end()
    if world > 1:
        t = torch.tensor([ms], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    units_step = g.nnz * n_v * s * world
    value = units_step / (ms * 1e-3)

    # ---- e2e through the public API with host (pinned) buffers ----
    pin_off = torch.tensor(np.array(g.row_offsets)).pin_memory()
    pin_cols = torch.tensor(np.array(g.col_indices)).pin_memory()
    pin_w = torch.tensor(np.array(g.weights)).pin_memory()
    e2e_times = []
    cfg = SlqConfig(n_v=n_v, s=s, seed=0)
    h2d = (g.n + 1) * 8 + g.nnz * 8
    for k in range(args.warmup + args.steps):
        gh = Graph(n=g.n, row_offsets=pin_off.numpy(), col_indices=pin_cols.numpy(), weights=pin_w.numpy(), m=g.m)
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        heat, wave = netlsd_heat_wave_slq(gh, grid, cfg, dtype=dtype, with_hash=False)
        torch.cuda.synchronize()
        if k >= args.warmup:
            e2e_times.append(time.perf_counter() - t0)
    # the same call with the descriptor's graph_hash (SHA-256 of the host CSR bytes, descriptors.py
    # graph_hash; SURVEY 8d asks for signature seconds with and without it)
    hash_times = []
    for k in range(2):
        gh = Graph(n=g.n, row_offsets=pin_off.numpy(), col_indices=pin_cols.numpy(), weights=pin_w.numpy(), m=g.m)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        heat, wave = netlsd_heat_wave_slq(gh, grid, cfg, dtype=dtype, with_hash=True)
        torch.cuda.synchronize()
        hash_times.append(time.perf_counter() - t0)
    d2h = 3 * 2 * WORKLOAD["T"] * 8
    e2e_s = float(np.mean(e2e_times))
    e2e_value = g.nnz * n_v * s / e2e_s

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    # ---- roofline of the dominant kernel class ----
    peak, peak_src = measured_peaks()
    ab = algorithmic_bytes(g, n_v, s, vb)
    per_class = {}
    for k, v in prof.items():
        if v["launches"] == 0:
            continue
        t_ms = v["ms"]
        per_class[k] = {"ms_per_step": t_ms / args.steps, "launches_per_step": v["launches"] / args.steps}
        if k in ab:
            per_class[k]["GB_per_step"] = ab[k] / 1e9
            per_class[k]["achieved_GBs"] = (ab[k] * args.steps / (t_ms * 1e-3) / 1e9) if t_ms > 0 else None
    dom = max(ab, key=lambda k: per_class.get(k, {}).get("ms_per_step", 0.0))
    ach = per_class[dom]["achieved_GBs"]
    traffic, traffic_src = args.traffic, "--traffic" if args.traffic else None
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_traffic_c2.json")
    if traffic is None and os.path.exists(tpath):
        with open(tpath) as f:
            tk = json.load(f)["kernels"].get(dom)
        if tk:
            traffic = tk["dram_bytes_per_launch"]
            traffic_src = "profiles/r1_traffic_c2.json (ncu --set full, dram read+write per launch, avg over a signature)"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": dtype, "data": "synthetic (seeded SBM, BASELINE configs[1] shape)",
        "config": dict(WORKLOAD, parallelism=f"probe-sharded x{world}" if world > 1 else "single GPU",
                       total_probes=total_probes, nnz=g.nnz),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": (ach / peak) if ach else None, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": ab[dom] / max(1.0, per_class[dom]["launches_per_step"]),
                     "peak_source": peak_src},
        "kernels": per_class,
        "ms_per_step_profiled": float(np.mean(ptimes)),
        "ms_steps": [round(t, 3) for t in times],
        "launch": "one CUDA-graph replay per step (the eager step's kernels)" if cuda_graph else
                  ("eager launches" + (f" (capture failed: {graph_note})" if graph_note else "")),
        "ms_per_step_eager": float(np.mean(times_eager)),
        "host_submit_ms_total": round(host_ms, 3),
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": UNIT, "seconds_per_signature": e2e_s,
                "ms_signatures": [round(1e3 * x, 3) for x in e2e_times],
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "netlsd_heat_wave_slq(Graph on pinned host arrays) incl. H2D, device prepare, D2H",
                "seconds_per_signature_with_graph_hash": float(np.min(hash_times))},
    }
    if not args.no_cpu_baseline and world == 1:
        v, dt, probes = cpu_baseline(g, n_v, s, grid.values, os.cpu_count() or 1, max_probes=args.ref_probes)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
                                "sample": f"first {probes} of {n_v} probes of the same C2 workload, {dt:.1f} s "
                                          "(oracle/slq_oracle.py: numpy+scipy port of the reference)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64")
    ap.add_argument("--ref-probes", type=int, default=None,
                    help="probes timed in the CPU arms (default: all n_v)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes/launch of the dominant kernel")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: --warmup < 3 violates the timing rules; using 3")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
