"""Run one BASELINE config on the GPU: device time per signature + parity against the oracle on a
probe prefix (per-probe rules are independent of the probe count, so a prefix is an exact check).

    python tools/run_config.py c4 [--reps 3] [--check-probes 8] [--dtype f64]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2003_01282_b200 import _lib, synth
from paper_2003_01282_b200.descriptors import TimeGrid
from paper_2003_01282_b200.device import DeviceGraph

CONFIGS = {
    "c1": dict(make=lambda: synth.barabasi_albert(1000, 3, seed=0), n_v=10, s=10, kinds=("nl", "p")),
    "c2": dict(make=lambda: synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0), n_v=100, s=15, kinds=("nl",)),
    "c4": dict(make=lambda: synth.rmat(20, 16, seed=0), n_v=100, s=15, kinds=("nl", "p")),
}
KIND = {"nl": "normalized_laplacian", "p": "density"}


def run_c3(args):
    """10,000 ER graphs (n ~ U{20..200}, p ~ U[0.05,0.3]) stacked block-diagonally, n_v=20, s=10,
    per-graph heat on 250 t; fp32 per BASELINE (fp64 also reported)."""
    from paper_2003_01282_b200.batched import BatchedGraphs, netlsd_slq_batch
    from paper_2003_01282_b200.slq import SlqConfig

    t0 = time.perf_counter()
    graphs = synth.er_batch(args.graphs, seed=0)
    batch = BatchedGraphs(graphs)
    gen_s = time.perf_counter() - t0
    grid = TimeGrid(1e-2, 1e2, 250)
    cfg = SlqConfig(n_v=20, s=10, seed=0)
    out = {"config": "c3", "graphs": len(graphs), "n": batch.stacked.n, "nnz": batch.stacked.nnz, "gen_s": gen_s}
    for dtype in ("f32", "f64"):
        times = []
        for _ in range(args.reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rules = batch.rules("normalized_laplacian", cfg, dtype)
            vals, stds = batch.integrate(rules, grid.values, _lib.FN_HEAT)
            e1.record()
            torch.cuda.synchronize()
            _lib.check_status(int(rules[3].item()))
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times[1:]))
        units = batch.stacked.nnz * cfg.n_v * cfg.s
        out[dtype] = {"ms": ms, "units_per_s": units / (ms * 1e-3), "graphs_per_s": len(graphs) / (ms * 1e-3),
                      "times": times}
    if args.check_probes:
        from oracle import slq_oracle as O

        k = min(50, len(graphs))
        t1 = time.perf_counter()
        ref = [O.heat_trace(graphs[j], grid.values, 20, 10, 0)[0] for j in range(k)]
        cpu_s = time.perf_counter() - t1
        for dtype in ("f64", "f32"):
            vals, _ = netlsd_slq_batch(batch, grid, cfg, dtype=dtype)
            errs = [float(np.linalg.norm(vals[j] - ref[j]) / np.linalg.norm(ref[j])) for j in range(k)]
            out[dtype]["parity_max_rel_l2_first50"] = max(errs)
        out["cpu_oracle_s_per_graph"] = cpu_s / k
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--check-probes", type=int, default=8)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--graphs", type=int, default=10_000)
    ap.add_argument("--graph", action="store_true", help="also time a CUDA-graph replay of the signature")
    args = ap.parse_args()
    if args.config == "c3":
        return run_c3(args)
    cfg = CONFIGS[args.config]
    t0 = time.perf_counter()
    g = cfg["make"]()
    gen_s = time.perf_counter() - t0
    dev = torch.device("cuda", 0)
    tgrid = torch.tensor(np.array(TimeGrid(1e-2, 1e2, 250).values), device=dev)
    dg = DeviceGraph(g, dev)
    out = {"config": args.config, "n": g.n, "nnz": g.nnz, "gen_s": gen_s, "dtype": args.dtype}
    for kind in cfg["kinds"]:
        fns = [_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM] if kind == "nl" else [_lib.FN_XLOGX]
        times = []
        for _ in range(args.reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rules = dg.rules(KIND[kind], 0, 0, cfg["n_v"], cfg["s"], dtype=args.dtype)
            vals, stds = rules.integrate(tgrid if kind == "nl" else None, fns)
            e1.record()
            torch.cuda.synchronize()
            rules.check()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times[1:]))
        units = g.nnz * cfg["n_v"] * cfg["s"]
        out[kind] = {"ms": ms, "units_per_s": units / (ms * 1e-3), "times": times}
        if args.graph:
            # the same signature captured once as a CUDA graph and replayed (device.CapturedSignature)
            from paper_2003_01282_b200.device import CapturedSignature

            cap = CapturedSignature(dg, KIND[kind], 0, cfg["n_v"], cfg["s"],
                                    tgrid.cpu().numpy() if kind == "nl" else None, fns, dtype=args.dtype)
            gt = []
            for _ in range(args.reps + 1):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                cap.replay()
                e1.record()
                torch.cuda.synchronize()
                gt.append(e0.elapsed_time(e1))
            cap.check()
            out[kind]["graph_replay_ms"] = float(np.median(gt[1:]))
        if args.check_probes:
            from oracle import slq_oracle as O

            okind = O.NORMALIZED_LAPLACIAN if kind == "nl" else O.DENSITY
            t1 = time.perf_counter()
            ref = O.slq_rules(O.make_block_operator(g, okind), args.check_probes, cfg["s"], 0,
                              threads=os.cpu_count())
            oracle_s = time.perf_counter() - t1
            got = dg.rules(KIND[kind], 0, 0, args.check_probes, cfg["s"], dtype=args.dtype)
            got.check()
            hi = 2.0 if kind == "nl" else 1.0
            steps_eq = bool(np.array_equal(got.steps.cpu().numpy(), ref.steps))
            dn = float(np.max(np.abs(got.nodes.cpu().numpy() - ref.nodes))) / hi
            tt = np.array(TimeGrid(1e-2, 1e2, 250).values)
            if kind == "nl":
                rh, _ = O.heat_from_rules(ref, g.n, tt)
                gv, _ = got.integrate(tt, [_lib.FN_HEAT])
                err = float(np.linalg.norm(gv.cpu().numpy()[0] - rh) / np.linalg.norm(rh))
            else:
                rv, _ = O.vnge_from_rules(ref, g.n)
                gv, _ = got.integrate(None, [_lib.FN_XLOGX])
                err = abs(-float(gv.cpu().numpy()[0, 0]) - rv) / abs(rv)
            out[kind]["parity"] = {"probes": args.check_probes, "steps_equal": steps_eq, "max_node_abs_over_hi": dn,
                                   "descriptor_rel_err": err, "oracle_s": oracle_s}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
