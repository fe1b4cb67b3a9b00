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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--check-probes", type=int, default=8)
    ap.add_argument("--dtype", default="f64")
    args = ap.parse_args()
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
