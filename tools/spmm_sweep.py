"""Per-kernel-class device time of one signature on C2 (SBM-100k, fp64, 100 probes) and a
device R-MAT (f32, 16 probes), for comparing builds (SLQ_LIB_PATH selects the library).

    SLQ_LIB_PATH=variants/a/libslq_b200.so python tools/spmm_sweep.py [--scale 25]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2003_01282_b200 import _lib, synth
from paper_2003_01282_b200.device import DeviceGraph

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=25)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--skip-c2", action="store_true")
ap.add_argument("--nv", type=int, default=16, help="probes of the R-MAT case (32: the folded C5 chunk width)")
ap.add_argument("--rmat-dtype", default="f32")
args = ap.parse_args()
dev = torch.device("cuda", 0)
out = {"lib": _lib.LIB_PATH, "env": {k: v for k, v in os.environ.items() if k.startswith("SLQ_")}}
cases = [("c2", lambda: DeviceGraph(synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0), dev), 100, "f64"),
         (f"drmat{args.scale}", lambda: DeviceGraph.rmat(args.scale, 16, seed=0, device=dev), args.nv, args.rmat_dtype)]
for name, make, nv, dt in cases[1:] if args.skip_c2 else cases:
    dg = make()
    for _ in range(2):
        dg.rules("normalized_laplacian", 0, 0, nv, 15, dtype=dt).check()
    best = None
    for _ in range(args.reps):
        _lib.profile_begin()
        dg.rules("normalized_laplacian", 0, 0, nv, 15, dtype=dt)
        torch.cuda.synchronize()
        prof = {k: round(v["ms"], 3) for k, v in _lib.profile_end().items() if v["launches"]}
        if best is None or prof["spmm"] < best["spmm"]:
            best = prof
    out[name] = best
    del dg
print(json.dumps(out))
