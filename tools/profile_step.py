"""Run a few C2 signature steps (for ncu launch lists / full captures; no timing printed)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2003_01282_b200 import _lib, synth
from paper_2003_01282_b200.descriptors import TimeGrid
from paper_2003_01282_b200.device import DeviceGraph

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--dtype", default="f64")
ap.add_argument("--graph", default="sbm")
ap.add_argument("--nv", type=int, default=100)
ap.add_argument("--s", type=int, default=15)
args = ap.parse_args()
dev = torch.device("cuda", 0)
if args.graph == "sbm":
    g = synth.sbm(100_000, 10, 1e-3, 1e-5, seed=0)
    dg = DeviceGraph(g, dev)
elif args.graph.startswith("drmat"):   # generated on the device (C5: drmat27)
    dg = DeviceGraph.rmat(int(args.graph.replace("drmat", "")), 16, seed=0, device=dev)
    g = dg
else:
    g = synth.rmat(int(args.graph.replace("rmat", "")), 16, seed=0)
    dg = DeviceGraph(g, dev)
grid = torch.tensor(np.array(TimeGrid(1e-2, 1e2, 250).values), device=dev)
for _ in range(args.steps):
    rules = dg.rules("normalized_laplacian", 0, 0, args.nv, args.s, dtype=args.dtype)
    for fn in (_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM):
        rules.estimate(rules.quadrature(grid, fn))
torch.cuda.synchronize()
print("ok", g.n, g.nnz)
