"""How concentrated are the SpMM gathers of an R-MAT graph on its highest-degree rows?

Column references of vertex v = deg(v) (symmetric CSR), so the share of gathered rows that hit the
top-K vertices by degree is the top-K degree mass.  Prints, for K rows = the row count that fits a
given number of MB at 128 bytes per row (32 fp32 probes), the fraction of all gathers.

    python tools/hub_share.py [--scale 27]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2003_01282_b200.device import DeviceGraph

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
args = ap.parse_args()
dg = DeviceGraph.rmat(args.scale, 16, 0.57, 0.19, 0.19, seed=0, device="cuda:0", fold=None)
d, _ = dg.degrees()
d = torch.sort(d, descending=True).values
cum = torch.cumsum(d, 0)
tot = float(cum[-1])
out = {"scale": args.scale, "n": dg.n, "nnz": dg.nnz, "nonisolated": int((d > 0).sum()), "max_degree": float(d[0])}
for mb in (8, 16, 32, 48, 64, 80, 96, 128, 256, 512, 1024):
    k = min(dg.n, int(mb * 1e6 / 128))
    out[f"top_{mb}MB_rows{k}"] = float(cum[k - 1]) / tot
print(json.dumps(out))
