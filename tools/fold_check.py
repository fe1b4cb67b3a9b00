"""Is the isolated-vertex fold degree-ordered?  Prints the first row lengths of the Lanczos graph of a
device R-MAT and the fraction of column references that hit its first K rows.
    python tools/fold_check.py [--scale 26]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2003_01282_b200.device import DeviceGraph

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
a = ap.parse_args()
dg = DeviceGraph.rmat(a.scale, 16, seed=0, device="cuda:0")
k = 1 << 20
lens, rows = dg.lanczos_row_lengths(k)
print(json.dumps({"scale": a.scale, "folded": dg.folded, "rows": rows, "first": lens[:8].tolist(),
                  "descending": bool(np.all(np.diff(lens) <= 0)),
                  "share_first_500k": float(lens[:500000].sum() / dg.nnz), "share_first_1M": float(lens.sum() / dg.nnz)}))
