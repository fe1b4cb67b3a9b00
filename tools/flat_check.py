"""A/B of the flat SpMM (spmm_flat.cu, SLQ_SPMM_FLAT=1) against the warp-per-row kernel
(SLQ_SPMM_FLAT=0) on a folded device R-MAT: tridiagonals must be bitwise equal.

    python tools/flat_check.py [--scale 16] [--time-scale 0]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r"""
import sys, json, hashlib, torch
sys.path.insert(0, %r)
from paper_2003_01282_b200 import _lib
from paper_2003_01282_b200.device import DeviceGraph
scale = int(sys.argv[1])
dg = DeviceGraph.rmat(scale, 16, seed=0, device=torch.device('cuda', 0))
out = {}
for kind in ('normalized_laplacian', 'density', 'laplacian'):
    for nv, dt in ((32, 'f32'), (24, 'f32'), (19, 'f32'), (16, 'f32'), (12, 'f32'), (8, 'f32'), (5, 'f32'),
                   (32, 'f64'), (19, 'f64'), (16, 'f64'), (11, 'f64'), (8, 'f64'), (3, 'f64')):
        a, b, s = dg.tridiagonals(kind, 0, 0, nv, 15, dtype=dt)
        h = hashlib.sha256(a.cpu().numpy().tobytes() + b.cpu().numpy().tobytes() + s.cpu().numpy().tobytes()).hexdigest()
        out[f'{kind}/{nv}/{dt}'] = [h[:16], float(a[0, 0]), float(a[-1, -1])]
print(json.dumps(out))
""" % ROOT

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=16)
args = ap.parse_args()
res = {}
for flat in ("0", "1"):
    env = dict(os.environ, SLQ_SPMM_FLAT=flat, SLQ_PRESCALE_MIN_N="0")
    r = subprocess.run([sys.executable, "-c", CHILD, str(args.scale)], env=env, capture_output=True, text=True, timeout=900)
    if r.returncode != 0:
        print(r.stdout[-2000:], r.stderr[-4000:])
        sys.exit(1)
    res[flat] = json.loads(r.stdout.strip().splitlines()[-1])
bad = [k for k in res["0"] if res["0"][k] != res["1"][k]]
print(json.dumps({"scale": args.scale, "cases": len(res["0"]), "mismatch": bad,
                  "detail": {k: [res["0"][k], res["1"][k]] for k in bad}}))
sys.exit(1 if bad else 0)
