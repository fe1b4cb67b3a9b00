"""Operator-pair chunk (slq_rules_pair_seeded) against two separate slq_rules_seeded calls: bitwise.
    SLQ_SPMM_FLAT=1 SLQ_PRESCALE_MIN_N=0 python tools/pair_check.py [--scale 16] [--time]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2003_01282_b200 import _lib
from paper_2003_01282_b200.device import DeviceGraph

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=16)
ap.add_argument("--time", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda", 0)
dg = DeviceGraph.rmat(args.scale, 16, seed=0, device=dev)
out = {"scale": args.scale, "cases": []}
for count, p0 in ((16, 0), (16, 48), (12, 3), (10, 0)):
    a, b, paired = dg.rules_pair(0, p0, count, 15)
    a.check()
    ra = dg.rules("normalized_laplacian", 0, p0, count, 15, dtype="f32")
    rb = dg.rules("density", 0, p0, count, 15, dtype="f32")
    ra.check(); rb.check()
    eq = all(torch.equal(x, y) for x, y in ((a.nodes, ra.nodes), (a.weights, ra.weights), (a.steps, ra.steps),
                                            (b.nodes, rb.nodes), (b.weights, rb.weights), (b.steps, rb.steps)))
    out["cases"].append({"count": count, "probe_begin": p0, "paired": paired, "bitwise_equal": eq,
                         "max_abs_nl": float((a.nodes - ra.nodes).abs().max()),
                         "max_abs_p": float((b.nodes - rb.nodes).abs().max())})
if args.time:
    def timed(fn, reps=3):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best
    out["pair16_s"] = timed(lambda: dg.rules_pair(0, 0, 16, 15))
    out["separate16_s"] = timed(lambda: (dg.rules("normalized_laplacian", 0, 0, 16, 15, dtype="f32"),
                                         dg.rules("density", 0, 0, 16, 15, dtype="f32")))
    out["one_op_32_s"] = timed(lambda: dg.rules("normalized_laplacian", 0, 0, 32, 15, dtype="f32"))
print(json.dumps(out))
sys.exit(0 if all(c["bitwise_equal"] and c["paired"] for c in out["cases"]) else 1)
