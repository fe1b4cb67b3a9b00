"""Device time of ONE rank's share of the C5 signature at a given world size, on one GPU: what a rank
of an N-GPU probe-sharded job computes (its probes of both operators; the all-gather of a few tens of
KB is not included).  With 9..16 probes per rank the operator-pair block (slq_rules_pair_seeded) is
compared with the two separate runs.  The pool has one GPU per call, so this is the evidence for the
1 -> 8 GPU scaling of the probe sharding.

    python tools/rank_share.py --scale 27 --worlds 1,2,4,8 > profiles/r2_rank_share_c5.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2003_01282_b200 import _lib
from paper_2003_01282_b200.device import DeviceGraph
from paper_2003_01282_b200.dist import pair_applies, probe_ranges

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--n-v", type=int, default=128)
ap.add_argument("--steps", type=int, default=15)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
dev = torch.device("cuda", 0)
dg = DeviceGraph.rmat(args.scale, 16, seed=0, device=dev)
tgrid = torch.tensor(np.geomspace(1e-2, 1e2, 250), device=dev)
NL_FNS, P_FNS = [_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM], [_lib.FN_XLOGX]


def share(b, e, pair):
    if pair:
        nl, dens, used = dg.rules_pair(0, b, e - b, args.steps)
        assert used
    else:
        nl = dg.rules("normalized_laplacian", 0, b, e - b, args.steps, dtype="f32")
        dens = dg.rules("density", 0, b, e - b, args.steps, dtype="f32")
    return nl.integrate(tgrid, NL_FNS), dens.integrate(None, P_FNS), nl, dens


def timed(fn):
    best = None
    for _ in range(args.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best, out


res = {"workload": f"R-MAT-{args.scale} ef 16, {args.n_v} probes x {args.steps} steps, fp32, heat+wave+VNGE; rank 0's share",
       "n": dg.n, "nnz": dg.nnz, "worlds": {}}
base = None
for w in [int(x) for x in args.worlds.split(",")]:
    b, e = probe_ranges(args.n_v, w)[0]
    entry = {"probes_per_rank": e - b}
    ms_sep, out_sep = timed(lambda: share(b, e, False))
    entry["separate_ms"] = round(ms_sep, 1)
    best = ms_sep
    if pair_applies(args.n_v, w, "f32"):
        ms_pair, out_pair = timed(lambda: share(b, e, True))
        entry["pair_ms"] = round(ms_pair, 1)
        entry["pair_bitwise_equal_separate"] = bool(
            torch.equal(out_pair[2].nodes, out_sep[2].nodes) and torch.equal(out_pair[2].weights, out_sep[2].weights) and
            torch.equal(out_pair[3].nodes, out_sep[3].nodes) and torch.equal(out_pair[3].weights, out_sep[3].weights))
        best = min(best, ms_pair)
    if base is None:
        base = best
    entry["speedup_vs_first_world"] = round(base / best, 2)
    entry["speedup_separate_only"] = round(base / ms_sep, 2)
    res["worlds"][str(w)] = entry
print(json.dumps(res, indent=1))
