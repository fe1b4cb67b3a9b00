"""BASELINE C5 on one GPU: R-MAT scale 27 (edge factor 16, a=.57 b=.19 c=.19), generated and
converted to CSR on the device; 128 Rademacher probes x 15 Lanczos steps in fp32 vector storage;
heat + wave traces (normalized Laplacian) and VNGE (density).  The oracle cannot run at this size,
so correctness is checked through size-independent properties:

  * alpha_0 of each probe equals z^T Op z / n computed through the exact operator-apply path;
  * fp32 and fp64 vector storage agree on a probe prefix (heat within 1e-4, the north_star fp32 bar);
  * per-probe quadrature weights sum to 1 and nodes lie in the spectrum interval;
  * a probe prefix of the full run is bitwise the rules of the prefix run (chunk independence).

    python tools/run_c5.py [--scale 27] [--probes 128] [--reps 1] [--check]
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/run_c5.py   # probes sharded over GPUs

Under torchrun every rank builds the same graph on its GPU, runs its contiguous probe range and
the rules are all-gathered (dist.sharded_rules); times are the max over ranks.  C5_DIST_BACKEND=gloo
lets several ranks share one GPU for testing at small scales.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2003_01282_b200 import _lib
from paper_2003_01282_b200.descriptors import TimeGrid
from paper_2003_01282_b200.device import DeviceGraph, device_probes
from paper_2003_01282_b200.dist import sharded_rules
from paper_2003_01282_b200.slq import SlqConfig


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=27)
    ap.add_argument("--probes", type=int, default=128)
    ap.add_argument("--steps", type=int, default=15)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--profile", action="store_true", help="per-kernel-class device time of one more NL run")
    ap.add_argument("--no-fold", action="store_true", help="keep the isolated vertices in the Lanczos vectors")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group(os.environ.get("C5_DIST_BACKEND", "nccl"))
    cfg_all = SlqConfig(n_v=args.probes, s=args.steps, seed=0)

    def max_over_ranks(ms):
        if world == 1:
            return ms
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t0 = time.perf_counter()
    dg, gen_ms = timed(lambda: DeviceGraph.rmat(args.scale, 16, 0.57, 0.19, 0.19, seed=0, device=dev, fold=None))
    folded, fold_ms = (0, 0.0) if args.no_fold else timed(lambda: dg.fold_isolated())
    out = {"config": "c5", "scale": args.scale, "n": dg.n, "nnz": dg.nnz, "gen_wall_s": time.perf_counter() - t0,
           "gen_ms": gen_ms, "folded_isolated": folded, "fold_ms": fold_ms, "probes": args.probes,
           "steps": args.steps, "dtype": args.dtype, "n_gpus": world}
    tgrid = torch.tensor(np.array(TimeGrid(1e-2, 1e2, 250).values), device=dev)
    units = dg.nnz * args.probes * args.steps
    total_ms = 0.0
    keep = {}
    for kind, fns in (("normalized_laplacian", [_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM]),
                      ("density", [_lib.FN_XLOGX])):
        times = []
        for _ in range(args.reps):
            def run():
                if world > 1:
                    r = sharded_rules(dg, kind, cfg_all, dtype=args.dtype)
                else:
                    r = dg.rules(kind, 0, 0, args.probes, args.steps, dtype=args.dtype)
                v, s = r.integrate(tgrid if kind == "normalized_laplacian" else None, fns)
                return r, v, s
            if world > 1:
                import torch.distributed as dist

                dist.barrier()
            (rules, vals, stds), ms = timed(run)
            rules.check()
            times.append(max_over_ranks(ms))
        keep[kind] = (rules, vals)
        ms = float(min(times))
        total_ms += ms
        out[kind] = {"ms": ms, "units_per_s": units / (ms * 1e-3), "times": times,
                     "value0": float(vals[0, 0]), "value_last": float(vals[0, -1])}
    out["signature_s"] = total_ms * 1e-3
    out["units_per_s_all"] = 2 * units / (total_ms * 1e-3)
    out["vnge"] = -float(keep["density"][1][0, 0])
    if world > 1:
        import torch.distributed as dist

        if rank == 0:
            print(json.dumps(out))
        dist.barrier()
        dist.destroy_process_group()
        return
    if args.profile:
        _lib.profile_begin()
        r = dg.rules("normalized_laplacian", 0, 0, args.probes, args.steps, dtype=args.dtype)
        r.integrate(tgrid, [_lib.FN_HEAT, _lib.FN_WAVE_RE, _lib.FN_WAVE_IM])
        torch.cuda.synchronize()
        out["profile_nl"] = {k: v for k, v in _lib.profile_end().items() if v["launches"]}
        del r
    if args.check:
        chk = {}
        rules, vals = keep["normalized_laplacian"]
        w = rules.weights.cpu().numpy()
        nodes = rules.nodes.cpu().numpy()
        st = rules.steps.cpu().numpy()
        sums = np.array([w[p, :st[p]].sum() for p in range(len(st))])
        chk["weight_sum_max_dev"] = float(np.max(np.abs(sums - 1.0)))
        chk["nodes_in_interval"] = bool(np.all((nodes >= 0) & (nodes <= 2.0)))
        # prefix (chunk) independence
        k = 8
        pre = dg.rules("normalized_laplacian", 0, 0, k, args.steps, dtype=args.dtype)
        chk["prefix_bitwise"] = bool(torch.equal(pre.nodes, rules.nodes[:k]) and torch.equal(pre.weights, rules.weights[:k]))
        # alpha_0 = z^T L z / n through the exact operator apply (fp64)
        a, _, _ = dg.tridiagonals("normalized_laplacian", 0, 0, 4, 2, dtype=args.dtype)
        z = device_probes(dg.n, 0, 0, 4, dev)
        y = dg.apply("normalized_laplacian", z)
        a0 = (z * y).sum(0) / dg.n
        chk["alpha0_rel_err"] = float(torch.max(torch.abs(a[:, 0] - a0) / torch.abs(a0)))
        del y, z
        # fp32 vs fp64 on a 4-probe prefix
        r64 = dg.rules("normalized_laplacian", 0, 0, 4, args.steps, dtype="f64")
        r32 = dg.rules("normalized_laplacian", 0, 0, 4, args.steps, dtype="f32")
        v64, _ = r64.integrate(tgrid, [_lib.FN_HEAT])
        v32, _ = r32.integrate(tgrid, [_lib.FN_HEAT])
        chk["heat_f32_vs_f64_rel_l2"] = float(torch.linalg.norm(v32 - v64) / torch.linalg.norm(v64))
        if folded:
            # the fold against the unfolded recurrence on the same 4-probe prefix (fp32 storage)
            dg.fold_isolated(-1.0)
            r_un = dg.rules("normalized_laplacian", 0, 0, 4, args.steps, dtype="f32")
            v_un, _ = r_un.integrate(tgrid, [_lib.FN_HEAT])
            chk["heat_fold_vs_unfolded_rel_l2"] = float(torch.linalg.norm(v32 - v_un) / torch.linalg.norm(v_un))
        out["checks"] = chk
    print(json.dumps(out))


if __name__ == "__main__":
    main()
