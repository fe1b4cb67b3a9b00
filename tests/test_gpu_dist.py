"""Probe sharding on the device path: two ranks (gloo, both on cuda:0 — their kernels never wait on
each other; the only exchange is the host all-gather of the rules) assemble exactly the rules and
descriptors of a single-rank run when every rank's chunk width falls in the same step-kernel slot
class as the single run's (DESIGN §4 determinism), and agree to rounding otherwise."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_v, dtype, out):
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import golden
    from paper_2003_01282_b200 import _lib
    from paper_2003_01282_b200.descriptors import TimeGrid
    from paper_2003_01282_b200.device import DeviceGraph
    from paper_2003_01282_b200.dist import sharded_rules
    from paper_2003_01282_b200.slq import SlqConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dg = DeviceGraph(golden.graph(golden.load("sbm5k.npz")), torch.device("cuda", 0))
    cfg = SlqConfig(n_v=n_v, s=15, seed=0)
    rules = sharded_rules(dg, "normalized_laplacian", cfg, dtype=dtype)
    vals, _ = rules.integrate(np.array(TimeGrid(1e-2, 1e2, 64).values), [_lib.FN_HEAT])
    if rank == 0:
        out.put((rules.nodes.cpu().numpy(), rules.weights.cpu().numpy(), rules.steps.cpu().numpy(),
                 vals.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _sharded(n_v, dtype):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_v, dtype, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _single(n_v, dtype):
    import golden
    from paper_2003_01282_b200 import _lib
    from paper_2003_01282_b200.descriptors import TimeGrid
    from paper_2003_01282_b200.device import DeviceGraph

    dg = DeviceGraph(golden.graph(golden.load("sbm5k.npz")), torch.device("cuda", 0))
    r = dg.rules("normalized_laplacian", 0, 0, n_v, 15, dtype=dtype)
    vals, _ = r.integrate(np.array(TimeGrid(1e-2, 1e2, 64).values), [_lib.FN_HEAT])
    return r.nodes.cpu().numpy(), r.weights.cpu().numpy(), r.steps.cpu().numpy(), vals.cpu().numpy()


@pytest.mark.parametrize("n_v,dtype", [(100, "f64"), (32, "f64"), (32, "f32")])
def test_two_ranks_bitwise_equal_single_rank(cuda_device, n_v, dtype):
    # 100 -> 50 + 50 (wide class both ways); 32 -> 16 + 16 (narrow class both ways)
    got, ref = _sharded(n_v, dtype), _single(n_v, dtype)
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)


def test_two_ranks_across_slot_classes_agree_to_rounding(cuda_device):
    # 40 probes on one rank (wide) vs 20 + 20 (narrow): same rules to rounding
    got, ref = _sharded(40, "f64"), _single(40, "f64")
    assert np.array_equal(got[2], ref[2])
    assert np.max(np.abs(got[0] - ref[0])) <= 1e-13
    assert np.max(np.abs(got[3] - ref[3]) / np.abs(ref[3])) <= 1e-13


def _worker_rmat(rank, world, port, out, env):
    import torch.distributed as dist

    os.environ.update(env)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2003_01282_b200 import _lib
    from paper_2003_01282_b200.descriptors import TimeGrid
    from paper_2003_01282_b200.device import DeviceGraph
    from paper_2003_01282_b200.dist import sharded_rules
    from paper_2003_01282_b200.slq import SlqConfig

    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    dg = DeviceGraph.rmat(14, 16, seed=5, device=torch.device("cuda", 0))
    cfg = SlqConfig(n_v=32, s=15, seed=0)
    if world > 1:
        rules = sharded_rules(dg, "normalized_laplacian", cfg, dtype="f32")
    else:
        rules = dg.rules("normalized_laplacian", 0, 0, 32, 15, dtype="f32")
    vals, _ = rules.integrate(np.array(TimeGrid(1e-2, 1e2, 64).values), [_lib.FN_HEAT])
    if rank == 0:
        out.put((dg.folded, rules.nodes.cpu().numpy(), rules.weights.cpu().numpy(), vals.cpu().numpy()))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _run_rmat(world, env):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_rmat, args=(r, world, port, q, env)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_two_ranks_folded_prescaled_bitwise_equal_single_rank(cuda_device):
    # the C5 configuration in miniature: a device-built R-MAT graph with its isolated vertices folded,
    # fp32, prescaled gathers forced on (SLQ_PRESCALE_MIN_N=0); one rank runs a 32-probe chunk (HALF2
    # SpMM), two ranks run 16 each (HALF SpMM) — same narrow class, so the rules are bitwise equal
    env = {"SLQ_PRESCALE_MIN_N": "0"}
    one, two = _run_rmat(1, env), _run_rmat(2, env)
    assert one[0] > 0 and one[0] == two[0]
    for a, b in zip(one[1:], two[1:]):
        assert np.array_equal(a, b)


def _batch_worker(rank, world, port, out):
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2003_01282_b200 import _lib, synth
    from paper_2003_01282_b200.dist import ShardedBatch
    from paper_2003_01282_b200.slq import SlqConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    graphs = synth.er_batch(61, seed=3)
    sb = ShardedBatch(graphs, device=torch.device("cuda", 0))
    t = np.geomspace(1e-2, 1e2, 32)
    vals, stds, status = sb.values("normalized_laplacian", SlqConfig(n_v=12, s=8, seed=0), t, _lib.FN_HEAT, "f32")
    out.put((rank, vals.cpu().numpy(), stds.cpu().numpy(), int(status.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_graph_range_sharding_bitwise_equals_single_gpu(cuda_device):
    """C3 over two ranks (dist.ShardedBatch: contiguous graph ranges, one all-gather of per-graph rows):
    every rank's assembled per-graph heat traces equal the single-GPU batched path bit for bit."""
    from paper_2003_01282_b200 import _lib, synth
    from paper_2003_01282_b200.batched import BatchedGraphs
    from paper_2003_01282_b200.slq import SlqConfig

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    batch = BatchedGraphs(synth.er_batch(61, seed=3), device=cuda_device)
    rules = batch.rules("normalized_laplacian", SlqConfig(n_v=12, s=8, seed=0), "f32")
    vals, stds = batch.integrate(rules, np.geomspace(1e-2, 1e2, 32), _lib.FN_HEAT)
    for _, v, s, st in res:
        assert st == 0
        assert np.array_equal(v, vals.cpu().numpy()) and np.array_equal(s, stds.cpu().numpy())


def _worker_pair(rank, world, port, out, env):
    import torch.distributed as dist

    os.environ.update(env)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2003_01282_b200.device import DeviceGraph
    from paper_2003_01282_b200.dist import pair_applies, sharded_rules_pair
    from paper_2003_01282_b200.slq import SlqConfig

    dg = DeviceGraph.rmat(14, 16, seed=5, device=torch.device("cuda", 0))
    cfg = SlqConfig(n_v=24, s=12, seed=0)
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        assert pair_applies(cfg.n_v, world, "f32")
        nl, dens = sharded_rules_pair(dg, cfg, dtype="f32")
    else:
        nl = dg.rules("normalized_laplacian", 0, 0, cfg.n_v, cfg.s, dtype="f32")
        dens = dg.rules("density", 0, 0, cfg.n_v, cfg.s, dtype="f32")
    nl.check()
    dens.check()
    if rank == 0:
        out.put((dg.folded, nl.nodes.cpu().numpy(), nl.weights.cpu().numpy(), nl.steps.cpu().numpy(),
                 dens.nodes.cpu().numpy(), dens.weights.cpu().numpy(), dens.steps.cpu().numpy()))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def test_two_ranks_operator_pair_bitwise_equal_single_rank(cuda_device):
    """C5 on 8 GPUs in miniature: 24 probes over two ranks = 12 per rank, so each rank runs ONE
    operator-pair block (normalized Laplacian + density interleaved, dist.sharded_rules_pair); the
    assembled rules of both operators are bitwise the single-rank separate runs' (24-probe chunks)."""
    env = {"SLQ_PRESCALE_MIN_N": "0", "SLQ_SPMM_FLAT": "1"}
    ctx = mp.get_context("spawn")
    res = []
    for world in (1, 2):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker_pair, args=(r, world, port, q, env)) for r in range(world)]
        for p in procs:
            p.start()
        res.append(q.get(timeout=300))
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
    one, two = res
    assert one[0] > 0 and one[0] == two[0]
    for a, b in zip(one[1:], two[1:]):
        assert np.array_equal(a, b)


def test_bench_eight_ranks_use_the_operator_pair_block(cuda_device, tmp_path):
    """`bench.py --gpus 8` as the driver launches it (torchrun, one process per rank; here gloo ranks
    on one GPU and a scale-14 stand-in graph): 128 probes over 8 ranks = 16 per rank, so every rank
    runs the operator-pair block; the line is the contract's and the end-to-end values equal the
    device-resident run's."""
    import json
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", BENCH_TEST_RMAT_SCALE="14", BENCH_NO_CLOCKS="1",
               SLQ_SPMM_FLAT="1", SLQ_PRESCALE_MIN_N="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "8", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "8", "--steps", "1", "--warmup", "3",
           "--no-cpu-baseline", "--e2e-reps", "1"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 8 and line["scaling"] == "strong"
    assert line["graph"]["probes_per_rank"] == 16 and line["graph"]["operator_pair_block"] is True
    assert line["config"]["workload"].startswith("TEST RUN")
    assert line["e2e"]["values_equal_device_resident_run"] is True
    assert line["gpu_launches"] > 0 and line["value"] > 0
