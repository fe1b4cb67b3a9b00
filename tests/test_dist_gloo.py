"""Multi-rank host logic of the probe sharding (world_size 2, gloo, CPU): balanced probe ranges,
the all-gather of per-rank rule blocks in probe order, and that the assembled rules — and so the
descriptors — equal the single-rank result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_01282_b200.dist import gather_rules_arrays, probe_ranges


def test_probe_ranges_balanced():
    assert probe_ranges(100, 8) == [(0, 13), (13, 26), (26, 39), (39, 52), (52, 64), (64, 76), (76, 88), (88, 100)]
    assert probe_ranges(3, 4) == [(0, 1), (1, 2), (2, 3), (3, 3)]
    for n_v in (1, 7, 128):
        for w in (1, 2, 3, 8):
            r = probe_ranges(n_v, w)
            assert r[0][0] == 0 and r[-1][1] == n_v
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [e - b for b, e in r]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rules_for(probes, width):
    # deterministic stand-in for per-probe rules: a pure function of the probe index
    rng = [np.random.default_rng(1000 + p) for p in probes]
    nodes = np.stack([np.sort(r.uniform(0, 2, width)) for r in rng]) if probes else np.zeros((0, width))
    weights = np.stack([r.dirichlet(np.ones(width)) for r in rng]) if probes else np.zeros((0, width))
    steps = np.array([width - (p % 3 == 0) for p in probes], dtype=np.int32)
    return nodes, weights, steps


def _worker(rank, world, port, n_v, width, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = probe_ranges(n_v, world)[rank]
    nodes, weights, steps = _rules_for(list(range(b, e)), width)
    # rank 1 reports a device error word (bit 1: eigensolver failure); it must reach EVERY rank through
    # the collective instead of one rank raising before it and leaving the other waiting
    status = torch.tensor([1 if rank == 1 else 0], dtype=torch.int32)
    gn, gw, gs, gst = gather_rules_arrays(torch.tensor(nodes), torch.tensor(weights), torch.tensor(steps), n_v,
                                          status=status)
    out.put((rank, gn.numpy(), gw.numpy(), gs.numpy(), int(gst.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_v,world", [(10, 2), (3, 2), (1, 2)])
def test_gather_rules_world2_matches_single(n_v, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_v, 6, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = _rules_for(list(range(n_v)), 6)
    for rank, *got, st in res:
        for a, b in zip(got, ref):
            assert np.array_equal(a, b)
        assert st == 1, f"rank {rank} did not see rank 1's device error"


def _rows_worker(rank, world, port, total, out):
    from paper_2003_01282_b200.dist import gather_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = probe_ranges(total, world)[rank]
    # a rank's per-graph signatures: a pure function of the graph index (C3 graph-range sharding)
    block = torch.tensor([[np.sin(g + 0.1 * t) for t in range(5)] for g in range(b, e)], dtype=torch.float64)
    block = block.reshape(e - b, 5)
    full = gather_rows(block, total)
    out.put((rank, full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total,world", [(10, 2), (3, 2), (1, 2)])
def test_graph_range_gather_world2(total, world):
    """C3 sharding over GPUs (dist.ShardedBatch): balanced contiguous graph ranges, one all-gather of the
    per-graph rows in graph order; every rank sees the single-rank array."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = np.array([[np.sin(g + 0.1 * t) for t in range(5)] for g in range(total)])
    for _, full in res:
        assert np.array_equal(full, ref)


class _FakeRules:
    def __init__(self, nodes, weights, steps):
        self.nodes, self.weights, self.steps = torch.tensor(nodes), torch.tensor(weights), torch.tensor(steps)


class _FakePairGraph:
    """Stands in for DeviceGraph.rules_pair on the CPU: rules are a pure function of (operator, probe)."""
    device = torch.device("cpu")
    n = 50

    def rules_pair(self, seed, probe_begin, count, steps, *, reorth=-1, dtype="f32", status=None):
        probes = list(range(probe_begin, probe_begin + count))
        nl = _FakeRules(*_rules_for(probes, steps))
        dens = _FakeRules(*_rules_for([1000 + p for p in probes], steps))
        return nl, dens, True


class _Cfg:
    n_v, s, seed = 24, 6, 0


def _pair_worker(rank, world, port, out):
    from paper_2003_01282_b200.dist import sharded_rules_pair

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nl, dens = sharded_rules_pair(_FakePairGraph(), _Cfg())
    out.put((rank, nl.nodes.numpy(), nl.weights.numpy(), nl.steps.numpy(), dens.nodes.numpy(),
             dens.weights.numpy(), dens.steps.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_pair_applies_only_for_9_to_16_fp32_probes_per_rank():
    from paper_2003_01282_b200.dist import pair_applies

    assert pair_applies(128, 8, "f32") and pair_applies(24, 2, "f32")
    assert not pair_applies(128, 4, "f32")      # 32 probes per rank: a full row per operator already
    assert not pair_applies(128, 16, "f32")     # 8 probes per rank
    assert not pair_applies(128, 8, "f64")
    assert pair_applies(100, 8, "f32")


def test_sharded_rules_pair_world2_matches_single():
    """Operator-pair sharding (dist.sharded_rules_pair): each rank's pair block covers its own probe
    range, one all-gather per operator puts both rule sets in probe order on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pair_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_nl = _rules_for(list(range(24)), 6)
    ref_p = _rules_for([1000 + p for p in range(24)], 6)
    for _, *got in res:
        for a, b in zip(got, list(ref_nl) + list(ref_p)):
            assert np.array_equal(a, b)
