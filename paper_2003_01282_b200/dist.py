"""Multi-GPU probe sharding: the CSR is replicated on every rank,
probes are split into balanced contiguous ranges, each rank builds the Gauss
rules of its own probes, and ONE all-gather of (nodes, weights, steps)
assembles every rule on every rank in ascending probe order.  Per-probe
arithmetic does not depend on the range a rank owns, so the result is
bitwise identical for any world size as long as each rank's chunks fall in
the same step-kernel slot class (<= 32 or > 32 vector columns) as the
single-rank run's, and equal to rounding otherwise (tests/test_gpu_dist.py).
The collective is a few tens of KB (latency-bound): NCCL over NVLink on
GPUs, gloo in the CPU tests.
"""
from __future__ import annotations

__all__ = ["probe_ranges", "gather_rules_arrays", "sharded_rules"]


def probe_ranges(n_v: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous [begin, end) ranges; the first n_v % world ranks take one extra."""
    base, extra = divmod(n_v, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < extra else 0)
        out.append((b, e))
        b = e
    return out


def gather_rules_arrays(nodes, weights, steps, n_v: int, group=None, status=None):
    """All-gather per-rank rule blocks (torch tensors of [count_r, s], [count_r, s], [count_r])
    into [n_v, s] / [n_v] blocks in probe order.  Works with any torch.distributed backend.

    ``status`` (a rank's device int32[1] error word) travels in the same collective: the returned
    4th element is the OR over all ranks, so every rank raises the same error AFTER the collective
    (no rank can leave the others waiting in it)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    ranges = probe_ranges(n_v, world)
    width = int(nodes.shape[1])
    cap = max(e - b for b, e in ranges)
    dev = nodes.device
    # pack [cap + 1, 2*width+1] float64 per rank (steps and the status word as float64 are exact)
    pack = torch.zeros((cap + 1, 2 * width + 1), dtype=torch.float64, device=dev)
    cnt = int(nodes.shape[0])
    pack[:cnt, :width] = nodes
    pack[:cnt, width:2 * width] = weights
    pack[:cnt, 2 * width] = steps.to(torch.float64)
    if status is not None:
        pack[cap, 0] = status.reshape(-1)[0].to(torch.float64)
    on_host = dist.get_backend(group) == "gloo" and pack.is_cuda   # gloo gathers host tensors
    if on_host:
        pack = pack.cpu()
    bufs = [torch.empty_like(pack) for _ in range(world)]
    dist.all_gather(bufs, pack, group=group)
    if on_host:
        bufs = [b.to(dev) for b in bufs]
    full = torch.cat([bufs[r][: e - b] for r, (b, e) in enumerate(ranges)], dim=0)
    words = torch.stack([b[cap, 0] for b in bufs]).to(torch.int32)
    combined = words[0:1].clone()
    for r in range(1, world):
        combined = torch.bitwise_or(combined, words[r:r + 1])
    return (full[:, :width].contiguous(), full[:, width:2 * width].contiguous(),
            full[:, 2 * width].to(torch.int32).contiguous(), combined)


def sharded_rules(dg, kind: str, cfg, *, dtype: str = "f64", reorth: int = -1, group=None):
    """Rules of probes 0..cfg.n_v-1 with the probes sharded over the ranks of ``group``; every rank
    gets all rules.  Device errors of any rank surface on EVERY rank (``DeviceRules.check``)."""
    import torch
    import torch.distributed as dist

    from .device import DeviceRules

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return dg.rules(kind, cfg.seed, 0, cfg.n_v, cfg.s, reorth=reorth, dtype=dtype)
    rank = dist.get_rank(group)
    b, e = probe_ranges(cfg.n_v, dist.get_world_size(group))[rank]
    status = torch.zeros(1, dtype=torch.int32, device=dg.device)
    if e > b:
        local = dg.rules(kind, cfg.seed, b, e - b, cfg.s, reorth=reorth, dtype=dtype, status=status)
        nodes, weights, steps = local.nodes, local.weights, local.steps
    else:
        width = min(cfg.s, dg.n)
        nodes = torch.zeros((0, width), dtype=torch.float64, device=dg.device)
        weights = torch.zeros_like(nodes)
        steps = torch.zeros(0, dtype=torch.int32, device=dg.device)
    nodes, weights, steps, combined = gather_rules_arrays(nodes, weights, steps, cfg.n_v, group, status=status)
    return DeviceRules(nodes, weights, steps, dg.n, status=combined)
