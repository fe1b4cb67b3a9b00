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

__all__ = ["probe_ranges", "gather_rules_arrays", "sharded_rules", "sharded_rules_pair", "pair_applies", "gather_rows",
           "ShardedBatch"]


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


def pair_applies(n_v: int, world: int, dtype: str) -> bool:
    """Whether every rank's probe share fits the operator-pair block (9..16 fp32 probes): the same
    decision on every rank, from the probe count and the world size only."""
    sizes = [e - b for b, e in probe_ranges(n_v, world)]
    return dtype in ("f32", "float32") and min(sizes) >= 9 and max(sizes) <= 16


def sharded_rules_pair(dg, cfg, *, dtype: str = "f32", reorth: int = -1, group=None):
    """Normalized-Laplacian AND density rules of probes 0..cfg.n_v-1 (heat/wave + VNGE of one
    signature), probes sharded over the ranks.  Each rank calls ``dg.rules_pair`` on its range: with
    9..16 probes per rank (128 probes on 8 GPUs) both Lanczos runs share every gathered row, so a
    rank makes ONE pass over the graph per step instead of two -- pure probe sharding then scales
    to 8 GPUs (a single operator's 16 probes would fill only half of each gathered 128-byte row).
    One all-gather per operator; returns ``(rules_nl, rules_density)`` on every rank, bitwise the
    rules of ``sharded_rules`` per operator."""
    import torch
    import torch.distributed as dist

    from .device import DeviceRules

    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    b, e = probe_ranges(cfg.n_v, world)[rank]
    status = torch.zeros(1, dtype=torch.int32, device=dg.device)
    width = min(cfg.s, dg.n)
    if e > b:
        nl, dens, _ = dg.rules_pair(cfg.seed, b, e - b, cfg.s, reorth=reorth, dtype=dtype, status=status)
        blocks = [(nl.nodes, nl.weights, nl.steps), (dens.nodes, dens.weights, dens.steps)]
    else:
        z = torch.zeros((0, width), dtype=torch.float64, device=dg.device)
        blocks = [(z, z.clone(), torch.zeros(0, dtype=torch.int32, device=dg.device))] * 2
    if world == 1:
        return tuple(DeviceRules(n_, w_, s_, dg.n, status=status) for n_, w_, s_ in blocks)
    out = []
    for n_, w_, s_ in blocks:
        nodes, weights, steps, combined = gather_rules_arrays(n_, w_, s_, cfg.n_v, group, status=status)
        out.append(DeviceRules(nodes, weights, steps, dg.n, status=combined))
    return tuple(out)


def gather_rows(block, total: int, group=None):
    """All-gather per-rank row blocks [count_r, ...] of a balanced contiguous partition of `total`
    rows (``probe_ranges``) into the full [total, ...] block in row order, on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    ranges = probe_ranges(total, world)
    cap = max(e - b for b, e in ranges)
    pack = torch.zeros((cap,) + tuple(block.shape[1:]), dtype=block.dtype, device=block.device)
    pack[:block.shape[0]] = block
    on_host = dist.get_backend(group) == "gloo" and pack.is_cuda
    if on_host:
        pack = pack.cpu()
    bufs = [torch.empty_like(pack) for _ in range(world)]
    dist.all_gather(bufs, pack, group=group)
    full = torch.cat([bufs[r][: e - b] for r, (b, e) in enumerate(ranges)], dim=0)
    return full.to(block.device) if on_host else full


class ShardedBatch:
    """C3 over several GPUs: the collection of small graphs is split into balanced
    contiguous GRAPH ranges, rank r stacks and solves its own range on its GPU (no data-path
    collective: graphs are independent), and one all-gather assembles the per-graph signatures in
    graph order.  Each graph's values are those of the single-GPU batched path bit for bit (the
    batched kernel's arithmetic for a graph does not depend on the other graphs in the stack)."""

    def __init__(self, graphs, device=None, group=None):
        import torch.distributed as dist

        from .batched import BatchedGraphs

        self.group = group
        self.total = len(graphs)
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        rank = dist.get_rank(group) if world > 1 else 0
        self.world = world
        self.begin, self.end = probe_ranges(self.total, world)[rank]
        self.local = BatchedGraphs(graphs[self.begin:self.end], device=device) if self.end > self.begin else None

    def values(self, kind: str, cfg, t, fn: int, dtype: str = "f64"):
        """(values [G, T], std_errors [G, T], status [1] int32) on every rank, device tensors; the status
        word is the OR over all graphs of all ranks (``_lib.check_status`` maps it to the exceptions)."""
        import torch

        T = 1 if t is None else len(t)
        if self.local is not None:
            rules = self.local.rules(kind, cfg, dtype)
            vals, stds = self.local.integrate(rules, t, fn)
            status = rules[3].to(torch.float64).reshape(1, 1).expand(vals.shape[0], 1)
            block = torch.cat([vals, stds, status], dim=1)
        else:
            import torch.distributed as dist

            dev = torch.device("cuda", torch.cuda.current_device())
            block = torch.zeros((0, 2 * T + 1), dtype=torch.float64, device=dev)
        if self.world > 1:
            full = gather_rows(block, self.total, self.group)
        else:
            full = block
        words = full[:, 2 * T].to(torch.int64)
        status = torch.zeros(1, dtype=torch.int64, device=full.device)
        for b in range(4):   # OR of the 4 status bits (rules.cu kSt*) over every graph
            if words.numel():
                status = status + (((words >> b) & 1).amax() << b)
        return full[:, :T], full[:, T:2 * T], status.to(torch.int32)
