"""Multi-GPU token (M) sharding of the fused chain.

M is never a reduction dimension of either GEMM (workload.py:6-7), so the
chain shards with no data-path collective: rank r of R takes rows
[r*M/R, (r+1)*M/R) of A and produces the same rows of E; the weights are
replicated.  Each shard gets its own plan (the search depends on M; plans are
cached by M in plan_cache).  The only collective is optional: an all-gather of
E for callers that want the full output on every rank (NCCL over NVLink).
"""

from __future__ import annotations

from dataclasses import replace
from typing import Optional

from .workload import GATED_FFN, ChainGraph, DimensionSpec, build_gated_ffn, build_standard_ffn

ROW_GRANULE = 16  # MIN_EXTENT of the chain description (workload.py:24)


def shard_bounds(m: int, world: int, rank: int, granule: int = ROW_GRANULE) -> tuple:
    """[lo, hi) rows of rank `rank`: contiguous, granule-aligned, sizes differ by
    at most one granule, every row covered exactly once."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    units = -(-m // granule)
    lo_u = units * rank // world
    hi_u = units * (rank + 1) // world
    return min(m, lo_u * granule), min(m, hi_u * granule)


def shard_graph(graph: ChainGraph, world: int, rank: int) -> Optional[ChainGraph]:
    """The chain a rank executes (None when the rank gets no rows)."""
    lo, hi = shard_bounds(graph.dims.m, world, rank)
    rows = hi - lo
    if rows <= 0:
        return None
    padded = max(rows, ROW_GRANULE)
    dims = replace(graph.dims, m=padded)
    if graph.kind == GATED_FFN:
        return build_gated_ffn(dims)
    return build_standard_ffn(dims, graph.activation, logical_m=rows if padded != rows else None)


def run_sharded(graph: ChainGraph, tensors: dict, group=None, gather: bool = False, exchange: str = "auto"):
    """Run this rank's M-shard of the chain on the current GPU.

    ``tensors`` holds the FULL A (or just this rank's rows when
    ``A.shape[0]`` equals the shard size) and the replicated weights.  Returns
    this rank's E rows, or the full E when ``gather`` (all-gather over the
    process group)."""
    import torch
    import torch.distributed as dist

    from . import runtime

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(graph.dims.m, world, rank)
    a = tensors["A"]
    local = a if a.shape[0] == hi - lo else a[lo:hi]
    sub = shard_graph(graph, world, rank)
    if sub is None:
        out = torch.empty((0, graph.dims.l), dtype=a.dtype, device=a.device)
    else:
        shard = dict(tensors)
        if sub.dims.m != local.shape[0]:  # pad tiny shards up to one row granule
            pad = torch.zeros((sub.dims.m - local.shape[0], local.shape[1]), dtype=local.dtype, device=local.device)
            local = torch.cat([local, pad])
        shard["A"] = local.contiguous()
        out = runtime.run(sub, None, shard, exchange=exchange)[: hi - lo]
    if not gather or world == 1:
        return out
    sizes = [shard_bounds(graph.dims.m, world, r) for r in range(world)]
    # NCCL gathers device tensors over NVLink; gloo (CPU process groups, ranks sharing
    # a GPU in tests) gathers host copies
    on_host = dist.get_backend(group) == "gloo"
    dev = torch.device("cpu") if on_host else out.device
    # all_gather wants equal-sized parts (gloo enforces it): shards differ by at most one
    # row granule, so every rank sends its rows padded to the largest shard
    rows = max(h - l_ for l_, h in sizes)
    send = torch.zeros((rows, graph.dims.l), dtype=out.dtype, device=dev)
    send[: out.shape[0]] = out.to(dev)
    parts = [torch.empty_like(send) for _ in sizes]
    dist.all_gather(parts, send, group=group)
    return torch.cat([p[: h - l_] for p, (l_, h) in zip(parts, sizes)]).to(out.device)
