"""Data-parallel plumbing: batch sharding + the one collective (SURVEY §8.1 row e).

The workload shards by batch element of the jagged GridBatch (conv_batch is an
independent per-grid loop, conv.py:381-382) and the weight gradient is additive
over elements, so the only exchange is one sum all-reduce of
each SparseConv3d's fp32 ``weight.grad`` ([Cout,Cin,3,3,3]: 442 KB at 64², 1.77 MB
at 128²) — NCCL over NVLink on B200 boxes, gloo in the CPU tests.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def partition_by_cost(costs, world_size):
    """Contiguous runs of batch elements per rank, balanced by cost (e.g. kernel-map pairs).

    Returns ``world_size`` (start, end) half-open ranges covering ``range(len(costs))``;
    deterministic, so every rank computes the same assignment without communication.
    """
    n = len(costs)
    if world_size <= 0:
        raise ValueError("world_size must be positive")
    total = float(sum(costs))
    bounds = [0]
    acc = 0.0
    k = 1
    for i, c in enumerate(costs):
        acc += float(c)
        while k < world_size and acc >= total * k / world_size and (i + 1) > bounds[-1]:
            bounds.append(i + 1)
            k += 1
    while len(bounds) < world_size:
        bounds.append(n)
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world_size)]


def shard(items, rank, world_size, costs=None):
    """This rank's contiguous share of ``items``."""
    costs = costs if costs is not None else [1] * len(items)
    s, e = partition_by_cost(costs, world_size)[rank]
    return items[s:e]


def allreduce_gradients(params, group=None, async_op=False):
    """Sum-all-reduce the gradients of ``params`` (one call per tensor; returns work handles)."""
    works = []
    if not (dist.is_available() and dist.is_initialized()):
        return works
    for p in params:
        g = p.grad if isinstance(p, torch.nn.Parameter) or hasattr(p, "grad") else p
        if g is None:
            continue
        works.append(dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group, async_op=async_op))
    return works
