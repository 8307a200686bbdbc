"""Multi-GPU plumbing: one process per GPU, fact tables row-partitioned across
ranks, dimension tables replicated, partial results exchanged once per query.

The reference is single-process; the data-parallel scheme is
SURVEY.md §8e: contiguous fact-table row ranges per GPU, each GPU runs every
pipeline on its shard, and the partial aggregates (AGGREGATE accumulators or
HASH_AGGREGATE group rows) are all-gathered and merged, then finalised.
torch.distributed (NCCL on GPUs, gloo on CPU) carries the exchange.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int, align: int = 64) -> tuple[int, int]:
    """Contiguous [begin, end) of rank's rows; boundaries aligned for 128-bit loads."""
    per = -(-n // world)
    per = -(-per // align) * align
    b = min(n, rank * per)
    return b, min(n, b + per)


def all_gather_rows(parts: np.ndarray, device=None) -> list[np.ndarray]:
    """All-gathers a (rows x width) int64 block from every rank (variable rows)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    dev = device if device is not None else torch.device("cpu")
    rows = torch.tensor([parts.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(rows) for _ in range(world)]
    dist.all_gather(counts, rows)
    counts = [int(c.item()) for c in counts]
    width = parts.shape[1] if parts.ndim == 2 else 1
    cap = max(1, max(counts))
    buf = torch.zeros((cap, width), dtype=torch.int64, device=dev)
    if parts.shape[0]:
        buf[: parts.shape[0]] = torch.from_numpy(np.ascontiguousarray(parts).reshape(-1, width)).to(dev)
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    return [o[:c].cpu().numpy() for o, c in zip(out, counts)]


def merge_partials_host(sink: int, aggs: list[tuple[int, int]], nkeys: int,
                        parts: list[np.ndarray]) -> np.ndarray:
    """Host reference of the partial merge (used by the CPU tests): SUM/COUNT
    add with int64 wrap, MIN/MAX select; aggs = [(fn, type)] per accumulator.
    sink 0 = AGGREGATE (1 x naggs), 1 = HASH_AGGREGATE (groups x (keys + aggs))."""
    def combine(fn, a, b):
        if fn in (0, 1):
            return (a + b) & 0xFFFFFFFFFFFFFFFF
        return min(a, b) if fn == 2 else max(a, b)

    def to_signed(x):
        return x - (1 << 64) if x >= 1 << 63 else x

    if sink == 0:
        acc = None
        for p in parts:
            row = [int(v) for v in p.reshape(-1)]
            acc = row if acc is None else [combine(f, a, b) for (f, _), a, b in zip(aggs, acc, row)]
        return np.array([[to_signed(v) if v >= 0 else v for v in acc]], dtype=np.int64)
    groups: dict[tuple, list[int]] = {}
    for p in parts:
        for row in p:
            key = tuple(int(v) for v in row[:nkeys])
            vals = [int(v) for v in row[nkeys:]]
            if key in groups:
                groups[key] = [combine(f, a, b) for (f, _), a, b in zip(aggs, groups[key], vals)]
            else:
                groups[key] = vals
    out = [list(k) + [to_signed(v) if v >= 0 else v for v in vals] for k, vals in sorted(groups.items())]
    return np.array(out, dtype=np.int64).reshape(len(out), nkeys + len(aggs))
