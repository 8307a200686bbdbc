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


def copartition_range(lineitem_begin: int, lineitem_end: int) -> tuple[int, int]:
    """The orders rows holding exactly the orderkeys of lineitem rows
    [begin, end): l_orderkey = i / 4 + 1 and o_orderkey = j + 1
    (include/hawk_gen.h), so lineitem shard boundaries that are multiples of
    4 cut orders at [begin / 4, end / 4). Each rank then builds the orders
    join table of its own shard only, and every lineitem row finds its order
    on its own GPU (TPC-H Q3)."""
    if lineitem_begin % 4 or (lineitem_end % 4 and lineitem_end != lineitem_begin):
        raise ValueError("lineitem shard boundaries must be multiples of 4")
    return lineitem_begin // 4, lineitem_end // 4


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
    """Host statement of the cross-shard merge the engine performs in
    Engine::finalize_partials (csrc/engine/engine.cpp), used by the CPU tests.

    Partials are int64 words: group keys, then one accumulator per aggregate,
    f64 accumulators as their IEEE bits. aggs = [(fn, type)] with fn HAWK_SUM=0,
    COUNT=1, MIN=2, MAX=3 and type HAWK_I64=0 / HAWK_F64=1. Integer SUM/COUNT
    add with int64 wrap-around (planner_reference.cpp:25-33); MIN/MAX select.
    sink 0 = AGGREGATE (1 x naggs), 1 = HASH_AGGREGATE (groups x (keys + aggs));
    groups come back sorted by key."""
    def f64(w: int) -> float:
        return float(np.array([w], dtype=np.int64).view(np.float64)[0])

    def bits(x: float) -> int:
        return int(np.array([x], dtype=np.float64).view(np.int64)[0])

    def combine(fn: int, ty: int, a: int, b: int) -> int:
        if ty == 1 and fn != 1:
            x, y = f64(a), f64(b)
            return bits(x + y if fn == 0 else min(x, y) if fn == 2 else max(x, y))
        if fn in (0, 1):
            return ((a + b + (1 << 63)) % (1 << 64)) - (1 << 63)
        return min(a, b) if fn == 2 else max(a, b)

    def fold(acc, row):
        return row if acc is None else [combine(f, t, a, b) for (f, t), a, b in zip(aggs, acc, row)]

    if sink == 0:
        acc = None
        for p in parts:
            if p.size:
                acc = fold(acc, [int(v) for v in p.reshape(-1)[: len(aggs)]])
        return np.array([acc if acc is not None else [0] * len(aggs)], dtype=np.int64)
    groups: dict[tuple, list[int]] = {}
    for p in parts:
        for row in p.reshape(-1, nkeys + len(aggs)):
            key = tuple(int(v) for v in row[:nkeys])
            groups[key] = fold(groups.get(key), [int(v) for v in row[nkeys:]])
    out = [list(k) + v for k, v in sorted(groups.items())]
    return np.array(out, dtype=np.int64).reshape(len(out), nkeys + len(aggs))
