"""Multi-GPU host logic on CPU (gloo, world_size 2): fact-table row sharding,
the variable-row all-gather of partials and the cross-shard merge.

Each rank runs the reference oracle (reference_execute, oracle/_ref) on ITS
shard of the fact table with the dimensions replicated — exactly what a GPU
rank computes with Engine.run_partial — the partial group rows are gathered
over torch.distributed and merged with distributed.merge_partials_host; rank 0
checks the merge against the oracle on the whole table.
"""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# a grouped query with every merge rule (SUM wraps, MIN/MAX select, COUNT adds)
MINMAX = ("select l_returnflag, l_linestatus, sum(l_quantity) as q, min(l_extendedprice) as lo, "
          "max(l_discount) as hi, count(*) as n from lineitem where l_shipdate <= 19980902 "
          "group by l_returnflag, l_linestatus")


def _case(name):
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    if name == "tpch_q3_copartitioned":
        sql, tables, fact = Q.BENCH["tpch_q3"]
        return sql, tables, fact, [0, 2, 3], [(1, 0, 0)]
    # (key positions, [(agg position, fn, type)]) with SUM=0 COUNT=1 MIN=2 MAX=3, I64=0
    if name == "minmax":
        return MINMAX, [dg.LINEITEM], dg.LINEITEM, [0, 1], [(2, 0, 0), (3, 2, 0), (4, 3, 0), (5, 1, 0)]
    sql, tables, fact = Q.BENCH[name]
    layout = {"tpch_q6": ([], [(0, 0, 0)]), "ssb_q11": ([], [(0, 0, 0)]),
              "ssb_q41": ([0, 1], [(2, 0, 0)]), "tpch_q3": ([0, 2, 3], [(1, 0, 0)])}[name]
    return sql, tables, fact, layout[0], layout[1]


def _rows(table, keys, aggs) -> np.ndarray:
    cols = [c.values for c in table.columns()]
    order = keys + [a[0] for a in aggs]
    if not cols or len(cols[0]) == 0:
        return np.zeros((0, len(order)), np.int64)
    return np.stack([np.asarray(cols[i], dtype=np.int64) for i in order], axis=1)


def _worker(rank, world, port, name, sf, seed, failures):
    import torch.distributed as dist
    sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
    from oracle_bridge import OraDb, OraTable
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200.distributed import (all_gather_rows, copartition_range,
                                                   merge_partials_host, shard_range)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        sql, tables, fact, keys, aggs = _case(name)
        n = dg.table_rows(fact, sf)
        b, e = shard_range(n, rank, world)
        db = OraDb()
        for t in tables:
            if t == fact:
                tname, cols = dg.host_table(t, sf, seed, b, e - b)
            elif name == "tpch_q3_copartitioned" and t == dg.ORDERS:
                # orders co-partitioned with the lineitem shard (bench.py load_tables)
                ob, oe = copartition_range(b, e)
                tname, cols = dg.host_table(t, sf, seed, ob, oe - ob)
            else:
                tname, cols = dg.host_table(t, sf, seed)
            db.add(OraTable.from_columns(tname, cols))
        part = _rows(db.execute(sql), keys, aggs)
        gathered = all_gather_rows(part)
        assert len(gathered) == world
        merged = merge_partials_host(1 if keys else 0, [(f, t) for _, f, t in aggs], len(keys), gathered)
        if rank == 0:
            full = OraDb()
            for t in tables:
                tname, cols = dg.host_table(t, sf, seed)
                full.add(OraTable.from_columns(tname, cols))
            want = _rows(full.execute(sql), keys, aggs)
            want = want[np.lexsort(want[:, ::-1].T)] if keys and len(want) else want
            if want.shape != merged.shape or not np.array_equal(want, merged):
                failures.put(f"{name}: merged {merged.shape} != oracle {want.shape}")
    except Exception as ex:  # noqa: BLE001 - surfaced through the queue
        failures.put(f"rank {rank}: {type(ex).__name__}: {ex}")
    finally:
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name", ["tpch_q6", "ssb_q11", "ssb_q41", "tpch_q3", "tpch_q3_copartitioned",
                                  "minmax"])
def test_sharded_partials_merge_to_oracle(name):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    failures = ctx.Queue()
    mp.start_processes(_worker, args=(2, _free_port(), name, 0.01, 42, failures), nprocs=2,
                       join=True, start_method="spawn")
    errs = []
    while not failures.empty():
        errs.append(failures.get())
    assert not errs, errs


def test_shard_range_partitions_rows():
    from paper_1709_00700_b200.distributed import shard_range
    for n in (0, 1, 63, 64, 65, 6_001_215, 59_986_052):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (b0, e0), (b1, _) in zip(spans, spans[1:]):
                assert e0 == b1 and b0 <= e0
            assert all(b % 64 == 0 or b == n for b, _ in spans)


def test_merge_partials_host_semantics():
    from paper_1709_00700_b200.distributed import merge_partials_host
    big = np.int64(2**62)
    f = lambda x: np.array([x], np.float64).view(np.int64)[0]  # noqa: E731
    # SUM wraps like int64; COUNT adds; MIN/MAX select; f64 SUM adds as doubles
    a = np.array([[big, 3, 10, -5, f(1.5)]], np.int64)
    b = np.array([[big, 4, 7, 9, f(2.25)]], np.int64)
    aggs = [(0, 0), (1, 0), (2, 0), (3, 0), (0, 1)]
    m = merge_partials_host(0, aggs, 0, [a, b])
    assert m.tolist()[0][:4] == [-(2**63), 7, 7, 9]
    assert m.view(np.float64)[0, 4] == 3.75
    # grouped: keys merge, output sorted by key, empty shards allowed
    g1 = np.array([[2, 5], [1, 1]], np.int64)
    g2 = np.array([[1, 10], [3, 0]], np.int64)
    empty = np.zeros((0, 2), np.int64)
    m = merge_partials_host(1, [(0, 0)], 1, [g1, empty, g2])
    assert m.tolist() == [[1, 11], [2, 5], [3, 0]]


def test_copartition_range():
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200.distributed import copartition_range, shard_range
    n = dg.table_rows(dg.LINEITEM, 0.01)
    for world in (2, 3, 8):
        spans = [copartition_range(*shard_range(n, r, world)) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == dg.table_rows(dg.ORDERS, 0.01)
        for (b0, e0), (b1, _) in zip(spans, spans[1:]):
            assert e0 == b1
    with pytest.raises(ValueError):
        copartition_range(2, 8)
