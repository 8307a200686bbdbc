"""TEST INFRASTRUCTURE / REFERENCE ARM: the reference's own CPU path
(reference_execute, /root/reference/proj/src/planner_reference.cpp:331,
compiled unmodified into oracle/_ref/libhawk_oracle.so) over a whole
BASELINE workload, on every host core.

reference_execute is single-threaded by design and reentrant
(no shared state), so the fact table is split into one contiguous row shard
per host thread, exactly as the GPU engine shards it across GPUs: each thread
runs reference_execute over its shard (dimension tables shared), and the
shard results are merged the way the engine merges partials (integer SUM /
COUNT add with int64 wrap-around, planner_reference.cpp:25-33; AVG = merged
SUM / merged COUNT, :305-308). Columns come from oracle/port's generator
(port_gen), so no product library is loaded on this path.

Used by bench.py (`--impl reference` and the cpu_baseline leg) and by
tests/test_oracle.py (the merged answer equals reference_execute on the whole
table).
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from oracle_bridge import OraDb, OraTable, port_gen
from paper_1709_00700_b200 import datagen as dg
from paper_1709_00700_b200 import queries as Q
from paper_1709_00700_b200.engine import INT64, STRING, Column

# per query: (SQL run on every shard, output positions of the group keys,
# positions that add, [(avg position, count position)] finalised after the merge)
_Q1_SHARD = Q.TPCH_Q1.replace("avg(l_quantity)", "sum(l_quantity)") \
    .replace("avg(l_extendedprice)", "sum(l_extendedprice)").replace("avg(l_discount)", "sum(l_discount)")
SHARDED = {
    "tpch_q6": (Q.TPCH_Q6, [], [0], []),
    "tpch_q1": (_Q1_SHARD, [0, 1], [2, 3, 4, 5, 6, 7, 8, 9], [(6, 9), (7, 9), (8, 9)]),
    "ssb_q11": (Q.SSB_Q11, [], [0], []),
    "ssb_q41": (Q.SSB_Q41, [0, 1], [2], []),
    "tpch_q3": (Q.TPCH_Q3, [0, 2, 3], [1], []),
}


def _referenced(query: str, table: int) -> list[int]:
    """Columns of `table` the query reads (fact tables: FACT_COLUMNS; the
    dimension tables are kept whole)."""
    name, cols = dg.SCHEMA[table]
    if table != Q.BENCH[query][2]:
        return list(range(len(cols)))
    want = set(Q.FACT_COLUMNS[query])
    return [i for i, (c, _) in enumerate(cols) if c in want]


def _table(table: int, sf: float, seed: int, begin: int, n: int, cols: list[int], threads: int) -> OraTable:
    name, schema = dg.SCHEMA[table]
    out = []
    for ci in cols:
        cname, lex = schema[ci]
        vals = port_gen(table, ci, sf, seed, begin, n, threads)
        if lex is None:
            out.append(Column(cname, INT64, vals))
        else:
            codes, order = dg.first_appearance(vals, lex)
            out.append(Column(cname, STRING, codes, order))
    return OraTable.from_columns(name, out)


class ShardedReference:
    """reference_execute over `threads` row shards of the fact table."""

    def __init__(self, query: str, sf: float, seed: int = 42, threads: int | None = None,
                 fact_rows: int | None = None, fact_begin: int = 0):
        self.query = query
        self.threads = threads or os.cpu_count() or 1
        _, tables, fact = Q.BENCH[query]
        n = dg.table_rows(fact, sf) - fact_begin if fact_rows is None else fact_rows
        self.fact_rows = n
        t0 = time.perf_counter()
        dims = [_table(t, sf, seed, 0, dg.table_rows(t, sf), _referenced(query, t), self.threads)
                for t in tables if t != fact]
        per = -(-n // self.threads)
        per = -(-per // 64) * 64
        spans = [(b, min(n, b + per)) for b in range(0, n, per)] or [(0, 0)]
        fcols = _referenced(query, fact)

        def shard(span):
            b, e = span
            return _table(fact, sf, seed, fact_begin + b, e - b, fcols, 1)
        with ThreadPoolExecutor(self.threads) as ex:
            facts = list(ex.map(shard, spans))
        self.dbs = []
        for f in facts:
            db = OraDb()
            for d in dims:
                db.add(d)
            db.add(f)
            self.dbs.append(db)
        self.build_s = time.perf_counter() - t0
        self.shards = len(self.dbs)

    def run(self) -> np.ndarray:
        """One execution of the whole workload: every shard's reference_execute
        concurrently, then the merge. Returns rows in SELECT order (int64
        words; AVG columns as float64 bit patterns), keys sorted."""
        sql, keys, adds, avgs = SHARDED[self.query]
        with ThreadPoolExecutor(self.threads) as ex:
            parts = list(ex.map(lambda db: db.execute(sql), self.dbs))
        blocks = []
        for p in parts:
            cols = [np.asarray(c.values) for c in p.columns()]
            if cols and len(cols[0]):
                blocks.append(np.stack([c.view(np.int64) if c.dtype == np.float64 else c.astype(np.int64)
                                        for c in cols], axis=1))
        width = len(keys) + len(adds) + (0 if keys else 0)
        width = max([b.shape[1] for b in blocks], default=max(keys + adds, default=0) + 1)
        if not blocks:
            allr = np.zeros((0, width), np.int64)
        else:
            allr = np.concatenate(blocks)
        if keys:
            uniq, inv = np.unique(allr[:, keys], axis=0, return_inverse=True)
            out = np.zeros((len(uniq), width), np.int64)
            out[:, keys] = uniq
            with np.errstate(over="ignore"):
                for a in adds:
                    np.add.at(out[:, a], inv.reshape(-1), allr[:, a])
        else:
            out = np.zeros((1, width), np.int64)
            with np.errstate(over="ignore"):
                for a in adds:
                    out[0, a] = allr[:, a].sum(dtype=np.int64) if len(allr) else 0
        for a, c in avgs:
            out[:, a] = (out[:, a].astype(np.float64) / out[:, c].astype(np.float64)).view(np.int64)
        return out

    def timed(self, reps: int = 1) -> list[float]:
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            self.run()
            times.append(time.perf_counter() - t0)
        return times


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_variant_rate(query: str, sf: float, seed: int = 42, threads: int | None = None):
    """The reference's CPU variant (cpu-o, oracle/cpu_o.cpp) over the whole
    workload on every host thread: (fact tuples/s, threads, fact rows)."""
    threads = threads or os.cpu_count() or 1
    _, tables, fact = Q.BENCH[query]
    db = OraDb()
    for t in tables:
        db.add(_table(t, sf, seed, 0, dg.table_rows(t, sf), _referenced(query, t), threads))
    sql = Q.BENCH[query][0]
    db.execute_cpu_o(sql, threads)
    t0 = time.perf_counter()
    db.execute_cpu_o(sql, threads)
    dt = time.perf_counter() - t0
    n = dg.table_rows(fact, sf)
    return n / dt, threads, n
