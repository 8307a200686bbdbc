"""TEST INFRASTRUCTURE: seeded random queries in the reference's SQL grammar
over the micro tables (gen_lineorder / gen_part / gen_supplier): filters with
literal and column operands, string equality, arithmetic with int and float
literals (including division), SUM / COUNT / MIN / MAX / AVG, group-by on one
or two columns, projections, and one- or two-join FROM lists. Used by the
GPU fuzz parity test; the oracle decides what each query means."""
from __future__ import annotations

import random

LO_INT = {  # column: (lo, hi) at gen_lineorder(1e5)
    "lo_quantity": (1, 50), "lo_discount": (0, 10), "lo_revenue": (120, 6_000_000),
    "lo_extendedprice": (12, 5_000_000), "lo_orderdate": (19920101, 19981228),
    "lo_partkey": (0, 19999), "lo_suppkey": (0, 999), "lo_custkey": (0, 1999), "lo_linenumber": (1, 100000),
}
LO_STR = {"lo_shipmode": ["AIR", "SHIP", "REG AIR", "FOB", "RAIL", "MAIL", "TRUCK", "NONE"]}
P_INT = {"p_size": (1, 50), "p_partkey": (0, 999)}
P_STR = {"p_category": ["MFGR#7", "MFGR#9", "MFGR#20", "MFGR#1", "MFGR#99"]}
S_INT = {"s_suppkey": (0, 999)}
S_STR = {"s_region": ["REGION#1", "REGION#3", "REGION#0", "REGION#9"]}
GROUP_SMALL = ["lo_quantity", "lo_discount"]  # string outputs are rejected by the reference (int keys only)
OPS = ["<", "<=", ">", ">=", "=", "<>"]


def _literal(rng: random.Random, lo: int, hi: int) -> str:
    r = rng.random()
    if r < 0.1:
        return str(rng.choice([lo - 1, hi + 1, lo, hi]))
    return str(rng.randint(lo, hi))  # int columns compare with int literals only


def _expr(rng: random.Random, ints: dict) -> str:
    a = rng.choice(list(ints))
    r = rng.random()
    if r < 0.4:
        return a
    if r < 0.7:
        b = rng.choice(list(ints))
        return f"{a} {rng.choice(['+', '-', '*'])} {b}"
    if r < 0.85:
        d = rng.choice(["lo_discount - 5", "lo_quantity - 25", "3", "-7", "lo_discount"])
        if "lo_" in d and not any(d.startswith(k) for k in ints):
            d = str(rng.randint(1, 9))
        return f"{a} / ({d})"
    return f"{a} * {rng.choice(['0.5', '1.25', '-0.75', '3'])}"


def random_query(rng: random.Random) -> str:
    joins = rng.random()
    ints = dict(LO_INT)
    strs = dict(LO_STR)
    preds = []
    if joins < 0.7:
        frm = "lineorder"
    elif joins < 0.85:
        frm = "part, lineorder"
        preds.append("lo_partkey = p_partkey")
        ints.update(P_INT)
        strs.update(P_STR)
    else:
        frm = "part, supplier, lineorder"
        preds += ["lo_partkey = p_partkey", "lo_suppkey = s_suppkey"]
        ints.update(P_INT)
        ints.update(S_INT)
        strs.update(P_STR)
        strs.update(S_STR)
    for _ in range(rng.randint(0, 3)):
        r = rng.random()
        if r < 0.6:
            c = rng.choice(list(ints))
            preds.append(f"{c} {rng.choice(OPS)} {_literal(rng, *ints[c])}")
        elif r < 0.8:
            c = rng.choice(list(strs))
            preds.append(f"{c} {rng.choice(['=', '<>'])} '{rng.choice(strs[c])}'")
        else:
            a, b = rng.sample([k for k in ints if k.startswith("lo_")], 2)
            preds.append(f"{a} {rng.choice(OPS)} {b}")
    where = f" where {' and '.join(preds)}" if preds else ""
    kind = rng.random()
    if kind < 0.15:  # projection (kept small by a selective filter)
        cols = rng.sample([k for k in ints if k.startswith("lo_")], rng.randint(1, 3))
        extra = " and " if where else " where "
        return f"select {', '.join(cols)} from {frm}{where}{extra}lo_linenumber < {rng.randint(1, 3000)}"
    aggs = []
    for _ in range(rng.randint(1, 4)):
        fn = rng.choice(["sum", "sum", "count", "min", "max", "avg"])
        a = "count(*)" if fn == "count" else f"{fn}({_expr(rng, ints)})"
        if a not in aggs:  # result column names must be distinct
            aggs.append(a)
    if kind < 0.55:
        return f"select {', '.join(aggs)} from {frm}{where}"
    pool = GROUP_SMALL + (["p_size"] if "part" in frm else [])
    if rng.random() < 0.15:
        pool = pool + ["lo_partkey"]  # many groups
    keys = rng.sample(pool, rng.randint(1, 2))
    return f"select {', '.join(keys)}, {', '.join(aggs)} from {frm}{where} group by {', '.join(keys)}"
