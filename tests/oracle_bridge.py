"""TEST INFRASTRUCTURE: ctypes bridge to the parity checker.

oracle/_ref/libhawk_oracle.so — the reference's own sources (reference_execute,
compare_result_tables, result_checksum, gen_lineorder ...) plus oracle/ref_shim.cpp.
oracle/_ref/libhawk_port.so   — our CPU restatement (oracle/port), pinned against it.

Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline use this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "oracle", "_ref")

i32, i64, u64, f64, vp, cp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p, C.c_char_p

_ora = None
_port = None


def _sig(lib, name, res, *args):
    fn = getattr(lib, name)
    fn.restype = res
    fn.argtypes = list(args)


def ora():
    global _ora
    if _ora is None:
        lib = C.CDLL(os.path.join(REF_DIR, "libhawk_oracle.so"), mode=C.RTLD_LOCAL)
        _sig(lib, "ora_table_new", vp, cp, i32, C.POINTER(cp), C.POINTER(i32), i64, C.POINTER(vp),
             C.POINTER(C.POINTER(cp)), C.POINTER(i64), cp, i32)
        _sig(lib, "ora_table_gen", vp, cp, i64, u64, cp, i32)
        _sig(lib, "ora_table_load_csv", vp, cp, cp, i32, C.POINTER(cp), C.POINTER(i32), C.c_char, i32, cp, i32)
        _sig(lib, "ora_table_free", None, vp)
        _sig(lib, "ora_table_rows", i64, vp)
        _sig(lib, "ora_table_ncols", i32, vp)
        _sig(lib, "ora_table_name", cp, vp)
        _sig(lib, "ora_table_col_name", cp, vp, i32)
        _sig(lib, "ora_table_col_kind", i32, vp, i32)
        _sig(lib, "ora_table_col_data", vp, vp, i32)
        _sig(lib, "ora_table_col_lexicon_size", i64, vp, i32)
        _sig(lib, "ora_table_col_lexicon", cp, vp, i32, i64)
        _sig(lib, "ora_table_col_distinct", i64, vp, i32)
        _sig(lib, "ora_table_checksum", u64, vp)
        _sig(lib, "ora_compare", i32, vp, vp, f64, cp, i32)
        _sig(lib, "ora_db_new", vp)
        _sig(lib, "ora_db_free", None, vp)
        _sig(lib, "ora_db_add", None, vp, vp)
        _sig(lib, "ora_execute", vp, vp, cp, C.POINTER(i32), cp, i32)
        _sig(lib, "ora_pipeline_count", i32, vp, cp, cp, i32)
        _sig(lib, "ora_execute_cpu_o", vp, vp, cp, i32, C.POINTER(i32), cp, i32)
        _ora = lib
    return _ora


def port():
    global _port
    if _port is None:
        lib = C.CDLL(os.path.join(REF_DIR, "libhawk_port.so"), mode=C.RTLD_LOCAL)
        _sig(lib, "port_gen", None, i32, i32, f64, u64, i64, i64, vp, i32)
        _sig(lib, "port_width", i32, i32)
        _sig(lib, "port_run", i64, i32, C.POINTER(vp), i64, C.POINTER(i64), C.POINTER(i64), i32,
             vp, i64)
        _sig(lib, "port_run_gen", i64, i32, f64, u64, i64, i64, C.POINTER(i64), i32, vp, i64)
        _port = lib
    return _port


class OraError(RuntimeError):
    def __init__(self, cls: int, msg: str):
        super().__init__(msg)
        self.cls = cls


class OraTable:
    """A reference hawk::Table (owned)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        try:
            if self.h:
                ora().ora_table_free(self.h)
        except Exception:
            pass

    @classmethod
    def from_columns(cls, name: str, columns) -> "OraTable":
        """columns: list of paper_1709_00700_b200.engine.Column"""
        lib = ora()
        n = len(columns[0].values) if columns else 0
        keep = []
        names = (cp * max(1, len(columns)))(*[c.name.encode() for c in columns])
        kinds = (i32 * max(1, len(columns)))(*[c.kind for c in columns])
        data = (vp * max(1, len(columns)))()
        lexs = (C.POINTER(cp) * max(1, len(columns)))()
        lsz = (i64 * max(1, len(columns)))()
        for i, c in enumerate(columns):
            arr = np.ascontiguousarray(c.values, dtype=np.float64 if c.kind == 1 else np.int64)
            keep.append(arr)
            data[i] = arr.ctypes.data
            if c.kind == 2:
                lx = (cp * max(1, len(c.lexicon)))(*[s.encode() for s in c.lexicon])
                keep.append(lx)
                lexs[i] = C.cast(lx, C.POINTER(cp))
                lsz[i] = len(c.lexicon)
        err = C.create_string_buffer(512)
        h = lib.ora_table_new(name.encode(), len(columns), names, kinds, n, data, lexs, lsz, err, 512)
        if not h:
            raise RuntimeError(err.value.decode())
        return cls(h)

    @classmethod
    def generated(cls, which: str, n: int, seed: int) -> "OraTable":
        err = C.create_string_buffer(512)
        h = ora().ora_table_gen(which.encode(), n, seed, err, 512)
        if not h:
            raise RuntimeError(err.value.decode())
        return cls(h)

    @classmethod
    def load_csv(cls, path: str, name: str, schema, delimiter: str = ",", header: bool = False) -> "OraTable":
        """The reference's own load_csv (storage_csv.cpp:111-155); raises
        RuntimeError with the reference's ParseError / IoError message."""
        names = (cp * len(schema))(*[n.encode() for n, _ in schema])
        kinds = (i32 * len(schema))(*[k for _, k in schema])
        err = C.create_string_buffer(1024)
        h = ora().ora_table_load_csv(path.encode(), name.encode(), len(schema), names, kinds,
                                     delimiter.encode(), int(header), err, 1024)
        if not h:
            raise RuntimeError(err.value.decode())
        return cls(h)

    @property
    def rows(self) -> int:
        return ora().ora_table_rows(self.h)

    @property
    def name(self) -> str:
        return ora().ora_table_name(self.h).decode()

    def columns(self):
        from paper_1709_00700_b200.engine import Column
        lib = ora()
        out = []
        n = self.rows
        for c in range(lib.ora_table_ncols(self.h)):
            kind = lib.ora_table_col_kind(self.h, c)
            ptr = lib.ora_table_col_data(self.h, c)
            ct = C.c_double if kind == 1 else C.c_int64
            vals = (np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy()
                    if n else np.zeros(0, np.float64 if kind == 1 else np.int64))
            lex = None
            if kind == 2:
                lex = [lib.ora_table_col_lexicon(self.h, c, i).decode()
                       for i in range(lib.ora_table_col_lexicon_size(self.h, c))]
            out.append(Column(lib.ora_table_col_name(self.h, c).decode(), kind, vals, lex))
        return out

    def distinct(self) -> list[int]:
        lib = ora()
        return [lib.ora_table_col_distinct(self.h, c) for c in range(lib.ora_table_ncols(self.h))]

    def checksum(self) -> int:
        return ora().ora_table_checksum(self.h)

    def compare(self, actual: "OraTable", rel_tol: float = 1e-9) -> str | None:
        """compare_result_tables(expected=self, actual): None when equal."""
        msg = C.create_string_buffer(2048)
        r = ora().ora_compare(self.h, actual.h, rel_tol, msg, 2048)
        return None if r == 0 else msg.value.decode()

    def canonical_rows(self) -> list[tuple]:
        cols = self.columns()
        rows = list(zip(*[c.decoded() for c in cols])) if cols else []
        return sorted(rows)


class OraDb:
    def __init__(self):
        self.h = ora().ora_db_new()
        self.tables: list[OraTable] = []

    def __del__(self):
        try:
            ora().ora_db_free(self.h)
        except Exception:
            pass

    def add(self, t: OraTable):
        self.tables.append(t)
        ora().ora_db_add(self.h, t.h)

    def execute(self, sql: str) -> OraTable:
        cls = i32()
        err = C.create_string_buffer(1024)
        h = ora().ora_execute(self.h, sql.encode(), C.byref(cls), err, 1024)
        if not h:
            raise OraError(cls.value, err.value.decode())
        return OraTable(h)

    def execute_cpu_o(self, sql: str, threads: int = 0) -> OraTable:
        """The reference's CPU variant (cpu-o, oracle/cpu_o.cpp) on `threads`
        host threads (0 = all)."""
        cls = i32()
        err = C.create_string_buffer(1024)
        h = ora().ora_execute_cpu_o(self.h, sql.encode(), threads or (os.cpu_count() or 1), C.byref(cls), err, 1024)
        if not h:
            raise OraError(cls.value, err.value.decode())
        return OraTable(h)

    def pipeline_count(self, sql: str) -> int:
        err = C.create_string_buffer(512)
        return ora().ora_pipeline_count(self.h, sql.encode(), err, 512)


def result_table(result) -> OraTable:
    """Engine Result -> reference Table for compare_result_tables."""
    return OraTable.from_columns("result", result.columns)


def port_gen(table: int, col: int, sf: float, seed: int, begin: int, n: int,
             threads: int = 0) -> np.ndarray:
    """Rows [begin, begin + n) of a generated column (include/hawk_gen.h) on
    the host, without the product library."""
    out = np.empty(max(n, 0), dtype=np.int64)
    if n > 0:
        port().port_gen(table, col, sf, seed, begin, n, out.ctypes.data, threads or (os.cpu_count() or 1))
    return out


def port_run_gen(query: int, sf: float, seed: int, codes: list[int], threads: int,
                 out_rows: int, row_begin: int = 0, n: int | None = None) -> np.ndarray:
    """The streaming restatement (oracle/port, port_run_gen): fact rows are
    regenerated chunk by chunk per worker, so SF100 needs no host table."""
    from paper_1709_00700_b200 import datagen as dg
    lib = port()
    fact = dg.LINEORDER if query in (2, 3) else dg.LINEITEM
    if n is None:
        n = dg.table_rows(fact, sf) - row_begin
    cds = (i64 * max(1, len(codes)))(*codes)
    w = lib.port_width(query)
    out = np.zeros((max(1, out_rows), w), dtype=np.int64)
    r = lib.port_run_gen(query, sf, seed, row_begin, n, cds, threads, out.ctypes.data, out_rows)
    if r < 0:
        raise RuntimeError("port output buffer too small")
    return out[:r]


def port_run(query: int, cols: list[np.ndarray], n: int, dim_rows: list[int], codes: list[int],
             threads: int, out_rows: int) -> np.ndarray:
    lib = port()
    arrs = [np.ascontiguousarray(c, dtype=np.int64) for c in cols]
    ptrs = (vp * len(arrs))(*[a.ctypes.data for a in arrs])
    dims = (i64 * max(1, len(dim_rows)))(*dim_rows)
    cds = (i64 * max(1, len(codes)))(*codes)
    w = lib.port_width(query)
    out = np.zeros((max(1, out_rows), w), dtype=np.int64)
    r = lib.port_run(query, ptrs, n, dims, cds, threads, out.ctypes.data, out_rows)
    if r < 0:
        raise RuntimeError("port output buffer too small")
    return out[:r]
