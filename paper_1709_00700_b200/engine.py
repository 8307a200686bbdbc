"""Python host mirror of the engine's C ABI (include/hawk_b200_engine.h).

Mirrors the reference CLI's `run` / `explore` / `learn` operations
 with the reference's error classes
(/root/reference/proj/include/hawk/error.hpp:9-54) raised as Python
exceptions of the same names. All work happens in libhawk_engine.so and the
sm_100a kernels of libhawk_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import _native

# ---- reference exception classes (hawk/error.hpp) ------------------------------


class HawkError(RuntimeError):
    code = 99


class UnsupportedPlan(HawkError):
    code = 1


class InvalidConfig(HawkError):
    code = 2


class Unsupported(HawkError):
    code = 3


class PlanTooLarge(HawkError):
    code = 4


class CapacityExceeded(HawkError):
    code = 5


class DuplicateKey(HawkError):
    code = 6


class EmptyAggregate(HawkError):
    code = 7


class DivergentPlan(HawkError):
    code = 8


class InvalidParams(HawkError):
    code = 9


class SyntaxError_(HawkError):
    code = 10


class UnknownTable(HawkError):
    code = 11


class UnknownAttribute(HawkError):
    code = 12


class TypeError_(HawkError):
    code = 13


class ParseError_(HawkError):
    code = 14


class IoError_(HawkError):
    code = 15


_BY_CODE = {c.code: c for c in (UnsupportedPlan, InvalidConfig, Unsupported, PlanTooLarge,
                                CapacityExceeded, DuplicateKey, EmptyAggregate, DivergentPlan,
                                InvalidParams, SyntaxError_, UnknownTable, UnknownAttribute,
                                TypeError_, ParseError_, IoError_)}
ERROR_NAMES = {1: "UnsupportedPlan", 2: "InvalidConfig", 3: "Unsupported", 4: "PlanTooLarge",
               5: "CapacityExceeded", 6: "DuplicateKey", 7: "EmptyAggregate",
               8: "DivergentPlan", 9: "InvalidParams", 10: "SyntaxError", 11: "UnknownTable",
               12: "UnknownAttribute", 13: "TypeError", 14: "ParseError", 15: "IoError"}


def _raise(status: int):
    lib = _native.engine()
    msg = lib.hawk_engine_last_error().decode(errors="replace")
    raise _BY_CODE.get(status, HawkError)(msg)


def _check(status: int):
    if status != 0:
        _raise(status)


INT64, FLOAT64, STRING = 0, 1, 2


@dataclass
class Column:
    name: str
    kind: int
    values: np.ndarray            # int64 / float64 / int64 codes
    lexicon: list[str] | None = None

    def decoded(self) -> list:
        if self.kind == STRING:
            return [self.lexicon[c] for c in self.values]
        return self.values.tolist()


class Partial(NamedTuple):
    """A shard's partial result (Engine.run_partial): AGGREGATE accumulators,
    HASH_AGGREGATE group rows (keys + accumulators) or projected rows."""
    rows: np.ndarray
    sink: int
    kernel_ms: float
    launches: int


class Result:
    """A query result. Columns are zero-copy views of the engine's result
    buffers, built on first access (as are the per-pipeline metrics), so a
    caller that only reads timings pays no per-column work."""

    def __init__(self, owner, lib, r):
        self._owner, self._lib, self._r = owner, lib, r
        self.kernel_ms = lib.hawk_result_kernel_ms(r)
        self.wall_ms = lib.hawk_result_wall_ms(r)
        self.input_tuples = lib.hawk_result_input_tuples(r)
        self.launches = lib.hawk_result_launches(r)
        self.rows = lib.hawk_result_rows(r)
        self._columns = None
        self._pipelines = None

    @property
    def columns(self) -> list[Column]:
        if self._columns is None:
            self._columns = _columns_of(self._lib, self._r, self._owner, self.rows)
        return self._columns

    @property
    def pipelines(self) -> list[dict]:
        if self._pipelines is None:
            pipes = []
            for line in self._lib.hawk_result_metrics_text(self._r).decode().splitlines():
                p = line.split()
                if len(p) >= 8:
                    pipes.append(dict(variant=p[0], kernel_ms=float(p[1]), launches=int(p[2]),
                                      rows_in=int(p[3]), rows_out=int(p[4]), grid=int(p[5]),
                                      block=int(p[6]), retries=int(p[7])))
            self._pipelines = pipes
        return self._pipelines

    def column(self, name: str) -> Column:
        for c in self.columns:
            if c.name == name:
                return c
        raise KeyError(name)


class _ResultOwner:
    """Frees a hawk_result once no column array views its memory any more."""

    def __init__(self, lib, r):
        self.lib, self.r = lib, r

    def __del__(self):
        try:
            self.lib.hawk_result_free(self.r)
        except Exception:
            pass


def _columns_of(lib, r, owner, n) -> list[Column]:
    cols = []
    for c in range(lib.hawk_result_ncols(r)):
        kind = lib.hawk_result_col_kind(r, c)
        name = lib.hawk_result_col_name(r, c).decode()
        ptr = lib.hawk_result_col_data(r, c)
        dtype = np.float64 if kind == FLOAT64 else np.int64
        if n:
            buf = ((C.c_double if kind == FLOAT64 else C.c_int64) * n).from_address(ptr)
            buf._owner = owner
            vals = np.ctypeslib.as_array(buf)
        else:
            vals = np.zeros(0, dtype)
        lex = None
        if kind == STRING:
            lex = [lib.hawk_result_col_lexicon(r, c, i).decode()
                   for i in range(lib.hawk_result_col_lexicon_size(r, c))]
        cols.append(Column(name, kind, vals, lex))
    return cols


def _result_from(lib, r) -> Result:
    """Result columns are zero-copy views of the engine's result buffers; the
    hawk_result lives as long as the Result or any of its column arrays
    (large results, e.g. TPC-H Q3 SF100's 1.2M groups, are not copied again)."""
    return Result(_ResultOwner(lib, r), lib, r)


class Engine:
    """One B200 engine (device column store + executor). device < 0 gives a
    planning-only engine: catalog, passes, variant space, lowering; no GPU."""

    def __init__(self, device: int = 0):
        self._lib = _native.engine()
        h = C.c_void_p()
        _check(self._lib.hawk_engine_create(device, C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self._lib.hawk_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def sm_count(self) -> int:
        return self._lib.hawk_engine_sm_count(self._h)

    @property
    def ctx(self) -> int:
        return self._lib.hawk_engine_ctx(self._h)

    # ---- tables ----
    def put_table(self, name: str, columns: list[Column], distinct: list[int] | None = None,
                  row_offset: int = 0):
        """Uploads host columns (H2D); string columns are codes + lexicon."""
        n = len(columns[0].values) if columns else 0
        keep = []
        names = (C.c_char_p * len(columns))(*[c.name.encode() for c in columns])
        kinds = (C.c_int32 * len(columns))(*[c.kind for c in columns])
        data = (C.c_void_p * len(columns))()
        lexs = (C.POINTER(C.c_char_p) * len(columns))()
        lsz = (C.c_int64 * len(columns))()
        for i, c in enumerate(columns):
            arr = np.ascontiguousarray(c.values, dtype=np.float64 if c.kind == FLOAT64 else np.int64)
            keep.append(arr)
            data[i] = arr.ctypes.data
            if c.kind == STRING:
                lx = (C.c_char_p * max(1, len(c.lexicon)))(*[s.encode() for s in c.lexicon])
                keep.append(lx)
                lexs[i] = C.cast(lx, C.POINTER(C.c_char_p))
                lsz[i] = len(c.lexicon)
        dist = None
        if distinct is not None:
            dist = (C.c_int64 * len(columns))(*distinct)
        _check(self._lib.hawk_engine_put_columns(self._h, name.encode(), len(columns), names, kinds,
                                                 n, data, lexs, lsz, dist, row_offset))

    def generate(self, table: int, sf: float, seed: int = 42, row_begin: int = 0, rows: int = -1):
        """Generates a synthetic table (include/hawk_gen.h) directly in HBM."""
        _check(self._lib.hawk_engine_generate(self._h, table, sf, seed, row_begin, rows))

    def load_csv(self, path: str, name: str, schema: list[tuple[str, int]], delimiter: str = ",",
                 header: bool = False):
        """A CSV file into device columns, parsed on the device with the
        reference's load_csv rules (storage_csv.cpp:111-155). schema: (column,
        kind) pairs, kind INT64 / FLOAT64 / STRING."""
        names = (C.c_char_p * len(schema))(*[n.encode() for n, _ in schema])
        kinds = (C.c_int32 * len(schema))(*[k for _, k in schema])
        _check(self._lib.hawk_engine_load_csv(self._h, path.encode(), name.encode(), len(schema), names,
                                              kinds, delimiter.encode(), int(header)))

    def drop(self, name: str):
        _check(self._lib.hawk_engine_drop(self._h, name.encode()))

    def table_rows(self, name: str) -> int:
        return self._lib.hawk_engine_table_rows(self._h, name.encode())

    def column_ptr(self, table: str, column: str) -> int:
        return self._lib.hawk_engine_column(self._h, table.encode(), column.encode()) or 0

    def flush_l2(self):
        _check(self._lib.hawk_engine_flush_l2(self._h))

    # ---- execution ----
    def run(self, sql: str, config: str = "") -> Result:
        r = C.c_void_p()
        _check(self._lib.hawk_engine_run(self._h, sql.encode(), config.encode(), C.byref(r)))
        return _result_from(self._lib, r)  # frees r when the columns are gone

    def run_sharded(self, sql: str, config: str, comm: "Communicator", root: int = 0) -> Result:
        """Multi-GPU: this rank's shard, NCCL gather of the partials to `root`
        over device buffers, device merge (Engine::execute_sharded). Non-root
        ranks get the query's columns with no rows."""
        r = C.c_void_p()
        _check(self._lib.hawk_engine_run_sharded(self._h, sql.encode(), config.encode(), comm.handle,
                                                 root, C.byref(r)))
        return _result_from(self._lib, r)

    def run_partial(self, sql: str, config: str = "") -> "Partial":
        """Shard execution: the (rows x width) int64 partials before the cross-GPU merge."""
        p = C.c_void_p()
        _check(self._lib.hawk_engine_run_partial(self._h, sql.encode(), config.encode(), C.byref(p)))
        try:
            rows = self._lib.hawk_partial_rows(p)
            width = self._lib.hawk_partial_width(p)
            n = rows * width
            ptr = self._lib.hawk_partial_data(p)
            data = (np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_int64)), shape=(n,)).copy()
                    if n else np.zeros(0, np.int64))
            return Partial(data.reshape(rows, width), self._lib.hawk_partial_sink(p),
                           self._lib.hawk_partial_kernel_ms(p), self._lib.hawk_partial_launches(p))
        finally:
            self._lib.hawk_partial_free(p)

    def finalize(self, sql: str, parts: list[np.ndarray], config: str = "") -> Result:
        arrs = [np.ascontiguousarray(p, dtype=np.int64) for p in parts]
        data = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        rows = (C.c_int64 * len(arrs))(*[a.shape[0] if a.ndim == 2 else 1 for a in arrs])
        r = C.c_void_p()
        _check(self._lib.hawk_engine_finalize(self._h, sql.encode(), config.encode(), len(arrs),
                                              data, rows, C.byref(r)))
        return _result_from(self._lib, r)  # frees r when the columns are gone

    # ---- IR introspection ----
    def pipeline_count(self, sql: str) -> int:
        n = C.c_int32()
        _check(self._lib.hawk_engine_pipeline_count(self._h, sql.encode(), C.byref(n)))
        return n.value

    def space_size(self, sql: str, pipeline: int) -> tuple[int, int]:
        n, s = C.c_int32(), C.c_int32()
        _check(self._lib.hawk_engine_space_size(self._h, sql.encode(), pipeline, C.byref(n),
                                                C.byref(s)))
        return n.value, s.value

    def space_config(self, sql: str, pipeline: int, i: int) -> str:
        buf = C.create_string_buffer(256)
        _check(self._lib.hawk_engine_space_config(self._h, sql.encode(), pipeline, i, buf, 256))
        return buf.value.decode()

    def validate(self, sql: str, config: str = "") -> str:
        buf = C.create_string_buffer(1 << 16)
        _check(self._lib.hawk_engine_validate(self._h, sql.encode(), config.encode(), buf, 1 << 16))
        return buf.value.decode()

    def compile_check(self, sql: str, config: str = "") -> str:
        """NVRTC-compiles every pipeline's generated program (no GPU needed)."""
        buf = C.create_string_buffer(1 << 16)
        _check(self._lib.hawk_engine_compile_check(self._h, sql.encode(), config.encode(), buf,
                                                   1 << 16))
        return buf.value.decode()

    def set_option(self, name: str, value: int):
        """Context knobs of libhawk_b200 (hawk_b200_ctx_set_option): jit, prefetch_passes, ..."""
        st = _native.b200().hawk_b200_ctx_set_option(self.ctx, name.encode(), int(value))
        if st != 0:
            raise InvalidParams(f"option {name}={value}: status {st}")

    def explain(self, sql: str, config: str = "") -> str:
        buf = C.create_string_buffer(1 << 16)
        _check(self._lib.hawk_engine_explain(self._h, sql.encode(), config.encode(), buf, 1 << 16))
        return buf.value.decode()

    # ---- optimizer ----
    def measure(self, sqls: list[str], config: str, prune_ms: float = 1000.0, reps: int = 3) -> float:
        arr = (C.c_char_p * len(sqls))(*[s.encode() for s in sqls])
        ms = C.c_double()
        _check(self._lib.hawk_engine_measure(self._h, arr, len(sqls), config.encode(), prune_ms,
                                             reps, C.byref(ms)))
        return ms.value

    def explore(self, sqls: list[str], kind: str = "aggregation", fixed: str = "",
                prune_ms: float = 1000.0, reps: int = 1, csv_path: str | None = None) -> dict:
        """full_exploration of one pipeline kind's space (32 projection / 896
        aggregation variants), the other kind fixed; CSV trace to csv_path."""
        arr = (C.c_char_p * len(sqls))(*[s.encode() for s in sqls])
        buf = C.create_string_buffer(512)
        ms, ev = C.c_double(), C.c_int32()
        _check(self._lib.hawk_engine_explore(self._h, arr, len(sqls), 0 if kind == "projection" else 1,
                                             fixed.encode(), prune_ms, reps,
                                             csv_path.encode() if csv_path else None, buf, 512,
                                             C.byref(ms), C.byref(ev)))
        return dict(config=buf.value.decode(), ms=ms.value, evaluations=ev.value)

    def learn_ex(self, sqls: list[str], q: int = 3, early: bool = True, prune_ms: float = 1000.0,
                 reps: int = 3, unroll_pass: bool = True, starts: list[str] | None = None,
                 trace_csv: str | None = None, config_path: str | None = None) -> dict:
        """Algorithm 1 with the unroll pass, restarts, and the trace CSV /
        key-value config file outputs."""
        arr = (C.c_char_p * len(sqls))(*[s.encode() for s in sqls])
        buf = C.create_string_buffer(512)
        ms, ev, sw = C.c_double(), C.c_int32(), C.c_int32()
        _check(self._lib.hawk_engine_learn_ex(
            self._h, arr, len(sqls), q, int(early), prune_ms, reps, int(unroll_pass),
            "|".join(starts).encode() if starts else None, trace_csv.encode() if trace_csv else None,
            config_path.encode() if config_path else None, buf, 512, C.byref(ms), C.byref(ev),
            C.byref(sw)))
        return dict(config=buf.value.decode(), ms=ms.value, evaluations=ev.value, sweeps=sw.value)

    def learn(self, sqls: list[str], q: int = 3, prune_ms: float = 1000.0, reps: int = 3) -> dict:
        arr = (C.c_char_p * len(sqls))(*[s.encode() for s in sqls])
        buf = C.create_string_buffer(512)
        ms, ev, sw = C.c_double(), C.c_int32(), C.c_int32()
        _check(self._lib.hawk_engine_learn(self._h, arr, len(sqls), q, prune_ms, reps, buf, 512,
                                           C.byref(ms), C.byref(ev), C.byref(sw)))
        return dict(config=buf.value.decode(), ms=ms.value, evaluations=ev.value, sweeps=sw.value)


class Communicator:
    """An NCCL communicator on an engine's device (include/hawk_b200_comm.h).
    `unique_id` (128 bytes) comes from Communicator.unique_id() on one rank and
    is shipped to the others by the launcher (torch.distributed in bench.py)."""

    def __init__(self, engine: Engine, world: int, rank: int, unique_id: bytes):
        lib = _native.b200()
        if not lib.hawk_nccl_available():
            raise Unsupported("libnccl.so.2 is not available")
        self._lib = lib
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        st = lib.hawk_nccl_comm_create(engine.ctx, world, rank, buf, C.byref(h))
        if st != 0:
            raise HawkError(f"ncclCommInitRank failed: status {st}")
        self.handle = h
        self.world, self.rank = world, rank

    @classmethod
    def _adopt(cls, lib, handle, world: int, rank: int) -> "Communicator":
        c = cls.__new__(cls)
        c._lib, c.handle, c.world, c.rank = lib, handle, world, rank
        return c

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        st = _native.b200().hawk_nccl_unique_id(buf)
        if st != 0:
            raise HawkError(f"ncclGetUniqueId failed: status {st}")
        return bytes(buf)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.hawk_nccl_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """N ranks of this process on one device (include/hawk_b200_comm.h): each
    rank is an Engine driven from its own host thread, and the collectives of
    its communicator are device-to-device copies between the ranks' buffers,
    sequenced by host barriers. It runs the multi-rank exchange of
    Engine.run_sharded where only one GPU is present; the NCCL communicator
    is the production path."""

    def __init__(self, world: int):
        self._lib = _native.b200()
        h = C.c_void_p()
        if self._lib.hawk_loopback_group_create(world, C.byref(h)) != 0:
            raise HawkError("loopback group: bad rank count")
        self.handle, self.world = h, world

    def communicator(self, engine: "Engine", rank: int) -> Communicator:
        h = C.c_void_p()
        if self._lib.hawk_loopback_comm_create(engine.ctx, self.handle, rank, C.byref(h)) != 0:
            raise HawkError(f"loopback communicator: bad rank {rank}")
        return Communicator._adopt(self._lib, h, self.world, rank)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.hawk_loopback_group_destroy(self.handle)
            self.handle = None


def save_config(config: str, path: str):
    """Writes a workload configuration ("<proj>;<agg>") as the key-value
    learned-configuration file."""
    _check(_native.engine().hawk_config_save(config.encode(), path.encode()))


def load_config(path: str) -> str:
    buf = C.create_string_buffer(512)
    _check(_native.engine().hawk_config_load(path.encode(), buf, 512))
    return buf.value.decode()
