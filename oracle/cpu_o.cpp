// TEST INFRASTRUCTURE / CPU BASELINE — never linked into the product.
//
// The reference's CPU variant: a host-parallel executor of the reference's
// own pipeline programs (PipelineSet from partition_into_pipelines,
// /root/reference/proj/src/planner_pipelines.cpp) under the configuration
// the paper learned for CPUs, "cpu-o":
//   single-pass projection (each worker appends to its own output region),
//   local hash tables for aggregation (one per worker, merged at the end),
//   sequential memory access (each worker scans one contiguous row range),
//   linear probing with murmur hashing for joins and groups,
//   branched predication, thread multiplier 1 (one worker per hardware
//   thread; host mode).
// The reference snapshot does not contain this executor (its runtime and
// codegen sources are missing, proj/CMakeLists.txt:24-39); this restates it
// from the IR semantics, and its results are checked against
// reference_execute (tests/test_oracle.py). Value semantics follow
// planner_reference.cpp: int64 wrap (:25-33), x/0 = 0 (:135), int -> double
// promotion (:114-128), SUM/COUNT/MIN/MAX/AVG and the empty-input rules
// (:233-308).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "hawk/error.hpp"
#include "hawk/planner/pipelines.hpp"
#include "hawk/sql/parser.hpp"

namespace hawk::cpu_o {

namespace {

using u64 = uint64_t;

u64 fmix64(u64 k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

int64_t wadd(int64_t a, int64_t b) { return static_cast<int64_t>(static_cast<u64>(a) + static_cast<u64>(b)); }
int64_t wsub(int64_t a, int64_t b) { return static_cast<int64_t>(static_cast<u64>(a) - static_cast<u64>(b)); }
int64_t wmul(int64_t a, int64_t b) { return static_cast<int64_t>(static_cast<u64>(a) * static_cast<u64>(b)); }

struct Val {
  bool f = false;  // double
  int64_t i = 0;
  double d = 0;
  double as_double() const { return f ? d : static_cast<double>(i); }
  u64 bits() const {
    if (!f) return static_cast<u64>(i);
    u64 b;
    std::memcpy(&b, &d, 8);
    return b;
  }
};

constexpr int64_t kEmpty = std::numeric_limits<int64_t>::min();

// linear probing, murmur: the join table of one descriptor (build row ids)
struct JoinTable {
  u64 mask = 0, seed = 0;
  std::unique_ptr<std::atomic<int64_t>[]> keys;
  std::unique_ptr<int64_t[]> rows;
  std::atomic<bool> duplicate{false};
  void init(int64_t build_rows, u64 s) {
    u64 cap = 16;
    while (cap < 2 * static_cast<u64>(std::max<int64_t>(build_rows, 1))) cap <<= 1;
    mask = cap - 1;
    seed = s;
    keys.reset(new std::atomic<int64_t>[cap]);
    rows.reset(new int64_t[cap]);
    for (u64 i = 0; i < cap; ++i) keys[i].store(kEmpty, std::memory_order_relaxed);
  }
  void insert(int64_t key, int64_t row) {
    u64 i = fmix64(static_cast<u64>(key) ^ seed) & mask;
    for (;;) {
      int64_t expect = kEmpty;
      if (keys[i].compare_exchange_strong(expect, key, std::memory_order_acq_rel)) {
        rows[i] = row;
        return;
      }
      if (expect == key) {
        duplicate = true;
        return;
      }
      i = (i + 1) & mask;
    }
  }
  int64_t find(int64_t key) const {
    if (key == kEmpty) return -1;
    u64 i = fmix64(static_cast<u64>(key) ^ seed) & mask;
    for (;;) {
      const int64_t k = keys[i].load(std::memory_order_relaxed);
      if (k == key) return rows[i];
      if (k == kEmpty) return -1;
      i = (i + 1) & mask;
    }
  }
};

struct Acc {
  int64_t isum = 0, count = 0, imin = std::numeric_limits<int64_t>::max(),
          imax = std::numeric_limits<int64_t>::min();
  double fsum = 0, fmin = HUGE_VAL, fmax = -HUGE_VAL;
  bool is_float = false;
  void add(const Val& v) {
    ++count;
    if (v.f) {
      is_float = true;
      fsum += v.d;
      fmin = std::min(fmin, v.d);
      fmax = std::max(fmax, v.d);
    } else {
      isum = wadd(isum, v.i);
      imin = std::min(imin, v.i);
      imax = std::max(imax, v.i);
    }
  }
  void merge(const Acc& o) {
    count += o.count;
    is_float |= o.is_float;
    isum = wadd(isum, o.isum);
    fsum += o.fsum;
    imin = std::min(imin, o.imin);
    imax = std::max(imax, o.imax);
    fmin = std::min(fmin, o.fmin);
    fmax = std::max(fmax, o.fmax);
  }
};

// a worker's local hash table of groups (linear probing, murmur of the
// combined key bits)
struct GroupTable {
  int nkeys = 0, naggs = 0;
  u64 mask = 0, seed = 0;
  std::vector<uint8_t> used;
  std::vector<u64> keys;
  std::vector<Val> keyvals;
  std::vector<Acc> accs;
  std::size_t groups = 0;
  void init(int k, int a, u64 s, u64 cap = 1024) {
    nkeys = k;
    naggs = a;
    seed = s;
    mask = cap - 1;
    used.assign(cap, 0);
    keys.assign(cap * static_cast<u64>(k), 0);
    keyvals.assign(cap * static_cast<u64>(k), Val{});
    accs.assign(cap * static_cast<u64>(a), Acc{});
    groups = 0;
  }
  u64 hash(const u64* k) const {
    u64 h = seed;
    for (int i = 0; i < nkeys; ++i) h = fmix64(h ^ k[i]) + 0x9e3779b97f4a7c15ull;
    return h;
  }
  Acc* find_or_insert(const u64* k, const Val* kv) {
    if ((groups + 1) * 2 > mask + 1) grow();
    u64 i = hash(k) & mask;
    for (;;) {
      if (!used[i]) {
        used[i] = 1;
        for (int j = 0; j < nkeys; ++j) {
          keys[i * nkeys + j] = k[j];
          keyvals[i * nkeys + j] = kv[j];
        }
        ++groups;
        return &accs[i * naggs];
      }
      bool eq = true;
      for (int j = 0; j < nkeys; ++j) eq &= keys[i * nkeys + j] == k[j];
      if (eq) return &accs[i * naggs];
      i = (i + 1) & mask;
    }
  }
  void grow() {
    GroupTable g;
    g.init(nkeys, naggs, seed, (mask + 1) * 2);
    for (u64 i = 0; i <= mask; ++i)
      if (used[i]) {
        Acc* a = g.find_or_insert(&keys[i * nkeys], &keyvals[i * nkeys]);
        for (int j = 0; j < naggs; ++j) a[j] = accs[i * naggs + j];
      }
    *this = std::move(g);
  }
};

class Executor {
 public:
  Executor(const PipelineSet& set, int threads) : set_(set), T_(std::max(1, threads)) {
    joins_.resize(set.descriptors.size());
  }

  Table run() {
    for (std::size_t p = 0; p < set_.pipelines.size(); ++p)
      if (static_cast<int>(p) != set_.terminal) build(set_.pipelines[p]);
    return terminal(set_.pipelines.at(static_cast<std::size_t>(set_.terminal)));
  }

 private:
  struct Worker {
    int64_t driver = 0;
    std::vector<int64_t> rid, aux;
    std::vector<Val> regs;
    std::vector<Acc> accs;
    GroupTable groups;
    std::vector<std::vector<Val>> rows;  // PROJECT output
  };

  const Table& table(int id) const { return *set_.tables.at(static_cast<std::size_t>(id)); }

  Val load(const Worker& w, const OpAttr& a) const {
    Val v;
    if (a.route == AttrRoute::Derived) return w.regs.at(static_cast<std::size_t>(a.column));
    int64_t row = w.driver;
    if (a.route == AttrRoute::BuildPayload) row = w.rid.at(static_cast<std::size_t>(a.descriptor));
    if (a.route == AttrRoute::CrossAux) row = w.aux.at(static_cast<std::size_t>(a.aux_op));
    const Column& c = table(a.table).column(static_cast<std::size_t>(a.column));
    if (c.kind() == ColumnKind::Float64) {
      v.f = true;
      v.d = c.floats()[static_cast<std::size_t>(row)];
    } else {
      v.i = c.ints()[static_cast<std::size_t>(row)];
    }
    return v;
  }

  Val operand(const Worker& w, const OpOperand& o) const {
    Val v;
    switch (o.kind) {
      case OpOperand::Kind::Attr: return load(w, o.attr);
      case OpOperand::Kind::IntLit: v.i = o.ival; return v;
      case OpOperand::Kind::FloatLit: v.f = true; v.d = o.fval; return v;
    }
    return v;
  }

  static bool compare(const Val& a, CompareOp op, const Val& b) {
    auto apply = [&](auto x, auto y) {
      switch (op) {
        case CompareOp::Lt: return x < y;
        case CompareOp::Le: return x <= y;
        case CompareOp::Eq: return x == y;
        case CompareOp::Ge: return x >= y;
        case CompareOp::Gt: return x > y;
        case CompareOp::Ne: return x != y;
      }
      return false;
    };
    if (a.f || b.f) return apply(a.as_double(), b.as_double());
    return apply(a.i, b.i);
  }

  static Val arith(ArithOp op, const Val& a, const Val& b) {
    Val r;
    if (a.f || b.f) {
      r.f = true;
      const double x = a.as_double(), y = b.as_double();
      r.d = op == ArithOp::Add ? x + y : op == ArithOp::Sub ? x - y : op == ArithOp::Mul ? x * y : x / y;
      return r;
    }
    switch (op) {
      case ArithOp::Add: r.i = wadd(a.i, b.i); break;
      case ArithOp::Sub: r.i = wsub(a.i, b.i); break;
      case ArithOp::Mul: r.i = wmul(a.i, b.i); break;
      case ArithOp::Div: r.i = b.i == 0 ? 0 : a.i / b.i; break;  // x/0 = 0
    }
    return r;
  }

  void prepare(Worker& w, const PipelineProgram& p) const {
    w.rid.assign(set_.descriptors.size(), -1);
    w.aux.assign(p.ops.size(), -1);
    int regs = 0;
    for (const PipelineOp& op : p.ops)
      if (op.kind == PipelineOpKind::Arithmetic) regs = std::max(regs, op.derived_id + 1);
    w.regs.assign(static_cast<std::size_t>(regs), Val{});
  }

  // the op chain from op k on for the worker's current row (branched: a
  // failing FILTER or a missing probe key ends the row)
  template <class Sink>
  void chain(Worker& w, const PipelineProgram& p, std::size_t k, Sink& sink) {
    for (; k < p.ops.size(); ++k) {
      const PipelineOp& op = p.ops[k];
      switch (op.kind) {
        case PipelineOpKind::Loop: break;
        case PipelineOpKind::Filter:
          for (const OpComparison& c : op.predicate)
            if (!compare(load(w, c.lhs), c.op, operand(w, c.rhs))) return;
          break;
        case PipelineOpKind::HashProbe: {
          const int64_t rid = joins_.at(static_cast<std::size_t>(op.descriptor))->find(load(w, op.keys.at(0)).i);
          if (rid < 0) return;
          w.rid[static_cast<std::size_t>(op.descriptor)] = rid;
          break;
        }
        case PipelineOpKind::CrossJoin: {
          const int64_t n = static_cast<int64_t>(table(op.table).row_count());
          for (int64_t a = 0; a < n; ++a) {
            w.aux[k] = a;
            chain(w, p, k + 1, sink);
          }
          return;
        }
        case PipelineOpKind::Arithmetic:
          w.regs[static_cast<std::size_t>(op.derived_id)] = arith(op.arith_op, operand(w, op.arith_lhs),
                                                                  operand(w, op.arith_rhs));
          break;
        default:
          sink(w, op);
          return;
      }
    }
  }

  template <class F>
  void parallel(int64_t n, F&& f) {
    std::vector<std::thread> pool;
    const int64_t chunk = (n + T_ - 1) / T_;
    for (int t = 0; t < T_; ++t)
      pool.emplace_back([&, t] { f(t, std::min(n, t * chunk), std::min(n, (t + 1) * chunk)); });
    for (std::thread& th : pool) th.join();
  }

  void build(const PipelineProgram& p) {
    const PipelineOp* put = nullptr;
    for (const PipelineOp& op : p.ops)
      if (op.kind == PipelineOpKind::HashPut) put = &op;
    if (!put) throw UnsupportedPlan("build pipeline without HASH_PUT");
    const HashTableDescriptor& d = set_.descriptors.at(static_cast<std::size_t>(put->descriptor));
    auto jt = std::make_unique<JoinTable>();
    const int64_t n = static_cast<int64_t>(table(p.driver_table).row_count());
    jt->init(n, d.seed);
    JoinTable* t = jt.get();
    joins_[static_cast<std::size_t>(put->descriptor)] = std::move(jt);
    parallel(n, [&](int, int64_t b, int64_t e) {
      Worker w;
      prepare(w, p);
      auto sink = [&](Worker& ww, const PipelineOp& op) {
        if (op.kind == PipelineOpKind::HashPut) t->insert(load(ww, op.keys.at(0)).i, ww.driver);
      };
      for (int64_t r = b; r < e; ++r) {
        w.driver = r;
        chain(w, p, 1, sink);
      }
    });
    if (t->duplicate)
      throw DuplicateKey("duplicate join build key (join build sides must be key-unique)");
  }

  Table terminal(const PipelineProgram& p) {
    const PipelineOp& last = p.ops.back();
    const int64_t n = static_cast<int64_t>(table(p.driver_table).row_count());
    const int naggs = static_cast<int>(last.aggregates.size());
    std::vector<Worker> workers(static_cast<std::size_t>(T_));
    parallel(n, [&](int t, int64_t b, int64_t e) {
      Worker& w = workers[static_cast<std::size_t>(t)];
      prepare(w, p);
      w.accs.assign(static_cast<std::size_t>(naggs), Acc{});
      if (last.kind == PipelineOpKind::HashAggregate)
        w.groups.init(static_cast<int>(last.keys.size()), naggs, 0x6a09e667f3bcc909ull);
      std::vector<u64> kb(last.keys.size());
      std::vector<Val> kv(last.keys.size());
      auto sink = [&](Worker& ww, const PipelineOp& op) {
        Acc* acc = ww.accs.data();
        if (op.kind == PipelineOpKind::HashAggregate) {
          for (std::size_t i = 0; i < op.keys.size(); ++i) {
            kv[i] = load(ww, op.keys[i]);
            kb[i] = kv[i].bits();
          }
          acc = ww.groups.find_or_insert(kb.data(), kv.data());
        } else if (op.kind == PipelineOpKind::Project) {
          std::vector<Val> row;
          for (const OpAttr& a : op.attrs) row.push_back(load(ww, a));
          ww.rows.push_back(std::move(row));
          return;
        }
        for (int a = 0; a < naggs; ++a) {
          const OpAggregate& g = op.aggregates[static_cast<std::size_t>(a)];
          if (g.fn == AggFunction::Count) ++acc[a].count;
          else acc[a].add(operand(ww, g.input));
        }
      };
      for (int64_t r = b; r < e; ++r) {
        w.driver = r;
        chain(w, p, 1, sink);
      }
    });
    return materialise(p, workers);
  }

  Value out_value(const OutputColumn& oc, const Val& v) const {
    if (oc.kind == ColumnKind::String)
      return table(oc.lexicon_table).column(static_cast<std::size_t>(oc.lexicon_column)).decode(v.i);
    if (oc.kind == ColumnKind::Float64) return v.as_double();
    return v.i;
  }

  static Val acc_value(const OpAggregate& g, const Acc& a) {
    Val v;
    const bool f = g.out_kind == ColumnKind::Float64;
    v.f = f;
    switch (g.fn) {
      case AggFunction::Sum: f ? v.d = a.fsum : v.i = a.isum; break;
      case AggFunction::Count: v.f = false; v.i = a.count; break;
      case AggFunction::Min: f ? v.d = a.fmin : v.i = a.imin; break;
      case AggFunction::Max: f ? v.d = a.fmax : v.i = a.imax; break;
    }
    return v;
  }

  Table materialise(const PipelineProgram& p, std::vector<Worker>& workers) const {
    Schema schema;
    for (const OutputColumn& oc : p.output) schema.push_back({oc.name, oc.kind});
    Table out("result", schema);
    const PipelineOp& last = p.ops.back();
    Row row;
    auto emit = [&](const Val* keys, const Acc* accs) {
      row.clear();
      for (const OutputColumn& oc : p.output) {
        switch (oc.source) {
          case OutputColumn::Source::ProjectAttr:
          case OutputColumn::Source::GroupKey:
            row.push_back(out_value(oc, keys[oc.index]));
            break;
          case OutputColumn::Source::Aggregate:
            row.push_back(out_value(oc, acc_value(last.aggregates[static_cast<std::size_t>(oc.index)], accs[oc.index])));
            break;
          case OutputColumn::Source::AvgDivide: {
            const Acc& s = accs[oc.index];
            const double sum = last.aggregates[static_cast<std::size_t>(oc.index)].out_kind == ColumnKind::Float64
                                   ? s.fsum
                                   : static_cast<double>(s.isum);
            row.emplace_back(sum / static_cast<double>(accs[oc.index2].count));
            break;
          }
        }
      }
      out.append_row(row);
    };
    if (last.kind == PipelineOpKind::Project) {
      for (Worker& w : workers)
        for (const std::vector<Val>& r : w.rows) emit(r.data(), nullptr);
    } else if (last.kind == PipelineOpKind::Aggregate) {
      std::vector<Acc> total(last.aggregates.size());
      for (Worker& w : workers)
        for (std::size_t a = 0; a < total.size(); ++a) total[a].merge(w.accs[a]);
      int64_t rows = 0;
      for (std::size_t a = 0; a < total.size(); ++a)
        if (last.aggregates[a].fn == AggFunction::Count) rows = total[a].count;
      if (rows == 0)
        for (const OutputColumn& oc : p.output)
          if (oc.source == OutputColumn::Source::AvgDivide ||
              (oc.source == OutputColumn::Source::Aggregate &&
               (last.aggregates[static_cast<std::size_t>(oc.index)].fn == AggFunction::Min ||
                last.aggregates[static_cast<std::size_t>(oc.index)].fn == AggFunction::Max)))
            throw EmptyAggregate("aggregate over empty input has no value");
      emit(nullptr, total.data());
    } else {  // merge the workers' local tables in worker order
      GroupTable all;
      all.init(static_cast<int>(last.keys.size()), static_cast<int>(last.aggregates.size()), 0x6a09e667f3bcc909ull);
      for (Worker& w : workers)
        for (u64 i = 0; i <= w.groups.mask; ++i)
          if (!w.groups.used.empty() && w.groups.used[i]) {
            Acc* a = all.find_or_insert(&w.groups.keys[i * w.groups.nkeys], &w.groups.keyvals[i * w.groups.nkeys]);
            for (int j = 0; j < all.naggs; ++j) a[j].merge(w.groups.accs[i * all.naggs + j]);
          }
      for (u64 i = 0; i <= all.mask; ++i)
        if (all.used[i]) emit(&all.keyvals[i * all.nkeys], &all.accs[i * all.naggs]);
    }
    out.finalize();
    return out;
  }

  const PipelineSet& set_;
  const int T_;
  std::vector<std::unique_ptr<JoinTable>> joins_;
};

}  // namespace

Table execute(const std::string& sql, const std::vector<TablePtr>& tables, int threads) {
  const PipelineSet set = partition_into_pipelines(sql::parse_query(sql, sql::make_catalog(tables)), tables);
  return Executor(set, threads).run();
}

}  // namespace hawk::cpu_o
