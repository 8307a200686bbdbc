// lower.cpp — pipeline-to-kernel lowering: a variant-applied
// hawk::PipelineProgram (ir/program.hpp:154-171) becomes the POD hawk_pipeline
// descriptor the sm_100a kernel family interprets. This replaces the
// reference's missing fragment generator / kernel assembler
// (proj/CMakeLists.txt:28-31): instead of emitting source per
// variant, the variant modes select a precompiled template instantiation and
// the per-query structure becomes kernel parameters.
//
// Value semantics mirror the oracle (proj/src/planner_reference.cpp):
//   comparisons int/int, double/double, string codes (:76-95)
//   int64 wrap, x/0 = 0, mixed -> double (:25-33, :106-141)
//   AVG = SUM + COUNT with host division (planner_pipelines.cpp:469-478)
#include <cstring>
#include <map>
#include <tuple>

#include "hawk_b200_engine.hpp"

namespace hawk::b200 {

namespace {

int type_of(ColumnKind k) { return k == ColumnKind::Float64 ? HAWK_F64 : HAWK_I64; }

struct Lowerer {
  const PipelineProgram& prog;
  const PipelineSet& set;
  LoweredProgram out;
  std::map<std::pair<int, int>, int> slot_of;       // (table, column) -> column slot
  std::map<int, int> probe_of_descriptor;           // descriptor -> device probe index
  std::map<int, int> reg_of_derived;                // derived id -> device register
  std::map<int, int> derived_type;                  // derived id -> HAWK_I64/F64

  Lowerer(const PipelineProgram& p, const PipelineSet& s) : prog(p), set(s) {}

  int column_slot(int table, int column) {
    auto key = std::make_pair(table, column);
    auto it = slot_of.find(key);
    if (it != slot_of.end()) return it->second;
    const int slot = static_cast<int>(out.column_of_slot.size());
    if (slot >= HAWK_MAX_COLUMNS) throw Unsupported("more than 32 distinct columns in a pipeline");
    out.column_of_slot.push_back(key);
    slot_of[key] = slot;
    return slot;
  }

  hawk_operand attr(const OpAttr& a) {
    hawk_operand o{};
    o.type = type_of(a.kind);
    switch (a.route) {
      case AttrRoute::Driver:
        o.kind = HAWK_OPND_COLUMN;
        o.index = column_slot(a.table, a.column);
        break;
      case AttrRoute::BuildPayload: {
        auto it = probe_of_descriptor.find(a.descriptor);
        if (it == probe_of_descriptor.end())
          throw UnsupportedPlan("payload attribute '" + a.name + "' used before its probe");
        o.kind = HAWK_OPND_PAYLOAD;
        o.index = column_slot(a.table, a.column);
        o.probe = it->second;
        break;
      }
      case AttrRoute::Derived: {
        auto it = reg_of_derived.find(a.column);
        if (it == reg_of_derived.end()) throw UnsupportedPlan("derived register used before definition");
        o.kind = HAWK_OPND_REG;
        o.index = it->second;
        o.type = derived_type.at(a.column);
        break;
      }
      case AttrRoute::CrossAux:
        throw Unsupported("CROSS_JOIN auxiliary attributes are not supported by the B200 executor");
    }
    return o;
  }

  hawk_operand operand(const OpOperand& x) {
    hawk_operand o{};
    switch (x.kind) {
      case OpOperand::Kind::Attr: return attr(x.attr);
      case OpOperand::Kind::IntLit:
        o.kind = HAWK_OPND_INT;
        o.type = HAWK_I64;
        o.bits = x.ival;
        return o;
      case OpOperand::Kind::FloatLit: {
        o.kind = HAWK_OPND_FLOAT;
        o.type = HAWK_F64;
        std::memcpy(&o.bits, &x.fval, 8);
        return o;
      }
    }
    return o;
  }

  static bool same(const hawk_operand& a, const hawk_operand& b) {
    return a.kind == b.kind && a.type == b.type && a.index == b.index && a.probe == b.probe &&
           a.bits == b.bits;
  }

  hawk_compare compare(const OpComparison& c) {
    hawk_compare h{};
    h.op = static_cast<int32_t>(c.op);
    h.lhs = attr(c.lhs);
    h.rhs = operand(c.rhs);
    // both sides compared in one domain: double if either is double
    h.type = (h.lhs.type == HAWK_F64 || h.rhs.type == HAWK_F64) ? HAWK_F64 : HAWK_I64;
    return h;
  }

  void run() {
    hawk_pipeline& p = out.pipe;
    std::memset(&p, 0, sizeof p);
    p.sink = -1;
    if (prog.ops.empty() || prog.ops.front().kind != PipelineOpKind::Loop)
      throw UnsupportedPlan("pipeline must start with LOOP");
    out.unroll = prog.unroll_factor;
    bool seen_probe = false;
    for (std::size_t i = 1; i < prog.ops.size(); ++i) {
      const PipelineOp& op = prog.ops[i];
      if (op.offset != 0) continue;  // unrolled replicas: the kernel's U template covers them
      if (p.sink >= 0 && op.kind != PipelineOpKind::Project)
        throw UnsupportedPlan(std::string("op after the pipeline sink: ") + to_string(op.kind));
      switch (op.kind) {
        case PipelineOpKind::Loop: throw UnsupportedPlan("nested LOOP");
        case PipelineOpKind::Filter:
          for (const OpComparison& c : op.predicate) {
            if (seen_probe || p.narith > 0) {
              if (p.narith > 0) throw Unsupported("FILTER after ARITHMETIC");
              if (p.npost >= HAWK_MAX_FILTERS) throw Unsupported("too many filter conjuncts");
              p.post[p.npost++] = compare(c);
            } else {
              if (p.nfilter >= HAWK_MAX_FILTERS) throw Unsupported("too many filter conjuncts");
              p.filter[p.nfilter++] = compare(c);
            }
          }
          break;
        case PipelineOpKind::HashProbe: {
          if (p.narith > 0) throw Unsupported("HASH_PROBE after ARITHMETIC");
          if (p.nprobe >= HAWK_MAX_PROBES) throw Unsupported("more than 4 probes in a pipeline");
          if (op.keys.size() != 1) throw Unsupported("composite join keys");
          hawk_probe pr{};
          pr.key = attr(op.keys[0]);
          pr.table = p.nprobe;
          probe_of_descriptor[op.descriptor] = p.nprobe;
          out.probe_descriptor.push_back(op.descriptor);
          p.probe[p.nprobe++] = pr;
          seen_probe = true;
          break;
        }
        case PipelineOpKind::CrossJoin:
          throw Unsupported("CROSS_JOIN is not supported by the B200 executor");
        case PipelineOpKind::Arithmetic: {
          hawk_arith a{};
          a.op = static_cast<int32_t>(op.arith_op);
          a.type = type_of(op.derived_kind);
          a.lhs = operand(op.arith_lhs);
          a.rhs = operand(op.arith_rhs);
          // value numbering: the reference lowering emits no CSE
          // (planner_pipelines.cpp:401-432); identical ops share a register
          int reg = -1;
          for (int r = 0; r < p.narith; ++r)
            if (p.arith[r].op == a.op && p.arith[r].type == a.type && same(p.arith[r].lhs, a.lhs) &&
                same(p.arith[r].rhs, a.rhs))
              reg = r;
          if (reg < 0) {
            if (p.narith >= HAWK_MAX_ARITH) throw Unsupported("more than 8 arithmetic registers");
            reg = p.narith;
            p.arith[p.narith++] = a;
          }
          reg_of_derived[op.derived_id] = reg;
          derived_type[op.derived_id] = a.type;
          break;
        }
        case PipelineOpKind::Aggregate:
        case PipelineOpKind::HashAggregate: {
          p.sink = op.kind == PipelineOpKind::Aggregate ? HAWK_SINK_AGGREGATE : HAWK_SINK_HASH_AGGREGATE;
          for (const OpAttr& k : op.keys) {
            if (p.nkeys >= HAWK_MAX_KEYS) throw Unsupported("more than 4 group keys");
            hawk_operand o = attr(k);
            if (o.type != HAWK_I64) throw Unsupported("float group keys");
            p.keys[p.nkeys++] = o;
          }
          for (const OpAggregate& g : op.aggregates) {
            hawk_agg a{};
            a.fn = static_cast<int32_t>(g.fn);
            a.type = g.fn == AggFunction::Count ? HAWK_I64 : type_of(g.out_kind);
            if (g.fn != AggFunction::Count) a.input = operand(g.input);
            else a.input = hawk_operand{HAWK_OPND_INT, HAWK_I64, 0, 0, 1};
            int slot = -1;
            for (int k = 0; k < p.naggs; ++k)
              if (p.aggs[k].fn == a.fn && p.aggs[k].type == a.type &&
                  (a.fn == HAWK_COUNT || same(p.aggs[k].input, a.input)))
                slot = k;
            if (slot < 0) {
              if (p.naggs >= HAWK_MAX_AGGS) throw Unsupported("more than 16 aggregates");
              slot = p.naggs;
              p.aggs[p.naggs++] = a;
            }
            out.agg_slot.push_back(slot);
            if (a.fn == HAWK_COUNT) out.count_agg = slot;
          }
          break;
        }
        case PipelineOpKind::Project:
          if (p.sink == HAWK_SINK_HASH_PUT) break;  // build-side payload: fetched by row id
          p.sink = HAWK_SINK_PROJECT;
          for (const OpAttr& a : op.attrs) {
            if (p.nproject >= HAWK_MAX_PROJECT) throw Unsupported("more than 16 projected attributes");
            p.project[p.nproject++] = attr(a);
          }
          break;
        case PipelineOpKind::HashPut:
          if (op.keys.size() != 1) throw Unsupported("composite join keys");
          p.sink = HAWK_SINK_HASH_PUT;
          p.keys[0] = attr(op.keys[0]);
          p.nkeys = 1;
          break;
      }
    }
    if (p.sink < 0) throw UnsupportedPlan("pipeline has no sink");
    // the non-grouped sink needs a row count for the empty-input rule
    // (planner_reference.cpp:269-278); the reference adds a hidden .rows
    if (p.sink == HAWK_SINK_AGGREGATE && out.count_agg < 0) {
      if (p.naggs >= HAWK_MAX_AGGS) throw Unsupported("more than 16 aggregates");
      out.count_agg = p.naggs;
      p.aggs[p.naggs++] = hawk_agg{HAWK_COUNT, HAWK_I64, hawk_operand{HAWK_OPND_INT, HAWK_I64, 0, 0, 1}};
    }
    p.ncolumns = static_cast<int32_t>(out.column_of_slot.size());
  }
};

}  // namespace

std::string describe(const hawk_pipeline& p) {
  static const char* kinds[] = {"col", "payload", "reg", "int", "float", "?", "?", "rowid"};
  static const char* cmps[] = {"<", "<=", "=", ">=", ">", "<>"};
  static const char* ariths[] = {"+", "-", "*", "/"};
  static const char* fns[] = {"sum", "count", "min", "max"};
  static const char* sinks[] = {"AGGREGATE", "HASH_AGGREGATE", "PROJECT", "HASH_PUT"};
  auto opnd = [&](const hawk_operand& o) {
    std::string s = kinds[o.kind & 7];
    if (o.kind == HAWK_OPND_INT) return s + "(" + std::to_string(o.bits) + ")";
    s += "(" + std::to_string(o.index);
    if (o.kind == HAWK_OPND_PAYLOAD) s += "@p" + std::to_string(o.probe);
    return s + (o.type == HAWK_F64 ? ":f64)" : ")");
  };
  std::string out;
  for (int i = 0; i < p.nfilter; ++i)
    out += std::string("FILTER ") + opnd(p.filter[i].lhs) + " " + cmps[p.filter[i].op] + " " + opnd(p.filter[i].rhs) + "\n";
  for (int i = 0; i < p.nprobe; ++i) out += "PROBE t" + std::to_string(p.probe[i].table) + " key " + opnd(p.probe[i].key) + "\n";
  for (int i = 0; i < p.npost; ++i)
    out += std::string("POST ") + opnd(p.post[i].lhs) + " " + cmps[p.post[i].op] + " " + opnd(p.post[i].rhs) + "\n";
  for (int i = 0; i < p.narith; ++i)
    out += "ARITH r" + std::to_string(i) + " = " + opnd(p.arith[i].lhs) + " " + ariths[p.arith[i].op] + " " + opnd(p.arith[i].rhs) + "\n";
  out += std::string("SINK ") + (p.sink >= 0 && p.sink < 4 ? sinks[p.sink] : "?") + "\n";
  for (int i = 0; i < p.nkeys; ++i) out += "KEY " + opnd(p.keys[i]) + "\n";
  for (int i = 0; i < p.naggs; ++i) out += std::string("AGG ") + fns[p.aggs[i].fn] + " " + opnd(p.aggs[i].input) + "\n";
  for (int i = 0; i < p.nproject; ++i) out += "OUT " + opnd(p.project[i]) + "\n";
  return out;
}

void reorder_probes(LoweredProgram& lp, const std::vector<double>& match_prob) {
  hawk_pipeline& p = lp.pipe;
  const int n = p.nprobe;
  if (n < 2 || static_cast<int>(match_prob.size()) != n) return;
  // greedy: the most selective probe whose key is available goes next
  std::vector<int> perm, inv(static_cast<std::size_t>(n), -1);
  std::vector<bool> placed(static_cast<std::size_t>(n), false);
  for (int k = 0; k < n; ++k) {
    int best = -1;
    for (int i = 0; i < n; ++i) {
      if (placed[static_cast<std::size_t>(i)]) continue;
      const hawk_operand& key = p.probe[i].key;
      if (key.kind == HAWK_OPND_PAYLOAD && !placed[static_cast<std::size_t>(key.probe)]) continue;
      if (best < 0 || match_prob[static_cast<std::size_t>(i)] < match_prob[static_cast<std::size_t>(best)])
        best = i;
    }
    if (best < 0) return;  // cyclic payload keys: keep the lowering's order
    placed[static_cast<std::size_t>(best)] = true;
    inv[static_cast<std::size_t>(best)] = k;
    perm.push_back(best);
  }
  auto remap = [&](hawk_operand& o) {
    if (o.kind == HAWK_OPND_PAYLOAD) o.probe = inv[static_cast<std::size_t>(o.probe)];
  };
  hawk_probe old[HAWK_MAX_PROBES];
  std::vector<int> old_desc = lp.probe_descriptor;
  for (int i = 0; i < n; ++i) old[i] = p.probe[i];
  for (int k = 0; k < n; ++k) {
    p.probe[k] = old[perm[static_cast<std::size_t>(k)]];
    p.probe[k].table = k;
    remap(p.probe[k].key);
    lp.probe_descriptor[static_cast<std::size_t>(k)] = old_desc[static_cast<std::size_t>(perm[static_cast<std::size_t>(k)])];
  }
  for (int i = 0; i < p.nfilter; ++i) remap(p.filter[i].lhs), remap(p.filter[i].rhs);
  for (int i = 0; i < p.npost; ++i) remap(p.post[i].lhs), remap(p.post[i].rhs);
  for (int i = 0; i < p.narith; ++i) remap(p.arith[i].lhs), remap(p.arith[i].rhs);
  for (int i = 0; i < p.nkeys; ++i) remap(p.keys[i]);
  for (int i = 0; i < p.naggs; ++i) remap(p.aggs[i].input);
  for (int i = 0; i < p.nproject; ++i) remap(p.project[i]);
}

// A probe is a pure semi-join when no operand of the program reads its build
// payload (TPC-H/SSB filter joins such as SSB Q4.1's supplier and part).
static void mark_filter_only_probes(hawk_pipeline& p) {
  bool used[HAWK_MAX_PROBES] = {};
  auto see = [&](const hawk_operand& o) {
    if (o.kind == HAWK_OPND_PAYLOAD && o.probe >= 0 && o.probe < HAWK_MAX_PROBES) used[o.probe] = true;
  };
  for (int i = 0; i < p.nprobe; ++i) see(p.probe[i].key);
  for (int i = 0; i < p.npost; ++i) see(p.post[i].lhs), see(p.post[i].rhs);
  for (int i = 0; i < p.nfilter; ++i) see(p.filter[i].lhs), see(p.filter[i].rhs);
  for (int i = 0; i < p.narith; ++i) see(p.arith[i].lhs), see(p.arith[i].rhs);
  for (int i = 0; i < p.nkeys; ++i) see(p.keys[i]);
  for (int i = 0; i < p.naggs; ++i) see(p.aggs[i].input);
  for (int i = 0; i < p.nproject; ++i) see(p.project[i]);
  for (int i = 0; i < p.nprobe; ++i) p.probe[i].filter_only = used[i] ? 0 : 1;
}

LoweredProgram lower_program(const PipelineProgram& program, const PipelineSet& set) {
  Lowerer l(program, set);
  l.run();
  mark_filter_only_probes(l.out.pipe);
  return l.out;
}

}  // namespace hawk::b200
