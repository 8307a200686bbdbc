// space.cpp — variant space enumeration,
// program validation, variant text formats.
#include <sstream>

#include "hawk_b200_engine.hpp"

namespace hawk::b200 {

namespace {

constexpr MemoryAccess kAccess[] = {MemoryAccess::Sequential, MemoryAccess::Coalesced};
constexpr PredicationMode kPred[] = {PredicationMode::Branched, PredicationMode::Predicated};
constexpr HashTableImpl kImpl[] = {HashTableImpl::LinearProbing, HashTableImpl::Cuckoo};
constexpr HashFunctionKind kFn[] = {HashFunctionKind::Murmur, HashFunctionKind::MultiplyShift};

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == sep) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += c;
    }
  }
  out.push_back(cur);
  return out;
}

}  // namespace

WorkloadConfig::WorkloadConfig() {
  projection.strategy = Strategy::SinglePass;
  aggregation.strategy = Strategy::LocalHash;
}

std::string WorkloadConfig::to_string() const {
  return projection.to_string() + ";" + aggregation.to_string();
}

VariantConfiguration parse_variant(const std::string& text) {
  VariantConfiguration c;
  auto parts = split(text, '/');
  if (parts.size() < 3) throw InvalidConfig("variant '" + text + "': expected strategy/access/predication");
  const std::string& s = parts[0];
  if (s == "single_pass") c.strategy = Strategy::SinglePass;
  else if (s == "multi_pass") c.strategy = Strategy::MultiPass;
  else if (s == "local_hash") c.strategy = Strategy::LocalHash;
  else if (s == "global_hash") c.strategy = Strategy::GlobalHash;
  else throw InvalidConfig("unknown strategy '" + s + "'");
  if (parts[1] == "sequential") c.memory_access = MemoryAccess::Sequential;
  else if (parts[1] == "coalesced") c.memory_access = MemoryAccess::Coalesced;
  else throw InvalidConfig("unknown memory access '" + parts[1] + "'");
  if (parts[2] == "branched") c.predication = PredicationMode::Branched;
  else if (parts[2] == "predicated") c.predication = PredicationMode::Predicated;
  else throw InvalidConfig("unknown predication '" + parts[2] + "'");
  for (std::size_t i = 3; i < parts.size(); ++i) {
    const std::string& p = parts[i];
    if (p == "linear_probing") c.hash_table_impl = HashTableImpl::LinearProbing;
    else if (p == "cuckoo") c.hash_table_impl = HashTableImpl::Cuckoo;
    else if (p == "murmur") c.hash_function = HashFunctionKind::Murmur;
    else if (p == "multiply_shift") c.hash_function = HashFunctionKind::MultiplyShift;
    else if (p.rfind("tm=", 0) == 0) c.thread_multiplier = std::stoi(p.substr(3));
    else if (p.rfind("wg=", 0) == 0) c.work_group_size = std::stoi(p.substr(3));
    else if (p.rfind("ht=", 0) == 0) c.hash_table_count_multiplier = std::stoi(p.substr(3));
    else if (p.rfind("u=", 0) == 0) c.unroll_factor = std::stoi(p.substr(2));
    else throw InvalidConfig("unknown variant field '" + p + "'");
  }
  return c;
}

WorkloadConfig parse_workload_config(const std::string& text) {
  WorkloadConfig w;
  auto parts = split(text, ';');
  for (const std::string& p : parts) {
    if (p.empty()) continue;
    VariantConfiguration c = parse_variant(p);
    if (c.strategy == Strategy::SinglePass || c.strategy == Strategy::MultiPass) w.projection = c;
    else w.aggregation = c;
  }
  return w;
}

std::vector<VariantConfiguration> enumerate_variant_space(const PipelineProgram& program) {
  std::vector<VariantConfiguration> out;
  if (program.kind == PipelineKind::Projection) {
    // (single_pass x 1 + multi_pass x 7 thread multipliers) x 2 access x 2 predication = 32
    for (int m = -1; m < 7; ++m)
      for (MemoryAccess a : kAccess)
        for (PredicationMode p : kPred) {
          VariantConfiguration c;
          c.strategy = m < 0 ? Strategy::SinglePass : Strategy::MultiPass;
          c.thread_multiplier = m < 0 ? 1 : kThreadMultipliers[m];
          c.memory_access = a;
          c.predication = p;
          out.push_back(c);
        }
  } else {
    // 2 access x 2 predication x 2 impl x 2 fn x (7 x 7 local + 7 global) = 896
    for (int h = -1; h < 7; ++h)
      for (int wg : kWorkGroupSizes)
        for (MemoryAccess a : kAccess)
          for (PredicationMode p : kPred)
            for (HashTableImpl i : kImpl)
              for (HashFunctionKind f : kFn) {
                VariantConfiguration c;
                c.strategy = h < 0 ? Strategy::GlobalHash : Strategy::LocalHash;
                c.hash_table_count_multiplier = h < 0 ? 1 : kTableCountMultipliers[h];
                c.work_group_size = wg;
                c.memory_access = a;
                c.predication = p;
                c.hash_table_impl = i;
                c.hash_function = f;
                out.push_back(c);
              }
  }
  return out;
}

std::vector<Diagnostic> validate_program(const PipelineProgram& program,
                                         const std::vector<HashTableDescriptor>* descriptors) {
  std::vector<Diagnostic> d;
  if (program.ops.empty() || program.ops.front().kind != PipelineOpKind::Loop)
    d.push_back({"LoopNotFirst", "the program must be headed by LOOP"});
  for (std::size_t i = 1; i < program.ops.size(); ++i)
    if (program.ops[i].kind == PipelineOpKind::Loop)
      d.push_back({"ExtraLoop", "LOOP at position " + std::to_string(i)});
  for (std::size_t i = 0; i < program.ops.size(); ++i) {
    const PipelineOp& op = program.ops[i];
    if (op.mode != program.predication)
      d.push_back({"MixedPredication", std::string("op ") + std::to_string(i) + " (" +
                                           to_string(op.kind) + ") is " + to_string(op.mode) +
                                           ", program is " + to_string(program.predication)});
    if (op.offset < 0 || op.offset >= program.unroll_factor)
      d.push_back({"BadOffset", "op " + std::to_string(i) + " offset " + std::to_string(op.offset)});
    const bool hash = op.kind == PipelineOpKind::HashPut || op.kind == PipelineOpKind::HashProbe ||
                      op.kind == PipelineOpKind::HashAggregate;
    if (hash && descriptors) {
      if (op.descriptor < 0 || static_cast<std::size_t>(op.descriptor) >= descriptors->size()) {
        d.push_back({"UnknownDescriptor", "op " + std::to_string(i)});
      } else {
        const HashTableDescriptor& h = (*descriptors)[static_cast<std::size_t>(op.descriptor)];
        if (h.impl != op.table_impl || h.function != op.hash_function)
          d.push_back({"HashTableMismatch",
                       "op " + std::to_string(i) + " uses " + to_string(op.table_impl) + "/" +
                           to_string(op.hash_function) + ", descriptor " +
                           std::to_string(h.id) + " is " + to_string(h.impl) + "/" +
                           to_string(h.function)});
      }
    }
  }
  const PipelineOpKind last = program.ops.empty() ? PipelineOpKind::Loop : program.ops.back().kind;
  const bool agg = last == PipelineOpKind::Aggregate || last == PipelineOpKind::HashAggregate;
  if (agg != (program.kind == PipelineKind::Aggregation))
    d.push_back({"KindMismatch", "pipeline kind does not match its last op"});
  return d;
}

// ---- workload dimensions, feature order first ---------------------

std::vector<Dimension> workload_dimensions() {
  std::vector<Dimension> dims;
  dims.push_back({"projection_strategy", {"single_pass", "multi_pass"}, [](WorkloadConfig& c, int v) {
                    c.projection.strategy = v == 0 ? Strategy::SinglePass : Strategy::MultiPass;
                  }});
  dims.push_back({"aggregation_strategy", {"local_hash", "global_hash"}, [](WorkloadConfig& c, int v) {
                    c.aggregation.strategy = v == 0 ? Strategy::LocalHash : Strategy::GlobalHash;
                  }});
  {
    Dimension d{"thread_multiplier", {}, [](WorkloadConfig& c, int v) {
                  c.projection.thread_multiplier = kThreadMultipliers[v];
                }};
    for (int t : kThreadMultipliers) d.values.push_back(std::to_string(t));
    dims.push_back(d);
  }
  {
    Dimension d{"work_group_size", {}, [](WorkloadConfig& c, int v) {
                  c.aggregation.work_group_size = kWorkGroupSizes[v];
                }};
    for (int t : kWorkGroupSizes) d.values.push_back(std::to_string(t));
    dims.push_back(d);
  }
  dims.push_back({"memory_access", {"sequential", "coalesced"}, [](WorkloadConfig& c, int v) {
                    c.projection.memory_access = c.aggregation.memory_access = kAccess[v];
                  }});
  {
    Dimension d{"hash_table_count_multiplier", {}, [](WorkloadConfig& c, int v) {
                  c.aggregation.hash_table_count_multiplier = kTableCountMultipliers[v];
                }};
    for (int t : kTableCountMultipliers) d.values.push_back(std::to_string(t));
    dims.push_back(d);
  }
  dims.push_back({"hash_table_impl", {"linear_probing", "cuckoo"}, [](WorkloadConfig& c, int v) {
                    c.projection.hash_table_impl = c.aggregation.hash_table_impl = kImpl[v];
                  }});
  dims.push_back({"hash_function", {"murmur", "multiply_shift"}, [](WorkloadConfig& c, int v) {
                    c.projection.hash_function = c.aggregation.hash_function = kFn[v];
                  }});
  dims.push_back({"predication", {"branched", "predicated"}, [](WorkloadConfig& c, int v) {
                    c.projection.predication = c.aggregation.predication = kPred[v];
                  }});
  return dims;
}

// The learned-configuration file ("key-value text file, one
// dimension per line"): every field of both pipeline kinds' variant.
std::string save_config_text(const WorkloadConfig& c) {
  std::ostringstream os;
  os << "# hawk-b200 variant configuration: <pipeline kind>.<dimension>=<value>\n";
  for (const auto& [kind, v] : {std::pair<const char*, const VariantConfiguration*>{"projection", &c.projection},
                                {"aggregation", &c.aggregation}}) {
    const auto parts = split(v->to_string(), '/');
    os << kind << ".strategy=" << parts[0] << "\n";
    os << kind << ".memory_access=" << parts[1] << "\n";
    os << kind << ".predication=" << parts[2] << "\n";
    os << kind << ".hash_table_impl="
       << (v->hash_table_impl == HashTableImpl::Cuckoo ? "cuckoo" : "linear_probing") << "\n";
    os << kind << ".hash_function="
       << (v->hash_function == HashFunctionKind::MultiplyShift ? "multiply_shift" : "murmur") << "\n";
    os << kind << ".thread_multiplier=" << v->thread_multiplier << "\n";
    os << kind << ".work_group_size=" << v->work_group_size << "\n";
    os << kind << ".hash_table_count_multiplier=" << v->hash_table_count_multiplier << "\n";
    os << kind << ".unroll_factor=" << v->unroll_factor << "\n";
  }
  return os.str();
}

WorkloadConfig load_config_text(const std::string& text) {
  WorkloadConfig w;
  std::istringstream is(text);
  std::string line;
  auto number = [](const std::string& key, const std::string& v) {
    try {
      std::size_t used = 0;
      const int n = std::stoi(v, &used);
      if (used != v.size()) throw std::invalid_argument(v);
      return n;
    } catch (const std::exception&) {
      throw InvalidConfig("config key '" + key + "': '" + v + "' is not an integer");
    }
  };
  while (std::getline(is, line)) {
    while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.pop_back();
    if (line.empty() || line[0] == '#') continue;
    auto eq = line.find('=');
    if (eq == std::string::npos) throw InvalidConfig("config line '" + line + "': expected key=value");
    std::string key = line.substr(0, eq), value = line.substr(eq + 1);
    if (key == "projection") {  // whole-variant form: projection=<to_string()>
      w.projection = parse_variant(value);
      continue;
    }
    if (key == "aggregation") {
      w.aggregation = parse_variant(value);
      continue;
    }
    const auto dot = key.find('.');
    const std::string kind = dot == std::string::npos ? "" : key.substr(0, dot);
    const std::string dim = dot == std::string::npos ? key : key.substr(dot + 1);
    VariantConfiguration* v = kind == "projection" ? &w.projection : kind == "aggregation" ? &w.aggregation : nullptr;
    if (!v) throw InvalidConfig("unknown config key '" + key + "'");
    if (dim == "strategy") {
      v->strategy = parse_variant(value + "/sequential/branched").strategy;
    } else if (dim == "memory_access") {
      v->memory_access = parse_variant("single_pass/" + value + "/branched").memory_access;
    } else if (dim == "predication") {
      v->predication = parse_variant("single_pass/sequential/" + value).predication;
    } else if (dim == "hash_table_impl") {
      v->hash_table_impl = parse_variant("single_pass/sequential/branched/" + value).hash_table_impl;
    } else if (dim == "hash_function") {
      v->hash_function = parse_variant("single_pass/sequential/branched/" + value).hash_function;
    } else if (dim == "thread_multiplier") {
      v->thread_multiplier = number(key, value);
    } else if (dim == "work_group_size") {
      v->work_group_size = number(key, value);
    } else if (dim == "hash_table_count_multiplier") {
      v->hash_table_count_multiplier = number(key, value);
    } else if (dim == "unroll_factor") {
      v->unroll_factor = number(key, value);
    } else {
      throw InvalidConfig("unknown config key '" + key + "'");
    }
  }
  // the parsed text must name an admissible configuration (value lists)
  parse_workload_config(w.to_string());
  return w;
}

}  // namespace hawk::b200
