// hawk-b200 — the command line of the executor (the reference's missing CLI,
// /root/reference/SPEC.md:493-536): data generation and CSV ingest, query
// execution under a variant configuration, full exploration and learning with
// CSV / key-value outputs, and kernel inspection.
//
//   hawk-b200 gen      --db tpch|ssb --sf S [--seed N] --out DIR
//   hawk-b200 run      (--sql STR | --query FILE) [--config FILE | --variant STR]
//                      (--data DIR | --db tpch|ssb --sf S) [--repeat K] [--out CSV]
//                      [--expect-rows N]
//   hawk-b200 explore  (--sql|--query) --kind aggregation|projection [--fixed STR]
//                      (--data|--db/--sf) --out CSV [--prune-threshold MS] [--reps N]
//   hawk-b200 learn    (--sql|--query)... --out CONFIG [--q N] [--no-early-stop]
//                      [--no-unroll] [--trace CSV] [--prune-threshold MS] [--reps N]
//                      (--data|--db/--sf)
//   hawk-b200 emit-kernel (--sql|--query) [--config|--variant] (--data|--db/--sf)
//
// --data DIR loads every DIR/<table>.csv with its DIR/<table>.schema
// ("<column> int64|float64|string" per line), as `gen` writes them.
// Exit codes: 0 success, 1 verification failure
// (--expect-rows), 2 usage error, 3 runtime / capacity error.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "hawk/sql/parser.hpp"
#include "hawk/storage/csv.hpp"
#include "hawk_b200_engine.hpp"
#include "hawk_gen.h"

namespace fs = std::filesystem;
using namespace hawk;
using namespace hawk::b200;

namespace {

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string cmd;
  std::multimap<std::string, std::string> opt;
  std::string get(const std::string& k, const std::string& def = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? def : it->second;
  }
  bool has(const std::string& k) const { return opt.count(k) > 0; }
  std::vector<std::string> all(const std::string& k) const {
    std::vector<std::string> v;
    for (auto [a, b] = opt.equal_range(k); a != b; ++a) v.push_back(a->second);
    return v;
  }
};

Args parse_args(int argc, char** argv) {
  if (argc < 2) throw Usage("missing command");
  Args a;
  a.cmd = argv[1];
  static const char* flags[] = {"--no-early-stop", "--no-unroll", nullptr};
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw Usage("unexpected argument '" + k + "'");
    bool flag = false;
    for (const char** f = flags; *f; ++f) flag |= k == *f;
    if (flag) {
      a.opt.emplace(k, "1");
      continue;
    }
    if (i + 1 >= argc) throw Usage("option " + k + " needs a value");
    a.opt.emplace(k, argv[++i]);
  }
  return a;
}

std::string read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot open '" + path + "'");
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

std::vector<std::string> sqls_of(const Args& a) {
  std::vector<std::string> out = a.all("--sql");
  for (const std::string& q : a.all("--query")) out.push_back(read_file(q));
  if (out.empty()) throw Usage("give --sql or --query");
  return out;
}

int db_tables(const std::string& db, std::vector<int>& t) {
  if (db == "tpch") t = {HG_LINEITEM, HG_ORDERS, HG_CUSTOMER};
  else if (db == "ssb") t = {HG_LINEORDER, HG_DDATE, HG_SCUSTOMER, HG_SUPPLIER, HG_PART};
  else throw Usage("--db must be tpch or ssb");
  return 0;
}

void load_data(Engine& e, const Args& a) {
  if (a.has("--data")) {
    for (const auto& entry : fs::directory_iterator(a.get("--data"))) {
      if (entry.path().extension() != ".csv") continue;
      const std::string name = entry.path().stem().string();
      fs::path schema_path = entry.path();
      schema_path.replace_extension(".schema");
      std::istringstream ss(read_file(schema_path.string()));
      Schema schema;
      std::string col, kind;
      while (ss >> col >> kind) {
        ColumnKind k = kind == "int64" ? ColumnKind::Int64 : kind == "float64" ? ColumnKind::Float64
                       : kind == "string" ? ColumnKind::String
                                          : throw Usage("bad kind '" + kind + "' in " + schema_path.string());
        schema.push_back({col, k});
      }
      e.load_csv(entry.path().string(), name, schema);
    }
    return;
  }
  if (!a.has("--db") || !a.has("--sf")) throw Usage("give --data DIR or --db and --sf");
  std::vector<int> tables;
  db_tables(a.get("--db"), tables);
  const double sf = std::stod(a.get("--sf"));
  const uint64_t seed = std::stoull(a.get("--seed", "42"));
  for (int t : tables) e.generate_table(t, sf, seed);
}

// a catalog-only engine for commands that need no device (emit-kernel)
void load_catalog(Engine& e, const Args& a) {
  if (a.has("--data")) throw Usage("emit-kernel plans against --db/--sf catalogs");
  std::vector<int> tables;
  db_tables(a.get("--db", "tpch"), tables);
  const double sf = std::stod(a.get("--sf", "1"));
  for (int t : tables) {
    Schema schema;
    std::vector<std::vector<std::string>> lex;
    std::vector<const void*> none;
    std::vector<int64_t> distinct;
    for (int c = 0; c < hg_table_ncols(t); ++c) {
      const bool str = hg_col_kind(t, c) == HG_KIND_STRING;
      schema.push_back({hg_col_name(t, c), str ? ColumnKind::String : ColumnKind::Int64});
      std::vector<std::string> l;
      for (int i = 0; i < hg_col_lexicon_size(t, c); ++i) l.emplace_back(hg_col_lexicon(t, c, i));
      lex.push_back(l);
      none.push_back(nullptr);
      distinct.push_back(hg_col_domain(t, c, sf));
    }
    e.put_columns(hg_table_name(t), schema, hg_table_rows(t, sf), none, lex, distinct);
  }
}

WorkloadConfig config_of(const Args& a) {
  if (a.has("--config")) return load_config_text(read_file(a.get("--config")));
  if (a.has("--variant")) return parse_workload_config(a.get("--variant"));
  return WorkloadConfig();
}

void write_csv(std::ostream& os, const ResultColumns& r) {
  for (std::size_t c = 0; c < r.columns.size(); ++c) os << (c ? "," : "") << r.columns[c].name;
  os << "\n";
  for (int64_t i = 0; i < r.rows; ++i) {
    for (std::size_t c = 0; c < r.columns.size(); ++c) {
      const ResultColumn& col = r.columns[c];
      if (c) os << ",";
      const std::size_t k = static_cast<std::size_t>(i);
      if (col.kind == ColumnKind::Float64) os << col.floats[k];
      else if (col.kind == ColumnKind::String) os << col.lexicon[static_cast<std::size_t>(col.ints[k])];
      else os << col.ints[k];
    }
    os << "\n";
  }
}

PipelineSet plan(Engine& e, const std::string& sql) {
  const std::vector<TablePtr> tables = e.catalog();
  return partition_into_pipelines(sql::parse_query(sql, sql::make_catalog(tables)), tables);
}

int cmd_gen(const Args& a) {
  std::vector<int> tables;
  db_tables(a.get("--db"), tables);
  if (!a.has("--sf") || !a.has("--out")) throw Usage("gen needs --sf and --out");
  const double sf = std::stod(a.get("--sf"));
  const uint64_t seed = std::stoull(a.get("--seed", "42"));
  fs::create_directories(a.get("--out"));
  for (int t : tables) {
    const fs::path base = fs::path(a.get("--out")) / hg_table_name(t);
    std::ofstream schema(base.string() + ".schema"), csv(base.string() + ".csv");
    const int nc = hg_table_ncols(t);
    for (int c = 0; c < nc; ++c)
      schema << hg_col_name(t, c) << " " << (hg_col_kind(t, c) == HG_KIND_STRING ? "string" : "int64") << "\n";
    const int64_t rows = hg_table_rows(t, sf);
    for (int64_t r = 0; r < rows; ++r) {
      for (int c = 0; c < nc; ++c) {
        const int64_t v = hg_value(t, c, r, sf, seed);
        if (c) csv << ",";
        if (hg_col_kind(t, c) == HG_KIND_STRING) csv << hg_col_lexicon(t, c, static_cast<int>(v));
        else csv << v;
      }
      csv << "\n";
    }
    std::printf("%s: %lld rows\n", base.string().c_str(), static_cast<long long>(rows));
  }
  return 0;
}

int cmd_run(const Args& a) {
  Engine e(std::stoi(a.get("--device", "0")));
  load_data(e, a);
  const WorkloadConfig cfg = config_of(a);
  const int repeat = std::stoi(a.get("--repeat", "1"));
  int status = 0;
  for (const std::string& sql : sqls_of(a)) {
    const PipelineSet set = plan(e, sql);
    ResultColumns r;
    ExecutionMetrics m;
    std::vector<VariantConfiguration> per;
    for (const PipelineProgram& p : set.pipelines)
      per.push_back(p.kind == PipelineKind::Projection ? cfg.projection : cfg.aggregation);
    for (int i = 0; i < repeat; ++i) r = e.execute_columns(set, per, &m);
    std::fprintf(stderr, "%lld rows, kernels %.3f ms, wall %.3f ms [%s]\n", static_cast<long long>(r.rows),
                 m.kernel_ms, m.wall_ms, cfg.to_string().c_str());
    if (a.has("--out")) {
      std::ofstream out(a.get("--out"));
      write_csv(out, r);
    } else {
      write_csv(std::cout, r);
    }
    if (a.has("--expect-rows") && r.rows != std::stoll(a.get("--expect-rows"))) status = 1;
  }
  return status;
}

int cmd_explore(const Args& a) {
  Engine e(std::stoi(a.get("--device", "0")));
  load_data(e, a);
  std::vector<WorkloadQuery> w;
  for (const std::string& s : sqls_of(a)) w.push_back({"q" + std::to_string(w.size()), s});
  const std::string kind = a.get("--kind", "aggregation");
  if (kind != "aggregation" && kind != "projection") throw Usage("--kind aggregation|projection");
  if (!a.has("--out")) throw Usage("explore needs --out CSV");
  const WorkloadConfig base = a.has("--fixed") ? parse_workload_config(a.get("--fixed")) : config_of(a);
  PipelineProgram shape;
  shape.kind = kind == "projection" ? PipelineKind::Projection : PipelineKind::Aggregation;
  std::vector<WorkloadConfig> space;
  for (const VariantConfiguration& v : enumerate_variant_space(shape)) {
    WorkloadConfig c = base;
    (kind == "projection" ? c.projection : c.aggregation) = v;
    space.push_back(c);
  }
  LearnOptions opt;
  opt.prune_threshold_ms = std::stod(a.get("--prune-threshold", "1000"));
  opt.repetitions = std::stoi(a.get("--reps", "3"));
  LearnResult r = full_exploration(e, w, space, opt);
  std::ofstream(a.get("--out")) << trace_csv(r.trace);
  std::printf("%s %.4f ms (%d configurations)\n", r.best.to_string().c_str(), r.best_ms, r.evaluations);
  return 0;
}

int cmd_learn(const Args& a) {
  Engine e(std::stoi(a.get("--device", "0")));
  load_data(e, a);
  std::vector<WorkloadQuery> w;
  for (const std::string& s : sqls_of(a)) w.push_back({"q" + std::to_string(w.size()), s});
  if (!a.has("--out")) throw Usage("learn needs --out CONFIG");
  LearnOptions opt;
  opt.max_iterations = std::stoi(a.get("--q", "3"));
  opt.early_termination = !a.has("--no-early-stop");
  opt.unroll_pass = !a.has("--no-unroll");
  opt.prune_threshold_ms = std::stod(a.get("--prune-threshold", "1000"));
  opt.repetitions = std::stoi(a.get("--reps", "3"));
  opt.starts = {WorkloadConfig(), b200_start_config()};
  LearnResult r = learn_variant_configuration(e, w, opt);
  std::ofstream(a.get("--out")) << save_config_text(r.best);
  if (a.has("--trace")) std::ofstream(a.get("--trace")) << trace_csv(r.trace);
  std::printf("%s %.4f ms (%d evaluations, %d sweeps)\n", r.best.to_string().c_str(), r.best_ms,
              r.evaluations, r.sweeps);
  return std::isfinite(r.best_ms) ? 0 : 3;
}

int cmd_emit(const Args& a) {
  Engine e(-1);  // planning only: no device needed
  load_catalog(e, a);
  const WorkloadConfig cfg = config_of(a);
  for (const std::string& sql : sqls_of(a)) {
    const PipelineSet set = rewrite_cross_joins(plan(e, sql));
    std::vector<HashTableDescriptor> desc;
    std::vector<VariantConfiguration> eff;
    std::vector<VariantConfiguration> per;
    for (const PipelineProgram& p : set.pipelines)
      per.push_back(p.kind == PipelineKind::Projection ? cfg.projection : cfg.aggregation);
    const std::vector<PipelineProgram> progs = apply_variants(set, per, desc, &eff);
    for (std::size_t i = 0; i < progs.size(); ++i) {
      LoweredProgram lp = lower_program(progs[i], set);
      hawk_variant v{};
      v.strategy = static_cast<int32_t>(eff[i].strategy);
      v.memory_access = static_cast<int32_t>(eff[i].memory_access);
      v.predication = static_cast<int32_t>(eff[i].predication);
      v.hash_table_impl = static_cast<int32_t>(eff[i].hash_table_impl);
      v.hash_function = static_cast<int32_t>(eff[i].hash_function);
      v.thread_multiplier = eff[i].thread_multiplier;
      v.work_group_size = eff[i].work_group_size;
      v.hash_table_count_multiplier = eff[i].hash_table_count_multiplier;
      v.unroll_factor = lp.unroll;
      std::vector<char> buf(1 << 20);
      if (hawk_b200_program_source(&lp.pipe, &v, buf.data(), static_cast<int32_t>(buf.size())) != HAWK_OK)
        throw Error("program source too large");
      std::printf("// ---- pipeline %zu [%s]\n%s\n", i, eff[i].to_string().c_str(), buf.data());
    }
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse_args(argc, argv);
    if (a.cmd == "gen") return cmd_gen(a);
    if (a.cmd == "run") return cmd_run(a);
    if (a.cmd == "explore") return cmd_explore(a);
    if (a.cmd == "learn") return cmd_learn(a);
    if (a.cmd == "emit-kernel") return cmd_emit(a);
    throw Usage("unknown command '" + a.cmd + "'");
  } catch (const Usage& u) {
    std::fprintf(stderr, "usage error: %s\n(commands: gen, run, explore, learn, emit-kernel)\n", u.what());
    return 2;
  } catch (const SyntaxError& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const InvalidConfig& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "usage error: bad number (%s)\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
