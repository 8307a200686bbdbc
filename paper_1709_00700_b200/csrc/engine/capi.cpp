// capi.cpp — extern "C" wrapper of the C++ engine (include/hawk_b200_engine.h).
// No exception crosses this boundary: each is mapped to its hawk_status class.
#include <cstring>
#include <fstream>
#include <sstream>
#include <unordered_map>

#include "hawk/sql/parser.hpp"
#include "hawk_b200_engine.h"
#include "hawk_b200_engine.hpp"

using namespace hawk;
using namespace hawk::b200;

struct hawk_engine {
  Engine engine;
  // parsed + partitioned plans by SQL text, valid for one catalog generation
  std::unordered_map<std::string, PipelineSet> plans;
  uint64_t plans_generation = ~0ull;
  explicit hawk_engine(int d) : engine(d) {}
};

struct hawk_result {
  ResultColumns table;
  ExecutionMetrics metrics;
  std::string metrics_text;
};

struct hawk_partial {
  PartialResult part;
  double kernel_ms = 0;
  int32_t launches = 0;
};

namespace {

thread_local std::string g_error;
thread_local int32_t g_error_class = 0;

int32_t classify(const std::exception& e) {
  if (dynamic_cast<const UnsupportedPlan*>(&e)) return HAWK_ERR_UNSUPPORTED_PLAN;
  if (dynamic_cast<const InvalidConfig*>(&e)) return HAWK_ERR_INVALID_CONFIG;
  if (dynamic_cast<const Unsupported*>(&e)) return HAWK_ERR_UNSUPPORTED;
  if (dynamic_cast<const PlanTooLarge*>(&e)) return HAWK_ERR_PLAN_TOO_LARGE;
  if (dynamic_cast<const CapacityExceeded*>(&e)) return HAWK_ERR_CAPACITY;
  if (dynamic_cast<const DuplicateKey*>(&e)) return HAWK_ERR_DUPLICATE_KEY;
  if (dynamic_cast<const EmptyAggregate*>(&e)) return HAWK_ERR_EMPTY_AGGREGATE;
  if (dynamic_cast<const DivergentPlan*>(&e)) return HAWK_ERR_DIVERGENT_PLAN;
  if (dynamic_cast<const InvalidParams*>(&e)) return HAWK_ERR_INVALID_PARAMS;
  // front-end errors: 10 SyntaxError, 11 UnknownTable, 12 UnknownAttribute, 13 TypeError
  if (dynamic_cast<const SyntaxError*>(&e)) return 10;
  if (dynamic_cast<const UnknownTable*>(&e)) return 11;
  if (dynamic_cast<const UnknownAttribute*>(&e)) return 12;
  if (dynamic_cast<const TypeError*>(&e)) return 13;
  if (dynamic_cast<const ParseError*>(&e)) return 14;
  if (dynamic_cast<const IoError*>(&e)) return 15;
  return 99;
}

template <typename F>
int32_t guard(F&& f) {
  try {
    f();
    g_error.clear();
    g_error_class = 0;
    return HAWK_OK;
  } catch (const std::exception& e) {
    g_error = e.what();
    g_error_class = classify(e);
    return g_error_class;
  } catch (...) {
    g_error = "unknown error";
    g_error_class = 99;
    return 99;
  }
}

PipelineSet plan_sql(Engine& engine, const std::string& sql) {
  const std::vector<TablePtr> tables = engine.catalog();
  auto plan = sql::parse_query(sql, sql::make_catalog(tables));
  return partition_into_pipelines(plan, tables);
}

// plan_sql with the engine's plan cache (parse + partition once per catalog state)
const PipelineSet& cached_plan(hawk_engine* e, const std::string& sql) {
  if (e->plans_generation != e->engine.catalog_generation()) {
    e->plans.clear();
    e->plans_generation = e->engine.catalog_generation();
  }
  auto it = e->plans.find(sql);
  if (it == e->plans.end()) {
    if (e->plans.size() > 256) e->plans.clear();
    it = e->plans.emplace(sql, plan_sql(e->engine, sql)).first;
  }
  return it->second;
}

// "<proj>;<agg>" workload config, or "c0|c1|..." one per pipeline
std::vector<VariantConfiguration> configs_for(const PipelineSet& set, const std::string& text) {
  std::vector<VariantConfiguration> out;
  if (text.find('|') != std::string::npos) {
    std::stringstream ss(text);
    std::string part;
    while (std::getline(ss, part, '|')) out.push_back(parse_variant(part));
    if (out.size() != set.pipelines.size()) throw InvalidConfig("one configuration per pipeline required");
    return out;
  }
  WorkloadConfig w = text.empty() ? WorkloadConfig() : parse_workload_config(text);
  for (const PipelineProgram& p : set.pipelines)
    out.push_back(p.kind == PipelineKind::Projection ? w.projection : w.aggregation);
  return out;
}

void fill_metrics_text(hawk_result* r) {
  std::ostringstream os;
  for (const PipelineMetrics& p : r->metrics.pipelines)
    os << p.variant << ' ' << p.kernel_ms << ' ' << p.launches << ' ' << p.rows_in << ' '
       << p.rows_out << ' ' << p.grid << ' ' << p.block << ' ' << p.retries << '\n';
  r->metrics_text = os.str();
}

void put_str(char* buf, int32_t len, const std::string& s) {
  if (!buf || len <= 0) return;
  std::strncpy(buf, s.c_str(), static_cast<std::size_t>(len - 1));
  buf[len - 1] = 0;
}

}  // namespace

extern "C" {

const char* hawk_engine_last_error(void) { return g_error.c_str(); }
int32_t hawk_engine_last_error_class(void) { return g_error_class; }

int32_t hawk_engine_create(int32_t device, hawk_engine** out) {
  return guard([&] { *out = new hawk_engine(device); });
}

void hawk_engine_destroy(hawk_engine* e) { delete e; }

int32_t hawk_engine_sm_count(hawk_engine* e) { return e->engine.sm_count(); }
void* hawk_engine_ctx(hawk_engine* e) { return e->engine.ctx(); }

int32_t hawk_engine_put_columns(hawk_engine* e, const char* name, int32_t ncols,
                                const char* const* names, const int32_t* kinds, int64_t rows,
                                const void* const* data, const char* const* const* lexicons,
                                const int64_t* lexicon_sizes, const int64_t* distinct,
                                int64_t row_offset) {
  return guard([&] {
    Schema schema;
    std::vector<const void*> cols;
    std::vector<std::vector<std::string>> lex(static_cast<std::size_t>(ncols));
    std::vector<int64_t> dist;
    for (int c = 0; c < ncols; ++c) {
      schema.push_back({names[c], static_cast<ColumnKind>(kinds[c])});
      cols.push_back(data[c]);
      if (kinds[c] == 2 && lexicons && lexicon_sizes)
        for (int64_t i = 0; i < lexicon_sizes[c]; ++i) lex[static_cast<std::size_t>(c)].emplace_back(lexicons[c][i]);
      dist.push_back(distinct ? distinct[c] : 0);
    }
    e->engine.put_columns(name, schema, rows, cols, lex, dist, row_offset);
  });
}

int32_t hawk_engine_generate(hawk_engine* e, int32_t table, double sf, uint64_t seed,
                             int64_t row_begin, int64_t rows) {
  return guard([&] { e->engine.generate_table(table, sf, seed, row_begin, rows); });
}

int32_t hawk_engine_load_csv(hawk_engine* e, const char* path, const char* name, int32_t ncols,
                             const char* const* names, const int32_t* kinds, char delimiter,
                             int32_t header) {
  return guard([&] {
    if (ncols < 1 || !names || !kinds) throw InvalidParams("load_csv: no columns");
    Schema schema;
    for (int i = 0; i < ncols; ++i) schema.push_back({names[i], static_cast<ColumnKind>(kinds[i])});
    CsvOptions opt;
    opt.delimiter = delimiter;
    opt.header = header != 0;
    e->engine.load_csv(path, name, schema, opt);
  });
}

int32_t hawk_engine_drop(hawk_engine* e, const char* name) {
  return guard([&] { e->engine.drop_table(name); });
}

int64_t hawk_engine_table_rows(hawk_engine* e, const char* name) {
  if (!e->engine.has_table(name)) return -1;
  return e->engine.table(name).rows;
}

const int64_t* hawk_engine_column(hawk_engine* e, const char* table, const char* column) {
  if (!e->engine.has_table(table)) return nullptr;
  const DeviceTable& t = e->engine.table(table);
  const int c = t.find(column);
  return c < 0 ? nullptr : t.columns[static_cast<std::size_t>(c)].d_data;
}

int32_t hawk_engine_flush_l2(hawk_engine* e) {
  return guard([&] { e->engine.flush_l2(); });
}

int32_t hawk_engine_run(hawk_engine* e, const char* sql, const char* config, hawk_result** out) {
  *out = nullptr;
  return guard([&] {
    const PipelineSet& set = cached_plan(e, sql);
    auto configs = configs_for(set, config ? config : "");
    auto* r = new hawk_result;
    try {
      r->table = e->engine.execute_columns(set, configs, &r->metrics);
    } catch (...) {
      delete r;
      throw;
    }
    fill_metrics_text(r);
    *out = r;
  });
}

int32_t hawk_engine_run_partial(hawk_engine* e, const char* sql, const char* config,
                                hawk_partial** out) {
  *out = nullptr;
  return guard([&] {
    const PipelineSet& set = cached_plan(e, sql);
    WorkloadConfig w = config && *config ? parse_workload_config(config) : WorkloadConfig();
    auto* p = new hawk_partial;
    ExecutionMetrics m;
    try {
      p->part = e->engine.execute_partial(set, w, &m);
    } catch (...) {
      delete p;
      throw;
    }
    p->kernel_ms = m.kernel_ms;
    p->launches = m.launches;
    *out = p;
  });
}

int32_t hawk_engine_run_sharded(hawk_engine* e, const char* sql, const char* config, hawk_comm* comm,
                                int32_t root, hawk_result** out) {
  *out = nullptr;
  return guard([&] {
    const PipelineSet& set = cached_plan(e, sql);
    WorkloadConfig w = config && *config ? parse_workload_config(config) : WorkloadConfig();
    auto* r = new hawk_result;
    try {
      r->table = e->engine.execute_sharded(set, w, comm, root, &r->metrics);
    } catch (...) {
      delete r;
      throw;
    }
    fill_metrics_text(r);
    *out = r;
  });
}

int64_t hawk_partial_rows(const hawk_partial* p) { return p->part.rows; }
int32_t hawk_partial_width(const hawk_partial* p) { return p->part.width; }
int32_t hawk_partial_sink(const hawk_partial* p) { return p->part.sink; }
const int64_t* hawk_partial_data(const hawk_partial* p) { return p->part.values.data(); }
double hawk_partial_kernel_ms(const hawk_partial* p) { return p->kernel_ms; }
int32_t hawk_partial_launches(const hawk_partial* p) { return p->launches; }
void hawk_partial_free(hawk_partial* p) { delete p; }

int32_t hawk_engine_finalize(hawk_engine* e, const char* sql, const char* config, int32_t nparts,
                             const int64_t* const* data, const int64_t* rows, hawk_result** out) {
  *out = nullptr;
  return guard([&] {
    const PipelineSet set = rewrite_cross_joins(cached_plan(e, sql));
    WorkloadConfig w = config && *config ? parse_workload_config(config) : WorkloadConfig();
    // widths come from the lowered terminal program
    const std::size_t T = static_cast<std::size_t>(set.terminal);
    PipelineProgram term = apply_variant(set.pipelines[T], set.pipelines[T].kind == PipelineKind::Projection
                                                               ? w.projection
                                                               : w.aggregation);
    LoweredProgram lp = lower_program(term, set);
    int width = lp.pipe.sink == HAWK_SINK_AGGREGATE   ? lp.pipe.naggs
                : lp.pipe.sink == HAWK_SINK_PROJECT ? lp.pipe.nproject
                                                    : lp.pipe.nkeys + lp.pipe.naggs;
    std::vector<PartialResult> parts(static_cast<std::size_t>(nparts));
    for (int i = 0; i < nparts; ++i) {
      PartialResult& p = parts[static_cast<std::size_t>(i)];
      p.sink = lp.pipe.sink;
      p.rows = rows[i];
      p.width = width;
      p.values.assign(data[i], data[i] + rows[i] * width);
    }
    auto* r = new hawk_result;
    try {
      r->table = e->engine.finalize_partials_columns(set, w, parts);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

int64_t hawk_result_rows(const hawk_result* r) { return r->table.rows; }
int32_t hawk_result_ncols(const hawk_result* r) { return static_cast<int32_t>(r->table.columns.size()); }
const char* hawk_result_col_name(const hawk_result* r, int32_t c) {
  return r->table.columns[static_cast<std::size_t>(c)].name.c_str();
}
int32_t hawk_result_col_kind(const hawk_result* r, int32_t c) {
  return static_cast<int32_t>(r->table.columns[static_cast<std::size_t>(c)].kind);
}
const void* hawk_result_col_data(const hawk_result* r, int32_t c) {
  const ResultColumn& col = r->table.columns[static_cast<std::size_t>(c)];
  if (col.kind == ColumnKind::Float64) return col.floats.data();
  return col.ints.data();
}
int64_t hawk_result_col_lexicon_size(const hawk_result* r, int32_t c) {
  return static_cast<int64_t>(r->table.columns[static_cast<std::size_t>(c)].lexicon.size());
}
const char* hawk_result_col_lexicon(const hawk_result* r, int32_t c, int64_t i) {
  return r->table.columns[static_cast<std::size_t>(c)].lexicon[static_cast<std::size_t>(i)].c_str();
}
double hawk_result_kernel_ms(const hawk_result* r) { return r->metrics.kernel_ms; }
double hawk_result_wall_ms(const hawk_result* r) { return r->metrics.wall_ms; }
int64_t hawk_result_input_tuples(const hawk_result* r) { return r->metrics.input_tuples; }
int32_t hawk_result_launches(const hawk_result* r) { return r->metrics.launches; }
const char* hawk_result_metrics_text(const hawk_result* r) { return r->metrics_text.c_str(); }
void hawk_result_free(hawk_result* r) { delete r; }

int32_t hawk_engine_pipeline_count(hawk_engine* e, const char* sql, int32_t* n) {
  return guard([&] { *n = static_cast<int32_t>(plan_sql(e->engine, sql).pipelines.size()); });
}

int32_t hawk_engine_space_size(hawk_engine* e, const char* sql, int32_t pipeline, int32_t* n,
                               int32_t* single_pass) {
  return guard([&] {
    PipelineSet set = plan_sql(e->engine, sql);
    auto space = enumerate_variant_space(set.pipelines.at(static_cast<std::size_t>(pipeline)));
    *n = static_cast<int32_t>(space.size());
    *single_pass = 0;
    for (const auto& c : space) *single_pass += c.strategy == Strategy::SinglePass;
  });
}

int32_t hawk_engine_space_config(hawk_engine* e, const char* sql, int32_t pipeline, int32_t i,
                                 char* buf, int32_t len) {
  return guard([&] {
    PipelineSet set = plan_sql(e->engine, sql);
    auto space = enumerate_variant_space(set.pipelines.at(static_cast<std::size_t>(pipeline)));
    put_str(buf, len, space.at(static_cast<std::size_t>(i)).to_string());
  });
}

int32_t hawk_engine_validate(hawk_engine* e, const char* sql, const char* config, char* buf,
                             int32_t len) {
  return guard([&] {
    PipelineSet set = rewrite_cross_joins(plan_sql(e->engine, sql));
    auto configs = configs_for(set, config ? config : "");
    std::vector<HashTableDescriptor> desc;
    std::vector<PipelineProgram> progs = apply_variants(set, configs, desc);
    std::ostringstream os;
    for (std::size_t i = 0; i < progs.size(); ++i)
      for (const Diagnostic& d : validate_program(progs[i], &desc))
        os << i << ':' << d.code << ':' << d.message << '\n';
    put_str(buf, len, os.str());
  });
}

// Generates and NVRTC-compiles the program of every pipeline (no GPU needed);
// `buf` receives one line per pipeline ("<i> ok <cubin bytes>" or the log).
int32_t hawk_engine_compile_check(hawk_engine* e, const char* sql, const char* config, char* buf,
                                  int32_t len) {
  return guard([&] {
    PipelineSet set = rewrite_cross_joins(plan_sql(e->engine, sql));
    auto configs = configs_for(set, config ? config : "");
    std::vector<HashTableDescriptor> desc;
    std::vector<VariantConfiguration> eff;
    std::vector<PipelineProgram> progs = apply_variants(set, configs, desc, &eff);
    std::ostringstream os;
    bool all_ok = true;
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
      std::string log(8192, '\0');
      size_t bytes = 0;
      const int32_t st = hawk_b200_program_compile(&lp.pipe, &v, log.data(), (int32_t)log.size(), &bytes);
      if (st == HAWK_OK) {
        // one line per pipeline: cubin bytes + the ptxas resource summary
        std::string info = log.c_str(), regs, spill;
        auto grab = [&](const char* key, std::string& out) {
          const auto at = info.find(key);
          if (at != std::string::npos) out = info.substr(at, info.find('\n', at) - at);
        };
        grab("Used ", regs);
        grab("bytes stack frame", spill);
        const auto dot = spill.find(',');
        os << i << " ok " << bytes << " [" << regs << (dot != std::string::npos ? ";" + spill.substr(dot + 1) : "")
           << "]\n";
      } else {
        all_ok = false;
        os << i << " error " << st << " " << log.c_str() << "\n";
      }
    }
    put_str(buf, len, os.str());
    if (!all_ok) throw Error("program compilation failed:\n" + os.str());
  });
}

int32_t hawk_engine_explain(hawk_engine* e, const char* sql, const char* config, char* buf,
                            int32_t len) {
  return guard([&] {
    PipelineSet set = rewrite_cross_joins(plan_sql(e->engine, sql));
    auto configs = configs_for(set, config ? config : "");
    std::ostringstream os;
    for (std::size_t i = 0; i < set.pipelines.size(); ++i) {
      PipelineProgram prog = apply_variant(set.pipelines[i], configs[i]);
      LoweredProgram lp = lower_program(prog, set);
      os << "pipeline " << i << (static_cast<int>(i) == set.terminal ? " (terminal)" : "") << " driver "
         << set.tables.at(static_cast<std::size_t>(prog.driver_table))->name() << " ["
         << configs[i].to_string() << "]\n"
         << describe(lp.pipe);
    }
    put_str(buf, len, os.str());
  });
}

int32_t hawk_engine_measure(hawk_engine* e, const char* const* sqls, int32_t n, const char* config,
                            double prune_ms, int32_t reps, double* ms) {
  return guard([&] {
    std::vector<WorkloadQuery> w;
    for (int i = 0; i < n; ++i) w.push_back({"q" + std::to_string(i), sqls[i]});
    LearnOptions opt;
    opt.prune_threshold_ms = prune_ms;
    opt.repetitions = reps;
    Measurement m = measure_variant(e->engine, parse_workload_config(config), w, opt);
    *ms = m.ms;
  });
}

int32_t hawk_engine_learn(hawk_engine* e, const char* const* sqls, int32_t n, int32_t q,
                          double prune_ms, int32_t reps, char* best, int32_t len, double* best_ms,
                          int32_t* evaluations, int32_t* sweeps) {
  return guard([&] {
    std::vector<WorkloadQuery> w;
    for (int i = 0; i < n; ++i) w.push_back({"q" + std::to_string(i), sqls[i]});
    LearnOptions opt;
    opt.max_iterations = q;
    opt.prune_threshold_ms = prune_ms;
    opt.repetitions = reps;
    // Algorithm 1 from the reference default, then from the B200 start
    opt.starts = {WorkloadConfig(), b200_start_config()};
    LearnResult r = learn_variant_configuration(e->engine, w, opt);
    put_str(best, len, r.best.to_string());
    *best_ms = r.best_ms;
    *evaluations = r.evaluations;
    *sweeps = r.sweeps;
  });
}

static void write_file(const char* path, const std::string& text) {
  if (!path || !*path) return;
  std::ofstream f(path, std::ios::binary);
  if (!f) throw Error(std::string("cannot write ") + path);
  f << text;
  if (!f) throw Error(std::string("cannot write ") + path);
}

int32_t hawk_config_save(const char* config, const char* path) {
  return guard([&] { write_file(path, save_config_text(parse_workload_config(config ? config : ""))); });
}

int32_t hawk_config_load(const char* path, char* buf, int32_t len) {
  return guard([&] {
    std::ifstream f(path ? path : "");
    if (!f) throw InvalidParams(std::string("cannot read config file ") + (path ? path : ""));
    std::stringstream ss;
    ss << f.rdbuf();
    put_str(buf, len, load_config_text(ss.str()).to_string());
  });
}

static std::vector<WorkloadQuery> workload_of(const char* const* sqls, int32_t n) {
  if (n < 1) throw InvalidParams("empty workload");
  std::vector<WorkloadQuery> w;
  for (int i = 0; i < n; ++i) w.push_back({"q" + std::to_string(i), sqls[i]});
  return w;
}

int32_t hawk_engine_explore(hawk_engine* e, const char* const* sqls, int32_t n, int32_t kind,
                            const char* fixed, double prune_ms, int32_t reps, const char* csv_path,
                            char* best, int32_t len, double* best_ms, int32_t* evaluations) {
  return guard([&] {
    const auto w = workload_of(sqls, n);
    const WorkloadConfig base = fixed && *fixed ? parse_workload_config(fixed) : WorkloadConfig();
    PipelineProgram shape;
    shape.kind = kind == 0 ? PipelineKind::Projection : PipelineKind::Aggregation;
    std::vector<WorkloadConfig> space;
    for (const VariantConfiguration& v : enumerate_variant_space(shape)) {
      WorkloadConfig c = base;
      (kind == 0 ? c.projection : c.aggregation) = v;
      space.push_back(c);
    }
    LearnOptions opt;
    opt.prune_threshold_ms = prune_ms;
    opt.repetitions = reps;
    LearnResult r = full_exploration(e->engine, w, space, opt);
    write_file(csv_path, trace_csv(r.trace));
    put_str(best, len, r.best.to_string());
    *best_ms = r.best_ms;
    *evaluations = r.evaluations;
  });
}

int32_t hawk_engine_learn_ex(hawk_engine* e, const char* const* sqls, int32_t n, int32_t q,
                             int32_t early_termination, double prune_ms, int32_t reps,
                             int32_t unroll_pass, const char* starts, const char* trace_csv_path,
                             const char* config_path, char* best, int32_t len, double* best_ms,
                             int32_t* evaluations, int32_t* sweeps) {
  return guard([&] {
    const auto w = workload_of(sqls, n);
    LearnOptions opt;
    opt.max_iterations = q;
    opt.early_termination = early_termination != 0;
    opt.prune_threshold_ms = prune_ms;
    opt.repetitions = reps;
    opt.unroll_pass = unroll_pass != 0;
    if (starts && *starts) {
      std::stringstream ss(starts);
      std::string part;
      while (std::getline(ss, part, '|')) opt.starts.push_back(parse_workload_config(part));
    }
    LearnResult r = learn_variant_configuration(e->engine, w, opt);
    write_file(trace_csv_path, trace_csv(r.trace));
    write_file(config_path, save_config_text(r.best));
    put_str(best, len, r.best.to_string());
    *best_ms = r.best_ms;
    *evaluations = r.evaluations;
    *sweeps = r.sweeps;
  });
}

int32_t hawk_coordinate_descent(int32_t ndims, const int32_t* sizes, hawk_index_cost_fn cost, void* user,
                                int32_t q, int32_t early_termination, int32_t* best, double* best_ms,
                                int32_t* evaluations, int32_t* sweeps, int32_t* sweep1_evaluations) {
  return guard([&] {
    if (ndims < 1 || !sizes || !cost || !best) throw InvalidParams("coordinate descent: bad arguments");
    std::vector<int> sz(sizes, sizes + ndims);
    for (int v : sz)
      if (v < 1) throw InvalidParams("coordinate descent: empty dimension");
    LearnOptions opt;
    opt.max_iterations = q;
    opt.early_termination = early_termination != 0;
    IndexDescent r = descend(sz, opt, {}, [&](const std::vector<int>& idx) {
      std::vector<int32_t> i32(idx.begin(), idx.end());
      return cost(i32.data(), ndims, user);
    });
    for (int d = 0; d < ndims; ++d) best[d] = r.best.empty() ? 0 : r.best[static_cast<std::size_t>(d)];
    *best_ms = r.best_ms;
    *evaluations = r.evaluations;
    *sweeps = r.sweeps;
    if (sweep1_evaluations) *sweep1_evaluations = r.evaluations_per_sweep.empty() ? 0 : r.evaluations_per_sweep[0];
  });
}

int32_t hawk_learn_with_cost(hawk_cost_fn cost, void* user, int32_t q, int32_t early_termination,
                             const char* starts, char* best, int32_t len, double* best_ms,
                             int32_t* evaluations, int32_t* sweeps) {
  return guard([&] {
    if (!cost) throw InvalidParams("no cost function");
    LearnOptions opt;
    opt.max_iterations = q;
    opt.early_termination = early_termination != 0;
    if (starts && *starts) {
      std::stringstream ss(starts);
      std::string part;
      while (std::getline(ss, part, '|')) opt.starts.push_back(parse_workload_config(part));
    }
    LearnResult r = coordinate_descent(workload_dimensions(), opt, [&](const WorkloadConfig& c) {
      Measurement m;
      m.ms = cost(c.to_string().c_str(), user);
      return m;
    });
    put_str(best, len, r.best.to_string());
    *best_ms = r.best_ms;
    *evaluations = r.evaluations;
    *sweeps = r.sweeps;
  });
}

}  // extern "C"
