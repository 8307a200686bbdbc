// learner.cpp — variant-configuration learning on the B200 (
// PAPER.md:1330-1421, Algorithm 1). Every candidate is timed with CUDA events
// on the device the way the paper times every variant on its processor.
#include <algorithm>
#include <cmath>
#include <functional>
#include <map>
#include <sstream>

#include "hawk/sql/parser.hpp"
#include "hawk_b200_engine.hpp"

namespace hawk::b200 {

namespace {

struct PreparedQuery {
  std::string name;
  PipelineSet set;
};

std::vector<PreparedQuery> prepare(Engine& engine, const std::vector<WorkloadQuery>& workload) {
  std::vector<PreparedQuery> out;
  const std::vector<TablePtr> tables = engine.catalog();
  for (const WorkloadQuery& q : workload) {
    auto plan = sql::parse_query(q.sql, sql::make_catalog(tables));
    out.push_back({q.name, partition_into_pipelines(plan, tables)});
  }
  return out;
}

// the reference exception class of a failed measurement (hawk/error.hpp:9-54)
std::string error_class(const std::exception& e) {
  if (dynamic_cast<const CapacityExceeded*>(&e)) return "CapacityExceeded";
  if (dynamic_cast<const DuplicateKey*>(&e)) return "DuplicateKey";
  if (dynamic_cast<const PlanTooLarge*>(&e)) return "PlanTooLarge";
  if (dynamic_cast<const InvalidConfig*>(&e)) return "InvalidConfig";
  if (dynamic_cast<const Unsupported*>(&e)) return "Unsupported";
  if (dynamic_cast<const UnsupportedPlan*>(&e)) return "UnsupportedPlan";
  if (dynamic_cast<const EmptyAggregate*>(&e)) return "EmptyAggregate";
  if (dynamic_cast<const DivergentPlan*>(&e)) return "DivergentPlan";
  return "Error";
}

std::vector<VariantConfiguration> per_kind(const PipelineSet& set, const WorkloadConfig& c) {
  std::vector<VariantConfiguration> v;
  for (const PipelineProgram& p : set.pipelines)
    v.push_back(p.kind == PipelineKind::Projection ? c.projection : c.aggregation);
  return v;
}

Measurement measure(Engine& engine, const WorkloadConfig& config,
                    const std::vector<PreparedQuery>& queries, const LearnOptions& opt) {
  Measurement m;
  m.config = config;
  double total = 0;
  for (const PreparedQuery& q : queries) {
    std::vector<double> times;
    try {
      for (int r = 0; r < std::max(1, opt.repetitions); ++r) {
        ExecutionMetrics em;
        engine.flush_l2();  // every run starts from HBM, as the paper's cold runs
        engine.execute_columns(q.set, per_kind(q.set, config), &em);
        times.push_back(em.kernel_ms);
        // slow variants are pruned after one run
        if (em.kernel_ms > opt.prune_threshold_ms) break;
      }
    } catch (const std::exception& e) {
      // variant errors count as +inf with a diagnostic
      m.error = q.name + ": " + error_class(e) + ": " + e.what();
      m.ms = std::numeric_limits<double>::infinity();
      return m;
    }
    std::sort(times.begin(), times.end());
    const double med = times[times.size() / 2];
    if (med > opt.prune_threshold_ms) {
      m.pruned = true;
      m.ms = std::numeric_limits<double>::infinity();
      return m;
    }
    total += med;
  }
  m.ms = total;
  return m;
}

}  // namespace

Measurement measure_variant(Engine& engine, const WorkloadConfig& config,
                            const std::vector<WorkloadQuery>& workload, const LearnOptions& opt) {
  return measure(engine, config, prepare(engine, workload), opt);
}

WorkloadConfig b200_start_config() {
  return parse_workload_config(
      "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8");
}

IndexDescent descend(const std::vector<int>& sizes, const LearnOptions& opt,
                     const std::vector<std::vector<int>>& starts_in,
                     const std::function<double(const std::vector<int>&)>& cost) {
  IndexDescent res;
  std::map<std::vector<int>, double> cache;  // measurements by configuration
  auto eval = [&](const std::vector<int>& idx) -> double {
    auto it = cache.find(idx);
    if (it != cache.end()) return it->second;
    const double ms = cost(idx);
    ++res.evaluations;
    if (!res.evaluations_per_sweep.empty()) ++res.evaluations_per_sweep.back();
    cache[idx] = ms;
    return ms;
  };
  std::vector<std::vector<int>> starts = starts_in;
  if (starts.empty()) starts.emplace_back(sizes.size(), 0);  // Algorithm 1 line 1
  bool first = true;
  for (std::vector<int> cur : starts) {
    int sweeps = 0;
    for (int sweep = 0; sweep < opt.max_iterations; ++sweep) {
      res.evaluations_per_sweep.push_back(0);
      bool changed = false;
      for (std::size_t d = 0; d < sizes.size(); ++d) {  // feature order
        int best_v = cur[d];
        double best = eval(cur);
        for (int v = 0; v < sizes[d]; ++v) {
          std::vector<int> cand = cur;
          cand[d] = v;
          const double ms = eval(cand);
          if (ms < best) {  // strict <: ties keep the earlier value
            best = ms;
            best_v = v;
          }
        }
        if (best_v != cur[d]) {
          cur[d] = best_v;
          changed = true;
        }
      }
      ++sweeps;
      if (opt.early_termination && !changed) break;  // Algorithm 1 lines 19-21
    }
    const double ms = eval(cur);
    if (first || ms < res.best_ms) {
      res.best = cur;
      res.best_ms = ms;
      res.sweeps = sweeps;
    }
    first = false;
  }
  return res;
}

LearnResult coordinate_descent(const std::vector<Dimension>& dims, const LearnOptions& opt,
                               const std::function<Measurement(const WorkloadConfig&)>& cost) {
  LearnResult res;
  auto config_of = [&](const std::vector<int>& idx) {
    WorkloadConfig c;
    if (!opt.starts.empty()) c = opt.starts.front();  // fields outside the dimensions
    for (std::size_t d = 0; d < dims.size(); ++d) dims[d].set(c, idx[d]);
    return c;
  };
  // dimension value indices of a configuration (values not on a dimension's
  // list fall back to its first value)
  auto index_of = [&](const WorkloadConfig& c) {
    std::vector<int> idx(dims.size(), 0);
    for (std::size_t d = 0; d < dims.size(); ++d)
      for (int v = 0; v < static_cast<int>(dims[d].values.size()); ++v) {
        WorkloadConfig t = c;
        dims[d].set(t, v);
        if (t.to_string() == c.to_string()) {
          idx[d] = v;
          break;
        }
      }
    return idx;
  };
  // distinct index vectors can name one configuration (e.g. thread
  // multipliers of a single-pass projection): measure each configuration once
  std::map<std::string, double> by_config;
  std::vector<int> sizes;
  for (const Dimension& d : dims) sizes.push_back(static_cast<int>(d.values.size()));
  std::vector<std::vector<int>> starts;
  for (const WorkloadConfig& c : opt.starts) starts.push_back(index_of(c));
  IndexDescent r = descend(sizes, opt, starts, [&](const std::vector<int>& idx) {
    const WorkloadConfig c = config_of(idx);
    const std::string key = c.to_string();
    auto it = by_config.find(key);
    if (it != by_config.end()) return it->second;
    Measurement m = cost(c);
    m.config = c;
    ++res.evaluations;
    res.trace.push_back(m);
    by_config[key] = m.ms;
    return m.ms;
  });
  res.best = config_of(r.best);
  res.best_ms = r.best_ms;
  res.sweeps = r.sweeps;
  return res;
}

std::vector<Dimension> unroll_dimensions() {
  std::vector<Dimension> dims;
  for (int kind = 0; kind < 2; ++kind) {
    Dimension d{kind == 0 ? "projection_unroll" : "aggregation_unroll", {}, nullptr};
    for (int u : kUnrollFactors) d.values.push_back(std::to_string(u));
    d.set = [kind](WorkloadConfig& c, int v) {
      (kind == 0 ? c.projection : c.aggregation).unroll_factor = kUnrollFactors[v];
    };
    dims.push_back(d);
  }
  return dims;
}

LearnResult learn_variant_configuration(Engine& engine, const std::vector<WorkloadQuery>& workload,
                                        const LearnOptions& opt) {
  const std::vector<PreparedQuery> queries = prepare(engine, workload);
  auto cost = [&](const WorkloadConfig& c) { return measure(engine, c, queries, opt); };
  LearnResult res = coordinate_descent(workload_dimensions(), opt, cost);
  if (!opt.unroll_pass || !std::isfinite(res.best_ms)) return res;
  // unroll is a code transformation outside the 32 / 896 space:
  // one coordinate pass over the projection and aggregation unroll factors,
  // starting from the learned configuration
  std::vector<Dimension> dims = unroll_dimensions();
  for (Dimension& d : dims) {
    auto set = d.set;
    const WorkloadConfig base = res.best;
    d.set = [set, base](WorkloadConfig& c, int v) {
      const int pu = c.projection.unroll_factor, au = c.aggregation.unroll_factor;
      c = base;
      c.projection.unroll_factor = pu;
      c.aggregation.unroll_factor = au;
      set(c, v);
    };
  }
  LearnOptions uo = opt;
  uo.max_iterations = 1;
  uo.starts = {res.best};
  LearnResult u = coordinate_descent(dims, uo, cost);
  res.evaluations += u.evaluations;
  for (Measurement& m : u.trace) res.trace.push_back(std::move(m));
  if (u.best_ms < res.best_ms) {
    res.best = u.best;
    res.best_ms = u.best_ms;
  }
  return res;
}

// Exploration / learning trace as CSV (config fields + metric
// columns): one row per measured configuration, in measurement order.
std::string trace_csv(const std::vector<Measurement>& trace) {
  std::ostringstream os;
  os << "index,projection,aggregation,ms,status,detail\n";
  int i = 0;
  for (const Measurement& m : trace) {
    std::string detail = m.error;
    for (char& ch : detail)
      if (ch == '"' || ch == '\n' || ch == '\r') ch = '\'';
    const char* status = !m.error.empty() ? "error" : m.pruned ? "pruned" : "ok";
    os << i++ << "," << m.config.projection.to_string() << "," << m.config.aggregation.to_string() << ",";
    if (std::isfinite(m.ms)) os << m.ms;
    else os << "inf";
    os << "," << status << ",\"" << detail << "\"\n";
  }
  return os.str();
}

LearnResult full_exploration(Engine& engine, const std::vector<WorkloadQuery>& workload,
                             const std::vector<WorkloadConfig>& space, const LearnOptions& opt) {
  const std::vector<PreparedQuery> queries = prepare(engine, workload);
  LearnResult res;
  for (const WorkloadConfig& c : space) {
    Measurement m = measure(engine, c, queries, opt);
    ++res.evaluations;
    if (m.ms < res.best_ms) {  // ties broken by enumeration order
      res.best_ms = m.ms;
      res.best = c;
    }
    res.trace.push_back(std::move(m));
  }
  return res;
}

}  // namespace hawk::b200
