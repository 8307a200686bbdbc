// learner.cpp — variant-configuration learning on the B200 (
// PAPER.md:1330-1421, Algorithm 1). Every candidate is timed with CUDA events
// on the device the way the paper times every variant on its processor.
#include <algorithm>
#include <cmath>
#include <functional>
#include <map>

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
      // variant errors count as +inf
      m.error = q.name + ": " + e.what();
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

LearnResult coordinate_descent(const std::vector<Dimension>& dims, const LearnOptions& opt,
                               const std::function<Measurement(const WorkloadConfig&)>& cost) {
  LearnResult res;
  auto config_of = [&](const std::vector<int>& idx) {
    WorkloadConfig c;
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
  std::map<std::string, Measurement> cache;  // measurements by configuration key
  auto eval = [&](const std::vector<int>& idx) -> double {
    WorkloadConfig c = config_of(idx);
    const std::string key = c.to_string();
    auto it = cache.find(key);
    if (it != cache.end()) return it->second.ms;
    Measurement m = cost(c);
    m.config = c;
    ++res.evaluations;
    res.trace.push_back(m);
    cache[key] = m;
    return m.ms;
  };
  std::vector<std::vector<int>> starts;
  if (opt.starts.empty()) starts.emplace_back(dims.size(), 0);  // Algorithm 1 line 1
  for (const WorkloadConfig& c : opt.starts) starts.push_back(index_of(c));
  bool first = true;
  for (std::vector<int> cur : starts) {
    int sweeps = 0;
    for (int sweep = 0; sweep < opt.max_iterations; ++sweep) {
      bool changed = false;
      for (std::size_t d = 0; d < dims.size(); ++d) {   // feature order
        int best_v = cur[d];
        double best = eval(cur);
        for (int v = 0; v < static_cast<int>(dims[d].values.size()); ++v) {
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
      res.best = config_of(cur);
      res.best_ms = ms;
      res.sweeps = sweeps;
    }
    first = false;
  }
  return res;
}

LearnResult learn_variant_configuration(Engine& engine, const std::vector<WorkloadQuery>& workload,
                                        const LearnOptions& opt) {
  const std::vector<PreparedQuery> queries = prepare(engine, workload);
  return coordinate_descent(workload_dimensions(), opt, [&](const WorkloadConfig& c) {
    return measure(engine, c, queries, opt);
  });
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
