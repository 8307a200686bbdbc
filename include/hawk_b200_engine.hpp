// hawk_b200_engine.hpp — the C++ host side of the B200 executor, speaking the
// reference's own pipeline-program types so it is a drop-in for the missing
// codegen/runtime/optimizer layers of Hawk (/root/reference/proj/CMakeLists.txt:24-39).
//
//   reference (declared, implementation missing)      here
//   ------------------------------------------------   -----------------------------
//   apply_variant & passes   ir/passes.hpp:9-26        defined in engine/passes.cpp
//   enumerate_variant_space  SPEC.md:244-252           hawk::b200::enumerate_variant_space
//   validate_program         SPEC.md:235-243           hawk::b200::validate_program
//   execute_kernel_plan      SPEC.md:372-380           hawk::b200::Engine::execute
//   exclusive_prefix_sum     SPEC.md:381-389           hawk_b200_exclusive_prefix_sum (C ABI)
//   eval_hash                SPEC.md:399-407           hawk_b200_eval_hash (C ABI)
//   measure_variant          SPEC.md:447-455           hawk::b200::measure_variant
//   learn_variant_config.    SPEC.md:456-464           hawk::b200::learn_variant_configuration
//   full_exploration         SPEC.md:465-473           hawk::b200::full_exploration
//
// Inputs are the reference's PipelineSet (planner/pipelines.hpp:11-16) as
// produced by partition_into_pipelines, and VariantConfiguration values
// (ir/program.hpp:190-203); the output is a reference Table
// (storage/table.hpp:23-52) comparable with compare_result_tables.
#pragma once

#include <cstdint>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "hawk/error.hpp"
#include "hawk/ir/passes.hpp"
#include "hawk/ir/program.hpp"
#include "hawk/planner/pipelines.hpp"
#include "hawk/storage/csv.hpp"
#include "hawk/storage/table.hpp"
#include "hawk_b200.h"
#include "hawk_b200_comm.h"

namespace hawk::b200 {

// ---- variant configurations ----------------------------------------------------

/// One VariantConfiguration per pipeline kind: the paper's per-processor
/// "variant configuration" covers projection and aggregation pipelines
/// (PAPER.md:2027-2034 learned-optimizer table).
struct WorkloadConfig {
  VariantConfiguration projection;
  VariantConfiguration aggregation;
  WorkloadConfig();
  std::string to_string() const;
  bool operator==(const WorkloadConfig&) const = default;
};

/// Parses VariantConfiguration::to_string() output
/// (/root/reference/proj/src/ir_program.cpp:84-96). Throws InvalidConfig.
VariantConfiguration parse_variant(const std::string& text);
WorkloadConfig parse_workload_config(const std::string& text);  // "proj;agg"

/// Exact variant space of one pipeline: 32 projection
/// configurations (4 single-pass) and 896 aggregation configurations.
std::vector<VariantConfiguration> enumerate_variant_space(const PipelineProgram& program);

struct Diagnostic {
  std::string code;  // MixedPredication, HashTableMismatch, LoopNotFirst, BadOffset, ...
  std::string message;
};
/// validate_program; never throws.
std::vector<Diagnostic> validate_program(const PipelineProgram& program,
                                         const std::vector<HashTableDescriptor>* descriptors = nullptr);

// ---- device column store ----------------------------------------------------------

struct DeviceColumn {
  std::string name;
  ColumnKind kind = ColumnKind::Int64;
  int64_t* d_data = nullptr;  // 8 bytes per row, padded to a multiple of 64 rows
  int64_t distinct = 0;       // exact or upper bound on distinct values; 0 = unknown
  bool range_known = false;   // [lo, hi] computed on the device on first use as a group key
  int64_t lo = 0, hi = 0;
};

struct DeviceTable {
  std::string name;
  int64_t rows = 0;
  int64_t row_offset = 0;  // global row id of local row 0 (fact-table shards)
  std::vector<DeviceColumn> columns;
  TablePtr catalog;        // schema + lexicons for the front end
  bool pooled = false;     // columns come from the engine's block pool (pair tables)
  int find(const std::string& column) const;
};

struct PipelineMetrics {
  std::string variant;
  double kernel_ms = 0;  // CUDA-event time of this pipeline's kernels
  int launches = 0;
  int64_t rows_in = 0;
  int64_t rows_out = 0;
  int grid = 0, block = 0;
  int retries = 0;
};

struct ExecutionMetrics {
  double kernel_ms = 0;     // sum over pipelines
  double wall_ms = 0;       // host wall time of execute()
  int64_t input_tuples = 0; // rows of every scanned table
  int launches = 0;
  std::vector<PipelineMetrics> pipelines;
};

/// std::vector whose resize leaves new elements uninitialised: result columns
/// are filled right after, and zero-filling 10 MB columns first cost a
/// measurable share of TPC-H Q3 SF100's host time.
template <class T>
struct default_init_allocator : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = default_init_allocator<U>;
  };
  using std::allocator<T>::allocator;
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};
template <class T>
using uvector = std::vector<T, default_init_allocator<T>>;

/// A query result as plain columns (the C ABI's result form). Strings are
/// codes into `lexicon` in first-appearance order, as a reference Table
/// encodes them (storage_table.cpp:127-135); to_table() builds that Table.
struct ResultColumn {
  std::string name;
  ColumnKind kind = ColumnKind::Int64;
  uvector<int64_t> ints;   // Int64 values / String codes
  uvector<double> floats;  // Float64 values
  std::vector<std::string> lexicon;
};
struct ResultColumns {
  std::vector<ResultColumn> columns;
  int64_t rows = 0;
  Table to_table() const;
};

/// Partial result of a fact-table shard, before the cross-GPU merge.
struct PartialResult {
  int sink = HAWK_SINK_AGGREGATE;
  std::vector<int64_t> values;  // AGGREGATE: naggs accs; HASH_AGGREGATE: groups x (K + A)
  int64_t rows = 0;
  int width = 0;
  hawk_pipeline program{};      // lowered terminal program (for merge semantics)
};

class Engine {
 public:
  explicit Engine(int device = 0);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  int device() const { return device_; }
  int sm_count() const;
  hawk_ctx* ctx() const { return ctx_; }

  /// Uploads a host table (H2D), keyed by its name.
  void put_table(const TablePtr& table);
  /// Uploads raw host columns (int64 / float64 bits / string codes).
  void put_columns(const std::string& name, const Schema& schema, int64_t rows,
                   const std::vector<const void*>& host_columns,
                   const std::vector<std::vector<std::string>>& lexicons,
                   const std::vector<int64_t>& distinct, int64_t row_offset = 0);
  /// Generates rows [row_begin, row_begin + rows) of a synthetic table
  /// (include/hawk_gen.h) directly in HBM; `rows` < 0 = the whole table.
  void generate_table(int hg_table, double sf, uint64_t seed, int64_t row_begin = 0,
                      int64_t rows = -1);
  /// CSV file -> device columns, parsed on the device with the reference's
  /// load_csv rules (storage_csv.cpp:111-155; include/hawk_b200_csv.h).
  void load_csv(const std::string& path, const std::string& name, const Schema& schema,
                const CsvOptions& options = {});
  void drop_table(const std::string& name);
  bool has_table(const std::string& name) const;
  const DeviceTable& table(const std::string& name) const;
  /// Catalog tables (schema + lexicon) for sql::parse_query / partition_into_pipelines.
  std::vector<TablePtr> catalog() const;

  /// execute_kernel_plan for a whole query: every pipeline in dependency
  /// order, `configs[i]` for pipeline i.
  Table execute(const PipelineSet& set, const std::vector<VariantConfiguration>& configs,
                ExecutionMetrics* metrics = nullptr);
  /// Same with one configuration per pipeline kind; the terminal pipeline's
  /// hash choice is propagated to the build descriptors (ir/passes.hpp:23-26).
  Table execute(const PipelineSet& set, const WorkloadConfig& config,
                ExecutionMetrics* metrics = nullptr);
  /// execute() returning plain columns: skips building the reference Table
  /// (whose finalize() hashes every column for its distinct counts).
  ResultColumns execute_columns(const PipelineSet& set, const std::vector<VariantConfiguration>& configs,
                                ExecutionMetrics* metrics = nullptr);
  /// Parses, partitions and executes a SQL query against the device store.
  Table run_sql(const std::string& sql, const WorkloadConfig& config,
                ExecutionMetrics* metrics = nullptr);

  /// Shard execution for multi-GPU: runs the query but stops before the
  /// result is finalised, returning the device partials (aggregations only).
  PartialResult execute_partial(const PipelineSet& set, const WorkloadConfig& config,
                                ExecutionMetrics* metrics = nullptr);
  /// Merges partials gathered from all shards and finalises the result Table.
  Table finalize_partials(const PipelineSet& set, const WorkloadConfig& config,
                          const std::vector<PartialResult>& parts);
  ResultColumns finalize_partials_columns(const PipelineSet& set, const WorkloadConfig& config,
                                          const std::vector<PartialResult>& parts);
  /// Multi-GPU execution over a fact-table shard per rank: runs the query on
  /// this rank's shard, gathers every rank's partial result to `root` with
  /// NCCL over device buffers (include/hawk_b200_comm.h) and merges it on the
  /// root's device. The root returns the query result; the other ranks an
  /// empty one (same columns, no rows).
  ResultColumns execute_sharded(const PipelineSet& set, const WorkloadConfig& config, hawk_comm* comm,
                                int root = 0, ExecutionMetrics* metrics = nullptr);
  /// Bumped by every change to the device store (plan caches key on it).
  uint64_t catalog_generation() const { return generation_; }

  /// Flushes L2 (timing hygiene).
  void flush_l2();

  struct Impl;  // opaque (engine.cpp)

 private:
  std::unique_ptr<Impl> impl_;
  int device_ = 0;
  uint64_t generation_ = 0;
  hawk_ctx* ctx_ = nullptr;
};

/// apply_variant over a whole PipelineSet: the terminal (probe-side)
/// pipeline's hash choice is propagated into the descriptors and imposed on
/// every build pipeline's HASH_PUT (ir/passes.hpp:23-26).
std::vector<PipelineProgram> apply_variants(const PipelineSet& set,
                                            const std::vector<VariantConfiguration>& configs,
                                            std::vector<HashTableDescriptor>& descriptors,
                                            std::vector<VariantConfiguration>* effective = nullptr);

/// CROSS_JOIN (planner_pipelines.cpp:337-352): a pair table of n_driver x
/// n_aux rows in driver-major order that replaces LOOP(driver) + CROSS_JOIN(aux).
struct CrossPairTable {
  std::string name;        // catalog name (unique per rewrite)
  int table = -1;          // its index in the rewritten PipelineSet::tables
  int driver = -1, aux = -1;
  int driver_columns = 0;  // pair columns [0, driver_columns) are the driver's
  std::vector<bool> used;  // pair columns the terminal program reads
};
/// The plan half of the CROSS_JOIN lowering: appends a pair-table catalog per
/// CROSS_JOIN of the terminal pipeline, reroutes CrossAux attributes to it and
/// drops the op. Needs no device; the identity when there is no CROSS_JOIN.
PipelineSet rewrite_cross_joins(const PipelineSet& set, std::vector<CrossPairTable>* pairs = nullptr);

/// Lowers one (variant-applied) program into the POD device descriptor; the
/// column slots are resolved against `tables` by the caller's binder.
struct LoweredProgram {
  hawk_pipeline pipe{};
  std::vector<std::pair<int, int>> column_of_slot;  // (storage table id, column)
  std::vector<int> agg_slot;       // lowered aggregate index -> device aggregate
  std::vector<int> probe_descriptor;  // device probe index -> descriptor id
  int count_agg = -1;              // a device COUNT aggregate (empty-input check)
  int unroll = 1;
};
LoweredProgram lower_program(const PipelineProgram& program, const PipelineSet& set);
/// Orders the probe chain by ascending match probability (inner joins
/// commute; a probe keyed by another probe's payload stays after it), so the
/// branched variants stop work on a row as early as possible.
void reorder_probes(LoweredProgram& lp, const std::vector<double>& match_prob);
/// Human-readable dump of a lowered device program (one op per line).
std::string describe(const hawk_pipeline& p);

// ---- optimizer ----------------------------

struct WorkloadQuery {
  std::string name;
  std::string sql;
};

struct LearnOptions {
  int max_iterations = 3;            // q
  bool early_termination = true;     // stop at the first unchanged sweep
  double prune_threshold_ms = 1000;  // slow-variant pruning
  int repetitions = 3;               // timed runs per query (median)
  /// After the descent, one coordinate pass over the projection and
  /// aggregation unroll factors {1, 2, 4} (outside the 32 / 896 space).
  bool unroll_pass = false;
  /// Starting configurations of the descent (Algorithm 1 line 1). Empty =
  /// the reference's default VariantConfiguration (every dimension's first
  /// value); more than one = restarts sharing one measurement cache, best
  /// result kept. Coordinate descent from the reference default can stall in
  /// a pruned region (e.g. TPC-H Q1: local_hash with wg=16/ht=1 is pruned, so
  /// global_hash wins dimension 2 and is never left).
  std::vector<WorkloadConfig> starts;
};

struct Measurement {
  WorkloadConfig config;
  double ms = std::numeric_limits<double>::infinity();  // sum over queries
  bool pruned = false;
  std::string error;
};

/// A dimension of the workload variant space; feature order = vector order.
struct Dimension {
  std::string name;
  std::vector<std::string> values;
  std::function<void(WorkloadConfig&, int)> set;
};
std::vector<Dimension> workload_dimensions();

/// measure_variant(config, workload, device): sum of
/// CUDA-event query times; failures and slow variants are +inf.
Measurement measure_variant(Engine& engine, const WorkloadConfig& config,
                            const std::vector<WorkloadQuery>& workload, const LearnOptions& opt);

struct LearnResult {
  WorkloadConfig best;
  double best_ms = std::numeric_limits<double>::infinity();
  int evaluations = 0;
  int sweeps = 0;
  std::vector<Measurement> trace;
};
/// Algorithm 1 coordinate descent, measurements cached
/// by configuration key, strict-< keeps the earlier value.
LearnResult learn_variant_configuration(Engine& engine, const std::vector<WorkloadQuery>& workload,
                                        const LearnOptions& opt);
/// Algorithm 1 over an abstract index space: dimension d takes values
/// 0..sizes[d]-1 in feature order; measurements cached by index vector.
struct IndexDescent {
  std::vector<int> best;
  double best_ms = std::numeric_limits<double>::infinity();
  int evaluations = 0;
  int sweeps = 0;
  std::vector<int> evaluations_per_sweep;
};
IndexDescent descend(const std::vector<int>& sizes, const LearnOptions& opt,
                     const std::vector<std::vector<int>>& starts,
                     const std::function<double(const std::vector<int>&)>& cost);
/// Algorithm 1 over any cost function (the learner above with `cost` =
/// measure_variant); used directly by the CPU tests with synthetic costs.
LearnResult coordinate_descent(const std::vector<Dimension>& dims, const LearnOptions& opt,
                               const std::function<Measurement(const WorkloadConfig&)>& cost);
/// The B200 starting point used as the learner's second start: single-pass
/// coalesced branched projections; local_hash, wg=256, ht=8, linear probing.
WorkloadConfig b200_start_config();
/// Brute force over explicit configurations.
LearnResult full_exploration(Engine& engine, const std::vector<WorkloadQuery>& workload,
                             const std::vector<WorkloadConfig>& space, const LearnOptions& opt);

/// The exploration / learning trace as CSV: index, projection, aggregation,
/// ms (inf = failed or pruned), status (ok / pruned / error), detail.
std::string trace_csv(const std::vector<Measurement>& trace);
/// Offline heuristic file: one `key=value` per line.
std::string save_config_text(const WorkloadConfig& c);
WorkloadConfig load_config_text(const std::string& text);

}  // namespace hawk::b200
