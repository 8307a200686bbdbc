// passes.cpp — the transformation passes the reference declares but does not
// ship (/root/reference/proj/include/hawk/ir/passes.hpp:9-26; the listed
// src/ir_passes.cpp is missing, proj/CMakeLists.txt:23). Semantics follow
// SPEC.md:226-234 (apply_variant) and :257-260 (design decisions).
#include <algorithm>
#include <string>

#include "hawk/error.hpp"
#include "hawk/ir/passes.hpp"

namespace hawk {

namespace {

bool is_hash_op(PipelineOpKind k) {
  return k == PipelineOpKind::HashPut || k == PipelineOpKind::HashProbe ||
         k == PipelineOpKind::HashAggregate;
}

template <typename T, std::size_t N>
bool admissible(const T (&values)[N], int v) {
  return std::find(std::begin(values), std::end(values), v) != std::end(values);
}

}  // namespace

// (1) execution strategy: projection pipelines run single- or multi-pass,
// aggregation pipelines local or global hash aggregation.
PipelineProgram set_strategy(PipelineProgram program, Strategy strategy) {
  const bool projection_strategy =
      strategy == Strategy::SinglePass || strategy == Strategy::MultiPass;
  if (projection_strategy != (program.kind == PipelineKind::Projection))
    throw InvalidConfig(std::string("strategy ") + to_string(strategy) + " is not valid for a " +
                        to_string(program.kind) + " pipeline");
  program.strategy = strategy;
  return program;
}

// (2) memory access on the LOOP and every element access.
PipelineProgram set_memory_access(PipelineProgram program, MemoryAccess access) {
  program.memory_access = access;
  return program;
}

// (3) predication mode on every op — uniform by construction.
PipelineProgram set_predication(PipelineProgram program, PredicationMode mode) {
  program.predication = mode;
  for (PipelineOp& op : program.ops) op.mode = mode;
  return program;
}

// (4) hash table implementation and function on every hash op.
PipelineProgram set_hash_tables(PipelineProgram program, HashTableImpl impl,
                                HashFunctionKind function) {
  for (PipelineOp& op : program.ops)
    if (is_hash_op(op.kind)) {
      op.table_impl = impl;
      op.hash_function = function;
    }
  return program;
}

// (5) unrolling, last so replicas inherit the final modes: the
// per-tuple body (every op after the head LOOP) is replicated `factor` times
// with access offsets 0..factor-1 and LOOP.step = factor.
PipelineProgram unroll(PipelineProgram program, int factor) {
  if (!admissible(kUnrollFactors, factor))
    throw InvalidConfig("unroll factor " + std::to_string(factor) + " not in {1,2,4}");
  if (program.ops.empty() || program.ops.front().kind != PipelineOpKind::Loop)
    throw UnsupportedPlan("pipeline must start with LOOP");
  if (program.unroll_factor != 1) throw InvalidConfig("program is already unrolled");
  std::vector<PipelineOp> body(program.ops.begin() + 1, program.ops.end());
  std::vector<PipelineOp> ops;
  ops.reserve(1 + body.size() * static_cast<std::size_t>(factor));
  PipelineOp loop = program.ops.front();
  loop.loop_step = factor;
  ops.push_back(loop);
  for (int o = 0; o < factor; ++o)
    for (PipelineOp op : body) {
      op.offset = o;
      ops.push_back(std::move(op));
    }
  program.ops = std::move(ops);
  program.unroll_factor = factor;
  return program;
}

PipelineProgram apply_variant(const PipelineProgram& program, const VariantConfiguration& config) {
  if (!admissible(kThreadMultipliers, config.thread_multiplier))
    throw InvalidConfig("thread multiplier " + std::to_string(config.thread_multiplier));
  if (!admissible(kWorkGroupSizes, config.work_group_size))
    throw InvalidConfig("work group size " + std::to_string(config.work_group_size));
  if (!admissible(kTableCountMultipliers, config.hash_table_count_multiplier))
    throw InvalidConfig("hash table count multiplier " +
                        std::to_string(config.hash_table_count_multiplier));
  PipelineProgram p = set_strategy(program, config.strategy);
  p = set_memory_access(std::move(p), config.memory_access);
  p = set_predication(std::move(p), config.predication);
  p = set_hash_tables(std::move(p), config.hash_table_impl, config.hash_function);
  if (config.unroll_factor != 1) p = unroll(std::move(p), config.unroll_factor);
  else if (!admissible(kUnrollFactors, config.unroll_factor))
    throw InvalidConfig("unroll factor");
  return p;
}

void propagate_hash_choice(std::vector<HashTableDescriptor>& descriptors,
                           const PipelineProgram& program) {
  for (const PipelineOp& op : program.ops) {
    if (!is_hash_op(op.kind) || op.descriptor < 0) continue;
    if (static_cast<std::size_t>(op.descriptor) >= descriptors.size())
      throw DivergentPlan("hash op references unknown descriptor " + std::to_string(op.descriptor));
    descriptors[static_cast<std::size_t>(op.descriptor)].impl = op.table_impl;
    descriptors[static_cast<std::size_t>(op.descriptor)].function = op.hash_function;
  }
}

}  // namespace hawk
