// launch.cuh — maps a runtime variant point to its template instantiation.
// Each role's .cu file instantiates all 2 x 2 x 2 x 2 x 3 variant points
// (access x predication x table impl x hash fn x unroll).
#pragma once

#include <cuda_runtime.h>

#include "pipeline_kernel.cuh"

namespace hk {

struct LaunchShape {
  dim3 grid, block;
  size_t smem;
  void* jit_fn = nullptr;  // compiled program (jit.cu) instead of the AOT instantiation
};

template <int ROLE, int A, int P, int I, int H, int U>
cudaError_t launch_one(const KParams& kp, const LaunchShape& s, cudaStream_t st) {
  auto fn = pipeline_kernel<ROLE, A, P, I, H, U>;
  if (s.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)s.smem);
    if (e != cudaSuccess) return e;
  }
  fn<<<s.grid, s.block, s.smem, st>>>(kp);
  return cudaGetLastError();
}

template <int ROLE, int A, int P, int I, int H, int U>
cudaError_t occupancy_one(int block, size_t smem, int* ctas) {
  auto fn = pipeline_kernel<ROLE, A, P, I, H, U>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas, fn, block, smem);
}

// Calls F<ROLE, A, P, I, H, U>::run(args...) for the runtime point.
#define HK_DISPATCH_U(ROLE, A, P, I, H, CALL)                 \
  switch (unroll) {                                           \
    case 1: return CALL(ROLE, A, P, I, H, 1);                 \
    case 2: return CALL(ROLE, A, P, I, H, 2);                 \
    default: return CALL(ROLE, A, P, I, H, 4);                \
  }
#define HK_DISPATCH_H(ROLE, A, P, I, CALL)                                      \
  if (hfn == HAWK_MURMUR) { HK_DISPATCH_U(ROLE, A, P, I, HAWK_MURMUR, CALL) }   \
  else { HK_DISPATCH_U(ROLE, A, P, I, HAWK_MULTIPLY_SHIFT, CALL) }
#define HK_DISPATCH_I(ROLE, A, P, CALL)                                                 \
  if (impl == HAWK_LINEAR_PROBING) { HK_DISPATCH_H(ROLE, A, P, HAWK_LINEAR_PROBING, CALL) } \
  else { HK_DISPATCH_H(ROLE, A, P, HAWK_CUCKOO, CALL) }
#define HK_DISPATCH_P(ROLE, A, CALL)                                               \
  if (pred == HAWK_BRANCHED) { HK_DISPATCH_I(ROLE, A, HAWK_BRANCHED, CALL) }        \
  else { HK_DISPATCH_I(ROLE, A, HAWK_PREDICATED, CALL) }

// Per-role entry points (defined in k_<role>.cu). `access` selects the file
// half so instantiations compile in parallel.
cudaError_t launch_role(int role, int access, int pred, int impl, int hfn, int unroll,
                        const KParams& kp, const LaunchShape& s, cudaStream_t st);
cudaError_t occupancy_role(int role, int access, int pred, int impl, int hfn, int unroll,
                           int block, size_t smem, int* ctas);

#define HK_DECLARE_ROLE_ACCESS(NAME)                                                         \
  cudaError_t launch_##NAME(int pred, int impl, int hfn, int unroll, const KParams& kp,      \
                            const LaunchShape& s, cudaStream_t st);                          \
  cudaError_t occupancy_##NAME(int pred, int impl, int hfn, int unroll, int block,           \
                               size_t smem, int* ctas);

#define HK_DEFINE_ROLE_ACCESS(NAME, ROLE, A)                                                 \
  cudaError_t launch_##NAME(int pred, int impl, int hfn, int unroll, const KParams& kp,      \
                            const LaunchShape& s, cudaStream_t st) {                         \
    HK_DISPATCH_P(ROLE, A, HK_LAUNCH_CALL)                                                   \
  }                                                                                          \
  cudaError_t occupancy_##NAME(int pred, int impl, int hfn, int unroll, int block,           \
                               size_t smem, int* ctas) {                                     \
    HK_DISPATCH_P(ROLE, A, HK_OCC_CALL)                                                      \
  }
#define HK_LAUNCH_CALL(ROLE, A, P, I, H, U) launch_one<ROLE, A, P, I, H, U>(kp, s, st)
#define HK_OCC_CALL(ROLE, A, P, I, H, U) occupancy_one<ROLE, A, P, I, H, U>(block, smem, ctas)

#define HK_ROLE_NAMES(X)            \
  X(agg_local_seq, K_AGG_LOCAL, HAWK_SEQUENTIAL) \
  X(agg_local_coa, K_AGG_LOCAL, HAWK_COALESCED)  \
  X(agg_global_seq, K_AGG_GLOBAL, HAWK_SEQUENTIAL) \
  X(agg_global_coa, K_AGG_GLOBAL, HAWK_COALESCED)  \
  X(hagg_local_seq, K_HAGG_LOCAL, HAWK_SEQUENTIAL) \
  X(hagg_local_coa, K_HAGG_LOCAL, HAWK_COALESCED)  \
  X(hagg_global_seq, K_HAGG_GLOBAL, HAWK_SEQUENTIAL) \
  X(hagg_global_coa, K_HAGG_GLOBAL, HAWK_COALESCED)  \
  X(proj_single_seq, K_PROJECT_SINGLE, HAWK_SEQUENTIAL) \
  X(proj_single_coa, K_PROJECT_SINGLE, HAWK_COALESCED)  \
  X(count_seq, K_COUNT, HAWK_SEQUENTIAL) \
  X(count_coa, K_COUNT, HAWK_COALESCED)  \
  X(scatter_seq, K_PROJECT_SCATTER, HAWK_SEQUENTIAL) \
  X(scatter_coa, K_PROJECT_SCATTER, HAWK_COALESCED)  \
  X(put_seq, K_PUT_SINGLE, HAWK_SEQUENTIAL) \
  X(put_coa, K_PUT_SINGLE, HAWK_COALESCED)

#define HK_DECLARE_X(NAME, ROLE, A) HK_DECLARE_ROLE_ACCESS(NAME)
HK_ROLE_NAMES(HK_DECLARE_X)
#undef HK_DECLARE_X

}  // namespace hk
