// jit.cuh — host interface of the compiled-program path (jit.cu).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "interp.cuh"

namespace hk {

// Generates, compiles (NVRTC, sm_100a) and caches the kernel of one pipeline
// role for one variant point; *fn is a CUfunction.
int32_t jit_function(const KParams& kp, int role, const hawk_variant& v, int block, void** fn,
                     std::string* error);
int32_t jit_occupancy(void* fn, int block, size_t smem, int* ctas);
int32_t jit_launch(void* fn, const KParams& kp, dim3 grid, dim3 block, size_t smem,
                   cudaStream_t stream);
// The generated translation unit (for inspection and tests).
std::string jit_source(const KParams& kp, int role, const hawk_variant& v);
// NVRTC compile without loading (needs libnvrtc only; no GPU).
int32_t jit_compile_only(const KParams& kp, int role, const hawk_variant& v, size_t* cubin_bytes,
                         std::string* error);

}  // namespace hk
