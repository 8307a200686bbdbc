// k_role.cu — compiled once per (role, access) pair (see csrc/Makefile);
// instantiates the pipeline kernel for every predication x table impl x
// hash function x unroll point of that pair.
#include "launch.cuh"

#ifndef HK_NAME
#error "compile with -DHK_NAME=<role_access> -DHK_ROLE=<K_*> -DHK_ACCESS=<HAWK_*>"
#endif

namespace hk {
#define HK_EXPAND_DEFINE(N, R, A) HK_DEFINE_ROLE_ACCESS(N, R, A)
HK_EXPAND_DEFINE(HK_NAME, HK_ROLE, HK_ACCESS)
}  // namespace hk
