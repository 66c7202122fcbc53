// ials_common.cuh -- small device helpers shared by the iALS++ kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define IALS_DEVI __device__ __forceinline__

namespace ials {

constexpr int kNumSMs = 148;

#define IALS_SMEM_U32_DEFINED
IALS_DEVI uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async 16 B / 4 B global -> shared (LDGSTS); .cg bypasses L1 for 16 B.
IALS_DEVI void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
IALS_DEVI void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src));
}
IALS_DEVI void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
IALS_DEVI void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Barrier over one "row team" (NW warps).  Team 0..k use named barriers 1..k+1;
// a single-warp team only needs __syncwarp.
template <int NW>
IALS_DEVI void team_sync(int team) {
  if constexpr (NW == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(team + 1), "r"(NW * 32) : "memory");
  }
}

IALS_DEVI float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G>
IALS_DEVI float group_sum(float v) {   // sum over aligned groups of G lanes
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Singular-row report: min over (side, row), first failing pivot of that row.
IALS_DEVI void report_singular(unsigned long long* err, int side, int row, int pivot) {
  unsigned long long key = (static_cast<unsigned long long>(side) << 62) |
                           (static_cast<unsigned long long>(static_cast<uint32_t>(row)) << 24) |
                           static_cast<unsigned long long>(pivot & 0xFFFFFF);
  atomicMin(err, key);
}

}  // namespace ials
