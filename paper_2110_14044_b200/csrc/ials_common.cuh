// ials_common.cuh -- small device helpers shared by the iALS++ kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define IALS_DEVI __device__ __forceinline__

// Checked builds (-DIALS_CHECKS, `python -m paper_2110_14044_b200.build --checked`):
// device-side bounds checks on every index-driven gather and scatter of the
// sweep kernels; a failure prints the site and traps (the launch then fails
// with an illegal-instruction error).  compute-sanitizer is not available on
// this GPU pool; the GPU test suite runs against the checked library instead.
#ifdef IALS_CHECKS
#include <cstdio>
#define IALS_CHECK(cond)                                                                    \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("IALS_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                             \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define IALS_CHECK(cond) \
  do {                   \
  } while (0)
#endif

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

// 32-byte read-only global load (LDG.E.256 on sm_100): one L1 wavefront per
// 32 B of a scattered row instead of two 16-byte loads; p 32-byte aligned
IALS_DEVI void ldg256(const float* p, float (&v)[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
                 "=f"(v[7])
               : "l"(p));
}

// Singular-row report: min over (side, row), first failing pivot of that row.
IALS_DEVI void report_singular(unsigned long long* err, int side, int row, int pivot) {
  unsigned long long key = (static_cast<unsigned long long>(side) << 62) |
                           (static_cast<unsigned long long>(static_cast<uint32_t>(row)) << 24) |
                           static_cast<unsigned long long>(pivot & 0xFFFFFF);
  atomicMin(err, key);
}

}  // namespace ials

namespace ials {
// Host f64 <-> device fp32 staging of ials_epoch_host64 (the reference's
// float64 model in place): 2-D strided casts, grid-stride over rows x cols.
// f64 -> fp32 rounds to nearest (what torch / NumPy .astype(float32) do).
__global__ void __launch_bounds__(256) k_f64_to_f32_2d(const double* __restrict__ src, int64_t lds,
                                                        float* __restrict__ dst, int64_t ldd,
                                                        int cols, int64_t rows) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[r * ldd + c] = __double2float_rn(src[r * lds + c]);
  }
}
__global__ void __launch_bounds__(256) k_f32_to_f64_2d(const float* __restrict__ src, int64_t lds,
                                                        double* __restrict__ dst, int64_t ldd,
                                                        int cols, int64_t rows) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[r * ldd + c] = (double)src[r * lds + c];
  }
}
}  // namespace ials
