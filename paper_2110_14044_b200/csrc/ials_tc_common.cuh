// ials_tc_common.cuh -- pieces shared by the tensor-core sweep kernels
// (ials_sweep_tc4.cuh, ials_sweep_pk.cuh, ials_sweep_wb.cuh): the aligned
// dynamic shared-memory base, the K-major no-swizzle panel operand layout and
// the packed alpha0 * slab[pi, pi] template.
#pragma once
#include "ials_sweep.cuh"
#include "ials_umma.cuh"

namespace ials {

// 128B-swizzled operands need 1024-byte aligned atoms: align the dynamic
// shared-memory base explicitly (the launch requests 1 KB of slack).
IALS_DEVI char* tc_smem_base(char* raw) {
  const uint32_t a = smem_u32(raw);
  return raw + ((1024u - (a & 1023u)) & 1023u);
}

// panel operand (128 x 8, K-major, no swizzle): 8-row groups of 256 B, two
// 4-element K chunks 128 B apart.
IALS_DEVI int pa_index(int m, int q) { return (m >> 3) * 64 + (q >> 2) * 32 + (m & 7) * 4 + (q & 3); }

constexpr int kTcPKS = 8448;  // packed floats per 128x128 lower triangle

IALS_DEVI int pk_off(int i) {
  const int q = i >> 2;
  return 4 * (2 * q * (q + 1) + (i - 4 * q) * (q + 1));
}

// alpha0 * slab[pi, pi] (identity on the padding) as packed lower rows: the
// same 33 KB for every row of the pass, read by the sweep kernels through L1.
__global__ void k_tc_template(SweepParams p, float* tpl) {
  const int i = blockIdx.x, b = p.b;
  for (int c = threadIdx.x; c < 4 * ((i >> 2) + 1); c += blockDim.x) {
    float v;
    if (i < b && c < b)
      v = p.alpha0 * p.slab[(size_t)(p.b0 + i) * b + c];
    else
      v = (c == i) ? 1.f : 0.f;
    tpl[pk_off(i) + c] = v;
  }
}

}  // namespace ials
