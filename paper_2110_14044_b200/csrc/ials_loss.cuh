// ials_loss.cuh -- device pieces of compute_loss (model.py:168-188), fp64
// accumulation with a fixed-order final reduction (deterministic).
#pragma once
#include "ials_common.cuh"

namespace ials {

constexpr int kLossBlocks = 296;

__device__ __forceinline__ double block_sum_d(double v) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// sum_e a_e (<w_u, h_i> - y_e)^2 over the user-major CSR
__global__ void __launch_bounds__(256)
    k_loss_observed(int n_rows, const int* __restrict__ ptr, const int* __restrict__ cols,
                    const float* __restrict__ labels, const float* __restrict__ weights,
                    const float* __restrict__ W, int ldw, const float* __restrict__ H, int ldh,
                    int d, double* __restrict__ red) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int row = gw; row < n_rows; row += nw) {
    const float* wr = W + (size_t)row * ldw;
    for (int e = ptr[row]; e < ptr[row + 1]; ++e) {
      const float* hr = H + (size_t)cols[e] * ldh;
      float s = 0.f;
      for (int t = lane; t < d; t += 32) s = fmaf(wr[t], hr[t], s);
      s = warp_sum(s);
      if (lane == 0) {
        const double y = labels ? labels[e] : 1.0;
        const double a = weights ? weights[e] : 1.0;
        const double err = (double)s - y;
        acc += a * err * err;
      }
    }
  }
  const double t = block_sum_d(acc);
  if (threadIdx.x == 0) red[blockIdx.x] = t;
}

__global__ void __launch_bounds__(256)
    k_loss_dot(const float* __restrict__ a, const float* __restrict__ b, size_t n,
               double* __restrict__ red) {
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    acc += (double)a[i] * (double)b[i];
  const double t = block_sum_d(acc);
  if (threadIdx.x == 0) red[blockIdx.x] = t;
}

// sum_r lam_r |M_r|^2
__global__ void __launch_bounds__(256)
    k_loss_rownorm(const float* __restrict__ M, int n, int ld, int d,
                   const float* __restrict__ lam, double* __restrict__ red) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int r = gw; r < n; r += nw) {
    const float* mr = M + (size_t)r * ld;
    double s = 0.0;
    for (int t = lane; t < d; t += 32) s += (double)mr[t] * (double)mr[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) acc += (double)lam[r] * s;
  }
  const double t = block_sum_d(acc);
  if (threadIdx.x == 0) red[blockIdx.x] = t;
}

__global__ void k_loss_final(const double* __restrict__ red, double* __restrict__ out) {
  if (threadIdx.x < 4) {
    double s = 0.0;
    for (int i = 0; i < kLossBlocks; ++i) s += red[threadIdx.x * kLossBlocks + i];
    out[threadIdx.x] = s;
  }
}

}  // namespace ials
