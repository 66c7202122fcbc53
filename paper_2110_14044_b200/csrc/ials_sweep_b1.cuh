// ials_sweep_b1.cuh -- block width 1 (the iCD special case, configs[2] b=1):
// a scalar Newton step per row, no matrix work.  For row r and column j = b0:
//   H = sum a_k h_k^2 + alpha0 G_jj + lam_r,  g = sum rho_k h_k + alpha0 (U_r . G_:j)
//   + lam_r U_rj,  d = g / H,  U_rj -= d,  yhat_k -= h_k d
// (solvers.py:152-186 with |pi| = 1; identical to the reference's iCD update
// _icd_side, solvers.py:189-207).  Light rows: one warp per row; heavy rows:
// one 256-thread CTA per row.
#pragma once
#include "ials_sweep.cuh"

namespace ials {

IALS_DEVI void b1_entry(const SweepParams& p, int e, float& h, float& a, int& pos, float& rho) {
  const int col = __ldg(p.side.cols + e);
  h = __ldg(p.fixed + (size_t)col * p.ldf + p.fb0);
  a = p.side.weights ? __ldg(p.side.weights + e) : 1.f;
  const float y = p.side.labels ? __ldg(p.side.labels + e) : 1.f;
  pos = p.side.pos ? __ldg(p.side.pos + e) : e;
  rho = a * (p.cache[pos] - y);
}

// sum over entries e = first, first + stride, ... < end of a h^2 and rho h,
// four entries in flight per thread
IALS_DEVI void b1_accumulate(const SweepParams& p, int first, int end, int stride, float& hh,
                             double& gg) {
  int e = first;
  for (; e + 3 * stride < end; e += 4 * stride) {
    float h[4], a[4], rho[4];
    int pos[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) b1_entry(p, e + u * stride, h[u], a[u], pos[u], rho[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      hh = fmaf(a[u] * h[u], h[u], hh);
      gg = fma((double)rho[u], (double)h[u], gg);
    }
  }
  for (; e < end; e += stride) {
    float h, a, rho;
    int pos;
    b1_entry(p, e, h, a, pos, rho);
    hh = fmaf(a * h, h, hh);
    gg = fma((double)rho, (double)h, gg);
  }
}

IALS_DEVI void b1_cache(const SweepParams& p, int first, int end, int stride, float dl) {
  int e = first;
  for (; e + 3 * stride < end; e += 4 * stride) {
    int col[4], pos[4];
    float h[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      col[u] = __ldg(p.side.cols + e + u * stride);
      pos[u] = p.side.pos ? __ldg(p.side.pos + e + u * stride) : e + u * stride;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) h[u] = __ldg(p.fixed + (size_t)col[u] * p.ldf + p.fb0);
#pragma unroll
    for (int u = 0; u < 4; ++u) p.cache[pos[u]] -= h[u] * dl;
  }
  for (; e < end; e += stride) {
    const int col = __ldg(p.side.cols + e);
    const float h = __ldg(p.fixed + (size_t)col * p.ldf + p.fb0);
    const int pos = p.side.pos ? __ldg(p.side.pos + e) : e;
    p.cache[pos] -= h * dl;
  }
}

IALS_DEVI float b1_solve(const SweepParams& p, int row, float hh, double gg) {
  const float lam = p.side.lam[row];
  const float H = hh + p.alpha0 * p.slab[p.b0] + lam;
  float* w = p.own + (size_t)row * p.ldo + p.b0;
  const double g = gg + (double)p.proj[row] + (double)lam * (double)(*w);
  float Hs = H;
  if (!(Hs > 0.f) || !(Hs < 3.0e38f)) {
    report_singular(p.err, p.side_id, row, 0);
    Hs = 1.f;
  }
  const float dl = (float)(g / (double)Hs);
  *w -= dl;
  p.drow[row] = dl;   // the entry-parallel cache kernel (k_b1_cache_flat) reads d by row
  return dl;
}

__global__ void __launch_bounds__(256) k_sweep_b1(SweepParams p) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int task = gw; task < p.n_light; task += nw) {
    const int row = p.light_rows[task];
    const int e0 = p.side.ptr[row], e1 = p.side.ptr[row + 1];
    float hh = 0.f;
    double gg = 0.0;
    b1_accumulate(p, e0 + lane, e1, 32, hh, gg);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      hh += __shfl_xor_sync(0xffffffffu, hh, o);
      gg += __shfl_xor_sync(0xffffffffu, gg, o);
    }
    float dl = 0.f;
    if (lane == 0) dl = b1_solve(p, row, hh, gg);
    dl = __shfl_sync(0xffffffffu, dl, 0);
    if (!p.b1_flat) b1_cache(p, e0 + lane, e1, 32, dl);
  }
}

// heavy rows: per slice (one warp) partial sums -> per row fixed-order sum
// and solve -> per slice cache update
__global__ void __launch_bounds__(256) k_b1_partial(SweepParams p) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int sl = gw; sl < p.n_slices; sl += nw) {
    float hh = 0.f;
    double gg = 0.0;
    b1_accumulate(p, p.slice_begin[sl] + lane, p.slice_end[sl], 32, hh, gg);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      hh += __shfl_xor_sync(0xffffffffu, hh, o);
      gg += __shfl_xor_sync(0xffffffffu, gg, o);
    }
    if (lane == 0) {
      p.hpart[sl] = hh;
      p.gpart[sl] = gg;
    }
  }
}

// warp per heavy row: lanes stride the row's slices, then a fixed shuffle
// tree (deterministic; the longest rows have hundreds of slices)
__global__ void __launch_bounds__(256) k_b1_solve(SweepParams p) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int h = gw; h < p.n_heavy; h += nw) {
    float hh = 0.f;
    double gg = 0.0;
    for (int sl = p.heavy_slice0[h] + lane; sl < p.heavy_slice0[h + 1]; sl += 32) {
      hh += p.hpart[sl];
      gg += p.gpart[sl];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      hh += __shfl_xor_sync(0xffffffffu, hh, o);
      gg += __shfl_xor_sync(0xffffffffu, gg, o);
    }
    if (lane == 0) p.hdelta[h] = b1_solve(p, p.heavy_rows[h], hh, gg);
  }
}

__global__ void __launch_bounds__(256) k_b1_cache(SweepParams p) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int sl = gw; sl < p.n_slices; sl += nw)
    b1_cache(p, p.slice_begin[sl] + lane, p.slice_end[sl], 32, p.hdelta[p.slice_heavy[sl]]);
}

// The pass's cache update walked in the OTHER side's entry order (x_rows = the
// fixed side's row of each entry, x_cols = this side's row, x_pos = the cache
// slot, NULL when that order is the cache's own): yhat -= f_u d_i with the
// cache and the ids streamed, f_u constant along a run and d (n_rows floats)
// resident in L1 / L2 -- the item pass otherwise scatters 4-byte updates over
// the cache through `pos`, a 32-byte sector each.  Four entries per thread in
// flight; every entry is written once (no atomics, deterministic).
template <bool SWAP>
__global__ void __launch_bounds__(256) k_b1_cache_flat(SweepParams p, long long nnz) {
  // SWAP: the other side's order; else this side's own order (rows = this side's row of
  // each entry), which only takes the update off the row's serial chain
  const int* __restrict__ FI = SWAP ? p.x_rows : p.side.cols;   // fixed-side id
  const int* __restrict__ DI = SWAP ? p.x_cols : p.side.rows;   // this side's row (d index)
  const int* __restrict__ PS = SWAP ? p.x_pos : p.side.pos;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; e + 3 * stride < nnz; e += 4 * stride) {
    int u[4], i[4];
    long long pos[4];
    float f[4], dv[4], c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u[k] = __ldg(FI + e + k * stride);
      i[k] = __ldg(DI + e + k * stride);
      pos[k] = PS ? (long long)__ldg(PS + e + k * stride) : e + k * stride;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      f[k] = __ldg(p.fixed + (size_t)u[k] * p.ldf + p.fb0);
      dv[k] = p.drow[i[k]];
      c[k] = p.cache[pos[k]];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) p.cache[pos[k]] = c[k] - f[k] * dv[k];
  }
  for (; e < nnz; e += stride) {
    const int u = __ldg(FI + e), i = __ldg(DI + e);
    const long long pos = PS ? (long long)__ldg(PS + e) : e;
    p.cache[pos] -= __ldg(p.fixed + (size_t)u * p.ldf + p.fb0) * p.drow[i];
  }
}

}  // namespace ials
