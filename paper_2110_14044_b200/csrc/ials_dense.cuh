// ials_dense.cuh -- K-pred (score-cache recompute), K-slab (partial Gramian)
// and K-proj (alpha0 * U @ slab), FP32 SIMT versions.
#pragma once
#include "ials_common.cuh"

namespace ials {

// ---------------------------------------------------------------- K-pred
// compute_predictions (model.py:153-165): out[e] = <W[row], H[cols[e]]> over
// the user-major CSR.  One warp per row (grid-stride); a group of LPN lanes
// per entry, each lane holding NV float4 of the row of W in registers.
// Work items are rows (seg_row == nullptr: item t = row t, entries ptr[t..t+1))
// or row segments (row seg_row[t], entries [seg_beg[t], seg_end[t])) so that a
// long row is spread over many warps.
struct Items {
  const int* ptr;
  const int* seg_row;
  const int* seg_beg;
  const int* seg_end;
  IALS_DEVI void get(int t, int& row, int& e0, int& e1) const {
    if (seg_row) {
      row = __ldg(seg_row + t); e0 = __ldg(seg_beg + t); e1 = __ldg(seg_end + t);
    } else {
      row = t; e0 = __ldg(ptr + t); e1 = __ldg(ptr + t + 1);
    }
  }
};

template <int LPN, int NV>
__global__ void __launch_bounds__(256)
    k_pred_vec(int n_items, Items it, const int* __restrict__ cols,
               const float* __restrict__ W, int ldw, const float* __restrict__ H, int ldh,
               int d, float* __restrict__ out) {
  constexpr int GPW = 32 / LPN;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int sub = lane / LPN, gl = lane % LPN;
  const int d4 = d >> 2;
  for (int t = gw; t < n_items; t += nw) {
    int row, e0, e1;
    it.get(t, row, e0, e1);
    float4 w[NV];
    const float4* wr = reinterpret_cast<const float4*>(W + (size_t)row * ldw);
#pragma unroll
    for (int m = 0; m < NV; ++m) {
      const int v = gl + m * LPN;
      w[m] = v < d4 ? __ldg(wr + v) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if constexpr (NV != 8) {   // one entry per step
      for (int eb = e0; eb < e1; eb += GPW) {
        const int e = eb + sub;
        float s = 0.f;
        if (e < e1) {
          const float4* hr = reinterpret_cast<const float4*>(H + (size_t)__ldg(cols + e) * ldh);
#pragma unroll
          for (int m = 0; m < NV; ++m) {
            const int v = gl + m * LPN;
            if (v < d4) {
              const float4 h = __ldg(hr + v);
              s = fmaf(w[m].x, h.x, s);
              s = fmaf(w[m].y, h.y, s);
              s = fmaf(w[m].z, h.z, s);
              s = fmaf(w[m].w, h.w, s);
            }
          }
        }
        s = group_sum<LPN>(s);
        if (e < e1 && gl == 0) out[e] = s;
      }
    } else {
    // two entries per group per step: both rows' loads are in flight before
    // the first dot product (latency-bound gathers); the next step's column
    // ids are loaded a step ahead.  Per entry the same fixed-order sum
    // (measured per epoch: d = 1024 (NV 8) 3.57 -> 2.70 ms; slower at NV 16,
    // d = 2048: 8.4 -> 17.7 ms, two rows of registers halve the occupancy; and
    // at NV 4, d = 64..512: 1.41 -> 2.04 ms at d = 512 -- NV 8 only).
    int nc0 = (e0 + sub < e1) ? __ldg(cols + e0 + sub) : -1;
    int nc1 = (e0 + GPW + sub < e1) ? __ldg(cols + e0 + GPW + sub) : -1;
    for (int eb = e0; eb < e1; eb += 2 * GPW) {
      const int c0 = nc0, c1 = nc1;
      {
        const int f0 = eb + 2 * GPW + sub, f1 = f0 + GPW;
        nc0 = f0 < e1 ? __ldg(cols + f0) : -1;
        nc1 = f1 < e1 ? __ldg(cols + f1) : -1;
      }
      float4 h0[NV], h1[NV];
      const float4* hr0 = reinterpret_cast<const float4*>(H + (size_t)max(c0, 0) * ldh);
      const float4* hr1 = reinterpret_cast<const float4*>(H + (size_t)max(c1, 0) * ldh);
#pragma unroll
      for (int m = 0; m < NV; ++m) {
        const int v = gl + m * LPN;
        h0[m] = (c0 >= 0 && v < d4) ? __ldg(hr0 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
        h1[m] = (c1 >= 0 && v < d4) ? __ldg(hr1 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float s0 = 0.f, s1 = 0.f;
#pragma unroll
      for (int m = 0; m < NV; ++m) {
        const int v = gl + m * LPN;
        if (v < d4) {
          s0 = fmaf(w[m].x, h0[m].x, s0);
          s0 = fmaf(w[m].y, h0[m].y, s0);
          s0 = fmaf(w[m].z, h0[m].z, s0);
          s0 = fmaf(w[m].w, h0[m].w, s0);
          s1 = fmaf(w[m].x, h1[m].x, s1);
          s1 = fmaf(w[m].y, h1[m].y, s1);
          s1 = fmaf(w[m].z, h1[m].z, s1);
          s1 = fmaf(w[m].w, h1[m].w, s1);
        }
      }
      s0 = group_sum<LPN>(s0);
      s1 = group_sum<LPN>(s1);
      if (c0 >= 0 && gl == 0) out[eb + sub] = s0;
      if (c1 >= 0 && gl == 0) out[eb + GPW + sub] = s1;
    }
    }
  }
}

__global__ void __launch_bounds__(256)
    k_pred_scalar(int n_items, Items it, const int* __restrict__ cols,
                  const float* __restrict__ W, int ldw, const float* __restrict__ H, int ldh,
                  int d, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < n_items; t += nw) {
    int row, e0, e1;
    it.get(t, row, e0, e1);
    const float* wr = W + (size_t)row * ldw;
    for (int e = e0; e < e1; ++e) {
      const float* hr = H + (size_t)cols[e] * ldh;
      float s = 0.f;
      for (int t = lane; t < d; t += 32) s = fmaf(wr[t], hr[t], s);
      s = warp_sum(s);
      if (lane == 0) out[e] = s;
    }
  }
}

// ---------------------------------------------------------------- K-corr
// Dual-cache delta correction of the sharded path:
// out[e] += <A[row, b0:b0+b], D[cols[e], 0:b]> over a (local) CSR, where D is
// the change of the other side's column block in the previous half-epoch.
// The same correction for b <= 128 with 16-byte rows (b0, lda, ldd, b multiples
// of 4): a warp keeps its segment's A[row, b0:b0+b] in registers (16 floats
// per lane) and takes 4 entries per step (8 lanes each), the next step's
// column ids loaded a step ahead, so the D-row gathers of a step are all in
// flight together instead of one warp-wide dot product and reduction per entry.
__global__ void __launch_bounds__(256)
    k_cache_correct_v(int n_items, Items it, const int* __restrict__ cols,
                      const float* __restrict__ A, int lda, int b0, const float* __restrict__ D,
                      int ldd, int b, float* __restrict__ out) {
  const int lane = threadIdx.x & 31, g = lane & 7, sub = lane >> 3;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < n_items; t += nw) {
    int row, e0, e1;
    it.get(t, row, e0, e1);
    const float* ar = A + (size_t)row * lda + b0;
    float4 av[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = 32 * q + 4 * g;
      av[q] = c < b ? __ldg(reinterpret_cast<const float4*>(ar + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    int ncol = e0 + sub < e1 ? __ldg(cols + e0 + sub) : -1;
    for (int eb = e0; eb < e1; eb += 4) {
      const int col = ncol;
      ncol = eb + 4 + sub < e1 ? __ldg(cols + eb + 4 + sub) : -1;
      float s = 0.f;
      if (col >= 0) {
        const float* dr = D + (size_t)col * ldd;
        float4 x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = 32 * q + 4 * g;
          x[q] = c < b ? __ldg(reinterpret_cast<const float4*>(dr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          s = fmaf(av[q].x, x[q].x, s);
          s = fmaf(av[q].y, x[q].y, s);
          s = fmaf(av[q].z, x[q].z, s);
          s = fmaf(av[q].w, x[q].w, s);
        }
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (col >= 0 && g == 0) out[eb + sub] += s;
    }
  }
}

__global__ void __launch_bounds__(256)
    k_cache_correct(int n_items, Items it, const int* __restrict__ cols,
                    const float* __restrict__ A, int lda, int b0, const float* __restrict__ D,
                    int ldd, int b, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = gw; t < n_items; t += nw) {
    int row, e0, e1;
    it.get(t, row, e0, e1);
    const float* ar = A + (size_t)row * lda + b0;
    float areg[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int j = lane + 32 * m;
      areg[m] = j < b ? ar[j] : 0.f;
    }
    for (int e = e0; e < e1; ++e) {
      const float* dr = D + (size_t)cols[e] * ldd;
      float s = 0.f;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int j = lane + 32 * m;
        if (j < b) s = fmaf(areg[m], __ldg(dr + j), s);
      }
      s = warp_sum(s);
      if (lane == 0) out[e] += s;
    }
  }
}

// ---------------------------------------------------------------- K-slab
// partial_gramian (linalg.py:39-45): slab[t][j] = sum_r M[r][t] M[r][b0+j].
// Split-K over rows; each CTA writes a 64x64 partial tile, a second kernel
// sums the splits in a fixed order (deterministic).
constexpr int GT = 64, GK = 16;

__global__ void __launch_bounds__(256)
    k_slab_partial(const float* __restrict__ M, int n, int ldm, int d, int b0, int b,
                   int rows_per_split, float* __restrict__ part) {
  __shared__ __align__(16) float As[GK][GT + 4];
  __shared__ __align__(16) float Bs[GK][GT + 4];
  const int t0 = blockIdx.x * GT, j0 = blockIdx.y * GT, split = blockIdx.z;
  const int r_beg = split * rows_per_split;
  const int r_end = min(n, r_beg + rows_per_split);
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  float acc[4][4] = {};
  for (int r0 = r_beg; r0 < r_end; r0 += GK) {
    for (int i = tid; i < GK * GT; i += 256) {
      const int rr = i / GT, cc = i % GT;
      const int r = r0 + rr;
      const bool rok = r < r_end;
      As[rr][cc] = (rok && t0 + cc < d) ? M[(size_t)r * ldm + t0 + cc] : 0.f;
      Bs[rr][cc] = (rok && j0 + cc < b) ? M[(size_t)r * ldm + b0 + j0 + cc] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < GK; ++rr) {
      const float4 a = *reinterpret_cast<const float4*>(&As[rr][ty * 4]);
      const float4 c = *reinterpret_cast<const float4*>(&Bs[rr][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], cv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* out = part + (size_t)split * d * b;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + ty * 4 + i;
    if (t >= d) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int jj = j0 + tx * 4 + j;
      if (jj < b) out[(size_t)t * b + jj] = acc[i][j];
    }
  }
}

// Narrow block widths (b <= 16): 128 (t) x 16 (j) tiles, 32 rows per
// k-step staged in shared memory; each thread owns 4 (t) x 2 (j) outputs.
__global__ void __launch_bounds__(256)
    k_slab_narrow(const float* __restrict__ M, int n, int ldm, int d, int b0, int b,
                  int rows_per_split, float* __restrict__ part) {
  __shared__ __align__(16) float As[32][128 + 4];
  __shared__ __align__(16) float Bs[32][16];
  const int t0 = blockIdx.x * 128, split = blockIdx.y;
  const int r_beg = split * rows_per_split;
  const int r_end = min(n, r_beg + rows_per_split);
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;   // t = 4tx.., j = 2ty..
  float acc[4][2] = {};
  for (int r0 = r_beg; r0 < r_end; r0 += 32) {
    for (int i = tid; i < 32 * 32; i += 256) {           // 32 rows x 32 float4
      const int rr = i >> 5, c4 = i & 31, r = r0 + rr, t = t0 + 4 * c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < r_end) {
        const float* src = M + (size_t)r * ldm + t;
        if (t + 3 < d && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
          v = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          if (t < d) v.x = src[0];
          if (t + 1 < d) v.y = src[1];
          if (t + 2 < d) v.z = src[2];
          if (t + 3 < d) v.w = src[3];
        }
      }
      *reinterpret_cast<float4*>(&As[rr][4 * c4]) = v;
    }
    for (int i = tid; i < 32 * 16; i += 256) {
      const int rr = i >> 4, j = i & 15, r = r0 + rr;
      Bs[rr][j] = (r < r_end && j < b) ? M[(size_t)r * ldm + b0 + j] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const float4 a = *reinterpret_cast<const float4*>(&As[rr][4 * tx]);
      const float2 c = *reinterpret_cast<const float2*>(&Bs[rr][2 * ty]);
      acc[0][0] = fmaf(a.x, c.x, acc[0][0]); acc[0][1] = fmaf(a.x, c.y, acc[0][1]);
      acc[1][0] = fmaf(a.y, c.x, acc[1][0]); acc[1][1] = fmaf(a.y, c.y, acc[1][1]);
      acc[2][0] = fmaf(a.z, c.x, acc[2][0]); acc[2][1] = fmaf(a.z, c.y, acc[2][1]);
      acc[3][0] = fmaf(a.w, c.x, acc[3][0]); acc[3][1] = fmaf(a.w, c.y, acc[3][1]);
    }
    __syncthreads();
  }
  float* out = part + (size_t)split * d * b;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + 4 * tx + i;
    if (t >= d) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int jj = 2 * ty + j;
      if (jj < b) out[(size_t)t * b + jj] = acc[i][j];
    }
  }
}

// Narrow block widths: proj = alpha0 * own @ slab with 128 (rows) x 16 (j)
// output tiles; K = d in steps of 32 staged in shared memory.
__global__ void __launch_bounds__(256)
    k_project_narrow(const float* __restrict__ own, int n_rows, int ldo, int d,
                     const float* __restrict__ slab, int b, float alpha0, float* __restrict__ proj) {
  __shared__ __align__(16) float As[32][128 + 4];   // As[k][r]
  __shared__ __align__(16) float Bs[32][16];        // Bs[k][j]
  const int r0 = blockIdx.x * 128;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  float acc[4][2] = {};
  for (int k0 = 0; k0 < d; k0 += 32) {
    for (int i = tid; i < 128 * 32; i += 256) {
      const int rr = i >> 5, kk = i & 31, r = r0 + rr, k = k0 + kk;
      As[kk][rr] = (r < n_rows && k < d) ? own[(size_t)r * ldo + k] : 0.f;
    }
    for (int i = tid; i < 32 * 16; i += 256) {
      const int kk = i >> 4, j = i & 15, k = k0 + kk;
      Bs[kk][j] = (k < d && j < b) ? slab[(size_t)k * b + j] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[kk][4 * tx]);
      const float2 c = *reinterpret_cast<const float2*>(&Bs[kk][2 * ty]);
      acc[0][0] = fmaf(a.x, c.x, acc[0][0]); acc[0][1] = fmaf(a.x, c.y, acc[0][1]);
      acc[1][0] = fmaf(a.y, c.x, acc[1][0]); acc[1][1] = fmaf(a.y, c.y, acc[1][1]);
      acc[2][0] = fmaf(a.z, c.x, acc[2][0]); acc[2][1] = fmaf(a.z, c.y, acc[2][1]);
      acc[3][0] = fmaf(a.w, c.x, acc[3][0]); acc[3][1] = fmaf(a.w, c.y, acc[3][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + 4 * tx + i;
    if (r >= n_rows) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int jj = 2 * ty + j;
      if (jj < b) proj[(size_t)r * b + jj] = alpha0 * acc[i][j];
    }
  }
}

__global__ void k_reduce_splits(const float* __restrict__ part, int nsplit, size_t count,
                                float* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < nsplit; ++k) s += part[(size_t)k * count + i];
    out[i] = s;
  }
}

// ---------------------------------------------------------------- K-proj
// proj[r][j] = alpha0 * sum_t own[r][t] slab[t][j]  (the alpha0 * w_r G[:, pi]
// gradient term of solvers.py:175), 64x64 output tiles, K = d.
__global__ void __launch_bounds__(256)
    k_project(const float* __restrict__ own, int n_rows, int ldo, int d,
              const float* __restrict__ slab, int b, float alpha0, float* __restrict__ proj) {
  __shared__ __align__(16) float As[GK][GT + 4];  // As[k][r]
  __shared__ __align__(16) float Bs[GK][GT + 4];  // Bs[k][j]
  const int r0 = blockIdx.x * GT, j0 = blockIdx.y * GT;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < d; k0 += GK) {
    for (int i = tid; i < GK * GT; i += 256) {
      const int rr = i / GK, kk = i % GK;  // own tile: 64 rows x 16 k (k fastest)
      const int r = r0 + rr, k = k0 + kk;
      As[kk][rr] = (r < n_rows && k < d) ? own[(size_t)r * ldo + k] : 0.f;
      const int kb = i / GT, jj = i % GT;
      Bs[kb][jj] = (k0 + kb < d && j0 + jj < b) ? slab[(size_t)(k0 + kb) * b + j0 + jj] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 c = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], cv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty * 4 + i;
    if (r >= n_rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int jj = j0 + tx * 4 + j;
      if (jj < b) proj[(size_t)r * b + jj] = alpha0 * acc[i][j];
    }
  }
}


// ---------------------------------------------------------------- b <= 4
// For the narrowest blocks (b = 1 is the iCD case) the slab and the
// projection are GEMVs over a whole factor matrix: bandwidth-bound, so they
// read each row once, coalesced, with many rows in flight.
//
// slab partial: part[split][k][j] = sum_{r in split} M[r][k] M[r][b0 + j];
// thread <-> column k, 8 rows per step (the M[r][b0+j] values are warp-wide
// broadcasts).
template <int B>
__global__ void __launch_bounds__(256)
    k_slab_gemv(const float* __restrict__ M, int n, int ldm, int d, int b0, int rows_per_split,
                float* __restrict__ part) {
  const int split = blockIdx.y;
  const int k = blockIdx.x * 256 + threadIdx.x;
  const int r_beg = split * rows_per_split, r_end = min(n, r_beg + rows_per_split);
  const bool ok = k < d;
  float a0[B], a1[B];
#pragma unroll
  for (int j = 0; j < B; ++j) a0[j] = a1[j] = 0.f;
  int r = r_beg;
  for (; r + 7 < r_end; r += 8) {
    float x[8], f[8][B];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float* row = M + (size_t)(r + u) * ldm;
      x[u] = ok ? __ldg(row + k) : 0.f;
#pragma unroll
      for (int j = 0; j < B; ++j) f[u][j] = __ldg(row + b0 + j);
    }
#pragma unroll
    for (int u = 0; u < 8; u += 2)
#pragma unroll
      for (int j = 0; j < B; ++j) {
        a0[j] = fmaf(x[u], f[u][j], a0[j]);
        a1[j] = fmaf(x[u + 1], f[u + 1][j], a1[j]);
      }
  }
  for (; r < r_end; ++r) {
    const float* row = M + (size_t)r * ldm;
    const float x = ok ? __ldg(row + k) : 0.f;
#pragma unroll
    for (int j = 0; j < B; ++j) a0[j] = fmaf(x, __ldg(row + b0 + j), a0[j]);
  }
  if (ok) {
    float* o = part + (size_t)split * d * B + (size_t)k * B;
#pragma unroll
    for (int j = 0; j < B; ++j) o[j] = a0[j] + a1[j];
  }
}

// projection: proj[r][j] = alpha0 * sum_k own[r][k] slab[k][j]; warp per
// row, 16-byte coalesced loads, shuffle reduction.
template <int B>
__global__ void __launch_bounds__(256)
    k_project_gemv(const float* __restrict__ own, int n_rows, int ldo, int d,
                   const float* __restrict__ slab, float alpha0, int vec, float* __restrict__ proj) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= n_rows) return;
  const float* row = own + (size_t)r * ldo;
  float acc[B];
#pragma unroll
  for (int j = 0; j < B; ++j) acc[j] = 0.f;
  if (vec) {
    for (int k4 = lane; 4 * k4 < d; k4 += 32) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(row) + k4);
      const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < B; ++j) acc[j] = fmaf(xs[q], __ldg(slab + (size_t)(4 * k4 + q) * B + j), acc[j]);
    }
  } else {
    for (int k = lane; k < d; k += 32) {
      const float x = __ldg(row + k);
#pragma unroll
      for (int j = 0; j < B; ++j) acc[j] = fmaf(x, __ldg(slab + (size_t)k * B + j), acc[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < B; ++j) {
    float v = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) proj[(size_t)r * B + j] = alpha0 * v;
  }
}


// out[r][j] = F[r][b0 + j] for j < b (0 for the padding up to ldc)
__global__ void k_compact_cols(const float* __restrict__ F, int n, int ldf, int b0, int b,
                               float* __restrict__ out, int ldc) {
  const long long cnt = (long long)n * ldc;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / ldc), j = (int)(i - (long long)r * ldc);
    out[i] = j < b ? __ldg(F + (size_t)r * ldf + b0 + j) : 0.f;
  }
}

// many splits (the b <= 4 GEMV slab): warp per output element, lanes stride
// the splits, fixed shuffle tree
__global__ void __launch_bounds__(256)
    k_reduce_splits_warp(const float* __restrict__ part, int nsplit, int count, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= count) return;
  float s = 0.f;
  for (int k = lane; k < nsplit; k += 32) s += part[(size_t)k * count + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[i] = s;
}
// Multi-GPU column-block exchange (distributed.py): recv holds every rank's
// rows of the block X[:, b0:b0+b] after the all-gather, rank r's at
// recv[r * nmax ..] (bounds[r]..bounds[r+1] global rows).  Per global row u:
// delta[u] = new - old (old = the rank's own pre-sweep copy for its rows, the
// replicated table for the others), and the remote rows are written into X.
__global__ void __launch_bounds__(256)
    k_apply_block(const float* __restrict__ recv, int nmax, const int* __restrict__ bounds, int world,
                  int rank, const float* __restrict__ old_local, float* X, int ldx, int b0, int b,
                  float* __restrict__ delta, int n_rows) {
  const long long n = (long long)n_rows * b;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int u = (int)(i / b), c = (int)(i - (long long)u * b);
    int r = 0;
    while (r + 1 < world && u >= bounds[r + 1]) ++r;
    const int lo = bounds[r];
    const float v = recv[((long long)r * nmax + (u - lo)) * b + c];
    float* x = X + (size_t)u * ldx + b0 + c;
    const float old = (r == rank) ? old_local[(size_t)(u - lo) * b + c] : *x;
    if (r != rank) *x = v;
    delta[i] = v - old;
  }
}

}  // namespace ials
