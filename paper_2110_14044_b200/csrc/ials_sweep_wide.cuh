// ials_sweep_wide.cuh -- side passes for block widths above 256: the dedicated
// iALS solve at d > 256 (solve_side_full / ials_epoch, solvers.py:216-233,
// 275-300: a Newton step of width d from an exact cache is the closed-form
// solve) and iALS++ partitions with blocks wider than 256 columns
// (_newton_side_pass, solvers.py:152-186).
//
// A b x b Hessian no longer fits a CTA's registers / TMEM, so the rows of a
// pass are taken in batches of R rows whose normal equations live in global
// memory (R * (b + 1) * lda floats; L2-resident for the widths up to ~512):
//
//   k_wide_build   grid (tile pairs + 1, R): CTA (s, r) forms one 64 x 64 lower
//                  tile of row r's Hessian  sum_k a_k x_k x_k^T + alpha0 G_pp +
//                  lam_r I  (register-tiled FP32 SYRK over the row's gathered
//                  sub-rows, cp.async double buffering, two-level summation);
//                  the extra CTA forms the gradient (fp64 row sum) as row b of
//                  the matrix.  Output tiles, not entries, are split across
//                  CTAs: deterministic without partial buffers, and a long
//                  (heavy) row is spread over all its tiles' CTAs.
//   k_wide_chol    one CTA per row: left-looking blocked Cholesky in place,
//                  64-column panels, the panel of every 64-row chunk formed by
//                  a register-tiled GEMM over the columns already factored,
//                  the diagonal block factored in shared memory and its
//                  explicit inverse applied to the chunks below (a GEMM);
//                  forward solve fused per panel, blocked backward solve;
//                  own[r, pi] -= d, drow[r] = d.
//   k_wide_cache   entry-parallel yhat[pos] -= x_k . d (warp per entry).
//
// FP32 SIMT throughout (the per-row cost is b^3/3: the cubic cost the paper
// holds against iALS).  A non-positive pivot is reported to the error word.
#pragma once
#include "ials_sweep.cuh"

namespace ials {

constexpr int kWT = 64;    // tile edge (Hessian tiles, Cholesky panels and row chunks)
constexpr int kWK = 16;    // entries (build) / columns (Cholesky GEMM) per staged chunk
constexpr int kWXLD = kWT + 4;   // k-major staging of the build: [k][tile column]
constexpr int kWALD = kWK + 4;   // row-major staging of the Cholesky GEMM: [row][k]
constexpr int kWTLD = kWT + 4;   // the 64 x 64 working blocks

struct WideParams {
  float* A;               // [R][(b + 1) * lda]; row b of a matrix: gradient -> y
  int lda;                // row stride, b rounded up to 4
  long long mat_stride;   // floats per matrix
  int i0, nb;             // this batch: rows [i0, i0 + nb) of heavy_rows ++ light_rows
};

IALS_DEVI int wide_row(const SweepParams& p, int i) {
  return i < p.n_heavy ? __ldg(p.heavy_rows + i) : __ldg(p.light_rows + (i - p.n_heavy));
}

// ---------------------------------------------------------------- build
// Stage entries [e0, e0 + nk) of the row, columns [c0, c0 + 64) of the block,
// k-major into X[kWK][kWXLD]; missing entries / columns beyond b are zeros.
IALS_DEVI void wide_stage(const SweepParams& p, float* X, int e0, int nk, int c0, int tid) {
  if (p.vec) {
    const int k = tid >> 4, v = tid & 15;
    float* dst = X + k * kWXLD + 4 * v;
    const int c = c0 + 4 * v;
    if (k < nk && c < p.b) {
      const int col = __ldg(p.side.cols + e0 + k);
      IALS_CHECK(col >= 0 && col < p.side.n_fixed);
      cp_async16(dst, p.fixed + (size_t)col * p.ldf + p.fb0 + c);
    } else {
      *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
    for (int i = tid; i < kWK * kWT; i += 256) {
      const int k = i >> 6, v = i & 63;
      const int c = c0 + v;
      float* dst = X + k * kWXLD + v;
      if (k < nk && c < p.b) {
        const int col = __ldg(p.side.cols + e0 + k);
        cp_async4(dst, p.fixed + (size_t)col * p.ldf + p.fb0 + c);
      } else {
        *dst = 0.f;
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_wide_build(SweepParams p, WideParams wp, int ntp) {
  __shared__ __align__(16) float Xi[2][kWK * kWXLD];
  __shared__ __align__(16) float Xj[2][kWK * kWXLD];
  __shared__ float aw[2][kWK];
  __shared__ float srho[32];
  __shared__ int scol[32];
  const int tid = threadIdx.x;
  const int row = wide_row(p, wp.i0 + blockIdx.y);
  const int ebeg = __ldg(p.side.ptr + row), eend = __ldg(p.side.ptr + row + 1);
  float* A = wp.A + (size_t)blockIdx.y * wp.mat_stride;
  const int b = p.b;
  const float lam = __ldg(p.side.lam + row);

  if ((int)blockIdx.x == ntp) {
    // gradient: g = sum_k rho_k x_k + alpha0 * (w G)[pi] + lam w[pi]; the
    // row sum in fp64 (it cancels strongly on long rows), each 32-entry
    // chunk's products in four fixed-order fp32 chains
    for (int jb = 0; jb < b; jb += 256 * 8) {
      double g[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) g[m] = 0.0;
      for (int e0 = ebeg; e0 < eend; e0 += 32) {
        __syncthreads();
        if (tid < 32) {
          const int e = e0 + tid;
          float r = 0.f;
          int col = 0;
          if (e < eend) {
            const float a = p.side.weights ? __ldg(p.side.weights + e) : 1.f;
            const float y = p.side.labels ? __ldg(p.side.labels + e) : 1.f;
            const int pos = p.side.pos ? __ldg(p.side.pos + e) : e;
            r = a * (p.cache[pos] - y);
            col = __ldg(p.side.cols + e);
          }
          srho[tid] = r;
          scol[tid] = col;
        }
        __syncthreads();
        const int nk = min(32, eend - e0);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int j = jb + tid + 256 * m;
          if (j >= b) break;
          const float* xc = p.fixed + p.fb0 + j;
          float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f;
          int k = 0;
          for (; k + 3 < nk; k += 4) {
            g0 = fmaf(srho[k], __ldg(xc + (size_t)scol[k] * p.ldf), g0);
            g1 = fmaf(srho[k + 1], __ldg(xc + (size_t)scol[k + 1] * p.ldf), g1);
            g2 = fmaf(srho[k + 2], __ldg(xc + (size_t)scol[k + 2] * p.ldf), g2);
            g3 = fmaf(srho[k + 3], __ldg(xc + (size_t)scol[k + 3] * p.ldf), g3);
          }
          for (; k < nk; ++k) g0 = fmaf(srho[k], __ldg(xc + (size_t)scol[k] * p.ldf), g0);
          g[m] += ((double)g0 + (double)g1) + ((double)g2 + (double)g3);
        }
      }
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int j = jb + tid + 256 * m;
        if (j >= b) break;
        const double v = g[m] + (double)__ldg(p.proj + (size_t)row * b + j) +
                         (double)lam * (double)p.own[(size_t)row * p.ldo + p.b0 + j];
        A[(size_t)b * wp.lda + j] = (float)v;
      }
    }
    return;
  }

  // tile pair s -> (ti, tj), tj <= ti
  int ti = 0;
  {
    const int s = blockIdx.x;
    while ((ti + 1) * (ti + 2) / 2 <= s) ++ti;
  }
  const int tj = blockIdx.x - ti * (ti + 1) / 2;
  const bool diag = ti == tj;
  const int ty = tid >> 4, tx = tid & 15;
  const bool unit = p.side.weights == nullptr;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  const int n = eend - ebeg;
  const int nch = (n + kWK - 1) / kWK;
  auto stage = [&](int c) {
    const int e0 = ebeg + c * kWK, nk = min(kWK, eend - e0), buf = c & 1;
    wide_stage(p, Xi[buf], e0, nk, ti * kWT, tid);
    if (!diag) wide_stage(p, Xj[buf], e0, nk, tj * kWT, tid);
    cp_async_commit();
    if (!unit && tid < kWK) aw[buf][tid] = tid < nk ? __ldg(p.side.weights + e0 + tid) : 0.f;
  };
  if (nch > 0) stage(0);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      stage(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* xi = Xi[c & 1] + ty * 4;
    const float* xj = (diag ? Xi[c & 1] : Xj[c & 1]) + tx * 4;
    float loc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) loc[i][j] = 0.f;
#pragma unroll
    for (int k = 0; k < kWK; ++k) {
      float4 a = *reinterpret_cast<const float4*>(xi + k * kWXLD);
      const float4 cc = *reinterpret_cast<const float4*>(xj + k * kWXLD);
      if (!unit) {
        const float w = aw[c & 1][k];
        a.x *= w; a.y *= w; a.z *= w; a.w *= w;
      }
      const float av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) loc[i][j] = fmaf(av[i], cv[j], loc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] += loc[i][j];
    __syncthreads();
  }
  // + alpha0 G_pp + lam I
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ti * kWT + ty * 4 + i;
    if (r >= b) continue;
    const float* srow = p.slab + (size_t)(p.b0 + r) * b;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = tj * kWT + tx * 4 + j;
      if (c >= b) continue;
      float v = acc[i][j] + p.alpha0 * __ldg(srow + c);
      if (r == c) v += lam;
      A[(size_t)r * wp.lda + c] = v;
    }
  }
}

// ---------------------------------------------------------------- factor / solve
struct WideSm {
  static constexpr int OFF_A = 0;                          // [2][64][kWALD]
  static constexpr int OFF_B = OFF_A + 2 * kWT * kWALD;    // [2][64][kWALD]
  static constexpr int OFF_T = OFF_B + 2 * kWT * kWALD;    // [64][kWTLD] working block
  static constexpr int OFF_LD = OFF_T + kWT * kWTLD;       // [64][kWTLD] diagonal factor
  static constexpr int OFF_LI = OFF_LD + kWT * kWTLD;      // [64][kWTLD] its inverse
  static constexpr int OFF_Y = OFF_LI + kWT * kWTLD;       // [b] y, then the step d
  static size_t bytes(int b) { return size_t(OFF_Y + ((b + 3) & ~3) + 64) * 4; }
};

// rows [r0, r0 + 64) x columns [k0, k0 + 16) of the matrix into S[64][kWALD]
// (rows beyond nrows as zeros); lda % 4 == 0 and 16-byte aligned base
IALS_DEVI void wide_stage_rows(float* S, const float* A, int lda, int r0, int nrows, int k0, int tid) {
  const int r = tid >> 2, v = tid & 3;
  float* dst = S + r * kWALD + 4 * v;
  if (r0 + r < nrows) {
    cp_async16(dst, A + (size_t)(r0 + r) * lda + k0 + 4 * v);
  } else {
    *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__global__ void __launch_bounds__(256, 2) k_wide_chol(SweepParams p, WideParams wp) {
  extern __shared__ __align__(16) float wsm[];
  float* As = wsm + WideSm::OFF_A;
  float* Bs = wsm + WideSm::OFF_B;
  float* T = wsm + WideSm::OFF_T;
  float* Ld = wsm + WideSm::OFF_LD;
  float* Li = wsm + WideSm::OFF_LI;
  float* ys = wsm + WideSm::OFF_Y;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31, warp = tid >> 5;
  const int row = wide_row(p, wp.i0 + blockIdx.x);
  float* A = wp.A + (size_t)blockIdx.x * wp.mat_stride;
  const int b = p.b, lda = wp.lda;
  const int nblk = (b + kWT - 1) / kWT;
  const float* grow = A + (size_t)b * lda;   // the gradient row

  for (int pb = 0; pb < nblk; ++pb) {
    const int c0 = pb * kWT, nc = min(kWT, b - c0);
    for (int rb = pb; rb < nblk; ++rb) {
      const int r0 = rb * kWT;
      // acc = L[r0.., :c0] L[c0.., :c0]^T: thread (ty, tx) holds rows ty*4+i,
      // columns tx + 16 j of the 64 x 64 chunk
      float acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
      const bool same = rb == pb;
      const int nkc = c0 / kWK;   // c0 is a multiple of 64
      auto stage = [&](int c) {
        const int buf = c & 1;
        wide_stage_rows(As + buf * kWT * kWALD, A, lda, r0, b, c * kWK, tid);
        if (!same) wide_stage_rows(Bs + buf * kWT * kWALD, A, lda, c0, b, c * kWK, tid);
        cp_async_commit();
      };
      if (nkc > 0) stage(0);
      for (int c = 0; c < nkc; ++c) {
        if (c + 1 < nkc) {
          stage(c + 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const float* a_ = As + (c & 1) * kWT * kWALD + (ty * 4) * kWALD;
        const float* b_ = (same ? As : Bs) + (c & 1) * kWT * kWALD + tx * kWALD;
#pragma unroll
        for (int k = 0; k < kWK; k += 4) {
          float4 av[4], bv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) av[i] = *reinterpret_cast<const float4*>(a_ + i * kWALD + k);
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = *reinterpret_cast<const float4*>(b_ + 16 * j * kWALD + k);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              acc[i][j] = fmaf(av[i].x, bv[j].x, acc[i][j]);
              acc[i][j] = fmaf(av[i].y, bv[j].y, acc[i][j]);
              acc[i][j] = fmaf(av[i].z, bv[j].z, acc[i][j]);
              acc[i][j] = fmaf(av[i].w, bv[j].w, acc[i][j]);
            }
        }
        __syncthreads();
      }
      // T = A[chunk, panel] - acc
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = ty * 4 + i;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = tx + 16 * j;
          float v = 0.f;
          if (r0 + r < b && c < nc) v = A[(size_t)(r0 + r) * lda + c0 + c] - acc[i][j];
          T[r * kWTLD + c] = v;
        }
      }
      __syncthreads();
      if (same) {
        // ---- factor the diagonal block in place (lower triangle of T)
        for (int j = 0; j < nc; ++j) {
          const float piv = T[j * kWTLD + j];
          float inv;
          if (!(piv > 0.f)) {
            if (tid == 0) report_singular(p.err, p.side_id, row, c0 + j);
            inv = 1.f;
          } else {
            inv = rsqrtf(piv);
            inv = inv * (1.5f - 0.5f * piv * inv * inv);   // one Newton step: full fp32 accuracy
          }
          __syncthreads();
          if (tid < nc && tid >= j) T[tid * kWTLD + j] = (tid == j) ? (piv > 0.f ? piv * inv : 1.f)
                                                                     : T[tid * kWTLD + j] * inv;
          __syncthreads();
          // trailing update of the lower triangle: (r, c), j < c <= r < nc
          for (int i = tid; i < kWT * kWT; i += 256) {
            const int r = i >> 6, c = i & 63;
            if (c > j && c <= r && r < nc) T[r * kWTLD + c] -= T[r * kWTLD + j] * T[c * kWTLD + j];
          }
          __syncthreads();
        }
        // Ld = tril(T) (identity beyond nc); written to the matrix
        for (int i = tid; i < kWT * kWT; i += 256) {
          const int r = i >> 6, c = i & 63;
          float v = (c <= r && r < nc) ? T[r * kWTLD + c] : (r == c ? 1.f : 0.f);
          Ld[r * kWTLD + c] = v;
          if (c <= r && r < nc) A[(size_t)(c0 + r) * lda + c0 + c] = v;
        }
        __syncthreads();
        // Li = Ld^-1: four lanes per column, the m-sum split over them
        {
          const int c = tid >> 2, q = tid & 3;
          for (int r = 0; r < kWT; ++r) {
            float s = 0.f;
            for (int m = c + q; m < r; m += 4) s = fmaf(Ld[r * kWTLD + m], Li[m * kWTLD + c], s);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            if (q == 0) Li[r * kWTLD + c] = r < c ? 0.f : ((r == c ? 1.f : 0.f) - s) / Ld[r * kWTLD + r];
            __syncwarp();
          }
        }
        __syncthreads();
        // ---- forward solve of the panel: y_blk = Ld^-1 (g_blk - L[blk, :c0] y[:c0])
        for (int rr = warp; rr < nc; rr += 8) {
          const float* lr = A + (size_t)(c0 + rr) * lda;
          float s = 0.f;
          for (int k = lane; k < c0; k += 32) s = fmaf(lr[k], ys[k], s);
          s = warp_sum(s);
          if (lane == 0) T[rr] = grow[c0 + rr] - s;   // T's first row: scratch (the block is in Ld)
        }
        __syncthreads();
        if (tid < nc) {
          float s = 0.f;
          for (int m = 0; m <= tid; ++m) s = fmaf(Li[tid * kWTLD + m], T[m], s);
          ys[c0 + tid] = s;
        }
        __syncthreads();
      } else {
        // ---- L[chunk, panel] = T Li^T  (out[r][c] = sum_{m <= c} T[r][m] Li[c][m])
        float o[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) o[i][j] = 0.f;
        const float* t_ = T + (ty * 4) * kWTLD;
        const float* l_ = Li + tx * kWTLD;
#pragma unroll 4
        for (int m = 0; m < kWT; m += 4) {
          float4 av[4], bv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) av[i] = *reinterpret_cast<const float4*>(t_ + i * kWTLD + m);
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = *reinterpret_cast<const float4*>(l_ + 16 * j * kWTLD + m);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              o[i][j] = fmaf(av[i].x, bv[j].x, o[i][j]);
              o[i][j] = fmaf(av[i].y, bv[j].y, o[i][j]);
              o[i][j] = fmaf(av[i].z, bv[j].z, o[i][j]);
              o[i][j] = fmaf(av[i].w, bv[j].w, o[i][j]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = r0 + ty * 4 + i;
          if (r >= b) continue;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = tx + 16 * j;
            if (c < nc) A[(size_t)r * lda + c0 + c] = o[i][j];
          }
        }
        __syncthreads();
      }
    }
    // the panel's columns of L are read (as rows' k-ranges) by later panels
    __threadfence_block();
    __syncthreads();
  }

  // ---- backward solve L^T d = y, block by block from the last
  for (int pb = nblk - 1; pb >= 0; --pb) {
    const int c0 = pb * kWT, nc = min(kWT, b - c0);
    for (int i = tid; i < kWT * kWT; i += 256) {
      const int r = i >> 6, c = i & 63;
      Ld[r * kWTLD + c] = (c <= r && r < nc) ? A[(size_t)(c0 + r) * lda + c0 + c] : 0.f;
    }
    __syncthreads();
    if (warp == 0) {
      for (int j = nc - 1; j >= 0; --j) {
        float s = 0.f;
        for (int m = j + 1 + lane; m < nc; m += 32) s = fmaf(Ld[m * kWTLD + j], ys[c0 + m], s);
        s = warp_sum(s);
        if (lane == 0) ys[c0 + j] = (ys[c0 + j] - s) / Ld[j * kWTLD + j];
        __syncwarp();
      }
    }
    __syncthreads();
    // y[:c0] -= L[blk, :c0]^T d_blk
    for (int k = tid; k < c0; k += 256) {
      float s = 0.f;
      for (int m = 0; m < nc; ++m) s = fmaf(A[(size_t)(c0 + m) * lda + k], ys[c0 + m], s);
      ys[k] -= s;
    }
    __syncthreads();
  }
  for (int j = tid; j < b; j += 256) {
    const float dj = ys[j];
    p.own[(size_t)row * p.ldo + p.b0 + j] -= dj;
    p.drow[(size_t)row * b + j] = dj;
  }
}

// ---------------------------------------------------------------- cache
// yhat[pos_e] -= x_e . d_row(e), warp per entry (both vectors are b floats)
__global__ void __launch_bounds__(256) k_wide_cache(SweepParams p, long long nnz) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * 8;
  for (long long e = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); e < nnz; e += nw) {
    int row;
    if (p.side.rows) {
      row = __ldg(p.side.rows + e);
    } else {   // largest row with ptr[row] <= e
      int lo = 0, hi = p.side.n_rows;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if ((long long)__ldg(p.side.ptr + mid) <= e) lo = mid; else hi = mid;
      }
      row = lo;
    }
    const int col = __ldg(p.side.cols + e);
    const float* x = p.fixed + (size_t)col * p.ldf + p.fb0;
    const float* dr = p.drow + (size_t)row * p.b;
    float s = 0.f;
    if (p.vec) {
      for (int j = 4 * lane; j < p.b; j += 128) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(x + j));
        const float4 c = __ldg(reinterpret_cast<const float4*>(dr + j));
        s = fmaf(a.x, c.x, s);
        s = fmaf(a.y, c.y, s);
        s = fmaf(a.z, c.z, s);
        s = fmaf(a.w, c.w, s);
      }
    } else {
      for (int j = lane; j < p.b; j += 32) s = fmaf(__ldg(x + j), __ldg(dr + j), s);
    }
    s = warp_sum(s);
    if (lane == 0) {
      const long long pos = p.side.pos ? (long long)__ldg(p.side.pos + e) : e;
      p.cache[pos] -= s;
    }
  }
}

}  // namespace ials
