// ials_sweep_w32.cuh -- light rows of a narrow block (17 <= b <= 32, b % 4 == 0)
// swept one row per WARP, FP32 SIMT.
//
// The packed tensor-core sweep (ials_sweep_pk.cuh) pays a CTA barrier and an
// MMA round trip per 8 entries of a 4-row tile, and its work is bound by
// instruction issue (~90 warp-instructions per entry at b = 32); at this width
// the Hessian is small enough for registers: one warp holds the 32 x 32
// Hessian as 32 lanes x (4 x 8) tiles, the row's sub-rows stream through a
// warp-private double buffer (cp.async, 16 entries a stage), and nothing in
// the row's chain synchronises wider than the warp (~40 warp-instructions per
// entry, 8 independent rows in flight per CTA).
//
// Per row r (_newton_side_pass, solvers.py:152-186, for one row):
//   accumulate  lane (ty, tx): H[4ty.., 8tx..] += x_k[4ty..] x_k[8tx..]^T (3
//               16-byte shared loads + 32 FMAs per entry); lane j: g_j +=
//               rho_k x_kj (fp32 per stage, fp64 across stages)
//   assemble    H += alpha0 G_pp (CTA-shared copy) + lam_r I;  g += proj + lam_r w
//   solve       lane i <-> row i of H in registers: right-looking Cholesky, the
//               column of l broadcast through shared memory, forward solve
//               fused; backward solve from L's rows in shared memory
//   write       own[r, pi] -= d, drow[r] = d (the pass's entry-parallel cache
//               kernel applies yhat -= x . d)
// A non-positive or non-finite pivot is the reference's SingularMatrixError:
// reported through the error word with its (side, row, pivot).
#pragma once
#include "ials_sweep.cuh"

namespace ials {

struct W32Lay {
  static constexpr int NW = 8, NT = NW * 32, KC = 16, XLD = 36, HLD = 36;   // 16-byte rows, conflict-free float4
  // per warp (floats): X [2][KC][XLD] (later H / L, 32 x HLD), RHO [2][KC], AW [2][KC], LC [2][32]
  static constexpr int OFF_X = 0;
  static constexpr int OFF_RHO = OFF_X + 2 * KC * XLD;
  static constexpr int OFF_AW = OFF_RHO + 2 * KC;
  static constexpr int OFF_LC = OFF_AW + 2 * KC;
  static constexpr int WARP_FLOATS = OFF_LC + 2 * 32;
  static constexpr int OFF_TPL = NW * WARP_FLOATS;   // [32][HLD] alpha0 * slab[pi, pi]
  static constexpr int BYTES = (OFF_TPL + 32 * HLD) * 4;
};
static_assert(2 * W32Lay::KC * W32Lay::XLD >= 32 * W32Lay::HLD, "H aliases the staging buffers");

template <bool UNIT>
__global__ void __launch_bounds__(W32Lay::NT, 3) k_sweep_w32(SweepParams p) {
  using L = W32Lay;
  extern __shared__ __align__(16) float w32_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* sm = w32_smem + warp * L::WARP_FLOATS;
  float* X = sm + L::OFF_X;
  float* RHO = sm + L::OFF_RHO;
  float* AW = sm + L::OFF_AW;
  float* LC = sm + L::OFF_LC;
  float* TPL = w32_smem + L::OFF_TPL;
  const int b = p.b;
  // alpha0 * G_pp (zero outside b x b), shared by the CTA's rows
  for (int i = threadIdx.x; i < 32 * 32; i += L::NT) {
    const int r = i >> 5, c = i & 31;
    TPL[r * L::HLD + c] = (r < b && c < b) ? p.alpha0 * __ldg(p.slab + (size_t)(p.b0 + r) * b + c) : 0.f;
  }
  // staging columns >= b are never written by the gathers: keep them zero
  for (int i = lane; i < 2 * L::KC * L::XLD; i += 32) X[i] = 0.f;
  __syncthreads();

  const int* lrows = p.light_rows;
  int n_light = p.n_light;
  if (p.chunk_tot) {   // ials_epoch_host's chunked first user pass: this launch's slice
    int off = 0;
    for (int k = 0; k < p.chunk; ++k) off += p.chunk_tot[k];
    lrows += off;
    n_light = p.chunk_tot[p.chunk];
  }
  const int ty = lane >> 2, tx = lane & 3;
  const int nq = b >> 2;   // 16-byte pieces of a sub-row
  int task = 0;
  if (lane == 0) task = atomicAdd(p.queue, 1);
  task = __shfl_sync(0xffffffffu, task, 0);
  while (task < n_light) {
    int nxt = 0;
    if (lane == 0) nxt = atomicAdd(p.queue, 1);
    const int row = __ldg(lrows + task);
    const int ebeg = __ldg(p.side.ptr + row), eend = __ldg(p.side.ptr + row + 1);
    const float lam = __ldg(p.side.lam + row);
    const int nst = (eend - ebeg + L::KC - 1) / L::KC;
    float acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
    double gacc = 0.0;
    // stage s -> buffer s & 1: lanes < KC fetch their entry's column id, cache
    // value (kept in a register until the stage is consumed) and weight /
    // label; every lane issues 4 of the 128 16-byte gathers
    float cval = 0.f, wval = 1.f, yval = 1.f;
    // (the column ids run one stage further ahead, so the gathers' addresses
    // never wait for their own index load)
    int col_next = (lane < eend - ebeg && lane < L::KC) ? __ldg(p.side.cols + ebeg + lane) : 0;
    auto issue = [&](int s) {
      const int e0 = ebeg + s * L::KC, nk = min(L::KC, eend - e0), buf = s & 1;
      const int col = col_next;
      col_next = (e0 + L::KC + lane < eend && lane < L::KC) ? __ldg(p.side.cols + e0 + L::KC + lane) : 0;
      cval = 0.f; wval = 1.f; yval = 1.f;
      if (lane < nk) {
        const int e = e0 + lane;
        IALS_CHECK(col >= 0 && col < p.side.n_fixed);
        const int pos = p.side.pos ? __ldg(p.side.pos + e) : e;
        IALS_CHECK(pos >= 0 && pos < p.side.nnz);
        cval = p.cache[pos];
        if (!UNIT) {
          if (p.side.weights) wval = __ldg(p.side.weights + e);
          if (p.side.labels) yval = __ldg(p.side.labels + e);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = (lane >> 3) + 4 * i, q = lane & 7;
        const int ce = __shfl_sync(0xffffffffu, col, e);
        float* dst = X + (buf * L::KC + e) * L::XLD + 4 * q;
        if (e < nk) {
          if (q < nq) cp_async16(dst, p.fixed + (size_t)ce * p.ldf + p.fb0 + 4 * q);
        } else if (q < nq) {   // a short last stage: rows past the end read as zeros
          *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      cp_async_commit();
    };
    if (nst > 0) issue(0);
    for (int s = 0; s < nst; ++s) {
      const int buf = s & 1;
      // this stage's residuals from the registers loaded when it was issued
      if (lane < L::KC) {
        const float rho = UNIT ? cval - 1.f : wval * (cval - yval);
        const bool in = ebeg + s * L::KC + lane < eend;
        RHO[buf * L::KC + lane] = in ? rho : 0.f;
        if (!UNIT) AW[buf * L::KC + lane] = in ? wval : 0.f;
      }
      if (s + 1 < nst) {
        issue(s + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      const float* xb = X + buf * L::KC * L::XLD;
      float gs = 0.f;
#pragma unroll 4   // (not 16: the unrolled kernel already overflows the instruction cache)
      for (int k = 0; k < L::KC; ++k) {
        const float* xr = xb + k * L::XLD;
        const float4 r4 = *reinterpret_cast<const float4*>(xr + 4 * ty);
        const float4 c0 = *reinterpret_cast<const float4*>(xr + 8 * tx);
        const float4 c1 = *reinterpret_cast<const float4*>(xr + 8 * tx + 4);
        float rv[4] = {r4.x, r4.y, r4.z, r4.w};
        const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        if (!UNIT) {
          const float a = AW[buf * L::KC + k];
#pragma unroll
          for (int r = 0; r < 4; ++r) rv[r] *= a;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(rv[r], cv[c], acc[r][c]);
        gs = fmaf(RHO[buf * L::KC + k], xr[lane], gs);
      }
      gacc += (double)gs;
      __syncwarp();   // the buffer is free for stage s + 2
    }
    // ---- assemble H (lower triangle suffices; the tiles are stored whole)
    float* HS = X;   // 32 x HLD
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      float4* dst = reinterpret_cast<float4*>(HS + (4 * ty + r) * L::HLD + 8 * tx);
      dst[0] = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
      dst[1] = make_float4(acc[r][4], acc[r][5], acc[r][6], acc[r][7]);
    }
    __syncwarp();
    // lam_r on the diagonal (identity on the padding rows, where H and G are zero)
    HS[lane * L::HLD + lane] += (lane < b) ? lam : 1.f;
    float a[32];
#pragma unroll
    for (int j4 = 0; j4 < 8; ++j4) {
      const float4 h = reinterpret_cast<const float4*>(HS + lane * L::HLD)[j4];
      const float4 g = reinterpret_cast<const float4*>(TPL + lane * L::HLD)[j4];
      a[4 * j4] = h.x + g.x; a[4 * j4 + 1] = h.y + g.y; a[4 * j4 + 2] = h.z + g.z; a[4 * j4 + 3] = h.w + g.w;
    }
    float ow = 0.f, t = 0.f;
    if (lane < b) {
      ow = p.own[(size_t)row * p.ldo + p.b0 + lane];
      t = (float)(gacc + (double)__ldg(p.proj + (size_t)row * b + lane) + (double)lam * (double)ow);
    }
    // ---- Cholesky (right-looking, lane i <-> row i) with the forward solve fused
    float rown = 1.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float dk = __shfl_sync(0xffffffffu, a[k], k);
      float r;   // MUFU.RSQ; a non-positive / non-finite pivot leaves a NaN, infinite or zero 1/sqrt
      asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(dk));
      if (lane == k) rown = r;
      const float lik = a[k] * r;          // l_ik (lane k: sqrt(d_k))
      a[k] = lik;
      const float yk = __shfl_sync(0xffffffffu, t, k) * r;
      if (lane == k) t = yk;                 // y_k, final
      else if (lane > k) t = fmaf(-lik, yk, t);   // (lanes < k: their y is final, their lik garbage)
      if (k < 31) {
        float* lc = LC + (k & 1) * 32;
        lc[lane] = lik;
        __syncwarp();
#pragma unroll
        for (int j4 = ((k + 1) >> 2) << 2; j4 < 32; j4 += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(lc + j4);
          if (j4 > k) a[j4] = fmaf(-lik, l4.x, a[j4]);
          if (j4 + 1 > k) a[j4 + 1] = fmaf(-lik, l4.y, a[j4 + 1]);
          if (j4 + 2 > k) a[j4 + 2] = fmaf(-lik, l4.z, a[j4 + 2]);
          if (j4 + 3 > k) a[j4 + 3] = fmaf(-lik, l4.w, a[j4 + 3]);
        }
      }
    }
    // (lanes < k keep garbage in a[k..]: row i only owns a[0..i])
    // ---- backward solve L^T d = y from L's rows in shared memory
    __syncwarp();
#pragma unroll
    for (int j4 = 0; j4 < 8; ++j4)
      reinterpret_cast<float4*>(HS + lane * L::HLD)[j4] = make_float4(a[4 * j4], a[4 * j4 + 1], a[4 * j4 + 2], a[4 * j4 + 3]);
    __syncwarp();
    // the first failing pivot, if any: lane k kept 1/sqrt(pivot k)
    const unsigned badmask = __ballot_sync(0xffffffffu, !(rown > 0.f && rown < 3.0e38f));
    const int bad = badmask ? __ffs(badmask) - 1 : -1;
    float dj = 0.f;
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      const float dk = __shfl_sync(0xffffffffu, t * rown, k);
      if (lane == k) dj = dk;
      if (lane < k) t = fmaf(-HS[k * L::HLD + lane], dk, t);
    }
    __syncwarp();   // HS (the staging buffers) is rewritten by the next row
    if (bad >= 0 && bad < b) {
      if (lane == 0) report_singular(p.err, p.side_id, row, bad);
      if (lane < b) p.drow[(size_t)row * b + lane] = 0.f;
    } else if (lane < b) {
      p.own[(size_t)row * p.ldo + p.b0 + lane] = ow - dj;
      p.drow[(size_t)row * b + lane] = dj;
    }
    // the staging columns >= b must read as zeros again (H overwrote them; at
    // b = 32 every element read is written by its stage's gathers or zero fill)
    if (b < 32)
      for (int i = lane; i < 2 * L::KC * L::XLD; i += 32) X[i] = 0.f;
    __syncwarp();
    task = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

}  // namespace ials
