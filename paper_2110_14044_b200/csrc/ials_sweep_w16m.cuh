// ials_sweep_w16m.cuh -- the two-rows-per-warp sweep of ials_sweep_w16.cuh (light
// rows of a block of 4 <= b <= 16 columns, b % 4 == 0) with the Hessians on the
// warp-level tensor path (mma.sync m16n8k8 TF32, 3xTF32, FP32 accumulators; see
// ials_sweep_w32m.cuh for the fragment algebra and for why not tcgen05 at this
// width).  A row's 16 x 16 Hessian is two m16n8 tiles; the warp's two rows take
// turns on the tensor path (every lane holds fragments of both Hessians), the
// staging, gradient, Cholesky and solves stay per half-warp as in
// ials_sweep_w16.cuh.
#pragma once
#include "ials_sweep_w16.cuh"
#include "ials_sweep_w32m.cuh"

namespace ials {

struct W16mLay {
  static constexpr int NW = 8, NT = NW * 32, KC = 16, XLD = 24, HLD = 20;   // XLD = -8 mod 32: conflict-free fragments
  // per half-warp (floats): X [2][KC][XLD] (later H / L, 16 x HLD, and behind it the
  // factorisation's column buffer LC [2][16]), RHO [2][KC], AW [2][KC]
  static constexpr int OFF_X = 0;
  static constexpr int OFF_LC = 16 * HLD;
  static constexpr int OFF_RHO = OFF_X + 2 * KC * XLD;
  static constexpr int OFF_AW = OFF_RHO + 2 * KC;
  // (a half's region is 16 mod 32 floats long: the two halves' 4-byte accesses
  // to the same offset fall on disjoint banks)
  static constexpr int HALF_FLOATS = OFF_AW + 2 * KC + 16;
  static constexpr int OFF_TPL = NW * 2 * HALF_FLOATS;   // [16][HLD] alpha0 * slab[pi, pi]
  static constexpr int BYTES = (OFF_TPL + 16 * HLD) * 4;
};
static_assert(2 * W16mLay::KC * W16mLay::XLD >= 16 * W16mLay::HLD + 32, "H and LC alias the staging buffers");
static_assert(W16mLay::HALF_FLOATS % 32 == 16, "bank offset of the second half");
static_assert(4 * (W16mLay::BYTES + 1024) <= 228 * 1024, "four CTAs per SM");

template <bool UNIT>
__global__ void __launch_bounds__(W16mLay::NT, 4) k_sweep_w16m(SweepParams p) {
  using L = W16mLay;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) float w16m_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, l16 = lane & 15;
  float* sm = w16m_smem + (warp * 2 + half) * L::HALF_FLOATS;
  float* X = sm + L::OFF_X;
  float* RHO = sm + L::OFF_RHO;
  float* AW = sm + L::OFF_AW;
  float* LC = sm + L::OFF_LC;
  float* TPL = w16m_smem + L::OFF_TPL;
  const int b = p.b;
  // alpha0 * G_pp (zero outside b x b), shared by the CTA's rows
  for (int i = threadIdx.x; i < 16 * 16; i += L::NT) {
    const int r = i >> 4, c = i & 15;
    TPL[r * L::HLD + c] = (r < b && c < b) ? p.alpha0 * __ldg(p.slab + (size_t)(p.b0 + r) * b + c) : 0.f;
  }
  // staging columns >= b are never written by the gathers: keep them zero
  for (int i = l16; i < 2 * L::KC * L::XLD; i += 16) X[i] = 0.f;
  __syncthreads();

  const int n_light = p.n_light, n_tasks = (n_light + 1) >> 1;
  const int g = lane >> 2, t4 = lane & 3;   // fragment coordinates
  float* X0 = w16m_smem + (warp * 2) * L::HALF_FLOATS + L::OFF_X;        // the warp's two rows
  float* X1 = X0 + L::HALF_FLOATS;
  const float* AW0 = w16m_smem + (warp * 2) * L::HALF_FLOATS + L::OFF_AW;
  const int nq = b >> 2;   // 16-byte pieces of a sub-row
  int task = 0;
  if (lane == 0) task = atomicAdd(p.queue, 1);
  task = __shfl_sync(FULL, task, 0);
  while (task < n_tasks) {
    int nxt = 0;
    if (lane == 0) nxt = atomicAdd(p.queue, 1);
    const int li = 2 * task + half;
    const int row = li < n_light ? __ldg(p.light_rows + li) : -1;
    const int ebeg = row >= 0 ? __ldg(p.side.ptr + row) : 0;
    const int eend = row >= 0 ? __ldg(p.side.ptr + row + 1) : 0;
    const float lam = row >= 0 ? __ldg(p.side.lam + row) : 1.f;
    int nst = (eend - ebeg + L::KC - 1) / L::KC;
    nst = max(nst, __shfl_xor_sync(FULL, nst, 16));   // the pair's stage count
    float acc[2][2][4];   // [row of the pair][column octet][fragment]
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][j][c] = 0.f;
    double gacc = 0.0;
    // stage s -> buffer s & 1: lane k of the half fetches entry k's column id
    // (one stage ahead of its gathers), cache value (kept in a register until
    // the stage is consumed) and weight / label; every lane issues 4 of the
    // half's 64 16-byte gathers
    float cval = 0.f, wval = 1.f, yval = 1.f;
    int col_next = (l16 < eend - ebeg) ? __ldg(p.side.cols + ebeg + l16) : 0;
    auto issue = [&](int s) {
      const int e0 = ebeg + s * L::KC, nk = min(L::KC, eend - e0), buf = s & 1;   // nk <= 0: the shorter row
      const int col = col_next;
      col_next = (e0 + L::KC + l16 < eend) ? __ldg(p.side.cols + e0 + L::KC + l16) : 0;
      cval = 0.f; wval = 1.f; yval = 1.f;
      if (l16 < nk) {
        const int e = e0 + l16;
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
        const int e = (l16 >> 2) + 4 * i, q = l16 & 3;
        const int ce = __shfl_sync(FULL, col, e, 16);
        float* dst = X + (buf * L::KC + e) * L::XLD + 4 * q;
        if (e < nk) {
          if (q < nq) cp_async16(dst, p.fixed + (size_t)ce * p.ldf + p.fb0 + 4 * q);
        } else if (q < nq) {   // past the row's end: zeros
          *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      cp_async_commit();
    };
    if (nst > 0) issue(0);
    for (int s = 0; s < nst; ++s) {
      const int buf = s & 1;
      // this stage's residuals from the registers loaded when it was issued
      {
        const float rho = UNIT ? cval - 1.f : wval * (cval - yval);
        const bool in = ebeg + s * L::KC + l16 < eend;
        RHO[buf * L::KC + l16] = in ? rho : 0.f;
        if (!UNIT) AW[buf * L::KC + l16] = in ? wval : 0.f;
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
      w16m_stage<UNIT>(acc[0], X0 + buf * L::KC * L::XLD, AW0 + buf * L::KC, g, t4);
      w16m_stage<UNIT>(acc[1], X1 + buf * L::KC * L::XLD, AW0 + L::HALF_FLOATS + buf * L::KC, g, t4);
#pragma unroll
      for (int k = 0; k < L::KC; k += 4) {
        const float4 rh = *reinterpret_cast<const float4*>(RHO + buf * L::KC + k);
        gs = fmaf(rh.x, xb[k * L::XLD + l16], gs);
        gs = fmaf(rh.y, xb[(k + 1) * L::XLD + l16], gs);
        gs = fmaf(rh.z, xb[(k + 2) * L::XLD + l16], gs);
        gs = fmaf(rh.w, xb[(k + 3) * L::XLD + l16], gs);
      }
      gacc += (double)gs;
      __syncwarp();   // the buffer is free for stage s + 2
    }
    // ---- assemble H: every lane stores its fragments of both rows' Hessians
    float* HS = X;   // 16 x HLD
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        float* dst = (i ? X1 : X0) + g * L::HLD + 8 * nb + 2 * t4;
        *reinterpret_cast<float2*>(dst) = make_float2(acc[i][nb][0], acc[i][nb][1]);
        *reinterpret_cast<float2*>(dst + 8 * L::HLD) = make_float2(acc[i][nb][2], acc[i][nb][3]);
      }
    __syncwarp();
    // lam_r on the diagonal (identity on the padding rows, where H and G are zero)
    HS[l16 * L::HLD + l16] += (l16 < b) ? lam : 1.f;
    const float diag0 = HS[l16 * L::HLD + l16] + TPL[l16 * L::HLD + l16];   // for the cancellation guard
    float a[16];
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) {
      const float4 h = reinterpret_cast<const float4*>(HS + l16 * L::HLD)[j4];
      const float4 g = reinterpret_cast<const float4*>(TPL + l16 * L::HLD)[j4];
      a[4 * j4] = h.x + g.x; a[4 * j4 + 1] = h.y + g.y; a[4 * j4 + 2] = h.z + g.z; a[4 * j4 + 3] = h.w + g.w;
    }
    float ow = 0.f, t = 0.f;
    if (l16 < b && row >= 0) {
      ow = p.own[(size_t)row * p.ldo + p.b0 + l16];
      t = (float)(gacc + (double)__ldg(p.proj + (size_t)row * b + l16) + (double)lam * (double)ow);
    }
    // ---- Cholesky (right-looking, lane i <-> row i) with the forward solve fused
    float rown = 1.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float dk = __shfl_sync(FULL, a[k], k, 16);
      float r;   // MUFU.RSQ; a non-positive / non-finite pivot leaves a NaN, infinite or zero 1/sqrt
      asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(dk));
      if (l16 == k) rown = r;
      const float lik = a[k] * r;          // l_ik (lane k: sqrt(d_k))
      a[k] = lik;
      const float yk = __shfl_sync(FULL, t, k, 16) * r;
      if (l16 == k) t = yk;                 // y_k, final
      else if (l16 > k) t = fmaf(-lik, yk, t);   // (lanes < k: their y is final, their lik garbage)
      if (k < 15) {
        float* lc = LC + (k & 1) * 16;
        lc[l16] = lik;
        __syncwarp();
#pragma unroll
        for (int j4 = ((k + 1) >> 2) << 2; j4 < 16; j4 += 4) {
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
    for (int j4 = 0; j4 < 4; ++j4)
      reinterpret_cast<float4*>(HS + l16 * L::HLD)[j4] = make_float4(a[4 * j4], a[4 * j4 + 1], a[4 * j4 + 2], a[4 * j4 + 3]);
    __syncwarp();
    // cancellation guard (lane k kept 1/sqrt(pivot k)): a pivot that lost more than
    // cond_max of its diagonal, or is not positive and finite, sends this half's row to
    // the FP32 SIMT sweep (the redo list), which also names a singular row
    const unsigned flagged =
        (__ballot_sync(FULL, l16 < b && !(rown > 0.f && rown < 3.0e38f && diag0 * (rown * rown) <= p.cond_max)) >>
         (16 * half)) & 0xffffu;
    float dj = 0.f;
#pragma unroll
    for (int k = 15; k >= 0; --k) {
      const float dk = __shfl_sync(FULL, t * rown, k, 16);
      if (l16 == k) dj = dk;
      if (l16 < k) t = fmaf(-HS[k * L::HLD + l16], dk, t);
    }
    __syncwarp();   // HS (the staging buffers) is rewritten by the next row
    if (row >= 0) {
      if (flagged) {
        if (l16 == 0) {
          p.redo_rows[atomicAdd(p.redo_cnt, 1)] = row;
          atomicAdd(p.redo_total, 1ull);
        }
        if (l16 < b) p.drow[(size_t)row * b + l16] = 0.f;
      } else if (l16 < b) {
        p.own[(size_t)row * p.ldo + p.b0 + l16] = ow - dj;
        p.drow[(size_t)row * b + l16] = dj;
      }
    }
    // the staging columns >= b must read as zeros again (H overwrote them; at
    // b = 16 every element read is written by its stage's gathers or zero fill)
    if (b < 16)
      for (int i = l16; i < 2 * L::KC * L::XLD; i += 16) X[i] = 0.f;
    __syncwarp();
    task = __shfl_sync(FULL, nxt, 0);
  }
}

}  // namespace ials
