// ials_sweep_w32m.cuh -- the warp-per-row sweep of ials_sweep_w32.cuh (light rows
// of a block of 17 <= b <= 32 columns, b % 4 == 0) with the Hessian on the
// warp-level tensor path: H = sum_k x_k x_k^T is accumulated 8 entries at a
// time by mma.sync m16n8k8 TF32 tiles, 3xTF32 (hi hi + lo hi + hi lo; x = hi +
// lo with hi = cvt.rna.tf32), FP32 accumulators in registers.
//
// Why not tcgen05 here: a 32 x 32 Hessian is a sixteenth of a 128-lane TMEM
// tile; the packed tcgen05 sweep (ials_sweep_pk.cuh) pays a CTA barrier and an
// MMA round trip per 8 entries of a 4-row tile and measured slower than the
// FP32 warp-per-row sweep (15.6 vs 11.1 ms at configs[1]).  The warp-level
// instruction keeps the row's chain inside one warp; what it replaces is the
// 32 FFMA + 3 LDS.128 per entry of the FP32 tiles (the kernel is bound by
// instruction issue: 72% issue slots, 45% FMA pipe).
//
// Fragments (g = lane >> 2, t = lane & 3): with xv[j][h] = X[k0 + t + 4h][8j + g]
// (8 shared loads per 8 entries, bank = 8t + g at a row stride of 40 floats),
//   A (16 x 8, rows = Hessian rows 16mb..)  = {xv[2mb][0], xv[2mb+1][0], xv[2mb][1], xv[2mb+1][1]}
//   B (8 x 8, cols = Hessian cols 8nb..)    = {xv[nb][0], xv[nb][1]}
// so A and B share registers (unit weights; weighted entries scale A's copy).
// Only the six tiles that meet the lower triangle are formed: (mb, nb) =
// (0, 0..1), (1, 0..3); the factorisation never reads above the diagonal.
// The gradient, assembly, Cholesky and solves are those of ials_sweep_w32.cuh; a row
// whose pivots cancel (H_kk / pivot_k > cond_max) is left to the FP32 SIMT sweep.
#pragma once
#include "ials_sweep_w32.cuh"

namespace ials {

struct W32mLay {
  static constexpr int NW = 8, NT = NW * 32, KC = 16, XLD = 40, HLD = 36;   // XLD = 8 mod 32: conflict-free fragments
  // per warp (floats): X [2][KC][XLD] (later H / L, 32 x HLD), RHO [2][KC], AW [2][KC], LC [2][32]
  static constexpr int OFF_X = 0;
  static constexpr int OFF_RHO = OFF_X + 2 * KC * XLD;
  static constexpr int OFF_AW = OFF_RHO + 2 * KC;
  static constexpr int OFF_LC = OFF_AW + 2 * KC;
  static constexpr int WARP_FLOATS = OFF_LC + 2 * 32;
  static constexpr int OFF_TPL = NW * WARP_FLOATS;   // [32][HLD] alpha0 * slab[pi, pi]
  static constexpr int BYTES = (OFF_TPL + 32 * HLD) * 4;
};
static_assert(2 * W32mLay::KC * W32mLay::XLD >= 32 * W32mLay::HLD, "H aliases the staging buffers");

// x = hi + lo: hi the TF32 rounding of x, lo the remainder (its low mantissa bits are
// ignored by the tensor core, an error of 2^-21 relative to x)
IALS_DEVI void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  lo = __float_as_uint(x - __uint_as_float(hi));
}
IALS_DEVI void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One 16-entry stage of a 32-wide row into the six lower-triangle tiles
// ([0] (0,0) [1] (0,1) [2..5] (1,0..3)); xb: [16][XLD = 40] staged sub-rows, aw: the
// stage's 16 entry weights (read only when !UNIT).
template <bool UNIT>
IALS_DEVI void w32m_stage(float (&acc)[6][4], const float* xb, const float* aw, int g, int t4) {
  constexpr int XLD = 40;
#pragma unroll
  for (int c8 = 0; c8 < 16; c8 += 8) {
    const float* xc = xb + c8 * XLD;
    uint32_t hi[4][2], lo[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) tf32_split(xc[(t4 + 4 * h) * XLD + 8 * j + g], hi[j][h], lo[j][h]);
    uint32_t ahi[4][2], alo[4][2];   // the A copy: a_k x_k for weighted entries
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (UNIT) {
          ahi[j][h] = hi[j][h];
          alo[j][h] = lo[j][h];
        } else {
          tf32_split(aw[c8 + t4 + 4 * h] * xc[(t4 + 4 * h) * XLD + 8 * j + g], ahi[j][h], alo[j][h]);
        }
      }
#pragma unroll
    for (int mb = 0; mb < 2; ++mb) {
      const uint32_t Ah[4] = {ahi[2 * mb][0], ahi[2 * mb + 1][0], ahi[2 * mb][1], ahi[2 * mb + 1][1]};
      const uint32_t Al[4] = {alo[2 * mb][0], alo[2 * mb + 1][0], alo[2 * mb][1], alo[2 * mb + 1][1]};
#pragma unroll
      for (int nb = 0; nb < 2 + 2 * mb; ++nb) {
        float(&d)[4] = acc[2 * mb + nb];
        mma_tf32(d, Al, hi[nb][0], hi[nb][1]);
        mma_tf32(d, Ah, lo[nb][0], lo[nb][1]);
        mma_tf32(d, Ah, hi[nb][0], hi[nb][1]);
      }
    }
  }
}

// One 16-entry stage of a 16-wide row into its two tiles (columns 0..7, 8..15);
// xb: [16][XLD = 24] staged sub-rows (24 = -8 mod 32: conflict-free fragments).
template <bool UNIT>
IALS_DEVI void w16m_stage(float (&acc)[2][4], const float* xb, const float* aw, int g, int t4) {
  constexpr int XLD = 24;
#pragma unroll
  for (int c8 = 0; c8 < 16; c8 += 8) {
    const float* xc = xb + c8 * XLD;
    uint32_t hi[2][2], lo[2][2];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) tf32_split(xc[(t4 + 4 * h) * XLD + 8 * j + g], hi[j][h], lo[j][h]);
    uint32_t Ah[4] = {hi[0][0], hi[1][0], hi[0][1], hi[1][1]};
    uint32_t Al[4] = {lo[0][0], lo[1][0], lo[0][1], lo[1][1]};
    if (!UNIT) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float a = aw[c8 + t4 + 4 * h];
        tf32_split(a * xc[(t4 + 4 * h) * XLD + g], Ah[2 * h], Al[2 * h]);
        tf32_split(a * xc[(t4 + 4 * h) * XLD + 8 + g], Ah[2 * h + 1], Al[2 * h + 1]);
      }
    }
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      mma_tf32(acc[nb], Al, hi[nb][0], hi[nb][1]);
      mma_tf32(acc[nb], Ah, lo[nb][0], lo[nb][1]);
      mma_tf32(acc[nb], Ah, hi[nb][0], hi[nb][1]);
    }
  }
}

template <bool UNIT, int MINB = 3>
__global__ void __launch_bounds__(W32mLay::NT, MINB) k_sweep_w32m(SweepParams p) {
  using L = W32mLay;
  extern __shared__ __align__(16) float w32m_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* sm = w32m_smem + warp * L::WARP_FLOATS;
  float* X = sm + L::OFF_X;
  float* RHO = sm + L::OFF_RHO;
  float* AW = sm + L::OFF_AW;
  float* LC = sm + L::OFF_LC;
  float* TPL = w32m_smem + L::OFF_TPL;
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
  const int g = lane >> 2, t4 = lane & 3;   // fragment coordinates
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
    // accumulator tiles (mb, nb): [0] (0,0) [1] (0,1) [2..5] (1,0..3)
    float acc[6][4];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
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
      w32m_stage<UNIT>(acc, xb, AW + buf * L::KC, g, t4);
#pragma unroll
      for (int k = 0; k < L::KC; k += 4) {
        const float4 rh = *reinterpret_cast<const float4*>(RHO + buf * L::KC + k);
        gs = fmaf(rh.x, xb[k * L::XLD + lane], gs);
        gs = fmaf(rh.y, xb[(k + 1) * L::XLD + lane], gs);
        gs = fmaf(rh.z, xb[(k + 2) * L::XLD + lane], gs);
        gs = fmaf(rh.w, xb[(k + 3) * L::XLD + lane], gs);
      }
      gacc += (double)gs;
      __syncwarp();   // the buffer is free for stage s + 2
    }
    // ---- assemble H: the six tiles of the lower triangle (the factorisation reads
    // row i's columns 0..i only; what the staging left above them is never used)
    float* HS = X;   // 32 x HLD
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int nb = 0; nb < 2 + 2 * mb; ++nb) {
        const float(&d)[4] = acc[2 * mb + nb];
        float* dst = HS + (16 * mb + g) * L::HLD + 8 * nb + 2 * t4;
        *reinterpret_cast<float2*>(dst) = make_float2(d[0], d[1]);
        *reinterpret_cast<float2*>(dst + 8 * L::HLD) = make_float2(d[2], d[3]);
      }
    __syncwarp();
    // lam_r on the diagonal (identity on the padding rows, where H and G are zero)
    HS[lane * L::HLD + lane] += (lane < b) ? lam : 1.f;
    const float diag0 = HS[lane * L::HLD + lane] + TPL[lane * L::HLD + lane];   // for the cancellation guard
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
    // cancellation guard (lane k kept 1/sqrt(pivot k)): the 3xTF32 Hessian carries an
    // error of ~1e-6 of its entries, so a pivot that lost more than cond_max of its
    // diagonal -- or is not positive and finite -- sends the row to the FP32 SIMT sweep
    // (the redo list), which also names a singular row
    const unsigned flagged = __ballot_sync(
        0xffffffffu, lane < b && !(rown > 0.f && rown < 3.0e38f && diag0 * (rown * rown) <= p.cond_max));
    float dj = 0.f;
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      const float dk = __shfl_sync(0xffffffffu, t * rown, k);
      if (lane == k) dj = dk;
      if (lane < k) t = fmaf(-HS[k * L::HLD + lane], dk, t);
    }
    __syncwarp();   // HS (the staging buffers) is rewritten by the next row
    if (flagged) {
      if (lane == 0) {
        p.redo_rows[atomicAdd(p.redo_cnt, 1)] = row;
        atomicAdd(p.redo_total, 1ull);
      }
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
