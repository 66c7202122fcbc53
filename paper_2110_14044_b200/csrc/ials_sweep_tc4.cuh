// ials_sweep_tc4.cuh -- fused tensor-core light-row sweep for block widths
// 33..128 (BT = 128; widths <= 64 are zero-padded), four CTAs (rows in
// flight) per SM.
//
// Per row, one CTA of 128 threads (thread i <-> TMEM lane i <-> matrix row i):
//   1. TMEM D := alpha0*slab[pi,pi] + lam*I   (tcgen05.st from the packed
//      template k_tc_template built once per pass; identity on the padding)
//   2. for each 16-entry chunk of the row (cp.async double-buffered gather):
//      fp64 gradient on the SIMT pipe; transpose + tf32 split into K-major
//      64B-swizzled operands (double-buffered, so the tensor core works on
//      chunk c while chunk c+1 is prepared); one thread issues
//      D += Xhi Xhi^T + Xhi Xlo^T + Xlo Xhi^T (3xTF32, M=N=128, K=8) straight
//      into the TMEM accumulator (no register row sum: that is what caps the
//      two-level-sum kernels at two CTAs per SM)
//   3. blocked Cholesky in TMEM: per 8-column panel the diagonal warp factors
//      the 8x8 block, every row solves against it (forward solve fused) and
//      writes its L entries back into TMEM; the trailing update is 3xTF32
//      MMAs restricted to the columns right of the panel (N = 128 - cs)
//   4. L is copied TMEM -> packed smem (reusing the operand buffers), then
//      backward solve, W update and the cache update yhat -= X d
// Shared memory ~55 KB and 128 TMEM columns per CTA -> 4 CTAs per SM.
#pragma once
#include "ials_tc_common.cuh"

namespace ials {

struct TcLay4 {
  static constexpr int BT = 128, NT = 128, KC = 16, XLD = BT;   // X rows as TMA gathers them
  static constexpr int MR = 8;   // metadata ring depth (chunks)
  // overlay region (1024-aligned), by phase:
  //   accumulate: XT hi/lo double buffer  4 x 8 KB (K-major SW64)
  //   factor + backward: packed L         33,024 B (written as it is factored)
  // the natural staging region holds the panel operands during the
  // factorisation and the diagonal-block inverses during the backward solve
  static constexpr int OFF_XT = 0;
  static constexpr int OFF_L = 0;
  static constexpr int OVL = 33792;
  static constexpr int OFF_X = OVL;                            // natural staging [2][KC][XLD]
  static constexpr int OFF_MC = OFF_X + 2 * KC * XLD * 4;      // ring [MR][KC]: cols
  static constexpr int OFF_MP = OFF_MC + MR * KC * 4;          //                positions
  static constexpr int OFF_MW = OFF_MP + MR * KC * 4;          //                weights
  static constexpr int OFF_MY = OFF_MW + MR * KC * 4;          //                labels
  static constexpr int OFF_CV = OFF_MY + MR * KC * 4;          // [4][KC] gathered yhat
  static constexpr int OFF_DG = OFF_CV + 4 * KC * 4;
  // factored diagonal block of the panel (DG 8x8, 1/pivots RV, y YP),
  // double-buffered by panel parity: buffer x = OFF_DG + x * 320
  static constexpr int OFF_RV = OFF_DG + 64 * 4;
  static constexpr int OFF_YP = OFF_RV + 8 * 4;
  static constexpr int OFF_Y = OFF_DG + 2 * 320;
  static constexpr int OFF_YF = OFF_Y + BT * 4;
  static constexpr int OFF_ID = OFF_YF + BT * 4;
  static constexpr int OFF_D = OFF_ID + BT * 4;
  static constexpr int OFF_PA_HI = OFF_X;          // factor: panel operands hi / lo (2 x 4 KB)
  static constexpr int OFF_LI = OFF_X + 8192;      // backward: 8 x 16x16 block inverses
  static constexpr int OFF_DIAG = OFF_D + BT * 4;  // H_kk before the factorisation
  static constexpr int OFF_FLAG = OFF_DIAG + BT * 4;
  static constexpr int OFF_BAR = OFF_FLAG + 16;    // MMA mbarriers [2], gather mbarriers [2], TMEM base
  static constexpr int OFF_RI = OFF_BAR + 48;      // [2][4]: row, entry begin / end, lam (row prefetch)
  static constexpr int BYTES = OFF_RI + 32 + 1024;
};

// K-major, 64B-swizzle float index of operand element (row m, k) of a
// 16-entry chunk: 8-row atoms of 512 B, 16-byte chunk (k/4) of row m at
// (k/4) ^ ((m/2) % 4).
IALS_DEVI int xt64_index(int m, int k) {
  return (m >> 3) * 128 + (m & 7) * 16 + ((((k >> 2) ^ ((m >> 1) & 3))) << 2) + (k & 3);
}

constexpr uint32_t kSwizzle64B = 4;

struct Tc4State {
  uint32_t tmem;
  uint32_t ph;      // bit x: phase parity of the next completion of bar[x]
  uint32_t gph;     // bit x: the same for the gather barrier of staging buffer x
  const CUtensorMap* fmap;   // fixed[:, fb0:fb0+128] rows for tile::gather4, or null (cp.async)
};

// step 1: TMEM row i := template row i (+ lam on the diagonal), zero above
// (lam I is added where the diagonal is consumed: the factorisation's
// diagonal block and the cancellation reference)
IALS_DEVI void tc4_init(const SweepParams& p, uint32_t row_addr, int tid) {
  const int i = tid;
  const float* tp = p.tpl + pk_off(i);
#pragma unroll 1
  for (int q = 0; q < 2; ++q) {
    float4 x[16];
#pragma unroll
    for (int c4 = 0; c4 < 16; ++c4)
      x[c4] = (64 * q + 4 * c4 <= i) ? __ldg(reinterpret_cast<const float4*>(tp + 64 * q) + c4)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int c8 = 0; c8 < 8; ++c8) {
      const float w8[8] = {x[2 * c8].x, x[2 * c8].y, x[2 * c8].z, x[2 * c8].w,
                           x[2 * c8 + 1].x, x[2 * c8 + 1].y, x[2 * c8 + 1].z, x[2 * c8 + 1].w};
      tmem_st8(row_addr + 64 * q + 8 * c8, w8);
    }
  }
}

// step 2: D += sum over the row's entries of a h h^T; fp64 gradient -> gacc.
//
// Every load is asynchronous and addressed from shared memory: the row's
// metadata (cols, positions, weights, labels) streams through a ring MR
// chunks deep, fetched 4 chunks ahead; the gathered sub-rows X and the
// predictions yhat[pos] are fetched 2 chunks ahead.  cp.async group g (one
// per iteration) = {X(g+2), yhat(g+2), meta(g+4)}, so waiting for group c-2
// at iteration c delivers X(c) and the metadata X(c+2) needs.
template <bool UNIT>
IALS_DEVI void tc4_meta(const SweepParams& p, char* smem, int ebeg, int eend, int c, int tid) {
  using L = TcLay4;
  const int e = ebeg + c * L::KC + (tid & 15);
  const int slot = (c & (L::MR - 1)) * L::KC + (tid & 15);
  if (e >= eend) return;
  if (UNIT && tid >= 32) return;   // all weights and labels are one: not staged
  switch (tid >> 4) {
    case 0: cp_async4(smem + L::OFF_MC + 4 * slot, p.side.cols + e); break;
    case 1: if (p.side.pos) cp_async4(smem + L::OFF_MP + 4 * slot, p.side.pos + e);
            else reinterpret_cast<int*>(smem + L::OFF_MP)[slot] = e;
            break;
    case 2: if (p.side.weights) cp_async4(smem + L::OFF_MW + 4 * slot, p.side.weights + e);
            else reinterpret_cast<float*>(smem + L::OFF_MW)[slot] = 1.f;
            break;
    case 3: if (p.side.labels) cp_async4(smem + L::OFF_MY + 4 * slot, p.side.labels + e);
            else reinterpret_cast<float*>(smem + L::OFF_MY)[slot] = 1.f;
            break;
    default: break;
  }
}

IALS_DEVI void tc4_gather(const SweepParams& p, char* smem, const Tc4State& st, int ebeg, int eend,
                          int c, int tid) {
  using L = TcLay4;
  const int nk = min(L::KC, eend - (ebeg + c * L::KC));
  if (nk <= 0) return;
  const int* mc = reinterpret_cast<const int*>(smem + L::OFF_MC) + (c & (L::MR - 1)) * L::KC;
  const int* mp = reinterpret_cast<const int*>(smem + L::OFF_MP) + (c & (L::MR - 1)) * L::KC;
  float* X = reinterpret_cast<float*>(smem + L::OFF_X) + (c & 1) * L::KC * L::XLD;
  if (st.fmap) {   // one thread (warp 1: warp 0 issues the MMAs): ceil(nk / 4) TMA
                   // gathers of 4 sub-rows (128 floats each)
    if (tid == 32) {
      uint64_t* gb = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR) + 2 + (c & 1);
      const int ng = (nk + 3) >> 2;
      mbar_expect_tx(gb, (uint32_t)ng * 4 * L::XLD * 4);
      for (int g = 0; g < ng; ++g) {
        const int k = 4 * g, last = nk - 1;
        for (int q = k; q < min(k + 4, nk); ++q) IALS_CHECK(mc[q] >= 0 && mc[q] < p.side.n_fixed);
        tma_gather4(smem_u32(X + k * L::XLD), st.fmap, p.fb0, mc[min(k, last)],
                    mc[min(k + 1, last)], mc[min(k + 2, last)], mc[min(k + 3, last)], gb);
      }
    }
  } else if (p.vec) {   // lane <-> 16-byte piece of a sub-row (b <= 128: 32 pieces), warp <-> entry
    const int lane = tid & 31, warp = tid >> 5;
    if (lane < (p.b >> 2)) {
      const float* src = p.fixed + p.fb0 + 4 * lane;
#pragma unroll
      for (int k = warp; k < L::KC; k += L::NT / 32)
        if (k < nk) cp_async16(X + k * L::XLD + 4 * lane, src + (size_t)mc[k] * p.ldf);
    }
  } else {
    for (int i = tid; i < nk * p.b; i += L::NT) {
      const int k = i / p.b, v = i - k * p.b;
      cp_async4(X + k * L::XLD + v, p.fixed + (size_t)mc[k] * p.ldf + p.fb0 + v);
    }
  }
  if (tid < nk) {
    IALS_CHECK(mp[tid] >= 0 && mp[tid] < p.side.nnz);
    cp_async4(smem + L::OFF_CV + 4 * ((c & 3) * L::KC + tid), p.cache + mp[tid]);
  }
}

// UNIT: every weight and label is one (the BASELINE configurations), so the
// residual is yhat - 1 and a h h^T = h h^T.
// SYM2 (heavy-row partials, symmetrised by their consumer): two MMAs per
// k-step, E += hi hi^T + hi (2 lo)^T, whose symmetric part (E + E^T) / 2 is the
// 3xTF32 sum hi hi^T + hi lo^T + lo hi^T (2 lo is exact).
template <bool UNIT, bool SYM2 = false>
IALS_DEVI int tc4_accumulate(const SweepParams& p, char* smem, Tc4State& st, double& gacc, int ebeg,
                             int eend, int tid) {
  using L = TcLay4;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  const int n = eend - ebeg;
  const int nch = (n + L::KC - 1) / L::KC;
  const uint32_t idesc = make_idesc_tf32(128, 128, 0, 0, 0);
  uint32_t pend = 0;   // bit x: bar[x] has an outstanding commit
  if (nch == 0) return 0;
  // prologue: metadata of chunks 0..3, then X / yhat of chunks 0 and 1
  for (int c = 0; c < 4 && c < nch; ++c) tc4_meta<UNIT>(p, smem, ebeg, eend, c, tid);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  tc4_gather(p, smem, st, ebeg, eend, 0, tid);
  tc4_gather(p, smem, st, ebeg, eend, 1, tid);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // one block barrier per chunk: it publishes chunk c's operands to the MMA
  // issuer, the yhat / metadata loads of the chunks ahead to every thread,
  // and frees chunk c's staging buffer for the gather of chunk c+2
  for (int c = 0; c < nch; ++c) {
    const int xb = c & 1;
    const int nk = min(L::KC, eend - (ebeg + c * L::KC));
    if (st.fmap) {   // the sub-rows of chunk c (TMA gather)
      mbar_wait(reinterpret_cast<uint64_t*>(smem + L::OFF_BAR) + 2 + xb, (st.gph >> xb) & 1u);
      st.gph ^= 1u << xb;
    }
    const float* X = reinterpret_cast<const float*>(smem + L::OFF_X) + xb * L::KC * L::XLD;
    const int ms = (c & (L::MR - 1)) * L::KC;
    const float* mw = reinterpret_cast<const float*>(smem + L::OFF_MW) + ms;
    const float* my = reinterpret_cast<const float*>(smem + L::OFF_MY) + ms;
    const float* cv = reinterpret_cast<const float*>(smem + L::OFF_CV) + (c & 3) * L::KC;
    // thread m <-> factor column m = operand row m: its 16 entries of the
    // chunk (conflict-free loads) feed the fp64 gradient and the hi/lo split
    float x[16];
    const bool colok = tid < p.b;   // columns >= b are not gathered
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = (colok && k < nk) ? X[k * L::XLD + tid] : 0.f;
    float wk[16];   // the chunk's weights: 16-byte broadcast reads of the rings
    {  // gradient: the chunk's 16 products in four fixed-order fp32 chains
       // (entries k mod 4), folded into the fp64 row sum (long rows cancel
       // across chunks, so the row sum itself stays fp64)
      float g[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const float4 c4 = reinterpret_cast<const float4*>(cv)[k4];
        const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
        float w[4] = {1.f, 1.f, 1.f, 1.f}, yy[4] = {1.f, 1.f, 1.f, 1.f};
        if (!UNIT) {
          const float4 w4 = reinterpret_cast<const float4*>(mw)[k4];
          const float4 y4 = reinterpret_cast<const float4*>(my)[k4];
          w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
          yy[0] = y4.x; yy[1] = y4.y; yy[2] = y4.z; yy[3] = y4.w;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = 4 * k4 + j;
          wk[k] = w[j];
          // (stale ring slots past nk may hold anything: select, do not multiply)
          const float r = (k < nk) ? (UNIT ? cc[j] - 1.f : w[j] * (cc[j] - yy[j])) : 0.f;
          g[j] = fmaf(r, x[k], g[j]);
        }
      }
      gacc += ((double)g[0] + (double)g[1]) + ((double)g[2] + (double)g[3]);
    }
    if (!UNIT && p.side.weights) {  // a h h^T = (sqrt(a) h)(sqrt(a) h)^T
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] *= (k < nk) ? sqrtf(wk[k]) : 0.f;
    }
    // the operand buffer xb was last read by chunk c-2's MMAs
    if (pend & (1u << xb)) {
      mbar_wait(bar + xb, (st.ph >> xb) & 1u);
      st.ph ^= 1u << xb;
      pend &= ~(1u << xb);
    }
    {  // row m of the K-major 64B-swizzled operands: 16-byte chunk c (entries
       // 4c..4c+3) at chunk c ^ ((m / 2) % 4) of the row's 64 bytes
      float* XTH = reinterpret_cast<float*>(smem + L::OFF_XT + xb * 16384);
      float* XTL = XTH + 2048;
      const int m = tid, rb = (m >> 3) * 128 + (m & 7) * 16, sw = (m >> 1) & 3;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float hi[4], lo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          hi[j] = tf32_rna(x[4 * c + j]);
          lo[j] = x[4 * c + j] - hi[j];   // fed as is: the MMA drops its low 13 bits
          if (SYM2) lo[j] *= 2.f;
        }
        const int o = rb + ((c ^ sw) << 2);
        *reinterpret_cast<float4*>(XTH + o) = make_float4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<float4*>(XTL + o) = make_float4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
    cp_async_wait<0>();   // this thread's yhat / metadata loads of the chunks ahead
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t hi = smem_u32(smem + L::OFF_XT + xb * 16384), lo = hi + 8192;
      const int ksteps = (nk + 7) >> 3;
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t ah = make_sdesc(hi + ks * 32, 16, 512, kSwizzle64B);
        const uint64_t al = make_sdesc(lo + ks * 32, 16, 512, kSwizzle64B);
        umma_tf32(st.tmem, ah, ah, idesc, 1);
        umma_tf32(st.tmem, ah, al, idesc, 1);
        if (!SYM2) umma_tf32(st.tmem, al, ah, idesc, 1);
      }
      umma_commit(bar + xb);
    }
    pend |= 1u << xb;
    // X / yhat of chunk c+2 (its staging buffer was consumed above), and the
    // metadata of chunk c+4
    if (c + 2 < nch) tc4_gather(p, smem, st, ebeg, eend, c + 2, tid);
    if (c + 4 < nch) tc4_meta<UNIT>(p, smem, ebeg, eend, c + 4, tid);
    cp_async_commit();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int xb = 0; xb < 2; ++xb)
    if (pend & (1u << xb)) {
      mbar_wait(bar + xb, (st.ph >> xb) & 1u);
      st.ph ^= 1u << xb;
    }
  tc_fence_after();
  return nch;
}

// step 3: Cholesky of the TMEM matrix + forward solve, written straight into
// the packed L the backward solve reads; 1/diag in OFF_ID, forward-solved y
// in OFF_YF.  Per 8-column panel (c0 = 8p):
//   * every row loads its panel entries from TMEM (fully updated: the
//     trailing MMA of the previous panel has completed);
//   * the 8 rows of the diagonal block are 8 consecutive lanes of one warp:
//     that warp gathers the block with shuffles, factors it (forward solve
//     included) and publishes it;
//   * every row below solves against the block (forward solve fused);
//   * l goes to the packed L and, split hi/lo, to the panel operand of the
//     3xTF32 trailing update D -= L_p L_p^T (columns >= cs only).
IALS_DEVI void tc4_factor(const SweepParams& p, char* smem, Tc4State& st, uint32_t row_addr, int row,
                          int tid, bool prof = false) {
  long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const bool watch = prof && (tid == 0 || tid == 64 || tid == 96);
  using L = TcLay4;
  float* ys = reinterpret_cast<float*>(smem + L::OFF_Y);
  float* yf = reinterpret_cast<float*>(smem + L::OFF_YF);
  float* invd = reinterpret_cast<float*>(smem + L::OFF_ID);
  const float* DIAG = reinterpret_cast<const float*>(smem + L::OFF_DIAG);
  int* FLAG = reinterpret_cast<int*>(smem + L::OFF_FLAG);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  float* lrow = reinterpret_cast<float*>(smem + L::OFF_L) + tid * (tid + 1) / 2;   // packed row
  const int b = p.b, i = tid, lane = tid & 31, warp = tid >> 5;
  const int np = (b + 7) >> 3;
  (void)row;
  float yi = ys[i];
  for (int pp = 0; pp < np; ++pp) {
    const int c0 = pp * 8;
    float* DG = reinterpret_cast<float*>(smem + L::OFF_DG + (pp & 1) * 320);
    float* RV = reinterpret_cast<float*>(smem + L::OFF_RV + (pp & 1) * 320);
    float* YP = reinterpret_cast<float*>(smem + L::OFF_YP + (pp & 1) * 320);
    float v[8];
    tmem_ld8(row_addr + c0, v);
    tmem_wait_ld();
    if (watch && pp == 8) acc[6] = clock64();
    if (warp == (c0 >> 5)) {
      // the diagonal block's rows are lanes base..base+7 of this warp: they
      // stage their panel entries and y in shared memory, every lane reads
      // the block back (18 broadcast loads instead of 44 shuffles: this warp's
      // instruction count is the panel's critical path) and factors it
      // redundantly (a short dependent chain), lane `base` publishes it
      const int base = c0 & 31;
      float* SG = reinterpret_cast<float*>(smem + L::OFF_LI);   // free until the backward solve
      if (lane >= base && lane < base + 8) {
        const int q = lane - base;
        reinterpret_cast<float4*>(SG)[2 * q] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(SG)[2 * q + 1] = make_float4(v[4], v[5], v[6], v[7]);
        SG[64 + q] = yi;
      }
      __syncwarp();
      float a[8][8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 x0 = reinterpret_cast<const float4*>(SG)[2 * q];
        const float4 x1 = reinterpret_cast<const float4*>(SG)[2 * q + 1];
        a[q][0] = x0.x; a[q][1] = x0.y; a[q][2] = x0.z; a[q][3] = x0.w;
        a[q][4] = x1.x; a[q][5] = x1.y; a[q][6] = x1.z; a[q][7] = x1.w;
      }
      float py[8];
      {
        const float4 y0 = reinterpret_cast<const float4*>(SG + 64)[0];
        const float4 y1 = reinterpret_cast<const float4*>(SG + 64)[1];
        py[0] = y0.x; py[1] = y0.y; py[2] = y0.z; py[3] = y0.w;
        py[4] = y1.x; py[5] = y1.y; py[6] = y1.z; py[7] = y1.w;
      }
      __syncwarp();   // SG is rewritten by the next panel's block
      float rinv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // a non-positive / non-finite pivot yields a NaN, infinite or zero
        // 1/pivot, which the cancellation test (record_block) flags; the
        // row's own numbers are then discarded and it is redone in FP32
        const float dk = a[k][k];
        float r;   // MUFU.RSQ without the denormal rescale (a denormal pivot is rejected anyway)
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(dk));
        rinv[k] = r;
        a[k][k] = dk * r;
#pragma unroll
        for (int q = k + 1; q < 8; ++q) a[q][k] *= r;
#pragma unroll
        for (int q = k + 1; q < 8; ++q)
#pragma unroll
          for (int m = k + 1; m <= q; ++m) a[q][m] = fmaf(-a[q][k], a[m][k], a[q][m]);
      }
      float yp[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float t = py[q];
#pragma unroll
        for (int m = 0; m < q; ++m) t = fmaf(-a[q][m], yp[m], t);
        yp[q] = t * rinv[q];
      }
      if (lane == base) {   // only what the other rows wait for
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float w[8];
#pragma unroll
          for (int m = 0; m < 8; ++m) w[m] = (m <= q) ? a[q][m] : 0.f;
          reinterpret_cast<float4*>(DG)[2 * q] = make_float4(w[0], w[1], w[2], w[3]);
          // readers use entries m <= q only: rows 0..3 have no upper half to store
          if (q >= 4) reinterpret_cast<float4*>(DG)[2 * q + 1] = make_float4(w[4], w[5], w[6], w[7]);
        }
        reinterpret_cast<float4*>(RV)[0] = make_float4(rinv[0], rinv[1], rinv[2], rinv[3]);
        reinterpret_cast<float4*>(RV)[1] = make_float4(rinv[4], rinv[5], rinv[6], rinv[7]);
        reinterpret_cast<float4*>(YP)[0] = make_float4(yp[0], yp[1], yp[2], yp[3]);
        reinterpret_cast<float4*>(YP)[1] = make_float4(yp[4], yp[5], yp[6], yp[7]);
      }
    }
    __syncthreads();
    if (watch && pp == 8) acc[1] = clock64();
    // the block's rows record their part of L, 1/pivot and y, and test the
    // pivot for cancellation: one that lost more than cond_max of its
    // diagonal is beyond what the 3xTF32 Hessian resolves (FP32 SIMT redo).
    // Runs in the shadow of the trailing MMA (buffers are double-buffered).
    auto record_block = [&]() {
      if (i >= c0 && i < c0 + 8) {
        const int j = i - c0;
        const float4 x0 = reinterpret_cast<const float4*>(DG)[2 * j];
        const float4 x1 = reinterpret_cast<const float4*>(DG)[2 * j + 1];
        const float w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
        for (int m = 0; m < 8; ++m)
          if (m <= j) lrow[c0 + m] = w[m];
        const float r = RV[j];
        invd[i] = r;
        yf[i] = YP[j];
        if (i < b && !(r > 0.f && DIAG[i] * (r * r) <= p.cond_max)) *FLAG = 1;
      }
    };
    float l[8];
    if (i >= c0 + 8 && i < b) {
      const float4 r0 = reinterpret_cast<const float4*>(RV)[0], r1 = reinterpret_cast<const float4*>(RV)[1];
      const float4 y0 = reinterpret_cast<const float4*>(YP)[0], y1 = reinterpret_cast<const float4*>(YP)[1];
      const float rinv[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
      const float yp[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 x0 = reinterpret_cast<const float4*>(DG)[2 * q];
        const float4 x1 = reinterpret_cast<const float4*>(DG)[2 * q + 1];
        const float w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        float tt = v[q];
#pragma unroll
        for (int m = 0; m < q; ++m) tt = fmaf(-l[m], w[m], tt);
        l[q] = tt * rinv[q];
        yi = fmaf(-l[q], yp[q], yi);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) lrow[c0 + q] = l[q];
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) l[q] = 0.f;   // no part in the trailing update
    }
    if (watch && pp == 8) acc[3] = clock64();
    if (pp + 1 < np) {
      float* PAH = reinterpret_cast<float*>(smem + L::OFF_PA_HI);
      float* PAL = PAH + 1024;   // 4 KB apart
      float hi[8], lo[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        hi[q] = tf32_rna(l[q]);
        lo[q] = l[q] - hi[q];
      }
      const int pa = pa_index(i, 0);   // q 0..3 contiguous, q 4..7 at +32
      *reinterpret_cast<float4*>(PAH + pa) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<float4*>(PAH + pa + 32) = make_float4(hi[4], hi[5], hi[6], hi[7]);
      *reinterpret_cast<float4*>(PAL + pa) = make_float4(lo[0], lo[1], lo[2], lo[3]);
      *reinterpret_cast<float4*>(PAL + pa + 32) = make_float4(lo[4], lo[5], lo[6], lo[7]);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      if (watch && pp == 8) acc[4] = clock64();
      if (tid == 0) {
        tc_fence_after();
        const int cs = ((c0 + 8) >> 4) << 4;   // N = 128 - cs, a multiple of 16
        const uint32_t idesc_neg = make_idesc_tf32(128, 128 - cs, 0, 0, 1);
        const uint32_t ph = smem_u32(PAH), pl = smem_u32(PAL);
        const uint64_t ah = make_sdesc(ph, 128, 256, kSwizzleNone);
        const uint64_t al = make_sdesc(pl, 128, 256, kSwizzleNone);
        const uint64_t bh = make_sdesc(ph + (cs >> 3) * 256, 128, 256, kSwizzleNone);
        const uint64_t bl = make_sdesc(pl + (cs >> 3) * 256, 128, 256, kSwizzleNone);
        umma_tf32(st.tmem + cs, ah, bh, idesc_neg, 1);
        umma_tf32(st.tmem + cs, ah, bl, idesc_neg, 1);
        umma_tf32(st.tmem + cs, al, bh, idesc_neg, 1);
        umma_commit(bar);
      }
      record_block();
      mbar_wait(bar, st.ph & 1u);
      if (watch && pp == 8) acc[5] = clock64();
      st.ph ^= 1u;
      tc_fence_after();
    } else {
      record_block();
    }
  }
  __syncthreads();
  if (watch) {
    const int w = tid == 0 ? 0 : (tid == 64 ? 1 : 2);
    for (int k = 0; k < 8; ++k) p.dbg[8192 + (blockIdx.x * 3 + w) * 8 + k] = acc[k];
  }
}

// Inverses of the 16x16 diagonal blocks of L (from the packed copy), all at
// once: thread t forms column q = t % 16 of block t / 16 by forward
// substitution with the stored reciprocal pivots.  LI[blk][m][q] (16 x 16,
// lower triangular).
IALS_DEVI void tc4_block_inverses(const SweepParams& p, char* smem, int tid) {
  using L = TcLay4;
  const float* Lp = reinterpret_cast<const float*>(smem + L::OFF_L);
  const float* invd = reinterpret_cast<const float*>(smem + L::OFF_ID);
  float* LI = reinterpret_cast<float*>(smem + L::OFF_LI);
  const int nb = (p.b + 15) >> 4, blk = tid >> 4, q = tid & 15, c0 = 16 * blk;
  if (blk >= nb) return;
  float x[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int gm = c0 + m;
    float t = (m == q) ? 1.f : 0.f;
    const float* lr = Lp + gm * (gm + 1) / 2 + c0;
    // x[k] = 0 for k < q, so those terms add exactly nothing; rows >= b read
    // unwritten packed rows, but their x is selected to zero below
#pragma unroll
    for (int k = 0; k < m; ++k) t = fmaf(-lr[k], x[k], t);
    x[m] = (m >= q && gm < p.b) ? t * invd[gm] : 0.f;
  }
#pragma unroll
  for (int m = 0; m < 16; ++m) LI[blk * 256 + m * 16 + q] = x[m];
}

// Backward solve L^T d = y by 16-wide blocks from the last: 16 threads form
// the block's unknowns d = L11^-T y_blk (dot products with the precomputed
// inverse), then every row r < c0 folds them into its own y_r.
IALS_DEVI void tc4_backward(const SweepParams& p, char* smem, int tid) {
  using L = TcLay4;
  const float* Lp = reinterpret_cast<const float*>(smem + L::OFF_L);
  const float* LI = reinterpret_cast<const float*>(smem + L::OFF_LI);
  float* yf = reinterpret_cast<float*>(smem + L::OFF_YF);
  float* ds = reinterpret_cast<float*>(smem + L::OFF_D);
  const int b = p.b;
  const int nb = (b + 15) >> 4;
  float yr = (tid < b) ? yf[tid] : 0.f;
  for (int pb = nb - 1; pb >= 0; --pb) {
    const int c0 = pb * 16;
    if (tid < 16) {   // d_q = sum_{m >= q} LI[m][q] y_m
      const int q = tid;
      const float* li = LI + pb * 256 + q;
      float t0 = 0.f, t1 = 0.f;
#pragma unroll
      for (int m = 0; m < 16; m += 2) {
        if (m >= q && c0 + m < b) t0 = fmaf(li[m * 16], yf[c0 + m], t0);
        if (m + 1 >= q && c0 + m + 1 < b) t1 = fmaf(li[(m + 1) * 16], yf[c0 + m + 1], t1);
      }
      if (c0 + q < b) ds[c0 + q] = t0 + t1;
    }
    __syncthreads();
    if (tid < c0) {
      const float4* dq = reinterpret_cast<const float4*>(ds + c0);
      float a0 = yr, a1 = 0.f;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const float4 dv = dq[q4];
        const int g = c0 + 4 * q4;   // rows >= b of the packed L were never written
        if (g < b) a0 = fmaf(-Lp[g * (g + 1) / 2 + tid], dv.x, a0);
        if (g + 1 < b) a1 = fmaf(-Lp[(g + 1) * (g + 2) / 2 + tid], dv.y, a1);
        if (g + 2 < b) a0 = fmaf(-Lp[(g + 2) * (g + 3) / 2 + tid], dv.z, a0);
        if (g + 3 < b) a1 = fmaf(-Lp[(g + 3) * (g + 4) / 2 + tid], dv.w, a1);
      }
      yr = a0 + a1;
      if (tid >= c0 - 16) yf[tid] = yr;   // the next block's entries
    }
    __syncthreads();
  }
}

template <bool UNIT>
__global__ void __launch_bounds__(128, 4) k_sweep_tc4(SweepParams p,
                                                          const __grid_constant__ CUtensorMap fmap,
                                                          int use_tma) {
  using L = TcLay4;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = tc_smem_base(smem_raw);
  const int tid = threadIdx.x;
  {  // finite staging everywhere (padding columns / short chunks read zeros)
    float4* x = reinterpret_cast<float4*>(smem + L::OFF_X);
    for (int i = tid; i < 2 * L::KC * L::XLD / 4; i += L::NT) x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L::OFF_BAR + 32);
  float* ys = reinterpret_cast<float*>(smem + L::OFF_Y);
  float* ds = reinterpret_cast<float*>(smem + L::OFF_D);
  ds[tid] = 0.f;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_init(bar + 2, 1);
    mbar_init(bar + 3, 1);
    if (use_tma) prefetch_tmap(&fmap);
  }
  if (tid < 32) tmem_alloc(tptr, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  Tc4State st;
  st.tmem = *tptr;
  st.ph = 0u;
  st.gph = 0u;
  st.fmap = use_tma ? &fmap : nullptr;
  const uint32_t row_addr = st.tmem + ((uint32_t)((tid >> 5) * 32) << 16);
  const int b = p.b;
  int ndone = 0;
  long long tph[8];
  // profiling: phase clocks of the CTA's rec_row-th row (dbg[32767] picks it; dbg holds 32K int64)
  const int rec_row = p.dbg ? (int)p.dbg[32767] : -1;
  // rows (descending degree) from a device queue (redo_cnt[2], zeroed per
  // pass): greedy longest-first; the next index is fetched while the current
  // row runs
  int* queue = p.redo_cnt + 2;
  int* next = reinterpret_cast<int*>(smem + L::OFF_FLAG) + 2;
  // the first user pass of ials_epoch_host sweeps the light rows chunk by
  // chunk as their rows of W arrive: this launch's slice of the grouped list
  const int* lrows = p.light_rows;
  int n_light = p.n_light;
  if (p.chunk_tot) {
    int off = 0;
    for (int k = 0; k < p.chunk; ++k) off += p.chunk_tot[k];
    lrows += off;
    n_light = p.chunk_tot[p.chunk];
  }
  // row info double buffer: the next row's id, entry range and lam are
  // fetched by thread 0 while the current row is factored
  int* RI = reinterpret_cast<int*>(smem + L::OFF_RI);
  auto put_row = [&](int rb, int r) {
    RI[4 * rb] = r;
    RI[4 * rb + 1] = p.side.ptr[r];
    RI[4 * rb + 2] = p.side.ptr[r + 1];
    reinterpret_cast<float*>(RI)[4 * rb + 3] = p.side.lam[r];
  };
  if (tid == 0) {
    const int t0 = atomicAdd(queue, 1);
    *next = t0;
    if (t0 < n_light) put_row(0, lrows[t0]);
  }
  __syncthreads();
  int task = *next;
  int rb = 0;
  while (task < n_light) {
    int nxt = 0;
    if (tid == 0) nxt = atomicAdd(queue, 1);   // consumed after the accumulate
    const bool rec = ndone == rec_row && tid == 0;
    if (rec) tph[0] = clock64();
    const int row = RI[4 * rb];
    const int ebeg = RI[4 * rb + 1], eend = RI[4 * rb + 2];
    const float lam = reinterpret_cast<const float*>(RI)[4 * rb + 3];
    // the projection and own value of this thread's column, used after the accumulate
    const float pj = (tid < b) ? __ldg(p.proj + (size_t)row * b + tid) : 0.f;
    const float ow = (tid < b) ? (p.rot ? __ldg(p.wq + (size_t)row * b + tid)
                                        : p.own[(size_t)row * p.ldo + p.b0 + tid]) : 0.f;
    tc4_init(p, row_addr, tid);
    if (rec) tph[1] = clock64();
    tmem_wait_st();
    tc_fence_before();   // the first chunk's barrier orders these stores before the MMAs
    double gacc = 0.0;
    const int nch = tc4_accumulate<UNIT>(p, smem, st, gacc, ebeg, eend, tid);
    const int nrow = (tid == 0 && nxt < n_light) ? lrows[nxt] : -1;   // lands during the factorisation
    if (rec) tph[2] = clock64();
    {  // + lam on the diagonal, and the diagonal itself (the cancellation
       // test's reference): lane l of warp w owns column 32w + l, reached with
       // 8-wide TMEM loads / stores of the warp's diagonal block and selects
       // (an indexed register read would go through local memory)
      const int lane = tid & 31, e = lane & 7;
      const float lv = (tid < b) ? lam : 0.f;
      float dg = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v[8];
        const uint32_t ca = row_addr + 32 * (tid >> 5) + 8 * j;
        tmem_ld8(ca, v);
        tmem_wait_ld();
        const bool mine = (lane >> 3) == j;
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] += (mine && m == e) ? lv : 0.f;
        tmem_st8(ca, v);
        const float a0 = (e & 1) ? v[1] : v[0], a1 = (e & 1) ? v[3] : v[2];
        const float a2 = (e & 1) ? v[5] : v[4], a3 = (e & 1) ? v[7] : v[6];
        const float b0 = (e & 2) ? a1 : a0, b1 = (e & 2) ? a3 : a2;
        if (mine) dg = (e & 4) ? b1 : b0;
      }
      tmem_wait_st();
      reinterpret_cast<float*>(smem + L::OFF_DIAG)[tid] = dg;
      if (tid == 0) *reinterpret_cast<int*>(smem + L::OFF_FLAG) = 0;
    }
    {
      float gv = 0.f;
      if (tid < b) gv = (float)(gacc + (double)pj + (double)lam * (double)ow);
      ys[tid] = gv;
    }
    __syncthreads();
    if (rec) tph[3] = clock64();
    tc4_factor(p, smem, st, row_addr, row, tid, ndone == rec_row);
    if (tid == 0) {
      if (nrow >= 0) put_row(rb ^ 1, nrow);
      *next = nxt;
    }
    if (rec) tph[4] = clock64();
    (void)nch;
    if (*reinterpret_cast<volatile int*>(smem + L::OFF_FLAG)) {
      // the SIMT sweep redoes this row (its own cache update included)
      if (tid == 0) {
        p.redo_rows[atomicAdd(p.redo_cnt, 1)] = row;
        atomicAdd(p.redo_total, 1ull);
      }
      if (tid < b) p.drow[(size_t)row * b + tid] = 0.f;
    } else {
      tc4_block_inverses(p, smem, tid);
      __syncthreads();
      tc4_backward(p, smem, tid);
      if (rec) tph[5] = clock64();
      if (tid < b) {
        if (!p.rot) p.own[(size_t)row * p.ldo + p.b0 + tid] = ow - ds[tid];
        p.drow[(size_t)row * b + tid] = ds[tid];   // for k_pass_cache (and the back-rotation)
      }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (rec) {
      tph[6] = clock64();
      tph[7] = eend - ebeg;
      for (int k = 0; k < 8; ++k) p.dbg[blockIdx.x * 8 + k] = tph[k];
    }
    ++ndone;
    task = *next;   // written after the factorisation, published by the barriers since
    rb ^= 1;
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free(st.tmem, 128);
}

// Heavy-row slices on the tensor core: each slice's partial Hessian is summed
// from zero in TMEM (same pipelined gather as the light rows, two MMAs per
// k-step: the non-symmetric E of tc4_accumulate<., true>) and written
// row-major with its fp64 partial gradient; k_heavy_solve<128, ., true>
// combines the slices of a row and takes the symmetric part.
template <bool UNIT>
__global__ void __launch_bounds__(128, 4) k_heavy_partial_tc4(SweepParams p,
                                                          const __grid_constant__ CUtensorMap fmap,
                                                          int use_tma) {
  using L = TcLay4;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = tc_smem_base(smem_raw);
  const int tid = threadIdx.x;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L::OFF_BAR + 32);
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_init(bar + 2, 1);
    mbar_init(bar + 3, 1);
    if (use_tma) prefetch_tmap(&fmap);
  }
  if (tid < 32) tmem_alloc(tptr, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  Tc4State st;
  st.tmem = *tptr;
  st.ph = 0u;
  st.gph = 0u;
  st.fmap = use_tma ? &fmap : nullptr;
  const uint32_t row_addr = st.tmem + ((uint32_t)((tid >> 5) * 32) << 16);
  // slices from a device queue (redo_cnt[1], zeroed per pass): CTAs that
  // start late -- beside the light-row sweep on another stream -- take fewer
  int* queue = p.redo_cnt + 1;
  int* next = reinterpret_cast<int*>(smem + L::OFF_FLAG) + 1;
  for (;;) {
    if (tid == 0) *next = atomicAdd(queue, 1);
    __syncthreads();
    const int sl = *next;
    __syncthreads();
    if (sl >= p.n_slices) break;
    {
      const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c8 = 0; c8 < 16; ++c8) tmem_st8(row_addr + 8 * c8, z);
      tmem_wait_st();
      tc_fence_before();   // ordered before the MMAs by the first chunk's barrier
    }
    double gacc = 0.0;
    tc4_accumulate<UNIT, true>(p, smem, st, gacc, p.slice_begin[sl], p.slice_end[sl], tid);
    float* hp = p.hpart + (size_t)sl * 128 * 128 + (size_t)tid * 128;
#pragma unroll
    for (int c32 = 0; c32 < 4; ++c32) {
      float v[32];
      tmem_ld32(row_addr + 32 * c32, v);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(hp + 32 * c32 + 4 * q) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    p.gpart[(size_t)sl * 128 + tid] = gacc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free(st.tmem, 128);
}

// yhat[pos] -= x . d for every entry of the pass: light rows take d from
// drow (the fused sweep's output; zero for rows the SIMT sweep redid), heavy
// slices from hdelta.  One CTA per row (or slice), 8 lanes per entry, 32
// entries in flight; lane g of an entry reads the 16-byte pieces 4g + 32q
// (q = 0..3), so each load instruction covers whole 128-byte lines.
// Bandwidth-bound gather: its own full-occupancy pass.
__global__ void __launch_bounds__(256) k_pass_cache(SweepParams p) {
  const int tid = threadIdx.x, g = tid & 7, slot = tid >> 3;
  const int blk = blockIdx.x;
  const float* d;
  int ebeg, eend;
  if (blk < p.n_light) {
    const int row = p.light_rows[blk];
    ebeg = p.side.ptr[row];
    eend = p.side.ptr[row + 1];
    d = p.drow + (size_t)row * p.b;
  } else {
    const int sl = blk - p.n_light;
    ebeg = p.slice_begin[sl];
    eend = p.slice_end[sl];
    d = p.hdelta + (size_t)p.slice_heavy[sl] * 128;
  }
  const int b = p.b;
  float dv[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = 32 * q + 4 * g;
    if (p.vec) {
      const float4 t = (c < b) ? __ldg(reinterpret_cast<const float4*>(d + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      dv[4 * q] = t.x; dv[4 * q + 1] = t.y; dv[4 * q + 2] = t.z; dv[4 * q + 3] = t.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) dv[4 * q + j] = (c + j < b) ? __ldg(d + c + j) : 0.f;
    }
  }
  for (int e0 = ebeg; e0 < eend; e0 += 32) {   // block-uniform trip count (shuffles below)
    const int e = e0 + slot;
    const bool live = e < eend;
    const int col = live ? __ldg(p.side.cols + e) : 0;
    const float* xr = p.fixed + (size_t)col * p.ldf + p.fb0;
    float s = 0.f;
    if (!live) {
    } else if (p.vec) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = 32 * q + 4 * g;
        if (c < b) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(xr + c));
          s = fmaf(x.x, dv[4 * q], s);
          s = fmaf(x.y, dv[4 * q + 1], s);
          s = fmaf(x.z, dv[4 * q + 2], s);
          s = fmaf(x.w, dv[4 * q + 3], s);
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = 32 * q + 4 * g + j;
          if (c < b) s = fmaf(__ldg(xr + c), dv[4 * q + j], s);
        }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (live && g == 0) {
      const int pos = p.side.pos ? __ldg(p.side.pos + e) : e;
      p.cache[pos] -= s;
    }
  }
}

// The same cache update, entry-parallel: every warp takes a contiguous run
// of the side's entries (storage order), 4 at a time (8 lanes each), and
// keeps the current row's d (drow[rows[e]]; heavy rows included --
// k_heavy_solve stores theirs there too -- and d = 0 for rows the SIMT sweep
// redid) in registers, reloading it only when its entries cross into the
// next row.  No per-row setup and no row-length imbalance.  Latency-bound
// (a dependent ids -> sub-row -> cache chain per entry): the loop is software
// pipelined -- the next step's ids are loaded one step ahead, and a step's
// 32 / LPE entries issue all their sub-row and cache loads before the dot
// product.  Per entry the sum is the same fixed-order chain as before
// (bit-identical results).  Measured at L1 (ncu, per launch): U = 1 at 4
// CTAs/SM 502 / 692 us (user / item side) against 539 / 972 us unpipelined;
// U = 2 (80 registers, 3 CTAs/SM) 568 / 812 us; capping registers for 5 or 6
// CTAs/SM spills (675 / 875, 1045 / 1155 us).  The vectorised variant (b % 4
// == 0, no per-element width tests) cut the instruction count 428M -> 271M
// (387 / 574 us); 4 lanes per entry executes 27% fewer instructions but needs
// 123 registers (2 CTAs/SM): 403 / 738 us.
// SWAP: walk the other side's view of the entries instead (x_rows / x_cols /
// x_pos): the vector held across a run is then the fixed side's sub-row and
// the gathered one this side's d (drow, n_rows x b: L2-resident when this
// side is the smaller one -- the item pass, whose fixed W[:, pi] is 70 MB at
// L1 and 292 MB at msd).  Each entry's sum is the same fixed-order chain of
// the same products (fma is commutative in its factors): bit-identical.
// BMAX: the widest block the instantiation serves (b <= 16 with LPE = 4: one
// float4 per lane, 8 entries per warp step; b <= 32 with LPE = 4: two).
template <bool VEC, int LPE, bool SWAP, int BMAX = 128>
__global__ void __launch_bounds__(256, (LPE == 8 || BMAX <= 64) ? 4 : 2) k_pass_cache_flat(SweepParams p, long long nnz) {
  constexpr int EPW = 32 / LPE, NQ = BMAX / (4 * LPE);   // entries per warp step, float4 per lane
  const int lane = threadIdx.x & 31, g = lane % LPE, sub = lane / LPE;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long per = ((nnz + nwarps - 1) / nwarps + EPW - 1) / EPW * EPW;
  const long long beg = wid * per, end = min(nnz, beg + per);
  const int b = p.b;
  const int* __restrict__ R = SWAP ? p.x_rows : p.side.rows;   // the run's (held) vector
  const int* __restrict__ C = SWAP ? p.x_cols : p.side.cols;   // the gathered vector
  const int* __restrict__ PS = SWAP ? p.x_pos : p.side.pos;
  int cur = -1, cur_skip_row = -1;
  bool cur_skip = false;
  float dv[4 * NQ];
#pragma unroll
  for (int j = 0; j < 4 * NQ; ++j) dv[j] = 0.f;
  int nrow, ncol;
  {
    const long long e = beg + sub;
    nrow = e < end ? __ldg(R + e) : -1;
    ncol = e < end ? __ldg(C + e) : 0;
  }
  for (long long e0 = beg; e0 < end; e0 += EPW) {   // warp-uniform trip count (shuffles below)
    const int row = nrow, col = ncol;
    {
      const long long e = e0 + EPW + sub;
      nrow = e < end ? __ldg(R + e) : -1;
      ncol = e < end ? __ldg(C + e) : 0;
    }
    bool live = row >= 0;
    if (!SWAP && p.flat_skip_deg > 0 && live) {   // rows whose solver updated their cache itself
      if (row != cur_skip_row) {
        cur_skip_row = row;
        cur_skip = __ldg(p.side.ptr + row + 1) - __ldg(p.side.ptr + row) <= p.flat_skip_deg;
      }
      live = !cur_skip;
    }
    float4 x[NQ];
    const float* xr = SWAP ? p.drow + (size_t)col * b : p.fixed + (size_t)col * p.ldf + p.fb0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = 4 * LPE * q + 4 * g;
      x[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (live && c < b) {
        if (VEC) {   // b % 4 == 0: c < b covers the whole float4
          x[q] = __ldg(reinterpret_cast<const float4*>(xr + c));
        } else {
          x[q].x = __ldg(xr + c);
          if (c + 1 < b) x[q].y = __ldg(xr + c + 1);
          if (c + 2 < b) x[q].z = __ldg(xr + c + 2);
          if (c + 3 < b) x[q].w = __ldg(xr + c + 3);
        }
      }
    }
    const long long e = e0 + sub;
    const long long pos = (live && g == 0) ? (PS ? (long long)__ldg(PS + e) : e) : 0;
    IALS_CHECK(!live || (col >= 0 && row >= 0 && pos >= 0 && pos < nnz));
    const float cold = (live && g == 0) ? p.cache[pos] : 0.f;
    if (live && row != cur) {
      const float* dr = SWAP ? p.fixed + (size_t)row * p.ldf + p.fb0 : p.drow + (size_t)row * b;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int c = 4 * LPE * q + 4 * g;
        if (VEC) {
          const float4 t = (c < b) ? __ldg(reinterpret_cast<const float4*>(dr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
          dv[4 * q] = t.x; dv[4 * q + 1] = t.y; dv[4 * q + 2] = t.z; dv[4 * q + 3] = t.w;
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) dv[4 * q + j] = (c + j < b) ? __ldg(dr + c + j) : 0.f;
        }
      }
      cur = row;
    }
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = 4 * LPE * q + 4 * g;
      if (c < b) {   // columns >= b are skipped (not added as +0 terms)
        s = fmaf(x[q].x, dv[4 * q], s);
        if (VEC || c + 1 < b) s = fmaf(x[q].y, dv[4 * q + 1], s);
        if (VEC || c + 2 < b) s = fmaf(x[q].z, dv[4 * q + 2], s);
        if (VEC || c + 3 < b) s = fmaf(x[q].w, dv[4 * q + 3], s);
      }
    }
#pragma unroll
    for (int o = 1; o < LPE; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (live && g == 0) p.cache[pos] = cold - s;
  }
}

}  // namespace ials
