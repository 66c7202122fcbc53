// ials_sweep_tc.cuh -- tensor-core (tcgen05) block sweep for block widths
// 33..128 (BT = 128).  Same math as k_sweep_light (ials_sweep.cuh), but the
// row's 128x128 Hessian lives in TMEM:
//
//   * TMEM D := alpha0*slab[pi,pi] + lam*I (tcgen05.st, one row per thread)
//   * per chunk of 32 gathered sub-rows (cp.async, double buffered): fp64
//     gradient sum on the SIMT pipe, then the chunk is transposed into
//     K-major 128B-swizzled operands X^T (hi) and X^T - tf32(X^T) (lo) and one
//     thread issues D += Xhi Xhi^T + Xhi Xlo^T + Xlo Xhi^T (3xTF32, fp32
//     accumulate; kind::tf32 M=128 N=128 K=8)
//   * blocked right-looking Cholesky on the TMEM matrix: per 8-column panel
//     every thread tcgen05.ld's its row's 8 panel values, the 8x8 diagonal
//     block is shared through smem and factored redundantly per thread, each
//     row is triangular-solved against it (forward solve fused), and the
//     trailing update D -= L_p L_p^T is three more 3xTF32 MMAs (a_negate)
//   * backward solve, W update and cache update as in the SIMT kernel.
// One CTA = 4 warps = 128 threads; thread i owns TMEM lane i = matrix row i.
#pragma once
#include "ials_common.cuh"
#include "ials_sweep.cuh"
#include "ials_umma.cuh"

namespace ials {

struct TcLay {
  static constexpr int BT = 128, NT = 128, KC = 32, XLD = BT + 4;
  // byte offsets (1024-aligned where an operand lives)
  static constexpr int OFF_XT_HI = 0;                         // 128 rows x 128 B (K-major SW128)
  static constexpr int OFF_XT_LO = OFF_XT_HI + 16384;
  static constexpr int OFF_PA_HI = OFF_XT_LO + 16384;         // 128 x 8 tf32 K-major, 4 KB
  static constexpr int OFF_PA_LO = OFF_PA_HI + 4096;
  static constexpr int OFF_X = OFF_PA_LO + 4096;              // natural staging [2][KC][XLD]
  static constexpr int OFF_AW = OFF_X + 2 * KC * XLD * 4;
  static constexpr int OFF_RH = OFF_AW + 2 * KC * 4;
  static constexpr int OFF_PS = OFF_RH + 2 * KC * 4;
  static constexpr int OFF_L = OFF_PS + 2 * KC * 4;           // packed lower L
  static constexpr int LP = BT * (BT + 1) / 2;
  static constexpr int OFF_DG = OFF_L + ((LP * 4 + 15) / 16) * 16;  // 8x8 diagonal block
  static constexpr int OFF_PY = OFF_DG + 64 * 4;
  static constexpr int OFF_RV = OFF_PY + 8 * 4;     // 1/diag of the panel
  static constexpr int OFF_YP = OFF_RV + 8 * 4;     // forward-solved y of the panel
  static constexpr int OFF_Y = OFF_YP + 8 * 4;
  static constexpr int OFF_YF = OFF_Y + BT * 4;
  static constexpr int OFF_ID = OFF_YF + BT * 4;
  static constexpr int OFF_D = OFF_ID + BT * 4;
  static constexpr int OFF_BAR = OFF_D + BT * 4;              // mbarrier (8 B) + tmem base
  static constexpr int BYTES = OFF_BAR + 16 + 1024;           // + slack to 1024-align the base
};

// 128B-swizzled operands need 1024-byte aligned atoms: align the dynamic
// shared-memory base explicitly (the launch requests 1 KB of slack).
IALS_DEVI char* tc_smem_base(char* raw) {
  const uint32_t a = smem_u32(raw);
  return raw + ((1024u - (a & 1023u)) & 1023u);
}

// K-major, 128B-swizzle float index of operand element (row m, k) for a
// 32-entry chunk: 8-row groups of 1 KB, chunk (k/4) of row m at (k/4) ^ (m%8).
IALS_DEVI int xt_index(int m, int k) {
  const int r = m & 7;
  return (m >> 3) * 256 + r * 32 + ((((k >> 2) ^ r)) << 2) + (k & 3);
}
// panel operand (128 x 8, K-major, no swizzle): 8-row groups of 256 B, two
// 4-element K chunks 128 B apart.
IALS_DEVI int pa_index(int m, int q) { return (m >> 3) * 64 + (q >> 2) * 32 + (m & 7) * 4 + (q & 3); }

template <int NT, int KC, int XLD>
IALS_DEVI void stage_entries(const SweepParams& p, float* X, float* aw, float* rh, int* ps, int ebeg,
                             int nk, int tid) {
  if (p.vec) {
    const int bv = p.b >> 2;
    for (int i = tid; i < nk * bv; i += NT) {
      const int k = i / bv, v = i - k * bv;
      const int col = __ldg(p.side.cols + ebeg + k);
      cp_async16(X + k * XLD + 4 * v, p.fixed + (size_t)col * p.ldf + p.fb0 + 4 * v);
    }
  } else {
    for (int i = tid; i < nk * p.b; i += NT) {
      const int k = i / p.b, v = i - k * p.b;
      const int col = __ldg(p.side.cols + ebeg + k);
      cp_async4(X + k * XLD + v, p.fixed + (size_t)col * p.ldf + p.fb0 + v);
    }
  }
  cp_async_commit();
  for (int k = tid; k < KC; k += NT) {
    float a = 0.f, r = 0.f;
    int pos = 0;
    if (k < nk) {
      const int e = ebeg + k;
      a = p.side.weights ? __ldg(p.side.weights + e) : 1.f;
      const float y = p.side.labels ? __ldg(p.side.labels + e) : 1.f;
      pos = p.side.pos ? __ldg(p.side.pos + e) : e;
      r = a * (p.cache[pos] - y);
    }
    aw[k] = a;
    rh[k] = r;
    ps[k] = pos;
  }
}

struct TcState {
  uint32_t tmem;   // TMEM base (lane 0, first column)
  uint32_t phase;  // mbarrier phase parity of the next completion
};

IALS_DEVI void tc_cta_sync() { __syncthreads(); }

// Adds the chunk sum held in TMEM (this thread's row) into the fp32 row sum.
IALS_DEVI void tc_flush(const TcState& st, float (&sum)[128], int tid) {
  const uint32_t row_addr = st.tmem + ((uint32_t)((tid >> 5) * 32) << 16);
#pragma unroll
  for (int c0 = 0; c0 < 128; c0 += 32) {
    float v[32];
    tmem_ld32(row_addr + c0, v);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) sum[c0 + j] += v[j];
  }
}

// Hessian + gradient over entries [ebeg, eend).  Each 32-entry chunk is
// summed from zero in TMEM by the tensor core (3xTF32) and then added into the
// fp32 register row sum `sum` (thread i holds row i): a two-level sum, so the
// tensor core's accumulation rounding only ever applies to one chunk's sum.
// Returns the number of chunks.
template <class L = TcLay>
IALS_DEVI int tc_accumulate(const SweepParams& p, char* smem, TcState& st, double& gacc,
                            float (&sum)[128], int ebeg, int eend, int tid) {
  float* XN = reinterpret_cast<float*>(smem + L::OFF_X);
  float* AW = reinterpret_cast<float*>(smem + L::OFF_AW);
  float* RH = reinterpret_cast<float*>(smem + L::OFF_RH);
  int* PS = reinterpret_cast<int*>(smem + L::OFF_PS);
  float* XTH = reinterpret_cast<float*>(smem + L::OFF_XT_HI);
  float* XTL = reinterpret_cast<float*>(smem + L::OFF_XT_LO);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  const int n = eend - ebeg;
  const int nch = (n + L::KC - 1) / L::KC;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t idesc = make_idesc_tf32(128, 128, 0, 0, 0);
  bool mma_pending = false;
  if (nch > 0) stage_entries<L::NT, L::KC, L::XLD>(p, XN, AW, RH, PS, ebeg, min(L::KC, n), tid);
  if (nch > 1) {
    const int s = ebeg + L::KC;
    stage_entries<L::NT, L::KC, L::XLD>(p, XN + L::KC * L::XLD, AW + L::KC, RH + L::KC,
                                        PS + L::KC, s, min(L::KC, eend - s), tid);
  }
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    const int nk = min(L::KC, eend - (ebeg + c * L::KC));
    if (c + 1 < nch) cp_async_wait<1>(); else cp_async_wait<0>();
    tc_cta_sync();
    const float* X = XN + buf * L::KC * L::XLD;
    const float* aw = AW + buf * L::KC;
    const float* rh = RH + buf * L::KC;
    // fp64 gradient (thread j <-> column j)
    {  // four independent fp64 chains (DFMA latency), combined in a fixed order
      double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
      int k = 0;
      for (; k + 3 < nk; k += 4) {
        g0 = fma((double)rh[k], (double)X[k * L::XLD + tid], g0);
        g1 = fma((double)rh[k + 1], (double)X[(k + 1) * L::XLD + tid], g1);
        g2 = fma((double)rh[k + 2], (double)X[(k + 2) * L::XLD + tid], g2);
        g3 = fma((double)rh[k + 3], (double)X[(k + 3) * L::XLD + tid], g3);
      }
      for (; k < nk; ++k) g0 = fma((double)rh[k], (double)X[k * L::XLD + tid], g0);
      gacc += (g0 + g1) + (g2 + g3);
    }
    // operands of the previous chunk must be consumed before overwriting;
    // its sum is then folded into the row sum
    if (mma_pending) {
      mbar_wait(bar, st.phase);
      st.phase ^= 1;
      mma_pending = false;
      tc_fence_after();
      tc_flush(st, sum, tid);
    }
    // transpose + tf32 split: lane <-> entry k, warp w <-> rows [32w, 32w+32)
    {
      const int k = lane;
      const bool ok = k < nk;
      const float sa = ok ? sqrtf(aw[k]) : 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int m0 = warp * 32 + q * 4;
        float4 v = ok ? *reinterpret_cast<const float4*>(X + k * L::XLD + m0)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
        const float e[4] = {v.x * sa, v.y * sa, v.z * sa, v.w * sa};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int idx = xt_index(m0 + i, k);
          XTH[idx] = e[i];
          XTL[idx] = tf32_lo(e[i]);
        }
      }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    tc_cta_sync();
    // the natural buffer is free again: prefetch chunk c + 2
    if (c + 2 < nch) {
      const int s = ebeg + (c + 2) * L::KC;
      stage_entries<L::NT, L::KC, L::XLD>(p, XN + buf * L::KC * L::XLD, AW + buf * L::KC,
                                          RH + buf * L::KC, PS + buf * L::KC, s,
                                          min(L::KC, eend - s), tid);
    }
    if (tid == 0) {
      tc_fence_after();
      const uint32_t hi = smem_u32(XTH), lo = smem_u32(XTL);
      const int ksteps = (nk + 7) >> 3;
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t ah = make_sdesc(hi + ks * 32, 16, 1024, kSwizzle128B);
        const uint64_t al = make_sdesc(lo + ks * 32, 16, 1024, kSwizzle128B);
        umma_tf32(st.tmem, ah, ah, idesc, ks > 0);
        umma_tf32(st.tmem, ah, al, idesc, 1);
        umma_tf32(st.tmem, al, ah, idesc, 1);
      }
      umma_commit(bar);
    }
    mma_pending = true;
  }
  if (mma_pending) {
    mbar_wait(bar, st.phase);
    st.phase ^= 1;
    tc_fence_after();
    tc_flush(st, sum, tid);
  }
  return nch;
}

// Row sum init: alpha0 * slab[pi, pi] + lam I on the b x b block, identity on
// the padding (thread i <-> row i).
IALS_DEVI void tc_init_rowsum(const SweepParams& p, float lam, float (&sum)[128], int tid) {
  const int b = p.b;
  const int i = tid;
  const float a0 = p.alpha0;
  const float* srow = p.slab + (size_t)(p.b0 + i) * b;
  if (i < b && (b & 3) == 0) {
    // all 32 row loads in flight at once (the slab stays L2-resident)
    float4 v[32];
#pragma unroll
    for (int c4 = 0; c4 < 32; ++c4)
      v[c4] = (4 * c4 < b) ? __ldg(reinterpret_cast<const float4*>(srow) + c4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int c4 = 0; c4 < 32; ++c4) {
      sum[4 * c4 + 0] = a0 * v[c4].x;
      sum[4 * c4 + 1] = a0 * v[c4].y;
      sum[4 * c4 + 2] = a0 * v[c4].z;
      sum[4 * c4 + 3] = a0 * v[c4].w;
    }
#pragma unroll
    for (int c = 0; c < 128; ++c)
      if (c == i) sum[c] += lam;
  } else {
#pragma unroll
    for (int c = 0; c < 128; ++c) {
      float x;
      if (i < b && c < b) {
        x = a0 * __ldg(srow + c);
        if (c == i) x += lam;
      } else {
        x = (c == i) ? 1.f : 0.f;
      }
      sum[c] = x;
    }
  }
}

// Write the row sum into TMEM (the matrix the factorisation works on).
IALS_DEVI void tc_store_rowsum(const TcState& st, const float (&sum)[128], int tid) {
  const uint32_t row_addr = st.tmem + ((uint32_t)((tid >> 5) * 32) << 16);
#pragma unroll
  for (int c0 = 0; c0 < 128; c0 += 8) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = sum[c0 + j];
    tmem_st8(row_addr + c0, v);
  }
  tmem_wait_st();
}

// Cholesky of the TMEM matrix + forward solve; leaves L (packed) in smem,
// y in OFF_YF, 1/diag in OFF_ID.  ys (OFF_Y) holds the gradient on entry.
template <class L = TcLay>
IALS_DEVI void tc_factor(const SweepParams& p, char* smem, TcState& st, int row, int tid) {
  float* Lp = reinterpret_cast<float*>(smem + L::OFF_L);
  float* DG = reinterpret_cast<float*>(smem + L::OFF_DG);
  float* PY = reinterpret_cast<float*>(smem + L::OFF_PY);
  float* ys = reinterpret_cast<float*>(smem + L::OFF_Y);
  float* yf = reinterpret_cast<float*>(smem + L::OFF_YF);
  float* invd = reinterpret_cast<float*>(smem + L::OFF_ID);
  float* PAH = reinterpret_cast<float*>(smem + L::OFF_PA_HI);
  float* PAL = reinterpret_cast<float*>(smem + L::OFF_PA_LO);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  const int b = p.b;
  const int i = tid;
  const uint32_t row_addr = st.tmem + ((uint32_t)((tid >> 5) * 32) << 16);
  const uint32_t idesc_neg = make_idesc_tf32(128, 128, 0, 0, 1);
  const int np = (b + 7) >> 3;
  float yi = ys[i];
  for (int pp = 0; pp < np; ++pp) {
    const int c0 = pp * 8;
    float v[8];
    tmem_ld8(row_addr + c0, v);
    tmem_wait_ld();
    if (i >= c0 && i < c0 + 8) {
#pragma unroll
      for (int m = 0; m < 8; ++m) DG[(i - c0) * 8 + m] = v[m];
      PY[i - c0] = yi;
    }
    tc_cta_sync();
    // the warp holding the diagonal rows factors the 8x8 block once
    float* RV = reinterpret_cast<float*>(smem + L::OFF_RV);
    float* YP = reinterpret_cast<float*>(smem + L::OFF_YP);
    if ((tid >> 5) == (c0 >> 5)) {
      float a[8][8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int m = 0; m <= q; ++m) a[q][m] = DG[q * 8 + m];
      float rinv[8];
      int bad = -1;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float dk = a[k][k];
        if (!(dk > 0.f) || !(dk < 3.0e38f)) {
          if (bad < 0) bad = k;
          dk = 1.f;
        }
        const float r = rsqrtf(dk);
        rinv[k] = r;
        a[k][k] = dk * r;
#pragma unroll
        for (int q = k + 1; q < 8; ++q) a[q][k] *= r;
#pragma unroll
        for (int q = k + 1; q < 8; ++q)
#pragma unroll
          for (int m = k + 1; m <= q; ++m) a[q][m] = fmaf(-a[q][k], a[m][k], a[q][m]);
      }
      if (bad >= 0 && c0 + bad < b && (tid & 31) == 0)
        report_singular(p.err, p.side_id, row, c0 + bad);
      float yp[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float t = PY[q];
#pragma unroll
        for (int m = 0; m < q; ++m) t = fmaf(-a[q][m], yp[m], t);
        yp[q] = t * rinv[q];
      }
      __syncwarp();
      if ((tid & 31) == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#pragma unroll
          for (int m = 0; m < 8; ++m) DG[q * 8 + m] = (m <= q) ? a[q][m] : 0.f;
          RV[q] = rinv[q];
          YP[q] = yp[q];
        }
      }
    }
    tc_cta_sync();
    float a[8][8], rinv[8], yp[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
#pragma unroll
      for (int m = 0; m <= q; ++m) a[q][m] = DG[q * 8 + m];
      rinv[q] = RV[q];
      yp[q] = YP[q];
    }
    // this row's panel entries
    float l[8];
    if (i >= c0 + 8 && i < b) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float t = v[q];
#pragma unroll
        for (int m = 0; m < q; ++m) t = fmaf(-l[m], a[q][m], t);
        l[q] = t * rinv[q];
      }
      float* lrow = Lp + i * (i + 1) / 2 + c0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        lrow[q] = l[q];
        yi = fmaf(-l[q], yp[q], yi);
      }
    } else if (i >= c0 && i < c0 + 8) {
      const int qq = i - c0;
      float* lrow = Lp + i * (i + 1) / 2 + c0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float t = 0.f, r = 0.f, y = 0.f;
#pragma unroll
        for (int z = 0; z < 8; ++z)
          if (z == qq) { t = (q <= z) ? a[z][q] : 0.f; r = rinv[z]; y = yp[z]; }
        l[q] = t;
        if (q <= qq) lrow[q] = t;
        if (q == 0) { invd[i] = r; yf[i] = y; }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) l[q] = 0.f;
    }
    if (pp + 1 < np) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        PAH[pa_index(i, q)] = l[q];
        PAL[pa_index(i, q)] = tf32_lo(l[q]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      tc_cta_sync();
      if (tid == 0) {
        tc_fence_after();
        const uint64_t ah = make_sdesc(smem_u32(PAH), 128, 256, kSwizzleNone);
        const uint64_t al = make_sdesc(smem_u32(PAL), 128, 256, kSwizzleNone);
        umma_tf32(st.tmem, ah, ah, idesc_neg, 1);
        umma_tf32(st.tmem, ah, al, idesc_neg, 1);
        umma_tf32(st.tmem, al, ah, idesc_neg, 1);
        umma_commit(bar);
      }
      mbar_wait(bar, st.phase);
      st.phase ^= 1;
      tc_fence_after();
    }
  }
  tc_cta_sync();
}

// Backward solve L^T d = y (warp 0), identical to the SIMT kernel's.
// Backward solve L^T d = y, panel by panel from the last: every thread
// back-substitutes the panel's 8 unknowns redundantly (from the packed L),
// then thread r < c0 folds them into its own y_r; one barrier per panel.
template <class L = TcLay>
IALS_DEVI void tc_backward(const SweepParams& p, char* smem, int tid) {
  const float* Lp = reinterpret_cast<const float*>(smem + L::OFF_L);
  float* yf = reinterpret_cast<float*>(smem + L::OFF_YF);
  const float* invd = reinterpret_cast<const float*>(smem + L::OFF_ID);
  float* ds = reinterpret_cast<float*>(smem + L::OFF_D);
  const int b = p.b;
  const int np = (b + 7) >> 3;
  float yr = (tid < b) ? yf[tid] : 0.f;   // this thread's running y_r
  for (int pp = np - 1; pp >= 0; --pp) {
    const int c0 = pp * 8;
    float dlt[8];
#pragma unroll
    for (int q = 7; q >= 0; --q) {
      const int gq = c0 + q;
      float v = (gq < b) ? yf[gq] : 0.f;
#pragma unroll
      for (int m = q + 1; m < 8; ++m) {
        const int gm = c0 + m;
        if (gm < b) v = fmaf(-Lp[gm * (gm + 1) / 2 + gq], dlt[m], v);
      }
      dlt[q] = (gq < b) ? v * invd[gq] : 0.f;
    }
    if (tid >= c0 && tid < c0 + 8 && tid < b) {  // ds[tid] = dlt[tid - c0], in registers
      const int e = tid - c0;
      const float a0 = (e & 1) ? dlt[1] : dlt[0], a1 = (e & 1) ? dlt[3] : dlt[2];
      const float a2 = (e & 1) ? dlt[5] : dlt[4], a3 = (e & 1) ? dlt[7] : dlt[6];
      const float b0 = (e & 2) ? a1 : a0, b1 = (e & 2) ? a3 : a2;
      ds[tid] = (e & 4) ? b1 : b0;
    }
    if (tid < c0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int gq = c0 + q;
        if (gq < b) yr = fmaf(-Lp[gq * (gq + 1) / 2 + tid], dlt[q], yr);
      }
    }
    __syncthreads();
    if (tid < c0 && tid >= c0 - 8) yf[tid] = yr;   // the next panel's entries
    __syncthreads();
  }
}

template <class L = TcLay>
IALS_DEVI void tc_cache_update(const SweepParams& p, char* smem, int ebeg, int eend, int nch,
                               int tid) {
  float* XN = reinterpret_cast<float*>(smem + L::OFF_X);
  float* AW = reinterpret_cast<float*>(smem + L::OFF_AW);
  float* RH = reinterpret_cast<float*>(smem + L::OFF_RH);
  int* PS = reinterpret_cast<int*>(smem + L::OFF_PS);
  const float* ds = reinterpret_cast<const float*>(smem + L::OFF_D);
  const int lane = tid & 31, warp = tid >> 5;
  const int n = eend - ebeg;
  // one thread per entry: all entries' dot products and cache updates in flight
  auto chunk = [&](int buf, int nk) {
    const float* X = XN + buf * L::KC * L::XLD;
    const int* ps = PS + buf * L::KC;
    (void)lane; (void)warp;
    if (tid < nk) {
      const float* xr = X + tid * L::XLD;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      int j = 0;
      if (p.vec) {
        for (; j + 3 < p.b; j += 4) {
          const float4 x = *reinterpret_cast<const float4*>(xr + j);
          const float4 dv = *reinterpret_cast<const float4*>(ds + j);
          s0 = fmaf(x.x, dv.x, s0);
          s1 = fmaf(x.y, dv.y, s1);
          s2 = fmaf(x.z, dv.z, s2);
          s3 = fmaf(x.w, dv.w, s3);
        }
      }
      for (; j < p.b; ++j) s0 = fmaf(xr[j], ds[j], s0);
      p.cache[ps[tid]] -= (s0 + s1) + (s2 + s3);
    }
  };
  if (nch <= 2) {
    for (int c = 0; c < nch; ++c) chunk(c, min(L::KC, n - c * L::KC));
    return;
  }
  for (int c = 0; c < nch; ++c) {
    const int s = ebeg + c * L::KC;
    const int nk = min(L::KC, eend - s);
    tc_cta_sync();
    stage_entries<L::NT, L::KC, L::XLD>(p, XN, AW, RH, PS, s, nk, tid);
    cp_async_wait<0>();
    tc_cta_sync();
    chunk(0, nk);
  }
}

__global__ void __launch_bounds__(128) k_sweep_tc128(SweepParams p) {
  using L = TcLay;
  extern __shared__ __align__(1024) char smem_tc[];
  char* smem = tc_smem_base(smem_tc);
  const int tid = threadIdx.x;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L::OFF_BAR + 8);
  {  // zero staging (stale rows must be finite)
    float4* x = reinterpret_cast<float4*>(smem + L::OFF_X);
    for (int i = tid; i < 2 * L::KC * L::XLD / 4; i += L::NT) x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (tid == 0) mbar_init(bar, 1);
  if (tid < 32) tmem_alloc(tptr, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  TcState st{*tptr, 0u};
  float* ys = reinterpret_cast<float*>(smem + L::OFF_Y);
  const float* ds = reinterpret_cast<const float*>(smem + L::OFF_D);
  for (int task = blockIdx.x; task < p.n_light; task += gridDim.x) {
    const int row = p.light_rows[task];
    const int ebeg = p.side.ptr[row], eend = p.side.ptr[row + 1];
    const float lam = p.side.lam[row];
    float sum[128];
    tc_init_rowsum(p, lam, sum, tid);
    double gacc = 0.0;
    const int nch = tc_accumulate(p, smem, st, gacc, sum, ebeg, eend, tid);
    tc_store_rowsum(st, sum, tid);
    tc_fence_before();
    {
      double g = 0.0;
      if (tid < p.b)
        g = gacc + (double)p.proj[(size_t)row * p.b + tid] +
            (double)lam * (double)p.own[(size_t)row * p.ldo + p.b0 + tid];
      ys[tid] = (float)g;
    }
    __syncthreads();
    tc_factor(p, smem, st, row, tid);
    tc_backward(p, smem, tid);
    if (tid < p.b) p.own[(size_t)row * p.ldo + p.b0 + tid] -= ds[tid];
    tc_cache_update(p, smem, ebeg, eend, nch, tid);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free(st.tmem, 128);
}

// Heavy-row slices on the tensor core: partial Hessian (full 128x128, row
// major, the layout k_heavy_solve<128> reads) + fp64 partial gradient.
__global__ void __launch_bounds__(128) k_heavy_partial_tc128(SweepParams p) {
  using L = TcLay;
  extern __shared__ __align__(1024) char smem_tc[];
  char* smem = tc_smem_base(smem_tc);
  const int tid = threadIdx.x;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L::OFF_BAR + 8);
  {
    float4* x = reinterpret_cast<float4*>(smem + L::OFF_X);
    for (int i = tid; i < 2 * L::KC * L::XLD / 4; i += L::NT) x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (tid == 0) mbar_init(bar, 1);
  if (tid < 32) tmem_alloc(tptr, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  TcState st{*tptr, 0u};
  for (int sl = blockIdx.x; sl < p.n_slices; sl += gridDim.x) {
    float sum[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) sum[c] = 0.f;
    double gacc = 0.0;
    tc_accumulate(p, smem, st, gacc, sum, p.slice_begin[sl], p.slice_end[sl], tid);
    float* hp = p.hpart + (size_t)sl * 128 * 128 + (size_t)tid * 128;
#pragma unroll
    for (int c0 = 0; c0 < 128; c0 += 4)
      *reinterpret_cast<float4*>(hp + c0) = make_float4(sum[c0], sum[c0 + 1], sum[c0 + 2], sum[c0 + 3]);
    p.gpart[(size_t)sl * 128 + tid] = gacc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free(st.tmem, 128);
}

}  // namespace ials
