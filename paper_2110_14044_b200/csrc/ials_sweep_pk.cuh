// ials_sweep_pk.cuh -- fused tensor-core light-row sweep for narrow blocks
// (b <= 64): G rows ("slots") share one 128-lane TMEM tile, so a CTA has G
// rows in flight and the per-row dependency chain (accumulate -> blocked
// Cholesky -> solves) is shared by G rows instead of being paid per row on a
// zero-padded 128 x 128 matrix.
//
//   G = 2: slots of NG = 64 lanes / columns (33 <= b <= 64)
//   G = 4: slots of NG = 32 lanes / columns (17 <= b <= 32)
//
// Thread t = g * NG + m <-> TMEM lane t <-> row m of slot g's matrix.  A tile
// is G consecutive rows of the descending-degree light list (similar lengths).
//   1. TMEM row t := [template row m of alpha0 * slab[pi, pi] (identity on the
//      padding m >= b) at columns g*NG.., zeros elsewhere]
//   2. per 8-entry chunk of every slot (TMA gather4 of NG-float boxes into a
//      natural [slot][entry][NG] staging, 3 chunks ahead; metadata 6 ahead):
//      thread (g, m) reads column m of its slot's entries -> fp64 gradient and
//      row t of the K-major operand (no swizzle, hi / lo split); one thread
//      issues D += A A^T (M = N = 128, K = 8, 3xTF32).  Row t of A holds slot
//      g's sub-rows, so the diagonal NG x NG blocks of D are the G Hessians
//      (the cross-slot blocks are never read).
//   3. lam on each slot's diagonal; the blocked Cholesky of all G matrices in
//      lockstep: per 8-column panel every slot's diagonal block is factored by
//      the warp holding it (G warps in parallel), the rows below solve, and one
//      3xTF32 rank-8 MMA updates all slots' trailing columns at once;
//   4. backward solve by 16-wide blocks (block inverses), per slot.
// The cancellation guard, the SIMT redo list, heavy rows (k_heavy_partial_tc4)
// and the entry-parallel cache pass are those of the b = 128 path.
#pragma once
#include "ials_sweep_tc4.cuh"

namespace ials {

template <int G>
struct PkLay {
  static constexpr int NT = 128, NG = 128 / G, KC = 8, EPC = G * KC, SW = NG;
  // pipeline depths (in chunks): sub-rows and yhat gathered GD ahead into NB
  // staging buffers, metadata MD ahead through an MR-deep ring, operands in
  // NXT buffers (one MMA barrier each)
  static constexpr int NB = 4, GD = 3, MR = 8, MD = 6, NXT = 3, NCV = 4;
  static constexpr int LPS = ((NG * (NG + 1) / 2) + 3) & ~3;   // packed L floats per slot
  // overlay, by phase -- accumulate: operands hi/lo x NXT (8 KB each) and the
  // natural staging [NB][G][KC][SW] (4 KB each); factor: packed L per slot,
  // the panel operands (8 KB), the diagonal-block staging, then the block
  // inverses (8 KB)
  static constexpr int OFF_XT = 0;
  static constexpr int OFF_X = NXT * 8192;
  static constexpr int OFF_L = 0;
  static constexpr int L_BYTES = G * LPS * 4;
  static constexpr int OFF_PA = ((L_BYTES + 1023) / 1024) * 1024;
  static constexpr int OFF_LI = OFF_PA + 8192;
  static constexpr int ACC_END = OFF_X + NB * KC * 128 * 4;
  static constexpr int OVL = (OFF_LI + 8192 > ACC_END) ? OFF_LI + 8192 : ACC_END;
  static constexpr int OFF_MC = OVL;                           // rings [MR][EPC]
  static constexpr int OFF_MP = OFF_MC + MR * EPC * 4;
  static constexpr int OFF_MW = OFF_MP + MR * EPC * 4;
  static constexpr int OFF_MY = OFF_MW + MR * EPC * 4;
  static constexpr int OFF_CV = OFF_MY + MR * EPC * 4;         // [NCV][EPC] gathered yhat
  static constexpr int OFF_DG = OFF_CV + NCV * EPC * 4;        // per slot, per panel parity: 320 B
  static constexpr int OFF_Y = OFF_DG + G * 640;
  static constexpr int OFF_YF = OFF_Y + 512;
  static constexpr int OFF_ID = OFF_YF + 512;
  static constexpr int OFF_D = OFF_ID + 512;
  static constexpr int OFF_DIAG = OFF_D + 512;
  static constexpr int OFF_TILE = OFF_DIAG + 512;              // [2][rows[4], beg[4], end[4], lam[4]]
  static constexpr int OFF_FLAG = OFF_TILE + 128;              // flags[G], next task
  // G = 4: the 32 x 32 packed template alpha0 * slab[pi, pi] in shared memory
  // (loaded once per launch; G = 2's 8.7 KB one is read through L1)
  static constexpr int TPL_FLOATS = G == 4 ? 576 : 0;
  static constexpr int OFF_BAR = OFF_FLAG + 32;                // MMA bars [NXT], gather bars [NB], TMEM base
  static constexpr int BAR_GATHER = NXT;
  static constexpr int OFF_TPTR = OFF_BAR + 8 * (NXT + NB);
  static constexpr int OFF_TPL = OFF_TPTR + 16;
  static constexpr int BYTES = OFF_TPL + TPL_FLOATS * 4 + 1024;
};

struct PkState {
  uint32_t tmem;
  uint32_t ph;    // bit x: phase parity of MMA barrier x
  uint32_t gph;   // bit x: phase parity of gather barrier x
  const CUtensorMap* fmap;
};

template <int G>
IALS_DEVI int pk_nk(const int* beg, const int* end, int g, int c) {
  return max(0, min(PkLay<G>::KC, end[g] - beg[g] - c * PkLay<G>::KC));
}

// metadata of chunk c for every slot: thread t -> array t / EPC, entry t % EPC
template <int G, bool UNIT>
IALS_DEVI void pk_meta(const SweepParams& p, char* smem, const int* beg, const int* end, int c, int tid) {
  using L = PkLay<G>;
  const int arr = tid / L::EPC, ei = tid - arr * L::EPC, g = ei / L::KC, j = ei - g * L::KC;
  if (arr >= (UNIT ? 2 : 4)) return;
  const int e = beg[g] + c * L::KC + j;
  if (e >= end[g]) return;
  const int slot = (c & (L::MR - 1)) * L::EPC + ei;
  switch (arr) {
    case 0: cp_async4(smem + L::OFF_MC + 4 * slot, p.side.cols + e); break;
    case 1: if (p.side.pos) cp_async4(smem + L::OFF_MP + 4 * slot, p.side.pos + e);
            else reinterpret_cast<int*>(smem + L::OFF_MP)[slot] = e;
            break;
    case 2: if (p.side.weights) cp_async4(smem + L::OFF_MW + 4 * slot, p.side.weights + e);
            else reinterpret_cast<float*>(smem + L::OFF_MW)[slot] = 1.f;
            break;
    default: if (p.side.labels) cp_async4(smem + L::OFF_MY + 4 * slot, p.side.labels + e);
             else reinterpret_cast<float*>(smem + L::OFF_MY)[slot] = 1.f;
             break;
  }
}

// sub-rows F[col, fb0 : fb0 + NG] of chunk c of every slot -> staging buffer
// c % NB, and the chunk's yhat[pos] -> CV ring
template <int G>
IALS_DEVI void pk_gather(const SweepParams& p, char* smem, const PkState& st, const int* beg,
                         const int* end, int c, int tid) {
  using L = PkLay<G>;
  const int* mc = reinterpret_cast<const int*>(smem + L::OFF_MC) + (c & (L::MR - 1)) * L::EPC;
  const int* mp = reinterpret_cast<const int*>(smem + L::OFF_MP) + (c & (L::MR - 1)) * L::EPC;
  float* X = reinterpret_cast<float*>(smem + L::OFF_X) + (c % L::NB) * G * L::KC * L::SW;
  if (st.fmap) {
    // each slot's gathers are issued by lane 0 of the first warp of the slot
    // (G issuers in parallel); the barrier expects G arrivals, each with its
    // slot's bytes (possibly 0), so it cannot complete before every slot's
    // gathers are registered
    if ((tid & 31) == 0 && (tid % L::NG) == 0) {
      const int g = tid / L::NG;
      const int nk = pk_nk<G>(beg, end, g, c), last = nk - 1;
      uint64_t* gb = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR) + L::BAR_GATHER + (c % L::NB);
      mbar_expect_tx(gb, (uint32_t)((nk + 3) >> 2) * 4 * L::SW * 4);
      const int* m = mc + g * L::KC;
      for (int q = 0; q < nk; ++q) IALS_CHECK(m[q] >= 0 && m[q] < p.side.n_fixed);
      for (int k = 0; k < nk; k += 4)
        tma_gather4(smem_u32(X + (g * L::KC + k) * L::SW), st.fmap, p.fb0, m[min(k, last)],
                    m[min(k + 1, last)], m[min(k + 2, last)], m[min(k + 3, last)], gb);
    }
  } else if (p.vec) {   // 16-byte pieces: thread <-> (entry, piece)
    constexpr int PV = L::SW / 4;
    for (int i = tid; i < L::EPC * PV; i += L::NT) {
      const int ei = i / PV, v = i - ei * PV, g = ei / L::KC, k = ei - g * L::KC;
      if (k < pk_nk<G>(beg, end, g, c) && 4 * v < p.b)
        cp_async16(X + ei * L::SW + 4 * v, p.fixed + (size_t)mc[ei] * p.ldf + p.fb0 + 4 * v);
    }
  } else {
    for (int i = tid; i < L::EPC * L::SW; i += L::NT) {
      const int ei = i / L::SW, v = i - ei * L::SW, g = ei / L::KC, k = ei - g * L::KC;
      if (k < pk_nk<G>(beg, end, g, c) && v < p.b)
        cp_async4(X + ei * L::SW + v, p.fixed + (size_t)mc[ei] * p.ldf + p.fb0 + v);
    }
  }
  if (tid < L::EPC) {
    const int g = tid / L::KC, k = tid - g * L::KC;
    if (k < pk_nk<G>(beg, end, g, c)) {
      IALS_CHECK(mp[tid] >= 0 && mp[tid] < p.side.nnz);
      cp_async4(smem + L::OFF_CV + 4 * ((c % L::NCV) * L::EPC + tid), p.cache + mp[tid]);
    }
  }
}

// step 2, per 8-entry chunk of every slot.  Every load is asynchronous: the
// metadata MD = 6 chunks ahead (ring of MR = 8), the sub-rows (TMA gather4)
// and yhat GD = 3 chunks ahead (NB = 4 staging buffers), so a chunk's loads
// have three iterations to land; cp.async group c (committed at the end of
// iteration c) = {X / yhat of chunk c + 3, metadata of chunk c + 6}, and
// iteration c waits for group c - 2 before its barrier (what iteration c + 1
// reads).  Operands go through NXT = 3 buffers, each freed by its MMA commit.
template <int G, bool UNIT>
IALS_DEVI void pk_accumulate(const SweepParams& p, char* smem, PkState& st, double& gacc,
                             const int* beg, const int* end, int nch, int tid) {
  using L = PkLay<G>;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  const uint32_t idesc = make_idesc_tf32(128, 128, 0, 0, 0);
  const int g = tid / L::NG, m = tid - g * L::NG;
  uint32_t pend = 0;   // bit x: MMA barrier x has an outstanding commit
  if (nch == 0) return;
  for (int c = 0; c < L::MD && c < nch; ++c) pk_meta<G, UNIT>(p, smem, beg, end, c, tid);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int c = 0; c < L::GD && c < nch; ++c) pk_gather<G>(p, smem, st, beg, end, c, tid);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int xb = c % L::NB, ob = c % L::NXT;
    const int nk = pk_nk<G>(beg, end, g, c);
    if (st.fmap) {
      mbar_wait(bar + L::BAR_GATHER + xb, (st.gph >> xb) & 1u);
      st.gph ^= 1u << xb;
    }
    const float* X = reinterpret_cast<const float*>(smem + L::OFF_X) + (xb * G + g) * L::KC * L::SW;
    const int ms = (c % L::MR) * L::EPC + g * L::KC;
    const float* mw = reinterpret_cast<const float*>(smem + L::OFF_MW) + ms;
    const float* my = reinterpret_cast<const float*>(smem + L::OFF_MY) + ms;
    const float* cv = reinterpret_cast<const float*>(smem + L::OFF_CV) + (c % L::NCV) * L::EPC + g * L::KC;
    float x[L::KC];
    const bool colok = m < p.b;
#pragma unroll
    for (int k = 0; k < L::KC; ++k) x[k] = (colok && k < nk) ? X[k * L::SW + m] : 0.f;
    float wk[L::KC];
    {
      float gs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k4 = 0; k4 < L::KC / 4; ++k4) {
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
          const float r = (k < nk) ? (UNIT ? cc[j] - 1.f : w[j] * (cc[j] - yy[j])) : 0.f;
          gs[j] = fmaf(r, x[k], gs[j]);
        }
      }
      gacc += ((double)gs[0] + (double)gs[1]) + ((double)gs[2] + (double)gs[3]);
    }
    if (!UNIT && p.side.weights) {
#pragma unroll
      for (int k = 0; k < L::KC; ++k) x[k] *= (k < nk) ? sqrtf(wk[k]) : 0.f;
    }
    if (pend & (1u << ob)) {   // operand buffer ob was last read by chunk c - NXT's MMAs
      mbar_wait(bar + ob, (st.ph >> ob) & 1u);
      st.ph ^= 1u << ob;
      pend &= ~(1u << ob);
    }
    {  // row tid of the K-major (no swizzle) operands: entries 0..3 | 4..7
      float* XTH = reinterpret_cast<float*>(smem + L::OFF_XT + ob * 8192);
      float* XTL = XTH + 1024;
      float hi[L::KC], lo[L::KC];
#pragma unroll
      for (int k = 0; k < L::KC; ++k) {
        hi[k] = tf32_rna(x[k]);
        lo[k] = x[k] - hi[k];   // fed as is: the MMA drops its low 13 bits
      }
      const int o = pa_index(tid, 0);
      *reinterpret_cast<float4*>(XTH + o) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<float4*>(XTH + o + 32) = make_float4(hi[4], hi[5], hi[6], hi[7]);
      *reinterpret_cast<float4*>(XTL + o) = make_float4(lo[0], lo[1], lo[2], lo[3]);
      *reinterpret_cast<float4*>(XTL + o + 32) = make_float4(lo[4], lo[5], lo[6], lo[7]);
    }
    cp_async_wait<1>();   // group c - 2: yhat / sub-rows of chunk c + 1, metadata of chunk c + 4
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t hi = smem_u32(smem + L::OFF_XT + ob * 8192), lo = hi + 4096;
      const uint64_t ah = make_sdesc(hi, 128, 256, kSwizzleNone);
      const uint64_t al = make_sdesc(lo, 128, 256, kSwizzleNone);
      umma_tf32(st.tmem, ah, ah, idesc, 1);
      umma_tf32(st.tmem, ah, al, idesc, 1);
      umma_tf32(st.tmem, al, ah, idesc, 1);
      umma_commit(bar + ob);
    }
    pend |= 1u << ob;
    // staging buffer (c + 3) % 4 was chunk c - 1's, read before this barrier
    if (c + L::GD < nch) pk_gather<G>(p, smem, st, beg, end, c + L::GD, tid);
    if (c + L::MD < nch) pk_meta<G, UNIT>(p, smem, beg, end, c + L::MD, tid);
    cp_async_commit();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int ob = 0; ob < L::NXT; ++ob)
    if (pend & (1u << ob)) {
      mbar_wait(bar + ob, (st.ph >> ob) & 1u);
      st.ph ^= 1u << ob;
    }
  tc_fence_after();
}

// step 3: blocked Cholesky + forward solve of the G slot matrices in lockstep
// (tc4_factor with per-slot diagonal warps, per-slot shared state and
// full-width trailing MMAs).  Returns with packed L (per slot), 1/pivots in
// OFF_ID and the forward-solved right-hand side in OFF_YF.
// UNIT_DIAG (the Woodbury tiles): the matrices in TMEM are C - I; the identity
// is added to a diagonal entry when its own row reads it for its panel (the
// trailing updates are additive, and nothing else reads the diagonal).
template <int G, class L = PkLay<G>, bool UNIT_DIAG = false>
IALS_DEVI void pk_factor(const SweepParams& p, char* smem, PkState& st, uint32_t row_addr, int tid,
                         const int b) {
  float* ys = reinterpret_cast<float*>(smem + L::OFF_Y);
  float* yf = reinterpret_cast<float*>(smem + L::OFF_YF);
  float* invd = reinterpret_cast<float*>(smem + L::OFF_ID);
  const float* DIAG = reinterpret_cast<const float*>(smem + L::OFF_DIAG);
  int* FLAG = reinterpret_cast<int*>(smem + L::OFF_FLAG);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  const int lane = tid & 31, warp = tid >> 5;
  const int g = tid / L::NG, i = tid - g * L::NG;   // slot, row within the slot
  float* lrow = reinterpret_cast<float*>(smem + L::OFF_L) + g * L::LPS + i * (i + 1) / 2;
  const int np = (b + 7) >> 3;
  float yi = ys[tid];
  for (int pp = 0; pp < np; ++pp) {
    const int c0 = pp * 8;
    float* DG = reinterpret_cast<float*>(smem + L::OFF_DG + g * 640 + (pp & 1) * 320);
    float* RV = DG + 64;
    float* YP = DG + 72;
    float v[8];
    tmem_ld8(row_addr + g * L::NG + c0, v);
    tmem_wait_ld();
    if (UNIT_DIAG && i >= c0 && i < c0 + 8) {   // (only the diagonal block's rows hold a diagonal entry)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (c0 + j == i) v[j] += 1.f;
    }
    if (warp == ((g * L::NG + c0) >> 5)) {   // this warp holds slot g's diagonal block
      const int base = (g * L::NG + c0) & 31;
      float* SG = reinterpret_cast<float*>(smem + L::OFF_LI) + g * 80;   // free until the backward solve
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
      __syncwarp();
      float rinv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float dk = a[k][k];
        float r;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(dk));
        rinv[k] = r;
        a[k][k] = dk * r;
#pragma unroll
        for (int q = k + 1; q < 8; ++q) a[q][k] *= r;
#pragma unroll
        for (int q = k + 1; q < 8; ++q)
#pragma unroll
          for (int mm = k + 1; mm <= q; ++mm) a[q][mm] = fmaf(-a[q][k], a[mm][k], a[q][mm]);
      }
      float yp[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float t = py[q];
#pragma unroll
        for (int mm = 0; mm < q; ++mm) t = fmaf(-a[q][mm], yp[mm], t);
        yp[q] = t * rinv[q];
      }
      if (lane == base) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float w[8];
#pragma unroll
          for (int mm = 0; mm < 8; ++mm) w[mm] = (mm <= q) ? a[q][mm] : 0.f;
          reinterpret_cast<float4*>(DG)[2 * q] = make_float4(w[0], w[1], w[2], w[3]);
          if (q >= 4) reinterpret_cast<float4*>(DG)[2 * q + 1] = make_float4(w[4], w[5], w[6], w[7]);
        }
        reinterpret_cast<float4*>(RV)[0] = make_float4(rinv[0], rinv[1], rinv[2], rinv[3]);
        reinterpret_cast<float4*>(RV)[1] = make_float4(rinv[4], rinv[5], rinv[6], rinv[7]);
        reinterpret_cast<float4*>(YP)[0] = make_float4(yp[0], yp[1], yp[2], yp[3]);
        reinterpret_cast<float4*>(YP)[1] = make_float4(yp[4], yp[5], yp[6], yp[7]);
      }
    }
    __syncthreads();
    auto record_block = [&]() {
      if (i >= c0 && i < c0 + 8) {
        const int j = i - c0;
        const float4 x0 = reinterpret_cast<const float4*>(DG)[2 * j];
        const float4 x1 = reinterpret_cast<const float4*>(DG)[2 * j + 1];
        const float w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
        for (int mm = 0; mm < 8; ++mm)
          if (mm <= j) lrow[c0 + mm] = w[mm];
        const float r = RV[j];
        invd[tid] = r;
        yf[tid] = YP[j];
        if (i < b && !(r > 0.f && DIAG[tid] * (r * r) <= p.cond_max)) FLAG[g] = 1;
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
        for (int mm = 0; mm < q; ++mm) tt = fmaf(-l[mm], w[mm], tt);
        l[q] = tt * rinv[q];
        yi = fmaf(-l[q], yp[q], yi);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) lrow[c0 + q] = l[q];
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) l[q] = 0.f;
    }
    if (pp + 1 < np) {
      float* PAH = reinterpret_cast<float*>(smem + L::OFF_PA);
      float* PAL = PAH + 1024;
      float hi[8], lo[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        hi[q] = tf32_rna(l[q]);
        lo[q] = l[q] - hi[q];
      }
      const int pa = pa_index(tid, 0);
      *reinterpret_cast<float4*>(PAH + pa) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<float4*>(PAH + pa + 32) = make_float4(hi[4], hi[5], hi[6], hi[7]);
      *reinterpret_cast<float4*>(PAL + pa) = make_float4(lo[0], lo[1], lo[2], lo[3]);
      *reinterpret_cast<float4*>(PAL + pa + 32) = make_float4(lo[4], lo[5], lo[6], lo[7]);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        // D -= L_p L_p^T over all 128 columns: the rows of each slot's
        // diagonal block and above carry zeros, so finished columns and the
        // other slots' columns of a row only see the (unread) cross blocks
        const uint32_t idesc_neg = make_idesc_tf32(128, 128, 0, 0, 1);
        const uint64_t ah = make_sdesc(smem_u32(PAH), 128, 256, kSwizzleNone);
        const uint64_t al = make_sdesc(smem_u32(PAL), 128, 256, kSwizzleNone);
        umma_tf32(st.tmem, ah, ah, idesc_neg, 1);
        umma_tf32(st.tmem, ah, al, idesc_neg, 1);
        umma_tf32(st.tmem, al, ah, idesc_neg, 1);
        umma_commit(bar);
      }
      record_block();
      mbar_wait(bar, st.ph & 1u);
      st.ph ^= 1u;
      tc_fence_after();
    } else {
      record_block();
    }
  }
  __syncthreads();
}

// 16 x 16 diagonal-block inverses of every slot's L: thread t -> block t / 16
// (slot (t / 16) / (NG / 16)), column q = t % 16
template <int G, class L = PkLay<G>>
IALS_DEVI void pk_block_inverses(char* smem, int tid, const int b) {
  constexpr int NBS = L::NG / 16;
  const float* invd = reinterpret_cast<const float*>(smem + L::OFF_ID);
  float* LI = reinterpret_cast<float*>(smem + L::OFF_LI);
  const int blk = tid >> 4, q = tid & 15, g = blk / NBS, c0 = 16 * (blk - g * NBS);
  const float* Lp = reinterpret_cast<const float*>(smem + L::OFF_L) + g * L::LPS;
  if (c0 >= b) return;
  float x[16];
#pragma unroll
  for (int mm = 0; mm < 16; ++mm) {
    const int gm = c0 + mm;
    float t = (mm == q) ? 1.f : 0.f;
    const float* lr = Lp + gm * (gm + 1) / 2 + c0;
#pragma unroll
    for (int k = 0; k < mm; ++k) t = fmaf(-lr[k], x[k], t);
    x[mm] = (mm >= q && gm < b) ? t * invd[g * L::NG + gm] : 0.f;
  }
#pragma unroll
  for (int mm = 0; mm < 16; ++mm) LI[blk * 256 + mm * 16 + q] = x[mm];
}

// backward solve L^T d = y of every slot, 16-wide blocks from the last
template <int G, class L = PkLay<G>>
IALS_DEVI void pk_backward(char* smem, int tid, const int b) {
  constexpr int NBS = L::NG / 16;
  const float* LI = reinterpret_cast<const float*>(smem + L::OFF_LI);
  float* yf = reinterpret_cast<float*>(smem + L::OFF_YF);
  float* ds = reinterpret_cast<float*>(smem + L::OFF_D);
  const int g = tid / L::NG, i = tid - g * L::NG;
  const float* Lp = reinterpret_cast<const float*>(smem + L::OFF_L) + g * L::LPS;
  float* yg = yf + g * L::NG;
  float* dg = ds + g * L::NG;
  const int nb = (b + 15) >> 4;
  float yr = (i < b) ? yg[i] : 0.f;
  for (int pb = nb - 1; pb >= 0; --pb) {
    const int c0 = pb * 16;
    if ((i >> 4) == pb) {   // d_q = sum_{m >= q} LI[m][q] y_m
      const int q = i & 15;
      const float* li = LI + (g * NBS + pb) * 256 + q;
      float t0 = 0.f, t1 = 0.f;
#pragma unroll
      for (int mm = 0; mm < 16; mm += 2) {
        if (mm >= q && c0 + mm < b) t0 = fmaf(li[mm * 16], yg[c0 + mm], t0);
        if (mm + 1 >= q && c0 + mm + 1 < b) t1 = fmaf(li[(mm + 1) * 16], yg[c0 + mm + 1], t1);
      }
      if (c0 + q < b) dg[c0 + q] = t0 + t1;
    }
    __syncthreads();
    if (i < c0) {
      const float4* dq = reinterpret_cast<const float4*>(dg + c0);
      float a0 = yr, a1 = 0.f;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const float4 dv = dq[q4];
        const int gg = c0 + 4 * q4;
        if (gg < b) a0 = fmaf(-Lp[gg * (gg + 1) / 2 + i], dv.x, a0);
        if (gg + 1 < b) a1 = fmaf(-Lp[(gg + 1) * (gg + 2) / 2 + i], dv.y, a1);
        if (gg + 2 < b) a0 = fmaf(-Lp[(gg + 2) * (gg + 3) / 2 + i], dv.z, a0);
        if (gg + 3 < b) a1 = fmaf(-Lp[(gg + 3) * (gg + 4) / 2 + i], dv.w, a1);
      }
      yr = a0 + a1;
      if (i >= c0 - 16) yg[i] = yr;
    }
    __syncthreads();
  }
}

template <int G, bool UNIT>
__global__ void __launch_bounds__(128, 4) k_sweep_pk(SweepParams p, const __grid_constant__ CUtensorMap fmap,
                                                        int use_tma) {
  using L = PkLay<G>;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = tc_smem_base(smem_raw);
  const int tid = threadIdx.x, g = tid / L::NG, m = tid - g * L::NG;
  {  // finite staging everywhere
    float4* x = reinterpret_cast<float4*>(smem + L::OFF_X);
    for (int i = tid; i < L::NB * G * L::KC * L::SW / 4; i += L::NT) x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L::OFF_TPTR);
  int* tinfo = reinterpret_cast<int*>(smem + L::OFF_TILE);   // [2][16]: rows, beg, end, lam
  int* FLAG = reinterpret_cast<int*>(smem + L::OFF_FLAG);
  float* ys = reinterpret_cast<float*>(smem + L::OFF_Y);
  float* ds = reinterpret_cast<float*>(smem + L::OFF_D);
  ds[tid] = 0.f;
  if (tid == 0) {
    for (int k = 0; k < L::NXT; ++k) mbar_init(bar + k, 1);
    for (int k = 0; k < L::NB; ++k) mbar_init(bar + L::BAR_GATHER + k, G);
    if (use_tma) prefetch_tmap(&fmap);
  }
  float* tpl_s = reinterpret_cast<float*>(smem + L::OFF_TPL);
  for (int k = tid; k < L::TPL_FLOATS; k += L::NT) tpl_s[k] = __ldg(p.tpl + k);
  if (tid < 32) tmem_alloc(tptr, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  PkState st;
  st.tmem = *tptr;
  st.ph = 0u;
  st.gph = 0u;
  st.fmap = use_tma ? &fmap : nullptr;
  const uint32_t row_addr = st.tmem + ((uint32_t)((tid >> 5) * 32) << 16);
  const int b = p.b;
  const int* lrows = p.light_rows;
  int n_light = p.n_light;
  if (p.chunk_tot) {   // ials_epoch_host's chunked first user pass
    int off = 0;
    for (int k = 0; k < p.chunk; ++k) off += p.chunk_tot[k];
    lrows += off;
    n_light = p.chunk_tot[p.chunk];
  }
  const int n_tiles = (n_light + G - 1) / G;
  int* queue = p.redo_cnt + 2;
  int* next = FLAG + 4;
  // tile t's rows (G consecutive rows of the longest-first list), their entry
  // ranges and lam into tile buffer tb (an empty slot solves I x = 0)
  auto tile_row = [&](int t, int s) { const int k = t * G + s; return k < n_light ? lrows[k] : -1; };
  auto put_tile = [&](int tb, int s, int r) {
    int* ti = tinfo + 16 * tb;
    ti[s] = r;
    ti[4 + s] = r >= 0 ? p.side.ptr[r] : 0;
    ti[8 + s] = r >= 0 ? p.side.ptr[r + 1] : 0;
    reinterpret_cast<float*>(ti)[12 + s] = r >= 0 ? p.side.lam[r] : 1.f;
  };
  if (tid == 0) *next = atomicAdd(queue, 1);
  __syncthreads();
  int task = *next;
  if (tid < G && task < n_tiles) put_tile(0, tid, tile_row(task, tid));
  if (tid < G) FLAG[tid] = 0;
  __syncthreads();
  int tb = 0;
  while (task < n_tiles) {
    if (tid == 0) *next = atomicAdd(queue, 1);   // read by all after the accumulate's barriers
    const int* trow = tinfo + 16 * tb;
    const int* tbeg = trow + 4;
    const int* tend = trow + 8;
    const float* tlam = reinterpret_cast<const float*>(trow + 12);
    const int row = trow[g];
    // this row's projection and own block value: loaded now, used after the accumulate
    const float pj = (row >= 0 && m < b) ? __ldg(p.proj + (size_t)row * b + m) : 0.f;
    const float ow = (row >= 0 && m < b) ? p.own[(size_t)row * p.ldo + p.b0 + m] : 0.f;
    {  // step 1: TMEM row := template row m in this slot's columns, zeros elsewhere
      const float* tp = (L::TPL_FLOATS ? tpl_s : p.tpl) + pk_off(m);
#pragma unroll 1
      for (int c8 = 0; c8 < 16; ++c8) {
        const int col = 8 * c8;   // warp-uniform
        float w8[8];
        const bool mine = col >= g * L::NG && col < (g + 1) * L::NG;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = col - g * L::NG + j;
          w8[j] = (mine && c <= m) ? tp[c] : 0.f;
        }
        tmem_st8(row_addr + col, w8);
      }
    }
    tmem_wait_st();
    tc_fence_before();
    int nch = 0;
#pragma unroll
    for (int s = 0; s < G; ++s) nch = max(nch, (tend[s] - tbeg[s] + L::KC - 1) / L::KC);
    double gacc = 0.0;
    pk_accumulate<G, UNIT>(p, smem, st, gacc, tbeg, tend, nch, tid);
    const int task_next = *next;   // published by the accumulate's barriers
    int nrow = -1;                 // the next tile's row of slot tid: its loads overlap the factorisation
    if (tid < G && task_next < n_tiles) nrow = tile_row(task_next, tid);
    const float lam = tlam[g];
    {  // lam on the diagonal (global column tid); the diagonal before factoring
      const int lane = tid & 31, e = lane & 7;
      const float lv = (m < b) ? lam : 0.f;
      float dg = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v[8];
        const uint32_t ca = row_addr + 32 * (tid >> 5) + 8 * j;
        tmem_ld8(ca, v);
        tmem_wait_ld();
        const bool mine = (lane >> 3) == j;
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] += (mine && q == e) ? lv : 0.f;
        tmem_st8(ca, v);
        const float a0 = (e & 1) ? v[1] : v[0], a1 = (e & 1) ? v[3] : v[2];
        const float a2 = (e & 1) ? v[5] : v[4], a3 = (e & 1) ? v[7] : v[6];
        const float b0 = (e & 2) ? a1 : a0, b1 = (e & 2) ? a3 : a2;
        if (mine) dg = (e & 4) ? b1 : b0;
      }
      tmem_wait_st();
      reinterpret_cast<float*>(smem + L::OFF_DIAG)[tid] = dg;
    }
    {
      float gv = 0.f;
      if (row >= 0 && m < b) gv = (float)(gacc + (double)pj + (double)lam * (double)ow);
      ys[tid] = gv;
    }
    __syncthreads();
    pk_factor<G>(p, smem, st, row_addr, tid, b);
    if (tid < G && task_next < n_tiles) put_tile(tb ^ 1, tid, nrow);
    pk_block_inverses<G>(smem, tid, b);
    __syncthreads();
    pk_backward<G>(smem, tid, b);
    const bool bad = FLAG[g] != 0;
    if (row >= 0 && m < b) {
      if (bad) {
        p.drow[(size_t)row * b + m] = 0.f;
      } else {
        p.own[(size_t)row * p.ldo + p.b0 + m] = ow - ds[tid];
        p.drow[(size_t)row * b + m] = ds[tid];
      }
    }
    if (bad && row >= 0 && m == 0) {   // the SIMT sweep redoes this row (cache update included)
      p.redo_rows[atomicAdd(p.redo_cnt, 1)] = row;
      atomicAdd(p.redo_total, 1ull);
    }
    tc_fence_before();
    __syncthreads();   // this tile's state (FLAG, tile buffer tb) is no longer read
    tc_fence_after();
    if (tid < G) FLAG[tid] = 0;
    task = task_next;
    tb ^= 1;
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free(st.tmem, 128);
}

}  // namespace ials

namespace ials {

// Heavy-row slices for b <= 64, G slices per tile: each slot's partial Hessian
// (its NG x NG diagonal block of the tile, summed from zero over the slice's
// entries with the packed pipeline) and fp64 partial gradient, written in the
// [slice][BT x BT] layout k_heavy_solve<BT = NG> reduces in a fixed order
// (BT x BT: 4 KB at b <= 32 instead of the 64 KB 128-wide tile).
template <int G, bool UNIT>
__global__ void __launch_bounds__(128, 4) k_heavy_partial_pk(SweepParams p,
                                                               const __grid_constant__ CUtensorMap fmap,
                                                               int use_tma) {
  using L = PkLay<G>;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = tc_smem_base(smem_raw);
  const int tid = threadIdx.x, g = tid / L::NG, m = tid - g * L::NG;
  {
    float4* x = reinterpret_cast<float4*>(smem + L::OFF_X);
    for (int i = tid; i < L::NB * G * L::KC * L::SW / 4; i += L::NT) x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L::OFF_TPTR);
  int* tinfo = reinterpret_cast<int*>(smem + L::OFF_TILE);   // beg[4] at +4, end[4] at +8
  int* next = reinterpret_cast<int*>(smem + L::OFF_FLAG) + 4;
  if (tid == 0) {
    for (int k = 0; k < L::NXT; ++k) mbar_init(bar + k, 1);
    for (int k = 0; k < L::NB; ++k) mbar_init(bar + L::BAR_GATHER + k, G);
    if (use_tma) prefetch_tmap(&fmap);
  }
  if (tid < 32) tmem_alloc(tptr, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  PkState st;
  st.tmem = *tptr;
  st.ph = 0u;
  st.gph = 0u;
  st.fmap = use_tma ? &fmap : nullptr;
  const uint32_t row_addr = st.tmem + ((uint32_t)((tid >> 5) * 32) << 16);
  const int n_tiles = (p.n_slices + G - 1) / G;
  int* queue = p.redo_cnt + 1;
  for (;;) {
    if (tid == 0) *next = atomicAdd(queue, 1);
    __syncthreads();
    const int task = *next;
    if (task >= n_tiles) break;
    if (tid < G) {
      const int sl = task * G + tid;
      tinfo[4 + tid] = sl < p.n_slices ? p.slice_begin[sl] : 0;
      tinfo[8 + tid] = sl < p.n_slices ? p.slice_end[sl] : 0;
    }
    {
      const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c8 = 0; c8 < 16; ++c8) tmem_st8(row_addr + 8 * c8, z);
      tmem_wait_st();
      tc_fence_before();
    }
    __syncthreads();
    const int* tbeg = tinfo + 4;
    const int* tend = tinfo + 8;
    int nch = 0;
#pragma unroll
    for (int s = 0; s < G; ++s) nch = max(nch, (tend[s] - tbeg[s] + L::KC - 1) / L::KC);
    double gacc = 0.0;
    pk_accumulate<G, UNIT>(p, smem, st, gacc, tbeg, tend, nch, tid);
    const int sl = task * G + g;
    if (sl < p.n_slices) {
      float* hp = p.hpart + (size_t)sl * L::NG * L::NG + (size_t)m * L::NG;
#pragma unroll
      for (int c32 = 0; c32 < L::NG; c32 += 32) {
        float v[32];
        tmem_ld32(row_addr + g * L::NG + c32, v);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(hp + c32 + 4 * q) =
              make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
      p.gpart[(size_t)sl * L::NG + m] = gacc;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free(st.tmem, 128);
}

}  // namespace ials
