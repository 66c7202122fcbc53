// ials_sweep_wb.cuh -- short rows of a rotated user pass (b = 128) solved
// through their Woodbury systems, G rows per 128-lane TMEM tile.
//
// In the rotated basis of ials_rot.cuh row r (n_r interactions, unit
// weights and labels) solves (D + X^T X) d = g, D = alpha0 L + lam_r I
// diagonal, X = the n_r gathered rows of F~ = F[:, pi] Q, g = X^T rho + p~
// (rho_k = yhat_k - 1, p~ = alpha0 (w @ slab) Q + lam_r w_pi Q).  With
// s = D^-1/2, Y = X diag(s) and z = s * g = Y^T rho + s * p~:
//     C = I + Y Y^T (n_r x n_r),  u = Y z,  v = C^-1 u,
//     d = s * (z - Y^T v)                        (Woodbury)
// -- an n_r x n_r factorisation instead of a b x b one.  And X d = v: the
// row's cache update is v itself (yhat_k -= v_k, no gather); the pass's
// entry-parallel cache kernel skips these rows.
//
// Thread t = g * NG + k <-> TMEM lane t <-> entry k of slot g (k < n_g <= NG).
//   pass 1  per 16-column chunk of b: each thread loads its entry's 16 values
//           of F~ (L2-resident, 64 B), forms y = s x and the chunk's hi/lo
//           operand row; one thread issues C += Y_c Y_c^T (M = N = 128,
//           K = 16, 3xTF32) into TMEM initialised to I;
//   u = Y z = Y (s p~) + Y Y^T rho: the first term accumulates in pass 1
//   (each thread's own entry), the second is (C - I) rho from the thread's
//   TMEM row of C -- z itself is never formed; the blocked Cholesky of the G
//   matrices C and the solves (the packed sweep's, on the max(n_g) leading
//   rows); pass 2: d~ = s z - s^2 X^T v = s^2 (p~ - X^T (v - rho)), the one
//   transposed product by a warp butterfly per 16 columns -> drow (the
//   back-rotation GEMM applies Q).  (u = Y q + (C - I) rho carries the 3xTF32 error of C times
//   |rho| instead of |z|: ~1e-7 absolute on d, far inside 1e-3 of the rows.)
// Work per row: 2 n_r b loads from L2 and an n_r/8-panel chain.
#pragma once
#include "ials_sweep_pk.cuh"

namespace ials {

template <int G>
struct WbLay {
  static constexpr int NT = 128, NG = 128 / G, B = 128, KCH = 16, NCH = B / KCH;
  static constexpr int LPS = ((NG * (NG + 1) / 2) + 3) & ~3;
  // overlay -- pass 1: operands hi / lo x 2 buffers (16 KB each); factor:
  // packed L per slot, the panel operands, the diagonal staging / inverses
  static constexpr int OFF_OP = 0;
  static constexpr int OFF_L = 0;
  static constexpr int L_BYTES = G * LPS * 4;
  static constexpr int OFF_PA = ((L_BYTES + 1023) / 1024) * 1024;
  static constexpr int OFF_LI = OFF_PA + 8192;
  static constexpr int OVL = (OFF_LI + 8192 > 32768) ? OFF_LI + 8192 : 32768;
  static constexpr int OFF_S = OVL;                      // [G][B] s = D^-1/2
  static constexpr int OFF_SZ = OFF_S + G * B * 4;       // [G][B] s^2 p~ (fp32, for Y q in pass 1)
  static constexpr int OFF_Z = OFF_SZ + G * B * 4;       // [G][B] s * z (fp64)
  static constexpr int OFF_ZP = OFF_Z + G * B * 8;       // [4 warps][B] column partials
  static constexpr int OFF_LAM = OFF_ZP + 4 * B * 4;     // [B] alpha0 * eigenvalues
  static constexpr int OFF_DG = OFF_LAM + B * 4;         // per slot, per panel parity: 320 B
  static constexpr int OFF_Y = OFF_DG + G * 640;
  static constexpr int OFF_YF = OFF_Y + 512;
  static constexpr int OFF_ID = OFF_YF + 512;
  static constexpr int OFF_D = OFF_ID + 512;
  static constexpr int OFF_DIAG = OFF_D + 512;
  static constexpr int OFF_TILE = OFF_DIAG + 512;        // [2][rows[4], beg[4], end[4], lam[4]]
  static constexpr int OFF_FLAG = OFF_TILE + 128;        // flags[G], next task
  static constexpr int OFF_RHO = OFF_FLAG + 32;          // [128] rho of every lane's entry
  static constexpr int OFF_BAR = OFF_RHO + 512;          // MMA bars [2]
  static constexpr int OFF_TPTR = OFF_BAR + 16;
  static constexpr int BYTES = OFF_TPTR + 16 + 1024;
};

// element (row m, k) of a 16-wide K-major operand without swizzle: 8 x 4 core
// matrices, LBO 128 B (K direction), SBO 512 B (8-row groups)
IALS_DEVI int wb_index(int m, int k) { return (m >> 3) * 128 + (k >> 2) * 32 + (m & 7) * 4 + (k & 3); }

// sum over the warp's 32 lanes of v[0..15]: lane l ends with the sum of
// column (l >> 1) & 15 (both lanes of a pair)
IALS_DEVI float butterfly16(float (&v)[16], int lane) {
  float a[8], b4[4], c2[2];
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4, h2 = lane & 2;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float send = h16 ? v[j] : v[j + 8];
    const float keep = h16 ? v[j + 8] : v[j];
    a[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float send = h8 ? a[j] : a[j + 4];
    const float keep = h8 ? a[j + 4] : a[j];
    b4[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const float send = h4 ? b4[j] : b4[j + 2];
    const float keep = h4 ? b4[j + 2] : b4[j];
    c2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  const float send = h2 ? c2[0] : c2[1];
  const float keep = h2 ? c2[1] : c2[0];
  float s = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}
// (column of lane l: bit 4 -> 8, bit 3 -> 4, bit 2 -> 2, bit 1 -> 1)
IALS_DEVI int butterfly16_col(int lane) {
  return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}

// rows lrows[row0 ..) in tiles of G (all with n <= NG): the rotated pass's
// fixed side F~ (n_fixed x 128, ld 128) is p.fixed, the rotated projection p~
// is p.proj, W[:, pi] Q is p.wq, alpha0 * eigenvalues p.rot_lam; d~ -> drow
// (tot / bucket: the host epoch's chunked first pass -- the rows are bucket
// `bucket` of the grouped light list, whose bucket sizes tot[] live on the device)
template <int G>
__global__ void __launch_bounds__(128, 4) k_sweep_wb(SweepParams p, int row0, int n_rows, int* queue,
                                                     const int* tot = nullptr, int bucket = 0) {
  using L = WbLay<G>;
  if (tot) {
    int off = 0;
    for (int k = 0; k < bucket; ++k) off += tot[k];
    row0 = off;
    n_rows = tot[bucket];
  }
  constexpr int B = L::B;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = tc_smem_base(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = tid / L::NG, k = tid - g * L::NG;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + L::OFF_TPTR);
  int* tinfo = reinterpret_cast<int*>(smem + L::OFF_TILE);
  int* FLAG = reinterpret_cast<int*>(smem + L::OFF_FLAG);
  float* S = reinterpret_cast<float*>(smem + L::OFF_S);
  float* SZ = reinterpret_cast<float*>(smem + L::OFF_SZ);
  double* Z = reinterpret_cast<double*>(smem + L::OFF_Z);
  float* ZP = reinterpret_cast<float*>(smem + L::OFF_ZP);
  float* LAM = reinterpret_cast<float*>(smem + L::OFF_LAM);
  float* ys = reinterpret_cast<float*>(smem + L::OFF_Y);
  float* ds = reinterpret_cast<float*>(smem + L::OFF_D);
  float* DIAG = reinterpret_cast<float*>(smem + L::OFF_DIAG);
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  LAM[tid] = p.alpha0 * p.rot_lam[tid];
  DIAG[tid] = 0.f;   // C = I + Y Y^T: pivots >= 1, the guard only rejects non-finite ones
  ds[tid] = 0.f;
  if (tid < 32) tmem_alloc(tptr, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  PkState st;
  st.tmem = *tptr;
  st.ph = 0u;
  st.gph = 0u;
  st.fmap = nullptr;
  const uint32_t row_addr = st.tmem + ((uint32_t)((tid >> 5) * 32) << 16);
  const int* lrows = p.light_rows + row0;
  const int n_tiles = (n_rows + G - 1) / G;
  int* next = FLAG + 4;
  auto tile_row = [&](int t, int s) { const int q = t * G + s; return q < n_rows ? lrows[q] : -1; };
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
  const uint32_t idesc = make_idesc_tf32(128, 128, 0, 0, 0);
  while (task < n_tiles) {
    if (tid == 0) *next = atomicAdd(queue, 1);
    const int* trow = tinfo + 16 * tb;
    const int row = trow[g], ebeg = trow[4 + g], n_g = trow[8 + g] - ebeg;
    int nmax = 0;
#pragma unroll
    for (int s = 0; s < G; ++s) nmax = max(nmax, trow[8 + s] - trow[4 + s]);
    const bool valid = row >= 0 && k < n_g;
    const int col = valid ? __ldg(p.side.cols + ebeg + k) : 0;
    IALS_CHECK(!valid || (col >= 0 && col < p.side.n_fixed && ebeg + k < p.side.nnz));
    const float rho = valid ? p.cache[ebeg + k] - 1.f : 0.f;   // user side: pos = e; UNIT
    const float* xr = p.fixed + (size_t)col * B;
    // per slot: s = D^-1/2 and z := s * p~ (column tid of every slot)
#pragma unroll
    for (int s = 0; s < G; ++s) {
      const int r = trow[s];
      const float lam_s = reinterpret_cast<const float*>(trow)[12 + s];
      const float sv = rsqrtf(LAM[tid] + lam_s);
      S[s * B + tid] = sv;
      double pt = 0.0;   // p~
      if (r >= 0)
        pt = (double)__ldg(p.proj + (size_t)r * B + tid) +
             (double)lam_s * (double)__ldg(p.wq + (size_t)r * B + tid);
      Z[s * B + tid] = (double)sv * pt;
      SZ[s * B + tid] = (float)((double)sv * (double)sv * pt);
    }
    reinterpret_cast<float*>(smem + L::OFF_RHO)[tid] = rho;
    // (TMEM is not initialised: the tile's first MMA overwrites it, and it holds
    // Y Y^T = C - I; the factorisation adds the identity as it reads the diagonal)
    tc_fence_before();
    __syncthreads();   // S, Z visible; the previous tile's TMEM reads are done
    // ---- pass 1: C += Y_c Y_c^T, Y^T rho
    float x[16], xn[16];
    auto load16 = [&](float (&v)[16], int c0) {   // two 32-byte loads (rows are 512 B aligned)
      float a[8], b8[8];
      if (valid) {
        ldg256(xr + c0, a);
        ldg256(xr + c0 + 8, b8);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = b8[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[j] = a[j];
        v[8 + j] = b8[j];
      }
    };
    load16(x, 0);
    uint32_t pend = 0;
    float uq = 0.f;   // y_k . (s p~) = x_k . (s^2 p~)
    for (int ch = 0; ch < L::NCH; ++ch) {
      const int c0 = ch * L::KCH, ob = ch & 1;
      if (ch + 1 < L::NCH) load16(xn, c0 + L::KCH);
      float y[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        y[j] = x[j] * S[g * B + c0 + j];
        uq = fmaf(x[j], SZ[g * B + c0 + j], uq);
      }
      if (pend & (1u << ob)) {   // buffer ob was read by chunk ch - 2's MMAs
        mbar_wait(bar + ob, (st.ph >> ob) & 1u);
        st.ph ^= 1u << ob;
        pend &= ~(1u << ob);
      }
      {
        float* OH = reinterpret_cast<float*>(smem + L::OFF_OP + ob * 16384);
        float* OL = OH + 2048;
        const int o = wb_index(tid, 0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float h[4], l[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            h[j] = tf32_rna(y[4 * q + j]);
            l[j] = y[4 * q + j] - h[j];
          }
          *reinterpret_cast<float4*>(OH + o + 32 * q) = make_float4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<float4*>(OL + o + 32 * q) = make_float4(l[0], l[1], l[2], l[3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t hi = smem_u32(smem + L::OFF_OP + ob * 16384), lo = hi + 8192;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint64_t ah = make_sdesc(hi + ks * 256, 128, 512, kSwizzleNone);
          const uint64_t al = make_sdesc(lo + ks * 256, 128, 512, kSwizzleNone);
          umma_tf32(st.tmem, ah, ah, idesc, (ch | ks) != 0);   // the tile's first MMA overwrites
          umma_tf32(st.tmem, ah, al, idesc, 1);
          umma_tf32(st.tmem, al, ah, idesc, 1);
        }
        umma_commit(bar + ob);
      }
      pend |= 1u << ob;
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = xn[j];
    }
#pragma unroll
    for (int ob = 0; ob < 2; ++ob)
      if (pend & (1u << ob)) {
        mbar_wait(bar + ob, (st.ph >> ob) & 1u);
        st.ph ^= 1u << ob;
      }
    tc_fence_after();
    const int task_next = *next;
    int nrow = -1;
    if (tid < G && task_next < n_tiles) nrow = tile_row(task_next, tid);
    // u_k = y_k . (s p~) + sum_j (C - I)_kj rho_j over the slot's entries: the
    // thread's TMEM row of Y Y^T (the diagonal |y_k|^2 included: TMEM holds
    // C - I, so it carries no added identity whose rounding would hide it)
    {
      const float* RH = reinterpret_cast<const float*>(smem + L::OFF_RHO) + g * L::NG;
      float cr = 0.f;
#pragma unroll
      for (int c32 = 0; c32 < L::NG; c32 += 32) {
        float cv[32];
        tmem_ld32(row_addr + g * L::NG + c32, cv);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) cr = fmaf(cv[j], RH[c32 + j], cr);
      }
      ys[tid] = valid ? uq + cr : 0.f;
    }
    __syncthreads();
    // ---- v = C^-1 u on the leading nmax rows of every slot
    const int nb = (nmax + 7) & ~7;
    pk_factor<G, L, true>(p, smem, st, row_addr, tid, nb);
    if (tid < G && task_next < n_tiles) put_tile(tb ^ 1, tid, nrow);
    pk_block_inverses<G, L>(smem, tid, nb);
    __syncthreads();
    pk_backward<G, L>(smem, tid, nb);
    // ---- pass 2: d~ = s z - s^2 X^T v with z = s p~ + s X^T rho, i.e.
    // d~ = s^2 (p~ - X^T (v - rho)): ONE transposed product, X^T (v - rho)
    // (butterfly per 16 columns), so pass 1 forms no column sums at all
    {
      const float vk = valid ? ds[tid] - rho : 0.f;
      load16(x, 0);
#pragma unroll 1
      for (int c0 = 0; c0 < B; c0 += 16) {
        if (c0 + 16 < B) load16(xn, c0 + 16);
        float v16[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v16[j] = x[j] * vk;
        const float cs = butterfly16(v16, lane);
        if (!(lane & 1)) ZP[warp * B + c0 + butterfly16_col(lane)] = cs;
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = xn[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < G; ++s) {
      const int r = trow[s];
      if (r < 0 || FLAG[s]) continue;
      float xv = 0.f;
#pragma unroll
      for (int w = 0; w < 4 / G; ++w) xv += ZP[(s * (4 / G) + w) * B + tid];
      const double sv = S[s * B + tid];
      p.drow[(size_t)r * B + tid] = (float)(sv * Z[s * B + tid] - sv * sv * (double)xv);
    }
    // X~ d~ = v: the row's cache update (unless the pass's cache kernel does it)
    if (p.flat_skip_deg > 0 && valid && !FLAG[g]) p.cache[ebeg + k] -= ds[tid];
    if (tid < G && trow[tid] >= 0 && FLAG[tid]) {   // non-finite pivot: the SIMT sweep redoes the row
      p.redo_rows[atomicAdd(p.redo_cnt, 1)] = trow[tid];
      atomicAdd(p.redo_total, 1ull);
    }
    tc_fence_before();
    __syncthreads();
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
