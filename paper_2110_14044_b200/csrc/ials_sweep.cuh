// ials_sweep.cuh -- the fused per-row block-Newton sweep (K-sweep / K-heavy).
//
// Replaces the reference's _newton_side_pass (solvers.py:152-186) and
// _solve_rows (solvers.py:101-114).  For a row r of the updated side and the
// block pi = [b0, b0+b):
//   1. gather h_k = F[col_k, pi] (staged in shared memory with cp.async)
//   2. rho_k = a_k (yhat_k - y_k);            g  = sum_k rho_k h_k
//   3. g += alpha0 * (U[r,:] @ slab) + lam_r U[r,pi]  (U @ slab precomputed: proj)
//   4. Hs = sum_k a_k h_k h_k^T + alpha0 slab[pi,:] + lam_r I  (lower triangle,
//      register-tiled: each warp owns 32x32 super-tiles, each lane a 4x8 tile)
//   5. Cholesky of Hs in the same register tiles (right-looking, one column per
//      step, the forward solve L y = g fused in), backward solve L^T d = y by one
//      warp from the packed L kept in shared memory
//   6. U[r,pi] -= d
//   7. yhat_k -= h_k . d   (cache slot pos_k; entries are re-staged when the row
//      has more than two chunks)
// Rows are independent and own disjoint cache slots, so there is
// no inter-row synchronisation.  Heavy rows (long item rows) are split into
// slices: partial (Hs, g) per slice -> fixed-order reduction + solve -> per-slice
// cache update, which keeps the result deterministic.
#pragma once
#include "ials_common.cuh"

namespace ials {

struct SideDev {
  int n_rows, n_fixed;
  const int* ptr;
  const int* cols;
  const float* labels;
  const float* weights;
  const int* pos;
  const float* lam;
  const int* rows;   // [nnz] row of each entry, or null
  long long nnz;
};

struct SweepParams {
  SideDev side;
  const float* fixed;
  int ldf;
  float* own;
  int ldo;
  int d, b0, b;
  const float* slab;  // d x b, ld b
  const float* proj;  // n_rows x b, ld b : alpha0 * own @ slab
  float alpha0;
  float* cache;
  int side_id;
  unsigned long long* err;
  int vec;  // 16-byte staging is legal (b % 4 == 0, b0 % 4 == 0, ldf % 4 == 0, aligned base)
  const int* light_rows;
  int n_light;
  const int* heavy_rows;
  const int* heavy_slice0;
  int n_heavy;
  const int* slice_heavy;
  const int* slice_begin;
  const int* slice_end;
  int n_slices;
  float* hpart;   // [n_slices][BT*BT]
  double* gpart;  // [n_slices][BT] (fp64: the gradient sum cancels strongly)
  float* hdelta;  // [n_heavy][BT]
  long long* dbg; // optional per-CTA phase timestamps (profiling builds only)
  const float* tpl;  // [8448] packed alpha0 * slab[pi, pi] (tensor-core plan)
  // fused tensor-core sweep: rows whose Cholesky pivots cancel more than
  // cond_max (H_kk / pivot_k) are left untouched and listed for the SIMT sweep
  int* redo_rows;
  int* redo_cnt;
  unsigned long long* redo_total;
  float cond_max;
  const int* n_light_dev;  // if set, k_sweep_light reads its row count here
  int* queue;              // if set, k_sweep_light takes its rows from this zeroed counter
  float* drow;             // [n_rows][b] per-row d of the fused sweep (k_pass_cache)
  int fb0;                 // column of the block in `fixed` (b0, or 0 for a compact copy)
  int fixed_cols;          // columns of `fixed` (d, or the compact copy's width)
  // rotated user pass (ials_rot.cuh): fixed = F[:, pi] Q, proj = the rotated
  // projection, slab[pi, pi] = diag(eigenvalues); the lam * w term reads
  // wq = W[:, pi] Q, and the row's d~ goes to drow only (own is updated by
  // the back-rotation GEMM, the cache by the pass's cache kernel)
  int rot;
  const float* wq;
  const float* rot_lam;
  int rot_n64, rot_n32;    // light rows with > 64 / > 32 entries (prefix lengths)
  int flat_skip_deg;       // k_pass_cache_flat skips rows with at most this many entries
                           // (their cache is updated by the kernel that solved them)
  const int* x_rows;       // the other side's view of the same entries (rows = fixed-side ids,
  const int* x_cols;       //   cols = this side's ids, x_pos = cache positions or NULL): the
  const int* x_pos;        //   cache pass may walk it instead (k_pass_cache_flat<., ., true>)
  const int* chunk_tot;    // if set (k_sweep_tc4): light rows grouped by row chunk, chunk_tot[k]
  int chunk;               //   rows in chunk k; this launch sweeps chunk `chunk` only
  int heavy_reduced;       // k_heavy_solve reads one slot per heavy row (k_heavy_reduce ran)
  int b1_flat;             // b = 1: the sweep leaves the cache to k_b1_cache_flat
};

template <int BT>
struct Cfg;
// ST: warp super-tile edge; SR x SC: per-lane tile; NW: warps per row team;
// RPC: row teams per CTA; KC: entries per staged chunk.
template <> struct Cfg<8>   { static constexpr int ST = 8,  SR = 1, SC = 2, NW = 1,  RPC = 4, KC = 32; };
template <> struct Cfg<16>  { static constexpr int ST = 16, SR = 2, SC = 4, NW = 1,  RPC = 4, KC = 32; };
template <> struct Cfg<32>  { static constexpr int ST = 16, SR = 2, SC = 4, NW = 1,  RPC = 4, KC = 16; };
template <> struct Cfg<64>  { static constexpr int ST = 32, SR = 4, SC = 8, NW = 3,  RPC = 1, KC = 32; };
template <> struct Cfg<128> { static constexpr int ST = 32, SR = 4, SC = 8, NW = 10, RPC = 1, KC = 32; };
template <> struct Cfg<256> { static constexpr int ST = 32, SR = 4, SC = 8, NW = 12, RPC = 1, KC = 16; };

template <int BT>
struct Lay {
  using C = Cfg<BT>;
  static constexpr int NW = C::NW, NT = NW * 32, KC = C::KC, ST = C::ST, SR = C::SR, SC = C::SC,
                       RPC = C::RPC;
  static constexpr int XLD = BT + 4;
  static constexpr int NS = BT / ST;
  static constexpr int NSUP = NS * (NS + 1) / 2;
  static constexpr int TPW = (NSUP + NW - 1) / NW;
  static constexpr int LP = BT * (BT + 1) / 2;
  static constexpr int MB = BT >= 32 ? BT / 32 : 1;
  static constexpr int OFF_X = 0;
  static constexpr int OFF_AW = OFF_X + 2 * KC * XLD;
  static constexpr int OFF_RH = OFF_AW + 2 * KC;
  static constexpr int OFF_PS = OFF_RH + 2 * KC;
  static constexpr int OFF_L = OFF_PS + 2 * KC;
  static constexpr int PLD = BT + 4;  // row stride of the transposed panel buffers
  static constexpr int OFF_PB = OFF_L + ((LP + 3) / 4) * 4;  // raw panel, [8][PLD]
  static constexpr int OFF_LB = OFF_PB + 8 * PLD;            // L panel,   [8][PLD]
  static constexpr int OFF_PY = OFF_LB + 8 * PLD;            // y of the panel [8]
  static constexpr int OFF_Y = OFF_PY + 8;
  static constexpr int OFF_YF = OFF_Y + BT;
  static constexpr int OFF_ID = OFF_YF + BT;
  static constexpr int OFF_D = OFF_ID + BT;
  static constexpr int OFF_Q = OFF_D + BT;   // the team's next row (device queue)
  static constexpr int FLOATS = OFF_Q + 4;
  static constexpr int TEAM_BYTES = FLOATS * 4;
  static constexpr int CTA_BYTES = TEAM_BYTES * RPC;
};

template <int N>
IALS_DEVI void lds_vec(float* dst, const float* src) {
  if constexpr (N == 8) {
    float4 a = *reinterpret_cast<const float4*>(src);
    float4 b = *reinterpret_cast<const float4*>(src + 4);
    dst[0] = a.x; dst[1] = a.y; dst[2] = a.z; dst[3] = a.w;
    dst[4] = b.x; dst[5] = b.y; dst[6] = b.z; dst[7] = b.w;
  } else if constexpr (N == 4) {
    float4 a = *reinterpret_cast<const float4*>(src);
    dst[0] = a.x; dst[1] = a.y; dst[2] = a.z; dst[3] = a.w;
  } else if constexpr (N == 2) {
    float2 a = *reinterpret_cast<const float2*>(src);
    dst[0] = a.x; dst[1] = a.y;
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) dst[i] = src[i];
  }
}

// Per-thread view of the register tiles of one row team.
template <int BT>
struct Tiles {
  using L = Lay<BT>;
  float acc[L::TPW][L::SR][L::SC];
  int roff[L::TPW], coff[L::TPW];
  bool valid[L::TPW];

  IALS_DEVI void init(int warp, int lane) {
#pragma unroll
    for (int t = 0; t < L::TPW; ++t) {
      int s = warp + L::NW * t;
      valid[t] = s < L::NSUP;
      int I = 0;
      while ((I + 1) * (I + 2) / 2 <= s) ++I;  // super-tile row (s = I(I+1)/2 + J)
      int J = s - I * (I + 1) / 2;
      roff[t] = I * L::ST + (lane >> 2) * L::SR;
      coff[t] = J * L::ST + (lane & 3) * L::SC;
#pragma unroll
      for (int i = 0; i < L::SR; ++i)
#pragma unroll
        for (int j = 0; j < L::SC; ++j) acc[t][i][j] = 0.f;
    }
  }
};

// Stage entries [ebeg, ebeg+nk) of the row into buffer `buf`.
template <int BT>
IALS_DEVI void stage_chunk(const SweepParams& p, float* sm, int buf, int ebeg, int nk, int tid) {
  using L = Lay<BT>;
  float* X = sm + L::OFF_X + buf * L::KC * L::XLD;
  if (p.vec) {
    // BT/4 float4 slots per entry (a power of two: shifts, no division);
    // slots beyond b/4 are skipped
    constexpr int SL = BT / 4 >= 1 ? BT / 4 : 1;
    constexpr int LG = SL == 1 ? 0 : SL == 2 ? 1 : SL == 4 ? 2 : SL == 8 ? 3 : SL == 16 ? 4
                       : SL == 32 ? 5 : 6;
    const int bv = p.b >> 2;
    for (int i = tid; i < nk * SL; i += L::NT) {
      const int k = i >> LG, v = i & (SL - 1);
      if (v >= bv) continue;
      const int col = __ldg(p.side.cols + ebeg + k);
      IALS_CHECK(col >= 0 && col < p.side.n_fixed);
      cp_async16(X + k * L::XLD + 4 * v, p.fixed + (size_t)col * p.ldf + p.fb0 + 4 * v);
    }
  } else {
    for (int i = tid; i < nk * p.b; i += L::NT) {
      int k = i / p.b, v = i - k * p.b;
      int col = __ldg(p.side.cols + ebeg + k);
      cp_async4(X + k * L::XLD + v, p.fixed + (size_t)col * p.ldf + p.fb0 + v);
    }
  }
  cp_async_commit();
  float* aw = sm + L::OFF_AW + buf * L::KC;
  float* rh = sm + L::OFF_RH + buf * L::KC;
  int* ps = reinterpret_cast<int*>(sm + L::OFF_PS) + buf * L::KC;
  for (int k = tid; k < L::KC; k += L::NT) {
    float a = 0.f, r = 0.f;
    int pos = 0;
    if (k < nk) {
      int e = ebeg + k;
      a = p.side.weights ? __ldg(p.side.weights + e) : 1.f;
      float y = p.side.labels ? __ldg(p.side.labels + e) : 1.f;
      pos = p.side.pos ? __ldg(p.side.pos + e) : e;
      r = a * (p.cache[pos] - y);
    }
    aw[k] = a;
    rh[k] = r;
    ps[k] = pos;
  }
}

// Hessian + gradient accumulation over one staged chunk.
template <int BT>
IALS_DEVI void accumulate_chunk(Tiles<BT>& T, double& gacc, const float* sm, int buf, int nk,
                                int tid, bool unit) {
  using L = Lay<BT>;
  const float* X = sm + L::OFF_X + buf * L::KC * L::XLD;
  const float* aw = sm + L::OFF_AW + buf * L::KC;
  const float* rh = sm + L::OFF_RH + buf * L::KC;
  const int nk4 = (nk + 3) & ~3;  // padded entries have a = 0 and finite stale rows
  // Two-level (blocked) summation: each chunk is summed into a zeroed local
  // tile that is then added to the running Hessian, as a blocked GEMM would;
  // a long row's sum is then ~sqrt(KC) times more accurate than one running
  // fp32 sum (matters for the ill-conditioned first epochs of heavy rows).
  // Tiles are visited outermost so one local tile suffices for any TPW.
#pragma unroll
  for (int t = 0; t < L::TPW; ++t) {
    if (!T.valid[t]) continue;
    float loc[L::SR][L::SC];
#pragma unroll
    for (int i = 0; i < L::SR; ++i)
#pragma unroll
      for (int j = 0; j < L::SC; ++j) loc[i][j] = 0.f;
    const float* xr0 = X + T.roff[t];
    const float* xc0 = X + T.coff[t];
    // unit weights: no per-entry scale, so stop at nk (stale padded rows
    // would otherwise contribute); weighted: padded entries carry a = 0
    const int kend = unit ? nk : nk4;
#pragma unroll 2
    for (int k = 0; k < kend; ++k) {
      float rv[L::SR], cv[L::SC];
      lds_vec<L::SR>(rv, xr0 + k * L::XLD);
      lds_vec<L::SC>(cv, xc0 + k * L::XLD);
      if (unit) {
#pragma unroll
        for (int i = 0; i < L::SR; ++i)
#pragma unroll
          for (int j = 0; j < L::SC; ++j) loc[i][j] = fmaf(rv[i], cv[j], loc[i][j]);
      } else {
        const float a = aw[k];
#pragma unroll
        for (int i = 0; i < L::SR; ++i) {
          const float ra = rv[i] * a;
#pragma unroll
          for (int j = 0; j < L::SC; ++j) loc[i][j] = fmaf(ra, cv[j], loc[i][j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < L::SR; ++i)
#pragma unroll
      for (int j = 0; j < L::SC; ++j) T.acc[t][i][j] += loc[i][j];
  }
  if (tid < BT) {
    // g = sum rho_k h_k + alpha0 w G + lam w cancels by orders of magnitude
    // on long rows, so the row sum is kept in double; each chunk's products
    // are summed in four fixed-order fp32 chains and folded in (4 fp64
    // conversions per chunk instead of 2 per entry: the conversion unit is
    // narrow).
    float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f;
    int k = 0;
    for (; k + 3 < nk; k += 4) {
      g0 = fmaf(rh[k], X[k * L::XLD + tid], g0);
      g1 = fmaf(rh[k + 1], X[(k + 1) * L::XLD + tid], g1);
      g2 = fmaf(rh[k + 2], X[(k + 2) * L::XLD + tid], g2);
      g3 = fmaf(rh[k + 3], X[(k + 3) * L::XLD + tid], g3);
    }
    for (; k < nk; ++k) g0 = fmaf(rh[k], X[k * L::XLD + tid], g0);
    gacc += ((double)g0 + (double)g1) + ((double)g2 + (double)g3);
  }
}

// Accumulate entries [ebeg, eend) with a double-buffered cp.async pipeline.
// Returns the number of chunks (so callers know whether buffers still hold them).
template <int BT>
IALS_DEVI int accumulate_range(const SweepParams& p, Tiles<BT>& T, double& gacc, float* sm,
                               int ebeg, int eend, int tid, int team) {
  using L = Lay<BT>;
  const int n = eend - ebeg;
  const int nch = (n + L::KC - 1) / L::KC;
  if (nch > 0) stage_chunk<BT>(p, sm, 0, ebeg, min(L::KC, n), tid);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      int s = ebeg + (c + 1) * L::KC;
      stage_chunk<BT>(p, sm, (c + 1) & 1, s, min(L::KC, eend - s), tid);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    team_sync<L::NW>(team);
    int s = ebeg + c * L::KC;
    accumulate_chunk<BT>(T, gacc, sm, c & 1, min(L::KC, eend - s), tid,
                         p.side.weights == nullptr);
    team_sync<L::NW>(team);
  }
  return nch;
}

// Steps 3-5: add the alpha0 slab / lambda terms, factor, solve; leaves the
// step d in sm[OFF_D .. +b).  A non-positive pivot is reported to the error
// word (the solve continues with pivot 1 so every value stays finite).
//
// Factorisation: right-looking blocked Cholesky with panels of 8 columns.
// The lower triangle lives in the same register tiles the Hessian was
// accumulated in.  Per panel:
//   A1  warp 0 factors the 8x8 diagonal block (every lane redundantly, in
//       registers) and forward-solves its part of the right-hand side;
//   A2  every row below the panel is triangular-solved against it (one thread
//       per row) and its RHS entry is updated;
//   B   the trailing matrix takes a rank-8 update in the register tiles
//       (vectorised panel loads, no masking: elements above the trailing block
//       are final or unused), then the owners publish the next raw panel.
// The backward solve L^T d = y runs on warp 0 panel by panel from the packed
// L kept in shared memory.
// GUARD (heavy rows whose Hessian partials came from the tensor core): the
// original diagonal is kept in the (unused) staging area, and a pivot that
// lost more than cond_max of it to cancellation flags the row (OFF_X + BT)
// for the FP32 redo instead of reporting it.
template <int BT, bool GUARD = false>
IALS_DEVI void finalize_and_solve(const SweepParams& p, Tiles<BT>& T, double gacc, float* sm,
                                  int row, int tid, int team) {
  using L = Lay<BT>;
  const int warp = tid >> 5, lane = tid & 31;
  const int b = p.b;
  float* Lp = sm + L::OFF_L;
  float* PB = sm + L::OFF_PB;
  float* LB = sm + L::OFF_LB;
  float* PY = sm + L::OFF_PY;
  float* ys = sm + L::OFF_Y;
  float* yf = sm + L::OFF_YF;
  float* invd = sm + L::OFF_ID;
  float* ds = sm + L::OFF_D;
  const float lam = p.side.lam[row];
  if (tid < BT && tid >= b) {  // padded rows: zero L panel rows keep them identity
#pragma unroll
    for (int q = 0; q < 8; ++q) LB[q * L::PLD + tid] = 0.f;
  }
  if (tid < BT) {
    double g = 0.0;
    if (tid < b)
      g = gacc + (double)p.proj[(size_t)row * b + tid] +
          (double)lam * (double)(p.rot ? p.wq[(size_t)row * b + tid]
                                       : p.own[(size_t)row * p.ldo + p.b0 + tid]);
    ys[tid] = (float)g;
  }
  const float a0 = p.alpha0;
  if (GUARD && tid == 0) reinterpret_cast<int*>(sm + L::OFF_X + BT)[0] = 0;
#pragma unroll
  for (int t = 0; t < L::TPW; ++t) {
    if (!T.valid[t]) continue;
#pragma unroll
    for (int i = 0; i < L::SR; ++i) {
      const int gi = T.roff[t] + i;
#pragma unroll
      for (int j = 0; j < L::SC; ++j) {
        const int gj = T.coff[t] + j;
        float v;
        if (gi < b && gj < b) {
          v = T.acc[t][i][j] + a0 * __ldg(p.slab + (size_t)(p.b0 + gi) * b + gj);
          if (gi == gj) {
            v += lam;
            if (GUARD) sm[L::OFF_X + gi] = v;
          }
        } else {
          v = (gi == gj) ? 1.f : 0.f;
        }
        T.acc[t][i][j] = v;
      }
    }
  }
  // 8-wide panels need SC >= 8 for the owner layout; BT = 8 / 16 tiles have
  // SC = 2 / 4, so their panels are assembled from 4 / 2 owner lanes.
  constexpr int PW = 8;
  const int np = (b + PW - 1) / PW;
  // publish panel 0 (raw)
#pragma unroll
  for (int t = 0; t < L::TPW; ++t) {
    if (!T.valid[t] || T.coff[t] >= PW) continue;
#pragma unroll
    for (int m = 0; m < L::SC; ++m) {
      float* dst = PB + (T.coff[t] + m) * L::PLD + T.roff[t];
#pragma unroll
      for (int i = 0; i < L::SR; ++i) dst[i] = T.acc[t][i][m];
    }
  }
  team_sync<L::NW>(team);
  for (int pp = 0; pp < np; ++pp) {
    const int c0 = pp * PW;
    // ---- A1: 8x8 diagonal block (warp 0, redundantly per lane)
    if (warp == 0) {
      float a[PW][PW];
#pragma unroll
      for (int q = 0; q < PW; ++q)
#pragma unroll
        for (int m = 0; m <= q; ++m) a[q][m] = PB[m * L::PLD + c0 + q];
      float rinv[PW];
      int bad = -1;
      bool cancel = false;
#pragma unroll
      for (int k = 0; k < PW; ++k) {
        float dk = a[k][k];
        if (GUARD && c0 + k < b && !(dk > 0.f && dk < 3.0e38f && sm[L::OFF_X + c0 + k] <= p.cond_max * dk))
          cancel = true;
        if (!(dk > 0.f) || !(dk < 3.0e38f)) {
          if (bad < 0) bad = k;
          dk = 1.f;
        }
        const float r = rsqrtf(dk);
        rinv[k] = r;
        a[k][k] = dk * r;
#pragma unroll
        for (int i = k + 1; i < PW; ++i) a[i][k] *= r;
#pragma unroll
        for (int i = k + 1; i < PW; ++i)
#pragma unroll
          for (int j = k + 1; j <= i; ++j) a[i][j] = fmaf(-a[i][k], a[j][k], a[i][j]);
      }
      if (GUARD) {
        if (cancel && lane == 0) reinterpret_cast<int*>(sm + L::OFF_X + BT)[0] = 1;
      } else if (bad >= 0 && c0 + bad < b && lane == 0) {
        report_singular(p.err, p.side_id, row, c0 + bad);
      }
      float y[PW];
#pragma unroll
      for (int q = 0; q < PW; ++q) {
        float v = ys[c0 + q];
#pragma unroll
        for (int m = 0; m < q; ++m) v = fmaf(-a[q][m], y[m], v);
        y[q] = v * rinv[q];
      }
      if (lane < PW) {
        const int q = lane;
        float yq = 0.f, rq = 0.f;
#pragma unroll
        for (int qq = 0; qq < PW; ++qq)
          if (qq == q) { yq = y[qq]; rq = rinv[qq]; }
        const int gq = c0 + q;
        invd[gq] = rq;
        yf[gq] = yq;
        PY[q] = yq;
        float* lrow = Lp + gq * (gq + 1) / 2 + c0;
#pragma unroll
        for (int qq = 0; qq < PW; ++qq) {
          if (qq != q) continue;
#pragma unroll
          for (int m = 0; m < PW; ++m) {
            const float v = (m <= qq) ? a[qq][m] : 0.f;
            LB[m * L::PLD + gq] = v;
            if (m <= qq) lrow[m] = v;
          }
        }
      }
    }
    team_sync<L::NW>(team);
    // ---- A2: rows below the panel (one thread per row)
    for (int t = c0 + PW + tid; t < b; t += L::NT) {
      float l[PW];
      float yv = ys[t];
      float* lrow = Lp + t * (t + 1) / 2 + c0;
#pragma unroll
      for (int q = 0; q < PW; ++q) {
        float v = PB[q * L::PLD + t];
#pragma unroll
        for (int m = 0; m < q; ++m) v = fmaf(-l[m], LB[m * L::PLD + c0 + q], v);
        l[q] = v * invd[c0 + q];
        LB[q * L::PLD + t] = l[q];
        lrow[q] = l[q];
        yv = fmaf(-l[q], PY[q], yv);
      }
      ys[t] = yv;
    }
    team_sync<L::NW>(team);
    // ---- B: rank-8 trailing update + publish the next raw panel
    const int cn = c0 + PW;
    if (cn < b) {
#pragma unroll
      for (int t = 0; t < L::TPW; ++t) {
        if (!T.valid[t]) continue;
        const int colend = T.coff[t] - (lane & 3) * L::SC + L::ST;  // super-tile column end
        if (colend <= cn) continue;                                 // no trailing columns
#pragma unroll
        for (int q = 0; q < PW; ++q) {
          float lr[L::SR], lc[L::SC];
          lds_vec<L::SR>(lr, LB + q * L::PLD + T.roff[t]);
          lds_vec<L::SC>(lc, LB + q * L::PLD + T.coff[t]);
#pragma unroll
          for (int i = 0; i < L::SR; ++i)
#pragma unroll
            for (int j = 0; j < L::SC; ++j) T.acc[t][i][j] = fmaf(-lr[i], lc[j], T.acc[t][i][j]);
        }
        if (T.coff[t] >= cn && T.coff[t] < cn + PW) {
#pragma unroll
          for (int m = 0; m < L::SC; ++m) {
            float* dst = PB + (T.coff[t] - cn + m) * L::PLD + T.roff[t];
#pragma unroll
            for (int i = 0; i < L::SR; ++i) dst[i] = T.acc[t][i][m];
          }
        }
      }
    }
    team_sync<L::NW>(team);
  }
  // ---- backward solve L^T d = y (warp 0, panel by panel)
  if (warp == 0) {
    for (int pp = np - 1; pp >= 0; --pp) {
      const int c0 = pp * PW;
      float z[PW], dlt[PW];
#pragma unroll
      for (int q = 0; q < PW; ++q) z[q] = (c0 + q < b) ? yf[c0 + q] : 0.f;
      // rows >= b are padding: their packed L entries outside the diagonal
      // block were never written, so they must not be read (NaN * 0 = NaN)
#pragma unroll
      for (int q = PW - 1; q >= 0; --q) {
        float v = z[q];
        const int gq = c0 + q;
#pragma unroll
        for (int m = q + 1; m < PW; ++m) {
          const int gm = c0 + m;
          if (gm < b) v = fmaf(-Lp[gm * (gm + 1) / 2 + gq], dlt[m], v);
        }
        dlt[q] = (gq < b) ? v * invd[gq] : 0.f;
      }
      if (lane < PW) {
#pragma unroll
        for (int q = 0; q < PW; ++q)
          if (q == lane && c0 + q < b) ds[c0 + q] = dlt[q];
      }
      for (int i = lane; i < c0; i += 32) {
        float v = yf[i];
#pragma unroll
        for (int q = 0; q < PW; ++q) {
          const int gq = c0 + q;
          if (gq < b) v = fmaf(-Lp[gq * (gq + 1) / 2 + i], dlt[q], v);
        }
        yf[i] = v;
      }
      __syncwarp();
    }
  }
  team_sync<L::NW>(team);
}

// Step 7 on one staged chunk: yhat[pos_k] -= x_k . d.  GL = BT/16 lanes
// cooperate on one entry, each covering 16 consecutive floats (4 LDS.128), so
// a team works on NW*32/GL entries at once.
template <int BT>
IALS_DEVI void cache_chunk(const SweepParams& p, const float* sm, int buf, int nk, int tid) {
  using L = Lay<BT>;
  constexpr int GL = BT >= 32 ? BT / 16 : 1;
  constexpr int EPW = 32 / GL;
  constexpr int SEG = BT >= 16 ? 16 : BT;
  const float* X = sm + L::OFF_X + buf * L::KC * L::XLD;
  const int* ps = reinterpret_cast<const int*>(sm + L::OFF_PS) + buf * L::KC;
  const float* ds = sm + L::OFF_D;
  const int warp = tid >> 5, lane = tid & 31;
  const int sub = lane / GL, gl = lane % GL;
  const int j0 = gl * SEG;
  for (int kb = 0; kb < nk; kb += L::NW * EPW) {
    const int k = kb + warp * EPW + sub;
    float s0 = 0.f, s1 = 0.f;
    if (k < nk && j0 < p.b) {
      const float* xr = X + k * L::XLD + j0;
      if (p.b - j0 >= SEG) {
#pragma unroll
        for (int j = 0; j < SEG; j += 4) {
          float xv[4], dv[4];
          lds_vec<4>(xv, xr + j);
          lds_vec<4>(dv, ds + j0 + j);
          s0 = fmaf(xv[0], dv[0], s0);
          s1 = fmaf(xv[1], dv[1], s1);
          s0 = fmaf(xv[2], dv[2], s0);
          s1 = fmaf(xv[3], dv[3], s1);
        }
      } else {
        for (int j = 0; j < p.b - j0; ++j) s0 = fmaf(xr[j], ds[j0 + j], s0);
      }
    }
    float sum = s0 + s1;
    if constexpr (GL > 1) sum = group_sum<GL>(sum);
    if (k < nk && gl == 0) p.cache[ps[k]] -= sum;
  }
}

template <int BT>
IALS_DEVI void cache_range(const SweepParams& p, float* sm, int ebeg, int eend, int nch_resident,
                           int tid, int team) {
  using L = Lay<BT>;
  const int n = eend - ebeg;
  const int nch = (n + L::KC - 1) / L::KC;
  if (nch <= 2 && nch == nch_resident) {
    for (int c = 0; c < nch; ++c) cache_chunk<BT>(p, sm, c & 1, min(L::KC, n - c * L::KC), tid);
    return;
  }
  if (nch > 0) stage_chunk<BT>(p, sm, 0, ebeg, min(L::KC, n), tid);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      int s = ebeg + (c + 1) * L::KC;
      stage_chunk<BT>(p, sm, (c + 1) & 1, s, min(L::KC, eend - s), tid);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    team_sync<L::NW>(team);
    cache_chunk<BT>(p, sm, c & 1, min(L::KC, eend - (ebeg + c * L::KC)), tid);
    team_sync<L::NW>(team);
  }
}

template <int BT>
IALS_DEVI void zero_stage(float* sm, int tid) {
  using L = Lay<BT>;
  float4* x = reinterpret_cast<float4*>(sm + L::OFF_X);
  for (int i = tid; i < 2 * L::KC * L::XLD / 4; i += L::NT) x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ---------------------------------------------------------------- kernels
template <int BT>
__global__ void __launch_bounds__(Lay<BT>::NT* Lay<BT>::RPC)
    k_sweep_light(SweepParams p) {
  using L = Lay<BT>;
  extern __shared__ __align__(16) float smem_all[];
  const int team = threadIdx.x / L::NT;
  const int tid = threadIdx.x - team * L::NT;
  float* sm = smem_all + team * L::FLOATS;
  zero_stage<BT>(sm, tid);
  team_sync<L::NW>(team);
  // persistent: rows are in descending-degree order, taken from a device
  // queue (greedy longest-first; the next index is fetched during the row)
  // or strided over the grid
  const int n_light = p.n_light_dev ? *p.n_light_dev : p.n_light;
  int* qslot = reinterpret_cast<int*>(sm + L::OFF_Q);
  int task = blockIdx.x * L::RPC + team;
  if (p.queue) {
    if (tid == 0) *qslot = atomicAdd(p.queue, 1);
    team_sync<L::NW>(team);
    task = *qslot;
    team_sync<L::NW>(team);
  }
  for (; task < n_light;) {
    int nxt = 0;
    if (p.queue && tid == 0) nxt = atomicAdd(p.queue, 1);
    const int row = p.light_rows[task];
    const int ebeg = p.side.ptr[row], eend = p.side.ptr[row + 1];
    Tiles<BT> T;
    T.init(tid >> 5, tid & 31);
    double gacc = 0.0;
    const int nch = accumulate_range<BT>(p, T, gacc, sm, ebeg, eend, tid, team);
    finalize_and_solve<BT>(p, T, gacc, sm, row, tid, team);
    const float* ds = sm + L::OFF_D;
    if (p.rot) {   // d~ for the back-rotation and the pass's cache kernel
      if (tid < p.b) p.drow[(size_t)row * p.b + tid] = ds[tid];
      if (eend - ebeg <= p.flat_skip_deg) cache_range<BT>(p, sm, ebeg, eend, nch, tid, team);
    } else {
      if (tid < p.b) p.own[(size_t)row * p.ldo + p.b0 + tid] -= ds[tid];
      cache_range<BT>(p, sm, ebeg, eend, nch, tid, team);
    }
    team_sync<L::NW>(team);
    if (p.queue) {
      if (tid == 0) *qslot = nxt;
      team_sync<L::NW>(team);
      task = *qslot;
      team_sync<L::NW>(team);
    } else {
      task += gridDim.x * L::RPC;
    }
  }
}

template <int BT>
__global__ void __launch_bounds__(Lay<BT>::NT* Lay<BT>::RPC)
    k_heavy_partial(SweepParams p) {
  using L = Lay<BT>;
  extern __shared__ __align__(16) float smem_all[];
  const int team = threadIdx.x / L::NT;
  const int tid = threadIdx.x - team * L::NT;
  const int sl = blockIdx.x * L::RPC + team;
  if (sl >= p.n_slices) return;
  float* sm = smem_all + team * L::FLOATS;
  zero_stage<BT>(sm, tid);
  team_sync<L::NW>(team);
  Tiles<BT> T;
  T.init(tid >> 5, tid & 31);
  double gacc = 0.0;
  accumulate_range<BT>(p, T, gacc, sm, p.slice_begin[sl], p.slice_end[sl], tid, team);
  float* hp = p.hpart + (size_t)sl * BT * BT;
#pragma unroll
  for (int t = 0; t < L::TPW; ++t) {
    if (!T.valid[t]) continue;
#pragma unroll
    for (int i = 0; i < L::SR; ++i)
#pragma unroll
      for (int j = 0; j < L::SC; ++j) hp[(T.roff[t] + i) * BT + T.coff[t] + j] = T.acc[t][i][j];
  }
  if (tid < BT) p.gpart[(size_t)sl * BT + tid] = gacc;
}

// SYM: the slice partials are the non-symmetric E of the tensor-core heavy
// partials; the Hessian is their symmetric part (E + E^T) / 2.
template <int BT, bool GUARD = false, bool SYM = false>
__global__ void __launch_bounds__(Lay<BT>::NT* Lay<BT>::RPC)
    k_heavy_solve(SweepParams p) {
  using L = Lay<BT>;
  extern __shared__ __align__(16) float smem_all[];
  const int team = threadIdx.x / L::NT;
  const int tid = threadIdx.x - team * L::NT;
  const int h = blockIdx.x * L::RPC + team;
  if (h >= p.n_heavy) return;
  float* sm = smem_all + team * L::FLOATS;
  const int row = p.heavy_rows[h];
  Tiles<BT> T;
  T.init(tid >> 5, tid & 31);
  double gacc = 0.0;
  // (heavy_reduced: k_heavy_reduce already summed the row's slices into the first slot)
  const int sl_first = p.heavy_slice0[h];
  const int sl_end = p.heavy_reduced ? min(sl_first + 1, p.heavy_slice0[h + 1]) : p.heavy_slice0[h + 1];
  for (int sl = sl_first; sl < sl_end; ++sl) {
    const float* hp = p.hpart + (size_t)sl * BT * BT;
#pragma unroll
    for (int t = 0; t < L::TPW; ++t) {
      if (!T.valid[t]) continue;
#pragma unroll
      for (int i = 0; i < L::SR; ++i) {
        float v[L::SC];
        lds_vec<L::SC>(v, hp + (T.roff[t] + i) * BT + T.coff[t]);
        if (SYM) {
#pragma unroll
          for (int j = 0; j < L::SC; ++j)
            v[j] = 0.5f * (v[j] + hp[(size_t)(T.coff[t] + j) * BT + T.roff[t] + i]);
        }
#pragma unroll
        for (int j = 0; j < L::SC; ++j) T.acc[t][i][j] += v[j];
      }
    }
    if (tid < BT) gacc += p.gpart[(size_t)sl * BT + tid];
  }
  finalize_and_solve<BT, GUARD>(p, T, gacc, sm, row, tid, team);
  const float* ds = sm + L::OFF_D;
  if (GUARD && reinterpret_cast<const int*>(sm + L::OFF_X + BT)[0]) {
    // cancelled pivot: the FP32 SIMT sweep redoes the whole row (its own
    // cache update included), so nothing of this solve is applied
    if (tid < p.b) {
      p.hdelta[(size_t)h * BT + tid] = 0.f;
      p.drow[(size_t)row * p.b + tid] = 0.f;
    }
    if (tid == 0) {
      p.redo_rows[atomicAdd(p.redo_cnt, 1)] = row;
      atomicAdd(p.redo_total, 1ull);
    }
    return;
  }
  if (tid < p.b) {
    p.own[(size_t)row * p.ldo + p.b0 + tid] -= ds[tid];
    p.hdelta[(size_t)h * BT + tid] = ds[tid];
    p.drow[(size_t)row * p.b + tid] = ds[tid];   // the entry-parallel cache pass reads d by row
  }
}

template <int BT>
__global__ void __launch_bounds__(Lay<BT>::NT* Lay<BT>::RPC)
    k_heavy_cache(SweepParams p) {
  using L = Lay<BT>;
  extern __shared__ __align__(16) float smem_all[];
  const int team = threadIdx.x / L::NT;
  const int tid = threadIdx.x - team * L::NT;
  const int sl = blockIdx.x * L::RPC + team;
  if (sl >= p.n_slices) return;
  float* sm = smem_all + team * L::FLOATS;
  const int h = p.slice_heavy[sl];
  float* ds = sm + L::OFF_D;
  if (tid < BT) ds[tid] = tid < p.b ? p.hdelta[(size_t)h * BT + tid] : 0.f;
  team_sync<L::NW>(team);
  cache_range<BT>(p, sm, p.slice_begin[sl], p.slice_end[sl], -1, tid, team);
}

}  // namespace ials
