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
};

template <int BT>
struct Cfg;
// ST: warp super-tile edge; SR x SC: per-lane tile; NW: warps per row team;
// RPC: row teams per CTA; KC: entries per staged chunk.
template <> struct Cfg<8>   { static constexpr int ST = 8,  SR = 1, SC = 2, NW = 1,  RPC = 4, KC = 32; };
template <> struct Cfg<16>  { static constexpr int ST = 16, SR = 2, SC = 4, NW = 1,  RPC = 4, KC = 32; };
template <> struct Cfg<32>  { static constexpr int ST = 32, SR = 4, SC = 8, NW = 1,  RPC = 4, KC = 32; };
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
  static constexpr int OFF_CB = OFF_L + ((LP + 3) / 4) * 4;
  static constexpr int OFF_Y = OFF_CB + 2 * BT;
  static constexpr int OFF_YF = OFF_Y + BT;
  static constexpr int OFF_ID = OFF_YF + BT;
  static constexpr int OFF_D = OFF_ID + BT;
  static constexpr int FLOATS = OFF_D + BT;
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
    const int bv = p.b >> 2;
    for (int i = tid; i < nk * bv; i += L::NT) {
      int k = i / bv, v = i - k * bv;
      int col = __ldg(p.side.cols + ebeg + k);
      cp_async16(X + k * L::XLD + 4 * v, p.fixed + (size_t)col * p.ldf + p.b0 + 4 * v);
    }
  } else {
    for (int i = tid; i < nk * p.b; i += L::NT) {
      int k = i / p.b, v = i - k * p.b;
      int col = __ldg(p.side.cols + ebeg + k);
      cp_async4(X + k * L::XLD + v, p.fixed + (size_t)col * p.ldf + p.b0 + v);
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
                                int tid) {
  using L = Lay<BT>;
  const float* X = sm + L::OFF_X + buf * L::KC * L::XLD;
  const float* aw = sm + L::OFF_AW + buf * L::KC;
  const float* rh = sm + L::OFF_RH + buf * L::KC;
  const int nk4 = (nk + 3) & ~3;  // padded entries have a = 0 and finite stale rows
  // Two-level (blocked) summation: each chunk is summed into a zeroed local
  // tile that is then added to the running Hessian, as a blocked GEMM would;
  // a long row's sum is then ~sqrt(KC) times more accurate than one running
  // fp32 sum (matters for the ill-conditioned first epochs of heavy rows).
  constexpr bool kBlocked = L::TPW == 1;
  float loc[kBlocked ? L::SR : 1][kBlocked ? L::SC : 1];
  if constexpr (kBlocked) {
#pragma unroll
    for (int i = 0; i < L::SR; ++i)
#pragma unroll
      for (int j = 0; j < L::SC; ++j) loc[i][j] = 0.f;
  }
#pragma unroll 2
  for (int k = 0; k < nk4; ++k) {
    const float a = aw[k];
    const float* xr = X + k * L::XLD;
#pragma unroll
    for (int t = 0; t < L::TPW; ++t) {
      if (!T.valid[t]) continue;
      float rv[L::SR], cv[L::SC];
      lds_vec<L::SR>(rv, xr + T.roff[t]);
      lds_vec<L::SC>(cv, xr + T.coff[t]);
#pragma unroll
      for (int i = 0; i < L::SR; ++i) {
        const float ra = rv[i] * a;
#pragma unroll
        for (int j = 0; j < L::SC; ++j) {
          if constexpr (kBlocked)
            loc[i][j] = fmaf(ra, cv[j], loc[i][j]);
          else
            T.acc[t][i][j] = fmaf(ra, cv[j], T.acc[t][i][j]);
        }
      }
    }
  }
  if constexpr (kBlocked) {
#pragma unroll
    for (int i = 0; i < L::SR; ++i)
#pragma unroll
      for (int j = 0; j < L::SC; ++j) T.acc[0][i][j] += loc[i][j];
  }
  if (tid < BT) {
    // fp64: g = sum rho_k h_k + alpha0 w G + lam w cancels by orders of magnitude
    // on long rows, so the sum is formed in double and rounded once.
    double g = gacc;
    for (int k = 0; k < nk; ++k) g = fma((double)rh[k], (double)X[k * L::XLD + tid], g);
    gacc = g;
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
    accumulate_chunk<BT>(T, gacc, sm, c & 1, min(L::KC, eend - s), tid);
    team_sync<L::NW>(team);
  }
  return nch;
}

// Steps 3-5: add the alpha0 slab / lambda terms, factor, solve; leaves the
// step d in sm[OFF_D .. +b).  Returns false (after reporting) on a bad pivot.
template <int BT>
IALS_DEVI void finalize_and_solve(const SweepParams& p, Tiles<BT>& T, double gacc, float* sm,
                                  int row, int tid, int team) {
  using L = Lay<BT>;
  const int warp = tid >> 5, lane = tid & 31;
  const int b = p.b;
  float* Lp = sm + L::OFF_L;
  float* cb = sm + L::OFF_CB;
  float* ys = sm + L::OFF_Y;
  float* yf = sm + L::OFF_YF;
  float* invd = sm + L::OFF_ID;
  float* ds = sm + L::OFF_D;
  const float lam = p.side.lam[row];
  if (tid < BT) {
    double g = 0.0;
    if (tid < b)
      g = gacc + (double)p.proj[(size_t)row * b + tid] +
          (double)lam * (double)p.own[(size_t)row * p.ldo + p.b0 + tid];
    ys[tid] = (float)g;
  }
  const float a0 = p.alpha0;
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
          if (gi == gj) v += lam;
        } else {
          v = (gi == gj) ? 1.f : 0.f;
        }
        T.acc[t][i][j] = v;
      }
    }
    // publish column 0
    if (T.coff[t] == 0) {
#pragma unroll
      for (int i = 0; i < L::SR; ++i) cb[T.roff[t] + i] = T.acc[t][i][0];
    }
  }
  team_sync<L::NW>(team);
  // Right-looking Cholesky, one column per step; forward solve fused.
  for (int j = 0; j < b; ++j) {
    const float* cj = cb + (j & 1) * BT;
    float piv = cj[j];
    if (!(piv > 0.f) || !(piv < 3.0e38f)) {
      if (tid == 0) report_singular(p.err, p.side_id, row, j);
      piv = 1.f;
    }
    const float rp = 1.0f / sqrtf(piv);
    const float yj = ys[j] * rp;
    if (tid < b) {
      if (tid > j) {
        const float l = cj[tid] * rp;
        Lp[tid * (tid + 1) / 2 + j] = l;
        ys[tid] -= l * yj;
      } else if (tid == j) {
        Lp[j * (j + 1) / 2 + j] = piv * rp;
        invd[j] = rp;
        yf[j] = yj;
      }
    }
    float* cn = cb + ((j + 1) & 1) * BT;
#pragma unroll
    for (int t = 0; t < L::TPW; ++t) {
      if (!T.valid[t]) continue;
      if (T.roff[t] - (lane >> 2) * L::SR + L::ST <= j + 1) continue;  // super-tile done
      float li[L::SR], lk[L::SC];
#pragma unroll
      for (int i = 0; i < L::SR; ++i) {
        const int gi = T.roff[t] + i;
        li[i] = (gi > j) ? cj[gi] * rp : 0.f;
      }
#pragma unroll
      for (int k = 0; k < L::SC; ++k) {
        const int gk = T.coff[t] + k;
        lk[k] = (gk > j) ? cj[gk] * rp : 0.f;
      }
#pragma unroll
      for (int i = 0; i < L::SR; ++i)
#pragma unroll
        for (int k = 0; k < L::SC; ++k) T.acc[t][i][k] = fmaf(-li[i], lk[k], T.acc[t][i][k]);
      // publish column j + 1 (owner lanes)
      const int jn = j + 1 - T.coff[t];
      if (jn >= 0 && jn < L::SC) {
#pragma unroll
        for (int i = 0; i < L::SR; ++i) {
#pragma unroll
          for (int k = 0; k < L::SC; ++k)
            if (k == jn) cn[T.roff[t] + i] = T.acc[t][i][k];
        }
      }
    }
    team_sync<L::NW>(team);
  }
  // Backward solve L^T d = y by warp 0 of the team.
  if (warp == 0) {
    float yv[L::MB];
#pragma unroll
    for (int m = 0; m < L::MB; ++m) {
      const int i = lane + 32 * m;
      yv[m] = (i < b) ? yf[i] : 0.f;
    }
#pragma unroll
    for (int mo = L::MB - 1; mo >= 0; --mo) {
      const int jtop = min(31, b - 1 - 32 * mo);
      for (int jj = jtop; jj >= 0; --jj) {
        const int j = mo * 32 + jj;
        const float dj = __shfl_sync(0xffffffffu, yv[mo], jj) * invd[j];
        if (lane == jj) yv[mo] = dj;
        const float* Lrow = Lp + j * (j + 1) / 2;
#pragma unroll
        for (int mm = 0; mm <= mo; ++mm) {
          const int i = lane + 32 * mm;
          if (i < j) yv[mm] = fmaf(-Lrow[i], dj, yv[mm]);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < L::MB; ++m) {
      const int i = lane + 32 * m;
      if (i < b) ds[i] = yv[m];
    }
  }
  team_sync<L::NW>(team);
}

// Step 7 on one staged chunk: yhat[pos_k] -= x_k . d
template <int BT>
IALS_DEVI void cache_chunk(const SweepParams& p, const float* sm, int buf, int nk, int tid) {
  using L = Lay<BT>;
  constexpr int GL = BT < 32 ? BT : 32;
  constexpr int EPW = 32 / GL;
  const float* X = sm + L::OFF_X + buf * L::KC * L::XLD;
  const int* ps = reinterpret_cast<const int*>(sm + L::OFF_PS) + buf * L::KC;
  const float* ds = sm + L::OFF_D;
  const int warp = tid >> 5, lane = tid & 31;
  const int sub = lane / GL, gl = lane % GL;
  for (int kb = 0; kb < nk; kb += L::NW * EPW) {
    const int k = kb + warp * EPW + sub;
    float s = 0.f;
    if (k < nk) {
      for (int j = gl; j < p.b; j += GL) s = fmaf(X[k * L::XLD + j], ds[j], s);
    }
    s = group_sum<GL>(s);
    if (k < nk && gl == 0) p.cache[ps[k]] -= s;
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
  const int task = blockIdx.x * L::RPC + team;
  if (task >= p.n_light) return;
  float* sm = smem_all + team * L::FLOATS;
  const int row = p.light_rows[task];
  const int ebeg = p.side.ptr[row], eend = p.side.ptr[row + 1];
  zero_stage<BT>(sm, tid);
  team_sync<L::NW>(team);
  Tiles<BT> T;
  T.init(tid >> 5, tid & 31);
  double gacc = 0.0;
  const int nch = accumulate_range<BT>(p, T, gacc, sm, ebeg, eend, tid, team);
  finalize_and_solve<BT>(p, T, gacc, sm, row, tid, team);
  const float* ds = sm + L::OFF_D;
  if (tid < p.b) p.own[(size_t)row * p.ldo + p.b0 + tid] -= ds[tid];
  cache_range<BT>(p, sm, ebeg, eend, nch, tid, team);
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

template <int BT>
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
  for (int sl = p.heavy_slice0[h]; sl < p.heavy_slice0[h + 1]; ++sl) {
    const float* hp = p.hpart + (size_t)sl * BT * BT;
#pragma unroll
    for (int t = 0; t < L::TPW; ++t) {
      if (!T.valid[t]) continue;
#pragma unroll
      for (int i = 0; i < L::SR; ++i) {
        float v[L::SC];
        lds_vec<L::SC>(v, hp + (T.roff[t] + i) * BT + T.coff[t]);
#pragma unroll
        for (int j = 0; j < L::SC; ++j) T.acc[t][i][j] += v[j];
      }
    }
    if (tid < BT) gacc += p.gpart[(size_t)sl * BT + tid];
  }
  finalize_and_solve<BT>(p, T, gacc, sm, row, tid, team);
  const float* ds = sm + L::OFF_D;
  if (tid < p.b) {
    p.own[(size_t)row * p.ldo + p.b0 + tid] -= ds[tid];
    p.hdelta[(size_t)h * BT + tid] = ds[tid];
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
