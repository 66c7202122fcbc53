// ials_sweep_w64m.cuh -- light rows of a block of 33 <= b <= 64 columns (b % 4 ==
// 0) swept one row per PAIR of warps, the Hessian on the warp-level tensor path
// (mma.sync m16n8k8 TF32, 3xTF32; fragment algebra in ials_sweep_w32m.cuh).
//
// The packed tcgen05 sweep (ials_sweep_pk.cuh, 2 rows per 128-lane TMEM tile)
// pays a CTA barrier and an MMA round trip per 8 entries and factors 64 x 64
// blocks in 8-column TMEM panels; here a row's chain never leaves its two
// warps (named barriers of 64 threads), four rows per CTA, two CTAs per SM.
//
// Per row r (_newton_side_pass, solvers.py:152-186, for one row):
//   accumulate  the 20 lower-triangle m16n8 tiles of the 64 x 64 Hessian, 10 per
//               warp (warp 0: Hessian rows 48..63 and 0..15, warp 1: rows 32..47
//               and 16..31), from sub-rows staged by cp.async (16 entries a
//               stage, row stride 72 floats = conflict-free fragment loads);
//               thread j: g_j += rho_k x_kj (fp32 per stage, fp64 across)
//   assemble    H += alpha0 G_pp (CTA-shared copy) + lam_r I;  g += proj + lam_r w
//   solve       thread i <-> row i of H in registers: right-looking Cholesky, column
//               k and the right-hand side broadcast through shared memory (one
//               pair barrier a step), forward solve fused; backward solve: the upper
//               warp's 32 unknowns by shuffles, one barrier, then the lower warp's
//   write       own[r, pi] -= d, drow[r] = d (the pass's entry-parallel cache
//               kernel applies yhat -= x . d)
// A non-positive or non-finite pivot is the reference's SingularMatrixError:
// reported through the error word with its (side, row, pivot).
#pragma once
#include "ials_sweep_w32m.cuh"

namespace ials {

struct W64mLay {
  static constexpr int TEAMS = 4, NT = TEAMS * 64, KC = 16, XLD = 72, HLD = 68;
  // per team (floats): HX [64][HLD] -- the staging buffers X [2][KC][XLD] first, then H / L;
  // RHO [2][KC], AW [2][KC], BC [2][128] (column k and the right-hand side of a step),
  // DV [64] (the solved unknowns), MISC [8] (task slot, failing pivot)
  static constexpr int OFF_X = 0;
  static constexpr int OFF_RHO = 64 * HLD;
  static constexpr int OFF_AW = OFF_RHO + 2 * KC;
  static constexpr int OFF_BC = OFF_AW + 2 * KC;
  static constexpr int OFF_DV = OFF_BC + 256;
  static constexpr int OFF_MISC = OFF_DV + 64;
  static constexpr int TEAM_FLOATS = OFF_MISC + 8;
  static constexpr int OFF_TPL = TEAMS * TEAM_FLOATS;   // [64][HLD] alpha0 * slab[pi, pi]
  static constexpr int BYTES = (OFF_TPL + 64 * HLD) * 4;
};
static_assert(2 * W64mLay::KC * W64mLay::XLD <= 64 * W64mLay::HLD, "the staging buffers sit inside H");
static_assert(W64mLay::TEAM_FLOATS % 4 == 0, "16-byte team regions");
static_assert(2 * (W64mLay::BYTES + 1024) <= 228 * 1024, "two CTAs per SM");

// One 16-entry stage into a warp's ten tiles.  ROLE 0: Hessian row blocks 3 (tiles
// 0..7 = column octets 0..7) and 0 (tiles 8..9 = octets 0..1); ROLE 1: row blocks 2
// (tiles 0..5) and 1 (tiles 6..9).
template <bool UNIT, int ROLE>
IALS_DEVI void w64m_stage(float (&acc)[10][4], const float* xb, const float* aw, int g, int t4) {
  constexpr int XLD = W64mLay::XLD;
  constexpr int MB0 = ROLE == 0 ? 3 : 2, MB1 = ROLE == 0 ? 0 : 1;
  constexpr int NJ = 2 * MB0 + 2;   // column octets this warp reads (8 or 6)
#pragma unroll
  for (int c8 = 0; c8 < 16; c8 += 8) {
    const float* xc = xb + c8 * XLD;
    uint32_t hi[NJ][2], lo[NJ][2];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) tf32_split(xc[(t4 + 4 * h) * XLD + 8 * j + g], hi[j][h], lo[j][h]);
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int mb = m == 0 ? MB0 : MB1;
      const int base = m == 0 ? 0 : 2 * MB0 + 2;
      uint32_t Ah[4] = {hi[2 * mb][0], hi[2 * mb + 1][0], hi[2 * mb][1], hi[2 * mb + 1][1]};
      uint32_t Al[4] = {lo[2 * mb][0], lo[2 * mb + 1][0], lo[2 * mb][1], lo[2 * mb + 1][1]};
      if (!UNIT) {   // a_k x_k on the A side
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float a = aw[c8 + t4 + 4 * h];
          tf32_split(a * xc[(t4 + 4 * h) * XLD + 16 * mb + g], Ah[2 * h], Al[2 * h]);
          tf32_split(a * xc[(t4 + 4 * h) * XLD + 16 * mb + 8 + g], Ah[2 * h + 1], Al[2 * h + 1]);
        }
      }
#pragma unroll
      for (int nb = 0; nb < 2 * mb + 2; ++nb) {
        float(&d)[4] = acc[base + nb];
        mma_tf32(d, Al, hi[nb][0], hi[nb][1]);
        mma_tf32(d, Ah, lo[nb][0], lo[nb][1]);
        mma_tf32(d, Ah, hi[nb][0], hi[nb][1]);
      }
    }
  }
}

template <bool UNIT>
__global__ void __launch_bounds__(W64mLay::NT, 2) k_sweep_w64m(SweepParams p) {
  using L = W64mLay;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) float w64m_smem[];
  const int team = threadIdx.x >> 6, tid = threadIdx.x & 63;
  const int lane = tid & 31, role = tid >> 5;   // warp of the pair
  float* sm = w64m_smem + team * L::TEAM_FLOATS;
  float* X = sm + L::OFF_X;
  float* RHO = sm + L::OFF_RHO;
  float* AW = sm + L::OFF_AW;
  float* BC = sm + L::OFF_BC;
  float* DV = sm + L::OFF_DV;
  int* MISC = reinterpret_cast<int*>(sm + L::OFF_MISC);
  float* TPL = w64m_smem + L::OFF_TPL;
  const int b = p.b;
  for (int i = threadIdx.x; i < 64 * 64; i += L::NT) {
    const int r = i >> 6, c = i & 63;
    TPL[r * L::HLD + c] = (r < b && c < b) ? p.alpha0 * __ldg(p.slab + (size_t)(p.b0 + r) * b + c) : 0.f;
  }
  // staging columns >= b are never written by the gathers: keep them zero
  for (int i = tid; i < 2 * L::KC * L::XLD; i += 64) X[i] = 0.f;
  __syncthreads();

  const int* lrows = p.light_rows;
  int n_light = p.n_light;
  if (p.chunk_tot) {   // ials_epoch_host's chunked first user pass: this launch's slice
    int off = 0;
    for (int k = 0; k < p.chunk; ++k) off += p.chunk_tot[k];
    lrows += off;
    n_light = p.chunk_tot[p.chunk];
  }
  const int g = lane >> 2, t4 = lane & 3;
  const int nq = b >> 2;   // 16-byte pieces of a sub-row
  if (tid == 0) MISC[0] = atomicAdd(p.queue, 1);
  team_sync<2>(team);
  int task = MISC[0];
  while (task < n_light) {
    team_sync<2>(team);   // every thread has read the slot
    if (tid == 0) {
      MISC[0] = atomicAdd(p.queue, 1);   // the next row, fetched during this one
      MISC[1] = 64;                       // first failing pivot (none)
    }
    const int row = __ldg(lrows + task);
    const int ebeg = __ldg(p.side.ptr + row), eend = __ldg(p.side.ptr + row + 1);
    const float lam = __ldg(p.side.lam + row);
    const int nst = (eend - ebeg + L::KC - 1) / L::KC;
    float acc[10][4];
#pragma unroll
    for (int i = 0; i < 10; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
    double gacc = 0.0;
    // stage s -> buffer s & 1: threads < KC fetch their entry's cache value (kept in a
    // register until the stage is consumed) and weight / label; every thread issues 4 of
    // the stage's 256 16-byte gathers (entry tid / 16 + 4 i, piece tid % 16)
    float cval = 0.f, wval = 1.f, yval = 1.f;
    auto issue = [&](int s) {
      const int e0 = ebeg + s * L::KC, nk = min(L::KC, eend - e0), buf = s & 1;
      cval = 0.f; wval = 1.f; yval = 1.f;
      if (tid < nk) {
        const int e = e0 + tid;
        const int pos = p.side.pos ? __ldg(p.side.pos + e) : e;
        IALS_CHECK(pos >= 0 && pos < p.side.nnz);
        cval = p.cache[pos];
        if (!UNIT) {
          if (p.side.weights) wval = __ldg(p.side.weights + e);
          if (p.side.labels) yval = __ldg(p.side.labels + e);
        }
      }
      const int q = tid & 15;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = (tid >> 4) + 4 * i;
        float* dst = X + (buf * L::KC + e) * L::XLD + 4 * q;
        if (e < nk) {
          const int ce = __ldg(p.side.cols + e0 + e);
          IALS_CHECK(ce >= 0 && ce < p.side.n_fixed);
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
      if (tid < L::KC) {
        const float rho = UNIT ? cval - 1.f : wval * (cval - yval);
        const bool in = ebeg + s * L::KC + tid < eend;
        RHO[buf * L::KC + tid] = in ? rho : 0.f;
        if (!UNIT) AW[buf * L::KC + tid] = in ? wval : 0.f;
      }
      if (s + 1 < nst) {
        issue(s + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      team_sync<2>(team);   // the stage's sub-rows and residuals are visible to both warps
      const float* xb = X + buf * L::KC * L::XLD;
      if (role == 0) w64m_stage<UNIT, 0>(acc, xb, AW + buf * L::KC, g, t4);
      else w64m_stage<UNIT, 1>(acc, xb, AW + buf * L::KC, g, t4);
      float gs = 0.f;
#pragma unroll
      for (int k = 0; k < L::KC; k += 4) {
        const float4 rh = *reinterpret_cast<const float4*>(RHO + buf * L::KC + k);
        gs = fmaf(rh.x, xb[k * L::XLD + tid], gs);
        gs = fmaf(rh.y, xb[(k + 1) * L::XLD + tid], gs);
        gs = fmaf(rh.z, xb[(k + 2) * L::XLD + tid], gs);
        gs = fmaf(rh.w, xb[(k + 3) * L::XLD + tid], gs);
      }
      gacc += (double)gs;
      team_sync<2>(team);   // the buffer is free for stage s + 2 (and, after the last, for H)
    }
    // ---- assemble H: the lower-triangle tiles (the factorisation reads row i's
    // columns 0..i only; what the staging left above them is never used)
    float* HS = X;   // 64 x HLD
    {
      const int mb0 = role == 0 ? 3 : 2, mb1 = role == 0 ? 0 : 1;
#pragma unroll
      for (int i = 0; i < 10; ++i) {
        const int first = i < 2 * mb0 + 2;
        const int mb = first ? mb0 : mb1, nb = first ? i : i - (2 * mb0 + 2);
        float* dst = HS + (16 * mb + g) * L::HLD + 8 * nb + 2 * t4;
        *reinterpret_cast<float2*>(dst) = make_float2(acc[i][0], acc[i][1]);
        *reinterpret_cast<float2*>(dst + 8 * L::HLD) = make_float2(acc[i][2], acc[i][3]);
      }
    }
    team_sync<2>(team);
    // thread i <-> row i: H + alpha0 G_pp + lam_r I (identity on the padding rows)
    float a[64];
#pragma unroll
    for (int j4 = 0; j4 < 16; ++j4) {
      const float4 h = reinterpret_cast<const float4*>(HS + tid * L::HLD)[j4];
      const float4 gg = reinterpret_cast<const float4*>(TPL + tid * L::HLD)[j4];
      a[4 * j4] = h.x + gg.x; a[4 * j4 + 1] = h.y + gg.y; a[4 * j4 + 2] = h.z + gg.z; a[4 * j4 + 3] = h.w + gg.w;
    }
    const float dadd = (tid < b) ? lam : 1.f;
    float ow = 0.f, t = 0.f;
    if (tid < b) {
      ow = p.own[(size_t)row * p.ldo + p.b0 + tid];
      t = (float)(gacc + (double)__ldg(p.proj + (size_t)row * b + tid) + (double)lam * (double)ow);
    }
    // ---- Cholesky (right-looking) with the forward solve fused.  Step k: every thread
    // posts its a_ik (thread k: the pivot, with the diagonal shift) and right-hand side;
    // l_ik = a_ik / sqrt(pivot); a_ij -= l_ik l_jk for k < j <= i.
    float rown = 1.f;
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      float* bc = BC + (k & 1) * 128;
      const float aik = (tid == k) ? a[k] + dadd : a[k];
      if (k < 32 || role == 1) {   // (rows above k are finished: the lower warp only keeps the barrier)
        bc[tid] = aik;
        bc[64 + tid] = t;
      }
      team_sync<2>(team);
      if (k < 32 || role == 1) {
        const float dk = bc[k];
        float r;   // MUFU.RSQ; a non-positive / non-finite pivot leaves a NaN, infinite or zero 1/sqrt
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(dk));
        if (tid == k) rown = r;
        const float lik = aik * r;
        a[k] = lik;
        const float yk = bc[64 + k] * r;
        if (tid == k) t = yk;
        else if (tid > k) t = fmaf(-lik, yk, t);
        const float m = -lik * r;   // a_ij -= l_ik (a_jk r)
#pragma unroll
        for (int j4 = ((k + 1) >> 2) << 2; j4 < 64; j4 += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(bc + j4);
          if (j4 > k) a[j4] = fmaf(m, l4.x, a[j4]);
          if (j4 + 1 > k) a[j4 + 1] = fmaf(m, l4.y, a[j4 + 1]);
          if (j4 + 2 > k) a[j4 + 2] = fmaf(m, l4.z, a[j4 + 2]);
          if (j4 + 3 > k) a[j4 + 3] = fmaf(m, l4.w, a[j4 + 3]);
        }
      }
    }
    // the first failing pivot, if any: thread k kept 1/sqrt(pivot k)
    if (!(rown > 0.f && rown < 3.0e38f)) atomicMin(&MISC[1], tid);
    // ---- backward solve L^T d = y: L's rows to shared memory, the upper warp's
    // unknowns by shuffles, then the lower warp's
    team_sync<2>(team);   // (every thread is past its last read of the staging / H region)
#pragma unroll
    for (int j4 = 0; j4 < 16; ++j4)
      reinterpret_cast<float4*>(HS + tid * L::HLD)[j4] = make_float4(a[4 * j4], a[4 * j4 + 1], a[4 * j4 + 2], a[4 * j4 + 3]);
    team_sync<2>(team);
    float dj = 0.f;
    if (role == 1) {
#pragma unroll
      for (int k = 31; k >= 0; --k) {   // unknown 32 + k
        const float dk = __shfl_sync(FULL, t * rown, k);
        if (lane == k) dj = dk;
        if (lane < k) t = fmaf(-HS[(32 + k) * L::HLD + 32 + lane], dk, t);
      }
      DV[32 + lane] = dj;
    }
    team_sync<2>(team);
    if (role == 0) {
#pragma unroll 8
      for (int k = 32; k < 64; ++k) t = fmaf(-HS[k * L::HLD + lane], DV[k], t);
#pragma unroll
      for (int k = 31; k >= 0; --k) {
        const float dk = __shfl_sync(FULL, t * rown, k);
        if (lane == k) dj = dk;
        if (lane < k) t = fmaf(-HS[k * L::HLD + lane], dk, t);
      }
    }
    const int bad = MISC[1];
    if (bad < b) {
      if (tid == 0) report_singular(p.err, p.side_id, row, bad);
      if (tid < b) p.drow[(size_t)row * b + tid] = 0.f;
    } else if (tid < b) {
      p.own[(size_t)row * p.ldo + p.b0 + tid] = ow - dj;
      p.drow[(size_t)row * b + tid] = dj;
    }
    team_sync<2>(team);   // H (the staging buffers) is rewritten by the next row
    // the staging columns >= b must read as zeros again (H overwrote them; at
    // b = 64 every element read is written by its stage's gathers or zero fill)
    if (b < 64)
      for (int i = tid; i < 2 * L::KC * L::XLD; i += 64) X[i] = 0.f;
    task = MISC[0];
  }
}

}  // namespace ials
