// ials_heavy_w64.cuh -- slice partials of the long rows of a block of 33 <= b <= 64
// columns (b % 4 == 0) on the warp-level tensor path (mma.sync m16n8k8 TF32, 3xTF32;
// fragment algebra in ials_sweep_w32m.cuh): a 2048-entry slice per PAIR of warps, the 20
// lower-triangle m16n8 tiles of E = sum_k a_k x_k x_k^T split ten and ten (warp 0: rows
// 48..63 and 0..15, warp 1: rows 32..47 and 16..31), the pair's sub-rows staged by
// cp.async (16 entries a stage, row stride 72 floats = conflict-free fragment loads),
// g = sum_k rho_k x_k by thread j <-> column j (fp32 per stage, fp64 across).  Stored as
// hpart[slice][64 x 64] (the tiles below the diagonal blocks mirrored: the whole
// symmetric matrix) / gpart[slice][64] for k_heavy_solve<64> (_newton_side_pass,
// solvers.py:152-186, for the rows the schedule cuts into slices).  It replaces the
// packed tcgen05 slice kernel (k_heavy_partial_pk<2>: 991 us per item pass at the
// configs[2] shape, b = 64), which pays a CTA barrier and an MMA round trip per 8 entries.
#pragma once
#include "ials_sweep_w32m.cuh"

namespace ials {

struct WH64Lay {
  static constexpr int TEAMS = 4, NT = TEAMS * 64, KC = 16, XLD = 72;
  // per team (floats): X [2][KC][XLD], RHO [2][KC], AW [2][KC]
  static constexpr int OFF_X = 0;
  static constexpr int OFF_RHO = 2 * KC * XLD;
  static constexpr int OFF_AW = OFF_RHO + 2 * KC;
  static constexpr int TEAM_FLOATS = OFF_AW + 2 * KC;
  static constexpr int BYTES = TEAMS * TEAM_FLOATS * 4;
};
static_assert(WH64Lay::TEAM_FLOATS % 4 == 0, "16-byte team regions");

// One 16-entry stage into a warp's ten tiles.  ROLE 0: Hessian row blocks 3 (tiles
// 0..7 = column octets 0..7) and 0 (tiles 8..9 = octets 0..1); ROLE 1: row blocks 2
// (tiles 0..5) and 1 (tiles 6..9).
template <bool UNIT, int ROLE>
IALS_DEVI void w64m_stage(float (&acc)[10][4], const float* xb, const float* aw, int g, int t4) {
  constexpr int XLD = WH64Lay::XLD;
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
__global__ void __launch_bounds__(WH64Lay::NT, 2) k_heavy_partial_wm64(SweepParams p) {
  using L = WH64Lay;
  extern __shared__ __align__(16) float wh64_smem[];
  const int team = threadIdx.x >> 6, tid = threadIdx.x & 63;
  const int lane = tid & 31, role = tid >> 5;   // warp of the pair
  float* sm = wh64_smem + team * L::TEAM_FLOATS;
  float* X = sm + L::OFF_X;
  float* RHO = sm + L::OFF_RHO;
  float* AW = sm + L::OFF_AW;
  const int b = p.b;
  // staging columns >= b are never written by the gathers: they stay zero
  for (int i = tid; i < 2 * L::KC * L::XLD; i += 64) X[i] = 0.f;
  team_sync<2>(team);
  const int g = lane >> 2, t4 = lane & 3;
  const int nq = b >> 2;   // 16-byte pieces of a sub-row
  for (int sl = blockIdx.x * L::TEAMS + team; sl < p.n_slices; sl += gridDim.x * L::TEAMS) {
    const int ebeg = __ldg(p.slice_begin + sl), eend = __ldg(p.slice_end + sl);
    const int nst = (eend - ebeg + L::KC - 1) / L::KC;
    float acc[10][4];
#pragma unroll
    for (int i = 0; i < 10; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
    double gacc = 0.0;
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
      for (int i = 0; i < 4; ++i) {   // entry tid / 16 + 4 i, piece tid % 16
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
      team_sync<2>(team);   // the buffer is free for stage s + 2
    }
    // fragment (rows 16 mb + g (+ 8), columns 8 nb + 2 t4 (+ 1)) -> hpart[slice][64 x 64]
    float* hp = p.hpart + (size_t)sl * 64 * 64;
    const int mb0 = role == 0 ? 3 : 2, mb1 = role == 0 ? 0 : 1;
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      const int first = i < 2 * mb0 + 2;
      const int mb = first ? mb0 : mb1, nb = first ? i : i - (2 * mb0 + 2);
      const int r0 = 16 * mb + g, c0 = 8 * nb + 2 * t4;
      *reinterpret_cast<float2*>(hp + (size_t)r0 * 64 + c0) = make_float2(acc[i][0], acc[i][1]);
      *reinterpret_cast<float2*>(hp + (size_t)(r0 + 8) * 64 + c0) = make_float2(acc[i][2], acc[i][3]);
      if (nb < 2 * mb) {   // below the diagonal block: the mirror image
        hp[(size_t)c0 * 64 + r0] = acc[i][0];
        hp[(size_t)(c0 + 1) * 64 + r0] = acc[i][1];
        hp[(size_t)c0 * 64 + r0 + 8] = acc[i][2];
        hp[(size_t)(c0 + 1) * 64 + r0 + 8] = acc[i][3];
      }
    }
    p.gpart[(size_t)sl * 64 + tid] = gacc;
  }
}

}  // namespace ials
