// ials_heavy_w.cuh -- slice partials of the long rows of a narrow block
// (b <= 32), FP32 SIMT in the register layout of the warp-per-row sweeps
// (ials_sweep_w32.cuh / ials_sweep_w16.cuh): a slice of a heavy row per warp
// (NB = 32) or per half-warp (NB = 16) accumulates
//   E = sum_k a_k x_k x_k^T (NB x NB, 4 x NB/4 register tiles),  g = sum_k rho_k x_k
// over its entries through a private cp.async double buffer and stores them as
// hpart[slice][bt x bt] / gpart[slice][bt] (bt = the width's block tile: 8, 16
// or 32); k_heavy_solve<bt> sums a row's slices in their fixed order and
// solves (_newton_side_pass, solvers.py:152-186, for the rows the schedule
// cuts into slices).  Slices have one length (the last of a row is shorter), so
// they are dealt round-robin, no queue.
#pragma once
#include "ials_sweep_w32m.cuh"

namespace ials {

template <int NB>
struct WHLay {
  static constexpr int NW = 8, NT = NW * 32, KC = 16, XLD = NB + 4, G = 32 / NB;   // G slices per warp
  // per slice group (floats): X [2][KC][XLD], RHO [2][KC], AW [2][KC]
  static constexpr int OFF_X = 0;
  static constexpr int OFF_RHO = OFF_X + 2 * KC * XLD;
  static constexpr int OFF_AW = OFF_RHO + 2 * KC;
  // (NB = 16: a group's region is 16 mod 32 floats long, so the two halves'
  // 4-byte accesses to the same offset fall on disjoint banks)
  static constexpr int GROUP_FLOATS = OFF_AW + 2 * KC + (NB == 16 ? 16 : 0);
  static constexpr int BYTES = NW * G * GROUP_FLOATS * 4;
};
static_assert(WHLay<16>::GROUP_FLOATS % 32 == 16, "bank offset of the second half");

template <int NB, bool UNIT>
__global__ void __launch_bounds__(WHLay<NB>::NT, NB == 16 ? 4 : 3) k_heavy_partial_w(SweepParams p, int bt) {
  using L = WHLay<NB>;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int TC = NB / 4;    // tile columns per lane (tile rows: 4)
  constexpr int NQL = NB / 4;   // 16-byte pieces of a padded sub-row = lanes sharing an entry's gather
  extern __shared__ __align__(16) float hw_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / NB, gl = lane % NB;
  float* sm = hw_smem + (warp * L::G + grp) * L::GROUP_FLOATS;
  float* X = sm + L::OFF_X;
  float* RHO = sm + L::OFF_RHO;
  float* AW = sm + L::OFF_AW;
  const int b = p.b;
  // staging columns >= b are never written by the gathers: they stay zero
  for (int i = gl; i < 2 * L::KC * L::XLD; i += NB) X[i] = 0.f;
  __syncwarp();
  const int ty = gl >> 2, tx = gl & 3;
  const int nq = b >> 2;
  for (int base = (blockIdx.x * L::NW + warp) * L::G; base < p.n_slices; base += gridDim.x * L::NW * L::G) {
    const int sl = base + grp;
    const bool live = sl < p.n_slices;
    const int ebeg = live ? __ldg(p.slice_begin + sl) : 0;
    const int eend = live ? __ldg(p.slice_end + sl) : 0;
    int nst = (eend - ebeg + L::KC - 1) / L::KC;
    if (L::G > 1) nst = max(nst, __shfl_xor_sync(FULL, nst, 16));
    float acc[4][TC];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < TC; ++c) acc[r][c] = 0.f;
    double gacc = 0.0;
    float cval = 0.f, wval = 1.f, yval = 1.f;
    int col_next = (gl < L::KC && gl < eend - ebeg) ? __ldg(p.side.cols + ebeg + gl) : 0;
    auto issue = [&](int s) {
      const int e0 = ebeg + s * L::KC, nk = min(L::KC, eend - e0), buf = s & 1;
      const int col = col_next;
      col_next = (gl < L::KC && e0 + L::KC + gl < eend) ? __ldg(p.side.cols + e0 + L::KC + gl) : 0;
      cval = 0.f; wval = 1.f; yval = 1.f;
      if (gl < nk) {   // (nk <= KC <= NB)
        const int e = e0 + gl;
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
      for (int i = 0; i < 4; ++i) {   // NB lanes cover NB / NQL = 4 entries a step
        const int e = gl / NQL + 4 * i, q = gl % NQL;
        const int ce = __shfl_sync(FULL, col, e, NB);
        float* dst = X + (buf * L::KC + e) * L::XLD + 4 * q;
        if (e < nk) {
          if (q < nq) cp_async16(dst, p.fixed + (size_t)ce * p.ldf + p.fb0 + 4 * q);
        } else if (q < nq) {
          *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      cp_async_commit();
    };
    if (nst > 0) issue(0);
    for (int s = 0; s < nst; ++s) {
      const int buf = s & 1;
      if (gl < L::KC) {
        const float rho = UNIT ? cval - 1.f : wval * (cval - yval);
        const bool in = ebeg + s * L::KC + gl < eend;
        RHO[buf * L::KC + gl] = in ? rho : 0.f;
        if (!UNIT) AW[buf * L::KC + gl] = in ? wval : 0.f;
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
#pragma unroll 4
      for (int k = 0; k < L::KC; ++k) {
        const float* xr = xb + k * L::XLD;
        const float4 r4 = *reinterpret_cast<const float4*>(xr + 4 * ty);
        float rv[4] = {r4.x, r4.y, r4.z, r4.w};
        float cv[TC];
#pragma unroll
        for (int c4 = 0; c4 < TC; c4 += 4) {
          const float4 c = *reinterpret_cast<const float4*>(xr + TC * tx + c4);
          cv[c4] = c.x; cv[c4 + 1] = c.y; cv[c4 + 2] = c.z; cv[c4 + 3] = c.w;
        }
        if (!UNIT) {
          const float a = AW[buf * L::KC + k];
#pragma unroll
          for (int r = 0; r < 4; ++r) rv[r] *= a;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < TC; ++c) acc[r][c] = fmaf(rv[r], cv[c], acc[r][c]);
        gs = fmaf(RHO[buf * L::KC + k], xr[gl], gs);
      }
      gacc += (double)gs;
      __syncwarp();   // the buffer is free for stage s + 2
    }
    if (live) {
      float* hp = p.hpart + (size_t)sl * bt * bt;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int rr = 4 * ty + r;
#pragma unroll
        for (int c4 = 0; c4 < TC; c4 += 4) {
          const int cc = TC * tx + c4;
          if (rr < bt && cc < bt)
            *reinterpret_cast<float4*>(hp + (size_t)rr * bt + cc) =
                make_float4(acc[r][c4], acc[r][c4 + 1], acc[r][c4 + 2], acc[r][c4 + 3]);
        }
      }
      if (gl < bt) p.gpart[(size_t)sl * bt + gl] = gacc;
    }
  }
}

// The same slices with E on the warp-level tensor path (3xTF32 m16n8k8 tiles,
// ials_sweep_w32m.cuh): NB = 32 a slice per warp, the six lower-triangle tiles
// (the two tiles below the diagonal blocks are mirrored into the upper right
// block on the way out: the stored partial is the whole symmetric matrix);
// NB = 16 two slices per warp, taking turns on the tensor path.
template <int NB>
struct WHmLay {
  static constexpr int NW = 8, NT = NW * 32, KC = 16, XLD = NB == 32 ? 40 : 24, G = 32 / NB;
  static constexpr int OFF_X = 0;
  static constexpr int OFF_RHO = OFF_X + 2 * KC * XLD;
  static constexpr int OFF_AW = OFF_RHO + 2 * KC;
  static constexpr int GROUP_FLOATS = OFF_AW + 2 * KC + (NB == 16 ? 16 : 0);
  static constexpr int BYTES = NW * G * GROUP_FLOATS * 4;
};
static_assert(WHmLay<16>::GROUP_FLOATS % 32 == 16, "bank offset of the second half");

template <int NB, bool UNIT>
__global__ void __launch_bounds__(WHmLay<NB>::NT, NB == 16 ? 4 : 3) k_heavy_partial_wm(SweepParams p, int bt) {
  using L = WHmLay<NB>;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NQL = NB / 4;
  constexpr int NACC = NB == 32 ? 6 : 4;   // NB = 16: [slice of the pair][column octet]
  extern __shared__ __align__(16) float hwm_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / NB, gl = lane % NB;
  float* wbase = hwm_smem + (warp * L::G) * L::GROUP_FLOATS;   // the warp's first group
  float* sm = wbase + grp * L::GROUP_FLOATS;
  float* X = sm + L::OFF_X;
  float* RHO = sm + L::OFF_RHO;
  float* AW = sm + L::OFF_AW;
  const int b = p.b;
  for (int i = gl; i < 2 * L::KC * L::XLD; i += NB) X[i] = 0.f;
  __syncwarp();
  const int g = lane >> 2, t4 = lane & 3;
  const int nq = b >> 2;
  for (int base = (blockIdx.x * L::NW + warp) * L::G; base < p.n_slices; base += gridDim.x * L::NW * L::G) {
    const int sl = base + grp;
    const bool live = sl < p.n_slices;
    const int ebeg = live ? __ldg(p.slice_begin + sl) : 0;
    const int eend = live ? __ldg(p.slice_end + sl) : 0;
    int nst = (eend - ebeg + L::KC - 1) / L::KC;
    if (L::G > 1) nst = max(nst, __shfl_xor_sync(FULL, nst, 16));
    float acc[NACC][4];
#pragma unroll
    for (int i = 0; i < NACC; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
    double gacc = 0.0;
    float cval = 0.f, wval = 1.f, yval = 1.f;
    int col_next = (gl < L::KC && gl < eend - ebeg) ? __ldg(p.side.cols + ebeg + gl) : 0;
    auto issue = [&](int s) {
      const int e0 = ebeg + s * L::KC, nk = min(L::KC, eend - e0), buf = s & 1;
      const int col = col_next;
      col_next = (gl < L::KC && e0 + L::KC + gl < eend) ? __ldg(p.side.cols + e0 + L::KC + gl) : 0;
      cval = 0.f; wval = 1.f; yval = 1.f;
      if (gl < nk) {
        const int e = e0 + gl;
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
        const int e = gl / NQL + 4 * i, q = gl % NQL;
        const int ce = __shfl_sync(FULL, col, e, NB);
        float* dst = X + (buf * L::KC + e) * L::XLD + 4 * q;
        if (e < nk) {
          if (q < nq) cp_async16(dst, p.fixed + (size_t)ce * p.ldf + p.fb0 + 4 * q);
        } else if (q < nq) {
          *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      cp_async_commit();
    };
    if (nst > 0) issue(0);
    for (int s = 0; s < nst; ++s) {
      const int buf = s & 1;
      if (gl < L::KC) {
        const float rho = UNIT ? cval - 1.f : wval * (cval - yval);
        const bool in = ebeg + s * L::KC + gl < eend;
        RHO[buf * L::KC + gl] = in ? rho : 0.f;
        if (!UNIT) AW[buf * L::KC + gl] = in ? wval : 0.f;
      }
      if (s + 1 < nst) {
        issue(s + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      const float* xb = X + buf * L::KC * L::XLD;
      if constexpr (NB == 32) {
        w32m_stage<UNIT>(acc, xb, AW + buf * L::KC, g, t4);
      } else {
        const float* x0 = wbase + L::OFF_X + buf * L::KC * L::XLD;
        const float* a0 = wbase + L::OFF_AW + buf * L::KC;
        w16m_stage<UNIT>(reinterpret_cast<float(&)[2][4]>(acc[0]), x0, a0, g, t4);
        w16m_stage<UNIT>(reinterpret_cast<float(&)[2][4]>(acc[2]), x0 + L::GROUP_FLOATS, a0 + L::GROUP_FLOATS, g, t4);
      }
      float gs = 0.f;
#pragma unroll
      for (int k = 0; k < L::KC; k += 4) {
        const float4 rh = *reinterpret_cast<const float4*>(RHO + buf * L::KC + k);
        gs = fmaf(rh.x, xb[k * L::XLD + gl], gs);
        gs = fmaf(rh.y, xb[(k + 1) * L::XLD + gl], gs);
        gs = fmaf(rh.z, xb[(k + 2) * L::XLD + gl], gs);
        gs = fmaf(rh.w, xb[(k + 3) * L::XLD + gl], gs);
      }
      gacc += (double)gs;
      __syncwarp();   // the buffer is free for stage s + 2
    }
    // fragment (row r0 = .. + g (+ 8), columns c0 = .. + 2 t4 (+ 1)) -> hpart[slice][bt x bt]
    if constexpr (NB == 32) {
      if (live) {
        float* hp = p.hpart + (size_t)sl * bt * bt;
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
          for (int nb = 0; nb < 2 + 2 * mb; ++nb) {
            const float(&d)[4] = acc[2 * mb + nb];
            const int r0 = 16 * mb + g, c0 = 8 * nb + 2 * t4;
            if (r0 < bt && c0 < bt) *reinterpret_cast<float2*>(hp + (size_t)r0 * bt + c0) = make_float2(d[0], d[1]);
            if (r0 + 8 < bt && c0 < bt) *reinterpret_cast<float2*>(hp + (size_t)(r0 + 8) * bt + c0) = make_float2(d[2], d[3]);
            if (mb == 1 && nb < 2) {   // below the diagonal blocks: the mirror image
              if (r0 < bt) { hp[(size_t)c0 * bt + r0] = d[0]; hp[(size_t)(c0 + 1) * bt + r0] = d[1]; }
              if (r0 + 8 < bt) { hp[(size_t)c0 * bt + r0 + 8] = d[2]; hp[(size_t)(c0 + 1) * bt + r0 + 8] = d[3]; }
            }
          }
        if (gl < bt) p.gpart[(size_t)sl * bt + gl] = gacc;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int sli = base + i;   // every lane holds fragments of both slices
        if (sli < p.n_slices) {
          float* hp = p.hpart + (size_t)sli * bt * bt;
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) {
            const float(&d)[4] = acc[2 * i + nb];
            const int c0 = 8 * nb + 2 * t4;
            if (g < bt && c0 < bt) *reinterpret_cast<float2*>(hp + (size_t)g * bt + c0) = make_float2(d[0], d[1]);
            if (g + 8 < bt && c0 < bt) *reinterpret_cast<float2*>(hp + (size_t)(g + 8) * bt + c0) = make_float2(d[2], d[3]);
          }
        }
      }
      if (live && gl < bt) p.gpart[(size_t)sl * bt + gl] = gacc;
    }
  }
}

// A heavy row's slice partials summed into its first slice's slot, in a fixed
// order, by one CTA: NGR groups of bt^2/4 threads each add every NGR-th slice
// (four loads in flight), then group 0 adds the groups' sums in group order.
// k_heavy_solve then reads one slot per row (SweepParams::heavy_reduced) -- the
// most popular item of the configs[1..3] shape has 549k entries, hundreds to
// thousands of slices that one warp otherwise adds one after the other.
template <int BT>
struct HRLay {
  static constexpr int V = BT * BT / 4, NGR = BT >= 32 ? 4 : 8, NT = V * NGR;   // 32: 1024, 16: 512, 8: 128
};

template <int BT>
__global__ void __launch_bounds__(HRLay<BT>::NT) k_heavy_reduce(SweepParams p) {
  using L = HRLay<BT>;
  __shared__ float4 part[L::NGR][L::V];
  __shared__ double gp[L::NGR][BT];
  const int h = blockIdx.x;
  const int sl0 = __ldg(p.heavy_slice0 + h), sl1 = __ldg(p.heavy_slice0 + h + 1);
  if (sl1 - sl0 <= 1) return;
  const int g = threadIdx.x / L::V, v = threadIdx.x % L::V;
  const float4* hp = reinterpret_cast<const float4*>(p.hpart);
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
  for (int sl = sl0 + g; sl < sl1; sl += L::NGR) {
    const float4 x = hp[(size_t)sl * L::V + v];
    a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
  }
  part[g][v] = a;
  if (v < BT) {
    double ga = 0.0;
#pragma unroll 4
    for (int sl = sl0 + g; sl < sl1; sl += L::NGR) ga += p.gpart[(size_t)sl * BT + v];
    gp[g][v] = ga;
  }
  __syncthreads();
  if (g == 0) {
    float4 t = part[0][v];
#pragma unroll
    for (int k = 1; k < L::NGR; ++k) {
      const float4 x = part[k][v];
      t.x += x.x; t.y += x.y; t.z += x.z; t.w += x.w;
    }
    reinterpret_cast<float4*>(p.hpart)[(size_t)sl0 * L::V + v] = t;
    if (v < BT) {
      double gt = gp[0][v];
#pragma unroll
      for (int k = 1; k < L::NGR; ++k) gt += gp[k][v];
      p.gpart[(size_t)sl0 * BT + v] = gt;
    }
  }
}

}  // namespace ials
