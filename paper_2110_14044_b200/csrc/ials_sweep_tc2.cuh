// ials_sweep_tc2.cuh -- the tensor-core side pass for block widths 33..128,
// split into three kernels per wave of rows so each runs at its own
// occupancy (the fused per-row kernel is bound by its per-row dependency
// chain with only two rows in flight per SM):
//
//   k_tc_hess   (2 CTAs/SM)  one slice of a row per iteration: gathered
//               sub-rows -> 3xTF32 MMAs into TMEM, flushed per 32-entry chunk
//               into an fp32 register row sum; fp64 gradient partial.  Writes
//               the packed lower triangle (rows padded to 4 floats) of the
//               slice's partial Hessian.
//   k_tc_factor (4 CTAs/SM)  per row: sum of its slices (fixed order) +
//               alpha0*slab + lam*I into TMEM, blocked Cholesky with 3xTF32
//               rank-8 trailing MMAs, forward/backward solve, U[r,pi] -= d.
//   k_tc_cache  (many CTAs)  per slice: re-gather, yhat[pos] -= h . d.
//
// A wave holds at most a few thousand slices so the partials (34 KB each)
// stay L2-resident between k_tc_hess and k_tc_factor.
#pragma once
#include "ials_sweep_tc.cuh"

namespace ials {

constexpr int kTcPKS = 8448;  // packed floats per 128x128 lower triangle

IALS_DEVI int pk_off(int i) {
  const int q = i >> 2;
  return 4 * (2 * q * (q + 1) + (i - 4 * q) * (q + 1));
}

struct TcLayH {
  static constexpr int BT = 128, NT = 128, KC = 32, XLD = BT + 4;
  static constexpr int OFF_XT_HI = 0;
  static constexpr int OFF_XT_LO = OFF_XT_HI + 16384;
  static constexpr int OFF_X = OFF_XT_LO + 16384;
  static constexpr int OFF_AW = OFF_X + 2 * KC * XLD * 4;
  static constexpr int OFF_RH = OFF_AW + 2 * KC * 4;
  static constexpr int OFF_PS = OFF_RH + 2 * KC * 4;
  static constexpr int OFF_BAR = OFF_PS + 2 * KC * 4;
  static constexpr int BYTES = OFF_BAR + 16 + 1024;
};

struct TcLayF {
  static constexpr int BT = 128, NT = 128;
  static constexpr int OFF_PA_HI = 0;
  static constexpr int OFF_PA_LO = OFF_PA_HI + 4096;
  static constexpr int LP = BT * (BT + 1) / 2;
  static constexpr int OFF_L = OFF_PA_LO + 4096;
  static constexpr int OFF_DG = OFF_L + ((LP * 4 + 15) / 16) * 16;
  static constexpr int OFF_PY = OFF_DG + 64 * 4;
  static constexpr int OFF_RV = OFF_PY + 8 * 4;
  static constexpr int OFF_YP = OFF_RV + 8 * 4;
  static constexpr int OFF_Y = OFF_YP + 8 * 4;
  static constexpr int OFF_YF = OFF_Y + BT * 4;
  static constexpr int OFF_ID = OFF_YF + BT * 4;
  static constexpr int OFF_D = OFF_ID + BT * 4;
  static constexpr int OFF_BAR = OFF_D + BT * 4;
  static constexpr int BYTES = OFF_BAR + 16 + 1024;
};

struct TcLayC {  // one thread per entry, 128-entry chunks
  static constexpr int BT = 128, NT = 128, KC = 128, XLD = BT + 4;
  static constexpr int OFF_X = 0;
  static constexpr int OFF_AW = OFF_X + KC * XLD * 4;
  static constexpr int OFF_RH = OFF_AW + KC * 4;
  static constexpr int OFF_PS = OFF_RH + KC * 4;
  static constexpr int OFF_D = OFF_PS + KC * 4;
  static constexpr int BYTES = OFF_D + BT * 4 + 16;
};

IALS_DEVI void tc_setup(char* smem, TcState& st, int off_bar, int tid) {
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + off_bar);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + off_bar + 8);
  if (tid == 0) mbar_init(bar, 1);
  if (tid < 32) tmem_alloc(tptr, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  st.tmem = *tptr;
  st.phase = 0u;
}

IALS_DEVI void tc_teardown(const TcState& st, int tid) {
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_free(st.tmem, 128);
}

// alpha0 * slab[pi, pi] (identity on the padding) as packed lower rows: the
// same 33 KB for every row of the pass, so k_tc_factor reads it from L1.
__global__ void k_tc_template(SweepParams p, float* tpl) {
  const int i = blockIdx.x, b = p.b;
  for (int c = threadIdx.x; c < 4 * ((i >> 2) + 1); c += blockDim.x) {
    float v;
    if (i < b && c < b)
      v = p.alpha0 * p.slab[(size_t)(p.b0 + i) * b + c];
    else
      v = (c == i) ? 1.f : 0.f;
    tpl[pk_off(i) + c] = v;
  }
}

__global__ void __launch_bounds__(128) k_tc_hess(SweepParams p) {
  using L = TcLayH;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = tc_smem_base(smem_raw);
  const int tid = threadIdx.x;
  {
    float4* x = reinterpret_cast<float4*>(smem + L::OFF_X);
    for (int i = tid; i < 2 * L::KC * L::XLD / 4; i += L::NT) x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  TcState st;
  tc_setup(smem, st, L::OFF_BAR, tid);
  const int nq = (tid >> 2) + 1;  // float4s of packed row tid
  int ndone = 0;
  for (int s = p.w_s0 + blockIdx.x; s < p.w_s1; s += gridDim.x) {
    const bool rec = p.dbg && ndone == 1 && tid == 0;
    long long t0 = 0, t1 = 0;
    if (rec) t0 = clock64();
    float sum[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) sum[c] = 0.f;
    double gacc = 0.0;
    tc_accumulate<L>(p, smem, st, gacc, sum, p.tc_slice_beg[s], p.tc_slice_end[s], tid);
    if (rec) t1 = clock64();
    float* hp = p.hbuf + (size_t)(s - p.w_s0) * kTcPKS + pk_off(tid);
#pragma unroll
    for (int c4 = 0; c4 < 32; ++c4)
      if (c4 < nq)
        *reinterpret_cast<float4*>(hp + 4 * c4) =
            make_float4(sum[4 * c4], sum[4 * c4 + 1], sum[4 * c4 + 2], sum[4 * c4 + 3]);
    p.gbuf[(size_t)(s - p.w_s0) * 128 + tid] = gacc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (rec) {
      const long long t2 = clock64();
      long long* o = p.dbg + 8 * 1024 + blockIdx.x * 4;
      o[0] = t1 - t0; o[1] = t2 - t1; o[2] = p.tc_slice_end[s] - p.tc_slice_beg[s];
    }
    ++ndone;
  }
  tc_teardown(st, tid);
}

__global__ void __launch_bounds__(128) k_tc_factor(SweepParams p) {
  using L = TcLayF;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = tc_smem_base(smem_raw);
  const int tid = threadIdx.x;
  TcState st;
  tc_setup(smem, st, L::OFF_BAR, tid);
  float* ys = reinterpret_cast<float*>(smem + L::OFF_Y);
  const float* ds = reinterpret_cast<const float*>(smem + L::OFF_D);
  const int b = p.b, i = tid;
  const uint32_t row_addr = st.tmem + ((uint32_t)((tid >> 5) * 32) << 16);
  int nrow_done = 0;
  long long tphase[8];
  for (int r = p.w_r0 + blockIdx.x; r < p.w_r1; r += gridDim.x) {
    const bool rec = p.dbg && nrow_done == 1 && tid == 0;
    if (rec) tphase[0] = clock64();
    const int row = p.tc_rows[r];
    const int s_beg = p.tc_row_slice0[r], s_end = p.tc_row_slice0[r + 1];
    const float lam = p.side.lam[row];
    // Hessian row i (lower part) = template (alpha0 * slab, L1-resident) +
    // sum of the row's slice partials (+ lam on the diagonal); 64 columns per
    // batch of loads, all in flight
    const float* tp = p.tpl + pk_off(i);
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      if (rec) tphase[5 + q] = clock64();
      if (64 * q > i) {
        float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) tmem_st8(row_addr + 64 * q + 8 * c8, z);
        continue;
      }
      float4 x[16];
#pragma unroll
      for (int c4 = 0; c4 < 16; ++c4)
        x[c4] = (64 * q + 4 * c4 <= i) ? __ldg(reinterpret_cast<const float4*>(tp + 64 * q) + c4)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = s_beg; s < s_end; ++s) {
        const float* hp = p.hbuf + (size_t)(s - p.w_s0) * kTcPKS + pk_off(i) + 64 * q;
        float4 y[16];
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4)
          y[c4] = (64 * q + 4 * c4 <= i) ? __ldcg(reinterpret_cast<const float4*>(hp) + c4)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4) {
          x[c4].x += y[c4].x; x[c4].y += y[c4].y; x[c4].z += y[c4].z; x[c4].w += y[c4].w;
        }
      }
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        float w8[8] = {x[2 * c8].x, x[2 * c8].y, x[2 * c8].z, x[2 * c8].w,
                       x[2 * c8 + 1].x, x[2 * c8 + 1].y, x[2 * c8 + 1].z, x[2 * c8 + 1].w};
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (64 * q + 8 * c8 + j == i && i < b) w8[j] += lam;
        tmem_st8(row_addr + 64 * q + 8 * c8, w8);
      }
    }
    tmem_wait_st();
    if (rec) tphase[7] = clock64();
    {
      double g = 0.0;
      for (int s = s_beg; s < s_end; ++s) g += p.gbuf[(size_t)(s - p.w_s0) * 128 + tid];
      float gv = 0.f;
      if (tid < b)
        gv = (float)(g + (double)p.proj[(size_t)row * b + tid] +
                     (double)lam * (double)p.own[(size_t)row * p.ldo + p.b0 + tid]);
      ys[tid] = gv;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (rec) tphase[1] = clock64();
    tc_factor<L>(p, smem, st, row, tid);
    if (rec) tphase[2] = clock64();
    tc_backward<L>(p, smem, tid);
    if (rec) tphase[3] = clock64();
    if (tid < b) {
      p.own[(size_t)row * p.ldo + p.b0 + tid] -= ds[tid];
      p.dbuf[(size_t)(r - p.w_r0) * 128 + tid] = ds[tid];
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (rec) {
      tphase[4] = clock64();
      for (int k = 0; k < 8; ++k) p.dbg[blockIdx.x * 8 + k] = tphase[k];
    }
    ++nrow_done;
  }
  tc_teardown(st, tid);
}

__global__ void __launch_bounds__(128) k_tc_cache(SweepParams p) {
  using L = TcLayC;
  extern __shared__ __align__(16) char smem_c[];
  char* smem = smem_c;
  const int tid = threadIdx.x;
  float* XN = reinterpret_cast<float*>(smem + L::OFF_X);
  float* AW = reinterpret_cast<float*>(smem + L::OFF_AW);
  float* RH = reinterpret_cast<float*>(smem + L::OFF_RH);
  int* PS = reinterpret_cast<int*>(smem + L::OFF_PS);
  float* DS = reinterpret_cast<float*>(smem + L::OFF_D);
  for (int s = p.w_s0 + blockIdx.x; s < p.w_s1; s += gridDim.x) {
    const int r = p.tc_slice_row[s];
    const int ebeg = p.tc_slice_beg[s], eend = p.tc_slice_end[s];
    if (eend <= ebeg) continue;
    __syncthreads();
    DS[tid] = tid < p.b ? p.dbuf[(size_t)(r - p.w_r0) * 128 + tid] : 0.f;
    for (int c0 = ebeg; c0 < eend; c0 += L::KC) {
      const int nk = min(L::KC, eend - c0);
      stage_entries<L::NT, L::KC, L::XLD>(p, XN, AW, RH, PS, c0, nk, tid);
      cp_async_wait<0>();
      __syncthreads();
      if (tid < nk) {
        const float* xr = XN + tid * L::XLD;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        int j = 0;
        if (p.vec) {
          for (; j + 3 < p.b; j += 4) {
            const float4 x = *reinterpret_cast<const float4*>(xr + j);
            const float4 dv = *reinterpret_cast<const float4*>(DS + j);
            s0 = fmaf(x.x, dv.x, s0);
            s1 = fmaf(x.y, dv.y, s1);
            s2 = fmaf(x.z, dv.z, s2);
            s3 = fmaf(x.w, dv.w, s3);
          }
        }
        for (; j < p.b; ++j) s0 = fmaf(xr[j], DS[j], s0);
        p.cache[PS[tid]] -= (s0 + s1) + (s2 + s3);
      }
      __syncthreads();
    }
  }
}

}  // namespace ials
