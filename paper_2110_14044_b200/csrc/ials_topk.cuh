// ials_topk.cuh -- ranking for fold-in evaluation:
// top_k_from_scores (/root/reference/pkg/src/blockals/metrics.py:31-57) on
// the device.  One CTA per score row: the row's excluded entries are set to
// -inf (k_topk_exclude, from a CSR of excluded columns), then k_topk finds the
// K-th largest finite score by an MSB-first 8-bit radix select over
// order-preserving integer keys, collects the K winners in index order (block
// scans; ties at the threshold taken by ascending index), and bitonic-sorts
// them by (score descending, index ascending) -- the reference's lexsort
// order.  -0 is folded into +0 (numpy compares them equal); NaN / -inf never
// rank, and fewer than k finite candidates return all of them.
#pragma once
#include <cstdint>
#include "ials_common.cuh"

namespace ials {

constexpr int kTopkThreads = 512, kTopkMax = 1024;

__global__ void k_topk_exclude(float* __restrict__ scores, int64_t lds, const int* __restrict__ ptr,
                               const int* __restrict__ cols) {
  const int r = blockIdx.x;
  for (int e = ptr[r] + threadIdx.x; e < ptr[r + 1]; e += blockDim.x)
    scores[(int64_t)r * lds + cols[e]] = -INFINITY;
}

IALS_DEVI uint32_t rank_key(float s) {   // ascending key <-> ascending score
  const uint32_t u = __float_as_uint(s + 0.0f);   // -0 -> +0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// exclusive block scan of v (kTopkThreads threads); returns the prefix, *tot = sum
IALS_DEVI int block_scan_excl(int v, int* sh, int* tot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < kTopkThreads / 32) ? sh[lane] : 0;
    int z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < kTopkThreads / 32) sh[lane] = z - w;
    if (lane == kTopkThreads / 32 - 1) sh[32] = z;
  }
  __syncthreads();
  const int r = sh[warp] + x - v;
  *tot = sh[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kTopkThreads) k_topk(const float* __restrict__ scores, int64_t lds,
                                                       int n, int k, int* __restrict__ out,
                                                       int* __restrict__ counts) {
  __shared__ int hist[256];
  __shared__ int sh[40];
  __shared__ unsigned long long buf[kTopkMax];
  __shared__ uint32_t sel[3];   // threshold key, ties needed, pool
  const int tid = threadIdx.x, r = blockIdx.x;
  const float* s = scores + (int64_t)r * lds;
  // pool = finite scores
  int cnt = 0;
  for (int i = tid; i < n; i += kTopkThreads) cnt += isfinite(s[i]) ? 1 : 0;
  int pool;
  block_scan_excl(cnt, sh, &pool);
  const int K = min(k, pool);
  if (K == 0) {
    for (int j = tid; j < k; j += kTopkThreads) out[(int64_t)r * k + j] = -1;
    if (tid == 0) counts[r] = 0;
    return;
  }
  // radix select of the K-th largest key among the finite scores
  uint32_t prefix = 0, mask = 0;
  int remaining = K;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kTopkThreads) {
      const float v = s[i];
      if (!isfinite(v)) continue;
      const uint32_t key = rank_key(v);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int c = 0, dgt = 255;
      for (; dgt > 0; --dgt) {
        if (c + hist[dgt] >= remaining) break;
        c += hist[dgt];
      }
      sel[0] = (uint32_t)dgt;
      sel[1] = (uint32_t)(remaining - c);
    }
    __syncthreads();
    prefix |= sel[0] << shift;
    mask |= 0xFFu << shift;
    remaining = (int)sel[1];
    __syncthreads();
  }
  const uint32_t T = prefix;
  const int need = remaining;      // entries equal to T to take (lowest indices first)
  const int G = K - need;          // entries strictly above T
  // collect in index order
  int gt_run = 0, eq_run = 0;
  for (int base = 0; base < n; base += kTopkThreads) {
    const int i = base + tid;
    uint32_t key = 0;
    bool gt = false, eq = false;
    if (i < n) {
      const float v = s[i];
      if (isfinite(v)) {
        key = rank_key(v);
        gt = key > T;
        eq = key == T;
      }
    }
    int tg, te;
    const int pg = block_scan_excl(gt ? 1 : 0, sh, &tg);
    const int pe = block_scan_excl(eq ? 1 : 0, sh, &te);
    const unsigned long long comp = ((unsigned long long)key << 32) | (0xFFFFFFFFu - (uint32_t)i);
    if (gt) buf[gt_run + pg] = comp;
    if (eq && eq_run + pe < need) buf[G + eq_run + pe] = comp;
    gt_run += tg;
    eq_run += te;
  }
  // bitonic sort (descending) of the K winners, padded to a power of two
  int P = 1;
  while (P < K) P <<= 1;
  for (int j = K + tid; j < P; j += kTopkThreads) buf[j] = 0ull;
  __syncthreads();
  for (int len = 2; len <= P; len <<= 1) {
    for (int st = len >> 1; st > 0; st >>= 1) {
      for (int a = tid; a < P; a += kTopkThreads) {
        const int b = a ^ st;
        if (b > a) {
          const bool desc = (a & len) == 0;
          const unsigned long long x = buf[a], y = buf[b];
          if ((x < y) == desc) {
            buf[a] = y;
            buf[b] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int j = tid; j < k; j += kTopkThreads)
    out[(int64_t)r * k + j] = (j < K) ? (int)(0xFFFFFFFFu - (uint32_t)(buf[j] & 0xFFFFFFFFull)) : -1;
  if (tid == 0) counts[r] = K;
}

}  // namespace ials

namespace ials {

// float64 scores (top_k_from_scores on the caller's f64 array, metrics.py:31-57):
// the same selection over 64-bit order-preserving keys (8 radix passes), the
// winners sorted by (score descending, index ascending) as (key, index) pairs.
IALS_DEVI uint64_t rank_key64(double s) {
  const uint64_t u = (uint64_t)__double_as_longlong(s + 0.0);   // -0 -> +0
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_topk_exclude64(double* __restrict__ scores, int64_t lds, const int* __restrict__ ptr,
                                 const int* __restrict__ cols) {
  const int r = blockIdx.x;
  for (int e = ptr[r] + threadIdx.x; e < ptr[r + 1]; e += blockDim.x)
    scores[(int64_t)r * lds + cols[e]] = -INFINITY;
}

__global__ void __launch_bounds__(kTopkThreads) k_topk64(const double* __restrict__ scores, int64_t lds,
                                                         int n, int k, int* __restrict__ out,
                                                         int* __restrict__ counts) {
  __shared__ int hist[256];
  __shared__ int sh[40];
  __shared__ uint64_t bkey[kTopkMax];
  __shared__ int bidx[kTopkMax];
  __shared__ uint64_t sel[2];
  const int tid = threadIdx.x, r = blockIdx.x;
  const double* s = scores + (int64_t)r * lds;
  int cnt = 0;
  for (int i = tid; i < n; i += kTopkThreads) cnt += isfinite(s[i]) ? 1 : 0;
  int pool;
  block_scan_excl(cnt, sh, &pool);
  const int K = min(k, pool);
  if (K == 0) {
    for (int j = tid; j < k; j += kTopkThreads) out[(int64_t)r * k + j] = -1;
    if (tid == 0) counts[r] = 0;
    return;
  }
  uint64_t prefix = 0, mask = 0;
  int remaining = K;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kTopkThreads) {
      const double v = s[i];
      if (!isfinite(v)) continue;
      const uint64_t key = rank_key64(v);
      if ((key & mask) == prefix) atomicAdd(&hist[(int)((key >> shift) & 255)], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int c = 0, dgt = 255;
      for (; dgt > 0; --dgt) {
        if (c + hist[dgt] >= remaining) break;
        c += hist[dgt];
      }
      sel[0] = (uint64_t)dgt;
      sel[1] = (uint64_t)(remaining - c);
    }
    __syncthreads();
    prefix |= sel[0] << shift;
    mask |= 0xFFull << shift;
    remaining = (int)sel[1];
    __syncthreads();
  }
  const uint64_t T = prefix;
  const int need = remaining, G = K - need;
  int gt_run = 0, eq_run = 0;
  for (int base = 0; base < n; base += kTopkThreads) {
    const int i = base + tid;
    uint64_t key = 0;
    bool gt = false, eq = false;
    if (i < n) {
      const double v = s[i];
      if (isfinite(v)) {
        key = rank_key64(v);
        gt = key > T;
        eq = key == T;
      }
    }
    int tg, te;
    const int pg = block_scan_excl(gt ? 1 : 0, sh, &tg);
    const int pe = block_scan_excl(eq ? 1 : 0, sh, &te);
    if (gt) { bkey[gt_run + pg] = key; bidx[gt_run + pg] = i; }
    if (eq && eq_run + pe < need) { bkey[G + eq_run + pe] = key; bidx[G + eq_run + pe] = i; }
    gt_run += tg;
    eq_run += te;
  }
  int P = 1;
  while (P < K) P <<= 1;
  for (int j = K + tid; j < P; j += kTopkThreads) { bkey[j] = 0ull; bidx[j] = 0x7FFFFFFF; }
  __syncthreads();
  // (key desc, index asc): x before y when x.key > y.key or (equal and x.idx < y.idx)
  for (int len = 2; len <= P; len <<= 1) {
    for (int st = len >> 1; st > 0; st >>= 1) {
      for (int a = tid; a < P; a += kTopkThreads) {
        const int b = a ^ st;
        if (b > a) {
          const bool desc = (a & len) == 0;
          const uint64_t ka = bkey[a], kb = bkey[b];
          const int ia = bidx[a], ib = bidx[b];
          const bool a_first = ka > kb || (ka == kb && ia < ib);
          if (a_first != desc) {
            bkey[a] = kb; bkey[b] = ka;
            bidx[a] = ib; bidx[b] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int j = tid; j < k; j += kTopkThreads) out[(int64_t)r * k + j] = (j < K) ? bidx[j] : -1;
  if (tid == 0) counts[r] = K;
}

}  // namespace ials
