// ials_csr.cuh -- device CSR construction, bit-exact with
// InteractionDataset.__init__ / user_view / item_view
// (/root/reference/pkg/src/blockals/data.py:98-134,148-162):
//   order      = argsort(users, stable)          -> user-major canonical order
//   user_cols  = items[order]                    (user view cols)
//   user_ptr   = [0, cumsum(bincount(users))]
//   item_order = argsort(user_cols, stable)      (item view cache_pos)
//   item_cols  = users[order][item_order]        (item view cols)
//   item_ptr   = [0, cumsum(bincount(items))]
//
// Stable sorts are LSD radix sorts with 8-bit digits (ceil(log2 K / 8) passes
// for keys in [0, K)).  One pass = per-tile digit histograms (digit-major) ->
// per-digit scan over the tiles (one CTA per digit) -> stable scatter, whose
// CTAs add the exclusive scan of the 256 bucket sizes: a tile of 2048 consecutive
// elements is ranked in eight rounds of 256 (round, warp, lane order = input
// order), within a warp by __match_any_sync, across warps by a per-round
// warp x digit prefix in shared memory.  Row pointers come from the sorted
// keys (every boundary k writes ptr[u] = k for the keys it skips), so there
// are no atomics anywhere and the result is deterministic.
#pragma once
#include <cstdint>
#include "ials_common.cuh"

namespace ials {

constexpr int kRadixThreads = 256, kRadixRounds = 8, kRadixTile = kRadixThreads * kRadixRounds;
constexpr int kRadixWarps = kRadixThreads / 32;

// hist[digit * ntiles + tile] = count of the digit in the tile (digit-major)
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const int* __restrict__ keys, int64_t n,
                                                              int shift, int* __restrict__ hist) {
  __shared__ int h[256];
  const int tid = threadIdx.x;
  h[tid] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
#pragma unroll
  for (int r = 0; r < kRadixRounds; ++r) {
    const int64_t j = base + r * kRadixThreads + tid;
    if (j < n) atomicAdd(&h[(__ldg(keys + j) >> shift) & 255], 1);
  }
  __syncthreads();
  hist[(int64_t)tid * gridDim.x + blockIdx.x] = h[tid];
}

// In place, one CTA per digit d: hist[d][t] <- sum_{t' < t} hist[d][t']
// (the tile's offset inside the digit's bucket); tot[d] = the bucket size.
// Thread k scans a contiguous run of tiles, runs are combined by a block scan.
__global__ void __launch_bounds__(256) k_radix_scan(int* __restrict__ hist, int ntiles, int* __restrict__ tot) {
  __shared__ int ws[8];
  const int d = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* h = hist + (int64_t)d * ntiles;
  const int per = (ntiles + 255) / 256, t0 = tid * per, t1 = min(ntiles, t0 + per);
  int s = 0;
  for (int t = t0; t < t1; ++t) s += h[t];
  int x = s;   // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  int wbase = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) wbase += (w < warp) ? ws[w] : 0;
  int run = wbase + x - s;   // exclusive prefix of this thread's run
  for (int t = t0; t < t1; ++t) {
    const int v = h[t];
    h[t] = run;
    run += v;
  }
  if (tid == 255) tot[d] = run;
}

// Stable scatter of (key, value) by digit; vals_in == nullptr means value = index.
__global__ void __launch_bounds__(kRadixThreads) k_radix_scatter(const int* __restrict__ keys_in,
                                                                 const int* __restrict__ vals_in, int64_t n,
                                                                 int shift, const int* __restrict__ hist,
                                                                 const int* __restrict__ tot,
                                                                 int* __restrict__ keys_out,
                                                                 int* __restrict__ vals_out) {
  __shared__ int cnt[256];                  // elements of each digit ranked so far in the tile
  __shared__ int wh[kRadixWarps][256];      // this round: per-warp digit counts -> warp prefix
  __shared__ int rtot[256];
  __shared__ int tbase[256];                // output position of the tile's first element per digit
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  cnt[tid] = 0;
  const int64_t tb = (int64_t)blockIdx.x * kRadixTile;
  {  // bucket starts: exclusive scan of the digit totals, + the tile's offset in its bucket
    const int v = tot[tid];
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) rtot[warp] = x;
    __syncthreads();
    int wbase = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) wbase += (w < warp) ? rtot[w] : 0;
    tbase[tid] = wbase + x - v + hist[(int64_t)tid * gridDim.x + blockIdx.x];
    __syncthreads();
  }
  for (int r = 0; r < kRadixRounds; ++r) {
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) wh[w][tid] = 0;
    __syncthreads();
    const int64_t j = tb + r * kRadixThreads + tid;
    const bool valid = j < n;
    const int key = valid ? __ldg(keys_in + j) : 0;
    const int dg = valid ? (key >> shift) & 255 : 256 + lane;   // invalid lanes match nobody
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const int lrank = __popc(peers & lt);
    if (valid && lrank == 0) wh[warp][dg] = __popc(peers);
    __syncthreads();
    {  // thread tid <-> digit tid: exclusive prefix over the warps of this round
      int run = 0;
#pragma unroll
      for (int w = 0; w < kRadixWarps; ++w) {
        const int v = wh[w][tid];
        wh[w][tid] = run;
        run += v;
      }
      rtot[tid] = run;
    }
    __syncthreads();
    if (valid) {
      const int64_t pos = (int64_t)tbase[dg] + cnt[dg] + wh[warp][dg] + lrank;
      keys_out[pos] = key;
      vals_out[pos] = vals_in ? __ldg(vals_in + j) : (int)j;
    }
    __syncthreads();
    cnt[tid] += rtot[tid];
  }
}

// ptr[u] = first sorted position whose key >= u, for u in [0, K]; skeys sorted.
__global__ void k_row_ptr(const int* __restrict__ skeys, int64_t n, int K, int* __restrict__ ptr) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k > n) return;
  const int lo = (k == 0) ? 0 : __ldg(skeys + k - 1) + 1;   // keys skipped between k-1 and k
  const int hi = (k == n) ? K : __ldg(skeys + k);
  for (int u = lo; u <= hi; ++u) ptr[u] = (int)k;
}

__global__ void k_gather_i32(const int* __restrict__ src, const int* __restrict__ idx, int64_t n,
                             int* __restrict__ dst) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[k] = __ldg(src + __ldg(idx + k));
}

// chunk of each row id (rows [c * per, (c + 1) * per) form chunk c)
__global__ void k_chunk_keys(const int* __restrict__ rows, int n, int per, int* __restrict__ keys) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) keys[k] = __ldg(rows + k) / per;
}

// the same with the rotated pass's three row classes inside every chunk:
// key = 3 * chunk + (0: more than 64 entries, 1: 33..64, 2: at most 32)
__global__ void k_chunk_class_keys(const int* __restrict__ rows, const int* __restrict__ ptr, int n, int per,
                                   int* __restrict__ keys) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) {
    const int r = __ldg(rows + k);
    const int deg = __ldg(ptr + r + 1) - __ldg(ptr + r);
    keys[k] = 3 * (r / per) + (deg > 64 ? 0 : (deg > 32 ? 1 : 2));
  }
}

__global__ void k_iota_i32(int64_t n, int* __restrict__ dst) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[k] = (int)k;
}

}  // namespace ials
