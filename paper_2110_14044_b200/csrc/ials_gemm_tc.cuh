// ials_gemm_tc.cuh -- the two dense GEMMs of an iALS++ block step on the
// tensor core (tcgen05, 3xTF32, TMA-fed), used by ials_epoch:
//
//   Gramian slab  G[:, pi] = F^T F[:, pi]          (d x b, K = rows of F)
//   projection    proj     = alpha0 * own G[:, pi] (rows x b, K = d)
//
// Both operands must be K-major for kind::tf32, so the epoch keeps, per
// factor matrix F (n x d), the transposed copy F^T (d x n); k_sync_copies
// refreshes it for the column block a side pass just changed
// (solvers.py:340-375 updates one block at a time).  The tf32 low parts
// x - trunc_tf32(x) are formed on chip, and
// D = A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T accumulates in TMEM.
//
// One CTA = 256 threads: warp 0 / lane 0 issues TMA loads of the raw fp32
// operands (the hi parts: the MMA drops their low 13 bits) into a 3-stage ring,
// warps 2..7 form the lo parts x - trunc_tf32(x) in shared memory (same
// swizzled layout: the map is elementwise), warp 1 / lane 0 issues the MMAs
// once both are there, and all eight warps drain the 128 x N accumulator
// (warp w: TMEM lanes 32 (w % 4).., column half w / 4).  Only the raw
// operands cross HBM, half of what stored lo copies would cost.
#pragma once
#include <cuda.h>
#include "ials_common.cuh"
#include "ials_umma.cuh"

namespace ials {

struct GemmJob {
  int m_rows;              // valid output rows (rows of A)
  int a_row0;              // first A row of tile 0 (row coordinate in the A maps)
  int b_row0;              // first B row
  int n;                   // valid output columns; the MMA runs N = bn = round_up(n, 16)
  int bn;
  int k_total;             // K extent
  int k_span;              // K per split (multiple of 32)
  float* out;              // out[split][row][col]
  int ldo;
  long long split_stride;  // floats between splits
  float scale;
  int b_lo_tma = 0;        // B's lo part is precomputed in memory (b_lo map): TMA-load it
  int n_tiles = 0;         // > 0: blockIdx.y walks N tiles of 128 output columns (B rows
                           // b_row0 + 128 y, out columns 128 y..), no K split (score GEMM)
  int a_k0 = 0;            // K coordinate of A's first column (a column block of A's map)
  int b_k0 = 0;            // the same for B
  int accumulate = 0;      // out += scale * acc instead of out = scale * acc
  int diag = 0;            // B rows follow the A tile (b_row0 + m0): diagonal blocks of F^T F
};

constexpr int kGemmStages = 3;
constexpr int kGemmKC = 32;  // K per stage: one 128-byte swizzle row
constexpr int kGemmThreads = 256, kGemmConv = kGemmThreads - 64;

struct GemmLay {
  static constexpr int A_BYTES = 128 * 128;  // 128 rows x 128 B
  static constexpr int B_BYTES = 128 * 128;  // up to 128 rows
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;   // A hi, A lo, B hi, B lo
  static constexpr int OFF_BAR = kGemmStages * STAGE;
  static constexpr int BYTES = OFF_BAR + 8 * (3 * kGemmStages + 1) + 16 + 1024;
};

IALS_DEVI void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm3_tf32(const __grid_constant__ CUtensorMap a_hi, const __grid_constant__ CUtensorMap b_hi,
                 const __grid_constant__ CUtensorMap b_lo, GemmJob job) {
  extern __shared__ __align__(1024) char smem_g[];
  char* smem = smem_g + ((1024u - (smem_u32(smem_g) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GemmLay::OFF_BAR);
  uint64_t* lo_ready = full + kGemmStages;
  uint64_t* empty = lo_ready + kGemmStages;
  uint64_t* done = empty + kGemmStages;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(done + 1);
  const int m0 = blockIdx.x * 128;
  const int ny = job.n_tiles ? (int)blockIdx.y : 0;   // N tile
  const int ks = job.n_tiles ? 0 : (int)blockIdx.y;   // K split
  const int b_row = job.b_row0 + 128 * ny + (job.diag ? m0 : 0);
  const int n_here = job.n_tiles ? min(128, job.n - 128 * ny) : job.n;
  const int kb = ks * job.k_span;
  const int ke = min(kb + job.k_span, job.k_total);
  const int nk = (ke - kb + kGemmKC - 1) / kGemmKC;
  if (tid == 0) {
    prefetch_tmap(&a_hi);
    prefetch_tmap(&b_hi);
    if (job.b_lo_tma) prefetch_tmap(&b_lo);
    for (int s = 0; s < kGemmStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(lo_ready + s, kGemmConv);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
  }
  if (warp == 2) tmem_alloc(tptr, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tptr;
  const uint32_t stage_bytes = GemmLay::A_BYTES + job.bn * 128 * (job.b_lo_tma ? 2 : 1);
  if (warp == 0 && (tid & 31) == 0) {  // TMA producer
    for (int c = 0; c < nk; ++c) {
      const int s = c % kGemmStages;
      if (c >= kGemmStages) mbar_wait(empty + s, ((c / kGemmStages) - 1) & 1);
      char* st = smem + s * GemmLay::STAGE;
      mbar_expect_tx(full + s, stage_bytes);
      const int kc = kb + c * kGemmKC;
      tma_load_2d(smem_u32(st), &a_hi, job.a_k0 + kc, job.a_row0 + m0, full + s);
      tma_load_2d(smem_u32(st + 2 * GemmLay::A_BYTES), &b_hi, job.b_k0 + kc, b_row, full + s);
      if (job.b_lo_tma)
        tma_load_2d(smem_u32(st + 2 * GemmLay::A_BYTES + GemmLay::B_BYTES), &b_lo, job.b_k0 + kc, b_row,
                    full + s);
    }
  } else if (warp == 1 && (tid & 31) == 0) {  // MMA issuer
    const uint32_t idesc = make_idesc_tf32(128, job.bn, 0, 0, 0);
    for (int c = 0; c < nk; ++c) {
      const int s = c % kGemmStages;
      mbar_wait(full + s, (c / kGemmStages) & 1);
      mbar_wait(lo_ready + s, (c / kGemmStages) & 1);
      tc_fence_after();
      const uint32_t base = smem_u32(smem + s * GemmLay::STAGE);
      const uint32_t ah = base, al = base + GemmLay::A_BYTES;
      const uint32_t bh = base + 2 * GemmLay::A_BYTES, bl = bh + GemmLay::B_BYTES;
#pragma unroll
      for (int ks = 0; ks < kGemmKC / 8; ++ks) {
        const uint64_t dah = make_sdesc(ah + ks * 32, 16, 1024, kSwizzle128B);
        const uint64_t dal = make_sdesc(al + ks * 32, 16, 1024, kSwizzle128B);
        const uint64_t dbh = make_sdesc(bh + ks * 32, 16, 1024, kSwizzle128B);
        const uint64_t dbl = make_sdesc(bl + ks * 32, 16, 1024, kSwizzle128B);
        umma_tf32(tmem, dah, dbh, idesc, (c | ks) > 0);
        umma_tf32(tmem, dah, dbl, idesc, 1);
        umma_tf32(tmem, dal, dbh, idesc, 1);
      }
      umma_commit(empty + s);   // frees the stage once these MMAs have read it
    }
    umma_commit(done);
  } else if (warp >= 2) {   // lo parts of the landed stage
    const int ct = tid - 64;
    const int na4 = GemmLay::A_BYTES / 16, nt4 = na4 + (job.b_lo_tma ? 0 : job.bn * 8);
    for (int c = 0; c < nk; ++c) {
      const int s = c % kGemmStages;
      mbar_wait(full + s, (c / kGemmStages) & 1);
      char* st = smem + s * GemmLay::STAGE;
      const float4* ahi = reinterpret_cast<const float4*>(st);
      float4* alo = reinterpret_cast<float4*>(st + GemmLay::A_BYTES);
      const float4* bhi = reinterpret_cast<const float4*>(st + 2 * GemmLay::A_BYTES);
      float4* blo = reinterpret_cast<float4*>(st + 2 * GemmLay::A_BYTES + GemmLay::B_BYTES);
      for (int i = ct; i < nt4; i += kGemmConv) {
        const bool isa = i < na4;
        const float4 v = isa ? ahi[i] : bhi[i - na4];
        const float4 l = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
        if (isa) alo[i] = l; else blo[i - na4] = l;
      }
      fence_proxy_async_smem();   // generic-proxy writes -> the MMA's async-proxy reads
      mbar_arrive(lo_ready + s);
    }
  }
  __syncwarp();
  // epilogue: warp w drains TMEM lanes 32 (w % 4).. (output rows m0 + lane), column half w / 4
  mbar_wait(done, 0);
  tc_fence_after();
  const int row = m0 + (warp & 3) * 32 + (tid & 31);
  float* o = job.out + (long long)ks * job.split_stride + (long long)row * job.ldo + 128 * ny;
  const uint32_t raddr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  for (int c32 = (warp >> 2) * 32; c32 < job.bn; c32 += 64) {   // warp-uniform
    float v[32];
    tmem_ld32(raddr + c32, v);
    tmem_wait_ld();
    if (row < job.m_rows && nk > 0 && job.accumulate) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c32 + j < n_here) o[c32 + j] += job.scale * v[j];
    } else if (row < job.m_rows && nk > 0) {
      if (c32 + 32 <= n_here && (job.ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(job.out) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)   // 16-byte stores: 8 per thread instead of 32
          *reinterpret_cast<float4*>(o + c32 + j) =
              make_float4(job.scale * v[j], job.scale * v[j + 1], job.scale * v[j + 2], job.scale * v[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c32 + j < n_here) o[c32 + j] = job.scale * v[j];
      }
    } else if (row < job.m_rows && !job.accumulate) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c32 + j < n_here) o[c32 + j] = 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_free(tmem, 128);
}

// slab[k][j] = sum_s P[s][k][j] (fixed split order), and its transpose
// split into tf32 hi / lo for the projection's B operand.
__global__ void k_gram_reduce(const float* __restrict__ P, int splits, long long split_stride, int d,
                              int b, float* slab, float* slabT_hi, float* slabT_lo) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= d * b) return;
  const int k = idx / b, j = idx - k * b;
  float s = 0.f;
  for (int t = 0; t < splits; ++t) s += P[(long long)t * split_stride + idx];
  slab[idx] = s;
  slabT_hi[(size_t)j * d + k] = s;
  if (slabT_lo) slabT_lo[(size_t)j * d + k] = tf32_lo(s);
}

// Refresh the K-major copies of F for columns [c0, c0 + cw): F^T, F^T_lo
// (d x ldt) and F_lo (n x ldl).  32 x 32 tiles through shared memory.
__global__ void k_sync_copies(const float* __restrict__ F, int n, int ldf, int c0, int cw,
                              float* FT, float* FT_lo, int ldt, float* F_lo, int ldl) {
  __shared__ float tile[32][33];
  const int r0 = blockIdx.x * 32, cb = c0 + blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int r = r0 + i, c = cb + tx;
    float x = 0.f;
    if (r < n && c < c0 + cw) {
      x = F[(size_t)r * ldf + c];
      if (F_lo) F_lo[(size_t)r * ldl + c] = tf32_lo(x);
    }
    tile[i][tx] = x;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int c = cb + i, r = r0 + tx;
    if (r < n && c < c0 + cw) {
      const float x = tile[tx][i];
      FT[(size_t)c * ldt + r] = x;
      if (FT_lo) FT_lo[(size_t)c * ldt + r] = tf32_lo(x);
    }
  }
}

}  // namespace ials
