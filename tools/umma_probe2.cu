// umma_probe2: try operand-layout variants for the MN-major tf32 Gram MMA.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2110_14044_b200/csrc/ials_umma.cuh"
using namespace ials;
constexpr int M = 128, KX = 16;

__global__ void probe(const float* X, float* out, int variant) {
  __shared__ __align__(1024) float xs[4096];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 4096; i += blockDim.x) xs[i] = 0.f;
  __syncthreads();
  for (int i = t; i < KX * M; i += blockDim.x) {
    int k = i / M, m = i % M;
    if (variant < 5 && k >= 8) continue;
    int idx;
    if (variant == 0 || variant == 1) idx = sw128_mn_index(m, k, 256, 1024);
    else if (variant == 2 || variant == 3) idx = (m / 4) * 32 + (k / 8) * 1024 + (k % 8) * 4 + (m % 4);  // no swizzle MN
    else if (variant == 4) { // K-major SW128: row m (128B = 32 k), chunk c = k/4 ^ (m%8), atom per 8 rows
      int r = m & 7; idx = (m >> 3) * 256 + r * 32 + ((((k >> 2)) ^ r) << 2) + (k & 3);
    } else { // K-major SW64: row m (64B = 16 k), chunk c = k/4 ^ ((m%8)>>1), atom 8 rows x 64B
      int r = m & 7; idx = (m >> 3) * 128 + r * 16 + ((((k >> 2)) ^ ((r >> 1) & 3)) << 2) + (k & 3);
    }
    xs[idx] = X[i];
  }
  if (t == 0) mbar_init(&bar, 1);
  if (w == 0) tmem_alloc(&tbase, 128);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (t == 0) {
    uint32_t idesc; uint64_t a;
    switch (variant) {
      case 0: idesc = make_idesc_tf32(128,128,1,1,0); a = make_sdesc(smem_u32(xs), 1024, 4096, kSwizzle128B); break;
      case 1: idesc = make_idesc_tf32(128,128,1,1,0); a = make_sdesc(smem_u32(xs), 4096, 1024, kSwizzle128B); break;
      case 2: idesc = make_idesc_tf32(128,128,1,1,0); a = make_sdesc(smem_u32(xs), 4096, 128, kSwizzleNone); break;
      case 3: idesc = make_idesc_tf32(128,128,1,1,0); a = make_sdesc(smem_u32(xs), 128, 4096, kSwizzleNone); break;
      case 4: idesc = make_idesc_tf32(128,128,0,0,0); a = make_sdesc(smem_u32(xs), 16, 1024, kSwizzle128B); break;
      default: idesc = make_idesc_tf32(128,128,0,0,0); a = make_sdesc(smem_u32(xs), 16, 512, 4); break;
    }
    umma_tf32(d, a, a, idesc, 0);
    if (variant == 6) {  // second K step of a 16-wide SW64 chunk: start + 32 B
      uint64_t a2 = make_sdesc(smem_u32(xs) + 32, 16, 512, 4);
      umma_tf32(d, a2, a2, idesc, 1);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < 128; c += 8) {
    float v[8];
    tmem_ld8(d + ((uint32_t)(32 * w) << 16) + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 8; ++j) out[t * 128 + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_free(tbase, 128);
}

int main() {
  std::vector<float> X(KX * M), o(M * M);
  srand(1);
  for (auto& x : X) x = (float)(rand() % 7 - 3);
  float *dX, *dO;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dO, o.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  for (int v = 0; v < 7; ++v) {
    cudaMemset(dO, 0, o.size() * 4);
    probe<<<1, 128>>>(dX, dO, v);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("variant %d: %s\n", v, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0; double s = 0;
    for (int i = 0; i < M; ++i) for (int j = 0; j < M; ++j) {
      double g = 0; const int kk = (v == 6) ? 16 : 8;
      for (int k = 0; k < kk; ++k) g += (double)X[k * M + i] * X[k * M + j];
      s += std::fabs(o[i * M + j]);
      if (std::fabs(o[i * M + j] - g) > 1e-3) ++bad;
    }
    printf("variant %d: mismatches %d  sum|D| %.1f  D[0][0..3] %.1f %.1f %.1f %.1f\n", v, bad, s, o[0], o[1], o[2], o[3]);
  }
  return 0;
}
