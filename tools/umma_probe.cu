// umma_probe.cu -- validates the tcgen05 building blocks used by the tensor-core
// sweep against a host reference (run on a B200):
//   1. TMEM alloc / tcgen05.ld / tcgen05.st / dealloc
//   2. tcgen05.mma kind::tf32, M=128 N=128 K=8, A = B = X^T with X staged
//      MN-major SWIZZLE_128B (the gathered-row layout of the Hessian)
//   3. the same with a_negate and K-major SWIZZLE_NONE operands (the rank-8
//      panel update of the Cholesky)
//   4. tcgen05.commit -> mbarrier completion
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2110_14044_b200/csrc/ials_umma.cuh"

using namespace ials;

constexpr int M = 128, KX = 16, KP = 8;

__global__ void probe(const float* X /*[KX][M]*/, const float* P /*[M][KP]*/, float* out0,
                      float* out1, int mode) {
  __shared__ __align__(1024) float xs[KX * M];   // 8 KB, SW128 MN-major atoms
  __shared__ __align__(1024) float ps[M * KP];   // 4 KB, K-major no swizzle
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < KX * M; i += blockDim.x) {
    int k = i / M, m = i % M;
    xs[sw128_mn_index(m, k, 256, 1024)] = X[i];  // LBO / SBO in floats: 1 KB / 4 KB
  }
  for (int i = t; i < M * KP; i += blockDim.x) {
    int m = i / KP, q = i % KP;
    ps[kmaj_none_index(m, q, 256 / 4, 128 / 4)] = P[i];
  }
  if (t == 0) mbar_init(&bar, 1);
  if (w == 0) tmem_alloc(&tbase, 128);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (t == 0 && mode >= 0) {
    const uint32_t idesc = make_idesc_tf32(128, 128, /*a_mn*/ 1, /*b_mn*/ 1, /*neg*/ 0);
    for (int s = 0; s < KX / 8; ++s) {
      uint64_t a = make_sdesc(smem_u32(xs) + s * 4096, 1024, 4096, kSwizzle128B);
      umma_tf32(d, a, a, idesc, s > 0);
    }
    if (mode == 1) {
      const uint32_t idn = make_idesc_tf32(128, 128, 0, 0, 1);
      uint64_t p = make_sdesc(smem_u32(ps), 128, 256, kSwizzleNone);
      umma_tf32(d, p, p, idn, 1);
    }
    umma_commit(&bar);
  }
  if (mode >= 0) mbar_wait(&bar, 0);
  tc_fence_after();
  float* out = mode <= 0 ? out0 : out1;
  for (int c = 0; c < 128; c += 8) {
    float v[8];
    tmem_ld8(d + ((uint32_t)(32 * w) << 16) + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 8; ++j) out[t * 128 + c + j] = v[j];
  }
  // tcgen05.st round trip: write row t + 1000 into column 0..7, read back
  float z[8];
  for (int j = 0; j < 8; ++j) z[j] = 1000.f + t + j;
  tmem_st8(d + ((uint32_t)(32 * w) << 16), z);
  tmem_wait_st();
  float v[8];
  tmem_ld8(d + ((uint32_t)(32 * w) << 16), v);
  tmem_wait_ld();
  for (int j = 0; j < 8; ++j)
    if (v[j] != z[j]) out[t * 128 + j] = -12345.f;
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_free(tbase, 128);
}

int main() {
  std::vector<float> X(KX * M), P(M * KP), o0(M * M), o1(M * M);
  srand(1);
  for (auto& x : X) x = (float)(rand() % 7 - 3);
  for (auto& p : P) p = (float)(rand() % 5 - 2);
  float *dX, *dP, *d0, *d1;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dP, P.size() * 4);
  cudaMalloc(&d0, o0.size() * 4); cudaMalloc(&d1, o1.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 4, cudaMemcpyHostToDevice);
  int stage = getenv("STAGE") ? atoi(getenv("STAGE")) : 9;
  probe<<<1, 128>>>(dX, dP, d0, d1, -1);
  cudaError_t e = cudaDeviceSynchronize();
  printf("stage -1 (tmem only): %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess || stage < 0) return 1;
  probe<<<1, 128>>>(dX, dP, d0, d1, 0);
  e = cudaDeviceSynchronize();
  printf("stage 0 (gram mma): %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  probe<<<1, 128>>>(dX, dP, d0, d1, 1);
  e = cudaDeviceSynchronize();
  printf("stage 1 (rank-8): %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(o0.data(), d0, o0.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(o1.data(), d1, o1.size() * 4, cudaMemcpyDeviceToHost);
  int bad0 = 0, bad1 = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) {
      double g = 0, pp = 0;
      for (int k = 0; k < KX; ++k) g += (double)X[k * M + i] * X[k * M + j];
      for (int q = 0; q < KP; ++q) pp += (double)P[i * KP + q] * P[j * KP + q];
      bool st_ok = true;
      if (j < 8) st_ok = o0[i * M + j] != -12345.f && o1[i * M + j] != -12345.f;
      if (j >= 8 && std::fabs(o0[i * M + j] - g) > 1e-3) { if (bad0++ < 5) printf("D0[%d][%d] %f vs %f\n", i, j, o0[i * M + j], g); }
      if (j >= 8 && std::fabs(o1[i * M + j] - (g - pp)) > 1e-3) { if (bad1++ < 5) printf("D1[%d][%d] %f vs %f\n", i, j, o1[i * M + j], g - pp); }
      if (!st_ok) { bad0++; }
    }
  printf("umma probe: gram mismatches %d, rank-8 update mismatches %d\n", bad0, bad1);
  return (bad0 || bad1) ? 2 : 0;
}
