// umma_latency: round-trip latency of (k x tcgen05.mma kind::tf32 M=128 N) + commit + mbarrier
// wait, measured with clock64 in one CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2110_14044_b200/csrc/ials_umma.cuh"
using namespace ials;

__global__ void lat(long long* out, int nmma, int N, int iters) {
  __shared__ __align__(1024) float ops[128 * 8 * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  const int t = threadIdx.x;
  for (int i = t; i < 128 * 16; i += blockDim.x) ops[i] = 0.001f * (i % 7);
  if (t == 0) mbar_init(&bar, 1);
  if (t < 32) tmem_alloc(&tb, 128);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t phase = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (t == 0) {
      tc_fence_after();
      const uint32_t id = make_idesc_tf32(128, N, 0, 0, 1);
      const uint64_t a = make_sdesc(smem_u32(ops), 128, 256, kSwizzleNone);
      for (int k = 0; k < nmma; ++k) umma_tf32(tb, a, a, id, 1);
      umma_commit(&bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc_fence_after();
    __syncthreads();
  }
  long long t1 = clock64();
  if (t == 0) out[0] = (t1 - t0) / iters;
  tc_fence_before();
  __syncthreads();
  if (t < 32) tmem_free(tb, 128);
}

__global__ void bar_lat(long long* out, int iters) {
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  for (int N : {128, 64}) for (int n : {1, 3, 6}) {
    lat<<<1, 128>>>(d, n, N, 200); cudaDeviceSynchronize();
    lat<<<1, 128>>>(d, n, N, 1000);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%d mmas=%d: %lld cycles per issue+commit+wait round trip (%s)\n", N, n, h, cudaGetErrorString(e));
  }
  bar_lat<<<1, 128>>>(d, 1000); cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (128 thr): %lld cycles\n", h);
  return 0;
}
