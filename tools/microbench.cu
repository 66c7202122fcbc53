// Microbenchmarks for the roofline denominators of the iALS++ sweep:
//  (1) FP32 FFMA throughput (register-tiled outer-product pattern, like the Hessian update)
//  (2) random row-gather bandwidth from an L2-resident and an HBM-resident table
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int NACC>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float acc[NACC];
  float x[4], y[8];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 4; i++) x[i] = a + i * 0.5f + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; i++) y[i] = b + i * 0.25f;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[i * 8 + j] = fmaf(x[i], y[j], acc[i * 8 + j]);
#pragma unroll
    for (int i = 0; i < 4; i++) x[i] = x[i] * 0.999f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// each warp gathers `rowf` floats (vectorised float4) from random rows
__global__ void gather_kernel(const float4* __restrict__ tab, const int* __restrict__ idx, int n, int rowv, int stridev, float* out) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  float s = 0;
  for (int k = warp; k < n; k += nw) {
    const float4* r = tab + (size_t)idx[k] * stridev;
    for (int v = lane; v < rowv; v += 32) { float4 q = __ldg(r + v); s += q.x + q.y + q.z + q.w; }
  }
  if (s == 123.456f) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d clock %d kHz l2 %d\n", p.name, p.multiProcessorCount, p.clockRate, p.l2CacheSize);
  float* out; CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int tpb : {256, 512}) for (int bps : {2, 4, 8}) {
    int grid = p.multiProcessorCount * bps;
    if (tpb * bps > 2048) continue;
    ffma_kernel<32><<<grid, tpb>>>(out, 100, 1.0f, 2.0f);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    ffma_kernel<32><<<grid, tpb>>>(out, iters, 1.0f, 2.0f);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 32 * iters * (double)grid * tpb;
    printf("ffma tpb=%d ctas/sm=%d : %.1f TFLOP/s\n", tpb, bps, flops / ms / 1e9);
  }
  // gather: table sizes 64 MB (L2-resident) and 2 GB (HBM)
  for (size_t tabMB : {16, 64, 2048}) for (int rowf : {32, 128, 512}) {
    int stridef = rowf < 256 ? 1024 : rowf;  // row stride like a d=1024 table with b-wide blocks
    size_t nrows = tabMB * (1 << 20) / (stridef * 4);
    float* tab; CK(cudaMalloc(&tab, nrows * stridef * 4));
    cudaMemset(tab, 0, nrows * stridef * 4);
    int n = 4 << 20;
    std::vector<int> h(n); uint64_t s = 88172645463325252ull;
    for (int i = 0; i < n; i++) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % nrows; }
    int* idx; CK(cudaMalloc(&idx, n * 4)); cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    gather_kernel<<<p.multiProcessorCount * 8, 256>>>((float4*)tab, idx, n, rowf / 4, stridef / 4, out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) gather_kernel<<<p.multiProcessorCount * 8, 256>>>((float4*)tab, idx, n, rowf / 4, stridef / 4, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("gather table %zu MB row %d B: %.1f GB/s\n", tabMB, rowf * 4, 5.0 * n * rowf * 4 / ms / 1e6);
    cudaFree(tab); cudaFree(idx);
  }
  return 0;
}
