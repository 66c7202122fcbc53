// tma_gather_probe: how does cp.async.bulk.tensor.2d ... tile::gather4 lay four
// gathered rows into shared memory, and with which tensor-map box?  Matrix
// M[r][c] = r * 1000 + c (n x 128 fp32); gather rows {7, 500, 3, 999}.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../paper_2110_14044_b200/csrc/ials_umma.cuh"
using namespace ials;

__global__ void probe(const __grid_constant__ CUtensorMap map, float* out, int tx_bytes, int* status) {
  __shared__ __align__(1024) float sm[4 * 128];
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  for (int i = t; i < 512; i += blockDim.x) sm[i] = -1.f;
  if (t == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (t == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)),
                 "r"(tx_bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(sm)),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(7), "r"(500), "r"(3), "r"(999),
        "r"(smem_u32(&bar))
        : "memory");
  }
  // bounded wait: a wrong transaction count must not hang the GPU
  uint32_t done = 0;
  for (int it = 0; it < (1 << 22) && !done; ++it) {
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
  }
  __syncthreads();
  if (t == 0) *status = done;
  for (int i = t; i < 512; i += blockDim.x) out[i] = sm[i];
}

int main() {
  const int n = 1000, w = 128;
  std::vector<float> M((size_t)n * w);
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < w; ++c) M[(size_t)r * w + c] = r * 1000.f + c;
  float *dM, *dO;
  int* dS;
  cudaMalloc(&dM, M.size() * 4);
  cudaMalloc(&dO, 512 * 4);
  cudaMalloc(&dS, 4);
  cudaMemcpy(dM, M.data(), M.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int boxes[2] = {1, 4};
  for (int bi = 0; bi < 2; ++bi) {
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)w, (cuuint64_t)n};
    cuuint64_t gstr[1] = {(cuuint64_t)w * 4};
    cuuint32_t box[2] = {128, (cuuint32_t)boxes[bi]};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dM, gdim, gstr, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("box {128,%d}: encode failed %d\n", boxes[bi], (int)r); continue; }
    cudaMemset(dO, 0, 512 * 4);
    probe<<<1, 128>>>(map, dO, 2048, dS);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("box {128,%d}: %s\n", boxes[bi], cudaGetErrorString(e)); return 1; }
    std::vector<float> o(512);
    int st = 0;
    cudaMemcpy(o.data(), dO, 2048, cudaMemcpyDeviceToHost);
    cudaMemcpy(&st, dS, 4, cudaMemcpyDeviceToHost);
    printf("box {128,%d}: barrier %s | row0 [%g %g .. %g] row1 [%g %g] row2 [%g] row3 [%g .. %g]\n",
           boxes[bi], st ? "completed (2048 B)" : "TIMEOUT", o[0], o[1], o[127], o[128], o[129],
           o[256], o[384], o[511]);
  }
  return 0;
}
