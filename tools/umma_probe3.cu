// umma_probe3: which shared-memory layouts does tcgen05.mma kind::tf32 accept
// as MN-major operands?  D = A B^T with A = B = X^T (X: K x M, M contiguous),
// checked against the exact Gram matrix; a K-major SW128 control first.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2110_14044_b200/csrc/ials_umma.cuh"
using namespace ials;
constexpr int M = 128, KX = 8;

struct Var {
  const char* name;
  int kmajor;        // operand layout: 1 = K-major SW128 (control), 0 = MN-major
  int swz;           // MN-major: 1 = SW128 atoms (32 MN x 8 K), 0 = interleave (4 MN x 8 K core)
  int a_mn, b_mn;    // idesc major bits
  uint32_t lbo, sbo; // descriptor byte offsets
  int lbo_mode;      // descriptor bit 52
};

// byte offset of element (m, k) for the layout family of v
__host__ __device__ inline int off_bytes(const Var& v, int m, int k) {
  if (v.kmajor) {
    const int r = m & 7;
    return ((m >> 3) * 256 + r * 32 + ((((k >> 2)) ^ r) << 2) + (k & 3)) * 4;
  }
  if (v.swz) {  // MN blocks of 32 at 1 KB, one k group (K = 8)
    const int r = k & 7, e = m & 31;
    return (m >> 5) * 1024 + r * 128 + ((((e >> 2) ^ r)) << 4) + (e & 3) * 4;
  }
  // interleave: core matrix = 8 K-rows x 16 B (4 MN), MN blocks of 4 at 128 B
  return (m >> 2) * 128 + (k & 7) * 16 + (m & 3) * 4;
}

__global__ void probe(const float* X, float* out, Var v) {
  __shared__ __align__(1024) float xs[4096];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 4096; i += blockDim.x) xs[i] = 0.f;
  __syncthreads();
  for (int i = t; i < KX * M; i += blockDim.x) {
    const int k = i / M, m = i % M;
    xs[off_bytes(v, m, k) / 4] = X[i];
  }
  if (t == 0) mbar_init(&bar, 1);
  if (w == 0) tmem_alloc(&tbase, 128);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (t == 0) {
    const uint32_t idesc = make_idesc_tf32(128, 128, v.a_mn, v.b_mn, 0);
    uint64_t a = make_sdesc(smem_u32(xs), v.lbo, v.sbo, v.kmajor || v.swz ? kSwizzle128B : kSwizzleNone);
    if (v.lbo_mode) a |= (uint64_t)1 << 52;
    umma_tf32(d, a, a, idesc, 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < 128; c += 8) {
    float r[8];
    tmem_ld8(d + ((uint32_t)(32 * w) << 16) + c, r);
    tmem_wait_ld();
    for (int j = 0; j < 8; ++j) out[t * 128 + c + j] = r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_free(tbase, 128);
}

int main() {
  const Var vars[] = {
      {"K-major SW128 control", 1, 1, 0, 0, 16, 1024, 0},
      {"MN SW128 lbo=1K sbo=4K", 0, 1, 1, 1, 1024, 4096, 0},
      {"MN SW128 lbo=4K sbo=1K", 0, 1, 1, 1, 4096, 1024, 0},
      {"MN SW128 lbo=1K sbo=1K", 0, 1, 1, 1, 1024, 1024, 0},
      {"MN SW128 lbo=1K sbo=4K mode1", 0, 1, 1, 1, 1024, 4096, 1},
      {"MN SW128 A only", 0, 1, 1, 0, 1024, 4096, 0},
      {"MN SW128 B only", 0, 1, 0, 1, 1024, 4096, 0},
      {"MN ilv lbo=4K sbo=128", 0, 0, 1, 1, 4096, 128, 0},
      {"MN ilv lbo=128 sbo=4K", 0, 0, 1, 1, 128, 4096, 0},
  };
  std::vector<float> X(KX * M), o(M * M);
  srand(1);
  for (auto& x : X) x = (float)(rand() % 7 - 3);
  float *dX, *dO;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dO, o.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  for (const Var& v : vars) {
    cudaMemset(dO, 0, o.size() * 4);
    probe<<<1, 128>>>(dX, dO, v);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%-32s: %s\n", v.name, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double s = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < M; ++j) {
        double g = 0;
        for (int k = 0; k < KX; ++k) g += (double)X[k * M + i] * X[k * M + j];
        s += std::fabs(o[i * M + j]);
        if (std::fabs(o[i * M + j] - g) > 1e-3) ++bad;
      }
    printf("%-32s: mismatches %5d  sum|D| %10.1f  D[0][0..3] %6.1f %6.1f %6.1f %6.1f\n", v.name, bad,
           s, o[0], o[1], o[2], o[3]);
  }
  return 0;
}
