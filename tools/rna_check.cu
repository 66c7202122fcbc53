#include <cstdio>
#include <cstdint>
#include <cstring>
__global__ void k(const float* x, unsigned* bad, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  float v = x[i]; uint32_t a; asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(a) : "f"(v));
  uint32_t b = (__float_as_uint(v) + 0x1000u) & 0xFFFFE000u;
  if (a != b) atomicAdd(bad, 1u);
}
int main() {
  const int n = 1 << 24; float* h = new float[n]; uint32_t s = 12345;
  for (int i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; uint32_t u = s;
    // random finite floats of all magnitudes / signs (exponents 1..253)
    uint32_t e = 1 + (u >> 8) % 253; u = (u & 0x807FFFFFu) | (e << 23); memcpy(&h[i], &u, 4); }
  float* d; unsigned* bad; cudaMalloc(&d, n * 4); cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice); k<<<n / 256, 256>>>(d, bad, n);
  unsigned hb; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost); printf("mismatches %u of %d\n", hb, n); }
