// ials_rot.cuh -- the rotated user pass of the fused sweep (b = 128).
//
// Every row r of a side pass solves (X_r^T X_r + A_r) d = g_r with
// A_r = alpha0 G_pp + lam_r I, G_pp = F[:, pi]^T F[:, pi] shared by all rows.
// With G_pp = Q L Q^T (one symmetric eigendecomposition per block),
// A_r = Q D_r Q^T, D_r = alpha0 L + lam_r I diagonal, so in the rotated basis
// (X~ = X Q, g~ = Q^T g, d = Q d~) every row's regulariser is diagonal and a
// row with n_r < b interactions can be solved through its n_r x n_r
// Woodbury system (ials_sweep_wb.cuh) instead of the b x b one.
//
// k_sym_eig: cyclic Jacobi on one symmetric b x b matrix per CTA (fp32 in
// shared memory, round-robin parallel ordering: b/2 disjoint rotations per
// round, rows then columns then the eigenvector columns), to an off-diagonal
// Frobenius norm below 1e-6 of the matrix norm or 20 sweeps.  Outputs Q^T
// (row j = eigenvector j), the eigenvalues, and the rotated block template
// (diag(L) at rows b0.. of a d x b buffer: what the sweep kernels read as
// slab[pi, pi]).  The sweep uses the same Q for X~, g~ and d = Q d~; what
// perturbs the solve is the dropped off-diagonal part of Q^T G Q (~1e-6 of |G|)
// and Q^T Q - I in the lam I term, which two Newton-Schulz steps keep at fp32
// level.
#pragma once
#include "ials_common.cuh"

namespace ials {

constexpr int kEigThreads = 512;

// in: G (b x b, ld ldg) per matrix z at G + z * stride_g; out: QT (b x b),
// lam (b), tpl rows [b0_z, b0_z + b) of a (d x b) buffer (b0_z = z * b), Qm.
// Gprev (optional, b x b per matrix): the input the outputs in place were
// computed from; unless `force`, a bit-identical G returns at once (the
// outputs are already its decomposition: the result is the same as
// recomputing it, so runs stay bitwise reproducible), and a computed G is
// stored there.
__global__ void __launch_bounds__(kEigThreads, 1)
    k_sym_eig(const float* __restrict__ G, int ldg, long long stride_g, int b, float* QT,
              float* lam, float* tpl, float* Qm, float* Gprev, int force) {
  extern __shared__ float es[];
  const int n = b;                       // even (b = 128 in the rotated pass)
  const int ld = n + 1;                  // padded rows: column sweeps are bank-conflict free
  float* A = es;                         // n x ld
  float* V = A + n * ld;                 // n x ld
  float* cs = V + n * ld;                // [n/2][4]: p, q, c, s
  const int tid = threadIdx.x, z = blockIdx.x;
  const float* g = G + z * stride_g;
  float* gp = Gprev ? Gprev + (size_t)z * n * n : nullptr;
  __shared__ int same;
  if (gp && !force) {
    if (tid == 0) same = 1;
    __syncthreads();
    int mine = 1;
    for (int i = tid; i < n * n; i += kEigThreads)
      if (__float_as_uint(g[(size_t)(i / n) * ldg + i % n]) != __float_as_uint(gp[i])) mine = 0;
    if (!mine) same = 0;
    __syncthreads();
    if (same) return;
  }
  for (int i = tid; i < n * n; i += kEigThreads) {
    const int r = i / n, c = i - r * n;
    A[r * ld + c] = 0.5f * (g[(size_t)r * ldg + c] + g[(size_t)c * ldg + r]);
    V[r * ld + c] = (r == c) ? 1.f : 0.f;
    if (gp) gp[i] = g[(size_t)r * ldg + c];
  }
  __syncthreads();
  const int half = n / 2;
  for (int sweep = 0; sweep < 20; ++sweep) {
    // convergence: off-diagonal vs total Frobenius norm
    __shared__ float ro[kEigThreads / 32], rt[kEigThreads / 32];
    __shared__ int conv;
    float off = 0.f, tot = 0.f;
    for (int i = tid; i < n * n; i += kEigThreads) {
      const int r = i / n, c = i - r * n;
      const float v = A[r * ld + c] * A[r * ld + c];
      tot += v;
      if (r != c) off += v;
    }
    off = warp_sum(off);
    tot = warp_sum(tot);
    if ((tid & 31) == 0) {
      ro[tid >> 5] = off;
      rt[tid >> 5] = tot;
    }
    __syncthreads();
    if (tid == 0) {
      float o = 0.f, t = 0.f;
      for (int w = 0; w < kEigThreads / 32; ++w) {
        o += ro[w];
        t += rt[w];
      }
      conv = o <= 1e-12f * t;   // off-diagonal norm below 1e-6 of the matrix norm
    }
    __syncthreads();
    if (conv) break;
    for (int round = 0; round < n - 1; ++round) {
      if (tid < half) {   // round-robin pairing: (n-1, round), (round+j, round-j) mod n-1
        int pp, qq;
        if (tid == 0) {
          pp = n - 1;
          qq = round;
        } else {
          pp = (round + tid) % (n - 1);
          qq = (round - tid + (n - 1)) % (n - 1);
        }
        if (pp > qq) {
          const int t = pp;
          pp = qq;
          qq = t;
        }
        const float apq = A[pp * ld + qq], app = A[pp * ld + pp], aqq = A[qq * ld + qq];
        float c = 1.f, s = 0.f;
        if (fabsf(apq) > 1e-30f * (fabsf(app) + fabsf(aqq)) && apq != 0.f) {
          const float th = (aqq - app) / (2.f * apq);
          const float t = copysignf(1.f, th) / (fabsf(th) + sqrtf(fmaf(th, th, 1.f)));
          c = rsqrtf(fmaf(t, t, 1.f));
          s = t * c;
        }
        cs[4 * tid] = __int_as_float(pp);
        cs[4 * tid + 1] = __int_as_float(qq);
        cs[4 * tid + 2] = c;
        cs[4 * tid + 3] = s;
      }
      __syncthreads();
      // rows p, q of A (A <- J^T A)
      for (int w = tid; w < half * n; w += kEigThreads) {
        const int j = w / n, k = w - j * n;
        const int pp = __float_as_int(cs[4 * j]), qq = __float_as_int(cs[4 * j + 1]);
        const float c = cs[4 * j + 2], s = cs[4 * j + 3];
        const float ap = A[pp * ld + k], aq = A[qq * ld + k];
        A[pp * ld + k] = c * ap - s * aq;
        A[qq * ld + k] = s * ap + c * aq;
      }
      __syncthreads();
      // columns p, q of A and V (A <- A J, V <- V J)
      for (int w = tid; w < half * n; w += kEigThreads) {
        const int j = w / n, k = w - j * n;
        const int pp = __float_as_int(cs[4 * j]), qq = __float_as_int(cs[4 * j + 1]);
        const float c = cs[4 * j + 2], s = cs[4 * j + 3];
        const float ap = A[k * ld + pp], aq = A[k * ld + qq];
        A[k * ld + pp] = c * ap - s * aq;
        A[k * ld + qq] = s * ap + c * aq;
        const float vp = V[k * ld + pp], vq = V[k * ld + qq];
        V[k * ld + pp] = c * vp - s * vq;
        V[k * ld + qq] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  // The accumulated rotations drift from orthogonality (~5e-4 in |V^T V - I|_F
  // after a cold decomposition) and the solve needs Q^T Q = I for the lam I
  // term of every row's Hessian: two Newton-Schulz steps V <- V (3I - V^T V)/2
  // bring V back to fp32 orthogonality (the error squares each step).  A's
  // storage holds V^T V, then G again for the final eigenvalues.
  __shared__ float evals[256];
  for (int it = 0; it < 2; ++it) {
    // T = (3 I - V^T V) / 2 -> A's storage
    for (int i = tid; i < n * n; i += kEigThreads) {
      const int r = i / n, c = i - r * n;
      float acc = 0.f;
      for (int k = 0; k < n; ++k) acc = fmaf(V[k * ld + r], V[k * ld + c], acc);
      A[r * ld + c] = ((r == c) ? 1.5f : 0.f) - 0.5f * acc;
    }
    __syncthreads();
    // V <- V T, row by row: every output of a row is formed before the row is rewritten
    for (int r0 = 0; r0 < n; r0 += kEigThreads / n) {
      const int r = r0 + tid / n, c = tid % n;
      float acc = 0.f;
      if (r < n)
        for (int k = 0; k < n; ++k) acc = fmaf(V[r * ld + k], A[k * ld + c], acc);
      __syncthreads();
      if (r < n) V[r * ld + c] = acc;
      __syncthreads();
    }
  }
  // the eigenvalues of the final basis: diag(V^T G V), G reloaded (symmetrised)
  // into A's storage; thread t sums the rows r = t / n (mod 4 parts) of column t % n
  for (int i = tid; i < n * n; i += kEigThreads) {
    const int r = i / n, c = i - r * n;
    A[r * ld + c] = 0.5f * (g[(size_t)r * ldg + c] + g[(size_t)c * ldg + r]);
  }
  __syncthreads();
  {
    constexpr int PARTS = kEigThreads / 128;
    __shared__ float epart[kEigThreads];
    const int i = tid % n, part = tid / n;
    float acc = 0.f;
    if (tid < n * PARTS)
      for (int r = part; r < n; r += PARTS) {
        float gv = 0.f;
        for (int c = 0; c < n; ++c) gv = fmaf(A[r * ld + c], V[c * ld + i], gv);
        acc = fmaf(V[r * ld + i], gv, acc);
      }
    epart[tid] = acc;
    __syncthreads();
    if (tid < n) {
      float s = 0.f;
      for (int q = 0; q < PARTS; ++q) s += epart[q * n + tid];
      evals[tid] = s;
    }
    __syncthreads();
  }
  float* qt = QT + (size_t)z * n * n;
  for (int i = tid; i < n * n; i += kEigThreads) {
    const int j = i / n, k = i - j * n;   // QT[j][k] = V[k][j]
    qt[i] = V[k * ld + j];
  }
  if (Qm) {
    float* qm = Qm + (size_t)z * n * n;
    for (int i = tid; i < n * n; i += kEigThreads) qm[i] = V[(i / n) * ld + i % n];
  }
  if (tid < n) lam[(size_t)z * n + tid] = evals[tid];
  if (tpl) {
    float* tp = tpl + (size_t)z * n * n;   // rows b0 = z * b of the d x b template
    for (int i = tid; i < n * n; i += kEigThreads) {
      const int r = i / n, c = i - r * n;
      tp[i] = (r == c) ? evals[r] : 0.f;
    }
  }
}

// out[i] = sum_s part[s * stride + i], fixed split order (i < count)
__global__ void k_reduce_splits_strided(const float* __restrict__ part, int nsplit, long long stride,
                                        size_t count, float* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < nsplit; ++s) acc += part[s * stride + i];
    out[i] = acc;
  }
}

constexpr int eig_smem_bytes(int b) { return (2 * b * (b + 1) + 2 * b) * 4; }

}  // namespace ials
