// ials_abi.cu -- C ABI of libials_b200.so (see include/ials_b200.h).
//
// Host-side launch logic for the iALS++ kernels.  Everything here is
// stream-ordered and allocation-free (scratch comes from the caller's
// workspace); the only device allocation is the session's error word.
#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <functional>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "../../include/ials_b200.h"
#include "ials_common.cuh"
#include "ials_dense.cuh"
#include "ials_csr.cuh"
#include "ials_topk.cuh"
#include "ials_sweep.cuh"
#include "ials_loss.cuh"
#include "ials_sweep_tc4.cuh"
#include "ials_sweep_pk.cuh"
#include "ials_rot.cuh"
#include "ials_sweep_wb.cuh"
#include "ials_gemm_tc.cuh"
#include "ials_sweep_b1.cuh"
#include "ials_sweep_wide.cuh"
#include "ials_sweep_w32.cuh"
#include "ials_sweep_w32m.cuh"
#include "ials_sweep_w16.cuh"
#include "ials_sweep_w16m.cuh"
#include "ials_heavy_w.cuh"
#include "ials_heavy_w64.cuh"

using namespace ials;

struct ials_session {
  int device;
  cudaStream_t copy_st = nullptr;             // ials_epoch_host: host <-> device staging
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  cudaStream_t aux_st = nullptr;              // heavy-row partials beside the light rows
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t rot_st = nullptr;              // the epoch's eigendecompositions beside the predictions
  cudaEvent_t ev_rot0 = nullptr, ev_rot1 = nullptr;
  cudaEvent_t ev_blk[64] = {};                // per block: its decomposition is ready
  const float* rot_qm = nullptr;              // where this session's last rotated epoch left its
  long long rot_key = 0;                      //   decompositions (and their inputs), and for what shape
  unsigned long long* err;  // device error word (ULLONG_MAX = clean)
  unsigned long long* redo; // rows the fused tensor-core sweep handed to SIMT
  const struct ChunkPlan* chunk = nullptr;   // set by ials_epoch_host around its first user pass
  // ials_epoch: a pass's entry-parallel cache update runs on its own stream beside
  // the NEXT pass's GEMM phase (slab, projection, K-major copies: none of them
  // touches the cache or the pass's per-row steps); the next sweep joins it
  cudaStream_t cache_st = nullptr;
  cudaEvent_t ev_cache_go = nullptr, ev_cache_done = nullptr;
  bool defer_cache = false;     // set by the epoch around a side pass whose layout allows it
  bool cache_pending = false;   // a deferred cache update has not been joined yet
  float* last_drow = nullptr;   // the per-row steps of the last side pass (the back-rotation's input)
  char msg[512];
};

// ials_epoch_host's first user pass: the light rows grouped by row chunk
// (stable, so each chunk keeps the longest-first order), and a prologue that
// queues chunk c's W copy, predictions and projection before its sweep
struct ChunkPlan {
  int nch;
  const int* rows;   // grouped light rows (device)
  const int* tot;    // rows per chunk (device)
  std::function<int(int)> prologue;
};


// Every entry point that takes a session runs on the session's device and
// restores the caller's current device on return (torch keeps its own notion
// of the current device; a session created for GPU 1 must not leave the
// thread on GPU 1, nor launch on GPU 0 when the caller's current device is 0).
struct DevGuard {
  int prev = -1, want = -1;
  explicit DevGuard(const ials_session* s);
  ~DevGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

static thread_local char g_msg[512];

static int fail(ials_session* s, int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  char* dst = s ? s->msg : g_msg;
  vsnprintf(dst, 512, fmt, ap);
  va_end(ap);
  return code;
}

#define CUDA_TRY(s, expr)                                                             \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return fail((s), IALS_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e),  \
                  __FILE__, __LINE__);                                                \
  } while (0)

// every kernel launch of the library is followed by exactly one LAUNCH_CHECK,
// which also counts it (ials_launch_count)
static std::atomic<long long> g_launches{0};

#define LAUNCH_CHECK(s)                                                               \
  do {                                                                                \
    g_launches.fetch_add(1, std::memory_order_relaxed);                               \
    cudaError_t _e = cudaGetLastError();                                              \
    if (_e != cudaSuccess)                                                            \
      return fail((s), IALS_E_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                \
  } while (0)


DevGuard::DevGuard(const ials_session* s) {
  if (!s) return;
  want = s->device;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  if (prev != want) cudaSetDevice(want);
}

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

int64_t ials_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
static inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

static bool tc4_enabled();
static bool w16_enabled();
static bool hw_enabled();
// Register/shared tile width of a block of b columns.  With the fused
// tensor-core sweep (the default) widths 33..64 also use the 128 tile (the
// padding is idle tensor-core work; the factorisation chain is half of the
// SIMT sweep's), under a stricter cancellation guard (tc_cond_for).
static int block_tile(int b) {
  if (b <= 8) return 8;
  if (b <= 16) return 16;
  if (b <= 32) return tc4_enabled() ? 128 : 32;   // packed tensor-core sweep, 4 rows per tile
  if (b <= 64) return tc4_enabled() ? 128 : 64;   // packed tensor-core sweep, 2 rows per tile
  if (b <= 128) return 128;
  return 256;
}

static constexpr int kMaxSplits = 64;

// Exported functions get C linkage from their declarations in ials_b200.h.

int ials_version(void) { return 1; }

int ials_session_create(int device, ials_session** out) {
  if (!out) return fail(nullptr, IALS_E_INVALID, "out is NULL");
  ials_session* s = new ials_session();
  s->device = device;
  s->msg[0] = 0;
  int prev = -1;
  if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(&s->err, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(s->err, 0xFF, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMalloc(&s->redo, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(s->redo, 0, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    fail(nullptr, IALS_E_CUDA, "session create: %s", cudaGetErrorString(e));
    delete s;
    if (prev >= 0) cudaSetDevice(prev);
    return IALS_E_CUDA;
  }
  if (prev >= 0 && prev != device) cudaSetDevice(prev);
  *out = s;
  return IALS_OK;
}

int ials_session_destroy(ials_session* s) {
  if (!s) return IALS_OK;
  DevGuard _dg(s);
  cudaFree(s->err);
  cudaFree(s->redo);
  if (s->copy_st) cudaStreamDestroy(s->copy_st);
  if (s->aux_st) cudaStreamDestroy(s->aux_st);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  if (s->rot_st) cudaStreamDestroy(s->rot_st);
  if (s->ev_rot0) cudaEventDestroy(s->ev_rot0);
  if (s->ev_rot1) cudaEventDestroy(s->ev_rot1);
  for (cudaEvent_t e : s->ev_blk)
    if (e) cudaEventDestroy(e);
  if (s->ev_a) cudaEventDestroy(s->ev_a);
  if (s->ev_b) cudaEventDestroy(s->ev_b);
  delete s;
  return IALS_OK;
}

int ials_last_error(ials_session* s, char* buf, size_t len) {
  if (!buf || len == 0) return IALS_E_INVALID;
  const char* m = s ? s->msg : g_msg;
  strncpy(buf, m, len - 1);
  buf[len - 1] = 0;
  return IALS_OK;
}

int ials_reset_singular(ials_session* s, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  CUDA_TRY(s, cudaMemsetAsync(s->err, 0xFF, sizeof(unsigned long long), S(stream)));
  return IALS_OK;
}

int ials_tc_redo_rows(ials_session* s, void* stream, int64_t* total, int32_t reset) {
  DevGuard _dg(s);
  if (!s || !total) return fail(s, IALS_E_INVALID, "tc_redo_rows: NULL argument");
  unsigned long long v = 0;
  CUDA_TRY(s, cudaMemcpyAsync(&v, s->redo, sizeof(v), cudaMemcpyDeviceToHost, S(stream)));
  if (reset) CUDA_TRY(s, cudaMemsetAsync(s->redo, 0, sizeof(v), S(stream)));
  CUDA_TRY(s, cudaStreamSynchronize(S(stream)));
  *total = static_cast<int64_t>(v);
  return IALS_OK;
}

int ials_check_singular(ials_session* s, void* stream, int64_t* row, int32_t* pivot,
                        int32_t* side) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  unsigned long long key = 0;
  CUDA_TRY(s, cudaMemcpyAsync(&key, s->err, sizeof(key), cudaMemcpyDeviceToHost, S(stream)));
  CUDA_TRY(s, cudaStreamSynchronize(S(stream)));
  if (key == ~0ull) return IALS_OK;
  const int sd = static_cast<int>(key >> 62);
  const int64_t r = static_cast<int64_t>((key >> 24) & 0xFFFFFFFFull);
  const int pv = static_cast<int>(key & 0xFFFFFF);
  if (row) *row = r;
  if (pivot) *pivot = pv;
  if (side) *side = sd;
  return fail(s, IALS_E_SINGULAR, "normal equations singular for %s row %lld (pivot %d)",
              sd == 0 ? "user" : "item", (long long)r, pv);
}

// Rows longer than the threshold are split into slices (partial Hessians
// reduced in a fixed order): a one-warp row team at small block widths is
// latency-bound on long rows, so it splits them early.
// (IALS_HEAVY / IALS_SLICE override both for every width: measurements)
int64_t ials_heavy_threshold(int32_t b) {
  static const long long ov = getenv("IALS_HEAVY") ? atoll(getenv("IALS_HEAVY")) : 0;
  if (ov > 0) return ov;
  const int bt = block_tile(b);
  // narrow blocks in the 128 tile: a long row is one warp's (b <= 32, the
  // warp-per-row sweep) or one tile slot's serial chain, while its slices spread
  // over the machine (measured at the configs[1] / [2] shapes: 512 at b = 32,
  // 15.6 -> 11.1 ms with the warp-per-row sweep; 2048 at b = 64)
  if (bt == 128 && b <= 32) return 512;
  if (bt == 128 && b <= 64) return 2048;
  return bt <= 16 ? 512 : bt == 32 ? 1024 : 4096;
}
int64_t ials_slice_len(int32_t b) {
  static const long long ov = getenv("IALS_SLICE") ? atoll(getenv("IALS_SLICE")) : 0;
  if (ov > 0) return ov;
  const int bt = block_tile(b);
  // (b <= 16 with the half-warp slice kernel and the parallel slice reduction of
  // ials_heavy_w.cuh: a 1024-entry slice is a 240 us serial chain, 256 stays)
  return bt <= 16 ? 256 : bt == 32 ? 512 : (bt == 256 ? 1024 : 2048);
}

static constexpr int kGemvSplits = 4 * 148;   // b <= 4: one GEMV split per 64+ rows

static size_t gram_ws(int32_t n, int32_t d, int32_t b) {
  (void)n;
  const size_t narrow = b <= 4 ? size_t(kGemvSplits) * d * b : 0;
  size_t splits = kMaxSplits;
  if (b > 256) {   // wide blocks: many 64 x 64 output tiles, few splits (gramian_impl's rule)
    const size_t tiles = size_t((d + GT - 1) / GT) * ((b + GT - 1) / GT);
    splits = std::min<size_t>(kMaxSplits, std::max<size_t>(1, (2 * kNumSMs + tiles - 1) / tiles));
  }
  return al256(std::max(splits * d * b, narrow) * sizeof(float));
}

// ---- wide blocks (b > 256, ials_sweep_wide.cuh): the rows of a pass are taken
// in batches whose normal equations live in the workspace
static int wide_min() {   // narrowest block taking the wide pass (IALS_WIDE_MIN: measurements)
  static const int v = getenv("IALS_WIDE_MIN") ? std::max(65, atoi(getenv("IALS_WIDE_MIN"))) : 257;
  return v;
}
static inline int wide_lda(int b) { return (b + 3) & ~3; }
static inline size_t wide_mat_floats(int b) { return size_t(b + 1) * wide_lda(b); }
static int wide_batch(int b) {   // rows per batch: a multiple of the SM count, <= 6 GB
  const size_t per = wide_mat_floats(b) * 4;
  const size_t fit = (size_t(6) << 30) / per;
  return (int)std::min<size_t>(8 * kNumSMs, std::max<size_t>(kNumSMs, fit / kNumSMs * kNumSMs));
}
static size_t wide_ws(int32_t n_rows, int32_t b) {
  const size_t R = std::min<size_t>(wide_batch(b), std::max(n_rows, 1));
  return 2 * al256(size_t(n_rows) * b * 4) + al256(R * wide_mat_floats(b) * 4);
}



// narrow blocks gather from a compact copy of the fixed side's column block
// (n_fixed x ldc): L2-resident, unlike the full d-wide rows
static constexpr int kCompactMaxB = 32;
static inline int compact_ld(int b) { return (b + 3) & ~3; }

static size_t pass_ws(int32_t n_rows, int32_t n_fixed, int32_t b, int32_t n_slices, int32_t n_heavy) {
  if (b >= wide_min()) return wide_ws(n_rows, b);
  const size_t bt = block_tile(b);
  return al256(size_t(n_rows) * b * 4) + al256(size_t(n_slices) * bt * bt * 4) +
         al256(size_t(n_slices) * bt * 8) + al256(size_t(n_heavy) * bt * 4) +
         al256(size_t(kTcPKS) * 4) + al256(size_t(n_rows) * 4 + 32) +
         al256(size_t(n_rows) * b * 4) +
         (b <= kCompactMaxB ? al256(size_t(n_fixed) * compact_ld(b) * 4) : 0);
}

size_t ials_workspace_bytes(int32_t n_rows_max, int32_t n_fixed_max, int32_t d, int32_t b,
                            int32_t n_slices_max, int32_t n_heavy_max) {
  // epoch layout: [slab d*b][gram partials][pass scratch]; loss needs at most
  // 2 d x d gramians + partials, covered separately by ials_loss_workspace.
  return al256(size_t(d) * b * 4) + gram_ws(std::max(n_rows_max, n_fixed_max), d, b) +
         pass_ws(std::max(n_rows_max, n_fixed_max), std::max(n_rows_max, n_fixed_max), b,
                 n_slices_max, n_heavy_max);
}

// ------------------------------------------------------------------ predictions
template <int LPN>
static void launch_pred_lpn(int nv, dim3 g, dim3 t, cudaStream_t st, int n_items, Items it,
                            const int* cols, const float* W, int ldw, const float* H, int ldh,
                            int d, float* out) {
  switch (nv) {
    case 1: k_pred_vec<LPN, 1><<<g, t, 0, st>>>(n_items, it, cols, W, ldw, H, ldh, d, out); break;
    case 2: k_pred_vec<LPN, 2><<<g, t, 0, st>>>(n_items, it, cols, W, ldw, H, ldh, d, out); break;
    case 4: k_pred_vec<LPN, 4><<<g, t, 0, st>>>(n_items, it, cols, W, ldw, H, ldh, d, out); break;
    case 8: k_pred_vec<LPN, 8><<<g, t, 0, st>>>(n_items, it, cols, W, ldw, H, ldh, d, out); break;
    default: k_pred_vec<LPN, 16><<<g, t, 0, st>>>(n_items, it, cols, W, ldw, H, ldh, d, out); break;
  }
}

static int predictions_impl(ials_session* s, int32_t n_items, Items it, const int32_t* cols,
                            const float* W, int32_t ldw, const float* H, int32_t ldh, int32_t d,
                            float* out, void* stream);

int ials_predictions(ials_session* s, int32_t n_rows, const int32_t* ptr, const int32_t* cols,
                     const float* W, int32_t ldw, const float* H, int32_t ldh, int32_t d,
                     float* out, void* stream) {
  DevGuard _dg(s);
  if (n_rows < 0) return fail(s, IALS_E_INVALID, "predictions: n_rows < 0");
  return predictions_impl(s, n_rows, Items{ptr, nullptr, nullptr, nullptr}, cols, W, ldw, H, ldh,
                          d, out, stream);
}

int ials_predictions_segments(ials_session* s, int32_t n_seg, const int32_t* seg_row,
                              const int32_t* seg_beg, const int32_t* seg_end, const int32_t* cols,
                              const float* W, int32_t ldw, const float* H, int32_t ldh, int32_t d,
                              float* out, void* stream) {
  DevGuard _dg(s);
  if (n_seg < 0 || (n_seg > 0 && (!seg_row || !seg_beg || !seg_end)))
    return fail(s, IALS_E_INVALID, "predictions_segments: bad segment list");
  return predictions_impl(s, n_seg, Items{nullptr, seg_row, seg_beg, seg_end}, cols, W, ldw, H,
                          ldh, d, out, stream);
}

static int predictions_impl(ials_session* s, int32_t n_rows, Items it, const int32_t* cols,
                            const float* W, int32_t ldw, const float* H, int32_t ldh, int32_t d,
                            float* out, void* stream) {
  if (d < 1 || ldw < d || ldh < d)
    return fail(s, IALS_E_INVALID, "predictions: bad shape (d=%d)", d);
  if (n_rows == 0) return IALS_OK;
  const int warps_needed = n_rows;
  const int blocks = std::min((warps_needed + 7) / 8, kNumSMs * 16);
  const bool vec = (d % 4 == 0) && (ldw % 4 == 0) && (ldh % 4 == 0) && d <= 2048 &&
                   (reinterpret_cast<uintptr_t>(W) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(H) % 16 == 0);
  if (vec) {
    const int d4 = d / 4;
    int lpn = 1;
    while (lpn * 2 <= std::max(1, d4 / 4) && lpn < 32) lpn *= 2;
    int nv = (d4 + lpn - 1) / lpn;
    int nvp = 1;
    while (nvp < nv) nvp *= 2;
    if (nvp > 16) { lpn = 32; nvp = 16; }
    dim3 g(blocks), t(256);
    switch (lpn) {
      case 1: launch_pred_lpn<1>(nvp, g, t, S(stream), n_rows, it, cols, W, ldw, H, ldh, d, out); break;
      case 2: launch_pred_lpn<2>(nvp, g, t, S(stream), n_rows, it, cols, W, ldw, H, ldh, d, out); break;
      case 4: launch_pred_lpn<4>(nvp, g, t, S(stream), n_rows, it, cols, W, ldw, H, ldh, d, out); break;
      case 8: launch_pred_lpn<8>(nvp, g, t, S(stream), n_rows, it, cols, W, ldw, H, ldh, d, out); break;
      case 16: launch_pred_lpn<16>(nvp, g, t, S(stream), n_rows, it, cols, W, ldw, H, ldh, d, out); break;
      default: launch_pred_lpn<32>(nvp, g, t, S(stream), n_rows, it, cols, W, ldw, H, ldh, d, out); break;
    }
  } else {
    k_pred_scalar<<<blocks, 256, 0, S(stream)>>>(n_rows, it, cols, W, ldw, H, ldh, d, out);
  }
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// ------------------------------------------------------------------ correction
int ials_cache_correct(ials_session* s, int32_t n_seg, const int32_t* seg_row,
                       const int32_t* seg_beg, const int32_t* seg_end, const int32_t* cols,
                       const float* A, int32_t lda, int32_t b0, const float* D, int32_t ldd,
                       int32_t b, float* out, void* stream) {
  DevGuard _dg(s);
  if (n_seg < 0 || b < 1 || b > 256 || b0 < 0 || lda < b0 + b || ldd < b)
    return fail(s, IALS_E_INVALID, "cache_correct: bad shape (b0=%d b=%d)", b0, b);
  if (n_seg == 0) return IALS_OK;
  const int blocks = std::min((n_seg + 7) / 8, kNumSMs * 16);
  const bool vec = b <= 128 && b % 4 == 0 && b0 % 4 == 0 && lda % 4 == 0 && ldd % 4 == 0 &&
                   reinterpret_cast<uintptr_t>(A) % 16 == 0 && reinterpret_cast<uintptr_t>(D) % 16 == 0;
  if (vec)
    k_cache_correct_v<<<blocks, 256, 0, S(stream)>>>(n_seg, Items{nullptr, seg_row, seg_beg, seg_end},
                                                     cols, A, lda, b0, D, ldd, b, out);
  else
    k_cache_correct<<<blocks, 256, 0, S(stream)>>>(n_seg, Items{nullptr, seg_row, seg_beg, seg_end},
                                                   cols, A, lda, b0, D, ldd, b, out);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// ------------------------------------------------------------------ gramian
static int gramian_impl(ials_session* s, const float* M, int32_t n, int32_t ldm, int32_t d,
                        int32_t b0, int32_t b, float* slab, float* part, size_t part_bytes,
                        cudaStream_t st) {
  const int tiles = ((d + GT - 1) / GT) * ((b + GT - 1) / GT);
  int nsplit = std::max(1, (2 * kNumSMs + tiles - 1) / tiles);
  nsplit = std::min(nsplit, std::max(1, (n + 255) / 256));
  nsplit = std::min(nsplit, kMaxSplits);
  while (nsplit > 1 && size_t(nsplit) * d * b * 4 > part_bytes) --nsplit;
  if (size_t(nsplit) * d * b * 4 > part_bytes)
    return fail(s, IALS_E_NOMEM, "partial_gramian: workspace too small");
  int rps = (n + nsplit - 1) / nsplit;
  rps = ((rps + GK - 1) / GK) * GK;
  if (n == 0) {
    CUDA_TRY(s, cudaMemsetAsync(slab, 0, size_t(d) * b * 4, st));
    return IALS_OK;
  }
  if (b <= 4) {  // GEMV: thread per column, split-K over rows (bandwidth-bound)
    const int ct = (d + 255) / 256;
    int ns = std::max(1, std::min((4 * kNumSMs + ct - 1) / ct, (n + 63) / 64));
    ns = std::min(ns, kGemvSplits);
    while (ns > 1 && size_t(ns) * d * b * 4 > part_bytes) --ns;
    nsplit = ns;
    rps = (n + nsplit - 1) / nsplit;
    nsplit = (n + rps - 1) / rps;
    dim3 g(ct, nsplit);
    switch (b) {
      case 1: k_slab_gemv<1><<<g, 256, 0, st>>>(M, n, ldm, d, b0, rps, part); break;
      case 2: k_slab_gemv<2><<<g, 256, 0, st>>>(M, n, ldm, d, b0, rps, part); break;
      case 3: k_slab_gemv<3><<<g, 256, 0, st>>>(M, n, ldm, d, b0, rps, part); break;
      default: k_slab_gemv<4><<<g, 256, 0, st>>>(M, n, ldm, d, b0, rps, part); break;
    }
  } else if (b <= 16) {  // narrow 128 x 16 tiles: no wasted 64-wide tile columns
    const int ct = (d + 127) / 128;
    int ns = std::max(1, std::min(2 * kNumSMs / ct, (n + 255) / 256));
    ns = std::min(ns, kMaxSplits);
    while (ns > 1 && size_t(ns) * d * b * 4 > part_bytes) --ns;
    nsplit = ns;
    rps = (n + nsplit - 1) / nsplit;
    rps = ((rps + 31) / 32) * 32;
    nsplit = (n + rps - 1) / rps;
    dim3 g(ct, nsplit);
    k_slab_narrow<<<g, 256, 0, st>>>(M, n, ldm, d, b0, b, rps, part);
  } else {
    dim3 g((d + GT - 1) / GT, (b + GT - 1) / GT, nsplit);
    k_slab_partial<<<g, 256, 0, st>>>(M, n, ldm, d, b0, b, rps, part);
  }
  LAUNCH_CHECK(s);
  const size_t cnt = size_t(d) * b;
  if (nsplit > 64 && cnt < (size_t(1) << 26)) {
    k_reduce_splits_warp<<<(unsigned)((cnt + 7) / 8), 256, 0, st>>>(part, nsplit, (int)cnt, slab);
  } else {
    const int rb = (int)std::min<size_t>((cnt + 255) / 256, 4096);
    k_reduce_splits<<<rb, 256, 0, st>>>(part, nsplit, cnt, slab);
  }
  LAUNCH_CHECK(s);
  return IALS_OK;
}

int ials_partial_gramian(ials_session* s, const float* M, int32_t n, int32_t ldm, int32_t d,
                         int32_t b0, int32_t b, float* slab, void* workspace, size_t ws_bytes,
                         void* stream) {
  DevGuard _dg(s);
  if (n < 0 || d < 1 || ldm < d || b < 1 || b0 < 0 || b0 + b > d)
    return fail(s, IALS_E_INVALID, "partial_gramian: bad shape (n=%d d=%d b0=%d b=%d)", n, d,
                b0, b);
  return gramian_impl(s, M, n, ldm, d, b0, b, slab, static_cast<float*>(workspace), ws_bytes,
                      S(stream));
}

// Kernel attributes (dynamic shared memory, carveout) are per device: the
// one-time setups below are tracked per device so that sessions of one
// process on several GPUs each get them.
static unsigned dev_bit() {
  int d = 0;
  cudaGetDevice(&d);
  return 1u << (d & 31);
}

// ------------------------------------------------------------------ rotation
static int g_rot = -1;   // -1: not yet read from IALS_ROT
static bool rot_enabled() {
  if (g_rot < 0) {
    const char* e = getenv("IALS_ROT");
    g_rot = (e && e[0] == '0') ? 0 : 1;
  }
  return g_rot == 1;
}
int ials_set_rotation(int enable) {
  rot_enabled();
  const int prev = g_rot;
  g_rot = enable ? 1 : 0;
  return prev;
}

static int eig_attrs(ials_session* s, int b) {
  static unsigned init = 0;
  if (!(init & dev_bit())) {
    CUDA_TRY(s, cudaFuncSetAttribute(k_sym_eig, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     eig_smem_bytes(128)));
    init |= dev_bit();
  }
  (void)b;
  return IALS_OK;
}

int ials_sym_eig(ials_session* s, int32_t n_mat, int32_t b, const float* A, int32_t lda,
                 int64_t stride, float* QT, float* lam, float* Q, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (n_mat < 0 || b < 2 || b > 128 || (b & 1) || lda < b || !A || !QT || !lam)
    return fail(s, IALS_E_INVALID, "sym_eig: bad arguments (b=%d, even, <= 128)", b);
  if (n_mat == 0) return IALS_OK;
  int rc = eig_attrs(s, b);
  if (rc) return rc;
  k_sym_eig<<<n_mat, kEigThreads, eig_smem_bytes(b), S(stream)>>>(A, lda, stride, b, QT, lam, nullptr, Q,
                                                                    nullptr, 1);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// ------------------------------------------------------------------ side pass
template <int BT>
static int set_smem_attrs(ials_session* s) {
  static unsigned done = 0;
  if (done & dev_bit()) return IALS_OK;
  const int bytes = Lay<BT>::CTA_BYTES;
  CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_light<BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CUDA_TRY(s, cudaFuncSetAttribute(k_heavy_partial<BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CUDA_TRY(s, cudaFuncSetAttribute(k_heavy_solve<BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CUDA_TRY(s, cudaFuncSetAttribute(k_heavy_solve<BT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CUDA_TRY(s, cudaFuncSetAttribute(k_heavy_solve<BT, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CUDA_TRY(s, cudaFuncSetAttribute(k_heavy_cache<BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done |= dev_bit();
  return IALS_OK;
}

static long long* g_dbg = nullptr;  // profiling: per-CTA phase timestamps
int ials_debug_timestamps(void* dev_buf) {
  g_dbg = static_cast<long long*>(dev_buf);
  return IALS_OK;
}

static int g_tc = -1;  // -1: not yet read from IALS_TC
// 2 (default): the fused tensor-core sweeps for b in 17..128; 0: the FP32
// SIMT sweep everywhere (IALS_TC=0).  (The round-1 mode 1 -- three kernels per
// wave of rows -- was slower than the fused sweep and is gone; 1 means 2.)
static bool tc4_enabled() {
  if (g_tc < 0) {
    const char* e = getenv("IALS_TC");
    g_tc = (e && e[0] == '0') ? 0 : 2;
  }
  return g_tc == 2;
}
static float g_cond = 0.f;
static float tc_cond_max() {
  if (g_cond == 0.f) {
    const char* e = getenv("IALS_TC_COND");
    g_cond = e ? static_cast<float>(atof(e)) : 256.f;
    if (!(g_cond > 1.f)) g_cond = 256.f;
  }
  return g_cond;
}

float ials_set_tc_cond_max(float v) {
  const float prev = tc_cond_max();
  if (v > 1.f) g_cond = v;
  return prev;
}
int ials_set_tensor_cores(int enable) {
  tc4_enabled();
  const int prev = g_tc;
  g_tc = enable ? 2 : 0;
  return prev;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encode(ials_session* s) {
  if (g_encode) return IALS_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUDA_TRY(s, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess)
    return fail(s, IALS_E_CUDA, "cuTensorMapEncodeTiled is unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return IALS_OK;
}

// 2-D fp32 map: `inner` contiguous elements per row, `rows` rows ld_floats
// apart; boxes of 32 x box_rows land 128B-swizzled (K-major operand rows)
static int make_map(ials_session* s, CUtensorMap* m, const float* ptr, uint64_t inner, uint64_t rows,
                    uint64_t ld_floats, uint32_t box_rows) {
  cuuint64_t gdim[2] = {inner, rows};
  cuuint64_t gstr[1] = {ld_floats * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), gdim,
                              gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(s, IALS_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return IALS_OK;
}

// rows of `fixed` (n_fixed x d, ld ldf) in boxes of 128 columns x 1 row: the
// tile::gather4 source of the fused sweep (out-of-range columns read as 0)
static int make_gather_map(ials_session* s, CUtensorMap* m, const float* ptr, uint64_t d, uint64_t rows,
                           uint64_t ld_floats, uint32_t box_w = 128) {
  cuuint64_t gdim[2] = {d, rows};
  cuuint64_t gstr[1] = {ld_floats * 4};
  cuuint32_t box[2] = {box_w, 1};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), gdim,
                              gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(s, IALS_E_CUDA, "cuTensorMapEncodeTiled (gather) failed (%d)", (int)r);
  return IALS_OK;
}

// BT = 128, b > 32: fused tensor-core light rows (k_sweep_tc4, 4 CTAs/SM),
// heavy rows on the SIMT slice kernels.
// the caller's stream waits for a deferred cache update (see ials_session)
static int join_cache(ials_session* s, cudaStream_t st) {
  if (s->cache_pending) {
    CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_cache_done, 0));
    s->cache_pending = false;
  }
  return IALS_OK;
}

// b 17..32: the warp-per-row FP32 sweep instead of the packed tensor-core one
// (IALS_W32=0 keeps the packed sweep)
static bool w32_enabled() {
  static const bool on = !(getenv("IALS_W32") && getenv("IALS_W32")[0] == '0');
  return on;
}

// b 4..16: the two-rows-per-warp FP32 sweep instead of the generic SIMT one
// (IALS_W16=0 keeps k_sweep_light<8 | 16>)
static bool w16_enabled() {
  static const bool on = !(getenv("IALS_W16") && getenv("IALS_W16")[0] == '0');
  return on;
}

// heavy-row slices of b <= 32 in the warp-per-row register layout
// (ials_heavy_w.cuh; IALS_HW=0 keeps k_heavy_partial<bt> / k_heavy_partial_pk<4>)
static bool hw_enabled() {
  static const bool on = !(getenv("IALS_HW") && getenv("IALS_HW")[0] == '0');
  return on;
}
// (IALS_W_MMA=0: the FP32 SIMT tiles instead of the warp-level 3xTF32 MMA tiles, in the
// b <= 16 sweep and in the slice kernels; IALS_W32_MMA=0 the same for the b 17..32 sweep)
// Cancellation limit (H_kk / pivot_k) of the warp-level MMA sweeps: their factorisation is
// FP32 and only the 3xTF32 Hessian carries an error (~1e-6 of its entries), so the limit
// sits above the packed tcgen05 sweep's 16 (whose trailing updates are 3xTF32 as well)
static constexpr float kWarpCond = 64.f;
static bool wmma_enabled() {
  static const bool on = !(getenv("IALS_W_MMA") && getenv("IALS_W_MMA")[0] == '0');
  return on;
}
template <int NB>
static int launch_heavy_w(ials_session* s, const SweepParams& p, int bt, cudaStream_t st) {
  const bool mma = wmma_enabled();
  const bool unit = !p.side.weights && !p.side.labels;
  auto kern = mma ? (unit ? k_heavy_partial_wm<NB, true> : k_heavy_partial_wm<NB, false>)
                  : (unit ? k_heavy_partial_w<NB, true> : k_heavy_partial_w<NB, false>);
  const int bytes = mma ? WHmLay<NB>::BYTES : WHLay<NB>::BYTES;
  static int per_sm = 0;
  static unsigned init = 0;
  if (!(init & dev_bit())) {
    CUDA_TRY(s, cudaFuncSetAttribute(k_heavy_partial_w<NB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, WHLay<NB>::BYTES));
    CUDA_TRY(s, cudaFuncSetAttribute(k_heavy_partial_w<NB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, WHLay<NB>::BYTES));
    CUDA_TRY(s, cudaFuncSetAttribute(k_heavy_partial_wm<NB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, WHmLay<NB>::BYTES));
    CUDA_TRY(s, cudaFuncSetAttribute(k_heavy_partial_wm<NB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, WHmLay<NB>::BYTES));
    init |= dev_bit();
  }
  if (per_sm == 0) {
    CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WHLay<NB>::NT, bytes));
    if (per_sm < 1) per_sm = 1;
  }
  const int per_cta = WHLay<NB>::NW * WHLay<NB>::G;
  const int grid = std::min((p.n_slices + per_cta - 1) / per_cta, per_sm * kNumSMs);
  kern<<<grid, WHLay<NB>::NT, bytes, st>>>(p, bt);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

static int wb_attrs(ials_session* s) {
  static unsigned winit = 0;
  if (!(winit & dev_bit())) {
    CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_wb<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, WbLay<2>::BYTES));
    CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_wb<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, WbLay<4>::BYTES));
    CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_wb<2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_wb<4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    winit |= dev_bit();
  }
  return IALS_OK;
}

static int launch_sweep_tc4(ials_session* s, const SweepParams& p, long long nnz, cudaStream_t st) {
  using L = Lay<128>;
  const bool unit = !p.side.weights && !p.side.labels;   // all ones: not staged
  int rc = set_smem_attrs<128>(s);
  if (rc) return rc;
  // [0] redo count, [1] slice queue, [2] light-row queue, [4] redo queue,
  // [5] / [6] the Woodbury tiles' queues (rotated user pass)
  CUDA_TRY(s, cudaMemsetAsync(p.redo_cnt, 0, 8 * sizeof(int), st));
  // sub-row gathers by TMA (tile::gather4) when the fixed matrix allows it
  CUtensorMap fmap;
  memset(&fmap, 0, sizeof(fmap));
  int use_tma = 0;
  // light rows: the fused sweep (b 65..128) or the packed one (b 17..64: G
  // rows per 128-lane tile, slot width 128 / G), boxes of the slot width
  const int G = p.b > 64 ? 1 : (p.b > 32 ? 2 : 4);
  // (the map's extent is the fixed matrix's own width: p.ldf columns when the
  // pass gathers from a compact column copy, d otherwise)
  const uint64_t fcols = (uint64_t)p.fixed_cols;
  if (p.vec && p.side.n_fixed > 0 && get_encode(s) == IALS_OK &&
      make_gather_map(s, &fmap, p.fixed, fcols, p.side.n_fixed, p.ldf, 128 / G) == IALS_OK)
    use_tma = 1;
  CUtensorMap hmap;   // heavy-row partials: the 128-wide tile
  memset(&hmap, 0, sizeof(hmap));
  int use_tma_h = use_tma;
  if (use_tma && G > 1)
    use_tma_h = make_gather_map(s, &hmap, p.fixed, fcols, p.side.n_fixed, p.ldf, 128) == IALS_OK;
  else
    hmap = fmap;
  // heavy-row partials run on a second stream beside the light rows (they
  // touch disjoint rows and only read the cache), so each kernel's last wave
  // is filled by the other's CTAs; joined before the heavy solve
  const bool fork = p.n_light > 0 && p.n_heavy > 0 && !s->chunk;   // chunked: heavy rows after
  cudaStream_t hst = st;                                          // the last chunk's data lands
  if (fork) {
    if (!s->aux_st) {
      CUDA_TRY(s, cudaStreamCreateWithFlags(&s->aux_st, cudaStreamNonBlocking));
      CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
      CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    }
    hst = s->aux_st;
    CUDA_TRY(s, cudaEventRecord(s->ev_fork, st));
    CUDA_TRY(s, cudaStreamWaitEvent(hst, s->ev_fork, 0));
  }
  if (p.n_light > 0) {
    static unsigned init = 0;
    if (!(init & dev_bit())) {
      for (auto k : {k_sweep_tc4<false>, k_sweep_tc4<true>}) {
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TcLay4::BYTES));
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      }
      for (auto k : {k_sweep_pk<2, false>, k_sweep_pk<2, true>}) {
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PkLay<2>::BYTES));
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      }
      for (auto k : {k_sweep_pk<4, false>, k_sweep_pk<4, true>}) {
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PkLay<4>::BYTES));
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      }
      init |= dev_bit();
    }
    k_tc_template<<<128, 128, 0, st>>>(p, const_cast<float*>(p.tpl));
    LAUNCH_CHECK(s);
    // rotated user pass: the b x b sweep takes the rows with > 64 entries,
    // the Woodbury tiles the rest (2 rows of <= 64, 4 rows of <= 32 per tile)
    const int n_b = p.rot ? p.rot_n64 : p.n_light;
    // TMEM: 4 x 128 columns per SM; the packed sweep takes G rows per task
    const int grid = std::min(std::max((n_b + G - 1) / G, 1), 4 * kNumSMs);
    const ChunkPlan* cp = s->chunk;
    for (int c = 0; c < (cp ? cp->nch : 1); ++c) {
      SweepParams q = p;
      q.n_light = n_b;
      if (cp) {
        rc = cp->prologue(c);
        if (rc) return rc;
        q.light_rows = cp->rows;
        q.chunk_tot = cp->tot;
        q.chunk = p.rot ? 3 * c : c;   // rotated: buckets (chunk, class) of the grouped list
        // the row queues [2], [5], [6] (and the idle [3], [4]) start over for every chunk
        if (c > 0) CUDA_TRY(s, cudaMemsetAsync(p.redo_cnt + 2, 0, 5 * sizeof(int), st));
      }
      if (n_b == 0) {
      } else if (G == 1) {
        if (unit)
          k_sweep_tc4<true><<<grid, 128, TcLay4::BYTES, st>>>(q, fmap, use_tma);
        else
          k_sweep_tc4<false><<<grid, 128, TcLay4::BYTES, st>>>(q, fmap, use_tma);
      } else if (G == 2) {
        // (IALS_PK_COND: the light rows' cancellation limit at b 33..64, default the pass's)
        static const float pk_cond = getenv("IALS_PK_COND") ? (float)atof(getenv("IALS_PK_COND")) : 0.f;
        if (pk_cond > 1.f) q.cond_max = pk_cond;
        if (unit)
          k_sweep_pk<2, true><<<grid, 128, PkLay<2>::BYTES, st>>>(q, fmap, use_tma);
        else
          k_sweep_pk<2, false><<<grid, 128, PkLay<2>::BYTES, st>>>(q, fmap, use_tma);
      } else if (w32_enabled() && p.vec) {
        // b 17..32: one row per warp (ials_sweep_w32m.cuh: the Hessian by warp-level
        // 3xTF32 MMA tiles; IALS_W32_MMA=0: the FP32 SIMT tiles of ials_sweep_w32.cuh)
        static const bool mma = !(getenv("IALS_W32_MMA") && getenv("IALS_W32_MMA")[0] == '0');
        static int w32_sm = 0;
        static unsigned w32_init = 0;
        static const bool occ4 = getenv("IALS_W32_OCC") && getenv("IALS_W32_OCC")[0] == '4';   // (measurement)
        auto kern = mma ? (occ4 ? (unit ? k_sweep_w32m<true, 4> : k_sweep_w32m<false, 4>)
                                : (unit ? k_sweep_w32m<true> : k_sweep_w32m<false>))
                        : (unit ? k_sweep_w32<true> : k_sweep_w32<false>);
        const int wbytes = mma ? W32mLay::BYTES : W32Lay::BYTES;
        if (!(w32_init & dev_bit())) {
          CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w32<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, W32Lay::BYTES));
          CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w32<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, W32Lay::BYTES));
          CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w32m<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, W32mLay::BYTES));
          CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w32m<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, W32mLay::BYTES));
          CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w32m<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, W32mLay::BYTES));
          CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w32m<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, W32mLay::BYTES));
          CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w32m<true, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
          CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w32m<false, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
          w32_init |= dev_bit();
        }
        if (w32_sm == 0) {
          CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&w32_sm, kern, W32Lay::NT, wbytes));
          if (w32_sm < 1) w32_sm = 1;
        }
        q.queue = p.redo_cnt + 2;   // zeroed with the redo count (and per chunk)
        q.cond_max = kWarpCond;
        const int wgrid = std::min((n_b + W32Lay::NW - 1) / W32Lay::NW, w32_sm * kNumSMs);
        kern<<<wgrid, W32Lay::NT, wbytes, st>>>(q);
      } else {
        if (unit)
          k_sweep_pk<4, true><<<grid, 128, PkLay<4>::BYTES, st>>>(q, fmap, use_tma);
        else
          k_sweep_pk<4, false><<<grid, 128, PkLay<4>::BYTES, st>>>(q, fmap, use_tma);
      }
      if (n_b > 0) LAUNCH_CHECK(s);
      if (cp && p.rot) {   // this chunk's Woodbury tiles (bucket sizes on the device)
        rc = wb_attrs(s);
        if (rc) return rc;
        SweepParams qw = p;
        qw.light_rows = cp->rows;
        const int n2 = p.rot_n32 - p.rot_n64, n4 = p.n_light - p.rot_n32;   // upper bounds
        if (n2 > 0) {
          k_sweep_wb<2><<<std::min((n2 + 1) / 2, 4 * kNumSMs), 128, WbLay<2>::BYTES, st>>>(
              qw, 0, 0, p.redo_cnt + 5, cp->tot, 3 * c + 1);
          LAUNCH_CHECK(s);
        }
        if (n4 > 0) {
          k_sweep_wb<4><<<std::min((n4 + 3) / 4, 4 * kNumSMs), 128, WbLay<4>::BYTES, st>>>(
              qw, 0, 0, p.redo_cnt + 6, cp->tot, 3 * c + 2);
          LAUNCH_CHECK(s);
        }
      }
    }
    if (p.rot && !cp) {
      rc = wb_attrs(s);
      if (rc) return rc;
      const int n2 = p.rot_n32 - p.rot_n64, n4 = p.n_light - p.rot_n32;
      if (n2 > 0) {
        k_sweep_wb<2><<<std::min((n2 + 1) / 2, 4 * kNumSMs), 128, WbLay<2>::BYTES, st>>>(p, p.rot_n64, n2, p.redo_cnt + 5);
        LAUNCH_CHECK(s);
      }
      if (n4 > 0) {
        k_sweep_wb<4><<<std::min((n4 + 3) / 4, 4 * kNumSMs), 128, WbLay<4>::BYTES, st>>>(p, p.rot_n32, n4, p.redo_cnt + 6);
        LAUNCH_CHECK(s);
      }
    }
  }
  bool heavy_reduced = false;
  if (p.n_heavy > 0) {
    static unsigned hinit = 0;
    if (!(hinit & dev_bit())) {
      for (auto k : {k_heavy_partial_tc4<false>, k_heavy_partial_tc4<true>}) {
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TcLay4::BYTES));
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      }
      hinit |= dev_bit();
    }
    const int threads = L::NT * L::RPC;
    if (G == 1) {
      const int hg = std::min(p.n_slices, 4 * kNumSMs);
      if (unit)
        k_heavy_partial_tc4<true><<<hg, 128, TcLay4::BYTES, hst>>>(p, hmap, use_tma_h);
      else
        k_heavy_partial_tc4<false><<<hg, 128, TcLay4::BYTES, hst>>>(p, hmap, use_tma_h);
      LAUNCH_CHECK(s);
    } else {   // b <= 64: G slices per tile, [slice][NG x NG] partials
      static unsigned pinit = 0;
      if (!(pinit & dev_bit())) {
        for (auto k : {k_heavy_partial_pk<2, false>, k_heavy_partial_pk<2, true>})
          CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PkLay<2>::BYTES));
        for (auto k : {k_heavy_partial_pk<4, false>, k_heavy_partial_pk<4, true>})
          CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PkLay<4>::BYTES));
        int rc2 = set_smem_attrs<32>(s);
        if (!rc2) rc2 = set_smem_attrs<64>(s);
        if (rc2) return rc2;
        pinit |= dev_bit();
      }
      const int hg = std::min((p.n_slices + G - 1) / G, 4 * kNumSMs);
      if (G == 4 && p.vec && w32_enabled() && hw_enabled()) {
        rc = launch_heavy_w<32>(s, p, 32, hst);
        if (rc) return rc;
        if (p.n_slices > p.n_heavy) {
          k_heavy_reduce<32><<<p.n_heavy, HRLay<32>::NT, 0, hst>>>(p);
          LAUNCH_CHECK(s);
          heavy_reduced = true;
        }
      } else if (G == 2 && p.vec && hw_enabled() && wmma_enabled()) {
        // b 33..64: a slice per pair of warps, warp-level 3xTF32 MMA tiles (ials_heavy_w64.cuh)
        static int h64_sm = 0;
        static unsigned h64_init = 0;
        if (!(h64_init & dev_bit())) {
          for (auto k : {k_heavy_partial_wm64<true>, k_heavy_partial_wm64<false>})
            CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, WH64Lay::BYTES));
          h64_init |= dev_bit();
        }
        if (h64_sm == 0) {
          CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h64_sm, k_heavy_partial_wm64<true>, WH64Lay::NT,
                                                                   WH64Lay::BYTES));
          if (h64_sm < 1) h64_sm = 1;
        }
        const int g64 = std::min((p.n_slices + WH64Lay::TEAMS - 1) / WH64Lay::TEAMS, h64_sm * kNumSMs);
        if (unit) k_heavy_partial_wm64<true><<<g64, WH64Lay::NT, WH64Lay::BYTES, hst>>>(p);
        else k_heavy_partial_wm64<false><<<g64, WH64Lay::NT, WH64Lay::BYTES, hst>>>(p);
      } else if (G == 2) {
        if (unit) k_heavy_partial_pk<2, true><<<hg, 128, PkLay<2>::BYTES, hst>>>(p, fmap, use_tma);
        else k_heavy_partial_pk<2, false><<<hg, 128, PkLay<2>::BYTES, hst>>>(p, fmap, use_tma);
      } else {
        if (unit) k_heavy_partial_pk<4, true><<<hg, 128, PkLay<4>::BYTES, hst>>>(p, fmap, use_tma);
        else k_heavy_partial_pk<4, false><<<hg, 128, PkLay<4>::BYTES, hst>>>(p, fmap, use_tma);
      }
      LAUNCH_CHECK(s);
    }
    if (fork) {
      CUDA_TRY(s, cudaEventRecord(s->ev_join, hst));
      CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_join, 0));
    }
    if (G == 1) {
      k_heavy_solve<128, true, true><<<(p.n_heavy + L::RPC - 1) / L::RPC, threads, L::CTA_BYTES, st>>>(p);
    } else if (G == 2) {
      using L64 = Lay<64>;
      k_heavy_solve<64, true><<<(p.n_heavy + L64::RPC - 1) / L64::RPC, L64::NT * L64::RPC, L64::CTA_BYTES, st>>>(p);
    } else {
      using L32 = Lay<32>;
      SweepParams ph = p;
      ph.heavy_reduced = heavy_reduced ? 1 : 0;
      k_heavy_solve<32, true><<<(p.n_heavy + L32::RPC - 1) / L32::RPC, L32::NT * L32::RPC, L32::CTA_BYTES, st>>>(ph);
    }
    LAUNCH_CHECK(s);
  }
  if (p.n_light + p.n_heavy > 0) {
    // rows the cancellation checks rejected (light or heavy): FP32 SIMT sweep
    // over the device list (persistent grid, the count is read on the device)
    // (at the block's own tile width: a 64- or 32-wide block redone in the
    // 128 tile would do 4x / 16x the arithmetic)
    SweepParams q = p;
    q.light_rows = p.redo_rows;
    q.n_light_dev = p.redo_cnt;
    q.queue = p.redo_cnt + 4;   // zeroed with the redo count
    if (G == 1) {
      static int simt_sm = 0;
      if (simt_sm == 0) {
        CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&simt_sm, k_sweep_light<128>,
                                                                 L::NT * L::RPC, L::CTA_BYTES));
        if (simt_sm < 1) simt_sm = 1;
      }
      k_sweep_light<128><<<simt_sm * kNumSMs, L::NT * L::RPC, L::CTA_BYTES, st>>>(q);
    } else if (G == 2) {
      using L64 = Lay<64>;
      static int simt_sm = 0;
      rc = set_smem_attrs<64>(s);
      if (rc) return rc;
      if (simt_sm == 0) {
        CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&simt_sm, k_sweep_light<64>,
                                                                 L64::NT * L64::RPC, L64::CTA_BYTES));
        if (simt_sm < 1) simt_sm = 1;
      }
      k_sweep_light<64><<<simt_sm * kNumSMs, L64::NT * L64::RPC, L64::CTA_BYTES, st>>>(q);
    } else {
      using L32 = Lay<32>;
      static int simt_sm = 0;
      rc = set_smem_attrs<32>(s);
      if (rc) return rc;
      if (simt_sm == 0) {
        CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&simt_sm, k_sweep_light<32>,
                                                                 L32::NT * L32::RPC, L32::CTA_BYTES));
        if (simt_sm < 1) simt_sm = 1;
      }
      k_sweep_light<32><<<simt_sm * kNumSMs, L32::NT * L32::RPC, L32::CTA_BYTES, st>>>(q);
    }
    LAUNCH_CHECK(s);
  }
  if (p.n_light + p.n_slices > 0) {
    cudaStream_t cst = st;
    if (s->defer_cache) {   // beside the next pass's GEMM phase; joined by the next sweep
      if (!s->cache_st) {
        CUDA_TRY(s, cudaStreamCreateWithFlags(&s->cache_st, cudaStreamNonBlocking));
        CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_cache_go, cudaEventDisableTiming));
        CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_cache_done, cudaEventDisableTiming));
      }
      CUDA_TRY(s, cudaEventRecord(s->ev_cache_go, st));
      CUDA_TRY(s, cudaStreamWaitEvent(s->cache_st, s->ev_cache_go, 0));
      cst = s->cache_st;
    }
    if (p.side.rows && nnz > 0) {   // entry-parallel: no per-row setup, full load balance
      const long long g = std::min<long long>((nnz + 31) / 32, 16LL * kNumSMs);
      // walk the other side's order when this side's d is the smaller gather
      const bool swap = p.x_rows && p.x_cols && p.side.n_rows < p.side.n_fixed;
      // narrow blocks: 4 lanes per entry, 2 (b <= 32) or 4 (b <= 64) float4 each -- configs[1]
      // epoch 8.89 -> 7.43 ms, sw-b64 26.6 -> 25.5 ms against the 8-lane 128-wide instantiation
      // (IALS_CACHE_NARROW=0 keeps that one; IALS_CACHE_LPE=2: two lanes per entry at b <= 32,
      // 7.52 vs 7.42 ms at configs[1])
      static const bool narrow = !(getenv("IALS_CACHE_NARROW") && getenv("IALS_CACHE_NARROW")[0] == '0');
      static const bool lpe2 = getenv("IALS_CACHE_LPE") && getenv("IALS_CACHE_LPE")[0] == '2';
      if (narrow && p.vec && p.b <= 32 && lpe2) {
        if (swap) k_pass_cache_flat<true, 2, true, 32><<<(int)g, 256, 0, cst>>>(p, nnz);
        else k_pass_cache_flat<true, 2, false, 32><<<(int)g, 256, 0, cst>>>(p, nnz);
      } else if (narrow && p.vec && p.b <= 32) {
        if (swap) k_pass_cache_flat<true, 4, true, 32><<<(int)g, 256, 0, cst>>>(p, nnz);
        else k_pass_cache_flat<true, 4, false, 32><<<(int)g, 256, 0, cst>>>(p, nnz);
      } else if (narrow && p.vec && p.b <= 64) {
        if (swap) k_pass_cache_flat<true, 4, true, 64><<<(int)g, 256, 0, cst>>>(p, nnz);
        else k_pass_cache_flat<true, 4, false, 64><<<(int)g, 256, 0, cst>>>(p, nnz);
      } else if (swap) {
        if (p.vec) k_pass_cache_flat<true, 8, true><<<(int)g, 256, 0, cst>>>(p, nnz);
        else k_pass_cache_flat<false, 8, true><<<(int)g, 256, 0, cst>>>(p, nnz);
      } else {
        if (p.vec) k_pass_cache_flat<true, 8, false><<<(int)g, 256, 0, cst>>>(p, nnz);
        else k_pass_cache_flat<false, 8, false><<<(int)g, 256, 0, cst>>>(p, nnz);
      }
    } else {
      k_pass_cache<<<p.n_light + p.n_slices, 256, 0, cst>>>(p);
    }
    LAUNCH_CHECK(s);
    if (s->defer_cache) {
      CUDA_TRY(s, cudaEventRecord(s->ev_cache_done, s->cache_st));
      s->cache_pending = true;
    }
  }
  return IALS_OK;
}

template <int BT>
static int launch_sweep(ials_session* s, const SweepParams& p, long long nnz, cudaStream_t st) {
  using L = Lay<BT>;
  if (BT == 128 && p.b > 16 && tc4_enabled()) return launch_sweep_tc4(s, p, nnz, st);
  int rc = set_smem_attrs<BT>(s);
  if (rc) return rc;
  const int threads = L::NT * L::RPC;
  // b 4..16 (16-byte sub-rows): two rows per warp, FP32 SIMT (ials_sweep_w16.cuh); the
  // cache update is the entry-parallel pass over drow, heavy rows included
  const bool w16 = BT <= 16 && p.b >= 4 && p.vec && p.side.rows && !p.rot && nnz > 0 && w16_enabled();
  // the long rows' slice partials (ials_heavy_w.cuh) run beside the light rows on the
  // second stream (disjoint rows, the cache only read), joined before their solve
  const bool hw = w16 && p.n_heavy > 0 && hw_enabled();
  const bool fork = hw && p.n_light > 0;
  // [0] the redo count (rows the MMA kernels' cancellation guards reject), [3] the light-row
  // queue, [4] the redo launch's queue
  if (w16) CUDA_TRY(s, cudaMemsetAsync(p.redo_cnt, 0, 8 * sizeof(int), st));
  const bool guard = w16 && wmma_enabled();
  if (hw) {
    cudaStream_t hst = st;
    if (fork) {
      if (!s->aux_st) {
        CUDA_TRY(s, cudaStreamCreateWithFlags(&s->aux_st, cudaStreamNonBlocking));
        CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
        CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
      }
      hst = s->aux_st;
      CUDA_TRY(s, cudaEventRecord(s->ev_fork, st));
      CUDA_TRY(s, cudaStreamWaitEvent(hst, s->ev_fork, 0));
    }
    rc = launch_heavy_w<16>(s, p, BT, hst);
    if (rc) return rc;
    if (fork) CUDA_TRY(s, cudaEventRecord(s->ev_join, hst));
  }
  if (w16 && p.n_light > 0) {
    static int w16_sm = 0;
    static unsigned w16_init = 0;
    const bool unit = !p.side.weights && !p.side.labels;
    const bool mma = wmma_enabled();
    auto kern = mma ? (unit ? k_sweep_w16m<true> : k_sweep_w16m<false>)
                    : (unit ? k_sweep_w16<true> : k_sweep_w16<false>);
    const int wbytes = mma ? W16mLay::BYTES : W16Lay::BYTES;
    if (!(w16_init & dev_bit())) {
      CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w16<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, W16Lay::BYTES));
      CUDA_TRY(s, cudaFuncSetAttribute(k_sweep_w16<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, W16Lay::BYTES));
      for (auto k : {k_sweep_w16m<true>, k_sweep_w16m<false>}) {
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, W16mLay::BYTES));
        CUDA_TRY(s, cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      }
      w16_init |= dev_bit();
    }
    if (w16_sm == 0) {
      CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&w16_sm, kern, W16Lay::NT, wbytes));
      if (w16_sm < 1) w16_sm = 1;
    }
    SweepParams q = p;
    q.queue = p.redo_cnt + 3;
    q.cond_max = kWarpCond;
    const int tasks = (p.n_light + 1) / 2;
    const int wgrid = std::min((tasks + W16Lay::NW - 1) / W16Lay::NW, w16_sm * kNumSMs);
    kern<<<wgrid, W16Lay::NT, wbytes, st>>>(q);
    LAUNCH_CHECK(s);
  } else if (p.n_light > 0) {
    static int per_sm = 0;
    if (per_sm == 0) {
      CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep_light<BT>,
                                                               threads, L::CTA_BYTES));
      if (per_sm < 1) per_sm = 1;
    }
    const int need = (p.n_light + L::RPC - 1) / L::RPC;
    const int grid = std::min(need, per_sm * kNumSMs);
    SweepParams q = p;
    q.queue = p.redo_cnt + 3;   // zeroed below; the redo launch of the fused path uses [4]
    CUDA_TRY(s, cudaMemsetAsync(q.queue, 0, sizeof(int), st));
    k_sweep_light<BT><<<grid, threads, L::CTA_BYTES, st>>>(q);
    LAUNCH_CHECK(s);
  }
  if (p.n_heavy > 0) {
    if (!hw) {
      k_heavy_partial<BT><<<(p.n_slices + L::RPC - 1) / L::RPC, threads, L::CTA_BYTES, st>>>(p);
      LAUNCH_CHECK(s);
    } else if (fork) {
      CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_join, 0));
    }
    SweepParams ph = p;
    if (hw && BT <= 32 && p.n_slices > p.n_heavy) {   // some row has several slices
      k_heavy_reduce<(BT <= 32 ? BT : 32)><<<p.n_heavy, HRLay<(BT <= 32 ? BT : 32)>::NT, 0, st>>>(p);
      LAUNCH_CHECK(s);
      ph.heavy_reduced = 1;
    }
    if (guard && hw)
      k_heavy_solve<BT, true><<<(p.n_heavy + L::RPC - 1) / L::RPC, threads, L::CTA_BYTES, st>>>(ph);
    else
      k_heavy_solve<BT><<<(p.n_heavy + L::RPC - 1) / L::RPC, threads, L::CTA_BYTES, st>>>(ph);
    LAUNCH_CHECK(s);
    if (!w16) {
      k_heavy_cache<BT><<<(p.n_slices + L::RPC - 1) / L::RPC, threads, L::CTA_BYTES, st>>>(p);
      LAUNCH_CHECK(s);
    }
  }
  if (guard && p.n_light + p.n_heavy > 0) {
    // rows the cancellation guards rejected: the FP32 SIMT sweep over the device list
    // (persistent grid, the count is read on the device; it updates their cache itself,
    // the entry-parallel pass below sees d = 0 for them)
    static int simt_sm = 0;
    if (simt_sm == 0) {
      CUDA_TRY(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&simt_sm, k_sweep_light<BT>, threads, L::CTA_BYTES));
      if (simt_sm < 1) simt_sm = 1;
    }
    SweepParams q = p;
    q.light_rows = p.redo_rows;
    q.n_light_dev = p.redo_cnt;
    q.queue = p.redo_cnt + 4;
    k_sweep_light<BT><<<simt_sm * kNumSMs, threads, L::CTA_BYTES, st>>>(q);
    LAUNCH_CHECK(s);
  }
  if (w16 && p.n_light + p.n_heavy > 0) {
    const long long g = std::min<long long>((nnz + 31) / 32, 16LL * kNumSMs);
    // walk the other side's order when this side's d is the smaller gather
    const bool swap = p.x_rows && p.x_cols && p.side.n_rows < p.side.n_fixed;
    static const bool lpe8 = getenv("IALS_W16_LPE8") != nullptr;   // (measurements)
    // two lanes x 2 float4 per entry (sw-b16 epoch 19.2 -> 17.4 ms against four lanes;
    // IALS_CACHE_LPE=4 keeps four)
    static const bool lpe2 = !(getenv("IALS_CACHE_LPE") && getenv("IALS_CACHE_LPE")[0] == '4');
    if (lpe8) {
      if (swap) k_pass_cache_flat<true, 8, true><<<(int)g, 256, 0, st>>>(p, nnz);
      else k_pass_cache_flat<true, 8, false><<<(int)g, 256, 0, st>>>(p, nnz);
    } else if (lpe2) {
      if (swap) k_pass_cache_flat<true, 2, true, 16><<<(int)g, 256, 0, st>>>(p, nnz);
      else k_pass_cache_flat<true, 2, false, 16><<<(int)g, 256, 0, st>>>(p, nnz);
    } else {   // 4 lanes x 16 bytes
      if (swap) k_pass_cache_flat<true, 4, true, 16><<<(int)g, 256, 0, st>>>(p, nnz);
      else k_pass_cache_flat<true, 4, false, 16><<<(int)g, 256, 0, st>>>(p, nnz);
    }
    LAUNCH_CHECK(s);
  }
  return IALS_OK;
}

// drow (n_rows x b, the per-row d of a pass) inside a pass workspace: the
// carve of side_pass_impl below
static float* pass_drow(char* ws, const ials_side* side, const ials_sched* sched, int b) {
  const size_t bt = block_tile(b);
  char* w = ws;
  w += al256(size_t(side->n_rows) * b * 4);             // proj
  w += al256(size_t(sched->n_slices) * bt * bt * 4);    // hpart
  w += al256(size_t(sched->n_slices) * bt * 8);         // gpart
  w += al256(size_t(sched->n_heavy) * bt * 4);          // hdelta
  w += al256(size_t(kTcPKS) * 4);                       // template
  w += al256(size_t(side->n_rows) * 4 + 32);            // redo list
  return reinterpret_cast<float*>(w);
}

// A pass of a block wider than 256 columns (ials_sweep_wide.cuh): projection,
// then per batch of rows the Hessians + gradients (k_wide_build) and the
// factorisations / solves (k_wide_chol), then the entry-parallel cache update.
static int wide_pass(ials_session* s, SweepParams p, char* ws, cudaStream_t st, bool proj_ready,
                     const float* proj_in) {
  const int b = p.b, n_rows = p.side.n_rows;
  char* w = ws;
  float* proj = reinterpret_cast<float*>(w);
  w += al256(size_t(n_rows) * b * 4);
  p.drow = reinterpret_cast<float*>(w);
  w += al256(size_t(n_rows) * b * 4);
  WideParams wp{};
  wp.A = reinterpret_cast<float*>(w);
  wp.lda = wide_lda(b);
  wp.mat_stride = (long long)wide_mat_floats(b);
  if (proj_in) proj = const_cast<float*>(proj_in);
  p.proj = proj;
  p.vec = p.vec && (p.ldf % 4 == 0);
  if (n_rows == 0) return IALS_OK;
  if (!proj_ready && !proj_in) {
    dim3 g((n_rows + GT - 1) / GT, (b + GT - 1) / GT);
    k_project<<<g, 256, 0, st>>>(p.own, n_rows, p.ldo, p.d, p.slab, b, p.alpha0, proj);
    LAUNCH_CHECK(s);
  }
  const size_t smem = WideSm::bytes(b);
  if (smem > 227 * 1024) return fail(s, IALS_E_INVALID, "side_pass: block width %d too wide", b);
  {
    int dev = 0;
    CUDA_TRY(s, cudaGetDevice(&dev));
    static size_t attr_bytes[64] = {};
    if (dev < 64 && attr_bytes[dev] < smem) {
      CUDA_TRY(s, cudaFuncSetAttribute(k_wide_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr_bytes[dev] = smem;
    }
  }
  const int R = std::min(wide_batch(b), n_rows);
  const int nt = (b + kWT - 1) / kWT, ntp = nt * (nt + 1) / 2;
  for (int i0 = 0; i0 < n_rows; i0 += R) {
    wp.i0 = i0;
    wp.nb = std::min(R, n_rows - i0);
    k_wide_build<<<dim3(ntp + 1, wp.nb), 256, 0, st>>>(p, wp, ntp);
    LAUNCH_CHECK(s);
    k_wide_chol<<<wp.nb, 256, smem, st>>>(p, wp);
    LAUNCH_CHECK(s);
  }
  if (p.side.nnz > 0) {
    const long long nw = (p.side.nnz + 7) / 8;
    k_wide_cache<<<(int)std::min<long long>(nw, 32 * kNumSMs), 256, 0, st>>>(p, p.side.nnz);
    LAUNCH_CHECK(s);
  }
  return IALS_OK;
}

// a rotated user pass (ials_rot.cuh): the pass sweeps F~ = F[:, pi] Q with the
// diagonal template diag(eigenvalues) (rslab's rows pi), reads W[:, pi] Q
// (wq) for the lam * w term and leaves d~ in drow for the back-rotation
struct RotPass {
  const float* Ft;      // n_fixed x b
  const float* wq;      // n_rows x b
  const float* lam;     // b eigenvalues
  const float* rslab;   // d x b: rows [b0, b0 + b) = diag(lam)
};

static int side_pass_impl(ials_session* s, const ials_side* side, const ials_sched* sched,
                          const float* fixed, int32_t ldf, float* own, int32_t ldo, int32_t d,
                          int32_t b0, int32_t b, const float* slab, float alpha0, float* cache,
                          int32_t side_id, char* ws, size_t ws_bytes, cudaStream_t st,
                          bool proj_ready = false, const float* proj_in = nullptr,
                          const ials_side* other = nullptr, const RotPass* rot = nullptr,
                          size_t defer_min_off = 0) {
  // defer_min_off > 0 (ials_epoch): this pass's cache update may run beside the
  // next pass's GEMM phase, whose projection overwrites the first defer_min_off
  // bytes of the scratch: the per-row steps it reads are kept above them
  if (!side || !sched || !fixed || !own || !slab || !cache)
    return fail(s, IALS_E_INVALID, "side_pass: NULL argument");
  {
    const int jr = join_cache(s, st);   // the previous pass's deferred cache update
    if (jr) return jr;
  }
  s->defer_cache = false;
  if (d < 1 || b < 1 || b0 < 0 || b0 + b > d || ldf < d || ldo < d)
    return fail(s, IALS_E_INVALID, "side_pass: bad block (d=%d b0=%d b=%d)", d, b0, b);
  const int bt = block_tile(b);
  const size_t need = pass_ws(side->n_rows, side->n_fixed, b, sched->n_slices, sched->n_heavy);
  if (need > ws_bytes)
    return fail(s, IALS_E_NOMEM, "side_pass: workspace %zu < %zu bytes", ws_bytes, need);
  SweepParams p{};
  p.side = SideDev{side->n_rows, side->n_fixed, side->ptr, side->cols, side->labels,
                   side->weights, side->pos, side->lam, side->rows, side->nnz};
  p.fixed = fixed;
  p.ldf = ldf;
  p.own = own;
  p.ldo = ldo;
  p.d = d;
  p.b0 = b0;
  p.fb0 = b0;
  p.fixed_cols = d;
  p.b = b;
  p.slab = slab;
  p.alpha0 = alpha0;
  p.cache = cache;
  p.side_id = side_id;
  p.err = s->err;
  p.vec = (b % 4 == 0) && (b0 % 4 == 0) && (ldf % 4 == 0) &&
          (reinterpret_cast<uintptr_t>(fixed) % 16 == 0);
  p.light_rows = sched->light_rows;
  p.n_light = sched->n_light;
  p.heavy_rows = sched->heavy_rows;
  p.heavy_slice0 = sched->heavy_slice0;
  p.n_heavy = sched->n_heavy;
  p.slice_heavy = sched->slice_heavy;
  p.slice_begin = sched->slice_begin;
  p.slice_end = sched->slice_end;
  p.n_slices = sched->n_slices;
  if (b >= wide_min()) return wide_pass(s, p, ws, st, proj_ready, proj_in);
  char* w = ws;
  float* proj = reinterpret_cast<float*>(w);
  w += al256(size_t(side->n_rows) * b * 4);
  p.hpart = reinterpret_cast<float*>(w);
  w += al256(size_t(sched->n_slices) * bt * bt * 4);
  p.gpart = reinterpret_cast<double*>(w);
  w += al256(size_t(sched->n_slices) * bt * 8);
  p.hdelta = reinterpret_cast<float*>(w);
  w += al256(size_t(sched->n_heavy) * bt * 4);
  float* tpl_simt = reinterpret_cast<float*>(w);
  w += al256(size_t(kTcPKS) * 4);
  p.redo_cnt = reinterpret_cast<int*>(w);
  p.redo_rows = reinterpret_cast<int*>(w + 32);   // [0..7]: redo count, work queues
  w += al256(size_t(side->n_rows) * 4 + 32);
  if (defer_min_off && bt == 128 && b > 16 && tc4_enabled()) {
    // (only the fused tensor-core path has the separate cache kernel)
    char* dr = std::max(w, ws + al256(defer_min_off));
    const size_t tail = al256(size_t(side->n_rows) * b * 4) +
                        (b <= kCompactMaxB ? al256(size_t(side->n_fixed) * compact_ld(b) * 4) : 0);
    if (size_t(dr - ws) + tail <= ws_bytes) {
      w = dr;
      s->defer_cache = true;
    }
  }
  p.drow = reinterpret_cast<float*>(w);
  s->last_drow = p.drow;
  w += al256(size_t(side->n_rows) * b * 4);
  if (b <= kCompactMaxB && side->n_fixed > 0) {
    // gather from a compact, L2-resident copy of fixed[:, b0:b0+b]
    const int ldc = compact_ld(b);
    float* compact = reinterpret_cast<float*>(w);
    const long long cnt = (long long)side->n_fixed * ldc;
    k_compact_cols<<<(int)std::min<long long>((cnt + 255) / 256, 65535), 256, 0, st>>>(
        fixed, side->n_fixed, ldf, b0, b, compact, ldc);
    LAUNCH_CHECK(s);
    p.fixed = compact;
    p.ldf = ldc;
    p.fb0 = 0;
    p.fixed_cols = ldc;
    p.vec = (b % 4 == 0) && (reinterpret_cast<uintptr_t>(compact) % 16 == 0);
  }
  p.redo_total = s->redo;
  p.rot = 0;
  p.flat_skip_deg = 0;
  if (rot) {
    p.rot = 1;
    p.fixed = rot->Ft;
    p.ldf = b;
    p.fb0 = 0;
    p.fixed_cols = b;
    p.vec = 1;
    p.slab = rot->rslab;
    p.wq = rot->wq;
    p.rot_lam = rot->lam;
    static const bool wb_off = getenv("IALS_WB") && getenv("IALS_WB")[0] == '0';   // (diagnostics)
    p.rot_n64 = wb_off ? sched->n_light : sched->n_deg_gt64;
    p.rot_n32 = wb_off ? sched->n_light : sched->n_deg_gt32;
    // the Woodbury tiles update their rows' cache themselves (yhat -= v) when
    // the pass's cache kernel walks this side's order and can skip their
    // rows; when it walks the other side's order (this side the smaller) it
    // updates every entry and the tiles leave the cache alone
    const bool walks_other = other && other->rows && other->cols && side->n_rows < side->n_fixed;
    p.flat_skip_deg = walks_other ? 0 : 64;
  }
  if (other && other->rows && other->cols && other->nnz == side->nnz) {   // same entries, other order
    p.x_rows = other->rows;
    p.x_cols = other->cols;
    p.x_pos = other->pos;
  }
  // narrow blocks in the 128 tile: a pivot losing more than 16x of its
  // diagonal already goes to the FP32 sweep (ill-conditioned heavy rows at
  // b = 64 slip under the 256x limit, tests/test_gpu_parity.py heavy rows)
  p.cond_max = b <= 64 ? std::min(tc_cond_max(), 16.f) : tc_cond_max();
  p.n_light_dev = nullptr;
  if (proj_in) {   // precomputed by the caller (ials_side_pass_projected)
    proj = const_cast<float*>(proj_in);
    proj_ready = true;
  }
  p.proj = proj;
  p.dbg = g_dbg;
  p.tpl = tpl_simt;
  if (side->n_rows > 0 && !proj_ready) {
    if (b <= 4) {
      const int g = (side->n_rows + 7) / 8;
      const int vec = (d % 4 == 0) && (ldo % 4 == 0) && (reinterpret_cast<uintptr_t>(own) % 16 == 0);
      switch (b) {
        case 1: k_project_gemv<1><<<g, 256, 0, st>>>(own, side->n_rows, ldo, d, slab, alpha0, vec, proj); break;
        case 2: k_project_gemv<2><<<g, 256, 0, st>>>(own, side->n_rows, ldo, d, slab, alpha0, vec, proj); break;
        case 3: k_project_gemv<3><<<g, 256, 0, st>>>(own, side->n_rows, ldo, d, slab, alpha0, vec, proj); break;
        default: k_project_gemv<4><<<g, 256, 0, st>>>(own, side->n_rows, ldo, d, slab, alpha0, vec, proj); break;
      }
    } else if (b <= 16) {
      k_project_narrow<<<(side->n_rows + 127) / 128, 256, 0, st>>>(own, side->n_rows, ldo, d, slab,
                                                                    b, alpha0, proj);
    } else {
      dim3 g((side->n_rows + GT - 1) / GT, (b + GT - 1) / GT);
      k_project<<<g, 256, 0, st>>>(own, side->n_rows, ldo, d, slab, b, alpha0, proj);
    }
    LAUNCH_CHECK(s);
  }
  if (b == 1) {  // scalar blocks: the iCD special case
    // the smaller side (items): the cache update walks the other side's entry order
    // (coalesced cache and ids, d in L1 / L2) instead of scattering through `pos`
    // (IALS_B1_FLAT: 0 = in the sweep, 2 = both sides entry-parallel; measured at the
    // configs[2] shape: 116.7 / 78.9 / 79.9 ms an epoch for 0 / 1 / 2)
    static const int b1_mode = getenv("IALS_B1_FLAT") ? atoi(getenv("IALS_B1_FLAT")) : 1;
    const bool b1_swap = b1_mode >= 1 && p.x_rows && p.x_cols && side->n_rows < side->n_fixed && side->nnz > 0;
    p.b1_flat = b1_swap || (b1_mode >= 2 && side->rows && side->nnz > 0);
    if (p.n_light > 0) {
      k_sweep_b1<<<std::min((p.n_light + 7) / 8, kNumSMs * 16), 256, 0, st>>>(p);
      LAUNCH_CHECK(s);
    }
    if (p.n_heavy > 0) {
      const int g = std::min((p.n_slices + 7) / 8, kNumSMs * 16);
      k_b1_partial<<<g, 256, 0, st>>>(p);
      LAUNCH_CHECK(s);
      k_b1_solve<<<(p.n_heavy + 7) / 8, 256, 0, st>>>(p);
      LAUNCH_CHECK(s);
      if (!p.b1_flat) {
        k_b1_cache<<<g, 256, 0, st>>>(p);
        LAUNCH_CHECK(s);
      }
    }
    if (p.b1_flat) {
      const long long g = std::min<long long>((side->nnz + 1023) / 1024, 32LL * kNumSMs);
      if (b1_swap) k_b1_cache_flat<true><<<(int)g, 256, 0, st>>>(p, side->nnz);
      else k_b1_cache_flat<false><<<(int)g, 256, 0, st>>>(p, side->nnz);
      LAUNCH_CHECK(s);
    }
    return IALS_OK;
  }
  switch (bt) {
    case 8: return launch_sweep<8>(s, p, side->nnz, st);
    case 16: return launch_sweep<16>(s, p, side->nnz, st);
    case 32: return launch_sweep<32>(s, p, side->nnz, st);
    case 64: return launch_sweep<64>(s, p, side->nnz, st);
    case 128: return launch_sweep<128>(s, p, side->nnz, st);
    default: return launch_sweep<256>(s, p, side->nnz, st);
  }
}

int ials_side_pass(ials_session* s, const ials_side* side, const ials_sched* sched,
                   const float* fixed, int32_t ldf, float* own, int32_t ldo, int32_t d,
                   int32_t b0, int32_t b, const float* slab, float alpha0, float* cache,
                   int32_t side_id, void* workspace, size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  return side_pass_impl(s, side, sched, fixed, ldf, own, ldo, d, b0, b, slab, alpha0, cache,
                        side_id, static_cast<char*>(workspace), ws_bytes, S(stream));
}

int ials_side_pass_projected(ials_session* s, const ials_side* side, const ials_sched* sched,
                             const float* fixed, int32_t ldf, float* own, int32_t ldo, int32_t d,
                             int32_t b0, int32_t b, const float* slab, const float* proj,
                             float alpha0, float* cache, int32_t side_id, void* workspace,
                             size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (!proj && side && side->n_rows > 0) return fail(s, IALS_E_INVALID, "side_pass_projected: NULL proj");
  return side_pass_impl(s, side, sched, fixed, ldf, own, ldo, d, b0, b, slab, alpha0, cache,
                        side_id, static_cast<char*>(workspace), ws_bytes, S(stream), true, proj);
}

// ------------------------------------------------------------------ tensor-core GEMMs (epoch)
static inline int rup(int x, int m) { return (x + m - 1) / m * m; }

// split-K plan of the Gramian: >= 2 CTAs per SM and at most 2048 rows
// accumulated in TMEM per CTA
static void gram_plan(int n, int d, int* splits, int* span) {
  const int mt = (d + 127) / 128;
  int S = std::max((n + 2047) / 2048, (2 * kNumSMs + mt - 1) / mt);
  S = std::max(1, std::min(S, std::max(1, n / 32)));
  // fill the last wave (one CTA per SM): as many splits as the waves hold
  const int waves = (mt * S + kNumSMs - 1) / kNumSMs;
  S = std::max(S, std::min(std::max(1, n / 32), waves * kNumSMs / mt));
  int sp = rup((n + S - 1) / S, kGemmKC);
  *span = std::max(sp, kGemmKC);
  *splits = std::max(1, (n + *span - 1) / *span);
}

struct TcCopies {   // K-major copies of one factor matrix F (n x d)
  float* FT;        // d x ldt
  float* FT_lo;
  float* F_lo;      // n x d
  int n, ldt;
};

// only F^T is stored: the GEMM forms the tf32 low parts on chip
static size_t copies_bytes(int n, int d) {
  const size_t ldt = rup(std::max(n, 1), 4);
  return al256(size_t(d) * ldt * 4);
}

static char* carve_copies(char* w, int n, int d, TcCopies* c) {
  c->n = n;
  c->ldt = rup(std::max(n, 1), 4);
  c->FT = reinterpret_cast<float*>(w);
  c->FT_lo = nullptr;
  c->F_lo = nullptr;
  return w + al256(size_t(d) * c->ldt * 4);
}

static size_t rot_bytes(int n_users, int n_items, int d, int b);
static size_t tc_gemm_bytes(int n_users, int n_items, int d, int b) {
  int su, spu, si, spi;
  gram_plan(std::max(n_users, 1), d, &su, &spu);
  gram_plan(std::max(n_items, 1), d, &si, &spi);
  return copies_bytes(n_users, d) + copies_bytes(n_items, d) +
         al256(size_t(std::max(su, si)) * d * b * 4) + 2 * al256(size_t(b) * d * 4) + 1024 +
         rot_bytes(n_users, n_items, d, b);
}

size_t ials_epoch_tc_bytes(int32_t n_users, int32_t n_items, int32_t d, int32_t b) {
  return tc_gemm_bytes(n_users, n_items, d, b);
}


static int sync_copies(ials_session* s, const float* F, int ldf, int d, int c0, int cw,
                       const TcCopies& c, cudaStream_t st) {
  if (c.n <= 0 || cw <= 0) return IALS_OK;
  dim3 g((c.n + 31) / 32, (cw + 31) / 32), t(32, 8);
  k_sync_copies<<<g, t, 0, st>>>(F, c.n, ldf, c0, cw, c.FT, c.FT_lo, c.ldt, c.F_lo, d);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

static int gemm_attrs(ials_session* s) {
  static unsigned init = 0;
  if (!(init & dev_bit())) {
    CUDA_TRY(s, cudaFuncSetAttribute(k_gemm3_tf32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     GemmLay::BYTES));
    init |= dev_bit();
  }
  return IALS_OK;
}

// slab = F^T F[:, b0:b0+bb] (d x bb) and slabT hi / lo (bb x d)
static int gram_tc(ials_session* s, const TcCopies& F, int d, int b0, int bb, float* P, float* slab,
                   float* slabT_hi, float* slabT_lo, cudaStream_t st) {
  int rc = gemm_attrs(s);
  if (rc) return rc;
  const int bn = rup(bb, 16);
  int S, span;
  gram_plan(F.n, d, &S, &span);
  CUtensorMap ah, bh;
  rc = make_map(s, &ah, F.FT, F.n, d, F.ldt, 128);
  if (!rc) rc = make_map(s, &bh, F.FT, F.n, d, F.ldt, bn);
  if (rc) return rc;
  GemmJob job{d, 0, b0, bb, bn, F.n, span, P, bb, (long long)d * bb, 1.f};
  k_gemm3_tf32<<<dim3((d + 127) / 128, S), kGemmThreads, GemmLay::BYTES, st>>>(ah, bh, bh, job);
  LAUNCH_CHECK(s);
  // slab^T hi and its tf32 lo part (the projection TMA-loads both)
  k_gram_reduce<<<(d * bb + 255) / 256, 256, 0, st>>>(P, S, (long long)d * bb, d, bb, slab,
                                                      slabT_hi, slabT_lo);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// proj = alpha0 * own @ slab (rows x bb)
static int proj_tc(ials_session* s, const float* own, int ldo, const TcCopies& O, int d, int bb,
                   const float* slabT_hi, const float* slabT_lo, float alpha0, float* proj,
                   cudaStream_t st) {
  if (O.n <= 0) return IALS_OK;
  int rc = gemm_attrs(s);
  if (rc) return rc;
  const int bn = rup(bb, 16);
  CUtensorMap ah, bh, bl;
  rc = make_map(s, &ah, own, d, O.n, ldo, 128);
  if (!rc) rc = make_map(s, &bh, slabT_hi, d, bb, d, bn);
  if (!rc && slabT_lo) rc = make_map(s, &bl, slabT_lo, d, bb, d, bn);
  if (rc) return rc;
  GemmJob job{O.n, 0, 0, bb, bn, d, rup(d, kGemmKC), proj, bb, 0, alpha0};
  // B = slab^T is the same for every CTA: its lo part comes precomputed
  // (k_gram_reduce) instead of being re-formed on chip by each CTA
  job.b_lo_tma = slabT_lo ? 1 : 0;
  k_gemm3_tf32<<<dim3((O.n + 127) / 128, 1), kGemmThreads, GemmLay::BYTES, st>>>(ah, bh, slabT_lo ? bl : bh, job);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// out (m x n, ld ldo) = scale * A[:, a_k0 : a_k0 + K] B[:, b_k0 : b_k0 + K]^T
// (+ out when acc): A (m x *), B (n x *) row-major fp32, the 3xTF32 TMA GEMM
static int gemm_nt(ials_session* s, const float* A, int m, int a_cols, int lda, int a_k0,
                   const float* Bm, int n, int b_cols, int ldb, int b_k0, int K, float* out,
                   int ldo, float scale, bool acc, cudaStream_t st) {
  if (m <= 0 || n <= 0) return IALS_OK;
  int rc = gemm_attrs(s);
  if (!rc) rc = get_encode(s);
  if (rc) return rc;
  CUtensorMap am, bm;
  rc = make_map(s, &am, A, a_cols, m, lda, 128);
  const int bn = n > 128 ? 128 : rup(n, 16);
  if (!rc) rc = make_map(s, &bm, Bm, b_cols, n, ldb, bn);
  if (rc) return rc;
  GemmJob job{m, 0, 0, n, bn, K, rup(K, kGemmKC), out, ldo, 0, scale};
  job.a_k0 = a_k0;
  job.b_k0 = b_k0;
  job.accumulate = acc ? 1 : 0;
  job.n_tiles = n > 128 ? (n + 127) / 128 : 0;
  k_gemm3_tf32<<<dim3((m + 127) / 128, std::max(job.n_tiles, 1)), kGemmThreads, GemmLay::BYTES, st>>>(
      am, bm, bm, job);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// rotated user passes: scratch of one epoch (b = 128)
struct RotWs {
  float *Gd, *Gprev, *Gpart, *QT, *Qm, *lam, *rslab, *Ft, *WQ, *slabQT;
};
static size_t rot_bytes(int n_users, int n_items, int d, int b) {
  if (b != 128 || d % b) return 0;
  int si, spi;
  gram_plan(std::max(n_items, 1), d, &si, &spi);
  return 6 * al256(size_t(d) * b * 4) + al256(size_t(si) * d * b * 4) + al256(size_t(d) * 4) +
         al256(size_t(std::max(n_items, 1)) * b * 4) + al256(size_t(std::max(n_users, 1)) * b * 4) + 1024;
}
static char* rot_carve(char* t, int n_users, int n_items, int d, int b, RotWs* r) {
  int si, spi;
  gram_plan(std::max(n_items, 1), d, &si, &spi);
  auto take = [&](size_t bytes) { float* p = reinterpret_cast<float*>(t); t += al256(bytes); return p; };
  r->Gd = take(size_t(d) * b * 4);
  r->Gprev = take(size_t(d) * b * 4);
  r->QT = take(size_t(d) * b * 4);
  r->Qm = take(size_t(d) * b * 4);
  r->rslab = take(size_t(d) * b * 4);
  r->slabQT = take(size_t(d) * b * 4);
  r->Gpart = take(size_t(si) * d * b * 4);
  r->lam = take(size_t(d) * 4);
  r->Ft = take(size_t(std::max(n_items, 1)) * b * 4);
  r->WQ = take(size_t(std::max(n_users, 1)) * b * 4);
  return t;
}

// ---- row shards (the multi-GPU host path): one factor shard's K-major
// copies + GEMM scratch in a caller workspace:
//   [copies(n, d)][split partials S x d x b][slab^T hi (b x d)][slab^T lo]
struct ShardWs {
  TcCopies c;
  float *P, *sth, *stl;
  int S, span;
};

static size_t shard_bytes(int n, int d, int b) {
  int S, span;
  gram_plan(std::max(n, 1), d, &S, &span);
  return copies_bytes(n, d) + al256(size_t(S) * d * b * 4) + 2 * al256(size_t(b) * d * 4) + 1024;
}

static int shard_carve(ials_session* s, void* ws, size_t ws_bytes, int n, int d, int b, ShardWs* w) {
  if (n < 0 || d < 1 || b < 1 || b > d) return fail(s, IALS_E_INVALID, "shard: bad sizes (n=%d d=%d b=%d)", n, d, b);
  if (!ws || ws_bytes < shard_bytes(n, d, b))
    return fail(s, IALS_E_NOMEM, "shard: workspace %zu < %zu bytes", ws_bytes, shard_bytes(n, d, b));
  char* t = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 1023) & ~uintptr_t(1023));
  t = carve_copies(t, n, d, &w->c);
  gram_plan(std::max(n, 1), d, &w->S, &w->span);
  w->P = reinterpret_cast<float*>(t);
  t += al256(size_t(w->S) * d * b * 4);
  w->sth = reinterpret_cast<float*>(t);
  t += al256(size_t(b) * d * 4);
  w->stl = reinterpret_cast<float*>(t);
  return IALS_OK;
}

size_t ials_shard_gemm_bytes(int32_t n_rows, int32_t d, int32_t b) { return shard_bytes(n_rows, d, b); }

int ials_shard_sync(ials_session* s, const float* F, int32_t ldf, int32_t n_rows, int32_t d, int32_t b,
                    int32_t c0, int32_t cw, void* ws, size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  ShardWs w;
  int rc = shard_carve(s, ws, ws_bytes, n_rows, d, b, &w);
  if (rc) return rc;
  if (c0 < 0 || cw < 0 || c0 + cw > d || (n_rows > 0 && (!F || ldf < d)))
    return fail(s, IALS_E_INVALID, "shard_sync: bad range");
  return sync_copies(s, F, ldf, d, c0, cw, w.c, S(stream));
}

int ials_shard_gramian(ials_session* s, int32_t n_rows, int32_t d, int32_t b, int32_t b0, int32_t bb,
                       float* slab, void* ws, size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  ShardWs w;
  int rc = shard_carve(s, ws, ws_bytes, n_rows, d, b, &w);
  if (rc) return rc;
  if (b0 < 0 || bb < 1 || bb > b || b0 + bb > d || !slab) return fail(s, IALS_E_INVALID, "shard_gramian: bad block");
  if (get_encode(s) != IALS_OK) return fail(s, IALS_E_CUDA, "shard_gramian: no cuTensorMapEncodeTiled");
  if (n_rows == 0) {
    CUDA_TRY(s, cudaMemsetAsync(slab, 0, size_t(d) * bb * 4, S(stream)));
    return IALS_OK;
  }
  return gram_tc(s, w.c, d, b0, bb, w.P, slab, w.sth, w.stl, S(stream));
}

int ials_shard_projection(ials_session* s, const float* F, int32_t ldf, int32_t n_rows, int32_t d,
                          int32_t b, int32_t bb, float* slab, float alpha0, float* proj, void* ws,
                          size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  ShardWs w;
  int rc = shard_carve(s, ws, ws_bytes, n_rows, d, b, &w);
  if (rc) return rc;
  if (bb < 1 || bb > b || !slab || (n_rows > 0 && (!F || !proj || ldf < d)))
    return fail(s, IALS_E_INVALID, "shard_projection: bad arguments");
  if (n_rows == 0) return IALS_OK;
  if (get_encode(s) != IALS_OK) return fail(s, IALS_E_CUDA, "shard_projection: no cuTensorMapEncodeTiled");
  cudaStream_t st = S(stream);
  // stage slab^T hi / lo from the (all-reduced) slab: the split reduction with one split
  k_gram_reduce<<<(d * bb + 255) / 256, 256, 0, st>>>(slab, 1, (long long)d * bb, d, bb, slab, w.sth, w.stl);
  LAUNCH_CHECK(s);
  return proj_tc(s, F, ldf, w.c, d, bb, w.sth, w.stl, alpha0, proj, st);
}

int ials_shard_apply_block(ials_session* s, const float* recv, int32_t nmax, const int32_t* bounds,
                           int32_t world, int32_t rank, const float* old_local, float* X, int32_t ldx,
                           int32_t b0, int32_t b, float* delta, int32_t n_rows, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (world < 1 || rank < 0 || rank >= world || nmax < 0 || b < 1 || b0 < 0 || ldx < b0 + b ||
      n_rows < 0 || !recv || !bounds || !X || !delta)
    return fail(s, IALS_E_INVALID, "shard_apply_block: bad arguments");
  if (n_rows == 0) return IALS_OK;
  const long long n = (long long)n_rows * b;
  k_apply_block<<<(int)std::min<long long>((n + 255) / 256, 16LL * kNumSMs), 256, 0, S(stream)>>>(
      recv, nmax, bounds, world, rank, old_local, X, ldx, b0, b, delta, n_rows);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// ---- rotated user passes over a row shard (the multi-GPU host path).  Every
// block's G_pp = H[:, pi]^T H[:, pi] is final at the start of an epoch, so the
// ranks form their partial diagonal blocks at once (ials_shard_diag_gramian),
// all-reduce the d x b stack, and every rank decomposes the same input
// (ials_shard_rot_prepare: one CTA per block, all blocks side by side).  A
// user pass then runs like ials_epoch's: rotated projection, F~ = H[:, pi] Q
// from the replicated H, W_loc[:, pi] Q, the rotated sweep, the back-rotation.
struct ShardRot {
  float *QT, *Qm, *rslab, *slabQT, *lam, *Ft, *WQ;
};
static size_t shard_rot_bytes(int n_rows, int n_fixed, int d, int b) {
  if (b != 128 || d % b) return 0;
  return 4 * al256(size_t(d) * b * 4) + al256(size_t(d) * 4) +
         al256(size_t(std::max(n_fixed, 1)) * b * 4) + al256(size_t(std::max(n_rows, 1)) * b * 4) + 1024;
}
static int shard_rot_carve(ials_session* s, void* ws, size_t bytes, int n_rows, int n_fixed, int d, int b,
                           ShardRot* r) {
  const size_t need = shard_rot_bytes(n_rows, n_fixed, d, b);
  if (!need) return fail(s, IALS_E_INVALID, "shard_rot: b must be 128 and divide d (d=%d b=%d)", d, b);
  if (!ws || bytes < need) return fail(s, IALS_E_NOMEM, "shard_rot: workspace %zu < %zu bytes", bytes, need);
  char* t = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 1023) & ~uintptr_t(1023));
  auto take = [&](size_t n) { float* p = reinterpret_cast<float*>(t); t += al256(n); return p; };
  r->QT = take(size_t(d) * b * 4);
  r->Qm = take(size_t(d) * b * 4);
  r->rslab = take(size_t(d) * b * 4);
  r->slabQT = take(size_t(d) * b * 4);
  r->lam = take(size_t(d) * 4);
  r->Ft = take(size_t(std::max(n_fixed, 1)) * b * 4);
  r->WQ = take(size_t(std::max(n_rows, 1)) * b * 4);
  return IALS_OK;
}

size_t ials_shard_rot_bytes(int32_t n_rows, int32_t n_fixed, int32_t d, int32_t b) {
  return shard_rot_bytes(n_rows, n_fixed, d, b);
}

int ials_rotation_available(int32_t d, int32_t b) {
  return (rot_enabled() && tc4_enabled() && b == 128 && d >= b && d % b == 0 && d / b <= 64) ? 1 : 0;
}

int ials_shard_diag_gramian(ials_session* s, int32_t n_rows, int32_t d, int32_t b, float* Gd, void* ws,
                            size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  ShardWs w;
  int rc = shard_carve(s, ws, ws_bytes, n_rows, d, b, &w);
  if (rc) return rc;
  if (!Gd || b != 128 || d % b) return fail(s, IALS_E_INVALID, "shard_diag_gramian: b must be 128 and divide d");
  cudaStream_t st = S(stream);
  if (n_rows == 0) {
    CUDA_TRY(s, cudaMemsetAsync(Gd, 0, size_t(d) * b * 4, st));
    return IALS_OK;
  }
  if (get_encode(s) != IALS_OK) return fail(s, IALS_E_CUDA, "shard_diag_gramian: no cuTensorMapEncodeTiled");
  rc = gemm_attrs(s);
  if (rc) return rc;
  CUtensorMap gm;   // F^T (d x n): A and B operands, B rows following the A tile
  rc = make_map(s, &gm, w.c.FT, w.c.n, d, w.c.ldt, 128);
  if (rc) return rc;
  const int nblk = d / b;
  GemmJob job{d, 0, 0, b, 128, w.c.n, w.span, w.P, b, (long long)d * b, 1.f};
  job.diag = 1;
  k_gemm3_tf32<<<dim3(nblk, w.S), kGemmThreads, GemmLay::BYTES, st>>>(gm, gm, gm, job);
  LAUNCH_CHECK(s);
  const size_t cnt = size_t(d) * b;
  k_reduce_splits_strided<<<(int)std::min<size_t>((cnt + 255) / 256, 4096), 256, 0, st>>>(
      w.P, w.S, (long long)d * b, cnt, Gd);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

int ials_shard_rot_prepare(ials_session* s, int32_t d, int32_t b, const float* Gd, int32_t n_rows,
                           int32_t n_fixed, void* rot_ws, size_t rot_bytes_, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  ShardRot r;
  int rc = shard_rot_carve(s, rot_ws, rot_bytes_, n_rows, n_fixed, d, b, &r);
  if (rc) return rc;
  if (!Gd) return fail(s, IALS_E_INVALID, "shard_rot_prepare: NULL Gd");
  rc = eig_attrs(s, b);
  if (rc) return rc;
  cudaStream_t st = S(stream);
  k_sym_eig<<<d / b, kEigThreads, eig_smem_bytes(b), st>>>(Gd, b, (long long)b * b, b, r.QT, r.lam, r.rslab,
                                                           r.Qm, nullptr, 1);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

int ials_shard_user_pass_rot(ials_session* s, const ials_side* side, const ials_sched* sched,
                             const float* fixed, int32_t ldf, float* own, int32_t ldo, int32_t d,
                             int32_t b0, int32_t b, float* slab, float alpha0, float* cache,
                             void* own_ws, size_t own_ws_bytes, void* rot_ws, size_t rot_bytes_,
                             void* workspace, size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (!side || !sched || !fixed || !own || !slab || !cache)
    return fail(s, IALS_E_INVALID, "shard_user_pass_rot: NULL argument");
  if (b != 128 || d % b || b0 % b || b0 < 0 || b0 + b > d)
    return fail(s, IALS_E_INVALID, "shard_user_pass_rot: bad block (d=%d b0=%d b=%d)", d, b0, b);
  if (sched->n_heavy != 0 || side->weights || side->labels)
    return fail(s, IALS_E_INVALID, "shard_user_pass_rot: unit weights and no heavy rows only");
  if (!tc4_enabled()) return fail(s, IALS_E_INVALID, "shard_user_pass_rot: the tensor-core sweep is disabled");
  if (side->n_rows == 0) return IALS_OK;
  ShardWs w;
  int rc = shard_carve(s, own_ws, own_ws_bytes, side->n_rows, d, b, &w);
  if (rc) return rc;
  ShardRot r;
  rc = shard_rot_carve(s, rot_ws, rot_bytes_, side->n_rows, side->n_fixed, d, b, &r);
  if (rc) return rc;
  if (get_encode(s) != IALS_OK) return fail(s, IALS_E_CUDA, "shard_user_pass_rot: no cuTensorMapEncodeTiled");
  cudaStream_t st = S(stream);
  char* pws = static_cast<char*>(workspace);
  const size_t need = pass_ws(side->n_rows, side->n_fixed, b, sched->n_slices, sched->n_heavy);
  if (!pws || ws_bytes < need)
    return fail(s, IALS_E_NOMEM, "shard_user_pass_rot: workspace %zu < %zu bytes", ws_bytes, need);
  const int zb = b0 / b;
  const float* qt = r.QT + size_t(zb) * b * b;
  // (slab Q)^T -> the rotated projection alpha0 W_loc slab Q; F~ = H[:, pi] Q; W_loc[:, pi] Q
  rc = gemm_nt(s, qt, b, b, b, 0, slab, d, b, b, 0, b, r.slabQT, d, 1.f, false, st);
  if (!rc) rc = proj_tc(s, own, ldo, w.c, d, b, r.slabQT, nullptr, alpha0, reinterpret_cast<float*>(pws), st);
  if (!rc) rc = gemm_nt(s, fixed, side->n_fixed, d, ldf, b0, qt, b, b, b, 0, b, r.Ft, b, 1.f, false, st);
  if (!rc) rc = gemm_nt(s, own, side->n_rows, d, ldo, b0, qt, b, b, b, 0, b, r.WQ, b, 1.f, false, st);
  if (rc) return rc;
  RotPass rp{r.Ft, r.WQ, r.lam + b0, r.rslab};
  rc = side_pass_impl(s, side, sched, fixed, ldf, own, ldo, d, b0, b, slab, alpha0, cache, 0, pws, ws_bytes,
                      st, true, nullptr, nullptr, &rp);
  if (rc) return rc;
  // W_loc[:, pi] -= d~ Q^T: the rows' steps back in the original basis
  return gemm_nt(s, pass_drow(pws, side, sched, b), side->n_rows, b, b, 0, r.Qm + size_t(zb) * b * b, b, b, b, 0,
                 b, own + b0, ldo, -1.f, true, st);
}

// optional phase events: 0 start, 1 after the cache, then per block
// (user Gramian, user pass, item Gramian, item pass) -> 2 + 4 * blocks
// (per host thread: the Python mirror sets them around one ials_epoch call
// and clears them after it, so concurrent epochs on other threads -- or other
// devices -- never record each other's events)
static thread_local cudaEvent_t g_ev[2 + 4 * 1024];
static thread_local int g_nev = 0;

int ials_epoch_events(void* const* events, int32_t n) {
  if (n < 0 || n > 2 + 4 * 1024 || (n > 0 && !events)) return IALS_E_INVALID;
  for (int i = 0; i < n; ++i) g_ev[i] = static_cast<cudaEvent_t>(events[i]);
  g_nev = n;
  return IALS_OK;
}

static cudaError_t rec_event(int k, cudaStream_t st) {
  if (k < g_nev && g_ev[k]) return cudaEventRecord(g_ev[k], st);
  return cudaSuccess;
}

// the eigendecompositions' side stream (highest priority: its CTAs take SMs as
// the predictions' retire) and its fork / join events
static int ensure_rot_stream(ials_session* s) {
  if (s->rot_st) return IALS_OK;
  int lo = 0, hi = 0;
  CUDA_TRY(s, cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CUDA_TRY(s, cudaStreamCreateWithPriority(&s->rot_st, cudaStreamNonBlocking, hi));
  CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_rot0, cudaEventDisableTiming));
  CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_rot1, cudaEventDisableTiming));
  return IALS_OK;
}

// ------------------------------------------------------------------ epoch
// host staging of ials_epoch_host (all pointers pinned host memory)
struct EpochHost {
  const void *W_in, *H_in;
  void *W_out, *H_out, *cache_out;
  int64_t ldw, ldh;
  // float64 host model (ials_epoch_host64): the copies go through device f64
  // staging (dense, ld = d) and cast kernels on the copy stream
  bool f64 = false;
  double *sW = nullptr, *sH = nullptr, *sC = nullptr;
};

static inline int cast_grid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8LL * kNumSMs));
}

// rows [r0, r1) of a host matrix (host ld in elements) -> device fp32 rows,
// on the copy stream (the caller orders it after / before the epoch's work)
static int host_rows_in(ials_session* s, const EpochHost* h, const void* src, int64_t lds, float* dst,
                        int ldd, int d, int r0, int r1, double* stage) {
  if (r1 <= r0 || d <= 0) return IALS_OK;
  const size_t rows = size_t(r1 - r0);
  if (!h->f64) {
    CUDA_TRY(s, cudaMemcpy2DAsync(dst + size_t(r0) * ldd, size_t(ldd) * 4,
                                  static_cast<const float*>(src) + size_t(r0) * lds, size_t(lds) * 4,
                                  size_t(d) * 4, rows, cudaMemcpyHostToDevice, s->copy_st));
    return IALS_OK;
  }
  double* sg = stage + size_t(r0) * d;
  CUDA_TRY(s, cudaMemcpy2DAsync(sg, size_t(d) * 8, static_cast<const double*>(src) + size_t(r0) * lds,
                                size_t(lds) * 8, size_t(d) * 8, rows, cudaMemcpyHostToDevice,
                                s->copy_st));
  k_f64_to_f32_2d<<<cast_grid(int64_t(rows) * d), 256, 0, s->copy_st>>>(sg, d, dst + size_t(r0) * ldd,
                                                                         ldd, d, int64_t(rows));
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// columns [c0, c0 + cw) of a device fp32 matrix (n rows) -> the host matrix,
// on the copy stream once the work queued on `st` so far has finished
static int host_cols_out(ials_session* s, cudaStream_t st, const EpochHost* h, void* dst, int64_t ldh_,
                         const float* src, int lds, int n, int d, int c0, int cw, double* stage) {
  if (n <= 0 || cw <= 0) return IALS_OK;
  CUDA_TRY(s, cudaEventRecord(s->ev_a, st));
  CUDA_TRY(s, cudaStreamWaitEvent(s->copy_st, s->ev_a, 0));
  if (!h->f64) {
    CUDA_TRY(s, cudaMemcpy2DAsync(static_cast<float*>(dst) + c0, size_t(ldh_) * 4, src + c0,
                                  size_t(lds) * 4, size_t(cw) * 4, size_t(n),
                                  cudaMemcpyDeviceToHost, s->copy_st));
    return IALS_OK;
  }
  k_f32_to_f64_2d<<<cast_grid(int64_t(n) * cw), 256, 0, s->copy_st>>>(src + c0, lds, stage + c0, d, cw, n);
  LAUNCH_CHECK(s);
  CUDA_TRY(s, cudaMemcpy2DAsync(static_cast<double*>(dst) + c0, size_t(ldh_) * 8, stage + c0,
                                size_t(d) * 8, size_t(cw) * 8, size_t(n), cudaMemcpyDeviceToHost,
                                s->copy_st));
  return IALS_OK;
}


// the passes of one epoch: p = 2 * block + side (0 user, 1 item); a range
// [pass0, pass0 + npass) runs exactly the code ials_epoch runs for them
struct PassRange {
  int pass0, npass;
  bool recompute;   // the prediction cache first (ials_epoch: yes)
};
static int epoch_impl(ials_session* s, const ials_side* users, const ials_sched* user_sched,
                      const ials_side* items, const ials_sched* item_sched, float* W, int32_t ldw,
                      float* H, int32_t ldh, int32_t d, int32_t b, float alpha0, float* cache,
                      void* workspace, size_t ws_bytes, void* stream, const EpochHost* host,
                      PassRange range = PassRange{0, 1 << 30, true});
static int radix_sort_index(ials_session* s, const int* keys, int64_t n, int K, int* keys_out,
                            int* vals_out, int* tk, int* tv, int* hist, int* tot, cudaStream_t st);

int ials_epoch(ials_session* s, const ials_side* users, const ials_sched* user_sched,
               const ials_side* items, const ials_sched* item_sched, float* W, int32_t ldw,
               float* H, int32_t ldh, int32_t d, int32_t b, float alpha0, float* cache,
               void* workspace, size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  return epoch_impl(s, users, user_sched, items, item_sched, W, ldw, H, ldh, d, b, alpha0, cache,
                    workspace, ws_bytes, stream, nullptr);
}

int ials_epoch_range(ials_session* s, const ials_side* users, const ials_sched* user_sched,
                     const ials_side* items, const ials_sched* item_sched, float* W, int32_t ldw,
                     float* H, int32_t ldh, int32_t d, int32_t b, float alpha0, float* cache,
                     void* workspace, size_t ws_bytes, void* stream, int32_t pass0, int32_t npass,
                     int32_t recompute_cache) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  const int nb = (b >= 1 && d >= 1) ? (d + b - 1) / b : 0;
  if (pass0 < 0 || npass < 0 || pass0 + npass > 2 * nb)
    return fail(s, IALS_E_INVALID, "epoch_range: passes [%d, %d) outside [0, %d)", pass0,
                pass0 + npass, 2 * nb);
  return epoch_impl(s, users, user_sched, items, item_sched, W, ldw, H, ldh, d, b, alpha0, cache,
                    workspace, ws_bytes, stream, nullptr,
                    PassRange{pass0, npass, recompute_cache != 0});
}

int ials_epoch_host(ials_session* s, const ials_side* users, const ials_sched* user_sched,
                    const ials_side* items, const ials_sched* item_sched, const float* W_in,
                    float* W_out, int64_t ldw_host, const float* H_in, float* H_out,
                    int64_t ldh_host, float* W, int32_t ldw, float* H, int32_t ldh, int32_t d,
                    int32_t b, float alpha0, float* cache, float* cache_out, void* workspace,
                    size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (!W_in || !W_out || !H_in || !H_out || ldw_host < d || ldh_host < d)
    return fail(s, IALS_E_INVALID, "epoch_host: bad host buffers");
  if (!s->copy_st) {
    CUDA_TRY(s, cudaStreamCreateWithFlags(&s->copy_st, cudaStreamNonBlocking));
    CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_a, cudaEventDisableTiming));
    CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_b, cudaEventDisableTiming));
  }
  const EpochHost h{W_in, H_in, W_out, H_out, cache_out, ldw_host, ldh_host};
  return epoch_impl(s, users, user_sched, items, item_sched, W, ldw, H, ldh, d, b, alpha0, cache,
                    workspace, ws_bytes, stream, &h);
}

int ials_host_register(void* ptr, size_t bytes) {
  if (!ptr || bytes == 0) return fail(nullptr, IALS_E_INVALID, "host_register: empty range");
  const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return IALS_OK;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, IALS_E_CUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
  }
  return IALS_OK;
}

int ials_host_unregister(void* ptr) {
  if (!ptr) return IALS_OK;
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(nullptr, IALS_E_CUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
  }
  return IALS_OK;
}

size_t ials_host64_staging_bytes(int32_t n_users, int32_t n_items, int32_t d, int64_t nnz) {
  return al256(size_t(std::max(n_users, 0)) * std::max(d, 0) * 8) +
         al256(size_t(std::max(n_items, 0)) * std::max(d, 0) * 8) + al256(size_t(std::max<int64_t>(nnz, 0)) * 8);
}

int ials_epoch_host64(ials_session* s, const ials_side* users, const ials_sched* user_sched,
                      const ials_side* items, const ials_sched* item_sched, const double* W_in,
                      double* W_out, int64_t ldw_host, const double* H_in, double* H_out,
                      int64_t ldh_host, float* W, int32_t ldw, float* H, int32_t ldh, int32_t d,
                      int32_t b, float alpha0, float* cache, double* cache_out, void* staging,
                      size_t staging_bytes, void* workspace, size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (!W_in || !W_out || !H_in || !H_out || ldw_host < d || ldh_host < d || !users || !items)
    return fail(s, IALS_E_INVALID, "epoch_host64: bad host buffers");
  if (!staging || staging_bytes < ials_host64_staging_bytes(users->n_rows, items->n_rows, d, users->nnz))
    return fail(s, IALS_E_NOMEM, "epoch_host64: staging %zu < %zu bytes", staging_bytes,
                ials_host64_staging_bytes(users->n_rows, items->n_rows, d, users->nnz));
  if (!s->copy_st) {
    CUDA_TRY(s, cudaStreamCreateWithFlags(&s->copy_st, cudaStreamNonBlocking));
    CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_a, cudaEventDisableTiming));
    CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_b, cudaEventDisableTiming));
  }
  EpochHost h{W_in, H_in, W_out, H_out, cache_out, ldw_host, ldh_host};
  char* t = static_cast<char*>(staging);
  h.f64 = true;
  h.sW = reinterpret_cast<double*>(t);
  t += al256(size_t(users->n_rows) * d * 8);
  h.sH = reinterpret_cast<double*>(t);
  t += al256(size_t(items->n_rows) * d * 8);
  h.sC = reinterpret_cast<double*>(t);
  return epoch_impl(s, users, user_sched, items, item_sched, W, ldw, H, ldh, d, b, alpha0, cache,
                    workspace, ws_bytes, stream, &h);
}

static int epoch_impl(ials_session* s, const ials_side* users, const ials_sched* user_sched,
                      const ials_side* items, const ials_sched* item_sched, float* W, int32_t ldw,
                      float* H, int32_t ldh, int32_t d, int32_t b, float alpha0, float* cache,
                      void* workspace, size_t ws_bytes, void* stream, const EpochHost* host,
                      PassRange range) {
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (!users || !items || !user_sched || !item_sched)
    return fail(s, IALS_E_INVALID, "epoch: NULL argument");
  if (b < 1 || b > d) return fail(s, IALS_E_INVALID, "epoch: bad block size %d", b);
  cudaStream_t st = S(stream);
  char* ws = static_cast<char*>(workspace);
  const size_t slab_bytes = al256(size_t(d) * b * 4);
  const size_t gbytes = gram_ws(0, d, b);
  if (ws_bytes < slab_bytes + gbytes) return fail(s, IALS_E_NOMEM, "epoch: workspace too small");
  float* slab = reinterpret_cast<float*>(ws);
  float* part = reinterpret_cast<float*>(ws + slab_bytes);
  char* pws = ws + slab_bytes + gbytes;
  size_t pbytes = ws_bytes - slab_bytes - gbytes;
  // tensor-core GEMMs (with the fused tensor-core sweep, b in 33..128): the
  // K-major copies live at the end of the workspace when it has room
  const size_t tcb = tc_gemm_bytes(users->n_rows, items->n_rows, d, b);
  const size_t pass_need =
      std::max(pass_ws(users->n_rows, users->n_fixed, b, user_sched->n_slices, user_sched->n_heavy),
               pass_ws(items->n_rows, items->n_fixed, b, item_sched->n_slices, item_sched->n_heavy));
  // the tensor-core region starts at the first 1 KB-aligned address at or
  // above ws + ws_bytes - tcb (tcb reserves the 1 KB this rounding can take),
  // so the pass scratch below it keeps all of ws_bytes - tcb
  char* tc_start = reinterpret_cast<char*>(
      (reinterpret_cast<uintptr_t>(ws) + (ws_bytes - std::min(tcb, ws_bytes)) + 1023) & ~uintptr_t(1023));
  // (b 8..16 keeps its FP32 SIMT sweep but takes the GEMMs: the slab and the
  // projection are bandwidth-bound reads of W / H, 145 + 68 us per block and side
  // on the SIMT kernels at d = 256, b = 16 against ~90 us here)
  const bool tc_sweep = tc4_enabled() && block_tile(b) == 128 && b > 16;
  const bool tc_gemm = tc4_enabled() && (tc_sweep || (b >= 8 && b <= 16 && b % 4 == 0)) && d % 4 == 0 &&
                       ldw % 4 == 0 && ldh % 4 == 0 && reinterpret_cast<uintptr_t>(W) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(H) % 16 == 0 && pbytes >= tcb &&
                       tc_start - pws >= (long long)pass_need && get_encode(s) == IALS_OK;
  TcCopies cw{}, ch{};
  float *P = nullptr, *sth = nullptr, *stl = nullptr;
  RotWs rw{};
  if (tc_gemm) {
    char* t = tc_start;
    pbytes = size_t(t - pws);
    t = carve_copies(t, users->n_rows, d, &cw);
    t = carve_copies(t, items->n_rows, d, &ch);
    int su, spu, si, spi;
    gram_plan(std::max(users->n_rows, 1), d, &su, &spu);
    gram_plan(std::max(items->n_rows, 1), d, &si, &spi);
    P = reinterpret_cast<float*>(t);
    t += al256(size_t(std::max(su, si)) * d * b * 4);
    sth = reinterpret_cast<float*>(t);
    t += al256(size_t(b) * d * 4);
    stl = reinterpret_cast<float*>(t);
    t += al256(size_t(b) * d * 4);
    if (rot_bytes(users->n_rows, items->n_rows, d, b))
      rot_carve(reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(t) + 1023) & ~uintptr_t(1023)),
                users->n_rows, items->n_rows, d, b, &rw);
  }
  if (host) {
    // H in full, then W in row chunks, host -> device on the copy stream; the
    // predictions of each user chunk start as soon as its rows have landed
    CUDA_TRY(s, cudaEventRecord(s->ev_a, st));   // W / H free on the device
    CUDA_TRY(s, cudaStreamWaitEvent(s->copy_st, s->ev_a, 0));
    int hr = host_rows_in(s, host, host->H_in, host->ldh, H, ldh, d, 0, items->n_rows, host->sH);
    if (hr) return hr;
  }
  if (tc_gemm && !host) {
    int rc = sync_copies(s, W, ldw, d, 0, d, cw, st);
    if (!rc) rc = sync_copies(s, H, ldh, d, 0, d, ch, st);
    if (rc) return rc;
  }
  // rotated user passes (ials_rot.cuh): every block's G_pp = H_pi^T H_pi is
  // final at the start of the epoch (H[:, pi] changes only in block pi's item
  // pass, after its user pass), so all eigendecompositions run here, on a
  // side stream beside the prediction cache
  const bool rot = tc_gemm && rot_enabled() && rw.Gd && d / b <= 64 && user_sched->n_heavy == 0 &&
                   !users->weights && !users->labels && user_sched->n_light > 0 && items->n_rows > 0;
  // Every block's G_pp = H_pi^T H_pi is final at the start of the epoch (H[:, pi]
  // changes only in block pi's item pass, after its user pass): the diagonal
  // Gram blocks are formed at once and decomposed one CTA per block on a
  // high-priority side stream, block pi's user pass waiting only for its own
  // (k_sym_eig returns at once for a G bit-identical to the one its outputs
  // were computed from -- the decompositions the previous epoch prepared for
  // this one, below).
  const int nblk = d / b;
  const long long rkey = ((long long)d << 40) ^ ((long long)items->n_rows << 8) ^ b;
  auto diag_gram = [&](int z0, int nz) -> int {   // Gd rows of blocks [z0, z0 + nz), on rot_st
    int S_i, span_i;
    gram_plan(std::max(items->n_rows, 1), d, &S_i, &span_i);
    CUtensorMap gm;   // H^T (d x n_items): A and B operands, B rows following the A tile
    int rc = make_map(s, &gm, ch.FT, ch.n, d, ch.ldt, 128);
    if (rc) return rc;
    GemmJob job{d, z0 * b, z0 * b, b, 128, ch.n, span_i, rw.Gpart, b, (long long)d * b, 1.f};
    job.diag = 1;
    k_gemm3_tf32<<<dim3(nz, S_i), kGemmThreads, GemmLay::BYTES, s->rot_st>>>(gm, gm, gm, job);
    LAUNCH_CHECK(s);
    // (the GEMM wrote rows [0, nz * b) of each split: rows of blocks z0.. relative to z0)
    const size_t cnt = size_t(nz) * b * b;
    k_reduce_splits_strided<<<(int)std::min<size_t>((cnt + 255) / 256, 4096), 256, 0, s->rot_st>>>(
        rw.Gpart, S_i, (long long)d * b, cnt, rw.Gd + size_t(z0) * b * b);
    LAUNCH_CHECK(s);
    return IALS_OK;
  };
  auto launch_eig = [&]() -> int {   // after H's K-major copy is current on st
    {
      const int rc0 = ensure_rot_stream(s);
      if (rc0) return rc0;
    }
    for (int z = 0; z < nblk; ++z)
      if (!s->ev_blk[z]) CUDA_TRY(s, cudaEventCreateWithFlags(&s->ev_blk[z], cudaEventDisableTiming));
    int rc = gemm_attrs(s);
    if (!rc) rc = eig_attrs(s, b);
    if (rc) return rc;
    CUDA_TRY(s, cudaEventRecord(s->ev_rot0, st));
    CUDA_TRY(s, cudaStreamWaitEvent(s->rot_st, s->ev_rot0, 0));
    rc = diag_gram(0, nblk);
    if (rc) return rc;
    // the outputs in place are trusted only if this session left them there
    // for this shape; otherwise every block is recomputed
    const int force = (s->rot_qm == rw.Qm && s->rot_key == rkey) ? 0 : 1;
    for (int z = 0; z < nblk; ++z) {
      const size_t o = size_t(z) * b * b;
      k_sym_eig<<<1, kEigThreads, eig_smem_bytes(b), s->rot_st>>>(rw.Gd + o, b, 0, b, rw.QT + o, rw.lam + z * b,
                                                                  rw.rslab + o, rw.Qm + o, rw.Gprev + o, force);
      LAUNCH_CHECK(s);
      CUDA_TRY(s, cudaEventRecord(s->ev_blk[z], s->rot_st));
    }
    s->rot_qm = rw.Qm;
    s->rot_key = rkey;
    return IALS_OK;
  };
  // after block zb's item pass (H[:, pi] final for the rest of the epoch, its
  // K-major copy synced on st): its decomposition for the next epoch
  auto prepare_next = [&](int zb) -> int {
    CUDA_TRY(s, cudaEventRecord(s->ev_rot0, st));
    CUDA_TRY(s, cudaStreamWaitEvent(s->rot_st, s->ev_rot0, 0));
    int rc = diag_gram(zb, 1);
    if (rc) return rc;
    const size_t o = size_t(zb) * b * b;
    k_sym_eig<<<1, kEigThreads, eig_smem_bytes(b), s->rot_st>>>(rw.Gd + o, b, 0, b, rw.QT + o, rw.lam + zb * b,
                                                                rw.rslab + o, rw.Qm + o, rw.Gprev + o, 0);
    LAUNCH_CHECK(s);
    return IALS_OK;
  };
  if (rot && !host) {
    const int rc = launch_eig();
    if (rc) return rc;
  }
  CUDA_TRY(s, rec_event(0, st));
  int rc = join_cache(s, st);   // (a failed earlier call may have left one pending)
  if (rc) return rc;
  // a pass's cache update beside the next pass's GEMM phase: opt-in (IALS_DEFER_CACHE=1).
  // Measured 88.1 -> 87.5 ms at L1 and 606 -> 604 ms at msd (the two contend for
  // L2 / HBM bandwidth), and it moves sweep work into the "gramian" phase events,
  // which would flatter the sweep's roofline fraction: off by default.
  static const bool kDefer = getenv("IALS_DEFER_CACHE") && getenv("IALS_DEFER_CACHE")[0] == '1';
  const bool defer = kDefer && tc_gemm && tc_sweep;
  // Host staging with the fused sweep: the first user pass runs chunk by
  // chunk of user rows, each chunk's sweep starting once its rows of W have
  // landed (with its predictions and projection), instead of after all of W.
  // Its light rows are grouped by chunk (stable: longest-first inside each)
  // in the split-partial scratch P, idle between the two Gramians of block 0.
  // (L1 e2e: 117.6 ms unchunked; 4 / 8 / 16 / 32 chunks 112.8 / 113.1 / 115.2 / 119.9 ms --
  // each chunk's sweep ends with its own tail; IALS_HOST_CHUNKS overrides, 0 or 1 = off)
  static const int kChunks = getenv("IALS_HOST_CHUNKS") ? std::max(1, std::min(64, atoi(getenv("IALS_HOST_CHUNKS")))) : 4;
  const int U = users->n_rows, per_chunk = (U + kChunks - 1) / kChunks;
  const int nl = user_sched->n_light;
  const size_t part_need = 4 * al256(size_t(std::max(nl, 1)) * 4) +
                           al256(size_t((nl + kRadixTile - 1) / kRadixTile + 1) * 256 * 4) + al256(256 * 4);
  // (rotated first pass: the grouped list is bucketed by (chunk, row class) and
  // each chunk runs its own b x b sweep and Woodbury tiles; IALS_HOST_CHUNKS_ROT=0
  // keeps the rotated first pass whole)
  static const bool kChunkRot = !(getenv("IALS_HOST_CHUNKS_ROT") && getenv("IALS_HOST_CHUNKS_ROT")[0] == '0');
  bool chunked = host && tc_gemm && tc_sweep && nl > 0 && kChunks > 1 && U >= kChunks &&
                 (!rot || (kChunkRot && b == 128));
  if (chunked) {
    int su, spu, si, spi;
    gram_plan(std::max(users->n_rows, 1), d, &su, &spu);
    gram_plan(std::max(items->n_rows, 1), d, &si, &spi);
    chunked = al256(size_t(std::max(su, si)) * d * b * 4) >= part_need;
  }
  ChunkPlan plan{};
  if (chunked) {
    CUDA_TRY(s, cudaEventRecord(s->ev_b, s->copy_st));   // H is on the device
    CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_b, 0));
    rc = sync_copies(s, H, ldh, d, 0, d, ch, st);
    if (!rc && rot) rc = launch_eig();   // the decompositions overlap W's upload
    if (rc) return rc;
    char* t = reinterpret_cast<char*>(P);
    int* keys = reinterpret_cast<int*>(t);
    t += al256(size_t(nl) * 4);
    int* skeys = reinterpret_cast<int*>(t);
    t += al256(size_t(nl) * 4);
    int* idx = reinterpret_cast<int*>(t);
    t += al256(size_t(nl) * 4);
    int* grouped = reinterpret_cast<int*>(t);
    t += al256(size_t(nl) * 4);
    int* tot = reinterpret_cast<int*>(t);
    t += al256(256 * 4);
    int* hist = reinterpret_cast<int*>(t);
    plan.nch = kChunks;
    plan.rows = grouped;
    plan.tot = tot;
    plan.prologue = [&, st, keys, skeys, idx, grouped, tot, hist](int c) -> int {
      if (c == 0) {   // after block 0's H Gramian, the last user of P before the sweep
        if (rot)
          k_chunk_class_keys<<<(nl + 255) / 256, 256, 0, st>>>(user_sched->light_rows, users->ptr, nl, per_chunk, keys);
        else
          k_chunk_keys<<<(nl + 255) / 256, 256, 0, st>>>(user_sched->light_rows, nl, per_chunk, keys);
        LAUNCH_CHECK(s);
        int r = radix_sort_index(s, keys, nl, rot ? 3 * kChunks : kChunks, skeys, idx, skeys, idx, hist, tot, st);
        if (r) return r;
        k_gather_i32<<<(nl + 255) / 256, 256, 0, st>>>(user_sched->light_rows, idx, nl, grouped);
        LAUNCH_CHECK(s);
      }
      const int r0 = c * per_chunk, r1 = std::min(U, r0 + per_chunk);
      if (r1 <= r0) return IALS_OK;
      int hr = host_rows_in(s, host, host->W_in, host->ldw, W, ldw, d, r0, r1, host->sW);
      if (hr) return hr;
      CUDA_TRY(s, cudaEventRecord(s->ev_b, s->copy_st));
      CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_b, 0));   // W rows [r0, r1) are on the device
      int r = ials_predictions(s, r1 - r0, users->ptr + r0, users->cols, W + size_t(r0) * ldw, ldw, H,
                               ldh, d, cache, stream);
      if (r) return r;
      TcCopies part = cw;
      part.n = r1 - r0;
      if (rot) {   // the chunk's rotated projection and its rows of W[:, pi] Q (block 0)
        r = proj_tc(s, W + size_t(r0) * ldw, ldw, part, d, b, rw.slabQT, nullptr, alpha0,
                    reinterpret_cast<float*>(pws) + size_t(r0) * b, st);
        if (!r)
          r = gemm_nt(s, W + size_t(r0) * ldw, r1 - r0, d, ldw, 0, rw.QT, b, b, b, 0, b,
                      rw.WQ + size_t(r0) * b, b, 1.f, false, st);
        return r;
      }
      return proj_tc(s, W + size_t(r0) * ldw, ldw, part, d, std::min(b, d), sth, stl, alpha0,
                     reinterpret_cast<float*>(pws) + size_t(r0) * std::min(b, d), st);
    };
  } else if (host) {
    if (tc_gemm && rot) {   // H first: its copies and the eigendecompositions overlap W's upload
      CUDA_TRY(s, cudaEventRecord(s->ev_b, s->copy_st));
      CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_b, 0));
      rc = sync_copies(s, H, ldh, d, 0, d, ch, st);
      if (!rc) rc = launch_eig();
      if (rc) return rc;
    }
    const int nch = 8;
    const int per = (U + nch - 1) / nch;
    for (int c = 0; c < nch && c * per < U; ++c) {
      const int r0 = c * per, r1 = std::min(U, r0 + per);
      rc = host_rows_in(s, host, host->W_in, host->ldw, W, ldw, d, r0, r1, host->sW);
      if (rc) return rc;
      CUDA_TRY(s, cudaEventRecord(s->ev_b, s->copy_st));
      CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_b, 0));   // H and W rows [0, r1) are on the device
      rc = ials_predictions(s, r1 - r0, users->ptr + r0, users->cols, W + size_t(r0) * ldw, ldw, H,
                            ldh, d, cache, stream);
      if (rc) return rc;
    }
    if (tc_gemm) {
      rc = sync_copies(s, W, ldw, d, 0, d, cw, st);
      if (!rc && !rot) rc = sync_copies(s, H, ldh, d, 0, d, ch, st);
      if (rc) return rc;
    }
  } else if (range.recompute) {
    rc = ials_predictions(s, users->n_rows, users->ptr, users->cols, W, ldw, H, ldh, d, cache,
                          stream);
    if (rc) return rc;
  }
  CUDA_TRY(s, rec_event(1, st));
  int ek = 2;
  for (int b0 = 0; b0 < d; b0 += b) {
    const int bb = std::min(b, d - b0);
    const bool first_chunked = chunked && b0 == 0;
    const int pu = 2 * (b0 / b);
    const bool do_u = pu >= range.pass0 && pu < range.pass0 + range.npass;
    const bool do_i = pu + 1 >= range.pass0 && pu + 1 < range.pass0 + range.npass;
    const int zb = b0 / b;
    const bool rot_u = rot && bb == 128;
    RotPass rp{rw.Ft, rw.WQ, rw.lam + b0, rw.rslab};
    if (do_u) {
    if (rot_u) CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_blk[zb], 0));   // this block's decomposition
    if (tc_gemm) {
      rc = gram_tc(s, ch, d, b0, bb, P, slab, sth, stl, st);
      if (!rc && rot_u) {
        // (slab Q)^T = Q^T slab^T -> the rotated projection alpha0 W slab Q;
        // F~ = H[:, pi] Q and W[:, pi] Q
        const float* qt = rw.QT + size_t(zb) * b * b;
        // (a chunked first pass forms its rows' projection and W Q chunk by chunk)
        rc = gemm_nt(s, qt, b, b, b, 0, slab, d, bb, bb, 0, b, rw.slabQT, d, 1.f, false, st);
        if (!rc && !first_chunked)
          rc = proj_tc(s, W, ldw, cw, d, bb, rw.slabQT, nullptr, alpha0, reinterpret_cast<float*>(pws), st);
        if (!rc) rc = gemm_nt(s, H, items->n_rows, d, ldh, b0, qt, b, b, b, 0, b, rw.Ft, b, 1.f, false, st);
        if (!rc && !first_chunked)
          rc = gemm_nt(s, W, users->n_rows, d, ldw, b0, qt, b, b, b, 0, b, rw.WQ, b, 1.f, false, st);
      } else if (!rc && !first_chunked) {
        rc = proj_tc(s, W, ldw, cw, d, bb, sth, stl, alpha0, reinterpret_cast<float*>(pws), st);
      }
    } else {
      rc = gramian_impl(s, H, items->n_rows, ldh, d, b0, bb, slab, part, gbytes, st);
    }
    if (rc) return rc;
    CUDA_TRY(s, rec_event(ek++, st));
    if (first_chunked) s->chunk = &plan;
    rc = side_pass_impl(s, users, user_sched, H, ldh, W, ldw, d, b0, bb, slab, alpha0, cache, 0,
                        pws, pbytes, st, tc_gemm, nullptr, items, rot_u ? &rp : nullptr,
                        defer ? al256(size_t(items->n_rows) * b * 4) : 0);
    s->chunk = nullptr;
    if (rc) return rc;
    if (rot_u) {   // W[:, pi] -= d~ Q^T: the rows' steps back in the original basis
      rc = gemm_nt(s, s->last_drow, users->n_rows, b, b, 0,
                   rw.Qm + size_t(zb) * b * b, b, b, b, 0, b, W + b0, ldw, -1.f, true, st);
      if (rc) return rc;
    }
    if (host) {   // W[:, b0:b0+bb] is final: back to the host beside the rest of the epoch
      rc = host_cols_out(s, st, host, host->W_out, host->ldw, W, ldw, users->n_rows, d, b0, bb,
                         host->sW);
      if (rc) return rc;
    }
    CUDA_TRY(s, rec_event(ek++, st));
    }   // do_u
    if (!do_i) continue;
    if (tc_gemm) {   // (chunked: W's copies are built here, after its first block)
      rc = first_chunked ? sync_copies(s, W, ldw, d, 0, d, cw, st)
                         : sync_copies(s, W, ldw, d, b0, bb, cw, st);
      if (!rc) rc = gram_tc(s, cw, d, b0, bb, P, slab, sth, stl, st);
      if (!rc) rc = proj_tc(s, H, ldh, ch, d, bb, sth, stl, alpha0, reinterpret_cast<float*>(pws), st);
    } else {
      rc = gramian_impl(s, W, users->n_rows, ldw, d, b0, bb, slab, part, gbytes, st);
    }
    if (rc) return rc;
    CUDA_TRY(s, rec_event(ek++, st));
    rc = side_pass_impl(s, items, item_sched, W, ldw, H, ldh, d, b0, bb, slab, alpha0, cache, 1,
                        pws, pbytes, st, tc_gemm, nullptr, users, nullptr,
                        defer ? al256(size_t(users->n_rows) * b * 4) : 0);
    if (rc) return rc;
    if (host) {
      rc = host_cols_out(s, st, host, host->H_out, host->ldh, H, ldh, items->n_rows, d, b0, bb,
                         host->sH);
      if (rc) return rc;
    }
    if (tc_gemm) {
      rc = sync_copies(s, H, ldh, d, b0, bb, ch, st);
      if (rc) return rc;
    }
    if (rot && zb + 1 < nblk) {   // (the last block's is prepared by the next epoch's start)
      rc = prepare_next(zb);
      if (rc) return rc;
    }
    CUDA_TRY(s, rec_event(ek++, st));
  }
  rc = join_cache(s, st);   // the last pass's cache update
  if (rc) return rc;
  if (rot) {   // the caller's stream covers the side stream's use of the workspace
    CUDA_TRY(s, cudaEventRecord(s->ev_rot1, s->rot_st));
    CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_rot1, 0));
  }
  if (host) {   // the maintained cache, then the caller's stream waits for every copy
    if (host->cache_out) {
      // one "row" of nnz entries (nnz < 2^31)
      rc = host_cols_out(s, st, host, host->cache_out, users->nnz, cache, (int)users->nnz, 1,
                         (int)users->nnz, 0, (int)users->nnz, host->sC);
      if (rc) return rc;
    }
    CUDA_TRY(s, cudaEventRecord(s->ev_b, s->copy_st));
    CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_b, 0));
  }
  return IALS_OK;
}

// ------------------------------------------------------------------ CSR
static int radix_passes(int K) {
  int p = 0;
  while (p < 4 && (int64_t(1) << (8 * p)) < int64_t(K)) ++p;
  return p;
}

size_t ials_build_csr_workspace_bytes(int64_t n) {
  const int64_t ntiles = (n + kRadixTile - 1) / kRadixTile;
  return 4 * al256(size_t(std::max<int64_t>(n, 1)) * 4) + al256(size_t(std::max<int64_t>(ntiles, 1)) * 256 * 4) +
         al256(256 * 4);
}

// stable sort of (keys, index) by keys in [0, K): LSD radix, 8-bit digits
static int radix_sort_index(ials_session* s, const int* keys, int64_t n, int K, int* keys_out,
                            int* vals_out, int* tk, int* tv, int* hist, int* tot, cudaStream_t st) {
  const int P = radix_passes(K);
  const int g = (int)((n + 255) / 256);
  if (P == 0) {   // one key: the identity permutation
    CUDA_TRY(s, cudaMemcpyAsync(keys_out, keys, size_t(n) * 4, cudaMemcpyDeviceToDevice, st));
    k_iota_i32<<<g, 256, 0, st>>>(n, vals_out);
    LAUNCH_CHECK(s);
    return IALS_OK;
  }
  const int ntiles = (int)((n + kRadixTile - 1) / kRadixTile);
  const int* ki = keys;
  const int* vi = nullptr;   // pass 0: value = index
  for (int p = 0; p < P; ++p) {
    // the last pass lands in keys_out / vals_out
    const bool to_out = ((P - 1 - p) % 2) == 0;
    int* ko = to_out ? keys_out : tk;
    int* vo = to_out ? vals_out : tv;
    k_radix_hist<<<ntiles, kRadixThreads, 0, st>>>(ki, n, 8 * p, hist);
    LAUNCH_CHECK(s);
    k_radix_scan<<<256, 256, 0, st>>>(hist, ntiles, tot);
    LAUNCH_CHECK(s);
    k_radix_scatter<<<ntiles, kRadixThreads, 0, st>>>(ki, vi, n, 8 * p, hist, tot, ko, vo);
    LAUNCH_CHECK(s);
    ki = ko;
    vi = vo;
  }
  return IALS_OK;
}

int ials_build_csr(ials_session* s, int32_t U, int32_t I, int64_t n, const int32_t* users,
                   const int32_t* items, int32_t* user_ptr, int32_t* user_cols, int32_t* order,
                   int32_t* item_ptr, int32_t* item_cols, int32_t* item_pos, void* workspace,
                   size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (U < 1 || I < 1 || n < 0 || n >= (int64_t(1) << 31))
    return fail(s, IALS_E_INVALID, "build_csr: bad sizes (U=%d I=%d n=%lld)", U, I, (long long)n);
  if (!user_ptr || !item_ptr || (n > 0 && (!users || !items || !user_cols || !order || !item_cols || !item_pos)))
    return fail(s, IALS_E_INVALID, "build_csr: NULL argument");
  if (ws_bytes < ials_build_csr_workspace_bytes(n))
    return fail(s, IALS_E_NOMEM, "build_csr: workspace %zu < %zu bytes", ws_bytes,
                ials_build_csr_workspace_bytes(n));
  cudaStream_t st = S(stream);
  char* w = static_cast<char*>(workspace);
  const size_t vb = al256(size_t(std::max<int64_t>(n, 1)) * 4);
  int* tk = reinterpret_cast<int*>(w);
  int* tv = reinterpret_cast<int*>(w + vb);
  int* su = reinterpret_cast<int*>(w + 2 * vb);   // users in canonical order
  int* si = reinterpret_cast<int*>(w + 3 * vb);   // user_cols in item order
  int* hist = reinterpret_cast<int*>(w + 4 * vb);
  int* tot = reinterpret_cast<int*>(w + 4 * vb + al256(size_t(std::max<int64_t>((n + kRadixTile - 1) / kRadixTile, 1)) * 256 * 4));
  const int g = (int)((n + 255) / 256);
  const int gp = (int)((n + 1 + 255) / 256);
  int rc = IALS_OK;
  if (n > 0) rc = radix_sort_index(s, users, n, U, su, order, tk, tv, hist, tot, st);
  if (rc) return rc;
  k_row_ptr<<<gp, 256, 0, st>>>(su, n, U, user_ptr);
  LAUNCH_CHECK(s);
  if (n == 0) {
    k_row_ptr<<<1, 256, 0, st>>>(su, 0, I, item_ptr);
    LAUNCH_CHECK(s);
    return IALS_OK;
  }
  k_gather_i32<<<g, 256, 0, st>>>(items, order, n, user_cols);
  LAUNCH_CHECK(s);
  rc = radix_sort_index(s, user_cols, n, I, si, item_pos, tk, tv, hist, tot, st);
  if (rc) return rc;
  k_row_ptr<<<gp, 256, 0, st>>>(si, n, I, item_ptr);
  LAUNCH_CHECK(s);
  k_gather_i32<<<g, 256, 0, st>>>(su, item_pos, n, item_cols);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// ------------------------------------------------------------------ ranking
int ials_topk(ials_session* s, int32_t n_rows, int32_t n_cols, float* scores, int64_t lds,
              const int32_t* ex_ptr, const int32_t* ex_cols, int32_t k, int32_t* out,
              int32_t* counts, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (n_rows < 0 || n_cols < 0 || lds < n_cols || k < 1 || k > kTopkMax)
    return fail(s, IALS_E_INVALID, "topk: bad sizes (rows=%d cols=%d k=%d, k <= %d)", n_rows, n_cols,
                k, kTopkMax);
  if (n_rows == 0) return IALS_OK;
  if (!scores || !out || !counts) return fail(s, IALS_E_INVALID, "topk: NULL argument");
  cudaStream_t st = S(stream);
  if (ex_ptr && ex_cols) {
    k_topk_exclude<<<n_rows, 256, 0, st>>>(scores, lds, ex_ptr, ex_cols);
    LAUNCH_CHECK(s);
  }
  k_topk<<<n_rows, kTopkThreads, 0, st>>>(scores, lds, n_cols, k, out, counts);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

int ials_topk64(ials_session* s, int32_t n_rows, int32_t n_cols, double* scores, int64_t lds,
                const int32_t* ex_ptr, const int32_t* ex_cols, int32_t k, int32_t* out,
                int32_t* counts, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (n_rows < 0 || n_cols < 0 || lds < n_cols || k < 1 || k > kTopkMax)
    return fail(s, IALS_E_INVALID, "topk64: bad sizes (rows=%d cols=%d k=%d, k <= %d)", n_rows,
                n_cols, k, kTopkMax);
  if (n_rows == 0) return IALS_OK;
  if (!scores || !out || !counts) return fail(s, IALS_E_INVALID, "topk64: NULL argument");
  cudaStream_t st = S(stream);
  if (ex_ptr && ex_cols) {
    k_topk_exclude64<<<n_rows, 256, 0, st>>>(scores, lds, ex_ptr, ex_cols);
    LAUNCH_CHECK(s);
  }
  k_topk64<<<n_rows, kTopkThreads, 0, st>>>(scores, lds, n_cols, k, out, counts);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// scores = E @ H^T (n_users x n_items) on the tensor core: the 3xTF32 TMA
// GEMM with blockIdx.y over 128-item tiles (FP32-accurate scores for
// rank_items / evaluate_holdout / ImplicitALS.recommend, metrics.py:57-119)
int ials_scores(ials_session* s, const float* E, int32_t lde, int32_t n_users, const float* H,
                int32_t ldh, int32_t n_items, int32_t d, float* out, int32_t ldo, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (n_users < 0 || n_items < 0 || d < 1 || lde < d || ldh < d || ldo < n_items)
    return fail(s, IALS_E_INVALID, "scores: bad shape (users=%d items=%d d=%d)", n_users, n_items, d);
  if (n_users == 0 || n_items == 0) return IALS_OK;
  if (!E || !H || !out || lde % 4 || ldh % 4 || reinterpret_cast<uintptr_t>(E) % 16 ||
      reinterpret_cast<uintptr_t>(H) % 16)
    return fail(s, IALS_E_INVALID, "scores: E / H must be 16-byte aligned with ld %% 4 == 0");
  int rc = gemm_attrs(s);
  if (!rc) rc = get_encode(s);
  if (rc) return rc;
  CUtensorMap am, bm;
  rc = make_map(s, &am, E, d, n_users, lde, 128);
  if (!rc) rc = make_map(s, &bm, H, d, n_items, ldh, 128);
  if (rc) return rc;
  const int nt = (n_items + 127) / 128;
  GemmJob job{n_users, 0, 0, n_items, 128, d, rup(d, kGemmKC), out, ldo, 0, 1.f};
  job.n_tiles = nt;
  k_gemm3_tf32<<<dim3((n_users + 127) / 128, nt), kGemmThreads, GemmLay::BYTES, S(stream)>>>(am, bm, bm, job);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// ------------------------------------------------------------------ loss
size_t ials_loss_workspace_bytes(int32_t d) {
  return 2 * al256(size_t(d) * d * 4) + gram_ws(0, d, d) +
         al256(size_t(kLossBlocks) * 4 * sizeof(double));
}

int ials_loss_terms(ials_session* s, const ials_side* users, const ials_side* items,
                    const float* W, int32_t ldw, const float* H, int32_t ldh, int32_t d,
                    double* out, void* workspace, size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (!users || !items || !W || !H || !out) return fail(s, IALS_E_INVALID, "loss: NULL argument");
  cudaStream_t st = S(stream);
  // workspace: [gw d*d][gh d*d][gram partials][block partials (doubles)]
  char* w = static_cast<char*>(workspace);
  const size_t gsz = al256(size_t(d) * d * 4);
  const size_t psz = gram_ws(0, d, d);
  const size_t rsz = al256(size_t(kLossBlocks) * 4 * sizeof(double));
  if (ws_bytes < 2 * gsz + psz + rsz) return fail(s, IALS_E_NOMEM, "loss: workspace too small");
  float* gw = reinterpret_cast<float*>(w);
  float* gh = reinterpret_cast<float*>(w + gsz);
  float* part = reinterpret_cast<float*>(w + 2 * gsz);
  double* red = reinterpret_cast<double*>(w + 2 * gsz + psz);
  int rc = gramian_impl(s, W, users->n_rows, ldw, d, 0, d, gw, part, psz, st);
  if (rc) return rc;
  rc = gramian_impl(s, H, items->n_rows, ldh, d, 0, d, gh, part, psz, st);
  if (rc) return rc;
  k_loss_observed<<<kLossBlocks, 256, 0, st>>>(users->n_rows, users->ptr, users->cols,
                                               users->labels, users->weights, W, ldw, H, ldh, d,
                                               red);
  LAUNCH_CHECK(s);
  k_loss_dot<<<kLossBlocks, 256, 0, st>>>(gw, gh, size_t(d) * d, red + kLossBlocks);
  LAUNCH_CHECK(s);
  k_loss_rownorm<<<kLossBlocks, 256, 0, st>>>(W, users->n_rows, ldw, d, users->lam,
                                              red + 2 * kLossBlocks);
  LAUNCH_CHECK(s);
  k_loss_rownorm<<<kLossBlocks, 256, 0, st>>>(H, items->n_rows, ldh, d, items->lam,
                                              red + 3 * kLossBlocks);
  LAUNCH_CHECK(s);
  k_loss_final<<<1, 256, 0, st>>>(red, out);
  LAUNCH_CHECK(s);
  return IALS_OK;
}

// ------------------------------------------------------------------ multi-GPU epoch
#include "ials_shard_epoch.cuh"
