/*
 * ials_b200.h -- C ABI of the B200-native iALS++ block solver (libials_b200.so).
 *
 * The reference (blockals 0.1.0, /root/reference/pkg/src/blockals) is a pure
 * Python/NumPy package and has no FFI.  Its drop-in boundary is its Python
 * API; every entry point below replaces the numerical core of one reference
 * function, and the host mirror (paper_2110_14044_b200/ Python modules, bound with
 * ctypes) keeps the reference names, argument meaning and error behaviour:
 *
 *   ials_predictions       <- compute_predictions   model.py:153-165
 *   ials_partial_gramian   <- partial_gramian       linalg.py:39-45
 *   ials_side_pass         <- _newton_side_pass     solvers.py:152-186
 *                             (+ _solve_rows :101-114, SingularMatrixError linalg.py:18-28)
 *   ials_epoch             <- ialspp_epoch          solvers.py:340-375
 *   ials_loss_terms        <- compute_loss          model.py:168-188 (device reductions)
 *   ials_build_csr         <- InteractionDataset.__init__ + user_view / item_view
 *                             data.py:98-134,148-162 (device stable radix sorts)
 *   ials_topk              <- top_k_from_scores     metrics.py:31-57 (fold-in evaluation)
 *
 * Conventions
 *   - All array arguments are DEVICE pointers (memory owned by the caller,
 *     e.g. torch tensors); no function allocates device memory except the
 *     session (error word).  Scratch comes from the caller's workspace, sized
 *     with ials_workspace_bytes().
 *   - Every call is stream-ordered on `stream` (a cudaStream_t passed as
 *     void*) and does not synchronise the host.
 *   - Return 0 on success or a negative IALS_E_* code.  The last error text
 *     is available from ials_last_error().  A singular block Hessian does not
 *     fail the launch: it sets the session's device error word, read back
 *     with ials_check_singular() (which synchronises the stream).
 *   - Factor tables are row-major fp32 with leading dimension ld >= d.
 *   - Indices are int32 (|S| < 2^31 is checked by the host mirror).
 */
#ifndef IALS_B200_H
#define IALS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IALS_OK 0
#define IALS_E_INVALID (-1)   /* -> ValueError                    */
#define IALS_E_SINGULAR (-2)  /* -> SingularMatrixError(row,pivot) */
#define IALS_E_CUDA (-3)      /* -> RuntimeError                  */
#define IALS_E_NOMEM (-4)     /* workspace too small -> ValueError */

/* One side of the interaction matrix (reference SideView, data.py:26-52).
 * Rows are users (user pass) or items (item pass); entry e of row r lives in
 * [ptr[r], ptr[r+1]).  pos[e] is the canonical (user-major) score-cache slot
 * of the entry (data.py:156-162); NULL means identity (user view).  labels /
 * weights NULL mean all ones. */
typedef struct ials_side {
  int32_t n_rows;          /* rows of the side being updated            */
  int32_t n_fixed;         /* rows of the opposite (fixed) side         */
  int64_t nnz;             /* entries                                   */
  const int32_t* ptr;      /* [n_rows + 1]                              */
  const int32_t* cols;     /* [nnz] fixed-side row of each entry        */
  const float* labels;     /* [nnz] y, or NULL                          */
  const float* weights;    /* [nnz] alpha, or NULL                      */
  const int32_t* pos;      /* [nnz] cache slot, or NULL                 */
  const float* lam;        /* [n_rows] effective_reg (model.py:144-150) */
  const int32_t* rows;     /* [nnz] row of each entry, or NULL (enables the
                              entry-parallel cache pass of the fused sweep) */
} ials_side;

/* Work schedule of one side for one block width (built once per dataset by
 * ials_schedule_* on the host mirror): light rows are solved by one fused
 * kernel in descending-degree order; heavy rows are split into slices whose
 * partial Hessians are reduced in a fixed order (deterministic). */
typedef struct ials_sched {
  int32_t n_light;
  const int32_t* light_rows;    /* [n_light]                                  */
  int32_t n_heavy;
  const int32_t* heavy_rows;    /* [n_heavy]                                  */
  const int32_t* heavy_slice0;  /* [n_heavy + 1] first slice of each heavy row */
  int32_t n_slices;
  const int32_t* slice_heavy;   /* [n_slices] heavy index of each slice        */
  const int32_t* slice_begin;   /* [n_slices] absolute entry range             */
  const int32_t* slice_end;     /* [n_slices]                                  */
  /* light rows (descending degree) with more than 64 / 32 interactions: the
   * prefix lengths that split the rotated user pass between the b x b sweep
   * and the Woodbury tiles of 2 and 4 rows */
  int32_t n_deg_gt64;
  int32_t n_deg_gt32;
} ials_sched;

/* Row segments of at most a few hundred entries each (the gather-dot kernels
 * of the multi-GPU path walk these instead of whole rows, so one long item
 * row does not serialise a warp): segment t covers entries [beg[t], end[t])
 * of local row row[t]. */
typedef struct ials_segs {
  int32_t n;
  const int32_t* row;
  const int32_t* beg;
  const int32_t* end;
} ials_segs;

typedef struct ials_session ials_session;
typedef struct ials_comm ials_comm;

int ials_version(void);
int ials_session_create(int device, ials_session** out);
int ials_session_destroy(ials_session* s);
/* Copies the last error message (NUL-terminated) into buf. */
int ials_last_error(ials_session* s, char* buf, size_t len);
/* Clear the device error word (stream-ordered). */
int ials_reset_singular(ials_session* s, void* stream);
/* Synchronises `stream`; returns IALS_E_SINGULAR and fills row/pivot/side
 * (0 user, 1 item) if a non-positive pivot was met since the last reset. */
int ials_check_singular(ials_session* s, void* stream, int64_t* row, int32_t* pivot,
                        int32_t* side);

/* Sweep engine for block widths 33..128: 0 = FP32 SIMT sweep, 1 = tcgen05
 * (3xTF32) wave kernels for b in 33..128, 2 = fused tcgen05 sweep for b in
 * 33..128 (4 rows in flight per SM; rows whose Cholesky pivots cancel more
 * than IALS_TC_COND (default 256) x -- 16 x for b <= 64 -- are re-solved by
 * the SIMT sweep).
 * Returns the previous setting.  The IALS_TC environment variable sets the
 * initial mode (default 2). */
int ials_set_tensor_cores(int enable);

/* Number of rows the fused tensor-core sweep handed to the SIMT sweep since
 * the session was created (or last reset); synchronises `stream`. */
int ials_tc_redo_rows(ials_session* s, void* stream, int64_t* total, int32_t reset);

/* The fused tensor-core sweep's cancellation limit (> 1); returns the
 * previous value.  IALS_TC_COND sets the initial value. */
float ials_set_tc_cond_max(float v);

/* Profiling only: a device buffer (>= 8 * 1024 int64) that kernels fill with
 * per-CTA phase timestamps (clock64), or NULL to disable. */
int ials_debug_timestamps(void* dev_buf);

/* Heavy-row threshold (entries) used by the schedule for block width b. */
int64_t ials_heavy_threshold(int32_t b);
/* Slice length (entries) of heavy rows for block width b. */
int64_t ials_slice_len(int32_t b);

/* Bytes of scratch ials_side_pass / ials_partial_gramian / ials_epoch need. */
size_t ials_workspace_bytes(int32_t n_rows_max, int32_t n_fixed_max, int32_t d, int32_t b,
                            int32_t n_slices_max, int32_t n_heavy_max);


/* out[e] = <W[user of e], H[col e]> for the user-major CSR (ptr, cols). */
int ials_predictions(ials_session* s, int32_t n_rows, const int32_t* ptr, const int32_t* cols,
                     const float* W, int32_t ldw, const float* H, int32_t ldh, int32_t d,
                     float* out, void* stream);

/* Same as ials_predictions over a list of row segments: segment t covers
 * entries [seg_beg[t], seg_end[t]) of row seg_row[t] (long rows spread over
 * many warps; used for the item-major cache of the sharded path). */
int ials_predictions_segments(ials_session* s, int32_t n_seg, const int32_t* seg_row,
                              const int32_t* seg_beg, const int32_t* seg_end, const int32_t* cols,
                              const float* W, int32_t ldw, const float* H, int32_t ldh, int32_t d,
                              float* out, void* stream);

/* Sharded path (dual-cache delta scheme): over row segments
 * of a local CSR, out[e] += <A[row][b0 .. b0+b), D[cols[e]][0 .. b)> -- the
 * score change the other side's last half-epoch (delta D of its column
 * block) caused.  No reference counterpart (the reference is single-process).
 * b <= 256. */
int ials_cache_correct(ials_session* s, int32_t n_seg, const int32_t* seg_row,
                       const int32_t* seg_beg, const int32_t* seg_end, const int32_t* cols,
                       const float* A, int32_t lda, int32_t b0, const float* D, int32_t ldd,
                       int32_t b, float* out, void* stream);

/* slab[t][j] = sum_r M[r][t] * M[r][b0 + j]  (d x b, row-major, ld = b). */
int ials_partial_gramian(ials_session* s, const float* M, int32_t n, int32_t ldm, int32_t d,
                         int32_t b0, int32_t b, float* slab, void* workspace, size_t ws_bytes,
                         void* stream);

/* One exact Newton step on columns [b0, b0+b) of every row of `side`
 * (reference _newton_side_pass, solvers.py:152-186): reads `fixed`
 * (n_fixed x d) and the slab (d x b, from ials_partial_gramian of `fixed`),
 * updates own[:, b0:b0+b] and the score cache in place.  side_id (0 user,
 * 1 item) only labels a singular-row report. */
int ials_side_pass(ials_session* s, const ials_side* side, const ials_sched* sched,
                   const float* fixed, int32_t ldf, float* own, int32_t ldo, int32_t d,
                   int32_t b0, int32_t b, const float* slab, float alpha0, float* cache,
                   int32_t side_id, void* workspace, size_t ws_bytes, void* stream);

/* One full iALS++ epoch (ialspp_epoch, solvers.py:340-375) over contiguous
 * blocks of width b (the last keeps the remainder): cache recompute, then
 * per block slab(H) -> user pass -> slab(W) -> item pass. */
/* Profiling: cudaEvent_t handles that ials_epoch records at its phase
 * boundaries (0: start, 1: after the prediction cache, then per block: after
 * the user-side Gramian, after the user pass, after the item-side Gramian,
 * after the item pass); n = 0 disables.  At most 2 + 4 * 1024 events. */
int ials_epoch_events(void* const* events, int32_t n);

/* Extra workspace ials_epoch can use for its tensor-core GEMM path (b in
 * 33..128 with the fused sweep): K-major copies of W and H and the Gramian
 * split partials.  Pass a workspace of ials_workspace_bytes(...) plus this
 * to enable it; with less, the epoch uses the FP32 SIMT GEMMs. */
size_t ials_epoch_tc_bytes(int32_t n_users, int32_t n_items, int32_t d, int32_t b);

int ials_epoch(ials_session* s, const ials_side* users, const ials_sched* user_sched,
               const ials_side* items, const ials_sched* item_sched, float* W, int32_t ldw,
               float* H, int32_t ldh, int32_t d, int32_t b, float alpha0, float* cache,
               void* workspace, size_t ws_bytes, void* stream);

/* The passes [pass0, pass0 + npass) of ials_epoch, pass p = 2 * block + side
 * (0 user, 1 item), with the prediction cache recomputed first when
 * recompute_cache != 0: exactly the code ials_epoch runs for those passes
 * (same GEMMs, sweep kernels and schedules), so a caller (the parity tests)
 * can inspect the state between passes.  ials_epoch == ials_epoch_range(...,
 * 0, 2 * ceil(d / b), 1). */
int ials_epoch_range(ials_session* s, const ials_side* users, const ials_sched* user_sched,
                     const ials_side* items, const ials_sched* item_sched, float* W, int32_t ldw,
                     float* H, int32_t ldh, int32_t d, int32_t b, float alpha0, float* cache,
                     void* workspace, size_t ws_bytes, void* stream, int32_t pass0, int32_t npass,
                     int32_t recompute_cache);

/* ials_epoch for a model held in (pinned) HOST memory, the reference's
 * in-place ialspp_epoch contract end to end: W_in / H_in are copied to the
 * device buffers W / H, the epoch runs, and W_out / H_out (may alias the
 * inputs) and cache_out (NULL to skip) receive the results.  The copies run
 * on a second stream and overlap the epoch: H and W (in row chunks, each
 * chunk's predictions starting as it lands) on the way in, each column block
 * W[:, pi] / H[:, pi] as soon as its side pass has finished it on the way
 * out.  With the tensor-core path the first user pass also runs by row chunk
 * (IALS_HOST_CHUNKS, default 4): each chunk's projection and sweep start once
 * its rows of W have landed.  Results are bit-identical to ials_epoch.  Host
 * leading dimensions in elements.  Stream-ordered on `stream`. */
int ials_epoch_host(ials_session* s, const ials_side* users, const ials_sched* user_sched,
                    const ials_side* items, const ials_sched* item_sched, const float* W_in,
                    float* W_out, int64_t ldw_host, const float* H_in, float* H_out,
                    int64_t ldh_host, float* W, int32_t ldw, float* H, int32_t ldh, int32_t d,
                    int32_t b, float alpha0, float* cache, float* cache_out, void* workspace,
                    size_t ws_bytes, void* stream);

/* ials_epoch_host for the reference's own float64 model (FactorModel's
 * C-contiguous f64 W / H, PredictionCache's f64 scores): the same overlapped
 * epoch, with every host copy going through device float64 staging and a cast
 * kernel on the copy stream (f64 -> fp32 round-to-nearest on the way in, exact
 * fp32 -> f64 on the way out), so the host does no conversion and no extra
 * pass over the model.  `staging` (device) holds ials_host64_staging_bytes.
 * Host buffers should be page-locked (cudaHostRegister) for the copies to
 * overlap; pageable buffers work but serialise. */
/* Multi-GPU column-block exchange (one process per GPU, replicated W / H):
 * after the all-gather of every rank's updated rows of X[:, b0:b0+b] into
 * recv (rank r's rows bounds[r]..bounds[r+1] at recv + r * nmax * b, b floats
 * per row), write the other ranks' rows into X and form the block's change
 * delta (n_rows x b, new - old; old_local = this rank's pre-sweep rows).
 * bounds: device array of world + 1 row offsets. */
int ials_shard_apply_block(ials_session* s, const float* recv, int32_t nmax, const int32_t* bounds,
                           int32_t world, int32_t rank, const float* old_local, float* X, int32_t ldx,
                           int32_t b0, int32_t b, float* delta, int32_t n_rows, void* stream);

/* Rotated user passes (b = 128, unit weights, no heavy user rows): per block
 * the eigendecomposition of G_pp, rows with <= 64 interactions solved through
 * their Woodbury systems (ials_rot.cuh, ials_sweep_wb.cuh).  Default on
 * (IALS_ROT=0 in the environment turns it off); returns the previous value. */
int ials_set_rotation(int enable);

/* Symmetric eigendecomposition of n_mat b x b matrices (b even, <= 128; cyclic
 * Jacobi, one CTA each, fp32): A_z at A + z * stride (ld lda) -> QT_z (b x b, row j =
 * eigenvector j), lam_z (b), and Q_z (b x b, column j = eigenvector j). */
int ials_sym_eig(ials_session* s, int32_t n_mat, int32_t b, const float* A, int32_t lda,
                 int64_t stride, float* QT, float* lam, float* Q, void* stream);

/* Page-lock (cudaHostRegister, portable) / release a caller's host range in
 * place, so ials_epoch_host64 copies overlap the epoch without a host-side
 * staging copy.  Registering an already registered range is not an error. */
int ials_host_register(void* ptr, size_t bytes);
int ials_host_unregister(void* ptr);
size_t ials_host64_staging_bytes(int32_t n_users, int32_t n_items, int32_t d, int64_t nnz);
int ials_epoch_host64(ials_session* s, const ials_side* users, const ials_sched* user_sched,
                      const ials_side* items, const ials_sched* item_sched, const double* W_in,
                      double* W_out, int64_t ldw_host, const double* H_in, double* H_out,
                      int64_t ldh_host, float* W, int32_t ldw, float* H, int32_t ldh, int32_t d,
                      int32_t b, float alpha0, float* cache, double* cache_out, void* staging,
                      size_t staging_bytes, void* workspace, size_t ws_bytes, void* stream);

/* Workspace bytes for ials_loss_terms at embedding dimension d. */
size_t ials_loss_workspace_bytes(int32_t d);

/* Device loss pieces (compute_loss, model.py:168-188), all in fp64:
 * out[0] = sum_e w_e (yhat_e - y_e)^2 over the user-major CSR,
 * out[1] = <W^T W, H^T H>, out[2] = sum_u lam_u |w_u|^2, out[3] = sum_i lam_i |h_i|^2. */
int ials_loss_terms(ials_session* s, const ials_side* users, const ials_side* items,
                    const float* W, int32_t ldw, const float* H, int32_t ldh, int32_t d,
                    double* out, void* workspace, size_t ws_bytes, void* stream);

/* Number of kernels this library has launched since it was loaded (every
 * launch site counts itself; stream captures count when captured, graph
 * replays do not).  bench.py reads it around its timed region. */
int64_t ials_launch_count(void);

/* ---- multi-GPU host path: tensor-core GEMMs on a ROW SHARD of a factor table
 * (one rank's contiguous rows of W or H; ials_epoch keeps its own copies).
 * The caller workspace (ials_shard_gemm_bytes) holds the shard's K-major TF32
 * copies -- refresh them with ials_shard_sync after the shard's rows change
 * -- and the GEMM scratch; b is the block width the workspace is sized for. */
size_t ials_shard_gemm_bytes(int32_t n_rows, int32_t d, int32_t b);
int ials_shard_sync(ials_session* s, const float* F, int32_t ldf, int32_t n_rows, int32_t d,
                    int32_t b, int32_t c0, int32_t cw, void* ws, size_t ws_bytes, void* stream);
/* partial slab over the shard: slab[d x bb] = F_shard^T F_shard[:, b0:b0+bb]
 * (partial_gramian, linalg.py:39-45; the caller all-reduces across ranks) */
int ials_shard_gramian(ials_session* s, int32_t n_rows, int32_t d, int32_t b, int32_t b0, int32_t bb,
                       float* slab, void* ws, size_t ws_bytes, void* stream);
/* proj[n_rows x bb] = alpha0 * F_shard @ slab (the alpha0 U[r,:] @ slab term of
 * _newton_side_pass, solvers.py:175), slab the all-reduced d x bb slab */
int ials_shard_projection(ials_session* s, const float* F, int32_t ldf, int32_t n_rows, int32_t d,
                          int32_t b, int32_t bb, float* slab, float alpha0, float* proj, void* ws,
                          size_t ws_bytes, void* stream);
/* ials_side_pass with the projection precomputed (proj: n_rows x b). */
int ials_side_pass_projected(ials_session* s, const ials_side* side, const ials_sched* sched,
                             const float* fixed, int32_t ldf, float* own, int32_t ldo, int32_t d,
                             int32_t b0, int32_t b, const float* slab, const float* proj,
                             float alpha0, float* cache, int32_t side_id, void* workspace,
                             size_t ws_bytes, void* stream);

/* Rotated user passes over a row shard (b = 128 dividing d, unit weights, no
 * heavy user rows): the sharded form of ials_epoch's rotated pass
 * (_newton_side_pass, solvers.py:152-186, in the eigenbasis of G_pp).
 *  1. ials_shard_diag_gramian: Gd (d x b; rows [z b, (z+1) b) = the partial
 *     G_zz = F_shard[:, z]^T F_shard[:, z] of every block z) from the ITEM
 *     shard's K-major copies (ws = its ials_shard_gemm_bytes workspace); the
 *     caller all-reduces Gd across ranks (every G_zz is final at epoch start);
 *  2. ials_shard_rot_prepare: every block's eigendecomposition into rot_ws
 *     (ials_shard_rot_bytes(local users, items, d, b)), one CTA per block;
 *  3. ials_shard_user_pass_rot: block b0's user pass on the local user rows
 *     (own = W_local, own_ws = its shard workspace, fixed = the replicated H,
 *     slab = the all-reduced d x b slab, workspace = ials_workspace_bytes). */
size_t ials_shard_rot_bytes(int32_t n_rows, int32_t n_fixed, int32_t d, int32_t b);
/* 1 when user passes of width b at dimension d can run rotated (b = 128
 * dividing d, at most 64 blocks, rotation and the tensor-core sweep enabled). */
int ials_rotation_available(int32_t d, int32_t b);
int ials_shard_diag_gramian(ials_session* s, int32_t n_rows, int32_t d, int32_t b, float* Gd, void* ws,
                            size_t ws_bytes, void* stream);
int ials_shard_rot_prepare(ials_session* s, int32_t d, int32_t b, const float* Gd, int32_t n_rows,
                           int32_t n_fixed, void* rot_ws, size_t rot_bytes, void* stream);
int ials_shard_user_pass_rot(ials_session* s, const ials_side* side, const ials_sched* sched,
                             const float* fixed, int32_t ldf, float* own, int32_t ldo, int32_t d,
                             int32_t b0, int32_t b, float* slab, float alpha0, float* cache,
                             void* own_ws, size_t own_ws_bytes, void* rot_ws, size_t rot_bytes,
                             void* workspace, size_t ws_bytes, void* stream);

/* ---- multi-GPU epoch (one process per GPU, contiguous row
 * shards of users and items, W and H replicated on every rank).  The
 * communicator wraps an NCCL communicator over the ranks' GPUs; libnccl.so.2 is
 * opened at run time (the process's own copy under a PyTorch host).
 *   rank 0:     ials_comm_unique_id(id)   -> 128 bytes, sent to every rank by
 *               the host's own means (MPI, a socket, torch.distributed ...)
 *   every rank: ials_comm_create(sess, id, rank, world, &comm)
 * With id == NULL and world == 1 the communicator is local (no NCCL). */
int ials_comm_unique_id(void* id128);
int ials_comm_create(ials_session* s, const void* id128, int32_t rank, int32_t world, ials_comm** out);
/* The same over a communicator the host already has (nccl_comm: its ncclComm_t
 * on this session's device); ials_comm_destroy then leaves it alive. */
int ials_comm_wrap(ials_session* s, void* nccl_comm, int32_t rank, int32_t world, ials_comm** out);
int ials_comm_destroy(ials_comm* c);

/* One rank's share of an iALS++ epoch (ialspp_epoch, solvers.py:340-375),
 * called collectively by all ranks of `comm`.
 *   user_bounds / item_bounds: HOST arrays of world + 1 row offsets (rank r owns
 *     rows [bounds[r], bounds[r+1]); bounds[world] = U / I);
 *   users / items: the LOCAL rows' CSR (ptr rebased to 0, cols = global ids of
 *     the other side, pos = NULL, lam = the local rows' regularisers, n_fixed =
 *     I / U) with their schedules and segment lists;
 *   W (U x d), H (I x d): the replicated tables on this rank's device, updated
 *     in place on every rank;
 *   Cu / Ci: this rank's score caches (its users' entries user-major, its
 *     items' entries item-major), recomputed at the start of the epoch;
 *   rotate: 1 to run the user passes rotated (b = 128 | d, unit weights, no
 *     local heavy user rows on ANY rank -- the flag must be the same on all
 *     ranks: it adds a collective); see ials_rotation_available.
 * Per block: all-reduce of the partial slab (NCCL, d x b floats), the local
 * sweep, the padded all-gather of the updated column block on the
 * communicator's stream beside the other side's partial slab GEMM, and the
 * dual-cache correction from the gathered block's change.  Block widths up to
 * 256.  Workspace: ials_epoch_sharded_bytes (n_slices_max / n_heavy_max: the
 * larger of the two local schedules'). */
size_t ials_epoch_sharded_bytes(const int32_t* user_bounds, const int32_t* item_bounds, int32_t world,
                                int32_t rank, int32_t d, int32_t b, int32_t n_slices_max,
                                int32_t n_heavy_max);
int ials_epoch_sharded(ials_session* s, ials_comm* comm, const ials_side* users, const ials_sched* user_sched,
                       const ials_segs* user_segs, const ials_side* items, const ials_sched* item_sched,
                       const ials_segs* item_segs, const int32_t* user_bounds, const int32_t* item_bounds,
                       float* W, int32_t ldw, float* H, int32_t ldh, int32_t d, int32_t b, float alpha0,
                       int32_t rotate, float* Cu, float* Ci, void* workspace, size_t ws_bytes, void* stream);

/* Workspace bytes for ials_build_csr over n interactions. */
size_t ials_build_csr_workspace_bytes(int64_t n);

/* Device CSR construction, bit-exact with the reference
 * (InteractionDataset.__init__, data.py:98-134; user_view / item_view,
 * data.py:148-162), from COO ids already range-checked by the caller
 * (0 <= users < U, 0 <= items < I):
 *   order[k]     = argsort(users, stable)[k]     (canonical user-major order)
 *   user_ptr     = [0, cumsum(bincount(users, minlength=U))]   (U+1)
 *   user_cols[k] = items[order[k]]
 *   item_pos[k]  = argsort(user_cols, stable)[k] (the item view's cache_pos)
 *   item_ptr     = [0, cumsum(bincount(items, minlength=I))]   (I+1)
 *   item_cols[k] = users[order[item_pos[k]]]
 * Labels / weights follow as gathers by `order` / `item_pos` on the caller's
 * side.  Deterministic (no atomics on the outputs).  n < 2^31. */
int ials_build_csr(ials_session* s, int32_t U, int32_t I, int64_t n, const int32_t* users,
                   const int32_t* items, int32_t* user_ptr, int32_t* user_cols, int32_t* order,
                   int32_t* item_ptr, int32_t* item_cols, int32_t* item_pos, void* workspace,
                   size_t ws_bytes, void* stream);

/* Ranking (top_k_from_scores, metrics.py:31-57) of n_rows score rows
 * scores[r * lds + c], c < n_cols.  If ex_ptr / ex_cols (a CSR over the rows)
 * are given, those entries are first set to -inf IN PLACE.  out (n_rows x k)
 * receives each row's k largest finite scores' column indices, ties by
 * ascending index, padded with -1 when fewer than k finite scores remain;
 * counts[r] = the number returned.  1 <= k <= 1024. */
int ials_topk(ials_session* s, int32_t n_rows, int32_t n_cols, float* scores, int64_t lds,
              const int32_t* ex_ptr, const int32_t* ex_cols, int32_t k, int32_t* out,
              int32_t* counts, void* stream);

/* ials_topk on float64 score rows (top_k_from_scores on the caller's f64
 * scores, metrics.py:31-57): the same order -- score descending, ties by
 * ascending index -- over 64-bit order-preserving keys, so no precision is
 * lost before ranking. */
int ials_topk64(ials_session* s, int32_t n_rows, int32_t n_cols, double* scores, int64_t lds,
                const int32_t* ex_ptr, const int32_t* ex_cols, int32_t k, int32_t* out,
                int32_t* counts, void* stream);

/* out[u][i] = <E[u], H[i]> (n_users x n_items, ld ldo) on the tensor core
 * (3xTF32, FP32-accurate; rank_items / evaluate_holdout / recommend,
 * metrics.py:57-119).  E, H 16-byte aligned with lde, ldh multiples of 4. */
int ials_scores(ials_session* s, const float* E, int32_t lde, int32_t n_users, const float* H,
                int32_t ldh, int32_t n_items, int32_t d, float* out, int32_t ldo, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* IALS_B200_H */
