// ials_shard_epoch.cuh -- the multi-GPU epoch behind the C ABI (included at the
// end of ials_abi.cu: host code over that file's static helpers).
//
// one process per GPU, users and items in contiguous row
// shards, W and H replicated.  ials_epoch_sharded is one rank's share of an
// iALS++ epoch (ialspp_epoch, solvers.py:340-375); every rank calls it
// collectively.  The collectives are NCCL's (ials_comm_*: libnccl.so.2 is
// opened at run time, so a single-GPU host needs no NCCL):
//
//   per epoch   all-reduce of the stacked diagonal Gram blocks (rotated passes)
//   per block   all-reduce of the partial slab (d x b floats), twice
//               all-gather of the updated rows of W[:, pi] / H[:, pi] (padded
//               to the largest shard), on the communicator's own stream beside
//               the other side's partial slab GEMM
//
// Score caches never move (the dual-cache scheme of distributed.py): C_u holds
// this rank's users' entries, C_i its items' entries, each corrected for the
// other side's last half-epoch from the gathered block's change.
//
// The same steps, kernel for kernel, as distributed.ShardedTrainer.epoch with
// GpuOps (the Python orchestration the gloo tests cover); at world size 1 the
// two are bit-identical (tests/test_gpu_parity.py).
#pragma once
#include <dlfcn.h>

struct IalsNcclId { char internal[128]; };   // ncclUniqueId (nccl.h: NCCL_UNIQUE_ID_BYTES 128)

struct NcclApi {
  void* lib = nullptr;
  int (*GetUniqueId)(IalsNcclId*) = nullptr;
  int (*CommInitRank)(void**, int, IalsNcclId, int) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
static constexpr int kNcclFloat = 7, kNcclSum = 0;   // ncclFloat32, ncclSum

static const NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.lib ? &api : nullptr;
  tried = true;
  // the process's own libnccl.so.2 when one is loaded (a PyTorch host), else the system's
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
  auto sym = [&](const char* n) { return dlsym(h, n); };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllReduce || !api.AllGather)
    return nullptr;
  api.lib = h;
  return &api;
}

struct ials_comm {
  void* nccl = nullptr;        // ncclComm_t (null at world size 1 without NCCL)
  bool owned = true;           // created here (ials_comm_create) or the host's own (ials_comm_wrap)
  int rank = 0, world = 1, device = 0;
  cudaStream_t st = nullptr;   // the all-gathers' stream
  cudaEvent_t ev_go = nullptr, ev_done = nullptr;
};

#define NCCL_TRY(s, call)                                                                     \
  do {                                                                                        \
    const int _r = (call);                                                                    \
    if (_r != 0)                                                                              \
      return fail(s, IALS_E_CUDA, "NCCL: %s (%s)",                                            \
                  nccl_api() && nccl_api()->GetErrorString ? nccl_api()->GetErrorString(_r) : "error", #call); \
  } while (0)

int ials_comm_unique_id(void* id128) {
  if (!id128) return IALS_E_INVALID;
  const NcclApi* a = nccl_api();
  if (!a) return fail(nullptr, IALS_E_CUDA, "comm: libnccl.so.2 not found");
  return a->GetUniqueId(static_cast<IalsNcclId*>(id128)) == 0 ? IALS_OK
                                                              : fail(nullptr, IALS_E_CUDA, "comm: ncclGetUniqueId failed");
}

int ials_comm_create(ials_session* s, const void* id128, int32_t rank, int32_t world, ials_comm** out) {
  DevGuard _dg(s);
  if (!s || !out || world < 1 || rank < 0 || rank >= world)
    return fail(s, IALS_E_INVALID, "comm_create: bad arguments (rank %d of %d)", rank, world);
  ials_comm* c = new ials_comm;
  c->rank = rank;
  c->world = world;
  c->device = s->device;
  if (world > 1 || id128) {
    const NcclApi* a = nccl_api();
    if (!a || !id128) {
      delete c;
      return fail(s, IALS_E_CUDA, "comm_create: %s", a ? "NULL unique id" : "libnccl.so.2 not found");
    }
    IalsNcclId id;
    memcpy(&id, id128, sizeof(id));
    const int r = a->CommInitRank(&c->nccl, world, id, rank);
    if (r != 0) {
      delete c;
      return fail(s, IALS_E_CUDA, "comm_create: ncclCommInitRank: %s", a->GetErrorString ? a->GetErrorString(r) : "error");
    }
  }
  cudaError_t e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_go, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    ials_comm_destroy(c);
    return fail(s, IALS_E_CUDA, "comm_create: %s", cudaGetErrorString(e));
  }
  *out = c;
  return IALS_OK;
}

// the host's own ncclComm_t (ials_set_comm): not destroyed with the wrapper
int ials_comm_wrap(ials_session* s, void* nccl_comm, int32_t rank, int32_t world, ials_comm** out) {
  DevGuard _dg(s);
  if (!s || !out || !nccl_comm || world < 1 || rank < 0 || rank >= world)
    return fail(s, IALS_E_INVALID, "comm_wrap: bad arguments (rank %d of %d)", rank, world);
  if (!nccl_api()) return fail(s, IALS_E_CUDA, "comm_wrap: libnccl.so.2 not found");
  ials_comm* c = new ials_comm;
  c->nccl = nccl_comm;
  c->owned = false;
  c->rank = rank;
  c->world = world;
  c->device = s->device;
  cudaError_t e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_go, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    ials_comm_destroy(c);
    return fail(s, IALS_E_CUDA, "comm_wrap: %s", cudaGetErrorString(e));
  }
  *out = c;
  return IALS_OK;
}

int ials_comm_destroy(ials_comm* c) {
  if (!c) return IALS_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  if (c->nccl && c->owned && nccl_api()) nccl_api()->CommDestroy(c->nccl);
  if (c->ev_go) cudaEventDestroy(c->ev_go);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->st) cudaStreamDestroy(c->st);
  if (prev >= 0) cudaSetDevice(prev);
  delete c;
  return IALS_OK;
}

// ---- workspace of one sharded epoch
struct ShardEpochWs {
  float* part;        // gram split partials (SIMT Gramian)
  size_t part_bytes;
  char* pass;         // the side passes' scratch
  size_t pass_bytes;
  void *sw, *sh;      // tensor-core shard workspaces of W_loc / H_loc
  size_t sw_bytes, sh_bytes;
  void* rot;
  size_t rot_bytes;
  float *g_h, *g_w, *gd, *old, *send, *recv, *dW, *dH, *proj;
  int* bounds;        // device: user bounds (world + 1), item bounds (world + 1)
};

static bool shard_tc_width(int d, int b) { return b > 32 && b <= 128 && d % 4 == 0; }

static size_t shard_epoch_carve(char* base, int nu, int ni, int U, int I, int d, int b, int n_slices,
                                int n_heavy, int world, int nmax, ShardEpochWs* w) {
  char* t = base;
  auto take = [&](size_t bytes) {
    char* p = t;
    t += al256(bytes);
    return p;
  };
  const int nloc = std::max(std::max(nu, ni), 1), nall = std::max(std::max(U, I), 1);
  const size_t gb = gram_ws(nloc, d, b);
  const size_t pb = std::max(pass_ws(std::max(nu, 1), std::max(I, 1), b, n_slices, n_heavy),
                             pass_ws(std::max(ni, 1), std::max(U, 1), b, n_slices, n_heavy));
  const size_t swb = shard_tc_width(d, b) ? shard_bytes(nu, d, b) : 0;
  const size_t shb = shard_tc_width(d, b) ? shard_bytes(ni, d, b) : 0;
  const size_t rb = shard_rot_bytes(nu, I, d, b);
  char* p;
  p = take(gb); if (w) { w->part = reinterpret_cast<float*>(p); w->part_bytes = gb; }
  p = take(pb); if (w) { w->pass = p; w->pass_bytes = pb; }
  p = take(swb + 1024); if (w) { w->sw = p; w->sw_bytes = swb; }
  p = take(shb + 1024); if (w) { w->sh = p; w->sh_bytes = shb; }
  p = take(rb + 1024); if (w) { w->rot = p; w->rot_bytes = rb; }
  const size_t slab = size_t(d) * b * 4;
  p = take(slab); if (w) w->g_h = reinterpret_cast<float*>(p);
  p = take(slab); if (w) w->g_w = reinterpret_cast<float*>(p);
  p = take(slab); if (w) w->gd = reinterpret_cast<float*>(p);
  p = take(size_t(nloc) * b * 4); if (w) w->old = reinterpret_cast<float*>(p);
  p = take(size_t(std::max(nmax, 1)) * b * 4); if (w) w->send = reinterpret_cast<float*>(p);
  p = take(size_t(world) * std::max(nmax, 1) * b * 4); if (w) w->recv = reinterpret_cast<float*>(p);
  p = take(size_t(nall) * b * 4); if (w) w->dW = reinterpret_cast<float*>(p);
  p = take(size_t(nall) * b * 4); if (w) w->dH = reinterpret_cast<float*>(p);
  p = take(size_t(nloc) * b * 4); if (w) w->proj = reinterpret_cast<float*>(p);
  p = take(size_t(2) * (world + 1) * 4); if (w) w->bounds = reinterpret_cast<int*>(p);
  return size_t(t - base);
}

static int shard_nmax(const int32_t* ub, const int32_t* ib, int world) {
  int m = 0;
  for (int r = 0; r < world; ++r) m = std::max(m, std::max(ub[r + 1] - ub[r], ib[r + 1] - ib[r]));
  return m;
}

size_t ials_epoch_sharded_bytes(const int32_t* user_bounds, const int32_t* item_bounds, int32_t world,
                                int32_t rank, int32_t d, int32_t b, int32_t n_slices_max,
                                int32_t n_heavy_max) {
  if (!user_bounds || !item_bounds || world < 1 || rank < 0 || rank >= world || d < 1 || b < 1) return 0;
  const int nu = user_bounds[rank + 1] - user_bounds[rank], ni = item_bounds[rank + 1] - item_bounds[rank];
  return shard_epoch_carve(nullptr, nu, ni, user_bounds[world], item_bounds[world], d, b, n_slices_max,
                           n_heavy_max, world, shard_nmax(user_bounds, item_bounds, world), nullptr) + 1024;
}

int ials_epoch_sharded(ials_session* s, ials_comm* comm, const ials_side* users, const ials_sched* user_sched,
                       const ials_segs* user_segs, const ials_side* items, const ials_sched* item_sched,
                       const ials_segs* item_segs, const int32_t* user_bounds, const int32_t* item_bounds,
                       float* W, int32_t ldw, float* H, int32_t ldh, int32_t d, int32_t b, float alpha0,
                       int32_t rotate, float* Cu, float* Ci, void* workspace, size_t ws_bytes, void* stream) {
  DevGuard _dg(s);
  if (!s) return fail(nullptr, IALS_E_INVALID, "session is NULL");
  if (!comm || !users || !items || !user_sched || !item_sched || !user_segs || !item_segs || !user_bounds ||
      !item_bounds || !W || !H || !workspace)
    return fail(s, IALS_E_INVALID, "epoch_sharded: NULL argument");
  if (b < 1 || b > d || b > 256) return fail(s, IALS_E_INVALID, "epoch_sharded: bad block size %d (<= 256)", b);
  const int world = comm->world, rank = comm->rank;
  const int U = user_bounds[world], I = item_bounds[world];
  const int ulo = user_bounds[rank], uhi = user_bounds[rank + 1];
  const int ilo = item_bounds[rank], ihi = item_bounds[rank + 1];
  const int nu = uhi - ulo, ni = ihi - ilo;
  if (users->n_rows != nu || items->n_rows != ni || users->n_fixed != I || items->n_fixed != U)
    return fail(s, IALS_E_INVALID, "epoch_sharded: local sides do not match the bounds");
  if ((nu > 0 && !Cu && users->nnz > 0) || (ni > 0 && !Ci && items->nnz > 0))
    return fail(s, IALS_E_INVALID, "epoch_sharded: NULL cache");
  const int nmax = shard_nmax(user_bounds, item_bounds, world);
  const int nsl = std::max(user_sched->n_slices, item_sched->n_slices);
  const int nhv = std::max(user_sched->n_heavy, item_sched->n_heavy);
  char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 1023) & ~uintptr_t(1023));
  ShardEpochWs w{};
  const size_t need = shard_epoch_carve(base, nu, ni, U, I, d, b, nsl, nhv, world, nmax, &w);
  if (size_t(base - static_cast<char*>(workspace)) + need > ws_bytes)
    return fail(s, IALS_E_NOMEM, "epoch_sharded: workspace %zu < %zu bytes", ws_bytes, need + 1024);
  cudaStream_t st = S(stream);
  const NcclApi* nc = comm->nccl ? nccl_api() : nullptr;
  if (world > 1 && !nc) return fail(s, IALS_E_INVALID, "epoch_sharded: world %d without an NCCL communicator", world);
  float* Wl = W + size_t(ulo) * ldw;
  float* Hl = H + size_t(ilo) * ldh;
  CUDA_TRY(s, cudaMemcpyAsync(w.bounds, user_bounds, size_t(world + 1) * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(s, cudaMemcpyAsync(w.bounds + world + 1, item_bounds, size_t(world + 1) * 4, cudaMemcpyHostToDevice, st));
  const int* ub_dev = w.bounds;
  const int* ib_dev = w.bounds + world + 1;

  // tensor-core GEMMs on the shards (K-major copies), as GpuOps.tc_enable
  const bool tc = shard_tc_width(d, b) && ldw % 4 == 0 && ldh % 4 == 0 &&
                  reinterpret_cast<uintptr_t>(Wl) % 16 == 0 && reinterpret_cast<uintptr_t>(Hl) % 16 == 0 &&
                  get_encode(s) == IALS_OK;
  ShardWs cw{}, ch{};
  int rc = IALS_OK;
  if (tc) {
    rc = shard_carve(s, w.sw, w.sw_bytes + 1024, nu, d, b, &cw);
    if (!rc) rc = shard_carve(s, w.sh, w.sh_bytes + 1024, ni, d, b, &ch);
    if (!rc) rc = sync_copies(s, Wl, ldw, d, 0, d, cw.c, st);
    if (!rc) rc = sync_copies(s, Hl, ldh, d, 0, d, ch.c, st);
    if (rc) return rc;
  }
  auto allreduce = [&](float* buf, size_t count) -> int {
    if (nc) NCCL_TRY(s, nc->AllReduce(buf, buf, count, kNcclFloat, kNcclSum, comm->nccl, st));
    return IALS_OK;
  };
  // partial slab of a shard: F_loc^T F_loc[:, b0:b0+bb]
  auto gram = [&](const float* F, int ldf, int n, const ShardWs& c, int b0, int bb, float* out) -> int {
    if (tc) {
      if (n == 0) {
        CUDA_TRY(s, cudaMemsetAsync(out, 0, size_t(d) * bb * 4, st));
        return IALS_OK;
      }
      return gram_tc(s, c.c, d, b0, bb, c.P, out, c.sth, c.stl, st);
    }
    if (n == 0) {
      CUDA_TRY(s, cudaMemsetAsync(out, 0, size_t(d) * bb * 4, st));
      return IALS_OK;
    }
    return gramian_impl(s, F, n, ldf, d, b0, bb, out, w.part, w.part_bytes, st);
  };
  // rotated user passes: one all-reduce of the stacked diagonal Gram blocks
  const bool rot = rotate && tc && ials_rotation_available(d, b) && U > 0 && I > 0 &&
                   user_sched->n_heavy == 0 && !users->weights && !users->labels;
  if (rotate && !rot)
    return fail(s, IALS_E_INVALID, "epoch_sharded: rotate set but the rotated pass does not apply "
                                   "(b = 128 | d, unit weights, no heavy user rows)");
  // (on the session's high-priority side stream, beside the two prediction
  // passes below; the first user pass waits for it)
  ShardRot sr{};
  if (rot) {
    rc = shard_rot_carve(s, w.rot, w.rot_bytes + 1024, nu, I, d, b, &sr);
    if (!rc) rc = ensure_rot_stream(s);
    if (rc) return rc;
    CUDA_TRY(s, cudaEventRecord(s->ev_rot0, st));   // H_loc's K-major copy is current
    CUDA_TRY(s, cudaStreamWaitEvent(s->rot_st, s->ev_rot0, 0));
    cudaStream_t main_st = st;
    st = s->rot_st;
    if (ni == 0) {
      CUDA_TRY(s, cudaMemsetAsync(w.gd, 0, size_t(d) * b * 4, st));
    } else {
      rc = gemm_attrs(s);
      if (rc) return rc;
      CUtensorMap gm;
      rc = make_map(s, &gm, ch.c.FT, ch.c.n, d, ch.c.ldt, 128);
      if (rc) return rc;
      GemmJob job{d, 0, 0, b, 128, ch.c.n, ch.span, ch.P, b, (long long)d * b, 1.f};
      job.diag = 1;
      k_gemm3_tf32<<<dim3(d / b, ch.S), kGemmThreads, GemmLay::BYTES, st>>>(gm, gm, gm, job);
      LAUNCH_CHECK(s);
      const size_t cnt = size_t(d) * b;
      k_reduce_splits_strided<<<(int)std::min<size_t>((cnt + 255) / 256, 4096), 256, 0, st>>>(
          ch.P, ch.S, (long long)d * b, cnt, w.gd);
      LAUNCH_CHECK(s);
    }
    CUDA_TRY(s, cudaEventRecord(comm->ev_go, st));   // the shard's split-partial scratch is free again
    rc = allreduce(w.gd, size_t(d) * b);
    if (!rc) rc = eig_attrs(s, b);
    if (rc) return rc;
    k_sym_eig<<<d / b, kEigThreads, eig_smem_bytes(b), st>>>(w.gd, b, (long long)b * b, b, sr.QT, sr.lam, sr.rslab,
                                                             sr.Qm, nullptr, 1);
    LAUNCH_CHECK(s);
    CUDA_TRY(s, cudaEventRecord(s->ev_rot1, st));
    st = main_st;
  }
  // both caches from the current factors
  rc = predictions_impl(s, user_segs->n, Items{nullptr, user_segs->row, user_segs->beg, user_segs->end},
                        users->cols, Wl, ldw, H, ldh, d, Cu, stream);
  if (!rc)
    rc = predictions_impl(s, item_segs->n, Items{nullptr, item_segs->row, item_segs->beg, item_segs->end},
                          items->cols, Hl, ldh, W, ldw, d, Ci, stream);
  if (rc) return rc;
  auto correct = [&](const ials_segs* sg, const ials_side* side, const float* A, int lda, int b0, int bb,
                     const float* D, float* out) -> int {
    if (sg->n == 0) return IALS_OK;
    const int blocks = std::min((sg->n + 7) / 8, kNumSMs * 16);
    const bool vec = bb <= 128 && bb % 4 == 0 && b0 % 4 == 0 && lda % 4 == 0 &&
                     reinterpret_cast<uintptr_t>(A) % 16 == 0 && reinterpret_cast<uintptr_t>(D) % 16 == 0;
    if (vec)
      k_cache_correct_v<<<blocks, 256, 0, st>>>(sg->n, Items{nullptr, sg->row, sg->beg, sg->end}, side->cols, A,
                                                lda, b0, D, bb, bb, out);
    else
      k_cache_correct<<<blocks, 256, 0, st>>>(sg->n, Items{nullptr, sg->row, sg->beg, sg->end}, side->cols, A, lda,
                                              b0, D, bb, bb, out);
    LAUNCH_CHECK(s);
    return IALS_OK;
  };
  // one side pass on the local rows (slab: the all-reduced d x bb slab)
  auto sweep = [&](const ials_side* side, const ials_sched* sched, const float* fixed, int ldf, float* own,
                   int ldo, int n, const ShardWs& c, int b0, int bb, float* slab, float* cache, int side_id) -> int {
    if (side_id == 0 && rot && bb == 128) {
      if (n == 0) return IALS_OK;
      const int zb = b0 / b;
      const float* qt = sr.QT + size_t(zb) * b * b;
      float* pj = reinterpret_cast<float*>(w.pass);
      int r = gemm_nt(s, qt, b, b, b, 0, slab, d, bb, bb, 0, b, sr.slabQT, d, 1.f, false, st);
      if (!r) r = proj_tc(s, own, ldo, c.c, d, bb, sr.slabQT, nullptr, alpha0, pj, st);
      if (!r) r = gemm_nt(s, fixed, side->n_fixed, d, ldf, b0, qt, b, b, b, 0, b, sr.Ft, b, 1.f, false, st);
      if (!r) r = gemm_nt(s, own, n, d, ldo, b0, qt, b, b, b, 0, b, sr.WQ, b, 1.f, false, st);
      if (r) return r;
      RotPass rp{sr.Ft, sr.WQ, sr.lam + b0, sr.rslab};
      r = side_pass_impl(s, side, sched, fixed, ldf, own, ldo, d, b0, bb, slab, alpha0, cache, 0, w.pass,
                         w.pass_bytes, st, true, nullptr, nullptr, &rp);
      if (!r)
        r = gemm_nt(s, pass_drow(w.pass, side, sched, bb), n, b, b, 0, sr.Qm + size_t(zb) * b * b, b, b, b, 0, b,
                    own + b0, ldo, -1.f, true, st);
      if (!r) r = sync_copies(s, own, ldo, d, b0, bb, c.c, st);
      return r;
    }
    if (tc && n > 0) {   // projection on the tensor core, then the sweep (ials_shard_projection)
      k_gram_reduce<<<(d * bb + 255) / 256, 256, 0, st>>>(slab, 1, (long long)d * bb, d, bb, slab, c.sth, c.stl);
      LAUNCH_CHECK(s);
      int r = proj_tc(s, own, ldo, c.c, d, bb, c.sth, c.stl, alpha0, w.proj, st);
      if (!r)
        r = side_pass_impl(s, side, sched, fixed, ldf, own, ldo, d, b0, bb, slab, alpha0, cache, side_id, w.pass,
                           w.pass_bytes, st, true, w.proj);
      if (!r) r = sync_copies(s, own, ldo, d, b0, bb, c.c, st);
      return r;
    }
    return side_pass_impl(s, side, sched, fixed, ldf, own, ldo, d, b0, bb, slab, alpha0, cache, side_id, w.pass,
                          w.pass_bytes, st);
  };
  // this rank's rows of X[:, b0:b0+bb] out to every rank (padded all-gather on the
  // communicator's stream); joined by finish(), which also writes the remote rows
  auto start_exchange = [&](const float* Xl, int ldx, int n, int b0, int bb) -> int {
    if (n > 0)
      CUDA_TRY(s, cudaMemcpy2DAsync(w.send, size_t(bb) * 4, Xl + b0, size_t(ldx) * 4, size_t(bb) * 4, n,
                                    cudaMemcpyDeviceToDevice, st));
    if (nc) {
      CUDA_TRY(s, cudaEventRecord(comm->ev_go, st));
      CUDA_TRY(s, cudaStreamWaitEvent(comm->st, comm->ev_go, 0));
      NCCL_TRY(s, nc->AllGather(w.send, w.recv, size_t(nmax) * bb, kNcclFloat, comm->nccl, comm->st));
      CUDA_TRY(s, cudaEventRecord(comm->ev_done, comm->st));
    }
    return IALS_OK;
  };
  auto finish_exchange = [&](float* X, int ldx, int n_all, const int* bdev, int b0, int bb, float* delta) -> int {
    if (nc) CUDA_TRY(s, cudaStreamWaitEvent(st, comm->ev_done, 0));
    if (n_all == 0) return IALS_OK;
    const long long n = (long long)n_all * bb;
    k_apply_block<<<(int)std::min<long long>((n + 255) / 256, 16LL * kNumSMs), 256, 0, st>>>(
        nc ? w.recv : w.send, nmax, bdev, world, rank, w.old, X, ldx, b0, bb, delta, n_all);
    LAUNCH_CHECK(s);
    return IALS_OK;
  };
  auto keep_old = [&](const float* Xl, int ldx, int n, int b0, int bb) -> int {
    if (n > 0)
      CUDA_TRY(s, cudaMemcpy2DAsync(w.old, size_t(bb) * 4, Xl + b0, size_t(ldx) * 4, size_t(bb) * 4, n,
                                    cudaMemcpyDeviceToDevice, st));
    return IALS_OK;
  };

  int prev_b0 = -1, prev_bb = 0;
  if (rot) CUDA_TRY(s, cudaStreamWaitEvent(st, comm->ev_go, 0));   // (the diagonal GEMM used ch.P)
  rc = gram(Hl, ldh, ni, ch, 0, std::min(b, d), w.g_h);
  if (rc) return rc;
  if (rot) CUDA_TRY(s, cudaStreamWaitEvent(st, s->ev_rot1, 0));   // the decompositions
  for (int b0 = 0; b0 < d; b0 += b) {
    const int bb = std::min(b, d - b0);
    // ---- user pass
    if (prev_b0 >= 0) rc = correct(user_segs, users, Wl, ldw, prev_b0, prev_bb, w.dH, Cu);
    if (!rc) rc = allreduce(w.g_h, size_t(d) * bb);
    if (!rc) rc = keep_old(Wl, ldw, nu, b0, bb);
    if (!rc) rc = sweep(users, user_sched, H, ldh, Wl, ldw, nu, cw, b0, bb, w.g_h, Cu, 0);
    if (!rc) rc = start_exchange(Wl, ldw, nu, b0, bb);
    if (!rc) rc = gram(Wl, ldw, nu, cw, b0, bb, w.g_w);   // beside the all-gather
    if (!rc) rc = finish_exchange(W, ldw, U, ub_dev, b0, bb, w.dW);
    // ---- item pass
    if (!rc) rc = correct(item_segs, items, Hl, ldh, b0, bb, w.dW, Ci);
    if (!rc) rc = allreduce(w.g_w, size_t(d) * bb);
    if (!rc) rc = keep_old(Hl, ldh, ni, b0, bb);
    if (!rc) rc = sweep(items, item_sched, W, ldw, Hl, ldh, ni, ch, b0, bb, w.g_w, Ci, 1);
    if (!rc) rc = start_exchange(Hl, ldh, ni, b0, bb);
    if (!rc && b0 + bb < d) rc = gram(Hl, ldh, ni, ch, b0 + bb, std::min(b, d - b0 - bb), w.g_h);
    if (!rc) rc = finish_exchange(H, ldh, I, ib_dev, b0, bb, w.dH);
    if (rc) return rc;
    prev_b0 = b0;
    prev_bb = bb;
  }
  if (prev_b0 >= 0) rc = correct(user_segs, users, Wl, ldw, prev_b0, prev_bb, w.dH, Cu);
  return rc;
}
