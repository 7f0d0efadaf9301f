// capi_train.cu -- C ABI: train steps (train_track's loop body), streaming steps, the multi-object
// scheduler and the Reptile exchange.
#include "capi_internal.cuh"

using namespace prenom;
using namespace prenom_capi;

extern "C" {
prenom_status prenom_train_step(prenom_object_t o, int n_steps, prenom_step_stats* stats) {
  NvtxRange nvtx_("prenom.train_step");
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (n_steps < 1) return fail(PRENOM_USAGE, "n_steps must be >= 1");
  if (o->frames.empty()) return fail(PRENOM_DATA, "train_step: object has no frames");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  STATUS_TRY(ensure_scratch(o, o->cfg.rays_per_iter, o->cfg.samples_per_ray));
  CUDA_TRY(o->stats.ensure((size_t)n_steps));
  cudaStream_t st = o->ctx->stream;
  CUDA_TRY(cudaMemsetAsync(o->stats.p, 0, sizeof(StepStatsDev) * n_steps, st));
  for (int it = 0; it < n_steps; ++it) STATUS_TRY(enqueue_step(o, o->stats.p + it, it + 1 < n_steps));
  o->last_n_steps = n_steps;
  if (stats) {
    std::vector<StepStatsDev> h(n_steps);
    CUDA_TRY(cudaMemcpyAsync(h.data(), o->stats.p, sizeof(StepStatsDev) * n_steps, cudaMemcpyDeviceToHost, st));
    STATUS_TRY(check_flag(o));
    for (int i = 0; i < n_steps; ++i) to_host_stats(h[i], &stats[i]);
  }
  return PRENOM_OK;
}

// Streaming variant: nothing on this call synchronizes. The stats of the
// call's steps (and the numeric flag) are copied device->host into a pinned
// slot behind the steps; prenom_wait_stats(ticket) waits for that copy only.
// prefetch_next issues the next step's ray sampling on the side stream right
// after this call's last backward (as consecutive steps of one call do), so a
// caller stepping one call per keyframe keeps the sampling overlapped with Adam.
prenom_status prenom_train_step_async(prenom_object_t o, int n_steps, int prefetch_next, uint64_t* ticket) {
  NvtxRange nvtx_("prenom.train_step_async");
  if (!o || !ticket) return fail(PRENOM_USAGE, "NULL argument");
  if (n_steps < 1) return fail(PRENOM_USAGE, "n_steps must be >= 1");
  if (o->frames.empty()) return fail(PRENOM_DATA, "train_step: object has no frames");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  STATUS_TRY(ensure_scratch(o, o->cfg.rays_per_iter, o->cfg.samples_per_ray));
  CUDA_TRY(o->stats.ensure((size_t)n_steps));
  cudaStream_t st = o->ctx->stream;
  auto& sl = o->slots[o->next_ticket % 4];
  if (sl.ev) CUDA_TRY(cudaEventSynchronize(sl.ev));  // the slot's previous copy (4 calls ago) has landed
  if (sl.cap < n_steps) {
    if (sl.host) CUDA_TRY(cudaFreeHost(sl.host));
    CUDA_TRY(cudaMallocHost(&sl.host, sizeof(StepStatsDev) * n_steps));
    sl.cap = n_steps;
  }
  if (!sl.flag) CUDA_TRY(cudaMallocHost(&sl.flag, sizeof(int)));
  if (!sl.ev) CUDA_TRY(cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming));
  CUDA_TRY(cudaMemsetAsync(o->stats.p, 0, sizeof(StepStatsDev) * n_steps, st));
  for (int it = 0; it < n_steps; ++it)
    STATUS_TRY(enqueue_step(o, o->stats.p + it, it + 1 < n_steps || prefetch_next != 0));
  o->last_n_steps = n_steps;
  CUDA_TRY(cudaMemcpyAsync(sl.host, o->stats.p, sizeof(StepStatsDev) * n_steps, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(sl.flag, o->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaEventRecord(sl.ev, st));
  sl.n = n_steps;
  sl.ticket = o->next_ticket++;
  *ticket = sl.ticket;
  return PRENOM_OK;
}

prenom_status prenom_wait_stats(prenom_object_t o, uint64_t ticket, prenom_step_stats* stats) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  for (auto& sl : o->slots) {
    if (sl.ticket != ticket || ticket == 0) continue;
    CUDA_TRY(cudaEventSynchronize(sl.ev));
    if (*sl.flag & 1) return fail(PRENOM_NUMERIC, "field_eval produced a non-finite output");
    if (*sl.flag & 2) return fail(PRENOM_NUMERIC, "batch_loss: non-finite loss");
    if (stats)
      for (int i = 0; i < sl.n; ++i) to_host_stats(sl.host[i], &stats[i]);
    return PRENOM_OK;
  }
  return fail(PRENOM_USAGE, "prenom_wait_stats: unknown or expired ticket (4 calls are kept)");
}

prenom_status prenom_object_frame_at(prenom_object_t o, int64_t step, int* frame) {
  if (!o || !frame) return fail(PRENOM_USAGE, "NULL argument");
  if (o->frames.empty()) return fail(PRENOM_DATA, "object has no frames");
  if (step < 0) return fail(PRENOM_USAGE, "negative step");
  *frame = frame_of_step(o, step);
  return PRENOM_OK;
}

prenom_status prenom_object_last_stats(prenom_object_t o, int n, prenom_step_stats* stats) {
  if (!o || !stats) return fail(PRENOM_USAGE, "NULL argument");
  n = std::min(n, o->last_n_steps);
  if (n <= 0) return PRENOM_OK;
  std::vector<StepStatsDev> h(n);
  CUDA_TRY(cudaMemcpyAsync(h.data(), o->stats.p + (o->last_n_steps - n), sizeof(StepStatsDev) * n,
                           cudaMemcpyDeviceToHost, o->ctx->stream));
  STATUS_TRY(check_flag(o));
  for (int i = 0; i < n; ++i) to_host_stats(h[i], &stats[i]);
  return PRENOM_OK;
}

prenom_status prenom_object_step(prenom_object_t o, int64_t* step) {
  if (!o || !step) return fail(PRENOM_USAGE, "NULL argument");
  *step = o->step;
  return PRENOM_OK;
}

prenom_status prenom_object_check(prenom_object_t o) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  return check_flag(o);
}

prenom_status prenom_train_step_many(prenom_object_t* objs, int n_objs, int n_steps) {
  NvtxRange nvtx_("prenom.train_step_many");
  if (!objs || n_objs < 1 || n_steps < 1) return fail(PRENOM_USAGE, "bad arguments");
  for (int i = 0; i < n_objs; ++i) {
    if (!objs[i]) return fail(PRENOM_USAGE, "NULL object");
    if (objs[i]->ctx != objs[0]->ctx) return fail(PRENOM_USAGE, "objects must share one context");
    if (objs[i]->frames.empty()) return fail(PRENOM_DATA, "train_step: object has no frames");
  }
  CUDA_TRY(cudaSetDevice(objs[0]->ctx->device));
  for (int i = 0; i < n_objs; ++i) {
    prenom_object_s* o = objs[i];
    STATUS_TRY(ensure_scratch(o, o->cfg.rays_per_iter, o->cfg.samples_per_ray));
    CUDA_TRY(o->stats.ensure((size_t)n_steps));
    CUDA_TRY(cudaMemsetAsync(o->stats.p, 0, sizeof(StepStatsDev) * n_steps, o->ctx->stream));
    o->last_n_steps = n_steps;
  }
  // Multi-object scheduler: objects are independent (own θ, Adam, grid, rng;
  // mapper.cpp:572-585), so their steps go round-robin onto K lane streams and
  // the kernels of different objects overlap (filling each other's ramp and
  // tail waves). The lanes fork from and join back to the context stream, so
  // callers still see one ordered stream. PRENOM_LANES overrides K (1 = serial).
  prenom_ctx_s* c = objs[0]->ctx;
  static const int lanes_env = [] {
    const char* v = getenv("PRENOM_LANES");
    return v ? atoi(v) : kDefaultLanes;
  }();
  // per-kernel event timing (prenom_ctx_profile) needs serial kernels: one lane
  const int K = c->prof ? 1 : std::max(1, std::min(n_objs, std::min(lanes_env, kMaxLanes)));
  if (K == 1) {
    for (int it = 0; it < n_steps; ++it)
      for (int i = 0; i < n_objs; ++i) STATUS_TRY(enqueue_step(objs[i], objs[i]->stats.p + it, it + 1 < n_steps));
    return PRENOM_OK;
  }
  while ((int)c->lanes.size() < K) {
    cudaStream_t l;
    cudaEvent_t e;
    CUDA_TRY(cudaStreamCreateWithFlags(&l, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->lanes.push_back(l);
    c->lane_ev.push_back(e);
  }
  if (!c->fork_ev) CUDA_TRY(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(c->fork_ev, c->stream));
  for (int k = 0; k < K; ++k) CUDA_TRY(cudaStreamWaitEvent(c->lanes[k], c->fork_ev, 0));
  for (int i = 0; i < n_objs; ++i) objs[i]->lane = c->lanes[i % K];
  prenom_status st = PRENOM_OK;
  struct MinTiles {  // small per-object batches: fewer, fuller persistent CTAs (kernels_tc.cu)
    MinTiles() { tc_set_min_tiles_per_cta(kLaneMinTilesPerCta); }
    ~MinTiles() { tc_set_min_tiles_per_cta(1); }
  } min_tiles_;
  for (int it = 0; it < n_steps && st == PRENOM_OK; ++it)
    for (int i = 0; i < n_objs && st == PRENOM_OK; ++i)
      st = enqueue_step(objs[i], objs[i]->stats.p + it, false);  // concurrency replaces the sample-ahead
  for (int i = 0; i < n_objs; ++i) objs[i]->lane = nullptr;
  for (int k = 0; k < K; ++k) {
    CUDA_TRY(cudaEventRecord(c->lane_ev[k], c->lanes[k]));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->lane_ev[k], 0));
  }
  return st;
}

prenom_status prenom_reptile_delta(prenom_object_t meta, prenom_object_t adapted, float* delta_dev) {
  if (!meta || !adapted || !delta_dev) return fail(PRENOM_USAGE, "NULL argument");
  if (meta->P != adapted->P) return fail(PRENOM_DATA, "reptile_update: parameter vectors differ in length");
  CUDA_TRY(cudaSetDevice(meta->ctx->device));
  if (adapted->ctx != meta->ctx) CUDA_TRY(cudaStreamSynchronize(adapted->ctx->stream));
  CUDA_TRY(launch_reptile_delta(meta->P, meta->params.p, adapted->params.p, delta_dev, meta->ctx->stream));
  meta->ctx->launches += 1;
  return PRENOM_OK;  // stream-ordered on the meta context's stream
}

prenom_status prenom_reptile_apply(prenom_object_t meta, const float* delta_dev, int n_tasks, float beta) {
  if (!meta || !delta_dev) return fail(PRENOM_USAGE, "NULL argument");
  if (n_tasks < 1) return fail(PRENOM_USAGE, "n_tasks must be >= 1");
  CUDA_TRY(cudaSetDevice(meta->ctx->device));
  CUDA_TRY(launch_reptile_apply(meta->P, meta->params.p, delta_dev, 1.f / (float)n_tasks, beta, meta->ctx->stream));
  meta->ctx->launches += 1;
  return PRENOM_OK;  // stream-ordered on the meta context's stream
}

prenom_status prenom_reptile_update(prenom_object_t meta, prenom_object_t adapted, float beta) {
  if (!meta || !adapted) return fail(PRENOM_USAGE, "NULL argument");
  if (meta->P != adapted->P) return fail(PRENOM_DATA, "reptile_update: parameter vectors differ in length");
  CUDA_TRY(cudaSetDevice(meta->ctx->device));
  CUDA_TRY(cudaStreamSynchronize(adapted->ctx->stream));
  CUDA_TRY(launch_reptile_update(meta->P, meta->params.p, adapted->params.p, beta, meta->ctx->stream));
  meta->ctx->launches += 1;
  return PRENOM_OK;
}
}  // extern "C"
