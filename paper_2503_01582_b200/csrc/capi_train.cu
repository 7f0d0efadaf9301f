// capi_train.cu -- C ABI: train steps (train_track's loop body), streaming steps, the multi-object
// scheduler and the Reptile exchange.
#include "capi_internal.cuh"

using namespace prenom;
using namespace prenom_capi;

namespace {
constexpr int kGroupJobChunk = 64;  // steps whose job arrays are uploaded at once

// Objects that can share grouped launches: one field architecture and batch /
// sampler shape, tensor-core MLP in the same mode (the grouped kernels are the
// per-object ones with an object table; everything else may differ).
bool same_group(const prenom_object_s* a, const prenom_object_s* b) {
  return uses_tc(a) && uses_tc(b) && tc_split(a) == tc_split(b) &&
         std::memcmp(&a->arch, &b->arch, sizeof(prenom_field_arch)) == 0 &&
         a->cfg.rays_per_iter == b->cfg.rays_per_iter && a->cfg.samples_per_ray == b->cfg.samples_per_ray &&
         a->cfg.prior_sampling == b->cfg.prior_sampling && a->cfg.coarse_samples == b->cfg.coarse_samples;
}

// n_steps train steps of the objects g[0..K) (same_group) through grouped
// launches on `st`: per step k_sample_grp -> k_fwd_wx<GRP> -> k_composite_grp ->
// k_bwd_tc<GRP> + k_mlp_grad_reduce_grp -> k_adam_grp, then each due grid refresh
// (mapper.cpp:182-183, per object). The launches cover every object's
// train_track step exactly as enqueue_step would (same Philox streams, keyframe
// picks, Adam corrections); only the MLP weight-gradient partials are summed in
// a different CTA order. The object table is uploaded once per call, the per-step
// job arrays once per kGroupJobChunk steps.
prenom_status enqueue_group_steps(prenom_ctx_s* c, GroupScratch* gs, const std::vector<prenom_object_s*>& g,
                                  int n_steps, cudaStream_t st) {
  const int K = (int)g.size();
  prenom_object_s* o0 = g[0];
  const int B = o0->cfg.rays_per_iter, S = o0->cfg.samples_per_ray;
  const long long per_obj_tiles = ((long long)B * S + kTile - 1) / kTile;
  std::vector<TcObj> tab(K);
  for (int j = 0; j < K; ++j) {
    prenom_object_s* o = g[j];
    TcObj& t = tab[j];
    t.params = o->params.p;
    t.grad = o->grad.p;
    t.count = o->count.p;
    t.pos = o->pos_depth.p;
    t.feat = o->feat_tc.p;
    t.out = o->out.p;
    t.dout = o->dout.p;
    t.part = o->mlp_part.p;
    t.flag = o->flag.p;
    t.n = (long long)B * S;
    t.tile0 = per_obj_tiles * j;
    if (o->upload_pending) CUDA_TRY(cudaStreamWaitEvent(st, o->ev_upload, 0));
    o->upload_pending = false;
  }
  const long long ntiles = per_obj_tiles * K;
  // [fwd next, fwd done] reset themselves after each forward; zeroed here once per call anyway
  CUDA_TRY(gs->ctr.ensure((size_t)(3 + K)));
  CUDA_TRY(cudaMemsetAsync(gs->ctr.p, 0, sizeof(int) * 2, st));
  CUDA_TRY(gs->objs.ensure((size_t)K));
  CUDA_TRY(cudaMemcpyAsync(gs->objs.p, tab.data(), sizeof(TcObj) * K, cudaMemcpyHostToDevice, st));
  // per-step jobs, [steps][K] SampleJob, CompositeArgs, AdamJob, built and uploaded in
  // chunks of kGroupJobChunk steps (the upload is stream-ordered behind the previous
  // chunk's launches, which read the same buffer)
  const size_t sj = sizeof(SampleJob) * K, cj = sizeof(CompositeArgs) * K, aj = sizeof(AdamJob) * K;
  const size_t per_step = (sj + cj + aj + 15) / 16 * 16;
  const int split = tc_split(o0);
  std::vector<unsigned char> h(per_step * std::min(n_steps, kGroupJobChunk));
  CUDA_TRY(gs->jobs.ensure(h.size()));
  for (int c0 = 0; c0 < n_steps; c0 += kGroupJobChunk) {
    const int nc = std::min(kGroupJobChunk, n_steps - c0);
    std::vector<std::vector<int>> refresh(nc);  // objects whose grid is refreshed after step it
    SamplerCfg cfg0{};
    for (int it = 0; it < nc; ++it) {
      SampleJob* sjob = reinterpret_cast<SampleJob*>(h.data() + per_step * it);
      CompositeArgs* cjob = reinterpret_cast<CompositeArgs*>(h.data() + per_step * it + sj);
      AdamJob* ajob = reinterpret_cast<AdamJob*>(h.data() + per_step * it + sj + cj);
      for (int j = 0; j < K; ++j) {
        prenom_object_s* o = g[j];
        const int64_t step = o->step + it;
        const int fi = frame_of_step(o, step);
        sjob[j].src = frame_source(o, fi);
        if (sjob[j].src.n_obj_px == 0) return fail(PRENOM_DATA, "generate_rays: no object pixels");
        sjob[j].cfg = sampler_cfg(o, B, o->cfg.prior_sampling, PRENOM_TAG_FINE, (uint32_t)step);
        sjob[j].out = bufs(o);
        if (it == 0 && j == 0) cfg0 = sjob[j].cfg;
        cjob[j] = train_composite_args(o, o->stats.p + c0 + it, (uint32_t)step, fi);
        AdamJob& a = ajob[j];
        a.n = o->P;
        a.p = o->params.p;
        a.g = o->grad.p;
        a.m = o->m.p;
        a.v = o->v.p;
        a.lr = o->cfg.eta;
        a.b1 = o->cfg.adam_beta1;
        a.b2 = o->cfg.adam_beta2;
        a.eps = o->cfg.adam_eps;
        adam_corrections(o, step, a.c1, a.c2);
        const int m = o->cfg.grid_refresh_every;
        if (m > 0 && (step + 1) % m == 0) refresh[it].push_back(j);
      }
    }
    CUDA_TRY(cudaMemcpyAsync(gs->jobs.p, h.data(), per_step * nc, cudaMemcpyHostToDevice, st));
    for (int it = 0; it < nc; ++it) {
      const unsigned char* base = gs->jobs.p + per_step * it;
      {
        ProfScope ps(c, PRENOM_K_SAMPLE, st);
        CUDA_TRY(launch_sample_group(reinterpret_cast<const SampleJob*>(base), K, cfg0, st));
      }
      {
        ProfScope ps(c, PRENOM_K_FIELD_FWD, st);
        CUDA_TRY(launch_fwd_tc_group(o0->fd, gs->objs.p, K, ntiles, S, gs->ctr.p, split, st));
      }
      {
        ProfScope ps(c, PRENOM_K_COMPOSITE, st);
        CUDA_TRY(launch_composite_group(reinterpret_cast<const CompositeArgs*>(base + sj), K, B, S, st));
      }
      {
        ProfScope ps(c, PRENOM_K_MLP_BWD, st);
        CUDA_TRY(launch_bwd_tc_group(o0->fd, gs->objs.p, K, ntiles, S, gs->ctr.p + 2, split, st));
      }
      {
        ProfScope ps(c, PRENOM_K_ADAM, st);
        CUDA_TRY(launch_adam_group(reinterpret_cast<const AdamJob*>(base + sj + cj), K, o0->P, st));
      }
      c->launches += 6;  // sample, fwd, composite, bwd, MLP-gradient reduce, Adam
      for (int j : refresh[it]) {
        prenom_object_s* o = g[j];
        ProfScope ps(c, PRENOM_K_REFRESH, st);
        CUDA_TRY(launch_refresh_grid(o->fd, o->params.p, o->R, o->grid.p, o->flag.p, st));
        c->launches += 1;
      }
    }
    for (auto* o : g) o->step += nc;
  }
  return PRENOM_OK;
}
}  // namespace

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
    for (int k = 0; k < i; ++k)
      if (objs[k] == objs[i]) return fail(PRENOM_USAGE, "train_step_many: an object is listed twice");
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
  // mapper.cpp:572-585). Objects of one architecture and batch shape form a
  // group that trains through grouped launches (one launch per stage for all of
  // them, enqueue_group_steps); the groups and the remaining objects go
  // round-robin onto K lane streams, so the kernels of different units overlap
  // (filling each other's ramp and tail waves). The lanes fork from and join
  // back to the context stream, so callers still see one ordered stream.
  // PRENOM_LANES overrides K (1 = serial).
  prenom_ctx_s* c = objs[0]->ctx;
  static const int lanes_env = [] {
    const char* v = getenv("PRENOM_LANES");
    return v ? atoi(v) : kDefaultLanes;
  }();
  static const int group_max = [] {  // objects per grouped unit (PRENOM_GROUP_MAX; 0 = no limit)
    const char* v = getenv("PRENOM_GROUP_MAX");
    return v ? atoi(v) : kGroupMaxDefault;
  }();
  std::vector<std::vector<prenom_object_s*>> units;  // a group (>= 2 objects) or one object
  {
    std::vector<bool> used(n_objs, false);
    for (int i = 0; i < n_objs; ++i) {
      if (used[i]) continue;
      std::vector<prenom_object_s*> u{objs[i]};
      used[i] = true;
      if (c->grouping)
        for (int k = i + 1; k < n_objs; ++k)
          if (!used[k] && (group_max <= 0 || (int)u.size() < group_max) && same_group(objs[i], objs[k])) {
            u.push_back(objs[k]);
            used[k] = true;
          }
      units.push_back(std::move(u));
    }
    for (auto& u : units)
      if (u.size() > 1)
        for (auto* o : u) STATUS_TRY(drop_prefetch(o));  // (a group samples every step itself)
  }
  const int n_units = (int)units.size();
  int n_groups = 0;
  for (auto& u : units) n_groups += u.size() > 1;
  while ((int)c->groups.size() < n_groups) c->groups.push_back(new GroupScratch);
  // per-kernel event timing (prenom_ctx_profile) needs serial kernels: one lane
  const int K = c->prof ? 1 : std::max(1, std::min(n_units, std::min(lanes_env, kMaxLanes)));
  if (K == 1) {
    int gi = 0;
    for (auto& u : units)
      if (u.size() > 1) STATUS_TRY(enqueue_group_steps(c, c->groups[gi++], u, n_steps, c->stream));
    for (int it = 0; it < n_steps; ++it)
      for (auto& u : units)
        if (u.size() == 1) STATUS_TRY(enqueue_step(u[0], u[0]->stats.p + it, it + 1 < n_steps));
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
  prenom_status st = PRENOM_OK;
  struct MinTiles {  // small per-object batches: fewer, fuller persistent CTAs (kernels_tc.cu)
    MinTiles() { tc_set_min_tiles_per_cta(kLaneMinTilesPerCta); }
    ~MinTiles() { tc_set_min_tiles_per_cta(1); }
  } min_tiles_;
  {
    int gi = 0;
    for (int u = 0; u < n_units && st == PRENOM_OK; ++u) {
      if (units[u].size() > 1)
        st = enqueue_group_steps(c, c->groups[gi++], units[u], n_steps, c->lanes[u % K]);
      else
        units[u][0]->lane = c->lanes[u % K];
    }
  }
  for (int it = 0; it < n_steps && st == PRENOM_OK; ++it)
    for (int u = 0; u < n_units && st == PRENOM_OK; ++u)
      if (units[u].size() == 1)
        st = enqueue_step(units[u][0], units[u][0]->stats.p + it, false);  // concurrency replaces the sample-ahead
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
