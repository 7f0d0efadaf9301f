// capi.cu -- C ABI: version, defaults, contexts, objects (create from prior / init), frames, state transfer.
#include "capi_internal.cuh"

using namespace prenom;
using namespace prenom_capi;

extern "C" {
const char* prenom_last_error(void) { return g_err.c_str(); }
int prenom_abi_version(void) { return PRENOM_ABI_VERSION; }

void prenom_default_train_cfg(prenom_train_cfg* c) {
  c->rays_per_iter = 128;
  c->bg_fraction = 0.25f;
  c->samples_per_ray = 24;
  c->lambda_d = 0.1f;
  c->lambda_sigma = 1e-4f;
  c->coarse_samples = 32;
  c->escape_eps = 1e-4f;
  c->grid_refresh_every = 50;
  c->eta = 1e-2f;
  c->prior_sampling = 1;
  c->band_px = 8;
  c->mlp_precision = PRENOM_MLP_FP32;
  c->adam_beta1 = 0.9f;
  c->adam_beta2 = 0.999f;
  c->adam_eps = 1e-8f;
}

prenom_status prenom_param_count(const prenom_field_arch* arch, size_t* total, size_t* hash) {
  STATUS_TRY(validate_arch(arch));
  const FieldDesc d = make_desc(*arch);
  if (total) *total = (size_t)d.hash_params + d.mlp_params;
  if (hash) *hash = (size_t)d.hash_params;
  return PRENOM_OK;
}

prenom_status prenom_level_resolution(const prenom_field_arch* arch, int level, int* res) {
  STATUS_TRY(validate_arch(arch));
  if (level < 0 || level >= arch->hash_levels) return fail(PRENOM_USAGE, "level out of range");
  *res = level_resolution_host(*arch, level);
  return PRENOM_OK;
}

prenom_status prenom_ctx_create(int device, prenom_ctx_t* out) {
  if (!out) return fail(PRENOM_USAGE, "out is NULL");
  int n = 0;
  CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(PRENOM_USAGE, "no such CUDA device");
  CUDA_TRY(cudaSetDevice(device));
  auto* c = new prenom_ctx_s;
  c->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  c->overlap = getenv("PRENOM_NO_OVERLAP") == nullptr;
  if (const char* g = getenv("PRENOM_GROUPED")) c->grouping = atoi(g) != 0;
  if (e != cudaSuccess) {
    delete c;
    return fail(PRENOM_CUDA, cudaGetErrorString(e));
  }
  *out = c;
  return PRENOM_OK;
}

prenom_status prenom_ctx_destroy(prenom_ctx_t ctx) {
  if (!ctx) return PRENOM_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto& u : ctx->ev_used) {
    cudaEventDestroy(u.second.first);
    cudaEventDestroy(u.second.second);
  }
  cudaStreamSynchronize(ctx->side);
  cudaStreamDestroy(ctx->side);
  comm_destroy(ctx);
  for (auto l : ctx->lanes) {
    cudaStreamSynchronize(l);
    cudaStreamDestroy(l);
  }
  for (auto e : ctx->lane_ev) cudaEventDestroy(e);
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PRENOM_OK;
}

prenom_status prenom_ctx_stream(prenom_ctx_t ctx, void** stream) {
  if (!ctx || !stream) return fail(PRENOM_USAGE, "NULL argument");
  *stream = (void*)ctx->stream;
  return PRENOM_OK;
}

prenom_status prenom_ctx_synchronize(prenom_ctx_t ctx) {
  if (!ctx) return fail(PRENOM_USAGE, "NULL ctx");
  CUDA_TRY(cudaSetDevice(ctx->device));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->side));  // a trailing sample-ahead / keyframe upload
  for (auto l : ctx->lanes) CUDA_TRY(cudaStreamSynchronize(l));
  return PRENOM_OK;
}

prenom_status prenom_ctx_launch_count(prenom_ctx_t ctx, int64_t* count) {
  if (!ctx || !count) return fail(PRENOM_USAGE, "NULL argument");
  *count = ctx->launches;
  return PRENOM_OK;
}

prenom_status prenom_ctx_profile(prenom_ctx_t ctx, int enable) {
  if (!ctx) return fail(PRENOM_USAGE, "NULL ctx");
  ctx->prof = enable != 0;
  return PRENOM_OK;
}

prenom_status prenom_ctx_set_grouping(prenom_ctx_t ctx, int enable) {
  if (!ctx) return fail(PRENOM_USAGE, "NULL ctx");
  ctx->grouping = enable != 0;
  return PRENOM_OK;
}

prenom_status prenom_ctx_kernel_times(prenom_ctx_t ctx, double* ms, int64_t* launches) {
  if (!ctx || !ms || !launches) return fail(PRENOM_USAGE, "NULL argument");
  CUDA_TRY(cudaSetDevice(ctx->device));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < PRENOM_K_COUNT; ++k) {
    ms[k] = 0.0;
    launches[k] = 0;
  }
  for (auto& u : ctx->ev_used) {
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, u.second.first, u.second.second));
    ms[u.first] += t;
    launches[u.first] += 1;
    ctx->ev_pool.push_back(u.second.first);
    ctx->ev_pool.push_back(u.second.second);
  }
  ctx->ev_used.clear();
  return PRENOM_OK;
}

prenom_status prenom_object_next_frame(prenom_object_t o, int* frame) {
  if (!o || !frame) return fail(PRENOM_USAGE, "NULL argument");
  if (o->frames.empty()) return fail(PRENOM_DATA, "object has no frames");
  *frame = (int)pdm_pick(philox_first(o->seed, PRENOM_TAG_FRAME, (uint32_t)o->step, 0, 0), (uint32_t)o->frames.size());
  return PRENOM_OK;
}

prenom_status prenom_object_create(prenom_ctx_t ctx, const prenom_field_arch* arch, const float* theta,
                                   const float* grid, int grid_res, uint64_t seed, const prenom_train_cfg* cfg,
                                   const float box_min[3], const float box_max[3], prenom_object_t* out) {
  if (!ctx || !out || !cfg || !box_min || !box_max) return fail(PRENOM_USAGE, "NULL argument");
  STATUS_TRY(validate_arch(arch));
  if (grid_res < 2 || grid_res > 1024) return fail(PRENOM_DATA, "grid resolution out of range");
  if (cfg->rays_per_iter < 1) return fail(PRENOM_USAGE, "generate_rays: n must be >= 1");
  if (cfg->samples_per_ray < 1 || cfg->samples_per_ray > 256) return fail(PRENOM_USAGE, "samples_per_ray must be in [1, 256]");
  if (cfg->prior_sampling && (cfg->coarse_samples < 1 || cfg->coarse_samples > 1024))
    return fail(PRENOM_USAGE, "coarse_samples must be in [1, 1024]");
  for (int a = 0; a < 3; ++a)
    if (!(box_max[a] > box_min[a])) return fail(PRENOM_DATA, "degenerate object box");
  if (cfg->mlp_precision != PRENOM_MLP_FP32 && cfg->mlp_precision != PRENOM_MLP_BF16 &&
      cfg->mlp_precision != PRENOM_MLP_BF16X3)
    return fail(PRENOM_USAGE, "unknown mlp_precision");
  if (cfg->mlp_precision != PRENOM_MLP_FP32 && !tc_supported(make_desc(*arch)))
    return fail(PRENOM_USAGE, "tensor-core MLP needs F=2, L*F<=32, W in {32,64}, H in {1,2}");
  CUDA_TRY(cudaSetDevice(ctx->device));
  auto* o = new prenom_object_s;
  o->ctx = ctx;
  o->arch = *arch;
  o->fd = make_desc(*arch);
  o->cfg = *cfg;
  o->P = param_count_host(*arch);
  o->R = grid_res;
  o->seed = seed;
  std::memcpy(o->bmin, box_min, sizeof o->bmin);
  std::memcpy(o->bmax, box_max, sizeof o->bmax);
  std::memset(&o->pose, 0, sizeof o->pose);
  o->pose.R[0] = o->pose.R[4] = o->pose.R[8] = 1.f;
  std::memcpy(o->Rt, o->pose.R, sizeof o->Rt);
  cudaStream_t st = ctx->stream;
  auto cleanup = [&](prenom_status s) {
    delete o;
    return s;
  };
  const size_t P4 = (o->P + 3) & ~size_t(3);
  if (o->params.ensure(P4) || o->grad.ensure(P4) || o->m.ensure(P4) || o->v.ensure(P4) ||
      o->grid.ensure((size_t)grid_res * grid_res * grid_res) || o->flag.ensure(1) || o->stats.ensure(16))
    return cleanup(fail(PRENOM_CUDA, "out of device memory creating object"));
  cudaMemsetAsync(o->grad.p, 0, P4 * sizeof(float), st);
  cudaMemsetAsync(o->m.p, 0, P4 * sizeof(float), st);
  cudaMemsetAsync(o->v.p, 0, P4 * sizeof(float), st);
  cudaMemsetAsync(o->flag.p, 0, sizeof(int), st);
  if (theta) {
    cudaMemcpyAsync(o->params.p, theta, o->P * sizeof(float), cudaMemcpyHostToDevice, st);
  } else {
    launch_init_params(o->fd, o->params.p, seed, st);
  }
  const size_t gv = (size_t)grid_res * grid_res * grid_res;
  if (grid)
    cudaMemcpyAsync(o->grid.p, grid, gv * sizeof(float), cudaMemcpyHostToDevice, st);
  else
    cudaMemsetAsync(o->grid.p, 0, gv * sizeof(float), st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cleanup(fail(PRENOM_CUDA, cudaGetErrorString(e)));
  *out = o;
  return PRENOM_OK;
}

prenom_status prenom_object_destroy(prenom_object_t obj) {
  if (!obj) return PRENOM_OK;
  cudaSetDevice(obj->ctx->device);
  // its work may sit on the main stream, the sampling stream (sample-ahead,
  // keyframe uploads) or a lane stream
  cudaStreamSynchronize(obj->ctx->stream);
  cudaStreamSynchronize(obj->ctx->side);
  for (auto l : obj->ctx->lanes) cudaStreamSynchronize(l);
  if (obj->ctx->mc_grid_owner == obj) obj->ctx->mc_grid_owner = nullptr;
  delete obj;
  return PRENOM_OK;
}

prenom_status prenom_object_set_frames(prenom_object_t o, int n, const prenom_camera* cams, const float* rgb,
                                       const float* depth, const uint8_t* mask, uint8_t inst,
                                       const prenom_pose* pose) {
  if (!o || !cams || !rgb || !depth || !mask || !pose) return fail(PRENOM_USAGE, "NULL argument");
  if (n < 1) return fail(PRENOM_DATA, "no frames");
  const int W = cams[0].width, H = cams[0].height;
  if (W < 1 || H < 1) return fail(PRENOM_DATA, "bad frame size");
  for (int i = 0; i < n; ++i)
    if (cams[i].width != W || cams[i].height != H)
      return fail(PRENOM_DATA, "generate_rays: mask does not match camera dimensions");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  STATUS_TRY(drop_prefetch(o));
  init_frames(o, n, cams, inst, pose);
  const size_t npx = (size_t)W * H;
  for (int i = 0; i < n; ++i)
    STATUS_TRY(set_frame_pixels(o, o->frames[i], rgb + 3 * npx * i, depth + npx * i, mask + npx * i));
  return PRENOM_OK;
}

prenom_status prenom_object_synth_frames(prenom_object_t o, int n, const prenom_camera* cams, int n_boxes,
                                         const prenom_box* boxes, float depth_noise, float missing_frac,
                                         uint64_t seed, const prenom_pose* pose) {
  if (!o || !cams || !boxes || !pose) return fail(PRENOM_USAGE, "NULL argument");
  if (n < 1) return fail(PRENOM_DATA, "no frames");
  if (n_boxes < 1 || n_boxes > kMaxSynthBoxes) return fail(PRENOM_USAGE, "n_boxes out of range [1, 16]");
  if (depth_noise < 0.f || missing_frac < 0.f || missing_frac > 1.f) return fail(PRENOM_USAGE, "bad noise");
  const int W = cams[0].width, H = cams[0].height;
  if (W < 1 || H < 1) return fail(PRENOM_DATA, "bad frame size");
  for (int i = 0; i < n; ++i)
    if (cams[i].width != W || cams[i].height != H) return fail(PRENOM_DATA, "views differ in size");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  STATUS_TRY(drop_prefetch(o));
  init_frames(o, n, cams, 1, pose);
  cudaStream_t st = o->ctx->stream;
  const size_t npx = (size_t)W * H;
  SynthView v;
  std::memset(&v, 0, sizeof v);
  v.n_boxes = n_boxes;
  for (int b = 0; b < n_boxes; ++b)
    for (int a = 0; a < 3; ++a) {
      v.boxes[b].lo[a] = boxes[b].lo[a];
      v.boxes[b].hi[a] = boxes[b].hi[a];
      v.boxes[b].albedo[a] = boxes[b].albedo[a];
    }
  v.depth_noise = depth_noise;
  v.missing_frac = missing_frac;
  v.seed = seed;
  CUDA_TRY(o->fscratch.mask.ensure(npx));
  for (int i = 0; i < n; ++i) {
    FrameDev* f = o->frames[i];
    CUDA_TRY(f->rgb.ensure(npx * 3));
    CUDA_TRY(f->depth.ensure(npx));
    v.cam = cams[i];
    v.view = i;
    CUDA_TRY(launch_synth_view(v, f->rgb.p, f->depth.p, o->fscratch.mask.p, st));
    CUDA_TRY(build_pixel_lists(o->fscratch.mask.p, W, H, 1, o->cfg.band_px, o->fscratch, f->obj_px, f->bg_px,
                               &f->n_obj_px, &f->n_bg_px, st));
    o->ctx->launches += 10;
  }
  return PRENOM_OK;
}

prenom_status prenom_object_get_frame(prenom_object_t o, int frame, float* rgb, float* depth, int* n_obj_px,
                                      int* n_bg_px, int* obj_px, int* bg_px) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (frame < 0 || frame >= (int)o->frames.size()) return fail(PRENOM_USAGE, "frame index out of range");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  cudaStream_t st = o->ctx->stream;
  const FrameDev* f = o->frames[frame];
  const size_t npx = (size_t)o->W * o->H;
  if (rgb) CUDA_TRY(cudaMemcpyAsync(rgb, f->rgb.p, 3 * sizeof(float) * npx, cudaMemcpyDeviceToHost, st));
  if (depth) CUDA_TRY(cudaMemcpyAsync(depth, f->depth.p, sizeof(float) * npx, cudaMemcpyDeviceToHost, st));
  if (obj_px && f->n_obj_px)
    CUDA_TRY(cudaMemcpyAsync(obj_px, f->obj_px.p, sizeof(int) * f->n_obj_px, cudaMemcpyDeviceToHost, st));
  if (bg_px && f->n_bg_px)
    CUDA_TRY(cudaMemcpyAsync(bg_px, f->bg_px.p, sizeof(int) * f->n_bg_px, cudaMemcpyDeviceToHost, st));
  if (n_obj_px) *n_obj_px = f->n_obj_px;
  if (n_bg_px) *n_bg_px = f->n_bg_px;
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

prenom_status prenom_object_upload_frame(prenom_object_t o, int frame, const float* rgb, const float* depth,
                                         const uint8_t* mask) {
  NvtxRange nvtx_("prenom.upload_frame");
  if (!o || !rgb || !depth) return fail(PRENOM_USAGE, "NULL argument");
  if (frame < 0 || frame >= (int)o->frames.size()) return fail(PRENOM_USAGE, "frame index out of range");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  // On the sampling stream: ordered after any sampling already issued (which
  // may still read this frame) and before the next one; the main stream only
  // waits for it when it samples itself (enqueue_step).
  // It also waits for the work already on the main stream (whose sampling may
  // read the frame), but not for steps enqueued after it.
  cudaStream_t side = o->ctx->overlap ? o->ctx->side : o->ctx->stream;
  // samples already prefetched from this very frame would be stale: re-sample
  if (o->sample_ready && o->prefetch_frame == frame) STATUS_TRY(drop_prefetch(o));
  if (!o->ev_upload) {
    CUDA_TRY(cudaEventCreateWithFlags(&o->ev_upload, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&o->ev_main, cudaEventDisableTiming));
  }
  if (side != o->ctx->stream) {
    CUDA_TRY(cudaEventRecord(o->ev_main, o->ctx->stream));
    CUDA_TRY(cudaStreamWaitEvent(side, o->ev_main, 0));
  }
  STATUS_TRY(set_frame_pixels(o, o->frames[frame], rgb, depth, mask, side));
  CUDA_TRY(cudaEventRecord(o->ev_upload, side));
  o->upload_pending = true;
  return PRENOM_OK;
}


prenom_status prenom_get_params(prenom_object_t o, float* theta) {
  if (!o || !theta) return fail(PRENOM_USAGE, "NULL argument");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  CUDA_TRY(cudaMemcpyAsync(theta, o->params.p, o->P * sizeof(float), cudaMemcpyDeviceToHost, o->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  return PRENOM_OK;
}

prenom_status prenom_set_params(prenom_object_t o, const float* theta) {
  if (!o || !theta) return fail(PRENOM_USAGE, "NULL argument");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  CUDA_TRY(cudaMemcpyAsync(o->params.p, theta, o->P * sizeof(float), cudaMemcpyHostToDevice, o->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  return PRENOM_OK;
}

prenom_status prenom_get_grid(prenom_object_t o, int* res, float* grid) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (res) *res = o->R;
  if (grid) {
    CUDA_TRY(cudaSetDevice(o->ctx->device));
    CUDA_TRY(cudaMemcpyAsync(grid, o->grid.p, sizeof(float) * o->R * o->R * o->R, cudaMemcpyDeviceToHost,
                             o->ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  }
  return PRENOM_OK;
}

prenom_status prenom_set_grid(prenom_object_t o, int R, const float* grid) {
  if (!o || !grid) return fail(PRENOM_USAGE, "NULL argument");
  if (R < 2 || R > 1024) return fail(PRENOM_DATA, "grid resolution out of range");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  const size_t n = (size_t)R * R * R;
  STATUS_TRY(drop_prefetch(o));  // (the prefetched samples read the old grid)
  CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  CUDA_TRY(o->grid.ensure(n));
  o->R = R;
  CUDA_TRY(cudaMemcpyAsync(o->grid.p, grid, n * sizeof(float), cudaMemcpyHostToDevice, o->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  return PRENOM_OK;
}

prenom_status prenom_get_adam(prenom_object_t o, float* m, float* v, int64_t* step) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  if (m) CUDA_TRY(cudaMemcpyAsync(m, o->m.p, o->P * sizeof(float), cudaMemcpyDeviceToHost, o->ctx->stream));
  if (v) CUDA_TRY(cudaMemcpyAsync(v, o->v.p, o->P * sizeof(float), cudaMemcpyDeviceToHost, o->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  if (step) *step = o->step;
  return PRENOM_OK;
}

// Resume: restore a checkpointed Adam state (the reference never saves it,
// SURVEY §5; this makes train_track resumable: the step also keys the
// Philox draws, so a resumed object continues the same sample stream).
prenom_status prenom_set_adam(prenom_object_t o, const float* m, const float* v, int64_t step) {
  if (!o || !m || !v) return fail(PRENOM_USAGE, "NULL argument");
  if (step < 0) return fail(PRENOM_USAGE, "negative step");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  STATUS_TRY(drop_prefetch(o));  // the step keys the draws
  CUDA_TRY(cudaMemcpyAsync(o->m.p, m, o->P * sizeof(float), cudaMemcpyHostToDevice, o->ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(o->v.p, v, o->P * sizeof(float), cudaMemcpyHostToDevice, o->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  o->step = step;
  return PRENOM_OK;
}

prenom_status prenom_reset_adam(prenom_object_t o) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  STATUS_TRY(drop_prefetch(o));  // the step keys the draws
  const size_t P4 = (o->P + 3) & ~size_t(3);
  CUDA_TRY(cudaMemsetAsync(o->m.p, 0, P4 * sizeof(float), o->ctx->stream));
  CUDA_TRY(cudaMemsetAsync(o->v.p, 0, P4 * sizeof(float), o->ctx->stream));
  CUDA_TRY(cudaMemsetAsync(o->grad.p, 0, P4 * sizeof(float), o->ctx->stream));
  o->step = 0;
  return PRENOM_OK;
}

prenom_status prenom_object_set_seed(prenom_object_t o, uint64_t seed) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (o->sample_ready) {
    CUDA_TRY(cudaSetDevice(o->ctx->device));
    STATUS_TRY(drop_prefetch(o));  // the seed keys the draws
  }
  o->seed = seed;
  return PRENOM_OK;
}

prenom_status prenom_object_copy_params(prenom_object_t dst, prenom_object_t src) {
  if (!dst || !src) return fail(PRENOM_USAGE, "NULL argument");
  if (dst->P != src->P) return fail(PRENOM_DATA, "parameter vectors differ in length");
  CUDA_TRY(cudaSetDevice(dst->ctx->device));
  CUDA_TRY(cudaStreamSynchronize(src->ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(dst->params.p, src->params.p, src->P * sizeof(float), cudaMemcpyDeviceToDevice,
                           dst->ctx->stream));
  return prenom_reset_adam(dst);
}
}  // extern "C"
