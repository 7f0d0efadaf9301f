// capi.cu -- host side of the C ABI in include/prenom/prenom_gpu.h.
//
// Owns per-GPU contexts and per-object device state, and orchestrates the
// train step (train_track's loop body, mapper.cpp:150-184) as a sequence of
// kernel launches on the context stream:
//   k_sample -> k_fwd_tile -> k_composite (+stats) -> k_bwd_tile ->
//   k_encode_bwd -> k_adam [-> k_field_points (grid refresh every m steps)]
// The host never touches sample data: per step it only draws the keyframe
// index (one Philox call, TAG_FRAME) and computes the Adam bias corrections
// with glibc powf (field.cpp:300-301), like the reference.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include "prenom_device.cuh"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: host ranges for nsys/ncu timelines

using namespace prenom;

namespace {

thread_local std::string g_err;

prenom_status fail(prenom_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return fail(PRENOM_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));          \
  } while (0)

#define STATUS_TRY(expr)                 \
  do {                                   \
    prenom_status _s = (expr);           \
    if (_s != PRENOM_OK) return _s;      \
  } while (0)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t ensure(size_t count) {
    if (count <= n && p) return cudaSuccess;
    release();
    n = std::max<size_t>(count, 1);
    return cudaMalloc(&p, n * sizeof(T));
  }
};

int level_resolution_host(const prenom_field_arch& a, int level) {
  const double r = a.base_resolution * std::pow((double)a.per_level_scale, level);  // field.cpp:113-116
  return std::max(1, (int)r);
}

prenom_status validate_arch(const prenom_field_arch* a) {
  if (!a) return fail(PRENOM_USAGE, "arch is NULL");
  if (a->hash_levels < 1 || a->features_per_level < 1 || a->log2_table_size < 0 || a->base_resolution < 1 ||
      a->per_level_scale < 1.f || a->hidden_width < 1 || a->hidden_layers < 1)
    return fail(PRENOM_DATA, "invalid architecture description");  // field.cpp arch_from_text
  if (a->hash_levels > kMaxLevels) return fail(PRENOM_USAGE, "hash_levels exceeds 24");
  if (a->features_per_level > 4) return fail(PRENOM_USAGE, "features_per_level exceeds 4");
  if (a->hash_levels * a->features_per_level > kMaxIn) return fail(PRENOM_USAGE, "L*F exceeds 64");
  if (a->hidden_width > kMaxWidth) return fail(PRENOM_USAGE, "hidden_width exceeds 64");
  if (a->hidden_layers > kMaxHidden) return fail(PRENOM_USAGE, "hidden_layers exceeds 3");
  if (a->log2_table_size > 26) return fail(PRENOM_USAGE, "log2_table_size exceeds 26");
  if (a->density_activation != PRENOM_ACT_EXP_CLAMPED && a->density_activation != PRENOM_ACT_SOFTPLUS)
    return fail(PRENOM_DATA, "unknown density activation");
  return PRENOM_OK;
}

FieldDesc make_desc(const prenom_field_arch& a) {
  FieldDesc d;
  std::memset(&d, 0, sizeof d);
  d.L = a.hash_levels;
  d.F = a.features_per_level;
  d.T = a.log2_table_size;
  d.W = a.hidden_width;
  d.H = a.hidden_layers;
  d.act = a.density_activation;
  d.in_dim = d.L * d.F;
  d.rows = 1ll << d.T;
  d.row_mask = (uint32_t)(d.rows - 1);
  d.hash_params = (long long)d.L * d.F * d.rows;
  for (int l = 0; l < d.L; ++l) {
    d.res[l] = level_resolution_host(a, l);
    const uint64_t v = (uint64_t)d.res[l] + 1;
    d.dense_verts[l] = (v * v * v <= (uint64_t)d.rows) ? (uint32_t)v : 0u;  // field.cpp:143-146
  }
  int off = 0, in = d.in_dim;
  for (int l = 0; l <= d.H; ++l) {
    const int out = l < d.H ? d.W : 4;
    d.w_off[l] = off;
    d.b_off[l] = off + out * in;
    off += out * in + out;
    in = out;
  }
  d.mlp_params = off;
  return d;
}

size_t param_count_host(const prenom_field_arch& a) {
  const FieldDesc d = make_desc(a);
  return (size_t)d.hash_params + (size_t)d.mlp_params;
}

void mat_vec(const float* M, const float* v, float* out) {
  out[0] = M[0] * v[0] + M[1] * v[1] + M[2] * v[2];
  out[1] = M[3] * v[0] + M[4] * v[1] + M[5] * v[2];
  out[2] = M[6] * v[0] + M[7] * v[1] + M[8] * v[2];
}

uint32_t philox_first(uint64_t seed, uint32_t tag, uint32_t step, uint32_t ray, uint32_t idx) {
  const uint32_t ctr[4] = {idx, ray, step, tag};
  uint32_t out[4];
  pdm_philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32), out);
  return out[0];
}

}  // namespace

constexpr int kDefaultLanes = 8;  // B200, with >= 8 tiles per persistent CTA: cfg3 4 lanes 1.35e9, 8 lanes 1.41e9;
                                  // cfg5 4: 1.10e9, 8: 1.12e9 (1 lane: cfg3 1.00e9)
constexpr int kMaxLanes = 16;
constexpr int kLaneMinTilesPerCta = 8;

struct prenom_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // ray sampling of step t+1 overlaps Adam of step t
  bool overlap = true;          // PRENOM_NO_OVERLAP=1 disables (A/B measurement)
  // multi-object scheduler: independent objects' steps run on these streams
  // concurrently (prenom_train_step_many), forked from and joined back to `stream`
  std::vector<cudaStream_t> lanes;
  std::vector<cudaEvent_t> lane_ev;
  cudaEvent_t fork_ev = nullptr;
  int64_t launches = 0;
  McMesh mc_dbg;  // prenom_debug_marching_cubes result
  McScratch mc;   // extraction scratch shared by the context's objects
  const void* mc_grid_owner = nullptr;  // object whose lattice mc.grid holds
  // optional per-kernel event timing
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used;
  cudaEvent_t get_event() {
    if (ev_pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
};

namespace {
// NVTX range over a host API call; free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct ProfScope {
  prenom_ctx_s* c;
  int k;
  cudaStream_t s;
  cudaEvent_t b = nullptr, e = nullptr;
  ProfScope(prenom_ctx_s* ctx, int kind, cudaStream_t st = nullptr) : c(ctx), k(kind), s(st ? st : ctx->stream) {
    if (c->prof) {
      b = c->get_event();
      e = c->get_event();
      cudaEventRecord(b, s);
    }
  }
  ~ProfScope() {
    if (c->prof) {
      cudaEventRecord(e, s);
      c->ev_used.push_back({k, {b, e}});
    }
  }
};
}  // namespace

struct FrameDev {
  DevBuf<float> rgb, depth;
  MeshBuf<int> obj_px, bg_px;  // dilation_band / pixel lists, built on the device (kernels_data.cu)
  int n_obj_px = 0, n_bg_px = 0;
  prenom_camera cam;
  float origin[3];  // world_to_obj.apply(camera.t)
};

struct prenom_object_s {
  prenom_ctx_s* ctx = nullptr;
  prenom_field_arch arch;
  FieldDesc fd;
  prenom_train_cfg cfg;
  size_t P = 0;
  DevBuf<float> params, grad, m, v;
  int R = 0;
  DevBuf<float> grid;
  DevBuf<float> query;  // prenom_density_query output (swapped with grid on update)
  uint64_t seed = 0;
  float bmin[3], bmax[3];
  int64_t step = 0;
  int64_t render_calls = 0;
  // frames
  std::vector<FrameDev*> frames;
  int W = 0, H = 0;
  uint8_t inst = 1;
  prenom_pose pose;
  float Rt[9];
  // scratch
  DevBuf<float4> pos_depth, target, out, dout;
  DevBuf<float> delta, feat_t, dfeat_t, t_entry, t_exit;
  DevBuf<unsigned char> feat_tc;  // bf16 feature tiles (tensor-core path)
  DevBuf<int> tile_ctr;           // dynamic tile-scheduler counters (fwd, bwd)
  DevBuf<int> kind, count;
  DevBuf<StepStatsDev> stats;
  int last_n_steps = 0;
  // sample-ahead pipelining (k_sample(t+1) on ctx->side while k_adam(t) runs)
  cudaEvent_t ev_bwd = nullptr, ev_sample = nullptr;
  bool sample_ready = false;
  cudaStream_t lane = nullptr;  // set while prenom_train_step_many runs this object on a lane stream
  // streaming: frame uploads go on ctx->side (the sampling stream); a step
  // whose sampling runs on the main stream waits for ev_upload first
  cudaEvent_t ev_upload = nullptr, ev_main = nullptr;
  bool upload_pending = false;
  // prenom_train_step_async: ring of pinned host stat slots
  struct AsyncSlot {
    uint64_t ticket = 0;
    int n = 0;
    StepStatsDev* host = nullptr;  // pinned
    int* flag = nullptr;           // pinned
    int cap = 0;
    cudaEvent_t ev = nullptr;
  };
  AsyncSlot slots[4];
  uint64_t next_ticket = 1;
  DevBuf<int> flag;
  McMesh mesh;  // prenom_extract_mesh result (device)
  FrameScratch fscratch;  // band / pixel-list construction
  ~prenom_object_s() {
    for (auto* f : frames) delete f;
    if (ev_bwd) cudaEventDestroy(ev_bwd);
    if (ev_sample) cudaEventDestroy(ev_sample);
    if (ev_upload) cudaEventDestroy(ev_upload);
    if (ev_main) cudaEventDestroy(ev_main);
    for (auto& sl : slots) {
      if (sl.ev) cudaEventDestroy(sl.ev);
      if (sl.host) cudaFreeHost(sl.host);
      if (sl.flag) cudaFreeHost(sl.flag);
    }
  }
};

namespace {

prenom_status ensure_scratch(prenom_object_s* o, int B, int S) {
  const size_t N = (size_t)B * S;
  const size_t Npad = ((N + kTile - 1) / kTile) * kTile;
  CUDA_TRY(o->pos_depth.ensure(Npad));
  CUDA_TRY(o->delta.ensure(Npad));
  CUDA_TRY(o->out.ensure(Npad));
  CUDA_TRY(o->dout.ensure(Npad));
  if (o->cfg.mlp_precision == PRENOM_MLP_BF16) {
    CUDA_TRY(o->feat_tc.ensure(tc_feature_bytes(o->fd, (long long)N)));
    if (!o->tile_ctr.p) {  // [fwd next, fwd done (self-resetting), bwd next (memset per launch), -]
      CUDA_TRY(o->tile_ctr.ensure(4));
      CUDA_TRY(cudaMemset(o->tile_ctr.p, 0, 4 * sizeof(int)));
    }
  } else {
    CUDA_TRY(o->feat_t.ensure(Npad * o->fd.in_dim));
    CUDA_TRY(o->dfeat_t.ensure(Npad * o->fd.in_dim));
  }
  CUDA_TRY(o->target.ensure(B));
  CUDA_TRY(o->kind.ensure(B));
  CUDA_TRY(o->count.ensure(B));
  CUDA_TRY(o->t_entry.ensure(B));
  CUDA_TRY(o->t_exit.ensure(B));
  return PRENOM_OK;
}

SampleBufs bufs(prenom_object_s* o) {
  SampleBufs sb;
  std::memset(&sb, 0, sizeof sb);
  sb.pos_depth = o->pos_depth.p;
  sb.delta = o->delta.p;
  sb.target = o->target.p;
  sb.kind = o->kind.p;
  sb.count = o->count.p;
  sb.t_entry = o->t_entry.p;
  sb.t_exit = o->t_exit.p;
  return sb;
}

prenom_status check_flag(prenom_object_s* o) {
  int f = 0;
  CUDA_TRY(cudaMemcpyAsync(&f, o->flag.p, sizeof(int), cudaMemcpyDeviceToHost, o->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  if (f & 1) return fail(PRENOM_NUMERIC, "field_eval produced a non-finite output");
  if (f & 2) return fail(PRENOM_NUMERIC, "batch_loss: non-finite loss");
  return PRENOM_OK;
}

RaySource frame_source(prenom_object_s* o, int fi) {
  const FrameDev* f = o->frames[fi];
  RaySource src;
  std::memset(&src, 0, sizeof src);
  src.mode = 0;
  src.rgb = f->rgb.p;
  src.depth = f->depth.p;
  src.obj_px = f->obj_px.p;
  src.bg_px = f->bg_px.p;
  src.n_obj_px = f->n_obj_px;
  src.n_bg_px = f->n_bg_px;
  const int B = o->cfg.rays_per_iter;
  // render.cpp:66-68
  int n_bg = f->n_bg_px == 0 ? 0 : (int)std::lround((float)B * o->cfg.bg_fraction);
  n_bg = std::min(n_bg, B);
  src.n_obj = B - n_bg;
  src.width = f->cam.width;
  src.fx = f->cam.fx;
  src.fy = f->cam.fy;
  src.cx = f->cam.cx;
  src.cy = f->cam.cy;
  std::memcpy(src.Rc, f->cam.R, sizeof src.Rc);
  std::memcpy(src.Rt, o->Rt, sizeof src.Rt);
  std::memcpy(src.origin, f->origin, sizeof src.origin);
  return src;
}

SamplerCfg sampler_cfg(prenom_object_s* o, int B, int prior, uint32_t tag, uint32_t step) {
  SamplerCfg c;
  std::memset(&c, 0, sizeof c);
  c.B = B;
  c.S = o->cfg.samples_per_ray;
  c.prior = prior;
  c.n_coarse = o->cfg.coarse_samples;
  c.eps = o->cfg.escape_eps;
  c.grid_res = o->R;
  c.grid = o->grid.p;
  std::memcpy(c.bmin, o->bmin, sizeof c.bmin);
  std::memcpy(c.bmax, o->bmax, sizeof c.bmax);
  c.seed = o->seed;
  c.tag = tag;
  c.step = step;
  return c;
}

int frame_of_step(const prenom_object_s* o, int64_t step) {  // keyframe pick (mapper.cpp:151)
  return (int)pdm_pick(philox_first(o->seed, PRENOM_TAG_FRAME, (uint32_t)step, 0, 0), (uint32_t)o->frames.size());
}

// generate_rays + sample_ray for `step` (render.cpp:47-102, density_grid.cpp:110-117)
prenom_status enqueue_sample(prenom_object_s* o, int64_t step, cudaStream_t st) {
  const RaySource src = frame_source(o, frame_of_step(o, step));
  if (src.n_obj_px == 0) return fail(PRENOM_DATA, "generate_rays: no object pixels");
  ProfScope ps(o->ctx, PRENOM_K_SAMPLE, st);
  CUDA_TRY(launch_sample(src, sampler_cfg(o, o->cfg.rays_per_iter, o->cfg.prior_sampling, PRENOM_TAG_FINE,
                                          (uint32_t)step), bufs(o), nullptr, st));
  return PRENOM_OK;
}

// One iteration of train_track's loop body (mapper.cpp:150-184). With
// has_next, the next step's ray sampling is issued on the side stream as
// soon as this step's backward has consumed the sample buffers, so it runs
// concurrently with this step's Adam (it only reads frames and the grid;
// steps that refresh the grid keep the serial order).
prenom_status enqueue_step(prenom_object_s* o, StepStatsDev* stats, bool has_next = false) {
  NvtxRange nvtx_("prenom.step");
  cudaStream_t st = o->lane ? o->lane : o->ctx->stream;
  const prenom_train_cfg& c = o->cfg;
  const int B = c.rays_per_iter, S = c.samples_per_ray;
  const uint32_t step = (uint32_t)o->step;
  const int fi = frame_of_step(o, o->step);
  const SampleBufs sb = bufs(o);
  if (o->sample_ready) {
    CUDA_TRY(cudaStreamWaitEvent(st, o->ev_sample, 0));
    o->sample_ready = false;
  } else {
    if (o->upload_pending) CUDA_TRY(cudaStreamWaitEvent(st, o->ev_upload, 0));
    STATUS_TRY(enqueue_sample(o, o->step, st));
  }
  o->upload_pending = false;  // any later sampling is ordered after this step's
  const bool tc = c.mlp_precision == PRENOM_MLP_BF16;
  {
    ProfScope ps(o->ctx, PRENOM_K_FIELD_FWD, st);
    if (tc)
      CUDA_TRY(launch_fwd_tc(o->fd, o->params.p, (long long)B * S, S, sb.count, sb.pos_depth, o->feat_tc.p, o->out.p,
                             o->flag.p, o->tile_ctr.p, st));
    else
      CUDA_TRY(launch_field_fwd_train(o->fd, o->params.p, B, S, sb, o->feat_t.p, o->out.p, o->flag.p, st));
  }
  CompositeArgs ca;
  std::memset(&ca, 0, sizeof ca);
  ca.B = B;
  ca.S = S;
  ca.pos_depth = sb.pos_depth;
  ca.delta = sb.delta;
  ca.target = sb.target;
  ca.kind = sb.kind;
  ca.count = sb.count;
  ca.out = o->out.p;
  ca.bg_colors = nullptr;
  ca.seed = o->seed;
  ca.step = step;
  ca.lambda_d = c.lambda_d;
  ca.lambda_sigma = c.lambda_sigma;
  ca.dout = o->dout.p;
  ca.stats = stats;
  ca.flag = o->flag.p;
  ca.frame = fi;
  {
    ProfScope ps(o->ctx, PRENOM_K_COMPOSITE, st);
    CUDA_TRY(launch_composite(ca, st));
  }
  if (tc) {
    ProfScope ps(o->ctx, PRENOM_K_MLP_BWD, st);  // MLP backward + fused table-gradient scatter
    CUDA_TRY(launch_bwd_tc(o->fd, o->params.p, o->grad.p, (long long)B * S, S, sb.count, sb.pos_depth,
                           o->feat_tc.p, o->dout.p, o->tile_ctr.p + 2, st));
  } else {
    {
      ProfScope ps(o->ctx, PRENOM_K_MLP_BWD, st);
      CUDA_TRY(launch_mlp_bwd_train(o->fd, o->params.p, o->grad.p, B, S, sb.count, o->feat_t.p, o->dout.p,
                                    o->dfeat_t.p, st));
    }
    {
      ProfScope ps(o->ctx, PRENOM_K_ENCODE_BWD, st);
      CUDA_TRY(launch_encode_bwd(o->fd, o->params.p, o->grad.p, B, S, sb.count, sb.pos_depth, o->dfeat_t.p, st));
    }
  }
  const bool refresh_now = c.grid_refresh_every > 0 && (o->step + 1) % c.grid_refresh_every == 0;
  if (has_next && !refresh_now && o->ctx->overlap) {
    if (!o->ev_bwd) {
      CUDA_TRY(cudaEventCreateWithFlags(&o->ev_bwd, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&o->ev_sample, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventRecord(o->ev_bwd, st));
    CUDA_TRY(cudaStreamWaitEvent(o->ctx->side, o->ev_bwd, 0));
    STATUS_TRY(enqueue_sample(o, o->step + 1, o->ctx->side));
    CUDA_TRY(cudaEventRecord(o->ev_sample, o->ctx->side));
    o->sample_ready = true;
  }
  // adam_step (field.cpp:295-310); grad zeroed in the same pass (mapper.cpp:175)
  const float stepf = (float)(o->step + 1);
  const float c1 = 1.f - std::pow(c.adam_beta1, stepf);
  const float c2 = 1.f - std::pow(c.adam_beta2, stepf);
  {
    ProfScope ps(o->ctx, PRENOM_K_ADAM, st);
    CUDA_TRY(launch_adam(o->P, o->params.p, o->grad.p, o->m.p, o->v.p, c.eta, c.adam_beta1, c.adam_beta2,
                         c.adam_eps, c1, c2, 1, st));
  }
  o->ctx->launches += tc ? 5 : 6;  // sample, fwd, composite, bwd (+ encode_bwd), adam
  o->step += 1;
  // grid refresh every m iterations (mapper.cpp:182-183)
  if (c.grid_refresh_every > 0 && o->step % c.grid_refresh_every == 0) {
    ProfScope ps(o->ctx, PRENOM_K_REFRESH, st);
    CUDA_TRY(launch_refresh_grid(o->fd, o->params.p, o->R, o->grid.p, o->flag.p, st));
    o->ctx->launches += 1;
  }
  return PRENOM_OK;
}

void to_host_stats(const StepStatsDev& d, prenom_step_stats* s) {
  s->total = d.total;
  s->color_term = d.color;
  s->depth_term = d.depth;
  s->sigma_term = d.sigma;
  s->n_samples = (int64_t)d.n_samples;
  s->n_rays_escaped = d.escaped;
  s->frame_index = d.frame;
}

prenom_status set_frame_pixels(prenom_object_s* o, FrameDev* f, const float* rgb, const float* depth,
                               const uint8_t* mask, cudaStream_t st = nullptr) {
  const size_t npx = (size_t)o->W * o->H;
  if (!st) st = o->ctx->stream;
  CUDA_TRY(f->rgb.ensure(npx * 3));
  CUDA_TRY(f->depth.ensure(npx));
  CUDA_TRY(cudaMemcpyAsync(f->rgb.p, rgb, npx * 3 * sizeof(float), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(f->depth.p, depth, npx * sizeof(float), cudaMemcpyHostToDevice, st));
  if (mask) {
    CUDA_TRY(o->fscratch.mask.ensure(npx));
    CUDA_TRY(cudaMemcpyAsync(o->fscratch.mask.p, mask, npx, cudaMemcpyHostToDevice, st));
    CUDA_TRY(build_pixel_lists(o->fscratch.mask.p, o->W, o->H, o->inst, o->cfg.band_px, o->fscratch, f->obj_px,
                               f->bg_px, &f->n_obj_px, &f->n_bg_px, st));
    o->ctx->launches += 9;
  }
  return PRENOM_OK;
}

// Frame records (camera, object-frame ray origin) for n views; pixel data
// is filled by set_frame_pixels or the device renderer.
void init_frames(prenom_object_s* o, int n, const prenom_camera* cams, uint8_t inst, const prenom_pose* pose) {
  for (auto* f : o->frames) delete f;
  o->frames.clear();
  o->W = cams[0].width;
  o->H = cams[0].height;
  o->inst = inst;
  o->pose = *pose;
  // Pose::inverse (geom.hpp:127-130)
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o->Rt[i * 3 + j] = pose->R[j * 3 + i];
  float tt[3];
  mat_vec(o->Rt, pose->t, tt);
  const float tinv[3] = {-tt[0], -tt[1], -tt[2]};
  for (int i = 0; i < n; ++i) {
    auto* f = new FrameDev;
    o->frames.push_back(f);
    f->cam = cams[i];
    float wt[3];
    mat_vec(o->Rt, cams[i].t, wt);
    for (int k = 0; k < 3; ++k) f->origin[k] = wt[k] + tinv[k];
  }
}

}  // namespace

// =========================================================== C ABI
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
  if (cfg->mlp_precision == PRENOM_MLP_BF16 && !tc_supported(make_desc(*arch)))
    return fail(PRENOM_USAGE, "bf16 tensor-core MLP needs F=2, L*F<=32, W in {32,64}, H in {1,2}");
  if (cfg->mlp_precision != PRENOM_MLP_FP32 && cfg->mlp_precision != PRENOM_MLP_BF16)
    return fail(PRENOM_USAGE, "unknown mlp_precision");
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

prenom_status prenom_render(prenom_object_t o, int n_rays, const float* origins, const float* dirs,
                            float* rgb_out, float* depth_out) {
  NvtxRange nvtx_("prenom.render");
  if (!o || !origins || !dirs) return fail(PRENOM_USAGE, "NULL argument");
  if (n_rays < 1) return fail(PRENOM_USAGE, "n_rays must be >= 1");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  const int S = o->cfg.samples_per_ray;
  STATUS_TRY(ensure_scratch(o, n_rays, S));
  cudaStream_t st = o->ctx->stream;
  DevBuf<float> d_o, d_d, d_rgb, d_dep;
  CUDA_TRY(d_o.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_d.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_rgb.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_dep.ensure(n_rays));
  CUDA_TRY(cudaMemcpyAsync(d_o.p, origins, 3 * sizeof(float) * n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_d.p, dirs, 3 * sizeof(float) * n_rays, cudaMemcpyHostToDevice, st));
  RaySource src;
  std::memset(&src, 0, sizeof src);
  src.mode = 1;
  src.origins = d_o.p;
  src.dirs = d_d.p;
  const SampleBufs sb = bufs(o);
  CUDA_TRY(launch_sample(src, sampler_cfg(o, n_rays, o->cfg.prior_sampling, PRENOM_TAG_RENDER,
                                          (uint32_t)o->render_calls++), sb, nullptr, st));
  if (o->cfg.mlp_precision == PRENOM_MLP_BF16)
    CUDA_TRY(launch_fwd_tc(o->fd, o->params.p, (long long)n_rays * S, S, sb.count, sb.pos_depth, o->feat_tc.p,
                           o->out.p, o->flag.p, o->tile_ctr.p, st));
  else
    CUDA_TRY(launch_field_fwd_train(o->fd, o->params.p, n_rays, S, sb, o->feat_t.p, o->out.p, o->flag.p, st));
  CompositeArgs ca;
  std::memset(&ca, 0, sizeof ca);
  ca.B = n_rays;
  ca.S = S;
  ca.pos_depth = sb.pos_depth;
  ca.delta = sb.delta;
  ca.target = sb.target;
  ca.kind = sb.kind;
  ca.count = sb.count;
  ca.out = o->out.p;
  ca.color_out = d_rgb.p;
  ca.depth_out = d_dep.p;
  CUDA_TRY(cudaMemsetAsync(d_rgb.p, 0, 3 * sizeof(float) * n_rays, st));
  CUDA_TRY(cudaMemsetAsync(d_dep.p, 0, sizeof(float) * n_rays, st));
  CUDA_TRY(launch_composite(ca, st));
  o->ctx->launches += 3;
  if (rgb_out) CUDA_TRY(cudaMemcpyAsync(rgb_out, d_rgb.p, 3 * sizeof(float) * n_rays, cudaMemcpyDeviceToHost, st));
  if (depth_out) CUDA_TRY(cudaMemcpyAsync(depth_out, d_dep.p, sizeof(float) * n_rays, cudaMemcpyDeviceToHost, st));
  return check_flag(o);
}

prenom_status prenom_density_query(prenom_object_t o, int R, float* out, int update) {
  NvtxRange nvtx_("prenom.density_query");
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (R < 2 || R > 1024) return fail(PRENOM_DATA, "grid resolution out of range");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  cudaStream_t st = o->ctx->stream;
  const size_t n = (size_t)R * R * R;
  DevBuf<float>& d = o->query;  // kept across calls (no per-query cudaMalloc/cudaFree)
  CUDA_TRY(d.ensure(n));
  CUDA_TRY(launch_refresh_grid(o->fd, o->params.p, R, d.p, o->flag.p, st));
  o->ctx->launches += 1;
  if (out) CUDA_TRY(cudaMemcpyAsync(out, d.p, n * sizeof(float), cudaMemcpyDeviceToHost, st));
  if (update) {
    CUDA_TRY(cudaStreamSynchronize(st));
    std::swap(o->grid.p, d.p);
    std::swap(o->grid.n, d.n);
    o->R = R;
  }
  return check_flag(o);
}

// train_track's tail (mapper.cpp:186-187): refresh_grid at R, choose_iso
// (density_grid.cpp:134-136) unless iso is given, marching_cubes
// (marching_cubes.cpp:125-180) -- all on the device; the mesh stays in the
// object until prenom_get_mesh copies it out.
prenom_status prenom_extract_mesh(prenom_object_t o, int R, float iso, float iso_floor, float* iso_used,
                                  int64_t* n_vertices, int64_t* n_triangles) {
  NvtxRange nvtx_("prenom.extract_mesh");
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (R < 2 || R > 1024) return fail(PRENOM_DATA, "grid resolution out of range");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  cudaStream_t st = o->ctx->stream;
  const size_t n = (size_t)R * R * R;
  McScratch& m = o->ctx->mc;
  CUDA_TRY(m.grid.ensure(n));
  o->ctx->mc_grid_owner = nullptr;
  CUDA_TRY(launch_refresh_grid(o->fd, o->params.p, R, m.grid.p, o->flag.p, st));
  o->ctx->launches += 1;
  STATUS_TRY(check_flag(o));
  float level = iso;
  if (std::isnan(iso)) {
    CUDA_TRY(m.gmax.ensure(1));
    CUDA_TRY(launch_grid_max(m.grid.p, (long long)n, m.gmax.p, st));
    o->ctx->launches += 1;
    float mx = 0.f;
    CUDA_TRY(cudaMemcpyAsync(&mx, m.gmax.p, sizeof(float), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    level = std::fmax(0.5f * mx, iso_floor);
  }
  int launches = 0;
  o->mesh.R = R;
  o->ctx->mc_grid_owner = o;
  CUDA_TRY(run_marching_cubes(m.grid.p, R, level, m, o->mesh, st, &launches));
  o->ctx->launches += launches;
  if (iso_used) *iso_used = level;
  if (n_vertices) *n_vertices = o->mesh.n_vertices;
  if (n_triangles) *n_triangles = o->mesh.n_triangles;
  return PRENOM_OK;
}

prenom_status prenom_get_mesh_grid(prenom_object_t o, int* res, float* grid) {
  if (!o || !res) return fail(PRENOM_USAGE, "NULL argument");
  if (o->mesh.R < 2) return fail(PRENOM_USAGE, "prenom_get_mesh_grid: no mesh extracted yet");
  if (o->ctx->mc_grid_owner != o)
    return fail(PRENOM_USAGE, "prenom_get_mesh_grid: the lattice was replaced by a later extraction on this context");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  *res = o->mesh.R;
  if (grid) {
    const size_t n = (size_t)o->mesh.R * o->mesh.R * o->mesh.R;
    CUDA_TRY(cudaMemcpyAsync(grid, o->ctx->mc.grid.p, n * sizeof(float), cudaMemcpyDeviceToHost, o->ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  }
  return PRENOM_OK;
}

prenom_status prenom_get_mesh(prenom_object_t o, float* vertices, int32_t* triangles) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  cudaStream_t st = o->ctx->stream;
  const McMesh& m = o->mesh;
  if (vertices && m.n_vertices)
    CUDA_TRY(cudaMemcpyAsync(vertices, m.verts.p, 3 * sizeof(float) * m.n_vertices, cudaMemcpyDeviceToHost, st));
  if (triangles && m.n_triangles)
    CUDA_TRY(cudaMemcpyAsync(triangles, m.tris.p, 3 * sizeof(int32_t) * m.n_triangles, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

prenom_status prenom_debug_marching_cubes(prenom_ctx_t c, int R, const float* grid, float iso, int64_t* n_vertices,
                                          int64_t* n_triangles) {
  if (!c || !grid) return fail(PRENOM_USAGE, "NULL argument");
  if (R < 1 || R > 1024) return fail(PRENOM_DATA, "grid resolution out of range");
  CUDA_TRY(cudaSetDevice(c->device));
  McScratch& m = c->mc;
  c->mc_grid_owner = nullptr;
  const size_t n = (size_t)R * R * R;
  CUDA_TRY(m.grid.ensure(n));
  CUDA_TRY(cudaMemcpyAsync(m.grid.p, grid, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  int launches = 0;
  CUDA_TRY(run_marching_cubes(m.grid.p, R, iso, m, c->mc_dbg, c->stream, &launches));
  c->launches += launches;
  if (n_vertices) *n_vertices = c->mc_dbg.n_vertices;
  if (n_triangles) *n_triangles = c->mc_dbg.n_triangles;
  return PRENOM_OK;
}

prenom_status prenom_debug_mesh_get(prenom_ctx_t c, float* vertices, int32_t* triangles) {
  if (!c) return fail(PRENOM_USAGE, "NULL context");
  CUDA_TRY(cudaSetDevice(c->device));
  const McMesh& m = c->mc_dbg;
  if (vertices && m.n_vertices)
    CUDA_TRY(cudaMemcpyAsync(vertices, m.verts.p, 3 * sizeof(float) * m.n_vertices, cudaMemcpyDeviceToHost,
                             c->stream));
  if (triangles && m.n_triangles)
    CUDA_TRY(cudaMemcpyAsync(triangles, m.tris.p, 3 * sizeof(int32_t) * m.n_triangles, cudaMemcpyDeviceToHost,
                             c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return PRENOM_OK;
}

int prenom_mc_case_triangles(int config, int* edges) {
  if (!edges) return -1;
  return mc_case_triangles(config, edges);
}

// metrics.cpp:14-22's nearest-neighbour step (kernels_metrics.cu): per query,
// the exact minimum squared distance to the cloud.
prenom_status prenom_nearest_sq(prenom_ctx_t c, int n_queries, const float* queries, int n_points,
                                const float* points, float* min_sq) {
  if (!c || (n_queries > 0 && (!queries || !min_sq)) || (n_points > 0 && !points))
    return fail(PRENOM_USAGE, "NULL argument");
  if (n_queries < 0 || n_points < 1) return fail(PRENOM_DATA, "nearest_sq: empty cloud");
  CUDA_TRY(cudaSetDevice(c->device));
  DevBuf<float> dq, dp, dout;
  CUDA_TRY(dq.ensure(3 * (size_t)n_queries));
  CUDA_TRY(dp.ensure(3 * (size_t)n_points));
  CUDA_TRY(dout.ensure((size_t)n_queries));
  CUDA_TRY(cudaMemcpyAsync(dq.p, queries, 12 * (size_t)n_queries, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(dp.p, points, 12 * (size_t)n_points, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(launch_nearest_sq(n_queries, dq.p, n_points, dp.p, dout.p, c->stream));
  c->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(min_sq, dout.p, 4 * (size_t)n_queries, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return PRENOM_OK;
}

prenom_status prenom_field_eval(prenom_object_t o, int n, const float* xyz, float* sigma, float* rgb) {
  if (!o || !xyz) return fail(PRENOM_USAGE, "NULL argument");
  if (n < 0) return fail(PRENOM_USAGE, "n < 0");
  if (n == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  cudaStream_t st = o->ctx->stream;
  DevBuf<float> dx, ds, dr;
  CUDA_TRY(dx.ensure(3 * (size_t)n));
  CUDA_TRY(ds.ensure(n));
  CUDA_TRY(dr.ensure(3 * (size_t)n));
  CUDA_TRY(cudaMemcpyAsync(dx.p, xyz, 3 * sizeof(float) * n, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_field_points(o->fd, o->params.p, n, dx.p, ds.p, dr.p, nullptr, nullptr, o->flag.p, st));
  o->ctx->launches += 1;
  if (sigma) CUDA_TRY(cudaMemcpyAsync(sigma, ds.p, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
  if (rgb) CUDA_TRY(cudaMemcpyAsync(rgb, dr.p, 3 * sizeof(float) * n, cudaMemcpyDeviceToHost, st));
  return check_flag(o);
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
  CUDA_TRY(cudaMemcpyAsync(o->m.p, m, o->P * sizeof(float), cudaMemcpyHostToDevice, o->ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(o->v.p, v, o->P * sizeof(float), cudaMemcpyHostToDevice, o->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  o->step = step;
  return PRENOM_OK;
}

prenom_status prenom_reset_adam(prenom_object_t o) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  const size_t P4 = (o->P + 3) & ~size_t(3);
  CUDA_TRY(cudaMemsetAsync(o->m.p, 0, P4 * sizeof(float), o->ctx->stream));
  CUDA_TRY(cudaMemsetAsync(o->v.p, 0, P4 * sizeof(float), o->ctx->stream));
  CUDA_TRY(cudaMemsetAsync(o->grad.p, 0, P4 * sizeof(float), o->ctx->stream));
  o->step = 0;
  return PRENOM_OK;
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

prenom_status prenom_object_set_seed(prenom_object_t o, uint64_t seed) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
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

// ------------------------------------------------------------- debug
prenom_status prenom_debug_philox(prenom_ctx_t ctx, int n, const uint32_t* ck, uint32_t* out) {
  if (!ctx || !ck || !out || n < 0) return fail(PRENOM_USAGE, "bad arguments");
  CUDA_TRY(cudaSetDevice(ctx->device));
  DevBuf<uint32_t> a, b;
  CUDA_TRY(a.ensure(6 * (size_t)n));
  CUDA_TRY(b.ensure(4 * (size_t)n));
  CUDA_TRY(cudaMemcpyAsync(a.p, ck, 6 * sizeof(uint32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(launch_philox(n, a.p, b.p, ctx->stream));
  ctx->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(out, b.p, 4 * sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return PRENOM_OK;
}

prenom_status prenom_debug_hash_encode(prenom_ctx_t ctx, const prenom_field_arch* arch, const float* params, int n,
                                       const float* xyz, float* features) {
  if (!ctx || !params || !xyz || !features || n < 0) return fail(PRENOM_USAGE, "bad arguments");
  STATUS_TRY(validate_arch(arch));
  if (n == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  const FieldDesc fd = make_desc(*arch);
  const size_t P = param_count_host(*arch);
  DevBuf<float> dp, dx, df;
  DevBuf<int> flag;
  CUDA_TRY(dp.ensure(P));
  CUDA_TRY(dx.ensure(3 * (size_t)n));
  CUDA_TRY(df.ensure((size_t)n * fd.in_dim));
  CUDA_TRY(flag.ensure(1));
  cudaStream_t st = ctx->stream;
  CUDA_TRY(cudaMemcpyAsync(dp.p, params, P * sizeof(float), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dx.p, xyz, 3 * sizeof(float) * n, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_field_points(fd, dp.p, n, dx.p, nullptr, nullptr, nullptr, df.p, flag.p, st));
  ctx->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(features, df.p, sizeof(float) * n * fd.in_dim, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

namespace {
// Points as B = n one-sample "rays" through the train-path tile kernels.
struct PointBatch {
  DevBuf<float> params, feat_t, dfeat_t, grad;
  DevBuf<unsigned char> feat_tc;
  DevBuf<float4> pos, out, dout;
  DevBuf<int> count, flag, ctr;
  SampleBufs sb;
  prenom_status init(const FieldDesc& fd, size_t P, int n, const float* h_params, const float* xyz,
                     cudaStream_t st) {
    const size_t npad = ((size_t)n + kTile - 1) / kTile * kTile;
    CUDA_TRY(params.ensure(P));
    CUDA_TRY(feat_t.ensure(npad * fd.in_dim));
    CUDA_TRY(dfeat_t.ensure(npad * fd.in_dim));
    if (tc_supported(fd)) CUDA_TRY(feat_tc.ensure(tc_feature_bytes(fd, n)));
    CUDA_TRY(pos.ensure(npad));
    CUDA_TRY(out.ensure(npad));
    CUDA_TRY(dout.ensure(npad));
    CUDA_TRY(count.ensure(n));
    CUDA_TRY(flag.ensure(1));
    CUDA_TRY(ctr.ensure(4));
    CUDA_TRY(cudaMemset(ctr.p, 0, 4 * sizeof(int)));
    CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    CUDA_TRY(cudaMemcpyAsync(params.p, h_params, P * sizeof(float), cudaMemcpyHostToDevice, st));
    std::vector<float4> hp(n);
    std::vector<int> hc(n, 1);
    for (int i = 0; i < n; ++i) hp[i] = make_float4(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], 0.f);
    CUDA_TRY(cudaMemcpyAsync(pos.p, hp.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(count.p, hc.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    std::memset(&sb, 0, sizeof sb);
    sb.pos_depth = pos.p;
    sb.count = count.p;
    return PRENOM_OK;
  }
};
}  // namespace

prenom_status prenom_debug_field_eval(prenom_ctx_t ctx, const prenom_field_arch* arch, const float* params, int n,
                                      const float* xyz, float* sigma, float* rgb, float* raw, int precision) {
  if (!ctx || !params || !xyz || n < 0) return fail(PRENOM_USAGE, "bad arguments");
  STATUS_TRY(validate_arch(arch));
  if (n == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  const FieldDesc fd = make_desc(*arch);
  const size_t P = param_count_host(*arch);
  cudaStream_t st = ctx->stream;
  int hflag = 0;
  if (precision == PRENOM_MLP_FP32) {
    DevBuf<float> dp, dx, ds, dr, dw;
    DevBuf<int> flag;
    CUDA_TRY(dp.ensure(P));
    CUDA_TRY(dx.ensure(3 * (size_t)n));
    CUDA_TRY(ds.ensure(n));
    CUDA_TRY(dr.ensure(3 * (size_t)n));
    CUDA_TRY(dw.ensure(4 * (size_t)n));
    CUDA_TRY(flag.ensure(1));
    CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    CUDA_TRY(cudaMemcpyAsync(dp.p, params, P * sizeof(float), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dx.p, xyz, 3 * sizeof(float) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(launch_field_points(fd, dp.p, n, dx.p, ds.p, dr.p, dw.p, nullptr, flag.p, st));
    ctx->launches += 1;
    if (sigma) CUDA_TRY(cudaMemcpyAsync(sigma, ds.p, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    if (rgb) CUDA_TRY(cudaMemcpyAsync(rgb, dr.p, 3 * sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    if (raw) CUDA_TRY(cudaMemcpyAsync(raw, dw.p, 4 * sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&hflag, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  } else if (precision == 2 || precision == PRENOM_MLP_BF16) {
    // the train-path tile forward: fp32 smem GEMMs (2) or bf16 tcgen05 (1)
    if (precision == PRENOM_MLP_BF16 && !tc_supported(fd)) return fail(PRENOM_USAGE, "arch not supported by the bf16 path");
    PointBatch pb;
    STATUS_TRY(pb.init(fd, P, n, params, xyz, st));
    if (precision == PRENOM_MLP_BF16)
      CUDA_TRY(launch_fwd_tc(fd, pb.params.p, n, 1, pb.count.p, pb.pos.p, pb.feat_tc.p, pb.out.p, pb.flag.p, pb.ctr.p,
                             st));
    else
      CUDA_TRY(launch_field_fwd_train(fd, pb.params.p, n, 1, pb.sb, pb.feat_t.p, pb.out.p, pb.flag.p, st));
    ctx->launches += 1;
    std::vector<float4> h(n);
    CUDA_TRY(cudaMemcpyAsync(h.data(), pb.out.p, sizeof(float4) * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&hflag, pb.flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    for (int i = 0; i < n; ++i) {
      if (sigma) sigma[i] = h[i].x;
      if (rgb) {
        rgb[3 * i] = h[i].y;
        rgb[3 * i + 1] = h[i].z;
        rgb[3 * i + 2] = h[i].w;
      }
    }
    if (raw) std::memset(raw, 0, sizeof(float) * 4 * n);
  } else {
    return fail(PRENOM_USAGE, "unsupported mlp precision for debug_field_eval");
  }
  if (hflag) return fail(PRENOM_NUMERIC, "field_eval produced a non-finite output");
  return PRENOM_OK;
}

prenom_status prenom_debug_field_backward(prenom_ctx_t ctx, const prenom_field_arch* arch, const float* params,
                                          int n, const float* xyz, const float* d_sigma, const float* d_rgb,
                                          float* grad, int precision) {
  if (!ctx || !params || !xyz || !d_sigma || !d_rgb || !grad || n < 0) return fail(PRENOM_USAGE, "bad arguments");
  STATUS_TRY(validate_arch(arch));
  const FieldDesc fd = make_desc(*arch);
  const size_t P = param_count_host(*arch);
  if (n == 0) {
    std::memset(grad, 0, P * sizeof(float));
    return PRENOM_OK;
  }
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  PointBatch pb;
  STATUS_TRY(pb.init(fd, P, n, params, xyz, st));
  CUDA_TRY(pb.grad.ensure(P));
  CUDA_TRY(cudaMemsetAsync(pb.grad.p, 0, P * sizeof(float), st));
  std::vector<float4> hd(n);
  for (int i = 0; i < n; ++i) hd[i] = make_float4(d_sigma[i], d_rgb[3 * i], d_rgb[3 * i + 1], d_rgb[3 * i + 2]);
  CUDA_TRY(cudaMemcpyAsync(pb.dout.p, hd.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, st));
  if (precision == PRENOM_MLP_BF16) {
    if (!tc_supported(fd)) return fail(PRENOM_USAGE, "arch not supported by the bf16 path");
    CUDA_TRY(launch_fwd_tc(fd, pb.params.p, n, 1, pb.count.p, pb.pos.p, pb.feat_tc.p, pb.out.p, pb.flag.p, pb.ctr.p,
                           st));
    CUDA_TRY(launch_bwd_tc(fd, pb.params.p, pb.grad.p, n, 1, pb.count.p, pb.pos.p, pb.feat_tc.p, pb.dout.p,
                           pb.ctr.p + 2, st));
  } else {
    CUDA_TRY(launch_field_fwd_train(fd, pb.params.p, n, 1, pb.sb, pb.feat_t.p, pb.out.p, pb.flag.p, st));
    CUDA_TRY(launch_mlp_bwd_train(fd, pb.params.p, pb.grad.p, n, 1, pb.count.p, pb.feat_t.p, pb.dout.p,
                                  pb.dfeat_t.p, st));
    CUDA_TRY(launch_encode_bwd(fd, pb.params.p, pb.grad.p, n, 1, pb.count.p, pb.pos.p, pb.dfeat_t.p, st));
  }
  ctx->launches += 3;
  CUDA_TRY(cudaMemcpyAsync(grad, pb.grad.p, P * sizeof(float), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

prenom_status prenom_debug_adam(prenom_ctx_t ctx, size_t n, float* params, const float* grads, float* m, float* v,
                                int64_t* step, float lr, float b1, float b2, float eps) {
  if (!ctx || !params || !grads || !m || !v || !step) return fail(PRENOM_USAGE, "NULL argument");
  if (n == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  DevBuf<float> dp, dg, dm, dv;
  CUDA_TRY(dp.ensure(n));
  CUDA_TRY(dg.ensure(n));
  CUDA_TRY(dm.ensure(n));
  CUDA_TRY(dv.ensure(n));
  CUDA_TRY(cudaMemcpyAsync(dp.p, params, n * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dg.p, grads, n * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dm.p, m, n * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dv.p, v, n * 4, cudaMemcpyHostToDevice, st));
  *step += 1;
  const float c1 = 1.f - std::pow(b1, (float)*step), c2 = 1.f - std::pow(b2, (float)*step);
  CUDA_TRY(launch_adam(n, dp.p, dg.p, dm.p, dv.p, lr, b1, b2, eps, c1, c2, 0, st));
  ctx->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(params, dp.p, n * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(m, dm.p, n * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(v, dv.p, n * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

prenom_status prenom_debug_sample_rays(prenom_ctx_t ctx, int n_rays, const float* origins, const float* dirs,
                                       const float box_min[3], const float box_max[3], int prior, int grid_res,
                                       const float* grid, int n_coarse, int n_fine, float eps, uint64_t seed,
                                       int64_t step, float* depths, float* deltas, float* positions, int* count,
                                       float* t_entry, float* t_exit) {
  if (!ctx || !origins || !dirs || !box_min || !box_max || n_rays < 0) return fail(PRENOM_USAGE, "bad arguments");
  if (prior && (!grid || grid_res < 2)) return fail(PRENOM_USAGE, "prior sampling needs a grid");
  if (n_fine < 1 || n_fine > 1024 || (prior && (n_coarse < 1 || n_coarse > 1024)))
    return fail(PRENOM_USAGE, "sample counts out of range");
  if (n_rays == 0) return PRENOM_OK;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t N = (size_t)n_rays * n_fine;
  DevBuf<float> d_o, d_d, d_g, d_delta, d_te, d_tx;
  DevBuf<float4> d_pd, d_tgt;
  DevBuf<int> d_kind, d_cnt;
  CUDA_TRY(d_o.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_d.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_pd.ensure(N));
  CUDA_TRY(d_delta.ensure(N));
  CUDA_TRY(d_tgt.ensure(n_rays));
  CUDA_TRY(d_kind.ensure(n_rays));
  CUDA_TRY(d_cnt.ensure(n_rays));
  CUDA_TRY(d_te.ensure(n_rays));
  CUDA_TRY(d_tx.ensure(n_rays));
  CUDA_TRY(cudaMemcpyAsync(d_o.p, origins, 12 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_d.p, dirs, 12 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  if (prior) {
    const size_t gv = (size_t)grid_res * grid_res * grid_res;
    CUDA_TRY(d_g.ensure(gv));
    CUDA_TRY(cudaMemcpyAsync(d_g.p, grid, gv * 4, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(cudaMemsetAsync(d_pd.p, 0, N * sizeof(float4), st));
  CUDA_TRY(cudaMemsetAsync(d_delta.p, 0, N * sizeof(float), st));
  RaySource src;
  std::memset(&src, 0, sizeof src);
  src.mode = 1;
  src.origins = d_o.p;
  src.dirs = d_d.p;
  SamplerCfg c;
  std::memset(&c, 0, sizeof c);
  c.B = n_rays;
  c.S = n_fine;
  c.prior = prior;
  c.n_coarse = n_coarse;
  c.eps = eps;
  c.grid_res = grid_res;
  c.grid = d_g.p;
  std::memcpy(c.bmin, box_min, 12);
  std::memcpy(c.bmax, box_max, 12);
  c.seed = seed;
  c.tag = PRENOM_TAG_FINE;
  c.step = (uint32_t)step;
  SampleBufs sb;
  std::memset(&sb, 0, sizeof sb);
  sb.pos_depth = d_pd.p;
  sb.delta = d_delta.p;
  sb.target = d_tgt.p;
  sb.kind = d_kind.p;
  sb.count = d_cnt.p;
  sb.t_entry = d_te.p;
  sb.t_exit = d_tx.p;
  CUDA_TRY(launch_sample(src, c, sb, nullptr, st));
  ctx->launches += 1;
  std::vector<float4> hpd(N);
  CUDA_TRY(cudaMemcpyAsync(hpd.data(), d_pd.p, N * sizeof(float4), cudaMemcpyDeviceToHost, st));
  if (deltas) CUDA_TRY(cudaMemcpyAsync(deltas, d_delta.p, N * 4, cudaMemcpyDeviceToHost, st));
  if (count) CUDA_TRY(cudaMemcpyAsync(count, d_cnt.p, 4 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  if (t_entry) CUDA_TRY(cudaMemcpyAsync(t_entry, d_te.p, 4 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  if (t_exit) CUDA_TRY(cudaMemcpyAsync(t_exit, d_tx.p, 4 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (size_t i = 0; i < N; ++i) {
    if (depths) depths[i] = hpd[i].w;
    if (positions) {
      positions[3 * i] = hpd[i].x;
      positions[3 * i + 1] = hpd[i].y;
      positions[3 * i + 2] = hpd[i].z;
    }
  }
  return PRENOM_OK;
}

prenom_status prenom_debug_batch_loss(prenom_ctx_t ctx, int n_rays, int S, const int* kind, const float* target_rgb,
                                      const float* target_depth, const int* count, const float* deltas,
                                      const float* depths, const float* sigma, const float* rgb,
                                      const float* bg_colors, float lambda_d, float lambda_sigma, double* terms,
                                      float* d_sigma, float* d_rgb, float* color_out, float* depth_out) {
  if (!ctx || !kind || !target_rgb || !target_depth || !count || !deltas || !depths || !sigma || !rgb || !bg_colors ||
      !terms || n_rays < 0 || S < 1 || S > 256)
    return fail(PRENOM_USAGE, "bad arguments");
  if (n_rays == 0) return fail(PRENOM_DATA, "batch_loss: no rays");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  const size_t N = (size_t)n_rays * S;
  std::vector<float4> hpd(N), hout(N), htgt(n_rays);
  for (size_t i = 0; i < N; ++i) {
    hpd[i] = make_float4(0.f, 0.f, 0.f, depths[i]);
    hout[i] = make_float4(sigma[i], rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
  }
  for (int r = 0; r < n_rays; ++r) {
    if (count[r] != 0 && count[r] != S) return fail(PRENOM_USAGE, "count must be 0 or S");
    htgt[r] = make_float4(target_rgb[3 * r], target_rgb[3 * r + 1], target_rgb[3 * r + 2], target_depth[r]);
  }
  DevBuf<float4> d_pd, d_out, d_dout, d_tgt;
  DevBuf<float> d_delta, d_bg, d_col, d_dep;
  DevBuf<int> d_kind, d_cnt, d_flag;
  DevBuf<StepStatsDev> d_stats;
  CUDA_TRY(d_pd.ensure(N));
  CUDA_TRY(d_out.ensure(N));
  CUDA_TRY(d_dout.ensure(N));
  CUDA_TRY(d_tgt.ensure(n_rays));
  CUDA_TRY(d_delta.ensure(N));
  CUDA_TRY(d_bg.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_col.ensure(3 * (size_t)n_rays));
  CUDA_TRY(d_dep.ensure(n_rays));
  CUDA_TRY(d_kind.ensure(n_rays));
  CUDA_TRY(d_cnt.ensure(n_rays));
  CUDA_TRY(d_flag.ensure(1));
  CUDA_TRY(d_stats.ensure(1));
  CUDA_TRY(cudaMemcpyAsync(d_pd.p, hpd.data(), N * sizeof(float4), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_out.p, hout.data(), N * sizeof(float4), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_tgt.p, htgt.data(), n_rays * sizeof(float4), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_delta.p, deltas, N * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_bg.p, bg_colors, 12 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_kind.p, kind, 4 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_cnt.p, count, 4 * (size_t)n_rays, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(d_dout.p, 0, N * sizeof(float4), st));
  CUDA_TRY(cudaMemsetAsync(d_col.p, 0, 12 * (size_t)n_rays, st));
  CUDA_TRY(cudaMemsetAsync(d_dep.p, 0, 4 * (size_t)n_rays, st));
  CUDA_TRY(cudaMemsetAsync(d_flag.p, 0, 4, st));
  CUDA_TRY(cudaMemsetAsync(d_stats.p, 0, sizeof(StepStatsDev), st));
  CompositeArgs ca;
  std::memset(&ca, 0, sizeof ca);
  ca.B = n_rays;
  ca.S = S;
  ca.pos_depth = d_pd.p;
  ca.delta = d_delta.p;
  ca.target = d_tgt.p;
  ca.kind = d_kind.p;
  ca.count = d_cnt.p;
  ca.out = d_out.p;
  ca.bg_colors = d_bg.p;
  ca.lambda_d = lambda_d;
  ca.lambda_sigma = lambda_sigma;
  ca.dout = d_dout.p;
  ca.color_out = d_col.p;
  ca.depth_out = d_dep.p;
  ca.stats = d_stats.p;
  ca.flag = d_flag.p;
  CUDA_TRY(launch_composite(ca, st));
  ctx->launches += 2;
  StepStatsDev hs;
  std::vector<float4> hd(N);
  int hflag = 0;
  CUDA_TRY(cudaMemcpyAsync(&hs, d_stats.p, sizeof hs, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(hd.data(), d_dout.p, N * sizeof(float4), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&hflag, d_flag.p, 4, cudaMemcpyDeviceToHost, st));
  if (color_out) CUDA_TRY(cudaMemcpyAsync(color_out, d_col.p, 12 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  if (depth_out) CUDA_TRY(cudaMemcpyAsync(depth_out, d_dep.p, 4 * (size_t)n_rays, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  terms[0] = hs.total;
  terms[1] = hs.color;
  terms[2] = hs.depth;
  terms[3] = hs.sigma;
  for (size_t i = 0; i < N; ++i) {
    if (d_sigma) d_sigma[i] = hd[i].x;
    if (d_rgb) {
      d_rgb[3 * i] = hd[i].y;
      d_rgb[3 * i + 1] = hd[i].z;
      d_rgb[3 * i + 2] = hd[i].w;
    }
  }
  if (hflag) return fail(PRENOM_NUMERIC, "batch_loss: non-finite loss");
  return PRENOM_OK;
}

prenom_status prenom_debug_generate_rays(prenom_object_t o, int frame, int64_t step, float* origins, float* dirs,
                                         int* kind, float* target_rgb, float* target_depth, int* pick_px) {
  if (!o) return fail(PRENOM_USAGE, "NULL object");
  if (frame < 0 || frame >= (int)o->frames.size()) return fail(PRENOM_USAGE, "frame index out of range");
  CUDA_TRY(cudaSetDevice(o->ctx->device));
  const int B = o->cfg.rays_per_iter;
  STATUS_TRY(ensure_scratch(o, B, o->cfg.samples_per_ray));
  const RaySource src = frame_source(o, frame);
  if (src.n_obj_px == 0) return fail(PRENOM_DATA, "generate_rays: no object pixels");
  cudaStream_t st = o->ctx->stream;
  DevBuf<float> d_o, d_d;
  DevBuf<int> d_pick;
  CUDA_TRY(d_o.ensure(3 * (size_t)B));
  CUDA_TRY(d_d.ensure(3 * (size_t)B));
  CUDA_TRY(d_pick.ensure(B));
  SampleBufs sb = bufs(o);
  sb.ray_o = d_o.p;
  sb.ray_d = d_d.p;
  sb.pick_px = d_pick.p;
  CUDA_TRY(launch_sample(src, sampler_cfg(o, B, 0, PRENOM_TAG_FINE, (uint32_t)step), sb, nullptr, st));
  o->ctx->launches += 1;
  std::vector<float4> tg(B);
  if (origins) CUDA_TRY(cudaMemcpyAsync(origins, d_o.p, 12 * (size_t)B, cudaMemcpyDeviceToHost, st));
  if (dirs) CUDA_TRY(cudaMemcpyAsync(dirs, d_d.p, 12 * (size_t)B, cudaMemcpyDeviceToHost, st));
  if (pick_px) CUDA_TRY(cudaMemcpyAsync(pick_px, d_pick.p, 4 * (size_t)B, cudaMemcpyDeviceToHost, st));
  if (kind) CUDA_TRY(cudaMemcpyAsync(kind, sb.kind, 4 * (size_t)B, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(tg.data(), sb.target, sizeof(float4) * B, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int r = 0; r < B; ++r) {
    if (target_rgb) {
      target_rgb[3 * r] = tg[r].x;
      target_rgb[3 * r + 1] = tg[r].y;
      target_rgb[3 * r + 2] = tg[r].z;
    }
    if (target_depth) target_depth[r] = tg[r].w;
  }
  return PRENOM_OK;
}

prenom_status prenom_debug_umma_gemm(prenom_ctx_t ctx, int M, int N, int K, int a_mn, int b_mn, const float* A,
                                     const float* B, float* D) {
  if (!ctx || !A || !B || !D) return fail(PRENOM_USAGE, "NULL argument");
  if ((M != 64 && M != 128) || N < 8 || N > 256 || N % 8 || K < 16 || K % 16 || K > 256 ||
      (M == 128 && N % 16))
    return fail(PRENOM_USAGE, "unsupported UMMA shape");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  DevBuf<float> a, b, d;
  CUDA_TRY(a.ensure((size_t)M * K));
  CUDA_TRY(b.ensure((size_t)N * K));
  CUDA_TRY(d.ensure((size_t)M * N));
  CUDA_TRY(cudaMemcpyAsync(a.p, A, sizeof(float) * M * K, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(b.p, B, sizeof(float) * N * K, cudaMemcpyHostToDevice, st));
  CUDA_TRY(launch_umma_gemm(M, N, K, a_mn, b_mn, a.p, b.p, d.p, st));
  ctx->launches += 1;
  CUDA_TRY(cudaMemcpyAsync(D, d.p, sizeof(float) * M * N, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return PRENOM_OK;
}

}  // extern "C"
