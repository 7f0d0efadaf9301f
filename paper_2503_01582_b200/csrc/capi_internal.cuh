// capi_internal.cuh -- host-side internals shared by the C-ABI translation units
// (capi.cu: contexts, objects, frames, state; capi_train.cu: train steps,
// multi-object scheduler, Reptile; capi_query.cu: render, density query,
// mesh, field eval, metric NN; capi_debug.cu: single-stage parity entry points).
//
// Owns per-GPU contexts and per-object device state, and orchestrates the
// train step (train_track's loop body, mapper.cpp:150-184) as a sequence of
// kernel launches on the context stream:
//   k_sample -> k_fwd_tc | k_fwd_tile -> k_composite (+stats) ->
//   k_bwd_tc | k_bwd_tile + k_encode_bwd -> k_adam [-> k_field_points (refresh every m)]
// The host never touches sample data: per step it only draws the keyframe
// index (one Philox call, TAG_FRAME) and computes the Adam bias corrections
// with glibc powf (field.cpp:300-301), like the reference.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include "prenom_device.cuh"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: host ranges for nsys/ncu timelines

using namespace prenom;  // internal header of the C-ABI translation units only
namespace prenom_capi {}
using namespace prenom_capi;


namespace prenom_capi {

inline thread_local std::string g_err;

void comm_destroy(prenom_ctx_t ctx);  // capi_comm.cu

inline prenom_status fail(prenom_status s, const std::string& msg) {
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

inline int level_resolution_host(const prenom_field_arch& a, int level) {
  const double r = a.base_resolution * std::pow((double)a.per_level_scale, level);  // field.cpp:113-116
  return std::max(1, (int)r);
}

inline prenom_status validate_arch(const prenom_field_arch* a) {
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

inline FieldDesc make_desc(const prenom_field_arch& a) {
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

inline size_t param_count_host(const prenom_field_arch& a) {
  const FieldDesc d = make_desc(a);
  return (size_t)d.hash_params + (size_t)d.mlp_params;
}

inline void mat_vec(const float* M, const float* v, float* out) {
  out[0] = M[0] * v[0] + M[1] * v[1] + M[2] * v[2];
  out[1] = M[3] * v[0] + M[4] * v[1] + M[5] * v[2];
  out[2] = M[6] * v[0] + M[7] * v[1] + M[8] * v[2];
}

inline uint32_t philox_first(uint64_t seed, uint32_t tag, uint32_t step, uint32_t ray, uint32_t idx) {
  const uint32_t ctr[4] = {idx, ray, step, tag};
  uint32_t out[4];
  pdm_philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32), out);
  return out[0];
}

}  // namespace

constexpr int kDefaultLanes = 8;  // B200, with >= 8 tiles per persistent CTA: cfg3 4 lanes 1.35e9, 8 lanes 1.41e9;
                                  // cfg5 4: 1.10e9, 8: 1.12e9 (1 lane: cfg3 1.00e9)
constexpr int kMaxLanes = 16;
constexpr int kGroupMaxDefault = 0;  // objects per grouped unit of the multi-object scheduler (0 = all)
constexpr int kLaneMinTilesPerCta = 16;  // split mode, B200: cfg3 1.13 -> 1.22e9, cfg5 1.01 -> 1.06e9, cfg4 0.81 -> 0.85e9 vs 8 (32: within 1%)
constexpr int kL2PersistDefault = 0;  // off: measured on cfg2, persisting the table (1) or its gradient (2)
                                       // slows the step 0.657 -> 0.745 / 0.772 ms (Adam 0.10 -> 0.17 ms)

// Device scratch of one grouped launch sequence (multi-object scheduler): the
// object table of the grouped forward / backward, their tile counters and the
// per-step job arrays of the grouped sampling, compositing and Adam launches.
struct GroupScratch {
  DevBuf<TcObj> objs;
  DevBuf<int> ctr;  // [fwd next, fwd done (self-resetting), bwd next, part slots of objects 0..K-1]
  DevBuf<unsigned char> jobs;
};

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
  // objects of one architecture and batch shape train through grouped launches
  // (one launch per stage for all of them) when on: prenom_ctx_set_grouping /
  // PRENOM_GROUPED=1. Off by default: measured on B200 the grouped launches are
  // 13-31% faster per launch, but the lanes overlap one object's Adam with
  // another's backward, which a grouped step cannot (multi-object scheduler)
  bool grouping = false;
  std::vector<GroupScratch*> groups;
  ~prenom_ctx_s() {
    for (auto* g : groups) delete g;
  }
  int64_t launches = 0;
  // NCCL communicator of the Reptile all-reduce (prenom_ctx_init_comm; an
  // opaque ncclComm_t, NCCL is loaded at run time) and its buffers
  void* comm = nullptr;
  int comm_size = 1, comm_rank = 0;
  DevBuf<float> reptile_sum;          // this rank's sum of task deltas, all-reduced in place
  DevBuf<const float*> reptile_ptrs;  // adapted parameter vectors of one reptile step
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

namespace prenom_capi {
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
  DevBuf<float> mlp_part;         // per-CTA MLP weight-gradient partials of the tensor-core backward
  DevBuf<int> tile_ctr;           // dynamic tile-scheduler counters (fwd, bwd)
  DevBuf<int> kind, count;
  DevBuf<StepStatsDev> stats;
  int last_n_steps = 0;
  // sample-ahead pipelining (k_sample(t+1) on ctx->side while k_adam(t) runs)
  cudaEvent_t ev_bwd = nullptr, ev_sample = nullptr;
  bool sample_ready = false;
  int prefetch_frame = -1;  // keyframe the prefetched samples were drawn from
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

namespace prenom_capi {

// tensor-core MLP modes (bf16 / split bf16) and their split flag
inline bool uses_tc(const prenom_object_s* o) { return o->cfg.mlp_precision != PRENOM_MLP_FP32; }
inline int tc_split(const prenom_object_s* o) { return o->cfg.mlp_precision == PRENOM_MLP_BF16X3 ? 1 : 0; }

inline prenom_status ensure_scratch(prenom_object_s* o, int B, int S) {
  const size_t N = (size_t)B * S;
  const size_t Npad = ((N + kTile - 1) / kTile) * kTile;
  CUDA_TRY(o->pos_depth.ensure(Npad));
  CUDA_TRY(o->delta.ensure(Npad));
  CUDA_TRY(o->out.ensure(Npad));
  CUDA_TRY(o->dout.ensure(Npad));
  if (uses_tc(o)) {
    unsigned char* before = o->feat_tc.p;
    CUDA_TRY(o->feat_tc.ensure(tc_feature_bytes(o->fd, (long long)N, tc_split(o))));
    if (o->feat_tc.p != before)
      CUDA_TRY(init_feature_tiles(o->fd, o->feat_tc.p, o->feat_tc.n, tc_split(o), o->ctx->stream));
    CUDA_TRY(o->mlp_part.ensure(tc_mlp_part_floats(o->fd)));
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

inline SampleBufs bufs(prenom_object_s* o) {
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

inline prenom_status check_flag(prenom_object_s* o) {
  int f = 0;
  CUDA_TRY(cudaMemcpyAsync(&f, o->flag.p, sizeof(int), cudaMemcpyDeviceToHost, o->ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(o->ctx->stream));
  if (f & 1) return fail(PRENOM_NUMERIC, "field_eval produced a non-finite output");
  if (f & 2) return fail(PRENOM_NUMERIC, "batch_loss: non-finite loss");
  return PRENOM_OK;
}

inline RaySource frame_source(prenom_object_s* o, int fi) {
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

inline SamplerCfg sampler_cfg(prenom_object_s* o, int B, int prior, uint32_t tag, uint32_t step) {
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

inline int frame_of_step(const prenom_object_s* o, int64_t step) {  // keyframe pick (mapper.cpp:151)
  return (int)pdm_pick(philox_first(o->seed, PRENOM_TAG_FRAME, (uint32_t)step, 0, 0), (uint32_t)o->frames.size());
}

// generate_rays + sample_ray for `step` (render.cpp:47-102, density_grid.cpp:110-117)
inline prenom_status enqueue_sample(prenom_object_s* o, int64_t step, cudaStream_t st) {
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
// L2 residency (SURVEY §7 hard part 4): an access-policy window over one of
// the object's 64 MiB-class arrays marks its lines persisting in L2, so
// Adam's 256 MiB stream does not evict them between steps. Mode from
// PRENOM_L2_PERSIST: 0 off, 1 the hash table (gathers), 2 the table
// gradient (scatter RMW).
inline int l2_persist_mode() {
  static const int m = [] {
    const char* e = getenv("PRENOM_L2_PERSIST");
    return e ? atoi(e) : kL2PersistDefault;
  }();
  return m;
}

inline cudaError_t set_l2_window(prenom_object_s* o, cudaStream_t st) {
  const int mode = l2_persist_mode();
  if (mode == 0) return cudaSuccess;
  static size_t max_persist = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, dev);
    if (v > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)v);
    return (size_t)(v > 0 ? v : 0);
  }();
  static size_t max_window = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    return (size_t)(v > 0 ? v : 0);
  }();
  if (!max_persist || !max_window) return cudaSuccess;
  const size_t bytes = std::min<size_t>((size_t)o->fd.hash_params * sizeof(float), max_window);
  cudaStreamAttrValue a;
  std::memset(&a, 0, sizeof a);
  a.accessPolicyWindow.base_ptr = mode == 2 ? (void*)o->grad.p : (void*)o->params.p;
  a.accessPolicyWindow.num_bytes = bytes;
  a.accessPolicyWindow.hitRatio = std::min(1.f, (float)max_persist / (float)bytes);
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  return cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a);
}

// composite_backward + batch_loss arguments of a train step (render.cpp:156-243)
inline CompositeArgs train_composite_args(prenom_object_s* o, StepStatsDev* stats, uint32_t step, int fi) {
  const SampleBufs sb = bufs(o);
  CompositeArgs ca;
  std::memset(&ca, 0, sizeof ca);
  ca.B = o->cfg.rays_per_iter;
  ca.S = o->cfg.samples_per_ray;
  ca.pos_depth = sb.pos_depth;
  ca.delta = sb.delta;
  ca.target = sb.target;
  ca.kind = sb.kind;
  ca.count = sb.count;
  ca.out = o->out.p;
  ca.bg_colors = nullptr;
  ca.seed = o->seed;
  ca.step = step;
  ca.lambda_d = o->cfg.lambda_d;
  ca.lambda_sigma = o->cfg.lambda_sigma;
  ca.dout = o->dout.p;
  ca.stats = stats;
  ca.flag = o->flag.p;
  ca.frame = fi;
  return ca;
}

// Adam bias corrections of step `step` (0-based) with glibc powf, like the reference (field.cpp:300-301)
inline void adam_corrections(const prenom_object_s* o, int64_t step, float& c1, float& c2) {
  const float stepf = (float)(step + 1);
  c1 = 1.f - std::pow(o->cfg.adam_beta1, stepf);
  c2 = 1.f - std::pow(o->cfg.adam_beta2, stepf);
}

inline prenom_status enqueue_step(prenom_object_s* o, StepStatsDev* stats, bool has_next = false) {
  NvtxRange nvtx_("prenom.step");
  cudaStream_t st = o->lane ? o->lane : o->ctx->stream;
  CUDA_TRY(set_l2_window(o, st));
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
  const bool tc = uses_tc(o);
  int mlp_nparts = 0;  // per-CTA MLP-gradient partials the backward left for Adam
  {
    ProfScope ps(o->ctx, PRENOM_K_FIELD_FWD, st);
    if (tc)
      CUDA_TRY(launch_fwd_tc(o->fd, o->params.p, (long long)B * S, S, sb.count, sb.pos_depth, o->feat_tc.p, o->out.p,
                             o->flag.p, o->tile_ctr.p, tc_split(o), st));
    else
      CUDA_TRY(launch_field_fwd_train(o->fd, o->params.p, B, S, sb, o->feat_t.p, o->out.p, o->flag.p, st));
  }
  const CompositeArgs ca = train_composite_args(o, stats, step, fi);
  {
    ProfScope ps(o->ctx, PRENOM_K_COMPOSITE, st);
    CUDA_TRY(launch_composite(ca, st));
  }
  if (tc) {
    ProfScope ps(o->ctx, PRENOM_K_MLP_BWD, st);  // MLP backward + fused table-gradient scatter
    // (the MLP-gradient reduction is folded into this step's Adam: launch_adam_fused)
    CUDA_TRY(launch_bwd_tc(o->fd, o->params.p, o->grad.p, (long long)B * S, S, sb.count, sb.pos_depth,
                           o->feat_tc.p, o->dout.p, o->tile_ctr.p + 2, tc_split(o), o->mlp_part.p, o->mlp_part.n,
                           st, &mlp_nparts));
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
  // (per-kernel timing serialises the sampler: its events then time the kernel alone)
  if (has_next && !refresh_now && o->ctx->overlap && !o->ctx->prof) {
    if (!o->ev_bwd) {
      CUDA_TRY(cudaEventCreateWithFlags(&o->ev_bwd, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&o->ev_sample, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventRecord(o->ev_bwd, st));
    CUDA_TRY(cudaStreamWaitEvent(o->ctx->side, o->ev_bwd, 0));
    STATUS_TRY(enqueue_sample(o, o->step + 1, o->ctx->side));
    CUDA_TRY(cudaEventRecord(o->ev_sample, o->ctx->side));
    o->sample_ready = true;
    o->prefetch_frame = frame_of_step(o, o->step + 1);
  }
  // adam_step (field.cpp:295-310); grad zeroed in the same pass (mapper.cpp:175)
  float c1, c2;
  adam_corrections(o, o->step, c1, c2);
  {
    ProfScope ps(o->ctx, PRENOM_K_ADAM, st);
    if (mlp_nparts > 0)
      CUDA_TRY(launch_adam_fused(o->P, (size_t)o->fd.hash_params, o->fd.mlp_params, o->params.p, o->grad.p, o->m.p,
                                 o->v.p, c.eta, c.adam_beta1, c.adam_beta2, c.adam_eps, c1, c2, o->mlp_part.p,
                                 mlp_nparts, st));
    else
      CUDA_TRY(launch_adam(o->P, o->params.p, o->grad.p, o->m.p, o->v.p, c.eta, c.adam_beta1, c.adam_beta2,
                           c.adam_eps, c1, c2, 1, st));
  }
  // sample, fwd, composite, bwd (+ encode_bwd on the SIMT path, + the MLP-gradient reduce when it was not
  // folded into Adam), adam
  o->ctx->launches += (tc && mlp_nparts > 0) ? 5 : 6;
  o->step += 1;
  // grid refresh every m iterations (mapper.cpp:182-183)
  if (c.grid_refresh_every > 0 && o->step % c.grid_refresh_every == 0) {
    ProfScope ps(o->ctx, PRENOM_K_REFRESH, st);
    CUDA_TRY(launch_refresh_grid(o->fd, o->params.p, o->R, o->grid.p, o->flag.p, st));
    o->ctx->launches += 1;
  }
  return PRENOM_OK;
}

// A prefetched sample set (enqueue_step with has_next) was drawn for
// (step + 1, seed, grid, frames) as they stood. Every call that changes one of
// them drops it, after ordering the context stream behind the sampling kernel
// (which may still be reading the grid / frame being replaced), so the next
// step re-samples from the new state (resumed objects continue the
// same sample stream; a new grid or keyframe is what the next step samples).
inline prenom_status drop_prefetch(prenom_object_s* o) {
  if (!o->sample_ready) return PRENOM_OK;
  CUDA_TRY(cudaStreamWaitEvent(o->ctx->stream, o->ev_sample, 0));
  o->sample_ready = false;
  o->prefetch_frame = -1;
  return PRENOM_OK;
}

inline void to_host_stats(const StepStatsDev& d, prenom_step_stats* s) {
  s->total = d.total;
  s->color_term = d.color;
  s->depth_term = d.depth;
  s->sigma_term = d.sigma;
  s->n_samples = (int64_t)d.n_samples;
  s->n_rays_escaped = d.escaped;
  s->frame_index = d.frame;
}

inline prenom_status set_frame_pixels(prenom_object_s* o, FrameDev* f, const float* rgb, const float* depth,
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
inline void init_frames(prenom_object_s* o, int n, const prenom_camera* cams, uint8_t inst, const prenom_pose* pose) {
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
