// prenom_device.cuh -- device-side types and helpers shared by the sm_100a
// kernels of the per-object train step. Host code includes it for the
// descriptor structs and launch prototypes.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "prenom/prenom_detmath.h"
#include "prenom/prenom_gpu.h"

namespace prenom {

constexpr int kMaxLevels = 24;   // L <= 24 (BASELINE archs use 8..16)
constexpr int kMaxIn = 64;       // L*F <= 64
constexpr int kMaxWidth = 64;    // hidden width <= 64 (fp32 tile kernels)
constexpr int kMaxHidden = 3;    // hidden layers 1..3
constexpr int kTile = 128;       // samples per MLP tile (= UMMA M)
constexpr int kLd = kTile + 4;   // smem row stride (floats) of [dim][sample] tiles
constexpr uint32_t kPrime1 = 2654435761u, kPrime2 = 805459861u;  // field.cpp:20

// Field architecture + derived per-level constants (field.cpp:113-148),
// passed by value (constant bank) to every field kernel.
struct FieldDesc {
  int L, F, T, W, H, act;
  int in_dim;
  uint32_t row_mask;              // 2^T - 1
  long long rows;                 // 2^T
  long long hash_params;          // L*F*2^T = offset of the MLP block
  int res[kMaxLevels];            // level_resolution
  uint32_t dense_verts[kMaxLevels];  // res+1 when (res+1)^3 <= 2^T, else 0 (hashed)
  // MLP layer l (0..H, H = output layer): W at w_off[l], b at b_off[l],
  // relative to the MLP block start.
  int w_off[kMaxHidden + 1], b_off[kMaxHidden + 1];
  int mlp_params;
};

// Per-step statistics kept on the device (one slot per step of a call).
struct StepStatsDev {
  double total, color, depth, sigma;
  unsigned long long n_samples;
  int escaped;
  int frame;
  unsigned int blocks_done;  // k_composite's last block finishes the step's totals
  int pad_;
};

// Persistent-kernel tile scheduler counters [next tile, CTAs done, backward's next
// tile] of the forward: the last CTA to leave resets all three, so neither the
// forward nor the backward that follows it needs a memset node in front of it
// (a memset between the compositing kernel and the backward would keep the
// backward's prologue from overlapping the compositing kernel under PDL).
// (A self-reset inside the backward itself made k_bwd_tc 2.5x slower --
// unexplained, measured.)
__device__ __forceinline__ void tile_sched_exit(int* ctr) {
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      ctr[2] = 0;
    }
  }
}

// ---- programmatic dependent launch (PDL) between the step's kernels.
// A dependent kernel may start (prologue: smem carve, weight tiles, TMEM
// alloc, barriers) while its predecessor drains; griddepcontrol.wait then
// blocks until the predecessor grid has completed and its writes are
// visible, so every read of predecessor outputs sits after pdl_wait().
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
int num_sms();  // SMs of the current device (kernels_optim.cu)
bool pdl_enabled();  // PRENOM_NO_PDL=1 disables (A/B)

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}


// Ray-sample buffers of one batch: B rays x S slots.
struct SampleBufs {
  float4* pos_depth;  // [B*S] (x, y, z) in [0,1]^3 + depth (m)
  float* delta;       // [B*S]
  float4* target;     // [B] target rgb + target depth (-1 = absent)
  int* kind;          // [B] PRENOM_KIND_*
  int* count;         // [B] S or 0 (escaped)
  float* t_entry;     // [B] (debug)
  float* t_exit;      // [B] (debug)
  float* ray_o;       // [B][3] (debug, may be NULL)
  float* ray_d;       // [B][3] (debug, may be NULL)
  int* pick_px;       // [B] x + W*y (debug, frame mode, may be NULL)
};

// Source of the rays of one sampling launch.
struct RaySource {
  // mode 0: pixel picks from one frame (generate_rays); 1: explicit rays.
  int mode;
  // frame mode (render.cpp:47-102)
  const float* rgb;      // [H][W][3]
  const float* depth;    // [H][W]
  const int* obj_px;     // object pixel list (row-major scan order)
  const int* bg_px;      // band pixel list
  int n_obj_px, n_bg_px; // list sizes
  int n_obj;             // rays [0, n_obj) are object rays, the rest background
  int width;
  float fx, fy, cx, cy;
  float Rc[9];           // camera -> world rotation
  float Rt[9];           // world -> object rotation (obj pose transposed)
  float origin[3];       // world_to_obj.apply(camera.t), computed on the host
  // explicit mode
  const float* origins;  // [B][3]
  const float* dirs;     // [B][3]
};

struct SamplerCfg {
  int B, S;              // rays, fine samples per ray (n_fine)
  int prior;             // sample_ray (1) or uniform_samples (0)
  int n_coarse;
  float eps;
  int grid_res;
  const float* grid;     // R^3 x-fastest
  float bmin[3], bmax[3];
  uint64_t seed;
  uint32_t tag;          // PRENOM_TAG_FINE or PRENOM_TAG_RENDER
  uint32_t step;         // Philox c2
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ float clamp01(float v) { return v < 0.f ? 0.f : (1.f < v ? 1.f : v); }

__device__ __forceinline__ void philox_draw(uint64_t seed, uint32_t tag, uint32_t step,
                                            uint32_t ray, uint32_t idx, uint32_t out[4]) {
  const uint32_t ctr[4] = {idx, ray, step, tag};
  pdm_philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32), out);
}

// field.cpp:141-148 (bit-exact).
__device__ __forceinline__ uint32_t table_row(const FieldDesc& fd, int l, uint32_t x, uint32_t y,
                                              uint32_t z) {
  const uint32_t V = fd.dense_verts[l];
  if (V) return x + V * (y + V * z);
  return (x ^ (y * kPrime1) ^ (z * kPrime2)) & fd.row_mask;
}

// Level cell + fractional position (field.cpp:80-86), bit-exact.
struct LevelCell {
  int cx, cy, cz;
  float fx, fy, fz;
};

__device__ __forceinline__ LevelCell level_cell(int res, float px, float py, float pz) {
  LevelCell c;
  const float r = (float)res;
  const float gx = __fmul_rn(px, r), gy = __fmul_rn(py, r), gz = __fmul_rn(pz, r);
  c.cx = min((int)gx, res - 1);
  c.cy = min((int)gy, res - 1);
  c.cz = min((int)gz, res - 1);
  c.fx = __fsub_rn(gx, (float)c.cx);
  c.fy = __fsub_rn(gy, (float)c.cy);
  c.fz = __fsub_rn(gz, (float)c.cz);
  return c;
}

// The 8 corner rows of a level cell, factored: identical values to
// table_row(fd, l, cx + (k & 1), cy + (k >> 1 & 1), cz + (k >> 2 & 1)) (the
// dense index is affine mod 2^32; the hash XORs per-axis terms).
__device__ __forceinline__ void corner_rows(const FieldDesc& fd, int l, const LevelCell& c, uint32_t rows[8]) {
  const uint32_t V = fd.dense_verts[l];
  const uint32_t x = (uint32_t)c.cx, y = (uint32_t)c.cy, z = (uint32_t)c.cz;
  if (V) {
    const uint32_t b = x + V * (y + V * z), VV = V * V;
#pragma unroll
    for (int k = 0; k < 8; ++k) rows[k] = b + (k & 1 ? 1u : 0u) + (k & 2 ? V : 0u) + (k & 4 ? VV : 0u);
  } else {
    const uint32_t hy0 = y * kPrime1, hy1 = hy0 + kPrime1, hz0 = z * kPrime2, hz1 = hz0 + kPrime2;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      rows[k] = ((x + (k & 1 ? 1u : 0u)) ^ (k & 2 ? hy1 : hy0) ^ (k & 4 ? hz1 : hz0)) & fd.row_mask;
  }
}

// All 8 trilinear weights, same product order as corner_weight.
__device__ __forceinline__ void corner_weights(const LevelCell& c, float w[8]) {
  const float wx[2] = {__fsub_rn(1.f, c.fx), c.fx}, wy[2] = {__fsub_rn(1.f, c.fy), c.fy},
              wz[2] = {__fsub_rn(1.f, c.fz), c.fz};
  float wxy[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) wxy[k] = __fmul_rn(wx[k & 1], wy[k >> 1]);
#pragma unroll
  for (int k = 0; k < 8; ++k) w[k] = __fmul_rn(wxy[k & 3], wz[k >> 2]);
}

// Trilinear corner weight, same product order as field.cpp:88.
__device__ __forceinline__ float corner_weight(const LevelCell& c, int corner) {
  const float wx = (corner & 1) ? c.fx : __fsub_rn(1.f, c.fx);
  const float wy = (corner & 2) ? c.fy : __fsub_rn(1.f, c.fy);
  const float wz = (corner & 4) ? c.fz : __fsub_rn(1.f, c.fz);
  return __fmul_rn(__fmul_rn(wx, wy), wz);
}

// One level of encode_point (field.cpp:75-98); feat[F] accumulated in
// corner order with separate mul/add roundings (no FMA), skipping w == 0.
template <int F>
__device__ __forceinline__ void encode_level(const FieldDesc& fd, const float* __restrict__ params,
                                             int l, float px, float py, float pz, float* feat) {
  const LevelCell c = level_cell(fd.res[l], px, py, pz);
  const float* tab = params + (long long)l * F * fd.rows;
  float e[8][F];
  float w[8];
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    const uint32_t row = table_row(fd, l, (uint32_t)(c.cx + (corner & 1)),
                                   (uint32_t)(c.cy + ((corner >> 1) & 1)),
                                   (uint32_t)(c.cz + ((corner >> 2) & 1)));
    w[corner] = corner_weight(c, corner);
    if constexpr (F == 2) {
      const float2 v = __ldg(reinterpret_cast<const float2*>(tab + (size_t)row * 2));
      e[corner][0] = v.x;
      e[corner][1] = v.y;
    } else {
#pragma unroll
      for (int f = 0; f < F; ++f) e[corner][f] = __ldg(tab + (size_t)row * F + f);
    }
  }
#pragma unroll
  for (int f = 0; f < F; ++f) feat[f] = 0.f;
#pragma unroll
  for (int corner = 0; corner < 8; ++corner)
    if (w[corner] != 0.f) {
#pragma unroll
      for (int f = 0; f < F; ++f) feat[f] = __fadd_rn(feat[f], __fmul_rn(w[corner], e[corner][f]));
    }
}

// Two levels at once (16 independent corner gathers in flight), same
// per-level arithmetic and accumulation order as encode_level.
template <int F>
__device__ __forceinline__ void encode_level_pair(const FieldDesc& fd, const float* __restrict__ params, int la,
                                                  int lb, float px, float py, float pz, float* fa, float* fb) {
  const LevelCell ca = level_cell(fd.res[la], px, py, pz);
  const LevelCell cb = level_cell(fd.res[lb], px, py, pz);
  const float* ta = params + (long long)la * F * fd.rows;
  const float* tb = params + (long long)lb * F * fd.rows;
  float ea[8][F], eb[8][F], wa[8], wb[8];
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    const uint32_t ra = table_row(fd, la, (uint32_t)(ca.cx + (corner & 1)), (uint32_t)(ca.cy + ((corner >> 1) & 1)),
                                  (uint32_t)(ca.cz + ((corner >> 2) & 1)));
    const uint32_t rb = table_row(fd, lb, (uint32_t)(cb.cx + (corner & 1)), (uint32_t)(cb.cy + ((corner >> 1) & 1)),
                                  (uint32_t)(cb.cz + ((corner >> 2) & 1)));
    wa[corner] = corner_weight(ca, corner);
    wb[corner] = corner_weight(cb, corner);
    if constexpr (F == 2) {
      const float2 va = __ldg(reinterpret_cast<const float2*>(ta + (size_t)ra * 2));
      const float2 vb = __ldg(reinterpret_cast<const float2*>(tb + (size_t)rb * 2));
      ea[corner][0] = va.x;
      ea[corner][1] = va.y;
      eb[corner][0] = vb.x;
      eb[corner][1] = vb.y;
    } else {
#pragma unroll
      for (int f = 0; f < F; ++f) {
        ea[corner][f] = __ldg(ta + (size_t)ra * F + f);
        eb[corner][f] = __ldg(tb + (size_t)rb * F + f);
      }
    }
  }
#pragma unroll
  for (int f = 0; f < F; ++f) fa[f] = fb[f] = 0.f;
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    if (wa[corner] != 0.f)
#pragma unroll
      for (int f = 0; f < F; ++f) fa[f] = __fadd_rn(fa[f], __fmul_rn(wa[corner], ea[corner][f]));
    if (wb[corner] != 0.f)
#pragma unroll
      for (int f = 0; f < F; ++f) fb[f] = __fadd_rn(fb[f], __fmul_rn(wb[corner], eb[corner][f]));
  }
}

// Runtime-F variant (tiny test archs).
__device__ __forceinline__ void encode_level_rt(const FieldDesc& fd, const float* __restrict__ params,
                                                int l, float px, float py, float pz, float* feat) {
  const int F = fd.F;
  const LevelCell c = level_cell(fd.res[l], px, py, pz);
  const float* tab = params + (long long)l * F * fd.rows;
  for (int f = 0; f < F; ++f) feat[f] = 0.f;
  for (int corner = 0; corner < 8; ++corner) {
    const uint32_t row = table_row(fd, l, (uint32_t)(c.cx + (corner & 1)),
                                   (uint32_t)(c.cy + ((corner >> 1) & 1)),
                                   (uint32_t)(c.cz + ((corner >> 2) & 1)));
    const float w = corner_weight(c, corner);
    if (w == 0.f) continue;
    for (int f = 0; f < F; ++f)
      feat[f] = __fadd_rn(feat[f], __fmul_rn(w, __ldg(tab + (size_t)row * F + f)));
  }
}

// field.cpp:23-41. expf/log1pf are CUDA's (<= 2 ulp from glibc).
__device__ __forceinline__ float stable_sigmoid(float x) {
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}

__device__ __forceinline__ float density_forward(int act, float x) {
  if (act == PRENOM_ACT_EXP_CLAMPED) return fminf(expf(fminf(x, 10.f)), 1e4f);
  return x > 0.f ? x + log1pf(expf(-x)) : log1pf(expf(x));
}

__device__ __forceinline__ float density_derivative(int act, float x, float sigma) {
  if (act == PRENOM_ACT_EXP_CLAMPED) return sigma < 1e4f ? sigma : 0.f;
  return stable_sigmoid(x);
}

__device__ __forceinline__ bool all_finite4(float a, float b, float c, float d) {
  return isfinite(a) && isfinite(b) && isfinite(c) && isfinite(d);
}

// ------------------------------------------------------- launch wrappers
// (defined in the .cu files; all enqueue on `st` and return cudaGetLastError)
cudaError_t launch_sample(const RaySource& src, const SamplerCfg& cfg, SampleBufs out,
                          StepStatsDev* stats, cudaStream_t st);
// One object's sampling launch inside a grouped one (multi-object scheduler).
struct SampleJob {
  RaySource src;
  SamplerCfg cfg;
  SampleBufs out;
};
// jobs_dev[0..njobs) on the device; they share cfg0's B, S, prior and n_coarse
cudaError_t launch_sample_group(const SampleJob* jobs_dev, int njobs, const SamplerCfg& cfg0, cudaStream_t st);
cudaError_t launch_field_points(const FieldDesc& fd, const float* params, int n,
                                const float* xyz, float* sigma, float* rgb, float* raw,
                                float* features, int* flag, cudaStream_t st);
cudaError_t launch_field_fwd_train(const FieldDesc& fd, const float* params, int B, int S,
                                   const SampleBufs& sb, float* features_t, float4* out,
                                   int* flag, cudaStream_t st);
struct CompositeArgs {
  int B, S;
  const float4* pos_depth;
  const float* delta;
  const float4* target;
  const int* kind;
  const int* count;
  const float4* out;        // sigma, rgb per sample
  const float* bg_colors;   // [B][3] explicit, or NULL -> Philox TAG_BG
  uint64_t seed;
  uint32_t step;
  float lambda_d, lambda_sigma;
  float4* dout;             // d_sigma, d_rgb per sample (NULL: forward only)
  float* color_out;         // [B][3] or NULL
  float* depth_out;         // [B] or NULL
  StepStatsDev* stats;      // loss terms accumulated here (NULL: none)
  int* flag;                // numeric flag
  int frame;                // keyframe index recorded in stats
};
cudaError_t launch_composite(const CompositeArgs& a, cudaStream_t st);
// grouped: jobs_dev[0..njobs) (device), one per object, all with this B and S
cudaError_t launch_composite_group(const CompositeArgs* jobs_dev, int njobs, int B, int S, cudaStream_t st);
cudaError_t launch_mlp_bwd_train(const FieldDesc& fd, const float* params, float* grad, int B,
                                 int S, const int* count, const float* features_t,
                                 const float4* dout, float* dfeat_t, cudaStream_t st);
cudaError_t launch_encode_bwd(const FieldDesc& fd, const float* params, float* grad, int B, int S,
                              const int* count, const float4* pos_depth, const float* dfeat_t,
                              cudaStream_t st);
cudaError_t launch_adam(size_t n, float* p, float* g, float* m, float* v, float lr, float b1,
                        float b2, float eps, float c1, float c2, int zero_grad, cudaStream_t st);
// Adam with the backward's MLP-gradient reduction folded in: the MLP block's gradient is
// the sum of nparts per-CTA partials (part, [nparts][P_mlp]), summed by the first blocks
// of the launch while the others stream the hash table
cudaError_t launch_adam_fused(size_t n, size_t hash_params, int mlp_params, float* p, float* g, float* m, float* v,
                              float lr, float b1, float b2, float eps, float c1, float c2, const float* part,
                              int nparts, cudaStream_t st);
// grouped Adam (gradient zeroed): one job per object, blockIdx.y = job
struct AdamJob {
  size_t n;
  float *p, *g, *m, *v;
  float lr, b1, b2, eps, c1, c2;
};
cudaError_t launch_adam_group(const AdamJob* jobs_dev, int njobs, size_t n_max, cudaStream_t st);
cudaError_t launch_refresh_grid(const FieldDesc& fd, const float* params, int R, float* out,
                                int* flag, cudaStream_t st);
cudaError_t launch_init_params(const FieldDesc& fd, float* params, uint64_t seed, cudaStream_t st);
cudaError_t launch_philox(int n, const uint32_t* ctr_key, uint32_t* out, cudaStream_t st);
cudaError_t launch_reptile_delta(size_t n, const float* meta, const float* adapted, float* delta,
                                 cudaStream_t st);
cudaError_t launch_reptile_apply(size_t n, float* meta, const float* delta, float inv_n,
                                 float beta, cudaStream_t st);
cudaError_t launch_reptile_delta_sum(size_t n, const float* meta, const float* const* adapted_dev, int k, float* out,
                                     cudaStream_t st);
cudaError_t launch_reptile_update(size_t n, float* meta, const float* adapted, float beta, cudaStream_t st);
cudaError_t launch_l2_read(const float4* buf, size_t n4, int reps, float* sink, cudaStream_t st, float* ms);
// ---- isosurface (mesh.cu)
template <typename T>
struct MeshBuf {
  T* p = nullptr;
  size_t n = 0;
  MeshBuf() = default;
  MeshBuf(const MeshBuf&) = delete;
  MeshBuf& operator=(const MeshBuf&) = delete;
  ~MeshBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t ensure(size_t want) {
    if (want <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, (want ? want : 1) * sizeof(T));
    if (e == cudaSuccess) n = want ? want : 1;
    return e;
  }
};
// A mesh in the reference layout (mesh.hpp:12-17) on the device (per object).
struct McMesh {
  MeshBuf<float> verts;  // [n_vertices][3]
  MeshBuf<int> tris;     // [n_triangles][3]
  int64_t n_vertices = 0, n_triangles = 0;
  int R = 0;  // lattice resolution of the last extraction
};
// Extraction scratch, one per context (extractions are stream-ordered):
// the R^3 lattice, its max, and the count/emit/weld buffers (first_use is
// 3 R^3 keys, 200 MB at R = 256 -- allocated once, not per object).
struct McScratch {
  MeshBuf<uint32_t> block, tmp, keep, keep_off, first_use, mark, vid, total;
  MeshBuf<uint4> tri_keys, kept;
  MeshBuf<float> grid, gmax;
};
// ---- device-side data path (kernels_data.cu)
struct SynthBox {
  float lo[3], hi[3], albedo[3];
};
constexpr int kMaxSynthBoxes = 16;
struct SynthView {
  prenom_camera cam;  // camera -> world (scene frame)
  int view;
  int n_boxes;
  SynthBox boxes[kMaxSynthBoxes];
  float depth_noise, missing_frac;
  uint64_t seed;
};
struct FrameScratch {
  MeshBuf<uint8_t> mask, obj, rowdil;
  MeshBuf<uint32_t> f_obj, f_bg, o_obj, o_bg, tmp, total;
};
cudaError_t launch_synth_view(const SynthView& v, float* rgb, float* depth, uint8_t* mask, cudaStream_t st);
// dilation_band + object/band pixel lists (render.cpp:17-45, 57-66) of one
// device mask; synchronizes st (list sizes are read back)
cudaError_t build_pixel_lists(const uint8_t* d_mask, int W, int H, uint8_t inst, int band_px, FrameScratch& s,
                              MeshBuf<int>& obj_px, MeshBuf<int>& bg_px, int* n_obj, int* n_bg, cudaStream_t st);
int mc_case_triangles(int config, int* edges);  // host table (marching_cubes.cpp:24-107)
// exclusive scan of n u32 into out; *h_total = sum (host read, synchronizes st)
cudaError_t scan_exclusive_u32(const uint32_t* in, long long n, uint32_t* out, MeshBuf<uint32_t>& tmp,
                               uint32_t* d_total, uint32_t* h_total, cudaStream_t st);
cudaError_t launch_grid_max(const float* grid, long long n, float* d_out, cudaStream_t st);
cudaError_t launch_nearest_sq(int nq, const float* q, int np, const float* p, float* out, cudaStream_t st);
cudaError_t run_marching_cubes(const float* d_grid, int R, float iso, McScratch& m, McMesh& out, cudaStream_t st,
                               int* launches);

// bf16 tensor-core MLP path (kernels_tc.cu)
bool tc_supported(const FieldDesc& fd);
cudaError_t tc_bwd_trace(long long* mlp /* 64 x 16 */, long long* scat /* 64 x 4 */, long long* cta /* 1024 x 5 */);
void tc_set_min_tiles_per_cta(int v);  // persistent-grid hint for the calling host thread (multi-object)
bool tc_concurrent_objects();          // that hint is set: objects run concurrently on lane streams
size_t tc_feature_bytes(const FieldDesc& fd, long long n, int split);
// writes the constant ones / zero core matrices of a stored-feature buffer (once per allocation)
cudaError_t init_feature_tiles(const FieldDesc& fd, void* feat, size_t bytes, int split, cudaStream_t st);
// tile_ctr (dynamic tile scheduler): the forward uses [0], [1] and leaves [0..2]
// zeroed; the backward of the same step gets tile_ctr + 2 (zero on entry: the
// buffer is zeroed at allocation and after every forward)
cudaError_t launch_fwd_tc(const FieldDesc& fd, const float* params, long long n, int S, const int* count,
                          const float4* pos, void* feat_tiles, float4* out, int* flag, int* tile_ctr, int split,
                          cudaStream_t st);
// defer_nparts (optional): do not launch the MLP-gradient reduction; *defer_nparts =
// the number of per-CTA partials left in mlp_part (0: flushed with atomics), for
// launch_adam_fused to sum
cudaError_t launch_bwd_tc(const FieldDesc& fd, const float* params, float* grad, long long n, int S,
                          const int* count, const float4* pos, const void* feat_tiles, const float4* dout,
                          int* tile_ctr, int split, float* mlp_part, size_t part_cap, cudaStream_t st,
                          int* defer_nparts = nullptr);
// floats of per-CTA MLP-gradient partials launch_bwd_tc can use (else it flushes with atomics)
size_t tc_mlp_part_floats(const FieldDesc& fd);
// Grouped launches (multi-object scheduler): the objects of one architecture
// and samples-per-ray share ONE forward / backward launch over an object-major
// tile space; obj[j] covers tiles [tile0, tile0 + ceil(n / 128)).
struct TcObj {
  const float* params;
  float* grad;
  const int* count;
  const float4* pos;
  void* feat;          // stored feature tiles (tc_feature_bytes)
  float4* out;
  const float4* dout;
  float* part;         // per-CTA MLP-gradient partial slots (tc_mlp_part_floats)
  int* flag;
  long long n;         // samples (B * S)
  long long tile0;     // first tile in the launch
};
// ctr: [fwd next, fwd done] (self-resetting); ctr_bwd: [bwd next, part slots of
// obj 0..nobj-1], zeroed by the launcher. The tile space is object-major and
// claimed in order, so the CTAs work through the objects together (one or two
// objects' tables hot in L2 at a time; measured: giving each CTA a home object
// instead -- fewer weight reloads, every table hot at once -- is slower).
cudaError_t launch_fwd_tc_group(const FieldDesc& fd, const TcObj* objs_dev, int nobj, long long ntiles, int S,
                                int* ctr, int split, cudaStream_t st);
cudaError_t launch_bwd_tc_group(const FieldDesc& fd, const TcObj* objs_dev, int nobj, long long ntiles, int S,
                                int* ctr_bwd, int split, cudaStream_t st);
cudaError_t launch_umma_gemm(int M, int N, int K, int a_mn, int b_mn, const float* A, const float* B,
                             float* D, cudaStream_t st);

}  // namespace prenom
