// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI shim over the *unmodified* reference sources (compiled in place from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/). It lets
// the Python tests and bench.py's CPU-baseline leg call the reference's own
// public API (noma::field_eval, noma::sample_ray, noma::batch_loss, ...)
// through ctypes. Nothing here re-implements reference arithmetic: every
// numeric result comes from the reference object code. The only fresh code
// is argument marshalling and `ref_train_object`, a restatement of the
// anonymous-namespace loop `train_track` (mapper.cpp:150-184) that calls the
// same public functions in the same order, because mapper.cpp cannot link
// here (it needs Eigen through icp_refine, mapper.cpp:552).
//
// RNG "replay" helpers: several reference functions consume a std::mt19937
// internally. To pin the Philox restatement in oracle/prenom_oracle.c, the
// shim replays the very same distribution calls on a copy of the generator
// and returns the drawn values, so the oracle can be fed identical draws.

#include <chrono>
#include <cstdio>
#include <string>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <vector>

#include "noma/density_grid.hpp"
#include "noma/errors.hpp"
#include "noma/field.hpp"
#include "noma/marching_cubes.hpp"
#include "noma/mesh.hpp"
#include "noma/meta.hpp"
#include "noma/metrics.hpp"
#include "noma/search.hpp"
#include "noma/prior_bundle.hpp"
#include "noma/shapes.hpp"
#include "noma/render.hpp"
#include "noma/task.hpp"

using namespace noma;

extern "C" {

struct RefArch {
  int hash_levels, features_per_level, log2_table_size, base_resolution;
  float per_level_scale;
  int hidden_width, hidden_layers, density_activation;
};

struct RefCamera {
  float fx, fy, cx, cy;
  int width, height;
  float R[9];
  float t[3];
};

struct RefTrainCfg {
  int rays_per_iter;
  float bg_fraction;
  int samples_per_ray;
  float lambda_d, lambda_sigma;
  int coarse_samples;
  float escape_eps;
  int grid_refresh_every;
  float eta;
  int prior_sampling;
};

}  // extern "C"

namespace {

FieldArch to_arch(const RefArch* a) {
  FieldArch r;
  r.hash_levels = a->hash_levels;
  r.features_per_level = a->features_per_level;
  r.log2_table_size = a->log2_table_size;
  r.base_resolution = a->base_resolution;
  r.per_level_scale = a->per_level_scale;
  r.hidden_width = a->hidden_width;
  r.hidden_layers = a->hidden_layers;
  r.density_activation =
      a->density_activation ? DensityActivation::kSoftplus : DensityActivation::kExpClamped;
  return r;
}

Vec3 v3(const float* p) { return {p[0], p[1], p[2]}; }
void put3(float* dst, const Vec3& v) {
  dst[0] = v.x;
  dst[1] = v.y;
  dst[2] = v.z;
}

Pose to_pose(const float* R, const float* t) {
  Pose p;
  for (int i = 0; i < 9; ++i) p.R.m[static_cast<std::size_t>(i)] = R[i];
  p.t = v3(t);
  return p;
}

Camera to_camera(const RefCamera* c) {
  Camera cam;
  cam.fx = c->fx;
  cam.fy = c->fy;
  cam.cx = c->cx;
  cam.cy = c->cy;
  cam.width = c->width;
  cam.height = c->height;
  cam.pose = to_pose(c->R, c->t);
  return cam;
}

ColorImage to_color(int w, int h, const float* rgb) {
  ColorImage img(w, h);
  for (std::size_t i = 0; i < img.data.size(); ++i) img.data[i] = v3(rgb + 3 * i);
  return img;
}

DepthImage to_depth(int w, int h, const float* d) {
  DepthImage img(w, h);
  std::memcpy(img.data.data(), d, img.data.size() * sizeof(float));
  return img;
}

MaskImage to_mask(int w, int h, const std::uint8_t* m) {
  MaskImage img(w, h);
  std::memcpy(img.data.data(), m, img.data.size());
  return img;
}

DensityGrid to_grid(int R, const float* vals) {
  DensityGrid g(R);
  std::memcpy(g.values.data(), vals, g.values.size() * sizeof(float));
  return g;
}

void put_set(const RaySampleSet& s, float* depths, float* deltas, float* pos, float* t_entry,
             float* t_exit) {
  for (std::size_t i = 0; i < s.size(); ++i) {
    if (depths) depths[i] = s.depths[i];
    if (deltas) deltas[i] = s.deltas[i];
    if (pos) put3(pos + 3 * i, s.positions[i]);
  }
  if (t_entry) *t_entry = s.t_entry;
  if (t_exit) *t_exit = s.t_exit;
}

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define REF_GUARD_BEGIN try {
#define REF_GUARD_END                                   \
  }                                                     \
  catch (const UsageError& e) { return fail(e, 1); }    \
  catch (const DataError& e) { return fail(e, 2); }     \
  catch (const NumericError& e) { return fail(e, 3); }  \
  catch (const std::exception& e) { return fail(e, 5); }

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

std::size_t ref_param_count(const RefArch* a) { return param_count(to_arch(a)); }
std::size_t ref_hash_param_count(const RefArch* a) { return hash_param_count(to_arch(a)); }
int ref_level_resolution(const RefArch* a, int level) {
  return level_resolution(to_arch(a), level);
}
std::uint32_t ref_vertex_table_row(const RefArch* a, int level, std::uint32_t x, std::uint32_t y,
                                   std::uint32_t z) {
  return vertex_table_row(to_arch(a), level, x, y, z);
}

void ref_init_params(const RefArch* a, std::uint64_t seed, float* out) {
  const ParamVector p = init_params(to_arch(a), seed);
  std::memcpy(out, p.data(), p.size() * sizeof(float));
}

// field.cpp:168-172, one call per point.
void ref_hash_encode(const RefArch* a, const float* params, int n, const float* xyz, float* out) {
  const FieldArch arch = to_arch(a);
  const ParamVector p(params, params + param_count(arch));
  const std::size_t nf = static_cast<std::size_t>(arch.hash_levels) * arch.features_per_level;
  for (int i = 0; i < n; ++i) {
    const auto f = hash_encode(arch, p, v3(xyz + 3 * i));
    std::memcpy(out + nf * i, f.data(), nf * sizeof(float));
  }
}

// field.cpp:174-217. Optional cache outputs (any may be NULL): features
// [n][L*F], pre/hidden [n][H*W], raw [n][4].
int ref_field_eval(const RefArch* a, const float* params, int n, const float* xyz, float* sigma,
                   float* rgb, float* feat, float* pre, float* hidden, float* raw) {
  REF_GUARD_BEGIN
  const FieldArch arch = to_arch(a);
  const ParamVector p(params, params + param_count(arch));
  const std::size_t nf = static_cast<std::size_t>(arch.hash_levels) * arch.features_per_level;
  const std::size_t nh = static_cast<std::size_t>(arch.hidden_layers) * arch.hidden_width;
  FieldEvalCache cache;
  for (int i = 0; i < n; ++i) {
    const FieldOutput o = field_eval(arch, p, v3(xyz + 3 * i), &cache);
    if (sigma) sigma[i] = o.sigma;
    if (rgb) put3(rgb + 3 * i, o.rgb);
    if (feat) std::memcpy(feat + nf * i, cache.features.data(), nf * sizeof(float));
    if (pre) std::memcpy(pre + nh * i, cache.pre.data(), nh * sizeof(float));
    if (hidden) std::memcpy(hidden + nh * i, cache.hidden.data(), nh * sizeof(float));
    if (raw) std::memcpy(raw + 4 * i, cache.raw.data(), 4 * sizeof(float));
  }
  return 0;
  REF_GUARD_END
}

// field.cpp:227-293: per point field_eval(&cache) then field_backward into
// one accumulated gradient (points in order).
int ref_field_backward(const RefArch* a, const float* params, int n, const float* xyz,
                       const float* d_sigma, const float* d_rgb, float* grad) {
  REF_GUARD_BEGIN
  const FieldArch arch = to_arch(a);
  const std::size_t P = param_count(arch);
  const ParamVector p(params, params + P);
  ParamVector g(grad, grad + P);
  FieldEvalCache cache;
  for (int i = 0; i < n; ++i) {
    field_eval(arch, p, v3(xyz + 3 * i), &cache);
    field_backward(arch, p, cache, d_sigma[i], v3(d_rgb + 3 * i), g);
  }
  std::memcpy(grad, g.data(), P * sizeof(float));
  return 0;
  REF_GUARD_END
}

// field.cpp:295-310; *step is the state's step counter (in/out).
int ref_adam_step(std::size_t n, float* params, const float* grads, float* m, float* v,
                  std::int64_t* step, float lr, float b1, float b2, float eps) {
  REF_GUARD_BEGIN
  AdamState st(n, lr);
  st.beta1 = b1;
  st.beta2 = b2;
  st.eps = eps;
  st.step = *step;
  std::memcpy(st.m.data(), m, n * sizeof(float));
  std::memcpy(st.v.data(), v, n * sizeof(float));
  ParamVector p(params, params + n);
  const ParamVector g(grads, grads + n);
  adam_step(st, p, g);
  std::memcpy(params, p.data(), n * sizeof(float));
  std::memcpy(m, st.m.data(), n * sizeof(float));
  std::memcpy(v, st.v.data(), n * sizeof(float));
  *step = st.step;
  return 0;
  REF_GUARD_END
}

// render.cpp:104-132. Returns 1 when escaped.
int ref_uniform_samples(const float* o, const float* d, const float* bmin, const float* bmax,
                        int n, float* depths, float* deltas, float* pos, float* t_entry,
                        float* t_exit) {
  ObjectRay ray;
  ray.origin = v3(o);
  ray.direction = v3(d);
  const RaySampleSet s = uniform_samples(ray, Box3{v3(bmin), v3(bmax)}, n);
  if (s.escaped) return 1;
  put_set(s, depths, deltas, pos, t_entry, t_exit);
  return 0;
}

float ref_trilerp(int R, const float* vals, const float* p) {
  return trilerp(to_grid(R, vals), v3(p));
}

// density_grid.cpp:43-70 over uniform_samples(ray, box, n_coarse).
// Returns 1 when escaped (coarse escape -> 2).
int ref_build_ray_cdf(int R, const float* vals, const float* o, const float* d, const float* bmin,
                      const float* bmax, int n_coarse, float eps, float* term_probs, float* cdf) {
  ObjectRay ray;
  ray.origin = v3(o);
  ray.direction = v3(d);
  const RaySampleSet coarse = uniform_samples(ray, Box3{v3(bmin), v3(bmax)}, n_coarse);
  if (coarse.escaped) return 2;
  const RayCdf c = build_ray_cdf(to_grid(R, vals), coarse, eps);
  for (int i = 0; i < n_coarse; ++i) term_probs[i] = c.term_probs[static_cast<std::size_t>(i)];
  if (c.escaped) return 1;
  for (int i = 0; i < n_coarse; ++i) cdf[i] = c.cdf[static_cast<std::size_t>(i)];
  return 0;
}

// density_grid.cpp:72-108 with the coarse set uniform_samples(ray, box,
// n_coarse) and an explicit cdf. `uniforms` (2*n) receives the two draws per
// sample in consumption order, replayed on a copy of mt19937(seed).
int ref_inverse_transform_sample(const float* o, const float* d, const float* bmin,
                                 const float* bmax, int n_coarse, const float* cdf, int n,
                                 std::uint32_t seed, float* depths, float* deltas, float* pos,
                                 float* uniforms) {
  REF_GUARD_BEGIN
  ObjectRay ray;
  ray.origin = v3(o);
  ray.direction = v3(d);
  const RaySampleSet coarse = uniform_samples(ray, Box3{v3(bmin), v3(bmax)}, n_coarse);
  if (coarse.escaped) return 2;
  std::mt19937 rng(seed);
  std::mt19937 replay = rng;
  const std::vector<float> c(cdf, cdf + n_coarse);
  const RaySampleSet fine = inverse_transform_sample(coarse, c, n, rng);
  put_set(fine, depths, deltas, pos, nullptr, nullptr);
  if (uniforms) {
    std::uniform_real_distribution<float> unit(0.f, 1.f);
    for (int s = 0; s < 2 * n; ++s) uniforms[s] = unit(replay);
  }
  return 0;
  REF_GUARD_END
}

// density_grid.cpp:110-117. Returns 1 when the final set is escaped.
int ref_sample_ray(int R, const float* vals, const float* o, const float* d, const float* bmin,
                   const float* bmax, int n_coarse, int n_fine, float eps, std::uint32_t seed,
                   float* depths, float* deltas, float* pos, float* t_entry, float* t_exit) {
  REF_GUARD_BEGIN
  ObjectRay ray;
  ray.origin = v3(o);
  ray.direction = v3(d);
  std::mt19937 rng(seed);
  const RaySampleSet s =
      sample_ray(to_grid(R, vals), ray, Box3{v3(bmin), v3(bmax)}, n_coarse, n_fine, eps, rng);
  if (s.escaped) return 1;
  put_set(s, depths, deltas, pos, t_entry, t_exit);
  return 0;
  REF_GUARD_END
}

// render.cpp:134-154.
void ref_composite(int n, const float* sigmas, const float* rgb, const float* deltas,
                   const float* depths, float* color, float* depth, float* term_probs) {
  std::vector<float> s(sigmas, sigmas + n), dl(deltas, deltas + n), dp(depths, depths + n);
  std::vector<Vec3> c(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) c[static_cast<std::size_t>(i)] = v3(rgb + 3 * i);
  const CompositeResult r = composite(s, c, dl, dp);
  put3(color, r.color);
  *depth = r.depth;
  if (term_probs)
    for (int i = 0; i < n; ++i) term_probs[i] = r.term_probs[static_cast<std::size_t>(i)];
}

// render.cpp:156-185 (fresh zero grads).
void ref_composite_backward(int n, const float* sigmas, const float* rgb, const float* deltas,
                            const float* depths, const float* d_color, float d_depth,
                            float* d_sigma, float* d_rgb) {
  std::vector<float> s(sigmas, sigmas + n), dl(deltas, deltas + n), dp(depths, depths + n);
  std::vector<Vec3> c(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) c[static_cast<std::size_t>(i)] = v3(rgb + 3 * i);
  std::vector<SampleGrad> g;
  composite_backward(s, c, dl, dp, v3(d_color), d_depth, g);
  for (int i = 0; i < n; ++i) {
    d_sigma[i] = g[static_cast<std::size_t>(i)].d_sigma;
    put3(d_rgb + 3 * i, g[static_cast<std::size_t>(i)].d_rgb);
  }
}

// render.cpp:187-243. Rays are flat: ray r owns samples [offsets[r],
// offsets[r+1]); a ray with escaped[r] != 0 or no samples is skipped.
// target_depth < 0 means "absent". terms = {total, color, depth, sigma}.
// bg_colors (3 per ray, NaN when not drawn) replays the colours drawn.
int ref_batch_loss(int n_rays, const int* kind, const float* target_rgb, const float* target_depth,
                   const int* escaped, const int* offsets, const float* deltas,
                   const float* depths, const float* sigma, const float* rgb, float lambda_d,
                   float lambda_sigma, std::uint32_t seed, double* terms, float* d_sigma,
                   float* d_rgb, float* bg_colors) {
  REF_GUARD_BEGIN
  std::vector<ObjectRay> rays(static_cast<std::size_t>(n_rays));
  std::vector<RaySampleSet> sets(static_cast<std::size_t>(n_rays));
  std::vector<std::vector<FieldOutput>> outs(static_cast<std::size_t>(n_rays));
  for (int r = 0; r < n_rays; ++r) {
    ObjectRay& ray = rays[static_cast<std::size_t>(r)];
    ray.kind = kind[r] ? RayKind::kBackground : RayKind::kObject;
    ray.target_color = v3(target_rgb + 3 * r);
    if (target_depth[r] >= 0.f) ray.target_depth = target_depth[r];
    RaySampleSet& s = sets[static_cast<std::size_t>(r)];
    s.escaped = escaped[r] != 0;
    for (int i = offsets[r]; i < offsets[r + 1]; ++i) {
      s.depths.push_back(depths[i]);
      s.deltas.push_back(deltas[i]);
      s.positions.push_back({});
      FieldOutput fo;
      fo.sigma = sigma[i];
      fo.rgb = v3(rgb + 3 * i);
      outs[static_cast<std::size_t>(r)].push_back(fo);
    }
  }
  std::mt19937 rng(seed);
  std::mt19937 replay = rng;
  LossWeights w;
  w.lambda_d = lambda_d;
  w.lambda_sigma = lambda_sigma;
  const LossResult L = batch_loss(rays, sets, outs, w, rng);
  terms[0] = L.total;
  terms[1] = L.color_term;
  terms[2] = L.depth_term;
  terms[3] = L.sigma_term;
  for (int r = 0; r < n_rays; ++r) {
    const auto& g = L.grads[static_cast<std::size_t>(r)];
    for (std::size_t i = 0; i < g.size(); ++i) {
      const int k = offsets[r] + static_cast<int>(i);
      d_sigma[k] = g[i].d_sigma;
      put3(d_rgb + 3 * k, g[i].d_rgb);
    }
  }
  if (bg_colors) {
    std::uniform_real_distribution<float> unit(0.f, 1.f);
    for (int r = 0; r < n_rays; ++r) {
      float* c = bg_colors + 3 * r;
      c[0] = c[1] = c[2] = std::nanf("");
      const RaySampleSet& s = sets[static_cast<std::size_t>(r)];
      if (s.escaped || s.size() == 0 || !kind[r]) continue;
      c[0] = unit(replay);
      c[1] = unit(replay);
      c[2] = unit(replay);
    }
  }
  return 0;
  REF_GUARD_END
}

// render.cpp:17-45.
void ref_dilation_band(int w, int h, const std::uint8_t* mask, std::uint8_t value, int band_px,
                       std::uint8_t* out) {
  const MaskImage band = dilation_band(to_mask(w, h, mask), value, band_px);
  std::memcpy(out, band.data.data(), band.data.size());
}

// render.cpp:47-102 with the picks replayed: pick_px[i] = x + W*y of ray i.
// target_depth: -1 when absent. kinds: 0 object, 1 background.
int ref_generate_rays(const RefCamera* cam, const float* rgb, const float* depth,
                      const std::uint8_t* mask, std::uint8_t inst, const float* obj_R,
                      const float* obj_t, int n, float bg_fraction, std::uint32_t seed,
                      int band_px, float* origins, float* dirs, int* kinds, float* target_rgb,
                      float* target_depth, int* pick_px) {
  REF_GUARD_BEGIN
  const Camera c = to_camera(cam);
  const int W = c.width, H = c.height;
  const MaskImage m = to_mask(W, H, mask);
  std::mt19937 rng(seed);
  std::mt19937 replay = rng;
  const auto rays = generate_rays(c, to_color(W, H, rgb), to_depth(W, H, depth), m, inst,
                                  to_pose(obj_R, obj_t), Vec3{1.f, 1.f, 1.f}, n, bg_fraction,
                                  rng, band_px);
  for (std::size_t i = 0; i < rays.size(); ++i) {
    put3(origins + 3 * i, rays[i].origin);
    put3(dirs + 3 * i, rays[i].direction);
    kinds[i] = rays[i].kind == RayKind::kBackground ? 1 : 0;
    put3(target_rgb + 3 * i, rays[i].target_color);
    target_depth[i] = rays[i].target_depth ? *rays[i].target_depth : -1.f;
  }
  if (pick_px) {
    std::vector<int> obj_px, bg_px;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        if (m.at(x, y) == inst) obj_px.push_back(x + W * y);
    const MaskImage band = dilation_band(m, inst, band_px);
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        if (band.at(x, y)) bg_px.push_back(x + W * y);
    int n_bg = bg_px.empty() ? 0 : static_cast<int>(std::lround(n * bg_fraction));
    n_bg = std::min(n_bg, n);
    const int n_obj = n - n_bg;
    std::uniform_int_distribution<std::size_t> po(0, obj_px.size() - 1);
    for (int i = 0; i < n_obj; ++i) pick_px[i] = obj_px[po(replay)];
    if (n_bg > 0) {
      std::uniform_int_distribution<std::size_t> pb(0, bg_px.size() - 1);
      for (int i = 0; i < n_bg; ++i) pick_px[n_obj + i] = bg_px[pb(replay)];
    }
  }
  return static_cast<int>(rays.size()) == n ? 0 : 5;
  REF_GUARD_END
}

// density_grid.cpp:119-132.
int ref_refresh_grid(const RefArch* a, const float* params, int R, float* out) {
  REF_GUARD_BEGIN
  const FieldArch arch = to_arch(a);
  const ParamVector p(params, params + param_count(arch));
  const DensityGrid g = refresh_grid(arch, p, R);
  std::memcpy(out, g.values.data(), g.values.size() * sizeof(float));
  return 0;
  REF_GUARD_END
}

// marching_cubes.cpp:125-180 (+ cleanup_mesh). The mesh is kept here until
// ref_mesh_get copies it out (two-call pattern: sizes first).
static thread_local Mesh g_ref_mesh;

int ref_marching_cubes(int R, const float* vals, float iso, std::int64_t* nv, std::int64_t* nt) {
  REF_GUARD_BEGIN
  DensityGrid g(R);
  std::memcpy(g.values.data(), vals, sizeof(float) * g.values.size());
  g_ref_mesh = marching_cubes(g, iso);
  *nv = (std::int64_t)g_ref_mesh.vertices.size();
  *nt = (std::int64_t)g_ref_mesh.triangles.size();
  return 0;
  REF_GUARD_END
}

void ref_mesh_get(float* verts, int* tris) {
  for (std::size_t i = 0; i < g_ref_mesh.vertices.size(); ++i) {
    verts[3 * i] = g_ref_mesh.vertices[i].x;
    verts[3 * i + 1] = g_ref_mesh.vertices[i].y;
    verts[3 * i + 2] = g_ref_mesh.vertices[i].z;
  }
  for (std::size_t i = 0; i < g_ref_mesh.triangles.size(); ++i)
    for (int k = 0; k < 3; ++k) tris[3 * i + k] = g_ref_mesh.triangles[i][k];
}

int ref_cube_case_triangles(int config, int* edges) {
  const auto& t = cube_case_triangles(config);
  for (std::size_t i = 0; i < t.size(); ++i)
    for (int k = 0; k < 3; ++k) edges[3 * i + k] = t[i][k];
  return (int)t.size();
}

float ref_choose_iso(int R, const float* vals, float floor_value) {
  DensityGrid g(R);
  std::memcpy(g.values.data(), vals, sizeof(float) * g.values.size());
  return choose_iso(g, floor_value);
}

// ---- prior bundles (prior_bundle.cpp:103-220; bake_prior density_grid.cpp:138-143)
// Genome fields as two arrays: gi = {hash_levels, log2_table_size,
// features_per_level, hidden_width, hidden_layers, meta_steps, inner_iters,
// density_activation}, gf = {eta, beta, per_level_scale, lambda_d, lambda_sigma}.
int ref_save_prior(const char* path, const char* category, const RefArch* a, const float* theta, int R,
                   const float* grid, std::int64_t nv, const float* verts, std::int64_t nt, const int* tris,
                   std::uint64_t search_seed, int population, int generations, const int* gi, const float* gf) {
  REF_GUARD_BEGIN
  PriorBundle b;
  b.category = category_from_string(category);
  b.arch = to_arch(a);
  b.theta.assign(theta, theta + param_count(b.arch));
  b.grid = DensityGrid(R);
  std::memcpy(b.grid.values.data(), grid, sizeof(float) * b.grid.values.size());
  b.mesh.vertices.resize((std::size_t)nv);
  for (std::int64_t i = 0; i < nv; ++i) b.mesh.vertices[i] = {verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]};
  b.mesh.triangles.resize((std::size_t)nt);
  for (std::int64_t i = 0; i < nt; ++i) b.mesh.triangles[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
  b.provenance.search_seed = search_seed;
  b.provenance.population = population;
  b.provenance.generations = generations;
  Genome& g = b.provenance.genome;
  g.hash_levels = gi[0], g.log2_table_size = gi[1], g.features_per_level = gi[2], g.hidden_width = gi[3];
  g.hidden_layers = gi[4], g.meta_steps = gi[5], g.inner_iters = gi[6];
  g.density_activation = gi[7] ? DensityActivation::kSoftplus : DensityActivation::kExpClamped;
  g.eta = gf[0], g.beta = gf[1], g.per_level_scale = gf[2], g.lambda_d = gf[3], g.lambda_sigma = gf[4];
  save_prior(b, path);
  return 0;
  REF_GUARD_END
}

// load_prior then prior_summary text (0 = ok; else the error class, message
// in ref_last_error). out receives the summary (truncated to cap).
int ref_prior_summary(const char* path, char* out, int cap) {
  REF_GUARD_BEGIN
  const std::string s = prior_summary(path);
  std::snprintf(out, (std::size_t)cap, "%s", s.c_str());
  return 0;
  REF_GUARD_END
}

// load_prior: sizes first (theta count, R, nv, nt), arrays when the pointers are non-NULL.
int ref_load_prior(const char* path, RefArch* a, std::int64_t* sizes, float* theta, float* grid, float* verts,
                   int* tris) {
  REF_GUARD_BEGIN
  const PriorBundle b = load_prior(path);
  a->hash_levels = b.arch.hash_levels, a->features_per_level = b.arch.features_per_level;
  a->log2_table_size = b.arch.log2_table_size, a->base_resolution = b.arch.base_resolution;
  a->per_level_scale = b.arch.per_level_scale, a->hidden_width = b.arch.hidden_width;
  a->hidden_layers = b.arch.hidden_layers;
  a->density_activation = b.arch.density_activation == DensityActivation::kSoftplus ? 1 : 0;
  sizes[0] = (std::int64_t)b.theta.size(), sizes[1] = b.grid.resolution;
  sizes[2] = (std::int64_t)b.mesh.vertices.size(), sizes[3] = (std::int64_t)b.mesh.triangles.size();
  if (theta) std::memcpy(theta, b.theta.data(), b.theta.size() * sizeof(float));
  if (grid) std::memcpy(grid, b.grid.values.data(), b.grid.values.size() * sizeof(float));
  if (verts)
    for (std::size_t i = 0; i < b.mesh.vertices.size(); ++i) {
      verts[3 * i] = b.mesh.vertices[i].x, verts[3 * i + 1] = b.mesh.vertices[i].y;
      verts[3 * i + 2] = b.mesh.vertices[i].z;
    }
  if (tris)
    for (std::size_t i = 0; i < b.mesh.triangles.size(); ++i)
      for (int k = 0; k < 3; ++k) tris[3 * i + k] = b.mesh.triangles[i][k];
  return 0;
  REF_GUARD_END
}

// bake_prior (density_grid.cpp:138-143): grid -> out_grid, mesh kept for ref_mesh_get.
int ref_bake_prior(const RefArch* a, const float* params, int R, float iso, float* out_grid, std::int64_t* nv,
                   std::int64_t* nt) {
  REF_GUARD_BEGIN
  const FieldArch arch = to_arch(a);
  const ParamVector p(params, params + param_count(arch));
  BakedPrior baked = bake_prior(arch, p, R, iso);
  std::memcpy(out_grid, baked.grid.values.data(), baked.grid.values.size() * sizeof(float));
  g_ref_mesh = std::move(baked.mesh);
  *nv = (std::int64_t)g_ref_mesh.vertices.size();
  *nt = (std::int64_t)g_ref_mesh.triangles.size();
  return 0;
  REF_GUARD_END
}

// ---- genome evaluation pieces (search.cpp:214-228; mesh.cpp:70-104; metrics.cpp:14-22)
double ref_iter_cost_model(const RefArch* a, int rays_per_iter, int samples_per_ray) {
  InnerOptions inner;
  inner.rays_per_iter = rays_per_iter;
  inner.samples_per_ray = samples_per_ray;
  return iter_cost_model(to_arch(a), inner);
}

static Mesh make_mesh(std::int64_t nv, const float* verts, std::int64_t nt, const int* tris) {
  Mesh m;
  m.vertices.resize((std::size_t)nv);
  for (std::int64_t i = 0; i < nv; ++i) m.vertices[i] = {verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]};
  m.triangles.resize((std::size_t)nt);
  for (std::int64_t i = 0; i < nt; ++i) m.triangles[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
  return m;
}

int ref_sample_surface(std::int64_t nv, const float* verts, std::int64_t nt, const int* tris, int n,
                       std::uint64_t seed, float* out) {
  REF_GUARD_BEGIN
  const auto pts = sample_surface(make_mesh(nv, verts, nt, tris), n, seed);
  for (std::size_t i = 0; i < pts.size(); ++i) {
    out[3 * i] = pts[i].x, out[3 * i + 1] = pts[i].y, out[3 * i + 2] = pts[i].z;
  }
  return 0;
  REF_GUARD_END
}

int ref_transformed(std::int64_t nv, const float* verts, const float* scale, const float* t, float* out) {
  REF_GUARD_BEGIN
  Mesh m = make_mesh(nv, verts, 0, nullptr);
  Pose pose{};
  pose.t = {t[0], t[1], t[2]};
  const Mesh r = transformed(m, {scale[0], scale[1], scale[2]}, pose);
  for (std::size_t i = 0; i < r.vertices.size(); ++i) {
    out[3 * i] = r.vertices[i].x, out[3 * i + 1] = r.vertices[i].y, out[3 * i + 2] = r.vertices[i].z;
  }
  return 0;
  REF_GUARD_END
}

int ref_chamfer(std::int64_t na, const float* a, std::int64_t nb, const float* b, double* out) {
  REF_GUARD_BEGIN
  std::vector<Vec3> pa((std::size_t)na), pb((std::size_t)nb);
  for (std::int64_t i = 0; i < na; ++i) pa[i] = {a[3 * i], a[3 * i + 1], a[3 * i + 2]};
  for (std::int64_t i = 0; i < nb; ++i) pb[i] = {b[3 * i], b[3 * i + 1], b[3 * i + 2]};
  *out = chamfer(pa, pb);
  return 0;
  REF_GUARD_END
}

// meta.cpp:83-92.
int ref_reptile_update(std::size_t n, const float* meta, const float* adapted, float beta,
                       float* out) {
  REF_GUARD_BEGIN
  const ParamVector a(meta, meta + n), b(adapted, adapted + n);
  const ParamVector r = reptile_update(a, b, beta);
  std::memcpy(out, r.data(), n * sizeof(float));
  return 0;
  REF_GUARD_END
}

// meta_train's task order (meta.cpp:101-110): `order` starts as iota and is
// reshuffled in place at every epoch by std::shuffle over
// std::mt19937(derive_seed(seed, 0xE9C6 + epoch)) -- this toolchain's
// libstdc++, as the reference binary would run it. derive_seed lives in
// meta.cpp's anonymous namespace (meta.cpp:14-20) and is restated here.
// out: n_epochs x n_tasks indices, epoch-major.
int ref_meta_task_order(std::size_t n_tasks, std::uint64_t seed, int n_epochs, std::int64_t* out) {
  REF_GUARD_BEGIN
  auto derive = [](std::uint64_t base, std::uint64_t salt) {
    std::uint64_t s = base * 0x9E3779B97F4A7C15ULL + salt * 0xBF58476D1CE4E5B9ULL + 1;
    s ^= s >> 31;
    s *= 0x94D049BB133111EBULL;
    s ^= s >> 29;
    return static_cast<std::uint32_t>(s ^ (s >> 32));
  };
  std::vector<std::size_t> order(n_tasks);
  for (std::size_t i = 0; i < n_tasks; ++i) order[i] = i;
  for (int e = 0; e < n_epochs; ++e) {
    std::mt19937 shuffle_rng(derive(seed, 0xE9C6ULL + static_cast<std::size_t>(e)));
    std::shuffle(order.begin(), order.end(), shuffle_rng);
    for (std::size_t i = 0; i < n_tasks; ++i) out[(std::size_t)e * n_tasks + i] = (std::int64_t)order[i];
  }
  return 0;
  REF_GUARD_END
}

}  // extern "C"

// Restatement of train_track (mapper.cpp:130-184) on the public API with
// the reference's own mt19937 stream, as a persistent handle so repeated
// steps time only reference compute (frames are converted once).
struct RefTrainer {
  FieldArch arch;
  ParamVector theta, grad;
  DensityGrid g;
  int grid_R = 0;
  AdamState adam;
  Box3 box;
  Pose pose;
  std::uint8_t inst = 1;
  std::vector<Camera> cameras;
  std::vector<ColorImage> rgbs;
  std::vector<DepthImage> depths;
  std::vector<MaskImage> masks;
  LossWeights weights;
  RefTrainCfg cfg;
  std::mt19937 rng;
  std::vector<RaySampleSet> samples;
  std::vector<std::vector<FieldOutput>> outputs;
  std::vector<std::vector<FieldEvalCache>> caches;
  int it = 0;
};

extern "C" {

void* ref_trainer_create(const RefArch* a, const float* params, int grid_R, const float* grid, int n_frames,
                         const RefCamera* cams, const float* rgb, const float* depth, const std::uint8_t* mask,
                         std::uint8_t inst, const float* obj_R, const float* obj_t, const float* bmin,
                         const float* bmax, const RefTrainCfg* cfg, std::uint32_t seed) {
  try {
    auto* t = new RefTrainer;
    t->arch = to_arch(a);
    const std::size_t P = param_count(t->arch);
    t->theta.assign(params, params + P);
    t->grad.assign(P, 0.f);
    t->grid_R = grid_R;
    t->g = grid ? to_grid(grid_R, grid) : DensityGrid(grid_R, 0.f);
    t->adam = AdamState(P, cfg->eta);
    t->box = Box3{v3(bmin), v3(bmax)};
    t->pose = to_pose(obj_R, obj_t);
    t->inst = inst;
    for (int f = 0; f < n_frames; ++f) {
      t->cameras.push_back(to_camera(cams + f));
      const int W = cams[f].width, H = cams[f].height;
      const std::size_t px = static_cast<std::size_t>(W) * H;
      t->rgbs.push_back(to_color(W, H, rgb + 3 * px * f));
      t->depths.push_back(to_depth(W, H, depth + px * f));
      t->masks.push_back(to_mask(W, H, mask + px * f));
    }
    t->weights.lambda_d = cfg->lambda_d;
    t->weights.lambda_sigma = cfg->lambda_sigma;
    t->cfg = *cfg;
    t->rng.seed(seed);
    return t;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_trainer_destroy(void* h) { delete static_cast<RefTrainer*>(h); }

// `iters` iterations of train_track's loop body (mapper.cpp:150-184).
// losses: iters x {total, color, depth, sigma} (may be NULL).
int ref_trainer_step(void* h, int iters, double* losses) {
  REF_GUARD_BEGIN
  RefTrainer& t = *static_cast<RefTrainer*>(h);
  std::uniform_int_distribution<std::size_t> pick_kf(0, t.cameras.size() - 1);
  for (int k = 0; k < iters; ++k) {
    const std::size_t fi = pick_kf(t.rng);
    const auto rays = generate_rays(t.cameras[fi], t.rgbs[fi], t.depths[fi], t.masks[fi], t.inst, t.pose,
                                    t.box.size(), t.cfg.rays_per_iter, t.cfg.bg_fraction, t.rng);
    t.samples.clear();
    t.outputs.clear();
    t.caches.clear();
    for (const ObjectRay& ray : rays) {
      RaySampleSet set = t.cfg.prior_sampling
                             ? sample_ray(t.g, ray, t.box, t.cfg.coarse_samples, t.cfg.samples_per_ray,
                                          t.cfg.escape_eps, t.rng)
                             : uniform_samples(ray, t.box, t.cfg.samples_per_ray);
      std::vector<FieldOutput> outs(set.size());
      std::vector<FieldEvalCache> cache(set.size());
      for (std::size_t i = 0; i < set.size(); ++i)
        outs[i] = field_eval(t.arch, t.theta, set.positions[i], &cache[i]);
      t.samples.push_back(std::move(set));
      t.outputs.push_back(std::move(outs));
      t.caches.push_back(std::move(cache));
    }
    const LossResult loss = batch_loss(rays, t.samples, t.outputs, t.weights, t.rng);
    std::fill(t.grad.begin(), t.grad.end(), 0.f);
    for (std::size_t r = 0; r < rays.size(); ++r)
      for (std::size_t i = 0; i < loss.grads[r].size(); ++i)
        field_backward(t.arch, t.theta, t.caches[r][i], loss.grads[r][i].d_sigma, loss.grads[r][i].d_rgb,
                       t.grad);
    adam_step(t.adam, t.theta, t.grad);
    if (losses) {
      losses[4 * k + 0] = loss.total;
      losses[4 * k + 1] = loss.color_term;
      losses[4 * k + 2] = loss.depth_term;
      losses[4 * k + 3] = loss.sigma_term;
    }
    t.it += 1;
    if (t.cfg.grid_refresh_every > 0 && t.it % t.cfg.grid_refresh_every == 0)
      t.g = refresh_grid(t.arch, t.theta, t.grid_R);
  }
  return 0;
  REF_GUARD_END
}

// Samples evaluated in the last step (for throughput accounting).
long long ref_trainer_last_samples(void* h) {
  const RefTrainer& t = *static_cast<RefTrainer*>(h);
  long long n = 0;
  for (const auto& s : t.samples) n += static_cast<long long>(s.size());
  return n;
}

void ref_trainer_get_params(void* h, float* out) {
  const RefTrainer& t = *static_cast<RefTrainer*>(h);
  std::memcpy(out, t.theta.data(), t.theta.size() * sizeof(float));
}

int ref_train_object(const RefArch* a, float* params, int grid_R, float* grid, int n_frames,
                     const RefCamera* cams, const float* rgb, const float* depth,
                     const std::uint8_t* mask, std::uint8_t inst, const float* obj_R,
                     const float* obj_t, const float* bmin, const float* bmax,
                     const RefTrainCfg* cfg, std::uint32_t seed, int iters, double* losses,
                     double* seconds) {
  const auto t0 = std::chrono::steady_clock::now();
  void* h = ref_trainer_create(a, params, grid_R, grid, n_frames, cams, rgb, depth, mask, inst, obj_R, obj_t,
                               bmin, bmax, cfg, seed);
  if (!h) return 5;
  const int st = ref_trainer_step(h, iters, losses);
  RefTrainer& t = *static_cast<RefTrainer*>(h);
  std::memcpy(params, t.theta.data(), t.theta.size() * sizeof(float));
  if (grid) std::memcpy(grid, t.g.values.data(), t.g.values.size() * sizeof(float));
  ref_trainer_destroy(h);
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return st;
}

// meta.cpp:24-81 (inner_adapt) on a one-task Task built from flat frames.
// theta_out receives the adapted parameters; losses (q) the batch losses.
int ref_inner_adapt(const RefArch* a, const float* theta, int n_frames, const RefCamera* cams,
                    const float* rgb, const float* depth, const std::uint8_t* mask,
                    const float* obj_R, const float* obj_t, const float* center,
                    const float* size, int q, float eta, std::uint32_t seed, int rays_per_iter,
                    float bg_fraction, int samples_per_ray, float lambda_d, float lambda_sigma,
                    float* theta_out, double* losses) {
  REF_GUARD_BEGIN
  const FieldArch arch = to_arch(a);
  const std::size_t P = param_count(arch);
  Task task;
  task.gt_pose = to_pose(obj_R, obj_t);
  task.gt_center = v3(center);
  task.gt_size = v3(size);
  for (int f = 0; f < n_frames; ++f) {
    const int W = cams[f].width, H = cams[f].height;
    const std::size_t px = static_cast<std::size_t>(W) * H;
    Frame fr;
    fr.rgb = to_color(W, H, rgb + 3 * px * f);
    fr.depth = to_depth(W, H, depth + px * f);
    fr.mask = to_mask(W, H, mask + px * f);
    task.frames.push_back(std::move(fr));
    task.cameras.push_back(to_camera(cams + f));
  }
  InnerOptions opt;
  opt.rays_per_iter = rays_per_iter;
  opt.bg_fraction = bg_fraction;
  opt.samples_per_ray = samples_per_ray;
  opt.weights.lambda_d = lambda_d;
  opt.weights.lambda_sigma = lambda_sigma;
  std::mt19937 rng(seed);
  std::vector<double> log;
  const ParamVector th(theta, theta + P);
  const ParamVector out = inner_adapt(th, arch, task, q, eta, rng, opt, &log);
  std::memcpy(theta_out, out.data(), P * sizeof(float));
  if (losses)
    for (std::size_t i = 0; i < log.size(); ++i) losses[i] = log[i];
  return 0;
  REF_GUARD_END
}

}  // extern "C"
