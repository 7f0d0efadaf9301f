// integration/gpu_trainer.cpp -- the reference-side adapter a maintainer would add to
// noma::core (core/src/gpu_trainer.cpp) to run the per-object train step on a B200
// through the C ABI of include/prenom/prenom_gpu.h. It replaces the body of the
// anonymous train_track (core/src/mapper.cpp:130-197): create from the category prior
// (mapper.cpp:133-137), iters_per_object steps with the every-m grid refresh
// (mapper.cpp:150-184), then the final refresh_grid + choose_iso + marching_cubes
// (mapper.cpp:186-187) and the world transform (mapper.cpp:188-194).
//
// Compiled against the reference's own headers by tests/test_integration.py
// (g++ -std=c++20 -fsyntax-only -I<reference>/core/include -Iinclude); linking needs
// libprenom_b200.so and noma::core (for noma::transformed).
#include <array>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "noma/errors.hpp"
#include "noma/mapper.hpp"
#include "noma/mesh.hpp"
#include "prenom/prenom_gpu.h"

namespace noma {
namespace gpu {

// mapper.cpp:20-26 lives in an anonymous namespace there; restated.
inline std::uint32_t mix_seed(std::uint64_t base, std::uint64_t salt) {
  std::uint64_t s = base * 0x9E3779B97F4A7C15ULL + salt * 0xC2B2AE3D27D4EB4FULL + 1;
  s ^= s >> 31;
  s *= 0x94D049BB133111EBULL;
  s ^= s >> 29;
  return static_cast<std::uint32_t>(s ^ (s >> 32));
}

// prenom_status -> the reference's exception classes (errors.hpp:9-24).
inline void check(prenom_status s) {
  if (s == PRENOM_OK) return;
  const std::string m = prenom_last_error();
  if (s == PRENOM_USAGE) throw UsageError(m);
  if (s == PRENOM_DATA) throw DataError(m);
  throw NumericError(m);  // PRENOM_NUMERIC, PRENOM_CUDA
}

inline prenom_field_arch to_c(const FieldArch& a) {
  prenom_field_arch c{};
  c.hash_levels = a.hash_levels;
  c.features_per_level = a.features_per_level;
  c.log2_table_size = a.log2_table_size;
  c.base_resolution = a.base_resolution;
  c.per_level_scale = a.per_level_scale;
  c.hidden_width = a.hidden_width;
  c.hidden_layers = a.hidden_layers;
  c.density_activation =
      a.density_activation == DensityActivation::kSoftplus ? PRENOM_ACT_SOFTPLUS : PRENOM_ACT_EXP_CLAMPED;
  return c;
}

inline prenom_train_cfg to_c(const MapperConfig& cfg, int mlp_precision) {
  prenom_train_cfg tc;
  prenom_default_train_cfg(&tc);
  tc.rays_per_iter = cfg.inner.rays_per_iter;
  tc.bg_fraction = cfg.inner.bg_fraction;
  tc.samples_per_ray = cfg.inner.samples_per_ray;
  tc.lambda_d = cfg.inner.weights.lambda_d;
  tc.lambda_sigma = cfg.inner.weights.lambda_sigma;
  tc.coarse_samples = cfg.coarse_samples;
  tc.escape_eps = cfg.escape_eps;
  tc.grid_refresh_every = cfg.grid_refresh_every;
  tc.eta = cfg.eta;
  tc.prior_sampling = cfg.prior_sampling ? 1 : 0;
  tc.mlp_precision = mlp_precision;
  return tc;
}

struct GpuTrainOutput {  // train_track's TrainOutput (mapper.cpp:123-128)
  Mesh mesh_world;
  int iterations = 0;
  std::string note;
  std::vector<prenom_step_stats> losses;
};

// RAII handle so a thrown reference error never leaks the device object.
struct Object {
  prenom_object_t h = nullptr;
  ~Object() {
    if (h) prenom_object_destroy(h);
  }
};

inline GpuTrainOutput train_track_gpu(prenom_ctx_t ctx, const ObjectTrack& track,
                                      const std::vector<SequenceFrame>& frames, const PriorBundle* prior,
                                      const MapperConfig& cfg, int mlp_precision = PRENOM_MLP_BF16X3) {
  if (track.keyframes.empty()) throw DataError("train_track: track has no keyframes");
  const FieldArch arch = prior ? prior->arch : FieldArch{};
  const prenom_field_arch ca = to_c(arch);
  const prenom_train_cfg tc = to_c(cfg, mlp_precision);
  const int R = prior ? prior->grid.resolution : cfg.grid_resolution;
  const Box3 box = track.object_box();
  const float bmin[3] = {box.min.x, box.min.y, box.min.z}, bmax[3] = {box.max.x, box.max.y, box.max.z};
  // theta: the prior's, else init_params on the device from the same seed role
  // (mapper.cpp:134-135: mix_seed(seed, 0x1217 + id)); the sampler's Philox key is
  // the role of train_track's mt19937(mix_seed(seed, 0x77AA + id)) (mapper.cpp:143)
  Object obj;
  check(prenom_object_create(ctx, &ca, prior ? prior->theta.data() : nullptr,
                             prior ? prior->grid.values.data() : nullptr, R,
                             mix_seed(cfg.seed, 0x77AAULL + static_cast<std::uint64_t>(track.id)), &tc, bmin, bmax,
                             &obj.h));
  // the track's keyframes as packed views (one camera each); the object's mask value is
  // remapped to 1 per keyframe (kf.instance_value differs between frames)
  std::vector<prenom_camera> cams;
  std::vector<float> rgb, depth;
  std::vector<std::uint8_t> mask;
  for (const KeyframeRef& kf : track.keyframes) {
    const SequenceFrame& f = frames.at(static_cast<std::size_t>(kf.frame_index));
    prenom_camera c{};
    c.fx = f.camera.fx;
    c.fy = f.camera.fy;
    c.cx = f.camera.cx;
    c.cy = f.camera.cy;
    c.width = f.camera.width;
    c.height = f.camera.height;
    for (int i = 0; i < 9; ++i) c.R[i] = f.camera.pose.R.m[static_cast<std::size_t>(i)];
    c.t[0] = f.camera.pose.t.x;
    c.t[1] = f.camera.pose.t.y;
    c.t[2] = f.camera.pose.t.z;
    cams.push_back(c);
    for (const Vec3& px : f.rgb.data) {
      rgb.push_back(px.x);
      rgb.push_back(px.y);
      rgb.push_back(px.z);
    }
    depth.insert(depth.end(), f.depth.data.begin(), f.depth.data.end());
    for (std::uint8_t m : f.mask.data) mask.push_back(m == kf.instance_value ? 1 : 0);
  }
  const Pose pose = track.obj_to_world();
  prenom_pose cp{};
  for (int i = 0; i < 9; ++i) cp.R[i] = pose.R.m[static_cast<std::size_t>(i)];
  cp.t[0] = pose.t.x;
  cp.t[1] = pose.t.y;
  cp.t[2] = pose.t.z;
  check(prenom_object_set_frames(obj.h, static_cast<int>(cams.size()), cams.data(), rgb.data(), depth.data(),
                                 mask.data(), 1, &cp));
  GpuTrainOutput out;
  out.losses.resize(static_cast<std::size_t>(cfg.iters_per_object));
  check(prenom_train_step(obj.h, cfg.iters_per_object, out.losses.data()));  // refresh every m inside
  out.iterations = cfg.iters_per_object;
  // mapper.cpp:186-187: refresh_grid, choose_iso (floor 5), marching_cubes -- on the device
  float iso = 0.f;
  std::int64_t nv = 0, nt = 0;
  check(prenom_extract_mesh(obj.h, R, NAN, 5.f, &iso, &nv, &nt));
  if (nt == 0) {
    out.note = "empty reconstruction";
    return out;
  }
  Mesh unit;
  std::vector<float> v(static_cast<std::size_t>(nv) * 3);
  std::vector<std::int32_t> t(static_cast<std::size_t>(nt) * 3);
  check(prenom_get_mesh(obj.h, v.data(), t.data()));
  for (std::int64_t i = 0; i < nv; ++i) unit.vertices.push_back({v[3 * i], v[3 * i + 1], v[3 * i + 2]});
  for (std::int64_t i = 0; i < nt; ++i) unit.triangles.push_back({t[3 * i], t[3 * i + 1], t[3 * i + 2]});
  // mapper.cpp:188-194
  const Mat3 Rw = pose.R;
  const Vec3 shift = pose.t - Rw * (track.size * 0.5f);
  out.mesh_world = transformed(unit, track.size, Pose{Rw, shift});
  return out;
}

}  // namespace gpu
}  // namespace noma
