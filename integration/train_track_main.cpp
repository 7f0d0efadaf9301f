// integration/train_track_main.cpp -- drives noma::gpu::train_track_gpu (gpu_trainer.cpp)
// with the reference's own types: a track (ObjectTrack + KeyframeRefs), SequenceFrames
// (Camera, ColorImage, DepthImage, MaskImage), MapperConfig, and no prior. The views come
// from a binary scene file (written by tests/test_integration.py):
//   int32 n, W, H, inst; float32 box_size[3]; float32 pose_R[9], pose_t[3];
//   per view: float32 fx, fy, cx, cy, R[9], t[3]; then rgb [n][H][W][3] f32,
//   depth [n][H][W] f32, mask [n][H][W] u8.
// Prints one JSON line: per-step losses, mesh size, note.
// Usage: train_track_main <scene.bin> <iters> <rays> <samples> <seed> <track_id> <mlp_precision>
#include <cstdio>
#include <cstdlib>
#include <fstream>

#include "gpu_trainer.cpp"

int main(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s scene.bin iters rays samples seed track_id mlp_precision\n", argv[0]);
    return 1;
  }
  std::ifstream in(argv[1], std::ios::binary);
  auto rd = [&](void* p, std::size_t n) {
    in.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
    if (!in) throw noma::DataError("short scene file");
  };
  try {
    std::int32_t hdr[4];
    rd(hdr, sizeof hdr);
    const int n = hdr[0], W = hdr[1], H = hdr[2];
    const std::uint8_t inst = static_cast<std::uint8_t>(hdr[3]);
    float size[3], pr[9], pt[3];
    rd(size, sizeof size);
    rd(pr, sizeof pr);
    rd(pt, sizeof pt);
    std::vector<noma::SequenceFrame> frames(static_cast<std::size_t>(n));
    for (auto& f : frames) {
      float c[16];
      rd(c, sizeof c);
      f.camera.fx = c[0];
      f.camera.fy = c[1];
      f.camera.cx = c[2];
      f.camera.cy = c[3];
      f.camera.width = W;
      f.camera.height = H;
      for (int i = 0; i < 9; ++i) f.camera.pose.R.m[static_cast<std::size_t>(i)] = c[4 + i];
      f.camera.pose.t = {c[13], c[14], c[15]};
    }
    const std::size_t npx = static_cast<std::size_t>(W) * H;
    std::vector<float> buf(npx * 3);
    for (auto& f : frames) {
      rd(buf.data(), npx * 3 * sizeof(float));
      f.rgb = noma::ColorImage(W, H);
      for (std::size_t i = 0; i < npx; ++i) f.rgb.data[i] = {buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]};
    }
    for (auto& f : frames) {
      f.depth = noma::DepthImage(W, H, 0.f);
      rd(f.depth.data.data(), npx * sizeof(float));
    }
    for (auto& f : frames) {
      f.mask = noma::MaskImage(W, H, 0);
      rd(f.mask.data.data(), npx);
    }
    // the track: pose = rot_z(yaw) + position (mapper.hpp ObjectTrack::obj_to_world); the
    // scene file's object pose is given as R, t -- the adapter reads the track's pose, so
    // the scenes used here have yaw 0 (R = I) and position t
    noma::ObjectTrack track;
    track.id = std::atoi(argv[6]);
    track.position = {pt[0], pt[1], pt[2]};
    track.yaw = 0.f;
    track.size = {size[0], size[1], size[2]};
    for (int i = 0; i < n; ++i) {
      noma::KeyframeRef kf;
      kf.frame_index = i;
      kf.instance_value = inst;
      track.keyframes.push_back(kf);
    }
    noma::MapperConfig cfg;
    cfg.iters_per_object = std::atoi(argv[2]);
    cfg.inner.rays_per_iter = std::atoi(argv[3]);
    cfg.inner.samples_per_ray = std::atoi(argv[4]);
    cfg.seed = std::strtoull(argv[5], nullptr, 10);
    cfg.prior_sampling = false;  // no prior: the reference trains on midpoints over a zero grid
    cfg.grid_refresh_every = 0;
    prenom_ctx_t ctx;
    noma::gpu::check(prenom_ctx_create(0, &ctx));
    const auto out = noma::gpu::train_track_gpu(ctx, track, frames, nullptr, cfg, std::atoi(argv[7]));
    std::printf("{\"iterations\": %d, \"n_vertices\": %zu, \"n_triangles\": %zu, \"note\": \"%s\", \"losses\": [",
                out.iterations, out.mesh_world.vertices.size(), out.mesh_world.triangles.size(), out.note.c_str());
    for (std::size_t i = 0; i < out.losses.size(); ++i)
      std::printf("%s%.17g", i ? ", " : "", out.losses[i].total);
    std::printf("]}\n");
    prenom_ctx_destroy(ctx);
  } catch (const noma::UsageError& e) {
    std::fprintf(stderr, "usage error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
