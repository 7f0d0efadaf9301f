// kernels_data.cu -- the device-side data path:
//   * dilation_band + the object / band pixel lists of a keyframe
//     (render.cpp:17-45, 57-66), built on the device at upload instead of a
//     host BFS over every pixel;
//   * a synthetic RGB-D renderer of axis-aligned box unions straight into an
//     object's frame buffers (the device twin of scenes.box_union_scene; it
//     stands in for the reference's sdf_render.cpp at cfg5 scale, where
//     100 views x 512^2 x 256 objects cannot sensibly be made on the host).
//
// Band: the reference's 8-connected BFS from the instance pixels marks every
// pixel at Chebyshev distance 1..band_px (the BFS never leaves the image, and
// in a rectangle the 8-connected path length is the Chebyshev distance), i.e.
// band = dilate_box(mask, band_px) & !mask -- a separable max filter.
// Lists: indices in row-major scan order = stable stream compaction.
#include "prenom_device.cuh"

namespace prenom {
namespace {

__global__ void k_mask_flags(const uint8_t* mask, int npx, uint8_t inst, uint8_t* obj) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npx) obj[i] = mask[i] == inst ? 1 : 0;
}

// horizontal pass: rowdil[y][x] = any obj in row y within |dx| <= band
__global__ void k_dilate_rows(const uint8_t* obj, int W, int H, int band, uint8_t* rowdil) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W * H) return;
  const int x = i % W, y = i / W;
  const int x0 = max(0, x - band), x1 = min(W - 1, x + band);
  uint8_t any = 0;
  for (int xx = x0; xx <= x1; ++xx) any |= obj[y * W + xx];
  rowdil[i] = any;
}

// vertical pass + flags: bg = dilated & !obj
__global__ void k_band_flags(const uint8_t* obj, const uint8_t* rowdil, int W, int H, int band, uint32_t* f_obj,
                             uint32_t* f_bg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W * H) return;
  const int x = i % W, y = i / W;
  const int y0 = max(0, y - band), y1 = min(H - 1, y + band);
  uint8_t any = 0;
  for (int yy = y0; yy <= y1; ++yy) any |= rowdil[yy * W + x];
  const uint32_t o = obj[i];
  f_obj[i] = o;
  f_bg[i] = (band > 0 && any && !o) ? 1u : 0u;
}

__global__ void k_compact_idx(const uint32_t* flag, const uint32_t* off, int n, int* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) out[off[i]] = i;
}

// One view of a box union: pixel rays through Camera::pixel_direction
// (render.hpp:20-22), slab tests in the world frame, nearest hit wins;
// depth = hit distance (+ N(0, noise) from Philox TAG_SYNTH, c0 = pixel,
// c1 = view; out[0..1] Box-Muller, out[2] the missing-depth draw).
__global__ void k_synth_view(SynthView v, float* rgb, float* depth, uint8_t* mask) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int W = v.cam.width, H = v.cam.height;
  if (i >= W * H) return;
  const float u = (float)(i % W), vv = (float)(i / W);
  float dx = (u - v.cam.cx) / v.cam.fx, dy = (vv - v.cam.cy) / v.cam.fy, dz = 1.f;
  const float n = sqrtf(dx * dx + dy * dy + dz * dz);
  dx /= n;
  dy /= n;
  dz /= n;
  const float* R = v.cam.R;
  const float d[3] = {R[0] * dx + R[1] * dy + R[2] * dz, R[3] * dx + R[4] * dy + R[5] * dz,
                      R[6] * dx + R[7] * dy + R[8] * dz};
  const float* o = v.cam.t;
  float best = INFINITY;
  int hit_box = -1;
  for (int b = 0; b < v.n_boxes; ++b) {
    float t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float inv = 1.f / (fabsf(d[a]) < 1e-12f ? 1e-12f : d[a]);
      const float ta = (v.boxes[b].lo[a] - o[a]) * inv, tb = (v.boxes[b].hi[a] - o[a]) * inv;
      t0 = fmaxf(t0, fminf(ta, tb));
      t1 = fminf(t1, fmaxf(ta, tb));
    }
    if (t0 <= t1 && t1 > 0.f) {
      const float t = fmaxf(t0, 0.f);
      if (t < best) {
        best = t;
        hit_box = b;
      }
    }
  }
  float dep = 0.f;
  float c[3] = {0.f, 0.f, 0.f};
  if (hit_box >= 0) {
    dep = best;
    uint32_t x4[4];
    philox_draw(v.seed, PRENOM_TAG_SYNTH, 0u, (uint32_t)v.view, (uint32_t)i, x4);
    if (v.depth_noise > 0.f) {
      const float u1 = 1.f - pdm_u01(x4[0]), u2 = pdm_u01(x4[1]);  // u1 in (0, 1]
      dep += v.depth_noise * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
    }
    if (v.missing_frac > 0.f && pdm_u01(x4[2]) < v.missing_frac) dep = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = v.boxes[hit_box].albedo[a];
  }
  rgb[3 * (size_t)i + 0] = c[0];
  rgb[3 * (size_t)i + 1] = c[1];
  rgb[3 * (size_t)i + 2] = c[2];
  depth[i] = dep;
  mask[i] = hit_box >= 0 ? 1 : 0;
}

}  // namespace

cudaError_t launch_synth_view(const SynthView& v, float* rgb, float* depth, uint8_t* mask, cudaStream_t st) {
  const int npx = v.cam.width * v.cam.height;
  k_synth_view<<<(npx + 255) / 256, 256, 0, st>>>(v, rgb, depth, mask);
  return cudaGetLastError();
}

cudaError_t build_pixel_lists(const uint8_t* d_mask, int W, int H, uint8_t inst, int band_px, FrameScratch& s,
                              MeshBuf<int>& obj_px, MeshBuf<int>& bg_px, int* n_obj, int* n_bg, cudaStream_t st) {
  const int npx = W * H;
  cudaError_t e;
  if ((e = s.obj.ensure(npx)) != cudaSuccess || (e = s.rowdil.ensure(npx)) != cudaSuccess ||
      (e = s.f_obj.ensure(npx)) != cudaSuccess || (e = s.f_bg.ensure(npx)) != cudaSuccess ||
      (e = s.o_obj.ensure(npx)) != cudaSuccess || (e = s.o_bg.ensure(npx)) != cudaSuccess ||
      (e = s.total.ensure(1)) != cudaSuccess)
    return e;
  const int g = (npx + 255) / 256;
  k_mask_flags<<<g, 256, 0, st>>>(d_mask, npx, inst, s.obj.p);
  k_dilate_rows<<<g, 256, 0, st>>>(s.obj.p, W, H, band_px, s.rowdil.p);
  k_band_flags<<<g, 256, 0, st>>>(s.obj.p, s.rowdil.p, W, H, band_px, s.f_obj.p, s.f_bg.p);
  uint32_t no = 0, nb = 0;
  if ((e = scan_exclusive_u32(s.f_obj.p, npx, s.o_obj.p, s.tmp, s.total.p, &no, st)) != cudaSuccess) return e;
  if ((e = scan_exclusive_u32(s.f_bg.p, npx, s.o_bg.p, s.tmp, s.total.p, &nb, st)) != cudaSuccess) return e;
  if ((e = obj_px.ensure(no)) != cudaSuccess || (e = bg_px.ensure(nb)) != cudaSuccess) return e;
  k_compact_idx<<<g, 256, 0, st>>>(s.f_obj.p, s.o_obj.p, npx, obj_px.p);
  k_compact_idx<<<g, 256, 0, st>>>(s.f_bg.p, s.o_bg.p, npx, bg_px.p);
  *n_obj = (int)no;
  *n_bg = (int)nb;
  return cudaGetLastError();
}

}  // namespace prenom
