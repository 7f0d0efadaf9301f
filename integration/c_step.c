/* integration/c_step.c -- a plain C11 caller of include/prenom/prenom_gpu.h, linked against
 * libprenom_b200.so with no Python and no C++: context, an object created from device
 * init_params, synthetic box-union RGB-D views rendered on the device, N train steps
 * (prior-CDF sampler, tensor-core MLP), a density query, and the status/error mapping.
 * Prints the per-step loss and exits 0 when the loss went down.
 *   c_step [steps] [mlp_precision] */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "prenom/prenom_gpu.h"

#define TRY(x)                                                                     \
  do {                                                                             \
    prenom_status s_ = (x);                                                        \
    if (s_ != PRENOM_OK) {                                                         \
      fprintf(stderr, "%s failed (%d): %s\n", #x, (int)s_, prenom_last_error());   \
      return 10 + (int)s_;                                                         \
    }                                                                              \
  } while (0)

int main(int argc, char** argv) {
  const int steps = argc > 1 ? atoi(argv[1]) : 50;
  const int mlp = argc > 2 ? atoi(argv[2]) : PRENOM_MLP_BF16X3;
  prenom_ctx_t ctx;
  TRY(prenom_ctx_create(0, &ctx));
  prenom_field_arch a = {16, 2, 16, 16, 1.3195080f, 64, 2, PRENOM_ACT_EXP_CLAMPED};
  prenom_train_cfg cfg;
  prenom_default_train_cfg(&cfg);
  cfg.rays_per_iter = 1024;
  cfg.samples_per_ray = 48;
  cfg.prior_sampling = 0;
  cfg.grid_refresh_every = 0;
  cfg.mlp_precision = mlp;
  const float bmin[3] = {-0.5f, -0.5f, -0.5f}, bmax[3] = {0.5f, 0.5f, 0.5f};
  prenom_object_t obj;
  TRY(prenom_object_create(ctx, &a, NULL, NULL, 16, 7, &cfg, bmin, bmax, &obj));
  /* 12 views at 64^2 on a ring of radius 1.5 looking at the origin (camera -> world) */
  enum { NV = 12, RES = 64 };
  prenom_camera cams[NV];
  for (int i = 0; i < NV; ++i) {
    const float th = 6.2831853f * (float)i / NV, ph = 0.4f * (float)((i % 3) - 1);
    const float c[3] = {1.5f * cosf(th) * cosf(ph), 1.5f * sinf(th) * cosf(ph), 1.5f * sinf(ph)};
    float z[3] = {-c[0], -c[1], -c[2]}, up[3] = {0.f, 0.f, 1.f}, x[3], y[3];
    const float zn = sqrtf(z[0] * z[0] + z[1] * z[1] + z[2] * z[2]);
    for (int k = 0; k < 3; ++k) z[k] /= zn;
    x[0] = up[1] * z[2] - up[2] * z[1];  /* x = up x z */
    x[1] = up[2] * z[0] - up[0] * z[2];
    x[2] = up[0] * z[1] - up[1] * z[0];
    const float xn = sqrtf(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
    for (int k = 0; k < 3; ++k) x[k] /= xn;
    y[0] = z[1] * x[2] - z[2] * x[1];    /* y = z x x */
    y[1] = z[2] * x[0] - z[0] * x[2];
    y[2] = z[0] * x[1] - z[1] * x[0];
    prenom_camera* cm = &cams[i];
    cm->fx = cm->fy = 64.f;
    cm->cx = cm->cy = RES / 2.f;
    cm->width = cm->height = RES;
    for (int r = 0; r < 3; ++r) { /* columns = camera axes in world */
      cm->R[3 * r + 0] = x[r];
      cm->R[3 * r + 1] = y[r];
      cm->R[3 * r + 2] = z[r];
      cm->t[r] = c[r];
    }
  }
  prenom_box boxes[2] = {{{-0.2f, -0.15f, -0.1f}, {0.1f, 0.2f, 0.15f}, {0.8f, 0.3f, 0.2f}},
                         {{0.0f, -0.3f, -0.25f}, {0.25f, 0.0f, 0.05f}, {0.2f, 0.5f, 0.9f}}};
  prenom_pose pose = {{1, 0, 0, 0, 1, 0, 0, 0, 1}, {0, 0, 0}};
  TRY(prenom_object_synth_frames(obj, NV, cams, 2, boxes, 0.005f, 0.f, 11, &pose));
  prenom_step_stats* st = (prenom_step_stats*)calloc((size_t)steps, sizeof *st);
  TRY(prenom_train_step(obj, steps, st));
  double first = 0, last = 0;
  for (int i = 0; i < steps; ++i) {
    if (i < 5) first += st[i].total / 5;
    if (i >= steps - 5) last += st[i].total / 5;
  }
  printf("{\"steps\": %d, \"mlp_precision\": %d, \"loss_first5\": %.6f, \"loss_last5\": %.6f, \"samples\": %lld}\n", steps,
         mlp, first, last, (long long)st[steps - 1].n_samples);
  float* q = (float*)malloc(sizeof(float) * 32 * 32 * 32);
  TRY(prenom_density_query(obj, 32, q, 0));
  /* the reference's error classes come back as status codes */
  if (prenom_train_step(obj, 0, NULL) != PRENOM_USAGE) return 3;
  free(q);
  free(st);
  TRY(prenom_object_destroy(obj));
  TRY(prenom_ctx_destroy(ctx));
  return last < first ? 0 : 4;
}
