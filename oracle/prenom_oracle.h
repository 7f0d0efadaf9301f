/* TEST INFRASTRUCTURE ONLY -- the CPU oracle. Never linked into the product.
 *
 * Plain-C restatement of the reference hot path (/root/reference/proj/core)
 * with the reference's std::mt19937 consumers replaced by the Philox counter
 * layout documented in include/prenom/prenom_gpu.h. Every function cites the
 * reference file:line it follows. Pinned against the reference itself
 * (oracle/_ref/libnoma_ref.so, built from the untouched sources) in
 * tests/test_oracle_vs_ref.py: bit-exact where the reference arithmetic is
 * deterministic, identical-draw replay for the RNG consumers, tolerance for
 * the CDF (det_exp vs glibc exp) -- see DESIGN.md "Oracle".
 */
#ifndef PRENOM_ORACLE_H
#define PRENOM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "prenom/prenom_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* RNG (independent implementation; Random123 KAT in tests). */
void po_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
float po_u01(uint32_t x);
uint32_t po_pick(uint32_t x, uint32_t n);
void po_draw(uint64_t seed, uint32_t tag, int64_t step, uint32_t ray, uint32_t idx,
             uint32_t out[4]);

double po_det_exp(double x);

/* field.cpp */
int po_level_resolution(const prenom_field_arch* a, int level);
size_t po_hash_param_count(const prenom_field_arch* a);
size_t po_param_count(const prenom_field_arch* a);
uint32_t po_vertex_table_row(const prenom_field_arch* a, int level, uint32_t x, uint32_t y,
                             uint32_t z);
void po_hash_encode(const prenom_field_arch* a, const float* params, const float p[3],
                    float* feat, uint32_t* rows, float* w);
/* cache buffers (may be NULL): feat[L*F], pre[H*W], hidden[H*W], raw[4],
 * rows[L*8], w[L*8]. Returns 0, or 3 (NumericError) on non-finite output. */
int po_field_eval(const prenom_field_arch* a, const float* params, const float p[3],
                  float* sigma, float rgb[3], float* feat, float* pre, float* hidden, float* raw,
                  uint32_t* rows, float* w);
void po_field_backward(const prenom_field_arch* a, const float* params, const float p[3],
                       float d_sigma, const float d_rgb[3], float* grad);
void po_adam_step(size_t n, float* p, const float* g, float* m, float* v, int64_t* step,
                  float lr, float b1, float b2, float eps);

/* render.cpp / geom.hpp */
int po_ray_box(const float o[3], const float d[3], const float bmin[3], const float bmax[3],
               float* t_near, float* t_far);
int po_uniform_samples(const float o[3], const float d[3], const float bmin[3],
                       const float bmax[3], int n, float* depths, float* deltas, float* pos,
                       float* t_entry, float* t_exit);
void po_composite(int n, const float* sigma, const float* rgb, const float* deltas,
                  const float* depths, float color[3], float* depth, float* term_probs);
void po_composite_backward(int n, const float* sigma, const float* rgb, const float* deltas,
                           const float* depths, const float d_color[3], float d_depth,
                           float* d_sigma, float* d_rgb);
int po_batch_loss(int n_rays, const int* kind, const float* target_rgb,
                  const float* target_depth, const int* escaped, const int* offsets,
                  const float* deltas, const float* depths, const float* sigma,
                  const float* rgb, const float* bg_colors, float lambda_d, float lambda_sigma,
                  double terms[4], float* d_sigma, float* d_rgb, float* color_out,
                  float* depth_out);
void po_dilation_band(int w, int h, const uint8_t* mask, uint8_t value, int band_px,
                      uint8_t* out);
/* picks: n entries; first n_obj index the object-pixel list, the rest the band list. */
int po_generate_rays(const prenom_camera* cam, const float* rgb, const float* depth,
                     const uint8_t* mask, uint8_t inst, const prenom_pose* obj_pose, int n,
                     float bg_fraction, int band_px, const uint32_t* picks, float* origins,
                     float* dirs, int* kinds, float* target_rgb, float* target_depth,
                     int* pick_px, int* n_obj_out);
int po_generate_rays_philox(const prenom_camera* cam, const float* rgb, const float* depth,
                            const uint8_t* mask, uint8_t inst, const prenom_pose* obj_pose,
                            int n, float bg_fraction, int band_px, uint64_t seed, int64_t step,
                            float* origins, float* dirs, int* kinds, float* target_rgb,
                            float* target_depth, int* pick_px);

/* density_grid.cpp */
float po_trilerp(int R, const float* vals, const float p[3]);
int po_build_ray_cdf(int R, const float* vals, int n, const float* deltas, const float* pos,
                     float eps, float* term_probs, float* cdf);
void po_inverse_transform_sample(const float o[3], const float d[3], const float bmin[3],
                                 const float bmax[3], float t_entry, float t_exit, int n_c,
                                 const float* c_depths, const float* c_deltas, const float* cdf,
                                 int n, const float* uniforms, float* depths, float* deltas,
                                 float* pos);
int po_sample_ray(int R, const float* vals, const float o[3], const float d[3],
                  const float bmin[3], const float bmax[3], int n_c, int n_f, float eps,
                  const float* uniforms, float* depths, float* deltas, float* pos,
                  float* t_entry, float* t_exit);
int po_sample_ray_philox(int R, const float* vals, const float o[3], const float d[3],
                         const float bmin[3], const float bmax[3], int n_c, int n_f, float eps,
                         uint64_t seed, uint32_t tag, int64_t step, uint32_t ray,
                         float* depths, float* deltas, float* pos, float* t_entry,
                         float* t_exit);
int po_refresh_grid(const prenom_field_arch* a, const float* params, int R, float* out);

/* meta.cpp */
void po_reptile_update(size_t n, const float* meta, const float* adapted, float beta,
                       float* out);

/* train_track loop body (mapper.cpp:150-184) with Philox draws. */
typedef struct po_object po_object;
po_object* po_object_create(const prenom_field_arch* a, const float* theta, const float* grid,
                            int grid_res, uint64_t seed, const prenom_train_cfg* cfg,
                            const float bmin[3], const float bmax[3]);
void po_object_destroy(po_object* o);
int po_object_set_frames(po_object* o, int n, const prenom_camera* cams, const float* rgb,
                         const float* depth, const uint8_t* mask, uint8_t inst,
                         const prenom_pose* pose);
int po_object_train_step(po_object* o, int n_steps, prenom_step_stats* stats);
void po_object_get_params(const po_object* o, float* theta);
void po_object_get_grid(const po_object* o, float* grid);
int64_t po_object_step(const po_object* o);

#ifdef __cplusplus
}
#endif
#endif
