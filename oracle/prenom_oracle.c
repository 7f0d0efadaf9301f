/* TEST INFRASTRUCTURE ONLY -- CPU oracle (see prenom_oracle.h).
 *
 * Compile with -ffp-contract=off and without -ffast-math (oracle/Makefile):
 * every float/double expression below is evaluated as the same sequence of
 * IEEE operations the reference performs (reference compiled for x86-64
 * without FMA), which is what makes the bit-exact comparisons meaningful.
 */
#include "prenom_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "prenom/prenom_detmath.h"

/* ------------------------------------------------------------------ RNG */

void po_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t x[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  uint32_t k[2] = {key[0], key[1]};
  for (int r = 0; r < 10; ++r) {
    const uint64_t a = (uint64_t)0xD2511F53u * x[0];
    const uint64_t b = (uint64_t)0xCD9E8D57u * x[2];
    const uint32_t y0 = (uint32_t)(b >> 32) ^ x[1] ^ k[0];
    const uint32_t y1 = (uint32_t)b;
    const uint32_t y2 = (uint32_t)(a >> 32) ^ x[3] ^ k[1];
    const uint32_t y3 = (uint32_t)a;
    x[0] = y0;
    x[1] = y1;
    x[2] = y2;
    x[3] = y3;
    k[0] += 0x9E3779B9u;
    k[1] += 0xBB67AE85u;
  }
  memcpy(out, x, sizeof x);
}

float po_u01(uint32_t x) { return (float)(x >> 8) * (1.0f / 16777216.0f); }

uint32_t po_pick(uint32_t x, uint32_t n) { return (uint32_t)(((uint64_t)x * n) >> 32); }

void po_draw(uint64_t seed, uint32_t tag, int64_t step, uint32_t ray, uint32_t idx,
             uint32_t out[4]) {
  const uint32_t ctr[4] = {idx, ray, (uint32_t)step, tag};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  po_philox(ctr, key, out);
}

double po_det_exp(double x) { return pdm_det_exp(x); }

/* --------------------------------------------------------------- helpers */

static float clampf01(float v) { return v < 0.f ? 0.f : (1.f < v ? 1.f : v); } /* std::clamp */

/* ---------------------------------------------------------------- field */

/* field.cpp:113-116 */
int po_level_resolution(const prenom_field_arch* a, int level) {
  const double r = a->base_resolution * pow((double)a->per_level_scale, level);
  const int ir = (int)r;
  return ir > 1 ? ir : 1;
}

/* field.cpp:122-139 */
size_t po_hash_param_count(const prenom_field_arch* a) {
  return (size_t)a->hash_levels * a->features_per_level * ((size_t)1 << a->log2_table_size);
}

size_t po_param_count(const prenom_field_arch* a) {
  size_t n = 0;
  int in = a->hash_levels * a->features_per_level;
  for (int l = 0; l < a->hidden_layers; ++l) {
    n += (size_t)a->hidden_width * in + a->hidden_width;
    in = a->hidden_width;
  }
  n += (size_t)4 * in + 4;
  return po_hash_param_count(a) + n;
}

/* field.cpp:141-148 */
uint32_t po_vertex_table_row(const prenom_field_arch* a, int level, uint32_t x, uint32_t y,
                             uint32_t z) {
  const uint32_t verts = (uint32_t)po_level_resolution(a, level) + 1u;
  const uint64_t dense = (uint64_t)verts * verts * verts;
  const uint64_t rows = (uint64_t)1 << a->log2_table_size;
  if (dense <= rows) return x + verts * (y + verts * z);
  const uint32_t h = (x * 1u) ^ (y * 2654435761u) ^ (z * 805459861u);
  return h & (uint32_t)(rows - 1u);
}

/* field.cpp:64-99 (encode_point) */
void po_hash_encode(const prenom_field_arch* a, const float* params, const float p_in[3],
                    float* feat, uint32_t* rows_out, float* w_out) {
  const int L = a->hash_levels, F = a->features_per_level;
  const size_t rows = (size_t)1 << a->log2_table_size;
  for (int i = 0; i < L * F; ++i) feat[i] = 0.f;
  const float px = clampf01(p_in[0]), py = clampf01(p_in[1]), pz = clampf01(p_in[2]);
  for (int l = 0; l < L; ++l) {
    const int res = po_level_resolution(a, l);
    const size_t level_off = (size_t)l * F * rows;
    const float gx = px * (float)res, gy = py * (float)res, gz = pz * (float)res;
    int cx = (int)gx, cy = (int)gy, cz = (int)gz;
    if (cx > res - 1) cx = res - 1;
    if (cy > res - 1) cy = res - 1;
    if (cz > res - 1) cz = res - 1;
    const float fx = gx - (float)cx, fy = gy - (float)cy, fz = gz - (float)cz;
    for (int corner = 0; corner < 8; ++corner) {
      const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
      const float w = (dx ? fx : 1.f - fx) * (dy ? fy : 1.f - fy) * (dz ? fz : 1.f - fz);
      const uint32_t row = po_vertex_table_row(a, l, (uint32_t)(cx + dx), (uint32_t)(cy + dy),
                                               (uint32_t)(cz + dz));
      if (rows_out) rows_out[l * 8 + corner] = row;
      if (w_out) w_out[l * 8 + corner] = w;
      if (w == 0.f) continue;
      const float* entry = params + level_off + (size_t)row * F;
      for (int f = 0; f < F; ++f) feat[l * F + f] += w * entry[f];
    }
  }
}

/* field.cpp:23-41 */
static float stable_sigmoid(float x) {
  if (x >= 0.f) {
    const float e = expf(-x);
    return 1.f / (1.f + e);
  }
  const float e = expf(x);
  return e / (1.f + e);
}

static float density_forward(int act, float x) {
  if (act == PRENOM_ACT_EXP_CLAMPED) return fminf(expf(fminf(x, 10.f)), 1e4f);
  return x > 0.f ? x + log1pf(expf(-x)) : log1pf(expf(x));
}

static float density_derivative(int act, float x, float sigma) {
  if (act == PRENOM_ACT_EXP_CLAMPED) return sigma < 1e4f ? sigma : 0.f;
  return stable_sigmoid(x);
}

/* field.cpp:48-62: offsets of layer l's W and b (l == H is the output layer). */
static void mlp_offsets(const prenom_field_arch* a, int layer, size_t* w_off, size_t* b_off,
                        int* in_dim, int* out_dim) {
  size_t off = po_hash_param_count(a);
  int in = a->hash_levels * a->features_per_level;
  for (int l = 0; l < layer; ++l) {
    off += (size_t)a->hidden_width * in + a->hidden_width;
    in = a->hidden_width;
  }
  const int out = layer < a->hidden_layers ? a->hidden_width : 4;
  *w_off = off;
  *b_off = off + (size_t)out * in;
  *in_dim = in;
  *out_dim = out;
}

/* field.cpp:174-217 */
int po_field_eval(const prenom_field_arch* a, const float* params, const float p[3],
                  float* sigma, float rgb[3], float* feat_out, float* pre_out,
                  float* hidden_out, float* raw_out, uint32_t* rows, float* w) {
  const int L = a->hash_levels, F = a->features_per_level, W = a->hidden_width,
            H = a->hidden_layers;
  float* feat = feat_out ? feat_out : (float*)malloc(sizeof(float) * (size_t)(L * F));
  float* pre = pre_out ? pre_out : (float*)malloc(sizeof(float) * (size_t)(H * W));
  float* hid = hidden_out ? hidden_out : (float*)malloc(sizeof(float) * (size_t)(H * W));
  po_hash_encode(a, params, p, feat, rows, w);
  const float* in = feat;
  for (int l = 0; l < H; ++l) {
    size_t wo, bo;
    int ni, no;
    mlp_offsets(a, l, &wo, &bo, &ni, &no);
    float* pr = pre + (size_t)l * W;
    float* ac = hid + (size_t)l * W;
    for (int o = 0; o < no; ++o) {
      const float* wrow = params + wo + (size_t)o * ni;
      float s = params[bo + o];
      for (int i = 0; i < ni; ++i) s += wrow[i] * in[i];
      pr[o] = s;
      ac[o] = s > 0.f ? s : 0.f;
    }
    in = ac;
  }
  float raw[4];
  {
    size_t wo, bo;
    int ni, no;
    mlp_offsets(a, H, &wo, &bo, &ni, &no);
    for (int o = 0; o < 4; ++o) {
      const float* wrow = params + wo + (size_t)o * ni;
      float s = params[bo + o];
      for (int i = 0; i < ni; ++i) s += wrow[i] * in[i];
      raw[o] = s;
    }
  }
  if (raw_out) memcpy(raw_out, raw, sizeof raw);
  const float sg = density_forward(a->density_activation, raw[0]);
  const float r0 = stable_sigmoid(raw[1]), r1 = stable_sigmoid(raw[2]),
              r2 = stable_sigmoid(raw[3]);
  if (sigma) *sigma = sg;
  if (rgb) {
    rgb[0] = r0;
    rgb[1] = r1;
    rgb[2] = r2;
  }
  if (!feat_out) free(feat);
  if (!pre_out) free(pre);
  if (!hidden_out) free(hid);
  if (!isfinite(sg) || !isfinite(r0) || !isfinite(r1) || !isfinite(r2)) return 3;
  return 0;
}

/* field.cpp:227-293 (recomputes the forward cache for the point). */
void po_field_backward(const prenom_field_arch* a, const float* params, const float p[3],
                       float d_sigma, const float d_rgb[3], float* grad) {
  const int L = a->hash_levels, F = a->features_per_level, W = a->hidden_width,
            H = a->hidden_layers;
  const size_t rows_n = (size_t)1 << a->log2_table_size;
  float* feat = (float*)malloc(sizeof(float) * (size_t)(L * F));
  float* pre = (float*)malloc(sizeof(float) * (size_t)(H * W + 1));
  float* hid = (float*)malloc(sizeof(float) * (size_t)(H * W + 1));
  uint32_t* rows = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(L * 8));
  float* cw = (float*)malloc(sizeof(float) * (size_t)(L * 8));
  const int maxd = (L * F > W ? L * F : W);
  float* d_in = (float*)calloc((size_t)maxd, sizeof(float));
  float* d_prev = (float*)calloc((size_t)maxd, sizeof(float));
  float raw[4], sg, rgb[3];
  po_field_eval(a, params, p, &sg, rgb, feat, pre, hid, raw, rows, cw);

  float g_raw[4];
  g_raw[0] = d_sigma * density_derivative(a->density_activation, raw[0], sg);
  for (int k = 0; k < 3; ++k) g_raw[k + 1] = d_rgb[k] * rgb[k] * (1.f - rgb[k]);

  size_t wo, bo;
  int ni, no;
  mlp_offsets(a, H, &wo, &bo, &ni, &no);
  const float* last = H > 0 ? hid + (size_t)(H - 1) * W : feat;
  for (int i = 0; i < ni; ++i) d_in[i] = 0.f;
  for (int o = 0; o < 4; ++o) {
    const float g = g_raw[o];
    if (g == 0.f) continue;
    float* gw = grad + wo + (size_t)o * ni;
    const float* wrow = params + wo + (size_t)o * ni;
    for (int i = 0; i < ni; ++i) {
      gw[i] += g * last[i];
      d_in[i] += g * wrow[i];
    }
    grad[bo + o] += g;
  }
  for (int l = H - 1; l >= 0; --l) {
    mlp_offsets(a, l, &wo, &bo, &ni, &no);
    const float* pr = pre + (size_t)l * W;
    const float* in = l > 0 ? hid + (size_t)(l - 1) * W : feat;
    for (int i = 0; i < ni; ++i) d_prev[i] = 0.f;
    for (int o = 0; o < no; ++o) {
      if (pr[o] <= 0.f) continue;
      const float g = d_in[o];
      if (g == 0.f) continue;
      float* gw = grad + wo + (size_t)o * ni;
      const float* wrow = params + wo + (size_t)o * ni;
      for (int i = 0; i < ni; ++i) {
        gw[i] += g * in[i];
        d_prev[i] += g * wrow[i];
      }
      grad[bo + o] += g;
    }
    float* t = d_in;
    d_in = d_prev;
    d_prev = t;
  }
  for (int l = 0; l < L; ++l) {
    const size_t level_off = (size_t)l * F * rows_n;
    for (int corner = 0; corner < 8; ++corner) {
      const float w = cw[l * 8 + corner];
      if (w == 0.f) continue;
      float* ge = grad + level_off + (size_t)rows[l * 8 + corner] * F;
      for (int f = 0; f < F; ++f) ge[f] += w * d_in[l * F + f];
    }
  }
  free(feat);
  free(pre);
  free(hid);
  free(rows);
  free(cw);
  free(d_in);
  free(d_prev);
}

/* field.cpp:295-310 */
void po_adam_step(size_t n, float* p, const float* g, float* m, float* v, int64_t* step,
                  float lr, float b1, float b2, float eps) {
  *step += 1;
  const float c1 = 1.f - powf(b1, (float)*step);
  const float c2 = 1.f - powf(b2, (float)*step);
  for (size_t i = 0; i < n; ++i) {
    const float gi = g[i];
    m[i] = b1 * m[i] + (1.f - b1) * gi;
    v[i] = b2 * v[i] + (1.f - b2) * gi * gi;
    const float mhat = m[i] / c1;
    const float vhat = v[i] / c2;
    p[i] -= lr * mhat / (sqrtf(vhat) + eps);
  }
}

/* --------------------------------------------------------------- render */

/* geom.hpp:141-162 */
int po_ray_box(const float o[3], const float d[3], const float bmin[3], const float bmax[3],
               float* t_near, float* t_far) {
  float t0 = -INFINITY, t1 = INFINITY;
  for (int ax = 0; ax < 3; ++ax) {
    const float oo = o[ax], dd = d[ax];
    if (fabsf(dd) < 1e-12f) {
      if (oo < bmin[ax] || oo > bmax[ax]) return 0;
      continue;
    }
    const float inv = 1.f / dd;
    float ta = (bmin[ax] - oo) * inv;
    float tb = (bmax[ax] - oo) * inv;
    if (ta > tb) {
      const float t = ta;
      ta = tb;
      tb = t;
    }
    t0 = fmaxf(t0, ta);
    t1 = fminf(t1, tb);
  }
  if (t0 > t1) return 0;
  *t_near = t0;
  *t_far = t1;
  return 1;
}

/* render.cpp:11-15 */
static void normalize_in_box(const float o[3], const float d[3], float t, const float bmin[3],
                             const float bmax[3], float out[3]) {
  for (int ax = 0; ax < 3; ++ax) {
    const float pt = o[ax] + d[ax] * t;
    const float s = bmax[ax] - bmin[ax];
    out[ax] = clampf01((pt - bmin[ax]) / s);
  }
}

/* render.cpp:104-132; returns 1 when escaped. */
int po_uniform_samples(const float o[3], const float d[3], const float bmin[3],
                       const float bmax[3], int n, float* depths, float* deltas, float* pos,
                       float* t_entry, float* t_exit) {
  float t0, t1;
  if (!po_ray_box(o, d, bmin, bmax, &t0, &t1) || t1 <= 0.f) return 1;
  t0 = fmaxf(t0, 0.f);
  if (t1 - t0 < 1e-9f) return 1;
  if (t_entry) *t_entry = t0;
  if (t_exit) *t_exit = t1;
  const float step = (t1 - t0) / (float)n;
  for (int i = 0; i < n; ++i) {
    const float dd = t0 + ((float)i + 0.5f) * step;
    if (depths) depths[i] = dd;
    if (deltas) deltas[i] = step;
    if (pos) normalize_in_box(o, d, dd, bmin, bmax, pos + 3 * i);
  }
  return 0;
}

/* render.cpp:134-154 */
void po_composite(int n, const float* sigma, const float* rgb, const float* deltas,
                  const float* depths, float color[3], float* depth, float* term_probs) {
  double cr = 0.0, cg = 0.0, cb = 0.0, dep = 0.0, T = 1.0;
  for (int i = 0; i < n; ++i) {
    const double a = 1.0 - exp(-(double)sigma[i] * deltas[i]);
    const double rho = a * T;
    if (term_probs) term_probs[i] = (float)rho;
    cr += rho * rgb[3 * i + 0];
    cg += rho * rgb[3 * i + 1];
    cb += rho * rgb[3 * i + 2];
    dep += rho * depths[i];
    T *= 1.0 - a;
  }
  color[0] = (float)cr;
  color[1] = (float)cg;
  color[2] = (float)cb;
  *depth = (float)dep;
}

/* render.cpp:156-185 (accumulates into d_sigma / d_rgb). */
void po_composite_backward(int n, const float* sigma, const float* rgb, const float* deltas,
                           const float* depths, const float d_color[3], float d_depth,
                           float* d_sigma, float* d_rgb) {
  double* a = (double*)malloc(sizeof(double) * (size_t)(3 * n + 1));
  double* rho = a + n;
  double* tb = rho + n;
  double T = 1.0;
  for (int i = 0; i < n; ++i) {
    a[i] = 1.0 - exp(-(double)sigma[i] * deltas[i]);
    tb[i] = T;
    rho[i] = a[i] * T;
    T *= 1.0 - a[i];
  }
  double* s = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  for (int i = 0; i < n; ++i) {
    s[i] = (double)d_color[0] * rgb[3 * i] + (double)d_color[1] * rgb[3 * i + 1] +
           (double)d_color[2] * rgb[3 * i + 2] + (double)d_depth * depths[i];
    const float r = (float)rho[i];
    d_rgb[3 * i + 0] += d_color[0] * r;
    d_rgb[3 * i + 1] += d_color[1] * r;
    d_rgb[3 * i + 2] += d_color[2] * r;
  }
  double suffix = 0.0;
  for (int k = n - 1; k >= 0; --k) {
    double denom = 1.0 - a[k];
    if (denom < 1e-300) denom = 1e-300;
    const double da = s[k] * tb[k] - suffix / denom;
    d_sigma[k] += (float)(da * deltas[k] * (1.0 - a[k]));
    suffix += s[k] * rho[k];
  }
  free(a);
  free(s);
}

/* render.cpp:187-243 with the background targets given explicitly
 * (bg_colors: 3 per ray, read for background rays only). d_sigma / d_rgb are
 * zeroed then filled for every sample of every ray. Returns 3 on a
 * non-finite total (NumericError, render.cpp:241). */
int po_batch_loss(int n_rays, const int* kind, const float* target_rgb,
                  const float* target_depth, const int* escaped, const int* offsets,
                  const float* deltas, const float* depths, const float* sigma,
                  const float* rgb, const float* bg_colors, float lambda_d, float lambda_sigma,
                  double terms[4], float* d_sigma, float* d_rgb, float* color_out,
                  float* depth_out) {
  double color_term = 0.0, depth_term = 0.0, sigma_term = 0.0;
  const int total_s = offsets[n_rays];
  for (int i = 0; i < total_s; ++i) {
    d_sigma[i] = 0.f;
    d_rgb[3 * i] = d_rgb[3 * i + 1] = d_rgb[3 * i + 2] = 0.f;
  }
  for (int r = 0; r < n_rays; ++r) {
    const int b = offsets[r], n = offsets[r + 1] - offsets[r];
    if (color_out) color_out[3 * r] = color_out[3 * r + 1] = color_out[3 * r + 2] = 0.f;
    if (depth_out) depth_out[r] = 0.f;
    if (escaped[r] || n == 0) continue;
    float c[3], dep;
    po_composite(n, sigma + b, rgb + 3 * b, deltas + b, depths + b, c, &dep, NULL);
    if (color_out) memcpy(color_out + 3 * r, c, sizeof c);
    if (depth_out) depth_out[r] = dep;
    const float* tgt = kind[r] ? bg_colors + 3 * r : target_rgb + 3 * r;
    const float e0 = c[0] - tgt[0], e1 = c[1] - tgt[1], e2 = c[2] - tgt[2];
    const float cn = sqrtf(e0 * e0 + e1 * e1 + e2 * e2);
    color_term += cn;
    float dc[3] = {0.f, 0.f, 0.f};
    if (cn > 1e-12f) {
      dc[0] = e0 / cn;
      dc[1] = e1 / cn;
      dc[2] = e2 / cn;
    }
    float dd = 0.f;
    if (!kind[r] && target_depth[r] >= 0.f) {
      const float derr = dep - target_depth[r];
      depth_term += fabsf(derr);
      dd = lambda_d * (derr > 0.f ? 1.f : (derr < 0.f ? -1.f : 0.f));
    }
    po_composite_backward(n, sigma + b, rgb + 3 * b, deltas + b, depths + b, dc, dd,
                          d_sigma + b, d_rgb + 3 * b);
    if (kind[r])
      for (int i = 0; i < n; ++i) {
        sigma_term += sigma[b + i];
        d_sigma[b + i] += lambda_sigma;
      }
  }
  terms[1] = color_term;
  terms[2] = depth_term;
  terms[3] = sigma_term;
  terms[0] = color_term + lambda_d * depth_term + lambda_sigma * sigma_term;
  return isfinite(terms[0]) ? 0 : 3;
}

/* render.cpp:17-45: 8-connected BFS = Chebyshev distance <= band_px, minus
 * the region itself. */
void po_dilation_band(int w, int h, const uint8_t* mask, uint8_t value, int band_px,
                      uint8_t* out) {
  const size_t npx = (size_t)w * h;
  int* dist = (int*)malloc(sizeof(int) * npx);
  int* queue = (int*)malloc(sizeof(int) * npx);
  size_t head = 0, tail = 0;
  for (size_t i = 0; i < npx; ++i) {
    out[i] = 0;
    dist[i] = -1;
    if (mask[i] == value) {
      dist[i] = 0;
      queue[tail++] = (int)i;
    }
  }
  while (head < tail) {
    const int idx = queue[head++];
    const int x = idx % w, y = idx / w, d = dist[idx];
    if (d >= band_px) continue;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int nx = x + dx, ny = y + dy;
        if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
        const size_t ni = (size_t)ny * w + nx;
        if (dist[ni] >= 0) continue;
        dist[ni] = d + 1;
        out[ni] = 1;
        queue[tail++] = (int)ni;
      }
  }
  free(dist);
  free(queue);
}

static void mat_vec(const float* M, const float v[3], float out[3]) {
  out[0] = M[0] * v[0] + M[1] * v[1] + M[2] * v[2];
  out[1] = M[3] * v[0] + M[4] * v[1] + M[5] * v[2];
  out[2] = M[6] * v[0] + M[7] * v[1] + M[8] * v[2];
}

static int build_pixel_lists(int W, int H, const uint8_t* mask, uint8_t inst, int band_px,
                             int** obj_px, int* n_obj_px, int** bg_px, int* n_bg_px) {
  const size_t npx = (size_t)W * H;
  uint8_t* band = (uint8_t*)malloc(npx);
  po_dilation_band(W, H, mask, inst, band_px, band);
  *obj_px = (int*)malloc(sizeof(int) * (npx + 1));
  *bg_px = (int*)malloc(sizeof(int) * (npx + 1));
  *n_obj_px = *n_bg_px = 0;
  for (size_t i = 0; i < npx; ++i) {
    if (mask[i] == inst) (*obj_px)[(*n_obj_px)++] = (int)i;
    if (band[i]) (*bg_px)[(*n_bg_px)++] = (int)i;
  }
  free(band);
  return 0;
}

/* render.cpp:47-102 with explicit picks. */
int po_generate_rays(const prenom_camera* cam, const float* rgb, const float* depth,
                     const uint8_t* mask, uint8_t inst, const prenom_pose* obj_pose, int n,
                     float bg_fraction, int band_px, const uint32_t* picks, float* origins,
                     float* dirs, int* kinds, float* target_rgb, float* target_depth,
                     int* pick_px, int* n_obj_out) {
  if (n < 1) return 1;
  const int W = cam->width, H = cam->height;
  int *obj_px, *bg_px, n_op, n_bp;
  build_pixel_lists(W, H, mask, inst, band_px, &obj_px, &n_op, &bg_px, &n_bp);
  if (n_op == 0) {
    free(obj_px);
    free(bg_px);
    return 2;
  }
  int n_bg = n_bp == 0 ? 0 : (int)lroundf((float)n * bg_fraction);
  if (n_bg > n) n_bg = n;
  const int n_obj = n - n_bg;
  if (n_obj_out) *n_obj_out = n_obj;
  /* Pose::inverse (geom.hpp:127-130) */
  float Rt[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Rt[i * 3 + j] = obj_pose->R[j * 3 + i];
  float tt[3], org[3], wt[3];
  mat_vec(Rt, obj_pose->t, tt);
  const float tinv[3] = {-tt[0], -tt[1], -tt[2]};
  mat_vec(Rt, cam->t, wt);
  for (int k = 0; k < 3; ++k) org[k] = wt[k] + tinv[k];
  for (int i = 0; i < n; ++i) {
    const int is_bg = i >= n_obj;
    const int px = is_bg ? bg_px[picks[i]] : obj_px[picks[i]];
    const int x = px % W, y = px / W;
    if (pick_px) pick_px[i] = px;
    /* Camera::pixel_direction (render.hpp:20-22) + geom.hpp normalized */
    const float v[3] = {((float)x - cam->cx) / cam->fx, ((float)y - cam->cy) / cam->fy, 1.f};
    const float nn = sqrtf(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    float dc[3] = {0.f, 0.f, 0.f};
    if (nn > 0.f) {
      dc[0] = v[0] / nn;
      dc[1] = v[1] / nn;
      dc[2] = v[2] / nn;
    }
    float dw[3], dobj[3];
    mat_vec(cam->R, dc, dw);
    mat_vec(Rt, dw, dobj);
    memcpy(origins + 3 * i, org, sizeof org);
    memcpy(dirs + 3 * i, dobj, sizeof dobj);
    kinds[i] = is_bg;
    memcpy(target_rgb + 3 * i, rgb + 3 * (size_t)px, 3 * sizeof(float));
    target_depth[i] = -1.f;
    if (!is_bg && depth[px] > 0.f) target_depth[i] = depth[px];
  }
  free(obj_px);
  free(bg_px);
  return 0;
}

int po_generate_rays_philox(const prenom_camera* cam, const float* rgb, const float* depth,
                            const uint8_t* mask, uint8_t inst, const prenom_pose* obj_pose,
                            int n, float bg_fraction, int band_px, uint64_t seed, int64_t step,
                            float* origins, float* dirs, int* kinds, float* target_rgb,
                            float* target_depth, int* pick_px) {
  const int W = cam->width, H = cam->height;
  int *obj_px, *bg_px, n_op, n_bp;
  build_pixel_lists(W, H, mask, inst, band_px, &obj_px, &n_op, &bg_px, &n_bp);
  free(obj_px);
  free(bg_px);
  if (n < 1) return 1;
  if (n_op == 0) return 2;
  int n_bg = n_bp == 0 ? 0 : (int)lroundf((float)n * bg_fraction);
  if (n_bg > n) n_bg = n;
  const int n_obj = n - n_bg;
  uint32_t* picks = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    uint32_t r[4];
    po_draw(seed, PRENOM_TAG_PIXEL, step, (uint32_t)i, 0, r);
    picks[i] = po_pick(r[0], (uint32_t)(i < n_obj ? n_op : n_bp));
  }
  const int st = po_generate_rays(cam, rgb, depth, mask, inst, obj_pose, n, bg_fraction,
                                  band_px, picks, origins, dirs, kinds, target_rgb,
                                  target_depth, pick_px, NULL);
  free(picks);
  return st;
}

/* --------------------------------------------------------- density grid */

/* density_grid.cpp:20-41 */
float po_trilerp(int R, const float* g, const float p_in[3]) {
  const float px = clampf01(p_in[0]), py = clampf01(p_in[1]), pz = clampf01(p_in[2]);
  const float gx = px * (float)(R - 1), gy = py * (float)(R - 1), gz = pz * (float)(R - 1);
  int i = (int)gx, j = (int)gy, k = (int)gz;
  if (i > R - 2) i = R - 2;
  if (j > R - 2) j = R - 2;
  if (k > R - 2) k = R - 2;
  const float fx = gx - (float)i, fy = gy - (float)j, fz = gz - (float)k;
#define AT(a, b, c) g[(size_t)(a) + (size_t)R * ((size_t)(b) + (size_t)R * (size_t)(c))]
  const float c00 = AT(i, j, k) * (1.f - fx) + AT(i + 1, j, k) * fx;
  const float c10 = AT(i, j + 1, k) * (1.f - fx) + AT(i + 1, j + 1, k) * fx;
  const float c01 = AT(i, j, k + 1) * (1.f - fx) + AT(i + 1, j, k + 1) * fx;
  const float c11 = AT(i, j + 1, k + 1) * (1.f - fx) + AT(i + 1, j + 1, k + 1) * fx;
#undef AT
  const float c0 = c00 * (1.f - fy) + c10 * fy;
  const float c1 = c01 * (1.f - fy) + c11 * fy;
  return c0 * (1.f - fz) + c1 * fz;
}

/* density_grid.cpp:43-70, with pdm_det_exp in place of std::exp (the one
 * tolerance-pinned substitution). Returns 1 when escaped. */
int po_build_ray_cdf(int R, const float* vals, int n, const float* deltas, const float* pos,
                     float eps, float* term_probs, float* cdf) {
  double T = 1.0, total = 0.0;
  for (int i = 0; i < n; ++i) {
    const double sigma = po_trilerp(R, vals, pos + 3 * i);
    const double a = 1.0 - pdm_det_exp(-sigma * deltas[i]);
    const double rho = a * T;
    term_probs[i] = (float)rho;
    total += rho;
    T *= 1.0 - a;
  }
  if (total < eps) return 1;
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc += term_probs[i];
    cdf[i] = (float)(acc / total);
  }
  cdf[n - 1] = 1.f;
  return 0;
}

static int cmp_float(const void* a, const void* b) {
  const float x = *(const float*)a, y = *(const float*)b;
  return (x > y) - (x < y);
}

/* density_grid.cpp:72-108 with explicit uniforms (2 per sample, in the
 * reference's consumption order: bin draw, then in-bin draw). */
void po_inverse_transform_sample(const float o[3], const float d[3], const float bmin[3],
                                 const float bmax[3], float t_entry, float t_exit, int n_c,
                                 const float* c_depths, const float* c_deltas, const float* cdf,
                                 int n, const float* u, float* depths, float* deltas,
                                 float* pos) {
  for (int s = 0; s < n; ++s) {
    const float uu = u[2 * s];
    int bin = 0; /* std::lower_bound: first cdf[i] >= uu */
    {
      int lo = 0, cnt = n_c;
      while (cnt > 0) {
        const int half = cnt / 2;
        if (cdf[lo + half] < uu) {
          lo = lo + half + 1;
          cnt -= half + 1;
        } else {
          cnt = half;
        }
      }
      bin = lo;
    }
    if (bin > n_c - 1) bin = n_c - 1;
    float lo = c_depths[bin] - 0.5f * c_deltas[bin];
    float hi = c_depths[bin] + 0.5f * c_deltas[bin];
    lo = fmaxf(lo, t_entry);
    hi = fminf(hi, t_exit);
    depths[s] = lo + u[2 * s + 1] * (hi - lo);
  }
  qsort(depths, (size_t)n, sizeof(float), cmp_float);
  for (int i = 1; i < n; ++i)
    if (depths[i] <= depths[i - 1]) depths[i] = depths[i - 1] + 1e-6f;
  for (int i = 0; i + 1 < n; ++i) deltas[i] = depths[i + 1] - depths[i];
  deltas[n - 1] = fmaxf(t_exit - depths[n - 1], 1e-6f);
  for (int i = 0; i < n; ++i) normalize_in_box(o, d, depths[i], bmin, bmax, pos + 3 * i);
}

/* density_grid.cpp:110-117; returns 1 when the final set is escaped. */
int po_sample_ray(int R, const float* vals, const float o[3], const float d[3],
                  const float bmin[3], const float bmax[3], int n_c, int n_f, float eps,
                  const float* u, float* depths, float* deltas, float* pos, float* t_entry,
                  float* t_exit) {
  float* cd = (float*)malloc(sizeof(float) * (size_t)(7 * n_c));
  float* cdl = cd + n_c;
  float* cp = cdl + n_c;
  float* tp = cp + 3 * n_c;
  float* cdf = tp + n_c;
  float te = 0.f, tx = 0.f;
  int esc = po_uniform_samples(o, d, bmin, bmax, n_c, cd, cdl, cp, &te, &tx);
  if (!esc) esc = po_build_ray_cdf(R, vals, n_c, cdl, cp, eps, tp, cdf) ? 2 : 0;
  int out;
  if (esc) {
    out = po_uniform_samples(o, d, bmin, bmax, n_f, depths, deltas, pos, t_entry, t_exit);
  } else {
    po_inverse_transform_sample(o, d, bmin, bmax, te, tx, n_c, cd, cdl, cdf, n_f, u, depths,
                                deltas, pos);
    if (t_entry) *t_entry = te;
    if (t_exit) *t_exit = tx;
    out = 0;
  }
  free(cd);
  return out;
}

int po_sample_ray_philox(int R, const float* vals, const float o[3], const float d[3],
                         const float bmin[3], const float bmax[3], int n_c, int n_f, float eps,
                         uint64_t seed, uint32_t tag, int64_t step, uint32_t ray,
                         float* depths, float* deltas, float* pos, float* t_entry,
                         float* t_exit) {
  float* u = (float*)malloc(sizeof(float) * (size_t)(2 * n_f + 4));
  for (int s = 0; s < n_f; s += 2) {
    uint32_t r[4];
    po_draw(seed, tag, step, ray, (uint32_t)(s / 2), r);
    u[2 * s + 0] = po_u01(r[0]);
    u[2 * s + 1] = po_u01(r[1]);
    u[2 * s + 2] = po_u01(r[2]);
    u[2 * s + 3] = po_u01(r[3]);
  }
  const int st = po_sample_ray(R, vals, o, d, bmin, bmax, n_c, n_f, eps, u, depths, deltas, pos,
                               t_entry, t_exit);
  free(u);
  return st;
}

/* density_grid.cpp:119-132 */
int po_refresh_grid(const prenom_field_arch* a, const float* params, int R, float* out) {
  const float scale = 1.f / (float)(R - 1);
  int st = 0;
  for (int k = 0; k < R; ++k)
    for (int j = 0; j < R; ++j)
      for (int i = 0; i < R; ++i) {
        const float p[3] = {(float)i * scale, (float)j * scale, (float)k * scale};
        float s;
        if (po_field_eval(a, params, p, &s, NULL, NULL, NULL, NULL, NULL, NULL, NULL)) st = 3;
        out[(size_t)i + (size_t)R * ((size_t)j + (size_t)R * k)] = s;
      }
  return st;
}

/* meta.cpp:83-92 */
void po_reptile_update(size_t n, const float* meta, const float* adapted, float beta,
                       float* out) {
  const float keep = 1.f - beta;
  for (size_t i = 0; i < n; ++i) out[i] = keep * meta[i] + beta * adapted[i];
}

/* ------------------------------------------------------- trainer object */

struct po_object {
  prenom_field_arch arch;
  prenom_train_cfg cfg;
  size_t P;
  float *params, *m, *v, *grad;
  int64_t step;
  int R;
  float* grid;
  uint64_t seed;
  float bmin[3], bmax[3];
  int n_frames, W, H;
  prenom_camera* cams;
  float *rgb, *depth;
  uint8_t* mask;
  uint8_t inst;
  prenom_pose pose;
};

po_object* po_object_create(const prenom_field_arch* a, const float* theta, const float* grid,
                            int grid_res, uint64_t seed, const prenom_train_cfg* cfg,
                            const float bmin[3], const float bmax[3]) {
  po_object* o = (po_object*)calloc(1, sizeof(po_object));
  o->arch = *a;
  o->cfg = *cfg;
  o->P = po_param_count(a);
  o->params = (float*)malloc(sizeof(float) * o->P);
  memcpy(o->params, theta, sizeof(float) * o->P);
  o->m = (float*)calloc(o->P, sizeof(float));
  o->v = (float*)calloc(o->P, sizeof(float));
  o->grad = (float*)calloc(o->P, sizeof(float));
  o->R = grid_res;
  const size_t nv = (size_t)grid_res * grid_res * grid_res;
  o->grid = (float*)calloc(nv, sizeof(float));
  if (grid) memcpy(o->grid, grid, sizeof(float) * nv);
  o->seed = seed;
  memcpy(o->bmin, bmin, sizeof o->bmin);
  memcpy(o->bmax, bmax, sizeof o->bmax);
  return o;
}

void po_object_destroy(po_object* o) {
  if (!o) return;
  free(o->params);
  free(o->m);
  free(o->v);
  free(o->grad);
  free(o->grid);
  free(o->cams);
  free(o->rgb);
  free(o->depth);
  free(o->mask);
  free(o);
}

int po_object_set_frames(po_object* o, int n, const prenom_camera* cams, const float* rgb,
                         const float* depth, const uint8_t* mask, uint8_t inst,
                         const prenom_pose* pose) {
  o->n_frames = n;
  o->W = cams[0].width;
  o->H = cams[0].height;
  const size_t px = (size_t)o->W * o->H * n;
  o->cams = (prenom_camera*)malloc(sizeof(prenom_camera) * (size_t)n);
  memcpy(o->cams, cams, sizeof(prenom_camera) * (size_t)n);
  o->rgb = (float*)malloc(sizeof(float) * px * 3);
  memcpy(o->rgb, rgb, sizeof(float) * px * 3);
  o->depth = (float*)malloc(sizeof(float) * px);
  memcpy(o->depth, depth, sizeof(float) * px);
  o->mask = (uint8_t*)malloc(px);
  memcpy(o->mask, mask, px);
  o->inst = inst;
  o->pose = *pose;
  return 0;
}

/* mapper.cpp:150-184, one iteration per step, Philox draws with c2 = step. */
/* ---- optional threading of the oracle's train step (env PO_THREADS, default
 * 1 = the sequential restatement every parity test uses). Only long
 * full-size evidence runs set it: field evaluations are independent; the
 * backward gives each thread a contiguous sample block and a private gradient,
 * summed in thread order -- deterministic for a given thread count, not the
 * sequential summation order. */
static int po_threads(void) {
  const char* e = getenv("PO_THREADS");
  const int n = e ? atoi(e) : 1;
  return n < 1 ? 1 : (n > 64 ? 64 : n);
}

typedef struct {
  const prenom_field_arch* a;
  const float* params;
  const float* pos;
  float* sg;
  float* rgb;
  const float* dsg;
  const float* drgb;
  float* grad;
  size_t P;
  int n;
  int nt;
  int status;
} po_par_job;

typedef struct {
  po_par_job* job;
  int t;
  float* priv;
  int status;
} po_par_arg;

static void* po_eval_block(void* p) {
  po_par_arg* w = (po_par_arg*)p;
  po_par_job* j = w->job;
  const int lo = (int)((long long)j->n * w->t / j->nt), hi = (int)((long long)j->n * (w->t + 1) / j->nt);
  for (int i = lo; i < hi && w->status == 0; ++i)
    w->status = po_field_eval(j->a, j->params, j->pos + 3 * (size_t)i, j->sg + i, j->rgb + 3 * (size_t)i, NULL,
                              NULL, NULL, NULL, NULL, NULL);
  return NULL;
}

static void* po_backward_block(void* p) {
  po_par_arg* w = (po_par_arg*)p;
  po_par_job* j = w->job;
  const int lo = (int)((long long)j->n * w->t / j->nt), hi = (int)((long long)j->n * (w->t + 1) / j->nt);
  for (int i = lo; i < hi; ++i)
    po_field_backward(j->a, j->params, j->pos + 3 * (size_t)i, j->dsg[i], j->drgb + 3 * (size_t)i, w->priv);
  return NULL;
}

static void po_run_parallel(po_par_job* job, void* (*fn)(void*)) {
  const int nt = po_threads();
  job->nt = nt;
  job->status = 0;
  po_par_arg args[64];
  pthread_t th[64];
  const int backward = fn == po_backward_block;
  for (int t = 0; t < nt; ++t) {
    args[t].job = job;
    args[t].t = t;
    args[t].status = 0;
    args[t].priv = backward ? (float*)calloc(job->P, sizeof(float)) : NULL;
  }
  for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, fn, &args[t]);
  fn(&args[0]);
  for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
  for (int t = 0; t < nt; ++t) job->status |= args[t].status;
  if (backward) {
    for (size_t k = 0; k < job->P; ++k) {
      float acc = 0.f;
      for (int t = 0; t < nt; ++t) acc += args[t].priv[k];
      job->grad[k] = acc;
    }
    for (int t = 0; t < nt; ++t) free(args[t].priv);
  }
}

int po_object_train_step(po_object* o, int n_steps, prenom_step_stats* stats) {
  const prenom_train_cfg* c = &o->cfg;
  const prenom_field_arch* a = &o->arch;
  const int B = c->rays_per_iter, S = c->samples_per_ray;
  float* org = (float*)malloc(sizeof(float) * (size_t)B * 3);
  float* dir = (float*)malloc(sizeof(float) * (size_t)B * 3);
  int* kind = (int*)malloc(sizeof(int) * (size_t)B);
  float* trgb = (float*)malloc(sizeof(float) * (size_t)B * 3);
  float* tdep = (float*)malloc(sizeof(float) * (size_t)B);
  float* bg = (float*)malloc(sizeof(float) * (size_t)B * 3);
  int* esc = (int*)malloc(sizeof(int) * (size_t)B);
  int* off = (int*)malloc(sizeof(int) * (size_t)(B + 1));
  const size_t NS = (size_t)B * S;
  float* dep = (float*)malloc(sizeof(float) * NS);
  float* dlt = (float*)malloc(sizeof(float) * NS);
  float* pos = (float*)malloc(sizeof(float) * NS * 3);
  float* sg = (float*)malloc(sizeof(float) * NS);
  float* rgb = (float*)malloc(sizeof(float) * NS * 3);
  float* dsg = (float*)malloc(sizeof(float) * NS);
  float* drgb = (float*)malloc(sizeof(float) * NS * 3);
  int status = 0;
  const size_t fpx = (size_t)o->W * o->H;
  for (int it = 0; it < n_steps && status == 0; ++it) {
    const int64_t step = o->step;
    uint32_t r4[4];
    po_draw(o->seed, PRENOM_TAG_FRAME, step, 0, 0, r4);
    const int fi = (int)po_pick(r4[0], (uint32_t)o->n_frames);
    status = po_generate_rays_philox(&o->cams[fi], o->rgb + 3 * fpx * fi, o->depth + fpx * fi,
                                     o->mask + fpx * fi, o->inst, &o->pose, B, c->bg_fraction,
                                     c->band_px, o->seed, step, org, dir, kind, trgb, tdep,
                                     NULL);
    if (status) break;
    int n_samples = 0, n_esc = 0;
    off[0] = 0;
    for (int r = 0; r < B; ++r) {
      float* dd = dep + (size_t)off[r];
      int e;
      if (c->prior_sampling)
        e = po_sample_ray_philox(o->R, o->grid, org + 3 * r, dir + 3 * r, o->bmin, o->bmax,
                                 c->coarse_samples, S, c->escape_eps, o->seed, PRENOM_TAG_FINE,
                                 step, (uint32_t)r, dd, dlt + off[r], pos + 3 * (size_t)off[r],
                                 NULL, NULL);
      else
        e = po_uniform_samples(org + 3 * r, dir + 3 * r, o->bmin, o->bmax, S, dd,
                               dlt + off[r], pos + 3 * (size_t)off[r], NULL, NULL);
      esc[r] = e;
      off[r + 1] = off[r] + (e ? 0 : S);
      n_esc += e ? 1 : 0;
      po_draw(o->seed, PRENOM_TAG_BG, step, (uint32_t)r, 0, r4);
      bg[3 * r + 0] = po_u01(r4[0]);
      bg[3 * r + 1] = po_u01(r4[1]);
      bg[3 * r + 2] = po_u01(r4[2]);
    }
    n_samples = off[B];
    {
      po_par_job job = {a, o->params, pos, sg, rgb, dsg, drgb, NULL, o->P, n_samples, 0, 0};
      po_run_parallel(&job, po_eval_block);
      status = job.status;
    }
    if (status) break;
    double terms[4];
    status = po_batch_loss(B, kind, trgb, tdep, esc, off, dlt, dep, sg, rgb, bg, c->lambda_d,
                           c->lambda_sigma, terms, dsg, drgb, NULL, NULL);
    if (status) break;
    memset(o->grad, 0, sizeof(float) * o->P);
    if (po_threads() <= 1) {
      for (int i = 0; i < n_samples; ++i)
        po_field_backward(a, o->params, pos + 3 * i, dsg[i], drgb + 3 * i, o->grad);
    } else {
      po_par_job job = {a, o->params, pos, sg, rgb, dsg, drgb, o->grad, o->P, n_samples, 0, 0};
      po_run_parallel(&job, po_backward_block);
    }
    po_adam_step(o->P, o->params, o->grad, o->m, o->v, &o->step, c->eta, c->adam_beta1,
                 c->adam_beta2, c->adam_eps);
    if (stats) {
      prenom_step_stats* s = &stats[it];
      s->total = terms[0];
      s->color_term = terms[1];
      s->depth_term = terms[2];
      s->sigma_term = terms[3];
      s->n_samples = n_samples;
      s->n_rays_escaped = n_esc;
      s->frame_index = fi;
    }
    if (c->grid_refresh_every > 0 && o->step % c->grid_refresh_every == 0)
      status = po_refresh_grid(a, o->params, o->R, o->grid);
  }
  free(org);
  free(dir);
  free(kind);
  free(trgb);
  free(tdep);
  free(bg);
  free(esc);
  free(off);
  free(dep);
  free(dlt);
  free(pos);
  free(sg);
  free(rgb);
  free(dsg);
  free(drgb);
  return status;
}

void po_object_get_params(const po_object* o, float* theta) {
  memcpy(theta, o->params, sizeof(float) * o->P);
}

void po_object_get_grid(const po_object* o, float* grid) {
  memcpy(grid, o->grid, sizeof(float) * (size_t)o->R * o->R * o->R);
}

int64_t po_object_step(const po_object* o) { return o->step; }
