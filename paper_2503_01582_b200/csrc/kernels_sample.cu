// kernels_sample.cu -- ray generation + prior-CDF probabilistic ray sampling.
//
// One warp per ray. Replaces, per ray:
//   generate_rays' pixel pick and ray construction   render.cpp:47-102
//   ray_box_intersect / uniform_samples              geom.hpp:141-162, render.cpp:104-132
//   build_ray_cdf (trilerp of the prior grid)        density_grid.cpp:20-70
//   inverse_transform_sample + sort + tie fix        density_grid.cpp:72-108
//   sample_ray's two escape fallbacks                density_grid.cpp:110-117
// Every float/double operation that feeds a sample position, depth, delta
// or bin index is spelled with a *_rn intrinsic (never contracted to FMA)
// and exp is pdm_det_exp, so the result is bit-identical to the CPU oracle
// (oracle/prenom_oracle.c) under the same Philox draws.
//
// Memory: the prior grid (32^3..128^3 fp32, 128 KiB..8 MiB) is read through
// L1/L2 with __ldg (8 corners x n_coarse per ray); outputs are one float4
// (x, y, z, depth) + one float (delta) per sample, written coalesced.
#include "prenom_device.cuh"

namespace prenom {
namespace {

constexpr int kWarpsPerBlock = 4;

__device__ __forceinline__ void mat_vec_rn(const float* M, const float v[3], float out[3]) {
  out[0] = __fadd_rn(__fadd_rn(__fmul_rn(M[0], v[0]), __fmul_rn(M[1], v[1])), __fmul_rn(M[2], v[2]));
  out[1] = __fadd_rn(__fadd_rn(__fmul_rn(M[3], v[0]), __fmul_rn(M[4], v[1])), __fmul_rn(M[5], v[2]));
  out[2] = __fadd_rn(__fadd_rn(__fmul_rn(M[6], v[0]), __fmul_rn(M[7], v[1])), __fmul_rn(M[8], v[2]));
}

// geom.hpp:141-162
__device__ __forceinline__ bool ray_box(const float o[3], const float d[3], const float bmin[3],
                                        const float bmax[3], float& t_near, float& t_far) {
  float t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (fabsf(d[a]) < 1e-12f) {
      if (o[a] < bmin[a] || o[a] > bmax[a]) return false;
      continue;
    }
    const float inv = __fdiv_rn(1.f, d[a]);
    float ta = __fmul_rn(__fsub_rn(bmin[a], o[a]), inv);
    float tb = __fmul_rn(__fsub_rn(bmax[a], o[a]), inv);
    if (ta > tb) {
      const float t = ta;
      ta = tb;
      tb = t;
    }
    t0 = fmaxf(t0, ta);
    t1 = fminf(t1, tb);
  }
  if (t0 > t1) return false;
  t_near = t0;
  t_far = t1;
  return true;
}

// render.cpp:11-15 applied to origin + direction * t.
__device__ __forceinline__ float3 normalize_in_box(const float o[3], const float d[3], float t,
                                                   const float bmin[3], const float bmax[3]) {
  float r[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float p = __fadd_rn(o[a], __fmul_rn(d[a], t));
    r[a] = clamp01(__fdiv_rn(__fsub_rn(p, bmin[a]), __fsub_rn(bmax[a], bmin[a])));
  }
  return make_float3(r[0], r[1], r[2]);
}

// density_grid.cpp:20-41 (same operation order).
__device__ __forceinline__ float trilerp(const float* __restrict__ g, int R, float3 p) {
  const float px = clamp01(p.x), py = clamp01(p.y), pz = clamp01(p.z);
  const float rm1 = (float)(R - 1);
  const float gx = __fmul_rn(px, rm1), gy = __fmul_rn(py, rm1), gz = __fmul_rn(pz, rm1);
  const int i = min((int)gx, R - 2), j = min((int)gy, R - 2), k = min((int)gz, R - 2);
  const float fx = __fsub_rn(gx, (float)i), fy = __fsub_rn(gy, (float)j), fz = __fsub_rn(gz, (float)k);
  auto at = [&](int a, int b, int c) {
    return __ldg(g + (size_t)a + (size_t)R * ((size_t)b + (size_t)R * (size_t)c));
  };
  const float ofx = __fsub_rn(1.f, fx), ofy = __fsub_rn(1.f, fy), ofz = __fsub_rn(1.f, fz);
  const float c00 = __fadd_rn(__fmul_rn(at(i, j, k), ofx), __fmul_rn(at(i + 1, j, k), fx));
  const float c10 = __fadd_rn(__fmul_rn(at(i, j + 1, k), ofx), __fmul_rn(at(i + 1, j + 1, k), fx));
  const float c01 = __fadd_rn(__fmul_rn(at(i, j, k + 1), ofx), __fmul_rn(at(i + 1, j, k + 1), fx));
  const float c11 = __fadd_rn(__fmul_rn(at(i, j + 1, k + 1), ofx), __fmul_rn(at(i + 1, j + 1, k + 1), fx));
  const float c0 = __fadd_rn(__fmul_rn(c00, ofy), __fmul_rn(c10, fy));
  const float c1 = __fadd_rn(__fmul_rn(c01, ofy), __fmul_rn(c11, fy));
  return __fadd_rn(__fmul_rn(c0, ofz), __fmul_rn(c1, fz));
}

__device__ __forceinline__ float uniform_depth(float t0, float step, int i) {
  return __fadd_rn(t0, __fmul_rn(__fadd_rn((float)i, 0.5f), step));
}

// Bitonic sort (ascending) of the warp's p2 = 32*E slots held in registers,
// slot i = lane*E + e: partners j < E are in the same lane, j >= E one
// shuffle away (lane ^ j/E). The sorted multiset is unique, so the result is
// the one std::sort gives (density_grid.cpp:96).
template <int E>
__device__ __forceinline__ void warp_bitonic_sort(float (&v)[E], int lane) {
  constexpr int n = 32 * E;
#pragma unroll
  for (int k = 2; k <= n; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < E) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int f = e ^ j;
          if (f > e) {
            const bool up = ((lane * E + e) & k) == 0;
            const float a = v[e], b = v[f];
            if ((a > b) == up) {
              v[e] = b;
              v[f] = a;
            }
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = lane * E + e;
          const float p = __shfl_xor_sync(0xffffffffu, v[e], j / E);
          const bool want_min = ((i & j) == 0) == ((i & k) == 0);
          v[e] = want_min ? fminf(v[e], p) : fmaxf(v[e], p);
        }
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void sort_slots(float* SORT, int lane) {
  float v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = SORT[lane * E + e];
  __syncwarp();
  warp_bitonic_sort<E>(v, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) SORT[lane * E + e] = v[e];
  __syncwarp();
}

__device__ __forceinline__ void sample_body(const RaySource& src, const SamplerCfg& cfg, const SampleBufs& out,
                                            int nc_cap, int p2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * kWarpsPerBlock + warp;
  if (r >= cfg.B) return;  // warp-uniform
  // per-warp scratch: double A[nc_cap], ACC[nc_cap]; float CDF[nc_cap], SORT[p2]
  const size_t per_warp = (size_t)nc_cap * 16 + (size_t)nc_cap * 4 + (size_t)p2 * 4;
  unsigned char* base = smem_raw + per_warp * warp;
  double* A = reinterpret_cast<double*>(base);
  double* ACC = A + nc_cap;
  float* CDF = reinterpret_cast<float*>(ACC + nc_cap);
  float* SORT = CDF + nc_cap;

  const int S = cfg.S;
  float o[3], d[3];
  float4 tgt = make_float4(0.f, 0.f, 0.f, -1.f);
  int kind = PRENOM_KIND_OBJECT;
  int picked = -1;
  if (src.mode == 0) {
    // generate_rays (render.cpp:63-101): object rays first, then band rays.
    const bool bg = r >= src.n_obj;
    uint32_t x4[4];
    philox_draw(cfg.seed, PRENOM_TAG_PIXEL, cfg.step, (uint32_t)r, 0u, x4);
    const int idx = (int)pdm_pick(x4[0], (uint32_t)(bg ? src.n_bg_px : src.n_obj_px));
    const int px = bg ? src.bg_px[idx] : src.obj_px[idx];
    picked = px;
    const int x = px % src.width, y = px / src.width;
    // Camera::pixel_direction + normalized (render.hpp:20-22, geom.hpp:31-34)
    const float v[3] = {__fdiv_rn(__fsub_rn((float)x, src.cx), src.fx),
                        __fdiv_rn(__fsub_rn((float)y, src.cy), src.fy), 1.f};
    const float nn = __fsqrt_rn(
        __fadd_rn(__fadd_rn(__fmul_rn(v[0], v[0]), __fmul_rn(v[1], v[1])), __fmul_rn(v[2], v[2])));
    float dc[3] = {0.f, 0.f, 0.f};
    if (nn > 0.f) {
      dc[0] = __fdiv_rn(v[0], nn);
      dc[1] = __fdiv_rn(v[1], nn);
      dc[2] = __fdiv_rn(v[2], nn);
    }
    float dw[3];
    mat_vec_rn(src.Rc, dc, dw);
    mat_vec_rn(src.Rt, dw, d);
    o[0] = src.origin[0];
    o[1] = src.origin[1];
    o[2] = src.origin[2];
    const float* c = src.rgb + 3 * (size_t)px;
    const float dep = src.depth[px];
    kind = bg ? PRENOM_KIND_BACKGROUND : PRENOM_KIND_OBJECT;
    tgt = make_float4(c[0], c[1], c[2], (!bg && dep > 0.f) ? dep : -1.f);
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      o[a] = src.origins[3 * r + a];
      d[a] = src.dirs[3 * r + a];
    }
  }

  // uniform_samples' escape tests (render.cpp:108-117)
  float t0 = 0.f, t1 = 0.f;
  bool esc = !ray_box(o, d, cfg.bmin, cfg.bmax, t0, t1) || t1 <= 0.f;
  if (!esc) {
    t0 = fmaxf(t0, 0.f);
    esc = __fsub_rn(t1, t0) < 1e-9f;
  }
  if (lane == 0 && out.ray_o) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      out.ray_o[3 * r + a] = o[a];
      out.ray_d[3 * r + a] = d[a];
    }
    if (out.pick_px) out.pick_px[r] = picked;
  }
  if (lane == 0) {
    out.target[r] = tgt;
    out.kind[r] = kind;
    out.count[r] = esc ? 0 : S;
    if (out.t_entry) out.t_entry[r] = esc ? 0.f : t0;
    if (out.t_exit) out.t_exit[r] = esc ? 0.f : t1;
  }
  if (esc) return;
  const size_t base_s = (size_t)r * S;

  bool uniform = !cfg.prior;
  double total = 0.0;
  const int nc = cfg.n_coarse;
  float cstep = 0.f;
  if (!uniform) {
    // build_ray_cdf over the n_coarse midpoints (density_grid.cpp:43-70)
    cstep = __fdiv_rn(__fsub_rn(t1, t0), (float)nc);
    for (int i = lane; i < nc; i += 32) {
      const float dc = uniform_depth(t0, cstep, i);
      const float3 p = normalize_in_box(o, d, dc, cfg.bmin, cfg.bmax);
      const double sg = (double)trilerp(cfg.grid, cfg.grid_res, p);
      A[i] = __dsub_rn(1.0, pdm_det_exp(__dmul_rn(-sg, (double)cstep)));
    }
    __syncwarp();
    int escaped_cdf = 0;
    if (lane == 0) {
      double T = 1.0;
      for (int i = 0; i < nc; ++i) {
        const double a = A[i];
        const double rho = __dmul_rn(a, T);
        CDF[i] = (float)rho;  // term_probs[i]
        total = __dadd_rn(total, rho);
        T = __dmul_rn(T, __dsub_rn(1.0, a));
      }
      escaped_cdf = total < (double)cfg.eps;
      if (!escaped_cdf) {
        double acc = 0.0;
        for (int i = 0; i < nc; ++i) {
          acc = __dadd_rn(acc, (double)CDF[i]);
          ACC[i] = acc;
        }
      }
    }
    escaped_cdf = __shfl_sync(0xffffffffu, escaped_cdf, 0);
    total = __shfl_sync(0xffffffffu, total, 0);
    __syncwarp();
    uniform = escaped_cdf;
    if (!uniform) {
      for (int i = lane; i < nc; i += 32) CDF[i] = (i == nc - 1) ? 1.f : (float)__ddiv_rn(ACC[i], total);
      __syncwarp();
    }
  }

  if (uniform) {
    // uniform_samples(ray, box, n_fine) (render.cpp:118-131)
    const float step = __fdiv_rn(__fsub_rn(t1, t0), (float)S);
    for (int s = lane; s < S; s += 32) {
      const float dd = uniform_depth(t0, step, s);
      const float3 p = normalize_in_box(o, d, dd, cfg.bmin, cfg.bmax);
      out.pos_depth[base_s + s] = make_float4(p.x, p.y, p.z, dd);
      out.delta[base_s + s] = step;
    }
    return;
  }

  // inverse_transform_sample (density_grid.cpp:83-95): two draws per sample.
  const int npairs = (S + 1) >> 1;
  for (int pr = lane; pr < npairs; pr += 32) {
    uint32_t x4[4];
    philox_draw(cfg.seed, cfg.tag, cfg.step, (uint32_t)r, (uint32_t)pr, x4);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int s = 2 * pr + j;
      if (s >= S) break;
      const float u = pdm_u01(x4[2 * j]), u2 = pdm_u01(x4[2 * j + 1]);
      int lo_i = 0, cnt = nc;  // std::lower_bound
      while (cnt > 0) {
        const int half = cnt >> 1;
        if (CDF[lo_i + half] < u) {
          lo_i += half + 1;
          cnt -= half + 1;
        } else {
          cnt = half;
        }
      }
      const int bin = min(lo_i, nc - 1);
      const float db = uniform_depth(t0, cstep, bin);
      const float hd = __fmul_rn(0.5f, cstep);
      const float lo = fmaxf(__fsub_rn(db, hd), t0);
      const float hi = fminf(__fadd_rn(db, hd), t1);
      SORT[s] = __fadd_rn(lo, __fmul_rn(u2, __fsub_rn(hi, lo)));
    }
  }
  for (int s = S + lane; s < p2; s += 32) SORT[s] = INFINITY;
  __syncwarp();
  // std::sort: bitonic network over p2 slots (the sorted multiset is unique),
  // in registers + shuffles for p2 <= 256, else through shared memory.
  if (p2 == 32) {
    sort_slots<1>(SORT, lane);
  } else if (p2 == 64) {
    sort_slots<2>(SORT, lane);
  } else if (p2 == 128) {
    sort_slots<4>(SORT, lane);
  } else if (p2 == 256) {
    sort_slots<8>(SORT, lane);
  } else {
    for (int k = 2; k <= p2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = lane; i < p2; i += 32) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const float a = SORT[i], b = SORT[ixj];
            const bool up = (i & k) == 0;
            if ((a > b) == up) {
              SORT[i] = b;
              SORT[ixj] = a;
            }
          }
        }
        __syncwarp();
      }
    }
  }
  // strictly increasing fix-up (density_grid.cpp:97-98), sequential when needed
  bool tie = false;
  for (int i = lane + 1; i < S; i += 32) tie |= SORT[i] <= SORT[i - 1];
  if (__any_sync(0xffffffffu, tie)) {
    if (lane == 0)
      for (int i = 1; i < S; ++i)
        if (SORT[i] <= SORT[i - 1]) SORT[i] = __fadd_rn(SORT[i - 1], 1e-6f);
    __syncwarp();
  }
  for (int s = lane; s < S; s += 32) {
    const float dd = SORT[s];
    const float dl = (s + 1 < S) ? __fsub_rn(SORT[s + 1], dd) : fmaxf(__fsub_rn(t1, dd), 1e-6f);
    const float3 p = normalize_in_box(o, d, dd, cfg.bmin, cfg.bmax);
    out.pos_depth[base_s + s] = make_float4(p.x, p.y, p.z, dd);
    out.delta[base_s + s] = dl;
  }
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_sample(RaySource src, SamplerCfg cfg, SampleBufs out, int nc_cap, int p2) {
  sample_body(src, cfg, out, nc_cap, p2);
}

// grouped (multi-object scheduler): blockIdx.y = object
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_sample_grp(const SampleJob* __restrict__ jobs, int nc_cap, int p2) {
  const SampleJob& j = jobs[blockIdx.y];
  sample_body(j.src, j.cfg, j.out, nc_cap, p2);
}

}  // namespace

cudaError_t launch_sample(const RaySource& src, const SamplerCfg& cfg, SampleBufs out,
                          StepStatsDev* /*stats*/, cudaStream_t st) {
  if (cfg.B <= 0) return cudaSuccess;
  const int nc_cap = cfg.prior ? ((cfg.n_coarse + 1) & ~1) : 2;
  int p2 = 32;
  while (p2 < cfg.S) p2 <<= 1;
  const size_t per_warp = (size_t)nc_cap * 20 + (size_t)p2 * 4;
  const size_t smem = per_warp * kWarpsPerBlock;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int blocks = (cfg.B + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_sample<<<blocks, kWarpsPerBlock * 32, smem, st>>>(src, cfg, out, nc_cap, p2);
  return cudaGetLastError();
}

// jobs of one group share B, S, prior and n_coarse (the shared-memory shape)
cudaError_t launch_sample_group(const SampleJob* jobs_dev, int njobs, const SamplerCfg& cfg0, cudaStream_t st) {
  if (cfg0.B <= 0 || njobs <= 0) return cudaSuccess;
  const int nc_cap = cfg0.prior ? ((cfg0.n_coarse + 1) & ~1) : 2;
  int p2 = 32;
  while (p2 < cfg0.S) p2 <<= 1;
  const size_t smem = ((size_t)nc_cap * 20 + (size_t)p2 * 4) * kWarpsPerBlock;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_sample_grp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const dim3 g((cfg0.B + kWarpsPerBlock - 1) / kWarpsPerBlock, njobs);
  k_sample_grp<<<g, kWarpsPerBlock * 32, smem, st>>>(jobs_dev, nc_cap, p2);
  return cudaGetLastError();
}

}  // namespace prenom
