// kernels_render.cu -- front-to-back compositing + batch loss + compositing
// backward, one warp per ray.
//
// Replaces composite (render.cpp:134-154), composite_backward
// (render.cpp:156-185) and batch_loss (render.cpp:187-243). Like the
// reference, all compositing arithmetic is fp64 (B200 runs fp64 at half the
// fp32 rate; this kernel moves 40 B/sample and is nowhere near either
// bound). The transmittance product and the suffix sum of
// composite_backward are warp scans instead of sequential loops, so results
// agree with the reference to fp64 rounding (tolerance-checked), not bitwise.
// Background targets are Philox draws (TAG_BG, c1 = ray) or explicit.
#include "prenom_device.cuh"

namespace prenom {
namespace {

constexpr int kWarps = 8;
constexpr int kMaxChunk = 8;  // S <= 256; a lane holds K = ceil(S/32) <= kMaxChunk samples

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// K (samples per lane) is a template parameter so the per-lane arrays are
// sized to the batch (S = 96 -> 3): registers, and so occupancy, follow S.
template <int K>
__device__ __forceinline__ void composite_body(const CompositeArgs& a, int frame) {
  __shared__ double red[kWarps][4];
  __shared__ unsigned long long red_n[kWarps];
  __shared__ int red_e[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * kWarps + warp;
  pdl_wait();  // field outputs of the forward kernel
  pdl_trigger();
  double t_color = 0.0, t_depth = 0.0, t_sigma = 0.0;
  int cnt = 0;
  if (r < a.B) {
    cnt = a.count[r];
    const size_t base = (size_t)r * a.S;
    const int k = (a.S + 31) >> 5;  // <= K
    const int i0 = lane * k;
    float sg[K], dl[K], dp[K], cr[K], cg[K], cb[K];
    double av[K], tb[K], rho[K];
    double prod = 1.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int i = i0 + j;
      sg[j] = dl[j] = dp[j] = cr[j] = cg[j] = cb[j] = 0.f;
      av[j] = 0.0;
      if (j < k && i < cnt) {
        const float4 o = a.out[base + i];
        sg[j] = o.x;
        cr[j] = o.y;
        cg[j] = o.z;
        cb[j] = o.w;
        dl[j] = a.delta[base + i];
        dp[j] = a.pos_depth[base + i].w;
        av[j] = 1.0 - exp(-(double)sg[j] * (double)dl[j]);
        prod *= 1.0 - av[j];
      }
    }
    // exclusive multiplicative scan of per-lane survival products
    double incl = prod;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl *= v;
    }
    double T = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) T = 1.0;
    double pc_r = 0.0, pc_g = 0.0, pc_b = 0.0, pd = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      tb[j] = T;
      rho[j] = av[j] * T;
      pc_r += rho[j] * cr[j];
      pc_g += rho[j] * cg[j];
      pc_b += rho[j] * cb[j];
      pd += rho[j] * dp[j];
      T *= 1.0 - av[j];
    }
    const float C0 = (float)warp_sum(pc_r), C1 = (float)warp_sum(pc_g), C2 = (float)warp_sum(pc_b);
    const float D = (float)warp_sum(pd);
    if (cnt > 0) {
      const float4 tg = a.target[r];
      const int bg = a.kind[r] == PRENOM_KIND_BACKGROUND;
      float t0 = tg.x, t1 = tg.y, t2 = tg.z;
      if (bg) {
        if (a.bg_colors) {
          t0 = a.bg_colors[3 * r];
          t1 = a.bg_colors[3 * r + 1];
          t2 = a.bg_colors[3 * r + 2];
        } else {
          uint32_t x4[4];
          philox_draw(a.seed, PRENOM_TAG_BG, a.step, (uint32_t)r, 0u, x4);
          t0 = pdm_u01(x4[0]);
          t1 = pdm_u01(x4[1]);
          t2 = pdm_u01(x4[2]);
        }
      }
      if (lane == 0) {
        if (a.color_out) {
          a.color_out[3 * r] = C0;
          a.color_out[3 * r + 1] = C1;
          a.color_out[3 * r + 2] = C2;
        }
        if (a.depth_out) a.depth_out[r] = D;
      }
      // batch_loss (render.cpp:212-236)
      const float e0 = C0 - t0, e1 = C1 - t1, e2 = C2 - t2;
      const float cn = sqrtf(__fadd_rn(__fadd_rn(__fmul_rn(e0, e0), __fmul_rn(e1, e1)), __fmul_rn(e2, e2)));
      float dc0 = 0.f, dc1 = 0.f, dc2 = 0.f;
      if (cn > 1e-12f) {
        dc0 = e0 / cn;
        dc1 = e1 / cn;
        dc2 = e2 / cn;
      }
      float dd = 0.f;
      t_color = cn;
      if (!bg && tg.w >= 0.f) {
        const float derr = D - tg.w;
        t_depth = fabsf(derr);
        dd = a.lambda_d * (derr > 0.f ? 1.f : (derr < 0.f ? -1.f : 0.f));
      }
      if (bg) {
        double sd = 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) sd += (double)sg[j];
        t_sigma = warp_sum(sd);
      }
      if (a.dout) {
        // composite_backward (render.cpp:171-184)
        double sv[K];
        double q = 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          sv[j] = (double)dc0 * cr[j] + (double)dc1 * cg[j] + (double)dc2 * cb[j] + (double)dd * dp[j];
          q += sv[j] * rho[j];
        }
        // exclusive suffix sum over lanes > lane
        double incl_s = q;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double v = __shfl_down_sync(0xffffffffu, incl_s, o);
          if (lane + o < 32) incl_s += v;
        }
        double suffix = incl_s - q;
#pragma unroll
        for (int j = K - 1; j >= 0; --j) {
          const int i = i0 + j;
          if (j < k && i < cnt) {
            const double denom = fmax(1.0 - av[j], 1e-300);
            const double da = sv[j] * tb[j] - suffix / denom;
            float ds = (float)(da * (double)dl[j] * (1.0 - av[j]));
            if (bg) ds += a.lambda_sigma;
            const float rf = (float)rho[j];
            a.dout[base + i] = make_float4(ds, dc0 * rf, dc1 * rf, dc2 * rf);
          }
          suffix += sv[j] * rho[j];
        }
      }
    }
    if (cnt > 0 && !(isfinite(t_color) && isfinite(t_depth) && isfinite(t_sigma)) && a.flag)
      atomicOr(a.flag, 2);
  }
  if (a.stats) {
    if (lane == 0) {
      red[warp][0] = t_color;
      red[warp][1] = t_depth;
      red[warp][2] = t_sigma;
      red_n[warp] = (r < a.B) ? (unsigned long long)cnt : 0ull;
      red_e[warp] = (r < a.B && cnt == 0) ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double c = 0.0, d = 0.0, s = 0.0;
      unsigned long long n = 0;
      int e = 0;
      for (int w = 0; w < kWarps; ++w) {
        c += red[w][0];
        d += red[w][1];
        s += red[w][2];
        n += red_n[w];
        e += red_e[w];
      }
      atomicAdd(&a.stats->color, c);
      atomicAdd(&a.stats->depth, d);
      atomicAdd(&a.stats->sigma, s);
      atomicAdd(&a.stats->n_samples, n);
      atomicAdd(&a.stats->escaped, e);
      if (blockIdx.x == 0) a.stats->frame = frame;
      // the last block to finish forms the total (render.cpp:238-240):
      // total = color + lambda_d * depth + lambda_sigma * sigma
      __threadfence();
      if (atomicAdd(&a.stats->blocks_done, 1u) == gridDim.x - 1) {
        __threadfence();
        StepStatsDev* st = a.stats;
        const double cc = atomicAdd(&st->color, 0.0), dd = atomicAdd(&st->depth, 0.0),
                     ss = atomicAdd(&st->sigma, 0.0);
        st->total = cc + (double)a.lambda_d * dd + (double)a.lambda_sigma * ss;
        if (!isfinite(st->total) && a.flag) atomicOr(a.flag, 2);
      }
    }
  }
}

// 4 blocks/SM caps it at 64 registers (94 unbounded; a 32-byte spill):
// 32 resident warps hide the fp64 scans' latency (cfg2 0.0285 -> 0.0241 ms;
// 5 blocks/SM, 48 registers, spills more and is slower)
template <int K>
__global__ void __launch_bounds__(kWarps * 32, 4) k_composite(CompositeArgs a, int frame) {
  composite_body<K>(a, frame);
}

// grouped (multi-object scheduler): blockIdx.y = object, its arguments jobs[y]
template <int K>
__global__ void __launch_bounds__(kWarps * 32, 4) k_composite_grp(const CompositeArgs* __restrict__ jobs) {
  const CompositeArgs a = jobs[blockIdx.y];
  composite_body<K>(a, a.frame);
}

}  // namespace

cudaError_t launch_composite(const CompositeArgs& a, cudaStream_t st) {
  if (a.B <= 0) return cudaSuccess;
  if (a.S > 32 * kMaxChunk) return cudaErrorInvalidValue;
  const int blocks = (a.B + kWarps - 1) / kWarps;
  const int k = (a.S + 31) >> 5;
  const dim3 g(blocks), b(kWarps * 32);
  if (k <= 1) return launch_pdl(k_composite<1>, g, b, 0, st, a, a.frame);
  if (k <= 2) return launch_pdl(k_composite<2>, g, b, 0, st, a, a.frame);
  if (k <= 3) return launch_pdl(k_composite<3>, g, b, 0, st, a, a.frame);
  if (k <= 4) return launch_pdl(k_composite<4>, g, b, 0, st, a, a.frame);
  return launch_pdl(k_composite<kMaxChunk>, g, b, 0, st, a, a.frame);
}

cudaError_t launch_composite_group(const CompositeArgs* jobs_dev, int njobs, int B, int S, cudaStream_t st) {
  if (B <= 0 || njobs <= 0) return cudaSuccess;
  if (S > 32 * kMaxChunk) return cudaErrorInvalidValue;
  const dim3 g((B + kWarps - 1) / kWarps, njobs), b(kWarps * 32);
  const int k = (S + 31) >> 5;
  if (k <= 1) return launch_pdl(k_composite_grp<1>, g, b, 0, st, jobs_dev);
  if (k <= 2) return launch_pdl(k_composite_grp<2>, g, b, 0, st, jobs_dev);
  if (k <= 3) return launch_pdl(k_composite_grp<3>, g, b, 0, st, jobs_dev);
  if (k <= 4) return launch_pdl(k_composite_grp<4>, g, b, 0, st, jobs_dev);
  return launch_pdl(k_composite_grp<kMaxChunk>, g, b, 0, st, jobs_dev);
}

}  // namespace prenom
