// kernels_optim.cu -- the dense parameter passes of the step and of Reptile:
//   k_adam            adam_step (field.cpp:295-310), bit-exact, fused grad zeroing
//   k_init_params     init_params' distributions from Philox (field.cpp:150-166)
//   k_reptile_*       reptile_update (meta.cpp:83-92), its delta/apply split for NCCL
//   k_philox          Philox4x32-10 known-answer entry point
#include <algorithm>
#include <cstdlib>

#include "prenom_device.cuh"

namespace prenom {
namespace {
// ------------------------------------------------------------------ Adam
// field.cpp:295-310, dense, same operation order with *_rn intrinsics;
// grad zeroed in the same pass (train_track zeroes it before each backward,
// mapper.cpp:175). c1 = 1 - b1^step, c2 = 1 - b2^step come from the host
// (glibc powf, like the reference).
__device__ __forceinline__ void adam1(float& p, float& g, float& m, float& v, float lr, float b1, float b2,
                                      float eps, float c1, float c2) {
  m = __fadd_rn(__fmul_rn(b1, m), __fmul_rn(__fsub_rn(1.f, b1), g));
  v = __fadd_rn(__fmul_rn(b2, v), __fmul_rn(__fmul_rn(__fsub_rn(1.f, b2), g), g));
  const float mhat = __fdiv_rn(m, c1);
  const float vhat = __fdiv_rn(v, c2);
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(lr, mhat), __fadd_rn(__fsqrt_rn(vhat), eps)));
}

__device__ __forceinline__ void adam_body(size_t n, float* __restrict__ p, float* __restrict__ g,
                                          float* __restrict__ m, float* __restrict__ v, float lr, float b1, float b2,
                                          float eps, float c1, float c2, int zero_grad, int bid = -1, int nblk = -1) {
  if (bid < 0) {
    bid = blockIdx.x;
    nblk = gridDim.x;
  }
  const size_t n4 = n / 4;
  const size_t stride = (size_t)nblk * blockDim.x;
  // two float4 groups per thread per iteration: 8 independent 16 B loads in flight
  for (size_t i0 = (size_t)bid * blockDim.x + threadIdx.x; i0 < n4; i0 += 2 * stride) {
    float4 pp[2], gg[2], mm[2], vv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const size_t i = i0 + u * stride;
      if (i < n4) {
        pp[u] = __ldcs(reinterpret_cast<float4*>(p) + i);
        gg[u] = __ldcs(reinterpret_cast<float4*>(g) + i);
        mm[u] = __ldcs(reinterpret_cast<float4*>(m) + i);
        vv[u] = __ldcs(reinterpret_cast<float4*>(v) + i);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const size_t i = i0 + u * stride;
      if (i < n4) {
        adam1(pp[u].x, gg[u].x, mm[u].x, vv[u].x, lr, b1, b2, eps, c1, c2);
        adam1(pp[u].y, gg[u].y, mm[u].y, vv[u].y, lr, b1, b2, eps, c1, c2);
        adam1(pp[u].z, gg[u].z, mm[u].z, vv[u].z, lr, b1, b2, eps, c1, c2);
        adam1(pp[u].w, gg[u].w, mm[u].w, vv[u].w, lr, b1, b2, eps, c1, c2);
        reinterpret_cast<float4*>(p)[i] = pp[u];
        __stcs(reinterpret_cast<float4*>(m) + i, mm[u]);
        __stcs(reinterpret_cast<float4*>(v) + i, vv[u]);
        if (zero_grad) reinterpret_cast<float4*>(g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  if (bid == 0 && threadIdx.x < n - n4 * 4) {
    const size_t i = n4 * 4 + threadIdx.x;
    float gi = g[i];
    adam1(p[i], gi, m[i], v[i], lr, b1, b2, eps, c1, c2);
    if (zero_grad) g[i] = 0.f;
  }
}

__global__ void __launch_bounds__(256) k_adam(size_t n, float* __restrict__ p, float* __restrict__ g,
                                              float* __restrict__ m, float* __restrict__ v, float lr, float b1,
                                              float b2, float eps, float c1, float c2, int zero_grad) {
  pdl_wait();  // the backward's gradient
  adam_body(n, p, g, m, v, lr, b1, b2, eps, c1, c2, zero_grad);
}

// Adam + the backward's MLP-gradient reduction (k_mlp_grad_reduce's job): blocks
// [0, nmlp) each reduce 32 MLP parameters over the nparts per-CTA partials (8 row
// groups per parameter, summed in fixed order: deterministic) and update them; the
// remaining blocks run the dense Adam over the hash table [0, hash_params). The
// reducing blocks come first, so they run in the first wave under the table stream.
__global__ void __launch_bounds__(256) k_adam_fused(size_t hash_params, int mlp_params, float* __restrict__ p,
                                                    float* __restrict__ g, float* __restrict__ m,
                                                    float* __restrict__ v, float lr, float b1, float b2, float eps,
                                                    float c1, float c2, const float* __restrict__ part, int nparts,
                                                    int nmlp) {
  pdl_wait();  // the backward's table gradient and partials
  if ((int)blockIdx.x >= nmlp) {
    adam_body(hash_params, p, g, m, v, lr, b1, b2, eps, c1, c2, 1, (int)blockIdx.x - nmlp, (int)gridDim.x - nmlp);
    return;
  }
  __shared__ float red[8][33];
  const int c = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int k = blockIdx.x * 32 + c;
  float a0 = 0.f, a1 = 0.f;
  if (k < mlp_params) {
    int r = grp;
    for (; r + 8 < nparts; r += 16) {
      a0 += part[(size_t)r * mlp_params + k];
      a1 += part[(size_t)(r + 8) * mlp_params + k];
    }
    if (r < nparts) a0 += part[(size_t)r * mlp_params + k];
  }
  red[grp][c] = a0 + a1;
  __syncthreads();
  if (grp == 0 && k < mlp_params) {
    float acc = red[0][c];
#pragma unroll
    for (int q = 1; q < 8; ++q) acc += red[q][c];
    const size_t i = hash_params + k;
    float gi = g[i] + acc;
    adam1(p[i], gi, m[i], v[i], lr, b1, b2, eps, c1, c2);
    g[i] = 0.f;
  }
}

// grouped (multi-object scheduler): blockIdx.y = object
__global__ void __launch_bounds__(256) k_adam_grp(const AdamJob* __restrict__ jobs) {
  pdl_wait();
  const AdamJob& j = jobs[blockIdx.y];
  adam_body(j.n, j.p, j.g, j.m, j.v, j.lr, j.b1, j.b2, j.eps, j.c1, j.c2, 1);
}

// --------------------------------------------------------- device init
// Same distributions as init_params (field.cpp:150-166): tables
// U(-1e-4, 1e-4), weights N(0,1)*sqrt(2/fan_in) (Box-Muller on Philox
// TAG_INIT draws), biases 0. Not the reference's mt19937 bits.
__global__ void k_init_params(FieldDesc fd, float* params, uint64_t seed) {
  const long long n = fd.hash_params + fd.mlp_params;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float val;
    if (i < fd.hash_params) {
      uint32_t x4[4];
      philox_draw(seed, PRENOM_TAG_INIT, 0u, 0u, (uint32_t)(i >> 2), x4);
      val = -1e-4f + 2e-4f * pdm_u01(x4[i & 3]);
    } else {
      const int j = (int)(i - fd.hash_params);
      int layer = 0;
      for (int l = 0; l <= fd.H; ++l)
        if (j >= fd.w_off[l]) layer = l;
      const int in = layer == 0 ? fd.in_dim : fd.W;
      if (j >= fd.b_off[layer]) {
        val = 0.f;
      } else {
        uint32_t x4[4];
        philox_draw(seed, PRENOM_TAG_INIT, 1u, 0u, (uint32_t)(j >> 1), x4);
        const int q = (j & 1) * 2;
        const float u1 = fmaxf(pdm_u01(x4[q]), 1e-7f), u2 = pdm_u01(x4[q + 1]);
        const float nrm = sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
        val = sqrtf(2.f / (float)in) * nrm;
      }
    }
    params[i] = val;
  }
}

__global__ void k_philox(int n, const uint32_t* ck, uint32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t ctr[4] = {ck[6 * i], ck[6 * i + 1], ck[6 * i + 2], ck[6 * i + 3]};
  uint32_t o[4];
  pdm_philox4x32_10(ctr, ck[6 * i + 4], ck[6 * i + 5], o);
  for (int j = 0; j < 4; ++j) out[4 * i + j] = o[j];
}

__global__ void k_reptile_delta(size_t n, const float* meta, const float* adapted, float* delta) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    delta[i] = __fsub_rn(adapted[i], meta[i]);
}

// Sum over a rank's adapted tasks of (theta_j - theta_meta), j in order, in one
// pass (k + 1 streams in, one out) -- the buffer the NCCL all-reduce sums
// across ranks. float4 main body, scalar tail.
__global__ void k_reptile_delta_sum(size_t n, const float* __restrict__ meta, const float* const* __restrict__ adapted,
                                    int k, float* __restrict__ out) {
  const size_t n4 = n / 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 m = reinterpret_cast<const float4*>(meta)[i];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(adapted[j]) + i);
      acc.x = __fadd_rn(acc.x, __fsub_rn(a.x, m.x));
      acc.y = __fadd_rn(acc.y, __fsub_rn(a.y, m.y));
      acc.z = __fadd_rn(acc.z, __fsub_rn(a.z, m.z));
      acc.w = __fadd_rn(acc.w, __fsub_rn(a.w, m.w));
    }
    reinterpret_cast<float4*>(out)[i] = acc;
  }
  for (size_t i = 4 * n4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float acc = 0.f;
    for (int j = 0; j < k; ++j) acc = __fadd_rn(acc, __fsub_rn(adapted[j][i], meta[i]));
    out[i] = acc;
  }
}

// meta.cpp:83-92 with adapted = meta + delta_sum / n_tasks.
__global__ void k_reptile_apply(size_t n, float* meta, const float* delta, float inv_n, float beta) {
  const float keep = __fsub_rn(1.f, beta);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float adapted = __fadd_rn(meta[i], __fmul_rn(delta[i], inv_n));
    meta[i] = __fadd_rn(__fmul_rn(keep, meta[i]), __fmul_rn(beta, adapted));
  }
}

// meta.cpp:83-92: out = keep * meta + beta * adapted (keep = 1 - beta), in place.
__global__ void k_reptile_update(size_t n, float* meta, const float* adapted, float beta) {
  const float keep = __fsub_rn(1.f, beta);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    meta[i] = __fadd_rn(__fmul_rn(keep, meta[i]), __fmul_rn(beta, adapted[i]));
}




}  // namespace

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_adam(size_t n, float* p, float* g, float* m, float* v, float lr, float b1, float b2, float eps,
                        float c1, float c2, int zero_grad, cudaStream_t st) {
  const size_t n4 = std::max<size_t>(n / 4, 1);
  // blocks per SM (4 resident at 64 registers): 20 for a step that has the GPU to itself
  // (cfg2: 0.1053 -> 0.1011 ms vs 8; 16-48 within 1%), 8 beside concurrent objects' kernels
  // on the lane streams (cfg3 0.9% slower at 24); PRENOM_ADAM_BLOCKS_PER_SM overrides
  static const int per_sm_env = [] {
    const char* e = getenv("PRENOM_ADAM_BLOCKS_PER_SM");
    return e ? atoi(e) : 0;
  }();
  const int per_sm = per_sm_env > 0 ? per_sm_env : (tc_concurrent_objects() ? 8 : 20);
  const unsigned grid = (unsigned)std::min<size_t>((n4 + 255) / 256, (size_t)num_sms() * per_sm);
  return launch_pdl(k_adam, dim3(grid), dim3(256), 0, st, n, p, g, m, v, lr, b1, b2, eps, c1, c2, zero_grad);
}

cudaError_t launch_adam_fused(size_t n, size_t hash_params, int mlp_params, float* p, float* g, float* m, float* v,
                              float lr, float b1, float b2, float eps, float c1, float c2, const float* part,
                              int nparts, cudaStream_t st) {
  if (!part || nparts <= 0 || hash_params % 4 != 0 || n != hash_params + (size_t)mlp_params)
    return cudaErrorInvalidValue;
  static const int per_sm_env = [] {
    const char* e = getenv("PRENOM_ADAM_BLOCKS_PER_SM");
    return e ? atoi(e) : 0;
  }();
  const int per_sm = per_sm_env > 0 ? per_sm_env : (tc_concurrent_objects() ? 8 : 20);
  const size_t n4 = std::max<size_t>(hash_params / 4, 1);
  const unsigned gmain = (unsigned)std::min<size_t>((n4 + 255) / 256, (size_t)num_sms() * per_sm);
  const int nmlp = (mlp_params + 31) / 32;
  return launch_pdl(k_adam_fused, dim3(gmain + (unsigned)nmlp), dim3(256), 0, st, hash_params, mlp_params, p, g, m, v,
                    lr, b1, b2, eps, c1, c2, part, nparts, nmlp);
}

cudaError_t launch_adam_group(const AdamJob* jobs_dev, int njobs, size_t n_max, cudaStream_t st) {
  if (njobs <= 0) return cudaSuccess;
  const size_t n4 = std::max<size_t>(n_max / 4, 1);
  const unsigned gx = (unsigned)std::max<size_t>(1, std::min<size_t>((n4 + 255) / 256, (size_t)num_sms() * 8 / njobs));
  return launch_pdl(k_adam_grp, dim3(gx, (unsigned)njobs), dim3(256), 0, st, jobs_dev);
}

cudaError_t launch_init_params(const FieldDesc& fd, float* params, uint64_t seed, cudaStream_t st) {
  k_init_params<<<num_sms() * 4, 256, 0, st>>>(fd, params, seed);
  return cudaGetLastError();
}

cudaError_t launch_philox(int n, const uint32_t* ck, uint32_t* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_philox<<<(n + 127) / 128, 128, 0, st>>>(n, ck, out);
  return cudaGetLastError();
}

cudaError_t launch_reptile_delta(size_t n, const float* meta, const float* adapted, float* delta, cudaStream_t st) {
  k_reptile_delta<<<num_sms() * 4, 256, 0, st>>>(n, meta, adapted, delta);
  return cudaGetLastError();
}

cudaError_t launch_reptile_delta_sum(size_t n, const float* meta, const float* const* adapted_dev, int k, float* out,
                                     cudaStream_t st) {
  k_reptile_delta_sum<<<num_sms() * 4, 256, 0, st>>>(n, meta, adapted_dev, k, out);
  return cudaGetLastError();
}

// L2 read probe: every thread sums float4s of a grid-stride walk over the buffer, reps times
__global__ void k_l2_read(const float4* __restrict__ buf, size_t n4, int reps, float* sink) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 v = __ldcg(buf + i);
      acc += (v.x + v.y) + (v.z + v.w);
    }
  sink[(blockIdx.x * blockDim.x + threadIdx.x) & ((1 << 20) - 1)] = acc;
}

cudaError_t launch_l2_read(const float4* buf, size_t n4, int reps, float* sink, cudaStream_t st, float* ms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  k_l2_read<<<num_sms() * 8, 512, 0, st>>>(buf, n4, reps, sink);
  cudaEventRecord(b, st);
  cudaError_t e = cudaEventSynchronize(b);
  if (ms) cudaEventElapsedTime(ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_reptile_update(size_t n, float* meta, const float* adapted, float beta, cudaStream_t st) {
  k_reptile_update<<<num_sms() * 4, 256, 0, st>>>(n, meta, adapted, beta);
  return cudaGetLastError();
}

cudaError_t launch_reptile_apply(size_t n, float* meta, const float* delta, float inv_n, float beta,
                                 cudaStream_t st) {
  k_reptile_apply<<<num_sms() * 4, 256, 0, st>>>(n, meta, delta, inv_n, beta);
  return cudaGetLastError();
}


}  // namespace prenom
