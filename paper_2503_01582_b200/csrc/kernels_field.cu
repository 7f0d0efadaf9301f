// kernels_field.cu -- hash-grid encode (fwd/bwd), the density+colour MLP
// (fp32 SIMT path), dense Adam, density query, device init.
//
// Replaces field.cpp: encode_point (64-99), field_eval (174-217),
// field_backward (227-293), adam_step (295-310), init_params (150-166) and
// density_grid.cpp: refresh_grid (119-132).
//
// Train-step data flow (per 128-sample tile, samples of one ray contiguous):
//   k_fwd_tile  : encode -> features (smem [in][128] + global SoA [in][N])
//                 -> MLP forward (smem GEMMs) -> (sigma, rgb) float4 / sample
//   (composite kernel: dL/dsigma, dL/drgb per sample)
//   k_bwd_tile  : MLP forward recompute from stored features -> g_raw ->
//                 backprop through the layers; weight grads accumulated per CTA
//                 in smem, one atomicAdd per weight per CTA; d_features -> SoA
//   k_encode_bwd: d_features x trilinear weights scattered into the table
//                 gradient (float2 vector atomics in L2)
//   k_adam      : dense, fused grad-zero, float4 vectorised
#include <cstdlib>

#include "prenom_device.cuh"

namespace prenom {
namespace {

constexpr int kFwdThreads = 256;
constexpr int kBwdThreads = 256;

// ------------------------------------------------------------ smem GEMMs
// Y[m][s] = epi( bias[m] + sum_k Wt(m,k) * X[k][s] ) over one 128-sample tile.
// Wt(m,k) = Wsm[m*rs + k*cs]. Lane owns samples 4*lane..4*lane+3 (float4),
// warp w owns rows w, w+nw, ... (weights are warp-broadcast smem reads).
// epi: 0 = identity, 1 = ReLU, 2 = gate by the existing Y (Y > 0 ? v : 0).
template <int NT, int MT>
__device__ __forceinline__ void tile_gemm(const float* __restrict__ Wsm, int rs, int cs,
                                          const float* __restrict__ bias, int M, int K,
                                          const float* X, float* Y, int ldy, int epi) {
  constexpr int nw = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int m0 = warp; m0 < M; m0 += nw * MT) {
    float4 acc[MT];
#pragma unroll
    for (int j = 0; j < MT; ++j) {
      const int m = m0 + j * nw;
      const float b = (bias && m < M) ? bias[m] : 0.f;
      acc[j] = make_float4(b, b, b, b);
    }
    for (int k = 0; k < K; ++k) {
      const float4 x = *reinterpret_cast<const float4*>(X + k * kLd + 4 * lane);
#pragma unroll
      for (int j = 0; j < MT; ++j) {
        const int m = m0 + j * nw;
        if (m < M) {
          const float w = Wsm[m * rs + k * cs];
          acc[j].x = fmaf(w, x.x, acc[j].x);
          acc[j].y = fmaf(w, x.y, acc[j].y);
          acc[j].z = fmaf(w, x.z, acc[j].z);
          acc[j].w = fmaf(w, x.w, acc[j].w);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < MT; ++j) {
      const int m = m0 + j * nw;
      if (m >= M) continue;
      float4* y = reinterpret_cast<float4*>(Y + (size_t)m * ldy + 4 * lane);
      float4 v = acc[j];
      if (epi == 1) {
        v.x = fmaxf(v.x, 0.f);
        v.y = fmaxf(v.y, 0.f);
        v.z = fmaxf(v.z, 0.f);
        v.w = fmaxf(v.w, 0.f);
      } else if (epi == 2) {
        const float4 g = *y;
        v.x = g.x > 0.f ? v.x : 0.f;
        v.y = g.y > 0.f ? v.y : 0.f;
        v.z = g.z > 0.f ? v.z : 0.f;
        v.w = g.w > 0.f ? v.w : 0.f;
      }
      *y = v;
    }
  }
}

// Register-blocked variant for the wide layers: Y[m][s] = epi(bias[m] +
// sum_k Wk[k*ldt + m] X[k][s]) with the weights k-major (a transposed copy
// for the forward, the reference layout W[o][i] itself for the backward
// data products). Warp w owns rows [w*MR, w*MR+MR) (M = 8*MR), lane owns
// samples 4*lane..4*lane+3: per k one conflict-free LDS.128 of X and MR/4
// broadcast LDS.128 of weights feed 4*MR FMAs (tile_gemm: 2 loads per 8).
template <int MR>
__device__ __forceinline__ void tile_gemm_rb(const float* Wk, int ldt, const float* bias, int K, const float* X,
                                             float* Y, int ldy, int epi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m0 = warp * MR;
  float4 acc[MR];
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    const float b = bias ? bias[m0 + j] : 0.f;
    acc[j] = make_float4(b, b, b, b);
  }
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    const float4 x = *reinterpret_cast<const float4*>(X + k * kLd + 4 * lane);
    float w[MR];
    if constexpr (MR % 4 == 0) {
#pragma unroll
      for (int q = 0; q < MR / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(Wk + k * ldt + m0 + 4 * q);
        w[4 * q] = v.x;
        w[4 * q + 1] = v.y;
        w[4 * q + 2] = v.z;
        w[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < MR; ++j) w[j] = Wk[k * ldt + m0 + j];
    }
#pragma unroll
    for (int j = 0; j < MR; ++j) {
      acc[j].x = fmaf(w[j], x.x, acc[j].x);
      acc[j].y = fmaf(w[j], x.y, acc[j].y);
      acc[j].z = fmaf(w[j], x.z, acc[j].z);
      acc[j].w = fmaf(w[j], x.w, acc[j].w);
    }
  }
#pragma unroll
  for (int j = 0; j < MR; ++j) {
    float4* y = reinterpret_cast<float4*>(Y + (size_t)(m0 + j) * ldy + 4 * lane);
    float4 v = acc[j];
    if (epi == 1) {
      v.x = fmaxf(v.x, 0.f);
      v.y = fmaxf(v.y, 0.f);
      v.z = fmaxf(v.z, 0.f);
      v.w = fmaxf(v.w, 0.f);
    } else if (epi == 2) {
      const float4 g = *y;
      v.x = g.x > 0.f ? v.x : 0.f;
      v.y = g.y > 0.f ? v.y : 0.f;
      v.z = g.z > 0.f ? v.z : 0.f;
      v.w = g.w > 0.f ? v.w : 0.f;
    }
    *y = v;
  }
}

// Y = epi(bias + W·X) for M output rows with k-major weights Wk[k*ldt + m]:
// the register-blocked kernel when 8 warps split M evenly (M = 16..64),
// else tile_gemm on the same layout (rs = 1, cs = ldt).
template <int NT>
__device__ __forceinline__ void gemm_kmajor(const float* Wk, int ldt, const float* bias, int M, int K,
                                            const float* X, float* Y, int ldy, int epi) {
  static_assert(NT == 256, "8 warps");
  switch (M) {
    case 64: tile_gemm_rb<8>(Wk, ldt, bias, K, X, Y, ldy, epi); return;
    case 32: tile_gemm_rb<4>(Wk, ldt, bias, K, X, Y, ldy, epi); return;
    case 24: tile_gemm_rb<3>(Wk, ldt, bias, K, X, Y, ldy, epi); return;
    case 16: tile_gemm_rb<2>(Wk, ldt, bias, K, X, Y, ldy, epi); return;
    default: tile_gemm<NT, 1>(Wk, 1, ldt, bias, M, K, X, Y, ldy, epi);
  }
}

// Stage the MLP block transposed (per layer W[o][i] -> Wt[i][o] at the same
// offset; biases as they are) for gemm_kmajor's forward products.
__device__ __forceinline__ void stage_mlp_transposed(const FieldDesc& fd, const float* __restrict__ mlp, float* Wt,
                                                     int nt) {
  int in = fd.in_dim;
  for (int l = 0; l <= fd.H; ++l) {
    const int out = l < fd.H ? fd.W : 4;
    const float* W = mlp + fd.w_off[l];
    float* T = Wt + fd.w_off[l];
    for (int i = threadIdx.x; i < out * in; i += nt) {
      const int o = i / in, k = i % in;
      T[k * out + o] = __ldg(W + i);
    }
    for (int i = threadIdx.x; i < out; i += nt) Wt[fd.b_off[l] + i] = __ldg(mlp + fd.b_off[l] + i);
    in = out;
  }
}

// acc[m*ldw + k] += sum_s A[m][s] * B[k][s] over the tile (weight gradient).
// Warp tile 16(m) x 32(k): lane (tm = lane>>3, tk = lane&7) owns rows
// tm + 4i and columns tk + 8j (i, j < 4), so the 8 lanes of an LDS.128
// wavefront read 8 consecutive B rows (distinct bank groups with kLd = 132)
// and share one A row (broadcast).
template <int NT>
__device__ __forceinline__ void tile_wgrad(const float* A, int M, const float* B, int K,
                                           float* acc, int ldw) {
  constexpr int nw = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tm = lane >> 3, tk = lane & 7;
  const int mt = (M + 15) / 16, kt = (K + 31) / 32;
  for (int t = warp; t < mt * kt; t += nw) {
    const int mb = (t / kt) * 16 + tm, kb = (t % kt) * 32 + tk;
    float c[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
    for (int s = 0; s < kTile; s += 4) {
      float4 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = mb + 4 * i;
        a[i] = m < M ? *reinterpret_cast<const float4*>(A + m * kLd + s) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = kb + 8 * j;
        b[j] = k < K ? *reinterpret_cast<const float4*>(B + k * kLd + s) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          c[i][j] = fmaf(a[i].x, b[j].x, c[i][j]);
          c[i][j] = fmaf(a[i].y, b[j].y, c[i][j]);
          c[i][j] = fmaf(a[i].z, b[j].z, c[i][j]);
          c[i][j] = fmaf(a[i].w, b[j].w, c[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int m = mb + 4 * i, k = kb + 8 * j;
        if (m < M && k < K) acc[m * ldw + k] += c[i][j];
      }
  }
}

// acc[m] += sum_s A[m][s] (bias gradient)
template <int NT>
__device__ __forceinline__ void tile_bgrad(const float* A, int M, float* acc) {
  for (int m = threadIdx.x; m < M; m += NT) {
    float s = 0.f;
    for (int i = 0; i < kTile; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(A + m * kLd + i);
      s += (v.x + v.y) + (v.z + v.w);
    }
    acc[m] += s;
  }
}

__device__ __forceinline__ bool sample_valid(long long s, long long n_total, int S,
                                             const int* __restrict__ count) {
  if (s >= n_total) return false;
  return __ldg(count + s / S) > 0;
}

// Encode one tile into smem X[in][kLd] (and global SoA), 2 threads/sample.
template <int F>
__device__ __forceinline__ void encode_tile(const FieldDesc& fd, const float* __restrict__ params,
                                            long long tile0, long long n_total, int S,
                                            const int* count, const float4* __restrict__ pos,
                                            float* X, float* feat_t, long long ld_t) {
  const int s = threadIdx.x & (kTile - 1);
  const int half = threadIdx.x >> 7;  // 0/1 (kFwdThreads == 256)
  const long long gs = tile0 + s;
  const bool valid = sample_valid(gs, n_total, S, count);
  float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) p = pos[gs];
  const float px = clamp01(p.x), py = clamp01(p.y), pz = clamp01(p.z);
  for (int l = half; l < fd.L; l += 2) {
    float f[F];
    if (valid) {
      encode_level<F>(fd, params, l, px, py, pz, f);
    } else {
#pragma unroll
      for (int j = 0; j < F; ++j) f[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < F; ++j) {
      X[(l * F + j) * kLd + s] = f[j];
      if (feat_t && gs < n_total) feat_t[(long long)(l * F + j) * ld_t + gs] = f[j];
    }
  }
}

__device__ __forceinline__ void encode_tile_rt(const FieldDesc& fd, const float* __restrict__ params,
                                               long long tile0, long long n_total, int S,
                                               const int* count, const float4* __restrict__ pos,
                                               float* X, float* feat_t, long long ld_t) {
  const int s = threadIdx.x & (kTile - 1);
  const int half = threadIdx.x >> 7;
  const long long gs = tile0 + s;
  const bool valid = sample_valid(gs, n_total, S, count);
  float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) p = pos[gs];
  const float px = clamp01(p.x), py = clamp01(p.y), pz = clamp01(p.z);
  for (int l = half; l < fd.L; l += 2) {
    float f[4] = {0.f, 0.f, 0.f, 0.f};
    if (valid) encode_level_rt(fd, params, l, px, py, pz, f);
    for (int j = 0; j < fd.F; ++j) {
      X[(l * fd.F + j) * kLd + s] = f[j];
      if (feat_t && gs < n_total) feat_t[(long long)(l * fd.F + j) * ld_t + gs] = f[j];
    }
  }
}

// Forward MLP over the tile: X (in) -> hidden buffers Hb[l] -> RAW[4][kLd];
// Wt = the MLP block staged by stage_mlp_transposed.
template <int NT>
__device__ __forceinline__ void mlp_forward_tile(const FieldDesc& fd, const float* Wt, const float* X,
                                                 float* Hb, float* RAW) {
  const float* in = X;
  int in_dim = fd.in_dim;
  for (int l = 0; l < fd.H; ++l) {
    float* out = Hb + (size_t)l * fd.W * kLd;
    gemm_kmajor<NT>(Wt + fd.w_off[l], fd.W, Wt + fd.b_off[l], fd.W, in_dim, in, out, kLd, 1);
    __syncthreads();
    in = out;
    in_dim = fd.W;
  }
  gemm_kmajor<NT>(Wt + fd.w_off[fd.H], 4, Wt + fd.b_off[fd.H], 4, in_dim, in, RAW, kLd, 0);
  __syncthreads();
}

// ------------------------------------------------------------ fwd (train)
__global__ void __launch_bounds__(kFwdThreads) k_fwd_tile(FieldDesc fd, const float* __restrict__ params,
                                                          long long n_total, int S, const int* count,
                                                          const float4* __restrict__ pos, float* feat_t,
                                                          long long ld_t, float4* out, int* flag) {
  extern __shared__ __align__(16) float sm[];
  float* X = sm;
  float* Hb = X + (size_t)fd.in_dim * kLd;
  float* RAW = Hb + (size_t)fd.H * fd.W * kLd;
  float* Wsm = RAW + 4 * kLd;
  stage_mlp_transposed(fd, params + fd.hash_params, Wsm, kFwdThreads);
  const long long ntiles = (n_total + kTile - 1) / kTile;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long tile0 = t * kTile;
    if (fd.F == 2)
      encode_tile<2>(fd, params, tile0, n_total, S, count, pos, X, feat_t, ld_t);
    else
      encode_tile_rt(fd, params, tile0, n_total, S, count, pos, X, feat_t, ld_t);
    __syncthreads();
    mlp_forward_tile<kFwdThreads>(fd, Wsm, X, Hb, RAW);  // Wsm holds the transposed block
    if (threadIdx.x < kTile) {
      const int s = threadIdx.x;
      const long long gs = tile0 + s;
      if (gs < n_total) {
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        if (sample_valid(gs, n_total, S, count)) {
          o.x = density_forward(fd.act, RAW[s]);
          o.y = stable_sigmoid(RAW[kLd + s]);
          o.z = stable_sigmoid(RAW[2 * kLd + s]);
          o.w = stable_sigmoid(RAW[3 * kLd + s]);
          if (!all_finite4(o.x, o.y, o.z, o.w)) atomicOr(flag, 1);
        }
        out[gs] = o;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ bwd (train)
__global__ void __launch_bounds__(kBwdThreads) k_bwd_tile(FieldDesc fd, const float* __restrict__ params,
                                                          float* grad, long long n_total, int S,
                                                          const int* count, const float* __restrict__ feat_t,
                                                          long long ld_t, const float4* __restrict__ dout,
                                                          float* dfeat_t) {
  extern __shared__ __align__(16) float sm[];
  float* X = sm;
  float* Hb = X + (size_t)fd.in_dim * kLd;
  float* RAW = Hb + (size_t)fd.H * fd.W * kLd;
  float* G = RAW + 4 * kLd;
  float* Wsm = G + 4 * kLd;                            // reference layout (backward products)
  float* Acc = Wsm + ((fd.mlp_params + 3) & ~3);
  float* Wt = Acc + ((fd.mlp_params + 3) & ~3);         // transposed (forward recompute)
  const float* mlp = params + fd.hash_params;
  for (int i = threadIdx.x; i < fd.mlp_params; i += kBwdThreads) {
    Wsm[i] = __ldg(mlp + i);
    Acc[i] = 0.f;
  }
  stage_mlp_transposed(fd, mlp, Wt, kBwdThreads);
  __syncthreads();
  const long long ntiles = (n_total + kTile - 1) / kTile;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long tile0 = t * kTile;
    // stored features (SoA, coalesced) -> X; invalid samples -> 0
    for (int i = threadIdx.x; i < fd.in_dim * (kTile / 4); i += kBwdThreads) {
      const int row = i / (kTile / 4), q = i % (kTile / 4);
      const long long gs = tile0 + 4 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gs + 3 < n_total) {
        v = *reinterpret_cast<const float4*>(feat_t + (long long)row * ld_t + gs);
      } else {
        float tmp[4] = {0.f, 0.f, 0.f, 0.f};
        for (int j = 0; j < 4; ++j)
          if (gs + j < n_total) tmp[j] = feat_t[(long long)row * ld_t + gs + j];
        v = make_float4(tmp[0], tmp[1], tmp[2], tmp[3]);
      }
      *reinterpret_cast<float4*>(X + row * kLd + 4 * q) = v;
    }
    __syncthreads();
    mlp_forward_tile<kBwdThreads>(fd, Wt, X, Hb, RAW);
    // g_raw (field.cpp:233-238)
    if (threadIdx.x < kTile) {
      const int s = threadIdx.x;
      const long long gs = tile0 + s;
      float g0 = 0.f, g1 = 0.f, g2 = 0.f, g3 = 0.f;
      if (sample_valid(gs, n_total, S, count)) {
        const float4 d = dout[gs];
        const float r0 = RAW[s];
        const float sg = density_forward(fd.act, r0);
        g0 = d.x * density_derivative(fd.act, r0, sg);
        const float s1 = stable_sigmoid(RAW[kLd + s]);
        const float s2 = stable_sigmoid(RAW[2 * kLd + s]);
        const float s3 = stable_sigmoid(RAW[3 * kLd + s]);
        g1 = d.y * s1 * (1.f - s1);
        g2 = d.z * s2 * (1.f - s2);
        g3 = d.w * s3 * (1.f - s3);
      }
      G[s] = g0;
      G[kLd + s] = g1;
      G[2 * kLd + s] = g2;
      G[3 * kLd + s] = g3;
    }
    __syncthreads();
    // output layer
    const int H = fd.H;
    const float* last = H > 0 ? Hb + (size_t)(H - 1) * fd.W * kLd : X;
    const int last_dim = H > 0 ? fd.W : fd.in_dim;
    tile_wgrad<kBwdThreads>(G, 4, last, last_dim, Acc + fd.w_off[H], last_dim);
    tile_bgrad<kBwdThreads>(G, 4, Acc + fd.b_off[H]);
    __syncthreads();
    // D_{H-1} = gate(H_{H-1}) * (W_out^T G), in place
    gemm_kmajor<kBwdThreads>(Wsm + fd.w_off[H], last_dim, nullptr, last_dim, 4, G,
                             Hb + (size_t)(H - 1) * fd.W * kLd, kLd, 2);
    __syncthreads();
    for (int l = H - 1; l >= 0; --l) {
      float* D = Hb + (size_t)l * fd.W * kLd;
      const float* prev = l > 0 ? Hb + (size_t)(l - 1) * fd.W * kLd : X;
      const int prev_dim = l > 0 ? fd.W : fd.in_dim;
      tile_wgrad<kBwdThreads>(D, fd.W, prev, prev_dim, Acc + fd.w_off[l], prev_dim);
      tile_bgrad<kBwdThreads>(D, fd.W, Acc + fd.b_off[l]);
      __syncthreads();
      if (l > 0) {
        gemm_kmajor<kBwdThreads>(Wsm + fd.w_off[l], prev_dim, nullptr, prev_dim, fd.W, D,
                                 Hb + (size_t)(l - 1) * fd.W * kLd, kLd, 2);
      } else {
        // d_features straight to global SoA (no gate)
        if (tile0 + kTile <= n_total) {
          gemm_kmajor<kBwdThreads>(Wsm + fd.w_off[0], fd.in_dim, nullptr, fd.in_dim, fd.W, D, dfeat_t + tile0,
                                   (int)ld_t, 0);
        } else {
          gemm_kmajor<kBwdThreads>(Wsm + fd.w_off[0], fd.in_dim, nullptr, fd.in_dim, fd.W, D, X, kLd, 0);
          __syncthreads();
          for (int i = threadIdx.x; i < fd.in_dim * kTile; i += kBwdThreads) {
            const int row = i / kTile, s = i % kTile;
            if (tile0 + s < n_total) dfeat_t[(long long)row * ld_t + tile0 + s] = X[row * kLd + s];
          }
        }
      }
      __syncthreads();
    }
  }
  // one atomic per MLP parameter per CTA
  float* gm = grad + fd.hash_params;
  for (int i = threadIdx.x; i < fd.mlp_params; i += kBwdThreads)
    if (Acc[i] != 0.f) atomicAdd(gm + i, Acc[i]);
}

// ------------------------------------------------------- encode backward
// thread per (sample, level); blockIdx.y = level (warp-uniform dense/hash).
template <int F>
__global__ void __launch_bounds__(256) k_encode_bwd(FieldDesc fd, float* grad, long long n_total, int S,
                                                    const int* count, const float4* __restrict__ pos,
                                                    const float* __restrict__ dfeat_t, long long ld_t) {
  // Consecutive lanes = consecutive depth-sorted samples of a ray: equal
  // (ray, cell) keys form contiguous runs; a segmented suffix sum leaves each
  // run's corner totals in its first lane, which alone issues the atomics.
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y, lane = threadIdx.x & 31;
  const bool valid = sample_valid(s, n_total, S, count);
  float d[F];
#pragma unroll
  for (int j = 0; j < F; ++j) d[j] = valid ? dfeat_t[(long long)(l * F + j) * ld_t + s] : 0.f;
  float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) p = pos[s];
  const LevelCell c = level_cell(fd.res[l], clamp01(p.x), clamp01(p.y), clamp01(p.z));
  const unsigned long long key =
      (valid && fd.res[l] < 4096)
          ? (((unsigned long long)(s / S) << 36) | ((unsigned long long)c.cz << 24) | ((unsigned long long)c.cy << 12) |
             (unsigned long long)c.cx)
          : (~0ull - (unsigned long long)lane);
  float v[8][F];
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    const float w = corner_weight(c, corner);
#pragma unroll
    for (int j = 0; j < F; ++j) v[corner][j] = w * d[j];
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long ok = __shfl_down_sync(0xffffffffu, key, off);
    const bool take = (lane + off < 32) && ok == key;
    if (!__any_sync(0xffffffffu, take)) break;  // no run longer than off
#pragma unroll
    for (int corner = 0; corner < 8; ++corner)
#pragma unroll
      for (int j = 0; j < F; ++j) {
        const float t = __shfl_down_sync(0xffffffffu, v[corner][j], off);
        if (take) v[corner][j] += t;
      }
  }
  const unsigned long long pk = __shfl_up_sync(0xffffffffu, key, 1);
  if (!valid || (lane != 0 && pk == key)) return;
  float* g = grad + (long long)l * F * fd.rows;
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    bool any = false;
#pragma unroll
    for (int j = 0; j < F; ++j) any |= v[corner][j] != 0.f;
    if (!any) continue;
    const uint32_t row = table_row(fd, l, (uint32_t)(c.cx + (corner & 1)), (uint32_t)(c.cy + ((corner >> 1) & 1)),
                                   (uint32_t)(c.cz + ((corner >> 2) & 1)));
    if constexpr (F == 2) {
      atomicAdd(reinterpret_cast<float2*>(g + (size_t)row * 2), make_float2(v[corner][0], v[corner][1]));
    } else {
#pragma unroll
      for (int j = 0; j < F; ++j) atomicAdd(g + (size_t)row * F + j, v[corner][j]);
    }
  }
}

__global__ void __launch_bounds__(256) k_encode_bwd_rt(FieldDesc fd, float* grad, long long n_total, int S,
                                                       const int* count, const float4* __restrict__ pos,
                                                       const float* __restrict__ dfeat_t, long long ld_t) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y, F = fd.F;
  if (!sample_valid(s, n_total, S, count)) return;
  const float4 p = pos[s];
  const LevelCell c = level_cell(fd.res[l], clamp01(p.x), clamp01(p.y), clamp01(p.z));
  float* g = grad + (long long)l * F * fd.rows;
  for (int corner = 0; corner < 8; ++corner) {
    const float w = corner_weight(c, corner);
    if (w == 0.f) continue;
    const uint32_t row = table_row(fd, l, (uint32_t)(c.cx + (corner & 1)), (uint32_t)(c.cy + ((corner >> 1) & 1)),
                                   (uint32_t)(c.cz + ((corner >> 2) & 1)));
    for (int j = 0; j < F; ++j) {
      const float d = dfeat_t[(long long)(l * F + j) * ld_t + s];
      if (d != 0.f) atomicAdd(g + (size_t)row * F + j, w * d);
    }
  }
}

// ------------------------------------------------- per-point exact field
// field_eval for arbitrary points, one thread per point, operation order of
// field.cpp:174-217 with *_rn intrinsics (pre-activations bit-exact).
__global__ void __launch_bounds__(128) k_field_points(FieldDesc fd, const float* __restrict__ params, int n,
                                                      const float* __restrict__ xyz, int grid_R, float* sigma,
                                                      float* rgb, float* raw_out, float* feat_out, int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float px, py, pz;
  if (grid_R > 0) {  // refresh_grid lattice point (density_grid.cpp:121-128)
    const float scale = __fdiv_rn(1.f, (float)(grid_R - 1));
    const int ix = i % grid_R, iy = (i / grid_R) % grid_R, iz = i / (grid_R * grid_R);
    px = __fmul_rn((float)ix, scale);
    py = __fmul_rn((float)iy, scale);
    pz = __fmul_rn((float)iz, scale);
  } else {
    px = xyz[3 * i];
    py = xyz[3 * i + 1];
    pz = xyz[3 * i + 2];
  }
  px = clamp01(px);
  py = clamp01(py);
  pz = clamp01(pz);
  float x[kMaxIn > kMaxWidth ? kMaxIn : kMaxWidth];
  float h[kMaxWidth];
  for (int l = 0; l < fd.L; ++l) encode_level_rt(fd, params, l, px, py, pz, x + l * fd.F);
  if (feat_out)
    for (int j = 0; j < fd.in_dim; ++j) feat_out[(size_t)i * fd.in_dim + j] = x[j];
  const float* mlp = params + fd.hash_params;
  int in = fd.in_dim;
  for (int l = 0; l < fd.H; ++l) {
    const float* Wl = mlp + fd.w_off[l];
    const float* bl = mlp + fd.b_off[l];
    for (int o = 0; o < fd.W; ++o) {
      float s = __ldg(bl + o);
      for (int k = 0; k < in; ++k) s = __fadd_rn(s, __fmul_rn(__ldg(Wl + o * in + k), x[k]));
      h[o] = s > 0.f ? s : 0.f;
    }
    for (int o = 0; o < fd.W; ++o) x[o] = h[o];
    in = fd.W;
  }
  float raw[4];
  const float* Wo = mlp + fd.w_off[fd.H];
  const float* bo = mlp + fd.b_off[fd.H];
  for (int o = 0; o < 4; ++o) {
    float s = __ldg(bo + o);
    for (int k = 0; k < in; ++k) s = __fadd_rn(s, __fmul_rn(__ldg(Wo + o * in + k), x[k]));
    raw[o] = s;
  }
  const float sg = density_forward(fd.act, raw[0]);
  const float c0 = stable_sigmoid(raw[1]), c1 = stable_sigmoid(raw[2]), c2 = stable_sigmoid(raw[3]);
  if (!all_finite4(sg, c0, c1, c2) && flag) atomicOr(flag, 1);
  if (sigma) sigma[i] = sg;
  if (rgb) {
    rgb[3 * i] = c0;
    rgb[3 * i + 1] = c1;
    rgb[3 * i + 2] = c2;
  }
  if (raw_out)
    for (int o = 0; o < 4; ++o) raw_out[4 * (size_t)i + o] = raw[o];
}

// Specialised exact field for the BASELINE family (F = 2, L*F = INP, hidden
// width W, H hidden layers): identical per-point arithmetic to
// k_field_points (same *_rn sums, each output's terms added in the same
// ascending k order, so the same bits), laid out for throughput:
//   * the MLP is staged once per CTA in shared memory TRANSPOSED ([in][out]),
//     read as warp-broadcast float4 over outputs;
//   * a layer walks k in a rolled loop and updates all W accumulators
//     (registers) per step -- W independent add chains, small code;
//   * activations live in a per-thread shared-memory column act[k][tid]
//     (conflict-free), so the loop index stays dynamic without local memory.
// (The generic kernel keeps runtime-sized x[]/h[] in local memory and
// re-reads each weight through L1 per multiply.) Used for refresh_grid,
// density queries and field_eval (cfg5: 128^3 refreshes, the 256^3 query).
constexpr int kFpThreads = 128;
template <int INP, int W, int H>
struct FpSmem {
  static constexpr int kW0 = 0, kB0 = INP * W, kL1 = kB0 + W;
  static constexpr int kWo = kL1 + (H - 1) * (W * W + W), kBo = kWo + 4 * W;
  static constexpr int kWeights = (kBo + 4 + 3) / 4 * 4;
  static constexpr int kAct = (INP > W ? INP : W) * kFpThreads;  // act[k][tid]
  static constexpr size_t kBytes = (size_t)(kWeights + kAct) * sizeof(float);
};

// out[o] = b[o] + sum_k W[o][k] act[k], k ascending (field.cpp:181-211)
template <int NIN, int NOUT>
__device__ __forceinline__ void fp_layer(const float* WT, const float* b, const float* act, float* out) {
#pragma unroll
  for (int o = 0; o < NOUT; ++o) out[o] = b[o];
#pragma unroll 2
  for (int k = 0; k < NIN; ++k) {
    const float xk = act[k * kFpThreads];
    const float4* wr = reinterpret_cast<const float4*>(WT + k * NOUT);
#pragma unroll
    for (int o4 = 0; o4 < NOUT / 4; ++o4) {
      const float4 w = wr[o4];
      out[4 * o4] = __fadd_rn(out[4 * o4], __fmul_rn(w.x, xk));
      out[4 * o4 + 1] = __fadd_rn(out[4 * o4 + 1], __fmul_rn(w.y, xk));
      out[4 * o4 + 2] = __fadd_rn(out[4 * o4 + 2], __fmul_rn(w.z, xk));
      out[4 * o4 + 3] = __fadd_rn(out[4 * o4 + 3], __fmul_rn(w.w, xk));
    }
  }
}

template <int INP, int W, int H>
__global__ void __launch_bounds__(kFpThreads) k_field_points_t(FieldDesc fd, const float* __restrict__ params, int n,
                                                               const float* __restrict__ xyz, int grid_R, float* sigma,
                                                               float* rgb, float* raw_out, float* feat_out, int* flag) {
  using SM = FpSmem<INP, W, H>;
  extern __shared__ __align__(16) float wsm[];
  {
    const float* mlp = params + fd.hash_params;  // reference layout: W[out][in], b[out] per layer
    for (int j = threadIdx.x; j < INP * W; j += blockDim.x) wsm[SM::kW0 + j] = __ldg(mlp + (j % W) * INP + j / W);
    for (int j = threadIdx.x; j < W; j += blockDim.x) wsm[SM::kB0 + j] = __ldg(mlp + W * INP + j);
    if constexpr (H == 2) {
      const float* m1 = mlp + W * INP + W;
      for (int j = threadIdx.x; j < W * W; j += blockDim.x) wsm[SM::kL1 + j] = __ldg(m1 + (j % W) * W + j / W);
      for (int j = threadIdx.x; j < W; j += blockDim.x) wsm[SM::kL1 + W * W + j] = __ldg(m1 + W * W + j);
    }
    const float* mo = mlp + W * INP + W + (H - 1) * (W * W + W);
    for (int j = threadIdx.x; j < 4 * W; j += blockDim.x) wsm[SM::kWo + j] = __ldg(mo + (j % 4) * W + j / 4);
    if (threadIdx.x < 4) wsm[SM::kBo + threadIdx.x] = __ldg(mo + 4 * W + threadIdx.x);
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float* act = wsm + SM::kWeights + threadIdx.x;  // act[k * kFpThreads]
  float px, py, pz;
  if (grid_R > 0) {  // refresh_grid lattice point (density_grid.cpp:121-128)
    const float scale = __fdiv_rn(1.f, (float)(grid_R - 1));
    const int ix = i % grid_R, iy = (i / grid_R) % grid_R, iz = i / (grid_R * grid_R);
    px = __fmul_rn((float)ix, scale);
    py = __fmul_rn((float)iy, scale);
    pz = __fmul_rn((float)iz, scale);
  } else {
    px = xyz[3 * i];
    py = xyz[3 * i + 1];
    pz = xyz[3 * i + 2];
  }
  px = clamp01(px);
  py = clamp01(py);
  pz = clamp01(pz);
  for (int l = 0; l < INP / 2; ++l) {
    float f2[2];
    encode_level<2>(fd, params, l, px, py, pz, f2);
    act[(2 * l) * kFpThreads] = f2[0];
    act[(2 * l + 1) * kFpThreads] = f2[1];
    if (feat_out) {
      feat_out[(size_t)i * INP + 2 * l] = f2[0];
      feat_out[(size_t)i * INP + 2 * l + 1] = f2[1];
    }
  }
  float h[W];
  fp_layer<INP, W>(wsm + SM::kW0, wsm + SM::kB0, act, h);
#pragma unroll
  for (int o = 0; o < W; ++o) act[o * kFpThreads] = h[o] > 0.f ? h[o] : 0.f;
  if constexpr (H == 2) {
    fp_layer<W, W>(wsm + SM::kL1, wsm + SM::kL1 + W * W, act, h);
#pragma unroll
    for (int o = 0; o < W; ++o) act[o * kFpThreads] = h[o] > 0.f ? h[o] : 0.f;
  }
  float raw[4];
  fp_layer<W, 4>(wsm + SM::kWo, wsm + SM::kBo, act, raw);
  const float sg = density_forward(fd.act, raw[0]);
  const float c0 = stable_sigmoid(raw[1]), c1 = stable_sigmoid(raw[2]), c2 = stable_sigmoid(raw[3]);
  if (!all_finite4(sg, c0, c1, c2) && flag) atomicOr(flag, 1);
  if (sigma) sigma[i] = sg;
  if (rgb) {
    rgb[3 * i] = c0;
    rgb[3 * i + 1] = c1;
    rgb[3 * i + 2] = c2;
  }
  if (raw_out)
#pragma unroll
    for (int o = 0; o < 4; ++o) raw_out[4 * (size_t)i + o] = raw[o];
}

template <int INP, int W, int H>
cudaError_t run_field_points_t(const FieldDesc& fd, const float* params, int n, const float* xyz, int R, float* sigma,
                               float* rgb, float* raw, float* features, int* flag, cudaStream_t st) {
  const size_t smem = FpSmem<INP, W, H>::kBytes;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_field_points_t<INP, W, H>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_field_points_t<INP, W, H><<<(unsigned)((n + kFpThreads - 1) / kFpThreads), kFpThreads, smem, st>>>(
      fd, params, n, xyz, R, sigma, rgb, raw, features, flag);
  return cudaGetLastError();
}

// true (and launched) when the arch has a specialised exact kernel
bool field_points_fast(const FieldDesc& fd, const float* params, int n, const float* xyz, int R, float* sigma,
                       float* rgb, float* raw, float* features, int* flag, cudaStream_t st, cudaError_t* err) {
  if (fd.F != 2 || fd.mlp_params != fd.b_off[fd.H] + 4) return false;
#define PRENOM_FP_CASE(L_, W_, H_)                                                                       \
  if (fd.L == L_ && fd.W == W_ && fd.H == H_) {                                                        \
    *err = run_field_points_t<2 * L_, W_, H_>(fd, params, n, xyz, R, sigma, rgb, raw, features, flag, st); \
    return true;                                                                                       \
  }
  PRENOM_FP_CASE(8, 32, 1) PRENOM_FP_CASE(8, 32, 2) PRENOM_FP_CASE(8, 64, 1) PRENOM_FP_CASE(8, 64, 2)
  PRENOM_FP_CASE(12, 32, 1) PRENOM_FP_CASE(12, 32, 2) PRENOM_FP_CASE(12, 64, 1) PRENOM_FP_CASE(12, 64, 2)
  PRENOM_FP_CASE(16, 32, 1) PRENOM_FP_CASE(16, 32, 2) PRENOM_FP_CASE(16, 64, 1) PRENOM_FP_CASE(16, 64, 2)
#undef PRENOM_FP_CASE
  return false;
}

}  // namespace

static size_t fwd_smem_bytes(const FieldDesc& fd) {
  return sizeof(float) * ((size_t)fd.in_dim * kLd + (size_t)fd.H * fd.W * kLd + 4 * kLd +
                          ((fd.mlp_params + 3) & ~3));
}

static size_t bwd_smem_bytes(const FieldDesc& fd) {
  return sizeof(float) * ((size_t)fd.in_dim * kLd + (size_t)fd.H * fd.W * kLd + 8 * kLd +
                          3 * ((fd.mlp_params + 3) & ~3));
}

cudaError_t launch_field_fwd_train(const FieldDesc& fd, const float* params, int B, int S,
                                   const SampleBufs& sb, float* features_t, float4* out, int* flag,
                                   cudaStream_t st) {
  const long long n = (long long)B * S;
  if (n == 0) return cudaSuccess;
  const size_t smem = fwd_smem_bytes(fd);
  cudaError_t e = cudaFuncSetAttribute(k_fwd_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long ntiles = (n + kTile - 1) / kTile;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fwd_tile, kFwdThreads, smem);
  const long long grid = std::min<long long>(ntiles, (long long)num_sms() * std::max(per_sm, 1));
  const long long ld = ((n + kTile - 1) / kTile) * kTile;
  k_fwd_tile<<<(unsigned)grid, kFwdThreads, smem, st>>>(fd, params, n, S, sb.count, sb.pos_depth, features_t, ld,
                                                        out, flag);
  return cudaGetLastError();
}

cudaError_t launch_mlp_bwd_train(const FieldDesc& fd, const float* params, float* grad, int B, int S,
                                 const int* count, const float* features_t, const float4* dout, float* dfeat_t,
                                 cudaStream_t st) {
  const long long n = (long long)B * S;
  if (n == 0) return cudaSuccess;
  const size_t smem = bwd_smem_bytes(fd);
  cudaError_t e = cudaFuncSetAttribute(k_bwd_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long ntiles = (n + kTile - 1) / kTile;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bwd_tile, kBwdThreads, smem);
  const long long grid = std::min<long long>(ntiles, (long long)num_sms() * std::max(per_sm, 1));
  const long long ld = ((n + kTile - 1) / kTile) * kTile;
  k_bwd_tile<<<(unsigned)grid, kBwdThreads, smem, st>>>(fd, params, grad, n, S, count, features_t, ld, dout,
                                                        dfeat_t);
  return cudaGetLastError();
}

cudaError_t launch_encode_bwd(const FieldDesc& fd, const float* /*params*/, float* grad, int B, int S,
                              const int* count, const float4* pos_depth, const float* dfeat_t, cudaStream_t st) {
  const long long n = (long long)B * S;
  if (n == 0) return cudaSuccess;
  const long long ld = ((n + kTile - 1) / kTile) * kTile;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)fd.L);
  if (fd.F == 2)
    k_encode_bwd<2><<<grid, 256, 0, st>>>(fd, grad, n, S, count, pos_depth, dfeat_t, ld);
  else
    k_encode_bwd_rt<<<grid, 256, 0, st>>>(fd, grad, n, S, count, pos_depth, dfeat_t, ld);
  return cudaGetLastError();
}

cudaError_t launch_field_points(const FieldDesc& fd, const float* params, int n, const float* xyz, float* sigma,
                                float* rgb, float* raw, float* features, int* flag, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  if (!getenv("PRENOM_GENERIC_FIELD") && field_points_fast(fd, params, n, xyz, 0, sigma, rgb, raw, features, flag, st, &e))
    return e;
  k_field_points<<<(n + 127) / 128, 128, 0, st>>>(fd, params, n, xyz, 0, sigma, rgb, raw, features, flag);
  return cudaGetLastError();
}

cudaError_t launch_refresh_grid(const FieldDesc& fd, const float* params, int R, float* out, int* flag,
                                cudaStream_t st) {
  const long long n = (long long)R * R * R;
  cudaError_t e = cudaSuccess;
  if (!getenv("PRENOM_GENERIC_FIELD") &&
      field_points_fast(fd, params, (int)n, nullptr, R, out, nullptr, nullptr, nullptr, flag, st, &e))
    return e;
  k_field_points<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(fd, params, (int)n, nullptr, R, out, nullptr, nullptr,
                                                              nullptr, flag);
  return cudaGetLastError();
}

}  // namespace prenom
