// kernels_tc.cu -- the density+colour MLP on 5th-gen tensor cores (tcgen05,
// fp32 accumulation in TMEM), fused with the hash-grid encode (forward) and the
// table-gradient scatter (backward).
//
// Replaces field_eval's MLP (field.cpp:181-211) and field_backward
// (field.cpp:227-293). Two operand modes (template SPL):
//   bf16        operands rounded to bf16 (1e-2 vs the fp32 oracle);
//   split bf16  x = hi + lo, three bf16 products per product (umma.cuh
//               mma_split): fp32-class results (1e-4), the headline mode.
// The encode itself is fp32 and bit-exact either way.
//
// Kernels (128-sample tiles, UMMA M = 128, the samples of a ray contiguous; one
// thread issues every tcgen05.mma, completion via tcgen05.commit -> mbarrier):
//   k_fwd_wx   (default) warp-specialised forward: encode warps write the bf16
//              features into TMEM, MLP warps run every layer from TMEM (TS form)
//   k_fwd_ws / k_fwd_ts / k_fwd_tc   earlier forwards (features in smem; no warp
//              specialisation; operands in smem) kept for A/B (PRENOM_FWD{,S}_TS)
//   k_bwd_tc   warp-specialised backward: MLP warps recompute the forward from the
//              stored features and backpropagate; scatter warps take d_features
//              from a TMEM slot and scatter them into the table gradient
//   k_mlp_grad_reduce  the backward CTAs' MLP-gradient partials, in CTA order
// Operand tiles use the core-matrix layout of umma.cuh, so the backward feeds
// forward activations/weights to the tensor core as MN-major (transposed)
// operands with no data movement:
//   fwd  H_l  = relu(H_{l-1} W_l^T + b_l)          A K-major,  B K-major
//   bwd  dH_l = D_{l+1} W_{l+1}                    A K-major,  B MN-major
//        dW_l += D_l^T [H_{l-1} | 1]               A MN-major, B MN-major (M=64)
// The appended ones column makes the bias gradient column `in` of dW_l. The
// weight-gradient accumulators live in TMEM for the whole persistent CTA and
// leave it once, as per-CTA partials (or one atomicAdd per weight).
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "prenom_device.cuh"
#include "umma.cuh"

namespace prenom {
namespace {

// forward launch shape (measured on B200, cfg2): see run_fwd
constexpr int kFwdThreadsDefault = 256;
constexpr int kFwdCtasDefault = 3;
constexpr int kFwdSmemKbDefault = 40;
// 3 CTAs x (40 + 1) KB fit a 132 KB carve-out, leaving 124 KB of L1 for the
// encode's gathers (was 57 KB/CTA padding, 196 KB carve-out, 60 KB of L1:
// k_fwd_tc 0.195 -> 0.186 ms on cfg2)
constexpr int kFwdCarveoutDefault = 58;
// bf16 forward: the warp-specialised kernel with features in TMEM (k_fwd_wx, ~15 KB
// per CTA), 2 CTAs in a 64 KB carve-out -> 192 KB of L1 (cfg2 0.157 ms vs 0.165 for
// k_fwd_ws, 0.177 for k_fwd_tc 3 x 256)
constexpr int kFwdTsDefault = 3;
constexpr int kFwdWsCarveout = 30;
// split-bf16 k_fwd_tc / k_fwd_ts shapes (~62 KB per CTA): two CTAs of 512 threads per SM
constexpr int kFwdSThreadsDefault = 512;
constexpr int kFwdSCtasDefault = 2;
constexpr int kFwdSCarveoutDefault = 58;  // 132 KB of shared memory, 124 KB of L1
// split forward: warp-specialised with the features and activations in TMEM
// (k_fwd_wx, weights-only shared memory, 2 CTAs per SM in a 64 KB carve-out: cfg2
// 0.188 ms vs 0.192 for k_fwd_ws (features in smem), 0.214 for k_fwd_ts at 512 x 2,
// 0.250 for k_fwd_tc); PRENOM_FWDS_TS=2 / 1 / 0 select those
constexpr int kFwdSTsDefault = 3;
constexpr int kFwdSTsThreads = 512;
constexpr int kFwdSTsCtas = 2;
constexpr int kFwdSTsCarveout = 30;
constexpr size_t kSmemPerSm = 228 * 1024;
constexpr int kSlack = 0;       // weight tiles are never over-read
// M=128 MN-major views of the (features|1) and (activations|1) tiles read
// past the tile end (finite garbage rows that are never flushed)
constexpr int kSlackX = 2048;
constexpr int kSlackH = 1024;

// bf16 copies of the MLP weights in core-matrix layouts + fp32 biases. With
// SPL (split-bf16 mode) a lo copy of every weight tile follows the hi copies
// at kLo bytes (umma.cuh split_bf16).
template <int INP, int W, int H, int SPL = 0>
struct WeightTiles {
  static constexpr int kW0 = W * INP * 2;
  static constexpr int kWl = W * W * 2;
  static constexpr int kWo = 16 * W * 2;
  static constexpr int kLo = kW0 + (H - 1) * kWl + kWo + kSlack;  // hi block bytes = lo offset
  static constexpr int kBytes = kLo * (SPL ? 2 : 1);
  unsigned char* w0;
  unsigned char* wl[2];
  unsigned char* wo;
  float* bias;  // H*W + 4

  __device__ void carve(unsigned char*& p) {
    unsigned char* q = p;
    w0 = q;
    q += kW0;
    for (int l = 1; l < H; ++l) {
      wl[l - 1] = q;
      q += kWl;
    }
    wo = q;
    p += kBytes;
    bias = reinterpret_cast<float*>(p);
    p += ((H * W + 4) * 4 + 15) / 16 * 16;
  }

  __device__ __forceinline__ static void put(unsigned char* t, uint32_t off, float v) {
    if (SPL) {
      __nv_bfloat16 hi, lo;
      umma::split_bf16(v, hi, lo);
      *reinterpret_cast<__nv_bfloat16*>(t + off) = hi;
      *reinterpret_cast<__nv_bfloat16*>(t + kLo + off) = lo;
    } else {
      *reinterpret_cast<__nv_bfloat16*>(t + off) = __float2bfloat16_rn(v);
    }
  }

  // threads [0, nt) cooperate (tix: this thread's index among them). One index
  // space over [W0 | W1..W_{H-1} | W_out (16 rows, 4 used) | biases]; each thread
  // issues 8 loads before it converts and stores them, so a reload inside a
  // grouped launch costs a few L2 round trips, not one per element.
  __device__ void load(const FieldDesc& fd, const float* __restrict__ mlp, int nt, int tix = -1) {
    const int IN = fd.in_dim;
    if (tix < 0) tix = threadIdx.x;
    constexpr int n0 = W * INP, nl = (H - 1) * W * W, no = 16 * W, nb = H * W + 4;
    constexpr int total = n0 + nl + no + nb;
    constexpr int U = 8;
    for (int base = tix; base < total; base += U * nt) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * nt;
        v[u] = 0.f;
        if (i < n0) {
          const int o = i / INP, k = i % INP;
          if (k < IN) v[u] = __ldg(mlp + fd.w_off[0] + o * IN + k);
        } else if (i < n0 + nl) {
          const int r = i - n0, l = 1 + r / (W * W), e = r % (W * W);
          v[u] = __ldg(mlp + fd.w_off[l] + e);
        } else if (i < n0 + nl + no) {
          const int r = i - n0 - nl, o = r / W;
          if (o < 4) v[u] = __ldg(mlp + fd.w_off[H] + r);
        } else if (i < total) {
          const int r = i - n0 - nl - no, l = r / W;
          v[u] = l < H ? __ldg(mlp + fd.b_off[l] + (r % W)) : __ldg(mlp + fd.b_off[H] + (r - H * W));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = base + u * nt;
        if (i < n0) {
          put(w0, umma::cm_offset(i / INP, i % INP, INP), v[u]);
        } else if (i < n0 + nl) {
          const int r = i - n0, l = 1 + r / (W * W), e = r % (W * W);
          put(wl[l - 1], umma::cm_offset(e / W, e % W, W), v[u]);
        } else if (i < n0 + nl + no) {
          const int r = i - n0 - nl;
          put(wo, umma::cm_offset(r / W, r % W, W), v[u]);
        } else if (i < total) {
          bias[i - n0 - nl - no] = v[u];
        }
      }
    }
  }
};

// Ray of a sample slot: 32-bit division (batches stay far below 2^31 slots;
// launch_*_tc check), not the ~70-instruction 64-bit one.
__device__ __forceinline__ uint32_t ray_of(long long gs, int S) { return (uint32_t)gs / (uint32_t)S; }

// Grouped launches: the object of global tile t. The tiles are object-major and
// every caller walks its tiles in increasing order, so the search starts at its
// previous object.
__device__ __forceinline__ int find_obj(const TcObj* __restrict__ g, int nobj, long long t, int j) {
  if (j < 0) j = 0;
  while (j + 1 < nobj && t >= g[j + 1].tile0) ++j;
  return j;
}

// (grouped launches) pull an object's MLP parameter block into L2 ahead of the
// weight-tile reload of its first tile; threads [0, nt) with index tix
__device__ __forceinline__ void prefetch_mlp_l2(const FieldDesc& fd, const float* params, int tix, int nt) {
  const char* p = reinterpret_cast<const char*>(params + fd.hash_params);
  const int lines = (fd.mlp_params * 4 + 127) / 128;
  for (int i = tix; i < lines; i += nt) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + (size_t)i * 128));
}

// Dynamic tile scheduler: CTAs pull 128-sample tiles from a global counter,
// so the tile load balances whatever number of CTAs the hardware co-locates
// on an SM (static striding left SMs with more resident CTAs as stragglers).
__device__ __forceinline__ long long next_tile(int* ctr, int* s_tile) {
  if (threadIdx.x == 0) *s_tile = atomicAdd(ctr, 1);
  __syncthreads();
  return *s_tile;
}

// Stored feature tiles (forward -> backward) use the backward's operand layout
// [128][INP + 8] per hi / lo half: the features plus the core matrix holding the
// ones column of [X | 1] (written once per buffer by init_feature_tiles), so the
// backward fetches a tile with ONE bulk copy. The forward's smem tile is
// [128][INP]; its 16 row groups go out as bulk copies into their slots.
template <int INP, int SPL>
__device__ __forceinline__ void store_features(uint4* feat_tiles, long long t, const unsigned char* X) {
  constexpr int XC = INP + 8;
  constexpr size_t kTileG = (size_t)128 * XC * 2 * (SPL ? 2 : 1);
  unsigned char* dst = reinterpret_cast<unsigned char*>(feat_tiles) + (size_t)t * kTileG;
#pragma unroll 1
  for (int h = 0; h < (SPL ? 2 : 1); ++h)
#pragma unroll 1
    for (int rg = 0; rg < 16; ++rg)
      umma::bulk_s2g_part(dst + h * 128 * XC * 2 + rg * (XC / 8) * 128, X + h * 128 * INP * 2 + rg * (INP / 8) * 128,
                          INP * 16);
  umma::bulk_commit();
}

// the ones / zero core matrices of every stored tile: hi [1, 0, ..., 0] per row, lo zeros
__global__ void k_feature_ones(unsigned char* feat, long long ntiles, int INP, int split) {
  const int XC = INP + 8;
  const long long tile_bytes = 128LL * XC * 2 * (split ? 2 : 1);
  const long long n = ntiles * 16 * 8 * (split ? 2 : 1);  // (tile, row group, row, half)
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    long long k = i;
    const int h = split ? (int)(k & 1) : 0;
    if (split) k >>= 1;
    const int r = (int)(k & 7), rg = (int)((k >> 3) & 15);
    const long long t = k >> 7;
    uint4* dst = reinterpret_cast<uint4*>(feat + t * tile_bytes + (long long)h * 128 * XC * 2 +
                                          (rg * (XC / 8) + INP / 8) * 128 + r * 16);
    *dst = make_uint4(h == 0 ? 0x3F80u : 0u, 0u, 0u, 0u);
  }
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void sync_for_mma() {
  umma::fence_proxy_async();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
}

__device__ __forceinline__ void wait_mma(uint64_t* bar, uint32_t& phase) {
  umma::mbar_wait(bar, phase);
  phase ^= 1u;
  umma::fence_after_sync();
}

// Epilogue: TMEM [128 x N] fp32 (cols c0..) -> +bias, ReLU -> bf16 tile [128][C].
// G column groups: warp w reads lane quadrant w%4, columns [(w/4)*N/G, ...).
template <int N, int G = 2, uint32_t LO = 0>
__device__ __forceinline__ void epi_relu(uint32_t tm, int col0, const float* bias, unsigned char* tile, int C) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = warp >> 2;
  const int row = 32 * q + lane;
  constexpr int NH = N / G;
  static_assert(NH % 8 == 0, "8-column TMEM loads");
#pragma unroll
  for (int c = 0; c < NH; c += 8) {
    const int col = half * NH + c;
    float v[8];
    umma::tmem_ld8(umma::taddr(tm, 32 * q, col0 + col), v);
    umma::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = fmaxf(v[j] + bias[col + j], 0.f);
    umma::st_row8_split(tile, row, col, C, v, LO);
  }
}

// epi_relu for the backward's forward recompute (G = 2); also returns this
// thread's ReLU gate, bit c = (bf16 H[row][half*N/2 + c] > 0), so the D_l
// epilogue needs no shared-memory read of H_l.
template <int N, int MG, uint32_t LO = 0>
__device__ __forceinline__ uint64_t epi_relu_gate(uint32_t tm, const float* bias, unsigned char* tile, int C) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = warp >> 2;
  const int row = 32 * q + lane;
  constexpr int NH = N / MG;
  static_assert(NH % 8 == 0 && NH <= 64, "8-column TMEM loads, 64-bit gate");
  uint64_t gate = 0;
#pragma unroll
  for (int c = 0; c < NH; c += 8) {
    const int col = half * NH + c;
    float v[8];
    umma::tmem_ld8(umma::taddr(tm, 32 * q, col), v);
    umma::tmem_wait_ld();
    uint32_t pk[4], pl[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float a0 = umma::operand_round(fmaxf(v[2 * i] + bias[col + 2 * i], 0.f)),
                  a1 = umma::operand_round(fmaxf(v[2 * i + 1] + bias[col + 2 * i + 1], 0.f));
      const __nv_bfloat162 b = __floats2bfloat162_rn(a0, a1);
      pk[i] = *reinterpret_cast<const uint32_t*>(&b);
      if (LO) {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(a0 - __low2float(b), a1 - __high2float(b));
        pl[i] = *reinterpret_cast<const uint32_t*>(&lo);
      }
      gate |= ((pk[i] & 0x7FFFu) ? 1ull : 0ull) << (c + 2 * i);
      gate |= ((pk[i] & 0x7FFF0000u) ? 1ull : 0ull) << (c + 2 * i + 1);
    }
    *reinterpret_cast<uint4*>(tile + umma::cm_offset(row, col, C)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    if (LO) *reinterpret_cast<uint4*>(tile + LO + umma::cm_offset(row, col, C)) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
  }
  return gate;
}

// ------------------------------------------------------------------ fwd
// NT threads: NT/128 threads per sample share the levels in the encode and
// the columns in the epilogues.
// SPL: split-bf16 operands (umma.cuh split_bf16); bit 0 of `split` turns the
// cross products on (the lo tiles are written either way).
template <int INP, int W, int H, int NT, int SPL>
__global__ void __launch_bounds__(NT) k_fwd_tc(FieldDesc fd, const float* __restrict__ params, long long n_total,
                                                     int S, const int* __restrict__ count,
                                                     const float4* __restrict__ pos, uint4* __restrict__ feat_tiles,
                                                     float4* __restrict__ out, int* flag, int* tile_ctr, int split) {
  using WT = WeightTiles<INP, W, H, SPL>;
  constexpr uint32_t XLO = SPL ? 128 * INP * 2 : 0;  // lo copies follow the hi tiles
  constexpr uint32_t HLO = SPL ? 128 * W * 2 : 0;
  constexpr uint32_t kXBytes = 128 * INP * 2 * (SPL ? 2 : 1);
  const bool sp = SPL && (split & 1);
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  WT wt;
  unsigned char* p = smem;
  wt.carve(p);
  // split mode: X overlays the activation tile (it is dead once the layer-0
  // MMA and the bulk store of the features have read it), so a CTA needs
  // ~62 KB and two fit an SM with 124 KB of L1 left for the gathers
  unsigned char* X = p;
  if (!SPL) p += kXBytes;
  // one activation tile: layer l+1's MMA completes (mbarrier) before layer
  // l+1's epilogue overwrites the tile it read
  unsigned char* Hb = p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_wait();  // params come from the previous step's Adam
  wt.load(fd, params + fd.hash_params, NT);
  constexpr int TPS = NT / 128;  // threads per sample
  for (int i = tid; i < (int)kXBytes / 2; i += NT) reinterpret_cast<__nv_bfloat16*>(X)[i] = __float2bfloat16_rn(0.f);
  // One 64-column TMEM region serves every layer: each MMA is issued only
  // after the previous epilogue drained it (sync_for_mma), so up to 8 CTAs fit.
  if (warp == 0) umma::tmem_alloc(&tbase, 64);
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = tbase;
  uint32_t phase = 0;
  constexpr uint32_t id_l0 = umma::idesc_bf16(128, W, false, false);
  constexpr uint32_t id_out = umma::idesc_bf16(128, 16, false, false);
  const long long ntiles = (n_total + kTile - 1) / kTile;
  __shared__ int s_tile;
  for (long long t = next_tile(tile_ctr, &s_tile); t < ntiles; t = next_tile(tile_ctr, &s_tile)) {
    const long long tile0 = t * kTile;
    // ---- encode (fp32, bit-exact) -> bf16 X tile; TPS threads per sample
    {
      const int s = tid & (kTile - 1), part = tid >> 7;
      const long long gs = tile0 + s;
      bool valid = gs < n_total && __ldg(count + ray_of(gs, S)) > 0;
      float4 pp = make_float4(0.f, 0.f, 0.f, 0.f);
      if (valid) pp = pos[gs];
      const float px = clamp01(pp.x), py = clamp01(pp.y), pz = clamp01(pp.z);
      // (batching two levels' gathers per thread measured slower: more distinct
      // lines in flight thrash L1, which serves the coarse levels)
      for (int l = part; l < fd.L; l += TPS) {
        float f[2] = {0.f, 0.f};
        if (valid) encode_level<2>(fd, params, l, px, py, pz, f);
        const __nv_bfloat162 hi = __floats2bfloat162_rn(f[0], f[1]);
        *reinterpret_cast<__nv_bfloat162*>(X + umma::cm_offset(s, 2 * l, INP)) = hi;
        if (SPL)
          *reinterpret_cast<__nv_bfloat162*>(X + XLO + umma::cm_offset(s, 2 * l, INP)) =
              __floats2bfloat162_rn(f[0] - __low2float(hi), f[1] - __high2float(hi));
      }
    }
    sync_for_mma();
    if (tid == 0) {
      for (int ks = 0; ks < INP / 16; ++ks)
        umma::mma_split(tm, umma::desc_kmajor(X, INP, ks), umma::desc_kmajor(wt.w0, INP, ks), id_l0, ks > 0, sp, XLO,
                        WT::kLo);
      umma::commit(&bar);
      // stored features for the backward pass (tile-major, same core-matrix
      // layout; split mode: hi tile then lo tile), written by the TMA engine:
      // no LSU work next to the gathers
      store_features<INP, SPL>(feat_tiles, t, X);
    }
    wait_mma(&bar, phase);
    if (SPL) {  // the bulk store must have read X before H overwrites it
      if (tid == 0) umma::bulk_wait_read();
      __syncthreads();
    }
    epi_relu<W, TPS, HLO>(tm, 0, wt.bias, Hb, W);
    for (int l = 1; l < H; ++l) {
      sync_for_mma();
      if (tid == 0) {
        for (int ks = 0; ks < W / 16; ++ks)
          umma::mma_split(tm, umma::desc_kmajor(Hb, W, ks), umma::desc_kmajor(wt.wl[l - 1], W, ks),
                          umma::idesc_bf16(128, W, false, false), ks > 0, sp, HLO, WT::kLo);
        umma::commit(&bar);
      }
      wait_mma(&bar, phase);
      epi_relu<W, TPS, HLO>(tm, 0, wt.bias + l * W, Hb, W);
    }
    sync_for_mma();
    if (tid == 0) {
      for (int ks = 0; ks < W / 16; ++ks)
        umma::mma_split(tm, umma::desc_kmajor(Hb, W, ks), umma::desc_kmajor(wt.wo, W, ks), id_out, ks > 0, sp, HLO,
                        WT::kLo);
      umma::commit(&bar);
    }
    wait_mma(&bar, phase);
    if (warp < 4) {
      const int row = 32 * warp + lane;
      float v[8];
      umma::tmem_ld8(umma::taddr(tm, 32 * warp, 0), v);
      umma::tmem_wait_ld();
      const long long gs = tile0 + row;
      if (gs < n_total) {
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        if (__ldg(count + ray_of(gs, S)) > 0) {
          const float* b = wt.bias + H * W;
          o.x = density_forward(fd.act, v[0] + b[0]);
          o.y = stable_sigmoid(v[1] + b[1]);
          o.z = stable_sigmoid(v[2] + b[2]);
          o.w = stable_sigmoid(v[3] + b[3]);
          if (!all_finite4(o.x, o.y, o.z, o.w)) atomicOr(flag, 1);
        }
        out[gs] = o;
      }
    }
    if (tid == 0) umma::bulk_wait_read();  // X is rewritten by the next tile's encode
    umma::fence_before_sync();
  }
  if (tid == 0) umma::bulk_wait_all();
#ifndef PRENOM_VAR_FWD_MEMSET
  tile_sched_exit(tile_ctr);
#endif
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 64);
}

// ------------------------------------------------------------------ fwd, TS form
// The same forward with the hidden activations kept in tensor memory: each
// epilogue reads the fp32 accumulator (tcgen05.ld), applies bias + ReLU,
// (split mode) splits hi/lo, packs bf16 pairs and writes them back with
// tcgen05.st; the next layer's MMA reads its A operand from TMEM
// (tcgen05.mma ... [d], [a], b_desc). Shared memory holds only the weights and
// the feature tile (~46 KB split, ~23 KB bf16), so more CTAs -- or more L1 for
// the encode's gathers -- fit an SM, and no epilogue touches shared memory.
// TMEM per CTA: accumulator [0, W), H hi [W, W + W/2), H lo [W + W/2, 2W).
template <int INP, int W, int H, int NT, int SPL>
__global__ void __launch_bounds__(NT) k_fwd_ts(FieldDesc fd, const float* __restrict__ params, long long n_total,
                                               int S, const int* __restrict__ count, const float4* __restrict__ pos,
                                               uint4* __restrict__ feat_tiles, float4* __restrict__ out, int* flag,
                                               int* tile_ctr, int split) {
  using WT = WeightTiles<INP, W, H, SPL>;
  constexpr uint32_t XLO = SPL ? 128 * INP * 2 : 0;
  constexpr uint32_t kXBytes = 128 * INP * 2 * (SPL ? 2 : 1);
  constexpr uint32_t kCols = 2 * W <= 64 ? 64 : 128;  // accumulator + H hi + H lo
  constexpr int kHhi = W, kHlo = W + W / 2;
  constexpr int TPS = NT / 128;  // threads per sample (encode) = column groups (epilogues)
  static_assert(W % (8 * TPS) == 0, "epilogue column groups of 8");
  const bool sp = SPL && (split & 1);
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ int s_tile, s_next;
  WT wt;
  unsigned char* p = smem;
  wt.carve(p);
  unsigned char* X = p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, g = warp >> 2, row = 32 * q + lane;
  pdl_wait();  // params come from the previous step's Adam
  wt.load(fd, params + fd.hash_params, NT);
  for (int i = tid; i < (int)kXBytes / 2; i += NT) reinterpret_cast<__nv_bfloat16*>(X)[i] = __float2bfloat16_rn(0.f);
  if (warp == 0) umma::tmem_alloc(&tbase, kCols);
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = tbase;
  const uint32_t lane_base = (uint32_t)(32 * q) << 16;
  uint32_t phase = 0;
  constexpr uint32_t id_h = umma::idesc_bf16(128, W, false, false);
  constexpr uint32_t id_out = umma::idesc_bf16(128, 16, false, false);
  // bias + ReLU of the accumulator -> bf16 (hi, lo) pairs in TMEM; column group g
  auto epilogue = [&](const float* bias) {
    constexpr int NG = W / TPS;
#pragma unroll
    for (int c = 0; c < NG; c += 8) {
      const int col = g * NG + c;
      float v[8];
      umma::tmem_ld8(tm + lane_base + col, v);
      umma::tmem_wait_ld();
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a0 = fmaxf(v[2 * i] + bias[col + 2 * i], 0.f), a1 = fmaxf(v[2 * i + 1] + bias[col + 2 * i + 1], 0.f);
        const __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
        hi[i] = *reinterpret_cast<const uint32_t*>(&h);
        if (SPL) {
          const __nv_bfloat162 l = __floats2bfloat162_rn(a0 - __low2float(h), a1 - __high2float(h));
          lo[i] = *reinterpret_cast<const uint32_t*>(&l);
        }
      }
      umma::tmem_st4(tm + lane_base + kHhi + col / 2, hi);
      if (SPL) umma::tmem_st4(tm + lane_base + kHlo + col / 2, lo);
    }
    umma::tmem_wait_st();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
  };
  const long long ntiles = (n_total + kTile - 1) / kTile;
  // the next tile is claimed at the start of this one (published by the first
  // barrier), so no claim round trip sits between tiles
  for (long long t = next_tile(tile_ctr, &s_tile); t < ntiles; t = s_next) {
    const long long tile0 = t * kTile;
    if (tid == 0) s_next = atomicAdd(tile_ctr, 1);
    {  // ---- encode (fp32, bit-exact) -> bf16 X tile (hi, lo)
      const int s = tid & (kTile - 1), part = tid >> 7;
      const long long gs = tile0 + s;
      bool valid = gs < n_total && __ldg(count + ray_of(gs, S)) > 0;
      float4 pp = make_float4(0.f, 0.f, 0.f, 0.f);
      if (valid) pp = pos[gs];
      const float px = clamp01(pp.x), py = clamp01(pp.y), pz = clamp01(pp.z);
      for (int l = part; l < fd.L; l += TPS) {
        float f[2] = {0.f, 0.f};
        if (valid) encode_level<2>(fd, params, l, px, py, pz, f);
        const __nv_bfloat162 hi = __floats2bfloat162_rn(f[0], f[1]);
        *reinterpret_cast<__nv_bfloat162*>(X + umma::cm_offset(s, 2 * l, INP)) = hi;
        if (SPL)
          *reinterpret_cast<__nv_bfloat162*>(X + XLO + umma::cm_offset(s, 2 * l, INP)) =
              __floats2bfloat162_rn(f[0] - __low2float(hi), f[1] - __high2float(hi));
      }
    }
    sync_for_mma();
    if (tid == 0) {
      for (int ks = 0; ks < INP / 16; ++ks)
        umma::mma_split(tm, umma::desc_kmajor(X, INP, ks), umma::desc_kmajor(wt.w0, INP, ks), id_h, ks > 0, sp, XLO,
                        WT::kLo);
      umma::commit(&bar);
      store_features<INP, SPL>(feat_tiles, t, X);  // stored features for the backward
    }
    wait_mma(&bar, phase);
    epilogue(wt.bias);
    for (int l = 1; l < H; ++l) {
      if (tid == 0) {
        for (int ks = 0; ks < W / 16; ++ks)
          umma::mma_split_ts(tm, tm + kHhi + ks * 8, umma::desc_kmajor(wt.wl[l - 1], W, ks), id_h, ks > 0, sp,
                             kHlo - kHhi, WT::kLo);
        umma::commit(&bar);
      }
      wait_mma(&bar, phase);
      epilogue(wt.bias + l * W);
    }
    if (tid == 0) {
      for (int ks = 0; ks < W / 16; ++ks)
        umma::mma_split_ts(tm, tm + kHhi + ks * 8, umma::desc_kmajor(wt.wo, W, ks), id_out, ks > 0, sp, kHlo - kHhi,
                           WT::kLo);
      umma::commit(&bar);
    }
    wait_mma(&bar, phase);
    if (warp < 4) {
      float v[8];
      umma::tmem_ld8(tm + lane_base, v);
      umma::tmem_wait_ld();
      const long long gs = tile0 + row;
      if (gs < n_total) {
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        if (__ldg(count + ray_of(gs, S)) > 0) {
          const float* b = wt.bias + H * W;
          o.x = density_forward(fd.act, v[0] + b[0]);
          o.y = stable_sigmoid(v[1] + b[1]);
          o.z = stable_sigmoid(v[2] + b[2]);
          o.w = stable_sigmoid(v[3] + b[3]);
          if (!all_finite4(o.x, o.y, o.z, o.w)) atomicOr(flag, 1);
        }
        out[gs] = o;
      }
    }
    if (tid == 0) umma::bulk_wait_read();  // X is rewritten by the next tile's encode
    umma::fence_before_sync();
    __syncthreads();  // (X reuse; s_next was published by the tile's first barrier)
  }
  if (tid == 0) umma::bulk_wait_all();
  tile_sched_exit(tile_ctr);
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, kCols);
}

// ------------------------------------------------------------------ fwd, warp-specialised
// k_fwd_ts with the encode and the MLP chain on different warps, so the gathers
// of tile t+1 run while tile t is on the tensor cores (in k_fwd_ts every warp
// waits for the chain). 16 encode warps (4 threads per sample, levels
// interleaved as before) fill a double-buffered feature tile (full / empty
// mbarriers); 4 MLP warps (one row per thread: TMEM lane quadrant = warp % 4)
// issue the MMAs, run the epilogues through TMEM and write (sigma, rgb).
// Tiles are claimed one ahead by the encode leader.
constexpr int kWsEncWarps = 16;  // k_fwd_ws's default shape
constexpr int kWsThreads = (kWsEncWarps + 4) * 32;
// k_fwd_wx's shape: encode warps + MLP warps (4 per epilogue column group). With
// two hidden layers the MLP chain bounds the split forward (cfg2: 0.124 ms without
// the layers after L0, 0.186 with them), so half the encoders make room for a
// second MLP warp per TMEM lane quadrant, each taking half the epilogue columns
// (cfg2 0.186 -> 0.175 ms, cfg1 0.052 -> 0.047; 12 + 8: 0.178; 16 + 8 spills at
// 40 registers: 0.191); one hidden layer keeps 16 + 4 (cfg3 / cfg5 archs are
// encode-bound: 8 + 8 is 1-6% slower there).
template <int H>
struct WxShape {
  static constexpr int kEnc = H >= 2 ? 8 : 16;
  static constexpr int kMlp = H >= 2 ? 8 : 4;
  static constexpr int kThreads = (kEnc + kMlp) * 32;
};

// NE encode warps (a multiple of 4: NE/4 threads per sample), MINB CTAs per SM.
template <int INP, int W, int H, int SPL, int NE = 16, int MINB = 2>
__global__ void __launch_bounds__((NE + 4) * 32, MINB) k_fwd_ws(FieldDesc fd, const float* __restrict__ params, long long n_total,
                                                    int S, const int* __restrict__ count, const float4* __restrict__ pos,
                                                    uint4* __restrict__ feat_tiles, float4* __restrict__ out, int* flag,
                                                    int* tile_ctr, int split) {
  using WT = WeightTiles<INP, W, H, SPL>;
  constexpr int kNE = NE;
  constexpr int kNT = (NE + 4) * 32;
  constexpr int kEnc = kNE * 32;
  constexpr int TPS = kEnc / 128;
  constexpr uint32_t XLO = SPL ? 128 * INP * 2 : 0;
  constexpr uint32_t kXBytes = 128 * INP * 2 * (SPL ? 2 : 1);
  constexpr uint32_t kCols = 2 * W <= 64 ? 64 : 128;
  constexpr int kHhi = W, kHlo = W + W / 2;
  const bool sp = SPL && (split & 1);
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[2], empty[2], bar;
  __shared__ uint32_t tbase;
  __shared__ long long claim[2], tile_of[2];
  WT wt;
  unsigned char* p = smem;
  wt.carve(p);
  unsigned char* const Xb0 = p;  // two feature buffers, kXBytes apart
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long ntiles = (n_total + kTile - 1) / kTile;
  pdl_wait();  // params come from the previous step's Adam
  wt.load(fd, params + fd.hash_params, kNT);
  for (int i = tid; i < (int)kXBytes; i += kNT) {  // (both buffers; padding levels stay 0)
    reinterpret_cast<__nv_bfloat16*>(Xb0)[i] = __float2bfloat16_rn(0.f);
  }
  if (warp == kNE) umma::tmem_alloc(&tbase, kCols);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&full[b], kEnc);
      umma::mbar_init(&empty[b], 1);
    }
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
    claim[0] = atomicAdd(tile_ctr, 1);
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = tbase;
  if (warp < kNE) {
    // ================= encode warps
    const int s = tid & (kTile - 1), part = tid >> 7;
    for (int i = 0;; ++i) {
      const int b = i & 1;
      umma::mbar_wait(&empty[b], ((uint32_t)(i >> 1) & 1u) ^ 1u);  // buffer b free (first pass: immediately)
      named_sync(2, kEnc);  // claim[b] of this iteration is published
      const long long t = claim[b];
      if (tid == 0 && t < ntiles) claim[b ^ 1] = atomicAdd(tile_ctr, 1);  // next iteration's tile
      if (t >= ntiles) {
        if (tid == 0) tile_of[b] = -1;  // sentinel for the MLP warps
        umma::mbar_arrive_plain(&full[b]);
        break;
      }
      if (tid == 0) tile_of[b] = t;
      unsigned char* X = Xb0 + b * kXBytes;
      const long long gs = t * kTile + s;
      const bool valid = gs < n_total && __ldg(count + ray_of(gs, S)) > 0;
      float4 pp = make_float4(0.f, 0.f, 0.f, 0.f);
      if (valid) pp = pos[gs];
      const float px = clamp01(pp.x), py = clamp01(pp.y), pz = clamp01(pp.z);
      for (int l = part; l < fd.L; l += TPS) {
        float f[2] = {0.f, 0.f};
        if (valid) encode_level<2>(fd, params, l, px, py, pz, f);
        const __nv_bfloat162 hi = __floats2bfloat162_rn(f[0], f[1]);
        *reinterpret_cast<__nv_bfloat162*>(X + umma::cm_offset(s, 2 * l, INP)) = hi;
        if (SPL)
          *reinterpret_cast<__nv_bfloat162*>(X + XLO + umma::cm_offset(s, 2 * l, INP)) =
              __floats2bfloat162_rn(f[0] - __low2float(hi), f[1] - __high2float(hi));
      }
      umma::fence_proxy_async();  // generic smem writes -> the tensor core and the TMA store
      umma::mbar_arrive_plain(&full[b]);
    }
  } else {
    // ================= MLP warps: one row per thread
    const int q = warp & 3, row = 32 * q + lane, mt = tid - kEnc;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    uint32_t phase = 0;
    constexpr uint32_t id_h = umma::idesc_bf16(128, W, false, false);
    constexpr uint32_t id_out = umma::idesc_bf16(128, 16, false, false);
    auto mlp_sync = [&]() {
      umma::fence_before_sync();
      named_sync(1, 128);
      umma::fence_after_sync();
    };
    auto epilogue = [&](const float* bias) {
#pragma unroll
      for (int c = 0; c < W; c += 16) {
        float v[16];
        umma::tmem_ld16(tm + lane_base + c, v);
        umma::tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int k = 8 * h + 2 * i;
            const float a0 = fmaxf(v[k] + bias[c + k], 0.f), a1 = fmaxf(v[k + 1] + bias[c + k + 1], 0.f);
            const __nv_bfloat162 hh = __floats2bfloat162_rn(a0, a1);
            hi[i] = *reinterpret_cast<const uint32_t*>(&hh);
            if (SPL) {
              const __nv_bfloat162 ll = __floats2bfloat162_rn(a0 - __low2float(hh), a1 - __high2float(hh));
              lo[i] = *reinterpret_cast<const uint32_t*>(&ll);
            }
          }
          umma::tmem_st4(tm + lane_base + kHhi + (c + 8 * h) / 2, hi);
          if (SPL) umma::tmem_st4(tm + lane_base + kHlo + (c + 8 * h) / 2, lo);
        }
      }
      umma::tmem_wait_st();
      mlp_sync();
    };
    for (int i = 0;; ++i) {
      const int b = i & 1;
      umma::mbar_wait(&full[b], (uint32_t)(i >> 1) & 1u);
      const long long t = tile_of[b];
      if (t < 0) break;
      umma::fence_after_sync();
      unsigned char* X = Xb0 + b * kXBytes;
      if (mt == 0) {
        for (int ks = 0; ks < INP / 16; ++ks)
          umma::mma_split(tm, umma::desc_kmajor(X, INP, ks), umma::desc_kmajor(wt.w0, INP, ks), id_h, ks > 0, sp, XLO,
                          WT::kLo);
        umma::commit(&bar);
      }
      // stored features for the backward: the lanes of MLP warp 0 issue one row-group
      // copy each (into the [X | 1] slots of the stored tile), in parallel
      constexpr int XCg = INP + 8;
      if (mt < 32 && mt < 16 * (SPL ? 2 : 1)) {
        const int h = mt >> 4, rg = mt & 15;
        unsigned char* dst = reinterpret_cast<unsigned char*>(feat_tiles) + (size_t)t * (128 * XCg * 2 * (SPL ? 2 : 1)) +
                             h * 128 * XCg * 2 + rg * (XCg / 8) * 128;
        umma::bulk_s2g_part(dst, X + h * 128 * INP * 2 + rg * (INP / 8) * 128, INP * 16);
        umma::bulk_commit();
      }
      wait_mma(&bar, phase);
      if (mt < 32) {  // the layer-0 MMA and the feature stores have read buffer b
        umma::bulk_wait_read();
        __syncwarp();
        if (mt == 0) umma::mbar_arrive_plain(&empty[b]);
      }
      epilogue(wt.bias);
      for (int l = 1; l < H; ++l) {
        if (mt == 0) {
          for (int ks = 0; ks < W / 16; ++ks)
            umma::mma_split_ts(tm, tm + kHhi + ks * 8, umma::desc_kmajor(wt.wl[l - 1], W, ks), id_h, ks > 0, sp,
                               kHlo - kHhi, WT::kLo);
          umma::commit(&bar);
        }
        wait_mma(&bar, phase);
        epilogue(wt.bias + l * W);
      }
      if (mt == 0) {
        for (int ks = 0; ks < W / 16; ++ks)
          umma::mma_split_ts(tm, tm + kHhi + ks * 8, umma::desc_kmajor(wt.wo, W, ks), id_out, ks > 0, sp,
                             kHlo - kHhi, WT::kLo);
        umma::commit(&bar);
      }
      wait_mma(&bar, phase);
      float v[8];
      umma::tmem_ld8(tm + lane_base, v);
      umma::tmem_wait_ld();
      const long long gs = t * kTile + row;
      if (gs < n_total) {
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        if (__ldg(count + ray_of(gs, S)) > 0) {
          const float* bb = wt.bias + H * W;
          o.x = density_forward(fd.act, v[0] + bb[0]);
          o.y = stable_sigmoid(v[1] + bb[1]);
          o.z = stable_sigmoid(v[2] + bb[2]);
          o.w = stable_sigmoid(v[3] + bb[3]);
          if (!all_finite4(o.x, o.y, o.z, o.w)) atomicOr(flag, 1);
        }
        out[gs] = o;
      }
      mlp_sync();  // the accumulator is free for the next tile's layer 0
    }
    if (mt < 32) umma::bulk_wait_all();
  }
  __syncthreads();
  tile_sched_exit(tile_ctr);
  if (warp == kNE) umma::tmem_dealloc(tm, kCols);
}

// ------------------------------------------------------------------ fwd, features in TMEM
// k_fwd_ws with the feature tile in tensor memory too: the encode threads write
// their level pairs (bf16 hi / lo, 32-bit columns) straight into a
// double-buffered TMEM X region with tcgen05.st (their sample row is their
// warp's TMEM lane quadrant), layer 0 reads A from TMEM, and the MLP warps copy
// the tile from TMEM into the stored-feature layout with 16-byte global stores.
// Shared memory holds only the weights (~29 KB per CTA), so the two CTAs of an
// SM leave ~190 KB of L1 to the gathers, and the encode issues no shared stores.
// TMEM: accumulator [0, W), H hi/lo [W, 2W), X[b] hi/lo [2W + b*INP, 2W + (b+1)*INP).
// GRP: grouped launch over the objects gobj[0..nobj) (n_total = all their tiles
// x 128; the per-object arguments are unused): the MLP warps reload the weight
// tiles when their tile's object changes.
template <int INP, int W, int H, int SPL, bool GRP = false>
__global__ void __launch_bounds__(WxShape<H>::kThreads, 2) k_fwd_wx(FieldDesc fd, const float* __restrict__ params,
                                                       long long n_total, int S, const int* __restrict__ count,
                                                       const float4* __restrict__ pos, uint4* __restrict__ feat_tiles,
                                                       float4* __restrict__ out, int* flag, int* tile_ctr, int split,
                                                       const TcObj* __restrict__ gobj, int nobj) {
  using WT = WeightTiles<INP, W, H, SPL>;
  constexpr int kWxEncWarps = WxShape<H>::kEnc, kWxMlpWarps = WxShape<H>::kMlp, kWxThreads = WxShape<H>::kThreads;
  constexpr int kEnc = kWxEncWarps * 32;
  constexpr int TPS = kEnc / 128;
  constexpr int kMlpT = kWxMlpWarps * 32;  // MLP threads
  constexpr int MG = kWxMlpWarps / 4;      // epilogue column groups per TMEM lane quadrant
  static_assert(kEnc % 128 == 0 && kWxMlpWarps % 4 == 0 && (W / MG) % 16 == 0, "k_fwd_wx shape");
  // Where the MLP chain bounds the forward (two hidden layers) and each of a sample's TPS
  // encode threads gets at least two 4-level chunks (one 16-byte core-matrix row of the
  // stored tile each; chunk c goes to part c % TPS, so a thread mixes coarse and fine
  // levels), the encoders store the backward's features themselves and the MLP warps skip
  // the copy-out (cfg2 forward 0.1752 -> 0.1725 ms; on the encode-bound one-hidden-layer
  // archs and on one chunk per thread it costs 1-5%).
  constexpr int NCH = INP / 8;
  constexpr bool kEncStores = H >= 2 && NCH % TPS == 0 && NCH / TPS >= 2;
  constexpr int XC = INP + 8;  // stored-tile row width ([X | 1])
  constexpr int kHhi = W, kHlo = W + W / 2;
  constexpr int kX0 = 2 * W;            // X[b] hi at kX0 + b * INP, lo at + INP / 2
  constexpr int kXcols = INP;           // per buffer: INP / 2 hi + INP / 2 lo columns
  constexpr uint32_t kCols = 2 * W + 2 * kXcols <= 128 ? 128 : 256;
  const bool sp = SPL && (split & 1);
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[2], empty[2], bar;
  __shared__ uint32_t tbase;
  __shared__ long long claim[2], tile_of[2];
  WT wt;
  unsigned char* p = smem;
  wt.carve(p);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long ntiles = (n_total + kTile - 1) / kTile;
  pdl_wait();  // params come from the previous step's Adam
  if (!GRP) wt.load(fd, params + fd.hash_params, kWxThreads);
  if (warp == kWxEncWarps) umma::tmem_alloc(&tbase, kCols);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      umma::mbar_init(&full[b], kEnc);
      umma::mbar_init(&empty[b], 1);
    }
    umma::mbar_init(&bar, 1);
    umma::fence_mbar_init();
    claim[0] = atomicAdd(tile_ctr, 1);
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = tbase;
  const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
  if (warp < kWxEncWarps) {
    // padding levels (L*F < INP) stay zero in both buffers: written once here
    const int part = tid >> 7;
    for (int b = 0; b < 2; ++b)
      for (int l = fd.L + part; l < INP / 2; l += TPS) {
        umma::tmem_st1(tm + lane_base + kX0 + b * kXcols + l, 0u);
        umma::tmem_st1(tm + lane_base + kX0 + b * kXcols + INP / 2 + l, 0u);
      }
    umma::tmem_wait_st();
  }
  if (warp < kWxEncWarps) {
    // ================= encode warps: features -> TMEM X[b]
    const int s = tid & (kTile - 1), part = tid >> 7;
    int ej = 0;
    for (int i = 0;; ++i) {
      const int b = i & 1;
      umma::mbar_wait(&empty[b], ((uint32_t)(i >> 1) & 1u) ^ 1u);  // buffer b free (first pass: immediately)
      umma::fence_after_sync();
      named_sync(2, kEnc);  // claim[b] of this iteration is published
      const long long t = claim[b];
      if (tid == 0 && t < ntiles) claim[b ^ 1] = atomicAdd(tile_ctr, 1);  // next iteration's tile
      if (t >= ntiles) {
        if (tid == 0) tile_of[b] = -1;  // sentinel for the MLP warps
        umma::mbar_arrive_plain(&full[b]);
        break;
      }
      if (tid == 0) tile_of[b] = t;
      const float* prm = params;
      const int* cnt = count;
      const float4* ps = pos;
      long long tl = t, nn = n_total;
      if (GRP) {
        const int pj = ej;
        ej = find_obj(gobj, nobj, t, ej);
        if (ej != pj && warp == 0) prefetch_mlp_l2(fd, gobj[ej].params, lane, 32);  // the MLP warps reload soon
        prm = gobj[ej].params;
        cnt = gobj[ej].count;
        ps = gobj[ej].pos;
        tl = t - gobj[ej].tile0;
        nn = gobj[ej].n;
      }
      const long long gs = tl * kTile + s;
      // the position is loaded next to the ray's sample count, not after it (two
      // independent L2 round trips instead of two serial ones); escaped rays'
      // slots hold stale positions, which `valid` discards
      float4 pp = make_float4(0.f, 0.f, 0.f, 0.f);
      bool valid = false;
      if (gs < nn) {
        pp = __ldg(ps + gs);
        valid = __ldg(cnt + ray_of(gs, S)) > 0;
      }
      if (!valid) pp = make_float4(0.f, 0.f, 0.f, 0.f);
      const float px = clamp01(pp.x), py = clamp01(pp.y), pz = clamp01(pp.z);
      const uint32_t xb = tm + lane_base + kX0 + b * kXcols;
      if constexpr (kEncStores) {
        uint4* fbp = feat_tiles;
        if (GRP) fbp = reinterpret_cast<uint4*>(gobj[ej].feat);
        unsigned char* dst = reinterpret_cast<unsigned char*>(fbp) + (size_t)tl * (128 * XC * 2 * (SPL ? 2 : 1)) +
                             (s >> 3) * (XC / 8) * 128 + (s & 7) * 16;
#pragma unroll 1
        for (int ch = part; ch < NCH; ch += TPS) {
          uint32_t hi4[4], lo4[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int l = 4 * ch + k;
            float f[2] = {0.f, 0.f};
            if (valid && l < fd.L) encode_level<2>(fd, prm, l, px, py, pz, f);
            f[0] = umma::operand_round(f[0]);
            f[1] = umma::operand_round(f[1]);
            const __nv_bfloat162 hi = __floats2bfloat162_rn(f[0], f[1]);
            hi4[k] = *reinterpret_cast<const uint32_t*>(&hi);
            if (SPL) {
              const __nv_bfloat162 lo = __floats2bfloat162_rn(f[0] - __low2float(hi), f[1] - __high2float(hi));
              lo4[k] = *reinterpret_cast<const uint32_t*>(&lo);
            }
          }
          umma::tmem_st4(xb + 4 * ch, hi4);
          *reinterpret_cast<uint4*>(dst + ch * 128) = make_uint4(hi4[0], hi4[1], hi4[2], hi4[3]);
          if (SPL) {
            umma::tmem_st4(xb + INP / 2 + 4 * ch, lo4);
            *reinterpret_cast<uint4*>(dst + 128 * XC * 2 + ch * 128) = make_uint4(lo4[0], lo4[1], lo4[2], lo4[3]);
          }
        }
      } else {
        for (int l = part; l < fd.L; l += TPS) {
          float f[2] = {0.f, 0.f};
          if (valid) encode_level<2>(fd, prm, l, px, py, pz, f);
          f[0] = umma::operand_round(f[0]);
          f[1] = umma::operand_round(f[1]);
          const __nv_bfloat162 hi = __floats2bfloat162_rn(f[0], f[1]);
          umma::tmem_st1(xb + l, *reinterpret_cast<const uint32_t*>(&hi));
          if (SPL) {
            const __nv_bfloat162 lo = __floats2bfloat162_rn(f[0] - __low2float(hi), f[1] - __high2float(hi));
            umma::tmem_st1(xb + INP / 2 + l, *reinterpret_cast<const uint32_t*>(&lo));
          }
        }
      }
      umma::tmem_wait_st();
      umma::fence_before_sync();
      umma::mbar_arrive_plain(&full[b]);
    }
  } else {
    // ================= MLP warps: one row per thread
    const int q = warp & 3, row = 32 * q + lane, mt = tid - kEnc, cg = mt >> 7;  // cg: column group
    uint32_t phase = 0;
    constexpr uint32_t id_h = umma::idesc_bf16(128, W, false, false);
    constexpr uint32_t id_out = umma::idesc_bf16(128, 16, false, false);
    auto mlp_sync = [&]() {
      umma::fence_before_sync();
      named_sync(1, kMlpT);
      umma::fence_after_sync();
    };
    auto epilogue = [&](const float* bias) {
#pragma unroll
      for (int c = cg * (W / MG); c < (cg + 1) * (W / MG); c += 16) {
        float v[16];
        umma::tmem_ld16(tm + lane_base + c, v);
        umma::tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int k = 8 * h + 2 * i;
            const float a0 = umma::operand_round(fmaxf(v[k] + bias[c + k], 0.f)),
                        a1 = umma::operand_round(fmaxf(v[k + 1] + bias[c + k + 1], 0.f));
            const __nv_bfloat162 hh = __floats2bfloat162_rn(a0, a1);
            hi[i] = *reinterpret_cast<const uint32_t*>(&hh);
            if (SPL) {
              const __nv_bfloat162 ll = __floats2bfloat162_rn(a0 - __low2float(hh), a1 - __high2float(hh));
              lo[i] = *reinterpret_cast<const uint32_t*>(&ll);
            }
          }
          umma::tmem_st4(tm + lane_base + kHhi + (c + 8 * h) / 2, hi);
          if (SPL) umma::tmem_st4(tm + lane_base + kHlo + (c + 8 * h) / 2, lo);
        }
      }
      umma::tmem_wait_st();
      mlp_sync();
    };
    int mj = -1;  // (GRP) object whose weights are in shared memory
    for (int i = 0;; ++i) {
      const int b = i & 1;
      umma::mbar_wait(&full[b], (uint32_t)(i >> 1) & 1u);
      const long long t = tile_of[b];
      if (t < 0) break;
      const int* cnt = count;
      uint4* fb = feat_tiles;
      float4* op = out;
      int* flg = flag;
      long long tl = t, nn = n_total;
      if (GRP) {
        const int j = find_obj(gobj, nobj, t, mj);
        if (j != mj) {  // no MMA is in flight: the previous tile's output layer was waited for
          wt.load(fd, gobj[j].params + fd.hash_params, kMlpT, mt);
          umma::fence_proxy_async();
          named_sync(1, kMlpT);
          mj = j;
        }
        cnt = gobj[j].count;
        fb = reinterpret_cast<uint4*>(gobj[j].feat);
        op = gobj[j].out;
        flg = gobj[j].flag;
        tl = t - gobj[j].tile0;
        nn = gobj[j].n;
      }
      umma::fence_after_sync();
      const uint32_t xa = tm + kX0 + b * kXcols;  // X[b] (lane 0 base: the MMA reads all 128 lanes)
      if (mt == 0) {
        for (int ks = 0; ks < INP / 16; ++ks)
          umma::mma_split_ts(tm, xa + ks * 8, umma::desc_kmajor(wt.w0, INP, ks), id_h, ks > 0, sp, INP / 2, WT::kLo);
        umma::commit(&bar);
      }
      // stored features for the backward (unless the encoders stored them): this thread's
      // row from TMEM into the [X | 1] slots of the stored tile (16-byte stores; the ones
      // columns were written once)
      if (!kEncStores) {
        unsigned char* dst = reinterpret_cast<unsigned char*>(fb) + (size_t)tl * (128 * XC * 2 * (SPL ? 2 : 1)) +
                             (row >> 3) * (XC / 8) * 128 + (row & 7) * 16;
#pragma unroll
        for (int h = 0; h < (SPL ? 2 : 1); ++h) {
          if (MG > 1 && h % MG != cg) continue;  // (column groups share the hi / lo halves)
          float v[INP / 2];
          if (INP / 2 == 16) {
            umma::tmem_ld16(tm + lane_base + kX0 + b * kXcols + h * (INP / 2), v);
          } else {
            umma::tmem_ld8(tm + lane_base + kX0 + b * kXcols + h * (INP / 2), v);
          }
          umma::tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < INP / 8; ++c)
            *reinterpret_cast<uint4*>(dst + h * 128 * XC * 2 + c * 128) =
                make_uint4(__float_as_uint(v[4 * c]), __float_as_uint(v[4 * c + 1]), __float_as_uint(v[4 * c + 2]),
                           __float_as_uint(v[4 * c + 3]));
        }
      }
      wait_mma(&bar, phase);
      // the layer-0 MMA and the copy-out have read X[b]: the encoders may refill it
      umma::fence_before_sync();
      named_sync(1, kMlpT);
      if (mt == 0) umma::mbar_arrive_plain(&empty[b]);
      umma::fence_after_sync();
      epilogue(wt.bias);
      for (int l = 1; l < H; ++l) {
        if (mt == 0) {
          for (int ks = 0; ks < W / 16; ++ks)
            umma::mma_split_ts(tm, tm + kHhi + ks * 8, umma::desc_kmajor(wt.wl[l - 1], W, ks), id_h, ks > 0, sp,
                               kHlo - kHhi, WT::kLo);
          umma::commit(&bar);
        }
        wait_mma(&bar, phase);
        epilogue(wt.bias + l * W);
      }
      if (mt == 0) {
        for (int ks = 0; ks < W / 16; ++ks)
          umma::mma_split_ts(tm, tm + kHhi + ks * 8, umma::desc_kmajor(wt.wo, W, ks), id_out, ks > 0, sp,
                             kHlo - kHhi, WT::kLo);
        umma::commit(&bar);
      }
      wait_mma(&bar, phase);
      float v[8];
      umma::tmem_ld8(tm + lane_base, v);
      umma::tmem_wait_ld();
      const long long gs = tl * kTile + row;
      if (cg == 0 && gs < nn) {
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        if (__ldg(cnt + ray_of(gs, S)) > 0) {
          const float* bb = wt.bias + H * W;
          o.x = density_forward(fd.act, v[0] + bb[0]);
          o.y = stable_sigmoid(v[1] + bb[1]);
          o.z = stable_sigmoid(v[2] + bb[2]);
          o.w = stable_sigmoid(v[3] + bb[3]);
          if (!all_finite4(o.x, o.y, o.z, o.w)) atomicOr(flg, 1);
        }
        op[gs] = o;
      }
      mlp_sync();  // the accumulator is free for the next tile's layer 0
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  tile_sched_exit(tile_ctr);
  if (warp == kWxEncWarps) umma::tmem_dealloc(tm, kCols);
}

// One level of the table-gradient scatter for the 32 consecutive samples of a
// warp (field.cpp:279-292). Samples of a ray are depth-sorted and a line
// enters each cell once, so equal cells form contiguous lane runs; each run's
// total is formed in its first lane, which alone issues the 8 corner atomics
// (de-duplicated scatter). Equal consecutive cells of different rays merge
// too (same rows, same sum), so the key is the cell alone.
// Two ways to form the run totals, chosen per level from the longest run R:
//  * R <= pull_max: the head pulls each later member's (fx, fy, fz, d0, d1)
//    -- 5 shuffles per member -- and accumulates w * d itself (ALU work);
//  * else a segmented tree over the 16 corner products, 16 shuffles per
//    round, log2(R) rounds.
// Shuffles share the LSU pipe with the atomics, which bounds this kernel, so
// the short runs of the fine levels go the pull way.
__device__ __forceinline__ void scatter_level(const FieldDesc& fd, float* __restrict__ grad, int l, bool valid,
                                              float px, float py, float pz, float dx, float dy, int lane, int skip,
                                              int pull_max) {
  const int res = fd.res[l];
  const LevelCell cell = level_cell(res, px, py, pz);
  const uint32_t key = valid ? ((uint32_t)cell.cz * (uint32_t)res + (uint32_t)cell.cy) * (uint32_t)res + (uint32_t)cell.cx
                             : 0xFFFFFFFFu - (uint32_t)lane;
  const float d0 = valid ? dx : 0.f, d1 = valid ? dy : 0.f;
  const uint32_t pk = __shfl_up_sync(0xffffffffu, key, 1);
  const bool head = lane == 0 || pk != key;
  const uint32_t heads = __ballot_sync(0xffffffffu, head);
  // a run = maximal block of consecutive lanes with one key; it ends at the
  // next head (equal keys need not be contiguous: rays can revisit a cell
  // another ray left, so run membership is positional, never key equality)
  const uint32_t above = heads & ~((2u << lane) - 1u);  // heads strictly above this lane
  const int run_end = above ? __ffs(above) - 1 : 32;
  const int rlen = head ? run_end - lane : 0;
  const int rmax = __reduce_max_sync(0xffffffffu, (unsigned)rlen);
  float w[8], c[16];
  corner_weights(cell, w);
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    c[2 * corner] = w[corner] * d0;
    c[2 * corner + 1] = w[corner] * d1;
  }
  if (rmax <= pull_max) {
    for (int j = 1; j < rmax; ++j) {  // warp-uniform
      const float fx = __shfl_down_sync(0xffffffffu, cell.fx, j), fy = __shfl_down_sync(0xffffffffu, cell.fy, j),
                  fz = __shfl_down_sync(0xffffffffu, cell.fz, j);
      const float e0 = __shfl_down_sync(0xffffffffu, d0, j), e1 = __shfl_down_sync(0xffffffffu, d1, j);
      if (j < rlen) {
        LevelCell m;
        m.fx = fx;
        m.fy = fy;
        m.fz = fz;
        float wm[8];
        corner_weights(m, wm);
#pragma unroll
        for (int corner = 0; corner < 8; ++corner) {
          c[2 * corner] = fmaf(wm[corner], e0, c[2 * corner]);
          c[2 * corner + 1] = fmaf(wm[corner], e1, c[2 * corner + 1]);
        }
      }
    }
  } else {
    // segmented suffix sums: once no run is longer than `off`, larger offsets cannot match
    for (int off = 1; off < rmax; off <<= 1) {
      const bool take = lane + off < run_end;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const float tv = __shfl_down_sync(0xffffffffu, c[kk], off);
        if (take) c[kk] += tv;
      }
    }
  }
  if (skip != 1 && valid && head) {  // (skip == 1: profiling, no atomics)
    // (grouped launches load `grad` from the object table: without the hint the
    // atomics compile to generic ATOM with a shared-window check instead of REDG)
    __builtin_assume(__isGlobal(grad));
    float* gl = grad + (long long)l * 2 * fd.rows;
    uint32_t rows[8];
    corner_rows(fd, l, cell, rows);
#pragma unroll
    for (int corner = 0; corner < 8; ++corner) {
      if (c[2 * corner] == 0.f && c[2 * corner + 1] == 0.f) continue;
      atomicAdd(reinterpret_cast<float2*>(gl + (size_t)rows[corner] * 2), make_float2(c[2 * corner], c[2 * corner + 1]));
    }
  }
}

// ------------------------------------------------------------------ bwd
// TMEM column map (fp32, M=128 lane layout everywhere; 256 columns per CTA so
// two CTAs share an SM). Weight gradients are accumulated transposed,
// dW_l^T = [H_{l-1} | 1]^T D_l (rows = input units + the ones row = bias),
// so every accumulator is an M=128 tile: the output layer needs 16 columns.
template <int INP, int W, int H>
struct BwdCols {
  // Output layer: dW_out^T = [H_{H-1} | 1]^T G, M = 128 (input units + the ones
  // row = bias), 16 columns. Hidden and input layers: dW_l = D_l^T [H_{l-1} | 1],
  // M = 64 (output units: rows 16q..16q+15 in lanes 32q..32q+15), N = the
  // previous tile's width incl. its ones column -- half the tensor work of the
  // M = 128 transposed form, whose M rows beyond in+1 were padding.
  static constexpr int kDWo = 0;                       // [128 x 16]
  static constexpr int kDWl = 16;                      // layers H-1..1: [64 x (W+8)] each
  static constexpr int kDW0 = kDWl + (H - 1) * (W + 8);  // [64 x (INP+8)]
  static constexpr int kR = (kDW0 + INP + 8 + 15) / 16 * 16;  // working region, 64 columns
  static constexpr int kDF = kR + 64;            // d_features of the tile being handed over
  static constexpr int kTotal = kDF + INP;
  static_assert(kTotal <= 256, "TMEM budget");
};

// Warp-specialized: warps 0-7 ("MLP warps", named barrier 1) run the
// tensor-core chain of a tile; its last MMA writes the fp32 d_features into a
// TMEM slot that warps 8-15 ("scatter warps") load straight into registers
// (TMEM lane quadrant = warp % 4 = their sample rows), guarded by full/empty
// mbarriers. A consumer releases the slot as soon as it holds the values, so
// the scatter of tile t overlaps the MMA chain of tile t+1 and no d_features
// pass through shared memory.
#ifndef PRENOM_BWD_MLP_WARPS
#define PRENOM_BWD_MLP_WARPS 8
#endif
constexpr int kMlpWarps = PRENOM_BWD_MLP_WARPS;  // 8: two column groups per row quadrant; 4: one
constexpr int kMG = kMlpWarps / 4;
constexpr int kMlpThreads = 32 * kMlpWarps;
constexpr int kScatThreads = 256;  // two warps per 32-sample group: level halves
constexpr int kBwdMlpLevels = 1;   // per half, scattered by the MLP warps (measured on cfg2)
constexpr int kBwdPullMax = 2;     // scatter_level: pull-reduce runs up to this length (round-2 split
                                   // backward: 2 vs 4 +0.4% cfg2, +0.5% cfg1, cfg3 / bf16 equal; 3 +0.25%,
                                   // 6 -0.9%; round 1: 6 / 8 / 12 slower by 0.3 / 1 / 3.5%: pulls cost ALU,
                                   // the tree shuffles)
constexpr int kBwdThreads = kMlpThreads + kScatThreads;
// MMA / slot waits (PRENOM_BWD_WAIT bits): 1 scatter warps sleep on the slot
// barrier, 2 one MLP warp polls each MMA barrier
constexpr int kBwdWaitDefault = 0;


__device__ __forceinline__ void mlp_sync_for_mma() {
  umma::fence_proxy_async();
  umma::fence_before_sync();
  named_sync(1, kMlpThreads);
  umma::fence_after_sync();
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive2(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], 2;" ::"r"(umma::smem_u32(bar)) : "memory");
}

// Phase trace of k_bwd_tc (PRENOM_BWD_WAIT bit 3): clock64 stamps of CTA 0's
// first 64 tiles, MLP thread 0 (slots 0..10: tile start, X in, L0, L1, out,
// G ready, dWo/dH1, dW1/dH0, dW0/dX, X re-fetched, slot free) and the first
// scatter thread (0 slot full, 1 slot released, 2 scatter done); read by
// prenom_debug_bwd_trace.
__device__ long long g_bwd_trace[64][16];
__device__ long long g_bwd_strace[64][4];
// per CTA (globaltimer ns): entry, after the prologue + pdl_wait, MLP loop end, exit; tiles
__device__ long long g_bwd_cta[1024][5];
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE_CTA(slot, v)                                                              \
  do {                                                                                  \
    if ((wait_mode & 8) && tid == 0 && blockIdx.x < 1024) g_bwd_cta[blockIdx.x][slot] = (v); \
  } while (0)
#define TRACE_MLP(slot)                                                                   \
  do {                                                                                    \
    if ((wait_mode & 8) && blockIdx.x == 0 && tid == 0 && iter < 64) g_bwd_trace[iter][slot] = clock64(); \
  } while (0)
#define TRACE_SCAT(slot)                                                                            \
  do {                                                                                              \
    if ((wait_mode & 8) && blockIdx.x == 0 && tid == kMlpThreads && k < 64) g_bwd_strace[k][slot] = clock64(); \
  } while (0)

template <int INP, int W, int H, int SPL>
struct BwdLayout {
  static constexpr bool kOverlay = SPL && H >= 2;
  static constexpr size_t kOperandBytes =
      kOverlay ? (size_t)(128 * 16 * 2 * 2 + H * 128 * (W + 8) * 2 * 2 + 1024)
               : (size_t)((128 * (INP + 8) * 2 + kSlackX) + H * (128 * (W + 8) * 2 + kSlackH) + 128 * 16 * 2) *
                     (SPL ? 2 : 1);
};

// SPL: split-bf16 operands; `split` bits: 0 forward recompute, 1 the data
// products (dH, dX), 2 the weight gradients.
// GRP: grouped launch over gobj[0..nobj) (n_total = all their tiles x 128). When
// the MLP warps' tile changes object they store the weight-gradient accumulators
// as the CTA's partial of the old object (slot from slots[obj]), reload the
// weight tiles and restart the accumulation; the scatter warps follow their
// tile's object.
template <int INP, int W, int H, int SPL, bool GRP = false>
__global__ void __launch_bounds__(kBwdThreads, (SPL && H < 2) ? 1 : 2)
    k_bwd_tc(FieldDesc fd, const float* __restrict__ params, float* __restrict__ grad, long long n_total, int S,
             const int* __restrict__ count, const float4* __restrict__ pos, const uint4* __restrict__ feat_tiles,
             const float4* __restrict__ dout, int* tile_ctr, int skip_scatter, int mlp_levels,
             int pull_max, int split, int wait_mode, float* __restrict__ mlp_part, const TcObj* __restrict__ gobj,
             int nobj, int* slots) {
  using CM = BwdCols<INP, W, H>;
  using WT = WeightTiles<INP, W, H, SPL>;
  constexpr int XC = INP + 8, HC = W + 8;
  // Split mode with >= 2 hidden layers: the feature tile X overlays the last
  // hidden tile H_{H-1} (X is dead from the layer-0 MMA until dW0, and is
  // re-fetched by TMA once D_{H-1} is dead), so the operand tiles fit two CTAs
  // per SM (~110 KB each); the MN-major over-reads land in the next buffer and
  // one slack block at the end.
  constexpr bool OV = BwdLayout<INP, W, H, SPL>::kOverlay;
  // lo copies sit one (tile + slack) after the hi copies
  constexpr uint32_t XLO = SPL ? 128 * XC * 2 + (OV ? 0 : kSlackX) : 0;
  constexpr uint32_t HLO = SPL ? 128 * HC * 2 + (OV ? 0 : kSlackH) : 0;
  constexpr uint32_t GLO = SPL ? 128 * 16 * 2 : 0;
  constexpr uint32_t kFeatBytes = 128 * XC * 2 * (SPL ? 2 : 1);  // one stored tile (store_features)
  const bool sp_f = SPL && (split & 1), sp_d = SPL && (split & 2), sp_w = SPL && (split & 4);
  constexpr int NH = INP / 2;  // d_feature columns per half: [h*NH, (h+1)*NH)
  constexpr int LH = INP / 4;  // levels per half
  extern __shared__ __align__(1024) unsigned char smem[];
  const long long t_entry = (wait_mode & 8) ? gtimer() : 0;
  __shared__ uint64_t bar, xbar, full_bar, empty_bar, xfree;
  __shared__ uint32_t tbase;
  __shared__ int s_tile, s_next, s_slot;
  __shared__ long long slot_tile;
  WT wt;
  unsigned char* p = smem;
  wt.carve(p);
  unsigned char* X;      // [128][INP+8]: features | ones
  unsigned char* Ht[2];  // [128][W+8] per hidden layer: activations | ones
  unsigned char* G;      // [128][16] g_raw (4 used)
  unsigned char* zero_begin = p;
  if (OV) {
    G = p;
    p += 128 * 16 * 2 * 2;
#pragma unroll
    for (int l = 0; l < H; ++l) {
      Ht[l] = p;
      p += 128 * HC * 2 * 2;
    }
    X = Ht[H - 1];
    p += 1024;
  } else {
    X = p;
    p += (128 * XC * 2 + kSlackX) * (SPL ? 2 : 1);
    for (int l = 0; l < H; ++l) {
      Ht[l] = p;
      p += (128 * HC * 2 + kSlackH) * (SPL ? 2 : 1);
    }
    G = p;
    p += 128 * 16 * 2 * (SPL ? 2 : 1);
  }
  // D_l = dH_l * relu'(H_l) is written over H_l itself (H_l is dead once its
  // ReLU gate is taken)
  unsigned char* zero_end = p;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (!GRP && tid < kMlpThreads) wt.load(fd, params + fd.hash_params, kMlpThreads);
  {
    uint4* z = reinterpret_cast<uint4*>(zero_begin);
    const int n16 = (int)((zero_end - zero_begin) / 16);
    for (int i = tid; i < n16; i += kBwdThreads) z[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  __syncthreads();
  const __nv_bfloat16 one = __float2bfloat16_rn(1.f);
  for (int r = tid; r < 128; r += kBwdThreads) {
    *reinterpret_cast<__nv_bfloat16*>(X + umma::cm_offset(r, INP, XC)) = one;
    for (int l = 0; l < H; ++l) *reinterpret_cast<__nv_bfloat16*>(Ht[l] + umma::cm_offset(r, W, HC)) = one;
  }
  if (warp == 0) umma::tmem_alloc(&tbase, 256);
  if (tid == 0) {
    umma::mbar_init(&bar, 1);
    umma::mbar_init(&xbar, 1);
    umma::mbar_init(&xfree, 1);  // (overlay) dW0 has read X: the next tile's features may land
    umma::mbar_init(&full_bar, 2);  // the MMA commit + the issuing thread (slot_tile written)
    // one arrival per consumer warp: the scatter warps, and the MLP warps when
    // they scatter levels themselves
    umma::mbar_init(&empty_bar, kScatThreads / 32 + (mlp_levels > 0 ? kMlpThreads / 32 : 0));
    umma::fence_mbar_init();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = tbase;
  const long long ntiles = (n_total + kTile - 1) / kTile;
  pdl_wait();  // (PDL) the prologue above may overlap the compositing kernel; dout / features from here on
  TRACE_CTA(0, t_entry);
  TRACE_CTA(1, gtimer());

  if (warp >= kMlpThreads / 32) {
    // ================= scatter warps: d_features -> table gradient
    const int r = (tid - kMlpThreads) & 127;  // sample row in the tile; warp = 32 consecutive samples
    const int lhalf = (tid - kMlpThreads) >> 7;  // levels [lhalf*L/2, ...)
    int sj = 0;
    for (uint32_t k = 0;; ++k) {
      if (wait_mode & 1)
        umma::mbar_wait_sleep(&full_bar, k & 1u, 20000u);  // (sleeping waiters leave issue slots to the chain)
      else
        umma::mbar_wait(&full_bar, k & 1u);
      const long long t = slot_tile;
      if (t < 0) break;
      TRACE_SCAT(0);
      umma::fence_after_sync();
      // this half's d_features: TMEM -> registers, then the slot is released
      float d[NH];
#pragma unroll
      for (int c = 0; c < NH; c += 8) umma::tmem_ld8(umma::taddr(tm + CM::kDF, 32 * (warp & 3), lhalf * NH + c), d + c);
      umma::tmem_wait_ld();
      umma::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar);
      TRACE_SCAT(1);
      float* gr = grad;
      const int* cnt = count;
      const float4* ps = pos;
      long long tl = t, nn = n_total;
      if (GRP) {
        sj = find_obj(gobj, nobj, t, sj);
        gr = gobj[sj].grad;
        cnt = gobj[sj].count;
        ps = gobj[sj].pos;
        tl = t - gobj[sj].tile0;
        nn = gobj[sj].n;
      }
      const long long gs = tl * kTile + r;
      float4 pp = make_float4(0.f, 0.f, 0.f, 0.f);  // (loaded beside the count, as in the forward)
      bool valid = false;
      if (gs < nn) {
        pp = __ldg(ps + gs);
        valid = __ldg(cnt + ray_of(gs, S)) > 0;
      }
      if (!valid) pp = make_float4(0.f, 0.f, 0.f, 0.f);
      const float px = clamp01(pp.x), py = clamp01(pp.y), pz = clamp01(pp.z);
      // levels [lhalf*LH, (lhalf+1)*LH) belong to this half; the MLP warps
      // scatter the first mlp_levels of them. The level's pair is always
      // d[0], d[1] (the array shifts down), so the loop stays rolled without
      // indexing registers dynamically.
      const int l_lo = lhalf * LH;
      const int l_hi = skip_scatter == 2 ? l_lo : min(fd.L, (lhalf + 1) * LH);
#pragma unroll 1
      for (int l = l_lo; l < l_hi; ++l) {  // warp-uniform
        if (l >= l_lo + mlp_levels)
          scatter_level(fd, gr, l, valid, px, py, pz, d[0], d[1], lane, skip_scatter, pull_max);
#pragma unroll
        for (int i = 0; i + 2 < NH; ++i) d[i] = d[i + 2];
      }
      TRACE_SCAT(2);
    }
  } else {
    // ================= MLP warps: tensor-core backward chain
    const uint32_t tr = tm + CM::kR;
    uint32_t phase = 0, xphase = 0, xfphase = 0;
    int iter = 0;
    const int q = warp & 3, half = warp >> 2, row = 32 * q + lane;
    // MMA completion: every MLP warp polls the mbarrier, or (wait_mode bit 1)
    // warp 0 polls and the others sleep on the named barrier
    auto wait_chain = [&](uint32_t& ph) {
      if (wait_mode & 2) {
        if (warp == 0) umma::mbar_wait(&bar, ph);
        named_sync(1, kMlpThreads);
        ph ^= 1u;
        umma::fence_after_sync();
      } else {
        wait_mma(&bar, ph);
      }
    };
    // (overlay) the ones column of [X | 1] and [H_{H-1} | 1], rewritten per tile:
    // one 16-byte core-matrix row [1, 0, ..., 0] (hi) and zeros (lo) per sample
    const uint4 ones_row = make_uint4(0x3F80u, 0u, 0u, 0u), zero_row = make_uint4(0u, 0u, 0u, 0u);
    auto set_ones = [&](unsigned char* tile, int col, int C, uint32_t lo) {
      if (tid < 128) {
        *reinterpret_cast<uint4*>(tile + umma::cm_offset(tid, col, C)) = ones_row;
        *reinterpret_cast<uint4*>(tile + lo + umma::cm_offset(tid, col, C)) = zero_row;
      }
    };
    int mj = -1, oit = 0;  // (GRP) object of the weight tiles / accumulators; its tiles in this CTA so far
    auto fetch_x = [&](long long t) {  // stored features [X | 1] (hi, lo) -> X: one bulk copy per half
      const unsigned char* src = reinterpret_cast<const unsigned char*>(feat_tiles) + (size_t)t * kFeatBytes;
      if (GRP) {
        const int j = find_obj(gobj, nobj, t, mj);
        src = reinterpret_cast<const unsigned char*>(gobj[j].feat) + (size_t)(t - gobj[j].tile0) * kFeatBytes;
      }
      umma::mbar_arrive_expect_tx(&xbar, kFeatBytes);
      if (!SPL || XLO == 128 * XC * 2) {
        umma::bulk_g2s(X, src, kFeatBytes, &xbar);  // (hi | lo contiguous in smem too)
      } else {
        umma::bulk_g2s(X, src, 128 * XC * 2, &xbar);
        umma::bulk_g2s(X + XLO, src + 128 * XC * 2, 128 * XC * 2, &xbar);
      }
    };
    auto fetch = [&]() -> long long {
      if (tid == 0) s_tile = atomicAdd(tile_ctr, 1);
      named_sync(1, kMlpThreads);
      return s_tile;
    };
    // ---- the TMEM weight-gradient accumulators -> memory (warps 0-3): row = input
    // unit (or the ones row = bias), column = output unit. With a partial buffer,
    // each CTA stores its partial sums (every MLP parameter once, zeros if it had
    // no tile) and k_mlp_grad_reduce adds them in CTA order: no same-address
    // atomics from all CTAs at once (measured 25-29 us of contention), and
    // deterministic MLP gradients. Without it: one atomicAdd per weight per CTA.
    auto store_dw = [&](float* part, float* gm, bool have) {
      auto put = [&](int idx, float val) {
        if (part) part[idx] = have ? val : 0.f;
        else atomicAdd(gm + idx, val);
      };
      auto flush = [&](int col0, int ncol, int n_out, int in, int bias_row, int w_off, int b_off) {
        for (int c = 0; c < ncol; c += 8) {
          float v[8];
          umma::tmem_ld8(umma::taddr(tm, 32 * warp, col0 + c), v);
          umma::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int o = c + j;
            if (o >= n_out) continue;
            if (row < in) put(w_off + o * in + row, v[j]);
            else if (row == bias_row) put(b_off + o, v[j]);
          }
        }
      };
      // M = 64 accumulators: output unit o = 16 * warp + lane (lanes < 16), column
      // = input unit (or the ones column = bias)
      auto flush64 = [&](int col0, int ncol, int in, int ones_col, int w_off, int b_off) {
        const int o = 16 * warp + lane;
        for (int c = 0; c < ncol; c += 8) {
          float v[8];
          umma::tmem_ld8(umma::taddr(tm, 32 * warp, col0 + c), v);
          umma::tmem_wait_ld();
          if (lane >= 16 || o >= W) continue;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int k = c + j;
            if (k < in) put(w_off + o * in + k, v[j]);
            else if (k == ones_col) put(b_off + o, v[j]);
          }
        }
      };
      flush(CM::kDWo, 16, 4, W, W, fd.w_off[H], fd.b_off[H]);
      for (int l = H - 1; l >= 1; --l) flush64(CM::kDWl + (H - 1 - l) * (W + 8), W + 8, W, W, fd.w_off[l], fd.b_off[l]);
      flush64(CM::kDW0, INP + 8, fd.in_dim, INP, fd.w_off[0], fd.b_off[0]);
    };
    // (GRP) object j's partial: a slot of its buffer, then the accumulators;
    // every MLP thread calls it (named barrier), after the last MMA completed
    auto store_part = [&](int j) {
      umma::fence_after_sync();
      if (tid == 0) s_slot = atomicAdd(slots + j, 1);
      named_sync(1, kMlpThreads);
      if (warp < 4) store_dw(gobj[j].part + (size_t)s_slot * fd.mlp_params, nullptr, true);
    };
    // The next tile is claimed at the start of this one (the atomic's result is
    // only consumed mid-tile, so its latency is hidden) and its features are
    // prefetched into X by a second thread as soon as this tile's dW0 has read X:
    // only the first tile waits for its copy. (knob 3 keeps the plain loop.)
    const bool pf = skip_scatter != 3;
    bool prefetched = false;
    long long claim_reg = 0;
    for (long long t = fetch(); t < ntiles; ++iter) {
      TRACE_MLP(0);
      if (pf && tid == 0) claim_reg = atomicAdd(tile_ctr, 1);
      const float4* dp = dout;
      const int* cnt = count;
      const float4* ps = pos;
      float* gr = grad;
      long long tl = t, nn = n_total;
      if (GRP) {
        const int j = find_obj(gobj, nobj, t, mj);
        if (j != mj) {  // the previous tile's MMAs have completed (its last wait_chain)
          // warps 0-3 store the old object's partials while warps 4-7 load the new
          // weight tiles (prefetched into L2 with this tile's features)
          if (mj >= 0 && oit > 0) store_part(mj);
          if (warp >= 4) wt.load(fd, gobj[j].params + fd.hash_params, kMlpThreads - 128, tid - 128);
          // (fenced by mlp_sync_for_mma below)
          mj = j;
          oit = 0;
        }
        dp = gobj[j].dout;
        cnt = gobj[j].count;
        ps = gobj[j].pos;
        gr = gobj[j].grad;
        tl = t - gobj[j].tile0;
        nn = gobj[j].n;
      }
      const int acc_it = GRP ? oit : iter;  // tiles already in the weight-gradient accumulators
      const long long gs = tl * kTile + row;
      // upstream gradient of this row, loaded now (beside the count): its latency
      // would otherwise sit on the chain at the g_raw epilogue (warps 0-3 own the rows there)
      float4 dpre = make_float4(0.f, 0.f, 0.f, 0.f);
      bool valid = false;
      if (gs < nn) {
        if (warp < 4) dpre = __ldg(dp + gs);
        valid = __ldg(cnt + ray_of(gs, S)) > 0;
      }
      if (!valid) dpre = make_float4(0.f, 0.f, 0.f, 0.f);
      // ---- stored bf16 features -> X by the TMA engine (no LSU work): one
      // bulk copy per 8-row group (the X row-group stride is longer: ones column)
      if (tid == 0 && !prefetched) fetch_x(t);  // ([X | 1]: the ones come with the tile)
      umma::mbar_wait(&xbar, xphase);
      xphase ^= 1u;
      TRACE_MLP(1);
      mlp_sync_for_mma();
      if (skip_scatter != 3) {  // (profiling knob 3: scatter-only timing -- the MLP chain is skipped)
      // ---- forward recompute (field.cpp:181-211), one TMEM region reused per layer
      if (tid == 0) {
        for (int ks = 0; ks < INP / 16; ++ks)
          umma::mma_split(tr, umma::desc_kmajor(X, XC, ks), umma::desc_kmajor(wt.w0, INP, ks),
                          umma::idesc_bf16(128, W, false, false), ks > 0, sp_f, XLO, WT::kLo);
        umma::commit(&bar);
      }
      wait_chain(phase);
      TRACE_MLP(2);
      if (OV) set_ones(Ht[H - 1], W, HC, HLO);  // X is dead until dW0
      uint64_t gate[2];
      gate[0] = epi_relu_gate<W, kMG, HLO>(tr, wt.bias, Ht[0], HC);
#pragma unroll
      for (int l = 1; l < H; ++l) {
        mlp_sync_for_mma();
        if (tid == 0) {
          for (int ks = 0; ks < W / 16; ++ks)
            umma::mma_split(tr, umma::desc_kmajor(Ht[l - 1], HC, ks), umma::desc_kmajor(wt.wl[l - 1], W, ks),
                            umma::idesc_bf16(128, W, false, false), ks > 0, sp_f, HLO, WT::kLo);
          umma::commit(&bar);
        }
        wait_chain(phase);
        TRACE_MLP(2 + l);
        gate[l] = epi_relu_gate<W, kMG, HLO>(tr, wt.bias + l * W, Ht[l], HC);
      }
      mlp_sync_for_mma();
      if (tid == 0) {
        for (int ks = 0; ks < W / 16; ++ks)
          umma::mma_split(tr, umma::desc_kmajor(Ht[H - 1], HC, ks), umma::desc_kmajor(wt.wo, W, ks),
                          umma::idesc_bf16(128, 16, false, false), ks > 0, sp_f, HLO, WT::kLo);
        umma::commit(&bar);
      }
      wait_chain(phase);
      TRACE_MLP(4);
      // ---- g_raw (field.cpp:233-238) -> G tile
      if (warp < 4) {
        float v[8];
        umma::tmem_ld8(umma::taddr(tr, 32 * q, 0), v);
        umma::tmem_wait_ld();
        float g[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (valid) {
          const float4 d = dpre;
          const float* b = wt.bias + H * W;
          const float r0 = v[0] + b[0];
          const float sg = density_forward(fd.act, r0);
          g[0] = d.x * density_derivative(fd.act, r0, sg);
          const float s1 = stable_sigmoid(v[1] + b[1]), s2 = stable_sigmoid(v[2] + b[2]),
                      s3 = stable_sigmoid(v[3] + b[3]);
          g[1] = d.y * s1 * (1.f - s1);
          g[2] = d.z * s2 * (1.f - s2);
          g[3] = d.w * s3 * (1.f - s3);
        }
        umma::st_row8_split(G, row, 0, 16, g, GLO);
      }
      mlp_sync_for_mma();
      TRACE_MLP(5);
      // ---- output layer: dW_out^T += [H_{H-1}|1]^T G;  dH_{H-1} = G W_out
      if (tid == 0) {
        for (int ks = 0; ks < 8; ++ks)
          umma::mma_split(tm + CM::kDWo, umma::desc_mnmajor(Ht[H - 1], HC, ks), umma::desc_mnmajor(G, 16, ks),
                          umma::idesc_bf16(128, 16, true, true), (acc_it > 0 || ks > 0), sp_w, HLO, GLO);
        umma::mma_split(tr, umma::desc_kmajor(G, 16, 0), umma::desc_mnmajor(wt.wo, W, 0),
                        umma::idesc_bf16(128, W, false, true), 0u, sp_d, GLO, WT::kLo);
        umma::commit(&bar);
      }
      wait_chain(phase);
      TRACE_MLP(6);
#pragma unroll
      for (int l = H - 1; l >= 0; --l) {
        if (OV && l == 0) {  // D_{H-1} is dead: X back into its place for dW0
          if (tid == 0) fetch_x(t);
        }
        // D_l = dH_l * relu'(H_l) -> D tile
        {
          constexpr int NHD = W / kMG;
#pragma unroll
          for (int c = 0; c < NHD; c += 8) {
            const int col = half * NHD + c;
            float v[8];
            umma::tmem_ld8(umma::taddr(tr, 32 * q, col), v);
            umma::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = (gate[l] >> (c + j)) & 1ull ? v[j] : 0.f;
            umma::st_row8_split(Ht[l], row, col, HC, v, HLO);  // D_l in place of H_l
          }
        }
        if (OV && l == 0) {
          umma::mbar_wait(&xbar, xphase);
          xphase ^= 1u;
          TRACE_MLP(9);
        }
        if (l == 0 && tid == 0) s_next = (int)claim_reg;  // published by the barrier below
        mlp_sync_for_mma();
        if (tid == 0) {
          const int dwc = l == 0 ? CM::kDW0 : CM::kDWl + (H - 1 - l) * (W + 8);
          const unsigned char* prev = l == 0 ? X : Ht[l - 1];
          const int pc = l == 0 ? XC : HC;
          const uint32_t plo = l == 0 ? XLO : HLO;
          // dW_l = D_l^T [prev | 1]: A = D_l (MN-major, M = 64 units), B = prev (MN-major, N = pc)
          for (int ks = 0; ks < 8; ++ks)
            umma::mma_split_terms(tm + dwc, umma::desc_mnmajor(Ht[l], HC, ks), umma::desc_mnmajor(prev, pc, ks),
                                  umma::idesc_bf16(64, pc, true, true), (acc_it > 0 || ks > 0), sp_w && !(split & 32),
                                  sp_w && !(split & 16), HLO, plo);
          if (pf && l == 0) umma::commit(&xfree);  // dW0 is the last reader of X
          if (l > 0) {
            for (int ks = 0; ks < W / 16; ++ks)
              umma::mma_split(tr, umma::desc_kmajor(Ht[l], HC, ks), umma::desc_mnmajor(wt.wl[l - 1], W, ks),
                              umma::idesc_bf16(128, W, false, true), ks > 0, sp_d, HLO, WT::kLo);
          } else {
            // d_features -> the TMEM slot, once every consumer holds the previous tile's
            umma::mbar_wait(&empty_bar, ((uint32_t)iter & 1u) ^ 1u);
            TRACE_MLP(10);
            slot_tile = t;
            for (int ks = 0; ks < W / 16; ++ks)
              umma::mma_split(tm + CM::kDF, umma::desc_kmajor(Ht[l], HC, ks), umma::desc_mnmajor(wt.w0, INP, ks),
                              umma::idesc_bf16(128, INP, false, true), ks > 0, sp_d, HLO, WT::kLo);
          }
          umma::commit(&bar);
          if (l == 0) {
            umma::commit(&full_bar);
            mbar_arrive(&full_bar);
          }
        }
        if (pf && l == 0 && tid == 32) {
          // a second thread copies the next tile's features into X once dW0 is done with
          // it, in parallel with the issuing thread's dX / slot hand-over
          umma::mbar_wait(&xfree, xfphase);
          xfphase ^= 1u;
          if (s_next < ntiles) {
            fetch_x(s_next);
            if (GRP) {
              const int nj = find_obj(gobj, nobj, s_next, mj);
              if (nj != mj) prefetch_mlp_l2(fd, gobj[nj].params, 0, 1);
            }
          }
        }
        wait_chain(phase);
        TRACE_MLP(7 + (H - 1 - l));
      }
      } else if (tid == 0) {  // (knob 3: no chain; hand over the stale slot)
        umma::mbar_wait(&empty_bar, ((uint32_t)iter & 1u) ^ 1u);
        slot_tile = t;
        mbar_arrive2(&full_bar);
      }
      // ---- this half's first mlp_levels levels, scattered by the MLP warps
      // straight from the slot, overlapping the scatter warps' share
      if (mlp_levels > 0) {
        // (knob 3 has no MMA to order this load after the slot's hand-over)
        if (skip_scatter == 3) umma::mbar_wait(&full_bar, (uint32_t)iter & 1u);
        float v[2 / kMG][8];
#pragma unroll
        for (int k = 0; k < 2 / kMG; ++k) umma::tmem_ld8(umma::taddr(tm + CM::kDF, 32 * q, (half + k) * NH), v[k]);
        umma::tmem_wait_ld();
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar);
        if (skip_scatter != 2) {
          float4 pp = make_float4(0.f, 0.f, 0.f, 0.f);
          if (valid) pp = ps[gs];
          const float px = clamp01(pp.x), py = clamp01(pp.y), pz = clamp01(pp.z);
#pragma unroll
          for (int k = 0; k < 2 / kMG; ++k) {
            const int l0 = (half + k) * LH;
#pragma unroll 1
            for (int j = 0; j < mlp_levels && l0 + j < fd.L; ++j) {  // warp-uniform
              scatter_level(fd, gr, l0 + j, valid, px, py, pz, v[k][0], v[k][1], lane, skip_scatter, pull_max);
#pragma unroll
              for (int i2 = 0; i2 < 6; ++i2) v[k][i2] = v[k][i2 + 2];
            }
          }
        }
      }
      ++oit;
      // next tile: claimed (and its features prefetched) by the issuing thread
      if (pf) {
        named_sync(1, kMlpThreads);
        t = s_next;
        prefetched = true;
      } else {
        t = fetch();
      }
    }
    TRACE_CTA(2, gtimer());
    TRACE_CTA(4, (long long)iter);
    // sentinel: stop the scatter warps
    if (tid == 0) {
      umma::mbar_wait(&empty_bar, ((uint32_t)iter & 1u) ^ 1u);
      slot_tile = -1;
      mbar_arrive2(&full_bar);
    }
    umma::fence_after_sync();
    if (GRP) {
      if (mj >= 0 && oit > 0) store_part(mj);
    } else if (warp < 4 && (iter > 0 || mlp_part)) {
      store_dw(mlp_part ? mlp_part + (size_t)blockIdx.x * fd.mlp_params : nullptr, grad + fd.hash_params, iter > 0);
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 256);
  TRACE_CTA(3, gtimer());
}

// MLP weight gradients: grad[i] += sum over the backward's CTAs of their partials.
// Block = 32 parameters x 32 row groups: each thread sums every 32nd CTA row (a
// short, independent load chain: the partials were just written and sit in L2),
// then the 32 group sums are added in fixed order -- deterministic.
__device__ __forceinline__ void mlp_grad_reduce(const float* __restrict__ part, int nparts, int P,
                                                float* __restrict__ g) {
  __shared__ float red[32][33];
  const int c = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + c;
  float a0 = 0.f, a1 = 0.f;
  if (i < P) {
    int r = grp;
    for (; r + 32 < nparts; r += 64) {
      a0 += part[(size_t)r * P + i];
      a1 += part[(size_t)(r + 32) * P + i];
    }
    if (r < nparts) a0 += part[(size_t)r * P + i];
  }
  red[grp][c] = a0 + a1;
  __syncthreads();
  if (grp == 0 && i < P) {
    float acc = red[0][c];
#pragma unroll 8
    for (int k = 1; k < 32; ++k) acc += red[k][c];
    g[i] += acc;
  }
}

__global__ void __launch_bounds__(1024) k_mlp_grad_reduce(const float* __restrict__ part, int nparts, int P,
                                                          float* __restrict__ g) {
  pdl_wait();
  mlp_grad_reduce(part, nparts, P, g);
}

// grouped: blockIdx.y = object, its partials = the slots its CTAs took
__global__ void __launch_bounds__(1024) k_mlp_grad_reduce_grp(const TcObj* __restrict__ gobj, const int* slots, int P,
                                                              long long hash_params) {
  pdl_wait();
  const TcObj& o = gobj[blockIdx.y];
  mlp_grad_reduce(o.part, slots[blockIdx.y], P, o.grad + hash_params);
}

// Persistent-grid sizing hint: under the multi-object scheduler (concurrent
// lane streams, ~1k tiles per object) each CTA takes at least 8 tiles, so the
// per-CTA prologue (weight tiles, TMEM alloc) is amortised and the lanes keep
// SMs for each other's kernels (cfg5 9.9e8 -> 1.12e9, cfg3 1.34e9 -> 1.41e9);
// a single object keeps the full grid (cfg4's 2k-tile steps lose 3% at 8).
// Set per host thread by prenom_train_step_many; PRENOM_MIN_TILES_PER_CTA overrides.
thread_local int t_min_tiles = 1;

int min_tiles_per_cta() {
  static const int env = [] {
    const char* e = getenv("PRENOM_MIN_TILES_PER_CTA");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  return env ? env : t_min_tiles;
}

int g_sms = 0;
int sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_sms;
}

template <int INP, int W, int H, int SPL>
size_t fwd_smem() {
  static_assert(W >= INP, "split-mode X overlays the activation tile");
  return WeightTiles<INP, W, H, SPL>::kBytes + ((H * W + 4) * 4 + 15) / 16 * 16 +
         (SPL ? 128 * W * 2 * 2 : 128 * INP * 2 + 128 * W * 2) + 1024;
}

template <int INP, int W, int H, int SPL>
size_t bwd_smem() {
  return WeightTiles<INP, W, H, SPL>::kBytes + ((H * W + 4) * 4 + 15) / 16 * 16 + BwdLayout<INP, W, H, SPL>::kOperandBytes +
         1024;
}

// cudaFuncSetAttribute only when a kernel's (shared memory, carve-out) changes:
// the attributes persist, and two driver calls per launch are host time on
// every step (the timed region enqueues ~7 launches per step).
// (Keyed by device too: function attributes belong to the device's context.)
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, std::pair<size_t, int>> g_attr;
template <class K>
cudaError_t set_attrs(K kern, size_t smem, int carveout) {
  int dev = 0;
  cudaError_t ed = cudaGetDevice(&dev);
  if (ed != cudaSuccess) return ed;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  const std::pair<int, const void*> key{dev, reinterpret_cast<const void*>(kern)};
  auto it = g_attr.find(key);
  if (it != g_attr.end() && it->second == std::make_pair(smem, carveout)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (carveout >= 0) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
    if (e != cudaSuccess) return e;
  }
  g_attr[key] = {smem, carveout};
  return cudaSuccess;
}

template <int INP, int W, int H, int SPL>
size_t fwd_ts_smem() {
  return WeightTiles<INP, W, H, SPL>::kBytes + ((H * W + 4) * 4 + 15) / 16 * 16 + 128 * INP * 2 * (SPL ? 2 : 1) + 1024;
}

template <int INP, int W, int H, int NT, int SPL>
cudaError_t run_fwd_nt(const FieldDesc& fd, const float* params, long long n, int S, const int* count,
                       const float4* pos, void* feat_tiles, float4* out, int* flag, int* tile_ctr, int ctas,
                       size_t min_smem, int carveout, int split, int ts, cudaStream_t st) {
  // ts: 1 = TMEM activations (k_fwd_ts), 2 = + warp-specialised encode (k_fwd_ws: 16 encode warps,
  // 2 CTAs/SM; measured on cfg2 split: 12 x 2 within 2%, 28 x 1 and 24 x 1 +40%: one MLP chain per SM)
  // ts == 3: k_fwd_wx (features in TMEM as well; weights-only shared memory)
  auto kern = ts == 2 ? k_fwd_ws<INP, W, H, SPL> : ts ? k_fwd_ts<INP, W, H, NT, SPL> : k_fwd_tc<INP, W, H, NT, SPL>;
  const size_t smem = std::max<size_t>(ts == 3   ? fwd_ts_smem<INP, W, H, SPL>() - 128 * INP * 2 * (SPL ? 2 : 1)
                                       : ts == 2 ? fwd_ts_smem<INP, W, H, SPL>() + 128 * INP * 2 * (SPL ? 2 : 1)
                                       : ts     ? fwd_ts_smem<INP, W, H, SPL>()
                                                : fwd_smem<INP, W, H, SPL>(),
                                       min_smem);
  const int nthreads = ts >= 2 ? kWsThreads : NT;
  // shared-memory carve-out (percent of the maximum): the rest of the 256 KB
  // array is L1, which serves the encode's gathers
  const long long ntiles = (n + kTile - 1) / kTile;
  const long long grid = std::min<long long>((ntiles + min_tiles_per_cta() - 1) / min_tiles_per_cta(), (long long)ctas * sms());
  if (ts == 3) {
    auto kx = k_fwd_wx<INP, W, H, SPL>;
    cudaError_t e = set_attrs(kx, smem, carveout);
    if (e != cudaSuccess) return e;
    return launch_pdl(kx, dim3((unsigned)grid), dim3(WxShape<H>::kThreads), smem, st, fd, params, n, S, count, pos,
                      reinterpret_cast<uint4*>(feat_tiles), out, flag, tile_ctr, split, (const TcObj*)nullptr, 0);
  }
  cudaError_t e = set_attrs(kern, smem, carveout);
  if (e != cudaSuccess) return e;
  return launch_pdl(kern, dim3((unsigned)grid), dim3(nthreads), smem, st, fd, params, n, S, count, pos,
                    reinterpret_cast<uint4*>(feat_tiles), out, flag, tile_ctr, split);
}

// grouped forward (k_fwd_wx<..., GRP>): same shape and carve-out as the single-object one
template <int INP, int W, int H>
cudaError_t run_fwd_grp(const FieldDesc& fd, const TcObj* objs, int nobj, long long ntiles, int S, int* ctr, int split,
                        cudaStream_t st) {
  const int carve = split ? kFwdSTsCarveout : kFwdWsCarveout;
  auto kx = split ? k_fwd_wx<INP, W, H, 1, true> : k_fwd_wx<INP, W, H, 0, true>;
  const size_t smem = split ? fwd_ts_smem<INP, W, H, 1>() - 128 * INP * 2 * 2 : fwd_ts_smem<INP, W, H, 0>() - 128 * INP * 2;
  cudaError_t e = set_attrs(kx, smem, carve);
  if (e != cudaSuccess) return e;
  const long long grid = std::min<long long>((ntiles + min_tiles_per_cta() - 1) / min_tiles_per_cta(), 2LL * sms());
  return launch_pdl(kx, dim3((unsigned)grid), dim3(WxShape<H>::kThreads), smem, st, fd, (const float*)nullptr, ntiles * kTile,
                    S, (const int*)nullptr, (const float4*)nullptr, (uint4*)nullptr, (float4*)nullptr, (int*)nullptr,
                    ctr, split, objs, nobj);
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <int INP, int W, int H>
cudaError_t run_fwd(const FieldDesc& fd, const float* params, long long n, int S, const int* count, const float4* pos,
                    void* feat_tiles, float4* out, int* flag, int* tile_ctr, int split, cudaStream_t st) {
  // CTAs per SM x threads per CTA trade gather latency hiding against L1
  // capacity (L1 = 256 KB - the shared-memory carve-out);
  // PRENOM_FWD{,S}_{CTAS,SMEM_KB,THREADS,CARVEOUT,TS} override the measured
  // defaults of the bf16 / split (S) forward; TS = activations in TMEM (k_fwd_ts)
  if (split) {
    static const int ts = env_int("PRENOM_FWDS_TS", kFwdSTsDefault);
    static const int nt = env_int("PRENOM_FWDS_THREADS", ts ? kFwdSTsThreads : kFwdSThreadsDefault) == 512 ? 512 : 256;
    static const int ctas = std::max(1, std::min(8, env_int("PRENOM_FWDS_CTAS", ts ? kFwdSTsCtas : kFwdSCtasDefault)));
    static const size_t min_smem = (size_t)env_int("PRENOM_FWDS_SMEM_KB", 0) * 1024;
    // carve-out per kernel: wx 64 KB (weights only), ws 132 KB (+ two feature buffers), ts 100 KB
    static const int carve = env_int("PRENOM_FWDS_CARVEOUT", ts == 3 ? kFwdSTsCarveout : ts == 2 ? 58 : ts ? 44
                                                                                                      : kFwdSCarveoutDefault);
    if (nt == 512)
      return run_fwd_nt<INP, W, H, 512, 1>(fd, params, n, S, count, pos, feat_tiles, out, flag, tile_ctr, ctas,
                                           min_smem, carve, split, ts, st);
    return run_fwd_nt<INP, W, H, 256, 1>(fd, params, n, S, count, pos, feat_tiles, out, flag, tile_ctr, ctas, min_smem,
                                         carve, split, ts, st);
  }
  static const int ts = env_int("PRENOM_FWD_TS", kFwdTsDefault);
  static const int nt = env_int("PRENOM_FWD_THREADS", kFwdThreadsDefault) == 512 ? 512 : 256;
  static const int ctas = std::max(1, std::min(8, env_int("PRENOM_FWD_CTAS", ts >= 2 ? 2 : kFwdCtasDefault)));
  static const size_t min_smem = (size_t)env_int("PRENOM_FWD_SMEM_KB", ts ? 0 : kFwdSmemKbDefault) * 1024;
  static const int carve = env_int("PRENOM_FWD_CARVEOUT", ts >= 2 ? kFwdWsCarveout : kFwdCarveoutDefault);  // (ws, wx: 64 KB)
  if (nt == 512)
    return run_fwd_nt<INP, W, H, 512, 0>(fd, params, n, S, count, pos, feat_tiles, out, flag, tile_ctr, ctas, min_smem,
                                         carve, 0, ts, st);
  return run_fwd_nt<INP, W, H, 256, 0>(fd, params, n, S, count, pos, feat_tiles, out, flag, tile_ctr, ctas, min_smem,
                                       carve, 0, ts, st);
}

template <int INP, int W, int H, int SPL>
cudaError_t run_bwd_s(const FieldDesc& fd, const float* params, float* grad, long long n, int S, const int* count,
                      const float4* pos, const void* feat_tiles, const float4* dout, int* tile_ctr, int split,
                      float* mlp_part, size_t part_cap, int* defer_nparts, cudaStream_t st) {
  // plain bf16: two CTAs (2 x 256 TMEM columns) per SM, the shared-memory
  // floor keeps a third CTA out; PRENOM_BWD_SMEM_KB / PRENOM_BWD_CARVEOUT for tuning
  static const size_t min_smem = (size_t)env_int("PRENOM_BWD_SMEM_KB", SPL ? 0 : 80) * 1024;
  static const int carveout = env_int("PRENOM_BWD_CARVEOUT", -1);
  auto kern = k_bwd_tc<INP, W, H, SPL>;
  const size_t smem = std::max<size_t>(bwd_smem<INP, W, H, SPL>(), min_smem);
  cudaError_t e = set_attrs(kern, smem, carveout);
  if (e != cudaSuccess) return e;
  const long long ntiles = (n + kTile - 1) / kTile;
  const int per_sm = std::max(1, (int)(kSmemPerSm / (smem + 1024)));
  const long long grid =
      std::min<long long>((ntiles + min_tiles_per_cta() - 1) / min_tiles_per_cta(), (long long)std::min(2, per_sm) * sms());
  // levels per half the MLP warps scatter themselves (they would otherwise
  // wait on the scatter warps); PRENOM_BWD_MLP_LEVELS overrides for tuning
  static const int mlp_env = env_int("PRENOM_BWD_MLP_LEVELS", -1);
  // the MLP warps load 8 slot columns: at most 4 levels per half
  // (split mode: 0 -- the MLP chain, not the scatter, bounds the kernel)
  const int mlp_levels =
      std::max(0, std::min(std::min(4, INP / 4), mlp_env >= 0 ? mlp_env : (SPL ? 0 : kBwdMlpLevels)));
  static const int skip = env_int("PRENOM_PROF_SKIP_SCATTER", 0);
  // longest run reduced by pulls (else by the shuffle tree); PRENOM_BWD_PULL_MAX overrides
  static const int pull_max = env_int("PRENOM_BWD_PULL_MAX", kBwdPullMax);
  static const int wait_mode = env_int("PRENOM_BWD_WAIT", kBwdWaitDefault);
  // tile_ctr[0] was zeroed by the forward of the same step (tile_sched_exit resets
  // its [2], which is this counter)
  float* part = mlp_part && (size_t)grid * fd.mlp_params <= part_cap ? mlp_part : nullptr;
  cudaError_t e2 = launch_pdl(kern, dim3((unsigned)grid), dim3(kBwdThreads), smem, st, fd, params, grad, n, S, count,
                              pos, reinterpret_cast<const uint4*>(feat_tiles), dout, tile_ctr, skip, mlp_levels,
                              pull_max, split, wait_mode, part, (const TcObj*)nullptr, 0, (int*)nullptr);
  if (defer_nparts) *defer_nparts = part ? (int)grid : 0;  // the caller's Adam sums the partials
  if (e2 != cudaSuccess || !part || defer_nparts) return e2;
  return launch_pdl(k_mlp_grad_reduce, dim3((unsigned)((fd.mlp_params + 31) / 32)), dim3(1024), 0, st,
                    (const float*)part, (int)grid, fd.mlp_params, grad + fd.hash_params);
}

// grouped backward + the per-object MLP-gradient reduction (blockIdx.y = object).
// Each object's partial buffer holds tc_mlp_part_floats: one slot per CTA at most
// (a CTA walks increasing tiles, so it leaves an object once).
template <int INP, int W, int H, int SPL>
cudaError_t run_bwd_grp_s(const FieldDesc& fd, const TcObj* objs, int nobj, long long ntiles, int S, int* ctr,
                          int split, cudaStream_t st) {
  static const size_t min_smem = (size_t)env_int("PRENOM_BWD_SMEM_KB", SPL ? 0 : 80) * 1024;
  static const int carveout = env_int("PRENOM_BWD_CARVEOUT", -1);
  auto kern = k_bwd_tc<INP, W, H, SPL, true>;
  const size_t smem = std::max<size_t>(bwd_smem<INP, W, H, SPL>(), min_smem);
  cudaError_t e = set_attrs(kern, smem, carveout);
  if (e != cudaSuccess) return e;
  const int per_sm = std::max(1, (int)(kSmemPerSm / (smem + 1024)));
  const long long grid =
      std::min<long long>((ntiles + min_tiles_per_cta() - 1) / min_tiles_per_cta(), (long long)std::min(2, per_sm) * sms());
  const int mlp_levels = SPL ? 0 : std::min(kBwdMlpLevels, INP / 4);
  static const int wait_mode = env_int("PRENOM_BWD_WAIT", kBwdWaitDefault);
  e = cudaMemsetAsync(ctr, 0, sizeof(int) * (1 + nobj), st);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kern, dim3((unsigned)grid), dim3(kBwdThreads), smem, st, fd, (const float*)nullptr, (float*)nullptr,
                 ntiles * kTile, S, (const int*)nullptr, (const float4*)nullptr, (const uint4*)nullptr,
                 (const float4*)nullptr, ctr, 0, mlp_levels, kBwdPullMax, split, wait_mode, (float*)nullptr, objs,
                 nobj, ctr + 1);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_mlp_grad_reduce_grp, dim3((unsigned)((fd.mlp_params + 31) / 32), (unsigned)nobj), dim3(1024), 0,
                    st, objs, (const int*)(ctr + 1), fd.mlp_params, fd.hash_params);
}

template <int INP, int W, int H>
cudaError_t run_bwd_grp(const FieldDesc& fd, const TcObj* objs, int nobj, long long ntiles, int S, int* ctr, int split,
                        cudaStream_t st) {
  if (split) return run_bwd_grp_s<INP, W, H, 1>(fd, objs, nobj, ntiles, S, ctr, split, st);
  return run_bwd_grp_s<INP, W, H, 0>(fd, objs, nobj, ntiles, S, ctr, 0, st);
}

template <int INP, int W, int H>
cudaError_t run_bwd(const FieldDesc& fd, const float* params, float* grad, long long n, int S, const int* count,
                    const float4* pos, const void* feat_tiles, const float4* dout, int* tile_ctr, int split,
                    float* mlp_part, size_t part_cap, int* defer_nparts, cudaStream_t st) {
  if (split)
    return run_bwd_s<INP, W, H, 1>(fd, params, grad, n, S, count, pos, feat_tiles, dout, tile_ctr, split, mlp_part,
                                   part_cap, defer_nparts, st);
  return run_bwd_s<INP, W, H, 0>(fd, params, grad, n, S, count, pos, feat_tiles, dout, tile_ctr, 0, mlp_part,
                                 part_cap, defer_nparts, st);
}

#define PRENOM_TC_DISPATCH(FN, ...)                                                          \
  do {                                                                                       \
    const int inp = fd.in_dim <= 16 ? 16 : 32;                                               \
    if (inp == 16 && fd.W == 32 && fd.H == 1) return FN<16, 32, 1>(__VA_ARGS__);             \
    if (inp == 16 && fd.W == 32 && fd.H == 2) return FN<16, 32, 2>(__VA_ARGS__);             \
    if (inp == 16 && fd.W == 64 && fd.H == 1) return FN<16, 64, 1>(__VA_ARGS__);             \
    if (inp == 16 && fd.W == 64 && fd.H == 2) return FN<16, 64, 2>(__VA_ARGS__);             \
    if (inp == 32 && fd.W == 32 && fd.H == 1) return FN<32, 32, 1>(__VA_ARGS__);             \
    if (inp == 32 && fd.W == 32 && fd.H == 2) return FN<32, 32, 2>(__VA_ARGS__);             \
    if (inp == 32 && fd.W == 64 && fd.H == 1) return FN<32, 64, 1>(__VA_ARGS__);             \
    if (inp == 32 && fd.W == 64 && fd.H == 2) return FN<32, 64, 2>(__VA_ARGS__);             \
    return cudaErrorInvalidValue;                                                            \
  } while (0)

}  // namespace

// On by default (cfg2, B200, interleaved 3x: 0.7001 -> 0.6940 ms/step);
// PRENOM_NO_PDL=1 disables for A/B.
void tc_set_min_tiles_per_cta(int v) { t_min_tiles = v < 1 ? 1 : v; }
bool tc_concurrent_objects() { return t_min_tiles > 1; }

bool pdl_enabled() {
  static const bool on = getenv("PRENOM_NO_PDL") == nullptr;
  return on;
}

cudaError_t tc_bwd_trace(long long* mlp, long long* scat, long long* cta) {
  cudaError_t e = cudaMemcpyFromSymbol(mlp, g_bwd_trace, sizeof(g_bwd_trace));
  if (e != cudaSuccess) return e;
  e = cudaMemcpyFromSymbol(scat, g_bwd_strace, sizeof(g_bwd_strace));
  if (e != cudaSuccess || !cta) return e;
  return cudaMemcpyFromSymbol(cta, g_bwd_cta, sizeof(g_bwd_cta));
}

bool tc_supported(const FieldDesc& fd) {
  for (int l = 0; l < fd.L; ++l)
    if (fd.res[l] > 1625) return false;  // scatter de-dup key: the cell index fits 32 bits (1625^3 < 2^32)
  return fd.F == 2 && fd.in_dim <= 32 && (fd.W == 32 || fd.W == 64) && (fd.H == 1 || fd.H == 2);
}

size_t tc_feature_bytes(const FieldDesc& fd, long long n, int split) {
  const int inp = fd.in_dim <= 16 ? 16 : 32;
  return (size_t)((n + kTile - 1) / kTile) * kTile * (inp + 8) * 2 * (split ? 2 : 1);
}

cudaError_t init_feature_tiles(const FieldDesc& fd, void* feat, size_t bytes, int split, cudaStream_t st) {
  const int inp = fd.in_dim <= 16 ? 16 : 32;
  const long long ntiles = (long long)(bytes / ((size_t)128 * (inp + 8) * 2 * (split ? 2 : 1)));
  if (ntiles <= 0) return cudaSuccess;
  k_feature_ones<<<std::max(1, std::min(4 * sms(), (int)((ntiles * 256 + 255) / 256))), 256, 0, st>>>(
      reinterpret_cast<unsigned char*>(feat), ntiles, inp, split);
  return cudaGetLastError();
}

// split: 0 = bf16 operands; else split-bf16 with the cross products enabled
// per bit (1 forward, 2 backward data products, 4 weight gradients; 16 / 32
// drop the D_lo*prev_hi / D_hi*prev_lo term of the hidden/input weight
// gradients -- numerics experiments).
// PRENOM_SPLIT_MASK overrides the mask of split-mode calls (bisection).
int split_mask(int split) {
  static const int m = env_int("PRENOM_SPLIT_MASK", 7);
  return split ? (m | 8) : 0;  // bit 3 keeps "split mode" set when the mask is 0
}

cudaError_t launch_fwd_tc(const FieldDesc& fd, const float* params, long long n, int S, const int* count,
                          const float4* pos, void* feat_tiles, float4* out, int* flag, int* tile_ctr, int split,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n + kTile >= (1LL << 31)) return cudaErrorInvalidValue;  // ray_of's 32-bit slot index
  split = split_mask(split);
  PRENOM_TC_DISPATCH(run_fwd, fd, params, n, S, count, pos, feat_tiles, out, flag, tile_ctr, split, st);
}

size_t tc_mlp_part_floats(const FieldDesc& fd) { return (size_t)2 * sms() * fd.mlp_params; }

cudaError_t launch_fwd_tc_group(const FieldDesc& fd, const TcObj* objs, int nobj, long long ntiles, int S, int* ctr,
                                int split, cudaStream_t st) {
  if (ntiles <= 0 || nobj <= 0) return cudaSuccess;
  split = split_mask(split);
  PRENOM_TC_DISPATCH(run_fwd_grp, fd, objs, nobj, ntiles, S, ctr, split, st);
}

cudaError_t launch_bwd_tc_group(const FieldDesc& fd, const TcObj* objs, int nobj, long long ntiles, int S, int* ctr,
                                int split, cudaStream_t st) {
  if (ntiles <= 0 || nobj <= 0) return cudaSuccess;
  split = split_mask(split);
  PRENOM_TC_DISPATCH(run_bwd_grp, fd, objs, nobj, ntiles, S, ctr, split, st);
}

cudaError_t launch_bwd_tc(const FieldDesc& fd, const float* params, float* grad, long long n, int S,
                          const int* count, const float4* pos, const void* feat_tiles, const float4* dout,
                          int* tile_ctr, int split, float* mlp_part, size_t part_cap, cudaStream_t st,
                          int* defer_nparts) {
  if (defer_nparts) *defer_nparts = 0;
  if (n <= 0) return cudaSuccess;
  if (n + kTile >= (1LL << 31)) return cudaErrorInvalidValue;  // ray_of's 32-bit slot index
  split = split_mask(split);
  PRENOM_TC_DISPATCH(run_bwd, fd, params, grad, n, S, count, pos, feat_tiles, dout, tile_ctr, split, mlp_part,
                     part_cap, defer_nparts, st);
}

}  // namespace prenom
