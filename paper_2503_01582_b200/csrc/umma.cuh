// umma.cuh -- minimal hand-written sm_100a tcgen05 (UMMA) toolkit:
// shared-memory matrix descriptors (SWIZZLE_NONE canonical "interleaved"
// core-matrix layouts), bf16 x bf16 -> fp32 tcgen05.mma issued by one thread,
// tcgen05.commit -> mbarrier completion, TMEM alloc/ld, and the proxy/thread
// fences that order them. Bit layouts follow the sm_100 descriptor formats
// (smem descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), layout type [61,64); instruction descriptor: D fmt
// [4,6), A fmt [7,10), B fmt [10,13), A/B major bits 15/16, N>>3 [17,23),
// M>>4 [24,29)).
//
// Operand tile layout used everywhere ("core-matrix interleaved"): a bf16
// buffer with R rows and C columns is stored as 8x8-element core matrices
// (128 contiguous bytes: 8 rows x 16 B, columns contiguous inside a row):
//     byte(r, c) = (r/8) * (C/8)*128 + (c/8) * 128 + (r%8) * 16 + (c%8) * 2
// The same buffer is a K-major operand when C is the MMA K dimension
// (LBO = 128, SBO = C/8*128) and an MN-major operand when C is the MMA M/N
// dimension (SBO = 128, LBO = C/8*128): the backward pass reuses forward
// activations and weights as transposed operands without copying them.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace prenom {
namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Byte offset of element (r, c) in a core-matrix-interleaved [R][C] tile.
__host__ __device__ __forceinline__ uint32_t cm_offset(int r, int c, int C) {
  return (uint32_t)((r >> 3) * (C >> 3) * 128 + (c >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // sm_100 descriptor version
  return d;                // base offset 0, SWIZZLE_NONE
}

// K-major operand view of a [rows][C] tile, MMA K-step `ks` (16 columns).
__device__ __forceinline__ uint64_t desc_kmajor(const void* tile, int C, int ks) {
  return make_desc(smem_u32(tile) + (uint32_t)ks * 256u, 128u, (uint32_t)(C >> 3) * 128u);
}

// MN-major operand view of a [rows][C] tile whose rows are the MMA K
// dimension and whose columns are the MMA M (or N) dimension; K-step `ks`
// covers buffer rows [16 ks, 16 ks + 16). mn0 selects the first M/N column.
__device__ __forceinline__ uint64_t desc_mnmajor(const void* tile, int C, int ks, int mn0 = 0) {
  return make_desc(smem_u32(tile) + (uint32_t)ks * 2u * (uint32_t)(C >> 3) * 128u + (uint32_t)(mn0 >> 3) * 128u,
                   (uint32_t)(C >> 3) * 128u, 128u);
}

// kind::f16 instruction descriptor: bf16 A/B, fp32 D.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T (one thread issues for the CTA).
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] * B[smem]^T: the A operand (M x K, K-major, 16-bit
// elements packed two per 32-bit column, lower k in the low half; row = lane)
// is read from tensor memory ("TS" form) -- activations produced by an
// epilogue never pass through shared memory.
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Arrive on an mbarrier when all prior tcgen05.mma of this thread complete.
__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  const uint32_t a = smem_u32(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}
// Same, but the waiting warp is suspended in hardware (up to `ns`) instead of
// re-polling: for waits that are long compared with the issue slots a spin
// would take from co-resident warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* mbar, uint32_t phase, uint32_t ns = 1000000u) {
  const uint32_t a = smem_u32(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(phase), "r"(ns)
        : "memory");
  }
}

__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Warp-collective TMEM allocation (power-of-2 columns >= 32).
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 lanes x 32-bit, 16 consecutive columns per thread (lane = warp quadrant row).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32-bit, 4 consecutive columns per thread (the inverse of tmem_ld).
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}

// 32 lanes x 32-bit, one column per thread.
__device__ __forceinline__ void tmem_st1(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// TMEM address of (lane, column) relative to an allocation base.
__device__ __forceinline__ uint32_t taddr(uint32_t base, int lane, int col) {
  return base + ((uint32_t)lane << 16) + (uint32_t)col;
}

// Plain arrive (count 1) on an mbarrier, release semantics for this thread's prior writes.
__device__ __forceinline__ void mbar_arrive_plain(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}

// TMA bulk copy global -> shared (no tensor map: 1-D, 16 B aligned, size % 16
// == 0), completing `bytes` of transaction count on the mbarrier.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}

// TMA bulk copy shared -> global (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// bulk store without the commit (several copies, one bulk group: bulk_commit)
__device__ __forceinline__ void bulk_s2g_part(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// the source shared memory of every committed bulk store has been read
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed bulk store has completed
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Store 8 consecutive bf16 of row r, columns [c0, c0+8) (c0 % 8 == 0) as one
// 16-byte vector into a core-matrix tile with C columns.
__device__ __forceinline__ void st_row8(unsigned char* tile, int r, int c0, int C, const float* v) {
  __nv_bfloat162 p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(tile + cm_offset(r, c0, C)) = *reinterpret_cast<uint4*>(p);
}

// Split-bf16 ("bf16x3") operands: x = hi + lo with hi = bf16(x) and
// lo = bf16(x - hi), so a product a*b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi keeps
// ~16 significand bits (the dropped a_lo b_lo term is 2^-16 relative) while
// every MMA stays kind::f16 at full bf16 tensor rate. The lo copy of a tile sits
// `lo_off` bytes after the hi copy, so its descriptor is the hi descriptor plus
// lo_off >> 4 in the start-address field.
// Numerics experiment (-DPRENOM_TF32_EMUL, never in the product build): every MLP
// operand rounded to tf32 (cvt.rna) before the hi/lo split, so the split MMAs
// compute exact products of tf32 operands -- what a kind::tf32 MLP would do.
__device__ __forceinline__ float operand_round(float x) {
#ifdef PRENOM_TF32_EMUL
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
#else
  return x;
#endif
}

__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  x = operand_round(x);
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

__device__ __forceinline__ uint64_t desc_add(uint64_t d, uint32_t byte_off) { return d + (uint64_t)(byte_off >> 4); }

// st_row8 of the hi and (when lo_off != 0) lo parts.
__device__ __forceinline__ void st_row8_split(unsigned char* tile, int r, int c0, int C, const float* v,
                                              uint32_t lo_off) {
  if (!lo_off) {
    st_row8(tile, r, c0, C, v);
    return;
  }
  __nv_bfloat16 h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) split_bf16(v[i], h[i], l[i]);
  *reinterpret_cast<uint4*>(tile + cm_offset(r, c0, C)) = *reinterpret_cast<uint4*>(h);
  *reinterpret_cast<uint4*>(tile + lo_off + cm_offset(r, c0, C)) = *reinterpret_cast<uint4*>(l);
}

// D (+)= A*B^T with split operands: hi*hi, then the two cross terms when `split`.
__device__ __forceinline__ void mma_split(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate, bool split, uint32_t a_lo, uint32_t b_lo) {
  mma_bf16(tmem_d, a, b, idesc, accumulate);
  if (split) {
    mma_bf16(tmem_d, a, desc_add(b, b_lo), idesc, 1u);
    mma_bf16(tmem_d, desc_add(a, a_lo), b, idesc, 1u);
  }
}

// mma_split with each cross term switchable (numerics experiments)
__device__ __forceinline__ void mma_split_terms(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                                uint32_t accumulate, bool a_hi_b_lo, bool a_lo_b_hi, uint32_t a_lo,
                                                uint32_t b_lo) {
  mma_bf16(tmem_d, a, b, idesc, accumulate);
  if (a_hi_b_lo) mma_bf16(tmem_d, a, desc_add(b, b_lo), idesc, 1u);
  if (a_lo_b_hi) mma_bf16(tmem_d, desc_add(a, a_lo), b, idesc, 1u);
}

// mma_split with the A operand in tensor memory: hi at tmem_a, lo at tmem_a + a_lo_cols.
__device__ __forceinline__ void mma_split_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                             uint32_t accumulate, bool split, uint32_t a_lo_cols, uint32_t b_lo) {
  mma_bf16_ts(tmem_d, tmem_a, b, idesc, accumulate);
  if (split) {
    mma_bf16_ts(tmem_d, tmem_a, desc_add(b, b_lo), idesc, 1u);
    mma_bf16_ts(tmem_d, tmem_a + a_lo_cols, b, idesc, 1u);
  }
}

}  // namespace umma
}  // namespace prenom
