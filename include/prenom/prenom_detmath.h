/* prenom_detmath.h -- deterministic arithmetic shared by the sm_100a kernels
 * and the CPU oracle, for the results the north star requires BIT-EXACT
 * (sample depths/positions, bin indices, table rows).
 *
 * Why: nvcc contracts a*b+c into FMA by default and CUDA's exp() is not
 * glibc's exp(). The reference's arithmetic (compiled for x86-64 without FMA)
 * is a plain sequence of IEEE-754 round-to-nearest operations, so the kernels
 * spell those operations with the *_rn intrinsics, which the compiler never
 * contracts, and use det_exp() below instead of exp(). On the host the same
 * code is plain C compiled with -ffp-contract=off.
 *
 * det_exp is NOT glibc's exp: it is a Cody-Waite reduction + degree-13
 * Taylor/Horner polynomial built only from +,-,*,floor, so it rounds
 * identically everywhere. It is within 2 ulp of glibc exp on the sampler's
 * domain (tests/test_detmath.py), which is how the reference's
 * build_ray_cdf (density_grid.cpp:43-70, std::exp in double) is pinned at
 * tolerance while kernel and oracle agree to the bit.
 */
#ifndef PRENOM_DETMATH_H
#define PRENOM_DETMATH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define PDM_FN __host__ __device__ __forceinline__
#else
#define PDM_FN static inline
#endif

#if defined(__CUDA_ARCH__)
#define PDM_FMUL(a, b) __fmul_rn((a), (b))
#define PDM_FADD(a, b) __fadd_rn((a), (b))
#define PDM_FSUB(a, b) __fsub_rn((a), (b))
#define PDM_FDIV(a, b) __fdiv_rn((a), (b))
#define PDM_FSQRT(a) __fsqrt_rn((a))
#define PDM_DMUL(a, b) __dmul_rn((a), (b))
#define PDM_DADD(a, b) __dadd_rn((a), (b))
#define PDM_DSUB(a, b) __dsub_rn((a), (b))
#define PDM_DDIV(a, b) __ddiv_rn((a), (b))
#else
#define PDM_FMUL(a, b) ((float)(a) * (float)(b))
#define PDM_FADD(a, b) ((float)(a) + (float)(b))
#define PDM_FSUB(a, b) ((float)(a) - (float)(b))
#define PDM_FDIV(a, b) ((float)(a) / (float)(b))
#define PDM_FSQRT(a) sqrtf((a))
#define PDM_DMUL(a, b) ((double)(a) * (double)(b))
#define PDM_DADD(a, b) ((double)(a) + (double)(b))
#define PDM_DSUB(a, b) ((double)(a) - (double)(b))
#define PDM_DDIV(a, b) ((double)(a) / (double)(b))
#endif

#if !defined(__CUDA_ARCH__)
#include <math.h>
#include <string.h>
#endif

PDM_FN double pdm_bits_to_double(uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)b);
#else
  double d;
  memcpy(&d, &b, sizeof d);
  return d;
#endif
}

/* exp(x) in double, bit-identical on host and device. */
PDM_FN double pdm_det_exp(double x) {
  if (x != x) return x;
  if (x > 709.782712893383973096) return pdm_bits_to_double(0x7ff0000000000000ull);
  if (x < -745.13321910194110842) return 0.0;
  const double inv_ln2 = 1.44269504088896338700e+00;
  /* ln2 split so that k * LN2_HI is exact for |k| < 2^21 (fdlibm constants). */
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double kd = floor(PDM_DADD(PDM_DMUL(x, inv_ln2), 0.5));
  const double hi = PDM_DSUB(x, PDM_DMUL(kd, ln2_hi));
  const double r = PDM_DSUB(hi, PDM_DMUL(kd, ln2_lo));
  /* exp(r), |r| <= 0.3466: Taylor to r^13 (truncation < 2^-60 relative). */
  double p = 1.6059043836821614599e-10; /* 1/13! */
  p = PDM_DADD(PDM_DMUL(p, r), 2.0876756987868098979e-09); /* 1/12! */
  p = PDM_DADD(PDM_DMUL(p, r), 2.5052108385441718775e-08); /* 1/11! */
  p = PDM_DADD(PDM_DMUL(p, r), 2.7557319223985890653e-07); /* 1/10! */
  p = PDM_DADD(PDM_DMUL(p, r), 2.7557319223985892510e-06); /* 1/9!  */
  p = PDM_DADD(PDM_DMUL(p, r), 2.4801587301587301566e-05); /* 1/8!  */
  p = PDM_DADD(PDM_DMUL(p, r), 1.9841269841269841253e-04); /* 1/7!  */
  p = PDM_DADD(PDM_DMUL(p, r), 1.3888888888888889419e-03); /* 1/6!  */
  p = PDM_DADD(PDM_DMUL(p, r), 8.3333333333333332177e-03); /* 1/5!  */
  p = PDM_DADD(PDM_DMUL(p, r), 4.1666666666666664354e-02); /* 1/4!  */
  p = PDM_DADD(PDM_DMUL(p, r), 1.6666666666666665741e-01); /* 1/3!  */
  p = PDM_DADD(PDM_DMUL(p, r), 0.5);
  p = PDM_DADD(PDM_DMUL(p, r), 1.0);
  p = PDM_DADD(PDM_DMUL(p, r), 1.0);
  const int k = (int)kd;
  if (k >= -1022) {
    if (k > 1023) return PDM_DMUL(PDM_DMUL(p, pdm_bits_to_double((uint64_t)(1023 + 1023) << 52)),
                                  pdm_bits_to_double((uint64_t)(k - 1023 + 1023) << 52));
    return PDM_DMUL(p, pdm_bits_to_double((uint64_t)(k + 1023) << 52));
  }
  /* subnormal result: one exact scaling, then a single rounding. */
  return PDM_DMUL(PDM_DMUL(p, pdm_bits_to_double((uint64_t)(k + 54 + 1023) << 52)),
                  pdm_bits_to_double((uint64_t)(-54 + 1023) << 52));
}

/* ---- Philox4x32-10 (Salmon et al., SC'11; Random123 constants) ---------- */
#define PDM_PHILOX_M0 0xD2511F53u
#define PDM_PHILOX_M1 0xCD9E8D57u
#define PDM_PHILOX_W0 0x9E3779B9u
#define PDM_PHILOX_W1 0xBB67AE85u

PDM_FN void pdm_philox4x32_10(const uint32_t ctr_in[4], uint32_t k0, uint32_t k1,
                              uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
#if defined(__CUDA_ARCH__)
    const uint32_t hi0 = __umulhi(PDM_PHILOX_M0, c0), lo0 = PDM_PHILOX_M0 * c0;
    const uint32_t hi1 = __umulhi(PDM_PHILOX_M1, c2), lo1 = PDM_PHILOX_M1 * c2;
#else
    const uint64_t p0 = (uint64_t)PDM_PHILOX_M0 * c0, p1 = (uint64_t)PDM_PHILOX_M1 * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += PDM_PHILOX_W0;
    k1 += PDM_PHILOX_W1;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

PDM_FN float pdm_u01(uint32_t x) { return (float)(x >> 8) * 5.9604644775390625e-08f; }
PDM_FN uint32_t pdm_pick(uint32_t x, uint32_t n) {
  return (uint32_t)(((uint64_t)x * (uint64_t)n) >> 32);
}

#endif /* PRENOM_DETMATH_H */
