/*
 * scg_rng.h -- the normative seeded random stream (INPUT GENERATOR ONLY).
 *
 * This header is the one piece of code shared by the CPU oracle (oracle/) and
 * the CUDA product path (paper_1912_02949_b200/csrc/).  It holds none of the
 * method's arithmetic: it only defines the random numbers the method draws,
 *   - the Gaussian test matrix Omega of the Nystrom sketch
 *     (PAPER.md:1151-1155 footnote "independent Gaussian random variable with
 *      mean zero and variance one"; Alg. 3 line "Omega <- randn(n, R)",
 *      PAPER.md:1228), and
 *   - the Gaussian start vector of every randomized Lanczos call
 *     (Alg. 2 line "v_1 <- randn(n, 1)"),
 * plus uniforms for the synthetic graph generators.  Because both sides draw
 * the same counter-based stream, a rank of a row-sharded run can generate
 * exactly its own rows.
 *
 * Definition:
 *   words   = Philox4x32-10(key = (seed_lo, seed_hi),
 *                           counter = (index_lo, index_hi, sub, stream))
 *   a       = ((w0 << 32) | w1) >> 11          (53-bit integer)
 *   b       = ((w2 << 32) | w3) >> 11
 *   u1      = (a + 1) * 2^-53   in (0, 1]
 *   u2      = b * 2^-53         in [0, 1)
 *   normal  = sqrt(-2 ln u1) * cos(2 pi u2)    (Box-Muller, cosine branch)
 * ln and cos are evaluated with the fixed IEEE-only routines below (explicit
 * fma, correctly rounded +,-,*,/,sqrt; no libm), so a host compiler with
 * -ffp-contract=off and nvcc with --fmad=false produce identical bits.
 *
 * Streams: 0 = Omega (sub = column k, index = row i), 1 = Lanczos start vector
 * (sub = iteration t, index = row), 2.. = graph generators.
 */
#ifndef SCG_RNG_H
#define SCG_RNG_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SCG_RNG_FN __host__ __device__ __forceinline__
#define SCG_FMA(a, b, c) fma((a), (b), (c))
#define SCG_SQRT(x) sqrt(x)
#include <math.h>
#else
#include <math.h>
#define SCG_RNG_FN static inline
#define SCG_FMA(a, b, c) fma((a), (b), (c))
#define SCG_SQRT(x) sqrt(x)
#endif

#define SCG_STREAM_OMEGA 0u
#define SCG_STREAM_LANCZOS 1u
#define SCG_STREAM_GRAPH 2u
#define SCG_STREAM_PHASE 3u /* phase retrieval instance: sub 0 unit phase, 1 magnitude, 2 signal */

typedef struct {
  uint32_t w[4];
} scg_philox_out;

SCG_RNG_FN void scg_mulhilo32(uint32_t a, uint32_t b, uint32_t *hi, uint32_t *lo) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  *lo = (uint32_t)p;
}

/* Philox4x32 with 10 rounds (Salmon et al., SC'11), counter c0..c3, key k0,k1. */
SCG_RNG_FN scg_philox_out scg_philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                            uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    scg_mulhilo32(M0, c0, &hi0, &lo0);
    scg_mulhilo32(M1, c2, &hi1, &lo1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0; k1 += W1;
  }
  scg_philox_out o;
  o.w[0] = c0; o.w[1] = c1; o.w[2] = c2; o.w[3] = c3;
  return o;
}

SCG_RNG_FN scg_philox_out scg_draw(uint64_t seed, uint32_t stream, uint32_t sub, uint64_t index) {
  return scg_philox4x32_10((uint32_t)index, (uint32_t)(index >> 32), sub, stream,
                           (uint32_t)seed, (uint32_t)(seed >> 32));
}

/* Uniform in [0, 1) with 53 random bits (first two words). */
SCG_RNG_FN double scg_uniform(uint64_t seed, uint32_t stream, uint32_t sub, uint64_t index) {
  scg_philox_out o = scg_draw(seed, stream, sub, index);
  uint64_t a = (((uint64_t)o.w[0] << 32) | (uint64_t)o.w[1]) >> 11;
  return (double)a * 0x1.0p-53;
}

/* ln(x) for x in (0, 1]; x = m 2^e with m in [sqrt(1/2), sqrt(2)),
 * ln m = 2 atanh(s), s = (m-1)/(m+1), atanh by its Taylor series to s^27. */
SCG_RNG_FN double scg_ln_unit(double x) {
  union { double d; uint64_t u; } v;
  v.d = x;
  int e = (int)((v.u >> 52) & 0x7ff) - 1023; /* x >= 2^-53: always normal */
  v.u = (v.u & 0x000fffffffffffffull) | 0x3ff0000000000000ull; /* m in [1,2) */
  double m = v.d;
  if (m > 0x1.6a09e667f3bcdp+0) { /* m > sqrt(2): halve (exact) */
    m = m * 0.5;
    e += 1;
  }
  double s = (m - 1.0) / (m + 1.0);
  double s2 = s * s;
  double p = 0x1.2f684bda12f68p-5;           /* 1/27 */
  p = SCG_FMA(p, s2, 0x1.47ae147ae147bp-5);  /* 1/25 */
  p = SCG_FMA(p, s2, 0x1.642c8590b2164p-5);  /* 1/23 */
  p = SCG_FMA(p, s2, 0x1.8618618618618p-5);  /* 1/21 */
  p = SCG_FMA(p, s2, 0x1.af286bca1af28p-5);  /* 1/19 */
  p = SCG_FMA(p, s2, 0x1.e1e1e1e1e1e1ep-5);  /* 1/17 */
  p = SCG_FMA(p, s2, 0x1.1111111111111p-4);  /* 1/15 */
  p = SCG_FMA(p, s2, 0x1.3b13b13b13b14p-4);  /* 1/13 */
  p = SCG_FMA(p, s2, 0x1.745d1745d1746p-4);  /* 1/11 */
  p = SCG_FMA(p, s2, 0x1.c71c71c71c71cp-4);  /* 1/9 */
  p = SCG_FMA(p, s2, 0x1.2492492492492p-3);  /* 1/7 */
  p = SCG_FMA(p, s2, 0x1.999999999999ap-3);  /* 1/5 */
  p = SCG_FMA(p, s2, 0x1.5555555555555p-2);  /* 1/3 */
  /* ln m = 2 s + 2 s^3 p(s^2) */
  double two_s = s + s;
  double lnm = SCG_FMA(two_s * s2, p, two_s);
  double de = (double)e;
  /* e ln2 split hi/lo */
  return SCG_FMA(de, 0x1.62e42fefa39efp-1, SCG_FMA(de, 0x1.abc9e3b39803fp-56, lnm));
}

/* cos and sin of th in [0, pi/4] by Taylor polynomials in th^2. */
SCG_RNG_FN double scg_cos_small(double th) {
  double t2 = th * th;
  double p = 0x1.e542ba4020225p-62;
  p = SCG_FMA(p, t2, -0x1.6827863b97d97p-53);
  p = SCG_FMA(p, t2, 0x1.ae7f3e733b81fp-45);
  p = SCG_FMA(p, t2, -0x1.93974a8c07c9dp-37);
  p = SCG_FMA(p, t2, 0x1.1eed8eff8d898p-29);
  p = SCG_FMA(p, t2, -0x1.27e4fb7789f5cp-22);
  p = SCG_FMA(p, t2, 0x1.a01a01a01a01ap-16);
  p = SCG_FMA(p, t2, -0x1.6c16c16c16c17p-10);
  p = SCG_FMA(p, t2, 0x1.5555555555555p-5);
  p = SCG_FMA(p, t2, -0x1.0000000000000p-1);
  return SCG_FMA(p, t2, 1.0);
}

SCG_RNG_FN double scg_sin_small(double th) {
  double t2 = th * th;
  double p = 0x1.71b8ef6dcf572p-66;
  p = SCG_FMA(p, t2, -0x1.2f49b46814157p-57);
  p = SCG_FMA(p, t2, 0x1.952c77030ad4ap-49);
  p = SCG_FMA(p, t2, -0x1.ae7f3e733b81fp-41);
  p = SCG_FMA(p, t2, 0x1.6124613a86d09p-33);
  p = SCG_FMA(p, t2, -0x1.ae64567f544e4p-26);
  p = SCG_FMA(p, t2, 0x1.71de3a556c734p-19);
  p = SCG_FMA(p, t2, -0x1.a01a01a01a01ap-13);
  p = SCG_FMA(p, t2, 0x1.1111111111111p-7);
  p = SCG_FMA(p, t2, -0x1.5555555555555p-3);
  return SCG_FMA(p * t2, th, th);
}

/* cos(2 pi u) for u in [0, 1): quadrant reduction is exact (4u exact).  With f the
 * fraction within the quadrant and th = (pi/2) f (f <= 1/2) or (pi/2)(1 - f) (f > 1/2), the
 * value is +-cos_small(th) or +-sin_small(th); only that one polynomial is evaluated, with its
 * coefficients selected per call (so a GPU warp runs one polynomial whatever its lanes need).
 * The sine's leading step fma(0, t2, s0) = s0 is exact, so both are the operations of
 * scg_cos_small / scg_sin_small above, bit for bit. */
SCG_RNG_FN double scg_cos_2pi(double u) {
  double x = 4.0 * u;
  int q = (int)x;           /* 0..3 */
  double f = x - (double)q; /* exact, in [0,1) */
  const int hi = f > 0.5;
  const double th = 0x1.921fb54442d18p+0 * (hi ? (1.0 - f) : f);
  /* q even needs cos(pi/2 f), q odd sin(pi/2 f); above 1/2 the two swap */
  const int use_cos = ((q & 1) == 0) != hi;
  const double t2 = th * th;
  double p = use_cos ? 0x1.e542ba4020225p-62 : 0.0;
  p = SCG_FMA(p, t2, use_cos ? -0x1.6827863b97d97p-53 : 0x1.71b8ef6dcf572p-66);
  p = SCG_FMA(p, t2, use_cos ? 0x1.ae7f3e733b81fp-45 : -0x1.2f49b46814157p-57);
  p = SCG_FMA(p, t2, use_cos ? -0x1.93974a8c07c9dp-37 : 0x1.952c77030ad4ap-49);
  p = SCG_FMA(p, t2, use_cos ? 0x1.1eed8eff8d898p-29 : -0x1.ae7f3e733b81fp-41);
  p = SCG_FMA(p, t2, use_cos ? -0x1.27e4fb7789f5cp-22 : 0x1.6124613a86d09p-33);
  p = SCG_FMA(p, t2, use_cos ? 0x1.a01a01a01a01ap-16 : -0x1.ae64567f544e4p-26);
  p = SCG_FMA(p, t2, use_cos ? -0x1.6c16c16c16c17p-10 : 0x1.71de3a556c734p-19);
  p = SCG_FMA(p, t2, use_cos ? 0x1.5555555555555p-5 : -0x1.a01a01a01a01ap-13);
  p = SCG_FMA(p, t2, use_cos ? -0x1.0000000000000p-1 : 0x1.1111111111111p-7);
  /* the sine has one coefficient less: its last step here is its -1/6 */
  const double v = use_cos ? SCG_FMA(p, t2, 1.0)
                           : SCG_FMA(SCG_FMA(p, t2, -0x1.5555555555555p-3) * t2, th, th);
  return (q == 1 || q == 2) ? -v : v;
}

/* One standard normal per counter (Box-Muller, cosine branch). */
SCG_RNG_FN double scg_normal(uint64_t seed, uint32_t stream, uint32_t sub, uint64_t index) {
  scg_philox_out o = scg_draw(seed, stream, sub, index);
  uint64_t a = (((uint64_t)o.w[0] << 32) | (uint64_t)o.w[1]) >> 11;
  uint64_t b = (((uint64_t)o.w[2] << 32) | (uint64_t)o.w[3]) >> 11;
  double u1 = (double)(a + 1) * 0x1.0p-53;
  double u2 = (double)b * 0x1.0p-53;
  double r = SCG_SQRT(-2.0 * scg_ln_unit(u1));
  return r * scg_cos_2pi(u2);
}

/* Omega[i, k] (column k, row i) -- PAPER.md:1228. */
SCG_RNG_FN double scg_omega(uint64_t seed, int64_t i, int32_t k) {
  return scg_normal(seed, SCG_STREAM_OMEGA, (uint32_t)k, (uint64_t)i);
}

/* Lanczos start vector of iteration t, entry i -- PAPER.md:1082. */
SCG_RNG_FN double scg_lanczos_start(uint64_t seed, int64_t t, int64_t i) {
  return scg_normal(seed, SCG_STREAM_LANCZOS, (uint32_t)t, (uint64_t)i);
}

#endif /* SCG_RNG_H */
