/* gen/philox_normal.h — the seeded synthetic-input generator (shared test infrastructure).
 *
 * This header holds NONE of the method's arithmetic (no factorisation, solve, Schur complement or assembly).
 * It is the counter-based generator of SURVEY.md Appendix A ("Philox"), implemented once as plain
 * +,-,*,/,sqrt code so that the host build (gcc -ffp-contract=off) and the device build (nvcc --fmad=false)
 * produce bit-identical doubles: every input the oracle and the CUDA path see is the same byte string.
 *
 *   Philox4x32-10 (Salmon et al., SC'11): key = (seed mod 2^32, seed div 2^32),
 *   counter = (g, id, tag, 0); one call yields 4 words -> two uniforms
 *   u = ((w_hi << 32 | w_lo) >> 11) * 2^-53 from words (0,1) and (2,3);
 *   Box-Muller: z0 = sqrt(-2 ln(1-u0)) cos(2 pi u1), z1 = sqrt(-2 ln(1-u0)) sin(2 pi u1).
 *
 * ln, cos and sin are evaluated by fixed polynomial/series code below (not libm), because libm and the
 * CUDA math library may round differently in the last bit. Accuracy is ~1e-16 relative; exactness against
 * libm is not required, only host/device determinism.
 */
#ifndef HDG_GEN_PHILOX_NORMAL_H
#define HDG_GEN_PHILOX_NORMAL_H

#include <stdint.h>

#if defined(__CUDACC__)
#define GEN_QUAL static __host__ __device__ __forceinline__
#else
#define GEN_QUAL static inline
#endif

/* tags */
enum { GEN_TAG_ADIAG = 0, GEN_TAG_A = 1, GEN_TAG_B = 2, GEN_TAG_C = 3, GEN_TAG_D = 4,
       GEN_TAG_RE = 5, GEN_TAG_RF = 6, GEN_TAG_P = 7, GEN_TAG_LAMBDA = 8 };

typedef struct { uint32_t x[4]; } gen_u32x4;

GEN_QUAL uint32_t gen_mulhilo(uint32_t a, uint32_t b, uint32_t* hi) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  return (uint32_t)p;
}

GEN_QUAL gen_u32x4 gen_philox4x32_10(gen_u32x4 c, uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, hi1;
    uint32_t lo0 = gen_mulhilo(0xD2511F53u, c.x[0], &hi0);
    uint32_t lo1 = gen_mulhilo(0xCD9E8D57u, c.x[2], &hi1);
    gen_u32x4 n;
    n.x[0] = hi1 ^ c.x[1] ^ k0;
    n.x[1] = lo1;
    n.x[2] = hi0 ^ c.x[3] ^ k1;
    n.x[3] = lo0;
    c = n;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

GEN_QUAL double gen_u01(uint32_t lo, uint32_t hi) {
  uint64_t w = ((uint64_t)hi << 32) | (uint64_t)lo;
  return (double)(w >> 11) * (1.0 / 9007199254740992.0); /* 2^-53, exact */
}

/* ln(x) for x in [2^-60, 1]: x = m 2^e with m in [sqrt(1/2), sqrt(2)); ln m = 2 atanh(t), t=(m-1)/(m+1). */
GEN_QUAL double gen_ln(double x) {
  int e = 0;
  while (x < 0.70710678118654752) { x = x * 2.0; e -= 1; }   /* exact scalings by 2 */
  const double t = (x - 1.0) / (x + 1.0);
  const double t2 = t * t;
  /* 2 * sum_{k=0}^{13} t^(2k+1)/(2k+1), Horner from the top; |t| <= 0.1716 -> truncation < 1e-19 */
  double s = 1.0 / 27.0;
  s = s * t2 + 1.0 / 25.0;
  s = s * t2 + 1.0 / 23.0;
  s = s * t2 + 1.0 / 21.0;
  s = s * t2 + 1.0 / 19.0;
  s = s * t2 + 1.0 / 17.0;
  s = s * t2 + 1.0 / 15.0;
  s = s * t2 + 1.0 / 13.0;
  s = s * t2 + 1.0 / 11.0;
  s = s * t2 + 1.0 / 9.0;
  s = s * t2 + 1.0 / 7.0;
  s = s * t2 + 1.0 / 5.0;
  s = s * t2 + 1.0 / 3.0;
  s = s * t2 + 1.0;
  const double lnm = 2.0 * t * s;
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  return ((double)e * ln2_hi + lnm) + (double)e * ln2_lo;
}

/* sin and cos of y in [0, pi/4] by Taylor series to degree 21/20 (truncation < 1e-19). */
GEN_QUAL void gen_sincos_small(double y, double* s, double* c) {
  const double y2 = y * y;
  double ps = 1.0 / 51090942171709440000.0;        /* 1/21! */
  ps = ps * (-y2) + 1.0 / 121645100408832000.0;     /* 1/19! */
  ps = ps * (-y2) + 1.0 / 355687428096000.0;        /* 1/17! */
  ps = ps * (-y2) + 1.0 / 1307674368000.0;          /* 1/15! */
  ps = ps * (-y2) + 1.0 / 6227020800.0;             /* 1/13! */
  ps = ps * (-y2) + 1.0 / 39916800.0;               /* 1/11! */
  ps = ps * (-y2) + 1.0 / 362880.0;                 /* 1/9!  */
  ps = ps * (-y2) + 1.0 / 5040.0;                   /* 1/7!  */
  ps = ps * (-y2) + 1.0 / 120.0;                    /* 1/5!  */
  ps = ps * (-y2) + 1.0 / 6.0;                      /* 1/3!  */
  ps = ps * (-y2) + 1.0;
  *s = y * ps;
  double pc = 1.0 / 2432902008176640000.0;          /* 1/20! */
  pc = pc * (-y2) + 1.0 / 6402373705728000.0;       /* 1/18! */
  pc = pc * (-y2) + 1.0 / 20922789888000.0;         /* 1/16! */
  pc = pc * (-y2) + 1.0 / 87178291200.0;            /* 1/14! */
  pc = pc * (-y2) + 1.0 / 479001600.0;              /* 1/12! */
  pc = pc * (-y2) + 1.0 / 3628800.0;                /* 1/10! */
  pc = pc * (-y2) + 1.0 / 40320.0;                  /* 1/8!  */
  pc = pc * (-y2) + 1.0 / 720.0;                    /* 1/6!  */
  pc = pc * (-y2) + 1.0 / 24.0;                     /* 1/4!  */
  pc = pc * (-y2) + 1.0 / 2.0;                      /* 1/2!  */
  pc = pc * (-y2) + 1.0;
  *c = pc;
}

/* (sin, cos) of 2 pi u, u in [0,1): quadrant split on 4u (exact), then fold to [0, pi/4]. */
GEN_QUAL void gen_sincos_2pi(double u, double* s, double* c) {
  const double v = 4.0 * u;
  const int q = (int)v;              /* 0..3 */
  double f = v - (double)q;          /* exact, in [0,1) */
  const double half_pi = 1.57079632679489661923;
  double sa, ca;
  if (f <= 0.5) {
    gen_sincos_small(f * half_pi, &sa, &ca);
  } else {
    double cb, sb;
    gen_sincos_small((1.0 - f) * half_pi, &cb, &sb); /* sin(pi/2 - y) = cos y */
    sa = sb; ca = cb;
    /* here sa = cos((1-f) pi/2) = sin(f pi/2), ca = sin((1-f) pi/2) = cos(f pi/2) */
  }
  switch (q) {
    case 0: *s = sa;  *c = ca;  break;
    case 1: *s = ca;  *c = -sa; break;
    case 2: *s = -sa; *c = -ca; break;
    default: *s = -ca; *c = sa; break;
  }
}

/* Normal draw number t (0-based, row-major within a block) of stream (seed, id, tag). */
GEN_QUAL double gen_normal(uint64_t seed, uint32_t id, uint32_t tag, uint64_t t) {
  gen_u32x4 ctr;
  ctr.x[0] = (uint32_t)(t >> 1);
  ctr.x[1] = id;
  ctr.x[2] = tag;
  ctr.x[3] = 0u;
  gen_u32x4 w = gen_philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double u0 = gen_u01(w.x[0], w.x[1]);
  const double u1 = gen_u01(w.x[2], w.x[3]);
  const double rad = sqrt(-2.0 * gen_ln(1.0 - u0));
  double sn, cs;
  gen_sincos_2pi(u1, &sn, &cs);
  return (t & 1) ? rad * sn : rad * cs;
}

/* Uniform draw number t of stream (seed, id, tag) (word pair (0,1)); used for the hp degree draw. */
GEN_QUAL double gen_uniform(uint64_t seed, uint32_t id, uint32_t tag, uint64_t t) {
  gen_u32x4 ctr;
  ctr.x[0] = (uint32_t)t;
  ctr.x[1] = id;
  ctr.x[2] = tag;
  ctr.x[3] = 0u;
  gen_u32x4 w = gen_philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
  return gen_u01(w.x[0], w.x[1]);
}

/* Value (i,j) of a generated block of element `id` (BASELINE.json configs):
 *   kind A: A_ij = s G_ij (i != j), A_ii = (2 + |z_i|) + s G_ii, s = 0.5/sqrt(n_e)   (G: tag 1, z: tag 0)
 *   kind B/C: G_ij * (1/sqrt(n_e))                                               (tags 2, 3)
 *   kind D: (0.5/sqrt(n_f)) H_ij + 2 delta_ij                                      (tag 4)
 *   kind RE/RF: N(0,1)                                                             (tags 5, 6)
 */
enum { GEN_KIND_A = 0, GEN_KIND_B = 1, GEN_KIND_C = 2, GEN_KIND_D = 3, GEN_KIND_RE = 4, GEN_KIND_RF = 5 };

GEN_QUAL double gen_block_value(uint64_t seed, uint32_t id, int kind, int ne, int nf, int cols, int i, int j) {
  const uint64_t t = (uint64_t)i * (uint64_t)cols + (uint64_t)j;
  switch (kind) {
    case GEN_KIND_A: {
      const double s = 0.5 / sqrt((double)ne);
      const double g = gen_normal(seed, id, GEN_TAG_A, t);
      if (i != j) return s * g;
      double z = gen_normal(seed, id, GEN_TAG_ADIAG, (uint64_t)i);
      if (z < 0.0) z = -z;
      return (2.0 + z) + s * g;
    }
    case GEN_KIND_B: return gen_normal(seed, id, GEN_TAG_B, t) * (1.0 / sqrt((double)ne));
    case GEN_KIND_C: return gen_normal(seed, id, GEN_TAG_C, t) * (1.0 / sqrt((double)ne));
    case GEN_KIND_D: {
      const double v = (0.5 / sqrt((double)nf)) * gen_normal(seed, id, GEN_TAG_D, t);
      return (i == j) ? v + 2.0 : v;
    }
    case GEN_KIND_RE: return gen_normal(seed, id, GEN_TAG_RE, t);
    default: return gen_normal(seed, id, GEN_TAG_RF, t);
  }
}

#endif
