/*
 * hgen.h -- seeded, counter-based input generator shared by the oracle side
 * (host) and the GPU tests/bench (device).  TEST/BENCH INFRASTRUCTURE: it holds
 * none of the H-matvec arithmetic, only the synthetic-input recipe of
 * DESIGN.md §3.
 *
 * The paper fills its benchmark H-matrices "by random numbers" and uses random
 * input vectors (§5 "Numerical Results"); BASELINE.json
 * fixes the distributions: U,V entries iid N(0,1)/sqrt(block rows), dense leaf
 * blocks iid N(0,1)/8, x iid U[-1,1].
 *
 * Every value is a pure function of (seed, tag, level, vec, global element
 * index), so any row slice can be generated independently (one rank's slice =
 * the same rows of a full generation), and host and device produce the SAME
 * BITS: the recipe uses only integer ops and IEEE-754 correctly rounded
 * +,-,*,/,sqrt -- no libm, no fma.  Host code is compiled with
 * -ffp-contract=off and device code with -fmad=false so that no contraction
 * changes the rounding.
 *
 *   splitmix64(z)            the standard 64-bit finaliser
 *   stream(seed,tag,lvl,vec) = splitmix64(seed ^ splitmix64(tag<<56 | lvl<<48 | vec))
 *   h(stream, idx, k)        = splitmix64(stream ^ splitmix64(2*idx + k)),  k in {0,1}
 *   u(h)                     = ((h >> 11) + 0.5) * 2^-53          in (0,1)
 *   normal                   = sqrt(-2 log u0) * cos(2 pi u1)     (Box-Muller)
 *   uniform11                = 2 u0 - 1
 *
 * idx is the element's index in the CANONICAL global panel: row*W + col for
 * U_l / V_l (W = (2^d-1) r), row*b + col for D, col*N + row for x (column col
 * of an N x nrhs column-major block).
 */
#ifndef HGEN_H
#define HGEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define HGEN_FN static __host__ __device__ __forceinline__
#else
#define HGEN_FN static inline
#endif

enum { HGEN_TAG_U = 1, HGEN_TAG_V = 2, HGEN_TAG_D = 3, HGEN_TAG_X = 4 };

HGEN_FN uint64_t hgen_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

HGEN_FN uint64_t hgen_stream(uint64_t seed, uint64_t tag, uint64_t level, uint64_t vec) {
  return hgen_splitmix64(seed ^ hgen_splitmix64((tag << 56) | (level << 48) | vec));
}

HGEN_FN double hgen_u01(uint64_t stream, uint64_t idx, uint64_t k) {
  uint64_t h = hgen_splitmix64(stream ^ hgen_splitmix64(2ull * idx + k));
  return ((double)(h >> 11) + 0.5) * 1.1102230246251565404e-16; /* 2^-53 */
}

/* Natural log of u in (0,1]: u = 2^e f with f in [sqrt(1/2), sqrt(2)],
 * log f = 2 atanh(s), s = (f-1)/(f+1), |s| <= 0.1716, series to s^25. */
HGEN_FN double hgen_log(double u) {
  union { double d; uint64_t i; } v;
  v.d = u;
  int e = (int)((v.i >> 52) & 0x7ff) - 1023;
  v.i = (v.i & 0x000fffffffffffffull) | 0x3ff0000000000000ull; /* f in [1,2) */
  double f = v.d;
  if (f > 1.4142135623730951) { f = f * 0.5; e += 1; }
  double s = (f - 1.0) / (f + 1.0);
  double s2 = s * s;
  double p = 1.0 / 25.0;
  p = p * s2 + 1.0 / 23.0;
  p = p * s2 + 1.0 / 21.0;
  p = p * s2 + 1.0 / 19.0;
  p = p * s2 + 1.0 / 17.0;
  p = p * s2 + 1.0 / 15.0;
  p = p * s2 + 1.0 / 13.0;
  p = p * s2 + 1.0 / 11.0;
  p = p * s2 + 1.0 / 9.0;
  p = p * s2 + 1.0 / 7.0;
  p = p * s2 + 1.0 / 5.0;
  p = p * s2 + 1.0 / 3.0;
  double lf = 2.0 * s + 2.0 * s * (s2 * p);
  const double ln2_hi = 6.93147180369123816490e-01; /* ln 2 rounded to 32 bits */
  const double ln2_lo = 1.90821492927058770002e-10; /* ln 2 - ln2_hi */
  return ((double)e * ln2_hi + lf) + (double)e * ln2_lo;
}

/* cos(2 pi u) for u in [0,1]: fold to w in [0,1/4] with a sign, then the
 * Taylor series of cos(phi), phi = 2 pi w in [0, pi/2], through phi^26/26!. */
HGEN_FN double hgen_cos2pi(double u) {
  double w = (u <= 0.5) ? u : 1.0 - u;      /* cos(2 pi u) = cos(2 pi (1-u)) */
  double sign = 1.0;
  if (w > 0.25) { w = 0.5 - w; sign = -1.0; } /* cos(pi - a) = -cos(a) */
  double phi = 6.283185307179586477 * w;
  double q = phi * phi;
  /* a_k = (-1)^k / (2k)!,  k = 0..13 */
  const double a[14] = {
      1.0,
      -1.0 / 2.0,
      1.0 / 24.0,
      -1.0 / 720.0,
      1.0 / 40320.0,
      -1.0 / 3628800.0,
      1.0 / 479001600.0,
      -1.0 / 87178291200.0,
      1.0 / 20922789888000.0,
      -1.0 / 6402373705728000.0,
      1.0 / 2432902008176640000.0,
      -1.0 / 1.1240007277776077e+21,
      1.0 / 6.2044840173323941e+23,
      -1.0 / 4.0329146112660565e+26,
  };
  double c = a[13];
  for (int k = 12; k >= 0; --k) c = a[k] + q * c;
  return sign * c;
}

/* N(0,1) sample number idx of a stream (Box-Muller on two independent draws). */
HGEN_FN double hgen_normal(uint64_t stream, uint64_t idx) {
  double u0 = hgen_u01(stream, idx, 0);
  double u1 = hgen_u01(stream, idx, 1);
  double rad = -2.0 * hgen_log(u0);
  if (rad < 0.0) rad = 0.0;
  return sqrt(rad) * hgen_cos2pi(u1);
}

/* U(-1,1) sample number idx of a stream. */
HGEN_FN double hgen_uniform11(uint64_t stream, uint64_t idx) {
  return 2.0 * hgen_u01(stream, idx, 0) - 1.0;
}

#endif
