/* gen_core.h -- seeded, counter-based synthetic-input generators.
 *
 * This header belongs to the `datagen` module, the ONLY code shared by the
 * CPU oracle side (tests) and the CUDA product side (bench / GPU tests).
 * It contains no arithmetic of the searched method (no search, no binning,
 * no interpolation): only random numbers and the value recipes of the
 * synthetic workloads.
 *
 * The same source is compiled by gcc (datagen/gen_host.c) and by nvcc
 * (datagen/gen_device.cu).  Every floating-point step is a single IEEE-754
 * correctly-rounded operation written out explicitly (GEN_MUL/GEN_ADD/
 * GEN_FMA/GEN_DIV, floor, exact power-of-two scaling), so host and device
 * produce bit-identical doubles; gcc must compile with -ffp-contract=off.
 */
#ifndef EOS_DATAGEN_GEN_CORE_H
#define EOS_DATAGEN_GEN_CORE_H

#include <stdint.h>

#ifdef __CUDACC__
#define GEN_FN __host__ __device__ __forceinline__
#else
#include <math.h>
#include <string.h>
#define GEN_FN static inline
#endif

#if defined(__CUDA_ARCH__)
#define GEN_MUL(a, b) __dmul_rn((a), (b))
#define GEN_ADD(a, b) __dadd_rn((a), (b))
#define GEN_SUB(a, b) __dsub_rn((a), (b))
#define GEN_DIV(a, b) __ddiv_rn((a), (b))
#define GEN_FMA(a, b, c) __fma_rn((a), (b), (c))
#define GEN_FLOOR(a) floor(a)
#define GEN_I2D(a) __ll2double_rn(a)
#else
#define GEN_MUL(a, b) ((a) * (b))
#define GEN_ADD(a, b) ((a) + (b))
#define GEN_SUB(a, b) ((a) - (b))
#define GEN_DIV(a, b) ((a) / (b))
#define GEN_FMA(a, b, c) fma((a), (b), (c))
#define GEN_FLOOR(a) floor(a)
#define GEN_I2D(a) ((double)(a))
#endif

/* splitmix64 finalizer (a bijection on 64-bit words). */
GEN_FN uint64_t gen_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* Key of one independent stream of a seeded config. */
GEN_FN uint64_t gen_key(uint64_t seed, uint64_t stream) {
  return gen_mix64(gen_mix64(seed + 0x632BE59BD9B4E019ULL) ^ (stream * 0xD1B54A32D192ED03ULL));
}

/* The i-th 64-bit random word of a stream: counter based, so any element of
 * the stream is addressable on its own (rank-invariant sharding). */
GEN_FN uint64_t gen_u64(uint64_t key, uint64_t i) {
  return gen_mix64(key ^ gen_mix64(i * 0x9E3779B97F4A7C15ULL + 0x2545F4914F6CDD1DULL));
}

/* Uniform double in [0, 1) with 53 random bits (exact conversion). */
GEN_FN double gen_unit(uint64_t r) {
  return GEN_MUL(GEN_I2D((int64_t)(r >> 11)), 1.1102230246251565404e-16 /* 2^-53 */);
}

GEN_FN double gen_bits2d(uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)b);
#else
  double d; memcpy(&d, &b, 8); return d;
#endif
}

/* 10^t for |t| <= ~300, built only from correctly rounded operations:
 *   z = t*log2(10), e = floor(z), f = z - e (exact), 2^f = exp(f ln2) by a
 *   degree-16 Taylor polynomial in Horner/FMA form, then exact scaling by 2^e.
 * Relative error vs the true 10^t is ~1e-15 -- irrelevant for a generator;
 * what matters is that host and device agree bit for bit. */
GEN_FN double gen_exp10(double t) {
  const double LOG2_10 = 3.321928094887362348;
  const double LN2 = 0.6931471805599453094;
  double z = GEN_MUL(t, LOG2_10);
  double e = GEN_FLOOR(z);
  double f = GEN_SUB(z, e);
  double g = GEN_MUL(f, LN2);
  /* 1/k! for k = 16..0 */
  const double c[17] = {
      4.779477332387385e-14, 7.647163731819816e-13, 1.1470745597729725e-11,
      1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,
      2.755731922398589e-07, 2.7557319223985893e-06, 2.48015873015873e-05,
      0.0001984126984126984, 0.001388888888888889, 0.008333333333333333,
      0.041666666666666664, 0.16666666666666666, 0.5, 1.0, 1.0};
  double p = c[0];
  for (int k = 1; k < 17; ++k) p = GEN_FMA(p, g, c[k]);
  int64_t ei = (int64_t)e;
  if (ei < -1022) ei = -1022;
  if (ei > 1023) ei = 1023;
  double scale = gen_bits2d((uint64_t)(ei + 1023) << 52);
  return GEN_MUL(p, scale);
}

/* ---- target recipes ---- */

/* log-uniform: log10(y) ~ U[a, a+w).  (cfg1, cfg2, cfg4, cfg5; P:224 read as
 * log-uniform.) */
GEN_FN double gen_loguniform(uint64_t key, uint64_t i, double a, double w) {
  double u = gen_unit(gen_u64(key, i));
  return gen_exp10(GEN_FMA(w, u, a));
}

/* cfg1: log-uniform, with ~1/copy_every of the positions replaced by an exact
 * copy of a table entry; position 0 -> X[0] and position 1 -> X[n-1]. */
GEN_FN double gen_with_copies(uint64_t key, uint64_t key2, uint64_t i, double a, double w,
                              const double* X, int64_t n, uint64_t copy_every) {
  if (i == 0) return X[0];
  if (i == 1) return X[n - 1];
  uint64_t r2 = gen_u64(key2, i);
  if (copy_every != 0 && (r2 % copy_every) == 0) return X[(r2 >> 32) % (uint64_t)n];
  return gen_loguniform(key, i, a, w);
}

/* cfg3 random walk: integer increments s_i = u0+u1+u2+u3 - 2^33 (Irwin-Hall(4)
 * of 32-bit uniforms, centred; approximately normal with sd 2^32/sqrt(3)).
 * The walk position is S_i = sum_{k<=i} s_k in wrapping 64-bit integers
 * (exact, so any summation order gives the same bits). */
GEN_FN int64_t gen_walk_step(uint64_t key, uint64_t i) {
  uint64_t r0 = gen_u64(key, 2 * i), r1 = gen_u64(key, 2 * i + 1);
  uint64_t s = (r0 & 0xFFFFFFFFULL) + (r0 >> 32) + (r1 & 0xFFFFFFFFULL) + (r1 >> 32);
  return (int64_t)(s - (1ULL << 33));
}

/* Map a walk position to a target: x = x0 + S*c (c = sigma*sqrt(3)/2^32 in
 * log10 units), reflected into [lo, hi] by folding with period 2(hi-lo),
 * then y = 10^x. */
GEN_FN double gen_walk_value(int64_t S, double x0, double c, double lo, double hi) {
  double x = GEN_FMA(GEN_I2D(S), c, x0);
  double P = GEN_MUL(2.0, GEN_SUB(hi, lo));
  double q = GEN_SUB(x, lo);
  double fl = GEN_FLOOR(GEN_DIV(q, P));
  double r = GEN_FMA(-fl, P, q);
  if (r < 0.0) r = 0.0;
  if (r >= P) r = 0.0;
  double span = GEN_SUB(hi, lo);
  if (r > span) r = GEN_SUB(P, r);
  return gen_exp10(GEN_ADD(lo, r));
}

#endif
