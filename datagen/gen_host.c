/* gen_host.c -- host (CPU) side of the datagen generators (see gen_core.h).
 * Built with: gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math
 * Exported with plain C linkage for ctypes.  Contains no method arithmetic. */
#include "gen_core.h"

uint64_t gen_stream_key(uint64_t seed, uint64_t stream) { return gen_key(seed, stream); }

double gen_exp10_host(double t) { return gen_exp10(t); }

/* out[j] = target at global index offset+j */
void gen_fill_loguniform(uint64_t seed, uint64_t stream, int64_t offset, int64_t count,
                         double a, double w, double* out) {
  uint64_t key = gen_key(seed, stream);
  for (int64_t j = 0; j < count; ++j) out[j] = gen_loguniform(key, (uint64_t)(offset + j), a, w);
}

/* out[j] = target at global index idx[j] (any order) */
void gen_sample_loguniform(uint64_t seed, uint64_t stream, const int64_t* idx, int64_t nidx,
                           double a, double w, double* out) {
  uint64_t key = gen_key(seed, stream);
  for (int64_t j = 0; j < nidx; ++j) out[j] = gen_loguniform(key, (uint64_t)idx[j], a, w);
}

void gen_fill_copies(uint64_t seed, int64_t offset, int64_t count, double a, double w,
                     const double* X, int64_t n, uint64_t copy_every, double* out) {
  uint64_t key = gen_key(seed, 0), key2 = gen_key(seed, 1);
  for (int64_t j = 0; j < count; ++j)
    out[j] = gen_with_copies(key, key2, (uint64_t)(offset + j), a, w, X, n, copy_every);
}

void gen_sample_copies(uint64_t seed, const int64_t* idx, int64_t nidx, double a, double w,
                       const double* X, int64_t n, uint64_t copy_every, double* out) {
  uint64_t key = gen_key(seed, 0), key2 = gen_key(seed, 1);
  for (int64_t j = 0; j < nidx; ++j)
    out[j] = gen_with_copies(key, key2, (uint64_t)idx[j], a, w, X, n, copy_every);
}

/* Sum of the walk steps s_i for i in [begin, end) (wrapping 64-bit: exact in any
 * split, so sub-range sums computed on separate threads add up to the same bits). */
uint64_t gen_walk_sum(uint64_t seed, int64_t begin, int64_t end) {
  uint64_t key = gen_key(seed, 0);
  uint64_t S = 0;
  for (int64_t i = begin; i < end; ++i) S += (uint64_t)gen_walk_step(key, (uint64_t)i);
  return S;
}

/* Random walk, global indices [offset, offset+count), given base = the sum of the
 * steps before offset (gen_walk_sum(seed, 0, offset)). */
void gen_fill_walk_from(uint64_t seed, int64_t offset, int64_t count, uint64_t base, double x0,
                        double c, double lo, double hi, double* out) {
  uint64_t key = gen_key(seed, 0);
  uint64_t S = base;
  for (int64_t j = 0; j < count; ++j) {
    S += (uint64_t)gen_walk_step(key, (uint64_t)(offset + j));
    out[j] = gen_walk_value((int64_t)S, x0, c, lo, hi);
  }
}

/* Random walk, global indices [offset, offset+count): sequential prefix sum. */
void gen_fill_walk(uint64_t seed, int64_t offset, int64_t count, double x0, double c, double lo,
                   double hi, double* out) {
  gen_fill_walk_from(seed, offset, count, gen_walk_sum(seed, 0, offset), x0, c, lo, hi, out);
}

/* Random walk at the sorted (non-decreasing) global indices idx[0..nidx). */
void gen_sample_walk(uint64_t seed, const int64_t* idx, int64_t nidx, double x0, double c,
                     double lo, double hi, double* out) {
  uint64_t key = gen_key(seed, 0);
  uint64_t S = 0;
  int64_t i = 0; /* next step to add */
  for (int64_t j = 0; j < nidx; ++j) {
    while (i <= idx[j]) { S += (uint64_t)gen_walk_step(key, (uint64_t)i); ++i; }
    out[j] = gen_walk_value((int64_t)S, x0, c, lo, hi);
  }
}
