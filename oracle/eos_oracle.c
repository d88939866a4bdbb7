/* eos_oracle.c -- the CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct C, fp64 throughout, written from the paper
 * (arXiv 2112.03229, /root/reference/PAPER.md, cited as P:<line>).  It shares
 * no code with the CUDA product path (paper_2112_03229_b200/), and only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load it.  Build: gcc -O2 -fno-fast-math -ffp-contract=off
 * (no FTZ/DAZ: subnormal compares must be exact IEEE; no FMA contraction).
 *
 * Pins (tests/test_oracle.py) -- every function below is pinned:
 *   oracle_lower_bound / oracle_search : brute-force linear count on tiny
 *       tables (exhaustive probe grids), the bracketing invariant, the
 *       hand-worked golden tables (tests/golden/), numpy.searchsorted /
 *       bisect (NaN masked), permutation invariance.
 *   oracle_interp2d : closed forms (bilinear reproduces a+b*r+c*t+d*r*t,
 *       node values exactly, 1-D reduction), convex-hull bound, scipy
 *       RegularGridInterpolator(method='linear').
 *   oracle_counters : recomputed from their definitions in numpy.
 */
#include <math.h>
#include <stdint.h>

/* Lower-bound search, P:54 (section "Methodology"):
 *   "returning an array of size m containing the index of the last element
 *    of X which is less than or equal to each element of Y.  If X contains
 *    no such lower bound for a given y, the index 0 is chosen.  In the case
 *    that the element is higher than the highest of X, the index n-1 is
 *    chosen."
 * i.e. idx(y) = max(0, #{j : X[j] <= y} - 1), "<=" the IEEE-754 comparison.
 * The count #{j : X[j] <= y} is found by plain bisection over the sorted X
 * (binary search): the predicate X[mid] <= y is true on a prefix of X.
 * NaN compares false, so a NaN target has count 0 and gets index 0 (the
 * literal P:54 reading; reading R4). */
int32_t oracle_lower_bound(const double* X, int64_t n, double y) {
  int64_t lo = 0, hi = n; /* invariant: X[j] <= y for j < lo; X[j] > y (or NaN y) for j >= hi */
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (X[mid] <= y)
      lo = mid + 1;
    else
      hi = mid;
  }
  /* lo == count of entries <= y */
  return (int32_t)(lo > 0 ? lo - 1 : 0);
}

/* Batch form, P:54 ("returning an array of size m"). */
void oracle_search(const double* X, int64_t n, const double* Y, int64_t m, int32_t* out) {
  for (int64_t i = 0; i < m; ++i) out[i] = oracle_lower_bound(X, n, Y[i]);
}

/* EOSPAC-style 2-D interpolation (EOSPAC "interpolate[s]" SESAME
 * data on density x temperature using the searched brackets; the paper gives
 * no formula -- DESIGN.md reading R14):
 *   i = idx_R(rho), j = idx_T(T)  (the P:54 lower bounds, returned as is)
 *   ci = min(i, nR-2), cj = min(j, nT-2)      (cell of the bracket)
 *   tx = (rho - R[ci]) / (R[ci+1] - R[ci]),  ty likewise, each clamped to
 *   [0,1] by comparisons (NaN stays NaN)
 *   P = (1-tx)*((1-ty)*G[ci][cj] + ty*G[ci][cj+1])
 *     +    tx *((1-ty)*G[ci+1][cj] + ty*G[ci+1][cj+1])
 * G is row-major [nR][nT] (T fastest).  Outputs may be NULL except P. */
static double clamp01(double t) { return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t); }

void oracle_interp2d(const double* R, int64_t nR, const double* Tax, int64_t nT, const double* G,
                     const double* rho, const double* T, int64_t m, double* P, int32_t* iR,
                     int32_t* iT) {
  for (int64_t q = 0; q < m; ++q) {
    int32_t i = oracle_lower_bound(R, nR, rho[q]);
    int32_t j = oracle_lower_bound(Tax, nT, T[q]);
    int64_t ci = i < nR - 2 ? i : nR - 2;
    int64_t cj = j < nT - 2 ? j : nT - 2;
    double tx = clamp01((rho[q] - R[ci]) / (R[ci + 1] - R[ci]));
    double ty = clamp01((T[q] - Tax[cj]) / (Tax[cj + 1] - Tax[cj]));
    double g00 = G[ci * nT + cj], g01 = G[ci * nT + cj + 1];
    double g10 = G[(ci + 1) * nT + cj], g11 = G[(ci + 1) * nT + cj + 1];
    P[q] = (1.0 - tx) * ((1.0 - ty) * g00 + ty * g01) + tx * ((1.0 - ty) * g10 + ty * g11);
    if (iR) iR[q] = i;
    if (iT) iT[q] = j;
  }
}

/* Derivatives of the interpolant above (EOSPAC returns F, dF/dx, dF/dy with
 * every interpolation; P:14, P:41 name the interpolation, the formula is
 * reading R23 in DESIGN.md): the partial derivatives of the bilinear form on
 * the bracket cell,
 *   dP/drho = ((1-ty)(G[ci+1][cj]-G[ci][cj]) + ty(G[ci+1][cj+1]-G[ci][cj+1]))
 *             / (R[ci+1]-R[ci])
 *   dP/dT   = ((1-tx)(G[ci][cj+1]-G[ci][cj]) + tx(G[ci+1][cj+1]-G[ci+1][cj]))
 *             / (T[cj+1]-T[cj])
 * inside the grid; outside the axis range the clamped interpolant is constant
 * along that axis, so the derivative is 0; a NaN coordinate gives NaN.
 * dPdrho / dPdT may be NULL. */
void oracle_interp2d_deriv(const double* R, int64_t nR, const double* Tax, int64_t nT,
                           const double* G, const double* rho, const double* T, int64_t m,
                           double* dPdrho, double* dPdT) {
  for (int64_t q = 0; q < m; ++q) {
    int32_t i = oracle_lower_bound(R, nR, rho[q]);
    int32_t j = oracle_lower_bound(Tax, nT, T[q]);
    int64_t ci = i < nR - 2 ? i : nR - 2;
    int64_t cj = j < nT - 2 ? j : nT - 2;
    double tx = clamp01((rho[q] - R[ci]) / (R[ci + 1] - R[ci]));
    double ty = clamp01((T[q] - Tax[cj]) / (Tax[cj + 1] - Tax[cj]));
    double g00 = G[ci * nT + cj], g01 = G[ci * nT + cj + 1];
    double g10 = G[(ci + 1) * nT + cj], g11 = G[(ci + 1) * nT + cj + 1];
    double sr = ((1.0 - ty) * (g10 - g00) + ty * (g11 - g01)) / (R[ci + 1] - R[ci]);
    double st = ((1.0 - tx) * (g01 - g00) + tx * (g11 - g10)) / (Tax[cj + 1] - Tax[cj]);
    int in_r = rho[q] >= R[0] && rho[q] <= R[nR - 1];
    int in_t = T[q] >= Tax[0] && T[q] <= Tax[nT - 1];
    if (dPdrho) dPdrho[q] = (rho[q] != rho[q]) ? rho[q] : (in_r ? sr : 0.0);
    if (dPdT) dPdT[q] = (T[q] != T[q]) ? T[q] : (in_t ? st : 0.0);
  }
}

/* Log-log bilinear interpolation (EOSPAC-style table variant, SURVEY §8(f)
 * f4; reading R24 in DESIGN.md): the same brackets and cells as
 * oracle_interp2d, but the interpolation runs on ln P over (ln rho, ln T):
 *   tx = clamp01((ln rho - ln R[ci]) / (ln R[ci+1] - ln R[ci])), ty likewise
 *   P  = exp((1-tx)((1-ty) ln G[ci][cj] + ty ln G[ci][cj+1])
 *            + tx ((1-ty) ln G[ci+1][cj] + ty ln G[ci+1][cj+1]))
 * The log differences are evaluated as ln(a) - ln(b) = log1p((a - b) / b),
 * the same real number (R24): written as a difference of two logs, fp64
 * loses ~|ln a| / (ln a - ln b) ulps of the weight to cancellation on narrow
 * cells, which the weight's error then carries into P (pinned against
 * 40-digit decimal logarithms in tests/test_oracle.py).
 * Requires R, T, G > 0.  Exact for power laws G = C rho^a T^b.  Derivatives
 * (NULL-able): dP/drho = P * s_rho / rho with s_rho the cell slope of ln P in
 * ln rho, 0 outside the axis range, NaN for NaN; likewise dP/dT. */
void oracle_interp2d_loglog(const double* R, int64_t nR, const double* Tax, int64_t nT,
                            const double* G, const double* rho, const double* T, int64_t m,
                            double* P, int32_t* iR, int32_t* iT, double* dPdrho, double* dPdT) {
  for (int64_t q = 0; q < m; ++q) {
    int32_t i = oracle_lower_bound(R, nR, rho[q]);
    int32_t j = oracle_lower_bound(Tax, nT, T[q]);
    int64_t ci = i < nR - 2 ? i : nR - 2;
    int64_t cj = j < nT - 2 ? j : nT - 2;
    double wr = log1p((R[ci + 1] - R[ci]) / R[ci]);    /* ln R[ci+1] - ln R[ci] */
    double wt = log1p((Tax[cj + 1] - Tax[cj]) / Tax[cj]);
    double tx = clamp01(log1p((rho[q] - R[ci]) / R[ci]) / wr);  /* (ln rho - ln R[ci]) / wr */
    double ty = clamp01(log1p((T[q] - Tax[cj]) / Tax[cj]) / wt);
    double l00 = log(G[ci * nT + cj]), l01 = log(G[ci * nT + cj + 1]);
    double l10 = log(G[(ci + 1) * nT + cj]), l11 = log(G[(ci + 1) * nT + cj + 1]);
    double lp = (1.0 - tx) * ((1.0 - ty) * l00 + ty * l01) + tx * ((1.0 - ty) * l10 + ty * l11);
    double p = exp(lp);
    P[q] = p;
    if (iR) iR[q] = i;
    if (iT) iT[q] = j;
    double sr = ((1.0 - ty) * (l10 - l00) + ty * (l11 - l01)) / wr;
    double st = ((1.0 - tx) * (l01 - l00) + tx * (l11 - l10)) / wt;
    int in_r = rho[q] >= R[0] && rho[q] <= R[nR - 1];
    int in_t = T[q] >= Tax[0] && T[q] <= Tax[nT - 1];
    if (dPdrho) dPdrho[q] = (rho[q] != rho[q]) ? rho[q] : (in_r ? p * sr / rho[q] : 0.0);
    if (dPdT) dPdT[q] = (T[q] != T[q]) ? T[q] : (in_t ? p * st / T[q] : 0.0);
  }
}

/* Validation counters over one shard (DESIGN.md
 * "Counters").  Accumulated (+=) into c[8], all sums modulo 2^64:
 *   c0 = number of targets
 *   c1 = sum of idx
 *   c2 = sum of mix64(mix64(global_position) ^ idx)     (position-aware checksum;
 *        DESIGN.md R25: mix64 is a bijection of 64-bit words, so for a fixed
 *        position distinct indices give distinct terms, at any n and position)
 *   c3 = #{y : !(y >= X[0])}   (below range or NaN: "no such lower bound")
 *   c4 = #{y : y > X[n-1]}     (above range: "higher than the highest")
 *   c5 = #{y : y is NaN}
 *   c6 = #{y : y == X[idx]}    (exact ties with a table entry)
 *   c7 = 0 (reserved)
 * mix64 is the splitmix64 finalizer, written out here independently; it is
 * pinned to the published splitmix64 output streams (tests/golden/
 * splitmix64_vectors.txt: output k of seed s is mix64(s + k * 0x9E3779B97F4A7C15)). */
uint64_t oracle_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void oracle_counters(const double* X, int64_t n, const double* Y, const int32_t* idx, int64_t m,
                     int64_t global_offset, uint64_t* c) {
  for (int64_t i = 0; i < m; ++i) {
    double y = Y[i];
    uint64_t k = (uint64_t)idx[i];
    c[0] += 1;
    c[1] += k;
    c[2] += oracle_mix64(oracle_mix64((uint64_t)(global_offset + i)) ^ k);
    c[3] += !(y >= X[0]);
    c[4] += (y > X[n - 1]);
    c[5] += (y != y);
    c[6] += (y == X[k]);
  }
}
