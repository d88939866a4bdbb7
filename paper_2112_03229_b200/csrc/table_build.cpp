// table_build.cpp -- host-side setup of a search table (runs once per table,
// P:276 "Hashtable generation time is O(n)", "search setup ... performed
// only once").  Validation, canonicalisation, bin key, count directory and the
// choice of hash.  Product path: shares no code with oracle/.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <thread>

#include "eos_internal.h"

namespace eos {

uint32_t key_hi(double v, int mode) {
  uint64_t b;
  if (mode == 0) {
    memcpy(&b, &v, 8);
    return (uint32_t)(b >> 32) & 0x7FFFFFFFu;
  }
  double c = v + 0.0;  // -0.0 -> +0.0 (round-to-nearest)
  memcpy(&b, &c, 8);
  uint32_t h = (uint32_t)(b >> 32);
  return (h & 0x80000000u) ? ~h : (h | 0x80000000u);
}

uint64_t key64(double v, int mode) {
  uint64_t b;
  if (mode == 0) {
    memcpy(&b, &v, 8);
    return b & 0x7FFFFFFFFFFFFFFFull;
  }
  double c = v + 0.0;  // -0.0 -> +0.0 (round-to-nearest)
  memcpy(&b, &c, 8);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

namespace {

int ceil_log2_plus1(int occ) {  // S = ceil(log2(occ + 1)), occ >= 0
  int s = 0;
  while ((1 << s) < occ + 1) ++s;
  return s;
}

int64_t pad16(int64_t b) { return (b + 15) & ~int64_t(15); }

// Key of the lowest binned entry.  Mode 0: the first strictly positive entry
// (a 0.0 head clamps into bin 0; R13); an all-zero table gives a
// single bin.  Mode 1: X[0].
uint32_t low_key(const std::vector<double>& X, int mode) {
  const int64_t n = (int64_t)X.size();
  if (mode == 1) return key_hi(X[0], 1);
  for (int64_t j = 0; j < n; ++j)
    if (X[j] > 0.0) return key_hi(X[j], 0);
  return key_hi(X[n - 1], 0);
}

// Bin parameters of a hash; returns the number of bins (0 if unusable).
struct HashParams {
  int kind, k;
  uint32_t hb, M, bmax;
  int64_t bins;
};

HashParams exponent_params(const std::vector<double>& X, int mode, int k) {
  HashParams h{EOS_HASH_EXPONENT, k, 0, 0, 0, 0};
  const int shift = 20 - k;
  const uint32_t lo = low_key(X, mode), top = key_hi(X.back(), mode);
  h.hb = lo & ~((1u << shift) - 1u);
  h.M = 1u << (12 + k);
  h.bins = (int64_t)((top - h.hb) >> shift) + 1;
  h.bmax = (uint32_t)(h.bins - 1);
  return h;
}

HashParams log_params(const std::vector<double>& X, int mode, int64_t H) {
  // Eq. 1: |H| bins of equal width in log2~ over [X_lo, X_max];
  // M = floor(|H| 2^32 / (span + 1)) keeps every bin index below |H|.
  HashParams h{EOS_HASH_LOG, -1, 0, 0, 0, 0};
  const uint32_t lo = low_key(X, mode), top = key_hi(X.back(), mode);
  h.hb = lo;
  const uint64_t span = (uint64_t)(top - lo) + 1;
  uint64_t M = ((uint64_t)H << 32) / span;
  M = std::max<uint64_t>(1, std::min<uint64_t>(M, 0xFFFFFFFFull));
  h.M = (uint32_t)M;
  h.bins = (int64_t)bin_of_key(top, h.hb, h.M, 0xFFFFFFFFu) + 1;
  h.bmax = (uint32_t)(h.bins - 1);
  return h;
}

int64_t image_of(int64_t n, int64_t bins, bool dir16 = false) {
  return pad16(8 * n) + pad16((dir16 ? 2 : 4) * bins);
}

double lifting_probes(int o, int S);
// Layout of a search table's lifting (kernels.cuh lookup_b), choose_layout below.
struct Layout {
  bool dir16 = false;
  int sf = 0;
  bool big = false;
  int64_t image = 0;
  double cost = 0.0;
};
Layout choose_layout(const std::vector<int64_t>& runs, int64_t n, int64_t bins, int steps,
                     double probes_per_bin, bool search);

eos_status build(const std::vector<double>& X, int mode, const HashParams& h, TablePlan* p,
                 bool search) {
  const int64_t n = (int64_t)X.size();
  if (h.bins < 1 || h.bins > (int64_t(1) << 22)) return EOS_ERR_UNSUPPORTED;
  std::vector<uint32_t> occ((size_t)h.bins, 0);
  for (int64_t j = 0; j < n; ++j) occ[bin_of_key(key_hi(X[j], mode), h.hb, h.M, h.bmax)]++;
  p->dir.assign((size_t)h.bins, 0);
  uint32_t lo = 0, mx = 0;
  for (int64_t b = 0; b < h.bins; ++b) {
    p->dir[b] = lo | (occ[b] << 16);
    lo += occ[b];
    mx = std::max(mx, occ[b]);
  }
  p->n = n;
  p->key_mode = mode;
  p->hash_kind = h.kind;
  p->k = h.k;
  p->hb = h.hb;
  p->M = h.M;
  p->bmax = h.bmax;
  p->bins = (int)h.bins;
  p->max_occ = (int)mx;
  p->steps = ceil_log2_plus1((int)mx);
  p->x_bytes = pad16(8 * n);
  p->image_bytes = image_of(n, h.bins);
  p->dir16 = false;
  p->fast_steps = p->steps;
  p->big = false;
  if (search) {  // directory format + fixed / rare steps (choose_layout)
    std::vector<int64_t> runs;
    double probes = 0.0;
    for (int64_t b = 0; b < h.bins; ++b)
      if (occ[b]) {
        runs.push_back(occ[b]);
        probes += lifting_probes((int)occ[b], p->steps);
      }
    const Layout L = choose_layout(runs, n, h.bins, p->steps, probes / (double)h.bins, true);
    p->dir16 = L.dir16;
    p->fast_steps = L.sf;
    p->big = L.big;
    p->image_bytes = L.image;
  }
  return EOS_OK;
}

// Expected executed (non-predicated) probes of S-step binary lifting in a bin
// holding `o` entries (o < 2^S), the target uniform among the o+1 gaps.
// Before the step of stride s the count c is the final count cf with its bits
// below 2s cleared, and the probe j = c + s executes iff j <= o: so the step
// executes for every cf whose block base (multiple of 2s) is <= o - s.  O(S).
double lifting_probes(int o, int S) {
  int64_t total = 0;
  for (int64_t s = S > 0 ? int64_t(1) << (S - 1) : 0; s > 0; s >>= 1) {
    const int64_t last = o - s;  // largest block base whose probe executes
    if (last < 0) continue;
    const int64_t nb = last / (2 * s) + 1;  // blocks with an executed probe
    const int64_t base = (nb - 1) * 2 * s;
    total += base + std::min<int64_t>(2 * s, o + 1 - base);
  }
  return (double)total / (o + 1);
}

// Modelled per-lookup cost of a plan (evaluate below), in shared-memory
// wavefronts per warp of 32 lookups plus issue and occupancy terms:
//   3.5 (random 4-B directory read) + 6.1 x E[executed 8-B probes]
//   + 1 per in-bin step (issue) + a launch-shape penalty.
// The shape (search_api.cu::pick_search) keeps the smem of all resident image
// copies <= ~144 KB per SM, leaving L1 for the in-flight streaming loads:
// image <= 32 KB: 4 CTAs x 256 threads (penalty 0); <= 72 KB: 2 x 512 (1);
// <= 144 KB: 1 x 1024 (1.5); up to 200 KB: 1 x 1024 with L1 squeezed (4.5).
// (Not modelled: n = 4096 log-uniform runs 11% faster with S = 3 at 95 KB than
// with S = 2 at 143 KB, but cfg5 loses 1-4% with the same trade.)
// Measured: for cfg5 a 198 KB directory loses 18% against 143 KB
// (profiles/r01_exp_hash_*.json), but for n = 16384 (128 KB of X alone) a
// 197 KB image with 4x the bins wins 39% over 146 KB
// (profiles/r01_exp_table_size.json): the penalty lets only a large probe
// saving buy the extra smem.  Targets are taken log-uniform over the table
// range, i.e. uniform over the bins (equal key width).
// Launch-shape term of the cost: <= 32 KB: 4 CTAs x 256 per SM;
// <= 72 KB: 2 x 512; <= 100 KB: 1 x 1024, and two 62-KB stages of the ring kernel
// still fit next to the image (search_api.cu: deep tables stream through it, cfg5
// 528 -> 562 Glookups/s); <= 144 KB: register kernel only; above: L1 squeezed.
double shape_cost(int64_t image_bytes) {
  return image_bytes <= 32 * 1024 ? 0.0
         : image_bytes <= 72 * 1024 ? 1.0
         : image_bytes <= 100 * 1024 ? 1.5
         : image_bytes <= 144 * 1024 ? 3.0
                                     : 4.5;
}

double cost_of(double mean_probes, double issue, int64_t image_bytes) {
  return 3.5 + 6.1 * mean_probes + issue + shape_cost(image_bytes);
}

// Layout of a search table's lifting (kernels.cuh lookup_b): S <= 3 runs all
// S steps as fixed, branch-free steps (SF = S); deeper tables run 3 fixed steps
// after a branch for their larger strides (big).  (A rare branch in front of
// fewer fixed steps -- SF < S for S <= 3 -- was measured 3-10% slower on cfg5
// in spite of 30% fewer instructions: each branch is a reconvergence point, so
// the 8 lookups of a thread no longer overlap their shared-memory latencies;
// DESIGN.md §12.)  16-bit directory entries (n <= 4096, occupancy <= 15) are
// taken whenever they fit (8 lo | occ: n <= 8192, occupancy <= 7): their unpack
// costs the same two instructions as the 32-bit entry's, and the image is smaller.
Layout choose_layout(const std::vector<int64_t>& runs, int64_t n, int64_t bins, int steps,
                     double probes_per_bin, bool search) {
  Layout best;
  best.sf = steps;
  best.image = image_of(n, bins);
  best.cost = cost_of(probes_per_bin, (double)steps, best.image);
  if (!search) return best;
  int64_t mx = 0;
  for (const int64_t r : runs) mx = std::max(mx, r);
  const bool can16 = n <= kDir16MaxN && mx <= kDir16MaxOcc;
  const int sf = std::min(steps, kMaxFastSteps);
  const bool big = steps > sf;
  const double issue = steps + (big ? 1.0 : 0.0);  // the deep strides' loop and branch
  best.sf = sf;
  best.big = big;
  best.cost = cost_of(probes_per_bin, issue, best.image);
  if (can16) {  // (unpacking either format takes two instructions; smaller image wins ties)
    const int64_t img = image_of(n, bins, true);
    const double c = cost_of(probes_per_bin, issue, img);
    if (c < best.cost + 1e-9) {
      best.dir16 = true;
      best.image = img;
      best.cost = c;
    }
  }
  return best;
}

// A candidate hash evaluated without building its directory: the table is
// sorted, so the bins of its keys are non-decreasing and every non-empty bin
// is one run of equal bin indices (empty bins execute no probe).  O(n) per
// candidate instead of O(n + bins) plus two allocations; the sum runs over
// the non-empty bins in bin order, as a sum over the whole directory would.
struct CandidateEval {
  bool ok = false;
  int steps = 0;
  double cost = 0.0;
  int64_t image_bytes = 0;
};

CandidateEval evaluate(const std::vector<uint32_t>& keys, const HashParams& h, bool compact,
                       bool search, std::vector<int64_t>& runs) {
  CandidateEval e;
  const int64_t n = (int64_t)keys.size();
  if (h.bins < 1 || h.bins > (int64_t(1) << 22)) return e;
  auto bin = [&](int64_t j) { return bin_of_key(keys[j], h.hb, h.M, h.bmax); };
  // runs of equal bins, each found by galloping: O(log run) bin evaluations
  runs.clear();
  int64_t mx = 0;
  for (int64_t j = 0; j < n;) {
    const uint32_t b = bin(j);
    int64_t lo = j, step = 1;  // bin(lo) == b; find the first r > j with bin(r) != b
    while (lo + step < n && bin(lo + step) == b) {
      lo += step;
      step *= 2;
    }
    int64_t hi = std::min(n, lo + step);  // bin(hi) != b or hi == n
    while (hi - lo > 1) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (bin(mid) == b) lo = mid; else hi = mid;
    }
    if (hi < n && bin(hi) < b) return e;  // unsorted keys: cannot happen for a validated table
    runs.push_back(hi - j);
    mx = std::max(mx, hi - j);
    j = hi;
  }
  e.ok = true;
  e.steps = ceil_log2_plus1((int)mx);
  e.image_bytes = image_of(n, h.bins);
  if (compact) {
    e.cost = (double)e.steps;
    return e;
  }
  double memo[64];
  for (double& m : memo) m = -1.0;
  double probes = 0.0;
  for (const int64_t len : runs) {
    const int o = (int)len;
    if (o < 64) {
      if (memo[o] < 0) memo[o] = lifting_probes(o, e.steps);
      probes += memo[o];
    } else {
      probes += lifting_probes(o, e.steps);
    }
  }
  const Layout L = choose_layout(runs, n, h.bins, e.steps, probes / (double)h.bins, search);
  e.cost = L.cost;
  e.image_bytes = L.image;
  return e;
}

// Automatic choice: the candidate of least plan_cost with an
// image within kAutoImageBudget; ties -> the smaller image, then the exponent
// hash.  Candidates: the exponent hash for every k, and the logarithm hash
// for |H| on a geometric grid (8 per octave).
// Grid axes (compact = true) use the smallest S, then the smallest image: the
// 2-D kernel's smem is dominated by the grid and its S = 1 cell lookup reads
// the probe unconditionally (kernels.cuh::axis_cell), so bigger directories
// buy nothing there.
// fill_budget > 0 (grid axes of REP 2 kernels, grid_api.cu): the smallest S,
// then the MOST bins within fill_budget bytes -- there a sparser directory
// makes the second cell-record read rarer (kernels.cuh axis_cell_rec).
// For search tables (!compact) fill_budget > 0 replaces the image budget
// (tiered sample tables, plan_tiered).
eos_status plan_auto(const std::vector<double>& X, int mode, bool compact, TablePlan* out,
                     int64_t fill_budget, bool search) {
  const int64_t n = (int64_t)X.size();
  const bool fill = compact && fill_budget > 0;
  const int64_t budget = fill_budget > 0 ? fill_budget
                                         : (compact ? kAxisImageBudget : kAutoImageBudget);
  std::vector<uint32_t> keys((size_t)n);
  for (int64_t j = 0; j < n; ++j) keys[j] = key_hi(X[j], mode);
  // candidates, in the order of preference of ties: exponent hash k = 0.., then
  // the logarithm hash on a geometric |H| grid
  std::vector<HashParams> cand;
  // (16-bit directory entries may fit twice the bins: search tables, n <= 4096)
  const bool may16 = search && n <= kDir16MaxN;
  for (int k = 0; k <= EOS_MAX_K; ++k) {
    HashParams h = exponent_params(X, mode, k);
    if (k > 0 && image_of(n, h.bins, may16) > budget) break;
    cand.push_back(h);
  }
  const int64_t max_bins = (budget - pad16(8 * n)) / (may16 ? 2 : 4);
  for (double H = 1.0; H <= (double)max_bins; H *= 1.0905077326652577 /* 2^(1/8) */)
    cand.push_back(log_params(X, mode, (int64_t)H));
  // evaluate them (independently: over host threads for large tables) ...
  std::vector<CandidateEval> ev(cand.size());
  auto eval_range = [&](size_t i0, size_t step) {
    std::vector<int64_t> runs;
    for (size_t i = i0; i < cand.size(); i += step)
      if (cand[i].bins >= 1) ev[i] = evaluate(keys, cand[i], compact, search, runs);
  };
  static const unsigned max_threads = std::min(std::max(1u, std::thread::hardware_concurrency()), 8u);
  const size_t nth = n >= 1024 ? max_threads : 1;
  if (nth > 1) {
    std::vector<std::thread> pool;
    try {
      for (size_t t = 1; t < nth; ++t) pool.emplace_back(eval_range, t, nth);
    } catch (...) {  // no threads available: the remaining ranges run here
      for (size_t t = pool.size() + 1; t < nth; ++t) eval_range(t, nth);
    }
    eval_range(0, nth);
    for (auto& th : pool) th.join();
  } else {
    eval_range(0, 1);
  }
  // ... then choose sequentially, in candidate order (deterministic)
  HashParams best;
  CandidateEval best_e;
  bool have = false;
  for (size_t i = 0; i < cand.size(); ++i) {
    const HashParams& h = cand[i];
    if (h.bins < 1) continue;
    const CandidateEval& e = ev[i];
    if (!e.ok) continue;
    if (have && (search ? e.image_bytes : image_of(n, h.bins)) > budget) continue;
    const double c = e.cost;
    if (have && fill && e.image_bytes > budget) continue;
    const bool tie_better = fill ? e.image_bytes > best_e.image_bytes : e.image_bytes < best_e.image_bytes;
    if (!have || c < best_e.cost - 1e-9 || (c < best_e.cost + 1e-9 && tie_better)) {
      best = h;
      best_e = e;
      have = true;
    }
  }
  if (!have) return EOS_ERR_UNSUPPORTED;
  return build(X, mode, best, out, search);  // the directory of the chosen hash only
}

}  // namespace

eos_status plan_table(const double* Xin, int64_t n, int kind, int64_t param, bool strict,
                      TablePlan* out, int64_t fill_budget, int64_t max_n, bool search) {
  if (!Xin || !out) return EOS_ERR_NULL;
  if (n < (strict ? 2 : 1) || n > max_n) return EOS_ERR_SIZE;
  if (kind == EOS_HASH_EXPONENT && (param < 0 || param > EOS_MAX_K)) return EOS_ERR_UNSUPPORTED;
  if (kind == EOS_HASH_LOG && (param < 1 || param > (int64_t(1) << 22))) return EOS_ERR_UNSUPPORTED;
  if (kind != EOS_HASH_AUTO && kind != EOS_HASH_EXPONENT && kind != EOS_HASH_LOG)
    return EOS_ERR_UNSUPPORTED;
  std::vector<double> X((size_t)n);
  for (int64_t j = 0; j < n; ++j) {
    double v = Xin[j];
    if (!isfinite(v)) return EOS_ERR_NONFINITE;
    X[j] = (v == 0.0) ? 0.0 : v;  // canonicalise -0.0 (R6)
  }
  for (int64_t j = 1; j < n; ++j) {
    if (strict ? !(X[j] > X[j - 1]) : (X[j] < X[j - 1])) return EOS_ERR_UNSORTED;
  }
  const int mode = (X[0] >= 0.0) ? 0 : 1;

  TablePlan p;
  eos_status st;
  if (kind == EOS_HASH_AUTO) {
    st = plan_auto(X, mode, strict, &p, fill_budget, search && !strict);
  } else {
    const HashParams h = kind == EOS_HASH_EXPONENT ? exponent_params(X, mode, (int)param)
                                                   : log_params(X, mode, param);
    st = build(X, mode, h, &p, search && !strict);
    // the staged image must fit shared memory: fp64 X + directory, or for the
    // sample table of a tiered table (the caller passing max_n = kMaxTopKeys)
    // its 32-bit keys + directory (make_key_image)
    const int64_t staged = max_n == kMaxTopKeys ? pad16(4 * n) + pad16(4 * p.bins) : p.image_bytes;
    if (st == EOS_OK && staged > kMaxImage) st = EOS_ERR_UNSUPPORTED;
  }
  if (st != EOS_OK) return st;
  p.X = std::move(X);
  *out = std::move(p);
  return EOS_OK;
}

eos_status plan_tiered(const double* Xin, int64_t n, int levels, int kind, int64_t param,
                       TieredPlan* out) {
  if (!Xin || !out) return EOS_ERR_NULL;
  if (n < 1 || n > EOS_MAX_TABLE_TIERED) return EOS_ERR_SIZE;
  auto pow8 = [](int d) { return int64_t(1) << (3 * d); };
  if (levels == EOS_LEVELS_AUTO) {
    levels = 0;
    if (n > EOS_MAX_TABLE) {
      levels = 1;
      while ((n + pow8(levels) - 1) / pow8(levels) > kMaxTopKeys) ++levels;
    }
  }
  if (levels < 0 || levels > kMaxLevels) return EOS_ERR_UNSUPPORTED;
  const int64_t stride = pow8(levels);  // 8^D
  const int64_t n1 = (n + stride - 1) / stride;
  if (n1 > (levels == 0 ? EOS_MAX_TABLE : kMaxTopKeys)) return EOS_ERR_SIZE;
  TieredPlan t;
  t.levels = levels;
  t.n = n;
  t.top_n = n1;
  if (levels == 0) {
    eos_status st = plan_table(Xin, n, kind, param, false, &t.top, 0, EOS_MAX_TABLE, true);
    if (st != EOS_OK) return st;
    t.x_last = t.top.X[n - 1];
    *out = std::move(t);
    return EOS_OK;
  }
  // F level 0 = the validated, canonicalised table (same rules as plan_table).
  const int64_t len0 = n1 * stride;
  int64_t total = 0;
  for (int d = 0; d < levels; ++d) total += len0 / pow8(d);
  try {
    t.lv.assign((size_t)total, NAN);
    t.keys.assign((size_t)total, 0xFFFFFFFFu);
  } catch (...) {
    return EOS_ERR_NOMEM;
  }
  const int64_t off0 = total - len0;
  double* L0 = t.lv.data() + off0;
  for (int64_t j = 0; j < n; ++j) {
    const double v = Xin[j];
    if (!isfinite(v)) return EOS_ERR_NONFINITE;
    L0[j] = (v == 0.0) ? 0.0 : v;  // canonicalise -0.0 (R6)
    if (j > 0 && L0[j] < L0[j - 1]) return EOS_ERR_UNSORTED;
  }
  const int mode = (L0[0] >= 0.0) ? 0 : 1;
  // Coarser F levels are strided samples of level 0 (NaN padding stays NaN);
  // K levels are the keys of the F entries (padding keeps 0xFFFFFFFF).
  int64_t off = off0, len = len0;
  for (int d = 0; d < levels; ++d) {
    if (d > 0) {
      len /= kFanout;
      off -= len;
    }
    const int64_t s = pow8(d);
    double* Fd = t.lv.data() + off;
    uint32_t* Kd = t.keys.data() + off;
    for (int64_t j = 0; j * s < n; ++j) {
      Fd[j] = L0[j * s];
      Kd[j] = key_hi(Fd[j], mode);
    }
  }
  std::vector<double> T1((size_t)n1);
  for (int64_t j = 0; j < n1; ++j) T1[j] = L0[j * stride];
  // Image budget of the sample table, measured (profiles/r01_exp_table_size.json,
  // r01_exp_tiered_bins.json): 4 n1 bytes of keys + max(48 KB, 8 n1) bytes of
  // directory (~2-3 bins per entry, S = 2), at most kTieredImageBudget.  At
  // n = 2^15 a 49-64 KB image runs at 196 Glookups/s and >= 80 KB at 131:
  // the smaller carveout leaves L1 room for the 128 KB top key level.
  // plan_table budgets fp64 entries, so it is given 4 n1 more.
  const int64_t budget = std::min<int64_t>(kTieredImageBudget,
                                           4 * n1 + std::max<int64_t>(48 * 1024, 8 * n1));
  eos_status st = plan_table(T1.data(), n1, kind, param, false, &t.top, budget + 4 * n1,
                             kMaxTopKeys);
  if (st != EOS_OK) return st;
  // key mode of T1 is that of X (T1[0] = X[0])
  t.x_last = L0[n - 1];
  *out = std::move(t);
  return EOS_OK;
}

// One depth of a packed plan: the sample table over X[15^D j] and its hash, the
// nodes of levels D-1 .. 0 (X must be validated).  EOS_ERR_UNSUPPORTED when the
// sample image does not fit `budget` at any residual width.
static eos_status plan_packed_depth(PackedPlan& p, int D, int64_t budget) {
  const int64_t n = p.n;
  int64_t stride = 1;  // 15^D
  for (int d = 0; d < D; ++d) stride *= kPackedNode;
  const int64_t n1 = (n + stride - 1) / stride;
  if (n1 > kPackedMaxTop) return EOS_ERR_SIZE;
  if (pad16(2 * n1) + 16 > budget) return EOS_ERR_UNSUPPORTED;
  p.depth = D;
  p.n1 = n1;
  p.sh = 0;
  const int mode = p.key_mode;
  std::vector<uint32_t> K1((size_t)n1);
  std::vector<double> T1((size_t)n1);
  for (int64_t j = 0; j < n1; ++j) {
    T1[j] = p.X[j * stride];
    K1[j] = key_hi(T1[j], mode);
  }
  const uint32_t lowk = low_key(T1, mode), top = K1[n1 - 1];
  // sample hash: the residual width sh (16 .. 1) with the fewest lifting
  // steps whose image fits; ties go to the smaller image
  const int64_t rbytes = pad16(2 * n1);
  std::vector<int32_t> cnt;
  for (int sh = 16; sh >= 1; --sh) {
    const uint32_t hb = lowk & ~((1u << sh) - 1u);
    const int64_t bins = (int64_t)((top > hb ? top - hb : 0) >> sh) + 1;
    if (rbytes + pad16(4 * ((bins + 1) / 2)) > budget) break;  // more bins at smaller sh
    cnt.assign((size_t)bins, 0);
    int max_occ = 0;
    for (int64_t j = 0; j < n1; ++j) {
      const uint32_t b = bin_of_key(K1[j], hb, 1u << (32 - sh), (uint32_t)(bins - 1));
      max_occ = std::max(max_occ, ++cnt[b]);
    }
    if (max_occ > (1 << kPackedMaxSteps) - 1) continue;
    const int S = ceil_log2_plus1(max_occ);
    if (p.sh == 0 || S < p.steps) {
      p.sh = sh;
      p.hb = hb;
      p.bins = (int)bins;
      p.bmax = (uint32_t)(bins - 1);
      p.max_occ = max_occ;
      p.steps = S;
    }
  }
  if (p.sh == 0) return EOS_ERR_UNSUPPORTED;
  const int sh = p.sh;
  // nodes of levels D-1 .. 0, coarsest first: level d has ceil(n / 15^(d+1)) nodes
  int64_t total = 0;
  for (int d = 0; d < D; ++d) {
    int64_t sd = kPackedNode;  // 15^(d+1)
    for (int e = 0; e < d; ++e) sd *= kPackedNode;
    total += (n + sd - 1) / sd;
  }
  const int64_t dbytes = pad16(4 * (((int64_t)p.bins + 1) / 2));
  try {  // residuals | directory | level table (int32 first node [4], 15^d [4])
    p.image.assign((size_t)(rbytes + dbytes + 32), 0);
    p.nodes.assign((size_t)(8 * total), 0);
  } catch (...) {
    return EOS_ERR_NOMEM;
  }
  // sample residuals (the kernel's rk of the entry's own key) and directory
  std::vector<uint32_t> lo((size_t)p.bins, 0), occ((size_t)p.bins, 0);
  for (int64_t j = 0; j < n1; ++j) {
    // the 16 bits of key64 - (hb << 32) right below the bin bits (entries >= hb)
    const uint32_t u = (K1[j] > p.hb ? K1[j] : p.hb) - p.hb;
    const uint64_t u64 = K1[j] >= p.hb ? key64(T1[j], mode) - ((uint64_t)p.hb << 32) : 0;
    const uint16_t r = (uint16_t)(u64 >> (16 + sh));
    memcpy(p.image.data() + 2 * j, &r, 2);
    const uint32_t b = std::min(u >> sh, p.bmax);
    if (occ[b]++ == 0) lo[b] = (uint32_t)j;
  }
  uint32_t next = 0;  // empty bins: lo = first entry of the next non-empty bin
  for (int64_t b = p.bins - 1; b >= 0; --b) {
    if (occ[b] == 0) lo[b] = next;
    else next = lo[b];
  }
  for (int64_t g = 0; 2 * g < p.bins; ++g) {  // bin pairs
    const uint32_t o1 = 2 * g + 1 < p.bins ? occ[2 * g + 1] : 0;
    const uint32_t d = lo[2 * g] | (occ[2 * g] << 20) | (o1 << 26);
    memcpy(p.image.data() + rbytes + 4 * g, &d, 4);
  }
  // nodes: node j of level d covers X[15^(d+1) j + 15^d t], t = 0..14
  int64_t off = 0;
  for (int d = D - 1; d >= 0; --d) {
    int64_t sd = 1;  // 15^d
    for (int e = 0; e < d; ++e) sd *= kPackedNode;
    const int64_t m = (n + kPackedNode * sd - 1) / (kPackedNode * sd);
    p.level_off[d] = off;
    p.level_stride[d] = sd;
    for (int64_t j = 0; j < m; ++j) {
      const int64_t i0 = kPackedNode * sd * j;
      const int64_t last = std::min<int64_t>(i0 + (kPackedNode - 1) * sd, (n - 1 - i0) / sd * sd + i0);
      const uint32_t Bm = key_hi(p.X[i0], mode) & ~63u;
      const uint64_t base = (uint64_t)Bm << 32;
      const uint64_t span = key64(p.X[last], mode) - base;
      uint32_t s = 0;
      while ((span >> s) > kPackedResMax) ++s;
      uint32_t* w = p.nodes.data() + 8 * (off + j);
      w[0] = Bm | s;
      for (int t = 1; t < kPackedNode; ++t) {
        const int64_t i = i0 + t * sd;
        const uint32_t r =
            i < n ? (uint32_t)((key64(p.X[i], mode) - base) >> s) + kPackedResBias : kPackedResPad;
        w[(t + 1) / 2] |= (t & 1) ? r : (r << 16);
      }
    }
    off += m;
  }
  int32_t lt[2 * kPackedMaxDepth] = {};
  for (int d = 0; d < D; ++d) {
    lt[d] = (int32_t)p.level_off[d];
    lt[kPackedMaxDepth + d] = (int32_t)p.level_stride[d];
  }
  memcpy(p.image.data() + rbytes + dbytes, lt, sizeof(lt));
  return EOS_OK;
}

eos_status plan_packed(const double* Xin, int64_t n, PackedPlan* out, int64_t budget, int depth) {
  if (!Xin || !out) return EOS_ERR_NULL;
  if (n < 1 || n > EOS_MAX_TABLE_TIERED) return EOS_ERR_SIZE;
  if (depth < 0 || depth > kPackedMaxDepth) return EOS_ERR_UNSUPPORTED;
  {  // fail early (before touching X) when no allowed depth can fit
    const int dmax = depth ? depth : kPackedMaxDepth;
    int64_t stride = 1;
    for (int d = 0; d < dmax; ++d) stride *= kPackedNode;
    if (pad16(2 * ((n + stride - 1) / stride)) + 16 > budget) return EOS_ERR_UNSUPPORTED;
  }
  PackedPlan p;
  p.n = n;
  try {
    p.X.resize((size_t)n);
  } catch (...) {
    return EOS_ERR_NOMEM;
  }
  for (int64_t j = 0; j < n; ++j) {  // same rules as plan_table
    const double v = Xin[j];
    if (!isfinite(v)) return EOS_ERR_NONFINITE;
    p.X[j] = (v == 0.0) ? 0.0 : v;  // canonicalise -0.0 (R6)
    if (j > 0 && p.X[j] < p.X[j - 1]) return EOS_ERR_UNSORTED;
  }
  p.key_mode = (p.X[0] >= 0.0) ? 0 : 1;
  p.x0 = p.X[0];
  p.x_last = p.X[n - 1];
  // the given depth, or the smallest that fits (each level is one more L2 gather)
  eos_status st = EOS_ERR_UNSUPPORTED;
  for (int D = depth ? depth : 1; D <= (depth ? depth : kPackedMaxDepth); ++D) {
    st = plan_packed_depth(p, D, budget);
    if (st == EOS_OK) break;
    if (st != EOS_ERR_UNSUPPORTED && st != EOS_ERR_SIZE) return st;
  }
  if (st != EOS_OK) return st;
  *out = std::move(p);
  return EOS_OK;
}

TablePlan packed_top(const PackedPlan& p) {
  TablePlan t;
  t.n = p.n1;
  t.key_mode = p.key_mode;
  t.hash_kind = EOS_HASH_EXPONENT;
  t.k = 20 - p.sh;
  t.hb = p.hb;
  t.M = 1u << (32 - p.sh);
  t.bmax = p.bmax;
  t.bins = p.bins;
  t.max_occ = p.max_occ;
  t.steps = p.steps;
  t.fast_steps = p.steps;
  t.x_bytes = pad16(2 * p.n1);
  t.image_bytes = (int64_t)p.image.size();
  t.dir16 = true;  // 2 B per bin (one u32 per bin pair)
  return t;
}

void fill_info(const PackedPlan& p, eos_table_info_t* info) {
  fill_info(packed_top(p), info);
  info->n = p.n;
  info->levels = p.depth;
  info->node_width = kPackedNode;
  info->top_n = p.n1;
  info->level_bytes = ((8 * p.n + 31) & ~int64_t(31)) + 4 * (int64_t)p.nodes.size();  // X, then the nodes
}

int64_t key_image_bytes(const TablePlan& p) { return pad16(4 * p.n) + pad16(4 * p.bins); }

std::vector<uint8_t> make_key_image(const TablePlan& p) {
  std::vector<uint8_t> img((size_t)key_image_bytes(p), 0);
  for (int64_t j = 0; j < p.n; ++j) {
    const uint32_t k = key_hi(p.X[j], p.key_mode);
    memcpy(img.data() + 4 * j, &k, 4);
  }
  memcpy(img.data() + pad16(4 * p.n), p.dir.data(), (size_t)(4 * p.bins));
  return img;
}

std::vector<uint8_t> make_image(const TablePlan& p) {
  std::vector<uint8_t> img((size_t)p.image_bytes, 0);
  memcpy(img.data(), p.X.data(), (size_t)(8 * p.n));
  if (p.dir16) {  // 8 lo | occ (kernels.cuh dir_entry)
    for (int64_t b = 0; b < p.bins; ++b) {
      const uint32_t d = p.dir[b];
      const uint16_t e = (uint16_t)(((d & 0xFFFFu) << 3) | (d >> 16));
      memcpy(img.data() + p.x_bytes + 2 * b, &e, 2);
    }
  } else {
    memcpy(img.data() + p.x_bytes, p.dir.data(), (size_t)(4 * p.bins));
  }
  return img;
}

void fill_info(const TablePlan& p, eos_table_info_t* info) {
  info->n = p.n;
  info->key_mode = p.key_mode;
  info->k = p.k;
  info->bins = p.bins;
  info->max_occ = p.max_occ;
  info->steps = p.steps;
  info->base = (int32_t)p.hb;
  info->image_bytes = p.image_bytes;
  info->device = -1;
  info->ctas_per_sm = 0;
  info->hash_kind = p.hash_kind;
  info->hash_mult = p.M;
  info->levels = 0;
  info->node_width = 0;
  info->top_n = p.n;
  info->level_bytes = 0;
  info->dir_entry_bytes = p.dir16 ? 2 : 4;
  info->fast_steps = p.fast_steps;
  info->rare_steps = p.big ? 1 : 0;
  info->ring_stages = 0;
  info->cell_map = 0;
}

void fill_info(const TieredPlan& t, eos_table_info_t* info) {
  fill_info(t.top, info);
  if (t.levels > 0) info->image_bytes = key_image_bytes(t.top);  // keys, not fp64
  info->n = t.n;
  info->levels = t.levels;
  info->node_width = t.levels > 0 ? 8 : 0;
  info->top_n = t.top_n;
  info->level_bytes = 12 * t.level_elems();  // fp64 F + u32 K per level entry
}

}  // namespace eos
