// table_build.cpp -- host-side setup of a search table (runs once per table,
// P:276 "Hashtable generation time is O(n)", "search setup ... performed
// only once").  Validation, canonicalisation, bin key, count directory and the
// choice of k.  Product path: shares no code with oracle/.
#include <math.h>
#include <string.h>

#include <algorithm>

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

namespace {

int ceil_log2_plus1(int occ) {  // S = ceil(log2(occ + 1)), occ >= 0
  int s = 0;
  while ((1 << s) < occ + 1) ++s;
  return s;
}

int64_t pad16(int64_t b) { return (b + 15) & ~int64_t(15); }

// Bin range for a given k (no directory yet).
void bin_range(const std::vector<double>& X, int mode, int k, uint32_t* base, uint32_t* top) {
  const int shift = 20 - k;
  const int64_t n = (int64_t)X.size();
  double lo = X[n - 1];
  if (mode == 0) {
    // lowest binned entry: first strictly positive one (a 0.0 head clamps into
    // bin 0; R13).  All-zero table -> a single bin.
    for (int64_t j = 0; j < n; ++j)
      if (X[j] > 0.0) { lo = X[j]; break; }
  } else {
    lo = X[0];
  }
  *base = key_hi(lo, mode) >> shift;
  *top = key_hi(X[n - 1], mode) >> shift;
}

eos_status build_for_k(const std::vector<double>& X, int mode, int k, TablePlan* p) {
  const int64_t n = (int64_t)X.size();
  uint32_t base, top;
  bin_range(X, mode, k, &base, &top);
  const int64_t bins = (int64_t)top - (int64_t)base + 1;
  if (bins < 1 || bins > (1 << 22)) return EOS_ERR_UNSUPPORTED;
  const int shift = 20 - k;
  std::vector<uint32_t> occ((size_t)bins, 0);
  for (int64_t j = 0; j < n; ++j) {
    uint32_t kb = key_hi(X[j], mode) >> shift;
    kb = std::min(std::max(kb, base), top);
    occ[kb - base]++;
  }
  p->dir.assign((size_t)bins, 0);
  uint32_t lo = 0, mx = 0;
  for (int64_t b = 0; b < bins; ++b) {
    p->dir[b] = lo | (occ[b] << 16);
    lo += occ[b];
    mx = std::max(mx, occ[b]);
  }
  p->n = n;
  p->key_mode = mode;
  p->k = k;
  p->shift = shift;
  p->base = base;
  p->top = top;
  p->bins = (int)bins;
  p->max_occ = (int)mx;
  p->steps = ceil_log2_plus1((int)mx);
  p->x_bytes = pad16(8 * n);
  p->image_bytes = p->x_bytes + pad16(4 * bins);
  return EOS_OK;
}

}  // namespace

eos_status plan_table(const double* Xin, int64_t n, int k_req, bool strict, TablePlan* out) {
  if (!Xin || !out) return EOS_ERR_NULL;
  if (n < (strict ? 2 : 1) || n > EOS_MAX_TABLE) return EOS_ERR_SIZE;
  if (k_req != EOS_K_AUTO && (k_req < 0 || k_req > EOS_MAX_K)) return EOS_ERR_UNSUPPORTED;
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

  if (k_req != EOS_K_AUTO) {
    TablePlan p;
    eos_status st = build_for_k(X, mode, k_req, &p);
    if (st != EOS_OK) return st;
    if (p.image_bytes > 200 * 1024) return EOS_ERR_UNSUPPORTED;  // does not fit in smem
    p.X = std::move(X);
    *out = std::move(p);
    return EOS_OK;
  }

  // Automatic k: the smallest fixed in-bin step count S
  // reachable with an image within kAutoImageBudget; ties -> smallest k
  // (smaller directory).  Bins only grow with k, so stop at the budget.
  TablePlan best;
  bool have = false;
  for (int k = 0; k <= EOS_MAX_K; ++k) {
    uint32_t base, top;
    bin_range(X, mode, k, &base, &top);
    int64_t bins = (int64_t)top - (int64_t)base + 1;
    int64_t img = pad16(8 * n) + pad16(4 * bins);
    if (have && img > kAutoImageBudget) break;
    TablePlan p;
    if (build_for_k(X, mode, k, &p) != EOS_OK) break;
    if (!have || p.steps < best.steps) {
      best = std::move(p);
      have = true;
    }
    if (best.steps <= 1) break;  // cannot do better than one probe
  }
  if (!have) return EOS_ERR_UNSUPPORTED;
  best.X = std::move(X);
  *out = std::move(best);
  return EOS_OK;
}

std::vector<uint8_t> make_image(const TablePlan& p) {
  std::vector<uint8_t> img((size_t)p.image_bytes, 0);
  memcpy(img.data(), p.X.data(), (size_t)(8 * p.n));
  memcpy(img.data() + p.x_bytes, p.dir.data(), (size_t)(4 * p.bins));
  return img;
}

void fill_info(const TablePlan& p, eos_table_info_t* info) {
  info->n = p.n;
  info->key_mode = p.key_mode;
  info->k = p.k;
  info->bins = p.bins;
  info->max_occ = p.max_occ;
  info->steps = p.steps;
  info->base = (int32_t)p.base;
  info->image_bytes = p.image_bytes;
  info->device = -1;
  info->ctas_per_sm = 0;
}

}  // namespace eos
