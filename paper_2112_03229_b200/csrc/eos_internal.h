// eos_internal.h -- host-side structures shared by the C-ABI translation units
// of libeossearch.so (product path; never includes or links oracle/ code).
#pragma once

#include <stdint.h>

#include <vector>

#include "eossearch.h"

namespace eos {

// Bin-key of a binary64 value, host side.  Must equal the device key in
// kernels.cuh bit for bit (tested through eos_plan_table vs the kernels).
//   mode 0 (X[0] >= 0): hi = upper 32 bits of |v| (sign masked).  For v >= 0
//     the upper word is (biased exponent << 20) | top 20 mantissa bits, so
//     hi >> (20 - k) is the paper's exponent hash refined by k
//     mantissa bits; it is monotone non-decreasing in v >= 0.
//   mode 1 (negatives present): order-preserving transform of the bits of
//     (v + 0.0) (canonicalises -0.0), monotone over all non-NaN doubles.
uint32_t key_hi(double v, int mode);

struct TablePlan {
  int64_t n = 0;
  int key_mode = 0;
  int k = 0;
  int shift = 20;          // 20 - k
  uint32_t base = 0;       // key_hi(X_lo) >> shift
  uint32_t top = 0;        // key_hi(X[n-1]) >> shift
  int bins = 0;            // top - base + 1
  int max_occ = 0;
  int steps = 0;           // ceil(log2(max_occ + 1))
  std::vector<double> X;   // canonicalised table (-0.0 -> +0.0)
  std::vector<uint32_t> dir;  // packed lo | occ << 16, size bins
  int64_t x_bytes = 0;     // X region in the image (16-B padded)
  int64_t image_bytes = 0; // X region + directory (16-B padded)
};

// Smem budget used by the automatic k choice (bytes of X + directory): one
// image copy per SM at the 1024-thread launch shape.  Measured: a larger
// image that removes an in-bin step wins (cfg5 k=9/S=3 at 138 KB beats
// k=7/S=4 at 59 KB by 6%; cfg1 k=9/S=1 beats k=5/S=2 by 3%).
constexpr int64_t kAutoImageBudget = 200 * 1024;

// Validate + build (eos_plan_table semantics).  k_req: EOS_K_AUTO or 0..EOS_MAX_K.
// strict: axes of a 2-D grid must be strictly increasing and n >= 2.
eos_status plan_table(const double* X, int64_t n, int k_req, bool strict, TablePlan* out);

// Serialise X | dir into a 16-B padded byte image.
std::vector<uint8_t> make_image(const TablePlan& p);

void fill_info(const TablePlan& p, eos_table_info_t* info);

}  // namespace eos
