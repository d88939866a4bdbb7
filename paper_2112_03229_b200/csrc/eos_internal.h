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
//     the upper word is (biased exponent << 20) | top 20 mantissa bits: a
//     fixed-point log2(v) (exact at powers of two, linear in the mantissa in
//     between), monotone non-decreasing in v >= 0.
//   mode 1 (negatives present): order-preserving transform of the bits of
//     (v + 0.0) (canonicalises -0.0), monotone over all non-NaN doubles.
uint32_t key_hi(double v, int mode);
// The whole 64-bit order-preserving key of which key_hi is the upper word (the
// packed tables' residuals take bits below it, PackedPlan).
uint64_t key64(double v, int mode);

// The one bin function of both hashes (host copy of kernels.cuh::bin_of):
//   bin(v) = min( umulhi( max(key_hi(v), hb) - hb, M ), bmax )
// Exponent hash with k mantissa bits: M = 2^(12+k), hb aligned
// down to a multiple of 2^(20-k)  =>  bin = (key >> (20-k)) - (hb >> (20-k)).
// Logarithm hash with |H| bins (Eqs. 1-2): M = |H| 2^32 / span,
// i.e. floor((log2~(v) - log2~(X_lo)) / log2~(b)) with the fixed-point log2~.
inline uint32_t bin_of_key(uint32_t key, uint32_t hb, uint32_t M, uint32_t bmax) {
  const uint32_t h = (key > hb ? key : hb) - hb;
  const uint32_t b = (uint32_t)(((uint64_t)h * (uint64_t)M) >> 32);
  return b < bmax ? b : bmax;
}

struct TablePlan {
  int64_t n = 0;
  int key_mode = 0;
  int hash_kind = 0;       // EOS_HASH_EXPONENT | EOS_HASH_LOG
  int k = 0;               // exponent hash: mantissa bits; log hash: -1
  uint32_t hb = 0;         // key of the lowest binned entry (aligned for the exponent hash)
  uint32_t M = 0;          // bin multiplier
  uint32_t bmax = 0;       // bins - 1
  int bins = 0;
  int max_occ = 0;
  int steps = 0;           // ceil(log2(max_occ + 1))
  // search tables (kernels.cuh lookup_b): directory entries of 16 bits
  // (8 lo | occ, n <= 8192 and max_occ <= 7) or 32 bits in the image;
  // fast_steps = SF fixed lifting steps (0: all S in a runtime loop); big =
  // some bin holds >= 2^SF entries (its larger strides run in a rare branch)
  bool dir16 = false;
  int fast_steps = 0;
  bool big = false;
  std::vector<double> X;   // canonicalised table (-0.0 -> +0.0)
  std::vector<uint32_t> dir;  // packed lo | occ << 16, size bins (canonical; the image may hold u16)
  int64_t x_bytes = 0;     // X region in the image (16-B padded)
  int64_t image_bytes = 0; // X region + directory (16-B padded)
};

// 16-bit directory entries: 8 lo | occ (8 (n - 1) + 7 < 2^16, occ <= 7)
constexpr int64_t kDir16MaxN = 8192;
constexpr int kDir16MaxOcc = 7;
constexpr int kMaxFastSteps = 3;  // fixed-step lifting bodies SF = 1..3 (kernels.cuh)

// Smem budget of the automatic hash choice (bytes of X + directory): one image
// copy per SM at the 1024-thread shape.  Images above 144 KB squeeze L1 and
// carry a cost penalty (table_build.cpp plan_cost).  Measured: a larger image
// that removes an in-bin step wins (cfg5 k=9/S=3 at 138 KB beats k=7/S=4 at
// 59 KB by 6%), a 198 KB image loses 18% on cfg5 but wins 39% at n = 16384.
constexpr int64_t kAutoImageBudget = 200 * 1024;
constexpr int64_t kAxisImageBudget = 16 * 1024;  // per axis of a 2-D grid (the grid owns smem)
constexpr int64_t kTieredImageBudget = 176 * 1024;  // cap of a tiered table's sample-table image
constexpr int64_t kMaxTopKeys = 32768;  // sample-table entries of a tiered table (32-bit keys)
constexpr int64_t kMaxImage = 200 * 1024;  // explicit requests beyond this do not fit in smem

// Validate + build (eos_plan_table_hash semantics).  kind/param: see
// eossearch.h (EOS_HASH_AUTO ignores param).  strict: axes of a 2-D grid must
// be strictly increasing and n >= 2.
// fill_budget: grid axes (strict): if > 0, among the automatic hash
// candidates with the smallest S take the one with the most bins whose image
// fits fill_budget bytes (instead of the smallest image); search tables: if
// > 0, the image budget of the automatic choice (default kAutoImageBudget).
// search: a single-level search table (16-bit directories and the fast-step /
// rare-branch split allowed; grid axes and tiered sample tables keep 32-bit
// entries and plain S-step lifting).
eos_status plan_table(const double* X, int64_t n, int kind, int64_t param, bool strict,
                      TablePlan* out, int64_t fill_budget = 0, int64_t max_n = EOS_MAX_TABLE,
                      bool search = false);

// Shared-memory image of a tiered table's sample table: the 32-bit keys of
// T1 (key_hi, the table's key mode) | directory, each 16-B padded.
std::vector<uint8_t> make_key_image(const TablePlan& p);
int64_t key_image_bytes(const TablePlan& p);

// Tables larger than shared memory (eossearch.h
// eos_search_create_levels).  D 8-ary levels in global memory under a
// shared-memory sample table T1[j] = X[j 8^D], j < n1 = ceil(n / 8^D) <=
// kMaxTopKeys, held as 32-bit keys (make_key_image).
// Level d (stride 8^d, d = 0..D-1) has n1 8^(D-d) entries
//   F_d[j] = X[j 8^d]            (fp64; NaN past n: never <= y)
//   K_d[j] = key_hi(F_d[j])      (u32 order-preserving upper word of the
//                                 key; 0xFFFFFFFF past n)
// A level step reads the 8 keys of a node (one 32-byte sector) and falls
// back to the node's 8 fp64 values only when a key equals the target's.
// Both arrays store their levels coarsest first (D-1, .., 0); level d starts
// at element n1 (8^(D-d) - 8) / 7 and F level 0 is X itself.
constexpr int kMaxLevels = 5;  // n <= 2^29 (EOS_MAX_TABLE_TIERED)
constexpr int kFanout = 8;
struct TieredPlan {
  int levels = 0;             // D (0: single-level smem table, `top` is the table)
  int64_t n = 0;              // entries of the full table
  int64_t top_n = 0;          // n1
  double x_last = 0.0;        // X[n-1]
  TablePlan top;              // T1 and its directory (the smem image)
  std::vector<double> lv;     // F levels (empty when levels == 0)
  std::vector<uint32_t> keys; // K levels
  int64_t level_elems() const { return (int64_t)lv.size(); }
};

// levels: EOS_LEVELS_AUTO (0 if n <= EOS_MAX_TABLE, else the smallest D with
// n1 <= kMaxTopKeys) or 0..kMaxLevels.  kind/param: the hash of T1.
eos_status plan_tiered(const double* X, int64_t n, int levels, int kind, int64_t param,
                       TieredPlan* out);

// Packed tables (eossearch.h EOS_LEVELS_PACKED): D levels of 32-byte nodes of
// 16-bit residual keys under a shared-memory sample table of 16-bit residual
// keys, so a lookup gathers D sectors from L2 -- one for tables up to ~1.5e6
// entries (the 8-ary levels gather ~log8 of n / 32768 more).  Level d (stored
// D-1 .. 0) holds ceil(n / 15^(d+1)) nodes; node j of level d covers the 15
// entries X[15^(d+1) j + 15^d t], t = 0..14 (below: d = 0, stride 1).
//   nodes:  node j covers X[15 j .. 15 j + 15) (kPackedNode entries); word 0 is
//           B_j | s_j with B_j = key_hi(X[15 j]) & ~63 and s_j (< 64) the
//           smallest shift with (key64(X[last of node]) - (B_j << 32)) >> s_j <=
//           0x77FF; words 1..7 hold the 14 residuals r_t = ((key64(X[15 j + t])
//           - (B_j << 32)) >> s_j) + 0x400, t = 1..14, two per word (t odd in the
//           low half), and 0x7C00 past n: as fp16 bit patterns these are normal
//           positive halves (or +inf past n) in the order of the keys, so the
//           kernel compares two per HSET2.  (64-bit keys: a node of a dense
//           table spans only a few hundred units of the 32-bit key, where equal
//           residuals -- each settled from X -- came for ~2% of lookups.)
//   sample: T1[j] = X[15^D j], j < n1 = ceil(n / 15^D), binned by the key-bit hash
//           bin = min((max(key, hb) - hb) >> sh, bmax) (hb aligned to 2^sh: the
//           exponent hash of k = 20 - sh mantissa bits); the image holds the
//           residuals -- the 16 key64 bits right below the bin bits, ((key64 -
//           (hb << 32)) >> (16 + sh)) & 0xFFFF, sh <= 16 -- as u16, then the
//           directory: one u32 per pair of bins (2g, 2g + 1), lo(2g) | occ(2g)
//           << 20 | occ(2g + 1) << 26 (occ <= 63, n1 <= 2^20), 16-B padded, then
//           the level table: int32 first node of level d [4], 15^d [4].
// Truncation keeps the order: r(X) < r(y) => X < y and r(X) > r(y) => X > y;
// equal residuals are settled from the fp64 values (X in device memory).
constexpr int kPackedNode = 15;
constexpr int kPackedMaxDepth = 4;  // levels of nodes (n <= 2^29 needs 4)
constexpr uint32_t kPackedResMax = 0x77FFu;   // largest residual (biased: 0x7BFF)
constexpr uint32_t kPackedResBias = 0x0400u;  // smallest normal fp16
constexpr uint32_t kPackedResPad = 0x7C00u;   // +inf: past n
constexpr int kPackedMaxSteps = 6;                 // occ <= 63 (6-bit fields)
constexpr int64_t kPackedMaxTop = int64_t(1) << 20;  // lo field
constexpr int64_t kPackedImageBudget = 224 * 1024;   // one 1024-thread CTA per SM
struct PackedPlan {
  int64_t n = 0;              // entries
  int depth = 1;              // D: levels of nodes; node j of level d covers X[15^(d+1) j + 15^d t]
  int64_t n1 = 0;             // sample entries T1[j] = X[15^D j] (= nodes of level D-1)
  int64_t level_off[kPackedMaxDepth] = {};     // first node of level d (levels D-1 .. 0 stored in that order)
  int64_t level_stride[kPackedMaxDepth] = {};  // 15^d
  int key_mode = 0;
  int sh = 0;                 // residual bits of the sample table
  uint32_t hb = 0, bmax = 0;
  int bins = 0, max_occ = 0, steps = 0;
  double x0 = 0.0, x_last = 0.0;
  std::vector<double> X;      // canonicalised table (device: X then the nodes)
  std::vector<uint32_t> nodes;  // 8 words per node, levels D-1 .. 0
  std::vector<uint8_t> image;   // smem image: u16 residuals | u32 directory
};
// EOS_ERR_UNSUPPORTED when no sh <= 16 gives an image within `budget` and bins of
// <= 63 entries (eos_search_create_levels then uses 8-ary levels under AUTO).
// depth 0: the smallest D <= kPackedMaxDepth whose sample table fits.
eos_status plan_packed(const double* X, int64_t n, PackedPlan* out,
                       int64_t budget = kPackedImageBudget, int depth = 0);
void fill_info(const PackedPlan& p, eos_table_info_t* info);
// The sample table of a packed plan as a TablePlan (hash fields, occupancy, T1).
TablePlan packed_top(const PackedPlan& p);

// Serialise X | dir into a 16-B padded byte image.
std::vector<uint8_t> make_image(const TablePlan& p);

void fill_info(const TablePlan& p, eos_table_info_t* info);
void fill_info(const TieredPlan& t, eos_table_info_t* info);

}  // namespace eos
