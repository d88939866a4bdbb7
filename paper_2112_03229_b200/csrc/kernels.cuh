// kernels.cuh -- sm_100a kernels of the hot path.
//
//   search1d_kernel        : per target y -> int32 lower bound
//   search1d_tiered_kernel : the same for tables larger than shared memory
//   search1d_direct_kernel : the same with the directory built on the device
//   interp2d_kernel        : per (rho, T) pair -> brackets + bilinear P (P:14,
//                            P:41), optionally dP/drho, dP/dT, log-log
//
// Design: HBM-bound streams.  The table X (fp64) and its
// hash count directory (u32) are staged once per CTA into shared memory
// (tables larger than shared memory: a sample of X, with the rest in L2-
// resident 8-ary key levels, search1d_tiered_kernel).  The grid has one CTA per tile of the target stream, but resident
// CTAs keep their staged image and steal the tiles of not-yet-launched CTAs
// with Blackwell cluster launch control (clusterlaunchcontrol.try_cancel):
// dynamic load balance at persistent-kernel cost, with no global counters.
// Tiles move with 128-bit streaming loads (ld.global.cs) and 64-bit
// streaming stores; the next tile's loads are issued before the current
// tile's results are stored.  Each target does a branchless bin lookup and a
// fixed-S-step branchless in-bin binary lifting (no warp divergence: S is a
// template constant of the launch).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "eossearch.h"

// Debug build (-DEOS_DEVICE_CHECKS, lib/libeossearch_checked.so): bounds checks
// on every shared/global access of the hot loops; a failure traps the kernel.
// (compute-sanitizer is not available on this GPU pool.)
#ifdef EOS_DEVICE_CHECKS
#include <cstdio>
#define EOS_DCHECK(c)                                                     \
  do {                                                                    \
    if (!(c)) {                                                           \
      printf("EOS_DCHECK failed: %s (%s:%d)\n", #c, __FILE__, __LINE__); \
      __trap();                                                           \
    }                                                                     \
  } while (0)
#else
#define EOS_DCHECK(c) \
  do {                \
  } while (0)
#endif

namespace eos {
namespace dev {

constexpr int kMaxTemplSteps = 8;  // S above this uses the runtime-S instantiation

struct AxisParams {
  int32_t n;        // entries
  int32_t x_off;    // byte offset of X (fp64[n]) in the smem image
  int32_t d_off;    // byte offset of the directory (u32[bins])
  uint32_t hb;      // key of the lowest binned entry
  uint32_t M;       // bin multiplier (exponent hash: 2^(12+k); log hash: |H| 2^32 / span)
  uint32_t bmax;    // bins - 1
  int32_t steps;    // S (used by the runtime-S path)
  int32_t mode;     // key mode (0: X[0] >= 0, sign-masked key; 1: order-preserving key)
  double x0;        // X[0]
  double xlast;     // X[n-1]
  // 2-D grid axes with a fitted cell map (axis_cell_rec, S = kMapped; grid_api.cu
  // fit_cell_map): cell(x) in {c, c + 1} for floor(map_a w(x) + map_b) = c (fp32),
  // w = log2 x (map_kind 1) or x (map_kind 2); map_kind 0: none
  float map_a;
  float map_b;
  int32_t map_kind;
};
// S of the 2-D kernels whose axes use their fitted cell maps instead of the
// directories (bank-pinned records only)
constexpr int kMapped = -1;

struct SearchArgs {
  const uint4* image;   // device image (16-B aligned)
  int32_t image_16;     // image size in 16-B words
  int32_t head;         // scalar-peeled leading elements (0/1) before the vector body
  int32_t vec_ok;       // 1: vector body usable (alignment)
  int32_t ring_ns;      // search1d_ring_kernel: shared-memory stages (2 .. kRingMaxStages)
  int64_t ntiles;       // tiles of the body (elements [head, count))
  AxisParams ax;
  const double* Y;
  int32_t* out;
  int64_t count;
  int64_t gofs;                  // global offset (counters)
  unsigned long long* counters;  // u64[8] or null
  // tiered tables (n > EOS_MAX_TABLE, search1d_tiered_kernel): the 8-ary
  // global levels, coarsest first (eos_internal.h TieredPlan); level d
  // (stride 8^d) holds n1 8^(D-d) entries: fp64 X[j 8^d] (NaN past the end)
  // at lv, their u32 keys (0xFFFFFFFF past the end) at kv.
  const double* lv;
  const uint32_t* kv;
  int64_t lv_top_len;            // 8 n1: length of level D-1
  int32_t levels;                // D (0: single-level smem table)
  int32_t sh;                    // packed tables: residual bits of the sample table
};

// splitmix64 finalizer (the checksum of counter c2; independent of oracle/)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Bin key of a target: upper word of the IEEE-754 bits, see eos_internal.h.
template <int MODE>
__device__ __forceinline__ uint32_t key_hi(double y) {
  if (MODE == 0) return (uint32_t)__double2hiint(y) & 0x7FFFFFFFu;
  const uint32_t h = (uint32_t)__double2hiint(__dadd_rn(y, 0.0));
  return h ^ ((uint32_t)((int32_t)h >> 31) | 0x80000000u);
}

// The whole 64-bit key (host: eos_internal.h key64); key_hi is its upper word.
template <int MODE>
__device__ __forceinline__ uint64_t key64(double y) {
  if (MODE == 0) return (uint64_t)__double_as_longlong(y) & 0x7FFFFFFFFFFFFFFFull;
  const uint64_t b = (uint64_t)__double_as_longlong(__dadd_rn(y, 0.0));
  return b ^ ((uint64_t)((int64_t)b >> 63) | 0x8000000000000000ull);
}

// The bin function of both hashes (host copy: eos_internal.h::bin_of_key).
__device__ __forceinline__ uint32_t bin_of(uint32_t key, const AxisParams& a) {
  return min(__umulhi(max(key, a.hb) - a.hb, a.M), a.bmax);
}
// Same function for mode-0 keys (key, hb < 2^31): max(key, hb) - hb ==
// max(key - hb, 0) in int32, one VIADDMNMX instead of VIMNMX + VIADD.
__device__ __forceinline__ uint32_t bin_of_m0(uint32_t key, const AxisParams& a) {
  return min(__umulhi((uint32_t)max((int32_t)(key - a.hb), 0), a.M), a.bmax);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Directory entry formats (eos_internal.h TablePlan::dir16): a 32-bit entry
// lo | occ << 16 (any table), or a 16-bit entry 8 lo | occ (search tables with
// n <= 8192 and every bin holding <= 7 entries: half the shared memory per bin,
// so twice the bins in the same image).  The 16-bit entry holds the byte offset
// of X[lo] with the occupancy in its three low (alignment) bits, so the entry's
// address is one add away: pa = &X[0] + d - occ.
// Sets pa = shared address of X[lo] and r = occ.
template <bool D16>
__device__ __forceinline__ void dir_entry(const void* __restrict__ sD, uint32_t b, uint32_t xa,
                                          uint32_t& pa, int32_t& r) {
  if (D16) {
    const uint32_t d = reinterpret_cast<const uint16_t*>(sD)[b];
    r = (int32_t)(d & 7u);
    pa = xa + d - (uint32_t)r;
  } else {
    const uint32_t d = reinterpret_cast<const uint32_t*>(sD)[b];
    r = (int32_t)(d >> 16);
    pa = xa + 8u * (d & 0xFFFFu);
  }
}

// One step of binary lifting with stride s over the rest of the bin, on the
// shared-memory byte address pa of the first entry not yet counted
// (X[lo + c]) and the r = occ - c entries that remain:
//   if (r >= s && X[lo + c + s - 1] <= y) { c += s; }
// The probe is an immediate offset from pa and is predicated off (moves no
// smem data) when the bin holds fewer than s more entries; the compare folds
// the range predicate in (DSETP.AND), the updates are predicated: 5 SASS
// instructions per step, 4 for the last one (no r update), no branches.
template <int S, bool LAST>
__device__ __forceinline__ void lift_step(double y, uint32_t& pa, int32_t& r, double& x) {
  // x: the probe register, defined once per lookup (its value is never used when the
  // probe is predicated off: the compare ANDs the range predicate in)
  if (LAST) {
    asm("{\n\t.reg .pred pi, pt;\n\t"
        "setp.ge.s32 pi, %2, %4;\n\t"
        "@pi ld.shared.f64 %1, [%0+%5];\n\t"
        "setp.le.and.f64 pt, %1, %3, pi;\n\t"
        "@pt add.u32 %0, %0, %6;\n\t}"
        : "+r"(pa), "+d"(x)
        : "r"(r), "d"(y), "n"(S), "n"(8 * (S - 1)), "n"(8 * S));
  } else {
    asm("{\n\t.reg .pred pi, pt;\n\t"
        "setp.ge.s32 pi, %1, %4;\n\t"
        "@pi ld.shared.f64 %2, [%0+%5];\n\t"
        "setp.le.and.f64 pt, %2, %3, pi;\n\t"
        "@pt add.u32 %0, %0, %6;\n\t"
        "@pt sub.s32 %1, %1, %4;\n\t}"
        : "+r"(pa), "+r"(r), "+d"(x)
        : "d"(y), "n"(S), "n"(8 * (S - 1)), "n"(8 * S));
  }
}
// the same with a runtime stride (rare branch / runtime-S loop)
__device__ __forceinline__ void lift_step_rt(double y, uint32_t& pa, int32_t& r, int32_t s) {
  asm("{\n\t.reg .pred pi, pt;\n\t.reg .f64 x;\n\t.reg .u32 q;\n\t"
      "setp.ge.s32 pi, %1, %3;\n\t"
      "shl.b32 q, %3, 3;\n\t"
      "add.u32 q, q, %0;\n\t"
      "mov.b64 x, 0;\n\t"
      "@pi ld.shared.f64 x, [q+-8];\n\t"
      "setp.le.and.f64 pt, x, %2, pi;\n\t"
      "@pt mov.u32 %0, q;\n\t"
      "@pt sub.s32 %1, %1, %3;\n\t}"
      : "+r"(pa), "+r"(r)
      : "d"(y), "r"(s));
}

// strides 2^(S-1) .. 1; only the stride-1 step (the last) skips the r update
template <int S>
__device__ __forceinline__ void lift_fixed(double y, uint32_t& pa, int32_t& r) {
  double x = 0.0;
  if (S >= 4) lift_step<8, false>(y, pa, r, x);
  if (S >= 3) lift_step<4, false>(y, pa, r, x);
  if (S >= 2) lift_step<2, false>(y, pa, r, x);
  if (S >= 1) lift_step<1, true>(y, pa, r, x);
}

// The hot per-target body:
//   bin b = min(umulhi(max(key, hb) - hb, M), B-1)          (exponent / log hash)
//   lo, occ = directory[b]                                  (count directory)
//   c = #{j < occ : X[lo + j] <= y}  by binary lifting (branchless steps)
//   idx = (y >= X[0]) ? lo + c - 1 : 0                      (P:54 fix-up; NaN -> 0)
// SF fixed steps (strides 2^(SF-1) .. 1) cover bins of up to 2^SF - 1
// entries.  BIG: the directory also holds deeper bins (up to 2^S - 1
// entries, S = a.steps); their larger strides run first, in a branch that only
// warps with a lane in such a bin take (the planner picks SF so that few warps
// diverge, table_build.cpp choose_layout).  SF = 0: every stride in a runtime
// loop.  Probes past the bin are predicated off, so they move no smem data:
// with fine bins most lanes probe nothing.  (Measured: dropping the occupancy
// test -- NaN-padded X -- is 11% slower on cfg2 and 34% on cfg5.)
// SF <= 4 here (kMaxFastSteps = 3 for search tables; grid axes use S <= 4).
template <int SF, bool BIG, int MODE, bool D16>
__device__ __forceinline__ int32_t lookup_b(double y, const double* __restrict__ sX,
                                            const void* __restrict__ sD, const AxisParams& a) {
  static_assert(SF >= 0 && SF <= 4, "fixed lifting steps");
  const uint32_t key = key_hi<MODE>(y);
  const uint32_t b = MODE == 0 ? bin_of_m0(key, a) : bin_of(key, a);
  EOS_DCHECK(b <= a.bmax);
  const uint32_t xa = smem_u32(sX);
  uint32_t pa;
  int32_t r;
  dir_entry<D16>(sD, b, xa, pa, r);
  EOS_DCHECK((int32_t)((pa - xa) >> 3) + r <= a.n && r < (1 << a.steps));
  if (SF == 0) {
    for (int32_t s = 1 << (a.steps - 1); s > 0; s >>= 1) lift_step_rt(y, pa, r, s);
  } else {
    if (BIG && r >= (1 << SF)) {  // rare: a bin deeper than the fixed steps
      for (int32_t s = 1 << (a.steps - 1); s >= (1 << SF); s >>= 1) lift_step_rt(y, pa, r, s);
    }
    lift_fixed<SF>(y, pa, r);
  }
  const int32_t idx = (int32_t)(pa - xa - 8u) >> 3;  // lo + c - 1
  return (y >= a.x0) ? idx : 0;
}

// S fixed steps (S = 0: runtime), 32-bit directory (grid axes, tiered sample
// tables, counters launches)
template <int S, int MODE>
__device__ __forceinline__ int32_t lookup(double y, const double* __restrict__ sX,
                                          const uint32_t* __restrict__ sD, const AxisParams& a) {
  return lookup_b<S, false, MODE, false>(y, sX, sD, a);
}

struct Counters {
  uint64_t c[7];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 7; ++i) c[i] = 0;
  }
  __device__ __forceinline__ void add(double y, int32_t idx, int64_t gpos, double x_idx,
                                      const AxisParams& a) {
    c[0] += 1;
    c[1] += (uint64_t)(uint32_t)idx;
    c[2] += mix64(mix64((uint64_t)gpos) ^ (uint64_t)(uint32_t)idx);  // DESIGN.md R25
    c[3] += !(y >= a.x0);
    c[4] += (y > a.xlast);
    c[5] += (y != y);
    c[6] += (y == x_idx);
  }
  __device__ __forceinline__ void flush(unsigned long long* g) {
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      uint64_t v = c[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
      if ((threadIdx.x & 31) == 0 && v) atomicAdd(g + i, (unsigned long long)v);
    }
  }
};

// Lookup policies of the streaming tile loop (search_body).  `many` maps the
// 2U targets of one thread's tile slice to their indices, `x_at(i)` = X[i]
// (counter c6 only).
//
// SmemLookup: the whole table and its directory are in shared memory.
template <int SF, bool BIG, int MODE, bool D16>
struct SmemLookup {
  static constexpr bool kBatchTail = true;  // ragged tiles: one batched lookup per thread
  static constexpr bool kEarlyLoad = true;  // static schedule: next tile's loads first
  const double* __restrict__ sX;
  const void* __restrict__ sD;
  AxisParams a;
  template <int N>
  __device__ __forceinline__ void many(const double (&y)[N], int32_t (&r)[N]) const {
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = lookup_b<SF, BIG, MODE, D16>(y[i], sX, sD, a);
  }
  __device__ __forceinline__ double x_at(int32_t i) const { return sX[i]; }
};

// Read-once target stream: 128-bit evict-first loads.  (A/B, DESIGN.md §12:
// the L2 256-byte prefetch hint and 256-bit loads / 128-bit stores per thread
// were within +-1.5%.)
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }

// One 32-byte sector with one 256-bit load (SASS LDG.E.NA.ENL2.256): one
// L1TEX wavefront per lane -- the gathers of a warp hit 32 different lines,
// so wavefronts, not bytes, bound the L1 stage.  L1::no_allocate: the levels
// are too large to live in L1 (measured faster than allocating).
__device__ __forceinline__ void ldg_keys8(const uint32_t* p, uint32_t (&k)[8]) {
  asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(k[0]), "=r"(k[1]), "=r"(k[2]), "=r"(k[3]), "=r"(k[4]), "=r"(k[5]), "=r"(k[6]),
        "=r"(k[7])
      : "l"(p));
}
__device__ __forceinline__ void ldg_f64x4(const double* p, double& a, double& b, double& c,
                                          double& d) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
      : "l"(p));
}

// TieredLookup (tables larger than shared memory): the smem
// table is the sample T1[j] = X[j 8^D] (n1 entries, as 32-bit keys:
// lookup_keys) with its directory; the
// full table lives in global memory (L2-resident) as D 8-ary levels, level d
// holding F_d[j] = X[j 8^d] (NaN past n) and their keys K_d[j] =
// key_hi(F_d[j]) (0xFFFFFFFF past n).  Per target:
//   b = max(#{T1 <= y} - 1, 0)                      (smem lookup, as above)
//   for d = D-1 .. 0:  node = K_d[8b .. 8b+8)         (one 32-B sector)
//     c = #{t : node[t] < key(y)}                      (key order = value order)
//     if some node[t] == key(y): c = #{t : F_d[8b+t] <= y}   (exact; rare)
//     b = 8b + max(c - 1, 0)
//   idx = (y >= X[0]) ? b : 0
// key_hi is the upper word of an order-preserving map of the fp64 bits, so
// key(X) < key(y) implies X < y and key(X) > key(y) implies X > y; only
// equal keys need the fp64 values.  Invariant: X[b 8^(d+1)] <= y <
// X[(b+1) 8^(d+1)] (or past the end), so c >= 1 for every y >= X[0].  At
// d = 0 the stride is 1 and b = #{X <= y} - 1.  All targets of a
// thread go through a level together so their sector loads overlap.
// The shared-memory sample table of a tiered table holds the 32-bit keys of
// T1 (4 B per entry, so up to 32768 entries fit), binned by the same hash.
// Lifting counts the bin's keys < key(y) -- key order is value order -- and
// the (rare) entries whose key equals key(y) are settled exactly from their
// fp64 values, T1[j] = F_{D-1}[8 j] in global memory.
template <int S, int MODE>
__device__ __forceinline__ int32_t lookup_keys(double y, uint32_t ky,
                                               const uint32_t* __restrict__ sK,
                                               const uint32_t* __restrict__ sD,
                                               const AxisParams& a,
                                               const double* __restrict__ ftop) {
  const uint32_t b = MODE == 0 ? bin_of_m0(ky, a) : bin_of(ky, a);
  EOS_DCHECK(b <= a.bmax);
  const uint32_t d = sD[b];
  const int32_t lo = (int32_t)(d & 0xFFFFu);
  const int32_t occ = (int32_t)(d >> 16);
  EOS_DCHECK(lo + occ <= a.n && occ < (1 << (S > 0 ? S : a.steps)));
  int32_t c = 0;
  if (S > 0) {
#pragma unroll
    for (int s = 1 << (S > 0 ? S - 1 : 0); s > 0; s >>= 1) {
      const int32_t j = c + s;
      if (j <= occ) {
        if (sK[lo + j - 1] < ky) c = j;
      }
    }
  } else {
    for (int s = 1 << (a.steps - 1); s > 0; s >>= 1) {
      const int32_t j = c + s;
      if (j <= occ) {
        if (sK[lo + j - 1] < ky) c = j;
      }
    }
  }
  if (c < occ && sK[lo + c] == ky) {
    // Equal keys (rare): binary lifting over the rest of the bin with the
    // exact values.  "key == key(y) and X <= y" holds on a prefix of it (the
    // equal keys come first, sorted by value; larger keys hold larger values).
    for (int32_t st = 1 << (31 - __clz(occ - c)); st > 0; st >>= 1) {
      const int32_t j = c + st;
      if (j <= occ && sK[lo + j - 1] == ky && __ldg(ftop + 8 * (int64_t)(lo + j - 1)) <= y) c = j;
    }
  }
  return (y >= a.x0) ? (lo + c - 1) : 0;
}

template <int S, int MODE>
struct TieredLookup {
  static constexpr bool kBatchTail = false;  // (batching the tail made the kernel spill)
  static constexpr bool kEarlyLoad = false;  // (n = 2^18: 185 -> 181; D = 2: +1.3%)
  const uint32_t* __restrict__ sK;  // keys of T1 (smem)
  const uint32_t* __restrict__ sD;
  AxisParams a;                   // of T1, except xlast = X[n-1] (counter c4)
  const double* __restrict__ lv;  // F level D-1 (global)
  const uint32_t* __restrict__ kv;  // K level D-1 (global)
  int64_t top_len;                // 8 n1
  int32_t levels;                 // D >= 1
  const double* __restrict__ x_full;  // F level 0 = X (counter c6)
  template <int N>
  __device__ __forceinline__ void many(const double (&y)[N], int32_t (&r)[N]) const {
    int32_t b[N];
    uint32_t ky[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      ky[i] = key_hi<MODE>(y[i]);
      b[i] = lookup_keys<S, MODE>(y[i], ky[i], sK, sD, a, lv);
    }
    const double* F = lv;
    const uint32_t* K = kv;
    int64_t len = top_len;
    for (int d = levels - 1; d >= 0; --d) {
      uint32_t k[N][8];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        EOS_DCHECK(b[i] >= 0 && 8 * (int64_t)b[i] + 7 < len);
        ldg_keys8(K + 8 * (int64_t)b[i], k[i]);
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        int32_t c = 0;
        bool tie = false;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          c += k[i][t] < ky[i];
          tie |= k[i][t] == ky[i];
        }
        if (tie) {  // exact count from the fp64 node (two sectors)
          const double* f = F + 8 * (int64_t)b[i];
          double v[8];
          ldg_f64x4(f, v[0], v[1], v[2], v[3]);
          ldg_f64x4(f + 4, v[4], v[5], v[6], v[7]);
          c = 0;
#pragma unroll
          for (int t = 0; t < 8; ++t) c += v[t] <= y[i];
        }
        b[i] = 8 * b[i] + max(c - 1, 0);
      }
      F += len;
      K += len;
      len *= 8;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = (y[i] >= a.x0) ? b[i] : 0;
  }
  __device__ __forceinline__ double x_at(int32_t i) const { return __ldg(x_full + i); }
};

// PackedLookup (packed tables, eossearch.h EOS_LEVELS_PACKED; layout in
// eos_internal.h PackedPlan): ONE L2 sector per lookup.  Per target:
//   sample (smem): u = max(key, hb) - hb, bin b = min(u >> sh, bmax), rk = the
//     16 bits of key64 - (hb << 32) below the bin bits (0xFFFF past the last
//     bin); lifting counts the bin's residuals <= rk, a run equal to rk settled
//     from X[15 j] (global); j = max(#{T1 <= y} - 1, 0)
//   node j (one 32-B sector, ld.global.nc, L1 no-allocate): B | s, r_1..r_14;
//     ry = min((max(key64, B << 32) - (B << 32)) >> s, 0x77FF); the residuals are sorted, so
//     lt = #{r_t < ry} and le = #{r_t <= ry} (fp16x2 compares of the biased
//     values, 14 at a time in 7 HSET2 each) bound the run of equal residuals,
//     settled from X[15 j + t] (rare)
//   idx = (y >= X[0]) ? 15 j + lt + #{ties <= y} : 0
// Invariant: X[15 j] <= y < X[15 (j + 1)] for X[0] <= y, so the node's first
// entry counts and idx = #{X <= y} - 1.
// Node residuals are stored biased by kResBias (the smallest normal fp16) so
// that two of them compare as one fp16x2 (HSET2): every stored value is a
// normal positive half or +inf (0x7C00, past the end), whose bit order is its
// value order.  eos_internal.h kPackedResMax / kPackedResBias.
constexpr int kPackedMaxDepthDev = 4;  // eos_internal.h kPackedMaxDepth
constexpr uint32_t kResMax = 0x77FFu;
constexpr uint32_t kResBias = 0x0400u;
__device__ __forceinline__ __half2 u32_as_h2(uint32_t w) {
  __half2 h;
  memcpy(&h, &w, 4);
  return h;
}
__device__ __forceinline__ uint32_t h2_as_u32(__half2 h) {
  uint32_t w;
  memcpy(&w, &h, 4);
  return w;
}

template <int S, int MODE, bool ML>
struct PackedLookup {
  static constexpr bool kBatchTail = false;
  static constexpr bool kEarlyLoad = true;
  const uint16_t* __restrict__ sR;  // sample residuals (smem)
  const uint32_t* __restrict__ sD;  // directory, one u32 per bin pair (smem)
  const int32_t* __restrict__ sL;   // level table (smem): first node of level d [0..3], 15^d [4..7]
  AxisParams a;                     // n = n1; hb, bmax of the sample hash; x0, xlast of X
  uint32_t sh;
  int32_t depth;                    // D levels of nodes; T1[j] = X[15^D j]
  const double* __restrict__ X;       // the table (global)
  const uint32_t* __restrict__ nodes;  // 8 words per node (global, 32-B aligned)

  // Sample lookups of N targets, step-major (the N lifting chains interleave).
  // Lifting counts the residuals <= rk and keeps the last one it accepted, which
  // is the bin's entry c - 1: equal to rk only when a run of equal residuals
  // may hold entries > y.  That run is settled after all chains, from its end,
  // in a branch taken rarely (no extra shared load on the common path).
  template <int N>
  __device__ __forceinline__ void sample(const double (&y)[N], const uint32_t (&ky)[N],
                                         int32_t (&j)[N]) const {
    uint32_t rk[N], last[N];
    int32_t lo[N], occ[N], c[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint32_t u =
          MODE == 0 ? (uint32_t)max((int32_t)(ky[i] - a.hb), 0) : max(ky[i], a.hb) - a.hb;
      const uint32_t q = u >> sh;
      const uint32_t b = min(q, a.bmax);
      // (u : low word of key64) >> (16 + sh), the low word 0 below hb
      const uint32_t lw = ky[i] >= a.hb ? (uint32_t)key64<MODE>(y[i]) : 0u;
      rk[i] = q > a.bmax ? 0xFFFFu : (__funnelshift_rc(lw, u, 16u + sh) & 0xFFFFu);
      // one u32 entry per bin pair: lo(pair) | occ(even bin) << 20 | occ(odd bin) << 26
      const uint32_t d = sD[b >> 1];
      const uint32_t o0 = (d >> 20) & 63u;
      lo[i] = (int32_t)((d & 0xFFFFFu) + ((b & 1u) ? o0 : 0u));
      occ[i] = (int32_t)((b & 1u) ? (d >> 26) : o0);
      c[i] = 0;
      last[i] = 0xFFFFFFFFu;
      EOS_DCHECK(lo[i] + occ[i] <= a.n && occ[i] < (1 << S));
    }
#pragma unroll
    for (int s = 1 << (S - 1); s > 0; s >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int32_t t = c[i] + s;
        const uint32_t v = t <= occ[i] ? (uint32_t)sR[lo[i] + t - 1] : 0xFFFFFFFFu;
        if (v <= rk[i]) {
          c[i] = t;
          last[i] = v;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (last[i] == rk[i]) {
        // entries lo .. lo + c - 1 are <= rk and the run of residuals == rk ends
        // at c - 1; its entries > y (fp64) form the run's tail
        while (c[i] > 0 && sR[lo[i] + c[i] - 1] == rk[i] &&
               !(__ldg(X + 15 * (ML ? (int64_t)sL[kPackedMaxDepthDev + depth - 1] : 1) *
                               (int64_t)(lo[i] + c[i] - 1)) <= y[i]))
          --c[i];
      }
      j[i] = max(lo[i] + c[i] - 1, 0);
    }
  }

  template <int N>
  __device__ __forceinline__ void many(const double (&y)[N], int32_t (&r)[N]) const {
    int32_t j[N];
    uint32_t ky[N];
#pragma unroll
    for (int i = 0; i < N; ++i) ky[i] = key_hi<MODE>(y[i]);
    sample(y, ky, j);
    // levels D-1 .. 0 (first node, entry stride 15^d from the image's level table);
    // ML = false: one level, no loop (the loop costs one-level tables 2%)
    if constexpr (ML) {
#pragma unroll 1
      for (int d = depth - 1; d >= 0; --d) level<N>(d, y, j);
    } else {
      EOS_DCHECK(depth == 1);
      level<N>(0, y, j);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) r[i] = (y[i] >= a.x0) ? j[i] : 0;
  }
  // One level d: j (nodes of level d) -> 15 j + #{entries of the node <= y} (nodes of
  // level d - 1; at d = 0 the index).
  template <int N>
  __device__ __forceinline__ void level(int d, const double (&y)[N], int32_t (&j)[N]) const {
    uint32_t k[N][8];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      EOS_DCHECK(j[i] >= 0 && (d < depth - 1 || j[i] < a.n));
      ldg_keys8(nodes + 8 * (int64_t)((ML ? sL[d] : 0) + j[i]), k[i]);
    }
    int32_t lt[N], le[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint64_t B = (uint64_t)(k[i][0] & ~63u) << 32;
      const uint32_t s = k[i][0] & 63u;
      const uint64_t k64 = key64<MODE>(y[i]);
      const uint32_t ry = (uint32_t)min((max(k64, B) - B) >> s, (uint64_t)kResMax) + kResBias;
      const __half2 hy = u32_as_h2(ry * 0x10001u);
      // lane sums start at 512 (ulp 0.5) so the final 1024 + count is exact
      __half2 a = u32_as_h2(0x60006000u), e = a;
#pragma unroll
      for (int w = 1; w < 8; ++w) {
        a = __hadd2(a, __hlt2(u32_as_h2(k[i][w]), hy));
        e = __hadd2(e, __hle2(u32_as_h2(k[i][w]), hy));
      }
      const uint32_t t = h2_as_u32(__hadd2(__lows2half2(a, e), __highs2half2(a, e)));
      lt[i] = (int32_t)(t & 0xFFFFu) - 0x6400;  // 1024.0 = 0x6400, ulp 1
      le[i] = (int32_t)(t >> 16) - 0x6400;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      int32_t cnt = lt[i];
      if (le[i] > lt[i]) {  // equal residuals (rare): the fp64 values of the run
        const int64_t stride = ML ? sL[kPackedMaxDepthDev + d] : 1;  // 15^d
        const double* f = X + stride * (15 * (int64_t)j[i] + 1);
#pragma unroll 1
        for (int32_t e = lt[i]; e < le[i]; ++e) cnt += __ldg(f + stride * e) <= y[i];
      }
      j[i] = 15 * j[i] + cnt;
    }
  }
  __device__ __forceinline__ double x_at(int32_t i) const { return __ldg(X + i); }
};

// ---- Blackwell cluster launch control + mbarrier (inline PTX, sm_100a) ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Wait for the phase of `bar` with parity `parity`.  try_wait suspends the
// thread until the phase completes or the suspend-time hint (ns) runs out, so
// waiting warps leave their issue slots to working ones instead of spinning.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!ok);
}
// Ask the hardware scheduler to cancel a not-yet-launched CTA of this grid;
// the 16-byte response lands in `resp` and completes `bar`.
__device__ __forceinline__ void clc_try_cancel(uint4* resp, uint64_t* bar) {
  asm volatile(
      "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];"
      ::"r"(smem_u32(resp)), "r"(smem_u32(bar))
      : "memory");
}
// Decode the response: returns the canceled CTA's blockIdx.x, or -1.
__device__ __forceinline__ int64_t clc_query(const uint4* resp) {
  uint32_t valid = 0, x = 0;
  asm volatile(
      "{\n\t.reg .b128 R;\n\t.reg .pred P;\n\t"
      "ld.shared.b128 R, [%2];\n\t"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 P, R;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t"
      "@P clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, R;\n\t}"
      : "=r"(valid), "=r"(x)
      : "r"(smem_u32(resp))
      : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  return valid ? (int64_t)x : -1;
}

// TMA 1-D bulk prefetch of [src, src + bytes) into L2 (16-B aligned, bytes a
// multiple of 16): no registers, no completion to wait for.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// TMA 1-D bulk copy global -> this CTA's shared memory, completing on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Stage the device image (L2-resident after the first CTA) into shared
// memory with TMA bulk copies (one thread issues them; everyone waits on the
// mbarrier).  SASS: UBLKCP.S.G + SYNCS.  All threads return with the image
// visible.  `bar` is single-use (phase 0).
__device__ __forceinline__ void stage_image(uint4* smem, const uint4* __restrict__ img, int n16,
                                            uint64_t* bar) {
  const uint32_t bytes = (uint32_t)n16 * 16u;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_arrive_expect_tx(bar, bytes);
    for (uint32_t off = 0; off < bytes; off += 32768u)
      bulk_g2s(reinterpret_cast<char*>(smem) + off, reinterpret_cast<const char*>(img) + off,
               min(32768u, bytes - off), bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
}

// Programmatic dependent launch (PDL): the part of a kernel before this call
// (CTA launch, barrier init, smem image staging -- none of it touches memory
// other kernels write) may overlap the tail of the previous kernel in the
// stream; every access to the caller's buffers comes after it.  Then let the
// next PDL launch in the stream start its own prologue.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Launch shape of search1d (compile-time): threads per CTA, double2 loads in
// flight per thread per tile, min resident CTAs per SM (register cap:
// 65536 / (THREADS*MINB) per thread), and the tile schedule:
// CLC = work stealing via cluster launch control over a one-CTA-per-tile
// grid; otherwise a static grid-stride loop over a persistent grid.
template <int THREADS, int UNROLL, int MINB, bool CLC>
struct Shape {
  static constexpr int kThreads = THREADS;
  static constexpr int kUnroll = UNROLL;
  static constexpr int kMinBlocks = MINB;
  static constexpr bool kClc = CLC;
  static constexpr int kTilePairs = THREADS * UNROLL;
  static constexpr int kTileElems = 2 * THREADS * UNROLL;
};
// Short in-bin searches (S <= 2) are HBM-bound: CLC tiles (measured best).
// Long ones (S >= 3) are smem/issue-bound: there the per-tile CTA barrier of
// the CLC loop costs more than the static schedule's tail.
using ShapeSmall = Shape<256, 4, 4, true>;      // image <= 32 KB: 4 CTAs x 256 threads per SM
using ShapeMid = Shape<512, 4, 2, true>;        // image <= 72 KB: 2 CTAs x 512
using ShapeDeepMid = Shape<512, 4, 2, false>;   // S >= 3, image <= 72 KB
using ShapeDeepBig = Shape<1024, 4, 1, false>;  // S >= 3, larger
using ShapeCnt = Shape<256, 4, 1, true>;        // validation launches (counters on)
// Tiered tables: 1024 threads x 4 level-major lookup chains, static
// schedule (profiles/r01_exp_tiered.json).
using ShapeTiered = Shape<1024, 2, 1, false>;

// The streaming tile loop of search1d (after the image is in smem): CLC or
// static tile schedule, 128-bit streaming loads, next-tile prefetch.  Full
// tiles (vector body) use pointer increments (static) or one multiply-add
// (CLC) per tile; ragged / unaligned tiles take the batched scalar path.  The
// unaligned leading element (args.head) goes with tile 0, in whichever CTA
// processes it (under CLC a not-yet-launched CTA 0 may be cancelled).
template <bool CNT, class SH, class LK>
__device__ __forceinline__ void search_body(const SearchArgs& args, const LK& lk, uint4* clc_resp_p,
                                            uint64_t* clc_bar_p) {
  const AxisParams& a = lk.a;
  constexpr int T = SH::kThreads;
  constexpr int U = SH::kUnroll;
  constexpr int TP = SH::kTilePairs;
  constexpr int TE = SH::kTileElems;
  static_assert(TE == 2 * U * T, "tile = 2U elements per thread");
  uint4& clc_resp = *clc_resp_p;
  uint64_t& clc_bar = *clc_bar_p;
  const double* __restrict__ Y = args.Y;
  int32_t* __restrict__ out = args.out;
  const int64_t count = args.count;
  const int64_t head = args.head;
  const int64_t body = count - head;
  const int64_t ntiles = args.ntiles;
  const int64_t nfull = args.vec_ok ? body / TE : 0;  // tiles of the vector body
  const double2* __restrict__ Y2 = reinterpret_cast<const double2*>(Y + head);
  int2* __restrict__ O2 = reinterpret_cast<int2*>(out + head);

  Counters cn;
  if (CNT) cn.zero();

  auto do_head = [&]() {  // the leading unaligned element (tile 0's)
    if (threadIdx.x == 0 && head) {
      const double y[1] = {Y[0]};
      int32_t r[1];
      lk.many(y, r);
      out[0] = r[0];
      if (CNT) cn.add(y[0], r[0], args.gofs, lk.x_at(r[0]), a);
    }
  };
  // full tile: 2U targets per thread, loaded into v before the call
  auto compute = [&](const double2 (&v)[U], int2 (&r)[U], int64_t t) {
    double y[2 * U];
    int32_t ri[2 * U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      y[2 * u] = v[u].x;
      y[2 * u + 1] = v[u].y;
    }
    lk.many(y, ri);
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = make_int2(ri[2 * u], ri[2 * u + 1]);
    if (CNT) {
      const int64_t p0 = t * TP + threadIdx.x;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t g = args.gofs + head + 2 * (p0 + u * T);
        cn.add(v[u].x, r[u].x, g, lk.x_at(r[u].x), a);
        cn.add(v[u].y, r[u].y, g + 1, lk.x_at(r[u].y), a);
      }
    }
  };
  // ragged / unaligned tile: each thread's (at most 2U) elements at stride T,
  // all loads first and one batched lookup, as in the vector body (a
  // one-at-a-time loop here waited a load latency per element)
  auto ragged = [&](int64_t t) {
    const int64_t e0 = head + t * TE;
    const int64_t e1 = min(count, e0 + TE);
    EOS_DCHECK(e0 >= 0 && t >= 0);
    if (!CNT && LK::kBatchTail) {
      double y[2 * U];
      int32_t r[2 * U];
#pragma unroll
      for (int k = 0; k < 2 * U; ++k) {
        const int64_t i = e0 + threadIdx.x + (int64_t)k * T;
        y[k] = i < e1 ? Y[i] : 0.0;
      }
      lk.many(y, r);
#pragma unroll
      for (int k = 0; k < 2 * U; ++k) {
        const int64_t i = e0 + threadIdx.x + (int64_t)k * T;
        if (i < e1) out[i] = r[k];
      }
    } else {  // counters / tiered tables: one element at a time (fewer live registers)
      for (int64_t i = e0 + threadIdx.x; i < e1; i += T) {
        const double y[1] = {Y[i]};
        int32_t r[1];
        lk.many(y, r);
        out[i] = r[0];
        if (CNT) cn.add(y[0], r[0], args.gofs + i, lk.x_at(r[0]), a);
      }
    }
  };
  if (!SH::kClc) {
    // static persistent schedule: tiles blockIdx.x + k gridDim.x, pointers advance
    // by gridDim.x tiles; the next tile's loads go out before this tile's stores
    int64_t t = blockIdx.x;
    if (t == 0) do_head();
    const int64_t step = (int64_t)gridDim.x * TP;
    const double2* yp = Y2 + t * TP + threadIdx.x;
    int2* op = O2 + t * TP + threadIdx.x;
    double2 v[U];
    if (t < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_stream(yp + u * T);
    }
    for (; t < nfull; t += gridDim.x) {
      int2 r[U];
      if constexpr (!CNT && LK::kEarlyLoad) {
        // the next tile's loads go out before this tile's lookups (a whole tile of
        // lookups to cover their latency, not just the stores); v is copied first.
        // Packed tables 191 -> 211 Glookups/s; single-level tables +1.5%; 8-ary
        // levels mixed
        double2 w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) w[u] = v[u];
        yp += step;
        if (t + gridDim.x < nfull) {
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = ld_stream(yp + u * T);
        }
        compute(w, r, t);
      } else {
      compute(v, r, t);
      yp += step;
      if (t + gridDim.x < nfull) {
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(yp + u * T);
      }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) __stcs(op + u * T, r[u]);
      op += step;
    }
    for (; t < ntiles; t += gridDim.x) ragged(t);
  } else {
    // CLC: this CTA's own tile, then tiles of cancelled (not yet launched) CTAs
    uint32_t phase = 0;
    int64_t t = blockIdx.x;
    if (ntiles == 0 && t == 0) do_head();
    double2 v[U];
    if (t < nfull) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_stream(Y2 + t * TP + threadIdx.x + u * T);
    }
    while (t < ntiles) {
      if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&clc_bar, 16);
        clc_try_cancel(&clc_resp, &clc_bar);
      }
      if (t == 0) do_head();
      int2 r[U];
      const bool f = t < nfull;
      if (f) compute(v, r, t);
      else ragged(t);
      mbar_wait(&clc_bar, phase);
      phase ^= 1u;
      const int64_t q = clc_query(&clc_resp);
      __syncthreads();  // everyone has read the response before it is reused
      const int64_t tn = q < 0 ? ntiles : q;
      if (tn < nfull) {  // before this tile's stores
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(Y2 + tn * TP + threadIdx.x + u * T);
      }
      if (f) {
        int2* op = O2 + t * TP + threadIdx.x;
#pragma unroll
        for (int u = 0; u < U; ++u) __stcs(op + u * T, r[u]);
      }
      t = tn;
    }
  }
  if (CNT) cn.flush(args.counters);
}

template <int SF, bool BIG, int MODE, bool D16, bool CNT, class SH>
__global__ void __launch_bounds__(SH::kThreads, SH::kMinBlocks) search1d_kernel(const SearchArgs args) {
  extern __shared__ __align__(128) uint4 smem[];
  __shared__ __align__(16) uint4 clc_resp;
  __shared__ __align__(8) uint64_t clc_bar, stage_bar;
  if (SH::kClc && threadIdx.x == 0) mbar_init(&clc_bar, 1);
  stage_image(smem, args.image, args.image_16, &stage_bar);
  pdl_enter();
  const AxisParams a = args.ax;
  EOS_DCHECK(a.d_off + (D16 ? 2 : 4) * ((int64_t)a.bmax + 1) <= 16 * (int64_t)args.image_16 &&
             a.x_off + 8 * (int64_t)a.n <= a.d_off);
  SmemLookup<SF, BIG, MODE, D16> lk;
  lk.sX = reinterpret_cast<const double*>(reinterpret_cast<const char*>(smem) + a.x_off);
  lk.sD = reinterpret_cast<const char*>(smem) + a.d_off;
  lk.a = a;
  search_body<CNT, SH>(args, lk, &clc_resp, &clc_bar);
}

// ---- streaming through a shared-memory ring (TMA bulk copies) ----------------
// The grid has one CTA per tile of 31 x 32 x PL targets; a resident CTA (one per SM,
// 1024 threads) keeps its staged image and takes over the tiles of CTAs that have
// not launched yet with cluster launch control, so tiles are processed in launch
// order.  Warp 31 is the producer: one elected lane claims the tiles (its own,
// then cancelled CTAs') and streams each into the next of NS shared-memory stages
// with cp.async.bulk (L2 evict-first: read once), completing on the stage's `full`
// mbarrier, the tile number in a shared slot.  Warps 0..30 consume: wait `full`,
// read their 128 targets (two conflict-free 16-byte loads per lane), release the
// stage (`empty`, one arrival per warp), look the targets up and store the int32
// indices with st.global.cs.  No CTA-wide barrier in the loop, and the loads in
// flight (up to NS stages) hold no registers.
// Measured on the same-mix stream (measure/probes.cu): a static
// persistent schedule reaches 6.35 TB/s with register prefetch and 6.63 with this
// ring, one CTA per tile 7.17, this ring with launch-order tiles 7.14: DRAM
// bandwidth follows the compactness of the address front, not the bytes in flight.
constexpr int kRingWarps = 31;                  // consumer warps
// targets per lane per stage: PL (template) = 4 or 8; a stage is 31 x 32 x PL targets
constexpr int kRingMaxStages = 6;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int PL, class LK>
__device__ __forceinline__ void ring_body(const SearchArgs& args, const LK& lk, double* ring,
                                          uint64_t* full, uint64_t* empty, int64_t* tile_of,
                                          uint4* clc_resp, uint64_t* clc_bar) {
  constexpr int ST = kRingWarps * 32 * PL;  // targets per stage
  const int NS = args.ring_ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* __restrict__ Y = args.Y;
  int32_t* __restrict__ out = args.out;
  const int64_t count = args.count;
  const int64_t head = args.head;
  const int64_t body = (count - head) & ~int64_t(1);  // even: whole 16-B pairs
  if (warp == kRingWarps) {  // producer
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int64_t t = blockIdx.x;
      uint32_t cph = 0, eph = 1;  // phases of the CLC barrier and of the empty barriers
      for (int k = 0, s = 0;; ++k) {
        if (k >= NS) mbar_wait(&empty[s], eph);
        tile_of[s] = t;
        if (t < 0) {  // no tile left: the stage carries the end mark
          mbar_arrive(&full[s]);
          break;
        }
        const int64_t e0 = t * ST;
        const uint32_t bytes = (uint32_t)(8 * min((int64_t)ST, body - e0));
        mbar_arrive_expect_tx(&full[s], bytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(ring + (size_t)s * ST)), "l"(Y + head + e0),
            "r"(bytes), "r"(smem_u32(&full[s])), "l"(pol)
            : "memory");
        mbar_arrive_expect_tx(clc_bar, 16);
        clc_try_cancel(clc_resp, clc_bar);
        mbar_wait(clc_bar, cph);
        cph ^= 1u;
        t = clc_query(clc_resp);
        if (++s == NS) {
          s = 0;
          eph ^= 1u;
        }
      }
    }
    return;
  }
  uint32_t fph = 0;  // phase of the full barriers
  for (int s = 0;;) {
    mbar_wait(&full[s], fph);
    const int64_t t = tile_of[s];
    if (t < 0) break;
    const double2* st = reinterpret_cast<const double2*>(ring + (size_t)s * ST + warp * 32 * PL);
    double y[PL];
#pragma unroll
    for (int h = 0; h < PL / 2; ++h) {
      const double2 v = st[32 * h + lane];
      y[2 * h] = v.x;
      y[2 * h + 1] = v.y;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // the stage's targets are in registers
    if (++s == NS) {
      s = 0;
      fph ^= 1u;
    }
    if (t == 0 && threadIdx.x == 0) {  // the scalar ends go with tile 0
      if (head) {
        const double y1[1] = {Y[0]};
        int32_t r1[1];
        lk.many(y1, r1);
        out[0] = r1[0];
      }
      if (head + body < count) {
        const double y1[1] = {Y[count - 1]};
        int32_t r1[1];
        lk.many(y1, r1);
        out[count - 1] = r1[0];
      }
    }
    int32_t r[PL];
    lk.many(y, r);
    const int64_t e0 = t * ST + warp * 32 * PL;  // first target of this warp's slice
    int2* o = reinterpret_cast<int2*>(out + head + e0);
    if (e0 + 32 * PL <= body) {
#pragma unroll
      for (int h = 0; h < PL / 2; ++h) __stcs(o + 32 * h + lane, make_int2(r[2 * h], r[2 * h + 1]));
    } else {  // the last tile
#pragma unroll
      for (int h = 0; h < PL / 2; ++h)
        if (e0 + 64 * h + 2 * lane < body) __stcs(o + 32 * h + lane, make_int2(r[2 * h], r[2 * h + 1]));
    }
  }
}

template <int SF, bool BIG, int MODE, bool D16, int PL>
__global__ void __launch_bounds__(1024, 1) search1d_ring_kernel(const SearchArgs args) {
  extern __shared__ __align__(128) uint4 smem[];
  __shared__ __align__(8) uint64_t full[kRingMaxStages], empty[kRingMaxStages], stage_bar, clc_bar;
  __shared__ __align__(16) uint4 clc_resp;
  __shared__ int64_t tile_of[kRingMaxStages];
  EOS_DCHECK(args.ring_ns >= 2 && args.ring_ns <= kRingMaxStages);
  if (threadIdx.x == 0) {
    for (int s = 0; s < args.ring_ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kRingWarps);
    }
    mbar_init(&clc_bar, 1);
  }
  stage_image(smem, args.image, args.image_16, &stage_bar);  // (its barrier orders the inits)
  pdl_enter();
  const AxisParams a = args.ax;
  SmemLookup<SF, BIG, MODE, D16> lk;
  lk.sX = reinterpret_cast<const double*>(reinterpret_cast<const char*>(smem) + a.x_off);
  lk.sD = reinterpret_cast<const char*>(smem) + a.d_off;
  lk.a = a;
  double* ring = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) +
                                           ((16 * (size_t)args.image_16 + 127) & ~size_t(127)));
  ring_body<PL>(args, lk, ring, full, empty, tile_of, &clc_resp, &clc_bar);
}

// Tables larger than shared memory (TieredLookup): the smem image holds the
// sample table T1 and its directory; the levels stay in global memory / L2.
template <int S, int MODE, bool CNT, class SH>
__global__ void __launch_bounds__(SH::kThreads, SH::kMinBlocks)
    search1d_tiered_kernel(const SearchArgs args) {
  extern __shared__ __align__(128) uint4 smem[];
  __shared__ __align__(16) uint4 clc_resp;
  __shared__ __align__(8) uint64_t clc_bar, stage_bar;
  if (SH::kClc && threadIdx.x == 0) mbar_init(&clc_bar, 1);
  stage_image(smem, args.image, args.image_16, &stage_bar);
  pdl_enter();
  const AxisParams a = args.ax;
  EOS_DCHECK(args.levels >= 1 && args.lv_top_len == 8 * (int64_t)a.n);
  TieredLookup<S, MODE> lk;
  lk.sK = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(smem) + a.x_off);
  lk.sD = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(smem) + a.d_off);
  lk.a = a;
  lk.lv = args.lv;
  lk.kv = args.kv;
  lk.top_len = args.lv_top_len;
  lk.levels = args.levels;
  // F level 0 (= X) follows levels D-1 .. 1: offset n1 (8^D - 8) / 7
  int64_t off = 0, len = args.lv_top_len;
  for (int d = args.levels - 1; d > 0; --d) {
    off += len;
    len *= 8;
  }
  lk.x_full = args.lv + off;
  search_body<CNT, SH>(args, lk, &clc_resp, &clc_bar);
}

// Packed tables (PackedLookup): the smem image holds the sample residuals and
// their directory; X and the nodes stay in global memory / L2.
template <int S, int MODE, bool CNT, class SH, bool ML = true>
__global__ void __launch_bounds__(SH::kThreads, SH::kMinBlocks)
    search1d_packed_kernel(const SearchArgs args) {
  extern __shared__ __align__(128) uint4 smem[];
  __shared__ __align__(16) uint4 clc_resp;
  __shared__ __align__(8) uint64_t clc_bar, stage_bar;
  if (SH::kClc && threadIdx.x == 0) mbar_init(&clc_bar, 1);
  stage_image(smem, args.image, args.image_16, &stage_bar);
  pdl_enter();
  const AxisParams a = args.ax;
  EOS_DCHECK(args.levels >= 1 && args.levels <= kPackedMaxDepthDev && args.sh >= 1 && args.sh <= 16 &&
             a.d_off + 4 * ((((int64_t)a.bmax + 2) / 2 + 3) & ~int64_t(3)) + 32 <=
                 16 * (int64_t)args.image_16 &&
             2 * (int64_t)a.n <= a.d_off);
  PackedLookup<S, MODE, ML> lk;
  lk.sR = reinterpret_cast<const uint16_t*>(reinterpret_cast<const char*>(smem) + a.x_off);
  lk.sD = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(smem) + a.d_off);
  // the level table follows the directory (16-B padded): eos_internal.h PackedPlan
  lk.sL = reinterpret_cast<const int32_t*>(lk.sD + ((((int64_t)a.bmax + 2) / 2 + 3) & ~int64_t(3)));
  lk.a = a;
  lk.sh = (uint32_t)args.sh;
  lk.depth = args.levels;
  lk.X = args.lv;
  lk.nodes = args.kv;
  search_body<CNT, SH>(args, lk, &clc_resp, &clc_bar);
}

// ------------------------------------------------ zero-setup search (f2) ----
// eos_search_direct: no host setup at all ("algorithms with zero setup
// cost may be a better choice" when tables are not known in advance).  Each
// CTA copies the device-resident table into smem, builds the count directory
// of a logarithm hash there (histogram + block scan, O(n + bins)), then runs
// the same streaming tile loop with a runtime in-bin step count.
constexpr int kDirectMaxTable = 4096;
#ifndef EOS_DIRECT_MAX_BINS
#define EOS_DIRECT_MAX_BINS 8192
#endif
constexpr int kDirectMaxBins = EOS_DIRECT_MAX_BINS;
using ShapeDirect = Shape<512, 4, 2, true>;

struct DirectArgs {
  SearchArgs s;          // image unused; ax filled in by the kernel
  const double* table;   // device fp64[n]
  int32_t n;
  int32_t bins_max;      // power of two <= kDirectMaxBins
  int32_t* status;       // nullable: receives EOS_ERR_UNSORTED / EOS_ERR_NONFINITE
};

template <int V>
struct IntTag {
  static constexpr int value = V;
};

template <class SH>
__global__ void __launch_bounds__(SH::kThreads, SH::kMinBlocks)
    search1d_direct_kernel(const DirectArgs A) {
  constexpr int T = SH::kThreads;
  extern __shared__ __align__(128) uint4 smem[];
  __shared__ __align__(16) uint4 clc_resp;
  __shared__ __align__(8) uint64_t clc_bar;
  __shared__ AxisParams sa;
  __shared__ uint32_t s_maxocc, s_bad, s_warp[T / 32];
  if (SH::kClc && threadIdx.x == 0) mbar_init(&clc_bar, 1);
  pdl_enter();  // the table may come from the previous kernel in the stream
  const int n = A.n;
  const int32_t x_bytes = (int32_t)((8 * n + 15) & ~15);
  double* sX = reinterpret_cast<double*>(smem);
  uint32_t* sD = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(smem) + x_bytes);
  uint32_t bad = 0;
  constexpr int LU = 8;  // all of a thread's table loads in flight at once (n <= 4096 = 8 T)
  for (int j0 = threadIdx.x; j0 < n; j0 += LU * T) {
    double v[LU];
#pragma unroll
    for (int u = 0; u < LU; ++u) v[u] = j0 + u * T < n ? __ldg(A.table + j0 + u * T) : 0.0;
#pragma unroll
    for (int u = 0; u < LU; ++u) {
      if (j0 + u * T < n) {
        if (!isfinite(v[u])) bad = EOS_ERR_NONFINITE;
        sX[j0 + u * T] = (v[u] == 0.0) ? 0.0 : v[u];  // canonicalise -0.0 (R6)
      }
    }
  }
  if (threadIdx.x == 0) {
    s_maxocc = 0;
    s_bad = 0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j + 1 < n; j += T)
    if (sX[j + 1] < sX[j]) bad = bad ? bad : EOS_ERR_UNSORTED;
  if (bad) atomicMax(&s_bad, bad);
  if (threadIdx.x == 0) {
    // hash over [lowest binned entry, X[n-1]] (R13): mode 0 bins from the
    // first entry > 0 (binary search), mode 1 from X[0]
    AxisParams a{};
    a.n = n;
    a.x_off = 0;
    a.d_off = x_bytes;
    a.mode = sX[0] >= 0.0 ? 0 : 1;
    int lo = 0;
    if (a.mode == 0) {
      int l = 0, h = n;  // first index with X > 0
      while (l < h) {
        const int m = (l + h) >> 1;
        if (sX[m] > 0.0) h = m; else l = m + 1;
      }
      lo = l < n ? l : n - 1;
    }
    const uint32_t klo = a.mode ? key_hi<1>(sX[lo]) : key_hi<0>(sX[lo]);
    const uint32_t khi = a.mode ? key_hi<1>(sX[n - 1]) : key_hi<0>(sX[n - 1]);
    const uint64_t span = (uint64_t)(khi - klo) + 1;
    uint64_t M = ((uint64_t)A.bins_max << 32) / span;
    M = M < 1 ? 1 : (M > 0xFFFFFFFFull ? 0xFFFFFFFFull : M);
    a.hb = klo;
    a.M = (uint32_t)M;
    a.bmax = __umulhi(khi - klo, a.M);
    a.x0 = sX[0];
    a.xlast = sX[n - 1];
    sa = a;
  }
  __syncthreads();
  const int bins = (int)sa.bmax + 1;
  for (int b = threadIdx.x; b < bins; b += T) sD[b] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += T) {
    const uint32_t key = sa.mode ? key_hi<1>(sX[j]) : key_hi<0>(sX[j]);
    atomicAdd(&sD[bin_of(key, sa)], 1u);
  }
  __syncthreads();
  // exclusive scan of the counts -> packed directory lo | occ << 16.  Each
  // warp owns a contiguous segment of bins and walks it 32 bins at a time
  // (lane l reads bin base + l: conflict-free), with a shuffle scan per chunk.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int W = T / 32;
  const int seg = ((bins + W - 1) / W + 31) & ~31;
  const int s0 = min(bins, warp * seg), s1 = min(bins, s0 + seg);
  uint32_t part = 0;
  for (int b = s0 + lane; b < s1; b += 32) part += sD[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, o);
  if (lane == 0) s_warp[warp] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int w = 0; w < W; ++w) {
      const uint32_t v = s_warp[w];
      s_warp[w] = run;
      run += v;
    }
  }
  __syncthreads();
  uint32_t carry = s_warp[warp], mx = 0;
  for (int c = s0; c < s1; c += 32) {
    const int b = c + lane;
    const uint32_t o = b < s1 ? sD[b] : 0u;
    uint32_t incl = o;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += v;
    }
    if (b < s1) sD[b] = (carry + incl - o) | (o << 16);
    carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    mx = max(mx, o);
  }
  atomicMax(&s_maxocc, mx);
  __syncthreads();
  if (threadIdx.x == 0 && s_bad && A.status) atomicExch(A.status, (int32_t)s_bad);
  AxisParams a = sa;
  int steps = 0;
  while ((1u << steps) < s_maxocc + 1) ++steps;
  a.steps = steps > 0 ? steps : 1;
  // S is known only now (block-uniform): fixed-S bodies for S <= 4, the
  // runtime-S body above
  auto body = [&](auto s_tag) {
    constexpr int S = decltype(s_tag)::value;
    if (a.mode) {
      const SmemLookup<S, false, 1, false> lk{sX, sD, a};
      search_body<false, SH>(A.s, lk, &clc_resp, &clc_bar);
    } else {
      const SmemLookup<S, false, 0, false> lk{sX, sD, a};
      search_body<false, SH>(A.s, lk, &clc_resp, &clc_bar);
    }
  };
  switch (a.steps) {
    case 1: body(IntTag<1>{}); break;
    case 2: body(IntTag<2>{}); break;
    case 3: body(IntTag<3>{}); break;
    case 4: body(IntTag<4>{}); break;
    default: body(IntTag<0>{}); break;
  }
}

// ------------------------------------------------------------------ 2-D ----
struct Interp2DArgs {
  const uint4* image;
  int32_t image_16;
  int32_t g_off;    // byte offset of G fp64[nR*nT] in the image
  int32_t rr_off;   // byte offset of the bank-pinned cell records of the R axis (REP 2
                    //   kernels): double2[2^rep_shift nR], (R[j], 1/(R[j+1]-R[j])), or
                    //   for LOGLOG grids (1/R[j], 1/ln(R[j+1]/R[j]))
  int32_t rt_off;   // the same for the T axis
  int32_t rep_shift;  // REP 2: log2 of the record copies per axis entry (3: 8 copies, the
                      //   conflict-free layout; fewer when smem is short: 2-way .. 8-way)
  int32_t narrow;     // LOGLOG: 2 if every cell of both axes has X[j+1]/X[j] <= 1.25, else 1 if <= 1.5, else 0
  int32_t pad3_;
  const double2* gq;  // GG / small kernels: the grid in device memory (ln G for LOGLOG) as
                      //   cell quads gq[2 (i (nT-1) + j)] = (G[i][j], G[i][j+1]),
                      //   gq[2 (i (nT-1) + j) + 1] = (G[i+1][j], G[i+1][j+1]) (32 B: one sector)
  int32_t vec_ok;
  int32_t pad_;
  int64_t ntiles;
  AxisParams r;     // density axis
  AxisParams t;     // temperature axis
  const double* rho;
  const double* T;
  double* P;
  int32_t* iR;      // nullable
  int32_t* iT;      // nullable
  double* dPr;      // nullable: dP/drho (DERIV kernels)
  double* dPt;      // nullable: dP/dT (DERIV kernels)
  int64_t count;
};

// 1/x for a normal x whose reciprocal is normal: the hardware estimate (ftz) and two
// Newton steps, within an ulp of the correctly rounded 1/x.
__device__ __forceinline__ double rcp_newton(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
  return __fma_rn(r, __fma_rn(-x, r, 1.0), r);
}

// ln(x / X) for the log-log weight of a cell [X, X r] with r <= 1.5 (grids whose
// cells all are, Interp2DArgs::narrow), X normal in [2^-1020, 2^1020]: the same real
// number as log1p((x - X)/X) (R24), as 2 atanh(u) with u = (x - X)/(x + X) -- inside
// the cell x - X is exact (Sterbenz) and u in [0, (r-1)/(r+1)] <= 0.2 -- by the odd
// series 2u (1 + u^2/3 + ... + u^(2K-2)/(2K-1)): K = 12 terms reach 2^-53 for u^2 <=
// 0.04 (r = 1.5), K = 8 for u^2 <= 1/81 (r = 1.25, narrow == 2; the first omitted term
// is <= 3.2e-17 relative).  One reciprocal estimate, K + 4 FMAs, no branch (the
// general log1p is a called routine).  The coefficients 2/(2i+1) live in the
// constant bank (as immediates each costs two uniform moves per call).  Outside the
// cell only the clamped weight matters: x < X gives a negative value, x above the
// cell a value above its log width (the partial sums grow with u), so both clamp as
// the exact logarithm would; x = +inf is held at 2^1021 (> every axis value: weight
// 1), x = +-0 gives u = -1, a negative value (weight 0, as ln 0 = -inf), x < 0 and
// NaN give NaN as log1p does.
__constant__ double kAtanhCoef[12] = {2.0,        2.0 / 3.0,  2.0 / 5.0,  2.0 / 7.0,
                                      2.0 / 9.0,  2.0 / 11.0, 2.0 / 13.0, 2.0 / 15.0,
                                      2.0 / 17.0, 2.0 / 19.0, 2.0 / 21.0, 2.0 / 23.0};
template <int K>
__device__ __forceinline__ double ln_ratio_cell(double x, double X) {
  static_assert(K >= 2 && K <= 12, "series length");
  const double xc = x > 0x1p1021 ? 0x1p1021 : x;  // (NaN passes through)
  const double u = __dmul_rn(__dsub_rn(xc, X), rcp_newton(__dadd_rn(xc, X)));
  const double u2 = __dmul_rn(u, u);
  double p = kAtanhCoef[K - 1];
#pragma unroll
  for (int i = K - 2; i >= 0; --i) p = __fma_rn(p, u2, kAtanhCoef[i]);
  const double r = __dmul_rn(u, p);
  return x < 0.0 ? __longlong_as_double(0x7FF8000000000000LL) : r;
}

// e^v for the log-log value P = exp(bilinear of ln G) (R24): n = rint(v / ln 2) by
// the 1.5 2^52 rounding constant, r = v - n ln 2 by two FMAs (ln 2 and its tail),
// |r| <= ln(2)/2, e^r by its Taylor polynomial of degree 13 (the first omitted term
// is < 5e-18 relative), scaled by 2^n in the exponent field.  Within ~2 ulp.
// |v| >= 708 (where 2^n could leave the normal range), inf and NaN take CUDA's exp.
__constant__ double kExpCoef[14] = {
    1.0,
    1.0,
    1.0 / 2.0,
    1.0 / 6.0,
    1.0 / 24.0,
    1.0 / 120.0,
    1.0 / 720.0,
    1.0 / 5040.0,
    1.0 / 40320.0,
    1.0 / 362880.0,
    1.0 / 3628800.0,
    1.0 / 39916800.0,
    1.0 / 479001600.0,
    1.0 / 6227020800.0};
__device__ __forceinline__ double exp_cell(double v) {
  if (!(fabs(v) < 708.0)) return exp(v);
  const double kd = __fma_rn(v, 0x1.71547652b82fep+0, 0x1.8p+52);  // v log2(e) + 1.5 2^52
  const double n = __dsub_rn(kd, 0x1.8p+52);
  double r = __fma_rn(-n, 0x1.62e42fefa39efp-1, v);  // ln 2 rounded ...
  r = __fma_rn(-n, 0x1.abc9e3b39803fp-56, r);        // ... and its tail
  double p = kExpCoef[13];
#pragma unroll
  for (int i = 12; i >= 0; --i) p = __fma_rn(p, r, kExpCoef[i]);
  return __hiloint2double(__double2hiint(p) + (__double2loint(kd) << 20), __double2loint(p));
}

__device__ __forceinline__ double clamp01(double t) {
  return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
}

// Bracket + cell endpoints on one axis: i (the P:54 lower bound), the cell
// ci = min(i, n-2) and its endpoints X[ci], X[ci+1].  With S = 1 (every bin
// holds at most one entry) the in-bin probe value X[lo] is always one of the
// two endpoints in the common case, so only one more gather is needed.

template <int S>
__device__ __forceinline__ void axis_cell(double y, const double* __restrict__ sX,
                                          const uint32_t* __restrict__ sD, const AxisParams& a,
                                          int32_t& i, int32_t& ci, double& xl, double& xr) {
  auto X = [&](int32_t j) { return sX[j]; };
  if (S == 1) {
    const uint32_t key = a.mode ? key_hi<1>(y) : key_hi<0>(y);
    const uint32_t d = sD[bin_of(key, a)];
    const int32_t lo = (int32_t)(d & 0xFFFFu);  // <= n-1: X[n-1] lies in the top bin
    const int32_t occ = (int32_t)(d >> 16);     // 0 or 1 when S == 1
    EOS_DCHECK(lo < a.n && occ <= 1);
    const double pv = X(lo);
    const int32_t c = (occ >= 1 && pv <= y) ? 1 : 0;
    i = (y >= a.x0) ? lo + c - 1 : 0;
    ci = min(i, a.n - 2);
    const bool left = (ci == lo), right = (ci + 1 == lo);
    const double ov = X(left ? lo + 1 : (right ? lo - 1 : ci));
    xl = left ? pv : ov;
    xr = left ? ov : (right ? pv : X(ci + 1));
    EOS_DCHECK(ci >= 0 && ci + 1 < a.n && (left ? lo + 1 : (right ? lo - 1 : ci)) < a.n);
  } else {
    i = a.mode ? lookup<S, 1>(y, sX, sD, a) : lookup<S, 0>(y, sX, sD, a);
    ci = min(i, a.n - 2);
    xl = X(ci);
    xr = X(ci + 1);
  }
}

// REP 2 (bank-pinned cell records): 16-byte records Rec[8 j + c] =
// (X[j], 1/(X[j+1] - X[j])), 8 copies, copy c in bank quad c.  A 128-bit
// shared load is served per quarter-warp, and lane l reads copy l mod 8, so
// the gathers are conflict-free (4 wavefronts per warp).  One record gives
// the cell's left endpoint and inverse width, so the interpolation weight
// needs no fp64 divide: t = (x - X[ci]) * (1/dX[ci]) (a few ulp from the
// divide; within the 1e-12 bar).  With S = 1: the first record is that of
// the bin's entry (occ = 1, also the probe) or of the cell left of the bin
// (occ = 0, then it is the cell); a second record is read only when the
// probe moves the cell.
//
// S = kMapped (axes whose nodes follow a fitted map, grid_api.cu fit_cell_map): no
// directory read.  p = floor(map_a w(y) + map_b), w = log2 y (MUFU.LG2) or y, in
// fp32 and clamped to [0, n-2], is the cell of y or the one above (the host checks
// every node against the device error bound), so the record at p is the cell's or,
// when y < X[p], the next record down is (read only then).
template <int S>
__device__ __forceinline__ void axis_cell_rec(double y, const double* __restrict__ sX,
                                              const uint32_t* __restrict__ sD, const AxisParams& a,
                                              int32_t& i, int32_t& ci, double& xl, double& inv,
                                              const double2* __restrict__ rec_, int32_t sh) {
  double2 r;
  int32_t p;
  if constexpr (S == kMapped) {
    const float yf = __double2float_rn(y);
    float l2;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(yf));
    const float w = a.map_kind == 1 ? l2 : yf;
    p = min(max(__float2int_rd(__fmaf_rn(w, a.map_a, a.map_b)), 0), a.n - 2);
    r = rec_[p << sh];
    // NaN: p = 0 (cvt of NaN), i = 0; y >= X[n-1]: p = n - 2 (the map), i = n - 1
    i = (y >= a.x0) ? ((y >= a.xlast) ? a.n - 1 : p - (y < r.x ? 1 : 0)) : 0;
    EOS_DCHECK(p >= 0 && p + 1 < a.n);
  } else if constexpr (S == 1) {
    const uint32_t key = a.mode ? key_hi<1>(y) : key_hi<0>(y);
    const uint32_t d = sD[bin_of(key, a)];
    const int32_t lo = (int32_t)(d & 0xFFFFu);  // <= n-1
    const int32_t occ = (int32_t)(d >> 16);     // 0 or 1
    p = occ >= 1 ? lo : max(lo - 1, 0);
    EOS_DCHECK(lo < a.n && occ <= 1 && p < a.n);
    r = rec_[p << sh];
    const int32_t c = (occ >= 1 && r.x <= y) ? 1 : 0;
    i = (y >= a.x0) ? lo + c - 1 : 0;
  } else {
    i = a.mode ? lookup<S, 1>(y, sX, sD, a) : lookup<S, 0>(y, sX, sD, a);
    p = -1;
  }
  ci = min(i, a.n - 2);
  if (ci != p) r = rec_[ci << sh];
  xl = r.x;
  inv = r.y;
}

// Bilinear on the bracket cell (R14).  Written with explicit
// round-to-nearest intrinsics (no FMA contraction), in the order of the
// formula in eossearch.h, so the value is the correctly-rounded evaluation
// of that formula (bit-identical to a plain evaluation in that order).
//
// GG (grids larger than shared memory): the grid stays in device memory
// (L2-resident up to a few 10^6 cells) as cell quads, so the 4 corners are one
// aligned 32-byte load (one L1/L2 sector).  The axes, their directories and
// records stay in smem.
// NK (log-log grids with bank-pinned records): 8 or 12 = the series length of every
// cell fixed at compile time (no launch-uniform branch, so a thread's two pairs
// interleave); 0 = chosen per launch from Interp2DArgs::narrow.
template <int S, bool DERIV, bool LOGLOG, int REP, bool GG, int NK = 0>
__device__ __forceinline__ double interp_one(double rho, double T, int32_t& i, int32_t& j,
                                             double& dpr, double& dpt, const char* sm,
                                             const Interp2DArgs& A) {
  const double* sR = reinterpret_cast<const double*>(sm + A.r.x_off);
  const double* sT = reinterpret_cast<const double*>(sm + A.t.x_off);
  const uint32_t* dR = reinterpret_cast<const uint32_t*>(sm + A.r.d_off);
  const uint32_t* dT = reinterpret_cast<const uint32_t*>(sm + A.t.d_off);
  const double* sG = reinterpret_cast<const double*>(sm + A.g_off);  // G, or ln G (LOGLOG)
  int32_t ci, cj;
  double r0, r1, t0, t1;
  double ir = 0.0, it = 0.0;  // REP 2: inverse cell widths (in x, or in ln x for LOGLOG)
  double wr = 0.0, wt = 0.0;  // REP 0: cell widths (in x, or in ln x for LOGLOG)
  double tx, ty;              // the bilinear weights
  if constexpr (LOGLOG) {
    // R24: t = (ln x - ln X[c]) / (ln X[c+1] - ln X[c]), evaluated as
    // log1p((x - X[c]) / X[c]) / log1p((X[c+1] - X[c]) / X[c]) -- the same real
    // numbers, without the cancellation of ln x - ln X[c] (which loses
    // ~|ln x| / (cell width in ln) ulps).  Brackets and X[c] from the plain axes.
    if constexpr (REP == 2) {
      // bank-pinned records (X[j], 1/ln(X[j+1]/X[j])), read as the linear grids read
      // theirs (the record is also the probe); no divides on the narrow-cell paths
      // (axes within [2^-1020, 2^1020], grid_api.cu)
      const int32_t sh = A.rep_shift, c = threadIdx.x & ((1 << sh) - 1);
      axis_cell_rec<S>(rho, sR, dR, A.r, i, ci, r0, ir,
                       reinterpret_cast<const double2*>(sm + A.rr_off) + c, sh);
      axis_cell_rec<S>(T, sT, dT, A.t, j, cj, t0, it,
                       reinterpret_cast<const double2*>(sm + A.rt_off) + c, sh);
      if constexpr (NK > 0) {
        tx = clamp01(__dmul_rn(ln_ratio_cell<NK>(rho, r0), ir));
        ty = clamp01(__dmul_rn(ln_ratio_cell<NK>(T, t0), it));
      } else if (A.narrow == 2) {  // every cell ratio <= 1.25: 8 terms (launch-uniform branch)
        tx = clamp01(__dmul_rn(ln_ratio_cell<8>(rho, r0), ir));
        ty = clamp01(__dmul_rn(ln_ratio_cell<8>(T, t0), it));
      } else if (A.narrow) {  // every cell ratio <= 1.5: 12 terms
        tx = clamp01(__dmul_rn(ln_ratio_cell<12>(rho, r0), ir));
        ty = clamp01(__dmul_rn(ln_ratio_cell<12>(T, t0), it));
      } else {  // wide cells: log1p((x - X)/X)
        tx = clamp01(__dmul_rn(log1p(__ddiv_rn(__dsub_rn(rho, r0), r0)), ir));
        ty = clamp01(__dmul_rn(log1p(__ddiv_rn(__dsub_rn(T, t0), t0)), it));
      }
    } else {
      axis_cell<S>(rho, sR, dR, A.r, i, ci, r0, r1);
      axis_cell<S>(T, sT, dT, A.t, j, cj, t0, t1);
      wr = log1p(__ddiv_rn(__dsub_rn(r1, r0), r0));
      wt = log1p(__ddiv_rn(__dsub_rn(t1, t0), t0));
      tx = clamp01(__ddiv_rn(log1p(__ddiv_rn(__dsub_rn(rho, r0), r0)), wr));
      ty = clamp01(__ddiv_rn(log1p(__ddiv_rn(__dsub_rn(T, t0), t0)), wt));
    }
  } else if constexpr (REP == 2) {
    const int32_t sh = A.rep_shift, c = threadIdx.x & ((1 << sh) - 1);  // this lane's copy
    axis_cell_rec<S>(rho, sR, dR, A.r, i, ci, r0, ir,
                     reinterpret_cast<const double2*>(sm + A.rr_off) + c, sh);
    axis_cell_rec<S>(T, sT, dT, A.t, j, cj, t0, it,
                     reinterpret_cast<const double2*>(sm + A.rt_off) + c, sh);
    tx = clamp01(__dmul_rn(__dsub_rn(rho, r0), ir));
    ty = clamp01(__dmul_rn(__dsub_rn(T, t0), it));
  } else {
    axis_cell<S>(rho, sR, dR, A.r, i, ci, r0, r1);
    axis_cell<S>(T, sT, dT, A.t, j, cj, t0, t1);
    wr = __dsub_rn(r1, r0);
    wt = __dsub_rn(t1, t0);
    tx = clamp01(__ddiv_rn(__dsub_rn(rho, r0), wr));
    ty = clamp01(__ddiv_rn(__dsub_rn(T, t0), wt));
  }
  EOS_DCHECK(ci >= 0 && cj >= 0 && ci + 1 < A.r.n && cj + 1 < A.t.n);
  double g00, g01, g10, g11;
  if (GG) {
    const int64_t w = A.t.n - 1;  // cells per row
    // one 256-bit load: the 4 corners share one 32-B sector
    ldg_f64x4(reinterpret_cast<const double*>(A.gq + 2 * ((int64_t)ci * w + cj)), g00, g01, g10,
              g11);
  } else {
    const double* g0 = sG + (int64_t)ci * A.t.n + cj;
    const double* g1 = g0 + A.t.n;
    g00 = g0[0];
    g01 = g0[1];
    g10 = g1[0];
    g11 = g1[1];
  }
  const double uy = __dsub_rn(1.0, ty);
  const double ux = __dsub_rn(1.0, tx);
  const double a0 = __dadd_rn(__dmul_rn(uy, g00), __dmul_rn(ty, g01));
  const double a1 = __dadd_rn(__dmul_rn(uy, g10), __dmul_rn(ty, g11));
  const double v = __dadd_rn(__dmul_rn(ux, a0), __dmul_rn(tx, a1));
  const double p = LOGLOG ? exp_cell(v) : v;
  if (DERIV) {
    // Partial derivatives of the interpolant on the cell (R23 / R24); 0
    // outside an axis range (the clamped interpolant is constant there); NaN
    // kept.  LOGLOG: dP/drho = P * (d ln P / d ln rho) / rho.
    const double nr = __dadd_rn(__dmul_rn(uy, __dsub_rn(g10, g00)), __dmul_rn(ty, __dsub_rn(g11, g01)));
    const double nt = __dadd_rn(__dmul_rn(ux, __dsub_rn(g01, g00)), __dmul_rn(tx, __dsub_rn(g11, g10)));
    const double sr = REP == 2 ? __dmul_rn(nr, ir) : __ddiv_rn(nr, wr);
    const double st = REP == 2 ? __dmul_rn(nt, it) : __ddiv_rn(nt, wt);
    const bool in_r = rho >= A.r.x0 && rho <= A.r.xlast;
    const bool in_t = T >= A.t.x0 && T <= A.t.xlast;
    const double dr = LOGLOG ? __ddiv_rn(__dmul_rn(p, sr), rho) : sr;
    const double dt = LOGLOG ? __ddiv_rn(__dmul_rn(p, st), T) : st;
    dpr = (rho != rho) ? rho : (in_r ? dr : 0.0);
    dpt = (T != T) ? T : (in_t ? dt : 0.0);
  }
  return p;
}

// default 2-D launch shape (165 KB image: 1 CTA/SM).  Static schedule: the
// 2-D body is smem/latency-bound, where the CLC loop's per-tile CTA barrier
// costs more than the static tail (profiles/r01_exp_interp.json).
using Shape2D = Shape<1024, 1, 1, false>;
using Shape2DDeriv = Shape<512, 1, 1, false>;  // derivative outputs need > 64 registers
// derivative kernels of log-log or device-memory grids with one-step (or mapped) axes
// and bank-pinned records: latency-bound at 16 warps per SM; they fit 768 threads (80
// registers) or, log-log grids in shared memory, 1024 (64) without spills
using Shape2DDerivWide = Shape<768, 1, 1, false>;
using Shape2DDerivFull = Shape<1024, 1, 1, false>;
// launches with fewer tiles than half the SMs: quarter-size tiles, the grid read from cell
// quads in device memory (grid_api.cu pick_interp_small)
using Shape2DSmallGG = Shape<256, 1, 1, false>;

template <int S, class SH, bool DERIV, bool LOGLOG = false, int REP = 0, bool GG = false, int NK = 0>
__global__ void __launch_bounds__(SH::kThreads, SH::kMinBlocks) interp2d_kernel(const Interp2DArgs A) {
  static_assert(S != kMapped || REP == 2, "fitted cell maps read the bank-pinned records");
  constexpr int T = SH::kThreads;
  constexpr int U = SH::kUnroll;
  constexpr int TP = SH::kTilePairs;
  constexpr int TE = SH::kTileElems;
  extern __shared__ __align__(128) uint4 smem[];
  __shared__ __align__(16) uint4 clc_resp;
  __shared__ __align__(8) uint64_t clc_bar, stage_bar;
  if (SH::kClc && threadIdx.x == 0) mbar_init(&clc_bar, 1);
  stage_image(smem, A.image, A.image_16, &stage_bar);
  pdl_enter();
  const char* sm = reinterpret_cast<const char*>(smem);
  const int64_t count = A.count;
  const int64_t ntiles = A.ntiles;
  const bool vec = A.vec_ok != 0;
  const bool br = A.iR != nullptr, bt = A.iT != nullptr;
  const double2* __restrict__ R2 = reinterpret_cast<const double2*>(A.rho);
  const double2* __restrict__ T2 = reinterpret_cast<const double2*>(A.T);
  double2* __restrict__ P2 = reinterpret_cast<double2*>(A.P);
  int2* __restrict__ IR2 = reinterpret_cast<int2*>(A.iR);
  int2* __restrict__ IT2 = reinterpret_cast<int2*>(A.iT);
  double2* __restrict__ DR2 = reinterpret_cast<double2*>(A.dPr);
  double2* __restrict__ DT2 = reinterpret_cast<double2*>(A.dPt);
  const bool bdr = DERIV && A.dPr != nullptr, bdt = DERIV && A.dPt != nullptr;

  uint32_t phase = 0;
  auto next_tile = [&](int64_t t) -> int64_t {
    if (!SH::kClc) return t + gridDim.x;
    mbar_wait(&clc_bar, phase);
    phase ^= 1u;
    const int64_t tn = clc_query(&clc_resp);
    __syncthreads();
    return tn < 0 ? ntiles : tn;
  };
  auto full = [&](int64_t t) { return vec && (t + 1) * TE <= count; };

  int64_t t = blockIdx.x;
  double2 vr[U], vt[U];
  if (t < ntiles && full(t)) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vr[u] = ld_stream(R2 + t * TP + threadIdx.x + u * T);
      vt[u] = ld_stream(T2 + t * TP + threadIdx.x + u * T);
    }
  }
  while (t < ntiles) {
    if (SH::kClc && threadIdx.x == 0) {
      mbar_arrive_expect_tx(&clc_bar, 16);
      clc_try_cancel(&clc_resp, &clc_bar);
    }
    int64_t tn;
    if (full(t)) {
      const int64_t p0 = t * TP + threadIdx.x;
      EOS_DCHECK(2 * (p0 + (U - 1) * T) + 1 < count);
      double2 p[U], dr[U], dt[U];
      int2 ir[U], it[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        p[u].x = interp_one<S, DERIV, LOGLOG, REP, GG, NK>(vr[u].x, vt[u].x, ir[u].x, it[u].x, dr[u].x, dt[u].x,
                                             sm, A);
        p[u].y = interp_one<S, DERIV, LOGLOG, REP, GG, NK>(vr[u].y, vt[u].y, ir[u].y, it[u].y, dr[u].y, dt[u].y,
                                             sm, A);
      }
      tn = next_tile(t);
      if (tn < ntiles && full(tn)) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          vr[u] = ld_stream(R2 + tn * TP + threadIdx.x + u * T);
          vt[u] = ld_stream(T2 + tn * TP + threadIdx.x + u * T);
        }
      }
#ifndef EOS_EXP_NO_L2_PREFETCH
      if (!SH::kClc && !GG && threadIdx.x == 0) {
        // the tile after next into L2 (static schedule): the register loads above,
        // issued only after this tile's pairs (a register double buffer issued
        // before them measured 175 -> 153 Gpairs/s at the 64-register cap), then
        // wait on L2, not DRAM.  (Not for grids in device memory, whose corner
        // gathers share L2: big2d 128 -> 120 with it.)
        const int64_t t2 = tn + gridDim.x;
        if (t2 < ntiles && full(t2)) {
          bulk_prefetch_l2(R2 + t2 * TP, (uint32_t)(TP * sizeof(double2)));
          bulk_prefetch_l2(T2 + t2 * TP, (uint32_t)(TP * sizeof(double2)));
        }
      }
#endif
#pragma unroll
      for (int u = 0; u < U; ++u) {
        __stcs(P2 + p0 + u * T, p[u]);
        if (br) __stcs(IR2 + p0 + u * T, ir[u]);
        if (bt) __stcs(IT2 + p0 + u * T, it[u]);
        if (bdr) __stcs(DR2 + p0 + u * T, dr[u]);
        if (bdt) __stcs(DT2 + p0 + u * T, dt[u]);
      }
    } else {
      const int64_t e0 = t * TE;
      const int64_t e1 = min(count, e0 + TE);
      // ragged tile: a thread's (2U) pairs at stride T; with U = 1 the second pair's
      // coordinates are loaded before the first pair is computed (not where the
      // 64-register cap of 1024-thread CTAs would make it spill: log-log, and
      // device-memory grids at 1024 threads)
      constexpr int E = (U == 1 && !LOGLOG && (!GG || T <= 512)) ? 2 : 1;
      for (int64_t q0 = e0 + threadIdx.x; q0 < e1; q0 += E * T) {
        double vr1[E], vt1[E];
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int64_t q = q0 + (int64_t)k * T;
          vr1[k] = q < e1 ? A.rho[q] : 1.0;
          vt1[k] = q < e1 ? A.T[q] : 1.0;
        }
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int64_t q = q0 + (int64_t)k * T;
          if (q < e1) {
            int32_t i, j;
            double dpr, dpt;
            const double pq = interp_one<S, DERIV, LOGLOG, REP, GG, NK>(vr1[k], vt1[k], i, j,
                                                                          dpr, dpt, sm, A);
            A.P[q] = pq;
            if (br) A.iR[q] = i;
            if (bt) A.iT[q] = j;
            if (bdr) A.dPr[q] = dpr;
            if (bdt) A.dPt[q] = dpt;
          }
        }
      }
      tn = next_tile(t);
      if (tn < ntiles && full(tn)) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          vr[u] = ld_stream(R2 + tn * TP + threadIdx.x + u * T);
          vt[u] = ld_stream(T2 + tn * TP + threadIdx.x + u * T);
        }
      }
    }
    t = tn;
  }
}

}  // namespace dev
}  // namespace eos
