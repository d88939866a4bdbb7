// search_api.cu -- the 1-D part of the C ABI (include/eossearch.h): table
// handles (single-level and tiered), the search launches, the zero-setup
// search, host-only planning.  Product path (never includes or links oracle/).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <new>
#include <vector>

#include "eos_internal.h"
#include "eossearch.h"
#include "kernels.cuh"
#include "runtime.h"

using eos::TablePlan;
namespace dv = eos::dev;
using namespace eos::rt;

struct eos_table_s {
  TablePlan plan;          // the shared-memory table (T1 of a tiered table)
  int levels = 0;          // D (tiered tables, eos_search_create_levels)
  int node_width = 0;      // 8: 8-ary key levels; 15: packed nodes (eos_internal.h PackedPlan)
  int sh = 0;              // packed: residual bits of the sample table
  const uint32_t* nodes_dev = nullptr;  // packed: the nodes (inside levels_dev, after X)
  int64_t n = 0;           // entries of the full table
  int64_t top_n = 0;       // n1
  int64_t level_bytes = 0;
  int64_t level_elems = 0;
  double* levels_dev = nullptr;  // the 8-ary levels: F (fp64) then K (u32), coarsest first
  int device = -1;
  int num_sms = 0;
  void* image_dev = nullptr;
  int64_t smem_bytes = 0;  // the staged image (fp64 table, or the keys of T1 when tiered)
  dv::AxisParams ax{};
  // launch configuration per counters on/off
  const void* fn[2] = {nullptr, nullptr};
  int grid[2] = {0, 0};
  int threads[2] = {256, 256};
  int unroll[2] = {4, 4};
  bool clc[2] = {true, true};
  int ctas_per_sm = 0;
  // large launches through the shared-memory ring (search1d_ring_kernel; nullptr: none)
  const void* fn_ring = nullptr;
  int ring_ns = 0, grid_ring = 0;
  int64_t ring_smem = 0;
  // small launches (pick_search_small; fn_small == nullptr: none)
  const void* fn_small = nullptr;
  int threads_small = 0, unroll_small = 0, grid_small = 0;
  bool clc_small = true;
};

namespace {

// ---------------------------------------------------------- kernel table ---
// The search kernel of a plan's lifting layout (eos_internal.h TablePlan):
// SF = 1..3 fixed steps (big: a rare branch for deeper bins) or SF = 0 (all
// steps in a runtime loop), key mode 0/1, 16- or 32-bit directory entries.
template <int SF, bool BIG, int MODE, bool D16, class SH>
const void* kfn() {
  return (const void*)dv::search1d_kernel<SF, BIG, MODE, D16, false, SH>;
}

template <class SH, int MODE, bool D16>
const void* search_fn_md(int sf, bool big) {
  switch (sf) {
    case 1: return big ? kfn<1, true, MODE, D16, SH>() : kfn<1, false, MODE, D16, SH>();
    case 2: return big ? kfn<2, true, MODE, D16, SH>() : kfn<2, false, MODE, D16, SH>();
    case 3: return big ? kfn<3, true, MODE, D16, SH>() : kfn<3, false, MODE, D16, SH>();
    default: return kfn<0, true, MODE, D16, SH>();
  }
}

template <class SH>
const void* search_fn(const TablePlan& p) {
  if (p.key_mode == 0)
    return p.dir16 ? search_fn_md<SH, 0, true>(p.fast_steps, p.big)
                   : search_fn_md<SH, 0, false>(p.fast_steps, p.big);
  return p.dir16 ? search_fn_md<SH, 1, true>(p.fast_steps, p.big)
                 : search_fn_md<SH, 1, false>(p.fast_steps, p.big);
}

// Validation launches (counters on): the runtime-step body, one shape.
const void* counters_fn(const TablePlan& p) {
  using SH = dv::ShapeCnt;
  if (p.key_mode == 0)
    return p.dir16 ? (const void*)dv::search1d_kernel<0, true, 0, true, true, SH>
                   : (const void*)dv::search1d_kernel<0, true, 0, false, true, SH>;
  return p.dir16 ? (const void*)dv::search1d_kernel<0, true, 1, true, true, SH>
                 : (const void*)dv::search1d_kernel<0, true, 1, false, true, SH>;
}

// tiered tables (levels >= 1): search1d_tiered_kernel
template <int S, int MODE, class SH>
const void* tiered_fn(bool cnt) {
  return cnt ? (const void*)dv::search1d_tiered_kernel<S, MODE, true, dv::ShapeCnt>
             : (const void*)dv::search1d_tiered_kernel<S, MODE, false, SH>;
}

template <int MODE, class SH>
const void* tiered_fn_mode(int steps, bool cnt) {
  switch (steps) {
    case 1: return tiered_fn<1, MODE, SH>(cnt);
    case 2: return tiered_fn<2, MODE, SH>(cnt);
    case 3: return tiered_fn<3, MODE, SH>(cnt);
    case 4: return tiered_fn<4, MODE, SH>(cnt);
    case 5: return tiered_fn<5, MODE, SH>(cnt);
    case 6: return tiered_fn<6, MODE, SH>(cnt);
    case 7: return tiered_fn<7, MODE, SH>(cnt);
    case 8: return tiered_fn<8, MODE, SH>(cnt);
    default: return tiered_fn<0, MODE, SH>(cnt);
  }
}

// packed tables: search1d_packed_kernel, S = 1..kPackedMaxSteps; ML = false: the
// one-level instantiation (no level loop) of the main launch shape
template <int MODE, class SH, bool CNT, bool ML>
const void* packed_fn(int steps) {
  switch (steps) {
    case 1: return (const void*)dv::search1d_packed_kernel<1, MODE, CNT, SH, ML>;
    case 2: return (const void*)dv::search1d_packed_kernel<2, MODE, CNT, SH, ML>;
    case 3: return (const void*)dv::search1d_packed_kernel<3, MODE, CNT, SH, ML>;
    case 4: return (const void*)dv::search1d_packed_kernel<4, MODE, CNT, SH, ML>;
    case 5: return (const void*)dv::search1d_packed_kernel<5, MODE, CNT, SH, ML>;
    default: return (const void*)dv::search1d_packed_kernel<6, MODE, CNT, SH, ML>;
  }
}
template <class SH, bool CNT, bool ML = true>
const void* packed_fn_mode(int mode, int steps) {
  return mode == 0 ? packed_fn<0, SH, CNT, ML>(steps) : packed_fn<1, SH, CNT, ML>(steps);
}
static_assert(eos::kPackedMaxSteps == 6, "packed_fn covers S = 1..6");

// Small launches of tiered tables: 512 x 1 tiles (a quarter of the default
// 1024 x 2), used like the single-level small shapes when the default tiles
// would leave most SMs idle.  big (n = 2^20) at 1e4 / 1e5 / 2.5e5 targets:
// 7.3 / 7.9 / 8.0 -> 3.7 / 4.6 / 6.9 us per launch.
template <int MODE>
const void* tiered_small_fn(int steps) {
  using SH = dv::Shape<512, 1, 1, false>;
  switch (steps) {
    case 1: return (const void*)dv::search1d_tiered_kernel<1, MODE, false, SH>;
    case 2: return (const void*)dv::search1d_tiered_kernel<2, MODE, false, SH>;
    case 3: return (const void*)dv::search1d_tiered_kernel<3, MODE, false, SH>;
    case 4: return (const void*)dv::search1d_tiered_kernel<4, MODE, false, SH>;
    default: return nullptr;
  }
}

// The ring kernel of a layout (search1d_ring_kernel; the stage count is a launch
// argument), 8 targets per lane per stage (62 KB stages): cfg5 (S = 3, 86 KB image,
// 2 stages) 528 -> 562 Glookups/s; 4 per lane 529; S = 1 tables equal either way
// (cfg2 580 vs 584), so those keep the register kernels.
template <int MODE, bool D16, int PL>
const void* ring_fn_md(int sf, bool big) {
  switch (sf) {
    case 1: return (const void*)dv::search1d_ring_kernel<1, false, MODE, D16, PL>;
    case 2: return (const void*)dv::search1d_ring_kernel<2, false, MODE, D16, PL>;
    case 3: return big ? (const void*)dv::search1d_ring_kernel<3, true, MODE, D16, PL>
                       : (const void*)dv::search1d_ring_kernel<3, false, MODE, D16, PL>;
    default: return (const void*)dv::search1d_ring_kernel<0, true, MODE, D16, PL>;
  }
}
constexpr int kRingPerLane = 8;
constexpr int kRingStage = dv::kRingWarps * 32 * kRingPerLane;  // 7936 targets, 62 KB
const void* ring_fn(const TablePlan& p) {
#ifndef EOS_EXPERIMENTS
  if (p.steps < 2) return nullptr;  // S = 1: the register kernels (measured equal)
#endif
  if (p.key_mode == 0)
    return p.dir16 ? ring_fn_md<0, true, kRingPerLane>(p.fast_steps, p.big)
                   : ring_fn_md<0, false, kRingPerLane>(p.fast_steps, p.big);
  return p.dir16 ? ring_fn_md<1, true, kRingPerLane>(p.fast_steps, p.big)
                 : ring_fn_md<1, false, kRingPerLane>(p.fast_steps, p.big);
}
int ring_stage() { return kRingStage; }
// Launches with at least this many ring stages per SM take the ring kernel.
constexpr int64_t kRingMinStagesPerSm = 4;

struct LaunchShape {
  const void* fn;
  int threads, unroll;
  bool clc;
};

template <class SH>
LaunchShape shape_of(const TablePlan& p) {
  return {search_fn<SH>(p), SH::kThreads, SH::kUnroll, SH::kClc};
}

// Default launch shape by image size: as many threads per SM as registers
// allow (~1024 at <= 64 regs), with all image copies of an SM <= ~144 KB of
// smem so L1 keeps room for the in-flight streaming loads.
// One 1024-thread CTA per SM (images > 72 KB) always takes the static
// schedule: its per-tile CTA barrier makes CLC 13-15% slower there even at
// S <= 2 (n = 4096 log-uniform, 143 KB image: 443 -> 508 Glookups/s;
// profiles/r01_exp_table_size.json).  Deep lifting (SF >= 3 or the runtime
// loop) is issue-bound: static schedule there too.
LaunchShape pick_search(const TablePlan& p, int64_t image_bytes) {
  const bool deep = p.fast_steps == 0 || p.fast_steps >= 3;
  if (image_bytes > 72 * 1024) return shape_of<dv::ShapeDeepBig>(p);
  if (deep) return shape_of<dv::ShapeDeepMid>(p);
  if (image_bytes <= 32 * 1024) return shape_of<dv::ShapeSmall>(p);
  return shape_of<dv::ShapeMid>(p);
}

// Small launches: the same shapes with one double2 per thread per tile (4x
// smaller tiles), used when the default tiling would leave most SMs idle (fewer
// tiles than half the SMs).  1e5 targets (25-49 default tiles): cfg1 37 -> 62,
// cfg2 39 -> 64, cfg5 34 -> 48 Glookups/s; between 1.5e5 and 3e5 targets the two
// are within launch noise, from 3.5e5 on they are the same kernel.
LaunchShape pick_search_small(const TablePlan& p, int64_t image_bytes) {
  const bool deep = p.fast_steps == 0 || p.fast_steps >= 3;
  if (image_bytes > 72 * 1024) return shape_of<dv::Shape<1024, 1, 1, false>>(p);
  if (deep) return shape_of<dv::Shape<512, 1, 2, false>>(p);
  if (image_bytes <= 32 * 1024) return shape_of<dv::Shape<256, 1, 4, true>>(p);
  return shape_of<dv::Shape<512, 1, 2, true>>(p);
}

#ifdef EOS_EXPERIMENTS
// ---- A/B experiments only (_build.py --exp: libeossearch_exp.so) ----------
// EOS_SEARCH_VARIANT=<name>: launch shape by name (single-level tables)
// EOS_TIERED_VARIANT=<name>: launch shape of tiered tables (mode 0, S <= 4)
// EOS_LAYOUT=<d16>,<sf>,<big>: force the lifting layout of a single-level table
// EOS_SMALL_TILES=0: small launches keep the default tiles
struct Variant {
  const char* name;
  LaunchShape (*get)(const TablePlan& p);
};
template <class SH>
LaunchShape vshape(const TablePlan& p) { return shape_of<SH>(p); }
const Variant kVariants[] = {
    {"static256u4", vshape<dv::Shape<256, 4, 4, false>>},
    {"static512u4", vshape<dv::Shape<512, 4, 2, false>>},
    {"static1024u4", vshape<dv::Shape<1024, 4, 1, false>>},
    {"static1024u2", vshape<dv::Shape<1024, 2, 1, false>>},
    {"clc256u4", vshape<dv::Shape<256, 4, 4, true>>},
    {"clc512u4", vshape<dv::Shape<512, 4, 2, true>>},
    {"clc1024u4", vshape<dv::Shape<1024, 4, 1, true>>},
    {"static512u8", vshape<dv::Shape<512, 8, 2, false>>},
};
template <class SH>
LaunchShape tvshape(const TablePlan& p) {
  switch (p.steps) {
    case 1: return {(const void*)dv::search1d_tiered_kernel<1, 0, false, SH>, SH::kThreads, SH::kUnroll, SH::kClc};
    case 2: return {(const void*)dv::search1d_tiered_kernel<2, 0, false, SH>, SH::kThreads, SH::kUnroll, SH::kClc};
    case 3: return {(const void*)dv::search1d_tiered_kernel<3, 0, false, SH>, SH::kThreads, SH::kUnroll, SH::kClc};
    default: return {(const void*)dv::search1d_tiered_kernel<4, 0, false, SH>, SH::kThreads, SH::kUnroll, SH::kClc};
  }
}
const Variant kTieredVariants[] = {
    {"static512u4", tvshape<dv::Shape<512, 4, 1, false>>},
    {"static1024u1", tvshape<dv::Shape<1024, 1, 1, false>>},
    {"clc1024u2", tvshape<dv::Shape<1024, 2, 1, true>>},
};
bool exp_variant(const TablePlan& p, bool tiered, LaunchShape* ls) {
  const char* want = getenv(tiered ? "EOS_TIERED_VARIANT" : "EOS_SEARCH_VARIANT");
  if (!want || (tiered && (p.key_mode != 0 || p.steps > 4))) return false;
  const Variant* vs = tiered ? kTieredVariants : kVariants;
  const size_t nv = tiered ? sizeof(kTieredVariants) / sizeof(Variant) : sizeof(kVariants) / sizeof(Variant);
  for (size_t i = 0; i < nv; ++i)
    if (strcmp(want, vs[i].name) == 0) {
      *ls = vs[i].get(p);
      return true;
    }
  return false;
}
void exp_layout(TablePlan* p) {
  const char* e = getenv("EOS_LAYOUT");
  int d16 = 0, sf = 0, big = 0;
  if (!e || sscanf(e, "%d,%d,%d", &d16, &sf, &big) != 3) return;
  if (d16 && (p->n > eos::kDir16MaxN || p->max_occ > eos::kDir16MaxOcc)) d16 = 0;
  if (sf > p->steps) sf = p->steps;
  p->dir16 = d16 != 0;
  p->fast_steps = sf;
  p->big = sf == 0 || p->steps > sf;
  p->image_bytes = p->x_bytes + ((((p->dir16 ? 2 : 4) * (int64_t)p->bins) + 15) & ~int64_t(15));
}
bool exp_small_off() {
  const char* e = getenv("EOS_SMALL_TILES");
  return e && e[0] == '0';
}
int exp_ring(int ns) {  // EOS_RING=<n>: at most n ring stages (0: none; unset: as the product)
  const char* e = getenv("EOS_RING");
  return e ? std::min(ns, atoi(e)) : ns;
}
#else
bool exp_small_off() { return false; }
int exp_ring(int ns) { return ns; }
#endif

eos_status launch_search(eos_table t, const double* Y, int64_t count, int32_t* out, int64_t gofs,
                         uint64_t* counters, cudaStream_t st_) {
  cudaStream_t st = st_;
  const bool cnt = counters != nullptr;
  dv::SearchArgs a{};
  a.image = (const uint4*)t->image_dev;
  a.image_16 = (int32_t)(t->smem_bytes / 16);
  a.ax = t->ax;
  a.Y = Y;
  a.out = out;
  a.count = count;
  a.gofs = gofs;
  a.counters = (unsigned long long*)counters;
  a.lv = t->levels_dev;
  a.kv = t->levels_dev ? reinterpret_cast<const uint32_t*>(t->levels_dev + t->level_elems) : nullptr;
  a.lv_top_len = 8 * t->top_n;
  a.levels = t->levels;
  if (t->node_width == eos::kPackedNode) {  // X, then the nodes
    a.kv = t->nodes_dev;
    a.lv_top_len = t->n;
    a.sh = t->sh;
  }
  // Vector body needs Y+head 16-B aligned and out+head 8-B aligned.
  const uintptr_t ya = (uintptr_t)Y, oa = (uintptr_t)out;
  a.head = (ya & 15) ? 1 : 0;
  a.vec_ok = ((ya & 7) == 0) && (((oa + 4 * (uintptr_t)a.head) & 7) == 0) && count > a.head;
  // One CTA per tile (CLC work stealing keeps ~#SM x occupancy of them
  // resident); the static schedule uses a persistent grid instead.
  // large launches with an aligned vector body: the shared-memory ring
  if (!cnt && t->fn_ring && a.vec_ok &&
      (count - a.head) / ring_stage() >= kRingMinStagesPerSm * t->num_sms) {
    a.ring_ns = t->ring_ns;
    const int64_t st = ((count - a.head) / 2 * 2 + ring_stage() - 1) / ring_stage();
    a.ntiles = st;
    void* params[] = {&a};  // one CTA per tile (cluster launch control, kernels.cuh ring_body)
    EOS_CUDA(launch(t->fn_ring, st, 1024, (size_t)t->ring_smem, st_, params));
    count_launch();
    return EOS_OK;
  }
  int64_t per_tile = (int64_t)t->threads[cnt] * t->unroll[cnt] * 2;
  int64_t tiles = (count - a.head + per_tile - 1) / per_tile;
  // fewer tiles than half the SMs: the small-tile shape spreads the launch over 4x more CTAs
  const bool sm = !cnt && t->fn_small && 2 * tiles < t->num_sms;
  if (sm) {
    per_tile = (int64_t)t->threads_small * t->unroll_small * 2;
    tiles = (count - a.head + per_tile - 1) / per_tile;
  }
  if (tiles > 0x7FFFFFFF) return EOS_ERR_SIZE;  // > 2^31 tiles (~4.4e12 targets) per call
  a.ntiles = tiles;
  const bool clc = sm ? t->clc_small : t->clc[cnt];
  int64_t grid = clc ? tiles : std::min<int64_t>(sm ? t->grid_small : t->grid[cnt], tiles);
  grid = std::max<int64_t>(grid, 1);
  void* params[] = {&a};
  EOS_CUDA(launch(sm ? t->fn_small : t->fn[cnt], grid, sm ? t->threads_small : t->threads[cnt],
                  (size_t)t->smem_bytes, st, params));
  count_launch();
  return EOS_OK;
}

}  // namespace

extern "C" {

static int kind_of_k(int32_t k) { return k == EOS_K_AUTO ? EOS_HASH_AUTO : EOS_HASH_EXPONENT; }

eos_status eos_plan_table(const double* table_host, int64_t n, int32_t k, eos_table_info_t* info,
                          uint32_t* dir_out, int64_t cap) {
  if (k != EOS_K_AUTO && k < 0) return EOS_ERR_UNSUPPORTED;
  return eos_plan_table_hash(table_host, n, kind_of_k(k), k, info, dir_out, cap);
}

eos_status eos_plan_table_hash(const double* table_host, int64_t n, int32_t kind, int64_t param,
                               eos_table_info_t* info, uint32_t* dir_out, int64_t cap) {
  if (!info) return EOS_ERR_NULL;
  TablePlan p;
  eos_status st = eos::plan_table(table_host, n, kind, param, false, &p, 0, EOS_MAX_TABLE, true);
  if (st != EOS_OK) return st;
  if (dir_out) {
    if (cap < p.bins) return EOS_ERR_SIZE;
    memcpy(dir_out, p.dir.data(), 4 * (size_t)p.bins);
  }
  eos::fill_info(p, info);
  return EOS_OK;
}

eos_status eos_search_create_ex(const double* table_host, int64_t n, int32_t k, eos_table* out) {
  if (k != EOS_K_AUTO && k < 0) return EOS_ERR_UNSUPPORTED;
  return eos_search_create_hash(table_host, n, kind_of_k(k), k, out);
}

eos_status eos_search_create_hash(const double* table_host, int64_t n, int32_t kind, int64_t param,
                                  eos_table* out) {
  return eos_search_create_levels(table_host, n, EOS_LEVELS_AUTO, kind, param, out);
}

// Packed plan for levels = EOS_LEVELS_PACKED, or EOS_LEVELS_AUTO above
// EOS_MAX_TABLE with the automatic hash (an explicit hash is honoured by the
// 8-ary levels).  *use = false: take the other structures (AUTO and the packed
// plan does not fit, or levels >= 0).
static eos_status try_packed(const double* table_host, int64_t n, int32_t levels, int32_t kind,
                             eos::PackedPlan* pp, bool* use) {
  *use = false;
  // AUTO: packed where the 8-ary structure needs two or more levels, i.e. two
  // or more L2 gathers per lookup (n > 8 kMaxTopKeys), and the packed depth is
  // not larger than the 8-ary depth; one 8-ary level beats a packed table's
  // deeper sample bins
  const bool explicit_depth =
      levels <= EOS_LEVELS_PACKED_DEPTH(1) && levels >= EOS_LEVELS_PACKED_DEPTH(eos::kPackedMaxDepth);
  const bool auto_packed = levels == EOS_LEVELS_AUTO && kind == EOS_HASH_AUTO && n > 8 * eos::kMaxTopKeys;
  if (levels != EOS_LEVELS_PACKED && !explicit_depth && !auto_packed) return EOS_OK;
  if (auto_packed && n > EOS_MAX_TABLE_TIERED) return EOS_OK;  // (plan_tiered reports it)
  const int depth = explicit_depth ? EOS_LEVELS_PACKED_DEPTH(0) - levels : 0;
  const eos_status st = eos::plan_packed(table_host, n, pp, eos::kPackedImageBudget, depth);
  if (st == EOS_OK) {
    if (auto_packed) {
      int d8 = 1;  // depth of the 8-ary structure: n1 = ceil(n / 8^D) <= kMaxTopKeys
      for (int64_t s = 8; (n + s - 1) / s > eos::kMaxTopKeys; s *= 8) ++d8;
      if (pp->depth > d8) return EOS_OK;
    }
    *use = true;
    return EOS_OK;
  }
  if (auto_packed && (st == EOS_ERR_UNSUPPORTED || st == EOS_ERR_SIZE)) return EOS_OK;
  return st;
}

eos_status eos_plan_table_levels(const double* table_host, int64_t n, int32_t levels, int32_t kind,
                                 int64_t param, eos_table_info_t* info) {
  if (!info) return EOS_ERR_NULL;
  {
    eos::PackedPlan pp;
    bool use = false;
    const eos_status st = try_packed(table_host, n, levels, kind, &pp, &use);
    if (st != EOS_OK) return st;
    if (use) {
      eos::fill_info(pp, info);
      return EOS_OK;
    }
  }
  eos::TieredPlan tp;
  eos_status st = eos::plan_tiered(table_host, n, levels, kind, param, &tp);
  if (st != EOS_OK) return st;
  eos::fill_info(tp, info);
  return EOS_OK;
}

// A packed table's handle: the sample image in smem, X and the nodes in one
// device allocation (X first; the nodes 32-B aligned after it).
static eos_status create_packed(eos::PackedPlan&& pp, eos_table* out) {
  eos_table t = new (std::nothrow) eos_table_s();
  if (!t) return EOS_ERR_NOMEM;
  auto fail = [&](eos_status st) {
    if (t->image_dev) cudaFree(t->image_dev);
    if (t->levels_dev) cudaFree(t->levels_dev);
    delete t;
    return st;
  };
  t->plan = eos::packed_top(pp);
  t->levels = pp.depth;
  t->node_width = eos::kPackedNode;
  t->sh = pp.sh;
  t->n = pp.n;
  t->top_n = pp.n1;
  t->smem_bytes = (int64_t)pp.image.size();
  const int64_t x_bytes = (8 * pp.n + 31) & ~int64_t(31);
  t->level_bytes = x_bytes + 4 * (int64_t)pp.nodes.size();
  dv::AxisParams& a = t->ax;
  a.n = (int32_t)pp.n1;
  a.x_off = 0;
  a.d_off = (int32_t)t->plan.x_bytes;
  a.hb = pp.hb;
  a.M = t->plan.M;
  a.bmax = pp.bmax;
  a.steps = pp.steps;
  a.mode = pp.key_mode;
  a.x0 = pp.x0;
  a.xlast = pp.x_last;
  cudaError_t e = cudaGetDevice(&t->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, t->device);
  if (e != cudaSuccess) return fail(cuda_status(e));
  eos_status st = upload(pp.image, &t->image_dev);
  if (st != EOS_OK) return fail(st);
  e = cudaMalloc((void**)&t->levels_dev, (size_t)t->level_bytes);
  if (e == cudaSuccess) e = cudaMemcpy(t->levels_dev, pp.X.data(), 8 * pp.X.size(), cudaMemcpyHostToDevice);
  t->nodes_dev = reinterpret_cast<const uint32_t*>(reinterpret_cast<char*>(t->levels_dev) + x_bytes);
  if (e == cudaSuccess)
    e = cudaMemcpy((void*)t->nodes_dev, pp.nodes.data(), 4 * pp.nodes.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(cuda_status(e));
  const int mode = pp.key_mode, S = pp.steps;
  t->fn[0] = pp.depth == 1 ? packed_fn_mode<dv::ShapeTiered, false, false>(mode, S)
                           : packed_fn_mode<dv::ShapeTiered, false>(mode, S);
  t->threads[0] = dv::ShapeTiered::kThreads;
  t->unroll[0] = dv::ShapeTiered::kUnroll;
  t->clc[0] = dv::ShapeTiered::kClc;
  t->fn[1] = packed_fn_mode<dv::ShapeCnt, true>(mode, S);
  t->threads[1] = dv::ShapeCnt::kThreads;
  t->unroll[1] = dv::ShapeCnt::kUnroll;
  t->clc[1] = dv::ShapeCnt::kClc;
  for (int c = 0; c < 2 && st == EOS_OK; ++c)
    st = configure(t->fn[c], t->threads[c], t->smem_bytes, t->num_sms, &t->grid[c],
                   c == 0 ? &t->ctas_per_sm : nullptr);
  if (st != EOS_OK) return fail(st);
  if (!exp_small_off()) {
    using SS = dv::Shape<512, 1, 1, false>;
    const void* fs = packed_fn_mode<SS, false>(mode, S);
    if (configure(fs, SS::kThreads, t->smem_bytes, t->num_sms, &t->grid_small, nullptr) == EOS_OK) {
      t->fn_small = fs;
      t->threads_small = SS::kThreads;
      t->unroll_small = SS::kUnroll;
      t->clc_small = SS::kClc;
    }
  }
  *out = t;
  return EOS_OK;
}

eos_status eos_search_create_levels(const double* table_host, int64_t n, int32_t levels,
                                    int32_t kind, int64_t param, eos_table* out) {
  if (!out) return EOS_ERR_NULL;
  *out = nullptr;
  {
    eos::PackedPlan pp;
    bool use = false;
    const eos_status st = try_packed(table_host, n, levels, kind, &pp, &use);
    if (st != EOS_OK) return st;
    if (use) return create_packed(std::move(pp), out);
  }
  eos_table t = new (std::nothrow) eos_table_s();
  if (!t) return EOS_ERR_NOMEM;
  std::vector<double> lv;
  std::vector<uint32_t> keys;
  {
    eos::TieredPlan tp;
    eos_status st = eos::plan_tiered(table_host, n, levels, kind, param, &tp);
    if (st != EOS_OK) { delete t; return st; }
    t->plan = std::move(tp.top);
#ifdef EOS_EXPERIMENTS
    if (tp.levels == 0) exp_layout(&t->plan);
#endif
    t->levels = tp.levels;
    t->node_width = tp.levels > 0 ? 8 : 0;
    t->n = tp.n;
    t->top_n = tp.top_n;
    t->level_bytes = 12 * tp.level_elems();
    lv = std::move(tp.lv);
    keys = std::move(tp.keys);
    t->ax = axis_params(t->plan, 0);
    t->ax.xlast = tp.x_last;  // X[n-1] of the full table (counter c4)
    if (t->levels > 0) {  // the sample table is staged as 32-bit keys
      t->ax.d_off = (int32_t)((4 * t->plan.n + 15) & ~int64_t(15));
      t->smem_bytes = eos::key_image_bytes(t->plan);
    } else {
      t->smem_bytes = t->plan.image_bytes;
    }
  }
  auto fail = [&](eos_status st) {
    if (t->image_dev) cudaFree(t->image_dev);
    if (t->levels_dev) cudaFree(t->levels_dev);
    delete t;
    return st;
  };
  cudaError_t e = cudaGetDevice(&t->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, t->device);
  if (e != cudaSuccess) return fail(cuda_status(e));
  eos_status st = upload(t->levels > 0 ? eos::make_key_image(t->plan) : eos::make_image(t->plan),
                         &t->image_dev);
  if (st != EOS_OK) return fail(st);
  if (t->levels > 0) {
    // [F levels fp64][K levels u32], both coarsest first
    e = cudaMalloc((void**)&t->levels_dev, (size_t)t->level_bytes);
    if (e == cudaSuccess)
      e = cudaMemcpy(t->levels_dev, lv.data(), 8 * lv.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(reinterpret_cast<char*>(t->levels_dev) + 8 * lv.size(), keys.data(),
                     4 * keys.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(cuda_status(e));
    t->level_elems = (int64_t)lv.size();
    std::vector<double>().swap(lv);
    std::vector<uint32_t>().swap(keys);
  }
  for (int c = 0; c < 2 && st == EOS_OK; ++c) {
    const bool cnt = c == 1;
    LaunchShape ls;
    if (t->levels > 0) {
      using SH = dv::ShapeTiered;
      ls.fn = t->plan.key_mode == 0 ? tiered_fn_mode<0, SH>(t->plan.steps, cnt)
                                    : tiered_fn_mode<1, SH>(t->plan.steps, cnt);
      ls.threads = cnt ? dv::ShapeCnt::kThreads : SH::kThreads;
      ls.unroll = cnt ? dv::ShapeCnt::kUnroll : SH::kUnroll;
      ls.clc = cnt ? dv::ShapeCnt::kClc : SH::kClc;
    } else if (cnt) {
      ls = {counters_fn(t->plan), dv::ShapeCnt::kThreads, dv::ShapeCnt::kUnroll, dv::ShapeCnt::kClc};
    } else {
      ls = pick_search(t->plan, t->smem_bytes);
    }
#ifdef EOS_EXPERIMENTS
    if (!cnt) exp_variant(t->plan, t->levels > 0, &ls);
#endif
    t->fn[c] = ls.fn;
    t->threads[c] = ls.threads;
    t->unroll[c] = ls.unroll;
    t->clc[c] = ls.clc;
    st = configure(t->fn[c], t->threads[c], t->smem_bytes, t->num_sms, &t->grid[c],
                   c == 0 ? &t->ctas_per_sm : nullptr);
  }
  if (st != EOS_OK) return fail(st);
  if (t->levels > 0 && !exp_small_off()) {
    const void* fs = t->plan.key_mode == 0 ? tiered_small_fn<0>(t->plan.steps)
                                           : tiered_small_fn<1>(t->plan.steps);
    if (fs && configure(fs, 512, t->smem_bytes, t->num_sms, &t->grid_small, nullptr) == EOS_OK) {
      t->fn_small = fs;
      t->threads_small = 512;
      t->unroll_small = 1;
      t->clc_small = false;
    }
  }
  if (t->levels == 0 && ring_fn(t->plan)) {  // the ring kernel: as many stages as fit
    const void* fr = ring_fn(t->plan);
    const int64_t img = (t->smem_bytes + 127) & ~int64_t(127);
    for (int ns = exp_ring(dv::kRingMaxStages); ns >= 2; --ns) {
      const int64_t smem = img + (int64_t)ns * ring_stage() * 8;
      int per_sm = 0;
      if (configure(fr, 1024, smem, t->num_sms, &t->grid_ring, &per_sm) == EOS_OK && per_sm >= 1) {
        t->fn_ring = fr;
        t->ring_ns = ns;
        t->ring_smem = smem;
        break;
      }
    }
  }
  if (t->levels == 0 && !exp_small_off()) {
    const LaunchShape ls = pick_search_small(t->plan, t->smem_bytes);
    if (ls.fn && configure(ls.fn, ls.threads, t->smem_bytes, t->num_sms, &t->grid_small,
                           nullptr) == EOS_OK) {
      t->fn_small = ls.fn;
      t->threads_small = ls.threads;
      t->unroll_small = ls.unroll;
      t->clc_small = ls.clc;
    }
  }
  *out = t;
  return EOS_OK;
}

eos_status eos_search_create(const double* table_host, int64_t n, eos_table* out) {
  return eos_search_create_ex(table_host, n, EOS_K_AUTO, out);
}

eos_status eos_search_ex(eos_table t, const double* targets_dev, int64_t count,
                         int32_t* idx_out_dev, int64_t global_offset, uint64_t* counters_dev,
                         void* stream) {
  if (!t) return EOS_ERR_NULL;
  if (count < 0 || count > (int64_t(1) << 62)) return EOS_ERR_SIZE;
  if (count == 0) return EOS_OK;
  if (!targets_dev || !idx_out_dev) return EOS_ERR_NULL;
  if (overlaps(targets_dev, 8 * count, idx_out_dev, 4 * count)) return EOS_ERR_ALIAS;
  eos_status st = check_device(t->device);
  if (st != EOS_OK) return st;
  return launch_search(t, targets_dev, count, idx_out_dev, global_offset, counters_dev,
                       (cudaStream_t)stream);
}

eos_status eos_search(eos_table t, const double* targets_dev, int64_t count, int32_t* idx_out_dev,
                      void* stream) {
  return eos_search_ex(t, targets_dev, count, idx_out_dev, 0, nullptr, stream);
}

eos_status eos_search_host(eos_table t, const double* targets_host, int64_t count,
                           int32_t* idx_out_host, void* stream) {
  if (!t) return EOS_ERR_NULL;
  if (count < 0 || count > (int64_t(1) << 62)) return EOS_ERR_SIZE;
  if (count == 0) return EOS_OK;
  if (!targets_host || !idx_out_host) return EOS_ERR_NULL;
  if (overlaps(targets_host, 8 * count, idx_out_host, 4 * count)) return EOS_ERR_ALIAS;
  eos_status st = check_device(t->device);
  if (st != EOS_OK) return st;
  const int64_t chunk = int64_t(1) << 23;  // 8 Mi targets: 64 MiB in + 32 MiB out per slot
  return host_pipeline(
      (cudaStream_t)stream, count, chunk, 12,
      [&](cudaStream_t s, char* stage, int64_t slot_elems, int64_t off, int64_t len) -> eos_status {
        double* dY = (double*)stage;
        int32_t* dI = (int32_t*)(stage + 8 * slot_elems);
        EOS_CUDA(cudaMemcpyAsync(dY, targets_host + off, 8 * len, cudaMemcpyHostToDevice, s));
        eos_status r = launch_search(t, dY, len, dI, off, nullptr, s);
        if (r != EOS_OK) return r;
        EOS_CUDA(cudaMemcpyAsync(idx_out_host + off, dI, 4 * len, cudaMemcpyDeviceToHost, s));
        return EOS_OK;
      });
}

eos_status eos_search_direct(const double* table_dev, int64_t n, const double* targets_dev,
                             int64_t count, int32_t* idx_out_dev, int32_t* status_dev,
                             void* stream) {
  if (n < 1 || n > dv::kDirectMaxTable) return EOS_ERR_SIZE;
  if (count < 0 || count > (int64_t(1) << 62)) return EOS_ERR_SIZE;
  if (!table_dev) return EOS_ERR_NULL;
  if (count == 0) return EOS_OK;
  if (!targets_dev || !idx_out_dev) return EOS_ERR_NULL;
  if (overlaps(targets_dev, 8 * count, idx_out_dev, 4 * count) ||
      overlaps(table_dev, 8 * n, idx_out_dev, 4 * count))
    return EOS_ERR_ALIAS;
  int dev = 0;
  EOS_CUDA(cudaGetDevice(&dev));
  using SH = dv::ShapeDirect;
  const void* fn = (const void*)dv::search1d_direct_kernel<SH>;
  int32_t bins_max = 1;
#ifndef EOS_DIRECT_BINS_PER_ENTRY
#define EOS_DIRECT_BINS_PER_ENTRY 4
#endif
  while (bins_max < EOS_DIRECT_BINS_PER_ENTRY * n && bins_max < dv::kDirectMaxBins) bins_max <<= 1;
  const int64_t smem = ((8 * n + 15) & ~int64_t(15)) + 4 * (int64_t)bins_max;
  {  // one-time per device: allow the largest dynamic smem this kernel uses
    static std::mutex mu;
    static bool done[64] = {false};
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 64 && !done[dev]) {
      const int64_t mx = ((8 * dv::kDirectMaxTable + 15) & ~int64_t(15)) + 4 * dv::kDirectMaxBins;
      EOS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx));
      done[dev] = true;
    }
  }
  dv::DirectArgs a{};
  a.table = table_dev;
  a.n = (int32_t)n;
  a.bins_max = bins_max;
  a.status = status_dev;
  a.s.Y = targets_dev;
  a.s.out = idx_out_dev;
  a.s.count = count;
  const uintptr_t ya = (uintptr_t)targets_dev, oa = (uintptr_t)idx_out_dev;
  a.s.head = (ya & 15) ? 1 : 0;
  a.s.vec_ok = ((ya & 7) == 0) && (((oa + 4 * (uintptr_t)a.s.head) & 7) == 0) && count > a.s.head;
  const int64_t per_tile = (int64_t)SH::kTileElems;
  const int64_t tiles = (count - a.s.head + per_tile - 1) / per_tile;
  if (tiles > 0x7FFFFFFF) return EOS_ERR_SIZE;
  a.s.ntiles = tiles;
  void* params[] = {&a};
  EOS_CUDA(launch(fn, std::max<int64_t>(tiles, 1), SH::kThreads, (size_t)smem,
                  (cudaStream_t)stream, params));
  count_launch();
  return EOS_OK;
}

eos_status eos_table_info(eos_table t, eos_table_info_t* out) {
  if (!t || !out) return EOS_ERR_NULL;
  eos::fill_info(t->plan, out);
  out->n = t->n;
  out->levels = t->levels;
  out->node_width = t->node_width;
  out->top_n = t->top_n;
  out->level_bytes = t->level_bytes;
  out->image_bytes = t->smem_bytes;
  out->device = t->device;
  out->ctas_per_sm = t->ctas_per_sm;
  out->ring_stages = t->fn_ring ? t->ring_ns : 0;
  return EOS_OK;
}

eos_status eos_search_destroy(eos_table t) {
  if (!t) return EOS_ERR_NULL;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != t->device) cudaSetDevice(t->device);
  cudaError_t e = cudaFree(t->image_dev);  // synchronises with in-flight work
  if (t->levels_dev) {
    cudaError_t e2 = cudaFree(t->levels_dev);
    if (e == cudaSuccess) e = e2;
  }
  if (cur != t->device && cur >= 0) cudaSetDevice(cur);
  delete t;
  return cuda_status(e);
}

}  // extern "C"
