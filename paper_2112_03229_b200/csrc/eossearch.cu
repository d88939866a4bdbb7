// eossearch.cu -- the C ABI of include/eossearch.h: handle management, device
// image upload, launch configuration and the end-to-end host-buffer pipelines.
// Product path (never includes or links oracle/).
//
// Tuning knobs, read at create / first use, for A/B experiments only (the
// defaults are the measured best):
//   EOS_SEARCH_VARIANT, EOS_TIERED_VARIANT  launch-shape variants by name
//   EOS_INTERP_VARIANT                      2-D launch variants by number
//   EOS_INTERP_REP=0                        2-D plain axes (no cell records)
//   EOS_GG_SMEM_KB                          smem cap of device-memory grids
//   EOS_PDL (0/1)                           programmatic dependent launch
//   EOS_HOST_SLOTS, EOS_HOST_CHUNK_LOG2     host-buffer pipeline depth / chunk
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <new>
#include <vector>

#include "eos_internal.h"
#include "eossearch.h"
#include "kernels.cuh"

using eos::TablePlan;
namespace dv = eos::dev;

static std::atomic<int64_t> g_launches{0};

struct eos_table_s {
  TablePlan plan;          // the shared-memory table (T1 of a tiered table)
  int levels = 0;          // D (tiered tables, eos_search_create_levels)
  int64_t n = 0;           // entries of the full table
  int64_t top_n = 0;       // n1
  int64_t level_bytes = 0;
  int64_t level_elems = 0;
  double* levels_dev = nullptr;  // the 8-ary levels: F (fp64) then K (u32), coarsest first
  int device = -1;
  int num_sms = 0;
  void* image_dev = nullptr;
  dv::AxisParams ax{};
  // launch configuration per counters on/off
  const void* fn[2] = {nullptr, nullptr};
  int grid[2] = {0, 0};
  int threads[2] = {256, 256};
  int unroll[2] = {4, 4};
  bool clc[2] = {true, true};
  int ctas_per_sm = 0;
};

struct eos_grid2d_s {
  TablePlan pr, pt;
  int device = -1;
  int num_sms = 0;
  void* image_dev = nullptr;
  int64_t image_bytes = 0;
  int32_t g_off = 0;
  dv::AxisParams ar{}, at{};
  const void* fn = nullptr;
  const void* fn_deriv = nullptr;
  int grid = 0, grid_deriv = 0;
  int threads_deriv = dv::Shape2DDeriv::kThreads, unroll_deriv = dv::Shape2DDeriv::kUnroll;
  int threads = 512, unroll = 2;
  bool clc = true;
  int32_t flags = 0;
  int32_t wr_off = 0, wt_off = 0, lr_off = 0, lt_off = 0;
  int32_t rr_off = 0, rt_off = 0;
  int rep = 0;  // 2: bank-pinned cell records in the image (REP kernels), 0: plain axes
  int32_t rep_shift = 0;       // REP 2: log2 of the record copies
  int64_t rep_bytes_axis = 0;  // image bytes per axis entry of the REP layout
  bool gg = false;          // grid in device memory (GG kernels)
  void* grid_dev = nullptr;  // GG: row pairs (double2[n_rho (n_T - 1)])
  int64_t grid_bytes = 0;
};

namespace {

// ---------------------------------------------------------- kernel table ---
template <int S, int MODE, class SH>
const void* search_fn(bool cnt) {
  return cnt ? (const void*)dv::search1d_kernel<S, MODE, true, SH>
             : (const void*)dv::search1d_kernel<S, MODE, false, SH>;
}

template <int MODE, class SH>
const void* search_fn_mode(int steps, bool cnt) {
  switch (steps) {
    case 1: return search_fn<1, MODE, SH>(cnt);
    case 2: return search_fn<2, MODE, SH>(cnt);
    case 3: return search_fn<3, MODE, SH>(cnt);
    case 4: return search_fn<4, MODE, SH>(cnt);
    case 5: return search_fn<5, MODE, SH>(cnt);
    case 6: return search_fn<6, MODE, SH>(cnt);
    case 7: return search_fn<7, MODE, SH>(cnt);
    case 8: return search_fn<8, MODE, SH>(cnt);
    default: return search_fn<0, MODE, SH>(cnt);  // runtime S
  }
}

template <class SH>
const void* search_fn_shape(int mode, int steps, bool cnt) {
  return mode == 0 ? search_fn_mode<0, SH>(steps, cnt) : search_fn_mode<1, SH>(steps, cnt);
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

// Launch-shape variants of the tiered kernel (EOS_TIERED_VARIANT=<name>,
// tuning experiments; mode 0, no counters, S <= 4).
template <class SH>
const void* tiered_variant_fn(int steps) {
  switch (steps) {
    case 1: return (const void*)dv::search1d_tiered_kernel<1, 0, false, SH>;
    case 2: return (const void*)dv::search1d_tiered_kernel<2, 0, false, SH>;
    case 3: return (const void*)dv::search1d_tiered_kernel<3, 0, false, SH>;
    case 4: return (const void*)dv::search1d_tiered_kernel<4, 0, false, SH>;
    default: return nullptr;
  }
}

struct LaunchShape {
  const void* fn;
  int threads, unroll;
  bool clc;
};

// Default launch shape by image size: as many threads per SM as registers
// allow (~1024 at <= 64 regs), with all image copies of an SM <= ~144 KB of
// smem so L1 keeps room for the in-flight streaming loads.
// One 1024-thread CTA per SM (images > 72 KB) always takes the static
// schedule: its per-tile CTA barrier makes CLC 13-15% slower there even at
// S <= 2 (n = 4096 log-uniform, 143 KB image: 443 -> 508 Glookups/s;
// profiles/r01_exp_table_size.json).
LaunchShape pick_search(int mode, int steps, bool cnt, int64_t image_bytes) {
  if (cnt) return {search_fn_shape<dv::ShapeCnt>(mode, steps, true), 256, 4, true};
  if (image_bytes > 72 * 1024)
    return {search_fn_shape<dv::ShapeDeepBig>(mode, steps, false), 1024, 4, false};
  if (steps >= 3)
    return {search_fn_shape<dv::ShapeDeepMid>(mode, steps, false), 512, 4, false};
  if (image_bytes <= 32 * 1024)
    return {search_fn_shape<dv::ShapeSmall>(mode, steps, false), 256, 4, true};
  return {search_fn_shape<dv::ShapeMid>(mode, steps, false), 512, 4, true};
}

// Launch-shape variants for tuning experiments (EOS_SEARCH_VARIANT=<name> at
// create time; mode 0, S <= 4, no counters).  Not part of the C ABI.
struct Variant {
  const char* name;
  int threads, unroll;
  bool clc;
  const void* (*get)(int steps);
};

template <class SH>
const void* variant_fn(int steps) {
  switch (steps) {
    case 1: return (const void*)dv::search1d_kernel<1, 0, false, SH>;
    case 2: return (const void*)dv::search1d_kernel<2, 0, false, SH>;
    case 3: return (const void*)dv::search1d_kernel<3, 0, false, SH>;
    case 4: return (const void*)dv::search1d_kernel<4, 0, false, SH>;
    default: return nullptr;
  }
}

const Variant kTieredVariants[] = {
    {"static512u4", 512, 4, false, tiered_variant_fn<dv::Shape<512, 4, 1, false>>},
    {"static1024u2", 1024, 2, false, tiered_variant_fn<dv::Shape<1024, 2, 1, false>>},
    {"clc1024u2", 1024, 2, true, tiered_variant_fn<dv::Shape<1024, 2, 1, true>>},
    {"static1024u1", 1024, 1, false, tiered_variant_fn<dv::Shape<1024, 1, 1, false>>},
};

const Variant kVariants[] = {
    {"static256u4", 256, 4, false, variant_fn<dv::Shape<256, 4, 4, false>>},
    {"static512u4", 512, 4, false, variant_fn<dv::Shape<512, 4, 2, false>>},
    {"clc256u4", 256, 4, true, variant_fn<dv::Shape<256, 4, 4, true>>},
    {"clc256u8", 256, 8, true, variant_fn<dv::Shape<256, 8, 4, true>>},
    {"clc256u2", 256, 2, true, variant_fn<dv::Shape<256, 2, 4, true>>},
    {"clc512u4", 512, 4, true, variant_fn<dv::Shape<512, 4, 2, true>>},
    {"clc512u2", 512, 2, true, variant_fn<dv::Shape<512, 2, 2, true>>},
    {"clc1024u4", 1024, 4, true, variant_fn<dv::Shape<1024, 4, 1, true>>},
    {"clc1024u2", 1024, 2, true, variant_fn<dv::Shape<1024, 2, 1, true>>},
    {"clc128u8", 128, 8, true, variant_fn<dv::Shape<128, 8, 8, true>>},
    {"static1024u4", 1024, 4, false, variant_fn<dv::Shape<1024, 4, 1, false>>},
};

template <int S>
const void* interp_fn_s(int variant) {
  switch (variant) {
    case 1: return (const void*)dv::interp2d_kernel<S, dv::Shape<512, 2, 1, false>, false, false>;
    case 2: return (const void*)dv::interp2d_kernel<S, dv::Shape<1024, 2, 1, false>, false, false>;
    case 3: return (const void*)dv::interp2d_kernel<S, dv::Shape<512, 4, 1, false>, false, false>;
    case 4: return (const void*)dv::interp2d_kernel<S, dv::Shape<512, 2, 1, true>, false, false>;
    case 5: return (const void*)dv::interp2d_kernel<S, dv::Shape<512, 2, 1, false>, true, false>;
    case 6: return (const void*)dv::interp2d_kernel<S, dv::Shape<1024, 1, 1, false>, true, false>;
    case 11: return (const void*)dv::interp2d_kernel<S, dv::Shape2D, false, false, false, 2>;
    default: return (const void*)dv::interp2d_kernel<S, dv::Shape2D, false, false>;
  }
}

template <int S>
const void* interp_deriv_fn_s(int rep) {
  switch (rep) {
    case 2: return (const void*)dv::interp2d_kernel<S, dv::Shape2DDeriv, false, true, false, 2>;
    default: return (const void*)dv::interp2d_kernel<S, dv::Shape2DDeriv, false, true>;
  }
}

template <int S>
const void* interp_loglog_fn_s(bool deriv, bool rep) {
  if (rep)
    return deriv ? (const void*)dv::interp2d_kernel<S, dv::Shape2DDeriv, false, true, true, 2>
                 : (const void*)dv::interp2d_kernel<S, dv::Shape2D, false, false, true, 2>;
  return deriv ? (const void*)dv::interp2d_kernel<S, dv::Shape2DDeriv, false, true, true>
               : (const void*)dv::interp2d_kernel<S, dv::Shape2D, false, false, true>;
}

struct Interp2DShape {
  const void* fn;
  const void* fn_deriv;  // with dP/drho and dP/dT outputs (Shape2DDeriv, static schedule)
  int threads, unroll;
  bool clc;
};

// EOS_INTERP_VARIANT (tuning experiments only): 0 static1024u1 (default
// without bank-pinned cell records), 1 static512u2, 2 static1024u2,
// 3 static512u4, 4 clc512u2, 5 static512u2+recip, 6 static1024u1+recip,
// 11 static1024u1 with bank-pinned cell records (REP 2, the default when they
// fit).
template <bool LOGLOG, int REP, int S>
Interp2DShape gg_shape() {
  return {(const void*)dv::interp2d_kernel<S, dv::Shape2D, false, false, LOGLOG, REP, true>,
          (const void*)dv::interp2d_kernel<S, dv::Shape2DDeriv, false, true, LOGLOG, REP, true>,
          dv::Shape2D::kThreads, dv::Shape2D::kUnroll, dv::Shape2D::kClc};
}

// Grids in device memory (GG): S = 1 or the runtime-S instantiation.
template <bool LOGLOG, int REP>
Interp2DShape gg_pick(int steps) {
  return steps == 1 ? gg_shape<LOGLOG, REP, 1>() : gg_shape<LOGLOG, REP, 0>();
}

Interp2DShape pick_interp(int steps, bool loglog, int rep, bool gg) {
  if (gg) {
    if (loglog) return rep == 2 ? gg_pick<true, 2>(steps) : gg_pick<true, 0>(steps);
    if (rep == 2) return gg_pick<false, 2>(steps);
    return gg_pick<false, 0>(steps);
  }
  if (loglog) {
    const void *fn, *fd;
    const bool r2 = rep == 2;
    switch (steps) {
      case 1: fn = interp_loglog_fn_s<1>(false, r2); fd = interp_loglog_fn_s<1>(true, r2); break;
      case 2: fn = interp_loglog_fn_s<2>(false, r2); fd = interp_loglog_fn_s<2>(true, r2); break;
      case 3: fn = interp_loglog_fn_s<3>(false, r2); fd = interp_loglog_fn_s<3>(true, r2); break;
      case 4: fn = interp_loglog_fn_s<4>(false, r2); fd = interp_loglog_fn_s<4>(true, r2); break;
      default: fn = interp_loglog_fn_s<0>(false, r2); fd = interp_loglog_fn_s<0>(true, r2); break;
    }
    return {fn, fd, dv::Shape2D::kThreads, dv::Shape2D::kUnroll, dv::Shape2D::kClc};
  }
  const int vdef = rep == 2 ? 11 : 0;
  int v = vdef;
  if (const char* e = getenv("EOS_INTERP_VARIANT")) v = atoi(e);
  static const int thr[12] = {1024, 512, 1024, 512, 512, 512, 1024, 0, 0, 0, 0, 1024};
  static const int unr[12] = {1, 2, 2, 4, 2, 2, 1, 0, 0, 0, 0, 1};
  static const bool clc[12] = {false, false, false, false, true, false, false,
                               false, false, false, false, false};
  // variants 10/11 need the image of the matching REP layout
  if (v < 0 || v > 11 || thr[v] == 0 || (v >= 10 && v != vdef)) v = vdef;
  const void* fn;
  const void* fd;
  switch (steps) {
    case 1: fn = interp_fn_s<1>(v); fd = interp_deriv_fn_s<1>(rep); break;
    case 2: fn = interp_fn_s<2>(v); fd = interp_deriv_fn_s<2>(rep); break;
    case 3: fn = interp_fn_s<3>(v); fd = interp_deriv_fn_s<3>(rep); break;
    case 4: fn = interp_fn_s<4>(v); fd = interp_deriv_fn_s<4>(rep); break;
    default: fn = interp_fn_s<0>(v); fd = interp_deriv_fn_s<0>(rep); break;
  }
  return {fn, fd, thr[v], unr[v], clc[v]};
}

dv::AxisParams axis_params(const TablePlan& p, int32_t x_off) {
  dv::AxisParams a{};
  a.n = (int32_t)p.n;
  a.x_off = x_off;
  a.d_off = x_off + (int32_t)p.x_bytes;
  a.hb = p.hb;
  a.M = p.M;
  a.bmax = p.bmax;
  a.steps = std::max(p.steps, 1);
  a.mode = p.key_mode;
  a.x0 = p.X[0];
  a.xlast = p.X[p.n - 1];
  return a;
}

eos_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return EOS_OK;
  if (e == cudaErrorMemoryAllocation) return EOS_ERR_NOMEM;
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return EOS_ERR_DEVICE;
  return EOS_ERR_CUDA;
}

#define EOS_CUDA(call)                              \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) return cuda_status(e_);  \
  } while (0)

eos_status check_device(int device) {
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_status(e);
  return cur == device ? EOS_OK : EOS_ERR_DEVICE;
}

bool overlaps(const void* a, int64_t abytes, const void* b, int64_t bbytes) {
  uintptr_t a0 = (uintptr_t)a, b0 = (uintptr_t)b;
  return a0 < b0 + (uintptr_t)bbytes && b0 < a0 + (uintptr_t)abytes;
}

// Configure a kernel for `smem` bytes of dynamic shared memory and return the
// persistent grid (#SM x resident CTAs per SM).
// The dynamic-smem limit is a per-function attribute shared by every handle
// that uses the same kernel instantiation, so it is raised to the device's
// opt-in maximum (never lowered to one table's size: a later, smaller table
// must not break launches of an earlier, larger one).  Occupancy still
// follows the actual per-launch size.
eos_status configure(const void* fn, int threads, int64_t smem, int num_sms, int* grid, int* per_sm) {
  int dev = 0, optin = 0;
  EOS_CUDA(cudaGetDevice(&dev));
  EOS_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  EOS_CUDA(cudaFuncGetAttributes(&fa, fn));
  const int64_t limit = (int64_t)optin - (int64_t)fa.sharedSizeBytes;
  if (smem > limit) return EOS_ERR_UNSUPPORTED;
  EOS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)limit));
  int occ = 0;
  EOS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, (size_t)smem));
  if (occ < 1) return EOS_ERR_UNSUPPORTED;
  *grid = occ * num_sms;
  if (per_sm) *per_sm = occ;
  return EOS_OK;
}

// Launch with programmatic stream serialization (PDL), so a kernel's prologue
// overlaps the previous kernel in the stream (see pdl_enter in kernels.cuh).
// EOS_PDL=0 disables it (A/B experiments).
cudaError_t launch(const void* fn, int64_t grid, int threads, size_t smem, cudaStream_t st,
                   void** params) {
  static const bool pdl = [] {
    const char* e = getenv("EOS_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, fn, params);
}

eos_status launch_search(eos_table t, const double* Y, int64_t count, int32_t* out, int64_t gofs,
                         uint64_t* counters, cudaStream_t st) {
  const bool cnt = counters != nullptr;
  dv::SearchArgs a{};
  a.image = (const uint4*)t->image_dev;
  a.image_16 = (int32_t)(t->plan.image_bytes / 16);
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
  // Vector body needs Y+head 16-B aligned and out+head 8-B aligned.
  const uintptr_t ya = (uintptr_t)Y, oa = (uintptr_t)out;
  a.head = (ya & 15) ? 1 : 0;
  a.vec_ok = ((ya & 7) == 0) && (((oa + 4 * (uintptr_t)a.head) & 7) == 0) && count > a.head;
  // One CTA per tile (CLC work stealing keeps ~#SM x occupancy of them
  // resident); the static schedule uses a persistent grid instead.
  const int64_t per_tile = (int64_t)t->threads[cnt] * t->unroll[cnt] * 2;
  const int64_t tiles = (count - a.head + per_tile - 1) / per_tile;
  if (tiles > 0x7FFFFFFF) return EOS_ERR_SIZE;  // > 2^31 tiles (~4.4e12 targets) per call
  a.ntiles = tiles;
  int64_t grid = t->clc[cnt] ? tiles : std::min<int64_t>(t->grid[cnt], tiles);
  grid = std::max<int64_t>(grid, 1);
  void* params[] = {&a};
  EOS_CUDA(launch(t->fn[cnt], grid, t->threads[cnt], (size_t)t->plan.image_bytes, st, params));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return EOS_OK;
}

eos_status launch_interp(eos_grid2d g, const double* rho, const double* T, int64_t count,
                         double* P, int32_t* iR, int32_t* iT, double* dPr, double* dPt,
                         cudaStream_t st) {
  const bool deriv = dPr != nullptr || dPt != nullptr;
  dv::Interp2DArgs a{};
  a.image = (const uint4*)g->image_dev;
  a.image_16 = (int32_t)(g->image_bytes / 16);
  a.g_off = g->g_off;
  a.wr_off = g->wr_off;
  a.wt_off = g->wt_off;
  a.lr_off = g->lr_off;
  a.lt_off = g->lt_off;
  a.rr_off = g->rr_off;
  a.rt_off = g->rt_off;
  a.gq = reinterpret_cast<const double2*>(g->grid_dev);
  a.rep_shift = g->rep_shift;
  a.r = g->ar;
  a.t = g->at;
  a.rho = rho;
  a.T = T;
  a.P = P;
  a.iR = iR;
  a.iT = iT;
  a.dPr = dPr;
  a.dPt = dPt;
  a.count = count;
  const uintptr_t al16 =
      (uintptr_t)rho | (uintptr_t)T | (uintptr_t)P | (uintptr_t)dPr | (uintptr_t)dPt;
  const uintptr_t al8 = (uintptr_t)iR | (uintptr_t)iT;
  a.vec_ok = ((al16 & 15) == 0) && ((al8 & 7) == 0);
  const int threads = deriv ? g->threads_deriv : g->threads;
  const int64_t per_tile = (int64_t)threads * (deriv ? g->unroll_deriv : g->unroll) * 2;
  const int64_t tiles = (count + per_tile - 1) / per_tile;
  if (tiles > 0x7FFFFFFF) return EOS_ERR_SIZE;
  a.ntiles = tiles;
  const bool clc = deriv ? dv::Shape2DDeriv::kClc : g->clc;
  int64_t grid = clc ? tiles : std::min<int64_t>(deriv ? g->grid_deriv : g->grid, tiles);
  grid = std::max<int64_t>(grid, 1);
  void* params[] = {&a};
  EOS_CUDA(launch(deriv ? g->fn_deriv : g->fn, grid, threads, (size_t)g->image_bytes, st,
                  params));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return EOS_OK;
}

eos_status upload(const std::vector<uint8_t>& img, void** dev) {
  EOS_CUDA(cudaMalloc(dev, img.size()));
  cudaError_t e = cudaMemcpy(*dev, img.data(), img.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(*dev);
    *dev = nullptr;
    return cuda_status(e);
  }
  return EOS_OK;
}

// Two-stream chunked pipeline over host buffers: chunk c uses slot c % 2 (its
// own stream and device staging), so H2D(c+1) overlaps search(c) / D2H(c).
template <class Body>
eos_status host_pipeline(cudaStream_t caller, int64_t count, int64_t chunk, int64_t bytes_per_elem,
                         Body body) {
  // tuning experiments: EOS_HOST_SLOTS (1..4), EOS_HOST_CHUNK_LOG2 (16..26)
  static const int slots_env = [] {
    const char* e = getenv("EOS_HOST_SLOTS");
    return e ? std::max(1, std::min(4, atoi(e))) : 2;
  }();
  static const int chunk_log2 = [] {
    const char* e = getenv("EOS_HOST_CHUNK_LOG2");
    return e ? std::max(16, std::min(26, atoi(e))) : 0;
  }();
  if (chunk_log2) chunk = (int64_t(1) << chunk_log2) * chunk / (int64_t(1) << 23);
  const int64_t nchunk = (count + chunk - 1) / chunk;
  const int nslot = (int)std::min<int64_t>(nchunk, slots_env);
  const int64_t slot_elems = (std::min(chunk, count) + 63) & ~int64_t(63);  // keeps 16-B alignment
  char* stage = nullptr;
  EOS_CUDA(cudaMallocAsync((void**)&stage, (size_t)(nslot * slot_elems * bytes_per_elem), caller));
  cudaStream_t s[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_start = nullptr, ev_done[4] = {nullptr, nullptr, nullptr, nullptr};
  eos_status st = EOS_OK;
  auto fail = [&](cudaError_t e) { if (st == EOS_OK && e != cudaSuccess) st = cuda_status(e); };
  fail(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
  for (int i = 0; i < nslot && st == EOS_OK; ++i) {
    fail(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
    fail(cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming));
  }
  if (st == EOS_OK) fail(cudaEventRecord(ev_start, caller));
  for (int i = 0; i < nslot && st == EOS_OK; ++i) fail(cudaStreamWaitEvent(s[i], ev_start, 0));
  for (int64_t c = 0; c < nchunk && st == EOS_OK; ++c) {
    const int slot = (int)(c % nslot);
    const int64_t off = c * chunk;
    const int64_t len = std::min(chunk, count - off);
    st = body(s[slot], stage + slot * slot_elems * bytes_per_elem, slot_elems, off, len);
  }
  for (int i = 0; i < nslot; ++i) {
    if (s[i] && ev_done[i]) {
      cudaEventRecord(ev_done[i], s[i]);
      cudaStreamWaitEvent(caller, ev_done[i], 0);
    }
  }
  cudaFreeAsync(stage, caller);
  for (int i = 0; i < nslot; ++i) {
    if (s[i]) cudaStreamDestroy(s[i]);
    if (ev_done[i]) cudaEventDestroy(ev_done[i]);
  }
  if (ev_start) cudaEventDestroy(ev_start);
  return st;
}

}  // namespace

extern "C" {

const char* eos_status_str(eos_status s) {
  switch (s) {
    case EOS_OK: return "ok";
    case EOS_ERR_NULL: return "null pointer or handle";
    case EOS_ERR_SIZE: return "size out of range";
    case EOS_ERR_NONFINITE: return "table or grid value is NaN or infinite";
    case EOS_ERR_UNSORTED: return "table not sorted (axes: not strictly increasing)";
    case EOS_ERR_DEVICE: return "no CUDA device or wrong current device";
    case EOS_ERR_CUDA: return "CUDA runtime error";
    case EOS_ERR_NOMEM: return "out of memory";
    case EOS_ERR_UNSUPPORTED: return "unsupported request";
    case EOS_ERR_ALIAS: return "output overlaps an input";
  }
  return "unknown status";
}

int32_t eos_abi_version(void) { return 2; }

int64_t eos_launch_count(void) { return g_launches.load(); }

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
  eos_status st = eos::plan_table(table_host, n, kind, param, false, &p);
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

eos_status eos_plan_table_levels(const double* table_host, int64_t n, int32_t levels, int32_t kind,
                                 int64_t param, eos_table_info_t* info) {
  if (!info) return EOS_ERR_NULL;
  eos::TieredPlan tp;
  eos_status st = eos::plan_tiered(table_host, n, levels, kind, param, &tp);
  if (st != EOS_OK) return st;
  eos::fill_info(tp, info);
  return EOS_OK;
}

eos_status eos_search_create_levels(const double* table_host, int64_t n, int32_t levels,
                                    int32_t kind, int64_t param, eos_table* out) {
  if (!out) return EOS_ERR_NULL;
  *out = nullptr;
  eos_table t = new (std::nothrow) eos_table_s();
  if (!t) return EOS_ERR_NOMEM;
  std::vector<double> lv;
  std::vector<uint32_t> keys;
  {
    eos::TieredPlan tp;
    eos_status st = eos::plan_tiered(table_host, n, levels, kind, param, &tp);
    if (st != EOS_OK) { delete t; return st; }
    t->plan = std::move(tp.top);
    t->levels = tp.levels;
    t->n = tp.n;
    t->top_n = tp.top_n;
    t->level_bytes = 12 * tp.level_elems();
    lv = std::move(tp.lv);
    keys = std::move(tp.keys);
    t->ax = axis_params(t->plan, 0);
    t->ax.xlast = tp.x_last;  // X[n-1] of the full table (counter c4)
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
  eos_status st = upload(eos::make_image(t->plan), &t->image_dev);
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
    if (t->levels > 0) {
      t->fn[c] = t->plan.key_mode == 0 ? tiered_fn_mode<0, dv::ShapeTiered>(t->plan.steps, cnt)
                                       : tiered_fn_mode<1, dv::ShapeTiered>(t->plan.steps, cnt);
      using SH = dv::ShapeTiered;
      t->threads[c] = cnt ? dv::ShapeCnt::kThreads : SH::kThreads;
      t->unroll[c] = cnt ? dv::ShapeCnt::kUnroll : SH::kUnroll;
      t->clc[c] = cnt ? dv::ShapeCnt::kClc : SH::kClc;
    } else {
      LaunchShape ls = pick_search(t->plan.key_mode, t->plan.steps, cnt, t->plan.image_bytes);
      t->fn[c] = ls.fn;
      t->threads[c] = ls.threads;
      t->unroll[c] = ls.unroll;
      t->clc[c] = ls.clc;
    }
    if (c == 0) {  // tuning experiments: launch-shape variants by name
      const bool tiered = t->levels > 0;
      const char* want = getenv(tiered ? "EOS_TIERED_VARIANT" : "EOS_SEARCH_VARIANT");
      const Variant* vs = tiered ? kTieredVariants : kVariants;
      const size_t nv = tiered ? sizeof(kTieredVariants) / sizeof(Variant)
                               : sizeof(kVariants) / sizeof(Variant);
      for (size_t i = 0; i < nv; ++i) {
        const Variant& v = vs[i];
        if (!want || strcmp(want, v.name) != 0 || t->plan.key_mode != 0) continue;
        const void* f = v.get(t->plan.steps);
        if (!f) break;
        t->fn[0] = f;
        t->threads[0] = v.threads;
        t->unroll[0] = v.unroll;
        t->clc[0] = v.clc;
      }
    }
    st = configure(t->fn[c], t->threads[c], t->plan.image_bytes, t->num_sms, &t->grid[c],
                   c == 0 ? &t->ctas_per_sm : nullptr);
  }
  if (st != EOS_OK) return fail(st);
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
  while (bins_max < 4 * n && bins_max < dv::kDirectMaxBins) bins_max <<= 1;
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
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return EOS_OK;
}

eos_status eos_table_info(eos_table t, eos_table_info_t* out) {
  if (!t || !out) return EOS_ERR_NULL;
  eos::fill_info(t->plan, out);
  out->n = t->n;
  out->levels = t->levels;
  out->top_n = t->top_n;
  out->level_bytes = t->level_bytes;
  out->device = t->device;
  out->ctas_per_sm = t->ctas_per_sm;
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

// -------------------------------------------------------------------- 2-D --
eos_status eos_grid2d_create(const double* rho_host, int64_t n_rho, const double* T_host,
                             int64_t n_T, const double* P_host, eos_grid2d* out) {
  return eos_grid2d_create_ex(rho_host, n_rho, T_host, n_T, P_host, EOS_GRID_LINEAR, out);
}

eos_status eos_grid2d_create_ex(const double* rho_host, int64_t n_rho, const double* T_host,
                                int64_t n_T, const double* P_host, int32_t flags,
                                eos_grid2d* out) {
  if (!out) return EOS_ERR_NULL;
  *out = nullptr;
  if (!rho_host || !T_host || !P_host) return EOS_ERR_NULL;
  if (flags & ~(EOS_GRID_LOGLOG | EOS_GRID_GLOBAL)) return EOS_ERR_UNSUPPORTED;
  const bool loglog = (flags & EOS_GRID_LOGLOG) != 0;
  if (n_rho > 0 && n_T > 0 && n_rho * n_T > EOS_MAX_GRID_CELLS) return EOS_ERR_SIZE;
  eos_grid2d g = new (std::nothrow) eos_grid2d_s();
  if (!g) return EOS_ERR_NOMEM;
  auto fail = [&](eos_status st) {
    if (g->image_dev) cudaFree(g->image_dev);
    if (g->grid_dev) cudaFree(g->grid_dev);
    delete g;
    return st;
  };
  eos_status st = eos::plan_table(rho_host, n_rho, EOS_HASH_AUTO, 0, true, &g->pr);
  if (st == EOS_OK) st = eos::plan_table(T_host, n_T, EOS_HASH_AUTO, 0, true, &g->pt);
  if (st != EOS_OK) return fail(st);
  g->flags = flags;
  const int64_t ncell = n_rho * n_T;
  for (int64_t q = 0; q < ncell; ++q)
    if (!isfinite(P_host[q])) return fail(EOS_ERR_NONFINITE);
  if (loglog) {  // ln of the axes and the grid must exist (R24)
    bool ok = g->pr.X[0] > 0.0 && g->pt.X[0] > 0.0;
    for (int64_t q = 0; q < ncell && ok; ++q) ok = P_host[q] > 0.0;
    if (!ok) return fail(EOS_ERR_UNSUPPORTED);
  }
  // image: [rho X | rho dir][T X | T dir][G][1/dR][1/dT (RECIP variants)][ln R][ln T][R recs][T recs]
  // G is absent for grids in device memory (GG: larger than ~220 KB, or
  // EOS_GRID_GLOBAL), which keep it as row pairs in g->grid_dev instead.
  int64_t r_bytes = g->pr.image_bytes, t_bytes = g->pt.image_bytes;
  // 1/dR, 1/dT arrays: only for the RECIP tuning variants (EOS_INTERP_VARIANT 5, 6)
  const char* ev = getenv("EOS_INTERP_VARIANT");
  const bool recip_arrays = ev && (atoi(ev) == 5 || atoi(ev) == 6);
  const int64_t wr_bytes = recip_arrays ? (8 * (n_rho - 1) + 15) & ~int64_t(15) : 0;
  const int64_t wt_bytes = recip_arrays ? (8 * (n_T - 1) + 15) & ~int64_t(15) : 0;
  const int64_t lr_bytes = loglog ? (8 * n_rho + 15) & ~int64_t(15) : 0;
  const int64_t lt_bytes = loglog ? (8 * n_T + 15) & ~int64_t(15) : 0;
  const int64_t axes_bytes = r_bytes + t_bytes + wr_bytes + wt_bytes + lr_bytes + lt_bytes;
  const int64_t smem_grid_bytes = (8 * ncell + 15) & ~int64_t(15);
  g->gg = (flags & EOS_GRID_GLOBAL) != 0 || axes_bytes + smem_grid_bytes > 220 * 1024;
  const int64_t g_bytes = g->gg ? 0 : smem_grid_bytes;
  g->image_bytes = axes_bytes + g_bytes;
  if (g->image_bytes > 220 * 1024) return fail(EOS_ERR_UNSUPPORTED);  // axes too long for smem
  // bank-pinned axis records (kernels.cuh axis_cell REP): 128 B per axis
  // entry, if the image still fits one CTA's shared memory (227 KB opt-in
  // less the kernel's static smem).  EOS_INTERP_REP=0/1/2 (default 2).
  {
    const char* e = getenv("EOS_INTERP_REP");  // 0: plain axes (A/B)
    const int want = (e && e[0] == '0') ? 0 : 2;
    // (log-log grids: records of the log axes.)  8 copies are conflict-free
    // (128 B per axis entry); take as many as fit, down to 1 (then the
    // records still save the divides)
    const int w = want;
    // Grids in device memory leave shared memory to L1, which holds their
    // in-flight corner loads: the image is capped (EOS_GG_SMEM_KB, default 96).
    const char* ec = getenv("EOS_GG_SMEM_KB");
    const int64_t cap = g->gg ? (ec ? atoi(ec) : 96) * int64_t(1024) : 226 * 1024;
    g->rep = 0;
    for (int sh = 3; w > 0 && sh >= 0; --sh) {
      const int64_t rep_bytes = (int64_t(16) << sh) * (n_rho + n_T);
      if (g->image_bytes + rep_bytes <= cap) {
        g->rep = w;
        g->rep_shift = sh;
        g->rep_bytes_axis = int64_t(16) << sh;
        g->image_bytes += rep_bytes;
        break;
      }
    }
    // REP 2: spend the rest of the shared memory (at most 64 KB) on sparser
    // axis directories (split by axis length), so the second record read is rare
    const int64_t spare = std::min<int64_t>(cap - g->image_bytes - 512, 64 * 1024);
    if (g->rep == 2 && !loglog && spare > 1024) {
      const int64_t avail = r_bytes + t_bytes + spare;
      const int64_t br = avail * n_rho / (n_rho + n_T), bt = avail - br;
      eos::TablePlan pr, pt;
      if (eos::plan_table(rho_host, n_rho, EOS_HASH_AUTO, 0, true, &pr, br) == EOS_OK &&
          eos::plan_table(T_host, n_T, EOS_HASH_AUTO, 0, true, &pt, bt) == EOS_OK &&
          pr.steps <= g->pr.steps && pt.steps <= g->pt.steps &&
          pr.image_bytes + pt.image_bytes <= avail) {
        g->image_bytes += pr.image_bytes + pt.image_bytes - r_bytes - t_bytes;
        g->pr = std::move(pr);
        g->pt = std::move(pt);
        r_bytes = g->pr.image_bytes;
        t_bytes = g->pt.image_bytes;
      }
    }
  }
  std::vector<uint8_t> img((size_t)g->image_bytes, 0);
  std::vector<uint8_t> ir = eos::make_image(g->pr), it = eos::make_image(g->pt);
  memcpy(img.data(), ir.data(), ir.size());
  memcpy(img.data() + r_bytes, it.data(), it.size());
  g->g_off = (int32_t)(r_bytes + t_bytes);
  g->wr_off = (int32_t)(g->g_off + g_bytes);
  g->wt_off = (int32_t)(g->wr_off + wr_bytes);
  g->lr_off = (int32_t)(g->wt_off + wt_bytes);
  g->lt_off = (int32_t)(g->lr_off + lr_bytes);
  g->rr_off = (int32_t)(g->lt_off + lt_bytes);
  g->rt_off = (int32_t)(g->rr_off + (g->rep ? g->rep_bytes_axis * n_rho : 0));
  auto put_rep = [&](const std::vector<double>& Xa, int32_t off) {
    std::vector<double> X(Xa);
    if (loglog)  // records of the log axis (the same host log as the ln R / ln T arrays)
      for (double& v : X) v = log(v);
    const int64_t n = (int64_t)X.size();
    for (int64_t q = 0; q < n; ++q) {
      // Rec[C q + c] = (X[q], 1/(X[q+1] - X[q])), C = 2^rep_shift copies; the
      // last record's width is unused
      const double rec[2] = {X[q], q + 1 < n ? 1.0 / (X[q + 1] - X[q]) : 0.0};
      const int C = 1 << g->rep_shift;
      for (int c = 0; c < C; ++c) memcpy(img.data() + off + 16 * (C * q + c), rec, 16);
    }
  };
  if (g->rep) {
    put_rep(g->pr.X, g->rr_off);
    put_rep(g->pt.X, g->rt_off);
  }
  // the grid values (ln G for log-log grids)
  auto gval = [&](int64_t q) { return loglog ? log(P_host[q]) : P_host[q]; };
  if (!g->gg) {
    for (int64_t q = 0; q < ncell; ++q) {
      const double v = gval(q);
      memcpy(img.data() + g->g_off + 8 * q, &v, 8);
    }
  }
  if (loglog) {  // ln of the axes
    for (int64_t q = 0; q < n_rho; ++q) {
      const double v = log(g->pr.X[q]);
      memcpy(img.data() + g->lr_off + 8 * q, &v, 8);
    }
    for (int64_t q = 0; q < n_T; ++q) {
      const double v = log(g->pt.X[q]);
      memcpy(img.data() + g->lt_off + 8 * q, &v, 8);
    }
  }
  for (int64_t q = 0; recip_arrays && q + 1 < n_rho; ++q) {
    const double w = 1.0 / (g->pr.X[q + 1] - g->pr.X[q]);
    memcpy(img.data() + g->wr_off + 8 * q, &w, 8);
  }
  for (int64_t q = 0; recip_arrays && q + 1 < n_T; ++q) {
    const double w = 1.0 / (g->pt.X[q + 1] - g->pt.X[q]);
    memcpy(img.data() + g->wt_off + 8 * q, &w, 8);
  }
  g->ar = axis_params(g->pr, 0);
  g->at = axis_params(g->pt, (int32_t)r_bytes);
  cudaError_t e = cudaGetDevice(&g->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device);
  if (e != cudaSuccess) return fail(cuda_status(e));
  st = upload(img, &g->image_dev);
  if (st != EOS_OK) return fail(st);
  if (g->gg) {  // row pairs gq[i (nT-1) + j] = (G[i][j], G[i][j+1])
    const int64_t w = n_T - 1;
    std::vector<double> q2;
    try {
      q2.resize((size_t)(2 * n_rho * w));
    } catch (...) {
      return fail(EOS_ERR_NOMEM);
    }
    for (int64_t i = 0; i < n_rho; ++i)
      for (int64_t j = 0; j < w; ++j) {
        q2[2 * (i * w + j)] = gval(i * n_T + j);
        q2[2 * (i * w + j) + 1] = gval(i * n_T + j + 1);
      }
    g->grid_bytes = 8 * (int64_t)q2.size();
    e = cudaMalloc(&g->grid_dev, (size_t)g->grid_bytes);
    if (e == cudaSuccess)
      e = cudaMemcpy(g->grid_dev, q2.data(), (size_t)g->grid_bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(cuda_status(e));
  }
  Interp2DShape sh = pick_interp(std::max(g->pr.steps, g->pt.steps), loglog, g->rep, g->gg);
  g->fn = sh.fn;
  g->fn_deriv = sh.fn_deriv;
  g->threads = sh.threads;
  g->unroll = sh.unroll;
  g->clc = sh.clc;
  st = configure(g->fn, g->threads, g->image_bytes, g->num_sms, &g->grid, nullptr);
  if (st == EOS_OK)
    st = configure(g->fn_deriv, g->threads_deriv, g->image_bytes, g->num_sms, &g->grid_deriv,
                   nullptr);
  if (st != EOS_OK) return fail(st);
  *out = g;
  return EOS_OK;
}

eos_status eos_interp2d_ex(eos_grid2d g, const double* rho_dev, const double* T_dev,
                           int64_t count, double* P_out_dev, int32_t* irho_out_dev,
                           int32_t* iT_out_dev, double* dPdrho_out_dev, double* dPdT_out_dev,
                           void* stream) {
  if (!g) return EOS_ERR_NULL;
  if (count < 0 || count > (int64_t(1) << 62)) return EOS_ERR_SIZE;
  if (count == 0) return EOS_OK;
  if (!rho_dev || !T_dev || !P_out_dev) return EOS_ERR_NULL;
  const void* ins[2] = {rho_dev, T_dev};
  const void* outs[5] = {P_out_dev, irho_out_dev, iT_out_dev, dPdrho_out_dev, dPdT_out_dev};
  const int64_t ob[5] = {8 * count, 4 * count, 4 * count, 8 * count, 8 * count};
  for (int o = 0; o < 5; ++o) {
    if (!outs[o]) continue;
    for (int i = 0; i < 2; ++i)
      if (overlaps(ins[i], 8 * count, outs[o], ob[o])) return EOS_ERR_ALIAS;
    for (int o2 = o + 1; o2 < 5; ++o2)
      if (outs[o2] && overlaps(outs[o], ob[o], outs[o2], ob[o2])) return EOS_ERR_ALIAS;
  }
  eos_status st = check_device(g->device);
  if (st != EOS_OK) return st;
  return launch_interp(g, rho_dev, T_dev, count, P_out_dev, irho_out_dev, iT_out_dev,
                       dPdrho_out_dev, dPdT_out_dev, (cudaStream_t)stream);
}

eos_status eos_interp2d(eos_grid2d g, const double* rho_dev, const double* T_dev, int64_t count,
                        double* P_out_dev, int32_t* irho_out_dev, int32_t* iT_out_dev,
                        void* stream) {
  return eos_interp2d_ex(g, rho_dev, T_dev, count, P_out_dev, irho_out_dev, iT_out_dev, nullptr,
                         nullptr, stream);
}

eos_status eos_interp2d_host(eos_grid2d g, const double* rho_host, const double* T_host,
                             int64_t count, double* P_out_host, int32_t* irho_out_host,
                             int32_t* iT_out_host, void* stream) {
  if (!g) return EOS_ERR_NULL;
  if (count < 0 || count > (int64_t(1) << 62)) return EOS_ERR_SIZE;
  if (count == 0) return EOS_OK;
  if (!rho_host || !T_host || !P_out_host) return EOS_ERR_NULL;
  eos_status st = check_device(g->device);
  if (st != EOS_OK) return st;
  const int64_t chunk = int64_t(1) << 22;
  return host_pipeline(
      (cudaStream_t)stream, count, chunk, 32,
      [&](cudaStream_t s, char* stage, int64_t se, int64_t off, int64_t len) -> eos_status {
        double* dR = (double*)stage;
        double* dT = (double*)(stage + 8 * se);
        double* dP = (double*)(stage + 16 * se);
        int32_t* dI = (int32_t*)(stage + 24 * se);
        int32_t* dJ = (int32_t*)(stage + 28 * se);
        EOS_CUDA(cudaMemcpyAsync(dR, rho_host + off, 8 * len, cudaMemcpyHostToDevice, s));
        EOS_CUDA(cudaMemcpyAsync(dT, T_host + off, 8 * len, cudaMemcpyHostToDevice, s));
        eos_status r = launch_interp(g, dR, dT, len, dP, irho_out_host ? dI : nullptr,
                                     iT_out_host ? dJ : nullptr, nullptr, nullptr, s);
        if (r != EOS_OK) return r;
        EOS_CUDA(cudaMemcpyAsync(P_out_host + off, dP, 8 * len, cudaMemcpyDeviceToHost, s));
        if (irho_out_host)
          EOS_CUDA(cudaMemcpyAsync(irho_out_host + off, dI, 4 * len, cudaMemcpyDeviceToHost, s));
        if (iT_out_host)
          EOS_CUDA(cudaMemcpyAsync(iT_out_host + off, dJ, 4 * len, cudaMemcpyDeviceToHost, s));
        return EOS_OK;
      });
}

eos_status eos_grid2d_info(eos_grid2d g, eos_table_info_t* rho_info, eos_table_info_t* T_info) {
  if (!g) return EOS_ERR_NULL;
  if (rho_info) { eos::fill_info(g->pr, rho_info); rho_info->device = g->device; }
  if (T_info) { eos::fill_info(g->pt, T_info); T_info->device = g->device; }
  return EOS_OK;
}

eos_status eos_grid2d_destroy(eos_grid2d g) {
  if (!g) return EOS_ERR_NULL;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != g->device) cudaSetDevice(g->device);
  cudaError_t e = cudaFree(g->image_dev);
  if (g->grid_dev) {
    cudaError_t e2 = cudaFree(g->grid_dev);
    if (e == cudaSuccess) e = e2;
  }
  if (cur != g->device && cur >= 0) cudaSetDevice(cur);
  delete g;
  return cuda_status(e);
}

}  // extern "C"
