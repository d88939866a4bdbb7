// grid_api.cu -- the 2-D part of the C ABI (include/eossearch.h): grid handles
// (shared-memory and device-memory grids, bank-pinned cell records) and the
// interpolation launches.  Product path (never includes or links oracle/).
#include <cuda_runtime.h>
#include <math.h>

#include <cmath>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <vector>

#include "eos_internal.h"
#include "eossearch.h"
#include "kernels.cuh"
#include "runtime.h"

using eos::TablePlan;
namespace dv = eos::dev;
using namespace eos::rt;

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
  int threads = dv::Shape2D::kThreads, unroll = dv::Shape2D::kUnroll;
  // small launches (fewer default tiles than half the SMs; no derivative outputs):
  // Shape2DSmall, 4x smaller tiles (nullptr: none)
  const void* fn_small = nullptr;        // ... without derivative outputs
  const void* fn_small_deriv = nullptr;  // ... with them
  int grid_small = 0, grid_small_deriv = 0, threads_small = 0;
  int64_t small_image_bytes = 0;  // the image without G (g_off)
  int32_t flags = 0;
  int32_t rr_off = 0, rt_off = 0;
  int rep = 0;  // 2: bank-pinned cell records in the image (REP kernels), 0: plain axes
  int narrow = 0;  // log-log: 2 if every cell ratio X[j+1]/X[j] <= 1.25, 1 if <= 1.5 (kernels.cuh log1p_cell)
  int32_t rep_shift = 0;       // REP 2: log2 of the record copies
  int64_t rep_bytes_axis = 0;  // image bytes per axis entry of the REP layout
  bool gg = false;          // grid in device memory (GG kernels)
  void* grid_dev = nullptr;  // cell quads double4[(n_rho - 1)(n_T - 1)] (GG and small kernels)
  int64_t grid_bytes = 0;
};

namespace {

// Fitted cell map of a grid axis (kernels.cuh axis_cell_rec, S = kMapped): the
// kernel takes p = floor(a w(x) + b) in fp32 (w = log2 x by lg2.approx.ftz.f32, or
// x), clamped to [0, n-2], and needs p in {c, c+1} for every x in cell c =
// [X[c], X[c+1]).  The exact map u(x) = a w(x) + b is monotone, so that holds if
// every node maps inside its own unit, c + E <= u(X[c]) <= c + 1 - E, where E
// bounds the device's error: the fp32 rounding of x (2^-24 relative: 2^-24/ln 2 of
// log2 x, or 2^-24 |x|), lg2.approx (2^-22 absolute plus the rounding of its
// exponent add, 2^-24 |log2 x|) and the fp32 fma (2^-24 |u|), times a, then 4x.
// b puts the nodes 1e-4 above their unit's floor, so p = c + 1 -- and a second
// record read -- is rare.  Kind 1 (log) is tried first; none fits: kind 0.
struct CellMap {
  int kind = 0;
  float a = 0.0f, b = 0.0f;
};
CellMap fit_cell_map(const std::vector<double>& X) {
  const int64_t n = (int64_t)X.size();
  for (int kind = 1; kind <= 2; ++kind) {
    if (kind == 1 ? !(X[0] >= 1e-30 && X[n - 1] <= 1e30)
                  : !(std::fabs(X[0]) <= 1e30 && std::fabs(X[n - 1]) <= 1e30))
      continue;
    std::vector<double> L((size_t)n);
    for (int64_t j = 0; j < n; ++j) L[j] = kind == 1 ? std::log2(X[j]) : X[j];
    const double a = (double)(n - 1) / (L[n - 1] - L[0]);
    if (!(a > 0.0 && a < 1e30)) continue;
    const float af = (float)a;
    const double lmax = std::max(std::fabs(L[0]), std::fabs(L[n - 1]));
    const double u24 = std::ldexp(1.0, -24);
    const double ew = kind == 1 ? u24 / M_LN2 + std::ldexp(1.0, -22) + lmax * u24 : lmax * u24;
    const double E = 4.0 * ((double)af * ew + (double)(n + 1) * u24) + 1e-6;
    double lo = HUGE_VAL;
    for (int64_t j = 0; j < n; ++j) lo = std::min(lo, (double)af * L[j] - (double)j);
    const float bf = (float)(E + 1e-4 - lo);
    bool ok = std::isfinite(bf);
    for (int64_t j = 0; j < n && ok; ++j) {
      const double v = (double)af * L[j] + (double)bf - (double)j;
      ok = v >= E && v <= 1.0 - E;
    }
    if (ok) return {kind, af, bf};
  }
  return {};
}

// Kernel of a grid: S = 1..4 or 0 (runtime), linear or log-log, REP 2 (bank-pinned
// cell records) or 0 (plain axes: EOS_GRID_EXACT, or when the records do not fit),
// grid in shared (GG = false) or device memory; with and without derivative outputs.
// S = 1 (the usual plan of a grid axis) runs 1024 threads per SM; deeper axes and
// derivative outputs need more than 64 registers per thread: 512 threads.
using Shape2DDeep = dv::Shape<512, 1, 1, false>;
struct InterpKernel {
  const void* fn;
  int threads;
  int unroll = 1;
};
// log-log grids in shared memory (issue-bound): the default 2-D shape; the experiment
// build takes -DEOS_EXP_LL_T=<threads> -DEOS_EXP_LL_U=<pairs of pairs per thread>
#if defined(EOS_EXPERIMENTS) && defined(EOS_EXP_LL_T)
using Shape2DLL = dv::Shape<EOS_EXP_LL_T, EOS_EXP_LL_U, 1, false>;
#else
using Shape2DLL = dv::Shape2D;
#endif

template <int S, bool LOGLOG, int REP, bool GG, int NK = 0>
InterpKernel interp_fn(bool deriv) {
  if (deriv) {
    if constexpr (LOGLOG && !GG && REP == 2 && (S == 1 || S == dv::kMapped))
      return {(const void*)dv::interp2d_kernel<S, dv::Shape2DDerivFull, true, LOGLOG, REP, GG, NK>,
              dv::Shape2DDerivFull::kThreads};
    if constexpr (GG && REP == 2 && (S == 1 || S == dv::kMapped))
      return {(const void*)dv::interp2d_kernel<S, dv::Shape2DDerivWide, true, LOGLOG, REP, GG>,
              dv::Shape2DDerivWide::kThreads};
    return {(const void*)dv::interp2d_kernel<S, dv::Shape2DDeriv, true, LOGLOG, REP, GG>,
            dv::Shape2DDeriv::kThreads};
  }
  if constexpr (LOGLOG && !GG && REP == 2 && NK > 0)
    return {(const void*)dv::interp2d_kernel<S, Shape2DLL, false, LOGLOG, REP, GG, NK>,
            Shape2DLL::kThreads, Shape2DLL::kUnroll};
  else if constexpr ((S == 1 || S == dv::kMapped) && !(LOGLOG && REP == 0))  // (plain log-log axes: 2 log1p per axis)
    return {(const void*)dv::interp2d_kernel<S, dv::Shape2D, false, LOGLOG, REP, GG, NK>,
            dv::Shape2D::kThreads};
  else
    return {(const void*)dv::interp2d_kernel<S, Shape2DDeep, false, LOGLOG, REP, GG>,
            Shape2DDeep::kThreads};
}

template <bool LOGLOG, int REP, bool GG>
InterpKernel interp_fn_steps(int steps, bool deriv, int narrow) {
  if constexpr (LOGLOG && REP == 2 && !GG) {  // the series length fixed at compile time
    if (narrow && (steps == dv::kMapped || steps == 1)) {
      if (steps == dv::kMapped)
        return narrow == 2 ? interp_fn<dv::kMapped, LOGLOG, REP, GG, 8>(deriv)
                           : interp_fn<dv::kMapped, LOGLOG, REP, GG, 12>(deriv);
      return narrow == 2 ? interp_fn<1, LOGLOG, REP, GG, 8>(deriv)
                         : interp_fn<1, LOGLOG, REP, GG, 12>(deriv);
    }
  }
  if constexpr (REP == 2) {
    if (steps == dv::kMapped) return interp_fn<dv::kMapped, LOGLOG, REP, GG>(deriv);
  }
  if constexpr (GG) {  // device-memory grids: S = 1 or the runtime loop
    return steps == 1 ? interp_fn<1, LOGLOG, REP, GG>(deriv) : interp_fn<0, LOGLOG, REP, GG>(deriv);
  } else {
    switch (steps) {
      case 1: return interp_fn<1, LOGLOG, REP, GG>(deriv);
      case 2: return interp_fn<2, LOGLOG, REP, GG>(deriv);
      case 3: return interp_fn<3, LOGLOG, REP, GG>(deriv);
      case 4: return interp_fn<4, LOGLOG, REP, GG>(deriv);
      default: return interp_fn<0, LOGLOG, REP, GG>(deriv);
    }
  }
}

InterpKernel pick_interp(int steps, bool loglog, int rep, bool gg, bool deriv, int narrow) {
  if (gg) {
    if (loglog) return rep == 2 ? interp_fn_steps<true, 2, true>(steps, deriv, narrow)
                                : interp_fn_steps<true, 0, true>(steps, deriv, narrow);
    return rep == 2 ? interp_fn_steps<false, 2, true>(steps, deriv, narrow)
                    : interp_fn_steps<false, 0, true>(steps, deriv, narrow);
  }
  if (loglog) return rep == 2 ? interp_fn_steps<true, 2, false>(steps, deriv, narrow)
                              : interp_fn_steps<true, 0, false>(steps, deriv, narrow);
  return rep == 2 ? interp_fn_steps<false, 2, false>(steps, deriv, narrow)
                  : interp_fn_steps<false, 0, false>(steps, deriv, narrow);
}

// The small-launch kernel: the default layouts (bank-pinned records, S = 1) only.
// Always the device-memory-grid flavour: a small launch stages only the image
// without G (axes, directories, records) and reads each cell's corners as one
// 32-B quad, so its many CTAs do not each copy the whole grid from L2.
const void* pick_interp_small(int steps, bool loglog, int rep, bool deriv) {
  using SG = dv::Shape2DSmallGG;
  if (rep != 2) return nullptr;
  if (steps == dv::kMapped) {
    if (deriv)
      return loglog ? (const void*)dv::interp2d_kernel<dv::kMapped, SG, true, true, 2, true>
                    : (const void*)dv::interp2d_kernel<dv::kMapped, SG, true, false, 2, true>;
    return loglog ? (const void*)dv::interp2d_kernel<dv::kMapped, SG, false, true, 2, true>
                  : (const void*)dv::interp2d_kernel<dv::kMapped, SG, false, false, 2, true>;
  }
  if (steps != 1) return nullptr;
  if (deriv)
    return loglog ? (const void*)dv::interp2d_kernel<1, SG, true, true, 2, true>
                  : (const void*)dv::interp2d_kernel<1, SG, true, false, 2, true>;
  return loglog ? (const void*)dv::interp2d_kernel<1, SG, false, true, 2, true>
                : (const void*)dv::interp2d_kernel<1, SG, false, false, 2, true>;
}

#ifdef EOS_EXPERIMENTS
bool exp_small_off() {  // EOS_SMALL_TILES=0: small launches keep the default tiles (A/B)
  const char* e = getenv("EOS_SMALL_TILES");
  return e && e[0] == '0';
}
#else
bool exp_small_off() { return false; }
#endif

eos_status launch_interp(eos_grid2d g, const double* rho, const double* T, int64_t count,
                         double* P, int32_t* iR, int32_t* iT, double* dPr, double* dPt,
                         cudaStream_t st) {
  const bool deriv = dPr != nullptr || dPt != nullptr;
  dv::Interp2DArgs a{};
  a.image = (const uint4*)g->image_dev;
  a.image_16 = (int32_t)(g->image_bytes / 16);
  a.g_off = g->g_off;
  a.rr_off = g->rr_off;
  a.rt_off = g->rt_off;
  a.gq = reinterpret_cast<const double2*>(g->grid_dev);
  a.rep_shift = g->rep_shift;
  a.narrow = g->narrow;
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
  int threads = deriv ? g->threads_deriv : g->threads;
  int64_t per_tile = (int64_t)threads * (deriv ? g->unroll_deriv : g->unroll) * 2;
  int64_t tiles = (count + per_tile - 1) / per_tile;
  // fewer tiles than half the SMs: the small-tile shape spreads the launch over more CTAs
  // (scripts/exp_small_tiles_2d.sh)
  const void* fsm = deriv ? g->fn_small_deriv : g->fn_small;
  const bool sm = fsm && 2 * tiles < g->num_sms;
  if (sm) {  // unroll 1, static schedule; G from the cell quads
    threads = g->threads_small;
    per_tile = (int64_t)threads * 2;
    tiles = (count + per_tile - 1) / per_tile;
    a.image_16 = (int32_t)(g->small_image_bytes / 16);
  }
  if (tiles > 0x7FFFFFFF) return EOS_ERR_SIZE;
  a.ntiles = tiles;
  const bool clc = sm ? false : (deriv ? dv::Shape2DDeriv::kClc : dv::Shape2D::kClc);
  const int pgrid = sm ? (deriv ? g->grid_small_deriv : g->grid_small)
                       : (deriv ? g->grid_deriv : g->grid);
  int64_t grid = clc ? tiles : std::min<int64_t>(pgrid, tiles);
  grid = std::max<int64_t>(grid, 1);
  void* params[] = {&a};
  EOS_CUDA(launch(sm ? fsm : (deriv ? g->fn_deriv : g->fn), grid, threads,
                  (size_t)(sm ? g->small_image_bytes : g->image_bytes), st, params));
  count_launch();
  return EOS_OK;
}

}  // namespace

extern "C" {

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
  if (flags & ~(EOS_GRID_LOGLOG | EOS_GRID_GLOBAL | EOS_GRID_EXACT | EOS_GRID_DIRECTORY))
    return EOS_ERR_UNSUPPORTED;
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
  // image: [rho X | rho dir][T X | T dir][R recs][T recs][G]
  // G is absent for grids in device memory (GG: larger than ~220 KB, or
  // EOS_GRID_GLOBAL), which keep it in g->grid_dev instead (cell quads or row pairs).
  int64_t r_bytes = g->pr.image_bytes, t_bytes = g->pt.image_bytes;
  const int64_t axes_bytes = r_bytes + t_bytes;
  const int64_t smem_grid_bytes = (8 * ncell + 15) & ~int64_t(15);
  g->gg = (flags & EOS_GRID_GLOBAL) != 0 || axes_bytes + smem_grid_bytes > 220 * 1024;
  const int64_t g_bytes = g->gg ? 0 : smem_grid_bytes;
  g->image_bytes = axes_bytes + g_bytes;
  if (g->image_bytes > 220 * 1024) return fail(EOS_ERR_UNSUPPORTED);  // axes too long for smem
  // bank-pinned axis records (kernels.cuh axis_cell_rec, REP 2): 128 B per axis
  // entry, if the image still fits one CTA's shared memory (227 KB opt-in
  // less the kernel's static smem).  EOS_GRID_EXACT: plain axes (REP 0), whose
  // weights divide exactly as the formula does.
  {
    // Log-log records need 1/X[c] on the device from the reciprocal estimate (its ftz
    // form): every axis value and its reciprocal must be normal doubles, else REP 0.
    bool rcp_ok = true;
    for (const std::vector<double>* ax : {&g->pr.X, &g->pt.X})
      rcp_ok = rcp_ok && ax->front() >= 0x1p-1020 && ax->back() <= 0x1p1020;
    const int want = ((flags & EOS_GRID_EXACT) || (loglog && !rcp_ok)) ? 0 : 2;
    // (log-log grids: records of the log axes.)  8 copies are conflict-free
    // (128 B per axis entry); take as many as fit, down to 1 (then the
    // records still save the divides)
    const int w = want;
    // Grids in device memory leave shared memory to L1, which holds their
    // in-flight corner loads: the image is capped at 96 KB (48-144 KB measured
    // within 1.5%).
    const int64_t cap = g->gg ? 96 * 1024 : 226 * 1024;
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
    if (g->rep == 2 && spare > 1024) {
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
  // G last: the image without it (the first g_off bytes) serves the small-launch
  // kernels, which read the corners from cell quads in device memory
  g->rr_off = (int32_t)(r_bytes + t_bytes);
  g->rt_off = (int32_t)(g->rr_off + (g->rep ? g->rep_bytes_axis * n_rho : 0));
  g->g_off = (int32_t)(g->rt_off + (g->rep ? g->rep_bytes_axis * n_T : 0));
  if (g->g_off + g_bytes != g->image_bytes) return fail(EOS_ERR_CUDA);  // layout invariant
  auto put_rep = [&](const std::vector<double>& X, int32_t off) {
    const int64_t n = (int64_t)X.size();
    for (int64_t q = 0; q < n; ++q) {
      // Rec[C q + c] = (X[q], 1/(X[q+1] - X[q])), or for log-log grids
      // (X[q], 1/ln(X[q+1]/X[q])) with ln(X[q+1]/X[q]) = log1p((X[q+1] - X[q])/X[q])
      // (R24); C = 2^rep_shift copies; the last record's width is unused
      const bool last = q + 1 >= n;
      const double rec[2] = {
          X[q],
          last ? 0.0 : (loglog ? 1.0 / log1p((X[q + 1] - X[q]) / X[q]) : 1.0 / (X[q + 1] - X[q]))};
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
  if (loglog) {  // the short log1p series of the weights: every cell ratio <= 1.5 (12
                 // terms) or <= 1.25 (8 terms), kernels.cuh log1p_cell
    bool n15 = true, n125 = true;
    for (const std::vector<double>* ax : {&g->pr.X, &g->pt.X})
      for (size_t q = 0; q + 1 < ax->size(); ++q) {
        n15 = n15 && (*ax)[q + 1] <= 1.5 * (*ax)[q];
        n125 = n125 && (*ax)[q + 1] <= 1.25 * (*ax)[q];
      }
    g->narrow = n125 ? 2 : (n15 ? 1 : 0);
  }
  g->ar = axis_params(g->pr, 0);
  g->at = axis_params(g->pt, (int32_t)r_bytes);
  // fitted cell maps: both axes, bank-pinned records, not EOS_GRID_DIRECTORY
  if (g->rep == 2 && !(flags & EOS_GRID_DIRECTORY)) {
    const CellMap mr = fit_cell_map(g->pr.X), mt = fit_cell_map(g->pt.X);
    if (mr.kind && mt.kind) {
      g->ar.map_kind = mr.kind;
      g->ar.map_a = mr.a;
      g->ar.map_b = mr.b;
      g->at.map_kind = mt.kind;
      g->at.map_a = mt.a;
      g->at.map_b = mt.b;
    }
  }
  cudaError_t e = cudaGetDevice(&g->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device);
  if (e != cudaSuccess) return fail(cuda_status(e));
  st = upload(img, &g->image_dev);
  if (st != EOS_OK) return fail(st);
  const bool small_ok = !exp_small_off();
  const int steps_max = g->ar.map_kind ? dv::kMapped : std::max(g->pr.steps, g->pt.steps);
  const void* fn_small = small_ok ? pick_interp_small(steps_max, loglog, g->rep, false) : nullptr;
  const void* fn_small_deriv =
      small_ok ? pick_interp_small(steps_max, loglog, g->rep, true) : nullptr;
  // shared-memory grids keep cell quads in device memory too, for the small-launch kernel
  const bool quads_for_small = !g->gg && fn_small && 32 * ncell <= (int64_t(64) << 20);
  if (g->gg || quads_for_small) {
    // cell quads: 32 B per cell, the 4 corners in one sector (4x the grid; at most
    // 8 GB for EOS_MAX_GRID_CELLS)
    const int64_t w = n_T - 1;
    std::vector<double> q2;
    try {
      q2.resize((size_t)(4 * (n_rho - 1) * w));
    } catch (...) {
      return fail(EOS_ERR_NOMEM);
    }
    for (int64_t i = 0; i + 1 < n_rho; ++i)
      for (int64_t j = 0; j < w; ++j) {
        double* c = q2.data() + 4 * (i * w + j);
        c[0] = gval(i * n_T + j);
        c[1] = gval(i * n_T + j + 1);
        c[2] = gval((i + 1) * n_T + j);
        c[3] = gval((i + 1) * n_T + j + 1);
      }
    g->grid_bytes = 8 * (int64_t)q2.size();
    e = cudaMalloc(&g->grid_dev, (size_t)g->grid_bytes);
    if (e == cudaSuccess)
      e = cudaMemcpy(g->grid_dev, q2.data(), (size_t)g->grid_bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(cuda_status(e));
  }
  const InterpKernel k0 = pick_interp(steps_max, loglog, g->rep, g->gg, false, g->narrow);
  const InterpKernel k1 = pick_interp(steps_max, loglog, g->rep, g->gg, true, g->narrow);
  g->fn = k0.fn;
  g->threads = k0.threads;
  g->unroll = k0.unroll;
  g->fn_deriv = k1.fn;
  g->threads_deriv = k1.threads;
  st = configure(g->fn, g->threads, g->image_bytes, g->num_sms, &g->grid, nullptr);
  if (st == EOS_OK)
    st = configure(g->fn_deriv, g->threads_deriv, g->image_bytes, g->num_sms, &g->grid_deriv,
                   nullptr);
  if (st != EOS_OK) return fail(st);
  if (fn_small && fn_small_deriv && g->grid_dev) {  // the small kernels read the quads
    const int ts = dv::Shape2DSmallGG::kThreads;
    if (configure(fn_small, ts, g->g_off, g->num_sms, &g->grid_small, nullptr) == EOS_OK &&
        configure(fn_small_deriv, ts, g->g_off, g->num_sms, &g->grid_small_deriv, nullptr) ==
            EOS_OK) {
      g->fn_small = fn_small;
      g->fn_small_deriv = fn_small_deriv;
      g->threads_small = ts;
      g->small_image_bytes = g->g_off;
    }
  }
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
  {  // outputs must not overlap the inputs or each other (as eos_interp2d_ex)
    const void* ins[2] = {rho_host, T_host};
    const void* outs[3] = {P_out_host, irho_out_host, iT_out_host};
    const int64_t ob[3] = {8 * count, 4 * count, 4 * count};
    for (int o = 0; o < 3; ++o) {
      if (!outs[o]) continue;
      for (int i = 0; i < 2; ++i)
        if (overlaps(ins[i], 8 * count, outs[o], ob[o])) return EOS_ERR_ALIAS;
      for (int o2 = o + 1; o2 < 3; ++o2)
        if (outs[o2] && overlaps(outs[o], ob[o], outs[o2], ob[o2])) return EOS_ERR_ALIAS;
    }
  }
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
  if (rho_info) {
    eos::fill_info(g->pr, rho_info);
    rho_info->device = g->device;
    rho_info->cell_map = g->ar.map_kind;
  }
  if (T_info) {
    eos::fill_info(g->pt, T_info);
    T_info->device = g->device;
    T_info->cell_map = g->at.map_kind;
  }
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
