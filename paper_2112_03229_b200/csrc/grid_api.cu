// grid_api.cu -- the 2-D part of the C ABI (include/eossearch.h): grid handles
// (shared-memory and device-memory grids, bank-pinned cell records) and the
// interpolation launches.  Product path (never includes or links oracle/).
#include <cuda_runtime.h>
#include <math.h>
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
  int threads = 512, unroll = 2;
  bool clc = true;
  // small launches (fewer default tiles than half the SMs; no derivative outputs):
  // Shape2DSmall, 4x smaller tiles (nullptr: none)
  const void* fn_small = nullptr;        // ... without derivative outputs
  const void* fn_small_deriv = nullptr;  // ... with them
  int grid_small = 0, grid_small_deriv = 0, threads_small = 0;
  int64_t small_image_bytes = 0;  // the image without G (g_off)
  int32_t flags = 0;
  int32_t wr_off = 0, wt_off = 0, lr_off = 0, lt_off = 0;
  int32_t rr_off = 0, rt_off = 0;
  int rep = 0;  // 2: bank-pinned cell records in the image (REP kernels), 0: plain axes
  int32_t rep_shift = 0;       // REP 2: log2 of the record copies
  int64_t rep_bytes_axis = 0;  // image bytes per axis entry of the REP layout
  bool gg = false;          // grid in device memory (GG kernels)
  void* grid_dev = nullptr;  // GG: cell quads (double4[(n_rho - 1)(n_T - 1)]) or row pairs
  bool gquad = false;        //     (double2[n_rho (n_T - 1)])
  int64_t grid_bytes = 0;
};

namespace {

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

// The small-launch kernel: the default layouts (bank-pinned records, S = 1) only.
// Always the device-memory-grid flavour: a small launch stages only the image
// without G (axes, directories, records) and reads each cell's corners as one
// 32-B quad, so its many CTAs do not each copy the whole grid from L2.
const void* pick_interp_small(int steps, bool loglog, int rep, bool deriv) {
  using SG = dv::Shape2DSmallGG;
  if (steps != 1 || rep != 2) return nullptr;
  if (deriv)
    return loglog ? (const void*)dv::interp2d_kernel<1, SG, false, true, true, 2, true>
                  : (const void*)dv::interp2d_kernel<1, SG, false, true, false, 2, true>;
  return loglog ? (const void*)dv::interp2d_kernel<1, SG, false, false, true, 2, true>
                : (const void*)dv::interp2d_kernel<1, SG, false, false, false, 2, true>;
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
  a.gquad = g->gquad ? 1 : 0;
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
    a.gquad = 1;
  }
  if (tiles > 0x7FFFFFFF) return EOS_ERR_SIZE;
  a.ntiles = tiles;
  const bool clc = sm ? false : (deriv ? dv::Shape2DDeriv::kClc : g->clc);
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
  // image: [rho X | rho dir][T X | T dir][1/dR][1/dT (RECIP variants)][ln R][ln T][R recs][T recs][G]
  // G is absent for grids in device memory (GG: larger than ~220 KB, or
  // EOS_GRID_GLOBAL), which keep it in g->grid_dev instead (cell quads or row pairs).
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
  // G last: the image without it (the first g_off bytes) serves the small-launch
  // kernels, which read the corners from cell quads in device memory
  g->wr_off = (int32_t)(r_bytes + t_bytes);
  g->wt_off = (int32_t)(g->wr_off + wr_bytes);
  g->lr_off = (int32_t)(g->wt_off + wt_bytes);
  g->lt_off = (int32_t)(g->lr_off + lr_bytes);
  g->rr_off = (int32_t)(g->lt_off + lt_bytes);
  g->rt_off = (int32_t)(g->rr_off + (g->rep ? g->rep_bytes_axis * n_rho : 0));
  g->g_off = (int32_t)(g->rt_off + (g->rep ? g->rep_bytes_axis * n_T : 0));
  if (g->g_off + g_bytes != g->image_bytes) return fail(EOS_ERR_CUDA);  // layout invariant
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
  const char* small_env = getenv("EOS_SMALL_TILES");  // "0": default tiles only
  const bool small_ok = !((small_env && small_env[0] == '0') || getenv("EOS_INTERP_VARIANT"));
  const int steps_max = std::max(g->pr.steps, g->pt.steps);
  const void* fn_small = small_ok ? pick_interp_small(steps_max, loglog, g->rep, false) : nullptr;
  const void* fn_small_deriv =
      small_ok ? pick_interp_small(steps_max, loglog, g->rep, true) : nullptr;
  // shared-memory grids keep cell quads in device memory too, for the small-launch kernel
  const bool quads_for_small = !g->gg && fn_small && 32 * ncell <= (int64_t(64) << 20);
  if (g->gg || quads_for_small) {
    // Cell quads (32 B per cell: the 4 corners in one sector) up to
    // EOS_GG_QUAD_MB (default 1024 MB of quads), else row pairs
    // gq[i (nT-1) + j] = (G[i][j], G[i][j+1]) (two 16-B loads per pair).
    const int64_t w = n_T - 1;
    const char* eq = getenv("EOS_GG_QUAD_MB");
    const int64_t quad_cap = (eq ? atoll(eq) : 1024) << 20;
    g->gquad = quads_for_small || 32 * (n_rho - 1) * w <= quad_cap;
    std::vector<double> q2;
    try {
      q2.resize((size_t)(g->gquad ? 4 * (n_rho - 1) * w : 2 * n_rho * w));
    } catch (...) {
      return fail(EOS_ERR_NOMEM);
    }
    if (g->gquad) {
      for (int64_t i = 0; i + 1 < n_rho; ++i)
        for (int64_t j = 0; j < w; ++j) {
          double* c = q2.data() + 4 * (i * w + j);
          c[0] = gval(i * n_T + j);
          c[1] = gval(i * n_T + j + 1);
          c[2] = gval((i + 1) * n_T + j);
          c[3] = gval((i + 1) * n_T + j + 1);
        }
    } else {
      for (int64_t i = 0; i < n_rho; ++i)
        for (int64_t j = 0; j < w; ++j) {
          q2[2 * (i * w + j)] = gval(i * n_T + j);
          q2[2 * (i * w + j) + 1] = gval(i * n_T + j + 1);
        }
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
  if (fn_small && fn_small_deriv && g->gquad) {  // the small kernels read quads (not row pairs)
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
