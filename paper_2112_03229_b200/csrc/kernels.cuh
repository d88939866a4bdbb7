// kernels.cuh -- sm_100a kernels of the hot path.
//
//   search1d_kernel : per target y -> int32 lower bound
//   interp2d_kernel : per (rho, T) pair -> brackets + bilinear P
//
// Design: HBM-bound streams.  The table X (fp64) and
// its exponent-hash count directory (u32) are staged once per CTA into shared
// memory; a persistent grid (#SM x resident CTAs) walks the target stream in
// tiles with 128-bit streaming loads (ld.global.cs) and 64-bit streaming
// stores; each target does a branchless bin lookup and a fixed-S-step
// branchless in-bin binary lifting (no warp divergence: S is a template
// constant of the launch).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace eos {
namespace dev {

constexpr int kThreads = 256;  // threads per CTA of search1d
constexpr int kUnroll = 4;     // double2 loads in flight per thread per tile
constexpr int kMaxTemplSteps = 8;  // S above this uses the runtime-S instantiation

struct AxisParams {
  int32_t n;        // entries
  int32_t x_off;    // byte offset of X (fp64[n]) in the smem image
  int32_t d_off;    // byte offset of the directory (u32[bins])
  int32_t shift;    // 20 - k
  uint32_t base;    // lowest bin key
  uint32_t top;     // highest bin key
  int32_t steps;    // S (used by the runtime-S path)
  int32_t pad_;
  double x0;        // X[0]
  double xlast;     // X[n-1]
};

struct SearchArgs {
  const uint4* image;   // device image (16-B aligned)
  int32_t image_16;     // image size in 16-B words
  int32_t head;         // scalar-peeled leading elements (0/1) before the vector body
  int32_t vec_ok;       // 1: vector body usable (alignment)
  int32_t pad_;
  AxisParams ax;
  const double* Y;
  int32_t* out;
  int64_t count;
  int64_t gofs;                  // global offset (counters)
  unsigned long long* counters;  // u64[8] or null
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

// The hot per-target body:
//   bin b = clamp(key >> shift, base, top) - base           (exponent hash + k bits)
//   lo, occ = directory[b]                                  (count directory)
//   c = #{j < occ : X[lo + j] <= y}  by S-step binary lifting (branchless)
//   idx = (y >= X[0]) ? lo + c - 1 : 0                      (P:54 fix-up; NaN -> 0)
template <int S, int MODE>
__device__ __forceinline__ int32_t lookup(double y, const double* __restrict__ sX,
                                          const uint32_t* __restrict__ sD, const AxisParams& a) {
  uint32_t kb = key_hi<MODE>(y) >> a.shift;
  kb = min(max(kb, a.base), a.top);
  const uint32_t d = sD[kb - a.base];
  const int32_t lo = (int32_t)(d & 0xFFFFu);
  const int32_t occ = (int32_t)(d >> 16);
  int32_t c = 0;
  if (S > 0) {
#pragma unroll
    for (int s = 1 << (S > 0 ? S - 1 : 0); s > 0; s >>= 1) {
      const int32_t j = c + s;
      if (j <= occ) {
        if (sX[lo + j - 1] <= y) c = j;
      }
    }
  } else {  // runtime S (large bins)
    for (int s = 1 << (a.steps - 1); s > 0; s >>= 1) {
      const int32_t j = c + s;
      if (j <= occ) {
        if (sX[lo + j - 1] <= y) c = j;
      }
    }
  }
  return (y >= a.x0) ? (lo + c - 1) : 0;
}

struct Counters {
  uint64_t c[7];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 7; ++i) c[i] = 0;
  }
  __device__ __forceinline__ void add(double y, int32_t idx, int64_t gpos, const double* sX,
                                      const AxisParams& a) {
    c[0] += 1;
    c[1] += (uint64_t)(uint32_t)idx;
    c[2] += mix64(((uint64_t)gpos << 20) | (uint64_t)(uint32_t)idx);
    c[3] += !(y >= a.x0);
    c[4] += (y > a.xlast);
    c[5] += (y != y);
    c[6] += (y == sX[idx]);
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

// Stage the device image (L2-resident after the first CTA) into shared memory.
__device__ __forceinline__ void stage_image(uint4* smem, const uint4* __restrict__ img, int n16) {
  for (int i = threadIdx.x; i < n16; i += blockDim.x) smem[i] = __ldg(img + i);
  __syncthreads();
}

// Launch shape of search1d (compile-time): threads per CTA, double2 loads in
// flight per thread per tile, min resident CTAs per SM (register cap), and
// whether the next tile's loads are issued before the current tile is
// searched (software prefetch).
template <int THREADS, int UNROLL, int MINB, bool PREFETCH>
struct Shape {
  static constexpr int kThreads = THREADS;
  static constexpr int kUnroll = UNROLL;
  static constexpr int kMinBlocks = MINB;
  static constexpr bool kPrefetch = PREFETCH;
  static constexpr int kTilePairs = THREADS * UNROLL;
};
using DefaultShape = Shape<kThreads, kUnroll, 4, false>;

template <int S, int MODE, bool CNT, class SH>
__global__ void __launch_bounds__(SH::kThreads, SH::kMinBlocks) search1d_kernel(const SearchArgs args) {
  constexpr int T = SH::kThreads;
  constexpr int U = SH::kUnroll;
  extern __shared__ __align__(16) uint4 smem[];
  stage_image(smem, args.image, args.image_16);
  const AxisParams a = args.ax;
  const double* __restrict__ sX =
      reinterpret_cast<const double*>(reinterpret_cast<const char*>(smem) + a.x_off);
  const uint32_t* __restrict__ sD =
      reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(smem) + a.d_off);
  const double* __restrict__ Y = args.Y;
  int32_t* __restrict__ out = args.out;
  const int64_t count = args.count;
  const int64_t gtid = (int64_t)blockIdx.x * T + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * T;

  Counters cn;
  if (CNT) cn.zero();

  if (!args.vec_ok) {
    for (int64_t i = gtid; i < count; i += gthreads) {
      const double y = Y[i];
      const int32_t r = lookup<S, MODE>(y, sX, sD, a);
      out[i] = r;
      if (CNT) cn.add(y, r, args.gofs + i, sX, a);
    }
  } else {
    const int64_t head = args.head;
    if (gtid < head) {
      const double y = Y[gtid];
      const int32_t r = lookup<S, MODE>(y, sX, sD, a);
      out[gtid] = r;
      if (CNT) cn.add(y, r, args.gofs + gtid, sX, a);
    }
    const double2* __restrict__ Y2 = reinterpret_cast<const double2*>(Y + head);
    int2* __restrict__ O2 = reinterpret_cast<int2*>(out + head);
    const int64_t npairs = (count - head) >> 1;
    const int64_t ntiles = npairs / SH::kTilePairs;
    int64_t t = blockIdx.x;
    double2 v[U];
    if (t < ntiles) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(Y2 + t * SH::kTilePairs + threadIdx.x + u * T);
    }
    while (t < ntiles) {
      const int64_t p0 = t * SH::kTilePairs + threadIdx.x;
      const int64_t tn = t + gridDim.x;
      double2 vn[U];
      if (SH::kPrefetch && tn < ntiles) {
#pragma unroll
        for (int u = 0; u < U; ++u) vn[u] = __ldcs(Y2 + tn * SH::kTilePairs + threadIdx.x + u * T);
      }
      int2 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        r[u].x = lookup<S, MODE>(v[u].x, sX, sD, a);
        r[u].y = lookup<S, MODE>(v[u].y, sX, sD, a);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) __stcs(O2 + p0 + u * T, r[u]);
      if (CNT) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t g = args.gofs + head + 2 * (p0 + u * T);
          cn.add(v[u].x, r[u].x, g, sX, a);
          cn.add(v[u].y, r[u].y, g + 1, sX, a);
        }
      }
      if (SH::kPrefetch) {
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = vn[u];
      } else if (tn < ntiles) {
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(Y2 + tn * SH::kTilePairs + threadIdx.x + u * T);
      }
      t = tn;
    }
    // remaining pairs (< one tile), then the odd last element
    for (int64_t p = ntiles * SH::kTilePairs + gtid; p < npairs; p += gthreads) {
      const double2 w = __ldcs(Y2 + p);
      int2 r;
      r.x = lookup<S, MODE>(w.x, sX, sD, a);
      r.y = lookup<S, MODE>(w.y, sX, sD, a);
      __stcs(O2 + p, r);
      if (CNT) {
        cn.add(w.x, r.x, args.gofs + head + 2 * p, sX, a);
        cn.add(w.y, r.y, args.gofs + head + 2 * p + 1, sX, a);
      }
    }
    const int64_t last = head + 2 * npairs;
    if (last < count && gtid == 0) {
      const double y = Y[last];
      const int32_t r = lookup<S, MODE>(y, sX, sD, a);
      out[last] = r;
      if (CNT) cn.add(y, r, args.gofs + last, sX, a);
    }
  }
  if (CNT) cn.flush(args.counters);
}

// ------------------------------------------------------------------ 2-D ----
constexpr int kThreads2D = 512;

struct Interp2DArgs {
  const uint4* image;
  int32_t image_16;
  int32_t g_off;    // byte offset of G fp64[nR*nT] in the image
  int32_t vec_ok;
  int32_t pad_;
  AxisParams r;     // density axis
  AxisParams t;     // temperature axis
  const double* rho;
  const double* T;
  double* P;
  int32_t* iR;      // nullable
  int32_t* iT;      // nullable
  int64_t count;
};

__device__ __forceinline__ double clamp01(double t) {
  return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
}

// Bilinear on the bracket cell (R14).  Written with explicit
// round-to-nearest intrinsics (no FMA contraction), in the order of the
// formula in eossearch.h, so the value is the correctly-rounded evaluation
// of that formula.
template <int S>
__device__ __forceinline__ double interp_one(double rho, double T, int32_t& i, int32_t& j,
                                             const char* sm, const Interp2DArgs& A) {
  const double* sR = reinterpret_cast<const double*>(sm + A.r.x_off);
  const double* sT = reinterpret_cast<const double*>(sm + A.t.x_off);
  const uint32_t* dR = reinterpret_cast<const uint32_t*>(sm + A.r.d_off);
  const uint32_t* dT = reinterpret_cast<const uint32_t*>(sm + A.t.d_off);
  const double* sG = reinterpret_cast<const double*>(sm + A.g_off);
  i = lookup<S, 0>(rho, sR, dR, A.r);
  j = lookup<S, 0>(T, sT, dT, A.t);
  const int32_t ci = min(i, A.r.n - 2);
  const int32_t cj = min(j, A.t.n - 2);
  const double r0 = sR[ci], r1 = sR[ci + 1];
  const double t0 = sT[cj], t1 = sT[cj + 1];
  const double tx = clamp01(__ddiv_rn(__dsub_rn(rho, r0), __dsub_rn(r1, r0)));
  const double ty = clamp01(__ddiv_rn(__dsub_rn(T, t0), __dsub_rn(t1, t0)));
  const double* g0 = sG + (int64_t)ci * A.t.n + cj;
  const double* g1 = g0 + A.t.n;
  const double g00 = g0[0], g01 = g0[1], g10 = g1[0], g11 = g1[1];
  const double uy = __dsub_rn(1.0, ty);
  const double a0 = __dadd_rn(__dmul_rn(uy, g00), __dmul_rn(ty, g01));
  const double a1 = __dadd_rn(__dmul_rn(uy, g10), __dmul_rn(ty, g11));
  return __dadd_rn(__dmul_rn(__dsub_rn(1.0, tx), a0), __dmul_rn(tx, a1));
}

template <int S>
__global__ void __launch_bounds__(kThreads2D, 1) interp2d_kernel(const Interp2DArgs A) {
  extern __shared__ __align__(16) uint4 smem[];
  stage_image(smem, A.image, A.image_16);
  const char* sm = reinterpret_cast<const char*>(smem);
  const int64_t count = A.count;
  const int64_t gtid = (int64_t)blockIdx.x * kThreads2D + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * kThreads2D;
  int64_t done = 0;
  if (A.vec_ok) {
    constexpr int U = 2;
    constexpr int kTilePairs = kThreads2D * U;  // in double2 units
    const double2* __restrict__ R2 = reinterpret_cast<const double2*>(A.rho);
    const double2* __restrict__ T2 = reinterpret_cast<const double2*>(A.T);
    double2* __restrict__ P2 = reinterpret_cast<double2*>(A.P);
    int2* __restrict__ IR2 = reinterpret_cast<int2*>(A.iR);
    int2* __restrict__ IT2 = reinterpret_cast<int2*>(A.iT);
    const int64_t npairs = count >> 1;
    const int64_t ntiles = npairs / kTilePairs;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t p0 = t * kTilePairs + threadIdx.x;
      double2 vr[U], vt[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        vr[u] = __ldcs(R2 + p0 + u * kThreads2D);
        vt[u] = __ldcs(T2 + p0 + u * kThreads2D);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int2 ir, it;
        double2 p;
        p.x = interp_one<S>(vr[u].x, vt[u].x, ir.x, it.x, sm, A);
        p.y = interp_one<S>(vr[u].y, vt[u].y, ir.y, it.y, sm, A);
        __stcs(P2 + p0 + u * kThreads2D, p);
        if (A.iR) __stcs(IR2 + p0 + u * kThreads2D, ir);
        if (A.iT) __stcs(IT2 + p0 + u * kThreads2D, it);
      }
    }
    done = ntiles * kTilePairs * 2;
  }
  for (int64_t q = done + gtid; q < count; q += gthreads) {
    int32_t i, j;
    const double p = interp_one<S>(A.rho[q], A.T[q], i, j, sm, A);
    A.P[q] = p;
    if (A.iR) A.iR[q] = i;
    if (A.iT) A.iT[q] = j;
  }
}

}  // namespace dev
}  // namespace eos
