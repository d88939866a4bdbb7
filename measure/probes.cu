// probes.cu -- roofline ceilings measured on the box by bench.py (harness code,
// not the product path; none of the method's arithmetic is here).
//
//  probe_stream  : the search's memory mix with no search: read fp64 targets,
//                  write one int32 per target (8 B in, 4 B out = 12 B per
//                  unit, the 1-D algorithmic bytes), and the 2-D mix (2 fp64
//                  in; fp64 + 2 int32 out = 32 B per pair).  The best of a few
//                  trivial launch shapes is the same-mix stream ceiling that
//                  bench.py reports next to the 1:1 copy peak of
//                  MEASURED_PEAKS.json (frac_vs_stream).
//  probe_gather  : random 32-byte sector gathers from an L2-resident buffer
//                  with the tiered kernel's load (ld.global.nc.L1::no_allocate
//                  .v8.u32, one sector per lane): the on-chip ceiling of the
//                  tiered-table level walk.
//  probe_stream_gather : the packed-table mix: the 1-D stream plus one random
//                  32-B sector gather per unit from an L2-resident buffer.
//  probe_interp_mix : the shared-memory grid interpolation mix: the 2-D stream
//                  plus two bank-pinned record reads and four random corner reads
//                  per pair from shared memory (interp2d_kernel's data-pipe traffic).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ double2 ldcs2(const double2* p) { return __ldcs(p); }

// out[i] = low word of the target's bits xor its high word: a value that
// depends on every loaded byte, so nothing is optimised away.
__device__ __forceinline__ int32_t fold(double v) {
  return __double2loint(v) ^ __double2hiint(v);
}

// shape A: one CTA per tile of T threads x U double2 (no persistence)
template <int T, int U>
__global__ void __launch_bounds__(T) k_stream_tiles(const double2* __restrict__ y,
                                                    int2* __restrict__ out, int64_t pairs) {
  const int64_t base = (int64_t)blockIdx.x * T * U + threadIdx.x;
  double2 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = base + (int64_t)u * T;
    v[u] = i < pairs ? ldcs2(y + i) : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = base + (int64_t)u * T;
    if (i < pairs) __stcs(out + i, make_int2(fold(v[u].x), fold(v[u].y)));
  }
}

// shape B: persistent grid-stride with the next tile's loads issued before the
// current tile's stores (the search kernel's static schedule)
template <int T, int U>
__global__ void __launch_bounds__(T, 1) k_stream_persist(const double2* __restrict__ y,
                                                         int2* __restrict__ out, int64_t pairs) {
  const int64_t tiles = pairs / ((int64_t)T * U);
  double2 v[U];
  int64_t t = blockIdx.x;
  if (t < tiles) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldcs2(y + t * T * U + threadIdx.x + u * T);
  }
  while (t < tiles) {
    const int64_t p0 = t * T * U + threadIdx.x;
    int2 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = make_int2(fold(v[u].x), fold(v[u].y));
    const int64_t tn = t + gridDim.x;
    if (tn < tiles) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldcs2(y + tn * T * U + threadIdx.x + u * T);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(out + p0 + u * T, r[u]);
    t = tn;
  }
  // tail pairs (not a whole tile): by CTA 0
  if (blockIdx.x == 0)
    for (int64_t i = tiles * T * U + threadIdx.x; i < pairs; i += T)
      __stcs(out + i, make_int2(fold(y[i].x), fold(y[i].y)));
}

// 2-D mix: per pair read rho, T (fp64), write P (fp64) and two int32
template <int T>
__global__ void __launch_bounds__(T) k_stream2d(const double2* __restrict__ a,
                                                const double2* __restrict__ b,
                                                double2* __restrict__ p, int2* __restrict__ i1,
                                                int2* __restrict__ i2, int64_t pairs2) {
  const int64_t i = (int64_t)blockIdx.x * T + threadIdx.x;
  if (i >= pairs2) return;
  const double2 x = ldcs2(a + i), z = ldcs2(b + i);
  __stcs(p + i, make_double2(x.x + z.x, x.y + z.y));
  __stcs(i1 + i, make_int2(fold(x.x), fold(x.y)));
  __stcs(i2 + i, make_int2(fold(z.x), fold(z.y)));
}

// shape C: persistent, 2U double2 per thread in flight (next tile loaded two ahead)
template <int T, int U>
__global__ void __launch_bounds__(T, 1) k_stream_persist2(const double2* __restrict__ y,
                                                          int2* __restrict__ out, int64_t pairs) {
  const int64_t tiles = pairs / ((int64_t)T * U);
  double2 v[2][U];
  int64_t t = blockIdx.x;
#pragma unroll
  for (int b = 0; b < 2; ++b)
    if (t + b * gridDim.x < tiles) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[b][u] = ldcs2(y + (t + b * gridDim.x) * T * U + threadIdx.x + u * T);
    }
  int cur = 0;
  while (t < tiles) {
    const int64_t p0 = t * T * U + threadIdx.x;
    int2 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = make_int2(fold(v[cur][u].x), fold(v[cur][u].y));
    const int64_t tn = t + 2 * (int64_t)gridDim.x;
    if (tn < tiles) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[cur][u] = ldcs2(y + tn * T * U + threadIdx.x + u * T);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(out + p0 + u * T, r[u]);
    t += gridDim.x;
    cur ^= 1;
  }
  if (blockIdx.x == 0)
    for (int64_t i = tiles * T * U + threadIdx.x; i < pairs; i += T)
      __stcs(out + i, make_int2(fold(y[i].x), fold(y[i].y)));
}

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
                 "selp.b32 %0, 1, 0, P;\n\t}"
                 : "=r"(ok) : "r"(s_u32(b)), "r"(parity) : "memory");
  } while (!ok);
}

// shape D: persistent TMA ring.  One producer warp streams tiles (31 x 32 x 4 targets)
// into NS shared-memory stages with cp.async.bulk (optionally with an L2 evict-first
// hint); 31 consumer warps wait on the stage's full barrier, read their targets from
// shared memory, store the int32 results with st.global.cs and release the stage.
template <int NS, bool HINT>
__global__ void __launch_bounds__(1024, 1) k_stream_tma(const double* __restrict__ y,
                                                       int32_t* __restrict__ out, int64_t n) {
  constexpr int CW = 31;
  constexpr int PL = 4;                 // targets per lane per stage
  constexpr int ST = CW * 32 * PL;      // targets per stage
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = (n + ST - 1) / ST;
  if (warp == CW) {
    if (lane == 0) {
      uint64_t pol = 0;
      if (HINT) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int k = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % NS;
        if (k >= NS) bar_wait(&empty[s], ((k / NS) - 1) & 1);
        const int64_t e0 = t * ST;
        const uint32_t bytes = (uint32_t)(8 * min((int64_t)ST, n - e0));
        bar_expect(&full[s], bytes);
        if (HINT)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
              "[%0], [%1], %2, [%3], %4;" ::"r"(s_u32(ring + s * ST)), "l"(y + e0), "r"(bytes),
              "r"(s_u32(&full[s])), "l"(pol) : "memory");
        else
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(s_u32(ring + s * ST)), "l"(y + e0), "r"(bytes), "r"(s_u32(&full[s])) : "memory");
      }
    }
    return;
  }
  int k = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % NS;
    bar_wait(&full[s], (k / NS) & 1);
    const double2* st = reinterpret_cast<const double2*>(ring + s * ST + warp * 32 * PL);
    const double2 a = st[lane], b = st[32 + lane];
    const int64_t e0 = t * ST + warp * 32 * PL;
    int2* o = reinterpret_cast<int2*>(out + e0);
    if (e0 + 32 * PL <= n) {
      __stcs(o + lane, make_int2(fold(a.x), fold(a.y)));
      __stcs(o + 32 + lane, make_int2(fold(b.x), fold(b.y)));
    } else {
      if (e0 + 2 * lane + 1 < n) __stcs(o + lane, make_int2(fold(a.x), fold(a.y)));
      if (e0 + 64 + 2 * lane + 1 < n) __stcs(o + 32 + lane, make_int2(fold(b.x), fold(b.y)));
    }
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[s]);
  }
}

__device__ __forceinline__ void clc_cancel(uint4* resp, uint64_t* bar) {
  asm volatile(
      "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];"
      ::"r"(s_u32(resp)), "r"(s_u32(bar)) : "memory");
}
__device__ __forceinline__ int64_t clc_get(const uint4* resp) {
  uint32_t valid = 0, x = 0;
  asm volatile(
      "{\n\t.reg .b128 R;\n\t.reg .pred P;\n\t"
      "ld.shared.b128 R, [%2];\n\t"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 P, R;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t"
      "@P clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, R;\n\t}"
      : "=r"(valid), "=r"(x) : "r"(s_u32(resp)) : "memory");
  return valid ? (int64_t)x : -1;
}

// shape E: TMA ring whose producer takes tiles with cluster launch control: the grid
// has one CTA per tile; a resident CTA's producer cancels not-yet-launched CTAs and
// streams their tiles, so tiles are processed in launch order (a compact front).
template <int NS>
__global__ void __launch_bounds__(1024, 1) k_stream_tma_clc(const double* __restrict__ y,
                                                           int32_t* __restrict__ out, int64_t n) {
  constexpr int CW = 31, PL = 4, ST = CW * 32 * PL;
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[NS], empty[NS], cbar;
  __shared__ __align__(16) uint4 resp;
  __shared__ int64_t tile_of[NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], CW);
    }
    bar_init(&cbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CW) {
    if (lane == 0) {
      int64_t t = blockIdx.x;
      uint32_t cph = 0;
      for (int k = 0;; ++k) {
        const int s = k % NS;
        if (k >= NS) bar_wait(&empty[s], ((k / NS) - 1) & 1);
        tile_of[s] = t;
        if (t < 0) {  // no more tiles: wake the consumers on this stage
          bar_arrive(&full[s]);
          break;
        }
        const int64_t e0 = t * ST;
        const uint32_t bytes = (uint32_t)(8 * min((int64_t)ST, n - e0));
        bar_expect(&full[s], bytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(s_u32(ring + s * ST)), "l"(y + e0), "r"(bytes), "r"(s_u32(&full[s])) : "memory");
        bar_expect(&cbar, 16);
        clc_cancel(&resp, &cbar);
        bar_wait(&cbar, cph);
        cph ^= 1;
        t = clc_get(&resp);
      }
    }
    return;
  }
  for (int k = 0;; ++k) {
    const int s = k % NS;
    bar_wait(&full[s], (k / NS) & 1);
    const int64_t t = tile_of[s];
    if (t < 0) break;
    const double2* st = reinterpret_cast<const double2*>(ring + s * ST + warp * 32 * PL);
    const double2 a = st[lane], b = st[32 + lane];
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[s]);
    const int64_t e0 = t * ST + warp * 32 * PL;
    int2* o = reinterpret_cast<int2*>(out + e0);
    if (e0 + 32 * PL <= n) {
      __stcs(o + lane, make_int2(fold(a.x), fold(a.y)));
      __stcs(o + 32 + lane, make_int2(fold(b.x), fold(b.y)));
    } else {
      if (e0 + 2 * lane + 1 < n) __stcs(o + lane, make_int2(fold(a.x), fold(a.y)));
      if (e0 + 64 + 2 * lane + 1 < n) __stcs(o + 32 + lane, make_int2(fold(b.x), fold(b.y)));
    }
  }
}

// shape F: persistent register loop (1024 x 4) whose tiles come from a global atomic
// counter (zeroed before the launch): tiles are taken in order, a compact front.
template <int T, int U>
__global__ void __launch_bounds__(T, 1) k_stream_atomic(const double2* __restrict__ y,
                                                        int2* __restrict__ out, int64_t pairs,
                                                        unsigned long long* ctr) {
  __shared__ int64_t nxt;
  const int64_t tiles = pairs / ((int64_t)T * U);
  if (threadIdx.x == 0) nxt = (int64_t)atomicAdd(ctr, 1ull);
  __syncthreads();
  int64_t t = nxt;
  double2 v[U];
  if (t < tiles) {
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldcs2(y + t * T * U + threadIdx.x + u * T);
  }
  while (t < tiles) {
    __syncthreads();
    if (threadIdx.x == 0) nxt = (int64_t)atomicAdd(ctr, 1ull);
    const int64_t p0 = t * T * U + threadIdx.x;
    int2 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = make_int2(fold(v[u].x), fold(v[u].y));
    __syncthreads();
    const int64_t tn = nxt;
    if (tn < tiles) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldcs2(y + tn * T * U + threadIdx.x + u * T);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(out + p0 + u * T, r[u]);
    t = tn;
  }
  if (blockIdx.x == 0)
    for (int64_t i = tiles * T * U + threadIdx.x; i < pairs; i += T)
      __stcs(out + i, make_int2(fold(y[i].x), fold(y[i].y)));
}

__device__ __forceinline__ uint64_t smix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// G independent gather chains per thread, `rounds` dependent rounds each: the
// next sector index depends on the loaded data (as in a level walk), so the
// loads cannot be hoisted.  One 32-B sector per lane per load.
template <int G>
__global__ void __launch_bounds__(1024, 1) k_gather(const uint32_t* __restrict__ buf,
                                                   uint64_t mask, int rounds,
                                                   uint32_t* __restrict__ sink) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t s[G];
  uint32_t acc = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) s[g] = smix(tid * G + g) & mask;
  for (int r = 0; r < rounds; ++r) {
    uint32_t k[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g)
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(k[g][0]), "=r"(k[g][1]), "=r"(k[g][2]), "=r"(k[g][3]), "=r"(k[g][4]),
                     "=r"(k[g][5]), "=r"(k[g][6]), "=r"(k[g][7])
                   : "l"(buf + 8 * s[g]));
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t x = k[g][0] ^ k[g][3] ^ k[g][7];
      acc += x;
      s[g] = (s[g] * 0x9E3779B97F4A7C15ULL + x + 1) & mask;
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;  // practically never: keeps the loads live
}

// Cooperative line gathers: groups of 4 lanes load the 4 sectors of one random 128-B
// line (one 256-bit load per lane), G chains per thread: how many random LINES per second
// the L1TEX t-stage serves when each line is requested whole by one instruction.
template <int G>
__global__ void __launch_bounds__(1024, 1) k_gather_line(const uint32_t* __restrict__ buf,
                                                        uint64_t lmask, int rounds,
                                                        uint32_t* __restrict__ sink) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int q = threadIdx.x & 3;             // this lane's sector of the group's line
  const uint64_t grp = tid >> 2;
  uint64_t s[G];
  uint32_t acc = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) s[g] = smix(grp * G + g) & lmask;
  for (int r = 0; r < rounds; ++r) {
    uint32_t k[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g)
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(k[g][0]), "=r"(k[g][1]), "=r"(k[g][2]), "=r"(k[g][3]), "=r"(k[g][4]),
                     "=r"(k[g][5]), "=r"(k[g][6]), "=r"(k[g][7])
                   : "l"(buf + 32 * s[g] + 8 * q));
#pragma unroll
    for (int g = 0; g < G; ++g) {
      uint32_t x = k[g][0] ^ k[g][3] ^ k[g][7];
      x ^= __shfl_xor_sync(0xFFFFFFFFu, x, 1);  // the group agrees on the next line
      x ^= __shfl_xor_sync(0xFFFFFFFFu, x, 2);
      acc += x;
      s[g] = (s[g] * 0x9E3779B97F4A7C15ULL + x + 1) & lmask;
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// The packed-table memory mix with no search: per unit, read an
// fp64 target (stream), gather ONE random 32-B sector of an L2-resident node
// buffer at an index hashed from the target's bits, write an int32 that
// depends on both.  One CTA per tile of T threads x U double2: the same-mix
// ceiling of a one-sector-per-lookup kernel.
template <int T, int U>
__global__ void __launch_bounds__(T) k_stream_gather(const double2* __restrict__ y,
                                                     int2* __restrict__ out, int64_t pairs,
                                                     const uint32_t* __restrict__ buf,
                                                     uint64_t mask) {
  const int64_t base = (int64_t)blockIdx.x * T * U + threadIdx.x;
  double2 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = base + (int64_t)u * T;
    v[u] = i < pairs ? ldcs2(y + i) : make_double2(0.0, 0.0);
  }
  uint32_t k[2 * U][8];
#pragma unroll
  for (int u = 0; u < 2 * U; ++u) {
    const double x = (u & 1) ? v[u >> 1].y : v[u >> 1].x;
    const uint64_t s = smix((uint64_t)__double_as_longlong(x)) & mask;
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(k[u][0]), "=r"(k[u][1]), "=r"(k[u][2]), "=r"(k[u][3]), "=r"(k[u][4]),
                   "=r"(k[u][5]), "=r"(k[u][6]), "=r"(k[u][7])
                 : "l"(buf + 8 * s));
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = base + (int64_t)u * T;
    const int2 r = make_int2(fold(v[u].x) ^ (int32_t)(k[2 * u][0] ^ k[2 * u][7]),
                             fold(v[u].y) ^ (int32_t)(k[2 * u + 1][0] ^ k[2 * u + 1][7]));
    if (i < pairs) __stcs(out + i, r);
  }
}

// The shared-memory grid interpolation mix with no search and no interpolation
// arithmetic: the 2-D stream (rho, T in; P, two int32 out) plus,
// per pair, one bank-pinned 16-B record read per axis (lane l reads copy l mod 8)
// and the 4 corner reads G[i][j], G[i][j+1], G[i+1][j], G[i+1][j+1] (8 B each) of a
// cell (i, j) hashed from the coordinates' bits, from a grid of nR x nT fp64 in
// shared memory: 1 CTA x 1024 threads per SM, static tiles, the next tile's loads
// after this tile's pairs and an L2 prefetch of the tile after next -- the launch
// shape of interp2d_kernel.  Its rate is the ceiling of that kernel's data-pipe
// traffic (shared wavefronts + the stream).
__device__ __forceinline__ void pf_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__global__ void __launch_bounds__(1024, 1) k_interp_mix(const double2* __restrict__ rho,
                                                       const double2* __restrict__ T,
                                                       double2* __restrict__ P, int2* __restrict__ iR,
                                                       int2* __restrict__ iT, int64_t pairs2,
                                                       int nR, int nT) {
  extern __shared__ __align__(16) double sm[];
  double* G = sm;                                                       // nR nT
  double2* recR = reinterpret_cast<double2*>(sm + (((int64_t)nR * nT + 1) & ~int64_t(1)));  // 8 nR
  double2* recT = recR + 8 * nR;                                        // 8 nT
  for (int q = threadIdx.x; q < nR * nT; q += blockDim.x) G[q] = 1.0 + q;
  for (int q = threadIdx.x; q < 8 * (nR + nT); q += blockDim.x) recR[q] = make_double2(q, 1.0 / (q + 1));
  __syncthreads();
  const int c8 = threadIdx.x & 7;
  const int64_t tiles = pairs2 / 1024;
  auto one = [&](double x, double y, int32_t& i, int32_t& j) {
    const uint32_t hx = (uint32_t)__double2loint(x) ^ (uint32_t)__double2hiint(x);
    const uint32_t hy = (uint32_t)__double2loint(y) ^ (uint32_t)__double2hiint(y);
    i = (int32_t)__umulhi(hx * 0x9E3779B1u, (uint32_t)(nR - 1));
    j = (int32_t)__umulhi(hy * 0x85EBCA77u, (uint32_t)(nT - 1));
    const double2 rr = recR[(i << 3) + c8], rt = recT[(j << 3) + c8];
    const double* g = G + i * nT + j;
    return ((g[0] + g[1]) * rr.y + (g[nT] + g[nT + 1]) * rt.y) + rr.x * rt.x;
  };
  int64_t t = blockIdx.x;
  double2 vr = make_double2(0, 0), vt = vr;
  if (t < tiles) {
    vr = ldcs2(rho + t * 1024 + threadIdx.x);
    vt = ldcs2(T + t * 1024 + threadIdx.x);
  }
  for (; t < tiles; t += gridDim.x) {
    int2 a, b;
    double2 p;
    p.x = one(vr.x, vt.x, a.x, b.x);
    p.y = one(vr.y, vt.y, a.y, b.y);
    const int64_t tn = t + gridDim.x;
    if (tn < tiles) {
      vr = ldcs2(rho + tn * 1024 + threadIdx.x);
      vt = ldcs2(T + tn * 1024 + threadIdx.x);
    }
    if (threadIdx.x == 0 && tn + gridDim.x < tiles) {
      pf_l2(rho + (tn + gridDim.x) * 1024, 1024 * 16);
      pf_l2(T + (tn + gridDim.x) * 1024, 1024 * 16);
    }
    const int64_t i = t * 1024 + threadIdx.x;
    __stcs(P + i, p);
    __stcs(iR + i, a);
    __stcs(iT + i, b);
  }
}

// The device-memory grid interpolation mix (big2d) with no search and
// no interpolation arithmetic: the 2-D stream plus, per pair, one bank-pinned 16-B
// record read per axis from shared memory (C copies, lane l reads copy l mod C) and one
// 32-B cell quad (the 4 corners) gathered from nR x nT quads in device memory
// (L2-resident) at a cell hashed from the coordinates' bits -- interp2d_kernel's GG
// traffic, in its launch shape (1 CTA x 1024 threads per SM, static tiles, next tile's
// loads after this tile's pairs).
__global__ void __launch_bounds__(1024, 1) k_interp_gg_mix(const double2* __restrict__ rho,
                                                          const double2* __restrict__ T,
                                                          double2* __restrict__ P, int2* __restrict__ iR,
                                                          int2* __restrict__ iT, int64_t pairs2,
                                                          const double* __restrict__ quads, int nR,
                                                          int nT, int csh) {
  extern __shared__ __align__(16) double sm[];
  double2* recR = reinterpret_cast<double2*>(sm);   // nR << csh
  double2* recT = recR + ((int64_t)nR << csh);      // nT << csh
  for (int q = threadIdx.x; q < ((nR + nT) << csh); q += blockDim.x) recR[q] = make_double2(q, 1.0 / (q + 1));
  __syncthreads();
  const int c = threadIdx.x & ((1 << csh) - 1);
  const int64_t tiles = pairs2 / 1024;
  auto one = [&](double x, double y, int32_t& i, int32_t& j) {
    const uint32_t hx = (uint32_t)__double2loint(x) ^ (uint32_t)__double2hiint(x);
    const uint32_t hy = (uint32_t)__double2loint(y) ^ (uint32_t)__double2hiint(y);
    i = (int32_t)__umulhi(hx * 0x9E3779B1u, (uint32_t)(nR - 1));
    j = (int32_t)__umulhi(hy * 0x85EBCA77u, (uint32_t)(nT - 1));
    const double2 rr = recR[(i << csh) + c], rt = recT[(j << csh) + c];
    double g0, g1, g2, g3;
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(g0), "=d"(g1), "=d"(g2), "=d"(g3)
        : "l"(quads + 4 * ((int64_t)i * (nT - 1) + j)));
    return ((g0 + g1) * rr.y + (g2 + g3) * rt.y) + rr.x * rt.x;
  };
  int64_t t = blockIdx.x;
  double2 vr = make_double2(0, 0), vt = vr;
  if (t < tiles) {
    vr = ldcs2(rho + t * 1024 + threadIdx.x);
    vt = ldcs2(T + t * 1024 + threadIdx.x);
  }
  for (; t < tiles; t += gridDim.x) {
    int2 a, b;
    double2 p;
    p.x = one(vr.x, vt.x, a.x, b.x);
    p.y = one(vr.y, vt.y, a.y, b.y);
    const int64_t tn = t + gridDim.x;
    if (tn < tiles) {
      vr = ldcs2(rho + tn * 1024 + threadIdx.x);
      vt = ldcs2(T + tn * 1024 + threadIdx.x);
    }
    const int64_t i = t * 1024 + threadIdx.x;
    __stcs(P + i, p);
    __stcs(iR + i, a);
    __stcs(iT + i, b);
  }
}

__global__ void k_fill(uint32_t* buf, uint64_t words) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += stride)
    buf[i] = (uint32_t)smix(i);
}

int sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace

extern "C" {

// Number of 1-D stream shapes (variant 0 .. probe_stream_variants()-1).
int probe_stream_variants(void) { return 11; }

// One launch of the 1-D same-mix stream over n targets (n even, y 16-B and
// out 8-B aligned).  Returns a cudaError_t.
int probe_stream(const double* y, int32_t* out, int64_t n, int variant, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t pairs = n / 2;
  const double2* y2 = reinterpret_cast<const double2*>(y);
  int2* o2 = reinterpret_cast<int2*>(out);
  switch (variant) {
    case 0: {
      const int64_t tiles = (pairs + 256 * 4 - 1) / (256 * 4);
      k_stream_tiles<256, 4><<<(unsigned)tiles, 256, 0, st>>>(y2, o2, pairs);
      break;
    }
    case 1: {
      const int64_t tiles = (pairs + 512 * 2 - 1) / (512 * 2);
      k_stream_tiles<512, 2><<<(unsigned)tiles, 512, 0, st>>>(y2, o2, pairs);
      break;
    }
    case 2:
      k_stream_persist<1024, 4><<<sms(), 1024, 0, st>>>(y2, o2, pairs);
      break;
    case 3:
      k_stream_persist<512, 4><<<2 * sms(), 512, 0, st>>>(y2, o2, pairs);
      break;
    case 4:
      k_stream_persist<1024, 8><<<sms(), 1024, 0, st>>>(y2, o2, pairs);
      break;
    case 5:
      k_stream_persist2<1024, 4><<<sms(), 1024, 0, st>>>(y2, o2, pairs);
      break;
    case 6:
    case 7:
    case 8: {  // TMA ring: 4 stages (127 KB), 4 stages + L2 evict-first, 6 stages (190 KB)
      const int ns = variant == 8 ? 6 : 4;
      const size_t smem = (size_t)ns * 31 * 32 * 4 * 8;
      const void* fn = variant == 6 ? (const void*)k_stream_tma<4, false>
                       : variant == 7 ? (const void*)k_stream_tma<4, true>
                                      : (const void*)k_stream_tma<6, false>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (variant == 6) k_stream_tma<4, false><<<sms(), 1024, smem, st>>>(y, out, 2 * pairs);
      else if (variant == 7) k_stream_tma<4, true><<<sms(), 1024, smem, st>>>(y, out, 2 * pairs);
      else k_stream_tma<6, false><<<sms(), 1024, smem, st>>>(y, out, 2 * pairs);
      break;
    }
    case 9: {
      const int64_t ntiles = (2 * pairs + 3967) / 3968;
      const size_t smem = (size_t)4 * 3968 * 8;
      cudaFuncSetAttribute((const void*)k_stream_tma_clc<4>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_stream_tma_clc<4><<<(unsigned)ntiles, 1024, smem, st>>>(y, out, 2 * pairs);
      break;
    }
    case 10: {
      static unsigned long long* ctr = nullptr;
      if (!ctr) cudaMalloc(&ctr, 8);
      cudaMemsetAsync(ctr, 0, 8, st);
      k_stream_atomic<1024, 4><<<sms(), 1024, 0, st>>>(y2, o2, pairs, ctr);
      break;
    }
    default:
      return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

// One launch of the 2-D same-mix stream over m pairs (m even, aligned).
int probe_stream2d(const double* rho, const double* T, double* P, int32_t* iR, int32_t* iT,
                   int64_t m, void* stream) {
  const int64_t p2 = m / 2;
  k_stream2d<256><<<(unsigned)((p2 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const double2*>(rho), reinterpret_cast<const double2*>(T),
      reinterpret_cast<double2*>(P), reinterpret_cast<int2*>(iR), reinterpret_cast<int2*>(iT), p2);
  return (int)cudaGetLastError();
}

// Fill `words` u32 of buf (device) with pseudo-random data.
int probe_fill(uint32_t* buf, uint64_t words, void* stream) {
  k_fill<<<4 * sms(), 256, 0, (cudaStream_t)stream>>>(buf, words);
  return (int)cudaGetLastError();
}

// One launch of the random-sector gather: every thread of a persistent grid
// (1 CTA x 1024 threads per SM) runs `chains` (1, 2, 4 or 8) chains of
// `rounds` dependent 32-B loads from buf[0 .. 8*sectors), sectors a power of two.  Sectors loaded =
// sms * 1024 * chains * rounds.
int probe_gather(const uint32_t* buf, uint64_t sectors, int chains, int rounds, uint32_t* sink,
                 void* stream) {
  if (sectors == 0 || (sectors & (sectors - 1))) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = sms();
  const uint64_t mask = sectors - 1;
  switch (chains) {
    case 1: k_gather<1><<<g, 1024, 0, st>>>(buf, mask, rounds, sink); break;
    case 2: k_gather<2><<<g, 1024, 0, st>>>(buf, mask, rounds, sink); break;
    case 4: k_gather<4><<<g, 1024, 0, st>>>(buf, mask, rounds, sink); break;
    default: k_gather<8><<<g, 1024, 0, st>>>(buf, mask, rounds, sink); break;
  }
  return (int)cudaGetLastError();
}

// Random 128-B line gathers by 4-lane groups (one 32-B sector per lane); lines loaded =
// sms * 1024 / 4 * chains * rounds.  lines a power of two.
int probe_gather_line(const uint32_t* buf, uint64_t lines, int chains, int rounds, uint32_t* sink,
                      void* stream) {
  if (lines == 0 || (lines & (lines - 1))) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = sms();
  const uint64_t mask = lines - 1;
  switch (chains) {
    case 1: k_gather_line<1><<<g, 1024, 0, st>>>(buf, mask, rounds, sink); break;
    case 2: k_gather_line<2><<<g, 1024, 0, st>>>(buf, mask, rounds, sink); break;
    case 4: k_gather_line<4><<<g, 1024, 0, st>>>(buf, mask, rounds, sink); break;
    default: k_gather_line<8><<<g, 1024, 0, st>>>(buf, mask, rounds, sink); break;
  }
  return (int)cudaGetLastError();
}

// Number of stream+gather shapes (variant 0 .. probe_stream_gather_variants()-1).
int probe_stream_gather_variants(void) { return 4; }

// One launch of the packed-table same mix over n targets (n even, aligned):
// read y, gather one 32-B sector of buf[0 .. 8*sectors) per target (sectors a
// power of two), write out.
int probe_stream_gather(const double* y, int32_t* out, int64_t n, const uint32_t* buf,
                        uint64_t sectors, int variant, void* stream) {
  if (sectors == 0 || (sectors & (sectors - 1))) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t pairs = n / 2;
  const double2* y2 = reinterpret_cast<const double2*>(y);
  int2* o2 = reinterpret_cast<int2*>(out);
  const uint64_t mask = sectors - 1;
  switch (variant) {
    case 0: k_stream_gather<256, 2><<<(unsigned)((pairs + 511) / 512), 256, 0, st>>>(y2, o2, pairs, buf, mask); break;
    case 1: k_stream_gather<256, 4><<<(unsigned)((pairs + 1023) / 1024), 256, 0, st>>>(y2, o2, pairs, buf, mask); break;
    case 2: k_stream_gather<512, 2><<<(unsigned)((pairs + 1023) / 1024), 512, 0, st>>>(y2, o2, pairs, buf, mask); break;
    case 3: k_stream_gather<1024, 2><<<(unsigned)((pairs + 2047) / 2048), 1024, 0, st>>>(y2, o2, pairs, buf, mask); break;
    default: return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

// One launch of the shared-memory interpolation mix over m pairs (m a multiple of
// 2048, aligned) with an nR x nT grid in shared memory (k_interp_mix).
int probe_interp_mix(const double* rho, const double* T, double* P, int32_t* iR, int32_t* iT,
                     int64_t m, int nR, int nT, void* stream) {
  const size_t smem = (size_t)((((int64_t)nR * nT + 1) & ~int64_t(1)) * 8 + 16 * 8 * ((int64_t)nR + nT));
  if (nR < 2 || nT < 2 || smem > 227 * 1024 || m % 2048) return (int)cudaErrorInvalidValue;
  cudaFuncSetAttribute((const void*)k_interp_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_interp_mix<<<sms(), 1024, smem, (cudaStream_t)stream>>>(
      reinterpret_cast<const double2*>(rho), reinterpret_cast<const double2*>(T),
      reinterpret_cast<double2*>(P), reinterpret_cast<int2*>(iR), reinterpret_cast<int2*>(iT), m / 2,
      nR, nT);
  return (int)cudaGetLastError();
}

// One launch of the device-memory-grid interpolation mix over m pairs (m a multiple of
// 2048, aligned): quads = (nR-1) x (nT-1) cells of 4 fp64 in device memory, 2^csh
// record copies per axis node in shared memory (k_interp_gg_mix).
int probe_interp_gg_mix(const double* rho, const double* T, double* P, int32_t* iR, int32_t* iT,
                        int64_t m, const double* quads, int nR, int nT, int csh, void* stream) {
  const size_t smem = (size_t)16 * (((int64_t)nR + nT) << csh);
  if (nR < 2 || nT < 2 || csh < 0 || csh > 3 || smem > 227 * 1024 || m % 2048)
    return (int)cudaErrorInvalidValue;
  cudaFuncSetAttribute((const void*)k_interp_gg_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_interp_gg_mix<<<sms(), 1024, smem, (cudaStream_t)stream>>>(
      reinterpret_cast<const double2*>(rho), reinterpret_cast<const double2*>(T),
      reinterpret_cast<double2*>(P), reinterpret_cast<int2*>(iR), reinterpret_cast<int2*>(iT), m / 2,
      quads, nR, nT, csh);
  return (int)cudaGetLastError();
}

int probe_sms(void) { return sms(); }

}  // extern "C"
