// Microbenchmark (GPU box): 4 random fp64 corner gathers per pair from a
// 200 x 100 fp64 grid in shared memory, as (a) 4 LDS.64 per lane (the
// interp2d kernel) and (b) 4-lane groups where lane p loads corner p of the
// group's 4 pairs and SHFLs redistribute them.  Prints pairs per SM-clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NR = 200, NT = 100, ITERS = 256;

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(const double* g, double* out, long long* clk) {
  extern __shared__ double sG[];
  for (int i = threadIdx.x; i < NR * NT; i += blockDim.x) sG[i] = g[i];
  __syncthreads();
  uint32_t s = hash(blockIdx.x * 1024 + threadIdx.x);
  double acc = 0;
  const int lane = threadIdx.x & 31, p = lane & 3;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    s = hash(s + it);
    const int ci = s % (NR - 1), cj = (s >> 12) % (NT - 1);
    const int b = ci * NT + cj;
    double c0, c1, c2, c3;
    if (MODE == 0) {
      c0 = sG[b]; c1 = sG[b + 1]; c2 = sG[b + NT]; c3 = sG[b + NT + 1];
    } else {
      const int off = (p & 1) + (p >> 1) * NT;  // this lane's corner
      double v[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int bq = __shfl_sync(0xffffffffu, b, (lane & ~3) | ((p + r) & 3));
        v[r] = sG[bq + off];
      }
      // lane q needs corner k from lane k: value v[(q - k) & 3]
      double w[4];
      w[0] = v[0];
#pragma unroll
      for (int s2 = 1; s2 < 4; ++s2)
        w[s2] = __shfl_sync(0xffffffffu, v[s2], (lane & ~3) | ((p - s2) & 3));
      // corner k arrived in round (p - k) & 3
      auto pick = [&](int k) {
        const int r = (p - k) & 3;
        return r == 0 ? w[0] : (r == 1 ? w[1] : (r == 2 ? w[2] : w[3]));
      };
      c0 = pick(0); c1 = pick(1); c2 = pick(2); c3 = pick(3);
    }
    acc += c0 * 0.1 + c1 * 0.2 + c2 * 0.3 + c3 * 0.4;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* g; double* out; long long* clk;
  cudaMalloc(&g, NR * NT * 8); cudaMemset(g, 0, NR * NT * 8);
  cudaMalloc(&out, sms * 1024 * 8); cudaMalloc(&clk, sms * 8);
  const int smem = NR * NT * 8;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      if (mode == 0) k<0><<<sms, 1024, smem>>>(g, out, clk); else k<1><<<sms, 1024, smem>>>(g, out, clk);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      printf("mode %d: %.3f ms, %lld clk on SM0, %.3f pairs/clk/SM\n", mode, ms, c,
             1024.0 * ITERS / (double)c);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
