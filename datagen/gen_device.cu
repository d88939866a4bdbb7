// gen_device.cu -- device (B200) side of the datagen generators (gen_core.h).
// Harness code, not the product path: fills target streams in HBM so that
// multi-GiB inputs never cross PCIe.  Bit-identical to gen_host.c (tested).
#include <cuda_runtime.h>
#include <stdint.h>
#include "gen_core.h"

namespace {

__global__ void k_loguniform(uint64_t key, int64_t offset, int64_t count, double a, double w,
                             double* __restrict__ out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride)
    out[j] = gen_loguniform(key, (uint64_t)(offset + j), a, w);
}

__global__ void k_copies(uint64_t key, uint64_t key2, int64_t offset, int64_t count, double a,
                         double w, const double* __restrict__ X, int64_t n, uint64_t copy_every,
                         double* __restrict__ out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride)
    out[j] = gen_with_copies(key, key2, (uint64_t)(offset + j), a, w, X, n, copy_every);
}

// ---- random walk: exact integer prefix sums in three passes ----
constexpr int WT = 256;             // threads per block
constexpr int WE = 16;              // elements per thread
constexpr int WCHUNK = WT * WE;     // elements per block

__global__ void k_walk_sum_range(uint64_t key, int64_t begin, int64_t end,
                                 unsigned long long* __restrict__ acc) {
  uint64_t s = 0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end; i += stride)
    s += (uint64_t)gen_walk_step(key, (uint64_t)i);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc, (unsigned long long)s);  // wrapping add: exact
}

__global__ void k_walk_chunk_sums(uint64_t key, int64_t offset, int64_t count,
                                  unsigned long long* __restrict__ sums) {
  __shared__ uint64_t red[WT / 32];
  int64_t base = offset + (int64_t)blockIdx.x * WCHUNK;
  int64_t end = offset + count;
  uint64_t s = 0;
  for (int e = threadIdx.x; e < WCHUNK; e += WT) {
    int64_t i = base + e;
    if (i < end) s += (uint64_t)gen_walk_step(key, (uint64_t)i);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int q = 0; q < WT / 32; ++q) t += red[q];
    sums[blockIdx.x] = t;
  }
}

// exclusive scan of chunk sums, seeded with the prefix before `offset`
__global__ void k_walk_scan_sums(unsigned long long* __restrict__ sums, int64_t nchunks,
                                 const unsigned long long* __restrict__ base) {
  uint64_t run = *base;
  for (int64_t c = 0; c < nchunks; ++c) {
    uint64_t v = sums[c];
    sums[c] = run;
    run += v;
  }
}

__global__ void k_walk_fill(uint64_t key, int64_t offset, int64_t count,
                            const unsigned long long* __restrict__ chunk_prefix, double x0,
                            double c, double lo, double hi, double* __restrict__ out) {
  __shared__ uint64_t sc[WT];
  int64_t cbase = (int64_t)blockIdx.x * WCHUNK + (int64_t)threadIdx.x * WE;  // local index
  uint64_t steps[WE];
  uint64_t tsum = 0;
#pragma unroll
  for (int e = 0; e < WE; ++e) {
    int64_t j = cbase + e;
    steps[e] = (j < count) ? (uint64_t)gen_walk_step(key, (uint64_t)(offset + j)) : 0;
    tsum += steps[e];
  }
  sc[threadIdx.x] = tsum;
  __syncthreads();
  // Hillis-Steele inclusive scan over thread totals
  for (int d = 1; d < WT; d <<= 1) {
    uint64_t v = (threadIdx.x >= d) ? sc[threadIdx.x - d] : 0;
    __syncthreads();
    sc[threadIdx.x] += v;
    __syncthreads();
  }
  uint64_t S = chunk_prefix[blockIdx.x] + sc[threadIdx.x] - tsum;
#pragma unroll
  for (int e = 0; e < WE; ++e) {
    int64_t j = cbase + e;
    S += steps[e];
    if (j < count) out[j] = gen_walk_value((int64_t)S, x0, c, lo, hi);
  }
}

int grid_for(int64_t count) {
  int64_t g = (count + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

extern "C" {

int gen_dev_fill_loguniform(uint64_t seed, uint64_t stream, int64_t offset, int64_t count,
                            double a, double w, double* out_dev, void* cu_stream) {
  if (count <= 0) return 0;
  k_loguniform<<<grid_for(count), 256, 0, (cudaStream_t)cu_stream>>>(gen_key(seed, stream), offset,
                                                                     count, a, w, out_dev);
  return (int)cudaGetLastError();
}

int gen_dev_fill_copies(uint64_t seed, int64_t offset, int64_t count, double a, double w,
                        const double* X_dev, int64_t n, uint64_t copy_every, double* out_dev,
                        void* cu_stream) {
  if (count <= 0) return 0;
  k_copies<<<grid_for(count), 256, 0, (cudaStream_t)cu_stream>>>(
      gen_key(seed, 0), gen_key(seed, 1), offset, count, a, w, X_dev, n, copy_every, out_dev);
  return (int)cudaGetLastError();
}

int gen_dev_fill_walk(uint64_t seed, int64_t offset, int64_t count, double x0, double c, double lo,
                      double hi, double* out_dev, void* cu_stream) {
  if (count <= 0) return 0;
  cudaStream_t st = (cudaStream_t)cu_stream;
  uint64_t key = gen_key(seed, 0);
  int64_t nchunks = (count + WCHUNK - 1) / WCHUNK;
  unsigned long long* ws = nullptr;
  cudaError_t err = cudaMallocAsync((void**)&ws, (size_t)(nchunks + 1) * 8, st);
  if (err != cudaSuccess) return (int)err;
  unsigned long long* base = ws + nchunks;
  cudaMemsetAsync(base, 0, 8, st);
  if (offset > 0) k_walk_sum_range<<<grid_for(offset), 256, 0, st>>>(key, 0, offset, base);
  k_walk_chunk_sums<<<(unsigned)nchunks, WT, 0, st>>>(key, offset, count, ws);
  k_walk_scan_sums<<<1, 1, 0, st>>>(ws, nchunks, base);
  k_walk_fill<<<(unsigned)nchunks, WT, 0, st>>>(key, offset, count, ws, x0, c, lo, hi, out_dev);
  err = cudaGetLastError();
  cudaFreeAsync(ws, st);
  return (int)err;
}

}  // extern "C"
