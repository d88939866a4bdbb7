// runtime.cu -- shared host runtime of libeossearch.so (runtime.h) and the
// status / version / launch-count entry points of the C ABI.
// Product path (never includes or links oracle/).
//
// The product library reads no environment variables: launch shapes and
// layouts follow from the plan alone.  A/B experiment knobs exist only in the
// experiment build (_build.py --exp, -DEOS_EXPERIMENTS: libeossearch_exp.so):
//   EOS_SEARCH_VARIANT, EOS_TIERED_VARIANT  launch-shape variants by name
//   EOS_LAYOUT=d16,sf,big                   lifting layout of a single-level table
//   EOS_SMALL_TILES=0                       small launches keep the default tiles
//   EOS_RING=<n>                            at most n ring stages (0: no ring kernel)
// and compile-time A/B flags of that build (-D...):
//   EOS_EXP_NO_L2_PREFETCH                  2-D kernels without the L2 prefetch of the
//                                           tile after next
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <new>
#include <vector>

#include "eos_internal.h"
#include "eossearch.h"
#include "kernels.cuh"
#include "runtime.h"

namespace eos {
namespace rt {

static std::atomic<int64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Staging for the host-buffer entry points: one stream-ordered pool per device
// that keeps up to 1 GiB reserved across synchronisations (the default pool
// returns its memory to the driver at every sync, and re-mapping it costs tens
// of microseconds per call).
cudaError_t stage_alloc(void** p, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, st);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      cudaMemPool_t np = nullptr;
      e = cudaMemPoolCreate(&np, &props);
      if (e != cudaSuccess) return e;
      uint64_t keep = uint64_t(1) << 30;
      e = cudaMemPoolSetAttribute(np, cudaMemPoolAttrReleaseThreshold, &keep);
      if (e != cudaSuccess) {
        cudaMemPoolDestroy(np);
        return e;
      }
      pools[dev] = np;
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

dev::AxisParams axis_params(const TablePlan& p, int32_t x_off) {
  dev::AxisParams a{};
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
cudaError_t launch(const void* fn, int64_t grid, int threads, size_t smem, cudaStream_t st,
                   void** params) {
  const bool pdl = true;
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

}  // namespace rt
}  // namespace eos

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

int32_t eos_abi_version(void) { return 5; }

int64_t eos_launch_count(void) { return eos::rt::g_launches.load(); }

}  // extern "C"
