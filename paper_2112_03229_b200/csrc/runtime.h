// runtime.h -- host-side helpers shared by the C-ABI translation units of
// libeossearch.so (runtime.cu, search_api.cu, grid_api.cu): CUDA status
// mapping, kernel configuration and launch (with programmatic dependent
// launch), image upload, the host-buffer pipeline.  Product path (never
// includes or links oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "eos_internal.h"
#include "eossearch.h"
#include "kernels.cuh"

namespace eos {
namespace rt {

eos_status cuda_status(cudaError_t e);

#define EOS_CUDA(call)                              \
  do {                                              \
    cudaError_t e_ = (call);                        \
    if (e_ != cudaSuccess) return cuda_status(e_);  \
  } while (0)

eos_status check_device(int device);
bool overlaps(const void* a, int64_t abytes, const void* b, int64_t bbytes);
// Configure a kernel for `smem` bytes of dynamic shared memory and return the
// persistent grid (#SM x resident CTAs per SM) and the CTAs per SM.
eos_status configure(const void* fn, int threads, int64_t smem, int num_sms, int* grid, int* per_sm);
// Launch with programmatic stream serialization (PDL).
cudaError_t launch(const void* fn, int64_t grid, int threads, size_t smem, cudaStream_t st,
                   void** params);
// Count one kernel launch (eos_launch_count).
void count_launch();
// Stream-ordered staging allocation from the library's per-device pool (freed
// with cudaFreeAsync).
cudaError_t stage_alloc(void** p, size_t bytes, cudaStream_t st);
eos_status upload(const std::vector<uint8_t>& img, void** dev);
// The smem-image axis parameters of a planned table at byte offset x_off.
dev::AxisParams axis_params(const TablePlan& p, int32_t x_off);

// Two-stream chunked pipeline over host buffers (one chunk: the caller stream
// alone): chunk c uses slot c % 2 (its
// own stream and device staging), so H2D(c+1) overlaps search(c) / D2H(c).
template <class Body>
eos_status host_pipeline(cudaStream_t caller, int64_t count, int64_t chunk, int64_t bytes_per_elem,
                         Body body) {
  // two slots; mid-sized calls: ~8 chunks (>= chunk / 32 each), so H2D overlaps
  // D2H (2-4 slots and 2^21-2^23-element chunks measured equal)
  const int slots_env = 2;
  {
    int64_t c = chunk / 32;
    while (c < chunk && 8 * c < count) c *= 2;
    chunk = c;
  }
  const int64_t nchunk = (count + chunk - 1) / chunk;
  const int nslot = (int)std::min<int64_t>(nchunk, slots_env);
  const int64_t slot_elems = (std::min(chunk, count) + 63) & ~int64_t(63);  // keeps 16-B alignment
  char* stage = nullptr;
  EOS_CUDA(stage_alloc((void**)&stage, (size_t)(nslot * slot_elems * bytes_per_elem), caller));
  if (nchunk == 1) {  // one chunk: nothing to overlap, so no side streams or events
    const eos_status st1 = body(caller, stage, slot_elems, 0, count);
    cudaFreeAsync(stage, caller);
    return st1;
  }
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

}  // namespace rt
}  // namespace eos
