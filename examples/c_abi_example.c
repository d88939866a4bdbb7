/* c_abi_example.c -- the boundary used from plain C (no Python, no torch):
 * create a table from host memory, search a device batch, read the indices
 * back, then the same through the host-buffer entry point, and a 2-D grid.
 *
 *   gcc -std=c11 -O2 -I include examples/c_abi_example.c \
 *       -L paper_2112_03229_b200/lib -leossearch -lcudart -o c_abi_example
 *
 * Usage: c_abi_example <table.f64> <targets.f64> <out_idx.i32> <out_host_idx.i32>
 * (raw little-endian arrays; sizes from the file lengths).  Exit code 0 on
 * success; any eos_status error is printed with eos_status_str. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "eossearch.h"

static void* slurp(const char* path, long* bytes) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  *bytes = ftell(f);
  fseek(f, 0, SEEK_SET);
  void* p = malloc((size_t)*bytes);
  if (p && fread(p, 1, (size_t)*bytes, f) != (size_t)*bytes) { free(p); p = NULL; }
  fclose(f);
  return p;
}

static int spill(const char* path, const void* p, size_t bytes) {
  FILE* f = fopen(path, "wb");
  if (!f) return 1;
  size_t w = fwrite(p, 1, bytes, f);
  fclose(f);
  return w != bytes;
}

#define CHECK(call)                                                            \
  do {                                                                         \
    eos_status s_ = (call);                                                    \
    if (s_ != EOS_OK) {                                                        \
      fprintf(stderr, "%s failed: %s\n", #call, eos_status_str(s_));          \
      return 2;                                                                \
    }                                                                          \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 5) {
    fprintf(stderr, "usage: %s table.f64 targets.f64 out_idx.i32 out_host_idx.i32\n", argv[0]);
    return 1;
  }
  long tb = 0, yb = 0;
  double* X = (double*)slurp(argv[1], &tb);
  double* Y = (double*)slurp(argv[2], &yb);
  if (!X || !Y) { fprintf(stderr, "cannot read inputs\n"); return 1; }
  const int64_t n = tb / 8, m = yb / 8;

  eos_table t = NULL;
  CHECK(eos_search_create(X, n, &t));
  eos_table_info_t info;
  CHECK(eos_table_info(t, &info));
  printf("n=%lld levels=%d bins=%d S=%d image=%lld abi=%d\n", (long long)info.n, info.levels,
         info.bins, info.steps, (long long)info.image_bytes, eos_abi_version());

  /* device path: caller-owned device buffers, default stream */
  double* dY = NULL;
  int32_t* dI = NULL;
  if (cudaMalloc((void**)&dY, 8 * (size_t)m) != cudaSuccess ||
      cudaMalloc((void**)&dI, 4 * (size_t)m) != cudaSuccess) { fprintf(stderr, "cudaMalloc\n"); return 3; }
  cudaMemcpy(dY, Y, 8 * (size_t)m, cudaMemcpyHostToDevice);
  CHECK(eos_search(t, dY, m, dI, NULL));
  int32_t* I = (int32_t*)malloc(4 * (size_t)m);
  if (cudaMemcpy(I, dI, 4 * (size_t)m, cudaMemcpyDeviceToHost) != cudaSuccess) return 3;

  /* host-buffer path (pipelined copies inside the library) */
  int32_t* Ih = (int32_t*)malloc(4 * (size_t)m);
  CHECK(eos_search_host(t, Y, m, Ih, NULL));
  if (cudaStreamSynchronize(0) != cudaSuccess) return 3;

  /* errors are reported, not crashed on */
  eos_table bad = NULL;
  const double unsorted[3] = {2.0, 1.0, 3.0};
  if (eos_search_create(unsorted, 3, &bad) != EOS_ERR_UNSORTED || bad != NULL) return 4;

  /* a 2-D grid from C: P = rho + 10 T on a 3 x 4 grid, one pair */
  const double R[3] = {1.0, 2.0, 4.0}, T[4] = {0.0, 1.0, 2.0, 3.0};
  double G[12];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 4; ++j) G[4 * i + j] = R[i] + 10.0 * T[j];
  eos_grid2d g = NULL;
  CHECK(eos_grid2d_create(R, 3, T, 4, G, &g));
  double *d2 = NULL, P = 0.0;
  cudaMalloc((void**)&d2, 3 * sizeof(double));
  const double in[2] = {3.0, 2.5};
  cudaMemcpy(d2, in, 2 * sizeof(double), cudaMemcpyHostToDevice);
  CHECK(eos_interp2d(g, d2, d2 + 1, 1, d2 + 2, NULL, NULL, NULL));
  cudaMemcpy(&P, d2 + 2, sizeof(double), cudaMemcpyDeviceToHost);
  printf("P(3.0, 2.5) = %.17g\n", P); /* bilinear reproduces rho + 10 T: 28 */
  if (P < 28.0 - 1e-12 || P > 28.0 + 1e-12) return 5;

  int rc = spill(argv[3], I, 4 * (size_t)m) | spill(argv[4], Ih, 4 * (size_t)m);
  CHECK(eos_grid2d_destroy(g));
  CHECK(eos_search_destroy(t));
  cudaFree(dY);
  cudaFree(dI);
  cudaFree(d2);
  free(X); free(Y); free(I); free(Ih);
  return rc;
}
