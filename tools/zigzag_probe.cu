// zigzag_probe.cu - standalone probe (tuning tool, not part of libuqg.so): how
// much of a vector that one kernel has just written is still in L2 when the
// next kernel reads it, if a group's kernels ran back to back on ONE group's
// vectors (66.8 MB each at C3) and the consumer swept the rows in the
// opposite direction of the producer?
//
// K1 (SpMV-like): reads a, b, writes c, forward.  K2 (update-like): reads d,
// c, e, writes d - forward (the library's order) or reverse.  Reports K2's
// algorithmic GB/s (4 arrays) for both orders and for a cold c.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/zz tools/zigzag_probe.cu
//   /tmp/zz [rows=261121] [S=32]
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t err_ = (x);                                                         \
    if (err_ != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(err_));         \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

// n2 = number of double2 elements; blocks take contiguous spans of 4 x 256 elements
__global__ void __launch_bounds__(256, 2) k1(size_t n2, const double2* __restrict__ a,
                                             const double2* __restrict__ b,
                                             double2* __restrict__ c) {
  const size_t span = 1024, nspan = (n2 + span - 1) / span;
  for (size_t s = blockIdx.x; s < nspan; s += gridDim.x) {
    double2 x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t i = s * span + u * 256 + threadIdx.x;
      if (i < n2) {
        x[u] = a[i];
        y[u] = b[i];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t i = s * span + u * 256 + threadIdx.x;
      if (i < n2) c[i] = make_double2(x[u].x * y[u].x, x[u].y * y[u].y);
    }
  }
}

template <int REV>
__global__ void __launch_bounds__(256, 2) k2(size_t n2, double2* __restrict__ d,
                                             const double2* __restrict__ c,
                                             const double2* __restrict__ e, double alpha) {
  const size_t span = 1024, nspan = (n2 + span - 1) / span;
  for (size_t s0 = blockIdx.x; s0 < nspan; s0 += gridDim.x) {
    const size_t s = REV ? nspan - 1 - s0 : s0;
    double2 x[4], y[4], z[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t i = s * span + u * 256 + threadIdx.x;
      if (i < n2) {
        x[u] = d[i];
        y[u] = c[i];
        z[u] = e[i];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t i = s * span + u * 256 + threadIdx.x;
      if (i < n2)
        d[i] = make_double2((x[u].x - alpha * y[u].x) * z[u].x, (x[u].y - alpha * y[u].y) * z[u].y);
    }
  }
}

int main(int argc, char** argv) {
  const size_t rows = argc > 1 ? atol(argv[1]) : 261121;
  const size_t S = argc > 2 ? atol(argv[2]) : 32;
  const size_t n = rows * S, n2 = n / 2;
  double *a, *b, *c, *d, *e, *junk;
  CK(cudaMalloc(&a, n * 8));
  CK(cudaMalloc(&b, n * 8));
  CK(cudaMalloc(&c, n * 8));
  CK(cudaMalloc(&d, n * 8));
  CK(cudaMalloc(&e, n * 8));
  const size_t junk_n = (size_t)64 << 20;  // 512 MB: flushes L2
  CK(cudaMalloc(&junk, junk_n * 8));
  CK(cudaMemset(a, 0, n * 8));
  CK(cudaMemset(b, 0, n * 8));
  CK(cudaMemset(d, 0, n * 8));
  CK(cudaMemset(e, 0, n * 8));
  const int grid = 296;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double bytes = 4.0 * n * 8;
  printf("vector %.1f MB, K2 moves %.1f MB\n", n * 8 / 1e6, bytes / 1e6);
  for (int mode = 0; mode < 3; ++mode) {  // 0 forward, 1 reverse, 2 cold (L2 flushed between)
    float tot = 0;
    const int reps = 20;
    for (int r = 0; r < reps + 2; ++r) {
      CK(cudaMemsetAsync(junk, 0, junk_n * 8));  // start from a flushed L2
      k1<<<grid, 256>>>(n2, (const double2*)a, (const double2*)b, (double2*)c);
      if (mode == 2) CK(cudaMemsetAsync(junk, 1, junk_n * 8));
      CK(cudaEventRecord(e0));
      if (mode == 1)
        k2<1><<<grid, 256>>>(n2, (double2*)d, (const double2*)c, (const double2*)e, 1e-3);
      else
        k2<0><<<grid, 256>>>(n2, (double2*)d, (const double2*)c, (const double2*)e, 1e-3);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) tot += ms;
    }
    printf("%s: K2 %.1f us, %.0f GB/s algorithmic\n",
           mode == 0 ? "forward after K1" : mode == 1 ? "reverse after K1" : "cold (L2 flushed)",
           tot / reps * 1e3, bytes / (tot / reps) / 1e6);
  }
  return 0;
}
