// stream_probe.cu - achievable HBM bandwidth of the PCG update pattern on B200
// (tuning tool, not part of libuqg.so): read r, Ap, dinv, write r
// (r -= alpha Ap, z = r dinv, per-thread r.r / r.z accumulation), 11.2 GB per
// pass like one C3 launch of pcg_update (42 groups x 4 x 66.85 MB).
//
// Variants (template): VB bytes per access per thread (16 or 32), U rows per
// step (loads of U rows issued before any store), NA: L1::no_allocate loads /
// streaming (.cs) stores.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sp tools/stream_probe.cu
//   /tmp/sp
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));           \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

template <int NA>
__device__ __forceinline__ double2 ld2(const double* p) {
  double2 v;
  if (NA)
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  else
    asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
template <int NA>
__device__ __forceinline__ void ld4(const double* p, double (&o)[4]) {
  if (NA)
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
  else
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
}
template <int NA>
__device__ __forceinline__ void st2(double* p, double2 v) {
  if (NA)
    asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
  else
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
template <int NA>
__device__ __forceinline__ void st4(double* p, const double (&o)[4]) {
  if (NA)
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(o[0]), "d"(o[1]),
                 "d"(o[2]), "d"(o[3]) : "memory");
  else
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(o[0]), "d"(o[1]),
                 "d"(o[2]), "d"(o[3]) : "memory");
}

// n doubles per array; each thread handles E = VB/8 consecutive doubles per row-step
template <int VB, int U, int NA>
__global__ void __launch_bounds__(256) upd(size_t n, double alpha, double* __restrict__ r,
                                           const double* __restrict__ ap,
                                           const double* __restrict__ d, double* out) {
  constexpr int E = VB / 8;
  const size_t nthreads = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double a0 = 0.0, a1 = 0.0;
  const size_t nvec = n / E;
  for (size_t base = tid; base < nvec; base += nthreads * U) {
    double rv[U][E], av[U][E], dv[U][E];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + (size_t)u * nthreads;
      ok[u] = i < nvec;
      if (ok[u]) {
        if constexpr (E == 4) {
          ld4<NA>(r + i * 4, rv[u]);
          ld4<NA>(ap + i * 4, av[u]);
          ld4<NA>(d + i * 4, dv[u]);
        } else {
          double2 x = ld2<NA>(r + i * 2), y = ld2<NA>(ap + i * 2), z = ld2<NA>(d + i * 2);
          rv[u][0] = x.x; rv[u][1 % E] = x.y;
          av[u][0] = y.x; av[u][1 % E] = y.y;
          dv[u][0] = z.x; dv[u][1 % E] = z.y;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
      const size_t i = base + (size_t)u * nthreads;
#pragma unroll
      for (int j = 0; j < E; ++j) {
        rv[u][j] = __dsub_rn(rv[u][j], __dmul_rn(alpha, av[u][j]));
        const double z = __dmul_rn(rv[u][j], dv[u][j]);
        a0 = __fma_rn(rv[u][j], rv[u][j], a0);
        a1 = __fma_rn(rv[u][j], z, a1);
      }
      if constexpr (E == 4) st4<NA>(r + i * 4, rv[u]);
      else st2<NA>(r + i * 2, make_double2(rv[u][0], rv[u][1 % E]));
    }
  }
  if (a0 == 12345.678) out[0] = a0 + a1;  // keep the sums alive
}

template <int VB, int U, int NA>
void run(size_t n, double* r, double* ap, double* d, double* out, int blocks_per_sm) {
  const int sms = 148;
  const int grid = sms * blocks_per_sm;
  upd<VB, U, NA><<<grid, 256>>>(n, 1e-3, r, ap, d, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int reps = 20;
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) upd<VB, U, NA><<<grid, 256>>>(n, 1e-3, r, ap, d, out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;
  int regs = 0;
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, upd<VB, U, NA>));
  regs = fa.numRegs;
  printf("VB=%2d U=%d NA=%d grid=%4d x256 regs=%3d: %.3f ms  %.1f GB/s\n", VB, U, NA, grid, regs, ms,
         4.0 * n * 8 / ms / 1e6);
}

int main() {
  const size_t n = (size_t)42 * 261121 * 32;  // one C3 vector pass: 42 groups
  double *r, *ap, *d, *out;
  CK(cudaMalloc(&r, n * 8));
  CK(cudaMalloc(&ap, n * 8));
  CK(cudaMalloc(&d, n * 8));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(r, 0, n * 8));
  CK(cudaMemset(ap, 0, n * 8));
  CK(cudaMemset(d, 0, n * 8));
  for (int bps : {4, 8}) {
    run<16, 2, 0>(n, r, ap, d, out, bps);
    run<16, 4, 0>(n, r, ap, d, out, bps);
    run<16, 2, 1>(n, r, ap, d, out, bps);
    run<16, 4, 1>(n, r, ap, d, out, bps);
    run<32, 1, 0>(n, r, ap, d, out, bps);
    run<32, 2, 0>(n, r, ap, d, out, bps);
    run<32, 1, 1>(n, r, ap, d, out, bps);
    run<32, 2, 1>(n, r, ap, d, out, bps);
  }
  // plain copy for reference (cudaMemcpy D2D: read + write)
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  for (int i = 0; i < 10; ++i) CK(cudaMemcpyAsync(ap, r, n * 8, cudaMemcpyDeviceToDevice));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("cudaMemcpy D2D: %.1f GB/s (read + write)\n", 2.0 * n * 8 * 10 / ms / 1e6);
  return 0;
}
