// grid_reduce_probe.cu - cost of one grid-wide (all-SM) deterministic
// reduction step on B200, by variant:
//   mode 0: arrival counter only (red.release + ld.acquire poll)
//   mode 1: counter + every CTA loads all partials into shared memory
//   mode 2: mode 1 + the fixed-order sums (16 strided sequential sums / lane, warp tree)
//   mode 3: no counter: partials written LL-style (value halves + phase flag in
//           8-byte words), every CTA polls/reads all of them, then the sums
// halo_kb: each CTA also writes halo_kb KB before arriving and reads its
// neighbour's after (modes 0-2 via the counter's release/acquire, modes 3-4
// LL-encoded with the same flags).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/grid_reduce_probe tools/grid_reduce_probe.cu
//   tools/grid_reduce_probe mode [ctas_per_sm] [halo_kb] [partials_per_cta]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ void arrive(unsigned* c) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
}
__device__ __forceinline__ unsigned poll(const unsigned* c) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
  return v;
}
__device__ __forceinline__ void st_ll(uint2* p, double v, unsigned flag) {
  const unsigned long long b = __double_as_longlong(v);
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"((unsigned)b), "r"(flag),
               "r"((unsigned)(b >> 32)), "r"(flag)
               : "memory");
}
__device__ __forceinline__ bool ld_ll(const uint2* p, unsigned flag, double& v) {
  unsigned a, f0, c, f1;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(f0), "=r"(c), "=r"(f1)
               : "l"(p)
               : "memory");
  v = __longlong_as_double(((unsigned long long)c << 32) | a);
  return f0 == flag && f1 == flag;
}

__global__ void __launch_bounds__(512, 1)
probe(int mode, int iters, int nparts, int halo_d, double* part, uint2* llp, double* halo,
      uint2* llh, unsigned* cnt, double* out) {
  __shared__ double sp[4096];
  __shared__ double s_tot[2];
  const int t = threadIdx.x, b = blockIdx.x, nb = gridDim.x;
  const int total = nparts * nb;  // per lane
  double acc = 1.0;
  unsigned target = 0, flag = 0;
  for (int it = 0; it < iters; ++it) {
    for (int ph = 0; ph < 2; ++ph) {
      ++flag;
      double h = 0.0;
      const int nbh = (b + 1) % nb;
      if (mode <= 2) {
        if (t < 2 * nparts) __stcg(&part[(size_t)b * 2 * nparts + t], acc + t + it);
        for (int i = t; i < halo_d; i += blockDim.x) __stcg(&halo[(size_t)b * halo_d + i], acc + i);
        __syncthreads();
        target += nb;
        if (t == 0) {
          arrive(cnt);
          while (poll(cnt) < target) {
          }
        }
        __syncthreads();
        if (mode >= 1)
          for (int i = t; i < 2 * total; i += blockDim.x) sp[i] = __ldcg(&part[i]);
        for (int i = t; i < halo_d; i += blockDim.x) h += __ldcg(&halo[(size_t)nbh * halo_d + i]);
      } else {
        // LL: the data carries the phase flag; no counter, no fence
        // double-buffered by phase parity: a CTA can only overwrite a buffer
        // after every CTA has published (hence finished reading) the one before
        uint2* lp = llp + (size_t)(flag & 1) * 2 * nb * 2 * nparts;
        uint2* lh = llh + (size_t)(flag & 1) * 2 * nb * (halo_d + 1);
        if (t < 2 * nparts) st_ll(&lp[2 * ((size_t)b * 2 * nparts + t)], acc + t + it, flag);
        for (int i = t; i < halo_d; i += blockDim.x)
          st_ll(&lh[2 * ((size_t)b * halo_d + i)], acc + i, flag);
        for (int i = t; i < 2 * total; i += blockDim.x) {
          double v;
          while (!ld_ll(&lp[2 * (size_t)i], flag, v)) {
          }
          sp[i] = v;
        }
        for (int i = t; i < halo_d; i += blockDim.x) {
          double v;
          while (!ld_ll(&lh[2 * ((size_t)nbh * halo_d + i)], flag, v)) {
          }
          h += v;
        }
      }
      __syncthreads();
      if (mode >= 2 && t < 32) {
        const int lane = t >> 4, jr = t & 15;
        double a = 0.0;
        for (int c = jr; c < total; c += 16) a += sp[2 * c + lane];
        for (int st = 8; st > 0; st >>= 1) {
          const double o = __shfl_down_sync(0xffffffffu, a, st, 16);
          if (jr < st) a += o;
        }
        if (jr == 0) s_tot[lane] = a;
      }
      __syncthreads();
      acc = s_tot[ph & 1] * 1e-30 + h * 1e-40 + 1.0;
    }
  }
  if (t == 0) out[b] = acc;
}

int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 2;
  const int per_sm = argc > 2 ? atoi(argv[2]) : 1;
  const int halo_kb = argc > 3 ? atoi(argv[3]) : 0;
  const int nparts = argc > 4 ? atoi(argv[4]) : 4;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nb = sms * per_sm;
  const int halo_d = halo_kb * 1024 / 8;
  double *part, *halo, *out;
  uint2 *llp, *llh;
  unsigned* cnt;
  cudaMalloc(&part, (size_t)nb * 2 * nparts * 8);
  cudaMalloc(&halo, (size_t)nb * (halo_d + 1) * 8);
  cudaMalloc(&llp, (size_t)nb * 2 * nparts * 32);
  cudaMalloc(&llh, (size_t)nb * (halo_d + 1) * 32);
  cudaMemset(llp, 0, (size_t)nb * 2 * nparts * 32);
  cudaMemset(llh, 0, (size_t)nb * (halo_d + 1) * 32);
  cudaMalloc(&out, nb * 8);
  cudaMalloc(&cnt, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 2000;
    cudaMemset(cnt, 0, 4);
    cudaMemset(llp, 0, (size_t)nb * 2 * nparts * 32);
    cudaMemset(llh, 0, (size_t)nb * (halo_d + 1) * 32);
    void* args[] = {&mode, &iters, (void*)&nparts, (void*)&halo_d, &part, &llp, &halo, &llh, &cnt, &out};
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)probe, nb, 512, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("launch failed: %s\n", cudaGetErrorString(e));
      return 1;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep)
      printf("mode=%d ctas=%d halo=%dKB parts/cta=%d: %.3f us per reduction\n", mode, nb, halo_kb,
             nparts, ms * 1e3 / iters / 2);
  }
  return 0;
}
