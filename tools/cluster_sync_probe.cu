// cluster_sync_probe.cu - latency floor of one "cluster reduction round" of
// the small-batch (C1) persistent PCG on B200 (tuning tool, not in libuqg.so).
//
// 22 groups, one 16-CTA cluster each (256 threads per CTA, 3-4 CTAs per SM),
// ITERS rounds of: every CTA pushes its NCL chunk partials (S lanes x NV
// values) into every CTA of the cluster over DSMEM, hardware cluster barrier,
// every CTA sums all C partials from its own shared memory in a fixed order
// (R-strided sequential sums + a binary tree over R rows), then a block
// barrier.  mode 0: partials through DSMEM; mode 1: partials through global
// memory (st + __ldcg after the barrier, the current kernel's pattern);
// mode 2: barrier only.  Prints microseconds per round.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/csp tools/cluster_sync_probe.cu
//   /tmp/csp [mode] [rounds_per_iteration]
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

namespace cg = cooperative_groups;

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));           \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

constexpr int S = 8, NV = 2, C = 63, NB = 16, T = 256, LP = 4, R = 64;

template <int MODE>
__global__ void __launch_bounds__(T) probe(int iters, double* gpart, double* out) {
  __shared__ double part[C * NV * S];
  __shared__ double red[NV * 2 * T];
  cg::cluster_group cl = cg::this_cluster();
  const int b = (int)cl.block_rank(), t = threadIdx.x, g = blockIdx.y;
  const int c0 = C * b / NB, c1 = C * (b + 1) / NB;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    // this CTA's chunk partials (fake values)
    const int nv = (c1 - c0) * NV * S;
    if (MODE == 0) {
      for (int e = t; e < nv * NB; e += T) {
        const int dst = e / nv, k = e % nv;
        double* rp = cl.map_shared_rank(part, dst);
        rp[c0 * NV * S + k] = (double)(it + k + b);
      }
    } else if (MODE == 1 || MODE == 3) {
      for (int e = t; e < nv; e += T) gpart[((size_t)g * C + c0) * NV * S + e] = (double)(it + e + b);
    }
    cl.sync();
    if (MODE == 3) {
      // warp-level final stage: combo (v, lane) = warp-strided; lanes hold jr and
      // jr + 32, first level in-thread, then shuffles 16..1 (same pairing)
      const int w = t / 32, l = t % 32;
      __shared__ double tot[NV * S];
      for (int cmb = w; cmb < NV * S; cmb += T / 32) {
        const int v = cmb / S, lane = cmb % S;
        auto ld = [&](int cc) {
          return cc < C ? __ldcg(&gpart[(size_t)g * C * NV * S + (cc * NV + v) * S + lane]) : 0.0;
        };
        double x = ld(l), y = ld(l + 32);
        x += y;
        for (int st = 16; st > 0; st >>= 1) x += __shfl_down_sync(0xffffffffu, x, st);
        if (l == 0) tot[cmb] = x;
      }
      __syncthreads();
      acc += tot[t % (NV * S)];
      __syncthreads();
    } else if (MODE != 2) {
      const int sl = t % LP, jr = t / LP;
      double a[NV * 2] = {};
      if (sl < S / 2)
        for (int cc = jr; cc < C; cc += R)
          for (int v = 0; v < NV; ++v)
            for (int j = 0; j < 2; ++j) {
              const int idx = (cc * NV + v) * S + 2 * sl + j;
              a[v * 2 + j] += MODE == 0 ? part[idx] : __ldcg(&gpart[(size_t)g * C * NV * S + idx]);
            }
      for (int v = 0; v < NV * 2; ++v) red[v * T + t] = a[v];
      __syncthreads();
      for (int st = R / 2; st > 0; st >>= 1) {
        if (jr < st)
          for (int v = 0; v < NV * 2; ++v) red[v * T + t] += red[v * T + t + st * LP];
        __syncthreads();
      }
      acc += red[t % (NV * 2 * T)];
      __syncthreads();
    }
  }
  if (t == 0 && b == 0) out[g] = acc;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int iters = 2000, G = 22;
  double *gpart, *out;
  CK(cudaMalloc(&gpart, (size_t)G * C * NV * S * 8));
  CK(cudaMalloc(&out, G * 8));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(NB, G, 1);
  cfg.blockDim = dim3(T, 1, 1);
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = NB;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  void (*fn)(int, double*, double*) = mode == 0 ? probe<0> : (mode == 1 ? probe<1> : (mode == 2 ? probe<2> : probe<3>));
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaLaunchKernelEx(&cfg, fn, iters, gpart, out));
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  CK(cudaLaunchKernelEx(&cfg, fn, iters, gpart, out));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("mode %d: %.3f us per round (22 clusters x 16 CTAs)\n", mode, ms * 1e3 / iters);
  return 0;
}
