// uqg_surrogate.cu - device evaluation of the grouping keys:
//   * the sparse-grid iteration surrogate (HierGrid.eval_many, hier_grid.py:317-359),
//   * the anisotropy indicator of the "par" strategy (random_field.py:254-270).
//
// Surrogate: out[i] = sum_j prod_d max(0, 1 - |y_id - c_jd| / w_jd) * s_j.  The
// per-node basis value is formed exactly as the reference forms it (one
// subtraction, one division, max, product over d in order), so on the
// iteration channel - integer data, dyadic grid - every term and partial sum is
// exact and the keys are bit-identical to the host's BLAS result whatever the
// summation order (checked in tests/test_gpu_surrogate.py).

#include <cuda_runtime.h>
#include <float.h>
#include <math.h>

#include "uqg_common.cuh"
#include "uqg_kernels.cuh"

namespace uqg {

constexpr int kSurrThreads = 256;

// one block per evaluation point; threads stride over the nodes; fixed tree.
__global__ void __launch_bounds__(kSurrThreads) surrogate_eval_kernel(
    const double* __restrict__ points, int n, int dim, const double* __restrict__ centers,
    const double* __restrict__ widths, const double* __restrict__ surplus, int n_nodes,
    double* __restrict__ out) {
  __shared__ double red[kSurrThreads];
  __shared__ double y[64];
  const int i = blockIdx.x, t = threadIdx.x;
  if (t < dim) y[t] = points[(size_t)i * dim + t];
  __syncthreads();
  double acc = 0.0;
  for (int j = t; j < n_nodes; j += kSurrThreads) {
    double b = 1.0;
    for (int d = 0; d < dim; ++d) {
      double v = __dsub_rn(1.0, __ddiv_rn(fabs(__dsub_rn(y[d], centers[(size_t)j * dim + d])),
                                          widths[(size_t)j * dim + d]));
      v = v > 0.0 ? v : 0.0;
      b = __dmul_rn(b, v);
    }
    acc = __fma_rn(b, surplus[j], acc);
  }
  red[t] = acc;
  __syncthreads();
  for (int st = kSurrThreads / 2; st > 0; st >>= 1) {
    if (t < st) red[t] += red[t + st];
    __syncthreads();
  }
  if (t == 0) out[i] = red[0];
}

// one block per lane (sample); threads over the points; max tree.
__global__ void __launch_bounds__(kSurrThreads) anisotropy_kernel(
    const double* __restrict__ modes, int P, int M, const double* __restrict__ sqrt_lam,
    const double* __restrict__ samples, double a_min, int a_hat_mode, double a_hat_value,
    int expansion, double a_hi, double a_lo, double* __restrict__ out, int* status) {
  __shared__ double red[kSurrThreads];
  const int l = blockIdx.x, t = threadIdx.x;
  const double* y = samples + (size_t)l * M;
  double ah = a_hat_value;
  if (a_hat_mode == 1) {
    double ss = 0.0;
    for (int m = 0; m < M; ++m) ss = __dadd_rn(ss, __dmul_rn(y[m], y[m]));
    const double r = sqrt(ss), d = 1.7320508075688772;
    ah = __dmul_rn(a_hat_value, r < d / 4.0 ? 1.0 : (r < d / 2.0 ? 100.0 : 10.0));
  }
  double mx = 0.0;
  for (int p = t; p < P; p += kSurrThreads) {
    double e = 0.0;
    for (int m = 0; m < M; ++m)
      e = __fma_rn(__dmul_rn(y[m], __ldg(&sqrt_lam[m])), __ldg(&modes[(size_t)m * P + p]), e);
    e = expansion == 0 ? exp(e) : __dadd_rn(1.0, e);
    const double a = __dadd_rn(a_min, __dmul_rn(ah, e));
    const double hi = a > a_hi ? a : a_hi, lo = a < a_lo ? a : a_lo;
    if (lo <= 0.0) atomicOr(status, 1);
    const double ratio = __ddiv_rn(hi, lo);
    mx = ratio > mx ? ratio : mx;
  }
  red[t] = mx;
  __syncthreads();
  for (int st = kSurrThreads / 2; st > 0; st >>= 1) {
    if (t < st) red[t] = red[t + st] > red[t] ? red[t + st] : red[t];
    __syncthreads();
  }
  if (t == 0) out[l] = red[0];
}

void launch_surrogate_eval(cudaStream_t s, const double* points, int n, int dim,
                           const double* centers, const double* widths, const double* surplus,
                           int n_nodes, double* out) {
  surrogate_eval_kernel<<<n, kSurrThreads, 0, s>>>(points, n, dim, centers, widths, surplus,
                                                   n_nodes, out);
}

void launch_anisotropy(cudaStream_t s, const double* modes, int P, int M, const double* sqrt_lam,
                       const double* samples, int L, double a_min, int a_hat_mode,
                       double a_hat_value, int expansion, double a_hi, double a_lo, double* out,
                       int* status) {
  anisotropy_kernel<<<L, kSurrThreads, 0, s>>>(modes, P, M, sqrt_lam, samples, a_min, a_hat_mode,
                                               a_hat_value, expansion, a_hi, a_lo, out, status);
}

}  // namespace uqg
