// uqg_kernels.cu - sm_100a kernels of the ensemble solve hot path.
//
// Layout: G groups x S lanes; matrix values
// [G][nnz][S], vectors [G][N][S]; one shared CSR graph.  All elementwise
// arithmetic that the reference performs with numpy is written with explicit
// round-to-nearest intrinsics (no FMA contraction; the library is also built
// with --fmad=false) so each lane reproduces numpy's rounding sequence.
// Only the order of the reductions (dots/norms) differs from numpy's BLAS.

#include <cuda_runtime.h>
#include <float.h>
#include <math.h>

#include "uqg_common.cuh"
#include "uqg_kernels.cuh"

namespace uqg {

// ===========================================================================
// KL coefficient (random_field.py:145-166)

__device__ __forceinline__ double a_hat_of(const double* y, int M, int mode, double value) {
  if (mode == 0) return value;
  // "test2" (random_field.py:126-132): piecewise amplitude over the sample radius
  double ss = 0.0;
  for (int m = 0; m < M; ++m) ss = __dadd_rn(ss, __dmul_rn(y[m], y[m]));
  const double r = sqrt(ss), d = 1.7320508075688772;  // sqrt(3.0)
  const double f = r < d / 4.0 ? 1.0 : (r < d / 2.0 ? 100.0 : 10.0);
  return __dmul_rn(value, f);
}

__device__ __forceinline__ double kl_finish(double e, int expansion, double a_min, double ahat) {
  e = expansion == 0 ? exp(e) : __dadd_rn(1.0, e);
  return __dadd_rn(a_min, __dmul_rn(ahat, e));
}

// The KL contraction fluct(node, lane) = sum_m (y_m sqrt(lam_m)) * mv_m(node)
// is a dense (P x M)(M x S) product per group followed by exp.  One CTA takes
// one group and a tile of kKlTile consecutive nodes: the lane coefficients
// c[m][s] = y_s[m] * sqrt(lam_m) and the tile's mode values mv[m][k] (rebuilt
// from the separable 1D tables, one rounded product each - bit-identical to
// the host mode table, so the (M x P) table is never streamed from HBM) are
// staged in shared memory once; every (node, lane) element then runs the
// M-term FMA chain in mode order from shared memory (mv broadcast across the
// warp's lanes) and the exp, and the store of a[g][node][lane] is coalesced.
// Same arithmetic, in the same order, as one thread per element recomputing
// everything (kl_sep2d_elem_kernel, kept for M x S too large to stage): same
// bits.  FP64-pipe bound (exp), not HBM bound: ncu in profiles/.
__global__ void __launch_bounds__(256) kl_sep2d_kernel(
    int n1, const double* __restrict__ table1d, const int* __restrict__ mode_p,
    const int* __restrict__ mode_q, const double* __restrict__ sqrt_lam, int M,
    const double* __restrict__ samples, const int* __restrict__ lane_ids, int G, int S,
    double a_min, int a_hat_mode, double a_hat_value, int expansion, double* __restrict__ a_out,
    int* status) {
  extern __shared__ double kl_sm[];
  double* c = kl_sm;                          // [M][S]
  double* ah = c + M * S;                     // [S]
  double* mv = ah + S + ((M * S + S) & 1);    // [M][kKlTile], 16-byte aligned
  const int g = blockIdx.y, t = threadIdx.x, T = blockDim.x;
  const int P = n1 * n1;
  const int p0 = blockIdx.x * kKlTile;
  const int tn = P - p0 < kKlTile ? P - p0 : kKlTile;
  for (int e = t; e < M * S; e += T) {
    const int m = e / S, s = e - m * S;
    const size_t lane = (size_t)g * S + s;
    const double* y = samples + (lane_ids ? (size_t)__ldg(&lane_ids[lane]) : lane) * M;
    c[e] = __dmul_rn(y[m], __ldg(&sqrt_lam[m]));
  }
  for (int s = t; s < S; s += T) {
    const size_t lane = (size_t)g * S + s;
    const double* y = samples + (lane_ids ? (size_t)__ldg(&lane_ids[lane]) : lane) * M;
    ah[s] = a_hat_of(y, M, a_hat_mode, a_hat_value);
  }
  for (int e = t; e < M * kKlTile; e += T) {
    const int m = e / kKlTile, k = e - m * kKlTile;
    if (k < tn) {
      const int p = p0 + k, i = p / n1, j = p - i * n1;
      mv[e] = __dmul_rn(__ldg(&table1d[(size_t)__ldg(&mode_p[m]) * n1 + i]),
                        __ldg(&table1d[(size_t)__ldg(&mode_q[m]) * n1 + j]));
    }
  }
  __syncthreads();
  double* out = a_out + ((size_t)g * P + p0) * S;
  bool bad = false;
  if (S <= T && T % S == 0) {
    // register blocking: a thread owns lane s and 4 consecutive nodes, so each
    // mode step is one c load (per lane) and two 16-byte mv loads (broadcast
    // across the lanes) for 4 FMAs - the chain per element is unchanged
    const int s = t % S, kr = t / S, RP = T / S;
    const double cs_ah = ah[s];
    for (int k0 = 4 * kr; k0 < tn; k0 += 4 * RP) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int m = 0; m < M; ++m) {
        const double cm = c[m * S + s];
        const double2 v01 = *reinterpret_cast<const double2*>(&mv[m * kKlTile + k0]);
        const double2 v23 = *reinterpret_cast<const double2*>(&mv[m * kKlTile + k0 + 2]);
        acc[0] = __fma_rn(cm, v01.x, acc[0]);
        acc[1] = __fma_rn(cm, v01.y, acc[1]);
        acc[2] = __fma_rn(cm, v23.x, acc[2]);
        acc[3] = __fma_rn(cm, v23.y, acc[3]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (k0 + q < tn) {
          const double a = kl_finish(acc[q], expansion, a_min, cs_ah);
          bad |= a <= 0.0;
          out[(size_t)(k0 + q) * S + s] = a;
        }
      }
    }
  } else {
    for (int e = t; e < tn * S; e += T) {
      const int k = e / S, s = e - k * S;
      double acc = 0.0;
      for (int m = 0; m < M; ++m) acc = __fma_rn(c[m * S + s], mv[m * kKlTile + k], acc);
      const double a = kl_finish(acc, expansion, a_min, ah[s]);
      bad |= a <= 0.0;
      out[e] = a;
    }
  }
  if (bad) atomicOr(status, 1);
}

// One thread per (group, node, lane), everything recomputed per element (for
// M x S beyond the shared-memory staging of kl_sep2d_kernel; same bits).
__global__ void kl_sep2d_elem_kernel(int n1, const double* __restrict__ table1d,
                                const int* __restrict__ mode_p, const int* __restrict__ mode_q,
                                const double* __restrict__ sqrt_lam, int M,
                                const double* __restrict__ samples,
                                const int* __restrict__ lane_ids, int G, int S, double a_min,
                                int a_hat_mode, double a_hat_value, int expansion,
                                double* __restrict__ a_out, int* status) {
  const long long P = (long long)n1 * n1;
  const long long total = (long long)G * P * S;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(idx % S);
    const long long gp = idx / S;
    const long long p = gp % P;
    const int g = (int)(gp / P);
    const int i = (int)(p / n1), j = (int)(p % n1);
    const size_t lane = (size_t)g * S + s;
    const double* y = samples + (lane_ids ? (size_t)__ldg(&lane_ids[lane]) : lane) * M;
    double e = 0.0;
    for (int m = 0; m < M; ++m) {
      const double mv = __dmul_rn(__ldg(&table1d[(size_t)__ldg(&mode_p[m]) * n1 + i]),
                                  __ldg(&table1d[(size_t)__ldg(&mode_q[m]) * n1 + j]));
      e = __fma_rn(__dmul_rn(y[m], __ldg(&sqrt_lam[m])), mv, e);
    }
    const double a = kl_finish(e, expansion, a_min, a_hat_of(y, M, a_hat_mode, a_hat_value));
    if (a <= 0.0) atomicOr(status, 1);
    a_out[idx] = a;
  }
}

// Dense-table form, output lane-major [L][P] (eval_a_batch's (S, P)).
__global__ void kl_table_kernel(const double* __restrict__ modes, int P, int M,
                                const double* __restrict__ sqrt_lam,
                                const double* __restrict__ samples, int L, double a_min,
                                int a_hat_mode, double a_hat_value, int expansion,
                                double* __restrict__ a_out, int* status) {
  const long long total = (long long)L * P;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(idx / P);
    const long long p = idx % P;
    const double* y = samples + (size_t)l * M;
    double e = 0.0;
    for (int m = 0; m < M; ++m)
      e = __fma_rn(__dmul_rn(y[m], __ldg(&sqrt_lam[m])), __ldg(&modes[(size_t)m * P + p]), e);
    const double a = kl_finish(e, expansion, a_min, a_hat_of(y, M, a_hat_mode, a_hat_value));
    if (a <= 0.0) atomicOr(status, 1);
    a_out[idx] = a;
  }
}

// ===========================================================================
// 2D 5-point FV assembly (oracle/fv2d.py; contract of fem3d.py:138-175)

__device__ __forceinline__ double harm(double a, double b) {
  return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, a), b), __dadd_rn(a, b));
}

__global__ void assemble_fv2d_kernel(int n, int G, int S, const double* __restrict__ a_nodes,
                                     double a_y, int a2_same, const int* __restrict__ row_offsets,
                                     double* __restrict__ vals, double* __restrict__ dinv) {
  const int m = n - 1, n1 = n + 1;
  const long long N = (long long)m * m, P = (long long)n1 * n1;
  const long long nnz = 5 * N - 4 * (long long)m;
  const long long total = (long long)G * N * S;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(idx % S);
    const long long gr = idx / S;
    const long long row = gr % N;
    const int g = (int)(gr / N);
    const int i = (int)(row / m) + 1, j = (int)(row % m) + 1;
    const double* a = a_nodes + (size_t)g * P * S + s;
    const long long c = (long long)i * n1 + j;
    const double ac = a[c * S];
    const double tw = harm(a[(c - n1) * S], ac);
    const double te = harm(ac, a[(c + n1) * S]);
    double ts = a_y, tn = a_y;
    if (a2_same) {
      ts = harm(a[(c - 1) * S], ac);
      tn = harm(ac, a[(c + 1) * S]);
    }
    const double diag = __dadd_rn(__dadd_rn(__dadd_rn(tw, te), ts), tn);
    double* v = vals + ((size_t)g * nnz + row_offsets[row]) * S + s;
    int k = 0;
    if (i > 1) v[(k++) * S] = -tw;
    if (j > 1) v[(k++) * S] = -ts;
    v[(k++) * S] = diag;
    if (j < m) v[(k++) * S] = -tn;
    if (i < m) v[(k++) * S] = -te;
    if (dinv) dinv[idx] = __ddiv_rn(1.0, diag);
  }
}

// Face form of the same operator (Fv2dOp in uqg_kernels.cuh): one thread per
// (group, face slot, lane).  Face slot q in [0, (m+1)*m) writes the x-face
// tx[q] (rows f = q / m and f + 1, column j = q % m + 1), the y-face ty[q]
// (row i = q / (m+1) + 1, columns k = q % (m+1) and k + 1) when the y
// coefficient is random, and - for q < N, cell q - the Jacobi inverse
// diagonal.  Same harmonic means and diagonal sum as assemble_fv2d_kernel.
__global__ void assemble_fv2d_faces_kernel(int n, int G, int S, const double* __restrict__ a_nodes,
                                           int a2_same, double a_y, double* __restrict__ tx,
                                           double* __restrict__ ty, double* __restrict__ dinv) {
  const int m = n - 1, n1 = n + 1;
  const long long N = (long long)m * m, F = N + m, P = (long long)n1 * n1;
  const long long total = (long long)G * F * S;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(idx % S);
    const long long gq = idx / S;
    const long long q = gq % F;
    const int g = (int)(gq / F);
    const double* a = a_nodes + (size_t)g * P * S + s;
    {
      const int f = (int)(q / m), j = (int)(q % m) + 1;
      tx[idx] = harm(a[((long long)f * n1 + j) * S], a[((long long)(f + 1) * n1 + j) * S]);
    }
    if (a2_same) {
      const int i = (int)(q / (m + 1)) + 1, k = (int)(q % (m + 1));
      ty[idx] = harm(a[((long long)i * n1 + k) * S], a[((long long)i * n1 + k + 1) * S]);
    }
    if (dinv && q < N) {
      const int i = (int)(q / m) + 1, j = (int)(q % m) + 1;
      const long long c = (long long)i * n1 + j;
      const double ac = a[c * S];
      const double tw = harm(a[(c - n1) * S], ac);
      const double te = harm(ac, a[(c + n1) * S]);
      double ts = a_y, tn = a_y;
      if (a2_same) {
        ts = harm(a[(c - 1) * S], ac);
        tn = harm(ac, a[(c + 1) * S]);
      }
      const double diag = __dadd_rn(__dadd_rn(__dadd_rn(tw, te), ts), tn);
      dinv[((size_t)g * N + q) * S + s] = __ddiv_rn(1.0, diag);
    }
  }
}

// ===========================================================================
// Jacobi inverse diagonal (ensemble.py:130-137,179-183).  The last diagonal
// entry of a row wins (numpy fancy assignment), an absent one reads 0.

__global__ void jacobi_dinv_kernel(long long N, int S, int G, long long nnz,
                                   const int* __restrict__ ro, const int* __restrict__ ci,
                                   const double* __restrict__ vals, double* __restrict__ dinv,
                                   int* status, int raw) {
  const long long total = (long long)G * N * S;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(idx % S);
    const long long gr = idx / S;
    const long long row = gr % N;
    const int g = (int)(gr / N);
    double d = 0.0;
    for (int k = ro[row]; k < ro[row + 1]; ++k)
      if (ci[k] == row) d = vals[((size_t)g * nnz + k) * S + s];
    if (raw) {
      dinv[idx] = d;
    } else {
      if (d <= 0.0) atomicOr(status, 1);
      dinv[idx] = __ddiv_rn(1.0, d);
    }
  }
}

// ===========================================================================
// 3D trilinear FEM (reference fem3d.py): coefficient at the Gauss points and
// gather-form assembly into the shared 27-point graph.

// a_out [G][E*8][S]; element e = (ex*m + ey)*m + ez, Gauss point q bit-ordered
// (x, y, z), z fastest; qtab[f][2*e_d + bit_d] = factor f at that abscissa.
__global__ void kl_sep3d_kernel(int m, const double* __restrict__ qtab,
                                const int* __restrict__ mode_p, const int* __restrict__ mode_q,
                                const int* __restrict__ mode_r,
                                const double* __restrict__ sqrt_lam, int M,
                                const double* __restrict__ samples,
                                const int* __restrict__ lane_ids, int G, int S, double a_min,
                                int a_hat_mode, double a_hat_value, int expansion,
                                double* __restrict__ a_out, int* status) {
  const long long Q = 8LL * m * m * m;
  const long long total = (long long)G * Q * S;
  const int w = 2 * m;  // table row length
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(idx % S);
    const long long gq = idx / S;
    const long long eq = gq % Q;
    const int g = (int)(gq / Q);
    const long long e = eq >> 3;
    const int q = (int)(eq & 7);
    const int ez = (int)(e % m), ey = (int)((e / m) % m), ex = (int)(e / ((long long)m * m));
    const int tx = 2 * ex + ((q >> 2) & 1), ty = 2 * ey + ((q >> 1) & 1), tz = 2 * ez + (q & 1);
    const size_t lane = (size_t)g * S + s;
    const double* y = samples + (lane_ids ? (size_t)__ldg(&lane_ids[lane]) : lane) * M;
    double acc = 0.0;
    for (int k = 0; k < M; ++k) {
      const double mv =
          __dmul_rn(__dmul_rn(__ldg(&qtab[(size_t)__ldg(&mode_p[k]) * w + tx]),
                              __ldg(&qtab[(size_t)__ldg(&mode_q[k]) * w + ty])),
                    __ldg(&qtab[(size_t)__ldg(&mode_r[k]) * w + tz]));
      acc = __fma_rn(__dmul_rn(y[k], __ldg(&sqrt_lam[k])), mv, acc);
    }
    const double a = kl_finish(acc, expansion, a_min, a_hat_of(y, M, a_hat_mode, a_hat_value));
    if (a <= 0.0) atomicOr(status, 1);
    a_out[idx] = a;
  }
}

// One thread per (group, row, lane).  For each neighbour j of row i (CSR
// order = lexicographic (dx, dy, dz)), sum the contributions of the elements
// holding both nodes in increasing element index (np.bincount's order over
// the (element, a, b) pairs):  K_e(a,b) = (sum_q a_q Dx[q][a][b]) + Kyz[a][b].
__global__ void assemble_fem3d_kernel(int m, int G, int S, const double* __restrict__ a_q,
                                      const double* __restrict__ dx_tab,
                                      const double* __restrict__ kyz_tab,
                                      const int* __restrict__ row_offsets,
                                      double* __restrict__ vals, double* __restrict__ dinv) {
  const int k = m - 1;
  const long long N = (long long)k * k * k;
  const long long nnz = row_offsets[N];
  const long long E = (long long)m * m * m;
  const long long total = (long long)G * N * S;
  __shared__ double sdx[512], skyz[64];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) sdx[i] = dx_tab[i];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) skyz[i] = kyz_tab[i];
  __syncthreads();
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(idx % S);
    const long long gr = idx / S;
    const long long row = gr % N;
    const int g = (int)(gr / N);
    const int iz = (int)(row % k) + 1, iy = (int)((row / k) % k) + 1,
              ix = (int)(row / ((long long)k * k)) + 1;
    const double* aq = a_q + (size_t)g * E * 8 * S + s;
    double* v = vals + ((size_t)g * nnz + row_offsets[row]) * S + s;
    int kk = 0;
    double diag = 0.0;
    for (int dx = -1; dx <= 1; ++dx) {
      const int jx = ix + dx;
      if (jx < 1 || jx > k) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int jy = iy + dy;
        if (jy < 1 || jy > k) continue;
        for (int dz = -1; dz <= 1; ++dz) {
          const int jz = iz + dz;
          if (jz < 1 || jz > k) continue;
          double sum = 0.0;
          for (int ex = max(ix, jx) - 1; ex <= min(ix, jx); ++ex) {
            for (int ey = max(iy, jy) - 1; ey <= min(iy, jy); ++ey) {
              for (int ez = max(iz, jz) - 1; ez <= min(iz, jz); ++ez) {
                const long long e = ((long long)ex * m + ey) * m + ez;
                const int a = (ix - ex) * 4 + (iy - ey) * 2 + (iz - ez);
                const int b = (jx - ex) * 4 + (jy - ey) * 2 + (jz - ez);
                double kx = 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  kx = __dadd_rn(kx, __dmul_rn(aq[(size_t)(e * 8 + q) * S], sdx[q * 64 + a * 8 + b]));
                sum = __dadd_rn(sum, __dadd_rn(kx, skyz[a * 8 + b]));
              }
            }
          }
          v[(size_t)(kk++) * S] = sum;
          if (dx == 0 && dy == 0 && dz == 0) diag = sum;
        }
      }
    }
    if (dinv) dinv[idx] = __ddiv_rn(1.0, diag);
  }
}

// ===========================================================================
// Grouping: stable rank sort + chunk/pad (grouping.py:83-122)

// Order-preserving 64-bit image of each key for the stable radix sort:
// +0.0 and -0.0 map to the same bits (numpy's stable argsort ties them and
// keeps generation order), negatives flip every bit, non-negatives flip the
// sign bit; ids[i] = i is the payload.  A non-finite key sets status bit 1.
__global__ void key_bits_kernel(const double* __restrict__ keys, int n,
                                unsigned long long* __restrict__ bits, int* __restrict__ ids,
                                int* status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double k = keys[i];
  if (!isfinite(k)) atomicOr(status, 2);
  const unsigned long long b = k == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(k);
  bits[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  ids[i] = i;
}

__global__ void chunk_kernel(const int* __restrict__ order, int n, int S, int K,
                             int* __restrict__ groups, int* __restrict__ pad) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx < (long long)K * S) {
    const long long src = idx < n ? idx : n - 1;  // replicate the last real sample
    groups[idx] = order ? order[src] : (int)src;
  }
  if (idx < K) pad[idx] = idx == K - 1 ? (int)((long long)K * S - n) : 0;
}

}  // namespace uqg
