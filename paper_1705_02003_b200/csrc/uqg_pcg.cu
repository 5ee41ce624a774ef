// uqg_pcg.cu - ensemble SpMV, per-lane dots and the device-resident Jacobi-PCG
// (reference ensemble.py:116-281), templated on V lanes per thread.
//
// One PCG iteration = three streaming kernels over every active group:
//   pcg_spmv   Ap = A p (CSR order, no FMA: bitwise scipy; CSR or the FV2D
//              face form), p.Ap; last chunk: freeze (p.Ap <= DBL_MIN), alpha
//   pcg_update r -= alpha Ap, r.r and r.z (z = dinv r)
//              last chunk: residual norm, history, breakdown, convergence,
//              termination, beta
//   pcg_dir    p = z + beta p, and the solution update x += alpha p:
//              kx = 1: in place every iteration (x's update deferred from
//              pcg_update to pcg_dir: same operands, same rounding);
//              kx > 1: p_{k+1} goes to the next of kx p buffers and
//              pcg_flush applies x += alpha_j p_j for kx iterations at a time
//              (every kx-th iteration, between pcg_update and pcg_dir, and for
//              the tail after the loop) - the same roundings in the same order.
// A group that terminates in pcg_update is in state FINISHING; its pcg_dir
// applies the last in-place x update (kx = 1) and moves it to DONE.  A DONE
// group turns every later launch into a no-op.
//
// Work distribution: blocks of group g (blockIdx.y) grid-stride over the
// group's reduction chunks (consecutive tiles of rows); see Geo.

#include <cuda_runtime.h>
#include <float.h>
#include <math.h>

#include "uqg_common.cuh"
#include "uqg_kernels.cuh"

namespace uqg {

// acc[j] = sum_k v_k[j] * x_{c_k}[j] in CSR order, separate roundings, starting
// from +0.0 exactly like scipy's csr_matvec.  Rows of up to ML entries fetch
// all column indices, then all values / vector entries, before the ordered sum
// (memory-level parallelism); longer rows take the plain loop.  ML = 5 fits
// the 2D 5-point stencil; ML = 8 otherwise.  Results do not depend on ML.
template <int V, int ML>
__device__ __forceinline__ void row_spmv(const int* __restrict__ ci, const double* __restrict__ v,
                                         const double* __restrict__ x, int k0, int k1, int S,
                                         double (&acc)[V]) {
#pragma unroll
  for (int j = 0; j < V; ++j) acc[j] = 0.0;
  const int len = k1 - k0;
  if (len <= ML) {
    int c[ML];
#pragma unroll
    for (int e = 0; e < ML; ++e) c[e] = e < len ? __ldg(&ci[k0 + e]) : 0;
    double a[ML][V], b[ML][V];
#pragma unroll
    for (int e = 0; e < ML; ++e) {
      if (e < len) {
        ldgv<V>(v + (size_t)(k0 + e) * S, a[e]);
        ldv<V>(x + (size_t)c[e] * S, b[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < ML; ++e) {
      if (e < len) {
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(a[e][j], b[e][j]));
      }
    }
  } else {
    for (int k = k0; k < k1; ++k) {
      double a[V], b[V];
      ldgv<V>(v + (size_t)k * S, a);
      ldv<V>(x + (size_t)__ldg(&ci[k]) * S, b);
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(a[j], b[j]));
    }
  }
}

// rows [r0, r1) of a chunk for this thread: row = tile * R + rr
struct ChunkRows {
  long long t0, t1;
};

__device__ __forceinline__ ChunkRows chunk_tiles(const Geo& geo, int chunk) {
  const long long t0 = (long long)chunk * geo.chunk_tiles;
  long long t1 = t0 + geo.chunk_tiles;
  if (t1 > geo.tiles) t1 = geo.tiles;
  return {t0, t1};
}

// ---------------------------------------------------------------------------

template <int V, int ML>
__global__ void __launch_bounds__(256) spmv_kernel(long long N, long long nnz, Geo geo,
                                                   const int* __restrict__ ro,
                                                   const int* __restrict__ ci,
                                                   const double* __restrict__ vals,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y) {
  const int g = blockIdx.y, t = threadIdx.x;
  const int sl = t % geo.Lp, rr = t / geo.Lp, S = geo.S;
  if (sl >= geo.L) return;
  const int o = V * sl;
  const double* vg = vals + (size_t)g * nnz * S + o;
  const double* xg = x + (size_t)g * N * S + o;
  double* yg = y + (size_t)g * N * S + o;
  for (int chunk = blockIdx.x; chunk < geo.chunks; chunk += gridDim.x) {
    const ChunkRows cr = chunk_tiles(geo, chunk);
    for (long long tile = cr.t0; tile < cr.t1; ++tile) {
      const long long row = tile * geo.R + rr;
      if (row < N) {
        double acc[V];
        row_spmv<V, ML>(ci, vg, xg, __ldg(&ro[row]), __ldg(&ro[row + 1]), S, acc);
        stv<V>(yg + row * S, acc);
      }
    }
  }
}

template <int V>
__global__ void __launch_bounds__(256) lane_dot_kernel(long long N, Geo geo,
                                                       const double* __restrict__ a,
                                                       const double* __restrict__ b,
                                                       double* __restrict__ out, double* part,
                                                       unsigned int* ticket) {
  extern __shared__ double red[];
  const int g = blockIdx.y, t = threadIdx.x;
  const int sl = t % geo.Lp, rr = t / geo.Lp, S = geo.S;
  const size_t base = (size_t)g * N * S + V * sl;
  for (int chunk = blockIdx.x; chunk < geo.chunks; chunk += gridDim.x) {
    double acc[1][V] = {};
    if (sl < geo.L) {
      const ChunkRows cr = chunk_tiles(geo, chunk);
      for (long long tile = cr.t0; tile < cr.t1; ++tile) {
        const long long row = tile * geo.R + rr;
        if (row < N) {
          double av[V], bv[V];
          ldv<V>(a + base + row * S, av);
          ldv<V>(b + base + row * S, bv);
#pragma unroll
          for (int j = 0; j < V; ++j) acc[0][j] = __fma_rn(av[j], bv[j], acc[0][j]);
        }
      }
    }
    if (reduce_lanes<1, V>(acc, red, part, ticket, g, chunk, geo) && t < geo.L) {
#pragma unroll
      for (int j = 0; j < V; ++j) out[(size_t)g * S + V * t + j] = red[j * geo.T + t];
    }
  }
}

// ---------------------------------------------------------------------------
// PCG

template <int V>
__global__ void __launch_bounds__(256) pcg_init_kernel(long long N, Geo geo, PcgState st,
                                                       const double* __restrict__ rhs,
                                                       double rhs_const,
                                                       const double* __restrict__ dinv,
                                                       double tol, int maxit,
                                                       double* __restrict__ x,
                                                       double* __restrict__ r,
                                                       double* __restrict__ p) {
  extern __shared__ double red[];
  const int g = blockIdx.y, t = threadIdx.x;
  const int sl = t % geo.Lp, rr = t / geo.Lp, S = geo.S;
  const size_t base = (size_t)g * N * S + V * sl;
  for (int chunk = blockIdx.x; chunk < geo.chunks; chunk += gridDim.x) {
    double acc[2][V] = {};  // b.b, r.z
    if (sl < geo.L) {
      const ChunkRows cr = chunk_tiles(geo, chunk);
      for (long long tile = cr.t0; tile < cr.t1; ++tile) {
        const long long row = tile * geo.R + rr;
        if (row < N) {
          const size_t o = base + row * S;
          double bv[V], zv[V], zero[V];
          if (rhs) {
            ldv<V>(rhs + o, bv);
          } else {
#pragma unroll
            for (int j = 0; j < V; ++j) bv[j] = rhs_const;
          }
          if (dinv) {
            double dv[V];
            ldgv<V>(dinv + o, dv);
#pragma unroll
            for (int j = 0; j < V; ++j) zv[j] = __dmul_rn(bv[j], dv[j]);
          } else {
#pragma unroll
            for (int j = 0; j < V; ++j) zv[j] = bv[j];
          }
#pragma unroll
          for (int j = 0; j < V; ++j) {
            zero[j] = 0.0;
            acc[0][j] = __fma_rn(bv[j], bv[j], acc[0][j]);
            acc[1][j] = __fma_rn(bv[j], zv[j], acc[1][j]);
          }
          stv<V>(x + o, zero);
          stv<V>(r + o, bv);
          stv<V>(p + o, zv);
        }
      }
    }
    if (!reduce_lanes<2, V>(acc, red, st.part, st.ticket, g, chunk, geo)) continue;
    __shared__ int s_all;
    if (t == 0) s_all = 1;
    __syncthreads();
    if (t < geo.L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const size_t l = (size_t)g * S + V * t + j;
        const double bn = sqrt(red[j * geo.T + t]);
        const double thr = tol * bn;
        const bool conv = bn <= thr;  // zero right-hand sides converge at iteration 0
        st.thr[l] = thr;
        st.rz[l] = red[(V + j) * geo.T + t];
        st.conv[l] = conv;
        st.frozen[l] = 0;
        st.iters[l] = 0;
        if (st.hist) st.hist[l] = bn;
        if (!conv) s_all = 0;
      }
    }
    __syncthreads();
    if (t == 0) {
      st.it[g] = 0;
      st.status[g] = 0;
      const int done = s_all || maxit == 0;  // x = 0 is final: no pending update
      st.done[g] = done ? kDone : kRunning;
      if (done) atomicAdd(st.ndone, 1);
    }
  }
}

template <int V, int ML>
__global__ void __launch_bounds__(256) pcg_spmv_kernel(long long N, long long nnz, Geo geo,
                                                       PcgState st, const int* __restrict__ ro,
                                                       const int* __restrict__ ci,
                                                       const double* __restrict__ vals,
                                                       const double* __restrict__ p,
                                                       double* __restrict__ ap) {
  extern __shared__ double red[];
  const int g = blockIdx.y, t = threadIdx.x;
  if (st.done[g] != kRunning) return;
  const int xs = xslot(st, st.it[g]);  // buffer of p_k / alpha_k
  p += (size_t)xs * st.pstride;
  const int sl = t % geo.Lp, rr = t / geo.Lp, S = geo.S;
  const double* vg = vals + (size_t)g * nnz * S + V * sl;
  const size_t base = (size_t)g * N * S + V * sl;
  const double* pg = p + base;
  for (int chunk = blockIdx.x; chunk < geo.chunks; chunk += gridDim.x) {
    double acc[1][V] = {};
    if (sl < geo.L) {
      const ChunkRows cr = chunk_tiles(geo, chunk);
      for (long long tile = cr.t0; tile < cr.t1; ++tile) {
        const long long row = tile * geo.R + rr;
        if (row < N) {
          double y[V], pv[V];
          row_spmv<V, ML>(ci, vg, pg, __ldg(&ro[row]), __ldg(&ro[row + 1]), S, y);
          stv<V>(ap + base + row * S, y);
          ldv<V>(pg + row * S, pv);
#pragma unroll
          for (int j = 0; j < V; ++j) acc[0][j] = __fma_rn(pv[j], y[j], acc[0][j]);
        }
      }
    }
    if (!reduce_lanes<1, V>(acc, red, st.part, st.ticket, g, chunk, geo)) continue;
    if (t < geo.L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const size_t l = (size_t)g * S + V * t + j;
        const double pap = red[j * geo.T + t];
        const unsigned char fr = st.frozen[l] | (unsigned char)(pap <= DBL_MIN);
        st.frozen[l] = fr;
        st.alpha[(size_t)xs * st.G * S + l] = fr ? 0.0 : __ddiv_rn(st.rz[l], pap);
      }
    }
    if (t == 0) st.it[g] += 1;
  }
}

// Face-form FV2D operator (Fv2dOp): same reduction chunks and state updates
// as pcg_spmv_kernel, the row's Ap re-derived from the faces (fv2d_row).
// One row of the face-form operator: loads, then the CSR-order sum.
// TY: -1 = y-face array decided at run time (tyg NULL or not), 0 = constant
// y-faces a_y (compile time), 1 = y-face array.
template <int V, int TY = -1>
struct FaceRow {
  double tw[V], te[V], ts[V], tn[V], pw[V], ps[V], pc[V], pn[V], pe[V];
  bool w, s, n, e;
  __device__ __forceinline__ void load(const double* __restrict__ txg,
                                       const double* __restrict__ tyg,
                                       const double* __restrict__ pg, double a_y, int m, int S,
                                       int row, int i0, int j0) {
    ldgv<V>(txg + row * S, tw);
    ldgv<V>(txg + (row + m) * S, te);
    if (TY == 1 || (TY < 0 && tyg)) {
      ldgv<V>(tyg + (row + i0) * S, ts);
      ldgv<V>(tyg + (row + i0 + 1) * S, tn);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) ts[j] = tn[j] = a_y;
    }
    w = i0 > 0;
    s = j0 > 0;
    n = j0 < m - 1;
    e = i0 < m - 1;
    if (w) ldgv<V>(pg + (row - m) * S, pw);
    if (s) ldgv<V>(pg + (row - 1) * S, ps);
    ldgv<V>(pg + row * S, pc);
    if (n) ldgv<V>(pg + (row + 1) * S, pn);
    if (e) ldgv<V>(pg + (row + m) * S, pe);
  }
  // y = row of A p (fv2d_row's arithmetic); acc += p[row] * y (fused)
  __device__ __forceinline__ void apply(double (&y)[V], double (&acc)[V]) const {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const double d = __dadd_rn(__dadd_rn(__dadd_rn(tw[j], te[j]), ts[j]), tn[j]);
      double a = 0.0;
      if (w) a = __dadd_rn(a, __dmul_rn(-tw[j], pw[j]));
      if (s) a = __dadd_rn(a, __dmul_rn(-ts[j], ps[j]));
      a = __dadd_rn(a, __dmul_rn(d, pc[j]));
      if (n) a = __dadd_rn(a, __dmul_rn(-tn[j], pn[j]));
      if (e) a = __dadd_rn(a, __dmul_rn(-te[j], pe[j]));
      y[j] = a;
      acc[j] = __fma_rn(pc[j], a, acc[j]);
    }
  }
};

// Chunks are reduced in batches of up to kFaceBatch (reduce_lanes_batch: one
// tree and one ticket per batch, same bits as per-chunk reduce_lanes).
#ifndef UQG_FACE_MINB
#define UQG_FACE_MINB 4
#endif
#ifndef UQG_FACE_BATCH
#define UQG_FACE_BATCH 8
#endif
constexpr int kFaceBatch = UQG_FACE_BATCH;
static_assert(kFaceBatch <= kMaxBatch, "batch exceeds reduce_lanes_batch's limit");

template <int V, int TY = -1>
__device__ __forceinline__ void face_spmv_body(long long N, const Geo& geo, const PcgState& st,
                                               const Fv2dOp& op, const double* __restrict__ p,
                                               double* __restrict__ ap) {
  extern __shared__ __align__(16) double red[];
  const int g = blockIdx.y, t = threadIdx.x;
  if (st.done[g] != kRunning) return;
  const int xs = xslot(st, st.it[g]);  // buffer of p_k / alpha_k
  p += (size_t)xs * st.pstride;
  const int sl = t % geo.Lp, rr = t / geo.Lp, S = geo.S, R = geo.R, m = op.m;
  const int n = (int)N, B = gridDim.x, T = geo.T;
  const size_t base = (size_t)g * N * S + V * sl;
  const double* pg = p + base;
  double* apg = ap + base;
  const size_t fo = (size_t)g * (N + m) * S + V * sl;
  const double* txg = op.tx + fo;
  const double* tyg = op.ty ? op.ty + fo : nullptr;
  const int ct = (int)geo.chunk_tiles;
  for (int c0 = blockIdx.x; c0 < geo.chunks; c0 += kFaceBatch * B) {
    int nk = (geo.chunks - 1 - c0) / B + 1;
    if (nk > kFaceBatch) nk = kFaceBatch;
    for (int k = 0; k < nk; ++k) {
      const int chunk = c0 + k * B;
      double acc[V] = {};
      if (sl < geo.L) {
        int row = chunk * ct * R + rr;  // first row of this thread in the chunk
        int rend = (chunk + 1) * ct * R;
        if (rend > n) rend = n;
        int i0 = row / m, j0 = row - i0 * m;
        for (; row < rend; row += R) {
          FaceRow<V, TY> f;
          f.load(txg, tyg, pg, op.a_y, m, S, row, i0, j0);
          double y[V];
          f.apply(y, acc);
          stv<V>(apg + row * S, y);
          j0 += R;
          while (j0 >= m) {
            j0 -= m;
            ++i0;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < V; ++j) red[(k * V + j) * T + t] = acc[j];
    }
    if (!reduce_lanes_batch<1, V>(red, st.part, st.ticket, g, c0, B, nk, geo)) continue;
    if (t < geo.L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const size_t l = (size_t)g * S + V * t + j;
        const double pap = red[j * geo.T + t];
        const unsigned char fr = st.frozen[l] | (unsigned char)(pap <= DBL_MIN);
        st.frozen[l] = fr;
        st.alpha[(size_t)xs * st.G * S + l] = fr ? 0.0 : __ddiv_rn(st.rz[l], pap);
      }
    }
    if (t == 0) st.it[g] += 1;
  }
}

template <int V, int TY = -1>
__global__ void __launch_bounds__(256, UQG_FACE_MINB) pcg_spmv_fv2d_kernel(
    long long N, Geo geo, PcgState st, Fv2dOp op, const double* __restrict__ p,
    double* __restrict__ ap) {
  face_spmv_body<V, TY>(N, geo, st, op, p, ap);
}

template <int V>
__global__ void __launch_bounds__(256) spmv_fv2d_kernel(long long N, Geo geo, Fv2dOp op,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y) {
  const int g = blockIdx.y, t = threadIdx.x;
  const int sl = t % geo.Lp, rr = t / geo.Lp, S = geo.S;
  if (sl >= geo.L) return;
  const size_t base = (size_t)g * N * S + V * sl;
  for (int chunk = blockIdx.x; chunk < geo.chunks; chunk += gridDim.x) {
    const ChunkRows cr = chunk_tiles(geo, chunk);
    for (long long tile = cr.t0; tile < cr.t1; ++tile) {
      const long long row = tile * geo.R + rr;
      if (row < N) {
        double acc[V], xc[V];
        fv2d_row<V, false>(op, N, S, g, V * sl, row, x + base, acc, xc);
        stv<V>(y + base + row * S, acc);
      }
    }
  }
}

// chunks per batched reduction in pcg_update (reduce_lanes_batch)
// Tiles per step of the streaming update / direction kernels (all loads of a
// step issued before any store) and their CTAs per SM: 4 tiles at 2 CTAs/SM
// (128 registers) keep 192 B per thread in flight - C3 level 10.64 -> 10.48 s,
// C2 1.455 -> 1.436 s against 2 tiles at 3 CTAs/SM (tools/runs/sweep_tiles*.sh;
// tools/stream_probe.cu: 7.17 TB/s for this 3-read / 1-write pattern at 4 rows
// per thread vs 6.99 at 2).  Per-thread rows are accumulated in tile order
// either way: same bits.
#ifndef UQG_UPDATE_TILES
#define UQG_UPDATE_TILES 4
#endif
constexpr int kUpdTiles = UQG_UPDATE_TILES;  // tiles per step in pcg_update
#ifndef UQG_DIR_TILES
#define UQG_DIR_TILES 4
#endif
constexpr int kDirTiles = UQG_DIR_TILES;  // tiles per step in pcg_dir
#ifndef UQG_DIR_MINB
#define UQG_DIR_MINB 2
#endif
#ifndef UQG_UPDATE_MINB
#define UQG_UPDATE_MINB 2
#endif
#ifndef UQG_UPDATE_BATCH
#define UQG_UPDATE_BATCH 4
#endif
constexpr int kUpdateBatch = UQG_UPDATE_BATCH;
static_assert(kUpdateBatch <= kMaxBatch, "batch exceeds reduce_lanes_batch's limit");

// HD: 1 = Jacobi scaling present (compiled in), -1 = decided by dinv at run time
template <int V, int HD = -1>
__global__ void __launch_bounds__(256, UQG_UPDATE_MINB) pcg_update_kernel(long long N, Geo geo, PcgState st,
                                                         const double* __restrict__ dinv,
                                                         int maxit, double* __restrict__ r,
                                                         const double* __restrict__ ap) {
  extern __shared__ double red[];
  const int g = blockIdx.y, t = threadIdx.x;
  if (st.done[g] != kRunning) return;
  const int sl = t % geo.Lp, rr = t / geo.Lp, S = geo.S;
  const size_t base = (size_t)g * N * S + V * sl;
  const int k_it = st.it[g] - 1;  // this is iteration k's update
  const size_t GS = (size_t)st.G * S, l0 = (size_t)g * S + V * sl;
  double alpha[V];
#pragma unroll
  for (int j = 0; j < V; ++j)
    alpha[j] = sl < geo.L ? st.alpha[(size_t)xslot(st, k_it) * GS + l0 + j] : 0.0;
  const int B = gridDim.x, T = geo.T;
  for (int c0 = blockIdx.x; c0 < geo.chunks; c0 += kUpdateBatch * B) {
    int nk = (geo.chunks - 1 - c0) / B + 1;
    if (nk > kUpdateBatch) nk = kUpdateBatch;
    for (int k = 0; k < nk; ++k) {
      const int chunk = c0 + k * B;
      double acc[2][V] = {};
      if (sl < geo.L) {
        const ChunkRows cr = chunk_tiles(geo, chunk);
        // kUpdTiles tiles per step: all loads of the step are issued before any store
        for (long long tile = cr.t0; tile < cr.t1; tile += kUpdTiles) {
          double rv[kUpdTiles][V], av[kUpdTiles][V], dv[kUpdTiles][V];
          bool ok[kUpdTiles];
          size_t o[kUpdTiles];
#pragma unroll
          for (int u = 0; u < kUpdTiles; ++u) {
            const long long row = (tile + u) * geo.R + rr;
            ok[u] = tile + u < cr.t1 && row < N;
            o[u] = base + (ok[u] ? row : 0) * S;
            if (ok[u]) {
              ldv<V>(r + o[u], rv[u]);
              ldv<V>(ap + o[u], av[u]);
              if (HD == 1 || (HD < 0 && dinv)) ldgv<V>(dinv + o[u], dv[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < kUpdTiles; ++u) {
            if (!ok[u]) continue;
            double zv[V];
#pragma unroll
            for (int j = 0; j < V; ++j) {
              rv[u][j] = __dsub_rn(rv[u][j], __dmul_rn(alpha[j], av[u][j]));
              zv[j] = (HD == 1 || (HD < 0 && dinv)) ? __dmul_rn(rv[u][j], dv[u][j]) : rv[u][j];
              acc[0][j] = __fma_rn(rv[u][j], rv[u][j], acc[0][j]);
              acc[1][j] = __fma_rn(rv[u][j], zv[j], acc[1][j]);
            }
            stv<V>(r + o[u], rv[u]);
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int j = 0; j < V; ++j) red[((k * 2 + v) * V + j) * T + t] = acc[v][j];
    }
    if (!reduce_lanes_batch<2, V>(red, st.part, st.ticket, g, c0, B, nk, geo)) continue;
    __shared__ int s_all, s_bad;
    if (t == 0) {
      s_all = 1;
      s_bad = 0;
    }
    __syncthreads();
    const int it = st.it[g];
    if (t < geo.L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const size_t l = (size_t)g * S + V * t + j;
        const double rn = sqrt(red[j * geo.T + t]);
        const double rz_new = red[(V + j) * geo.T + t];
        if (st.hist) {
          if (it <= st.hist_cap) st.hist[(size_t)it * st.G * S + l] = rn;
          else atomicOr(st.overflow, 1);
        }
        const bool live = !st.frozen[l];
        if (live && !isfinite(rn)) atomicOr(&s_bad, 1);
        bool conv = st.conv[l];
        if (live && !conv && rn <= st.thr[l]) {
          st.iters[l] = it;
          st.conv[l] = 1;
          conv = true;
        }
        if (live && !conv) atomicAnd(&s_all, 0);
        const double rz_old = st.rz[l];
        st.beta[l] = (live && rz_old > 0.0) ? __ddiv_rn(rz_new, rz_old) : 0.0;
        st.rz[l] = rz_new;
      }
    }
    __syncthreads();
    const bool finish = s_bad || s_all || it >= maxit;
    if (finish && t < geo.L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const size_t l = (size_t)g * S + V * t + j;
        if (!st.conv[l]) st.iters[l] = it;  // unconverged / frozen lanes: iterations run
      }
    }
    if (finish && t == 0) {
      if (s_bad) st.status[g] = 2;
      st.done[g] = kFinishing;  // pcg_dir applies this iteration's x update, then DONE
    }
  }
}

// kx = 1: x += alpha p (deferred here from pcg_update) and p = z + beta p in
// place.  kx > 1 (deferred solution update): only p_{k+1} = z + beta p_k, into
// the next buffer; x is updated by pcg_update's FLUSH iterations and pcg_flush.
template <int V>
__global__ void __launch_bounds__(256, UQG_DIR_MINB) pcg_dir_kernel(long long N, Geo geo, PcgState st,
                                                      const double* __restrict__ dinv,
                                                      const double* __restrict__ r,
                                                      double* __restrict__ x,
                                                      double* __restrict__ p) {
  const int g = blockIdx.y, t = threadIdx.x;
  const int state = st.done[g];
  if (state == kDone) return;
  const int sl = t % geo.Lp, rr = t / geo.Lp, S = geo.S;
  const bool running = state == kRunning, inplace = st.kx == 1;
  if (sl < geo.L && (running || inplace)) {
    const int it = st.it[g], k = it - 1;
    double alpha[V], beta[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      alpha[j] = st.alpha[(size_t)xslot(st, k) * st.G * S + (size_t)g * S + V * sl + j];
      beta[j] = st.beta[(size_t)g * S + V * sl + j];
    }
    const size_t base = (size_t)g * N * S + V * sl;
    const double* pk = p + (size_t)xslot(st, k) * st.pstride;
    double* pn = p + (size_t)xslot(st, it) * st.pstride;  // == pk when kx = 1
    for (int chunk = blockIdx.x; chunk < geo.chunks; chunk += gridDim.x) {
      const ChunkRows cr = chunk_tiles(geo, chunk);
      // kDirTiles tiles per step: all loads of the step are issued before any store
      for (long long tile = cr.t0; tile < cr.t1; tile += kDirTiles) {
        double xv[kDirTiles][V], pv[kDirTiles][V], rv[kDirTiles][V], dv[kDirTiles][V];
        bool ok[kDirTiles];
        size_t o[kDirTiles];
#pragma unroll
        for (int u = 0; u < kDirTiles; ++u) {
          const long long row = (tile + u) * geo.R + rr;
          ok[u] = tile + u < cr.t1 && row < N;
          o[u] = base + (ok[u] ? row : 0) * S;
          if (ok[u]) {
            if (inplace) ldv<V>(x + o[u], xv[u]);
            ldv<V>(pk + o[u], pv[u]);
            if (running) {
              ldv<V>(r + o[u], rv[u]);
              if (dinv) ldgv<V>(dinv + o[u], dv[u]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kDirTiles; ++u) {
          if (!ok[u]) continue;
          if (inplace) {
#pragma unroll
            for (int j = 0; j < V; ++j) xv[u][j] = __dadd_rn(xv[u][j], __dmul_rn(alpha[j], pv[u][j]));
            stv<V>(x + o[u], xv[u]);
          }
          if (running) {
#pragma unroll
            for (int j = 0; j < V; ++j) {
              const double zv = dinv ? __dmul_rn(rv[u][j], dv[u][j]) : rv[u][j];
              pv[u][j] = __dadd_rn(zv, __dmul_rn(beta[j], pv[u][j]));
            }
            stv<V>(pn + o[u], pv[u]);
          }
        }
      }
    }
  }
  if (state == kFinishing && last_block(st.ticket, g, gridDim.x, geo.tstride) && t == 0) {
    st.done[g] = kDone;
    atomicAdd(st.ndone, 1);
  }
}

// Deferred solution update (PcgState::kx > 1): x += alpha_j p_j over a window
// of iterations j, in increasing j.  in_loop: launched between pcg_update and
// pcg_dir of every kx-th iteration (it % kx == 0), window = the last kx
// iterations of every group not yet DONE - before pcg_dir overwrites the
// oldest p buffer.  Otherwise (after the loop): the it % kx updates still
// pending for each group.
// KX: the deepest window this instantiation handles (4 or 8 p buffers); the
// 4-deep kernel streams two tiles per step, the 8-deep one a single tile (the
// window's p values already keep 8 loads per thread in flight).
template <int V, int KX>
__global__ void __launch_bounds__(256, 2) pcg_flush_kernel(long long N, Geo geo, PcgState st,
                                                     double* __restrict__ x,
                                                     const double* __restrict__ p, int in_loop) {
  constexpr int U = KX <= 4 ? 2 : 1;  // tiles per step
  const int g = blockIdx.y, t = threadIdx.x;
  const int it = st.it[g], kx = st.kx;
  const int n = in_loop ? ((st.done[g] != kDone && it % kx == 0) ? kx : 0) : it % kx;
  const int sl = t % geo.Lp, rr = t / geo.Lp, S = geo.S;
  if (n == 0 || sl >= geo.L) return;
  const size_t base = (size_t)g * N * S + V * sl, GS = (size_t)st.G * S;
  const size_t l0 = (size_t)g * S + V * sl;
  double aj[KX][V];
  const double* pj[KX];
#pragma unroll
  for (int q = 0; q < KX; ++q) {  // oldest first: j = it - n + q
    const int sj = q < n ? xslot(st, it - n + q) : 0;
    pj[q] = p + (size_t)sj * st.pstride;
#pragma unroll
    for (int j = 0; j < V; ++j) aj[q][j] = q < n ? st.alpha[(size_t)sj * GS + l0 + j] : 0.0;
  }
  for (int chunk = blockIdx.x; chunk < geo.chunks; chunk += gridDim.x) {
    const ChunkRows cr = chunk_tiles(geo, chunk);
    // U tiles per step: all loads of the step are issued before any store
    for (long long tile = cr.t0; tile < cr.t1; tile += U) {
      double xv[U][V], pv[U][KX][V];
      bool ok[U];
      size_t o[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long row = (tile + u) * geo.R + rr;
        ok[u] = tile + u < cr.t1 && row < N;
        o[u] = base + (ok[u] ? row : 0) * S;
        if (ok[u]) {
          ldv<V>(x + o[u], xv[u]);
#pragma unroll
          for (int q = 0; q < KX; ++q)
            if (q < n) ldv<V>(pj[q] + o[u], pv[u][q]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int q = 0; q < KX; ++q)
          if (q < n)
#pragma unroll
            for (int j = 0; j < V; ++j)
              xv[u][j] = __dadd_rn(xv[u][j], __dmul_rn(aj[q][j], pv[u][q][j]));
        stv<V>(x + o[u], xv[u]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// TMA-staged PCG SpMV.  The matrix values of a tile of R consecutive rows are
// one contiguous span of [nnz][S] (CSR rows are consecutive), so one elected
// thread streams it into shared memory with a bulk async copy
// (cp.async.bulk ... mbarrier::complete_tx) NST tiles ahead of the consumers;
// threads then read values from shared memory and only gather p from global
// memory (mostly L1/L2 hits: p rows are reused by the neighbouring rows of
// the stencil).  Same arithmetic and order as pcg_spmv_kernel, so the results
// are bit-identical; used when S is even, the longest row is <= ML and the
// value array is 16-byte aligned.

constexpr int kStages = 3;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// tile index of the i-th tile a block processes (its chunks b, b+B, ...)
// (32-bit index math: tiles < 2^31, chunk_tiles <= tiles / kMaxChunks + 8)
__device__ __forceinline__ long long block_tile(const Geo& geo, int i, int& chunk) {
  const int ct = (int)geo.chunk_tiles;
  const int j = i / ct;
  chunk = (int)blockIdx.x + j * (int)gridDim.x;
  return (long long)chunk * ct + (i - j * ct);
}

__device__ __forceinline__ int block_tile_count(const Geo& geo) {
  const int nb = (geo.chunks - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  if (nb <= 0) return 0;
  const int last = blockIdx.x + (nb - 1) * gridDim.x;
  long long last_tiles = geo.tiles - (long long)last * geo.chunk_tiles;
  if (last_tiles > geo.chunk_tiles) last_tiles = geo.chunk_tiles;
  return (int)((nb - 1) * geo.chunk_tiles + last_tiles);
}

template <int ML, int NST = kStages, int MINB = 3>
__global__ void __launch_bounds__(256, MINB) pcg_spmv_tma_kernel(long long N, long long nnz, Geo geo,
                                                           PcgState st,
                                                           const int* __restrict__ ro,
                                                           const int* __restrict__ ci,
                                                           const double* __restrict__ vals,
                                                           const double* __restrict__ p,
                                                           double* __restrict__ ap,
                                                           BandHint bh) {
  constexpr int V = 2;
  extern __shared__ __align__(128) double red[];
  const int g = blockIdx.y, t = threadIdx.x;
  if (st.done[g] != kRunning) return;
  const int xs = xslot(st, st.it[g]);  // buffer of p_k / alpha_k
  p += (size_t)xs * st.pstride;
  const int S = geo.S, R = geo.R;
  const double* pg_all = p + (size_t)g * N * S;
  const size_t stage_doubles = (size_t)R * ML * S;
  double* stage = red + (size_t)V * geo.T;  // after the reduction scratch
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage + NST * stage_doubles);
  const double* vg = vals + (size_t)g * nnz * S;
  const int n_tiles = block_tile_count(geo);

  if (t == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int i) {  // thread 0 only
    int chunk;
    const long long tile = block_tile(geo, i, chunk);
    const long long r0 = tile * R;
    const long long r1 = r0 + R < N ? r0 + R : N;
    const int k0 = __ldg(&ro[r0]), k1 = __ldg(&ro[r1]);
    const uint32_t bytes = (uint32_t)(k1 - k0) * (uint32_t)S * 8u;
    uint64_t* bar = &bars[i % NST];
    fence_proxy_async();
    mbar_expect_tx(bar, bytes);
    if (bytes) bulk_g2s(stage + (size_t)(i % NST) * stage_doubles, vg + (size_t)k0 * S, bytes, bar);
    // banded graph: pull the p rows this tile will gather into L2 ahead of use
    // (the +m band is read here for the first time - a DRAM miss otherwise)
#pragma unroll
    for (int b = 0; b < kMaxBands; ++b) {
      if (b < bh.nb) {
        long long lo = r0 + bh.start[b], hi = lo + R + bh.extra[b];
        lo = lo < 0 ? 0 : lo;
        hi = hi > N ? N : hi;
        if (hi > lo) bulk_prefetch_l2(pg_all + lo * S, (uint32_t)(hi - lo) * S * 8u);
      }
    }
  };
  if (t == 0) {
    for (int i = 0; i < NST && i < n_tiles; ++i) issue(i);
  }

  const int sl = t % geo.Lp, rr = t / geo.Lp;
  const size_t base = (size_t)g * N * S + V * sl;
  const double* pg = p + base;
  double acc[1][V] = {};
  for (int i = 0; i < n_tiles; ++i) {
    int chunk;
    const long long tile = block_tile(geo, i, chunk);
    mbar_wait(&bars[i % NST], (uint32_t)((i / NST) & 1));
    if (sl < geo.L) {
      const long long row = tile * R + rr;
      if (row < N) {
        const int kt0 = __ldg(&ro[tile * R]);
        const int k0 = __ldg(&ro[row]), k1 = __ldg(&ro[row + 1]);
        const double* sv = stage + (size_t)(i % NST) * stage_doubles +
                           (size_t)(k0 - kt0) * S + V * sl;
        const int len = k1 - k0;
        int c[ML];
#pragma unroll
        for (int e = 0; e < ML; ++e) c[e] = e < len ? __ldg(&ci[k0 + e]) : 0;
        double b[ML][V];
#pragma unroll
        for (int e = 0; e < ML; ++e)
          if (e < len) ldgv<V>(pg + (size_t)c[e] * S, b[e]);
        double y[V] = {0.0, 0.0};
#pragma unroll
        for (int e = 0; e < ML; ++e) {
          if (e < len) {
            const double2 a = *reinterpret_cast<const double2*>(sv + (size_t)e * S);
            y[0] = __dadd_rn(y[0], __dmul_rn(a.x, b[e][0]));
            y[1] = __dadd_rn(y[1], __dmul_rn(a.y, b[e][1]));
          }
        }
        stv<V>(ap + base + row * S, y);
        double pv[V];
        ldgv<V>(pg + row * S, pv);
#pragma unroll
        for (int j = 0; j < V; ++j) acc[0][j] = __fma_rn(pv[j], y[j], acc[0][j]);
      }
    }
    __syncthreads();  // stage (i % NST) fully consumed
    if (t == 0 && i + NST < n_tiles) issue(i + NST);
    const bool chunk_end = ((i + 1) % geo.chunk_tiles == 0) || (tile == geo.tiles - 1);
    if (chunk_end) {
      if (reduce_lanes<1, V>(acc, red, st.part, st.ticket, g, chunk, geo)) {
        if (t < geo.L) {
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const size_t l = (size_t)g * S + V * t + j;
            const double pap = red[j * geo.T + t];
            const unsigned char fr = st.frozen[l] | (unsigned char)(pap <= DBL_MIN);
            st.frozen[l] = fr;
            st.alpha[(size_t)xs * st.G * S + l] = fr ? 0.0 : __ddiv_rn(st.rz[l], pap);
          }
        }
        if (t == 0) st.it[g] += 1;
      }
      acc[0][0] = acc[0][1] = 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// Cluster form of the face SpMV (S = 32, constant y-faces, reduction chunks of
// exactly m + 1 rows: C3).  The two CTAs of a thread-block cluster take two
// ADJACENT chunks and walk them tile by tile (16 rows).  A ninth warp's lane 0
// fetches, per tile, its chunk's 18 p rows and 17 x-face rows from L2 ONCE with
// cp.async.bulk ... .multicast::cluster into the shared memory of every CTA
// that uses them: the p rows of chunk X are the centre band of X, the east band
// of X - 1 and the west band of X + 1 (rows +- m = chunk rows -+ 1), its faces
// the west faces of X and the east faces of X - 1.  A stage holds three p slots
// (chunk mod 3) and two face slots (chunk mod 2), so a tile lands at the same
// offset in both CTAs; the cluster's outer bands are fetched by the CTA that
// needs them.  Per stage: a FULL mbarrier carrying the transaction bytes of all
// that lands in the stage, and an EMPTY mbarrier on which the eight consumer
// warps of both CTAs arrive (remotely for the other CTA) once they have read it.
// The consumers keep the cyclic row map (thread-row rr takes rows rr + 16 k of
// its chunk in order), FaceRow's arithmetic and the batched chunk reduction, so
// every bit equals pcg_spmv_fv2d_kernel's.  Every wait is bounded: a protocol
// failure raises the group's status instead of hanging.
// (tools/cluster_mc_probe.cu: 6.2 TB/s against 4.8-5.0 for the plain kernel.)
constexpr int kMcStages = 4;  // stages of one 16-row tile
constexpr int kMcBatch = 4;   // chunks per batched reduction (shared memory: 2 CTAs/SM)
constexpr int kMcT = 256;     // consumer threads (8 warps) + one producer warp
constexpr size_t kMcPSlot = 18 * 32, kMcTSlot = 17 * 32;  // doubles
constexpr size_t kMcStage = 3 * kMcPSlot + 2 * kMcTSlot;

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the barrier at the same offset in CTA `rank` of the cluster; relaxed:
// the stage reads it signals are complete once their values have been used
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, unsigned rank) {
  unsigned addr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr)
               : "memory");
}
// CLUSTER: acquire at cluster scope (the producer's wait on the EMPTY barrier, which the
// other CTA's warps signal); else CTA scope - enough for the FULL barrier, whose phase is
// completed by the bulk copies' own complete_tx (a cluster-scope acquire costs an L1
// invalidate, CCTL.IVALL, per wait: 22 % of the stall samples when the consumers used it)
template <bool CLUSTER>
__device__ __forceinline__ bool mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  const long long t0 = clock64();
  for (;;) {
    unsigned ok;
    if constexpr (CLUSTER) {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(bar)), "r"(parity)
          : "memory");
    } else {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(bar)), "r"(parity)
          : "memory");
    }
    if (ok) return true;
    if (clock64() - t0 > (1LL << 33)) return false;  // seconds: never hang
  }
}
__device__ __forceinline__ void bulk_g2s_mc(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, unsigned short mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

// rows [first, first + rows) clipped to [0, limit): first valid row and count
struct McSpan {
  long long lo;
  int n;
};
__device__ __forceinline__ McSpan mc_clip(long long first, int rows, long long limit) {
  const long long lo = first < 0 ? 0 : first;
  const long long hi = first + rows > limit ? limit : first + rows;
  return {lo, hi > lo ? (int)(hi - lo) : 0};
}

__global__ void __launch_bounds__(kMcT + 32, 2) pcg_spmv_fv2d_mc_kernel(
    long long N, Geo geo, PcgState st, Fv2dOp op, const double* __restrict__ p,
    double* __restrict__ ap) {
  constexpr int V = 2, S = 32, L = 16, R = 16, T = kMcT, NW = T / 32, NST = kMcStages;
  extern __shared__ __align__(16) double red[];
  double* stages = red + (size_t)kMcBatch * V * T;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)NST * kMcStage);
  uint64_t* empty = full + NST;
  const int g = blockIdx.y, t = threadIdx.x;
  if (st.done[g] != kRunning) return;  // the same for both CTAs of the cluster
  const int xs = xslot(st, st.it[g]);  // buffer of p_k / alpha_k
  p += (size_t)xs * st.pstride;
  const unsigned c = cluster_ctarank();  // 0: even chunk of the pair, 1: odd
  const int m = op.m, ct = (int)geo.chunk_tiles, crows = ct * R;  // crows == m + 1
  const int ncl = gridDim.x / 2, cid = blockIdx.x / 2;
  const int chunks = geo.chunks, npairs = (chunks + 1) / 2;
  const double* pg = p + (size_t)g * N * S;
  const double* txg = op.tx + (size_t)g * (N + m) * S;
  double* apg = ap + (size_t)g * N * S;
  const long long plim = N, tlim = N + m;
  const bool producer = t >= T;
  if (t == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2 * NW);  // the consumer warps of both CTAs
    }
    fence_mbar_init();
  }
  cluster_sync_all();
  int s = 0;
  unsigned ph = 0;  // parity of the FULL phase of the current pipeline iteration
  long long it = 0;
  bool ok = true;
  const int sl = t % L, rr = t / L;
  for (int q0 = cid; q0 < npairs && ok; q0 += kMcBatch * ncl) {
    int nkp = (npairs - 1 - q0) / ncl + 1;  // chunk pairs of this batch
    if (nkp > kMcBatch) nkp = kMcBatch;
    int nk_mine = 0;                        // ... and my existing chunks among them
    for (int k = 0; k < nkp && ok; ++k) {
      const int X = 2 * (q0 + k * ncl) + (int)c;  // my chunk (>= chunks: no rows)
      if (X < chunks) ++nk_mine;
      const size_t pc_slot = (size_t)(X % 3) * kMcPSlot, pw_slot = (size_t)((X + 2) % 3) * kMcPSlot,
                   pe_slot = (size_t)((X + 1) % 3) * kMcPSlot,
                   tw_slot = 3 * kMcPSlot + (size_t)(X % 2) * kMcTSlot,
                   te_slot = 3 * kMcPSlot + (size_t)((X + 1) % 2) * kMcTSlot;
      const long long c0 = (long long)X * crows;  // first row of my chunk
      if (producer) {
        // chunks X - 1, X, X + 1 entirely inside the vectors: every tile is whole
        const bool interior = c0 - crows - 1 >= 0 && c0 + 2LL * crows + 1 <= plim;
        for (int tile = 0; tile < ct; ++tile, ++it) {
          if ((t & 31) == 0 && interior) {
            double* stage = stages + (size_t)s * kMcStage;
            const size_t o = (size_t)(c0 - 1) * S + (size_t)tile * (R * S);  // row r0 - 1
            constexpr uint32_t pb = (R + 2) * S * 8u, tb = (R + 1) * S * 8u;
            const size_t nb = (size_t)crows * S;  // one chunk of rows
            if (it >= NST && !mbar_wait_bounded<true>(&empty[s], ph ^ 1u)) ok = false;
            if (ok) {
              fence_proxy_async();
              mbar_expect_tx(&full[s], 3 * pb + 2 * tb);
              bulk_g2s_mc(stage + pc_slot, pg + o, pb, &full[s], (unsigned short)3);
              bulk_g2s_mc(stage + tw_slot, txg + o, tb, &full[s], (unsigned short)(c == 0 ? 1 : 3));
              if (c == 0) {
                bulk_g2s(stage + pw_slot, pg + o - nb, pb, &full[s]);
              } else {
                bulk_g2s(stage + pe_slot, pg + o + nb, pb, &full[s]);
                bulk_g2s(stage + te_slot, txg + o + nb, tb, &full[s]);
              }
            }
          } else if ((t & 31) == 0) {
            double* stage = stages + (size_t)s * kMcStage;
            const long long r0 = c0 + (long long)tile * R;
            // tiles of chunks X - 1, X, X + 1 (their rows r0 -+ crows): what lands in my stage
            const McSpan pX = mc_clip(r0 - 1, R + 2, plim), tX = mc_clip(r0 - 1, R + 1, tlim);
            const McSpan pW = mc_clip(r0 - crows - 1, R + 2, plim);
            const McSpan pE = mc_clip(r0 + crows - 1, R + 2, plim),
                         tE = mc_clip(r0 + crows - 1, R + 1, tlim);
            const uint32_t expect = (uint32_t)(pX.n + tX.n + pW.n + pE.n + tE.n) * S * 8u;
            if (it >= NST && !mbar_wait_bounded<true>(&empty[s], ph ^ 1u)) ok = false;
            if (ok) {
              fence_proxy_async();
              if (expect) mbar_expect_tx(&full[s], expect);
              else mbar_arrive(&full[s]);
              // my chunk: p rows to both CTAs, faces to myself and to my west neighbour
              if (pX.n)
                bulk_g2s_mc(stage + pc_slot + (size_t)(pX.lo - (r0 - 1)) * S, pg + pX.lo * S,
                            (uint32_t)pX.n * S * 8u, &full[s], (unsigned short)3);
              if (tX.n)
                bulk_g2s_mc(stage + tw_slot + (size_t)(tX.lo - (r0 - 1)) * S, txg + tX.lo * S,
                            (uint32_t)tX.n * S * 8u, &full[s], (unsigned short)(c == 0 ? 1 : 3));
              if (c == 0) {  // the cluster's west edge: chunk X - 1 is nobody's
                if (pW.n)
                  bulk_g2s(stage + pw_slot + (size_t)(pW.lo - (r0 - crows - 1)) * S, pg + pW.lo * S,
                           (uint32_t)pW.n * S * 8u, &full[s]);
              } else {  // the east edge: chunk X + 1
                if (pE.n)
                  bulk_g2s(stage + pe_slot + (size_t)(pE.lo - (r0 + crows - 1)) * S, pg + pE.lo * S,
                           (uint32_t)pE.n * S * 8u, &full[s]);
                if (tE.n)
                  bulk_g2s(stage + te_slot + (size_t)(tE.lo - (r0 + crows - 1)) * S,
                           txg + tE.lo * S, (uint32_t)tE.n * S * 8u, &full[s]);
              }
            }
          }
          ok = __shfl_sync(0xffffffffu, (int)ok, 0) != 0;
          if (!ok) break;
          if (++s == NST) {
            s = 0;
            ph ^= 1u;
          }
        }
      } else {
        double acc[V] = {0.0, 0.0};
        long long row = c0 + rr;
        long long cend = c0 + crows;
        if (cend > N) cend = N;
        int i0 = (int)(row / m), j0 = (int)(row - (long long)i0 * m);
        for (int tile = 0; tile < ct; ++tile, ++it, row += R) {
          if (!mbar_wait_bounded<false>(&full[s], ph)) ok = false;
          ok = __all_sync(0xffffffffu, (int)ok) != 0;
          if (!ok) break;
          if (row < cend) {
            const double* stage = stages + (size_t)s * kMcStage + V * sl;
            const bool w = i0 > 0, sf = j0 > 0, nf = j0 < m - 1, e = i0 < m - 1;
            const double2 pc = *reinterpret_cast<const double2*>(stage + pc_slot + (size_t)(rr + 1) * S);
            const double2 ps = *reinterpret_cast<const double2*>(stage + pc_slot + (size_t)rr * S);
            const double2 pn = *reinterpret_cast<const double2*>(stage + pc_slot + (size_t)(rr + 2) * S);
            const double2 pw = *reinterpret_cast<const double2*>(stage + pw_slot + (size_t)(rr + 2) * S);
            const double2 pe = *reinterpret_cast<const double2*>(stage + pe_slot + (size_t)rr * S);
            const double2 tw = *reinterpret_cast<const double2*>(stage + tw_slot + (size_t)(rr + 1) * S);
            const double2 te = *reinterpret_cast<const double2*>(stage + te_slot + (size_t)rr * S);
            const double twv[V] = {tw.x, tw.y}, tev[V] = {te.x, te.y}, pwv[V] = {pw.x, pw.y},
                         psv[V] = {ps.x, ps.y}, pcv[V] = {pc.x, pc.y}, pnv[V] = {pn.x, pn.y},
                         pev[V] = {pe.x, pe.y};
            double y[V];
#pragma unroll
            for (int j = 0; j < V; ++j) {  // FaceRow::apply with constant y-faces a_y
              const double d = __dadd_rn(__dadd_rn(__dadd_rn(twv[j], tev[j]), op.a_y), op.a_y);
              double a = 0.0;
              if (w) a = __dadd_rn(a, __dmul_rn(-twv[j], pwv[j]));
              if (sf) a = __dadd_rn(a, __dmul_rn(-op.a_y, psv[j]));
              a = __dadd_rn(a, __dmul_rn(d, pcv[j]));
              if (nf) a = __dadd_rn(a, __dmul_rn(-op.a_y, pnv[j]));
              if (e) a = __dadd_rn(a, __dmul_rn(-tev[j], pev[j]));
              y[j] = a;
              acc[j] = __fma_rn(pcv[j], a, acc[j]);
            }
            stv<V>(apg + row * S + V * sl, y);
          }
          j0 += R;
          while (j0 >= m) {
            j0 -= m;
            ++i0;
          }
          // this warp has read stage s: tell both CTAs' producers
          __syncwarp();
          if ((t & 31) == 0) {
            mbar_arrive_cluster(&empty[s], 0);
            mbar_arrive_cluster(&empty[s], 1);
          }
          if (++s == NST) {
            s = 0;
            ph ^= 1u;
          }
        }
#pragma unroll
        for (int j = 0; j < V; ++j) red[(k * V + j) * T + t] = acc[j];
      }
    }
    if (producer || !ok) continue;
    // the batch's chunk partials and tickets (my chunks: 2 q0 + c, stride 2 ncl)
    if (nk_mine == 0) continue;
    if (!reduce_lanes_batch<1, V, kMcT>(red, st.part, st.ticket, g, 2 * q0 + (int)c, 2 * ncl,
                                        nk_mine, geo))
      continue;
    if (t < geo.L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const size_t l = (size_t)g * S + V * t + j;
        const double pap = red[j * geo.T + t];
        const unsigned char fr = st.frozen[l] | (unsigned char)(pap <= DBL_MIN);
        st.frozen[l] = fr;
        st.alpha[(size_t)xs * st.G * S + l] = fr ? 0.0 : __ddiv_rn(st.rz[l], pap);
      }
    }
    if (t == 0) st.it[g] += 1;
  }
  if (!ok && (t & 31) == 0) atomicOr(&st.status[g], 4);  // pipeline protocol failure
  cluster_sync_all();  // nobody exits while the other CTA may still signal its barriers
}

// ensemble_iterations = max over lanes (ensemble.py:277)
__global__ void pcg_finalize_kernel(PcgState st, int G, int S, int* ens_iters) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  int mx = 0;
  for (int s = 0; s < S; ++s) mx = max(mx, st.iters[(size_t)g * S + s]);
  ens_iters[g] = mx;
}

// ---------------------------------------------------------------------------
// host-side dispatch on V (and the unrolled row length ML)

#define UQG_DISPATCH_V(geo, KERNEL, GRID, SMEM, STREAM, ...)                     \
  do {                                                                           \
    if ((geo).V == 2)                                                            \
      KERNEL<2><<<(GRID), (geo).T, (SMEM), (STREAM)>>>(__VA_ARGS__);             \
    else                                                                         \
      KERNEL<1><<<(GRID), (geo).T, (SMEM), (STREAM)>>>(__VA_ARGS__);             \
  } while (0)

#define UQG_DISPATCH_VML(geo, KERNEL, GRID, SMEM, STREAM, ...)                        \
  do {                                                                                \
    const bool _short = (geo).maxrow >= 1 && (geo).maxrow <= 5;                       \
    if ((geo).V == 2) {                                                               \
      if (_short) KERNEL<2, 5><<<(GRID), (geo).T, (SMEM), (STREAM)>>>(__VA_ARGS__);   \
      else KERNEL<2, 8><<<(GRID), (geo).T, (SMEM), (STREAM)>>>(__VA_ARGS__);          \
    } else {                                                                          \
      if (_short) KERNEL<1, 5><<<(GRID), (geo).T, (SMEM), (STREAM)>>>(__VA_ARGS__);   \
      else KERNEL<1, 8><<<(GRID), (geo).T, (SMEM), (STREAM)>>>(__VA_ARGS__);          \
    }                                                                                 \
  } while (0)

static size_t red_bytes(const Geo& geo, int nv) { return (size_t)nv * geo.V * geo.T * sizeof(double); }

// Blocks per group sized to the kernel's residency (pick_blocks) for the
// geo.gact running groups.
template <class F>
static Geo sized(const Geo& geo, SlotCache& c, F fn, int T, size_t smem) {
  Geo gl = geo;
  gl.B = pick_blocks(geo.gact, geo.chunks, kernel_slots(c, fn, T, smem));
  return gl;
}


void launch_spmv(const Geo& geo, int G, cudaStream_t s, long long N, long long nnz, const int* ro,
                 const int* ci, const double* vals, const double* x, double* y) {
  const Geo gl = with_groups(geo, G);
  UQG_DISPATCH_VML(gl, spmv_kernel, dim3(gl.B, G), 0, s, N, nnz, gl, ro, ci, vals, x, y);
}

void launch_lane_dot(const Geo& geo, int G, cudaStream_t s, long long N, const double* a,
                     const double* b, double* out, double* part, unsigned* ticket) {
  const Geo gl = with_groups(geo, G);
  UQG_DISPATCH_V(gl, lane_dot_kernel, dim3(gl.B, G), red_bytes(gl, 1), s, N, gl, a, b, out, part,
                 ticket);
}

void launch_pcg_init(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                     const double* rhs, double rhs_const, const double* dinv, double tol,
                     int maxit, double* x, double* r, double* p) {
  const Geo gl = with_groups(geo, G);
  UQG_DISPATCH_V(gl, pcg_init_kernel, dim3(gl.B, G), red_bytes(gl, 2), s, N, gl, st, rhs,
                 rhs_const, dinv, tol, maxit, x, r, p);
}

template <int ML, int NST = kStages, int MINB = 3>
static void launch_spmv_tma(const Geo& gl, int G, cudaStream_t s, long long N, long long nnz,
                            const PcgState& st, const int* ro, const int* ci, const double* vals,
                            const double* p, double* ap, const BandHint* bands) {
  const size_t smem = (size_t)2 * gl.T * sizeof(double) +
                      (size_t)NST * gl.R * ML * gl.S * sizeof(double) + NST * 8;
  static size_t configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(pcg_spmv_tma_kernel<ML, NST, MINB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  BandHint bh{};  // L2 prefetch of the p bands (p must be 16-byte aligned)
  if (bands && (reinterpret_cast<uintptr_t>(p) & 15) == 0 && gl.S % 2 == 0) bh = *bands;
  pcg_spmv_tma_kernel<ML, NST, MINB><<<dim3(gl.B, G), gl.T, smem, s>>>(N, nnz, gl, st, ro, ci,
                                                                       vals, p, ap, bh);
}

void launch_spmv_fv2d(const Geo& geo, int G, cudaStream_t s, long long N, const Fv2dOp& op,
                      const double* x, double* y) {
  const Geo gl = with_groups(geo, G);
  UQG_DISPATCH_V(gl, spmv_fv2d_kernel, dim3(gl.B, G), 0, s, N, gl, op, x, y);
}

// UQG_FACE_CLUSTER=1: the cluster / TMA-multicast face SpMV where it applies
// (S = 32, constant y-faces, chunks of m + 1 rows, 16-byte aligned vectors);
// bit-identical to the plain kernel.
static bool face_cluster_enabled() {
  static const bool on = [] {
    const char* e = getenv("UQG_FACE_CLUSTER");
    return e && atoi(e) != 0;
  }();
  return on;
}

static bool launch_pcg_spmv_fv2d_mc(const Geo& geo, int G, cudaStream_t s, long long N,
                                    const PcgState& st, const Fv2dOp& op, const double* p,
                                    double* ap) {
  if (geo.V != 2 || geo.S != 32 || geo.Lp != 16 || geo.T != kMcT || op.ty) return false;
  if (geo.chunk_tiles * geo.R != (long long)op.m + 1 || geo.chunks < 2) return false;
  if ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(op.tx) |
       (uintptr_t)(st.pstride * sizeof(double))) & 15)
    return false;
  const size_t smem = ((size_t)kMcBatch * 2 * kMcT + (size_t)kMcStages * kMcStage) * sizeof(double) +
                      2 * kMcStages * sizeof(uint64_t);
  static int max_clusters = -1;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(kMcT + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  if (max_clusters < 0) {
    if (cudaFuncSetAttribute(pcg_spmv_fv2d_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess) {
      cudaGetLastError();
      max_clusters = 0;
    } else {
      cfg.gridDim = dim3(2, 1);
      int mc = 0;
      if (cudaOccupancyMaxActiveClusters(&mc, pcg_spmv_fv2d_mc_kernel, &cfg) != cudaSuccess) {
        cudaGetLastError();
        mc = 0;
      }
      max_clusters = mc;
    }
  }
  if (max_clusters < 1) return false;
  // clusters per group sized like blocks per group: pairs of chunks over resident clusters
  const int npairs = (geo.chunks + 1) / 2;
  const int b = pick_blocks(geo.gact, npairs, max_clusters);
  cfg.gridDim = dim3(2 * b, G);
  Geo gl = geo;
  gl.B = 2 * b;
  return cudaLaunchKernelEx(&cfg, pcg_spmv_fv2d_mc_kernel, N, gl, st, op, p, ap) == cudaSuccess;
}

void launch_pcg_spmv_fv2d(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                          const Fv2dOp& op, const double* p, double* ap) {
  if (face_cluster_enabled() && launch_pcg_spmv_fv2d_mc(geo, G, s, N, st, op, p, ap)) return;
  static SlotCache cf2, cf1;
  const Geo gl = geo.V == 2
                     ? sized(geo, cf2, pcg_spmv_fv2d_kernel<2>, geo.T,
                             red_bytes(geo, kFaceBatch))
                     : sized(geo, cf1, pcg_spmv_fv2d_kernel<1>, geo.T,
                             red_bytes(geo, kFaceBatch));
  const size_t smem = red_bytes(gl, kFaceBatch);
  // constant y-faces (a2 const, the BASELINE configs) compiled in: fewer live
  // registers, no spill of the y-face branch (C2 face SpMV 2,345 -> 2,277 ms);
  // a y-face array (a2 = "same") takes the run-time branch kernel (same bits).
  if (gl.V == 2 && !op.ty)
    pcg_spmv_fv2d_kernel<2, 0><<<dim3(gl.B, G), gl.T, smem, s>>>(N, gl, st, op, p, ap);
  else if (gl.V == 2)
    pcg_spmv_fv2d_kernel<2><<<dim3(gl.B, G), gl.T, smem, s>>>(N, gl, st, op, p, ap);
  else
    pcg_spmv_fv2d_kernel<1><<<dim3(gl.B, G), gl.T, smem, s>>>(N, gl, st, op, p, ap);
}

void launch_pcg_spmv(const Geo& geo, int G, cudaStream_t s, long long N, long long nnz,
                     const PcgState& st, const int* ro, const int* ci, const double* vals,
                     const double* p, double* ap, const BandHint* bands) {
  const Geo& gl = geo;  // B preset by the caller (blocks per ACTIVE group)
  // TMA-staged values (C2 4.73 TB/s with the band hint's L2 prefetch of the p
  // bands) when S is even, rows are short and the values 16-byte aligned;
  // else the register-gather kernel - identical bits.  (Warp-specialized,
  // 2/4-stage, metadata-staged, band-staged and paired-tile variants were
  // measured slower and removed.)
  const bool aligned = (reinterpret_cast<uintptr_t>(vals) & 15) == 0;
  if (gl.V == 2 && aligned && gl.maxrow >= 1 && gl.maxrow <= 8) {
    if (gl.maxrow <= 5)
      launch_spmv_tma<5>(gl, G, s, N, nnz, st, ro, ci, vals, p, ap, bands);
    else
      launch_spmv_tma<8>(gl, G, s, N, nnz, st, ro, ci, vals, p, ap, bands);
    return;
  }
  UQG_DISPATCH_VML(gl, pcg_spmv_kernel, dim3(gl.B, G), red_bytes(gl, 1), s, N, nnz, gl, st, ro,
                   ci, vals, p, ap);
}

void launch_pcg_update(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                       const double* dinv, int maxit, double* r, const double* ap) {
  static SlotCache c1, c2;
  const size_t smem = red_bytes(geo, 2 * kUpdateBatch);
  static size_t opted = 48 * 1024;  // > 48 KB of dynamic shared memory needs an opt-in
  if (smem > opted) {
    cudaFuncSetAttribute(pcg_update_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(pcg_update_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(pcg_update_kernel<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    opted = smem;
  }
  // Jacobi scaling compiled in (the solver's case); identity preconditioning
  // and V = 1 take the run-time branch kernel (same arithmetic)
  if (geo.V == 2 && dinv) {
    static SlotCache cj;
    const Geo gl = sized(geo, cj, pcg_update_kernel<2, 1>, geo.T, smem);
    pcg_update_kernel<2, 1><<<dim3(gl.B, G), gl.T, smem, s>>>(N, gl, st, dinv, maxit, r, ap);
    return;
  }
  const Geo gl = geo.V == 2 ? sized(geo, c2, pcg_update_kernel<2>, geo.T, smem)
                            : sized(geo, c1, pcg_update_kernel<1>, geo.T, smem);
  UQG_DISPATCH_V(gl, pcg_update_kernel, dim3(gl.B, G), smem, s, N, gl, st, dinv, maxit, r, ap);
}

void launch_pcg_flush(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                      double* x, const double* p, bool in_loop) {
  const Geo& gl = geo;  // B preset by the caller
  const int il = in_loop ? 1 : 0;
  if (st.kx <= 4) {
    if (gl.V == 2)
      pcg_flush_kernel<2, 4><<<dim3(gl.B, G), gl.T, 0, s>>>(N, gl, st, x, p, il);
    else
      pcg_flush_kernel<1, 4><<<dim3(gl.B, G), gl.T, 0, s>>>(N, gl, st, x, p, il);
  } else if (gl.V == 2) {
    pcg_flush_kernel<2, 8><<<dim3(gl.B, G), gl.T, 0, s>>>(N, gl, st, x, p, il);
  } else {
    pcg_flush_kernel<1, 8><<<dim3(gl.B, G), gl.T, 0, s>>>(N, gl, st, x, p, il);
  }
}

void launch_pcg_dir(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                    const double* dinv, const double* r, double* x, double* p) {
  // fixed with_groups target: measured faster for this pure stream than the
  // residency-sized grid (C2: 2043 vs 2099 ms)
  const Geo& gl = geo;
  UQG_DISPATCH_V(gl, pcg_dir_kernel, dim3(gl.B, G), 0, s, N, gl, st, dinv, r, x, p);
}

__global__ void pcg_loop_cond_kernel(cudaGraphConditionalHandle h, const int* ndone, int G,
                                     int* loops, int max_loops) {
  const int l = ++*loops;
  if (*ndone >= G || l >= max_loops) cudaGraphSetConditional(h, 0);
}

void launch_pcg_loop_cond(cudaStream_t s, cudaGraphConditionalHandle h, const int* ndone, int G,
                          int* loops, int max_loops) {
  pcg_loop_cond_kernel<<<1, 1, 0, s>>>(h, ndone, G, loops, max_loops);
}

void launch_pcg_finalize(int G, int S, cudaStream_t s, const PcgState& st, int* ens_iters) {
  pcg_finalize_kernel<<<(G + 127) / 128, 128, 0, s>>>(st, G, S, ens_iters);
}

}  // namespace uqg
