// uqg_persistent.cu - persistent (cooperative) ensemble PCG for small groups.
//
// For small problems (the C1 oracle case: 22 groups x 3,969 rows x 8 lanes, a
// few MB per group) the launch-per-phase loop of uqg_pcg.cu is latency-bound:
// every iteration pays three kernel launches, block scheduling and a
// last-block reduction tail.  Here ONE cooperative launch runs the whole
// solve: the blocks of a group iterate together, separated by group-local
// barriers (atomic arrive + generation flag; all blocks co-resident by
// construction of the cooperative launch), and every block reduces the chunk
// partials itself - in exactly the order of reduce_lanes' final stage - so all
// blocks hold identical per-lane alpha / beta / convergence state without a
// broadcast.  Per iteration: three phases, three barriers, no launches.
//
// Arithmetic and reduction trees are those of uqg_pcg.cu (same chunks, same
// in-chunk trees, same final order), so results are bit-identical to the
// launch-based path.  Loads of vectors written inside the launch bypass L1
// (ld.global.cg) since other SMs update them between phases.

#include <cuda_runtime.h>
#include <float.h>
#include <math.h>

#include "uqg_common.cuh"
#include "uqg_kernels.cuh"

namespace uqg {

namespace {

constexpr long long kBarrierTimeout = 1LL << 35;  // ~17 s at 1.9 GHz: abort, never hang

// Group-local barrier over the nb blocks of group g.
__device__ bool group_sync(unsigned* count, unsigned* gen, unsigned nb, int* abort_flag) {
  __shared__ int s_abort;
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = gen;
    volatile int* vab = abort_flag;
    const unsigned g0 = *vgen;
    __threadfence();
    const unsigned arrived = atomicAdd(count, 1u) + 1u;
    if (arrived == nb) {
      *count = 0u;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      const long long t0 = clock64();
      while (*vgen == g0) {
        if (*vab) break;
        if (clock64() - t0 > kBarrierTimeout) {
          atomicExch(abort_flag, 1);
          break;
        }
        __nanosleep(32);
      }
    }
    __threadfence();
    s_abort = *vab;
  }
  __syncthreads();
  return s_abort == 0;
}

// CL: the group is one thread-block cluster and the barrier is the hardware
// cluster barrier (release/acquire at cluster scope; no spinning, no atomics).
// Its release orders every prior write of the CTA - global partials and
// vectors included - before the other CTAs' acquire, so no separate gpu-scope
// fence is needed (measured: membar stalls were ~10% of the C1 solve).
template <bool CL>
__device__ __forceinline__ bool sync_group(unsigned* count, unsigned* gen, unsigned nb,
                                           int* abort_flag) {
  if constexpr (CL) {
    asm volatile(
        "barrier.cluster.arrive.release.aligned;\n\t"
        "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    return true;
  } else {
    return group_sync(count, gen, nb, abort_flag);
  }
}

// Final reduction over a group's chunk partials (second half of reduce_lanes,
// same order); result of value v, lane V*sl+j in red[(v*V+j)*T + sl].
template <int NV, int V>
__device__ void final_partials(double* red, const double* part, int g, const Geo& geo) {
  constexpr int NS = NV * V;
  const int t = threadIdx.x;
  const int T = geo.T, Lp = geo.Lp, R = geo.R, L = geo.L, S = geo.S, C = geo.chunks;
  __syncthreads();
  const int sl = t % Lp, jr = t / Lp;
  double acc[NS];
#pragma unroll
  for (int v = 0; v < NS; ++v) acc[v] = 0.0;
  if (sl < L) {
#pragma unroll 4
    for (int cc = jr; cc < C; cc += R) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int j = 0; j < V; ++j)
          acc[v * V + j] += __ldcg(&part[(((size_t)g * geo.pstride + cc) * NV + v) * S + V * sl + j]);
    }
  }
#pragma unroll
  for (int v = 0; v < NS; ++v) red[v * T + t] = acc[v];
  __syncthreads();
  tree_rows<NS>(red, T, Lp, R, t);
}

// Chunks are reduced in batches of up to kPersistBatch per in-block tree
// (batch_tree_partials: same partials, same bits as one tree per chunk).
constexpr int kPersistBatch = 4;

template <int NV, int V>
__device__ __forceinline__ void stash(const double (&acc)[NV][V], double* red, int kb, int T,
                                      int t) {
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int j = 0; j < V; ++j) red[((kb * NV + v) * V + j) * T + t] = acc[v][j];
}

__device__ __forceinline__ int batch_count(int c0, int C, int nb) {
  const int n = (C - 1 - c0) / nb + 1;
  return n < kPersistBatch ? n : kPersistBatch;
}

}  // namespace

// Lane state kept (identically) in every block's shared memory.
struct LaneSmem {
  double *alpha, *beta, *rz, *thr;
  int* iters;
  unsigned char *conv, *frozen;
};

template <int V, bool CL>
__global__ void __launch_bounds__(256, 4) pcg_persistent_kernel(
    long long N, long long nnz, Geo geo, PcgState st, const int* __restrict__ ro,
    const int* __restrict__ ci, const double* __restrict__ vals, Fv2dOp fv,
    const double* __restrict__ rhs,
    double rhs_const, const double* __restrict__ dinv, double tol, int maxit,
    double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
    double* __restrict__ ap, double* partA, double* partB, unsigned* bar_count, unsigned* bar_gen,
    int* abort_flag) {
  extern __shared__ __align__(16) double red[];
  const int g = blockIdx.y, t = threadIdx.x;
  const int S = geo.S, T = geo.T, L = geo.L, C = geo.chunks;
  const int sl = t % geo.Lp, rr = t / geo.Lp;
  const unsigned nb = gridDim.x;
  LaneSmem ls;
  ls.alpha = red + kPersistBatch * 2 * V * T;
  ls.beta = ls.alpha + S;
  ls.rz = ls.beta + S;
  ls.thr = ls.rz + S;
  ls.iters = reinterpret_cast<int*>(ls.thr + S);
  ls.conv = reinterpret_cast<unsigned char*>(ls.iters + S);
  ls.frozen = ls.conv + S;
  __shared__ int s_flags[2];  // [0] all converged/frozen, [1] breakdown
  unsigned* cnt = bar_count + g;
  unsigned* gen = bar_gen + g;
  const size_t base = (size_t)g * N * S + V * sl;
  const double* vg = vals ? vals + (size_t)g * nnz * S + V * sl : nullptr;

  // ---- init: x = 0, r = b, p = z, partials b.b and r.z
  for (int c0 = blockIdx.x; c0 < C; c0 += kPersistBatch * nb) {
    const int nk = batch_count(c0, C, nb);
    for (int kb = 0; kb < nk; ++kb) {
      const int chunk = c0 + kb * nb;
      double acc[2][V] = {};
      if (sl < L) {
        const long long t0 = (long long)chunk * geo.chunk_tiles;
        const long long t1 = t0 + geo.chunk_tiles < geo.tiles ? t0 + geo.chunk_tiles : geo.tiles;
        for (long long tile = t0; tile < t1; ++tile) {
          const long long row = tile * geo.R + rr;
          if (row >= N) continue;
          const size_t o = base + row * S;
          double bv[V], zv[V], zero[V];
          if (rhs) {
            ldgv<V>(rhs + o, bv);
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
      stash<2, V>(acc, red, kb, T, t);
    }
    batch_tree_partials<2, V>(red, partB, g, c0, nb, nk, geo);
  }
  if (!sync_group<CL>(cnt, gen, nb, abort_flag)) return;
  final_partials<2, V>(red, partB, g, geo);
  if (t == 0) s_flags[0] = 1;
  __syncthreads();
  if (t < L) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int s = V * t + j;
      const double bn = sqrt(red[j * T + t]);
      const double thr = tol * bn;
      ls.thr[s] = thr;
      ls.rz[s] = red[(V + j) * T + t];
      ls.conv[s] = bn <= thr;
      ls.frozen[s] = 0;
      ls.iters[s] = 0;
      if (blockIdx.x == 0 && st.hist) st.hist[(size_t)g * S + s] = bn;
      if (!(bn <= thr)) s_flags[0] = 0;
    }
  }
  __syncthreads();
  int it = 0;
  bool finish = s_flags[0] || maxit == 0;
  bool bad = false;

  while (!finish) {
    ++it;
    // ---- phase A: Ap = A p, partial p.Ap
    for (int c0 = blockIdx.x; c0 < C; c0 += kPersistBatch * nb) {
      const int nk = batch_count(c0, C, nb);
      for (int kb = 0; kb < nk; ++kb) {
        const int chunk = c0 + kb * nb;
        double acc[1][V] = {};
        if (sl < L) {
          const long long t0 = (long long)chunk * geo.chunk_tiles;
          const long long t1 = t0 + geo.chunk_tiles < geo.tiles ? t0 + geo.chunk_tiles : geo.tiles;
          for (long long tile = t0; tile < t1; ++tile) {
            const long long row = tile * geo.R + rr;
            if (row >= N) continue;
            double y[V], pv[V];
            if (fv.tx) {
              fv2d_row<V, true>(fv, N, S, g, V * sl, row, p + base, y, pv);
            } else {
              const int k0 = __ldg(&ro[row]), k1 = __ldg(&ro[row + 1]);
#pragma unroll
              for (int j = 0; j < V; ++j) y[j] = 0.0;
              for (int k = k0; k < k1; ++k) {
                double a[V], b[V];
                ldgv<V>(vg + (size_t)k * S, a);
                ldcgv<V>(p + base + (size_t)__ldg(&ci[k]) * S, b);
#pragma unroll
                for (int j = 0; j < V; ++j) y[j] = __dadd_rn(y[j], __dmul_rn(a[j], b[j]));
              }
              ldcgv<V>(p + base + row * S, pv);
            }
            stv<V>(ap + base + row * S, y);
#pragma unroll
            for (int j = 0; j < V; ++j) acc[0][j] = __fma_rn(pv[j], y[j], acc[0][j]);
          }
        }
        stash<1, V>(acc, red, kb, T, t);
      }
      batch_tree_partials<1, V>(red, partA, g, c0, nb, nk, geo);
    }
    if (!sync_group<CL>(cnt, gen, nb, abort_flag)) return;
    final_partials<1, V>(red, partA, g, geo);
    if (t < L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int s = V * t + j;
        const double pap = red[j * T + t];
        const unsigned char fr = ls.frozen[s] | (unsigned char)(pap <= DBL_MIN);
        ls.frozen[s] = fr;
        ls.alpha[s] = fr ? 0.0 : __ddiv_rn(ls.rz[s], pap);
      }
    }
    __syncthreads();
    // ---- phase B: r -= alpha Ap, partials r.r and r.z
    double alpha[V];
#pragma unroll
    for (int j = 0; j < V; ++j) alpha[j] = sl < L ? ls.alpha[V * sl + j] : 0.0;
    for (int c0 = blockIdx.x; c0 < C; c0 += kPersistBatch * nb) {
      const int nk = batch_count(c0, C, nb);
      for (int kb = 0; kb < nk; ++kb) {
        const int chunk = c0 + kb * nb;
        double acc[2][V] = {};
        if (sl < L) {
          const long long t0 = (long long)chunk * geo.chunk_tiles;
          const long long t1 = t0 + geo.chunk_tiles < geo.tiles ? t0 + geo.chunk_tiles : geo.tiles;
          for (long long tile = t0; tile < t1; ++tile) {
            const long long row = tile * geo.R + rr;
            if (row >= N) continue;
            const size_t o = base + row * S;
            double rv[V], av[V], zv[V];
            ldcgv<V>(r + o, rv);
            ldcgv<V>(ap + o, av);
#pragma unroll
            for (int j = 0; j < V; ++j) rv[j] = __dsub_rn(rv[j], __dmul_rn(alpha[j], av[j]));
            stv<V>(r + o, rv);
            if (dinv) {
              double dv[V];
              ldgv<V>(dinv + o, dv);
#pragma unroll
              for (int j = 0; j < V; ++j) zv[j] = __dmul_rn(rv[j], dv[j]);
            } else {
#pragma unroll
              for (int j = 0; j < V; ++j) zv[j] = rv[j];
            }
#pragma unroll
            for (int j = 0; j < V; ++j) {
              acc[0][j] = __fma_rn(rv[j], rv[j], acc[0][j]);
              acc[1][j] = __fma_rn(rv[j], zv[j], acc[1][j]);
            }
          }
        }
        stash<2, V>(acc, red, kb, T, t);
      }
      batch_tree_partials<2, V>(red, partB, g, c0, nb, nk, geo);
    }
    if (!sync_group<CL>(cnt, gen, nb, abort_flag)) return;
    final_partials<2, V>(red, partB, g, geo);
    if (t == 0) {
      s_flags[0] = 1;
      s_flags[1] = 0;
    }
    __syncthreads();
    if (t < L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int s = V * t + j;
        const double rn = sqrt(red[j * T + t]);
        const double rz_new = red[(V + j) * T + t];
        if (blockIdx.x == 0 && st.hist) {
          if (it <= st.hist_cap) st.hist[((size_t)it * st.G + g) * S + s] = rn;
          else atomicOr(st.overflow, 1);
        }
        const bool live = !ls.frozen[s];
        if (live && !isfinite(rn)) atomicOr(&s_flags[1], 1);
        if (live && !ls.conv[s] && rn <= ls.thr[s]) {
          ls.iters[s] = it;
          ls.conv[s] = 1;
        }
        if (live && !ls.conv[s]) atomicAnd(&s_flags[0], 0);
        const double rz_old = ls.rz[s];
        ls.beta[s] = (live && rz_old > 0.0) ? __ddiv_rn(rz_new, rz_old) : 0.0;
        ls.rz[s] = rz_new;
      }
    }
    __syncthreads();
    bad = s_flags[1] != 0;
    finish = bad || s_flags[0] || it >= maxit;
    // ---- phase C: x += alpha p ; p = z + beta p (skipped on the last iteration)
    double beta[V];
#pragma unroll
    for (int j = 0; j < V; ++j) beta[j] = sl < L ? ls.beta[V * sl + j] : 0.0;
    for (int chunk = blockIdx.x; chunk < C; chunk += nb) {
      if (sl >= L) continue;
      const long long t0 = (long long)chunk * geo.chunk_tiles;
      const long long t1 = t0 + geo.chunk_tiles < geo.tiles ? t0 + geo.chunk_tiles : geo.tiles;
      for (long long tile = t0; tile < t1; ++tile) {
        const long long row = tile * geo.R + rr;
        if (row >= N) continue;
        const size_t o = base + row * S;
        double xv[V], pv[V];
        ldcgv<V>(x + o, xv);
        ldcgv<V>(p + o, pv);
#pragma unroll
        for (int j = 0; j < V; ++j) xv[j] = __dadd_rn(xv[j], __dmul_rn(alpha[j], pv[j]));
        stv<V>(x + o, xv);
        if (!finish) {
          double rv[V], zv[V];
          ldcgv<V>(r + o, rv);
          if (dinv) {
            double dv[V];
            ldgv<V>(dinv + o, dv);
#pragma unroll
            for (int j = 0; j < V; ++j) zv[j] = __dmul_rn(rv[j], dv[j]);
          } else {
#pragma unroll
            for (int j = 0; j < V; ++j) zv[j] = rv[j];
          }
#pragma unroll
          for (int j = 0; j < V; ++j) pv[j] = __dadd_rn(zv[j], __dmul_rn(beta[j], pv[j]));
          stv<V>(p + o, pv);
        }
      }
    }
    if (!finish && !sync_group<CL>(cnt, gen, nb, abort_flag)) return;
  }
  // ---- outputs (block 0 of the group)
  if (blockIdx.x == 0) {
    if (t < L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int s = V * t + j;
        const size_t l = (size_t)g * S + s;
        st.iters[l] = ls.conv[s] ? ls.iters[s] : it;  // unconverged / frozen: iterations run
        st.conv[l] = ls.conv[s];
        st.frozen[l] = ls.frozen[s];
        st.alpha[l] = ls.alpha[s];
      }
    }
    if (t == 0) {
      st.it[g] = it;
      st.status[g] = bad ? 2 : 0;
      st.done[g] = kDone;
      atomicAdd(st.ndone, 1);
    }
  }
}

// Lets every persistent instantiation take `smem` bytes of dynamic shared
// memory (above the 48 KB default at large S); called before the occupancy
// queries and the launch.
static void allow_smem(size_t smem) {
  static size_t configured = 48 * 1024;
  if (smem <= configured) return;
  const void* fns[] = {(const void*)pcg_persistent_kernel<2, false>,
                       (const void*)pcg_persistent_kernel<1, false>,
                       (const void*)pcg_persistent_kernel<2, true>,
                       (const void*)pcg_persistent_kernel<1, true>};
  for (const void* f : fns)
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  configured = smem;
}

size_t persistent_smem(const Geo& geo) {
  return (size_t)kPersistBatch * 2 * geo.V * geo.T * sizeof(double) +
         (size_t)4 * geo.S * sizeof(double) +
         (size_t)geo.S * (sizeof(int) + 2) + 16;
}

template <bool CL>
static const void* persistent_fn(int V) {
  return V == 2 ? (const void*)pcg_persistent_kernel<2, CL> : (const void*)pcg_persistent_kernel<1, CL>;
}

// Cluster size (CTAs per group) for the cluster-barrier variant: up to 16
// (non-portable) and at most the group's chunk count; 0 if not launchable.
int persistent_cluster_size(const Geo& geo) {
  static int cached[2] = {-1, -1};
  static size_t cached_smem[2] = {0, 0};
  const int vi = geo.V == 2;
  const size_t smem = persistent_smem(geo);
  if (cached[vi] < 0 || cached_smem[vi] != smem) {  // per (V, shared-memory size)
    const void* fn = persistent_fn<true>(geo.V);
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, 1, 1);
    cfg.blockDim = dim3(geo.T, 1, 1);
    cfg.dynamicSmemBytes = smem;
    allow_smem(smem);
    cached_smem[vi] = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 16;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int cs = 0;
    if (cudaOccupancyMaxPotentialClusterSize(&cs, fn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      cs = 8;
    }
    cached[vi] = cs;
  }
  int c = cached[vi];
  if (c > 16) c = 16;
  if (c > geo.chunks) c = geo.chunks;
  return c;
}

// Blocks per group for a cooperative launch over G groups, or 0 if the
// groups cannot all be co-resident.
int persistent_blocks(const Geo& geo, int G) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = persistent_smem(geo);
  allow_smem(smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, persistent_fn<false>(geo.V), geo.T, smem);
  const long long cap = (long long)per_sm * sms;
  long long b = cap / (G < 1 ? 1 : G);
  if (b > geo.chunks) b = geo.chunks;
  return b < 1 ? 0 : (int)b;
}

cudaError_t launch_pcg_persistent(const Geo& geo, int G, int blocks, bool cluster, cudaStream_t s,
                                  long long N, long long nnz, const PcgState& st, const int* ro,
                                  const int* ci, const double* vals, const Fv2dOp& fv,
                                  const double* rhs,
                                  double rhs_const, const double* dinv, double tol, int maxit,
                                  double* x, double* r, double* p, double* ap, double* partA,
                                  double* partB, unsigned* bar_count, unsigned* bar_gen,
                                  int* abort_flag) {
  Geo gl = geo;
  gl.B = blocks;
  Fv2dOp op = fv;
  void* args[] = {&N,   &nnz,       &gl,   (void*)&st, &ro,    &ci,    &vals,  &op,
                  &rhs, &rhs_const, &dinv, &tol,       &maxit, &x,     &r,
                  &p,   &ap,        &partA, &partB,    &bar_count, &bar_gen, &abort_flag};
  const size_t smem = persistent_smem(gl);
  allow_smem(smem);
  if (!cluster)
    return cudaLaunchCooperativeKernel(persistent_fn<false>(gl.V), dim3(blocks, G), dim3(gl.T),
                                       args, smem, s);
  // one thread-block cluster per group: hardware cluster barriers
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks, G, 1);
  cfg.blockDim = dim3(gl.T, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = blocks;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, persistent_fn<true>(gl.V), args);
}

}  // namespace uqg
