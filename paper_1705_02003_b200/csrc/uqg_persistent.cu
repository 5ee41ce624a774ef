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

#include <cooperative_groups.h>

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

// ---------------------------------------------------------------------------
// Shared-memory-resident cluster PCG (face-form FV2D operator, small groups:
// the C1 oracle case).  A group is one thread-block cluster of NB CTAs and
// each CTA OWNS a contiguous run of reduction chunks: its rows of x, r, p (two
// buffers), Ap and dinv and the x-faces they touch live in its shared memory
// for the whole solve.  Cross-CTA traffic goes through distributed shared
// memory (DSMEM, ld.shared::cluster via map_shared_rank):
//   * chunk partials: each CTA keeps its chunks' partials; after the cluster
//     barrier every CTA sums all partials in the canonical order (same trees
//     as finish_chunks / final_partials), so every CTA holds the same lane
//     state without a broadcast;
//   * the SpMV's p halo (rows within m of the CTA's range): the direction
//     step forms p_{k+1} for the halo rows itself from the owner's r and p_k
//     (read over DSMEM; dinv's halo is a local copy), so the next SpMV needs
//     no barrier: two cluster barriers per iteration (after the SpMV partials
//     and after the update partials) instead of three.
// Hazards: p is double-buffered (a neighbour still reads p_k while p_{k+1} is
// written); r of iteration k+1 is written after barrier 1 of k+1, which every
// CTA reaches only after its halo reads of r_k; partial buffers are rewritten
// one barrier after their last remote read.
// Arithmetic and reduction order are those of the launch loop (x += alpha p
// moves into the update phase: the same values, so the same bits).

namespace cg = cooperative_groups;

struct SmemPlan {  // per-CTA shared-memory layout (doubles unless noted)
  int ncl;         // max chunks per CTA
  int nr;          // max rows per CTA
  int hm;          // halo rows on each side (min(m, N))
  size_t bytes;
};

__host__ __device__ inline SmemPlan smem_plan(const Geo& geo, int m, long long N, int nb) {
  SmemPlan sp;
  sp.ncl = (geo.chunks + nb - 1) / nb;
  sp.nr = (int)(sp.ncl * geo.chunk_tiles * geo.R);
  sp.hm = (int)(m < N ? m : N);
  const size_t S = geo.S;
  size_t d = 0;
  d += 6 * (size_t)sp.nr * S;             // x, r, p0, p1, ap, dinv
  d += (size_t)(sp.nr + m) * S;           // x-faces of the CTA's rows (w: row, e: row + m)
  d += 4 * (size_t)sp.hm * S;             // p halo (west, east) + dinv halo (west, east)
  d += 3 * (size_t)sp.ncl * S;            // partials: p.Ap, (r.r, r.z)
  d += (size_t)sp.ncl * 2 * geo.V * geo.T;  // batched in-block trees
  d += 4 * S;                             // alpha, beta, rz, thr
  sp.bytes = d * sizeof(double) + S * (sizeof(int) + 2) + 64;
  return sp;
}

__device__ __forceinline__ int chunk_lo(int C, int nb, int b) {
  return C * b / nb;  // C <= kMaxChunks, nb <= 16: no overflow
}
__device__ __forceinline__ int chunk_owner(int C, int nb, int c) {
  int b = c * nb / C;
  while (b + 1 < nb && chunk_lo(C, nb, b + 1) <= c) ++b;
  while (b > 0 && chunk_lo(C, nb, b) > c) --b;
  return b;
}

template <int V>
__global__ void __launch_bounds__(256, 1) pcg_cluster_smem_kernel(
    long long N_ll, Geo geo, PcgState st, Fv2dOp fv, const double* __restrict__ rhs,
    double rhs_const, const double* __restrict__ dinv_g, double tol, int maxit,
    double* __restrict__ x_g) {
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int N = (int)N_ll, m = fv.m;
  const int g = blockIdx.y, t = threadIdx.x, b = (int)cluster.block_rank();
  const int nb = (int)cluster.num_blocks();
  const int S = geo.S, T = geo.T, L = geo.L, Lp = geo.Lp, R = geo.R, C = geo.chunks;
  const int CR = (int)(geo.chunk_tiles * R);  // rows per chunk
  const int sl = t % Lp, rr = t / Lp;
  const SmemPlan sp = smem_plan(geo, m, N, nb);
  const int c0 = chunk_lo(C, nb, b), c1 = chunk_lo(C, nb, b + 1), ncl = c1 - c0;
  const int row0 = c0 * CR;
  int row1 = c1 * CR;
  if (row1 > N) row1 = N;
  const int hm = sp.hm;
  // layout (identical in every CTA, so DSMEM offsets are the owner's local ones)
  double* xs = sm;
  double* rs = xs + (size_t)sp.nr * S;
  double* pb[2] = {rs + (size_t)sp.nr * S, rs + 2 * (size_t)sp.nr * S};
  double* aps = pb[1] + (size_t)sp.nr * S;
  double* ds = aps + (size_t)sp.nr * S;
  double* txs = ds + (size_t)sp.nr * S;
  double* hw = txs + (size_t)(sp.nr + m) * S;   // p halo rows [row0 - hm, row0)
  double* he = hw + (size_t)hm * S;             // p halo rows [row1, row1 + hm)
  double* hdw = he + (size_t)hm * S;
  double* hde = hdw + (size_t)hm * S;
  double* pA = hde + (size_t)hm * S;            // [ncl][S]
  double* pB = pA + (size_t)sp.ncl * S;         // [ncl][2][S]
  double* red = pB + 2 * (size_t)sp.ncl * S;    // [ncl * 2 * V][T]
  double* la = red + (size_t)sp.ncl * 2 * V * T;
  double* lb = la + S;
  double* lrz = lb + S;
  double* lthr = lrz + S;
  int* lit = reinterpret_cast<int*>(lthr + S);
  unsigned char* lconv = reinterpret_cast<unsigned char*>(lit + S);
  unsigned char* lfr = lconv + S;
  __shared__ int s_flags[2];
  const size_t gb = (size_t)g * N * S;
  const size_t fo = (size_t)g * (N + m) * S;

  // ---- load the CTA's slice: dinv, x-faces, dinv halo; x = 0, r = b, p0 = z
  for (int e = t; e < (row1 - row0) * L; e += T) {
    const int q = row0 + e / L, l = V * (e % L);
    const size_t o = gb + (size_t)q * S + l, lo = (size_t)(q - row0) * S + l;
    double bv[V], dv[V], z[V], zero[V];
    if (rhs) {
      ldgv<V>(rhs + o, bv);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) bv[j] = rhs_const;
    }
    if (dinv_g) ldgv<V>(dinv_g + o, dv);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (!dinv_g) dv[j] = 1.0;
      z[j] = dinv_g ? __dmul_rn(bv[j], dv[j]) : bv[j];
      zero[j] = 0.0;
      xs[lo + j] = zero[j];
      rs[lo + j] = bv[j];
      ds[lo + j] = dv[j];
      pb[0][lo + j] = z[j];
    }
  }
  for (int e = t; e < (row1 - row0 + m) * L; e += T) {
    const int q = row0 + e / L, l = V * (e % L);
    double tv[V];
    ldgv<V>(fv.tx + fo + (size_t)q * S + l, tv);
#pragma unroll
    for (int j = 0; j < V; ++j) txs[(size_t)(q - row0) * S + l + j] = tv[j];
  }
  for (int e = t; e < 2 * hm * L; e += T) {
    const int h = e / L, l = V * (e % L);
    const int q = h < hm ? row0 - hm + h : row1 + (h - hm);
    double* dst = h < hm ? hdw + (size_t)h * S : hde + (size_t)(h - hm) * S;
#pragma unroll
    for (int j = 0; j < V; ++j)
      dst[l + j] = (q >= 0 && q < N) ? (dinv_g ? __ldg(dinv_g + gb + (size_t)q * S + l + j) : 1.0)
                                     : 0.0;
  }
  __syncthreads();

  // p of global row q from the current buffer (own rows or the local halo)
  auto p_at = [&](const double* pown, int q) -> const double* {
    if (q >= row0 && q < row1) return pown + (size_t)(q - row0) * S;
    if (q < row0) return hw + (size_t)(q - (row0 - hm)) * S;
    return he + (size_t)(q - row1) * S;
  };
  // halo p_{k+1} = r * dinv + beta * p_k from the owners' r and p_k (DSMEM);
  // init: beta = 0 and r = b gives p_0 = z.  A thread's halo items and their
  // owners' addresses are fixed for the solve: resolved once (kHaloItems per
  // thread cached, any further ones resolved per call).
  constexpr int kHaloItems = 2;
  const double* h_r[kHaloItems];
  const double* h_p[kHaloItems][2];
  auto halo_src = [&](int e, const double*& ro_, const double*& p0_, const double*& p1_) {
    const int h = e / L, l = V * (e % L);
    const int q = h < hm ? row0 - hm + h : row1 + (h - hm);
    if (q < 0 || q >= N) {
      ro_ = nullptr;
      return;
    }
    const int ob = chunk_owner(C, nb, q / CR);
    const size_t off = (size_t)(q - chunk_lo(C, nb, ob) * CR) * S + l;
    ro_ = cluster.map_shared_rank(rs, ob) + off;
    p0_ = cluster.map_shared_rank(pb[0], ob) + off;
    p1_ = cluster.map_shared_rank(pb[1], ob) + off;
  };
#pragma unroll
  for (int i = 0; i < kHaloItems; ++i) {
    h_r[i] = nullptr;
    const int e = t + i * T;
    if (e < 2 * hm * L) halo_src(e, h_r[i], h_p[i][0], h_p[i][1]);
  }
  auto form_item = [&](int e, const double* rr_o, const double* p0_, const double* p1_, int kb,
                       bool init) {
    {
      if (!rr_o) return;
      const int h = e / L, l = V * (e % L);
      const double* dh = (h < hm ? hdw + (size_t)h * S : hde + (size_t)(h - hm) * S) + l;
      double* dst = (h < hm ? hw + (size_t)h * S : he + (size_t)(h - hm) * S) + l;
      double rv[V];
#pragma unroll
      for (int j = 0; j < V; ++j) rv[j] = rr_o[j];
      if (init) {
#pragma unroll
        for (int j = 0; j < V; ++j) dst[j] = dinv_g ? __dmul_rn(rv[j], dh[j]) : rv[j];
      } else {
        const double* pk_o = kb ? p1_ : p0_;
        double pv[V];
#pragma unroll
        for (int j = 0; j < V; ++j) pv[j] = pk_o[j];
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const double z = dinv_g ? __dmul_rn(rv[j], dh[j]) : rv[j];
          dst[j] = __dadd_rn(z, __dmul_rn(lb[l + j], pv[j]));
        }
      }
    }
  };
  auto form_halo = [&](int kb, bool init) {
#pragma unroll
    for (int i = 0; i < kHaloItems; ++i)
      if (t + i * T < 2 * hm * L) form_item(t + i * T, h_r[i], h_p[i][0], h_p[i][1], kb, init);
    for (int e = t + kHaloItems * T; e < 2 * hm * L; e += T) {
      const double *rr_o, *p0_ = nullptr, *p1_ = nullptr;
      halo_src(e, rr_o, p0_, p1_);
      form_item(e, rr_o, p0_, p1_, kb, init);
    }
  };
  // canonical chunk partials of this CTA's chunks: per-thread values already
  // in red[((k*NV + v)*V + j)*T + t]; one tree pass for all chunks
  auto chunk_trees = [&](int NVv, double* part) {
    const int ns = ncl * NVv * V;
    __syncthreads();
    for (int s2 = R >> 1; s2 > 0; s2 >>= 1) {
      if ((t / Lp) < s2)
        for (int v = 0; v < ns; ++v) red[v * T + t] += red[v * T + t + s2 * Lp];
      __syncthreads();
    }
    if (t < L)
      for (int k = 0; k < ncl; ++k)
        for (int v = 0; v < NVv; ++v)
#pragma unroll
          for (int j = 0; j < V; ++j)
            part[((size_t)k * NVv + v) * S + V * t + j] = red[((k * NVv + v) * V + j) * T + t];
  };
  // all C partials in the canonical final order (finish_chunks' last stage):
  // totals of value v, lane V*sl+j in red[(v*V + j)*T + sl]
  auto final_sum = [&](int NVv, double* part) {
    double acc[2 * V];
#pragma unroll
    for (int v = 0; v < 2 * V; ++v) acc[v] = 0.0;
    if (sl < L) {
      for (int cc = rr; cc < C; cc += R) {
        const int ob = chunk_owner(C, nb, cc);
        const double* pr = cluster.map_shared_rank(part, ob) +
                           (size_t)(cc - chunk_lo(C, nb, ob)) * NVv * S;
        for (int v = 0; v < NVv; ++v)
#pragma unroll
          for (int j = 0; j < V; ++j) acc[v * V + j] += pr[(size_t)v * S + V * sl + j];
      }
    }
    __syncthreads();
    for (int v = 0; v < NVv * V; ++v) red[v * T + t] = acc[v];
    __syncthreads();
    for (int s2 = R >> 1; s2 > 0; s2 >>= 1) {
      if ((t / Lp) < s2)
        for (int v = 0; v < NVv * V; ++v) red[v * T + t] += red[v * T + t + s2 * Lp];
      __syncthreads();
    }
  };

  // ---- init partials b.b and r.z (r = b, z = p0)
  for (int k = 0; k < ncl; ++k) {
    double acc[2][V] = {};
    if (sl < L) {
      for (int q = (c0 + k) * CR + rr; q < (c0 + k + 1) * CR && q < N; q += R) {
        const size_t lo = (size_t)(q - row0) * S + V * sl;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          acc[0][j] = __fma_rn(rs[lo + j], rs[lo + j], acc[0][j]);
          acc[1][j] = __fma_rn(rs[lo + j], pb[0][lo + j], acc[1][j]);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int j = 0; j < V; ++j) red[((k * 2 + v) * V + j) * T + t] = acc[v][j];
  }
  chunk_trees(2, pB);
  cluster.sync();
  form_halo(0, true);
  final_sum(2, pB);
  if (t == 0) s_flags[0] = 1;
  __syncthreads();
  if (t < L) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int s = V * t + j;
      const double bn = sqrt(red[j * T + t]);
      const double thr = tol * bn;
      lthr[s] = thr;
      lrz[s] = red[(V + j) * T + t];
      lconv[s] = bn <= thr;
      lfr[s] = 0;
      lit[s] = 0;
      if (b == 0 && st.hist) st.hist[(size_t)g * S + s] = bn;
      if (!(bn <= thr)) s_flags[0] = 0;
    }
  }
  __syncthreads();
  int it = 0, kb = 0;  // kb: buffer of p_k
  bool finish = s_flags[0] || maxit == 0;
  bool bad = false;
  while (!finish) {
    ++it;
    // ---- phase A: Ap = A p_k (shared memory + halo), partial p.Ap
    const double* pk = pb[kb];
    for (int k = 0; k < ncl; ++k) {
      double acc[V] = {};
      if (sl < L) {
        for (int q = (c0 + k) * CR + rr; q < (c0 + k + 1) * CR && q < N; q += R) {
          const int i0 = q / m, j0 = q - i0 * m;
          const size_t lo = (size_t)(q - row0) * S + V * sl;
          const double* tw = txs + lo;
          const double* te = txs + lo + (size_t)m * S;
          const double ay = fv.a_y;
          const bool w = i0 > 0, s_ = j0 > 0, n_ = j0 < m - 1, e_ = i0 < m - 1;
          const double* pc = pk + lo;
          const double* pw = p_at(pk, q - m) + V * sl;
          const double* ps = p_at(pk, q - 1) + V * sl;
          const double* pn = p_at(pk, q + 1) + V * sl;
          const double* pe = p_at(pk, q + m) + V * sl;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const double d = __dadd_rn(__dadd_rn(__dadd_rn(tw[j], te[j]), ay), ay);
            double y = 0.0;
            if (w) y = __dadd_rn(y, __dmul_rn(-tw[j], pw[j]));
            if (s_) y = __dadd_rn(y, __dmul_rn(-ay, ps[j]));
            y = __dadd_rn(y, __dmul_rn(d, pc[j]));
            if (n_) y = __dadd_rn(y, __dmul_rn(-ay, pn[j]));
            if (e_) y = __dadd_rn(y, __dmul_rn(-te[j], pe[j]));
            aps[lo + j] = y;
            acc[j] = __fma_rn(pc[j], y, acc[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < V; ++j) red[(k * V + j) * T + t] = acc[j];
    }
    chunk_trees(1, pA);
    cluster.sync();  // barrier 1: p.Ap partials visible
    final_sum(1, pA);
    if (t < L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int s = V * t + j;
        const double pap = red[j * T + t];
        const unsigned char fr = lfr[s] | (unsigned char)(pap <= DBL_MIN);
        lfr[s] = fr;
        la[s] = fr ? 0.0 : __ddiv_rn(lrz[s], pap);
      }
    }
    __syncthreads();
    // ---- phase B: x += alpha p_k; r -= alpha Ap; partials r.r, r.z
    double alpha[V];
#pragma unroll
    for (int j = 0; j < V; ++j) alpha[j] = sl < L ? la[V * sl + j] : 0.0;
    for (int k = 0; k < ncl; ++k) {
      double acc[2][V] = {};
      if (sl < L) {
        for (int q = (c0 + k) * CR + rr; q < (c0 + k + 1) * CR && q < N; q += R) {
          const size_t lo = (size_t)(q - row0) * S + V * sl;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            xs[lo + j] = __dadd_rn(xs[lo + j], __dmul_rn(alpha[j], pk[lo + j]));
            const double rv = __dsub_rn(rs[lo + j], __dmul_rn(alpha[j], aps[lo + j]));
            rs[lo + j] = rv;
            const double zv = dinv_g ? __dmul_rn(rv, ds[lo + j]) : rv;
            acc[0][j] = __fma_rn(rv, rv, acc[0][j]);
            acc[1][j] = __fma_rn(rv, zv, acc[1][j]);
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int j = 0; j < V; ++j) red[((k * 2 + v) * V + j) * T + t] = acc[v][j];
    }
    chunk_trees(2, pB);
    cluster.sync();  // barrier 2: update partials (and every CTA's r) visible
    final_sum(2, pB);
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
        if (b == 0 && st.hist) {
          if (it <= st.hist_cap) st.hist[((size_t)it * st.G + g) * S + s] = rn;
          else atomicOr(st.overflow, 1);
        }
        const bool live = !lfr[s];
        if (live && !isfinite(rn)) atomicOr(&s_flags[1], 1);
        if (live && !lconv[s] && rn <= lthr[s]) {
          lit[s] = it;
          lconv[s] = 1;
        }
        if (live && !lconv[s]) atomicAnd(&s_flags[0], 0);
        const double rz_old = lrz[s];
        lb[s] = (live && rz_old > 0.0) ? __ddiv_rn(rz_new, rz_old) : 0.0;
        lrz[s] = rz_new;
      }
    }
    __syncthreads();
    bad = s_flags[1] != 0;
    finish = bad || s_flags[0] || it >= maxit;
    if (finish) break;
    // ---- phase C: p_{k+1} = z + beta p_k into the other buffer, own rows + halo
    double* pn = pb[kb ^ 1];
    for (int e = t; e < (row1 - row0) * L; e += T) {
      const size_t lo = (size_t)(e / L) * S + V * (e % L);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const double zv = dinv_g ? __dmul_rn(rs[lo + j], ds[lo + j]) : rs[lo + j];
        pn[lo + j] = __dadd_rn(zv, __dmul_rn(lb[V * (e % L) + j], pk[lo + j]));
      }
    }
    form_halo(kb, false);
    kb ^= 1;
    __syncthreads();
  }
  // ---- outputs: x rows, lane results (CTA 0 of the group)
  for (int e = t; e < (row1 - row0) * L; e += T) {
    const int q = row0 + e / L, l = V * (e % L);
    double xv[V];
#pragma unroll
    for (int j = 0; j < V; ++j) xv[j] = xs[(size_t)(q - row0) * S + l + j];
    stv<V>(x_g + gb + (size_t)q * S + l, xv);
  }
  if (b == 0) {
    if (t < L) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int s = V * t + j;
        const size_t l = (size_t)g * S + s;
        st.iters[l] = lconv[s] ? lit[s] : it;
        st.conv[l] = lconv[s];
        st.frozen[l] = lfr[s];
        st.alpha[l] = la[s];
      }
    }
    if (t == 0) {
      st.it[g] = it;
      st.status[g] = bad ? 2 : 0;
      st.done[g] = kDone;
      atomicAdd(st.ndone, 1);
    }
  }
  cluster.sync();  // no CTA leaves while another may still read its shared memory
}

// Cluster size and shared-memory bytes for the smem-resident kernel, or 0
// when the group does not fit (face form with constant y-faces only).
int cluster_smem_size(const Geo& geo, long long N, int m, size_t* smem_out) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (geo.sc != 1 || geo.T > 256) return 0;
  for (int nb = geo.chunks < 16 ? geo.chunks : 16; nb >= 1; --nb) {
    // every CTA must own at least one chunk and the smem plan must fit
    const SmemPlan sp = smem_plan(geo, m, N, nb);
    if ((long long)sp.bytes > optin) {
      if (nb == (geo.chunks < 16 ? geo.chunks : 16)) continue;
      return 0;  // fewer CTAs only makes each slice bigger
    }
    const void* fn = geo.V == 2 ? (const void*)pcg_cluster_smem_kernel<2>
                                : (const void*)pcg_cluster_smem_kernel<1>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.bytes);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb, 1, 1);
    cfg.blockDim = dim3(geo.T, 1, 1);
    cfg.dynamicSmemBytes = sp.bytes;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = nb;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (nclusters >= 1) {
      if (smem_out) *smem_out = sp.bytes;
      return nb;
    }
  }
  return 0;
}

cudaError_t launch_pcg_cluster_smem(const Geo& geo, int G, int nb, size_t smem, cudaStream_t s,
                                    long long N, const PcgState& st, const Fv2dOp& fv,
                                    const double* rhs, double rhs_const, const double* dinv,
                                    double tol, int maxit, double* x) {
  Geo gl = geo;
  gl.B = nb;
  Fv2dOp op = fv;
  PcgState sc = st;
  void* args[] = {&N, &gl, &sc, &op, (void*)&rhs, &rhs_const, (void*)&dinv, &tol, &maxit, &x};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb, G, 1);
  cfg.blockDim = dim3(gl.T, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = nb;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  const void* fn = gl.V == 2 ? (const void*)pcg_cluster_smem_kernel<2>
                             : (const void*)pcg_cluster_smem_kernel<1>;
  return cudaLaunchKernelExC(&cfg, fn, args);
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
