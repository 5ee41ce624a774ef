// uqg_common.cuh - shared geometry, error state, vector access and the
// deterministic per-lane reduction used by every kernel of libuqg.so.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>

namespace uqg {

// ---------------------------------------------------------------------------
// error reporting (thread-local last error, see uqg_last_error())

void set_error(const std::string& msg);

#define UQG_TRY_CUDA(expr)                                                        \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::uqg::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));       \
      return UQG_ECUDA;                                                           \
    }                                                                             \
  } while (0)

#define UQG_CHECK_LAUNCH()                                                        \
  do {                                                                            \
    cudaError_t _e = cudaGetLastError();                                          \
    if (_e != cudaSuccess) {                                                      \
      ::uqg::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e));  \
      return UQG_ECUDA;                                                           \
    }                                                                             \
  } while (0)

#define UQG_REQUIRE(cond, msg)        \
  do {                                \
    if (!(cond)) {                    \
      ::uqg::set_error(msg);          \
      return UQG_EINVAL;              \
    }                                 \
  } while (0)

// ---------------------------------------------------------------------------
// Launch geometry for lane-interleaved ensemble data.
//
// Each thread owns V consecutive lanes (V = 2 when S is even: one 16-byte
// load per access, else V = 1) of one row; L = S / V threads cover a row,
// rounded up to the power of two Lp so the per-lane reduction tree is a clean
// binary tree.  A block of T threads covers a "tile" of R = T / Lp rows.
//
// Reductions are organised by CHUNKS of consecutive tiles: every chunk yields
// one per-lane partial (fixed in-block tree), and the partials of a group are
// summed in chunk order.  V, Lp, R, the chunk size and the chunk count depend
// only on (N, S) - never on the number of groups, blocks or GPUs - so every
// lane's reduction tree, and hence every result bit, is independent of how
// groups are batched or sharded (hard part 2).  The number of
// blocks per group (each grid-strides over chunks) is then free to be sized
// for occupancy at launch time.
constexpr int kMaxChunks = 512;        // partials per group and reduction
constexpr int kTargetBlocks = 2368;    // ~2 waves of 148 SMs x 8 resident CTAs
constexpr int kMaxLanes = 512;         // S <= 512 keeps Lp <= 256 = block size
constexpr int kMaxBatch = 8;           // chunks per batched reduction (reduce_lanes_batch)

struct Geo {
  int S;          // lanes per group
  int V;          // lanes per thread (1 or 2)
  int L;          // threads per row = S / V
  int Lp;         // L rounded up to a power of two
  int T;          // threads per block
  int R;          // rows per tile
  long long tiles;
  long long chunk_tiles;  // tiles per reduction chunk
  int chunks;     // reduction chunks per group (<= kMaxChunks)
  int B;          // blocks per group in the launch (set by with_groups)
  int gact;       // groups still running (with_groups), for occupancy-aware sizing
  int maxrow;     // longest graph row if known (0 = unknown): picks the unrolled SpMV
  int sc;         // chunks per super-chunk (1 = no super level: chunks <= kMaxChunks)
  int nsc;        // super-chunks (sc > 1)
  int pstride;    // partial rows per group: chunks (+ nsc super-partials when sc > 1)
  int tstride;    // tickets per group: 1 (+ nsc super-chunk tickets when sc > 1)
};

inline Geo make_geo(long long N, int S, int maxrow = 0) {
  Geo g;
  g.S = S;
  g.maxrow = maxrow;
  g.V = S % 2 == 0 ? 2 : 1;
  g.L = S / g.V;
  g.Lp = 1;
  while (g.Lp < g.L) g.Lp <<= 1;
  g.T = g.Lp > 256 ? g.Lp : 256;
  g.R = g.T / g.Lp;
  g.tiles = (N + g.R - 1) / g.R;
  if (g.tiles < 1) g.tiles = 1;
  // Aim for >= 64 chunks of <= 8 tiles; groups with more tiles get longer
  // chunks (at most kMaxChunks of them), but a chunk never spans more rows than
  // ~sqrt(N) - the neighbour band of a 2D stencil - once that needs more than
  // kMaxChunks chunks: a block sweeps its chunks' tiles in order, and a chunk
  // longer than the band makes its own +m neighbours wait a whole band before
  // reuse, so at large N the concurrently swept bands no longer fit in L2.
  // Then consecutive chunks form super-chunks whose partials are summed (in
  // chunk order) by the block completing the super-chunk, and the final stage
  // sums the <= kMaxChunks super-partials.
  constexpr int ct_max = 8;
  long long ct = g.tiles / 64;
  ct = ct < 1 ? 1 : (ct > ct_max ? ct_max : ct);
  if ((g.tiles + ct - 1) / ct > kMaxChunks) {
    long long band = (long long)sqrt((double)N);  // floor(sqrt(N))
    while (band * band > N) --band;
    while ((band + 1) * (band + 1) <= N) ++band;
    long long ct_band = band / g.R;
    if (ct_band < ct) ct_band = ct;
    ct = (g.tiles + kMaxChunks - 1) / kMaxChunks;
    // within 10% of the band: keep the single-level reduction (C3), else cap
    // chunks at the band and add the super-chunk level (C4, C5: measured
    // 1.0-band chunks 4.6 / 4.8 TB/s vs 4.0 / 3.9 at 1.1 bands)
    if (ct * 10 > ct_band * 11) ct = ct_band;
  }
  g.chunk_tiles = ct;
  g.chunks = (int)((g.tiles + ct - 1) / ct);
  if (g.chunks > kMaxChunks) {
    g.sc = (g.chunks + kMaxChunks - 1) / kMaxChunks;
    g.nsc = (g.chunks + g.sc - 1) / g.sc;
    g.pstride = g.chunks + g.nsc;
    g.tstride = 1 + g.nsc;
  } else {
    g.sc = 1;
    g.nsc = g.chunks;
    g.pstride = g.chunks;
    g.tstride = 1;
  }
  g.B = g.chunks;
  g.gact = 1;
  return g;
}

// Blocks per group for a launch over G groups: fill ~2 waves of the GPU.
inline Geo with_groups(Geo g, int G) {
  long long b = (kTargetBlocks + G - 1) / (G < 1 ? 1 : G);
  if (b > g.chunks) b = g.chunks;
  g.B = b < 1 ? 1 : (int)b;
  g.gact = G < 1 ? 1 : G;
  return g;
}

// Blocks per group for G running groups of `chunks` chunks when `slots` CTAs
// of the kernel fit on the GPU at once: the grid-stride blocks all run about
// equally long, so the launch takes ceil(G*B / slots) "waves"; pick the B with
// the least idle tail (G*B / (waves*slots) largest; fewer waves on near-ties).
// Results do not depend on B (reductions follow the chunks).
inline int pick_blocks(int G, int chunks, int slots) {
  if (G < 1) G = 1;
  if (slots < 1) slots = 1;
  int best = 1;
  double best_score = -1.0;
  for (int b = 1; b <= chunks; ++b) {
    const long long blocks = (long long)G * b;
    const long long waves = (blocks + slots - 1) / slots;
    const double eff = (double)blocks / ((double)waves * slots);
    const double score = eff - 0.004 * (double)waves;
    if (score > best_score) {
      best_score = score;
      best = b;
    }
    if (waves > 64) break;
  }
  return best;
}

// Resident CTAs of `fn` on the whole GPU (cached per shared-memory size).
struct SlotCache {
  size_t smem = (size_t)-1;
  int slots = 0;
};
template <class F>
inline int kernel_slots(SlotCache& c, F fn, int T, size_t smem) {
  if (c.smem != smem) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, T, smem) != cudaSuccess) {
      cudaGetLastError();
      per = 1;
    }
    c.slots = (per < 1 ? 1 : per) * (sms < 1 ? 1 : sms);
    c.smem = smem;
  }
  return c.slots;
}

// ---------------------------------------------------------------------------
// V-lane vector access (16-byte loads/stores for V = 2).

// V = 4 (32-byte accesses, sm_100 LDG/STG.256) is used by the face SpMV only.
template <int V>
__device__ __forceinline__ void ldv(const double* p, double (&o)[V]) {
  if constexpr (V == 4) {
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
                 : "l"(p));
  } else if constexpr (V == 2) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    o[0] = t.x;
    o[1] = t.y;
  } else {
    o[0] = *p;
  }
}

// read-only path (matrix values, dinv): non-coherent cache
template <int V>
__device__ __forceinline__ void ldgv(const double* p, double (&o)[V]) {
  if constexpr (V == 4) {
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
        : "l"(p));
  } else if constexpr (V == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = t.x;
    o[1] = t.y;
  } else {
    o[0] = __ldg(p);
  }
}

// L2-only path (vectors written by other SMs inside the same launch)
template <int V>
__device__ __forceinline__ void ldcgv(const double* p, double (&o)[V]) {
  if constexpr (V == 4) {
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
                 : "l"(p));
  } else if constexpr (V == 2) {
    const double2 t = __ldcg(reinterpret_cast<const double2*>(p));
    o[0] = t.x;
    o[1] = t.y;
  } else {
    o[0] = __ldcg(p);
  }
}

template <int V>
__device__ __forceinline__ void stv(double* p, const double (&o)[V]) {
  if constexpr (V == 4) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(o[0]), "d"(o[1]),
                 "d"(o[2]), "d"(o[3])
                 : "memory");
  } else if constexpr (V == 2) {
    *reinterpret_cast<double2*>(p) = make_double2(o[0], o[1]);
  } else {
    *p = o[0];
  }
}

// ---------------------------------------------------------------------------
// Deterministic per-lane chunk reduction + "last chunk finishes" pattern.
//
// For one chunk, the block reduces NV x V per-thread values over the chunk's
// rows (fixed binary tree in shared memory), writes one partial per (group,
// chunk, value, lane), and takes a ticket.  The block that completes the last
// chunk of the group sums the chunk partials of each lane in a fixed order
// (strided sequential sums, then the same binary tree) and returns true with
// the total of value v, lane V*sl+j in red[(v*V + j)*T + sl].  With
// super-chunks (geo.sc > 1) the block completing a super-chunk first sums its
// chunk partials sequentially in chunk order into a super-partial, and the
// final stage runs over the super-partials.  No floating-point atomics: the
// result is a pure function of the inputs.
//
// Layout per group g: part rows [g*pstride + r][NV][S] (r < chunks: chunk
// partials, then super-partials); tickets [g*tstride]: group ticket, then one
// per super-chunk.

// NB = 0: the reducing threads are the whole block (__syncthreads); NB > 0: they
// are its first NB threads, synchronised by named barrier 1 (a kernel with
// extra warps that do not take part in reductions, e.g. a TMA producer warp).
template <int NB>
__device__ __forceinline__ void block_sync() {
  if constexpr (NB == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync 1, %0;" ::"n"(NB) : "memory");
  }
}

template <int NS, int NB = 0>
__device__ __forceinline__ void tree_rows(double* red, int T, int Lp, int R, int t) {
  for (int st = R >> 1; st > 0; st >>= 1) {
    if ((t / Lp) < st) {
#pragma unroll
      for (int v = 0; v < NS; ++v) red[v * T + t] += red[v * T + t + st * Lp];
    }
    block_sync<NB>();
  }
}

// Tickets of nk chunks (chunk0 + k*stride) whose partials are written and
// fenced (all threads call after a __syncthreads).  Returns true in the one
// block that completes the group, with the totals in red[].
template <int NV, int V, int NB = 0>
__device__ bool finish_chunks(double* red, double* part, unsigned int* ticket, int g, int chunk0,
                              int stride, int nk, const Geo& geo) {
  constexpr int NS = NV * V;
  const int t = threadIdx.x;
  const int T = geo.T, Lp = geo.Lp, R = geo.R, L = geo.L, S = geo.S, C = geo.chunks;
  unsigned int* gt = ticket + (size_t)g * geo.tstride;
  double* gp = part + (size_t)g * geo.pstride * NV * S;
  __shared__ int s_flag;
  int rows = C, row0 = 0;
  if (geo.sc == 1) {
    if (t == 0) {
      const unsigned int tk = atomicAdd(gt, (unsigned)nk);
      s_flag = (tk + (unsigned)nk == (unsigned)C);
    }
    block_sync<NB>();
    if (!s_flag) return false;
  } else {
    // one thread per chunk of the batch takes its super-chunk's ticket
    __shared__ int s_super[kMaxBatch];
    if (t < nk) {
      const int c = chunk0 + t * stride, si = c / geo.sc;
      const int c_lo = si * geo.sc, c_hi = c_lo + geo.sc < C ? c_lo + geo.sc : C;
      const unsigned int tk = atomicAdd(gt + 1 + si, 1u);
      s_super[t] = (tk + 1u == (unsigned)(c_hi - c_lo)) ? si : -1;
    }
    block_sync<NB>();
    // every super-chunk this batch completed: its partials summed in chunk order
    // (all completed super-chunks at once, the loads of one sum issued together)
    __threadfence();
    if (t < L) {
      for (int k = 0; k < nk; ++k) {
        const int si = s_super[k];
        if (si < 0) continue;
        const int c_lo = si * geo.sc, c_hi = c_lo + geo.sc < C ? c_lo + geo.sc : C;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int j = 0; j < V; ++j) {
            double a = 0.0;
            for (int c0 = c_lo; c0 < c_hi; c0 += 8) {
              double q[8];
#pragma unroll
              for (int u = 0; u < 8; ++u)
                q[u] = c0 + u < c_hi ? __ldcg(&gp[((size_t)(c0 + u) * NV + v) * S + V * t + j]) : 0.0;
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (c0 + u < c_hi) a += q[u];
            }
            gp[((size_t)(C + si) * NV + v) * S + V * t + j] = a;
          }
      }
    }
    __threadfence();
    block_sync<NB>();
    if (t == 0) {
      int fin = 0;
      for (int k = 0; k < nk; ++k) {
        const int si = s_super[k];
        if (si < 0) continue;
        gt[1 + si] = 0u;
        const unsigned int tk = atomicAdd(gt, 1u);
        if (tk + 1u == (unsigned)geo.nsc) fin = 1;
      }
      s_flag = fin;
    }
    block_sync<NB>();
    const bool last = s_flag;
    if (!last) return false;
    rows = geo.nsc;
    row0 = C;
  }
  __threadfence();
  const int sl = t % Lp, jr = t / Lp;
  double acc[NS];
#pragma unroll
  for (int v = 0; v < NS; ++v) acc[v] = 0.0;
  if (sl < L) {
#pragma unroll 4
    for (int cc = jr; cc < rows; cc += R) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int j = 0; j < V; ++j)
          acc[v * V + j] += __ldcg(&gp[((size_t)(row0 + cc) * NV + v) * S + V * sl + j]);
    }
  }
  block_sync<NB>();  // red[] may still hold the caller's tree values
#pragma unroll
  for (int v = 0; v < NS; ++v) red[v * T + t] = acc[v];
  block_sync<NB>();
  tree_rows<NS, NB>(red, T, Lp, R, t);
  if (t == 0) gt[0] = 0u;  // ready for the next reduction on this counter
  return true;
}

template <int NV, int V>
__device__ bool reduce_lanes(const double (&val)[NV][V], double* red, double* part,
                             unsigned int* ticket, int g, int chunk, const Geo& geo) {
  constexpr int NS = NV * V;
  const int t = threadIdx.x;
  const int T = geo.T, Lp = geo.Lp, R = geo.R, L = geo.L, S = geo.S;
  __syncthreads();  // red[] may still be read by the previous chunk's tree
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int j = 0; j < V; ++j) red[(v * V + j) * T + t] = val[v][j];
  __syncthreads();
  tree_rows<NS>(red, T, Lp, R, t);
  if (t < L) {
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int j = 0; j < V; ++j)
        part[(((size_t)g * geo.pstride + chunk) * NV + v) * S + V * t + j] =
            red[(v * V + j) * T + t];
  }
  __threadfence();
  __syncthreads();
  return finish_chunks<NV, V>(red, part, ticket, g, chunk, 1, 1, geo);
}

// reduce_lanes over a batch of nk chunks chunk0 + k*stride (k < nk) whose
// per-thread values the caller has stored in red[((k*NV + v)*V + j)*T + t]:
// one in-block tree for the whole batch (instead of one per chunk), then the
// chunks' tickets.  Every partial and the final sums are computed exactly as
// reduce_lanes<NV, V> computes them, so results are bit-identical (same result
// layout in red).  red must hold max(nk, 1) * NV * V * T doubles.
// The in-block half of reduce_lanes_batch: one tree pass over the rows for all
// nk chunks' values in red[((k*NV + v)*V + j)*T + t], then the chunk partials
// written to part (no fence, no ticket).
template <int NV, int V, int NB = 0>
__device__ void batch_tree_partials(double* red, double* part, int g, int chunk0, int stride,
                                    int nk, const Geo& geo) {
  constexpr int NS = NV * V;
  const int t = threadIdx.x;
  const int T = geo.T, Lp = geo.Lp, R = geo.R, L = geo.L, S = geo.S;
  const int ns = nk * NS;
  block_sync<NB>();
  for (int st = R >> 1; st > 0; st >>= 1) {
    if ((t / Lp) < st) {
      for (int v = 0; v < ns; ++v) red[v * T + t] += red[v * T + t + st * Lp];
    }
    block_sync<NB>();
  }
  if (t < L) {
    for (int k = 0; k < nk; ++k)
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int j = 0; j < V; ++j)
          part[(((size_t)g * geo.pstride + chunk0 + k * stride) * NV + v) * S + V * t + j] =
              red[((k * NV + v) * V + j) * T + t];
  }
}

template <int NV, int V, int NB = 0>
__device__ bool reduce_lanes_batch(double* red, double* part, unsigned int* ticket, int g,
                                   int chunk0, int stride, int nk, const Geo& geo) {
  batch_tree_partials<NV, V, NB>(red, part, g, chunk0, stride, nk, geo);
  __threadfence();
  block_sync<NB>();
  return finish_chunks<NV, V, NB>(red, part, ticket, g, chunk0, stride, nk, geo);
}

// "last block of the group" without values (for state transitions); uses the
// group ticket (slot 0 of the group's tickets).
__device__ __forceinline__ bool last_block(unsigned int* ticket, int g, int B, int tstride) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int* gt = ticket + (size_t)g * tstride;
    unsigned int tk = atomicAdd(gt, 1u);
    s_last = (tk == (unsigned)(B - 1));
    if (s_last) *gt = 0u;
  }
  __syncthreads();
  return s_last;
}

}  // namespace uqg
