// uqg_common.cuh - shared geometry, error state and the deterministic
// per-lane reduction used by every kernel of libuqg.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
// A block of T threads covers a "tile" of R = T / Sp consecutive rows; thread t
// owns lane s = t % Sp of row tile*R + t / Sp (lanes >= S idle).  Sp is S
// rounded up to a power of two so the per-lane reduction tree is a clean
// binary tree.  Each group gets B blocks that grid-stride over its tiles.
// B depends only on (N, S) - never on the number of groups or GPUs - so every
// lane's reduction tree, and hence every result bit, is independent of how
// groups are batched or sharded (hard part 2).
constexpr int kMaxBlocksPerGroup = 1184;  // 148 SMs x 8 resident 256-thread CTAs

struct Geo {
  int S;          // lanes per group
  int Sp;         // S rounded up to a power of two
  int T;          // threads per block
  int R;          // rows per tile
  long long tiles;
  int B;          // blocks per group
};

inline Geo make_geo(long long N, int S) {
  Geo g;
  g.S = S;
  g.Sp = 1;
  while (g.Sp < S) g.Sp <<= 1;
  g.T = g.Sp > 256 ? g.Sp : 256;
  g.R = g.T / g.Sp;
  g.tiles = (N + g.R - 1) / g.R;
  long long b = g.tiles < kMaxBlocksPerGroup ? g.tiles : kMaxBlocksPerGroup;
  g.B = b < 1 ? 1 : (int)b;
  return g;
}

// ---------------------------------------------------------------------------
// Deterministic per-lane block reduction + "last block finishes" pattern.
//
// Every block reduces NV per-thread values over its rows (fixed binary tree in
// shared memory), writes one partial per (group, block, value, lane), and takes
// a ticket.  The block that draws the last ticket sums the B partials of each
// lane in a fixed order (strided sequential sums, then the same binary tree)
// and returns true with the totals in red[v*T + s].  No floating-point atomics:
// the result is a pure function of the inputs.

template <int NV>
__device__ __forceinline__ void tree_rows(double* red, int T, int Sp, int R, int t) {
  for (int st = R >> 1; st > 0; st >>= 1) {
    if ((t / Sp) < st) {
#pragma unroll
      for (int v = 0; v < NV; ++v) red[v * T + t] += red[v * T + t + st * Sp];
    }
    __syncthreads();
  }
}

template <int NV>
__device__ bool reduce_lanes(const double (&val)[NV], double* red, double* part,
                             unsigned int* ticket, int g, const Geo& geo) {
  const int t = threadIdx.x;
  const int T = geo.T, Sp = geo.Sp, R = geo.R, S = geo.S, B = geo.B;
  const int b = blockIdx.x;
#pragma unroll
  for (int v = 0; v < NV; ++v) red[v * T + t] = val[v];
  __syncthreads();
  tree_rows<NV>(red, T, Sp, R, t);
  if (t < S) {
#pragma unroll
    for (int v = 0; v < NV; ++v)
      part[(((size_t)g * B + b) * NV + v) * S + t] = red[v * T + t];
  }
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (t == 0) {
    unsigned int tk = atomicAdd(&ticket[g], 1u);
    s_last = (tk == (unsigned)(B - 1));
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  const int s = t % Sp, j = t / Sp;
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  if (s < S) {
    for (int bb = j; bb < B; bb += R) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
        acc[v] += __ldcg(&part[(((size_t)g * B + bb) * NV + v) * S + s]);
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) red[v * T + t] = acc[v];
  __syncthreads();
  tree_rows<NV>(red, T, Sp, R, t);
  if (t == 0) ticket[g] = 0u;  // ready for the next reduction on this counter
  return true;
}

}  // namespace uqg
