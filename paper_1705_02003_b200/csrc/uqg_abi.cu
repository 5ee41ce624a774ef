// uqg_abi.cu - the C ABI of libuqg.so (include/uqg.h): argument validation,
// context / workspace management, launch accounting and the host side of the
// device-resident PCG loop.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/uqg.h"
#include "uqg_common.cuh"
#include "uqg_kernels.cuh"

namespace uqg {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace uqg

using namespace uqg;

struct uqg_ctx {
  int device = 0;
  int* status_dev = nullptr;       // sticky device status word
  int* pinned = nullptr;           // [4] pinned host scratch
  cudaEvent_t ev = nullptr;
  void* ws = nullptr;              // workspace (library-owned, grow-only)
  size_t ws_bytes = 0;
  void* ext = nullptr;             // caller-provided workspace (uqg_ctx_set_workspace)
  size_t ext_bytes = 0;
  // launch accounting / optional per-launch event timing (uqg_ctx_profile*)
  long long launches = 0;
  long long kind_launches[UQG_NKERN] = {};
  double kind_ms[UQG_NKERN] = {};
  bool prof = false;
  std::vector<cudaEvent_t> evpool;  // start/stop pairs
  std::vector<int> pend_kind;
  int pend = 0;
  BandHint bands{};                 // uqg_ctx_set_band_hint (nb = 0: none)
  // concurrent PCG parts (pcg_impl): extra non-blocking streams, their events,
  // pinned done-counter readbacks
  std::vector<cudaStream_t> aux;
  std::vector<cudaEvent_t> aux_ev;
  int* pinned_parts = nullptr;
  // graph launch loop (pcg_impl): capture stream, device pass counter, pinned readback
  cudaStream_t cap = nullptr;
  int* loops_dev = nullptr;
  int* loops_host = nullptr;
};

namespace {

// Timing events are harvested lazily (end of a solve, profile_read, or a full
// pool), so profiling adds two event records per launch and no host syncs.
constexpr int kEventPairs = 16384;

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int grid_for(long long total, int threads) {
  long long b = (total + threads - 1) / threads;
  long long cap = 148LL * 16;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

// Accumulate the elapsed times of all recorded (start, stop) pairs.
int harvest(uqg_ctx* ctx) {
  if (!ctx->pend) return UQG_OK;
  for (int i = 0; i < ctx->pend; ++i) {  // launches may sit on several streams
    float ms = 0.f;
    UQG_TRY_CUDA(cudaEventSynchronize(ctx->evpool[2 * i + 1]));
    UQG_TRY_CUDA(cudaEventElapsedTime(&ms, ctx->evpool[2 * i], ctx->evpool[2 * i + 1]));
    ctx->kind_ms[ctx->pend_kind[i]] += ms;
  }
  ctx->pend = 0;
  return UQG_OK;
}

// Every kernel launch of the library goes through here: it counts launches
// per kernel class and, when profiling is on, brackets the launch with CUDA
// events on the launching stream.
template <class F>
int launch(uqg_ctx* ctx, int kind, cudaStream_t s, F&& fn) {
  ctx->launches++;
  ctx->kind_launches[kind]++;
  if (ctx->prof) {
    if (ctx->pend == kEventPairs) {
      int rc = harvest(ctx);
      if (rc) return rc;
    }
    UQG_TRY_CUDA(cudaEventRecord(ctx->evpool[2 * ctx->pend], s));
    fn();
    UQG_TRY_CUDA(cudaEventRecord(ctx->evpool[2 * ctx->pend + 1], s));
    ctx->pend_kind[ctx->pend++] = kind;
  } else {
    fn();
  }
  UQG_CHECK_LAUNCH();
  return UQG_OK;
}

#define UQG_LAUNCH(kind, stream, ...)                                    \
  do {                                                                   \
    int _rc = launch(ctx, (kind), (stream), [&] { __VA_ARGS__; });       \
    if (_rc) return _rc;                                                 \
  } while (0)

// Workspace: the caller's buffer when it is large enough, else a grow-only
// library allocation.  ws_base() returns whichever ensure_ws selected.
void* ws_base(uqg_ctx* ctx, size_t bytes) {
  return (ctx->ext && bytes <= ctx->ext_bytes) ? ctx->ext : ctx->ws;
}

int ensure_ws(uqg_ctx* ctx, size_t bytes) {
  if (ctx->ext && bytes <= ctx->ext_bytes) return UQG_OK;
  if (bytes <= ctx->ws_bytes) return UQG_OK;
  if (ctx->ws) {
    cudaDeviceSynchronize();
    cudaFree(ctx->ws);
    ctx->ws = nullptr;
    ctx->ws_bytes = 0;
  }
  cudaError_t e = cudaMalloc(&ctx->ws, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("workspace allocation of " + std::to_string(bytes) + " bytes failed: " +
              cudaGetErrorString(e));
    return UQG_ENOMEM;
  }
  ctx->ws_bytes = bytes;
  return UQG_OK;
}

struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return p;
  }
};

struct PersistBufs {
  double* partA;
  unsigned* bar;  // [G] counts, [G] generations, [1] abort flag
};
thread_local PersistBufs g_persist;

// UQG_PCG_PERSISTENT: 2 = cluster kernel, 1 = cooperative kernel (when
// co-resident), 0 = never, unset = auto
// (small batches: the launch-per-phase loop would be latency-bound).
int persistent_mode() {
  static const int m = [] {
    const char* e = getenv("UQG_PCG_PERSISTENT");
    return e ? atoi(e) : -1;
  }();
  return m;
}

// UQG_X_DEFER: iterations per deferred solution update in the launch loop
// (PcgState::kx; 1 = x updated every iteration).  Results are identical for
// every value; the workspace grows by kx - 1 vectors per group.
int x_defer() {
  static const int k = [] {
    const char* e = getenv("UQG_X_DEFER");
    const int v = e ? atoi(e) : 8;
    return v < 1 ? 1 : (v > kMaxKx ? kMaxKx : v);
  }();
  return k;
}

// UQG_SOLVE_STREAMS: the launch loop splits the groups into this many parts
// solved concurrently on separate streams (default 2) when every part still
// moves >= 1 GB per iteration; kernels of two parts then share the SMs and
// fill each other's latency gaps (C2: 1,572 -> 1,496 ms per level).  Results
// do not depend on it (groups are independent).
constexpr int kMaxParts = 4;
int solve_streams() {  // read per solve: bench.py times kernels with one stream
  const char* e = getenv("UQG_SOLVE_STREAMS");
  const int v = e ? atoi(e) : 2;
  return v < 1 ? 1 : (v > kMaxParts ? kMaxParts : v);
}

// UQG_PCG_GRAPH: run the launch loop of a single-part solve as ONE CUDA graph
// launch - a while-conditional node repeating kx iterations, the condition
// cleared on the device once every group is DONE - instead of host-polled
// launch chunks (1 = on; read per solve).  Not used while profiling (per-launch
// events cannot be recorded inside a graph).
int graph_mode() {
  const char* e = getenv("UQG_PCG_GRAPH");
  return e ? atoi(e) : 0;
}

size_t pcg_layout(Carver& c, long long N, const Geo& geo, int G, PcgState* st, double** r,
                  double** p, double** ap, int kx = x_defer()) {
  const size_t vec = (size_t)G * N * geo.S;
  const size_t lanes = (size_t)G * geo.S;
  double* rr = c.take<double>(vec);
  double* pp = c.take<double>(vec * kx);
  double* aa = c.take<double>(vec);
  PcgState s{};
  s.G = G;
  s.kx = kx;
  s.pstride = vec;
  s.part = c.take<double>((size_t)G * geo.pstride * 2 * geo.S);
  s.ticket = c.take<unsigned int>((size_t)G * geo.tstride);
  s.rz = c.take<double>(lanes);
  s.thr = c.take<double>(lanes);
  s.alpha = c.take<double>(lanes * kx);
  s.beta = c.take<double>(lanes);
  s.it = c.take<int>(G);
  s.done = c.take<int>(G);
  s.status = c.take<int>(G);
  s.ndone = c.take<int>(1);
  s.overflow = c.take<int>(1);
  // persistent-path extras: phase-A partials, group barriers, abort flag
  double* partA = c.take<double>((size_t)G * geo.chunks * geo.S);
  unsigned* bar = c.take<unsigned>(2 * (size_t)G + 1);
  if (st) *st = s;
  if (r) *r = rr;
  if (p) *p = pp;
  if (ap) *ap = aa;
  if (st) {
    g_persist.partA = partA;
    g_persist.bar = bar;
  }
  return c.off + 256;
}

}  // namespace

extern "C" {

int uqg_version(void) { return 1; }

const char* uqg_last_error(void) { return g_last_error.c_str(); }

int uqg_ctx_create(int device, uqg_ctx** out) {
  UQG_REQUIRE(out != nullptr, "uqg_ctx_create: out is NULL");
  UQG_TRY_CUDA(cudaSetDevice(device));
  uqg_ctx* c = new uqg_ctx();
  c->device = device;
  cudaError_t e = cudaMalloc(&c->status_dev, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->status_dev, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaHostAlloc(&c->pinned, 4 * sizeof(int), cudaHostAllocDefault);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    set_error(std::string("uqg_ctx_create: ") + cudaGetErrorString(e));
    delete c;
    return UQG_ECUDA;
  }
  *out = c;
  return UQG_OK;
}

int uqg_ctx_destroy(uqg_ctx* ctx) {
  if (!ctx) return UQG_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->status_dev) cudaFree(ctx->status_dev);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->ev) cudaEventDestroy(ctx->ev);
  for (cudaEvent_t e : ctx->evpool) cudaEventDestroy(e);
  for (cudaStream_t a : ctx->aux) cudaStreamDestroy(a);
  for (cudaEvent_t e : ctx->aux_ev) cudaEventDestroy(e);
  if (ctx->pinned_parts) cudaFreeHost(ctx->pinned_parts);
  if (ctx->cap) cudaStreamDestroy(ctx->cap);
  if (ctx->loops_dev) cudaFree(ctx->loops_dev);
  if (ctx->loops_host) cudaFreeHost(ctx->loops_host);
  delete ctx;
  return UQG_OK;
}

int uqg_ctx_set_workspace(uqg_ctx* ctx, void* ptr, long long bytes) {
  UQG_REQUIRE(ctx && bytes >= 0, "uqg_ctx_set_workspace: bad argument");
  ctx->ext = ptr;
  ctx->ext_bytes = ptr ? (size_t)bytes : 0;
  return UQG_OK;
}

int uqg_ctx_set_band_hint(uqg_ctx* ctx, int nbands, const int* starts_host,
                          const int* extras_host, int graph_padded) {
  UQG_REQUIRE(ctx && nbands >= 0 && nbands <= kMaxBands, "uqg_ctx_set_band_hint: bad argument");
  UQG_REQUIRE(nbands == 0 || (starts_host && extras_host), "uqg_ctx_set_band_hint: NULL bands");
  BandHint h{};
  h.nb = nbands;
  for (int b = 0; b < nbands; ++b) {
    UQG_REQUIRE(extras_host[b] >= 0 && extras_host[b] <= 64, "band extra rows out of range");
    h.start[b] = starts_host[b];
    h.extra[b] = extras_host[b];
  }
  h.padded = graph_padded != 0;
  ctx->bands = h;
  return UQG_OK;
}

int uqg_ctx_profile(uqg_ctx* ctx, int enable) {
  UQG_REQUIRE(ctx, "uqg_ctx_profile: NULL ctx");
  if (enable && ctx->evpool.empty()) {
    ctx->evpool.resize(2 * kEventPairs);
    ctx->pend_kind.resize(kEventPairs);
    for (auto& e : ctx->evpool) UQG_TRY_CUDA(cudaEventCreate(&e));
  }
  if (!enable) {
    int rc = harvest(ctx);
    if (rc) return rc;
  }
  ctx->prof = enable != 0;
  return UQG_OK;
}

int uqg_ctx_profile_read(uqg_ctx* ctx, double* ms_host, long long* launches_host, int reset) {
  UQG_REQUIRE(ctx, "uqg_ctx_profile_read: NULL ctx");
  int rc = harvest(ctx);
  if (rc) return rc;
  for (int k = 0; k < UQG_NKERN; ++k) {
    if (ms_host) ms_host[k] = ctx->kind_ms[k];
    if (launches_host) launches_host[k] = ctx->kind_launches[k];
    if (reset) {
      ctx->kind_ms[k] = 0.0;
      ctx->kind_launches[k] = 0;
    }
  }
  return UQG_OK;
}

long long uqg_ctx_launch_count(uqg_ctx* ctx) { return ctx ? ctx->launches : -1; }

int uqg_status_sync(uqg_ctx* ctx, void* stream, int* status_host) {
  UQG_REQUIRE(ctx && status_host, "uqg_status_sync: NULL argument");
  cudaStream_t s = as_stream(stream);
  UQG_TRY_CUDA(cudaMemcpyAsync(ctx->pinned, ctx->status_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
  UQG_TRY_CUDA(cudaMemsetAsync(ctx->status_dev, 0, sizeof(int), s));
  UQG_TRY_CUDA(cudaStreamSynchronize(s));
  *status_host = ctx->pinned[0];
  return UQG_OK;
}

int uqg_kl_eval_sep2d(uqg_ctx* ctx, int n_cells, const double* table1d, int n_factors,
                      const int* mode_p, const int* mode_q, const double* sqrt_lam, int M,
                      const double* samples, const int* lane_ids, int G, int S, double a_min,
                      int a_hat_mode, double a_hat_value, int expansion, double* a_out,
                      void* stream) {
  UQG_REQUIRE(ctx && table1d && mode_p && mode_q && sqrt_lam && samples && a_out,
              "uqg_kl_eval_sep2d: NULL argument");
  UQG_REQUIRE(n_cells >= 2 && n_factors >= 1 && M >= 1 && G >= 1 && S >= 1,
              "uqg_kl_eval_sep2d: bad sizes");
  UQG_REQUIRE(a_hat_mode == 0 || a_hat_mode == 1, "unknown a_hat mode");
  UQG_REQUIRE(expansion == 0 || expansion == 1, "unknown expansion");
  const int n1 = n_cells + 1;
  UQG_REQUIRE((long long)n1 * n1 < 0x7fffffffLL, "uqg_kl_eval_sep2d: too many nodes");
  const long long total = (long long)G * n1 * n1 * S;
  cudaStream_t s = as_stream(stream);
  // tiled contraction with the lane coefficients and the tile's mode values
  // staged in shared memory; M x S too large to stage: per-element kernel
  const size_t smem = ((size_t)M * S + S + 1 + (size_t)M * kKlTile) * sizeof(double);
  static size_t opted = 48 * 1024;
  if (smem > opted && smem <= 200 * 1024) {
    UQG_TRY_CUDA(cudaFuncSetAttribute(kl_sep2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    opted = smem;
  }
  if (smem <= opted) {
    const dim3 grid((unsigned)((n1 * n1 + kKlTile - 1) / kKlTile), (unsigned)G);
    UQG_LAUNCH(UQG_K_KL, s,
               kl_sep2d_kernel<<<grid, 256, smem, s>>>(
                   n1, table1d, mode_p, mode_q, sqrt_lam, M, samples, lane_ids, G, S, a_min,
                   a_hat_mode, a_hat_value, expansion, a_out, ctx->status_dev));
  } else {
    UQG_LAUNCH(UQG_K_KL, s,
               kl_sep2d_elem_kernel<<<grid_for(total, 256), 256, 0, s>>>(
                   n1, table1d, mode_p, mode_q, sqrt_lam, M, samples, lane_ids, G, S, a_min,
                   a_hat_mode, a_hat_value, expansion, a_out, ctx->status_dev));
  }
  return UQG_OK;
}

int uqg_kl_eval_table(uqg_ctx* ctx, const double* modes, int P, int M, const double* sqrt_lam,
                      const double* samples, int L, double a_min, int a_hat_mode,
                      double a_hat_value, int expansion, double* a_out, void* stream) {
  UQG_REQUIRE(ctx && modes && sqrt_lam && samples && a_out, "uqg_kl_eval_table: NULL argument");
  UQG_REQUIRE(P >= 1 && M >= 1 && L >= 1, "uqg_kl_eval_table: bad sizes");
  UQG_REQUIRE(a_hat_mode == 0 || a_hat_mode == 1, "unknown a_hat mode");
  UQG_REQUIRE(expansion == 0 || expansion == 1, "unknown expansion");
  const long long total = (long long)L * P;
  cudaStream_t s = as_stream(stream);
  UQG_LAUNCH(UQG_K_KL, s,
             kl_table_kernel<<<grid_for(total, 256), 256, 0, s>>>(
                 modes, P, M, sqrt_lam, samples, L, a_min, a_hat_mode, a_hat_value, expansion,
                 a_out, ctx->status_dev));
  return UQG_OK;
}

int uqg_assemble_fv2d(uqg_ctx* ctx, int n_cells, int G, int S, const double* a_nodes,
                      double a_y, int a2_same, const int* row_offsets, double* vals,
                      double* dinv, void* stream) {
  UQG_REQUIRE(ctx && a_nodes && row_offsets && vals, "uqg_assemble_fv2d: NULL argument");
  UQG_REQUIRE(n_cells >= 2 && G >= 1 && S >= 1, "uqg_assemble_fv2d: bad sizes");
  const long long N = (long long)(n_cells - 1) * (n_cells - 1);
  const long long total = (long long)G * N * S;
  cudaStream_t s = as_stream(stream);
  UQG_LAUNCH(UQG_K_ASSEMBLE, s,
             assemble_fv2d_kernel<<<grid_for(total, 256), 256, 0, s>>>(
                 n_cells, G, S, a_nodes, a_y, a2_same, row_offsets, vals, dinv));
  return UQG_OK;
}

int uqg_kl_eval_sep3d(uqg_ctx* ctx, int m, const double* qtab, int n_factors, const int* mode_p,
                      const int* mode_q, const int* mode_r, const double* sqrt_lam, int M,
                      const double* samples, const int* lane_ids, int G, int S, double a_min,
                      int a_hat_mode, double a_hat_value, int expansion, double* a_out,
                      void* stream) {
  UQG_REQUIRE(ctx && qtab && mode_p && mode_q && mode_r && sqrt_lam && samples && a_out,
              "uqg_kl_eval_sep3d: NULL argument");
  UQG_REQUIRE(m >= 2 && n_factors >= 1 && M >= 1 && G >= 1 && S >= 1,
              "uqg_kl_eval_sep3d: bad sizes");
  UQG_REQUIRE(a_hat_mode == 0 || a_hat_mode == 1, "unknown a_hat mode");
  UQG_REQUIRE(expansion == 0 || expansion == 1, "unknown expansion");
  const long long total = (long long)G * 8 * m * m * m * S;
  cudaStream_t s = as_stream(stream);
  UQG_LAUNCH(UQG_K_KL, s,
             kl_sep3d_kernel<<<grid_for(total, 256), 256, 0, s>>>(
                 m, qtab, mode_p, mode_q, mode_r, sqrt_lam, M, samples, lane_ids, G, S, a_min,
                 a_hat_mode, a_hat_value, expansion, a_out, ctx->status_dev));
  return UQG_OK;
}

int uqg_assemble_fem3d(uqg_ctx* ctx, int m, int G, int S, const double* a_q, const double* dx_tab,
                       const double* kyz_tab, const int* row_offsets, double* vals, double* dinv,
                       void* stream) {
  UQG_REQUIRE(ctx && a_q && dx_tab && kyz_tab && row_offsets && vals,
              "uqg_assemble_fem3d: NULL argument");
  UQG_REQUIRE(m >= 2 && G >= 1 && S >= 1, "uqg_assemble_fem3d: bad sizes");
  const long long N = (long long)(m - 1) * (m - 1) * (m - 1);
  const long long total = (long long)G * N * S;
  cudaStream_t s = as_stream(stream);
  UQG_LAUNCH(UQG_K_ASSEMBLE, s,
             assemble_fem3d_kernel<<<grid_for(total, 256), 256, 0, s>>>(
                 m, G, S, a_q, dx_tab, kyz_tab, row_offsets, vals, dinv));
  return UQG_OK;
}

int uqg_jacobi_dinv(uqg_ctx* ctx, int N, int nnz, int S, int G, const int* row_offsets,
                    const int* col_indices, const double* vals, double* dinv, void* stream) {
  UQG_REQUIRE(ctx && row_offsets && dinv, "uqg_jacobi_dinv: NULL argument");
  UQG_REQUIRE(N >= 0 && nnz >= 0 && S >= 1 && G >= 1, "uqg_jacobi_dinv: bad sizes");
  int st = 0;
  int rc = uqg_status_sync(ctx, stream, &st);  // clear stale bits
  if (rc) return rc;
  const long long total = (long long)G * N * S;
  cudaStream_t s = as_stream(stream);
  if (total > 0) {
    UQG_LAUNCH(UQG_K_OTHER, s,
               jacobi_dinv_kernel<<<grid_for(total, 256), 256, 0, s>>>(
                   N, S, G, nnz, row_offsets, col_indices, vals, dinv, ctx->status_dev, 0));
  }
  rc = uqg_status_sync(ctx, stream, &st);
  if (rc) return rc;
  UQG_REQUIRE(!(st & 1), "Jacobi preconditioner needs strictly positive lane diagonals");
  return UQG_OK;
}

int uqg_diagonal(uqg_ctx* ctx, int N, int nnz, int S, int G, const int* row_offsets,
                 const int* col_indices, const double* vals, double* diag, void* stream) {
  UQG_REQUIRE(ctx && row_offsets && diag, "uqg_diagonal: NULL argument");
  UQG_REQUIRE(N >= 0 && nnz >= 0 && S >= 1 && G >= 1, "uqg_diagonal: bad sizes");
  const long long total = (long long)G * N * S;
  cudaStream_t s = as_stream(stream);
  if (total > 0) {
    UQG_LAUNCH(UQG_K_OTHER, s,
               jacobi_dinv_kernel<<<grid_for(total, 256), 256, 0, s>>>(
                   N, S, G, nnz, row_offsets, col_indices, vals, diag, ctx->status_dev, 1));
  }
  return UQG_OK;
}

int uqg_spmv(uqg_ctx* ctx, int N, int nnz, int max_row_len, int S, int G,
             const int* row_offsets, const int* col_indices, const double* vals, const double* x,
             double* y, void* stream) {
  UQG_REQUIRE(ctx && row_offsets && x && y, "uqg_spmv: NULL argument");
  UQG_REQUIRE(N >= 0 && nnz >= 0 && S >= 1 && S <= kMaxLanes && G >= 1, "uqg_spmv: bad sizes");
  if (N == 0) return UQG_OK;
  Geo geo = make_geo(N, S, max_row_len);
  cudaStream_t s = as_stream(stream);
  UQG_LAUNCH(UQG_K_SPMV, s,
             launch_spmv(geo, G, s, N, nnz, row_offsets, col_indices, vals, x, y));
  return UQG_OK;
}

int uqg_lane_dot(uqg_ctx* ctx, int N, int S, int G, const double* a, const double* b,
                 double* out, void* stream) {
  UQG_REQUIRE(ctx && a && b && out, "uqg_lane_dot: NULL argument");
  UQG_REQUIRE(N >= 0 && S >= 1 && S <= kMaxLanes && G >= 1, "uqg_lane_dot: bad sizes");
  cudaStream_t s = as_stream(stream);
  Geo geo = make_geo(N, S);
  size_t need = (size_t)G * geo.pstride * geo.S * sizeof(double) +
                (size_t)G * geo.tstride * sizeof(unsigned) + 1024;
  int rc = ensure_ws(ctx, need);
  if (rc) return rc;
  Carver c{(char*)ws_base(ctx, need)};
  double* part = c.take<double>((size_t)G * geo.pstride * geo.S);
  unsigned* ticket = c.take<unsigned>((size_t)G * geo.tstride);
  UQG_TRY_CUDA(cudaMemsetAsync(ticket, 0, (size_t)G * geo.tstride * sizeof(unsigned), s));
  UQG_LAUNCH(UQG_K_DOT, s, launch_lane_dot(geo, G, s, N, a, b, out, part, ticket));
  return UQG_OK;
}

int uqg_pcg_x_defer(void) { return x_defer(); }

long long uqg_pcg_workspace_bytes(int N, int nnz, int S, int G) {
  (void)nnz;
  if (N < 0 || S < 1 || G < 1) return -1;
  Geo geo = make_geo(N, S);
  Carver c{nullptr};
  return (long long)pcg_layout(c, N, geo, G, nullptr, nullptr, nullptr, nullptr);
}

}  // extern "C"

namespace {

// The operator of a PCG solve: shared-graph CSR (row_offsets / col_indices /
// vals) or the face form of the 2D FV operator (fv.tx != nullptr).
struct SpOp {
  const int* ro;
  const int* ci;
  const double* vals;
  Fv2dOp fv;
};

int pcg_impl(uqg_ctx* ctx, int N, int nnz, int max_row_len, int S, int G, const SpOp& op,
             const double* rhs, double rhs_const, const double* dinv, double tol, int maxit,
             double* x, int* iters, unsigned char* converged, unsigned char* frozen,
             int* ens_iters, double* hist_host, int hist_cap, int* hist_rows_host, void* stream);

}  // namespace

extern "C" {

int uqg_pcg(uqg_ctx* ctx, int N, int nnz, int max_row_len, int S, int G, const int* row_offsets,
            const int* col_indices, const double* vals, const double* rhs, double rhs_const,
            const double* dinv, double tol, int maxit, double* x, int* iters,
            unsigned char* converged, unsigned char* frozen, int* ens_iters,
            double* hist_host, int hist_cap, int* hist_rows_host, void* stream) {
  UQG_REQUIRE(ctx && row_offsets && x && iters && converged && frozen && ens_iters,
              "uqg_pcg: NULL argument");
  UQG_REQUIRE(N >= 0 && nnz >= 0 && S >= 1 && S <= kMaxLanes && G >= 1, "uqg_pcg: bad sizes");
  SpOp op{row_offsets, col_indices, vals, Fv2dOp{0, nullptr, nullptr, 0.0}};
  return pcg_impl(ctx, N, nnz, max_row_len, S, G, op, rhs, rhs_const, dinv, tol, maxit, x, iters,
                  converged, frozen, ens_iters, hist_host, hist_cap, hist_rows_host, stream);
}

int uqg_assemble_fv2d_faces(uqg_ctx* ctx, int n_cells, int G, int S, const double* a_nodes,
                            double a_y, int a2_same, double* tx, double* ty, double* dinv,
                            void* stream) {
  UQG_REQUIRE(ctx && a_nodes && tx && (!a2_same || ty), "uqg_assemble_fv2d_faces: NULL argument");
  UQG_REQUIRE(n_cells >= 2 && G >= 1 && S >= 1, "uqg_assemble_fv2d_faces: bad sizes");
  const long long m = n_cells - 1;
  const long long total = (long long)G * (m * m + m) * S;
  cudaStream_t s = as_stream(stream);
  UQG_LAUNCH(UQG_K_ASSEMBLE, s,
             assemble_fv2d_faces_kernel<<<grid_for(total, 256), 256, 0, s>>>(
                 n_cells, G, S, a_nodes, a2_same, a_y, tx, a2_same ? ty : nullptr, dinv));
  return UQG_OK;
}

int uqg_spmv_fv2d(uqg_ctx* ctx, int n_cells, int S, int G, const double* tx, const double* ty,
                  double a_y, const double* x, double* y, void* stream) {
  UQG_REQUIRE(ctx && tx && x && y, "uqg_spmv_fv2d: NULL argument");
  UQG_REQUIRE(n_cells >= 2 && S >= 1 && S <= kMaxLanes && G >= 1, "uqg_spmv_fv2d: bad sizes");
  const long long m = n_cells - 1, N = m * m;
  UQG_REQUIRE((N + m) * S <= 0x7fffffffLL, "uqg_spmv_fv2d: (N + m) * S must be < 2^31");
  Geo geo = make_geo(N, S, 5);
  cudaStream_t s = as_stream(stream);
  Fv2dOp op{(int)m, tx, ty, a_y};
  UQG_LAUNCH(UQG_K_SPMV, s, launch_spmv_fv2d(geo, G, s, N, op, x, y));
  return UQG_OK;
}

int uqg_pcg_fv2d(uqg_ctx* ctx, int n_cells, int S, int G, const double* tx, const double* ty,
                 double a_y, const double* rhs, double rhs_const, const double* dinv, double tol,
                 int maxit, double* x, int* iters, unsigned char* converged,
                 unsigned char* frozen, int* ens_iters, double* hist_host, int hist_cap,
                 int* hist_rows_host, void* stream) {
  UQG_REQUIRE(ctx && tx && x && iters && converged && frozen && ens_iters,
              "uqg_pcg_fv2d: NULL argument");
  UQG_REQUIRE(n_cells >= 2 && S >= 1 && S <= kMaxLanes && G >= 1, "uqg_pcg_fv2d: bad sizes");
  const long long m = n_cells - 1;
  UQG_REQUIRE((m * m + m) * S <= 0x7fffffffLL, "uqg_pcg_fv2d: (N + m) * S must be < 2^31");
  SpOp op{nullptr, nullptr, nullptr, Fv2dOp{(int)m, tx, ty, a_y}};
  return pcg_impl(ctx, (int)(m * m), 0, 5, S, G, op, rhs, rhs_const, dinv, tol, maxit, x, iters,
                  converged, frozen, ens_iters, hist_host, hist_cap, hist_rows_host, stream);
}

}  // extern "C"

namespace {

int pcg_impl(uqg_ctx* ctx, int N, int nnz, int max_row_len, int S, int G, const SpOp& op,
             const double* rhs, double rhs_const, const double* dinv, double tol, int maxit,
             double* x, int* iters, unsigned char* converged, unsigned char* frozen,
             int* ens_iters, double* hist_host, int hist_cap, int* hist_rows_host, void* stream) {
  UQG_REQUIRE(tol > 0.0 && tol <= 1.7976931348623157e308, "tol must be positive and finite");
  UQG_REQUIRE(maxit >= 0, "maxit must be >= 0");
  UQG_REQUIRE(!hist_host || (hist_cap >= 0 && hist_rows_host), "uqg_pcg: bad history buffer");
  cudaStream_t s = as_stream(stream);
  Geo geo = make_geo(N, S, max_row_len);
  // Small batches: one cooperative launch runs the whole solve (uqg_persistent.cu).
  // UQG_PCG_PERSISTENT: 2 = cluster-barrier kernel, 1 = cooperative kernel,
  // 0 = launch loop; auto = cluster kernel for small batches (< 512 MB per
  // iteration), launch loop otherwise.
  const int pmode = persistent_mode();
  const double op_elems = op.fv.tx ? (double)(N + op.fv.m) * (op.fv.ty ? 2 : 1) : (double)nnz;
  const double iter_bytes = 8.0 * S * (op_elems + 12.0 * N) * G;
  const bool small = iter_bytes < 512e6;
  bool use_cluster = false;
  int pblocks = 0;
  // (the persistent kernels reduce without super-chunks: geo.sc == 1 only)
  if (geo.sc == 1 && (pmode == 2 || (pmode < 0 && small))) {
    const int cs = persistent_cluster_size(geo);
    if (cs >= 2) {
      use_cluster = true;
      pblocks = cs;
    }
  }
  if (!use_cluster && geo.sc == 1 && (pmode == 1 || (pmode < 0 && small)))
    pblocks = persistent_blocks(geo, G);
  // workspace: the persistent kernel updates x in place (kx = 1)
  const int kx = pblocks > 0 ? 1 : x_defer();
  int P = 1;  // concurrent parts of the launch loop
  if (pblocks == 0 && !hist_host) {
    P = solve_streams();
    while (P > 1 && (iter_bytes / P < 1e9 || G / P < 1)) --P;
  }
  struct Part {
    int g0, G;
    PcgState st;
    double *r, *p, *ap;
    cudaStream_t s;
    SpOp op;
    bool done;
  } parts[kMaxParts];
  Carver probe{nullptr};
  size_t need = 0;
  for (int i = 0; i < P; ++i) {
    const int g0 = (int)((long long)G * i / P), g1 = (int)((long long)G * (i + 1) / P);
    need = pcg_layout(probe, N, geo, g1 - g0, nullptr, nullptr, nullptr, nullptr, kx);
  }
  size_t hist_elems = hist_host ? (size_t)(hist_cap + 1) * G * S : 0;
  need += hist_elems * sizeof(double) + 256;
  int rc = ensure_ws(ctx, need);
  if (rc) return rc;
  if (P > 1 && (int)ctx->aux.size() < P - 1) {  // lazily created part streams
    if (!ctx->pinned_parts)
      UQG_TRY_CUDA(cudaHostAlloc(&ctx->pinned_parts, kMaxParts * sizeof(int), cudaHostAllocDefault));
    while ((int)ctx->aux.size() < kMaxParts - 1) {
      cudaStream_t a;
      UQG_TRY_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
      ctx->aux.push_back(a);
    }
    while ((int)ctx->aux_ev.size() < kMaxParts) {
      cudaEvent_t e;
      UQG_TRY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ctx->aux_ev.push_back(e);
    }
  }
  Carver c{(char*)ws_base(ctx, need)};
  if (P > 1) {  // part streams start after everything queued on the caller's stream
    UQG_TRY_CUDA(cudaEventRecord(ctx->aux_ev[0], s));
    for (int i = 1; i < P; ++i) UQG_TRY_CUDA(cudaStreamWaitEvent(ctx->aux[i - 1], ctx->aux_ev[0], 0));
  }
  const size_t vs = (size_t)N * S;  // per-group vector stride
  for (int i = 0; i < P; ++i) {
    Part& q = parts[i];
    q.g0 = (int)((long long)G * i / P);
    q.G = (int)((long long)G * (i + 1) / P) - q.g0;
    // UQG_FACE_CLUSTER: the parts run one after the other on the caller's stream - the
    // cluster SpMV needs whole SMs (two co-scheduled CTAs of 104 KB shared memory each), and
    // kernels of another stream squeezed in between its clusters cost more than they fill
    static const bool one_stream = [] {
      const char* e = getenv("UQG_FACE_CLUSTER");
      return e && atoi(e) != 0;
    }();
    q.s = (i == 0 || one_stream) ? s : ctx->aux[i - 1];
    q.done = false;
    pcg_layout(c, N, geo, q.G, &q.st, &q.r, &q.p, &q.ap, kx);
    q.st.iters = iters + (size_t)q.g0 * S;
    q.st.conv = converged + (size_t)q.g0 * S;
    q.st.frozen = frozen + (size_t)q.g0 * S;
    q.st.hist = nullptr;
    q.st.hist_cap = hist_cap;
    q.op = op;
    if (op.vals) q.op.vals = op.vals + (size_t)q.g0 * nnz * S;
    if (op.fv.tx) q.op.fv.tx = op.fv.tx + (size_t)q.g0 * (N + op.fv.m) * S;
    if (op.fv.ty) q.op.fv.ty = op.fv.ty + (size_t)q.g0 * (N + op.fv.m) * S;
    UQG_TRY_CUDA(cudaMemsetAsync(q.st.ticket, 0, (size_t)q.G * geo.tstride * sizeof(unsigned), q.s));
    UQG_TRY_CUDA(cudaMemsetAsync(q.st.ndone, 0, sizeof(int), q.s));
    UQG_TRY_CUDA(cudaMemsetAsync(q.st.overflow, 0, sizeof(int), q.s));
  }
  // One PCG iteration of part q on stream qs, blocks per group from gl; flush:
  // the iteration closes a deferral window (pcg_flush before pcg_dir).
  auto launch_iteration = [&](const Part& q, const Geo& gl, cudaStream_t qs, bool flush) -> int {
    double* xq = x + (size_t)q.g0 * vs;
    const double* dq = dinv ? dinv + (size_t)q.g0 * vs : nullptr;
    if (q.op.fv.tx)
      UQG_LAUNCH(UQG_K_PCG_SPMV, qs,
                 launch_pcg_spmv_fv2d(gl, q.G, qs, N, q.st, q.op.fv, q.p, q.ap));
    else
      UQG_LAUNCH(UQG_K_PCG_SPMV, qs,
                 launch_pcg_spmv(gl, q.G, qs, N, nnz, q.st, q.op.ro, q.op.ci, q.op.vals, q.p,
                                 q.ap, ctx->bands.nb ? &ctx->bands : nullptr));
    UQG_LAUNCH(UQG_K_PCG_UPDATE, qs, launch_pcg_update(gl, q.G, qs, N, q.st, dq, maxit, q.r, q.ap));
    if (flush) UQG_LAUNCH(UQG_K_PCG_FLUSH, qs, launch_pcg_flush(gl, q.G, qs, N, q.st, xq, q.p, true));
    UQG_LAUNCH(UQG_K_PCG_DIR, qs, launch_pcg_dir(gl, q.G, qs, N, q.st, dq, q.r, xq, q.p));
    return UQG_OK;
  };
  PcgState& st = parts[0].st;  // single-part view (persistent path, history, status)
  st.hist = hist_host ? c.take<double>(hist_elems) : nullptr;
  double *r = parts[0].r, *p = parts[0].p, *ap = parts[0].ap;

  if (pblocks > 0) {
    PersistBufs pb = g_persist;
    UQG_TRY_CUDA(cudaMemsetAsync(pb.bar, 0, (2 * (size_t)G + 1) * sizeof(unsigned), s));
    cudaError_t le = cudaSuccess;
    UQG_LAUNCH(UQG_K_PCG_SPMV, s, {
      le = launch_pcg_persistent(geo, G, pblocks, use_cluster, s, N, nnz, st, op.ro, op.ci,
                                 op.vals, op.fv, rhs, rhs_const, dinv, tol, maxit, x, r, p, ap,
                                 pb.partA, st.part, pb.bar, pb.bar + G,
                                 reinterpret_cast<int*>(pb.bar + 2 * G));
    });
    if (le != cudaSuccess) {
      cudaGetLastError();
      set_error(std::string("cooperative launch: ") + cudaGetErrorString(le));
      return UQG_ECUDA;
    }
    UQG_TRY_CUDA(cudaMemcpyAsync(ctx->pinned + 2, pb.bar + 2 * G, sizeof(int),
                                 cudaMemcpyDeviceToHost, s));
    UQG_TRY_CUDA(cudaStreamSynchronize(s));
    if (ctx->pinned[2]) {
      set_error("uqg_pcg: persistent solve aborted (group barrier timeout)");
      return UQG_ECUDA;
    }
  } else if (P == 1 && !ctx->prof && graph_mode() > 0) {
    // Graph launch loop: the same kernels and per-iteration order as the
    // host-polled loop below, blocks sized for all G groups (finished groups'
    // blocks exit at once; results do not depend on the block count).
    UQG_LAUNCH(UQG_K_PCG_INIT, s,
               launch_pcg_init(geo, G, s, N, st, rhs, rhs_const, dinv, tol, maxit, x, r, p));
    if (!ctx->cap) {
      UQG_TRY_CUDA(cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
      UQG_TRY_CUDA(cudaMalloc(&ctx->loops_dev, sizeof(int)));
      UQG_TRY_CUDA(cudaHostAlloc(&ctx->loops_host, 2 * sizeof(int), cudaHostAllocDefault));
    }
    UQG_TRY_CUDA(cudaMemsetAsync(ctx->loops_dev, 0, sizeof(int), s));
    const Geo gl = with_groups(geo, G);
    const int max_loops = (maxit + 2) / kx + 2;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle hc;
    UQG_TRY_CUDA(cudaGraphCreate(&graph, 0));
    cudaError_t ge = cudaGraphConditionalHandleCreate(&hc, graph, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hc;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    if (ge == cudaSuccess) ge = cudaGraphAddNode(&node, graph, nullptr, 0, &cp);
    if (ge == cudaSuccess)
      ge = cudaStreamBeginCaptureToGraph(ctx->cap, cp.conditional.phGraph_out[0], nullptr, nullptr,
                                         0, cudaStreamCaptureModeRelaxed);
    int brc = UQG_OK;
    long long per_pass = 0;
    if (ge == cudaSuccess) {
      const long long before = ctx->launches;
      cudaStream_t cs = ctx->cap;
      brc = [&]() -> int {  // the body: iterations k = 0..kx-1 of a window
        for (int k = 0; k < kx; ++k) {
          const int rc = launch_iteration(parts[0], gl, cs, kx > 1 && k == kx - 1);
          if (rc) return rc;
        }
        UQG_LAUNCH(UQG_K_OTHER, cs,
                   launch_pcg_loop_cond(cs, hc, st.ndone, G, ctx->loops_dev, max_loops));
        return UQG_OK;
      }();
      cudaGraph_t body = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(ctx->cap, &body);
      if (ge == cudaSuccess) ge = ce;
      per_pass = ctx->launches - before;
    }
    if (ge == cudaSuccess && brc == UQG_OK) ge = cudaGraphInstantiate(&exec, graph, 0);
    if (ge == cudaSuccess && brc == UQG_OK) ge = cudaGraphLaunch(exec, s);
    if (exec) cudaGraphExecDestroy(exec);  // freed once the launch completes
    cudaGraphDestroy(graph);
    if (brc) return brc;
    if (ge != cudaSuccess) {
      cudaGetLastError();
      set_error(std::string("uqg_pcg graph loop: ") + cudaGetErrorString(ge));
      return UQG_ECUDA;
    }
    if (kx > 1)  // deferred x updates still pending at termination
      UQG_LAUNCH(UQG_K_PCG_FLUSH, s, launch_pcg_flush(gl, G, s, N, st, x, p, false));
    UQG_TRY_CUDA(cudaMemcpyAsync(ctx->loops_host, ctx->loops_dev, sizeof(int),
                                 cudaMemcpyDeviceToHost, s));
    UQG_TRY_CUDA(cudaMemcpyAsync(ctx->loops_host + 1, st.ndone, sizeof(int),
                                 cudaMemcpyDeviceToHost, s));
    UQG_TRY_CUDA(cudaStreamSynchronize(s));
    const int passes = ctx->loops_host[0];
    if (ctx->loops_host[1] < G) {
      set_error("uqg_pcg: device loop failed to terminate");
      return UQG_ECUDA;
    }
    // launch accounting: the body was counted once at capture
    ctx->launches += per_pass * (passes - 1);
    ctx->kind_launches[UQG_K_PCG_SPMV] += (long long)kx * (passes - 1);
    ctx->kind_launches[UQG_K_PCG_UPDATE] += (long long)kx * (passes - 1);
    ctx->kind_launches[UQG_K_PCG_DIR] += (long long)kx * (passes - 1);
    ctx->kind_launches[UQG_K_PCG_FLUSH] += (long long)(kx > 1) * (passes - 1);
    ctx->kind_launches[UQG_K_OTHER] += passes - 1;
  } else {
    // Launch loop: the host polls each part's device done-counter between
    // chunks of iterations and launches the next chunk for every part still
    // running, alternating parts per iteration.  Groups that have terminated
    // turn every later launch into a no-op, so the extra launches of the last
    // chunk cannot change any result.
    auto vec = [&](const Part& q, const double* v) { return v ? v + (size_t)q.g0 * vs : v; };
    auto vecw = [&](const Part& q, double* v) { return v + (size_t)q.g0 * vs; };
    for (int i = 0; i < P; ++i) {
      Part& q = parts[i];
      UQG_LAUNCH(UQG_K_PCG_INIT, q.s,
                 launch_pcg_init(geo, q.G, q.s, N, q.st, vec(q, rhs), rhs_const, vec(q, dinv), tol,
                                 maxit, vecw(q, x), q.r, q.p));
    }
    int* pin = P > 1 ? ctx->pinned_parts : ctx->pinned;
    long long launched = 0;
    int chunk = 2;
    for (;;) {
      bool all_done = true;
      for (int i = 0; i < P; ++i) {
        Part& q = parts[i];
        if (q.done) continue;
        UQG_TRY_CUDA(cudaMemcpyAsync(pin + i, q.st.ndone, sizeof(int), cudaMemcpyDeviceToHost, q.s));
        UQG_TRY_CUDA(cudaEventRecord(P > 1 ? ctx->aux_ev[i] : ctx->ev, q.s));
      }
      for (int i = 0; i < P; ++i) {
        Part& q = parts[i];
        if (q.done) continue;
        UQG_TRY_CUDA(cudaEventSynchronize(P > 1 ? ctx->aux_ev[i] : ctx->ev));
        q.done = pin[i] >= q.G;
        all_done = all_done && q.done;
      }
      if (all_done) break;
      if (launched > (long long)maxit + 1) {
        set_error("uqg_pcg: device loop failed to terminate");
        return UQG_ECUDA;
      }
      // Size blocks-per-group for the groups still running (finished groups'
      // blocks exit at once); the reduction chunks - hence the results - do
      // not depend on this.
      Geo gact[kMaxParts];
      for (int i = 0; i < P; ++i) gact[i] = with_groups(geo, std::max(1, parts[i].G - pin[i]));
      for (int k = 0; k < chunk; ++k) {
        for (int i = 0; i < P; ++i) {
          if (parts[i].done) continue;
          // iteration launched + k closes a deferral window: flush before pcg_dir
          const int rc = launch_iteration(parts[i], gact[i], parts[i].s,
                                          kx > 1 && (launched + k + 1) % kx == 0);
          if (rc) return rc;
        }
      }
      launched += chunk;
      chunk = std::min(chunk * 2, 64);
    }
    for (int i = 0; i < P; ++i) {
      Part& q = parts[i];
      if (kx > 1)  // deferred x updates still pending at termination
        UQG_LAUNCH(UQG_K_PCG_FLUSH, q.s,
                   launch_pcg_flush(with_groups(geo, q.G), q.G, q.s, N, q.st, vecw(q, x), q.p,
                                    false));
      if (i > 0) UQG_LAUNCH(UQG_K_OTHER, q.s, launch_pcg_finalize(q.G, S, q.s, q.st, ens_iters + q.g0));
    }
    for (int i = 1; i < P; ++i) {  // the caller's stream waits for every part
      UQG_TRY_CUDA(cudaEventRecord(ctx->aux_ev[i], parts[i].s));
      UQG_TRY_CUDA(cudaStreamWaitEvent(s, ctx->aux_ev[i], 0));
    }
  }
  UQG_LAUNCH(UQG_K_OTHER, s, launch_pcg_finalize(parts[0].G, S, s, st, ens_iters));
  // breakdown / history bookkeeping
  std::vector<int> h_status(G);
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < P && e == cudaSuccess; ++i)
    e = cudaMemcpyAsync(h_status.data() + parts[i].g0, parts[i].st.status,
                        parts[i].G * sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ctx->pinned + 1, st.overflow, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    set_error(std::string("uqg_pcg: ") + cudaGetErrorString(e));
    return UQG_ECUDA;
  }
  for (int g = 0; g < G; ++g) {
    if (h_status[g] & 4) {
      set_error("uqg_pcg: cluster SpMV pipeline failed (group " + std::to_string(g) + ")");
      return UQG_ECUDA;
    }
    if (h_status[g] == 2) {
      set_error("non-finite residual in active lane (group " + std::to_string(g) + ")");
      return UQG_EBREAKDOWN;
    }
  }
  if (hist_host) {
    if (ctx->pinned[1]) {
      set_error("residual history capacity exceeded");
      return UQG_ECAPACITY;
    }
    std::vector<int> h_it(G);
    e = cudaMemcpy(h_it.data(), st.it, G * sizeof(int), cudaMemcpyDeviceToHost);
    int rows = 1 + *std::max_element(h_it.begin(), h_it.end());
    if (e == cudaSuccess)
      e = cudaMemcpy(hist_host, st.hist, (size_t)rows * G * S * sizeof(double),
                     cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      set_error(std::string("uqg_pcg history: ") + cudaGetErrorString(e));
      return UQG_ECUDA;
    }
    *hist_rows_host = rows;
  }
  return UQG_OK;
}

}  // namespace

extern "C" {

int uqg_surrogate_eval(uqg_ctx* ctx, const double* points, int n, int dim, const double* centers,
                       const double* widths, const double* surplus, int n_nodes, double* out,
                       void* stream) {
  UQG_REQUIRE(ctx && out && (n == 0 || points), "uqg_surrogate_eval: NULL argument");
  UQG_REQUIRE(n >= 0 && dim >= 1 && dim <= 64 && n_nodes >= 0, "uqg_surrogate_eval: bad sizes");
  UQG_REQUIRE(n_nodes == 0 || (centers && widths && surplus), "uqg_surrogate_eval: NULL nodes");
  if (n == 0) return UQG_OK;
  cudaStream_t s = as_stream(stream);
  UQG_LAUNCH(UQG_K_GROUP, s,
             launch_surrogate_eval(s, points, n, dim, centers, widths, surplus, n_nodes, out));
  return UQG_OK;
}

int uqg_anisotropy_indicator(uqg_ctx* ctx, const double* modes, int P, int M,
                             const double* sqrt_lam, const double* samples, int L, double a_min,
                             int a_hat_mode, double a_hat_value, int expansion, double a_hi,
                             double a_lo, double* out, void* stream) {
  UQG_REQUIRE(ctx && modes && sqrt_lam && samples && out, "uqg_anisotropy_indicator: NULL argument");
  UQG_REQUIRE(P >= 1 && M >= 1 && L >= 1, "uqg_anisotropy_indicator: bad sizes");
  UQG_REQUIRE(a_hat_mode == 0 || a_hat_mode == 1, "unknown a_hat mode");
  UQG_REQUIRE(expansion == 0 || expansion == 1, "unknown expansion");
  int st = 0;
  int rc = uqg_status_sync(ctx, stream, &st);
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  UQG_LAUNCH(UQG_K_KL, s,
             launch_anisotropy(s, modes, P, M, sqrt_lam, samples, L, a_min, a_hat_mode,
                               a_hat_value, expansion, a_hi, a_lo, out, ctx->status_dev));
  rc = uqg_status_sync(ctx, stream, &st);
  if (rc) return rc;
  UQG_REQUIRE(!(st & 1), "anisotropy indicator needs strictly positive coefficients");
  return UQG_OK;
}

}  // extern "C"

namespace {

// Stable ascending sort of the keys (LSD radix sort over the order-preserving
// 64-bit images, cub::DeviceRadixSort - stable, so equal keys keep generation
// order) + chunking into width-S groups.  No host synchronisation: a
// non-finite key sets status bit 1, read by the caller's next status check.
int group_sort_impl(uqg_ctx* ctx, const double* keys, int n, int S, int* order, int* groups,
                    int* pad, cudaStream_t s) {
  const int K = (n + S - 1) / S;
  int* ord = order;
  if (keys) {
    size_t temp = 0;
    UQG_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, (unsigned long long*)nullptr,
                                                 (unsigned long long*)nullptr, (int*)nullptr,
                                                 (int*)nullptr, n, 0, 64, s));
    Carver probe{nullptr};
    probe.take<unsigned long long>(n);
    probe.take<unsigned long long>(n);
    probe.take<int>(n);
    probe.take<int>(n);
    probe.take<char>(temp);
    const size_t need = probe.off + 256;
    int rc = ensure_ws(ctx, need);
    if (rc) return rc;
    Carver c{(char*)ws_base(ctx, need)};
    unsigned long long* kin = c.take<unsigned long long>(n);
    unsigned long long* kout = c.take<unsigned long long>(n);
    int* ids = c.take<int>(n);
    int* ord_ws = c.take<int>(n);
    void* tmp = c.take<char>(temp);
    if (!ord) ord = ord_ws;
    UQG_LAUNCH(UQG_K_GROUP, s,
               key_bits_kernel<<<(n + 255) / 256, 256, 0, s>>>(keys, n, kin, ids, ctx->status_dev));
    cudaError_t se = cudaSuccess;  // cub launches its own kernels (counted as one)
    UQG_LAUNCH(UQG_K_GROUP, s,
               se = cub::DeviceRadixSort::SortPairs(tmp, temp, kin, kout, ids, ord, n, 0, 64, s));
    UQG_TRY_CUDA(se);
  } else {
    ord = nullptr;  // natural order
  }
  const long long slots = (long long)K * S;
  UQG_LAUNCH(UQG_K_GROUP, s,
             chunk_kernel<<<(int)((slots + 255) / 256), 256, 0, s>>>(ord, n, S, K, groups, pad));
  if (!keys && order) {
    UQG_TRY_CUDA(cudaMemcpyAsync(order, groups, (size_t)n * sizeof(int), cudaMemcpyDeviceToDevice, s));
  }
  return UQG_OK;
}

}  // namespace

extern "C" {

int uqg_group_sort(uqg_ctx* ctx, const double* keys, int n, int S, int* order, int* groups,
                   int* pad, void* stream) {
  UQG_REQUIRE(ctx && groups && pad, "uqg_group_sort: NULL argument");
  UQG_REQUIRE(n >= 1, "cannot group an empty sample set");
  UQG_REQUIRE(S >= 1, "ensemble size must be >= 1");
  cudaStream_t s = as_stream(stream);
  int st = 0;
  int rc = uqg_status_sync(ctx, stream, &st);  // clear stale bits
  if (rc) return rc;
  rc = group_sort_impl(ctx, keys, n, S, order, groups, pad, s);
  if (rc) return rc;
  rc = uqg_status_sync(ctx, stream, &st);
  if (rc) return rc;
  UQG_REQUIRE(!(st & 2), "grouping keys must be finite");
  return UQG_OK;
}

int uqg_group_sort_async(uqg_ctx* ctx, const double* keys, int n, int S, int* order, int* groups,
                         int* pad, void* stream) {
  UQG_REQUIRE(ctx && groups && pad, "uqg_group_sort_async: NULL argument");
  UQG_REQUIRE(n >= 1, "cannot group an empty sample set");
  UQG_REQUIRE(S >= 1, "ensemble size must be >= 1");
  return group_sort_impl(ctx, keys, n, S, order, groups, pad, as_stream(stream));
}

int uqg_status_clear(uqg_ctx* ctx, void* stream) {
  UQG_REQUIRE(ctx, "uqg_status_clear: NULL ctx");
  UQG_TRY_CUDA(cudaMemsetAsync(ctx->status_dev, 0, sizeof(int), as_stream(stream)));
  return UQG_OK;
}

}  // extern "C"
