// cluster_mc_probe.cu - standalone probe (tuning tool, not part of libuqg.so) of
// the TMA-multicast cluster form of the face SpMV.
//
// The CL CTAs of a thread-block cluster take CL adjacent grid lines (m rows each)
// and walk them 16 rows per step.  For every step each CTA's elected thread
// fetches ITS line's p rows (18) and x-face rows (16) from L2 once with
// cp.async.bulk ... .multicast::cluster into the shared memory of the CTAs that
// use them: p to {c-1, c, c+1} (east / centre / west band), faces to {c-1, c}
// (east / west faces).  A stage holds three p slots (line mod 3) and two face
// slots (line mod 2), so a line's tile lands at the same offset in every
// destination.  The cluster's edge CTAs fetch their outer bands themselves.
// Per stage and CTA: a FULL mbarrier (transaction bytes of everything that lands
// in the stage) and an EMPTY mbarrier on which the warps of every CTA that the
// owner multicasts into arrive (remote mbarrier.arrive) when they are done with
// the stage - CTAs and warps run ahead of one another, no cluster-wide barrier
// in the loop.  Arithmetic = the library's row; the reduction tree and chunk
// structure are not reproduced (memory-system probe).  Every wait is bounded
// (clock64): on a protocol error the kernel sets a flag and falls through.
//
// Result (round 2, C3 shape, one B200; every variant reproduces the reference
// kernel's Ap bit for bit and no bounded wait trips):
//  * first form - thread 0 of a consumer warp also produces, release-scoped remote
//    arrives, step / unit indices by division: 1.3-2.0 TB/s (ncu: 52 % of the stall
//    samples on the membar of the releasing arrive, which waits for the warp's Ap
//    stores);
//  * relaxed remote arrives (the stage reads are complete once their values are
//    used): 2.8-3.2 TB/s;
//  * plus a dedicated producer warp (9th warp, lane 0) that runs ahead of the
//    consumers, and no divisions in the loops: CL = 2 6.20 TB/s, CL = 4 5.99,
//    CL = 8 5.59 (4 stages of 16 rows, 2 CTAs/SM); 5 stages of 32 rows, CL = 2: 6.34
//    - against 4.8 TB/s for the cyclic kernel of tools/face_run_probe.cu and 5.0 for
//    the library's kernel in the bench.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/cmp tools/cluster_mc_probe.cu
//   timeout 60 /tmp/cmp [cells=512] [G=42]        (S = 32)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t err_ = (x);                                                      \
    if (err_ != cudaSuccess) {                                                   \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(err_));        \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

struct Args {
  int m, N, G;
  const double* tx;  // [G][N + m][S]
  const double* p;   // [G][N][S]
  double* ap;        // [G][N][S]
  double* out;
  int* err;
};

constexpr int S = 32, L = 16, T = 256, NW = T / 32;
// rows per step KR (template): 16 = one tile of the library at S = 32
__host__ __device__ constexpr size_t p_slot(int kr) { return (size_t)(kr + 2) * S; }  // doubles
__host__ __device__ constexpr size_t t_slot(int kr) { return (size_t)kr * S; }
__host__ __device__ constexpr size_t stage_doubles(int kr) { return 3 * p_slot(kr) + 2 * t_slot(kr); }

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// remote arrive on the barrier at the same offset in CTA `rank`
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, unsigned rank) {
  unsigned addr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, unsigned parity, int* err) {
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > (1LL << 31)) {  // ~1 s: protocol error, never hang
      atomicExch(err, 1);
      return false;
    }
  }
  return true;
}
__device__ __forceinline__ void bulk_mc(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                        unsigned short mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void bulk_uc(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ double2 ldg2(const double* q) {
  return __ldg(reinterpret_cast<const double2*>(q));
}

__device__ __forceinline__ double row1(double tw, double te, double pw, double ps, double pc,
                                       double pn, double pe, bool w, bool s, bool n, bool e) {
  const double ay = 1.0;
  const double d = __dadd_rn(__dadd_rn(__dadd_rn(tw, te), ay), ay);
  double a = 0.0;
  if (w) a = __dadd_rn(a, __dmul_rn(-tw, pw));
  if (s) a = __dadd_rn(a, __dmul_rn(-ay, ps));
  a = __dadd_rn(a, __dmul_rn(d, pc));
  if (n) a = __dadd_rn(a, __dmul_rn(-ay, pn));
  if (e) a = __dadd_rn(a, __dmul_rn(-te, pe));
  return a;
}

// rows [lo, hi) of a tile whose slot starts at row `first`, clipped to [0, limit)
struct Span {
  int lo, n;
};
__device__ __forceinline__ Span clip(int first, int rows, int limit) {
  int lo = first < 0 ? 0 : first, hi = first + rows > limit ? limit : first + rows;
  return {lo, hi > lo ? hi - lo : 0};
}

template <int CL, int NST, int KR>
__global__ void __launch_bounds__(T + 32, KR <= 16 ? 2 : 1) spmv_mc(Args a) {
  constexpr int kRows = KR;
  constexpr size_t kPSlot = p_slot(KR), kTSlot = t_slot(KR), kStage = stage_doubles(KR);
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)NST * kStage);
  uint64_t* empty = full + NST;
  const int m = a.m, N = a.N, t = threadIdx.x, sl = t % L, rr = t / L, warp = t / 32;
  const bool producer = warp == NW;  // warps 0..NW-1 consume, lane 0 of warp NW produces
  const unsigned c = cluster_rank();
  const int n_units = (m + CL - 1) / CL;
  const int n_clusters = gridDim.x / CL, cid = blockIdx.x / CL;
  const int steps = (m + kRows - 1) / kRows;
  const bool has_w = c > 0, has_e = c + 1 < CL;
  const int n_dest = 1 + (has_w ? 1 : 0) + (has_e ? 1 : 0);  // CTAs this CTA multicasts into
  if (t == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW * n_dest);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync();
  const unsigned short pmask = (unsigned short)((1u << c) | (has_w ? 1u << (c - 1) : 0u) |
                                                (has_e ? 1u << (c + 1) : 0u));
  const unsigned short tmask = (unsigned short)((1u << c) | (has_w ? 1u << (c - 1) : 0u));
  double2 acc = make_double2(0.0, 0.0);
  int s = 0, it = 0;
  unsigned ph = 0;  // parity of the FULL phase of the current iteration
  bool ok = true;
  // units of this cluster: cid, cid + n_clusters, ... over all groups
  for (int u = cid; u < n_units * a.G && ok; u += n_clusters) {
    const int g = u / n_units;
    int l0 = (u - g * n_units) * CL;
    if (l0 + CL > m) l0 = m - CL;  // last unit of a group shifted back: every CTA has a line
    const int i = l0 + (int)c;     // this CTA's line
    const bool w = i > 0, e = i + 1 < m;
    const double* pg = a.p + (size_t)g * N * S;
    const double* txg = a.tx + (size_t)g * (N + m) * S;
    const size_t pc_slot = (size_t)(i % 3) * kPSlot, pw_slot = (size_t)((i + 2) % 3) * kPSlot,
                 pe_slot = (size_t)((i + 1) % 3) * kPSlot, tw_slot = 3 * kPSlot + (size_t)(i % 2) * kTSlot,
                 te_slot = 3 * kPSlot + (size_t)((i + 1) % 2) * kTSlot;
    if (producer) {
      // the whole warp walks the loop (aligned cluster barrier at the end); lane 0 issues
      for (int st = 0; st < steps; ++st, ++it) {
        if ((t & 31) == 0) {
          double* stage = sm + (size_t)s * kStage;
          const int j0 = st * kRows;
          const Span ps = clip(j0 - 1, kRows + 2, m), ts = clip(j0, kRows, m);
          const unsigned pb = (unsigned)ps.n * S * 8, tb = (unsigned)ts.n * S * 8;
          // bytes landing in MY stage: own p + own faces, west p, east p (if any) + east faces
          const unsigned expect = pb + tb + (w ? pb : 0u) + (e ? pb : 0u) + tb;
          if (it >= NST && !mbar_wait(&empty[s], ph ^ 1u, a.err)) ok = false;
          if (ok) {
            fence_proxy_async();
            mbar_expect_tx(&full[s], expect);
            const size_t poff = (size_t)(ps.lo - (j0 - 1)) * S, toff = (size_t)(ts.lo - j0) * S;
            bulk_mc(stage + pc_slot + poff, pg + ((size_t)i * m + ps.lo) * S, pb, &full[s], pmask);
            bulk_mc(stage + tw_slot + toff, txg + ((size_t)i * m + ts.lo) * S, tb, &full[s], tmask);
            if (!has_w && w)  // cluster's west edge: line i - 1 is nobody's
              bulk_uc(stage + pw_slot + poff, pg + ((size_t)(i - 1) * m + ps.lo) * S, pb, &full[s]);
            if (!has_e) {  // cluster's east edge: line i + 1 (p only if it exists; faces always)
              if (e)
                bulk_uc(stage + pe_slot + poff, pg + ((size_t)(i + 1) * m + ps.lo) * S, pb, &full[s]);
              bulk_uc(stage + te_slot + toff, txg + ((size_t)(i + 1) * m + ts.lo) * S, tb, &full[s]);
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
      double* apl = a.ap + (size_t)g * N * S + (size_t)i * m * S + 2 * sl;
      for (int st = 0; st < steps; ++st, ++it) {
        if (!mbar_wait(&full[s], ph, a.err)) ok = false;
        ok = __all_sync(0xffffffffu, (int)ok) != 0;
        if (!ok) break;
        const double* stage = sm + (size_t)s * kStage;
#pragma unroll
        for (int q = 0; q < kRows / 16; ++q) {
          const int jl = q * 16 + rr, j = st * kRows + jl;
          if (j < m) {
            const bool sflag = j > 0, n = j < m - 1;
            const size_t po = (size_t)(jl + 1) * S + 2 * sl, to = (size_t)jl * S + 2 * sl;
            const double2 pc = *reinterpret_cast<const double2*>(stage + pc_slot + po);
            const double2 ps = *reinterpret_cast<const double2*>(stage + pc_slot + po - S);
            const double2 pn = *reinterpret_cast<const double2*>(stage + pc_slot + po + S);
            const double2 pw = *reinterpret_cast<const double2*>(stage + pw_slot + po);
            const double2 pe = *reinterpret_cast<const double2*>(stage + pe_slot + po);
            const double2 tw = *reinterpret_cast<const double2*>(stage + tw_slot + to);
            const double2 te = *reinterpret_cast<const double2*>(stage + te_slot + to);
            double2 y;
            y.x = row1(tw.x, te.x, pw.x, ps.x, pc.x, pn.x, pe.x, w, sflag, n, e);
            y.y = row1(tw.y, te.y, pw.y, ps.y, pc.y, pn.y, pe.y, w, sflag, n, e);
            *reinterpret_cast<double2*>(apl + (size_t)j * S) = y;
            acc.x = fma(pc.x, y.x, acc.x);
            acc.y = fma(pc.y, y.y, acc.y);
          }
        }
        // this warp is done with stage s: tell every CTA that writes into my stage
        __syncwarp();
        if ((t & 31) == 0) {
          mbar_arrive_remote(&empty[s], c);
          if (has_w) mbar_arrive_remote(&empty[s], c - 1);
          if (has_e) mbar_arrive_remote(&empty[s], c + 1);
        }
        if (++s == NST) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  }
  if (!producer) a.out[(size_t)blockIdx.x * T + t] = acc.x + acc.y;
  cluster_sync();  // nobody exits while a neighbour may still arrive on its barriers
}

__global__ void spmv_ref(Args a) {
  const int m = a.m, N = a.N;
  const int g = blockIdx.y;
  const double* pg = a.p + (size_t)g * N * S;
  const double* txg = a.tx + (size_t)g * (N + m) * S;
  double* apg = a.ap + (size_t)g * N * S;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < (long long)N * L;
       v += (long long)gridDim.x * blockDim.x) {
    const long long row = v / L;
    const int sl = (int)(v % L), i = (int)(row / m), j = (int)(row - (long long)i * m);
    const bool w = i > 0, s = j > 0, n = j < m - 1, e = i < m - 1;
    const double2 z = make_double2(0, 0);
    const double2 tw = ldg2(txg + row * S + 2 * sl), te = ldg2(txg + (row + m) * S + 2 * sl);
    const double2 pc = ldg2(pg + row * S + 2 * sl);
    const double2 pw = w ? ldg2(pg + (row - m) * S + 2 * sl) : z;
    const double2 pe = e ? ldg2(pg + (row + m) * S + 2 * sl) : z;
    const double2 ps = s ? ldg2(pg + (row - 1) * S + 2 * sl) : z;
    const double2 pn = n ? ldg2(pg + (row + 1) * S + 2 * sl) : z;
    double2 y;
    y.x = row1(tw.x, te.x, pw.x, ps.x, pc.x, pn.x, pe.x, w, s, n, e);
    y.y = row1(tw.y, te.y, pw.y, ps.y, pc.y, pn.y, pe.y, w, s, n, e);
    *reinterpret_cast<double2*>(apg + row * S + 2 * sl) = y;
  }
}

__global__ void fill(double* a, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u + seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    a[i] = 0.5 + (double)(h & 0xffffff) / 16777216.0;
  }
}

__global__ void diff(const double* x, const double* y, size_t n, unsigned long long* bad) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    if (x[i] != y[i]) atomicAdd(bad, 1ull);
}

template <int CL, int NST, int KR>
float run(const Args& a, int reps, bool* ok) {
  const size_t smem = (size_t)NST * stage_doubles(KR) * 8 + 2 * NST * 8;
  auto kern = spmv_mc<CL, NST, KR>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(T + 32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(148 * 2 / CL * CL);
  int maxc = 0;
  if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    maxc = 0;
  }
  if (maxc < 1) {
    *ok = false;
    return 0.f;
  }
  const int grid = maxc * CL;  // every cluster resident
  cfg.gridDim = dim3(grid);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaLaunchKernelEx(&cfg, kern, a));
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) CK(cudaLaunchKernelEx(&cfg, kern, a));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  *ok = true;
  printf("  [CL %d, %d stages of %d rows: grid %d CTAs, %zu B smem, %d clusters resident]", CL, NST,
         KR, grid, smem, maxc);
  return ms / reps;
}

int main(int argc, char** argv) {
  const int cells = argc > 1 ? atoi(argv[1]) : 512;
  const int G = argc > 2 ? atoi(argv[2]) : 42;
  Args a;
  a.m = cells - 1;
  a.N = a.m * a.m;
  a.G = G;
  const size_t nt = (size_t)G * (a.N + a.m) * S, nv = (size_t)G * a.N * S;
  double *tx, *p, *ap, *ap_ref, *out;
  int* err;
  CK(cudaMalloc(&tx, nt * 8));
  CK(cudaMalloc(&p, nv * 8));
  CK(cudaMalloc(&ap, nv * 8));
  CK(cudaMalloc(&ap_ref, nv * 8));
  CK(cudaMalloc(&out, (size_t)148 * 8 * T * 8));
  CK(cudaMalloc(&err, 4));
  CK(cudaMemset(err, 0, 4));
  fill<<<1184, 256>>>(tx, nt, 1u);
  fill<<<1184, 256>>>(p, nv, 2u);
  CK(cudaMemset(ap, 0, nv * 8));
  a.tx = tx;
  a.p = p;
  a.out = out;
  a.err = err;
  a.ap = ap_ref;
  spmv_ref<<<dim3(296, G), 256>>>(a);
  CK(cudaDeviceSynchronize());
  a.ap = ap;
  const double bytes = 8.0 * S * G * ((double)(a.N + a.m) + 2.0 * a.N);
  unsigned long long* bad;
  CK(cudaMalloc(&bad, 8));
  printf("cells %d S %d G %d: m %d\n", cells, S, G, a.m);
  auto check = [&]() {
    CK(cudaMemset(bad, 0, 8));
    diff<<<1184, 256>>>(ap, ap_ref, nv, bad);
    unsigned long long h = 0;
    int herr = 0;
    CK(cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost));
    printf("  check: %llu of %zu Ap entries differ from the reference kernel; protocol error flag %d\n",
           h, nv, herr);
    CK(cudaMemset(ap, 0, nv * 8));
    CK(cudaMemset(err, 0, 4));
  };
  bool ok;
  float ms;
#define RUN(CLV, NSTV, KRV)                                                              \
  ms = run<CLV, NSTV, KRV>(a, 10, &ok);                                                  \
  if (ok) {                                                                              \
    printf(" %.3f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);                               \
    check();                                                                             \
  }
  RUN(2, 4, 16) RUN(4, 4, 16) RUN(8, 4, 16) RUN(2, 4, 32) RUN(4, 4, 32) RUN(2, 5, 32)
  return 0;
}
