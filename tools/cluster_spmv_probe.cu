// cluster_spmv_probe.cu - standalone probe (tuning tool, not part of libuqg.so)
// of the cluster form of the face SpMV: the CL CTAs of a
// thread-block cluster take CL adjacent grid lines (m rows each) and walk them in
// lockstep, 64 rows per step.  Each CTA stages only its OWN line's p rows and
// x-faces of the step in shared memory (cp.async, 3 stages); the west / east
// neighbours' values - p[row - m], p[row + m], tx[row + m] - are read from the
// neighbouring CTAs' shared memory over DSMEM (ld.shared::cluster), so every p
// row and face row crosses L2 -> SM once per cluster (the cluster's two edge
// lines read their outer bands from global memory).  One cluster barrier per
// step.  Arithmetic = the library's row (CSR order, separate roundings, fused
// p.Ap accumulation per thread); the reduction tree and the chunk structure of
// the library are NOT reproduced: this measures the memory system only.
//
// Result (round 2, C3 shape, one B200): every variant reproduces the reference
// kernel's Ap bit for bit, and none is competitive - 2 CTAs/SM, 256 threads: CL = 2
// 2.64 TB/s, 4 2.61, 8 2.56, 16 2.21 (rows processed one by one); with the
// thread's rows' loads issued together 2.26 / 2.09 / 1.95; 512 threads per CTA
// 2.58 / 2.25 / 2.09 - against 5.0 TB/s for the library's kernel.  A step takes
// ~5.5 us per CTA where its copies need ~2: with one cluster barrier per step all
// warps of a CTA are in the same phase (wait, DSMEM loads, math, store) at the same
// time, so nothing hides the DSMEM latency and the barrier skew.  A competitive
// cluster form needs per-stage full/empty barriers across the CTAs (so that
// CTAs run ahead of one another) and TMA multicast instead of DSMEM reads.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/csp tools/cluster_spmv_probe.cu
//   timeout 60 /tmp/csp [cells=512] [S=32] [G=42]
#include <cuda_runtime.h>
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
  int m, N, S, G;
  const double* tx;  // [G][N + m][S]
  const double* p;   // [G][N][S]
  double* ap;        // [G][N][S]
  double* out;       // per-thread accumulators (keeps the sums alive)
};

constexpr int kRows = 64;  // rows per step
constexpr int kNst = 3;    // stages

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared-memory location in CTA `rank` of the cluster
__device__ __forceinline__ unsigned map_rank(const void* p, unsigned rank) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
__device__ __forceinline__ double2 ld_dsmem(unsigned addr) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
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

// Stage layout (doubles): p rows j0-1 .. j0+kRows (kRows + 2 rows), then tx rows
// j0 .. j0+kRows-1 (the line's west faces; the east faces of line i are the
// west faces of line i + 1).
template <int CL, int T, int L>
__global__ void __launch_bounds__(T, 2) spmv_cluster(Args a, int lines_per_group) {
  extern __shared__ __align__(16) double sm[];
  const int S = a.S, m = a.m, N = a.N;
  constexpr int R = T / L, NR = kRows / R;  // rows per thread and step
  const int t = threadIdx.x, sl = t % L, rr = t / L;
  const unsigned crank = cluster_rank();
  const int n_units = (lines_per_group + CL - 1) / CL;  // cluster units per group
  const int n_clusters = gridDim.x / CL, cid = blockIdx.x / CL;
  const size_t prow = (size_t)(kRows + 2) * S, stage_d = prow + (size_t)kRows * S;
  const int steps = (m + kRows - 1) / kRows;
  double2 acc = make_double2(0.0, 0.0);
  for (int u = cid; u < n_units * a.G; u += n_clusters) {
    const int g = u / n_units, i = (u - g * n_units) * CL + (int)crank;  // this CTA's line
    const bool live = i < m;  // the last unit of a group may be short
    const double* pg = a.p + (size_t)g * N * S;
    const double* txg = a.tx + (size_t)g * (N + m) * S;
    double* apg = a.ap + (size_t)g * N * S;
    const long long line0 = (long long)i * m;  // first row of the line
    auto issue = [&](int st) {
      if (!live) return;
      double* buf = sm + (size_t)(st % kNst) * stage_d;
      const int j0 = st * kRows;
      // p rows j0-1 .. j0+kRows of the line (clipped to the line's own rows)
      const int lo = j0 - 1 < 0 ? 0 : j0 - 1, hi = j0 + kRows + 1 > m ? m : j0 + kRows + 1;
      const int nvec = (hi - lo) * L;  // 16-byte pieces
      for (int v = t; v < nvec; v += T) {
        const int r = lo + v / L, c = v % L;
        cp16(buf + (size_t)(r - (j0 - 1)) * S + 2 * c, pg + (line0 + r) * S + 2 * c);
      }
      const int thi = j0 + kRows > m ? m : j0 + kRows;
      const int tvec = (thi - j0) * L;
      for (int v = t; v < tvec; v += T) {
        const int r = j0 + v / L, c = v % L;
        cp16(buf + prow + (size_t)(r - j0) * S + 2 * c, txg + (line0 + r) * S + 2 * c);
      }
    };
    // prologue: two steps in flight
    issue(0);
    cp_commit();
    if (steps > 1) issue(1);
    cp_commit();
    for (int st = 0; st < steps; ++st) {
      cp_wait<1>();      // this CTA's copies of step st have landed
      cluster_sync();    // ... and everybody's; everybody is done with step st - 1
      if (st + 2 < steps) issue(st + 2);
      cp_commit();
      if (live) {
        const double* buf = sm + (size_t)(st % kNst) * stage_d;
        const unsigned west = map_rank(buf, crank > 0 ? crank - 1 : 0);
        const unsigned east = map_rank(buf, crank + 1 < CL ? crank + 1 : crank);
        const bool w = i > 0, e = i < m - 1;
        const bool w_in = crank > 0, e_in = crank + 1 < CL && i + 1 < m;
        const int j0 = st * kRows;
        // all loads of the thread's NR rows first (local, DSMEM and edge-global), then the math
        double2 pc[NR], ps[NR], pn[NR], tw[NR], pw[NR], pe[NR], te[NR];
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int jl = q * R + rr, j = j0 + jl;
          pw[q] = pe[q] = te[q] = make_double2(0, 0);
          if (j < m) {
            const long long row = line0 + j;
            const size_t po = (size_t)(jl + 1) * S + 2 * sl;
            const size_t to = prow + (size_t)jl * S + 2 * sl;
            pc[q] = *reinterpret_cast<const double2*>(buf + po);
            ps[q] = *reinterpret_cast<const double2*>(buf + po - S);
            pn[q] = *reinterpret_cast<const double2*>(buf + po + S);
            tw[q] = *reinterpret_cast<const double2*>(buf + to);
            if (w) pw[q] = w_in ? ld_dsmem(west + (unsigned)(po * 8)) : ldg2(pg + (row - m) * S + 2 * sl);
            if (e_in) {
              pe[q] = ld_dsmem(east + (unsigned)(po * 8));
              te[q] = ld_dsmem(east + (unsigned)(to * 8));
            } else {
              if (e) pe[q] = ldg2(pg + (row + m) * S + 2 * sl);
              te[q] = ldg2(txg + (row + m) * S + 2 * sl);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const int jl = q * R + rr, j = j0 + jl;
          if (j < m) {
            const bool s = j > 0, n = j < m - 1;
            const long long row = line0 + j;
            double2 y;
            y.x = row1(tw[q].x, te[q].x, pw[q].x, ps[q].x, pc[q].x, pn[q].x, pe[q].x, w, s, n, e);
            y.y = row1(tw[q].y, te[q].y, pw[q].y, ps[q].y, pc[q].y, pn[q].y, pe[q].y, w, s, n, e);
            *reinterpret_cast<double2*>(apg + row * S + 2 * sl) = y;
            acc.x = fma(pc[q].x, y.x, acc.x);
            acc.y = fma(pc[q].y, y.y, acc.y);
          }
        }
      }
    }
    cp_wait<0>();
    cluster_sync();  // nobody still reads this unit's stages when the next unit refills them
  }
  a.out[(size_t)blockIdx.x * T + t] = acc.x + acc.y;
}

// reference: straightforward global-memory kernel, same arithmetic (for checking Ap)
__global__ void spmv_ref(Args a) {
  const int S = a.S, m = a.m, N = a.N, L = S / 2;
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

template <int CL, int T>
float run(const Args& a, int ctas_per_sm, int reps, bool* ok) {
  auto kern = spmv_cluster<CL, T, 16>;  // S = 32 only
  const size_t smem = (size_t)kNst * ((size_t)(kRows + 2) + kRows) * a.S * 8;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  int grid = 148 * ctas_per_sm;
  grid -= grid % CL;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(T);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int maxc = 0;
  if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    maxc = -1;
  }
  if (maxc >= 0 && maxc * CL < grid) {  // all clusters must be co-resident? no - but keep one wave
    grid = maxc * CL;
    cfg.gridDim = dim3(grid);
  }
  if (grid < CL) {
    *ok = false;
    return 0.f;
  }
  const int lines = a.m;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaLaunchKernelEx(&cfg, kern, a, lines));
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) CK(cudaLaunchKernelEx(&cfg, kern, a, lines));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  *ok = true;
  printf("  [CL %d T %d: grid %d CTAs, %zu B smem, max active clusters %d]", CL, T, grid, smem, maxc);
  return ms / reps;
}

int main(int argc, char** argv) {
  const int cells = argc > 1 ? atoi(argv[1]) : 512;
  const int S = argc > 2 ? atoi(argv[2]) : 32;
  const int G = argc > 3 ? atoi(argv[3]) : 42;
  Args a;
  a.m = cells - 1;
  a.N = a.m * a.m;
  a.S = S;
  a.G = G;
  const size_t nt = (size_t)G * (a.N + a.m) * S, nv = (size_t)G * a.N * S;
  double *tx, *p, *ap, *ap_ref, *out;
  CK(cudaMalloc(&tx, nt * 8));
  CK(cudaMalloc(&p, nv * 8));
  CK(cudaMalloc(&ap, nv * 8));
  CK(cudaMalloc(&ap_ref, nv * 8));
  CK(cudaMalloc(&out, (size_t)148 * 8 * 512 * 8));
  fill<<<1184, 256>>>(tx, nt, 1u);
  fill<<<1184, 256>>>(p, nv, 2u);
  CK(cudaMemset(ap, 0, nv * 8));
  a.tx = tx;
  a.p = p;
  a.out = out;
  a.ap = ap_ref;
  spmv_ref<<<dim3(296, G), 256>>>(a);
  CK(cudaDeviceSynchronize());
  a.ap = ap;
  const double bytes = 8.0 * S * G * ((double)(a.N + a.m) + 2.0 * a.N);
  unsigned long long* bad;
  CK(cudaMalloc(&bad, 8));
  printf("cells %d S %d G %d: m %d, %d steps of %d rows per line\n", cells, S, G, a.m,
         (a.m + kRows - 1) / kRows, kRows);
  auto check = [&](const char* name) {
    CK(cudaMemset(bad, 0, 8));
    diff<<<1184, 256>>>(ap, ap_ref, nv, bad);
    unsigned long long h = 0;
    CK(cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost));
    printf("  %s: %llu of %zu Ap entries differ from the reference kernel\n", name, h, nv);
    CK(cudaMemset(ap, 0, nv * 8));
  };
  bool ok;
  float ms;
  if (S != 32) {
    printf("this probe is instantiated for S = 32\n");
    return 1;
  }
#define RUN(CLV, TV)                                                                     \
  ms = run<CLV, TV>(a, 2, 10, &ok);                                                      \
  if (ok) printf(" CL %d, T %d: %.3f ms  %.0f GB/s\n", CLV, TV, ms, bytes / ms / 1e6), check("check");
  RUN(2, 256) RUN(4, 256) RUN(8, 256) RUN(2, 512) RUN(4, 512) RUN(8, 512)
  return 0;
}
