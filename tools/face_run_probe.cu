// face_run_probe.cu - standalone probe (tuning tool, not part of libuqg.so):
// does the face-form SpMV gain from giving each thread a RUN of consecutive
// rows of a reduction chunk (p[row-1], p[row], p[row+1] carried in registers:
// 5 loads per row instead of 7) instead of the library's cyclic rows
// rr, rr+R, rr+2R, ...?  Same chunks, same batched in-block tree, same exact
// CSR-order arithmetic as the library kernel; only the row -> thread map and
// the register carry differ.  Reports algorithmic GB/s (faces + p read, Ap
// write) and where the blocks of the 4-CTA/SM grid are placed.
//
// Result (round 2, C3 shape, one B200; profiles/r02_ncu_spmv_runmap.md): in
// this probe run+carry beats the probe's cyclic kernel (5.26 vs 4.80 TB/s),
// but the library's cyclic kernel is already at 5.0-5.5 TB/s (its 3 p-column
// loads of a tile are L1 hits: 303 M L2 sectors per launch), while a run map
// gets no L1 hits at all (398 M L2 sectors, 16% more DRAM reads).  Built into
// the library (all four p.Ap kernels moved to the run map, bit-identical to
// one another, GPU suite green) the C3 level went 10.53 -> 10.66 s, so the
// cyclic map stays.
//
// Also here: probe_il<KI>, KI ADJACENT chunks per block interleaved tile by tile
// (cyclic map, one accumulator per chunk; the east band of chunk c is the
// centre band of chunk c+1 and the west band of c+2, so those re-reads could be
// L1 hits).  C3 shape, 14 blocks per group: cyclic 4,805, KI = 1 4,768, 2 4,902,
// 4 3,827, 8 4,212 GB/s; C2 shape: slower for every KI > 1.  Not adopted.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/frp tools/face_run_probe.cu
//   /tmp/frp [cells=512] [S=32] [G=42] [random=1] [x] [ncu-mode]
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));           \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

struct Args {
  int m, N, S, G;
  const double* tx;
  const double* p;
  double* ap;
};

__device__ __forceinline__ double2 ld2(const double* q) {
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

// MAP 0: the library's cyclic map (row = base + rr + k R), 7 loads per row.
// MAP 1: run map (row = base + rr*CT + k), 7 loads per row (no carry).
// MAP 2: run map with the +-1 neighbours carried in registers, 5 loads per row.
// MAP 3: run map, carry, two rows per step (10 loads issued together).
template <int MAP, int MINB>
__global__ void __launch_bounds__(256, MINB) probe(Args a, int CT, double* part,
                                                   unsigned* ticket) {
  extern __shared__ double red[];
  const int S = a.S, m = a.m, N = a.N, L = S / 2, Lp = L, T = 256, R = T / Lp;
  const int tiles = (N + R - 1) / R, chunks = (tiles + CT - 1) / CT;
  const int g = blockIdx.y, B = gridDim.x, t = threadIdx.x;
  const int sl = t % Lp, rr = t / Lp;
  const double* txg = a.tx + (size_t)g * (N + m) * S + 2 * sl;
  const double* pg = a.p + (size_t)g * N * S + 2 * sl;
  double* apg = a.ap + (size_t)g * N * S + 2 * sl;
  for (int c0 = blockIdx.x; c0 < chunks; c0 += 8 * B) {
    int nk = (chunks - 1 - c0) / B + 1;
    if (nk > 8) nk = 8;
    for (int k = 0; k < nk; ++k) {
      const int chunk = c0 + k * B;
      double2 acc = make_double2(0.0, 0.0);
      const int cbase = chunk * CT * R;
      int cend = cbase + CT * R;
      if (cend > N) cend = N;
      if (MAP == 0) {
        int row = cbase + rr;
        int i0 = row / m, j0 = row - i0 * m;
        for (; row < cend; row += R) {
          const bool w = i0 > 0, s = j0 > 0, n = j0 < m - 1, e = i0 < m - 1;
          const double2 tw = ld2(txg + row * S), te = ld2(txg + (row + m) * S),
                        pc = ld2(pg + row * S);
          double2 pw = make_double2(0, 0), pe = pw, ps = pw, pn = pw;
          if (w) pw = ld2(pg + (row - m) * S);
          if (e) pe = ld2(pg + (row + m) * S);
          if (s) ps = ld2(pg + (row - 1) * S);
          if (n) pn = ld2(pg + (row + 1) * S);
          double2 y;
          y.x = row1(tw.x, te.x, pw.x, ps.x, pc.x, pn.x, pe.x, w, s, n, e);
          y.y = row1(tw.y, te.y, pw.y, ps.y, pc.y, pn.y, pe.y, w, s, n, e);
          *reinterpret_cast<double2*>(apg + row * S) = y;
          acc.x = fma(pc.x, y.x, acc.x);
          acc.y = fma(pc.y, y.y, acc.y);
          j0 += R;  // as the library kernel: no division per row
          while (j0 >= m) {
            j0 -= m;
            ++i0;
          }
        }
      } else {
        int row = cbase + rr * CT, rend = row + CT;
        if (rend > cend) rend = cend;
        if (row < rend) {
          int i0 = row / m, j0 = row - i0 * m;
          if (MAP == 1) {
            for (; row < rend; ++row) {
              const bool w = i0 > 0, s = j0 > 0, n = j0 < m - 1, e = i0 < m - 1;
              const double2 tw = ld2(txg + row * S), te = ld2(txg + (row + m) * S),
                            pc = ld2(pg + row * S);
              double2 pw = make_double2(0, 0), pe = pw, ps = pw, pn = pw;
              if (w) pw = ld2(pg + (row - m) * S);
              if (e) pe = ld2(pg + (row + m) * S);
              if (s) ps = ld2(pg + (row - 1) * S);
              if (n) pn = ld2(pg + (row + 1) * S);
              double2 y;
              y.x = row1(tw.x, te.x, pw.x, ps.x, pc.x, pn.x, pe.x, w, s, n, e);
              y.y = row1(tw.y, te.y, pw.y, ps.y, pc.y, pn.y, pe.y, w, s, n, e);
              *reinterpret_cast<double2*>(apg + row * S) = y;
              acc.x = fma(pc.x, y.x, acc.x);
              acc.y = fma(pc.y, y.y, acc.y);
              if (++j0 == m) {
                j0 = 0;
                ++i0;
              }
            }
          } else if (MAP == 2) {
            double2 ps = make_double2(0, 0), pc = ld2(pg + row * S);
            if (row > 0) ps = ld2(pg + (row - 1) * S);
            for (; row < rend; ++row) {
              const bool w = i0 > 0, s = j0 > 0, n = j0 < m - 1, e = i0 < m - 1;
              const double2 tw = ld2(txg + row * S), te = ld2(txg + (row + m) * S);
              double2 pw = make_double2(0, 0), pe = pw, pn = pw;
              if (row + 1 < N) pn = ld2(pg + (row + 1) * S);
              if (w) pw = ld2(pg + (row - m) * S);
              if (e) pe = ld2(pg + (row + m) * S);
              double2 y;
              y.x = row1(tw.x, te.x, pw.x, ps.x, pc.x, pn.x, pe.x, w, s, n, e);
              y.y = row1(tw.y, te.y, pw.y, ps.y, pc.y, pn.y, pe.y, w, s, n, e);
              *reinterpret_cast<double2*>(apg + row * S) = y;
              acc.x = fma(pc.x, y.x, acc.x);
              acc.y = fma(pc.y, y.y, acc.y);
              ps = pc;
              pc = pn;
              if (++j0 == m) {
                j0 = 0;
                ++i0;
              }
            }
          } else {  // MAP 3: two rows per step
            double2 ps = make_double2(0, 0), pc = ld2(pg + row * S);
            if (row > 0) ps = ld2(pg + (row - 1) * S);
            for (; row < rend; row += 2) {
              const bool two = row + 1 < rend;
              const bool w = i0 > 0, s = j0 > 0, n = j0 < m - 1, e = i0 < m - 1;
              int i1 = i0, j1 = j0 + 1;
              if (j1 == m) {
                j1 = 0;
                ++i1;
              }
              const bool w1 = i1 > 0, s1 = j1 > 0, n1 = j1 < m - 1, e1 = i1 < m - 1;
              const double2 z = make_double2(0, 0);
              const double2 tw = ld2(txg + row * S), te = ld2(txg + (row + m) * S);
              double2 pw = z, pe = z, pn = z, pw1 = z, pe1 = z, pn1 = z, tw1 = z, te1 = z;
              if (row + 1 < N) pn = ld2(pg + (row + 1) * S);
              if (w) pw = ld2(pg + (row - m) * S);
              if (e) pe = ld2(pg + (row + m) * S);
              if (two) {
                tw1 = ld2(txg + (row + 1) * S);
                te1 = ld2(txg + (row + 1 + m) * S);
                if (row + 2 < N) pn1 = ld2(pg + (row + 2) * S);
                if (w1) pw1 = ld2(pg + (row + 1 - m) * S);
                if (e1) pe1 = ld2(pg + (row + 1 + m) * S);
              }
              double2 y;
              y.x = row1(tw.x, te.x, pw.x, ps.x, pc.x, pn.x, pe.x, w, s, n, e);
              y.y = row1(tw.y, te.y, pw.y, ps.y, pc.y, pn.y, pe.y, w, s, n, e);
              *reinterpret_cast<double2*>(apg + row * S) = y;
              acc.x = fma(pc.x, y.x, acc.x);
              acc.y = fma(pc.y, y.y, acc.y);
              if (two) {
                y.x = row1(tw1.x, te1.x, pw1.x, pc.x, pn.x, pn1.x, pe1.x, w1, s1, n1, e1);
                y.y = row1(tw1.y, te1.y, pw1.y, pc.y, pn.y, pn1.y, pe1.y, w1, s1, n1, e1);
                *reinterpret_cast<double2*>(apg + (row + 1) * S) = y;
                acc.x = fma(pn.x, y.x, acc.x);
                acc.y = fma(pn.y, y.y, acc.y);
              }
              ps = pn;
              pc = pn1;
              i0 = i1;
              j0 = j1 + 1;
              if (j0 == m) {
                j0 = 0;
                ++i0;
              }
            }
          }
        }
      }
      red[(2 * k) * T + t] = acc.x;
      red[(2 * k + 1) * T + t] = acc.y;
    }
    __syncthreads();
    for (int st = R >> 1; st > 0; st >>= 1) {
      if (rr < st)
        for (int v = 0; v < 2 * nk; ++v) red[v * T + t] += red[v * T + t + st * Lp];
      __syncthreads();
    }
    if (t < L)
      for (int k = 0; k < nk; ++k)
        part[((size_t)g * chunks + c0 + k * B) * S + 2 * t] = red[(2 * k) * T + t];
    __threadfence();
    __syncthreads();
    if (t == 0) atomicAdd(&ticket[g], (unsigned)nk);
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


// KI adjacent chunks per block, interleaved tile by tile (cyclic map, per-chunk
// accumulators): the east band of chunk c is the centre band of chunk c+1 and
// the west band of chunk c+2, so with the chunks on one SM those re-reads can
// be L1 hits instead of L2 sectors.  Same chunk partials as MAP 0.
template <int KI>
__global__ void __launch_bounds__(256, 4) probe_il(Args a, int CT, double* part,
                                                   unsigned* ticket) {
  extern __shared__ double red[];
  const int S = a.S, m = a.m, N = a.N, L = S / 2, Lp = L, T = 256, R = T / Lp;
  const int tiles = (N + R - 1) / R, chunks = (tiles + CT - 1) / CT;
  const int units = (chunks + KI - 1) / KI;
  constexpr int UB = 8 / KI;  // units per batched tree (8 chunks)
  const int g = blockIdx.y, B = gridDim.x, t = threadIdx.x;
  const int sl = t % Lp, rr = t / Lp;
  const double* txg = a.tx + (size_t)g * (N + m) * S + 2 * sl;
  const double* pg = a.p + (size_t)g * N * S + 2 * sl;
  double* apg = a.ap + (size_t)g * N * S + 2 * sl;
  const int crows = CT * R;
  for (int u0 = blockIdx.x; u0 < units; u0 += UB * B) {
    int nu = (units - 1 - u0) / B + 1;
    if (nu > UB) nu = UB;
    for (int j = 0; j < nu; ++j) {
      const int c_first = (u0 + j * B) * KI;
      double2 acc[KI];
#pragma unroll
      for (int kk = 0; kk < KI; ++kk) acc[kk] = make_double2(0.0, 0.0);
      int row0 = c_first * crows + rr;
      int i0 = row0 / m, j0 = row0 - i0 * m;
      for (int tl = 0; tl < CT; ++tl) {
        int ik = i0, jk = j0;
#pragma unroll
        for (int kk = 0; kk < KI; ++kk) {
          const int row = row0 + kk * crows;
          int cend = (c_first + kk + 1) * crows;
          if (cend > N) cend = N;
          if (row < cend) {
            const bool w = ik > 0, s = jk > 0, n = jk < m - 1, e = ik < m - 1;
            const double2 z = make_double2(0, 0);
            const double2 tw = ld2(txg + row * S), te = ld2(txg + (row + m) * S);
            double2 pw = z, ps = z, pn = z, pe = z;
            if (w) pw = ld2(pg + (row - m) * S);
            if (s) ps = ld2(pg + (row - 1) * S);
            const double2 pc = ld2(pg + row * S);
            if (n) pn = ld2(pg + (row + 1) * S);
            if (e) pe = ld2(pg + (row + m) * S);
            double2 y;
            y.x = row1(tw.x, te.x, pw.x, ps.x, pc.x, pn.x, pe.x, w, s, n, e);
            y.y = row1(tw.y, te.y, pw.y, ps.y, pc.y, pn.y, pe.y, w, s, n, e);
            *reinterpret_cast<double2*>(apg + row * S) = y;
            acc[kk].x = fma(pc.x, y.x, acc[kk].x);
            acc[kk].y = fma(pc.y, y.y, acc[kk].y);
          }
          jk += crows;
          while (jk >= m) {
            jk -= m;
            ++ik;
          }
        }
        row0 += R;
        j0 += R;
        while (j0 >= m) {
          j0 -= m;
          ++i0;
        }
      }
#pragma unroll
      for (int kk = 0; kk < KI; ++kk) {
        red[(2 * (j * KI + kk)) * T + t] = acc[kk].x;
        red[(2 * (j * KI + kk) + 1) * T + t] = acc[kk].y;
      }
    }
    __syncthreads();
    for (int st = R >> 1; st > 0; st >>= 1) {
      if (rr < st)
        for (int v = 0; v < 2 * nu * KI; ++v) red[v * T + t] += red[v * T + t + st * Lp];
      __syncthreads();
    }
    if (t < L)
      for (int j = 0; j < nu; ++j)
        for (int kk = 0; kk < KI; ++kk) {
          const int c = (u0 + j * B) * KI + kk;
          if (c < chunks) part[((size_t)g * chunks + c) * S + 2 * t] = red[(2 * (j * KI + kk)) * T + t];
        }
    __threadfence();
    __syncthreads();
    if (t == 0) atomicAdd(&ticket[g], (unsigned)nu);
  }
}

template <int KI>
float run_il(const Args& a, int CT, int bpg, int reps, double* part, unsigned* ticket) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  dim3 grid(bpg, a.G);
  const size_t smem = 16 * 256 * 8;
  probe_il<KI><<<grid, 256, smem>>>(a, CT, part, ticket);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) probe_il<KI><<<grid, 256, smem>>>(a, CT, part, ticket);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

template <int MAP, int MINB>
float run(const Args& a, int CT, int bpg, int reps, double* part, unsigned* ticket) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  dim3 grid(bpg, a.G);
  const size_t smem = 16 * 256 * 8;
  probe<MAP, MINB><<<grid, 256, smem>>>(a, CT, part, ticket);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) probe<MAP, MINB><<<grid, 256, smem>>>(a, CT, part, ticket);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

// which SM each block of a (bpg, G) grid of the probe's shape lands on
__global__ void __launch_bounds__(256, 4) where(int* smid) {
  extern __shared__ double red[];
  if (threadIdx.x == 0) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    smid[blockIdx.y * gridDim.x + blockIdx.x] = (int)s;
    red[0] = 0.0;
  }
  // stay resident long enough for the whole grid to be placed
  const long long t0 = clock64();
  while (clock64() - t0 < 2000000) {
  }
}

template <int MAP, int MINB>
int slots() {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, probe<MAP, MINB>, 256, 16 * 256 * 8);
  return per;
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
  double *tx, *p, *ap;
  CK(cudaMalloc(&tx, nt * 8));
  CK(cudaMalloc(&p, nv * 8));
  CK(cudaMalloc(&ap, nv * 8));
  if (argc > 4 && atoi(argv[4]) == 0) {  // all-zero inputs
    CK(cudaMemset(tx, 0, nt * 8));
    CK(cudaMemset(p, 0, nv * 8));
  } else {
    fill<<<1184, 256>>>(tx, nt, 1u);
    fill<<<1184, 256>>>(p, nv, 2u);
    CK(cudaDeviceSynchronize());
  }
  a.tx = tx;
  a.p = p;
  a.ap = ap;
  const double bytes = 8.0 * S * G * ((double)(a.N + a.m) + 2.0 * a.N);
  double* part;
  unsigned* ticket;
  CK(cudaMalloc(&part, (size_t)G * 4096 * 256 * 8));
  CK(cudaMalloc(&ticket, G * sizeof(unsigned)));
  CK(cudaMemset(ticket, 0, G * sizeof(unsigned)));
  const int L = S / 2, R = 256 / L, tiles = (a.N + R - 1) / R;
  int ct = tiles / 64;
  ct = ct < 1 ? 1 : (ct > 8 ? 8 : ct);
  if ((tiles + ct - 1) / ct > 512) ct = (tiles + 511) / 512;
  const int chunks = (tiles + ct - 1) / ct;
  printf("cells %d S %d G %d: R %d, chunks of %d tiles (%d rows), %d chunks\n", cells, S, G, R,
         ct, ct * R, chunks);
  printf("resident CTAs/SM: map0 %d map1 %d map2 %d map3@4 %d map3@3 %d map3@2 %d\n",
         slots<0, 4>(), slots<1, 4>(), slots<2, 4>(), slots<3, 4>(), slots<3, 3>(), slots<3, 2>());
  if (argc > 6) {  // interleave mode: adjacent chunks per block, tile-interleaved
    for (int bpg : {12, 13, 14, 16}) {
      printf("blocks/group %2d: cyclic %.0f", bpg, bytes / run<0, 4>(a, ct, bpg, 10, part, ticket) / 1e6);
      printf("  il1 %.0f", bytes / run_il<1>(a, ct, bpg, 10, part, ticket) / 1e6);
      printf("  il2 %.0f", bytes / run_il<2>(a, ct, bpg, 10, part, ticket) / 1e6);
      printf("  il4 %.0f", bytes / run_il<4>(a, ct, bpg, 10, part, ticket) / 1e6);
      printf("  il8 %.0f GB/s\n", bytes / run_il<8>(a, ct, bpg, 10, part, ticket) / 1e6);
    }
    return 0;
  }
  if (argc > 5) {  // ncu mode: cyclic and run+carry only, 4 CTAs/SM, 2 launches each
    int bpg = 148 * 4 / G;
    if (bpg > chunks) bpg = chunks;
    printf("cyclic %.0f", bytes / run<0, 4>(a, ct, bpg, 1, part, ticket) / 1e6);
    printf("  run+carry %.0f GB/s\n", bytes / run<2, 4>(a, ct, bpg, 1, part, ticket) / 1e6);
    return 0;
  }
  // blocks per group: fill 148 SMs x resident CTAs with no partial wave
  for (int per = 2; per <= 4; ++per) {
    int bpg = 148 * per / G;
    if (bpg < 1) bpg = 1;
    if (bpg > chunks) bpg = chunks;
    printf("blocks/group %3d:", bpg);
    printf("  cyclic %.0f", bytes / run<0, 4>(a, ct, bpg, 20, part, ticket) / 1e6);
    printf("  run %.0f", bytes / run<1, 4>(a, ct, bpg, 20, part, ticket) / 1e6);
    printf("  run+carry %.0f", bytes / run<2, 4>(a, ct, bpg, 20, part, ticket) / 1e6);
    printf("  carry2@4 %.0f", bytes / run<3, 4>(a, ct, bpg, 20, part, ticket) / 1e6);
    printf("  carry2@3 %.0f", bytes / run<3, 3>(a, ct, bpg, 20, part, ticket) / 1e6);
    printf("  carry2@2 %.0f GB/s\n", bytes / run<3, 2>(a, ct, bpg, 20, part, ticket) / 1e6);
  }
  {  // block placement of the 4-CTA/SM grid
    const int bpg = 148 * 4 / G, nb = bpg * G;
    int* d;
    CK(cudaMalloc(&d, nb * sizeof(int)));
    where<<<dim3(bpg, G), 256, 16 * 256 * 8>>>(d);
    CK(cudaDeviceSynchronize());
    int* h = (int*)malloc(nb * sizeof(int));
    CK(cudaMemcpy(h, d, nb * sizeof(int), cudaMemcpyDeviceToHost));
    printf("smid of linear blocks 0..39:");
    for (int i = 0; i < 40 && i < nb; ++i) printf(" %d", h[i]);
    printf("\nblocks sharing SM of block 0:");
    for (int i = 0; i < nb; ++i)
      if (h[i] == h[0]) printf(" %d", i);
    printf("\nblocks sharing SM of block 1:");
    for (int i = 0; i < nb; ++i)
      if (h[i] == h[1]) printf(" %d", i);
    printf("\n");
  }
  return 0;
}
