// face_spmv_probe.cu - standalone probe of the face-form SpMV access pattern
// (tuning tool, not part of libuqg.so).  Times variants that add the face
// SpMV's loads one class at a time over C2-sized data (G groups x N rows x S
// lanes, lane-interleaved), reporting the algorithmic GB/s of the 3-pass
// stream (faces + p read, Ap write) so the cost of each load class shows.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe tools/face_spmv_probe.cu
//   /tmp/probe [cells=256] [S=16] [G=93]
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

// MODE 0: tx[row], p[row] -> ap            (pure 3-pass stream)
// MODE 1: + tx[row+m]                      (east face: second face stream)
// MODE 2: + p[row-m], p[row+m]             (vertical neighbours)
// MODE 3: + p[row-1], p[row+1]             (full 5-point face SpMV, no reduction)
template <int MODE>
__global__ void __launch_bounds__(256, 4) probe(Args a) {
  const int S = a.S, m = a.m, N = a.N;
  const int L = S / 2;  // threads per row (V = 2)
  const int rows_per_block = 256 / L;
  const int g = blockIdx.y;
  const int sl = threadIdx.x % L, rr = threadIdx.x / L;
  const double* txg = a.tx + (size_t)g * (N + m) * S + 2 * sl;
  const double* pg = a.p + (size_t)g * N * S + 2 * sl;
  double* apg = a.ap + (size_t)g * N * S + 2 * sl;
  for (int row = blockIdx.x * rows_per_block + rr; row < N; row += gridDim.x * rows_per_block) {
    double2 tw = ld2(txg + row * S), pc = ld2(pg + row * S);
    double2 y;
    y.x = tw.x * pc.x;
    y.y = tw.y * pc.y;
    if (MODE >= 1) {
      const double2 te = ld2(txg + (row + m) * S);
      y.x += te.x * pc.x;
      y.y += te.y * pc.y;
    }
    if (MODE >= 2) {
      const int i0 = row / m;
      if (i0 > 0) {
        const double2 pw = ld2(pg + (row - m) * S);
        y.x -= pw.x;
        y.y -= pw.y;
      }
      if (i0 < m - 1) {
        const double2 pe = ld2(pg + (row + m) * S);
        y.x -= pe.x;
        y.y -= pe.y;
      }
    }
    if (MODE >= 3) {
      const int j0 = row % m;
      if (j0 > 0) {
        const double2 ps = ld2(pg + (row - 1) * S);
        y.x -= ps.x;
        y.y -= ps.y;
      }
      if (j0 < m - 1) {
        const double2 pn = ld2(pg + (row + 1) * S);
        y.x -= pn.x;
        y.y -= pn.y;
      }
    }
    *reinterpret_cast<double2*>(apg + row * S) = y;
  }
}

// Chunked traversal of the library kernel: chunks of CT tiles (R rows each),
// blocks take chunks b, b+B, ...; per-thread p.Ap accumulated per chunk.
// RED = 0: the per-chunk accumulators go straight to global memory;
// RED = 1: + the library's batched in-block tree (8 chunks per tree) and a
// per-group atomic ticket per batch (no final stage); RED = 2: + the library's
// exact arithmetic (separate roundings, CSR term order, predicated terms).
template <int RED>
__global__ void __launch_bounds__(256, 4) probe_chunked(Args a, int CT, double* part,
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
      int row = chunk * CT * R + rr, rend = (chunk + 1) * CT * R;
      if (rend > N) rend = N;
      for (; row < rend; row += R) {
        const int i0 = row / m, j0 = row - i0 * m;
        const double2 tw = ld2(txg + row * S), te = ld2(txg + (row + m) * S),
                      pc = ld2(pg + row * S);
        double2 pw = make_double2(0, 0), pe = pw, ps = pw, pn = pw;
        if (i0 > 0) pw = ld2(pg + (row - m) * S);
        if (i0 < m - 1) pe = ld2(pg + (row + m) * S);
        if (j0 > 0) ps = ld2(pg + (row - 1) * S);
        if (j0 < m - 1) pn = ld2(pg + (row + 1) * S);
        double2 y;
        if (RED < 2) {
          y.x = (tw.x + te.x) * pc.x - tw.x * pw.x - te.x * pe.x - ps.x - pn.x;
          y.y = (tw.y + te.y) * pc.y - tw.y * pw.y - te.y * pe.y - ps.y - pn.y;
        } else {  // the library's exact CSR-order arithmetic (separate roundings)
          const double ay = 1.0;
          double d = __dadd_rn(__dadd_rn(__dadd_rn(tw.x, te.x), ay), ay), a = 0.0;
          if (i0 > 0) a = __dadd_rn(a, __dmul_rn(-tw.x, pw.x));
          if (j0 > 0) a = __dadd_rn(a, __dmul_rn(-ay, ps.x));
          a = __dadd_rn(a, __dmul_rn(d, pc.x));
          if (j0 < m - 1) a = __dadd_rn(a, __dmul_rn(-ay, pn.x));
          if (i0 < m - 1) a = __dadd_rn(a, __dmul_rn(-te.x, pe.x));
          y.x = a;
          d = __dadd_rn(__dadd_rn(__dadd_rn(tw.y, te.y), ay), ay);
          a = 0.0;
          if (i0 > 0) a = __dadd_rn(a, __dmul_rn(-tw.y, pw.y));
          if (j0 > 0) a = __dadd_rn(a, __dmul_rn(-ay, ps.y));
          a = __dadd_rn(a, __dmul_rn(d, pc.y));
          if (j0 < m - 1) a = __dadd_rn(a, __dmul_rn(-ay, pn.y));
          if (i0 < m - 1) a = __dadd_rn(a, __dmul_rn(-te.y, pe.y));
          y.y = a;
        }
        *reinterpret_cast<double2*>(apg + row * S) = y;
        acc.x = fma(pc.x, y.x, acc.x);
        acc.y = fma(pc.y, y.y, acc.y);
      }
      if (RED == 0) {
        part[((size_t)g * chunks + chunk) * 256 + t] = acc.x + acc.y;
      } else {
        red[(2 * k) * T + t] = acc.x;
        red[(2 * k + 1) * T + t] = acc.y;
      }
    }
    if (RED >= 1) {
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
}

template <int RED>
float run_chunked(const Args& a, int CT, int blocks_per_group, int reps, double* part,
                  unsigned* ticket) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  dim3 grid(blocks_per_group, a.G);
  const size_t smem = 16 * 256 * 8;
  probe_chunked<RED><<<grid, 256, smem>>>(a, CT, part, ticket);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) probe_chunked<RED><<<grid, 256, smem>>>(a, CT, part, ticket);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

template <int MODE>
float run(const Args& a, int blocks_per_group, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  dim3 grid(blocks_per_group, a.G);
  probe<MODE><<<grid, 256>>>(a);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) probe<MODE><<<grid, 256>>>(a);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

int main(int argc, char** argv) {
  const int cells = argc > 1 ? atoi(argv[1]) : 256;
  const int S = argc > 2 ? atoi(argv[2]) : 16;
  const int G = argc > 3 ? atoi(argv[3]) : 93;
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
  CK(cudaMemset(tx, 0, nt * 8));
  CK(cudaMemset(p, 0, nv * 8));
  a.tx = tx;
  a.p = p;
  a.ap = ap;
  // algorithmic bytes: faces (N+m rows) + p read + Ap write
  const double bytes = 8.0 * S * G * ((double)(a.N + a.m) + 2.0 * a.N);
  const int bpg[] = {8, 19, 26, 64};
  for (int b : bpg) {
    const float t0 = run<0>(a, b, 20), t1 = run<1>(a, b, 20), t2 = run<2>(a, b, 20),
                t3 = run<3>(a, b, 20);
    printf("blocks/group %3d: stream %.0f  +Te %.0f  +p(+-m) %.0f  +p(+-1) %.0f GB/s\n", b,
           bytes / t0 / 1e6, bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t3 / 1e6);
  }
  double* part;
  unsigned* ticket;
  CK(cudaMalloc(&part, (size_t)G * 4096 * 256 * 8));
  CK(cudaMalloc(&ticket, G * sizeof(unsigned)));
  CK(cudaMemset(ticket, 0, G * sizeof(unsigned)));
  const int L = S / 2, R = 256 / L, tiles = (a.N + R - 1) / R;
  int ct = tiles / 64;
  ct = ct < 1 ? 1 : (ct > 8 ? 8 : ct);
  if ((tiles + ct - 1) / ct > 512) ct = (tiles + 511) / 512;
  for (int b : bpg) {
    const float t4 = run_chunked<0>(a, ct, b, 20, part, ticket);
    const float t5 = run_chunked<1>(a, ct, b, 20, part, ticket);
    const float t6 = run_chunked<2>(a, ct, b, 20, part, ticket);
    printf("blocks/group %3d (chunks of %d tiles): chunked %.0f  +batched tree %.0f  "
           "+exact arithmetic %.0f GB/s\n", b, ct, bytes / t4 / 1e6, bytes / t5 / 1e6,
           bytes / t6 / 1e6);
  }
  return 0;
}
