// march_probe.cu - standalone probe (tuning tool, not part of libuqg.so) of a
// fused "direction + face SpMV" PCG pass that marches each (group, lane
// subset, row range) through the rows in order with the new direction
// p' = r * dinv + beta * p held in a shared-memory ring of 2m + 2R rows, so
// every stencil neighbour of p' is a shared-memory read and every HBM byte is
// read once: r, dinv, p (old), x-faces in; p' and Ap out (6 vector passes
// instead of the 7 of pcg_dir + pcg_spmv_fv2d).  Streams arrive through
// per-thread cp.async copies D steps ahead (no registers held in flight).
// The p.Ap partial of each reduction chunk follows the library's canonical
// order (per lane: row rr of every tile accumulated in tile order, then the
// binary tree over rr), checked here against a naive kernel.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/mp tools/march_probe.cu
//   /tmp/mp [cells=512] [S=32] [G=42] [ranges=16]
#include <cuda_runtime.h>
#include <stdint.h>
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

constexpr int R = 16;  // rows per tile (canonical geometry at S = 32: Lp = 16, T = 256)

struct Args {
  int m, N, S, G;
  int ct;          // tiles per chunk
  int chunks;      // chunks per group
  int ranges;      // row ranges per (group, lane subset)
  double a_y;
  const double* r;
  const double* dinv;
  const double* pk;
  const double* tx;
  const double* beta;  // [G][S]
  double* pn;
  double* ap;
  double* part;        // [G][chunks][S]
};

__device__ __forceinline__ void cp8(void* smem, const void* g) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// LS lanes per CTA (one per thread column), R rows per step, D stages ahead.
template <int LS, int D>
__global__ void __launch_bounds__(LS * R) march(Args a) {
  extern __shared__ __align__(16) double sm[];
  const int m = a.m, N = a.N, S = a.S;
  const int ring = 2 * m + 2 * R;
  double* rg = sm;                        // [ring][LS] p'
  double* st = rg + (size_t)ring * LS;    // [D][5][R][LS]: r, dinv, pk, te, tw
  double* red = st + (size_t)D * 5 * R * LS;  // [R][LS]
  const int t = threadIdx.x, li = t % LS, rr = t / LS;
  const int nsub = S / LS;
  int item = blockIdx.x;
  const int rgi = item % a.ranges;
  item /= a.ranges;
  const int sub = item % nsub;
  const int g = item / nsub;
  const int lane = sub * LS + li;
  // chunk range of this item
  const int c_a = (int)((long long)a.chunks * rgi / a.ranges);
  const int c_b = (int)((long long)a.chunks * (rgi + 1) / a.ranges);
  const int r0 = c_a * a.ct * R;
  int r1 = c_b * a.ct * R;
  if (r1 > N) r1 = N;
  const size_t vb = (size_t)g * N * S + lane;
  const size_t fb = (size_t)g * (N + m) * S + lane;
  const double beta = a.beta[(size_t)g * S + lane];
  // steps: cur from (r0 - 2m) rounded down to R, to r1 - 1 step R; producing
  // rows [cur + m, cur + m + R), consuming [cur, cur + R) when cur >= r0.
  const int cur0 = r0 - ((2 * m + R - 1) / R) * R;
  const int nsteps = (r1 - cur0 + R - 1) / R;
  auto issue = [&](int k) {  // stage of step k
    if (k < nsteps) {
      const int cur = cur0 + k * R;
      const int q = cur + m + rr;
      double* sb = st + ((size_t)(k % D) * 5 * R + rr) * LS + li;
      if (q >= 0 && q < N) {
        cp8(sb + 0 * R * LS, a.r + vb + (size_t)q * S);
        cp8(sb + 1 * R * LS, a.dinv + vb + (size_t)q * S);
        cp8(sb + 2 * R * LS, a.pk + vb + (size_t)q * S);
      }
      // te of consumer row cur + rr (boundary faces q < N + m included)
      if (cur >= r0 && cur + rr < r1) cp8(sb + 3 * R * LS, a.tx + fb + (size_t)q * S);
      const int row = cur + rr;
      if (cur >= r0 && row < r1) cp8(sb + 4 * R * LS, a.tx + fb + (size_t)row * S);
    }
    cp_commit();
  };
#pragma unroll
  for (int k = 0; k < D - 1; ++k) issue(k);
  double acc = 0.0;
  int tile_in_chunk = 0;
  int chunk = c_a;
  int slot_p = ((cur0 + m + rr) % ring + ring) % ring;  // ring slot of produced row
  for (int k = 0; k < nsteps; ++k) {
    issue(k + D - 1);
    cp_wait<D - 1>();
    const int cur = cur0 + k * R;
    const double* sb = st + ((size_t)(k % D) * 5 * R + rr) * LS + li;
    // produce p' for row q = cur + m + rr
    {
      const int q = cur + m + rr;
      double pv = 0.0;
      if (q >= 0 && q < N) {
        const double z = __dmul_rn(sb[0], sb[R * LS]);
        pv = __dadd_rn(z, __dmul_rn(beta, sb[2 * R * LS]));
        if (q >= r0 && q < r1) a.pn[vb + (size_t)q * S] = pv;
      }
      rg[(size_t)slot_p * LS + li] = pv;
    }
    __syncthreads();
    if (cur >= r0) {
      const int row = cur + rr;
      if (row < r1) {
        const int i0 = row / m, j0 = row - i0 * m;
        auto rs = [&](int rw) { int s2 = rw % ring; return s2 < 0 ? s2 + ring : s2; };
        const double pc = rg[(size_t)rs(row) * LS + li];
        const double tw = sb[4 * R * LS];
        // te of row = tx[row + m]: staged m rows ago as the producer's face?
        // no - the producer stage of THIS step holds tx[cur + m + rr], which is
        // exactly te of row = cur + rr.
        const double te = sb[3 * R * LS];
        const double d = __dadd_rn(__dadd_rn(__dadd_rn(tw, te), a.a_y), a.a_y);
        double y = 0.0;
        if (i0 > 0) y = __dadd_rn(y, __dmul_rn(-tw, rg[(size_t)rs(row - m) * LS + li]));
        if (j0 > 0) y = __dadd_rn(y, __dmul_rn(-a.a_y, rg[(size_t)rs(row - 1) * LS + li]));
        y = __dadd_rn(y, __dmul_rn(d, pc));
        if (j0 < m - 1) y = __dadd_rn(y, __dmul_rn(-a.a_y, rg[(size_t)rs(row + 1) * LS + li]));
        if (i0 < m - 1) y = __dadd_rn(y, __dmul_rn(-te, rg[(size_t)rs(row + m) * LS + li]));
        a.ap[vb + (size_t)row * S] = y;
        acc = __fma_rn(pc, y, acc);
      }
      if (++tile_in_chunk == a.ct || cur + R >= r1) {
        // canonical tree over rr for this chunk
        red[rr * LS + li] = acc;
        __syncthreads();
        for (int s2 = R / 2; s2 > 0; s2 >>= 1) {
          if (rr < s2) red[rr * LS + li] += red[(rr + s2) * LS + li];
          __syncthreads();
        }
        if (rr == 0) a.part[((size_t)g * a.chunks + chunk) * S + lane] = red[li];
        acc = 0.0;
        tile_in_chunk = 0;
        ++chunk;
      }
    }
    slot_p += R;
    if (slot_p >= ring) slot_p -= ring;
  }
  cp_wait<0>();
}


__device__ __forceinline__ void cp16(void* smem, const void* g) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}

// v2: two lanes per thread (16-byte cp.async / shared accesses), no integer
// division in the loop (row, i0, j0 and ring slots advanced incrementally).
template <int LS, int D>
__global__ void __launch_bounds__(LS / 2 * R) march2(Args a) {
  extern __shared__ __align__(16) double sm[];
  const int m = a.m, N = a.N, S = a.S;
  const int ring = 2 * m + 2 * R;
  constexpr int LP = LS / 2;  // threads per row
  double2* rg = reinterpret_cast<double2*>(sm);               // [ring][LP]
  double2* st = rg + (size_t)ring * LP;                       // [D][5][R][LP]
  double2* red = st + (size_t)D * 5 * R * LP;                 // [R][LP]
  const int t = threadIdx.x, li = t % LP, rr = t / LP;
  const int nsub = S / LS;
  int item = blockIdx.x;
  const int rgi = item % a.ranges;
  item /= a.ranges;
  const int sub = item % nsub;
  const int g = item / nsub;
  const int lane = sub * LS + 2 * li;
  const int c_a = (int)((long long)a.chunks * rgi / a.ranges);
  const int c_b = (int)((long long)a.chunks * (rgi + 1) / a.ranges);
  const int r0 = c_a * a.ct * R;
  int r1 = c_b * a.ct * R;
  if (r1 > N) r1 = N;
  const double* rp = a.r + (size_t)g * N * S + lane;
  const double* dp = a.dinv + (size_t)g * N * S + lane;
  const double* kp = a.pk + (size_t)g * N * S + lane;
  const double* tp = a.tx + (size_t)g * (N + m) * S + lane;
  double* pnp = a.pn + (size_t)g * N * S + lane;
  double* app = a.ap + (size_t)g * N * S + lane;
  const double2 beta = *reinterpret_cast<const double2*>(a.beta + (size_t)g * S + lane);
  const int cur0 = r0 - ((2 * m + R - 1) / R) * R;
  const int nsteps = (r1 - cur0 + R - 1) / R;
  // issue state (step ki): producer row q = cur + m + rr, consumer row cur + rr
  int ki = 0;
  auto issue = [&]() {
    if (ki < nsteps) {
      const int cur = cur0 + ki * R;
      const int q = cur + m + rr, row = cur + rr;
      double2* sb = st + ((size_t)(ki % D) * 5 * R + rr) * LP + li;
      if (q >= 0 && q < N) {
        cp16(sb + 0 * R * LP, rp + (size_t)q * S);
        cp16(sb + 1 * R * LP, dp + (size_t)q * S);
        cp16(sb + 2 * R * LP, kp + (size_t)q * S);
      }
      if (cur >= r0 && row < r1) {
        cp16(sb + 3 * R * LP, tp + (size_t)q * S);
        cp16(sb + 4 * R * LP, tp + (size_t)row * S);
      }
    }
    cp_commit();
    ++ki;
  };
#pragma unroll 1
  for (int k = 0; k < D - 1; ++k) issue();
  double acc0 = 0.0, acc1 = 0.0;
  int tile_in_chunk = 0, chunk = c_a;
  // ring slots: produced row q0 = cur0 + m + rr; consumer row r0 + rr (first
  // consumed step), neighbours at +-1, +-m
  int sp = ((cur0 + m + rr) % ring + ring) % ring;
  int sc = ((r0 + rr) % ring + ring) % ring;  // slot of consumer row (valid from cur = r0)
  int i0 = (r0 + rr) / m, j0 = (r0 + rr) - i0 * m;
  const int jstep_i = R / m, jstep_j = R - (R / m) * m;
  for (int k = 0; k < nsteps; ++k) {
    issue();
    cp_wait<D - 1>();
    const int cur = cur0 + k * R;
    const double2* sb = st + ((size_t)(k % D) * 5 * R + rr) * LP + li;
    {
      const int q = cur + m + rr;
      double2 pv = make_double2(0.0, 0.0);
      if (q >= 0 && q < N) {
        const double2 rv = sb[0], dv = sb[R * LP], ov = sb[2 * R * LP];
        pv.x = __dadd_rn(__dmul_rn(rv.x, dv.x), __dmul_rn(beta.x, ov.x));
        pv.y = __dadd_rn(__dmul_rn(rv.y, dv.y), __dmul_rn(beta.y, ov.y));
        if (q >= r0 && q < r1) *reinterpret_cast<double2*>(pnp + (size_t)q * S) = pv;
      }
      rg[(size_t)sp * LP + li] = pv;
    }
    __syncthreads();
    if (cur >= r0) {
      const int row = cur + rr;
      if (row < r1) {
        auto at = [&](int d) {
          int s2 = sc + d;
          s2 = s2 >= ring ? s2 - ring : (s2 < 0 ? s2 + ring : s2);
          return rg[(size_t)s2 * LP + li];
        };
        const double2 pc = at(0);
        const double2 tw = sb[4 * R * LP], te = sb[3 * R * LP];
        const double ay = a.a_y;
        double2 y;
        {
          const double d = __dadd_rn(__dadd_rn(__dadd_rn(tw.x, te.x), ay), ay);
          const double d2 = __dadd_rn(__dadd_rn(__dadd_rn(tw.y, te.y), ay), ay);
          double yx = 0.0, yy = 0.0;
          if (i0 > 0) {
            const double2 w = at(-m);
            yx = __dadd_rn(yx, __dmul_rn(-tw.x, w.x));
            yy = __dadd_rn(yy, __dmul_rn(-tw.y, w.y));
          }
          if (j0 > 0) {
            const double2 w = at(-1);
            yx = __dadd_rn(yx, __dmul_rn(-ay, w.x));
            yy = __dadd_rn(yy, __dmul_rn(-ay, w.y));
          }
          yx = __dadd_rn(yx, __dmul_rn(d, pc.x));
          yy = __dadd_rn(yy, __dmul_rn(d2, pc.y));
          if (j0 < m - 1) {
            const double2 w = at(1);
            yx = __dadd_rn(yx, __dmul_rn(-ay, w.x));
            yy = __dadd_rn(yy, __dmul_rn(-ay, w.y));
          }
          if (i0 < m - 1) {
            const double2 w = at(m);
            yx = __dadd_rn(yx, __dmul_rn(-te.x, w.x));
            yy = __dadd_rn(yy, __dmul_rn(-te.y, w.y));
          }
          y = make_double2(yx, yy);
        }
        *reinterpret_cast<double2*>(app + (size_t)row * S) = y;
        acc0 = __fma_rn(pc.x, y.x, acc0);
        acc1 = __fma_rn(pc.y, y.y, acc1);
      }
      sc += R;
      if (sc >= ring) sc -= ring;
      i0 += jstep_i;
      j0 += jstep_j;
      while (j0 >= m) { j0 -= m; ++i0; }
      if (++tile_in_chunk == a.ct || cur + R >= r1) {
        red[rr * LP + li] = make_double2(acc0, acc1);
        __syncthreads();
        for (int s2 = R / 2; s2 > 0; s2 >>= 1) {
          if (rr < s2) {
            double2 u = red[rr * LP + li];
            const double2 v = red[(rr + s2) * LP + li];
            u.x += v.x;
            u.y += v.y;
            red[rr * LP + li] = u;
          }
          __syncthreads();
        }
        if (rr == 0) *reinterpret_cast<double2*>(a.part + ((size_t)g * a.chunks + chunk) * S + lane) = red[li];
        acc0 = acc1 = 0.0;
        tile_in_chunk = 0;
        ++chunk;
      }
    }
    sp += R;
    if (sp >= ring) sp -= ring;
  }
  cp_wait<0>();
}


// v3: U tiles per step (U x R rows, T = U x R x LS/2 threads) sharing one
// ring; the canonical per-(lane, rr) fma chain over the tiles is restored by
// a serial fix-up: every thread stores its (p, Ap) pair, and after the next
// step's barrier the u = 0 threads run the U fmas in tile order.
template <int LS, int D, int U>
__global__ void __launch_bounds__(U * LS / 2 * R) march3(Args a) {
  extern __shared__ __align__(16) double sm[];
  const int m = a.m, N = a.N, S = a.S;
  constexpr int RS = U * R;               // rows per step
  const int ring = 2 * m + 2 * RS;
  constexpr int LP = LS / 2;
  double2* rg = reinterpret_cast<double2*>(sm);               // [ring][LP]
  double2* st = rg + (size_t)ring * LP;                       // [D][5][RS][LP]
  double2* fx = st + (size_t)D * 5 * RS * LP;                 // [2][RS][LP][2] (p, Ap)
  double2* red = fx + (size_t)2 * RS * LP * 2;                // [R][LP]
  const int t = threadIdx.x, li = t % LP, rs_ = t / LP;       // rs_ = row within step
  const int rr = rs_ % R, u = rs_ / R;
  const int nsub = S / LS;
  int item = blockIdx.x;
  const int rgi = item % a.ranges;
  item /= a.ranges;
  const int sub = item % nsub;
  const int g = item / nsub;
  const int lane = sub * LS + 2 * li;
  const int c_a = (int)((long long)a.chunks * rgi / a.ranges);
  const int c_b = (int)((long long)a.chunks * (rgi + 1) / a.ranges);
  const int r0 = c_a * a.ct * R;
  int r1 = c_b * a.ct * R;
  if (r1 > N) r1 = N;
  const double* rp = a.r + (size_t)g * N * S + lane;
  const double* dp = a.dinv + (size_t)g * N * S + lane;
  const double* kp = a.pk + (size_t)g * N * S + lane;
  const double* tp = a.tx + (size_t)g * (N + m) * S + lane;
  double* pnp = a.pn + (size_t)g * N * S + lane;
  double* app = a.ap + (size_t)g * N * S + lane;
  const double2 beta = *reinterpret_cast<const double2*>(a.beta + (size_t)g * S + lane);
  const int cur0 = r0 - ((2 * m + RS - 1) / RS) * RS;
  const int nsteps = (r1 - cur0 + RS - 1) / RS;
  int ki = 0;
  auto issue = [&]() {
    if (ki < nsteps) {
      const int cur = cur0 + ki * RS;
      const int q = cur + m + rs_, row = cur + rs_;
      double2* sb = st + ((size_t)(ki % D) * 5 * RS + rs_) * LP + li;
      if (q >= 0 && q < N) {
        cp16(sb + 0 * RS * LP, rp + (size_t)q * S);
        cp16(sb + 1 * RS * LP, dp + (size_t)q * S);
        cp16(sb + 2 * RS * LP, kp + (size_t)q * S);
      }
      if (cur >= r0 && row < r1) {
        cp16(sb + 3 * RS * LP, tp + (size_t)q * S);
        cp16(sb + 4 * RS * LP, tp + (size_t)row * S);
      }
    }
    cp_commit();
    ++ki;
  };
#pragma unroll 1
  for (int k = 0; k < D - 1; ++k) issue();
  double acc0 = 0.0, acc1 = 0.0;   // live in u == 0 threads
  int tiles_done = 0, chunk = c_a;
  int sp = ((cur0 + m + rs_) % ring + ring) % ring;
  int sc = ((r0 + rs_) % ring + ring) % ring;
  int i0 = (r0 + rs_) / m, j0 = (r0 + rs_) - i0 * m;
  const int jstep_i = RS / m, jstep_j = RS - (RS / m) * m;
  bool pending = false;   // fix-up of the previous consumer step outstanding
  int pend_buf = 0, pend_cur = 0;
  auto fixup = [&]() {
    // u == 0 threads: U fmas in tile order for (lane pair li, row rr)
    if (u == 0) {
      const double2* f = fx + (size_t)pend_buf * RS * LP * 2;
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int row = pend_cur + uu * R + rr;
        if (row < r1) {
          const double2 pv = f[((size_t)(uu * R + rr) * LP + li) * 2];
          const double2 yv = f[((size_t)(uu * R + rr) * LP + li) * 2 + 1];
          acc0 = __fma_rn(pv.x, yv.x, acc0);
          acc1 = __fma_rn(pv.y, yv.y, acc1);
        }
      }
    }
    tiles_done += U;
    if (tiles_done >= a.ct || pend_cur + RS >= r1) {  // chunk complete (ct % U == 0)
      if (u == 0) red[rr * LP + li] = make_double2(acc0, acc1);
      __syncthreads();
      for (int s2 = R / 2; s2 > 0; s2 >>= 1) {
        if (u == 0 && rr < s2) {
          double2 x = red[rr * LP + li];
          const double2 v = red[(rr + s2) * LP + li];
          x.x += v.x;
          x.y += v.y;
          red[rr * LP + li] = x;
        }
        __syncthreads();
      }
      if (t < LP) *reinterpret_cast<double2*>(a.part + ((size_t)g * a.chunks + chunk) * S + sub * LS + 2 * t) = red[t];
      acc0 = acc1 = 0.0;
      tiles_done = 0;
      ++chunk;
    }
    pending = false;
  };
  for (int k = 0; k < nsteps; ++k) {
    issue();
    cp_wait<D - 1>();
    const int cur = cur0 + k * RS;
    const double2* sb = st + ((size_t)(k % D) * 5 * RS + rs_) * LP + li;
    {
      const int q = cur + m + rs_;
      double2 pv = make_double2(0.0, 0.0);
      if (q >= 0 && q < N) {
        const double2 rv = sb[0], dv = sb[RS * LP], ov = sb[2 * RS * LP];
        pv.x = __dadd_rn(__dmul_rn(rv.x, dv.x), __dmul_rn(beta.x, ov.x));
        pv.y = __dadd_rn(__dmul_rn(rv.y, dv.y), __dmul_rn(beta.y, ov.y));
        if (q >= r0 && q < r1) *reinterpret_cast<double2*>(pnp + (size_t)q * S) = pv;
      }
      rg[(size_t)sp * LP + li] = pv;
    }
    __syncthreads();
    if (pending) fixup();
    if (cur >= r0) {
      const int row = cur + rs_;
      double2 pc = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
      if (row < r1) {
        auto at = [&](int d) {
          int s2 = sc + d;
          s2 = s2 >= ring ? s2 - ring : (s2 < 0 ? s2 + ring : s2);
          return rg[(size_t)s2 * LP + li];
        };
        pc = at(0);
        const double2 tw = sb[4 * RS * LP], te = sb[3 * RS * LP];
        const double ay = a.a_y;
        const double d = __dadd_rn(__dadd_rn(__dadd_rn(tw.x, te.x), ay), ay);
        const double d2 = __dadd_rn(__dadd_rn(__dadd_rn(tw.y, te.y), ay), ay);
        double yx = 0.0, yy = 0.0;
        if (i0 > 0) {
          const double2 w = at(-m);
          yx = __dadd_rn(yx, __dmul_rn(-tw.x, w.x));
          yy = __dadd_rn(yy, __dmul_rn(-tw.y, w.y));
        }
        if (j0 > 0) {
          const double2 w = at(-1);
          yx = __dadd_rn(yx, __dmul_rn(-ay, w.x));
          yy = __dadd_rn(yy, __dmul_rn(-ay, w.y));
        }
        yx = __dadd_rn(yx, __dmul_rn(d, pc.x));
        yy = __dadd_rn(yy, __dmul_rn(d2, pc.y));
        if (j0 < m - 1) {
          const double2 w = at(1);
          yx = __dadd_rn(yx, __dmul_rn(-ay, w.x));
          yy = __dadd_rn(yy, __dmul_rn(-ay, w.y));
        }
        if (i0 < m - 1) {
          const double2 w = at(m);
          yx = __dadd_rn(yx, __dmul_rn(-te.x, w.x));
          yy = __dadd_rn(yy, __dmul_rn(-te.y, w.y));
        }
        y = make_double2(yx, yy);
        *reinterpret_cast<double2*>(app + (size_t)row * S) = y;
      }
      double2* f = fx + (size_t)(k & 1) * RS * LP * 2;
      f[((size_t)rs_ * LP + li) * 2] = pc;
      f[((size_t)rs_ * LP + li) * 2 + 1] = y;
      pending = true;
      pend_buf = k & 1;
      pend_cur = cur;
      sc += RS;
      if (sc >= ring) sc -= ring;
      i0 += jstep_i;
      j0 += jstep_j;
      while (j0 >= m) { j0 -= m; ++i0; }
    }
    sp += RS;
    if (sp >= ring) sp -= ring;
  }
  __syncthreads();
  if (pending) fixup();
  cp_wait<0>();
}

// naive reference: p' then Ap (separate kernels), canonical partials
__global__ void naive_dir(Args a) {
  const size_t tot = (size_t)a.G * a.N * a.S;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot;
       i += (size_t)gridDim.x * blockDim.x) {
    const int lane = (int)(i % a.S);
    const int g = (int)(i / ((size_t)a.N * a.S));
    const double z = __dmul_rn(a.r[i], a.dinv[i]);
    a.pn[i] = __dadd_rn(z, __dmul_rn(a.beta[(size_t)g * a.S + lane], a.pk[i]));
  }
}
__global__ void naive_spmv(Args a) {
  const int m = a.m, N = a.N, S = a.S;
  const size_t tot = (size_t)a.G * N * S;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot;
       i += (size_t)gridDim.x * blockDim.x) {
    const int lane = (int)(i % S);
    const size_t gr = i / S;
    const int row = (int)(gr % N), g = (int)(gr / N);
    const double* p = a.pn + (size_t)g * N * S + lane;
    const double* tx = a.tx + (size_t)g * (N + m) * S + lane;
    const int i0 = row / m, j0 = row - i0 * m;
    const double tw = tx[(size_t)row * S], te = tx[(size_t)(row + m) * S];
    const double d = __dadd_rn(__dadd_rn(__dadd_rn(tw, te), a.a_y), a.a_y);
    double y = 0.0;
    if (i0 > 0) y = __dadd_rn(y, __dmul_rn(-tw, p[(size_t)(row - m) * S]));
    if (j0 > 0) y = __dadd_rn(y, __dmul_rn(-a.a_y, p[(size_t)(row - 1) * S]));
    y = __dadd_rn(y, __dmul_rn(d, p[(size_t)row * S]));
    if (j0 < m - 1) y = __dadd_rn(y, __dmul_rn(-a.a_y, p[(size_t)(row + 1) * S]));
    if (i0 < m - 1) y = __dadd_rn(y, __dmul_rn(-te, p[(size_t)(row + m) * S]));
    a.ap[i] = y;
  }
}
__global__ void naive_part(Args a) {
  // one thread per (g, chunk, lane): canonical accumulation + tree
  const size_t tot = (size_t)a.G * a.chunks * a.S;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot;
       i += (size_t)gridDim.x * blockDim.x) {
    const int lane = (int)(i % a.S);
    const size_t gc = i / a.S;
    const int c = (int)(gc % a.chunks), g = (int)(gc / a.chunks);
    double v[R];
    for (int rr = 0; rr < R; ++rr) {
      double acc = 0.0;
      for (int k = 0; k < a.ct; ++k) {
        const long long row = ((long long)c * a.ct + k) * R + rr;
        if (row >= a.N) break;
        const size_t o = ((size_t)g * a.N + row) * a.S + lane;
        acc = __fma_rn(a.pn[o], a.ap[o], acc);
      }
      v[rr] = acc;
    }
    for (int s2 = R / 2; s2 > 0; s2 >>= 1)
      for (int rr = 0; rr < s2; ++rr) v[rr] += v[rr + s2];
    a.part[i] = v[0];
  }
}

__global__ void fill(double* x, size_t n, uint64_t seed, double lo, double hi) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    x[i] = lo + (hi - lo) * ((z >> 11) * (1.0 / 9007199254740992.0));
  }
}

template <int LS, int D>
float run(Args a, int reps) {
  const int ring = 2 * a.m + 2 * R;
  const size_t smem = ((size_t)ring * LS + (size_t)D * 5 * R * LS + R * LS) * 8;
  CK(cudaFuncSetAttribute(march<LS, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, march<LS, D>, LS * R, smem));
  const int items = a.G * (a.S / LS) * a.ranges;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  march<LS, D><<<items, LS * R, smem>>>(a);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) march<LS, D><<<items, LS * R, smem>>>(a);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;
  const double vec = 8.0 * a.S * (double)a.N * a.G, faces = 8.0 * a.S * (double)(a.N + a.m) * a.G;
  const double bytes = 5 * vec + faces;
  printf("LS=%2d D=%d ranges=%3d smem=%6zu B ctas/SM=%d items=%d: %.3f ms  %.1f GB/s (6 passes)\n",
         LS, D, a.ranges, smem, per, items, ms, bytes / ms / 1e6);
  return ms;
}


template <int LS, int D>
float run2(Args a, int reps) {
  const int ring = 2 * a.m + 2 * R;
  const size_t smem = ((size_t)ring * LS + (size_t)D * 5 * R * LS + R * LS) * 8;
  CK(cudaFuncSetAttribute(march2<LS, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, march2<LS, D>, LS / 2 * R, smem));
  const int items = a.G * (a.S / LS) * a.ranges;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  march2<LS, D><<<items, LS / 2 * R, smem>>>(a);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) march2<LS, D><<<items, LS / 2 * R, smem>>>(a);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;
  const double vec = 8.0 * a.S * (double)a.N * a.G, faces = 8.0 * a.S * (double)(a.N + a.m) * a.G;
  printf("v2 LS=%2d D=%2d ranges=%3d smem=%6zu B ctas/SM=%d items=%d: %.3f ms  %.1f GB/s\n", LS, D,
         a.ranges, smem, per, items, ms, (5 * vec + faces) / ms / 1e6);
  return ms;
}


template <int LS, int D, int U>
float run3(Args a, int reps) {
  constexpr int RS = U * R;
  const int ring = 2 * a.m + 2 * RS;
  const size_t smem = ((size_t)ring * LS + (size_t)D * 5 * RS * LS + (size_t)2 * RS * LS * 2 + R * LS) * 8;
  const int T = U * LS / 2 * R;
  CK(cudaFuncSetAttribute(march3<LS, D, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, march3<LS, D, U>, T, smem));
  const int items = a.G * (a.S / LS) * a.ranges;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  march3<LS, D, U><<<items, T, smem>>>(a);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) march3<LS, D, U><<<items, T, smem>>>(a);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  ms /= reps;
  const double vec = 8.0 * a.S * (double)a.N * a.G, faces = 8.0 * a.S * (double)(a.N + a.m) * a.G;
  printf("v3 LS=%2d D=%d U=%d T=%d ranges=%3d smem=%6zu B ctas/SM=%d: %.3f ms  %.1f GB/s\n", LS, D,
         U, T, a.ranges, smem, per, ms, (5 * vec + faces) / ms / 1e6);
  return ms;
}

int main(int argc, char** argv) {
  const int cells = argc > 1 ? atoi(argv[1]) : 512;
  const int S = argc > 2 ? atoi(argv[2]) : 32;
  const int G = argc > 3 ? atoi(argv[3]) : 42;
  Args a{};
  a.m = cells - 1;
  a.N = a.m * a.m;
  a.S = S;
  a.G = G;
  // canonical geometry (make_geo) for this (N, S): ct tiles per chunk
  const long long tiles = (a.N + R - 1) / R;
  long long ct = tiles / 64;
  ct = ct < 1 ? 1 : (ct > 8 ? 8 : ct);
  if ((tiles + ct - 1) / ct > 512) ct = (tiles + 511) / 512;  // (C3: single level)
  a.ct = (int)ct;
  a.chunks = (int)((tiles + ct - 1) / ct);
  a.ranges = argc > 4 ? atoi(argv[4]) : 16;
  a.a_y = 1.0;
  const size_t nv = (size_t)G * a.N * S, nf = (size_t)G * (a.N + a.m) * S;
  double *r, *dinv, *pk, *tx, *beta, *pn, *ap, *part, *pn2, *ap2, *part2;
  CK(cudaMalloc(&r, nv * 8));
  CK(cudaMalloc(&dinv, nv * 8));
  CK(cudaMalloc(&pk, nv * 8));
  CK(cudaMalloc(&tx, nf * 8));
  CK(cudaMalloc(&beta, (size_t)G * S * 8));
  CK(cudaMalloc(&pn, nv * 8));
  CK(cudaMalloc(&ap, nv * 8));
  CK(cudaMalloc(&part, (size_t)G * a.chunks * S * 8));
  CK(cudaMalloc(&pn2, nv * 8));
  CK(cudaMalloc(&ap2, nv * 8));
  CK(cudaMalloc(&part2, (size_t)G * a.chunks * S * 8));
  fill<<<4096, 256>>>(r, nv, 1, -1, 1);
  fill<<<4096, 256>>>(dinv, nv, 2, 0.1, 1);
  fill<<<4096, 256>>>(pk, nv, 3, -1, 1);
  fill<<<4096, 256>>>(tx, nf, 4, 0.5, 2);
  fill<<<64, 256>>>(beta, (size_t)G * S, 5, 0, 1);
  CK(cudaDeviceSynchronize());
  a.r = r; a.dinv = dinv; a.pk = pk; a.tx = tx; a.beta = beta;
  // reference
  a.pn = pn2; a.ap = ap2; a.part = part2;
  naive_dir<<<4096, 256>>>(a);
  naive_spmv<<<4096, 256>>>(a);
  naive_part<<<1024, 128>>>(a);
  CK(cudaDeviceSynchronize());
  a.pn = pn; a.ap = ap; a.part = part;
  printf("cells=%d S=%d G=%d ct=%d chunks=%d: %.2f GB per fused pass\n", cells, S, G, a.ct,
         a.chunks, (5.0 * nv + nf) * 8 / 1e9);
  auto check = [&](const char* tag) {
    double* h1 = (double*)malloc(nv * 8);
    double* h2 = (double*)malloc(nv * 8);
    long long bad = 0;
    CK(cudaMemcpy(h1, pn, nv * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2, pn2, nv * 8, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < nv; ++i) bad += h1[i] != h2[i];
    CK(cudaMemcpy(h1, ap, nv * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2, ap2, nv * 8, cudaMemcpyDeviceToHost));
    long long bad2 = 0;
    for (size_t i = 0; i < nv; ++i) bad2 += h1[i] != h2[i];
    const size_t np = (size_t)G * a.chunks * S;
    CK(cudaMemcpy(h1, part, np * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2, part2, np * 8, cudaMemcpyDeviceToHost));
    long long bad3 = 0;
    for (size_t i = 0; i < np; ++i) bad3 += h1[i] != h2[i];
    printf("  %s: mismatches p' %lld, Ap %lld, partials %lld\n", tag, bad, bad2, bad3);
    free(h1);
    free(h2);
  };
  const int reps = 10;
  const int r_in = a.ranges;
  for (int rg : {r_in, 2 * r_in}) {
    a.ranges = rg;
    run3<8, 2, 4>(a, reps);
    run3<8, 3, 4>(a, reps);
    run3<4, 3, 4>(a, reps);
    run3<4, 4, 4>(a, reps);
    run3<4, 3, 8>(a, reps);
    run3<8, 2, 8>(a, reps);
    run3<8, 3, 2>(a, reps);
    run3<4, 4, 2>(a, reps);
  }
  a.ranges = r_in;
  CK(cudaMemset(pn, 0, nv * 8));
  CK(cudaMemset(ap, 0, nv * 8));
  CK(cudaMemset(part, 0, (size_t)G * a.chunks * S * 8));
  run3<8, 3, 4>(a, 1); check("v3 LS8 D3 U4");
  CK(cudaMemset(part, 0, (size_t)G * a.chunks * S * 8));
  run3<4, 3, 8>(a, 1); check("v3 LS4 D3 U8");
  run2<8, 4>(a, reps);
  return 0;
}
