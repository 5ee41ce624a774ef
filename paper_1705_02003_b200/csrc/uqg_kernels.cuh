// uqg_kernels.cuh - kernel declarations, launchers and the PCG per-group state.
#pragma once

#include "uqg_common.cuh"

namespace uqg {

// group states of the device PCG loop
constexpr int kRunning = 0;
constexpr int kFinishing = 1;  // terminated; pcg_dir still owes the last x update
constexpr int kDone = 2;

// Band hint for banded graphs (stencils): the columns of tile rows [r0, r0+R)
// lie in nb row bands [r0 + start[b], r0 + start[b] + R + extra[b]).  With a
// hint, the TMA CSR SpMV bulk-prefetches those p bands into L2 when it issues
// the tile's values (the hint only moves data earlier: any hint gives
// identical results).  padded != 0 promises >= 4 ints of readable slack after
// row_offsets[N] and col_indices[nnz-1].
constexpr int kMaxBands = 9;
struct BandHint {
  int nb;
  int start[kMaxBands];
  int extra[kMaxBands];
  int padded;
};

// Face storage of the 2D 5-point FV operator (fv2d.py contract; assembly in
// assemble_fv2d_kernel).  Every CSR value of a row is a face transmissibility
// (off-diagonals -T, diagonal ((Tw + Te) + Ts) + Tn), and each interior face
// is shared by two rows, so the operator is stored once per face and the
// SpMV re-derives the row in registers: 1 stream (2 with a random y
// coefficient) instead of the 5 value streams of CSR, same products in the
// same CSR column order - bit-identical to the CSR SpMV of the same matrix.
//   tx [G][(m+1)*m][S]  face f*m + (j-1) between cell rows f and f+1 (f = 0..m)
//                       at column j: row (i, j) has Tw = tx[row], Te = tx[row+m]
//   ty [G][m*(m+1)][S]  face (i-1)*(m+1) + k between columns k and k+1 of row i:
//                       Ts = ty[row + i - 1], Tn = ty[row + i]; nullptr = a_y
// (row = (i-1)*m + (j-1), cells 1-based; both arrays hold (m+1)*m faces.)
struct Fv2dOp {
  int m;
  const double* tx;
  const double* ty;
  double a_y;
};

// Ap of one row for lanes [lo, lo+V) of group g; p_g = p + g*N*S + lo.
// P_CG: load p through L2 only (persistent kernel).  Also returns p[row].
// In-group offsets are 32-bit: the ABI requires (N + m) * S < 2^31.
template <int V, bool P_CG>
__device__ __forceinline__ void fv2d_row(const Fv2dOp& op, long long N, int S, int g, int lo,
                                         long long row_ll, const double* __restrict__ p_g,
                                         double (&y)[V], double (&pc)[V]) {
  const int m = op.m, row = (int)row_ll;
  const int i0 = row / m, j0 = row - i0 * m;  // 0-based cell
  const size_t fo = (size_t)g * (N + m) * S + lo;
  const double* txg = op.tx + fo;
  double tw[V], te[V], ts[V], tn[V], pw[V], ps[V], pn[V], pe[V];
  ldgv<V>(txg + row * S, tw);
  ldgv<V>(txg + (row + m) * S, te);
  if (op.ty) {
    const double* tyg = op.ty + fo;
    ldgv<V>(tyg + (row + i0) * S, ts);
    ldgv<V>(tyg + (row + i0 + 1) * S, tn);
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j) ts[j] = tn[j] = op.a_y;
  }
  auto ldp = [&](int r, double (&o)[V]) {
    if constexpr (P_CG) ldcgv<V>(p_g + r * S, o);
    else ldgv<V>(p_g + r * S, o);
  };
  const bool w = i0 > 0, s = j0 > 0, n = j0 < m - 1, e = i0 < m - 1;
  if (w) ldp(row - m, pw);
  if (s) ldp(row - 1, ps);
  ldp(row, pc);
  if (n) ldp(row + 1, pn);
  if (e) ldp(row + m, pe);
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const double d = __dadd_rn(__dadd_rn(__dadd_rn(tw[j], te[j]), ts[j]), tn[j]);
    double acc = 0.0;
    if (w) acc = __dadd_rn(acc, __dmul_rn(-tw[j], pw[j]));
    if (s) acc = __dadd_rn(acc, __dmul_rn(-ts[j], ps[j]));
    acc = __dadd_rn(acc, __dmul_rn(d, pc[j]));
    if (n) acc = __dadd_rn(acc, __dmul_rn(-tn[j], pn[j]));
    if (e) acc = __dadd_rn(acc, __dmul_rn(-te[j], pe[j]));
    y[j] = acc;
  }
}

// Per-lane / per-group solver state living in device memory (ctx scratch), so
// the whole PCG loop - alpha, beta, freezing, convergence, termination - is
// decided on the device.  Lane index l = g*S + s.
struct PcgState {
  int G;
  double* part;            // [G][B][NV][S] block partials
  unsigned int* ticket;    // [G] last-block tickets
  double* rz;              // [G*S] r.z of the current iterate
  double* thr;             // [G*S] tol * ||b||
  double* alpha;           // [kx][G*S]
  double* beta;            // [G*S]
  int* iters;              // [G*S] -> caller's iterations_per_lane
  unsigned char* conv;     // [G*S] -> caller's converged_per_lane
  unsigned char* frozen;   // [G*S] -> caller's frozen_lanes
  int* it;                 // [G] iterations run
  int* done;               // [G] kRunning / kFinishing / kDone
  int* status;             // [G] 0 ok, 2 breakdown
  int* ndone;              // [1] number of DONE groups (host polls it)
  double* hist;            // [(hist_cap+1)][G][S] or nullptr
  int hist_cap;
  int* overflow;           // [1] history capacity exceeded
  // Deferred solution update (launch loop): p_k lives in buffer k % kx of p
  // ([kx][G][N][S], pstride doubles apart) and alpha_k in alpha[k % kx][G*S];
  // x += alpha_j p_j is applied for kx iterations at once by pcg_flush (every
  // kx-th iteration, and for the tail after the loop) in increasing j, i.e.
  // the same roundings in the same order as one update per iteration.
  // kx = 1: x and p updated in place every iteration by pcg_dir.
  int kx;
  size_t pstride;
};

constexpr int kMaxKx = 8;  // deepest supported deferral

// Buffer slot of iteration `it`'s p / alpha.
__device__ __forceinline__ int xslot(const PcgState& st, int it) {
  return st.kx > 1 ? it % st.kx : 0;
}

// uqg_kernels.cu: KL coefficient, assembly, diagonal, grouping
__global__ void kl_sep2d_kernel(int n1, const double* table1d, const int* mode_p,
                                const int* mode_q, const double* sqrt_lam, int M,
                                const double* samples, const int* lane_ids, int G, int S,
                                double a_min, int a_hat_mode, double a_hat_value, int expansion,
                                double* a_out, int* status);
__global__ void kl_sep2d_elem_kernel(int n1, const double* table1d, const int* mode_p,
                                const int* mode_q, const double* sqrt_lam, int M,
                                const double* samples, const int* lane_ids, int G, int S,
                                double a_min, int a_hat_mode, double a_hat_value, int expansion,
                                double* a_out, int* status);
constexpr int kKlTile = 128;  // nodes per CTA of kl_sep2d_kernel (multiple of 4)
__global__ void kl_table_kernel(const double* modes, int P, int M, const double* sqrt_lam,
                                const double* samples, int L, double a_min, int a_hat_mode,
                                double a_hat_value, int expansion, double* a_out, int* status);
__global__ void assemble_fv2d_kernel(int n, int G, int S, const double* a_nodes, double a_y,
                                     int a2_same, const int* row_offsets, double* vals,
                                     double* dinv);
__global__ void assemble_fv2d_faces_kernel(int n, int G, int S, const double* a_nodes,
                                           int a2_same, double a_y, double* tx, double* ty,
                                           double* dinv);
__global__ void jacobi_dinv_kernel(long long N, int S, int G, long long nnz, const int* ro,
                                   const int* ci, const double* vals, double* dinv, int* status,
                                   int raw);
__global__ void kl_sep3d_kernel(int m, const double* qtab, const int* mode_p, const int* mode_q,
                                const int* mode_r, const double* sqrt_lam, int M,
                                const double* samples, const int* lane_ids, int G, int S,
                                double a_min, int a_hat_mode, double a_hat_value, int expansion,
                                double* a_out, int* status);
__global__ void assemble_fem3d_kernel(int m, int G, int S, const double* a_q, const double* dx_tab,
                                      const double* kyz_tab, const int* row_offsets, double* vals,
                                      double* dinv);
__global__ void key_bits_kernel(const double* keys, int n, unsigned long long* bits, int* ids,
                                int* status);
__global__ void chunk_kernel(const int* order, int n, int S, int K, int* groups, int* pad);

// uqg_pcg.cu: launchers of the V-templated streaming kernels
void launch_spmv(const Geo& geo, int G, cudaStream_t s, long long N, long long nnz, const int* ro,
                 const int* ci, const double* vals, const double* x, double* y);
void launch_lane_dot(const Geo& geo, int G, cudaStream_t s, long long N, const double* a,
                     const double* b, double* out, double* part, unsigned* ticket);
void launch_pcg_init(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                     const double* rhs, double rhs_const, const double* dinv, double tol,
                     int maxit, double* x, double* r, double* p);
void launch_pcg_spmv(const Geo& geo, int G, cudaStream_t s, long long N, long long nnz,
                     const PcgState& st, const int* ro, const int* ci, const double* vals,
                     const double* p, double* ap, const BandHint* bands);
void launch_spmv_fv2d(const Geo& geo, int G, cudaStream_t s, long long N, const Fv2dOp& op,
                      const double* x, double* y);
void launch_pcg_spmv_fv2d(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                          const Fv2dOp& op, const double* p, double* ap);
void launch_pcg_update(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                       const double* dinv, int maxit, double* r, const double* ap);
void launch_pcg_flush(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                      double* x, const double* p, bool in_loop);
void launch_pcg_dir(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                    const double* dinv, const double* r, double* x, double* p);
void launch_pcg_finalize(int G, int S, cudaStream_t s, const PcgState& st, int* ens_iters);
// While-condition of the graph launch loop: one more pass of the body unless
// every group is DONE (ndone >= G) or the pass cap is reached (*loops counts
// the passes; the host turns a capped loop into an error).
void launch_pcg_loop_cond(cudaStream_t s, cudaGraphConditionalHandle h, const int* ndone, int G,
                          int* loops, int max_loops);

// uqg_surrogate.cu: grouping keys on the device
void launch_surrogate_eval(cudaStream_t s, const double* points, int n, int dim,
                           const double* centers, const double* widths, const double* surplus,
                           int n_nodes, double* out);
void launch_anisotropy(cudaStream_t s, const double* modes, int P, int M, const double* sqrt_lam,
                       const double* samples, int L, double a_min, int a_hat_mode,
                       double a_hat_value, int expansion, double a_hi, double a_lo, double* out,
                       int* status);

// uqg_persistent.cu: whole-solve cooperative kernel for small batches
int persistent_blocks(const Geo& geo, int G);
int persistent_cluster_size(const Geo& geo);
cudaError_t launch_pcg_persistent(const Geo& geo, int G, int blocks, bool cluster, cudaStream_t s,
                                  long long N, long long nnz, const PcgState& st, const int* ro,
                                  const int* ci, const double* vals, const Fv2dOp& fv,
                                  const double* rhs,
                                  double rhs_const, const double* dinv, double tol, int maxit,
                                  double* x, double* r, double* p, double* ap, double* partA,
                                  double* partB, unsigned* bar_count, unsigned* bar_gen,
                                  int* abort_flag);

}  // namespace uqg
