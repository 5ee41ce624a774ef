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
// hint, the PCG SpMV stages those p bands (and the tile's values, columns and
// row offsets) in shared memory by bulk async copies; a column outside every
// band falls back to a global load, so any hint gives identical results.
// padded != 0 promises >= 4 ints of readable slack after row_offsets[N] and
// col_indices[nnz-1] (bulk copies move 16-byte aligned spans).
constexpr int kMaxBands = 9;
struct BandHint {
  int nb;
  int start[kMaxBands];
  int extra[kMaxBands];
  int padded;
};

// Per-lane / per-group solver state living in device memory (ctx scratch), so
// the whole PCG loop - alpha, beta, freezing, convergence, termination - is
// decided on the device.  Lane index l = g*S + s.
struct PcgState {
  int G;
  double* part;            // [G][B][NV][S] block partials
  unsigned int* ticket;    // [G] last-block tickets
  double* rz;              // [G*S] r.z of the current iterate
  double* thr;             // [G*S] tol * ||b||
  double* alpha;           // [G*S]
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
};

// uqg_kernels.cu: KL coefficient, assembly, diagonal, grouping
__global__ void kl_sep2d_kernel(int n1, const double* table1d, const int* mode_p,
                                const int* mode_q, const double* sqrt_lam, int M,
                                const double* samples, const int* lane_ids, int G, int S,
                                double a_min, int a_hat_mode, double a_hat_value, int expansion,
                                double* a_out, int* status);
__global__ void kl_table_kernel(const double* modes, int P, int M, const double* sqrt_lam,
                                const double* samples, int L, double a_min, int a_hat_mode,
                                double a_hat_value, int expansion, double* a_out, int* status);
__global__ void assemble_fv2d_kernel(int n, int G, int S, const double* a_nodes, double a_y,
                                     int a2_same, const int* row_offsets, double* vals,
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
__global__ void rank_sort_kernel(const double* keys, int n, int* order, int* status);
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
void launch_pcg_update(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                       const double* dinv, int maxit, double* r, const double* ap);
void launch_pcg_dir(const Geo& geo, int G, cudaStream_t s, long long N, const PcgState& st,
                    const double* dinv, const double* r, double* x, double* p);
void launch_pcg_finalize(int G, int S, cudaStream_t s, const PcgState& st, int* ens_iters);

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
                                  const int* ci, const double* vals, const double* rhs,
                                  double rhs_const, const double* dinv, double tol, int maxit,
                                  double* x, double* r, double* p, double* ap, double* partA,
                                  double* partB, unsigned* bar_count, unsigned* bar_gen,
                                  int* abort_flag);

}  // namespace uqg
