/*
 * uqg.h - C ABI of the B200-native ensemble solve (libuqg.so).
 *
 * The reference (uqgroup, pure Python) has no FFI: its boundary is Python duck
 * typing.  These entry points are what a ctypes binding of the
 * reference's hot path binds; each names the reference interface it replaces.
 * Conventions:
 *   - every array argument is a DEVICE pointer unless its name ends in _host;
 *   - ensemble data is sample-interleaved: values [G][nnz][S], vectors [G][N][S],
 *     G independent groups ("ensembles") of S lanes ("samples") sharing one
 *     CSR graph (row_offsets [N+1], col_indices [nnz], int32, sorted per row);
 *   - `stream` is a cudaStream_t (may be NULL = legacy default stream); every
 *     call is stream-ordered; only uqg_pcg, uqg_status_sync and calls that
 *     return a validation verdict synchronise the stream;
 *   - return value: UQG_OK or an error code; uqg_last_error() gives a
 *     thread-local message for the last failing call.
 */
#ifndef UQG_H
#define UQG_H

#ifdef __cplusplus
extern "C" {
#endif

#define UQG_OK 0
#define UQG_EINVAL 1      /* -> EnsembleError / GroupingError / FemError       */
#define UQG_EBREAKDOWN 2  /* -> NumericalBreakdownError (ensemble.py:48-49)   */
#define UQG_ECUDA 3       /* CUDA runtime error                                */
#define UQG_ENOMEM 4      /* device allocation failed                          */
#define UQG_ECAPACITY 5   /* residual-history buffer too small; re-run larger  */

typedef struct uqg_ctx uqg_ctx;

int uqg_version(void);
const char* uqg_last_error(void);

/* One context per device per process; owns scratch workspace and events. */
int uqg_ctx_create(int device, uqg_ctx** out);
int uqg_ctx_destroy(uqg_ctx* ctx);

/* Hand the context a caller-owned device buffer to carve scratch from (e.g. a
 * torch allocation); calls needing more fall back to a library allocation.
 * ptr NULL detaches.  The buffer must outlive every call that uses it. */
int uqg_ctx_set_workspace(uqg_ctx* ctx, void* ptr, long long bytes);

/* Structure hint for banded graphs (stencils), used by uqg_pcg on this ctx
 * until replaced (nbands = 0 clears): the columns of rows [r0, r0+R) lie in
 * the row bands [r0 + starts[b], r0 + starts[b] + R + extras[b]).  With it the
 * TMA SpMV bulk-prefetches each tile's p bands into L2 when it issues the
 * tile's values; the hint only moves data earlier, so it never changes
 * results.  graph_padded != 0 promises >= 4 readable ints after
 * row_offsets[N] and after col_indices[nnz-1].  nbands <= 9. */
int uqg_ctx_set_band_hint(uqg_ctx* ctx, int nbands, const int* starts_host,
                          const int* extras_host, int graph_padded);

/* Kernel classes for launch accounting / timing. */
#define UQG_K_KL 0
#define UQG_K_ASSEMBLE 1
#define UQG_K_PCG_INIT 2
#define UQG_K_PCG_SPMV 3   /* Ap = A p + p.Ap                           */
#define UQG_K_PCG_UPDATE 4 /* r update + r.r, r.z                       */
#define UQG_K_PCG_DIR 5    /* p = z + beta p (x += alpha p when kx = 1)  */
#define UQG_K_DOT 6        /* lane_dot / qoi                             */
#define UQG_K_GROUP 7      /* key bits + radix sort + chunk              */
#define UQG_K_SPMV 8       /* standalone spmv                            */
#define UQG_K_OTHER 9      /* diagonal, jacobi, finalize                 */
#define UQG_K_PCG_FLUSH 10 /* deferred x += sum_j alpha_j p_j (every kx) */
#define UQG_NKERN 11

/* Per-launch CUDA-event timing on the launching stream (off by default).
 * uqg_ctx_profile_read returns accumulated milliseconds and launch counts per
 * kernel class (arrays of UQG_NKERN; either may be NULL) and optionally
 * resets them; it synchronises on the last recorded event.  Launch counts are
 * kept whether or not timing is on. */
int uqg_ctx_profile(uqg_ctx* ctx, int enable);
int uqg_ctx_profile_read(uqg_ctx* ctx, double* ms_host, long long* launches_host, int reset);
/* Total kernels this context has launched. */
long long uqg_ctx_launch_count(uqg_ctx* ctx);

/* Device-side sticky status word (bit 0: non-positive coefficient or diagonal,
 * bit 1: non-finite grouping key).  Synchronises `stream`, returns the word in
 * *status_host and clears it. */
int uqg_status_sync(uqg_ctx* ctx, void* stream, int* status_host);

/* KL coefficient at the (n+1)^2 nodes of the unit-square grid, separable modes.
 * Replaces KLDiffusionField.eval_a_batch (random_field.py:145-166) evaluated at
 * the mesh nodes with mode_values (random_field.py:135-143) = factor products.
 *   table1d [n_factors][n+1]: 1D factor f at x_i = i*h (np.interp, host setup)
 *   mode_p/mode_q [M]: factor ids of mode m; sqrt_lam [M] = sqrt(eigenvalues)
 *   samples [*][M] sample rows; lane_ids [G*S] (may be NULL = identity): lane
 *   g*S+s evaluates sample row lane_ids[g*S+s] - the grouping plan from
 *   uqg_group_sort feeds the solve without a host round trip;
 *   a_hat_mode 0=constant 1=test2; expansion 0=log 1=linear
 *   a_out [G][(n+1)^2][S].  a <= 0 anywhere sets status bit 0 (fem3d.py:153). */
int uqg_kl_eval_sep2d(uqg_ctx* ctx, int n_cells, const double* table1d, int n_factors,
                      const int* mode_p, const int* mode_q, const double* sqrt_lam, int M,
                      const double* samples, const int* lane_ids, int G, int S, double a_min,
                      int a_hat_mode, double a_hat_value, int expansion, double* a_out,
                      void* stream);

/* Dense form: a[l][p] = a_min + a_hat(y_l) * f(sum_m sqrt_lam[m] y_l[m] modes[m][p]),
 * output lane-major [L][P] exactly like eval_a_batch's (S, P) result. */
int uqg_kl_eval_table(uqg_ctx* ctx, const double* modes, int P, int M, const double* sqrt_lam,
                      const double* samples, int L, double a_min, int a_hat_mode,
                      double a_hat_value, int expansion, double* a_out, void* stream);

/* 2D 5-point FV ensemble assembly into the shared graph (
 * contract of assemble, fem3d.py:138-175).  a_nodes [G][(n+1)^2][S];
 * vals [G][nnz][S]; dinv [G][N][S] = 1/diag (may be NULL; jacobi_precond,
 * ensemble.py:179-183).  a2_same=0: y-faces use a_y (reference convention). */
int uqg_assemble_fv2d(uqg_ctx* ctx, int n_cells, int G, int S, const double* a_nodes,
                      double a_y, int a2_same, const int* row_offsets, double* vals,
                      double* dinv, void* stream);

/* 3D trilinear hex FEM (the reference's own operator, fem3d.py), m cells/dir.
 * uqg_kl_eval_sep3d: a at the 8 Gauss points of every element, a_out
 * [G][m^3*8][S] (element-major, q bit-ordered x,y,z), qtab [n_factors][2m] =
 * 1D factors at the Gauss abscissae; mode_p/q/r [M] factor ids; other
 * arguments as uqg_kl_eval_sep2d (random_field.py:145-166 at quad_points).
 * uqg_assemble_fem3d: vals [G][nnz][S] on the 27-point graph (row_offsets
 * [N+1], N=(m-1)^3), summing per nonzero the element matrices
 * sum_q a_q dx_tab[q][a][b] + kyz_tab[a][b] in increasing element order
 * (assemble, fem3d.py:138-175: einsum + bincount); dinv [G][N][S] = 1/diag
 * (may be NULL).  dx_tab [8][8][8] = _elem_mats[0], kyz_tab [8][8]. */
int uqg_kl_eval_sep3d(uqg_ctx* ctx, int m, const double* qtab, int n_factors, const int* mode_p,
                      const int* mode_q, const int* mode_r, const double* sqrt_lam, int M,
                      const double* samples, const int* lane_ids, int G, int S, double a_min,
                      int a_hat_mode, double a_hat_value, int expansion, double* a_out,
                      void* stream);
int uqg_assemble_fem3d(uqg_ctx* ctx, int m, int G, int S, const double* a_q, const double* dx_tab,
                       const double* kyz_tab, const int* row_offsets, double* vals, double* dinv,
                       void* stream);

/* Jacobi inverse diagonal from any shared-graph ensemble matrix
 * (EnsembleCsrMatrix.diagonal + jacobi_precond, ensemble.py:130-137,179-183).
 * Synchronises; returns UQG_EINVAL if any lane diagonal <= 0. */
int uqg_jacobi_dinv(uqg_ctx* ctx, int N, int nnz, int S, int G, const int* row_offsets,
                    const int* col_indices, const double* vals, double* dinv, void* stream);

/* Raw lane diagonals diag [G][N][S] (EnsembleCsrMatrix.diagonal,
 * ensemble.py:130-137): last diagonal entry of a row wins, absent reads 0. */
int uqg_diagonal(uqg_ctx* ctx, int N, int nnz, int S, int G, const int* row_offsets,
                 const int* col_indices, const double* vals, double* diag, void* stream);

/* y = A x per lane, sequential CSR order without FMA: bitwise equal to scipy
 * csr_matvec per lane (EnsembleCsrMatrix.spmv, ensemble.py:116-128).
 * max_row_len: longest row of the graph if known (selects the unrolled row
 * kernel: <=5 e.g. the 2D 5-point stencil, <=8), 0 = unknown; any value gives
 * identical results. */
int uqg_spmv(uqg_ctx* ctx, int N, int nnz, int max_row_len, int S, int G, const int* row_offsets,
             const int* col_indices, const double* vals, const double* x, double* y,
             void* stream);

/* out[g][s] = sum_j a[g][j][s] * b[g][j][s] (lane_dot, ensemble.py:155-161);
 * deterministic fixed-shape reduction tree.  Also serves qoi (fem3d.py:178-183). */
int uqg_lane_dot(uqg_ctx* ctx, int N, int S, int G, const double* a, const double* b,
                 double* out, void* stream);

/* Ensemble Jacobi-PCG on G independent groups at once (ensemble_pcg,
 * ensemble.py:205-281; exact semantics in SURVEY.md Appendix A).
 *   rhs [G][N][S] or NULL (then every entry is rhs_const);
 *   dinv [G][N][S] or NULL (IdentityPreconditioner, ensemble.py:164-166);
 *   x [G][N][S] out; iters [G][S] int32 out; converged/frozen [G][S] uint8 out;
 *   ens_iters [G] int32 out;
 *   hist_host: NULL, or host buffer [(hist_cap+1)][G][S] receiving the lane
 *   residual norms per iteration (row 0 = ||b||); *hist_rows_host = rows used.
 * Runs the whole loop on the device; the host only polls a done-counter.
 * Small batches run as one persistent launch (cluster barriers); large ones
 * as a launch loop, split into up to UQG_SOLVE_STREAMS concurrent parts on
 * context-owned streams that start after, and are joined back into,
 * `stream` - the call stays stream-ordered and results do not depend on the
 * split.  max_row_len as for uqg_spmv.
 * Returns UQG_EBREAKDOWN on a non-finite residual in an active lane. */
int uqg_pcg(uqg_ctx* ctx, int N, int nnz, int max_row_len, int S, int G, const int* row_offsets,
            const int* col_indices, const double* vals, const double* rhs, double rhs_const,
            const double* dinv, double tol, int maxit, double* x, int* iters,
            unsigned char* converged, unsigned char* frozen, int* ens_iters,
            double* hist_host, int hist_cap, int* hist_rows_host, void* stream);

/* Device bytes of scratch uqg_pcg needs for (N, S, G) (r, p, Ap, partials). */
long long uqg_pcg_workspace_bytes(int N, int nnz, int S, int G);

/* Iterations per deferred solution update in the launch loop (UQG_X_DEFER,
 * default 4; 1 = x updated every iteration): x += alpha_j p_j is applied kx
 * iterations at a time in increasing j - identical bits for every kx. */
int uqg_pcg_x_defer(void);

/* Face form of the 2D 5-point FV operator (same matrix as uqg_assemble_fv2d,
 * stored once per face instead of once per CSR entry; fv2d.py:46-80 values).
 * With m = n_cells - 1 and N = m*m unknowns:
 *   tx [G][(m+1)*m][S]: x-face f*m + (j-1) between cell rows f, f+1 at column
 *      j, i.e. row (i,j) has Tw = tx[row], Te = tx[row + m];
 *   ty [G][m*(m+1)][S]: y-face (i-1)*(m+1) + k between columns k, k+1 of row
 *      i (Ts = ty[row + i - 1], Tn = ty[row + i]); only when a2_same, else
 *      NULL and the y-faces are the constant a_y;
 *   dinv [G][N][S] = 1/diag (may be NULL).
 * uqg_spmv_fv2d / uqg_pcg_fv2d apply it with the products of the CSR row in
 * CSR column order: results are bit-identical to uqg_spmv / uqg_pcg on the
 * CSR form (arguments otherwise as uqg_pcg; the workspace size is
 * uqg_pcg_workspace_bytes(m*m, 0, S, G)). */
int uqg_assemble_fv2d_faces(uqg_ctx* ctx, int n_cells, int G, int S, const double* a_nodes,
                            double a_y, int a2_same, double* tx, double* ty, double* dinv,
                            void* stream);
int uqg_spmv_fv2d(uqg_ctx* ctx, int n_cells, int S, int G, const double* tx, const double* ty,
                  double a_y, const double* x, double* y, void* stream);
int uqg_pcg_fv2d(uqg_ctx* ctx, int n_cells, int S, int G, const double* tx, const double* ty,
                 double a_y, const double* rhs, double rhs_const, const double* dinv, double tol,
                 int maxit, double* x, int* iters, unsigned char* converged,
                 unsigned char* frozen, int* ens_iters, double* hist_host, int hist_cap,
                 int* hist_rows_host, void* stream);

/* Grouping keys on the device.
 * uqg_surrogate_eval: out[i] = sum_j prod_d max(0, 1 - |y[i][d] - c[j][d]| / w[j][d])
 * * surplus[j] (HierGrid.eval_many / _basis_block, hier_grid.py:317-359);
 * points [n][dim] canonical coordinates, centers/widths [n_nodes][dim],
 * dim <= 64.  On the iteration channel the result is exact (dyadic data), so it
 * equals the host's BLAS value bit for bit.
 * uqg_anisotropy_indicator: per sample l, max over P points of
 * max(a, a_hi) / min(a, a_lo) with a the KL coefficient from the dense mode
 * table modes [M][P] (anisotropy_indicator, random_field.py:254-270, with
 * a_hi = max(a_y, a_z), a_lo = min(a_y, a_z)); out [L].  Synchronises;
 * UQG_EINVAL if a coefficient bound is <= 0. */
int uqg_surrogate_eval(uqg_ctx* ctx, const double* points, int n, int dim, const double* centers,
                       const double* widths, const double* surplus, int n_nodes, double* out,
                       void* stream);
int uqg_anisotropy_indicator(uqg_ctx* ctx, const double* modes, int P, int M,
                             const double* sqrt_lam, const double* samples, int L, double a_min,
                             int a_hat_mode, double a_hat_value, int expansion, double a_hi,
                             double a_lo, double* out, void* stream);

/* Stable ascending sort of keys[n] (ties keep generation order) and chunking
 * into width-S groups, the short last group padded with its last sample
 * (group_by_key/_chunk, grouping.py:83-95,105-122).  keys NULL = natural
 * order (group_natural, grouping.py:98-102).  order [n] out (may be NULL),
 * groups [ceil(n/S)][S] out (indices into the input), pad [ceil(n/S)] out.
 * The sort is a stable LSD radix sort of order-preserving 64-bit key images
 * (+0.0 and -0.0 tie).  Synchronises; returns UQG_EINVAL on a non-finite key. */
int uqg_group_sort(uqg_ctx* ctx, const double* keys, int n, int S, int* order, int* groups,
                   int* pad, void* stream);
/* The same without any host synchronisation (the level pipeline): a
 * non-finite key sets status bit 1, seen by the caller's next
 * uqg_status_sync. */
int uqg_group_sort_async(uqg_ctx* ctx, const double* keys, int n, int S, int* order,
                         int* groups, int* pad, void* stream);
/* Clear the device status word, stream-ordered (no host synchronisation). */
int uqg_status_clear(uqg_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* UQG_H */
