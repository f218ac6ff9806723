/*
 * ipmg.h -- C ABI of the B200-native multilevel interior-penalty solver
 * (hot path of arXiv 2405.18982, Cui & Kanschat, "Multilevel Interior Penalty
 * Methods on GPUs").  Cites refer to /root/reference/PAPER.md line numbers.
 *
 * Problem: -Delta u = f on a Cartesian box of cubic cells,
 * u = 0 on the boundary, symmetric interior penalty DG with Q_k elements on
 * Gauss-Lobatto nodes, Ax = b.
 *
 * Conventions for every call below
 * --------------------------------
 *  - Returns ipmg_status; IPMG_OK = 0.  No exception crosses the ABI.  On any
 *    error a one-line diagnostic is available from ipmg_last_error().
 *  - Vector arguments are caller-owned, contiguous DEVICE pointers (e.g.
 *    torch tensors' data_ptr()) of the given precision (double for IPMG_FP64,
 *    float for IPMG_FP32) and exactly ipmg_level_info() ndofs elements of the level
 *    named, unless a call says "host".  NULL where a vector is required ->
 *    IPMG_ERR_INVALID_ARG.  Input and output vectors must not alias unless
 *    stated.
 *  - Vector layout ("library order"): on a level
 *    l >= 1 (all cell counts even) the dofs are grouped by parent cell:
 *      dof = ((parent_lex * 2^d + child_lex) * (k+1)^d + node_lex)
 *    parent_lex: lexicographic (x fastest) over the level-(l-1) cells,
 *    child_lex: x fastest over the 2^d children, node_lex: x fastest over the
 *    (k+1)^d Gauss-Lobatto nodes of the cell.  Level 0 is cell-wise
 *    lexicographic (Fig. 5 right).  ipmg_to_cellwise /
 *    ipmg_from_cellwise convert to/from plain cell-wise lexicographic order.
 *  - Work is enqueued on cfg.cuda_stream (NULL = legacy default stream) and
 *    calls return without synchronising, except ipmg_cg_solve (it reads the
 *    residual norm every iteration) and the host-only utilities.  Results of
 *    every call, the solvers' x included, are complete in stream order on
 *    cfg.cuda_stream: the mixed-precision CG applies its last solution update
 *    after the final residual check, so read x on that stream (or after
 *    ipmg_synchronize), as for every other output.
 *  - A handle must not be used by two host threads at once.
 */
#ifndef IPMG_H
#define IPMG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  IPMG_OK = 0,
  IPMG_ERR_INVALID_ARG = 1,
  IPMG_ERR_UNSUPPORTED = 2,
  IPMG_ERR_SIZE_MISMATCH = 3,
  IPMG_ERR_OUT_OF_MEMORY = 4,
  IPMG_ERR_CUDA = 5,
  IPMG_ERR_NCCL = 6,
  IPMG_ERR_NOT_CONVERGED = 7
} ipmg_status;

typedef enum { IPMG_FP64 = 0, IPMG_FP32 = 1 } ipmg_precision;

/* Local solver of the vertex-patch smoother: FULL = PAPER.md:199 (V_j = all patch
 * dofs, exact residual from the face neighbours); DIRICHLET = PAPER.md:212-225
 * (V_j without the outer nodes at mesh-interior patch faces, residual from the
 * patch cells only -- inconsistent, use GMRES; reading A20). */
typedef enum { IPMG_KERNEL_FULL = 0, IPMG_KERNEL_DIRICHLET = 1, IPMG_KERNEL_CLAMPED = 2 } ipmg_kernel;
/* CLAMPED = PAPER.md:226-231: V_j = patch functions with zero value and normal
 * derivative on the mesh-interior patch faces ((2k-2)^d dofs), exact residual
 * from the patch cells only; requires the Hermite-type basis. */

/* 1D basis of Q_k on every level: GLL Lagrange or the
 * Hermite-type basis of the clamped kernel (dual to v(0), v'(0), v at the k-3
 * interior Gauss points, -v'(1), v(1); k >= 3; reading A19).  All
 * vectors are coefficient vectors in the chosen basis. */
typedef enum { IPMG_BASIS_LAGRANGE = 0, IPMG_BASIS_HERMITE = 1 } ipmg_basis;

/* Multiplicative = Algorithm 1; additive = BASELINE.json
 * configs[4] (damped, omega default 1/2^d, reading A17). */
typedef enum { IPMG_MULTIPLICATIVE = 0, IPMG_ADDITIVE = 1 } ipmg_smoother;

/* Communicator of the slab decomposition (DESIGN.md
 * "Multi-GPU"): rank r of R owns a contiguous range of cell layers along the
 * slowest axis (y in 2D, z in 3D) on every level whose global layer count is
 * a multiple of 2R ("distributed" levels); coarser levels are replicated and
 * computed redundantly on every rank.  Library-owned; created by
 * ipmg_comm_create_nccl (one process per GPU) or ipmg_comm_create_local (an
 * in-process team: one handle per host thread, used to test the distributed
 * path on a single device). */
typedef struct ipmg_comm ipmg_comm;

typedef struct {
  int dim;                  /* 2 or 3 (else IPMG_ERR_INVALID_ARG)                         */
  int degree;               /* k = 1..7 (else IPMG_ERR_UNSUPPORTED)                       */
  int coarse_cells[3];      /* T_0 cells per direction, each 1 or 2; default 2 */
  int n_levels;             /* levels 0..n_levels-1, finest has coarse_cells*2^(n_levels-1)  */
  double h0;                /* T_0 cell size; unit cube with 2^d coarse cells -> 0.5       */
  int kernel;               /* ipmg_kernel                                                 */
  int smoother;             /* ipmg_smoother                                               */
  double additive_omega;    /* additive damping; <= 0 -> 1/2^d                            */
  int post_smooth_reverse;  /* 1: post-smoothing visits colours in reverse (symmetric V) */
  int vcycle_precision;     /* ipmg_precision of the V-cycle; FP32 = PAPER.md:465 mixed  */
  double penalty_scale;     /* gamma = penalty_scale * k(k+1)(1/h+ + 1/h-); default 1     */
  int device;               /* CUDA device ordinal                                         */
  void *cuda_stream;        /* cudaStream_t all work is enqueued on                        */
  ipmg_comm *comm;          /* NULL: one GPU; else this rank's communicator (not owned)    */
  int basis;                /* ipmg_basis; CLAMPED needs HERMITE, DIRICHLET needs LAGRANGE */
  int64_t dist_min_dofs;    /* with a communicator: distribute a level only if every rank keeps
                               >= this many of its dofs (else replicate it); 0: whenever possible */
  double boundary_penalty_scale; /* penalty on domain-boundary faces = this * the interior gamma
                               (PAPER.md:97-100 gives only the two-sided formula; reading A2:
                               h+ = h- = h, i.e. 1; 0.5 is the one-sided k(k+1)/h); <= 0 -> 1 */
} ipmg_config;

typedef struct ipmg_handle ipmg_handle;

typedef struct {
  int iterations;           /* n = number of A-applications until ||r_n|| <= rtol ||r_0|| */
  double nu;                /* fractional iteration count -8 n / log10(||r_n||/||r_0||) (reading A6) */
  double rel_residual;      /* ||r_n|| / ||r_0||                                           */
  double seconds;           /* host wall time of the solve (setup excluded)                */
  int history_len;          /* entries written to history                                  */
  double *history;          /* HOST, caller-owned, capacity history_cap: ||r_0||..||r_n|| */
  int history_cap;
} ipmg_solve_info;

/* Fill *cfg with defaults: dim 3, degree 4, coarse 2x2x2, 3 levels, h0 0.5, full
 * kernel, multiplicative, reverse post-smoothing, FP32 V-cycle, penalty 1. */
void ipmg_config_default(ipmg_config *cfg);

/* Host setup + device workspace (PAPER.md:142-147 hierarchy, 259-280 1D
 * eigenpairs).  *out is library-owned; free with ipmg_destroy.  Errors:
 * INVALID_ARG (dim, n_levels < 1, coarse_cells not in {1,2}, h0 <= 0),
 * UNSUPPORTED (degree), OUT_OF_MEMORY, CUDA. */
ipmg_status ipmg_create(const ipmg_config *cfg, ipmg_handle **out);
ipmg_status ipmg_destroy(ipmg_handle *h);

/* Level geometry of THIS rank.  ndofs = local cells * (k+1)^d; cells[3] local cells
 * (cells[2] = 1 in 2D); hsize = h0/2^l.  On a distributed level the local vector
 * is the contiguous range [zoff * layer, (zoff + cells[S]) * layer) of the global
 * library-order vector (layer = dofs per cell layer of the slowest axis S). */
ipmg_status ipmg_level_info(const ipmg_handle *h, int level, int64_t *ndofs, int cells[3],
                            double *hsize);

/* Partition of a level on this rank: *distributed (1: local slab, 0: replicated),
 * *zoff (first global cell layer of the slab along the slowest axis), *nglob
 * (global cell layers along it). */
ipmg_status ipmg_level_partition(const ipmg_handle *h, int level, int *distributed, int *zoff,
                                 int *nglob);

/* HOST-ONLY: the partition rule itself (no GPU needed).  out[0] distributed,
 * out[1] zoff, out[2] local layers, out[3] global layers of `level` for `rank`
 * of `nranks`.  Rule: level l >= 1 is distributed iff its global layer count
 * along the slowest axis is a multiple of 2*nranks (every rank owns an even
 * number >= 2 of layers, so colour-0 patches and parent cells never straddle
 * ranks) and every rank keeps >= min_local_dofs of its dofs (degree k sets the
 * dofs per cell); with nranks = 1 every level is "distributed" (zoff 0). */
ipmg_status ipmg_partition(int dim, const int coarse_cells[3], int n_levels, int nranks, int rank,
                           int level, int degree, int64_t min_local_dofs, int out[4]);

/* Communicators.  ipmg_nccl_unique_id writes 128 bytes (host) that rank 0
 * broadcasts (e.g. through torch.distributed) to every rank, which then calls
 * ipmg_comm_create_nccl with its rank, the world size and its CUDA device
 * (libnccl.so.2 is resolved at run time; IPMG_ERR_NCCL if absent or on NCCL
 * errors).  ipmg_comm_create_local fills out[0..nranks-1] with the members of
 * an in-process team on devices[r] (NULL: all device 0); member r must be
 * driven by its own host thread.  Failure behaviour: in the in-process team a peer
 * that fails or stalls for 120 s makes the others return IPMG_ERR_NCCL (host barriers
 * with a timeout).  With NCCL, ipmg_comm_create_nccl blocks until every rank has called
 * it (as ncclCommInitRank does); afterwards every host wait of the solvers polls the
 * stream and ncclCommGetAsyncError, and a communicator error or no progress for
 * IPMG_NCCL_TIMEOUT seconds (environment, default 120) aborts the communicator
 * (ncclCommAbort, which releases kernels blocked on a dead peer) and returns
 * IPMG_ERR_NCCL; the communicator is unusable afterwards.  Stream-ordered calls that do
 * not wait on the host (vmult, smooth, ...) return immediately; a later host wait
 * (a solver, ipmg_synchronize) reports the failure. */
ipmg_status ipmg_nccl_unique_id(void *id128);
ipmg_status ipmg_comm_create_nccl(const void *id128, int rank, int nranks, int device,
                                  ipmg_comm **out);
ipmg_status ipmg_comm_create_local(int nranks, const int *devices, ipmg_comm **out);
ipmg_status ipmg_comm_destroy(ipmg_comm *c);

/* y = A_l x, the SIPG operator on level l applied matrix-free, patch-wise over
 * the colour-0 vertex patches (Fig. 1).  x, y: level l. */
ipmg_status ipmg_vmult(ipmg_handle *h, int level, int precision, const void *x, void *y);

/* One smoothing step x <- S_l(x, b) on level l >= 1, in place.  Multiplicative:
 * Algorithm 1 with the full kernel, residual from the
 * pre-colour state, colours 0..2^d-1 (reverse != 0: reversed).
 * Additive: x <- x + omega sum_j R_j^T A_j^{-1} R_j (b - A x). */
ipmg_status ipmg_smooth(ipmg_handle *h, int level, int precision, void *x, const void *b,
                        int reverse);

/* One colour of Algorithm 1: x_out = x_in + sum_{j in colour} R_j^T A_j^{-1} R_j (b - A x_in)
 * (patches of the colour solved exactly; cells not covered by the colour are
 * copied).  x_in may be NULL (= zero vector).  x_out must not alias x_in. */
ipmg_status ipmg_smooth_colour(ipmg_handle *h, int level, int precision, const void *x_in,
                               const void *b, void *x_out, int colour);

/* r_c = P^T (b - A_l x) on level l >= 1 into level l-1 (restriction =
 * transpose of the canonical embedding, reading A4).  x may be NULL (= 0), giving
 * r_c = P^T b. */
ipmg_status ipmg_residual_restrict(ipmg_handle *h, int fine_level, int precision, const void *x,
                                   const void *b, void *r_c);

/* x_f += P e_c: canonical embedding from level fine_level-1. */
ipmg_status ipmg_prolongate_add(ipmg_handle *h, int fine_level, int precision, const void *e_c,
                                void *x_f);

/* x0 = A_0^{-1} b0 on level 0 by global fast diagonalisation (
 * eq. inverse2d/3d with global 1D eigenpairs, reading A10). */
ipmg_status ipmg_coarse_solve(ipmg_handle *h, int precision, const void *b0, void *x0);

/* z = P_L^{-1} r: one V-cycle on the finest level, in
 * cfg.vcycle_precision (converted on entry/exit).  r, z: double,
 * finest level, may not alias. */
ipmg_status ipmg_vcycle(ipmg_handle *h, const double *r, double *z);

/* GMG-preconditioned CG on the finest level (north star; PAPER.md:331 stopping
 * rule ||r_n||_2 <= rtol ||r_0||_2, x_0 = 0).  b, x: double device vectors;
 * info may be NULL.  Returns IPMG_ERR_NOT_CONVERGED (info still filled, x = the
 * max_it-th iterate, complete in stream order) when max_it is reached; b = 0 returns
 * OK with 0 iterations.  The host reads ||r|| once per iteration (a stream wait; with
 * an NCCL communicator the wait polls for communicator errors, see ipmg_comm_create_nccl).
 * info->seconds is host wall time up to the last residual check. */
ipmg_status ipmg_cg_solve(ipmg_handle *h, const double *b, double *x, double rtol, int max_it,
                          ipmg_solve_info *info);

/* Right-preconditioned GMRES without restart, modified Gram-Schmidt (the
 * paper's outer solver),
 * with the V-cycle of cfg (fp32 = mixed precision) as the preconditioner and the
 * solution assembled as x = sum_i y_i P^{-1} v_i.  x_0 = 0; stops when the
 * least-squares residual estimate |g_{j+1}| <= rtol ||b||_2.  history =
 * ||b||, |g_1|, .., |g_n| (host); nu = -8 n / log10(|g_n| / ||b||) is the
 * fractional iteration count of PAPER.md Tables 1/2/4.  b, x: double device
 * vectors of the finest level; max_it <= 1000 (the Krylov basis, 2 max_it
 * vectors, is library-owned and kept for later solves).  Returns
 * IPMG_ERR_NOT_CONVERGED (info filled) when max_it is reached. */
ipmg_status ipmg_gmres_solve(ipmg_handle *h, const double *b, double *x, double rtol, int max_it,
                             ipmg_solve_info *info);

/* Right-hand side b_i = int f phi_i on level `level`.  kind 0: f == 1.
 * kind 1: the manufactured solution u = prod_a sin(pi x_a / ell_a) of -Delta u = f with
 * f = pi^2 (sum_a ell_a^-2) u (ell_a = coarse_cells[a] * h0, the box extents; u = 0 on the
 * boundary), moments by Gauss quadrature with k+7 points per direction (SURVEY.md 4.2(3),
 * the L2-rate property test); Lagrange basis only (else UNSUPPORTED).  b: double device
 * vector of that level.  Errors: INVALID_ARG (level, kind, NULL b). */
ipmg_status ipmg_rhs(ipmg_handle *h, int level, int kind, double *b);

/* Layout conversion library order <-> cell-wise lexicographic order. */
ipmg_status ipmg_to_cellwise(ipmg_handle *h, int level, int precision, const void *x_lib,
                             void *x_cellwise);
ipmg_status ipmg_from_cellwise(ipmg_handle *h, int level, int precision, const void *x_cellwise,
                               void *x_lib);

/* Synchronise the handle's stream; returns IPMG_ERR_CUDA on an asynchronous fault
 * (IPMG_ERR_NCCL on a communicator failure, see ipmg_comm_create_nccl). */
ipmg_status ipmg_synchronize(ipmg_handle *h);

/* Instrumentation.  ipmg_profile(h, 1) clears and enables CUDA-event timing
 * of every kernel launched on the FINEST level (events recorded on the
 * handle's stream around each launch); 0 disables.  ipmg_profile_read
 * synchronises and returns, for kernel_class (0 smoother colour pass,
 * 1 operator apply / residual, 2 residual+restrict, 3 prolongate+add,
 * 4 coarse solve, 5 vector kernels, 6 additive colour pass, 7 the levels below the
 * finest in a V-cycle, timed as one block: the CUDA-graph replay of levels L-1..0), the number of
 * recorded launches, their summed device time in ms, and their summed
 * ALGORITHMIC HBM bytes.  ipmg_launch_count: total
 * kernels this handle has launched. */
ipmg_status ipmg_profile(ipmg_handle *h, int enable);
ipmg_status ipmg_profile_read(ipmg_handle *h, int kernel_class, int64_t *launches, double *total_ms,
                              double *total_bytes);
ipmg_status ipmg_launch_count(const ipmg_handle *h, int64_t *launches);

/* Measurement utility (no part of the method): CUDA-core peak of `device` in TFLOP/s,
 * the ALU denominator of the rooflines.  kind 0: packed fp32
 * FFMA2 (fma.rn.f32x2, 2 FMAs per instruction), 1: scalar FFMA, 2: DFMA.  Full
 * occupancy, 8 independent FMA chains per thread, best of `reps` timed launches (CUDA
 * events on a private stream, after one warm-up).  Restores the caller's current
 * device.  Errors: INVALID_ARG, CUDA. */
ipmg_status ipmg_alu_peak(int device, int kind, int reps, double *tflops);

/* One-line diagnostic of the last error on h (or of the last failed create
 * when h is NULL).  Library-owned string. */
const char *ipmg_last_error(const ipmg_handle *h);

/* HOST-ONLY utility (no GPU needed): the unit-h 1D tables of degree k the
 * kernels use, for inspection/tests.  `what`: 0 nodes (k+1), 1 mass (k+1)^2,
 * 2 stiffness (k+1)^2, 3+v patch matrix L^P_v (2k+2)^2 for variant v in 0..3
 * (bit0: low face on boundary, bit1: high face on boundary), 7+v patch
 * eigenvectors S_v (row-major, column m = mode m), 11+v eigenvalues (2k+2),
 * 15 prolongation (2k+2)x(k+1); Dirichlet kernel: 16+v residual patch matrix
 * (no mesh-interior outer faces), 20+v padded local eigenvectors, 24+v their
 * eigenvalues, 28+v mode activity (1/0).  Writes at most cap doubles to out (host);
 * *len = number of entries.  Errors: UNSUPPORTED (k), INVALID_ARG. */
ipmg_status ipmg_tables_1d(int k, double penalty_scale, int what, double *out, int cap, int *len);

#ifdef __cplusplus
}
#endif

#endif /* IPMG_H */
