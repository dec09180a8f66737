/*
 * sylv_sketch.h — C ABI of the B200 (sm_100a) sketched-and-truncated block Krylov
 * solver for the low-rank Sylvester equation
 *
 *        A X + X B = C1 C2^T,        X ~ X1 X2^T
 *
 * following Alg. 1 of Palitta, Schweitzer, Simoncini, arXiv 2311.16019
 * ("alg:whitening_krylov").  All arithmetic is IEEE fp64.
 *
 * The hot path (per block step d, for both K_d(A,C1) and K_d(B^T,C2)) runs in this
 * library's own CUDA kernels:
 *   a1  W~ = A U_d                          (Alg. 1 line 3,   PAPER.md:889)
 *   a2  h_{i,d} = U_i^T W~, W~ -= U_i h_{i,d}, i = max(1,d-k+1)..d
 *                                           (lines 4-7,       PAPER.md:890-895)
 *   a3  U_{d+1} h_{d+1,d} = W~              (line 8,          PAPER.md:896)
 *   a4  S U_{d+1} with a hashed sparse-sign S, never stored (BASELINE.json north star)
 *   a5  Q_{d+1} T_{d+1} = S [U_d, U_{d+1}]  (line 9,          PAPER.md:897-898; Prop. 2.1)
 * and, on the host at scheduled d:
 *   a6  projected Sylvester solve + sketched residual (lines 10-13, PAPER.md:899-903,
 *       eqs. reduced_sk PAPER.md:268-270 and resnorm_sk PAPER.md:323-325, hatted
 *       coefficients: DESIGN.md reading R4)
 * and once, on the device:
 *   a7  two-pass reconstruction X1 = U_d T_d^{-1} Y1 (lines 19-20).
 *
 * Conventions
 *  - Blocks (C1, C2, X1, X2, apply_sketch operands) are row-major: element (i, c) of
 *    an n x r block is at p[i*r + c] (X: p[i*ldx + c]).
 *  - Pointer arguments documented "host or device" are classified with
 *    cudaPointerGetAttributes; host memory may be pageable or pinned.
 *  - Ownership: the caller owns every pointer it passes; inputs are copied during
 *    the call, outputs are caller-allocated.  The library owns its workspace
 *    (allocated in init, released in destroy).
 *  - Errors: status codes only; no exceptions cross the ABI, no abort/exit.
 *    sylv_sketch_last_error() returns the context's last message.  After
 *    SYLV_E_BREAKDOWN / SYLV_E_SINGULAR / SYLV_E_NOT_CONVERGED / SYLV_E_LOST_INDEP the
 *    context stays valid for residual / solution / get_small / history (d <= d_done);
 *    after SYLV_E_BREAKDOWN or SYLV_E_LOST_INDEP it is terminal for stepping (step
 *    returns the same status again), and get_block only returns blocks still in the
 *    ring of the last step the device ran.
 *  - Concurrency: a context is not thread-safe; all device work is ordered on the
 *    stream given to init.
 *  - Supported shapes (round 1): r in {1,2,4,8}, 1 <= k <= 4, s % zeta == 0,
 *    s >= (d_max+1) r, n*zeta < 2^32.
 */
#ifndef SYLV_SKETCH_H
#define SYLV_SKETCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sylv_ctx sylv_ctx; /* opaque */

typedef enum {
  SYLV_OK = 0,
  SYLV_E_INVALID = 1,       /* bad argument / unsupported shape                          */
  SYLV_E_NOMEM = 2,         /* device or host allocation failed                          */
  SYLV_E_CUDA = 3,          /* CUDA runtime error (message in last_error)                */
  SYLV_E_NCCL = 4,          /* NCCL transport failure (comm create, collective)          */
  SYLV_E_BREAKDOWN = 5,     /* min diag h_{d+1,d} <= 1e-14 ||W~||_F (R11)      */
  SYLV_E_SINGULAR = 6,      /* projected Sylvester equation (numerically) singular       */
  SYLV_E_NOT_CONVERGED = 7, /* d_max reached without rho_rel < tol; state stays valid    */
  SYLV_E_STATE = 8,         /* call order violated (e.g. residual(d) with d > d_done)    */
  SYLV_E_LOST_INDEP = 9,    /* tau_{d+1} not positive definite: sketched basis deficient */
  SYLV_E_LAPACK = 10        /* host LAPACK not loadable (see sylv_set_lapack_path)       */
} sylv_status;

typedef enum { SYLV_OP_STENCIL2D = 1, SYLV_OP_STENCIL3D = 2, SYLV_OP_CSR = 3 } sylv_op_kind;

/* A coefficient matrix of the Sylvester equation (A, or B — NOT B^T; the library
 * forms B^T itself: for stencils by negating w (exact for central differences with
 * constant w, R16), for CSR by an explicit transpose at init).
 *  Stencil: -nu Laplace(u) + w . grad(u) on the unit square/cube, Dirichlet BCs,
 *           grid[0] = N interior nodes per direction, h = 1/(N+1), x fastest,
 *           n = N^2 or N^3  (BASELINE.json configs 0-3).
 *  CSR:     row_ptr[n+1] (int64), col_idx[nnz] (int32), val[nnz] (fp64); host or
 *           device; copied at init. */
typedef struct {
  int32_t kind;          /* sylv_op_kind */
  int64_t n;             /* global number of rows = columns                     */
  int32_t grid[3];       /* stencil: N (only grid[0] used; cubic/square grids)  */
  double nu;             /* stencil diffusion coefficient (BASELINE: 1.0)       */
  double w[3];           /* stencil convection vector                           */
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const double* val;
  int64_t nnz;
  int32_t is_transposed; /* CSR operator B only: 1 = the arrays already hold B^T (no
                            transpose at init); 0 = B (transposed on the device at init) */
} sylv_operator;

typedef struct {
  int32_t r;             /* block size (rank of C1, C2)                        */
  int32_t k;             /* truncation: orthogonalise against the last k blocks */
  int32_t d_max;         /* maxit                                              */
  int32_t zeta;          /* sparse-sign nonzeros per column (8)                */
  int64_t s;             /* sketch rows; s % zeta == 0, s >= (d_max+1) r       */
  uint64_t seed_u;       /* hash seed of S_U                                   */
  uint64_t seed_v;       /* hash seed of S_V                                   */
  double tol;            /* stop when rho_rel < tol (strict)                   */
  double rank_tol;       /* Y ~ Y1 Y2^T keeps sigma_i > rank_tol * sigma_1     */
  int32_t chunk;         /* second pass: blocks per X accumulation (0 = auto:   
                            up to 32, within half the free device memory)     */
  int32_t flags;         /* bit 0: time the n-space passes with CUDA events;
                            bit 1: run everything on one stream (isolated kernel
                            timings; default: U and V passes on two streams, each
                            sequence's sketch-space work on its own side stream);
                            bit 2: disable the 2.5-D TMA passes (3-D stencil, r = 8,
                            even N) and use the generic pass kernels;
                            bit 3: projected solves on the device for every d;
                            bit 4: projected solves on the host for every d
                            (default: device when d r >= 512, host below).
                            (Round 1's bit 5, a fused pass 2 + old-block pass 1,
                            measured slower and was removed in round 2: DESIGN.md §9) */
  int64_t row_begin;     /* sharded contexts: this rank's global rows [row_begin, */
  int64_t row_end;       /* row_end); 0, 0 = sylv_partition's balanced split.     */
                         /* Single-rank contexts: 0, 0 (or 0, n).                  */
  int32_t method;        /* SYLV_METHOD_*: 0 = sketched-and-truncated (Alg. 1, the
                            hot path); 1 = truncated Arnoldi without a sketch (Alg. 2,
                            PAPER.md:1178-1206: H_d Y + Y G_d^T = E1 b1 b2^T E1^T with
                            b = R(C), rho = the Prop. 3.2 bound sqrt(dr)(||Y E_d g^T|| +
                            ||h E_d^T Y||); s, zeta, seeds unused);
                            2 = full Arnoldi / Galerkin (every block
                            retained and orthonormalised against all previous ones by
                            block CGS2; k is ignored (= d_max); exact residual norm;
                            single-rank only; needs (d_max+1) n r doubles per sequence);
                            3 = sketched-and-truncated with the sketched inner product also
                            in the truncated Gram-Schmidt (h_{i,d} = (S U_i)^T
                            (S W~), S-orthonormal blocks; no inner product over n, hence no
                            n-space allreduce on several ranks) */
  int32_t sketch_kind;   /* SYLV_SKETCH_*: 0 = hashed sparse sign (zeta nonzeros per
                            column, seeds seed_u / seed_v; BASELINE); 1 = the paper's
                            SRDCT S = sqrt(n/s) D N E (scale read as
                            sqrt(n/s), R2): E = the n signs below (+-1),
                            N = orthonormal DCT-II, D = the s rows below; single-rank */
  const int8_t* srdct_signs_u;   /* SRDCT: n signs of E for S_U / S_V (host or device; */
  const int8_t* srdct_signs_v;   /* copied at init)                                   */
  const int64_t* srdct_rows_u;   /* SRDCT: s row indices of D in [0, n) for S_U / S_V  */
  const int64_t* srdct_rows_v;
} sylv_config;

enum { SYLV_SKETCH_SPARSE_SIGN = 0, SYLV_SKETCH_SRDCT = 1 };

enum { SYLV_METHOD_SKETCHED = 0, SYLV_METHOD_TRUNCATED = 1, SYLV_METHOD_FULL = 2, SYLV_METHOD_SKETCHED_GS = 3 };

/* Create a context and run Alg. 1 line 1: U1 ell = C1, V1 ell' = C2
 * (CholQR on the device), beta_1 = R(S_U C1), beta_2 = R(S_V C2), T_1 = tau_1 =
 * beta_1 ell^{-1} (R3).  C1, C2: n_local x r row-major (this rank's rows),
 * host or device.  stream: a cudaStream_t (NULL = legacy default stream).
 * nccl_comm: NULL (single rank) or a sylv_comm* (row-sharded context, SURVEY §8(e):
 * z-slabs / y-line ranges of the 2-D/3-D stencils, ranges of 32-row groups of a CSR matrix;
 * every rank calls every function of the context collectively, in the same order, with
 * identical cfg).  CSR operators of a sharded context describe the GLOBAL matrices (every
 * rank passes the same arrays, A and B, not B^T); each rank keeps its rows of A and of B^T
 * with local column indices, and its halo width is the band max |col - row| of the matrix
 * (every rank must own at least band rows; c4: 4096).  Each rank keeps
 * its rows of every basis block (plus ghost planes/rows filled by halo exchange); the
 * Gram-Schmidt inner products, Grams and partial sketches are summed over the ranks
 * (bit-identical on all ranks), the sketch-space QR and the projected solves are
 * replicated.  sylv_sketch_solution / get_block / apply_sketch work on local rows
 * (apply_sketch returns the global S X on every rank). */
sylv_status sylv_sketch_init(const sylv_operator* A, const sylv_operator* B,
                             const double* C1, const double* C2,
                             const sylv_config* cfg, void* nccl_comm, void* stream,
                             sylv_ctx** out);

/* Advance both sequences by up to nsteps block steps (Alg. 1 lines 3-9).  On return
 * *d_done = number of completed steps d (the basis holds d+1 blocks).  Returns
 * SYLV_E_BREAKDOWN (state valid, d_done = breakdown step), SYLV_E_LOST_INDEP (tau_{d+1}
 * not positive definite; d_done = last good step) or SYLV_E_NOT_CONVERGED when d_max is
 * reached before nsteps.  After BREAKDOWN / LOST_INDEP further calls return that status. */
sylv_status sylv_sketch_step(sylv_ctx* ctx, int32_t nsteps, int32_t* d_done);

/* Projected solve at 1 <= d <= d_done (Alg. 1 lines 10-13): M_U Y + Y M_V^T =
 * E1 beta1 beta2^T E1^T with M_U = [T_d | T_H] H_und_d T_d^{-1} (R6), then
 * rho^2 = ||hhat E_d^T Y||^2 + ||Y E_d ghat^T||^2, rho_rel = rho / ||beta1 beta2^T||_F.
 * Solver: host Bartels-Stewart (LAPACK) for d r < 512; above, on the device: the sign-function
 * iteration, else (where it fails: spec(M_V) not in Re > 0) an eigendecomposition solve
 * accepted only when its refined projected residual is at rounding level, else the host.
 * Y is kept in the context for sylv_sketch_solution(ctx, d, ...). */
sylv_status sylv_sketch_residual(sylv_ctx* ctx, int32_t d, double* rho, double* rho_rel);

/* Second pass (Alg. 1 lines 19-20): truncated SVD of the Y of the last residual(d)
 * call (computed here if absent), Z = T_d^{-1} Y1, and the device replay of the
 * Arnoldi recurrence from the stored coefficients, X1 = U_d Z1, X2 = V_d Z2.
 * X1, X2: n x max_rank row-major with leading dimension ldx >= max_rank, host or
 * device; columns >= *rank are zeroed. */
sylv_status sylv_sketch_solution(sylv_ctx* ctx, int32_t d, double* X1, double* X2,
                                 int64_t ldx, int32_t max_rank, int32_t* rank);

/* Driver: step + canonical check schedule + search of the last bracket (R9:
 * crossing prediction, safeguarded regula falsi on log rho_rel with bisection steps;
 * all checks exact unless SYLV_APPROX_CHECKS=1).  On success *d_star is a passing d
 * whose checked predecessor in the bracket failed (with rho_rel monotone on the bracket:
 * the first crossing, as bisection finds it).  Residual history is available through
 * sylv_sketch_history. */
sylv_status sylv_sketch_solve(sylv_ctx* ctx, int32_t* d_star, double* rho_rel);

/* Test / introspection entries -------------------------------------------------- */

/* Y = S X for an n x r block X (row-major, host or device); which = 0: S_U, 1: S_V.
 * Y: s x r row-major, host or device. */
sylv_status sylv_sketch_apply_sketch(sylv_ctx* ctx, int32_t which, const double* X,
                                     int32_t r, double* Y);

/* Small matrices of sequence `which` after d <= d_done steps, row-major:
 * H: (d+1)r x dr (H_und_d), T: (d+1)r x (d+1)r (T_{d+1}), beta: r x r. Any may be NULL. */
sylv_status sylv_sketch_get_small(sylv_ctx* ctx, int32_t which, int32_t d, double* H,
                                  double* T, double* beta);

/* Normalised basis block U_j (which=0) / V_j (which=1), n x r row-major, host or
 * device; j must still be in the window (d_done+1-k <= j <= d_done+1). */
sylv_status sylv_sketch_get_block(sylv_ctx* ctx, int32_t which, int32_t j, double* out);

/* Residual history of the last sylv_sketch_solve / residual calls: up to cap
 * entries (d, rho_rel); returns the count in *count. */
sylv_status sylv_sketch_history(sylv_ctx* ctx, int32_t cap, int32_t* d, double* rho_rel,
                                int32_t* count);

typedef struct {
  int64_t launches;          /* kernels launched by this context so far           */
  int64_t steps;             /* block steps done                                  */
  double ms_pass1, ms_pass2; /* summed CUDA-event times of the n-space passes     */
  int64_t n_pass1, n_pass2;  /* timed launches (flags bit 0)                      */
  double ms_skqr;            /* summed time of the sketch-space QR (flags bit 0)  */
  int64_t n_skqr;
  double ms_sketch;          /* summed time of the sparse-sign sketch kernels (a4) */
  int64_t n_sketch;
  double host_solve_s;       /* wall seconds spent in host projected solves       */
  int64_t host_solves;
  double kappa_T_u, kappa_T_v; /* reserved                                        */
  int64_t gpu_solves;        /* projected solves done on the device (sign iteration or
                                certified eigendecomposition)                        */
  double gpu_solve_s;        /* wall seconds in them                               */
  int64_t gpu_solve_fallbacks; /* device solves that did not converge -> host BS   */
  int64_t gpu_approx_checks;   /* solve driver: checks decided "rho_rel > 3 tol" by a
                                  device solve that ended off the identity          */
} sylv_stats;

sylv_status sylv_sketch_stats(sylv_ctx* ctx, sylv_stats* out);
void sylv_sketch_reset_stats(sylv_ctx* ctx);

const char* sylv_sketch_last_error(const sylv_ctx* ctx);
void sylv_sketch_destroy(sylv_ctx* ctx);

/* ---- Row-sharded contexts (north star: "row-sharded by grid slabs, with NCCL
 * halo exchange ... an allreduce of the Gram-Schmidt coefficients and ... of partial
 * sketches (S is linear in rows)") ------------------------------------------------------ */
typedef struct sylv_comm sylv_comm; /* opaque transport handle */

/* Balanced split of an operator over nranks: rank gets the global rows
 * [*row_begin, *row_end) = whole z-planes (3-D) or y-lines (2-D), or (kind = SYLV_OP_CSR; N is
 * ignored) a range of 32-row groups; every range starts at a multiple of 32 rows (the sketch
 * hash groups rows by 32).  Host only.  SYLV_E_INVALID if there are fewer
 * plane/row groups than ranks. */
sylv_status sylv_partition(int32_t kind, int32_t N, int64_t n, int32_t nranks, int32_t rank,
                           int64_t* row_begin, int64_t* row_end);

/* NCCL transport (one process per GPU).  Rank 0 calls sylv_comm_nccl_unique_id and the
 * caller broadcasts the 128 bytes (e.g. with torch.distributed); then every rank calls
 * sylv_comm_create_nccl collectively.  libnccl.so.2 is dlopen'ed (SYLV_E_NCCL if absent). */
sylv_status sylv_comm_nccl_unique_id(uint8_t id[128]);
sylv_status sylv_comm_create_nccl(int32_t nranks, int32_t rank, const uint8_t id[128], sylv_comm** out);
/* NCCL transport over a communicator the CALLER owns (an ncclComm_t, passed as void*): the
 * library splits its per-channel communicators from it (collective over its ranks) and
 * destroys only those splits in sylv_comm_destroy; the caller's communicator stays the
 * caller's (destroy it after sylv_comm_destroy). */
sylv_status sylv_comm_wrap_nccl(void* nccl_comm, sylv_comm** out);

/* In-process transport: nranks virtual ranks of ONE process on one GPU, one host thread per
 * rank calling the context functions collectively (parity tests of the sharded path on a
 * single GPU; sums and ghost copies are plain kernels/copies ordered by CUDA events and host
 * barriers, no kernel waits on another).  The group outlives its comms. */
sylv_status sylv_local_group_create(int32_t nranks, void** group);
void sylv_local_group_destroy(void* group);
sylv_status sylv_comm_create_local(void* group, int32_t rank, sylv_comm** out);

/* Destroy a transport handle (after every context using it). */
void sylv_comm_destroy(sylv_comm* comm);

/* Host LAPACK (dgees/dtrsyl/dgemm/dtrsm/dgesvd with the `scipy_` symbol prefix of
 * SciPy's bundled OpenBLAS, LP64).  Must be set before the first residual call;
 * returns SYLV_E_LAPACK if the library or a symbol cannot be loaded. */
sylv_status sylv_set_lapack_path(const char* path);

/* Host-only entries of the a6 step (no device work; used by the CPU test suite).
 * sylv_host_projected: M = [T_d | T_H] H_und_d T_d^{-1} (R6) from T (col-major,
 *   ld ldT, >= (d+1)r square) and the per-step coefficient layout of the library:
 *   H[j*(k+1)*r*r + slot*r*r + a*r + c], slot i < min(k,j) -> h_{j-min(k,j)+1+i, j},
 *   slot k -> h_{j+1,j} (row-major r x r blocks).  M: dr x dr col-major.
 * sylv_host_sylvester: Bartels-Stewart for MU Y + Y MV^T = E1 B E1^T (B r x r row-major),
 *   MU, MV, Y: m x m col-major (MU, MV are overwritten).  Returns SYLV_E_SINGULAR when
 *   the solve breaks down, SYLV_E_LAPACK when LAPACK is missing. */
sylv_status sylv_host_projected(int32_t d, int32_t r, int32_t k, const double* T, int64_t ldT,
                                const double* H, double* M);
sylv_status sylv_host_sylvester(int32_t m, int32_t r, double* MU, double* MV, const double* B,
                                double* Y);

/* Library version string. */
const char* sylv_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SYLV_SKETCH_H */
