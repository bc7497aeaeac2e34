/*
 * mpbjac.h — C-ABI of libmpbjac.so, the B200 (sm_100a) hot path of the
 * mixed-precision block-Jacobi preconditioned CG of arXiv 2407.15973.
 *
 * Every pointer argument is a DEVICE pointer unless its name starts with h_
 * (host).  All calls are stream-ordered on the handle's stream and never
 * allocate on the solve path: the caller owns matrix, vector, trace and
 * workspace buffers; the handle owns only small per-plan tables and a scratch
 * area for the standalone (non-solve) entry points.  Return value: 0 ok,
 * negative = invalid argument (the reference raises ValueError there),
 * positive = a cudaError_t.  mpb_status_string() names both kinds.
 *
 * Reference interface each entry point replaces (paths relative to the
 * reference's pkg/src/mpcg/):
 *   mpb_csr_matvec_f64/_f32        kernels_numba.py:37-45  csr_matvec
 *                                  (via sparse.py:175-183  spmv)
 *   mpb_block_jacobi_sweeps_*      kernels_numba.py:48-70  block_jacobi_sweeps
 *   mpb_dot_f64 / mpb_dot_f32      kernels_numba.py:18-24  dot_seq
 *                                  (via sparse.py:186-192  dot)
 *   mpb_norm_sq_f64 / _f32         kernels_numba.py:27-34  norm_sq_f64
 *                                  (via sparse.py:195-199  norm2)
 *   mpb_narrow_f64_f32             sparse.py:202-230       convert_precision(.., F32)
 *   mpb_widen_f32_f64              sparse.py:202-230       convert_precision(.., F64)
 *   mpb_setup_diag_f64/_f32        bjac.py:171-185         setup (diag checks)
 *   mpb_convert_values_f32         bjac.py:175 / sparse.py:202-214 (matrix values)
 *   mpb_plan_create                bjac.py:29-75           BlockPartition
 *   mpb_bjac_apply_f64/_f32        bjac.py:127-149         BjacPreconditioner.apply
 *   mpb_bjac_inner_apply_*         bjac.py:106-125         BjacPreconditioner.inner_apply
 *   mpb_fmp_apply                  policies.py:154-160     fmp_apply
 *   mpb_pcg_solve                  solver.py:101-184       pcg_solve (whole loop,
 *                                  with policies.py:102-183 apply_policy on device)
 *   mpb_true_relres                solver.py:93-98         true_relres
 */
#ifndef MPBJAC_H
#define MPBJAC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPB_VERSION 100

/* status codes (negative: argument errors) */
#define MPB_OK 0
#define MPB_ERR_ARG (-1)        /* null pointer / bad size                */
#define MPB_ERR_SHAPE (-2)      /* inconsistent lengths                   */
#define MPB_ERR_PARTITION (-3)  /* partition does not cover the matrix    */
#define MPB_ERR_SWEEPS (-4)     /* k < 1 or t < 1                          */
#define MPB_ERR_INDEX32 (-5)    /* nnz or n does not fit int32 indexing    */
#define MPB_ERR_POLICY (-6)     /* unknown policy kind / missing instance  */
#define MPB_ERR_WORKSPACE (-7)  /* workspace too small                     */
#define MPB_ERR_LAYOUT (-8)     /* SELL-32 layout / values missing         */
#define MPB_ERR_COMM (-9)       /* NCCL missing or a collective failed     */

/* policy kinds (policies.py:30-37) */
#define MPB_UNIFORM 0
#define MPB_FIXED_LOW 1
#define MPB_ADAPTIVE_HL 2
#define MPB_ADAPTIVE_LH 3

/* numerical outcomes of a solve (solver.py:31-44, sparse.py:23-24) */
#define MPB_SOLVE_OK 0
#define MPB_SOLVE_BREAKDOWN 1        /* r'z == 0            -> BreakdownError */
#define MPB_SOLVE_INDEF_PRECOND 2    /* r'z < 0             -> IndefiniteOperatorError */
#define MPB_SOLVE_INDEF_MATRIX 3     /* p'Ap <= 0           -> IndefiniteOperatorError */
#define MPB_SOLVE_NONFINITE 4        /* ||r|| not finite    -> NonFiniteResidualError */
#define MPB_SOLVE_NARROW_OVERFLOW 5  /* fp32 narrowing     -> NarrowingOverflowError */

typedef struct mpb_handle mpb_handle;
typedef struct mpb_plan mpb_plan;
/* SELL-32 layout of a CSR structure (slice height 32 = one warp, rows in
 * original order): entry j of row r at slice_ptr[r/32] + 32 j + r%32.  The
 * hot kernels read the matrix in this layout (coalesced, thread per row,
 * ascending column order); the library owns slice_ptr and the column array,
 * the caller owns value arrays packed with mpb_sell_pack_*. */
typedef struct mpb_sell mpb_sell;

/* CSR matrix on the device.  int32 row_ptr/col_idx (n and nnz < 2^31),
 * columns strictly ascending within each row (sparse.py:59-104).  The
 * sell / sell_val* fields carry the same matrix in SELL-32 layout; they are
 * required by the preconditioner, solve and true-residual entry points. */
typedef struct mpb_csr {
  int64_t n;
  int64_t nnz;
  const int32_t *row_ptr; /* n+1 */
  const int32_t *col_idx; /* nnz */
  const double *val64;    /* nnz, A.values (also the fp64 instance's values) */
  const float *val32;     /* nnz, fp32 instance's values, NULL if unused     */
  const mpb_sell *sell;   /* SELL-32 structure of row_ptr/col_idx            */
  const double *sell_val64; /* val64 packed in SELL-32 (mpb_sell_nnz entries) */
  const float *sell_val32;  /* val32 packed in SELL-32, NULL if unused        */
  /* in-block entries only, in the plan's in-block SELL-32 layout
   * (mpb_plan_pack_inblock_*); read by the first BJAC pass */
  const double *ib_val64;
  const float *ib_val32;
  /* the solved operator's fp64 values in SELL-32 when they differ from the
   * fp64 preconditioner values above (a preconditioner set up from another
   * matrix of the same structure, e.g. diag_augment(A, p)): the outer SpMV
   * and the true residuals read these (solver.py:154, 93-98).  NULL: the
   * operator is sell_val64. */
  const double *op_sell_val64;
  /* op_sell_val64 in the plan-packed layout (mpb_plan_pack_inblock_f64), so
   * that the outer SpMV can use the plan's offset-slot layout; NULL: the
   * SELL kernel runs.  Ignored when op_sell_val64 is NULL (ib_val64 is the
   * operator's then). */
  const double *op_ib_val64;
} mpb_csr;

typedef struct mpb_solve_options {
  int kind;            /* MPB_UNIFORM ...                                  */
  double adp_tol;      /* adaptive threshold (policies.py:40-43 defaults)  */
  int k, t;            /* outer passes, inner sweeps                       */
  double res_tol;      /* SolveConfig.res_tol                              */
  int64_t max_iter;    /* iteration cap (SolveConfig.iteration_cap)        */
  int64_t true_stride; /* record_true_residual_every (0: off)              */
  int has_x0;          /* x holds x0 on entry; else x is zeroed            */
  int graph_iters;     /* iterations per CUDA-graph replay (0: default)    */
} mpb_solve_options;

typedef struct mpb_solve_result {
  int converged;
  int error;              /* MPB_SOLVE_*                                   */
  int64_t iterations;
  int64_t err_iteration;
  double err_value;
  double r0_norm;
  double final_true_relres;
  int64_t overflow_count; /* narrowing overflow details                    */
  int64_t overflow_index;
  double device_seconds;  /* CUDA-event time of the iteration loop         */
  int64_t kernel_launches;
} mpb_solve_result;

/* ---- library / handle ---------------------------------------------------- */
int mpb_version(void);
const char *mpb_status_string(int status);
int mpb_create(int device, void *stream, mpb_handle **out);
int mpb_destroy(mpb_handle *h);
int mpb_set_stream(mpb_handle *h, void *stream);
int mpb_synchronize(mpb_handle *h);
/* Number of kernels this handle launched so far (for bench accounting). */
int64_t mpb_launch_count(const mpb_handle *h);

/* ---- partition / tile plan (host-only math, include/mpbjac_order.h) ---- */
/* h_tile_lo must hold nb + n/MPB_TILE_MAX_ROWS + 2 entries; returns ntiles.
 * No GPU needed. */
int64_t mpb_plan_tiles_host(int64_t nb, const int64_t *h_offsets,
                            const int64_t *h_row_ptr, int64_t *h_tile_lo,
                            int *h_large);
int mpb_plan_create(mpb_handle *h, int64_t n, int64_t nb,
                    const int64_t *h_offsets, const int64_t *h_row_ptr,
                    mpb_plan **out);
int mpb_plan_destroy(mpb_plan *p);
/* Build the plan's per-row static structure (row length, diagonal slot,
 * in-block slot range) against a SELL-32 layout of the matrix; required
 * before the plan is used with that matrix by the preconditioner / solve. */
int mpb_plan_bind_sell(mpb_handle *h, mpb_plan *p, const mpb_sell *sell);
/* The bound plan's packed value buffer: each row's entries inside its own
 * block in an in-block SELL-32 layout (ascending column; read by the first
 * BJAC pass), followed -- for plans with an offset-slot layout, see
 * mpb_plan_offset_slot_info -- by the values in that layout (and its near
 * slots alone).  mpb_plan_inblock_nnz: the entry count of the whole buffer
 * (the caller allocates it in the values' precision); mpb_plan_pack_inblock_*:
 * fill it from SELL-32 values of the bound structure. */
int64_t mpb_plan_inblock_nnz(const mpb_plan *p);
int mpb_plan_pack_inblock_f64(mpb_handle *h, const mpb_plan *p,
                              const double *sell_val, double *ib_val);
int mpb_plan_pack_inblock_f32(mpb_handle *h, const mpb_plan *p,
                              const float *sell_val, float *ib_val);
int mpb_plan_info(const mpb_plan *p, int64_t *h_ntiles, int *h_large,
                  int64_t *h_max_tile_nnz);
/* Row patterns of the bound SELL structure (after mpb_plan_bind_sell): rows
 * whose column offsets match one of *h_npat (<= 128) patterns carry no column
 * index on the hot path; *h_ngeneric rows read their SELL columns. */
int mpb_plan_layout_info(const mpb_plan *p, int *h_npat, int64_t *h_ngeneric);
/* Offset-slot layout of the bound plan: when every row pattern draws its
 * column offsets from the same 7 ascending values with 0 in the middle (a
 * 7-point stencil on any grid) and every block has 64 rows, the hot kernels
 * read slot k of every row as the entry at column row + offset[k] (no
 * pattern lookups; absent entries masked).  *h_slots: 7, or 0 without the
 * layout; *h_inblock_slots: bit k set = slot k is in-block in some row;
 * *h_near: the fused x/r update + first pass also runs on it (in-block
 * entries only at the diagonal and its two neighbouring offsets). */
int mpb_plan_offset_slot_info(const mpb_plan *p, int *h_slots, int *h_inblock_slots, int *h_near);

/* ---- SELL-32 layout (hot-path matrix format) ----------------------------- */
/* Builds slice pointers (from the host row_ptr) and packs the column array on
 * the device. */
int mpb_sell_create(mpb_handle *h, int64_t n, const int64_t *h_row_ptr,
                    const int32_t *row_ptr, const int32_t *col_idx,
                    mpb_sell **out);
int mpb_sell_destroy(mpb_sell *s);
/* Padded entry count (length of every SELL value array). */
int64_t mpb_sell_nnz(const mpb_sell *s);
/* Pack CSR values into SELL-32 order (padding zero-filled). */
int mpb_sell_pack_f64(mpb_handle *h, const mpb_sell *s, const int32_t *row_ptr,
                      const double *csr_val, double *sell_val);
int mpb_sell_pack_f32(mpb_handle *h, const mpb_sell *s, const int32_t *row_ptr,
                      const float *csr_val, float *sell_val);

/* ---- reference backend kernels (kernels_numba.py) ------------------------ */
int mpb_csr_matvec_f64(mpb_handle *h, int64_t n, const int32_t *row_ptr,
                       const int32_t *col_idx, const double *val,
                       const double *x, double *y);
int mpb_csr_matvec_f32(mpb_handle *h, int64_t n, const int32_t *row_ptr,
                       const int32_t *col_idx, const float *val,
                       const float *x, float *y);
/* in_block: one byte per nonzero (bjac.py:187-188); tmp: n entries */
int mpb_block_jacobi_sweeps_f64(mpb_handle *h, const int32_t *row_ptr,
                                const int32_t *col_idx, const double *val,
                                const uint8_t *in_block, const double *diag,
                                int t, const double *r, double *y, double *tmp,
                                int64_t row_start, int64_t row_end);
int mpb_block_jacobi_sweeps_f32(mpb_handle *h, const int32_t *row_ptr,
                                const int32_t *col_idx, const float *val,
                                const uint8_t *in_block, const float *diag,
                                int t, const float *r, float *y, float *tmp,
                                int64_t row_start, int64_t row_end);
/* Device-order sums (mpbjac_order.h).  plan may be NULL: then 512-row
 * tiles.  Result is written to h_out after a stream synchronize. */
int mpb_dot_f64(mpb_handle *h, const mpb_plan *plan, int64_t n,
                const double *x, const double *y, double *h_out);
int mpb_dot_f32(mpb_handle *h, const mpb_plan *plan, int64_t n, const float *x,
                const float *y, float *h_out);
int mpb_norm_sq_f64(mpb_handle *h, const mpb_plan *plan, int64_t n,
                    const double *x, double *h_out);
int mpb_norm_sq_f32(mpb_handle *h, const mpb_plan *plan, int64_t n,
                    const float *x, double *h_out);

/* ---- conversions and setup (sparse.py:202-230, bjac.py:152-190) -------- */
/* RN-even narrowing; counts finite values that land on +-inf.  Synchronous. */
int mpb_narrow_f64_f32(mpb_handle *h, int64_t n, const double *src, float *dst,
                       int64_t *h_overflow_count, int64_t *h_first_index);
int mpb_widen_f32_f64(mpb_handle *h, int64_t n, const float *src, double *dst);
/* Extract diag (the stored a_ii) and report the first row with no stored
 * diagonal (h_missing) and the first row whose diagonal is zero (h_zero);
 * -1 when none.  For the fp32 variant val32 is checked and val64 tells an
 * underflow (nonzero fp64 diag) from a true zero.  Synchronous. */
int mpb_setup_diag_f64(mpb_handle *h, int64_t n, const int32_t *row_ptr,
                       const int32_t *col_idx, const double *val64,
                       double *diag, int64_t *h_missing, int64_t *h_zero);
int mpb_setup_diag_f32(mpb_handle *h, int64_t n, const int32_t *row_ptr,
                       const int32_t *col_idx, const float *val32,
                       float *diag, int64_t *h_missing, int64_t *h_zero);
int mpb_convert_values_f32(mpb_handle *h, int64_t nnz, const double *val64,
                           float *val32, int64_t *h_overflow_count,
                           int64_t *h_first_index);

/* ---- the preconditioner (bjac.py:106-149, policies.py:154-160) --------- */
int mpb_bjac_apply_f64(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A,
                       int k, int t, const double *r, double *z);
int mpb_bjac_apply_f32(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A,
                       int k, int t, const float *r, float *z);
/* narrow(r) -> fp32 apply -> widen, fused; overflow reported like
 * mpb_narrow_f64_f32 (z is not written when it overflows).  Synchronous. */
int mpb_fmp_apply(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A, int k,
                  int t, const double *r, double *z,
                  int64_t *h_overflow_count, int64_t *h_first_index);
/* t sweeps on block b alone: r_b/y_b hold the block's rows. */
int mpb_bjac_inner_apply_f64(mpb_handle *h, const mpb_csr *A, int64_t row_lo,
                             int64_t row_hi, int t, const double *r_b,
                             double *y_b);
int mpb_bjac_inner_apply_f32(mpb_handle *h, const mpb_csr *A, int64_t row_lo,
                             int64_t row_hi, int t, const float *r_b,
                             float *y_b);

/* ---- the whole PCG loop on the device (solver.py:101-184) -------------- */
int64_t mpb_solve_workspace_bytes(const mpb_plan *plan, int64_t n);
/* b, x: n fp64 (x: in x0 if has_x0, out solution).  Trace arrays hold
 * max_iter entries: implicit relres, true relres (NaN = not recorded),
 * branch (0 high / 1 low), wall time since the loop started (s). */
int mpb_pcg_solve(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A,
                  const mpb_solve_options *opt, const double *b, double *x,
                  double *tr_relres, double *tr_true, int32_t *tr_branch,
                  double *tr_time, void *workspace, int64_t workspace_bytes,
                  mpb_solve_result *res);
/* Per-kernel timing of one PCG iteration (for the roofline report):
 * launches each kernel of an iteration `reps` times on the solve stream,
 * bracketing every launch with CUDA events, using the buffers of a prior
 * mpb_pcg_solve with the same arguments (the solver state is reset to a
 * mid-solve state before each launch).  branch: 0 fp64 / 1 fp32 instance.
 * h_ms[18] receives the mean ms per launch of: 0 first BJAC pass,
 * 1 middle passes (all of them, 0 when k < 3), 2 last BJAC pass,
 * 3 SpMV q = A p with the fused p.q step, 4 x/r update (fused relres
 * step), 5 x/r update fused with the next iteration's first pass (what the
 * solve runs when k >= 2 on one GPU; 0 otherwise), 6 whole iteration (sum of
 * the kernels the solve runs), 7 p-update p = z + beta p; each launched
 * alone between two events ("cold").  h_ms[8 + i]: the same kernels, `reps`
 * launches back to back with programmatic dependent launch as the solve
 * graph chains them ("chained").  h_ms[16] / h_ms[17]: the wave kernel
 * (x/r update + first pass + the next iteration's last pass, what the solve
 * runs for fixed-branch policies with k = 2 on one GPU; 0 otherwise), cold /
 * chained; the whole iteration (6 / 14) is then the SpMV plus the wave. */
int mpb_profile_iteration(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A,
                          const mpb_solve_options *opt, const double *b, double *x,
                          void *workspace, int64_t workspace_bytes, int branch,
                          int reps, double *h_ms);
/* ---- multi-GPU: z-slab row sharding over NCCL (one process per GPU) ---- */
typedef struct mpb_comm mpb_comm;
/* Ghost rows of one slab.  Own rows are 0..n-1 of the local matrix; columns
 * outside the slab are renumbered to n..n+recv_lo-1 (rows just below the slab,
 * owned by rank_lo) and n+recv_lo..n+recv_lo+recv_hi-1 (rows just above,
 * owned by rank_hi), keeping every row's stored (ascending global column)
 * order.  Each rank sends its first send_lo own rows to rank_lo and its last
 * send_hi own rows to rank_hi (-1: no neighbour). */
typedef struct mpb_halo {
  int rank_lo, rank_hi;
  int64_t recv_lo, recv_hi;
  int64_t send_lo, send_hi;
} mpb_halo;
/* 128-byte NCCL unique id (rank 0 creates it, the ranks share it). */
int mpb_comm_unique_id(void *h_id);
int mpb_comm_create(mpb_handle *h, int rank, int nranks, const void *h_id,
                    mpb_comm **out);
int mpb_comm_destroy(mpb_comm *c);
/* In-process group of nranks slab ranks on ONE device (tests of the
 * multi-GPU path with fewer GPUs than ranks): the ranks' host threads call
 * mpb_pcg_solve_dist concurrently with comms from mpb_comm_create_local;
 * every rank's work goes to the group's one stream and each halo exchange /
 * all-reduce is a host barrier at which rank 0 enqueues plain copies and a
 * rank-ordered sum for all ranks.  No kernel waits on another rank. */
int mpb_local_group_create(int device, int nranks, void **out);
int mpb_local_group_destroy(void *group);
/* the group's stream (cudaStream_t): the ranks' handles and their callers'
 * copies use it, so nothing orders through the legacy default stream */
void *mpb_local_group_stream(void *group);
int mpb_comm_create_local(void *group, int rank, mpb_comm **out);
int64_t mpb_solve_workspace_bytes_dist(const mpb_plan *plan, int64_t n,
                                       int64_t ghosts);
/* mpb_pcg_solve on this rank's slab: b has n entries, x has n + ghosts
 * (ghost part is scratch).  Halos of p and of the preconditioner's pass
 * outputs are exchanged with ncclSend/ncclRecv, the three dot products are
 * fp64 ncclAllReduce(sum) of the per-rank device-order sums; everything is
 * captured in the iteration graph.  Every rank gets the same scalars, trace
 * and stopping decision. */
int mpb_pcg_solve_dist(mpb_handle *h, const mpb_comm *comm, const mpb_halo *halo,
                       const mpb_plan *plan, const mpb_csr *A,
                       const mpb_solve_options *opt, const double *b, double *x,
                       double *tr_relres, double *tr_true, int32_t *tr_branch,
                       double *tr_time, void *workspace, int64_t workspace_bytes,
                       mpb_solve_result *res);
/* mpb_profile_iteration on one slab (x and the workspace sized with
 * `ghosts` as for mpb_pcg_solve_dist): the local kernels only, no halo or
 * all-reduce (those are timed by the whole-solve measurement). */
int mpb_profile_iteration_dist(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A,
                               const mpb_solve_options *opt, int64_t ghosts,
                               const double *b, double *x, void *workspace,
                               int64_t workspace_bytes, int branch, int reps,
                               double *h_ms);

/* ---- GPU-side problem assembly (setup; problems.py restated) ------------- */
/* Entries of the 7-point finite-volume operator on an n^3 grid (7 n^3 - 6 n^2). */
int64_t mpb_stencil_nnz(int64_t n);
/* The operator of problems.py diffusion_matrix / stencil_csr from a device
 * cell field kappa (n^3, x fastest): rows in order, entries zm ym xm diag xp
 * yp zp, interior faces w*2ab/(a+b), boundary faces w*kappa, off-diagonals
 * -(face*scale), diagonal ((((xm+xp)+ym)+yp)+zm)+zp)*scale.  Bit-identical
 * to the host generator.  row_ptr (n^3+1), col_idx, values: device. */
int mpb_assemble_stencil(mpb_handle *h, int64_t n, const double *kappa,
                         double wx, double wy, double wz, double scale,
                         int32_t *row_ptr, int32_t *col_idx, double *values);
/* Config 4's 3-temperature operator (problems.py three_temperature) from
 * the 7-point operator of its D field (rp1/col1/val1, mpb_assemble_stencil)
 * and the per-cell exchange rates w_re / w_ei (device, ncell each): rows
 * 3p+c with the cell's coupling block between the lower and upper stencil
 * entries (3 * nnz1 + 4 ncell entries; row_ptr 3 ncell + 1).  Bit-identical
 * to the host generator. */
int mpb_expand_3t(mpb_handle *h, int64_t ncell, const int32_t *rp1, const int32_t *col1,
                  const double *val1, const double *w_re, const double *w_ei,
                  double time_term, int32_t *row_ptr, int32_t *col_idx, double *values);
/* a * u_i + b for the first count SplitMix64 uniforms of seed
 * (problems.py splitmix64_stream; a = 1, b = 0: the stream itself). */
int mpb_splitmix64_uniform(mpb_handle *h, uint64_t seed, int64_t count,
                           double a, double b, double *out);

/* ---- row features (features.py:41-211 on the device) --------------------- */
/* Per row of a CSR matrix (device row_ptr (n+1), col_idx, values: exactly one
 * of val64 / val32): tau = max/min |a_ij| over stored nonzero off-diagonals
 * (NaN when undefined: none, or a non-finite maximum), dom = |a_ii| /
 * sum_{j!=i} |a_ij| (inf when that sum is 0), row_sum = sum a_ij, abs_sum =
 * sum |a_ij|, diag = stored a_ii (0 if missing); all in fp64, sums in
 * numpy's add.reduceat order (bit-identical to the reference).  Any output
 * may be NULL.  Replaces features.py:27-55 / 127-152 / 190-196. */
int mpb_row_features(mpb_handle *h, int64_t n, const int32_t *row_ptr,
                     const int32_t *col_idx, const double *val64,
                     const float *val32, double *tau, double *dom,
                     double *row_sum, double *abs_sum, double *diag);
/* Lower-inclusive histogram of the non-NaN tau over h_edges (ascending,
 * <= 64 host values; the last bin unbounded) and the NaN (undefined) count
 * (features.py:94-113).  Synchronous. */
int mpb_tau_histogram(mpb_handle *h, int64_t n, const double *tau,
                      const double *h_edges, int nedges, int64_t *h_counts,
                      int64_t *h_undefined);
/* min, median (mean of the middle two for even n), max of x with numpy's NaN
 * propagation, and the count of x > thresh (features.py:144-152).
 * Synchronous. */
int mpb_vector_stats(mpb_handle *h, int64_t n, const double *x, double thresh,
                     double *h_min, double *h_median, double *h_max,
                     int64_t *h_count_gt);
/* The first k (<= 1024) violations in index order of an M-matrix sign check
 * (features.py:182-203): kind 0 rows with !(a_i > 0) (a = diag); kind 1 rows
 * with a_i < -(tol * b_i) (a = row sums, b = absolute row sums); kind 2
 * entries (n = nnz) off the diagonal with a value > 0 (row_ptr / nrows /
 * col_idx / values of the matrix).  *h_found = how many were written.
 * Synchronous. */
int mpb_first_violations(mpb_handle *h, int kind, int64_t n, const double *a,
                         const double *b, double tol, const int32_t *row_ptr,
                         int64_t nrows, const int32_t *col_idx,
                         const double *val64, const float *val32, int k,
                         int64_t *h_idx, int64_t *h_found);

/* ||b - A x|| / r0_norm in device order.  Synchronous. */
int mpb_true_relres(mpb_handle *h, const mpb_plan *plan, const mpb_csr *A,
                    const double *x, const double *b, double r0_norm,
                    double *h_out);

#ifdef __cplusplus
}
#endif
#endif
