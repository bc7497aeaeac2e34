/*
 * mpbjac_oracle.c — CPU restatement of the reference's PCG / block-Jacobi hot
 * path.  TEST INFRASTRUCTURE, NOT PRODUCT CODE: only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's CPU-baseline / --impl reference
 * legs may load this library, and only as the checker or the CPU baseline.
 * The product path (paper_2407_15973_b200) never calls it.
 *
 * Every function below restates one reference function (file:line relative
 * to the reference's pkg/src/mpcg/):
 *   orc_csr_matvec_*      kernels_numba.py:37-45   (row-sequential, no FMA)
 *   orc_sweeps_*          kernels_numba.py:48-70   (masked Jacobi sweeps)
 *   orc_dot_seq_*         kernels_numba.py:18-24
 *   orc_norm_sq_*         kernels_numba.py:27-34
 *   orc_narrow            sparse.py:202-214        (RN-even + overflow count)
 *   orc_bjac_apply_*      bjac.py:127-149          (k outer x t inner)
 *   orc_pcg_solve         solver.py:101-184 + policies.py:102-183
 * plus the "device order" reductions of include/mpbjac_order.h
 * (orc_plan_tiles, orc_tree_*), which replay the GPU's fixed summation
 * order so a GPU solve can be compared with this oracle bit for bit.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).  Row loops of
 * matvec and sweeps are OpenMP-parallel; every row is still accumulated
 * sequentially in ascending column order, so results do not depend on the
 * thread count.  Dots in sequential mode stay single-threaded (they define
 * the reference's order).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/mpbjac_order.h"

typedef int64_t i64;
typedef int32_t i32;
typedef uint8_t u8;

#define OMP_FOR _Pragma("omp parallel for schedule(static)")

/* ------------------------------------------------------------------------ */
/* primitives: kernels_numba.py                                             */
/* ------------------------------------------------------------------------ */

#define DEF_PRIMS(SUF, T)                                                     \
  void orc_csr_matvec_##SUF(i64 n, const i64 *rp, const i32 *ci,            \
                            const T *v, const T *x, T *out) {                 \
    OMP_FOR for (i64 i = 0; i < n; i++) {                                     \
      T acc = (T)0;                                                           \
      for (i64 jj = rp[i]; jj < rp[i + 1]; jj++) acc += v[jj] * x[ci[jj]];   \
      out[i] = acc;                                                           \
    }                                                                         \
  }                                                                           \
  void orc_sweeps_##SUF(const i64 *rp, const i32 *ci, const T *v,             \
                        const u8 *in_block, const T *diag, int t, const T *r, \
                        T *y, T *tmp, i64 rs, i64 re) {                       \
    OMP_FOR for (i64 i = rs; i < re; i++) y[i] = r[i] / diag[i];              \
    for (int s = 0; s < t - 1; s++) {                                         \
      OMP_FOR for (i64 i = rs; i < re; i++) {                                 \
        T acc = (T)0;                                                         \
        for (i64 jj = rp[i]; jj < rp[i + 1]; jj++)                            \
          if (in_block[jj]) acc += v[jj] * y[ci[jj]];                         \
        tmp[i] = acc;                                                         \
      }                                                                       \
      OMP_FOR for (i64 i = rs; i < re; i++)                                   \
        y[i] = y[i] + (r[i] - tmp[i]) / diag[i];                              \
    }                                                                         \
  }                                                                           \
  T orc_dot_seq_##SUF(i64 n, const T *x, const T *y) {                        \
    T acc = (T)0;                                                             \
    for (i64 i = 0; i < n; i++) acc += x[i] * y[i];                           \
    return acc;                                                               \
  }                                                                           \
  double orc_norm_sq_##SUF(i64 n, const T *x) {                               \
    double acc = 0.0;                                                         \
    for (i64 i = 0; i < n; i++) {                                             \
      double v = (double)x[i];                                                \
      acc += v * v;                                                           \
    }                                                                         \
    return acc;                                                               \
  }                                                                           \
  /* bjac.py:127-149.  work must hold 3n T values. */                         \
  void orc_bjac_apply_##SUF(i64 n, const i64 *rp, const i32 *ci, const T *v, \
                            const u8 *in_block, const T *diag, int k, int t,  \
                            const T *r, T *z, T *work) {                      \
    T *tmp = work, *az = work + n, *w = work + 2 * n;                         \
    orc_sweeps_##SUF(rp, ci, v, in_block, diag, t, r, z, tmp, 0, n);          \
    for (int pass = 1; pass < k; pass++) {                                    \
      orc_csr_matvec_##SUF(n, rp, ci, v, z, az);                              \
      OMP_FOR for (i64 i = 0; i < n; i++) az[i] = r[i] - az[i];               \
      orc_sweeps_##SUF(rp, ci, v, in_block, diag, t, az, w, tmp, 0, n);       \
      OMP_FOR for (i64 i = 0; i < n; i++) z[i] = z[i] + w[i];                 \
    }                                                                         \
  }

DEF_PRIMS(f64, double)
DEF_PRIMS(f32, float)

/* sparse.py:202-214: RN-even narrowing; a finite value landing on +-inf is
 * counted, the first such index reported.  Returns the count. */
i64 orc_narrow(i64 n, const double *src, float *dst, i64 *first_bad) {
  i64 count = 0;
  *first_bad = -1;
  for (i64 i = 0; i < n; i++) {
    float f = (float)src[i];
    dst[i] = f;
    if (isinf(f) && isfinite(src[i])) {
      if (count == 0) *first_bad = i;
      count++;
    }
  }
  return count;
}

/* ------------------------------------------------------------------------ */
/* device-order reductions (include/mpbjac_order.h)                         */
/* ------------------------------------------------------------------------ */

/* Tile plan.  tile_lo receives ntiles+1 row offsets (caller sizes it
 * nb + n/MPB_TILE_MAX_ROWS + 2).  *large is set when some block was cut. */
i64 orc_plan_tiles(i64 nb, const i64 *offs, const i64 *rp, i64 *tile_lo,
                   int *large) {
  i64 nt = 0, cur_lo = 0, cur_rows = 0, cur_nnz = 0;
  *large = 0;
  for (i64 b = 0; b < nb; b++) {
    i64 lo = offs[b], hi = offs[b + 1];
    i64 br = hi - lo, bz = rp[hi] - rp[lo];
    if (br > MPB_TILE_MAX_ROWS) {
      if (cur_rows > 0) { tile_lo[nt++] = cur_lo; }
      for (i64 s = lo; s < hi; s += MPB_TILE_MAX_ROWS) tile_lo[nt++] = s;
      cur_lo = hi; cur_rows = 0; cur_nnz = 0;
      *large = 1;
      continue;
    }
    if (cur_rows > 0 &&
        (cur_rows + br > MPB_TILE_MAX_ROWS || cur_nnz + bz > MPB_TILE_PACK_NNZ)) {
      tile_lo[nt++] = cur_lo;
      cur_lo = lo; cur_rows = 0; cur_nnz = 0;
    }
    cur_rows += br;
    cur_nnz += bz;
  }
  if (cur_rows > 0) tile_lo[nt++] = cur_lo;
  tile_lo[nt] = offs[nb];
  return nt;
}

static double butterfly32(double *a) {
  for (int o = 16; o >= 1; o >>= 1)
    for (int l = 0; l < o; l++) a[l] = a[l] + a[l + o];
  return a[0];
}

/* Steps 1-3 of the tile sum over `count` values given by get(i). */
static double lane_tree(i64 count, int lanes, const double *vals) {
  double s[MPB_FIN_THREADS];
  double wsum[32];
  int nw = lanes / 32;
  for (int j = 0; j < lanes; j++) {
    double acc = 0.0;
    for (i64 i = j; i < count; i += lanes) acc = acc + vals[i];
    s[j] = acc;
  }
  for (int w = 0; w < nw; w++) wsum[w] = butterfly32(s + 32 * w);
  for (int w = nw; w < 32; w++) wsum[w] = 0.0;
  return butterfly32(wsum);
}

/* Sum of per-row values vals[0..n) in device order. */
double orc_tree_sum(i64 ntiles, const i64 *tile_lo, const double *vals) {
  double *part = (double *)malloc(sizeof(double) * (ntiles > 0 ? ntiles : 1));
  OMP_FOR for (i64 t = 0; t < ntiles; t++)
    part[t] = lane_tree(tile_lo[t + 1] - tile_lo[t], MPB_TILE_THREADS,
                        vals + tile_lo[t]);
  if (ntiles <= MPB_ONE_LEVEL_TILES) {
    double total1 = lane_tree(ntiles, MPB_FIN_THREADS, part);
    free(part);
    return total1;
  }
  /* two-level global sum: chunk sums, then the sum of the chunk sums */
  i64 nch = (ntiles + MPB_CHUNK_TILES - 1) / MPB_CHUNK_TILES;
  double *csum = (double *)malloc(sizeof(double) * (nch > 0 ? nch : 1));
  for (i64 c = 0; c < nch; c++) {
    i64 t0 = c * MPB_CHUNK_TILES, t1 = t0 + MPB_CHUNK_TILES < ntiles ? t0 + MPB_CHUNK_TILES : ntiles;
    csum[c] = lane_tree(t1 - t0, MPB_CHUNK_TILES, part + t0);
  }
  double total = lane_tree(nch, MPB_FIN_THREADS, csum);
  free(csum);
  free(part);
  return total;
}

static double tree_dot(i64 n, i64 ntiles, const i64 *tile_lo, const double *x,
                       const double *y, double *scratch) {
  OMP_FOR for (i64 i = 0; i < n; i++) scratch[i] = x[i] * y[i];
  return orc_tree_sum(ntiles, tile_lo, scratch);
}

double orc_tree_dot(i64 n, i64 ntiles, const i64 *tile_lo, const double *x,
                    const double *y) {
  double *s = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
  double d = tree_dot(n, ntiles, tile_lo, x, y, s);
  free(s);
  return d;
}

/* ------------------------------------------------------------------------ */
/* PCG: solver.py:101-184 with apply_policy (policies.py:102-183)           */
/* ------------------------------------------------------------------------ */

enum { K_UNIFORM = 0, K_FIXED_LOW = 1, K_ADAPTIVE_HL = 2, K_ADAPTIVE_LH = 3 };
enum {
  E_OK = 0, E_BREAKDOWN = 1, E_INDEF_PREC = 2, E_INDEF_MAT = 3,
  E_NONFINITE = 4, E_NARROW = 5, E_BAD_RELRES = 6
};

typedef struct {
  /* matrix (fp64) and preconditioner instances */
  i64 n;
  const i64 *rp;
  const i32 *ci;
  const double *val64; /* A.values == p_high.values (bitwise copy) */
  const float *val32;  /* p_low.values (may be NULL if unused)      */
  const double *diag64;
  const float *diag32;
  const u8 *in_block;
  int k, t;
  /* policy */
  int kind;
  double adp_tol;
  /* config */
  double res_tol;
  i64 cap;
  i64 stride;
  int order; /* 0: sequential (reference numba), 1: device tile-tree */
  i64 ntiles;
  const i64 *tile_lo;
  /* fp64 preconditioner values when the preconditioner was set up from
   * another matrix of the same structure (policies.build_mixed(A2, ..) used
   * to solve A); NULL: val64.  The outer SpMV and true residuals always use
   * val64 (solver.py:154, 93-98). */
  const double *pval64;
} orc_problem;

typedef struct {
  int converged;
  i64 iterations;
  double final_true_relres;
  double r0_norm;
  int error;
  i64 err_it;
  double err_val;
  i64 overflow_count;
  i64 overflow_index;
} orc_result;

static int choose_branch(int kind, double tol, double relres, int *err) {
  /* returns 0 high, 1 low (policies.py:102-116) */
  *err = 0;
  if (!isfinite(relres) || relres < 0) { *err = 1; return 0; }
  if (kind == K_UNIFORM) return 0;
  if (kind == K_FIXED_LOW) return 1;
  if (kind == K_ADAPTIVE_HL) return relres >= tol ? 0 : 1;
  return relres >= tol ? 1 : 0;
}

static double o_dot(const orc_problem *P, const double *x, const double *y,
                    double *scratch) {
  if (P->order == 0) return orc_dot_seq_f64(P->n, x, y);
  return tree_dot(P->n, P->ntiles, P->tile_lo, x, y, scratch);
}

static double o_norm(const orc_problem *P, const double *x, double *scratch) {
  if (P->order == 0) return sqrt(orc_norm_sq_f64(P->n, x));
  return sqrt(tree_dot(P->n, P->ntiles, P->tile_lo, x, x, scratch));
}

static double o_true_relres(const orc_problem *P, const double *x,
                            const double *b, double r0, double *tmp,
                            double *scratch) {
  orc_csr_matvec_f64(P->n, P->rp, P->ci, P->val64, x, tmp);
  for (i64 i = 0; i < P->n; i++) tmp[i] = b[i] - tmp[i];
  return o_norm(P, tmp, scratch) / r0;
}

/* x holds x0 on entry (zeros when the caller passed None, has_x0 = 0).
 * trace arrays hold cap entries; true_relres NaN means "None". */
int orc_pcg_solve(const orc_problem *P, const double *b, int has_x0, double *x,
                  double *tr_relres, double *tr_true, int *tr_branch,
                  orc_result *res) {
  i64 n = P->n;
  memset(res, 0, sizeof(*res));
  res->overflow_index = -1;
  double *r = malloc(sizeof(double) * n), *z = malloc(sizeof(double) * n);
  double *p = malloc(sizeof(double) * n), *q = malloc(sizeof(double) * n);
  double *tmp = malloc(sizeof(double) * n), *scr = malloc(sizeof(double) * n);
  double *work64 = malloc(sizeof(double) * 3 * n);
  float *r32 = malloc(sizeof(float) * n), *z32 = malloc(sizeof(float) * n);
  float *work32 = malloc(sizeof(float) * 3 * n);

  if (has_x0) {
    orc_csr_matvec_f64(n, P->rp, P->ci, P->val64, x, tmp);
    for (i64 i = 0; i < n; i++) r[i] = b[i] - tmp[i];
  } else {
    memcpy(r, b, sizeof(double) * n);
  }
  double r0 = o_norm(P, r, scr);
  res->r0_norm = r0;
  if (r0 == 0.0) {
    res->converged = 1;
    goto done;
  }
  double relres = 1.0, rho_prev = 0.0;
  int have_p = 0;
  for (i64 it = 1; it <= P->cap; it++) {
    int bad;
    int branch = choose_branch(P->kind, P->adp_tol, relres, &bad);
    if (bad) { res->error = E_BAD_RELRES; res->err_it = it; res->err_val = relres; goto done; }
    if (branch == 0) {
      orc_bjac_apply_f64(n, P->rp, P->ci, P->pval64 ? P->pval64 : P->val64, P->in_block, P->diag64,
                         P->k, P->t, r, z, work64);
    } else {
      i64 fb;
      i64 cnt = orc_narrow(n, r, r32, &fb);
      if (cnt) {
        res->error = E_NARROW; res->err_it = it;
        res->overflow_count = cnt; res->overflow_index = fb;
        res->err_val = r[fb];
        goto done;
      }
      orc_bjac_apply_f32(n, P->rp, P->ci, P->val32, P->in_block, P->diag32,
                         P->k, P->t, r32, z32, work32);
      for (i64 i = 0; i < n; i++) z[i] = (double)z32[i];
    }
    double rho = o_dot(P, r, z, scr);
    if (rho == 0.0) { res->error = E_BREAKDOWN; res->err_it = it; res->err_val = rho; goto done; }
    if (rho < 0.0) { res->error = E_INDEF_PREC; res->err_it = it; res->err_val = rho; goto done; }
    if (!have_p) {
      memcpy(p, z, sizeof(double) * n);
      have_p = 1;
    } else {
      double beta = rho / rho_prev;
      for (i64 i = 0; i < n; i++) p[i] = z[i] + beta * p[i];
    }
    orc_csr_matvec_f64(n, P->rp, P->ci, P->val64, p, q);
    double pq = o_dot(P, p, q, scr);
    if (pq <= 0.0) { res->error = E_INDEF_MAT; res->err_it = it; res->err_val = pq; goto done; }
    double alpha = rho / pq;
    for (i64 i = 0; i < n; i++) x[i] = x[i] + alpha * p[i];
    for (i64 i = 0; i < n; i++) r[i] = r[i] - alpha * q[i];
    rho_prev = rho;
    double rnorm = o_norm(P, r, scr);
    if (!isfinite(rnorm)) { res->error = E_NONFINITE; res->err_it = it; res->err_val = rnorm; goto done; }
    relres = rnorm / r0;
    tr_relres[it - 1] = relres;
    tr_branch[it - 1] = branch;
    tr_true[it - 1] = (P->stride && it % P->stride == 0)
                          ? o_true_relres(P, x, b, r0, tmp, scr)
                          : NAN;
    res->iterations = it;
    if (relres <= P->res_tol) { res->converged = 1; break; }
  }
  res->final_true_relres = o_true_relres(P, x, b, r0, tmp, scr);
  /* solver.py:179-182: a converged run's last entry gets the final value */
  if (res->converged && res->iterations > 0 && isnan(tr_true[res->iterations - 1]))
    tr_true[res->iterations - 1] = res->final_true_relres;
done:
  free(r); free(z); free(p); free(q); free(tmp); free(scr); free(work64);
  free(r32); free(z32); free(work32);
  return res->error;
}

/* thread control for the CPU baseline (bench.py reports the count used) */
#ifdef _OPENMP
#include <omp.h>
void orc_set_threads(int n) { omp_set_num_threads(n); }
int orc_get_threads(void) { return omp_get_max_threads(); }
#else
void orc_set_threads(int n) { (void)n; }
int orc_get_threads(void) { return 1; }
#endif
