// mpbjac_kernels.cuh — the sm_100a kernels of the mixed-precision BJAC-PCG
// hot path.  Thread-per-row, ascending-column accumulation without FMA
// everywhere a row sum is formed: that is what makes every kernel here
// bit-identical to the reference's row-sequential numba kernels
// (pkg/src/mpcg/kernels_numba.py:37-70).  Dot products follow the fixed
// tile-tree order of include/mpbjac_order.h.
#pragma once
#include "mpbjac_device.cuh"

namespace mpb {

// ---------------------------------------------------------------------------
// fused block-Jacobi pass: z_out = z_in + D_b^{-1}(r - A z_in)
// (bjac.py:127-149 one outer pass; kernels_numba.py:48-70 the t inner sweeps)
// ---------------------------------------------------------------------------
template <typename T>
struct PassArgs {
  const int *rp;
  const int *ci;
  const T *val;
  const int *tile_lo;  // ntiles+1 row offsets
  const int *tile_bf;  // first block overlapping each tile
  const int *tile_bl;  // last block overlapping each tile
  const int *boff;     // nb+1 block offsets
  int t;
  int cap_e;           // staged entries per tile (smem capacity)
  const double *r64;   // fp64 residual, narrowed on load for T=float ...
  const T *rT;         // ... or a residual already in T (when r64 == null)
  const T *zin;        // previous pass output (null on the first pass)
  T *zout;             // storage-precision output (may be null)
  double *zout64;      // widened output (may be null)
  double *part;        // r.z tile partials (last pass, needs r64)
  unsigned long long *ovf_count;  // narrowing overflow (first pass, T=float)
  long long *ovf_first;
  // large-block path buffers
  T *resbuf;
  T *dbuf;
  const SolverState *st;  // gate: skip when done or branch mismatch
  int want_branch;
};

__host__ __device__ constexpr uint32_t tile_smem_bytes(int cap_e, int es) {
  return region_bytes(cap_e, es) + region_bytes(cap_e, 4) +
         ((kTileRows * es + 15) / 16) * 16 + ((kTileRows + 2) * 4 + 15) / 16 * 16;
}

template <typename T>
__device__ __forceinline__ bool gated_off(const PassArgs<T> &a) {
  return a.st != nullptr && (a.st->done || a.st->branch != a.want_branch);
}

template <typename T>
__device__ __forceinline__ T load_residual(const PassArgs<T> &a, int row, bool check_ovf) {
  if (a.r64 != nullptr) {
    const double r = a.r64[row];
    const T v = narrow_or_copy<T>(r);
    if (sizeof(T) == 4 && check_ovf && a.ovf_count != nullptr && isinf(v) && isfinite(r)) {
      atomicAdd(a.ovf_count, 1ull);
      atomicMin(a.ovf_first, static_cast<long long>(row));
    }
    return v;
  }
  return a.rT[row];
}

// block [blo, bhi) containing local row rl; s_boff holds nbk+1 local offsets
__device__ __forceinline__ void find_block(const int *s_boff, int nbk, int rl, int &blo, int &bhi) {
  int L = 0, H = nbk;
  while (H - L > 1) {
    const int M = (L + H) >> 1;
    if (s_boff[M] <= rl) L = M; else H = M;
  }
  blo = s_boff[L];
  bhi = s_boff[L + 1];
}

template <typename T, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kTileThreads) k_bjac_tile(const PassArgs<T> a) {
  if (gated_off(a)) return;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ double ws[32];
  constexpr int R = kRowsPerThread;
  const int tid = threadIdx.x, tile = blockIdx.x;
  const int lo = a.tile_lo[tile], hi = a.tile_lo[tile + 1];
  const int e0 = a.rp[lo], e1 = a.rp[hi];
  const uint32_t RV = region_bytes(a.cap_e, sizeof(T)), RC = region_bytes(a.cap_e, 4);
  unsigned char *s_vraw = smem, *s_craw = smem + RV;
  T *s_w = reinterpret_cast<T *>(smem + RV + RC);
  int *s_boff = reinterpret_cast<int *>(smem + RV + RC + ((kTileRows * sizeof(T) + 15) / 16) * 16);
  const Window wv = window_of(a.val, e0, e1), wc = window_of(a.ci, e0, e1);
  const bool staged = e1 > e0 && wv.bytes <= RV && wc.bytes <= RC;
  if (staged && tid == 0) mbar_init(&mbar, 1);
  __syncthreads();
  if (staged && tid == 0) {
    mbar_arrive_expect_tx(&mbar, wv.bytes + wc.bytes);
    bulk_g2s(s_vraw, reinterpret_cast<const void *>(wv.g0), wv.bytes, &mbar);
    bulk_g2s(s_craw, reinterpret_cast<const void *>(wc.g0), wc.bytes, &mbar);
  }
  const T *sv = reinterpret_cast<const T *>(s_vraw + wv.skew);
  const int *sc = reinterpret_cast<const int *>(s_craw + wc.skew);
  const int bf = a.tile_bf[tile], nbk = a.tile_bl[tile] - bf + 1;
  for (int i = tid; i <= nbk; i += kTileThreads) s_boff[i] = a.boff[bf + i] - lo;

  // independent global loads while the bulk copies fly
  int rs[R], re[R];
  T rv[R];
#pragma unroll
  for (int m = 0; m < R; m++) {
    const int row = lo + tid + m * kTileThreads;
    rs[m] = re[m] = 0;
    rv[m] = T(0);
    if (row < hi) {
      rs[m] = a.rp[row];
      re[m] = a.rp[row + 1];
      rv[m] = load_residual(a, row, FIRST);
    }
  }
  __syncthreads();
  if (staged) mbar_wait(&mbar, 0);

  auto VAL = [&](int e) -> T { return staged ? sv[e - e0] : __ldg(a.val + e); };
  auto COL = [&](int e) -> int { return staged ? sc[e - e0] : __ldg(a.ci + e); };

  T res[R], d[R], w[R];
  int ib0[R], ib1[R];
#pragma unroll
  for (int m = 0; m < R; m++) {
    const int row = lo + tid + m * kTileThreads;
    res[m] = d[m] = w[m] = T(0);
    ib0[m] = ib1[m] = 0;
    if (row >= hi) continue;
    int blo, bhi;
    find_block(s_boff, nbk, row - lo, blo, bhi);
    blo += lo;
    bhi += lo;
    T az = T(0), dd = T(0);
    int i0 = re[m], i1 = re[m];
    for (int e = rs[m]; e < re[m]; e++) {
      const int c = COL(e);
      const T v = VAL(e);
      if (!FIRST) az = add_rn(az, mul_rn(v, __ldg(a.zin + c)));
      if (c == row) dd = v;
      if (c >= blo && i0 == re[m]) i0 = e;
      if (c >= bhi && i1 == re[m]) i1 = e;
    }
    res[m] = FIRST ? rv[m] : sub_rn(rv[m], az);
    d[m] = dd;
    ib0[m] = i0;
    ib1[m] = i1;
    w[m] = div_rn(res[m], dd);
    s_w[row - lo] = w[m];
  }
  for (int s = 1; s < a.t; s++) {
    __syncthreads();
    T tmp[R];
#pragma unroll
    for (int m = 0; m < R; m++) {
      T acc = T(0);
      for (int e = ib0[m]; e < ib1[m]; e++) acc = add_rn(acc, mul_rn(VAL(e), s_w[COL(e) - lo]));
      tmp[m] = acc;
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < R; m++) {
      const int row = lo + tid + m * kTileThreads;
      if (row >= hi) continue;
      w[m] = add_rn(w[m], div_rn(sub_rn(res[m], tmp[m]), d[m]));
      s_w[row - lo] = w[m];
    }
  }
  double part = 0.0;
#pragma unroll
  for (int m = 0; m < R; m++) {
    const int row = lo + tid + m * kTileThreads;
    if (row >= hi) continue;
    const T zo = FIRST ? w[m] : add_rn(__ldg(a.zin + row), w[m]);
    if (a.zout != nullptr) a.zout[row] = zo;
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
    if (LAST && a.part != nullptr) part = __dadd_rn(part, __dmul_rn(a.r64[row], static_cast<double>(zo)));
  }
  if (LAST && a.part != nullptr) {
    const double tot = block_tree<kTileThreads>(part, ws);
    if (tid == 0) a.part[tile] = tot;
  }
}

// ---- large blocks (> kTileRows rows): one launch per inner sweep ----------
// pass prologue: res = r - A z_in, d = diag, w0 = res / d
template <typename T, bool FIRST>
__global__ void __launch_bounds__(kTileThreads) k_big_resid(const PassArgs<T> a, T *w0) {
  if (gated_off(a)) return;
  const int lo = a.tile_lo[blockIdx.x], hi = a.tile_lo[blockIdx.x + 1];
  for (int row = lo + threadIdx.x; row < hi; row += kTileThreads) {
    const T rv = load_residual(a, row, FIRST);
    T az = T(0), dd = T(0);
    for (int e = a.rp[row]; e < a.rp[row + 1]; e++) {
      const int c = __ldg(a.ci + e);
      const T v = __ldg(a.val + e);
      if (!FIRST) az = add_rn(az, mul_rn(v, __ldg(a.zin + c)));
      if (c == row) dd = v;
    }
    const T res = FIRST ? rv : sub_rn(rv, az);
    a.resbuf[row] = res;
    a.dbuf[row] = dd;
    w0[row] = div_rn(res, dd);
  }
}

// one inner sweep: w_new = w + (res - A_b w) / d  (A_b: in-block entries)
template <typename T>
__global__ void __launch_bounds__(kTileThreads) k_big_sweep(const PassArgs<T> a, const T *wsrc, T *wdst) {
  if (gated_off(a)) return;
  const int tile = blockIdx.x;
  const int lo = a.tile_lo[tile], hi = a.tile_lo[tile + 1];
  const int bf = a.tile_bf[tile], bl = a.tile_bl[tile];
  for (int row = lo + threadIdx.x; row < hi; row += kTileThreads) {
    int L = bf, H = bl + 1;
    while (H - L > 1) {
      const int M = (L + H) >> 1;
      if (a.boff[M] <= row) L = M; else H = M;
    }
    const int blo = a.boff[L], bhi = a.boff[L + 1];
    T acc = T(0);
    for (int e = a.rp[row]; e < a.rp[row + 1]; e++) {
      const int c = __ldg(a.ci + e);
      if (c >= blo && c < bhi) acc = add_rn(acc, mul_rn(__ldg(a.val + e), wsrc[c]));
    }
    wdst[row] = add_rn(wsrc[row], div_rn(sub_rn(a.resbuf[row], acc), a.dbuf[row]));
  }
}

template <typename T, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kTileThreads) k_big_finish(const PassArgs<T> a, const T *w) {
  if (gated_off(a)) return;
  __shared__ double ws[32];
  const int tile = blockIdx.x;
  const int lo = a.tile_lo[tile], hi = a.tile_lo[tile + 1];
  double part = 0.0;
  for (int row = lo + threadIdx.x; row < hi; row += kTileThreads) {
    const T zo = FIRST ? w[row] : add_rn(a.zin[row], w[row]);
    if (a.zout != nullptr) a.zout[row] = zo;
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
    if (LAST && a.part != nullptr) part = __dadd_rn(part, __dmul_rn(a.r64[row], static_cast<double>(zo)));
  }
  if (LAST && a.part != nullptr) {
    const double tot = block_tree<kTileThreads>(part, ws);
    if (threadIdx.x == 0) a.part[tile] = tot;
  }
}

// ---------------------------------------------------------------------------
// fused p-update + fp64 SpMV + p.q partial (solver.py:150-155)
//   p = z (first iteration) | z + beta * p_old ; q = A p
// The gathered p_j are recomputed from z_j and p_old_j (bitwise the same
// value every CTA computes), so p never makes a separate HBM round trip.
// ---------------------------------------------------------------------------
struct SpmvArgs {
  const int *rp;
  const int *ci;
  const double *val;
  const int *tile_lo;
  int cap_e;
  const float *z32;   // low-branch z (fp32; widening is exact)
  const double *z64;  // high-branch z
  double *p0, *p1;    // p ping-pong: new = p[it & 1]
  double *q;
  double *part;
  const SolverState *st;
};

__global__ void __launch_bounds__(kTileThreads) k_spmv_pq(const SpmvArgs a) {
  if (a.st->done) return;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ double ws[32];
  constexpr int R = kRowsPerThread;
  const bool low = a.st->branch == 1;
  const bool first = a.st->first != 0;
  const double beta = a.st->beta;
  const bool odd = (a.st->it & 1) != 0;
  const double *pold = odd ? a.p0 : a.p1;
  double *pnew = odd ? a.p1 : a.p0;
  const int tid = threadIdx.x, tile = blockIdx.x;
  const int lo = a.tile_lo[tile], hi = a.tile_lo[tile + 1];
  const int e0 = a.rp[lo], e1 = a.rp[hi];
  const uint32_t RV = region_bytes(a.cap_e, 8), RC = region_bytes(a.cap_e, 4);
  unsigned char *s_vraw = smem, *s_craw = smem + RV;
  const Window wv = window_of(a.val, e0, e1), wc = window_of(a.ci, e0, e1);
  const bool staged = e1 > e0 && wv.bytes <= RV && wc.bytes <= RC;
  if (staged && tid == 0) mbar_init(&mbar, 1);
  __syncthreads();
  if (staged && tid == 0) {
    mbar_arrive_expect_tx(&mbar, wv.bytes + wc.bytes);
    bulk_g2s(s_vraw, reinterpret_cast<const void *>(wv.g0), wv.bytes, &mbar);
    bulk_g2s(s_craw, reinterpret_cast<const void *>(wc.g0), wc.bytes, &mbar);
  }
  const double *sv = reinterpret_cast<const double *>(s_vraw + wv.skew);
  const int *sc = reinterpret_cast<const int *>(s_craw + wc.skew);
  auto PJ = [&](int j) -> double {
    const double zj = low ? static_cast<double>(__ldg(a.z32 + j)) : __ldg(a.z64 + j);
    return first ? zj : __dadd_rn(zj, __dmul_rn(beta, __ldg(pold + j)));
  };
  int rs[R], re[R];
  double pi[R];
#pragma unroll
  for (int m = 0; m < R; m++) {
    const int row = lo + tid + m * kTileThreads;
    rs[m] = re[m] = 0;
    pi[m] = 0.0;
    if (row < hi) {
      rs[m] = a.rp[row];
      re[m] = a.rp[row + 1];
      pi[m] = PJ(row);
    }
  }
  if (staged) mbar_wait(&mbar, 0);
  double part = 0.0;
#pragma unroll
  for (int m = 0; m < R; m++) {
    const int row = lo + tid + m * kTileThreads;
    if (row >= hi) continue;
    double acc = 0.0;
    for (int e = rs[m]; e < re[m]; e++) {
      const int c = staged ? sc[e - e0] : __ldg(a.ci + e);
      const double v = staged ? sv[e - e0] : __ldg(a.val + e);
      acc = __dadd_rn(acc, __dmul_rn(v, PJ(c)));
    }
    pnew[row] = pi[m];
    a.q[row] = acc;
    part = __dadd_rn(part, __dmul_rn(pi[m], acc));
  }
  const double tot = block_tree<kTileThreads>(part, ws);
  if (tid == 0) a.part[tile] = tot;
}

// x += alpha p ; r -= alpha q ; r.r partial   (solver.py:160-165)
__global__ void __launch_bounds__(kTileThreads)
    k_update(const int *tile_lo, double *x, const double *p0, const double *p1, const double *q,
             double *r, double *part, const SolverState *st) {
  if (st->done) return;
  __shared__ double ws[32];
  const double alpha = st->alpha;
  const double *p = (st->it & 1) ? p1 : p0;
  const int lo = tile_lo[blockIdx.x], hi = tile_lo[blockIdx.x + 1];
  double acc = 0.0;
  for (int row = lo + threadIdx.x; row < hi; row += kTileThreads) {
    x[row] = __dadd_rn(x[row], __dmul_rn(alpha, p[row]));
    const double rn = __dsub_rn(r[row], __dmul_rn(alpha, q[row]));
    r[row] = rn;
    acc = __dadd_rn(acc, __dmul_rn(rn, rn));
  }
  const double tot = block_tree<kTileThreads>(acc, ws);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// res = b - A x (or b), optionally stored; res.res partial.
// gate: 0 always, 1 only when st->true_pending (strided true residual)
template <bool HAS_X>
__global__ void __launch_bounds__(kTileThreads)
    k_resid(const int *rp, const int *ci, const double *val, const int *tile_lo, const double *b,
            const double *x, double *rout, double *part, const SolverState *st, int gate) {
  if (gate == 1 && (st == nullptr || !st->true_pending)) return;
  __shared__ double ws[32];
  const int lo = tile_lo[blockIdx.x], hi = tile_lo[blockIdx.x + 1];
  double acc = 0.0;
  for (int row = lo + threadIdx.x; row < hi; row += kTileThreads) {
    double res = b[row];
    if (HAS_X) {
      double ax = 0.0;
      for (int e = rp[row]; e < rp[row + 1]; e++)
        ax = __dadd_rn(ax, __dmul_rn(__ldg(val + e), __ldg(x + __ldg(ci + e))));
      res = __dsub_rn(res, ax);
    }
    if (rout != nullptr) rout[row] = res;
    acc = __dadd_rn(acc, __dmul_rn(res, res));
  }
  const double tot = block_tree<kTileThreads>(acc, ws);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// ---------------------------------------------------------------------------
// scalar steps of the recurrence, one CTA (solver.py:128-177, policies.py:102-116)
// ---------------------------------------------------------------------------
enum ScalarStep { kStepR0 = 0, kStepRho = 1, kStepPq = 2, kStepRr = 3, kStepTrue = 4, kStepFinal = 5, kStepStart = 6 };

__device__ __forceinline__ int choose_branch(int kind, double tol, double relres) {
  if (kind == 0) return 0;
  if (kind == 1) return 1;
  if (kind == 2) return relres >= tol ? 0 : 1;
  return relres >= tol ? 1 : 0;
}

__device__ __forceinline__ void fail(SolverState *st, int code, double val) {
  st->error = code;
  st->err_it = st->it;
  st->err_val = val;
  st->done = 1;
}

__global__ void __launch_bounds__(kFinThreads)
    k_scalar(int step, const double *part, long long nparts, SolverState *st, double *tr_relres,
             double *tr_true, int *tr_branch, double *tr_time) {
  __shared__ double ws[32];
  if (step == kStepStart) {
    if (threadIdx.x == 0) st->t0_ns = globaltimer_ns();
    return;
  }
  if (step == kStepTrue) {
    if (!st->true_pending) return;
  } else if (step != kStepFinal && step != kStepR0 && st->done) {
    return;
  }
  const double tot = fin_sum(part, nparts, ws);
  if (threadIdx.x != 0) return;
  switch (step) {
    case kStepR0: {
      st->r0 = sqrt(tot);
      st->relres = 1.0;
      st->it = 1;
      st->first = 1;
      st->branch = choose_branch(st->kind, st->adp_tol, 1.0);
      if (st->r0 == 0.0) {
        st->converged = 1;
        st->done = 1;
      }
      break;
    }
    case kStepRho: {
      if (st->ovf_count != 0ull) {
        fail(st, kNarrowOverflow, 0.0);
        break;
      }
      st->rho = tot;
      if (tot == 0.0) { fail(st, kBreakdown, tot); break; }
      if (tot < 0.0) { fail(st, kIndefPrecond, tot); break; }
      st->beta = st->first ? 0.0 : tot / st->rho_prev;
      break;
    }
    case kStepPq: {
      st->pq = tot;
      if (tot <= 0.0) { fail(st, kIndefMatrix, tot); break; }
      st->alpha = st->rho / tot;
      break;
    }
    case kStepRr: {
      const double rnorm = sqrt(tot);
      st->rnorm = rnorm;
      st->rho_prev = st->rho;
      st->first = 0;
      if (!isfinite(rnorm)) { fail(st, kNonFinite, rnorm); break; }
      const double relres = rnorm / st->r0;
      st->relres = relres;
      const long long it = st->it;
      tr_relres[it - 1] = relres;
      tr_branch[it - 1] = st->branch;
      tr_time[it - 1] = 1e-9 * static_cast<double>(globaltimer_ns() - st->t0_ns);
      st->last_it = it;
      st->true_pending = (st->stride > 0 && it % st->stride == 0) ? 1 : 0;
      if (relres <= st->res_tol) {
        st->converged = 1;
        st->done = 1;
      } else if (it >= st->cap) {
        st->done = 1;
      } else {
        st->it = it + 1;
        st->branch = choose_branch(st->kind, st->adp_tol, relres);
      }
      break;
    }
    case kStepTrue: {
      tr_true[st->last_it - 1] = sqrt(tot) / st->r0;
      st->true_pending = 0;
      break;
    }
    case kStepFinal: {
      const double v = sqrt(tot) / st->r0;
      st->final_true = v;
      if (st->converged && st->last_it > 0 && isnan(tr_true[st->last_it - 1])) tr_true[st->last_it - 1] = v;
      break;
    }
  }
}

__global__ void k_fill(double *p, long long n, double v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

// ---------------------------------------------------------------------------
// reference backend kernels (plugin level; kernels_numba.py)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_matvec(long long n, const int *rp, const int *ci, const T *val, const T *x, T *y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++) acc = add_rn(acc, mul_rn(__ldg(val + e), __ldg(x + __ldg(ci + e))));
    y[i] = acc;
  }
}

template <typename T>
__global__ void k_msweep_init(long long rs, long long re, const T *r, const T *diag, T *y) {
  for (long long i = rs + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < re; i += (long long)gridDim.x * blockDim.x)
    y[i] = div_rn(r[i], diag[i]);
}
template <typename T>
__global__ void k_msweep_tmp(long long rs, long long re, const int *rp, const int *ci, const T *val,
                             const uint8_t *mask, const T *y, T *tmp) {
  for (long long i = rs + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < re; i += (long long)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++)
      if (mask[e]) acc = add_rn(acc, mul_rn(val[e], y[ci[e]]));
    tmp[i] = acc;
  }
}
template <typename T>
__global__ void k_msweep_upd(long long rs, long long re, const T *r, const T *diag, const T *tmp, T *y) {
  for (long long i = rs + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < re; i += (long long)gridDim.x * blockDim.x)
    y[i] = add_rn(y[i], div_rn(sub_rn(r[i], tmp[i]), diag[i]));
}

// inner_apply on one block [lo, hi): block-local vectors, mask = [lo, hi)
template <typename T>
__global__ void k_inner_init(int lo, int hi, const int *rp, const int *ci, const T *val, const T *rb, T *db, T *yb) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    T dd = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++)
      if (ci[e] == i) dd = val[e];
    db[i - lo] = dd;
    yb[i - lo] = div_rn(rb[i - lo], dd);
  }
}
template <typename T>
__global__ void k_inner_sweep(int lo, int hi, const int *rp, const int *ci, const T *val, const T *rb, const T *db,
                              const T *ysrc, T *ydst) {
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++) {
      const int c = ci[e];
      if (c >= lo && c < hi) acc = add_rn(acc, mul_rn(val[e], ysrc[c - lo]));
    }
    ydst[i - lo] = add_rn(ysrc[i - lo], div_rn(sub_rn(rb[i - lo], acc), db[i - lo]));
  }
}

// per-tile sum of x*y (SQ: y ignored, x widened and squared); tile_lo may be
// null (uniform kTileRows-row tiles)
template <typename T, typename ACC, bool SQ>
__global__ void __launch_bounds__(kTileThreads)
    k_tile_dot(long long n, const int *tile_lo, const T *x, const T *y, ACC *part) {
  __shared__ ACC ws[32];
  long long lo, hi;
  if (tile_lo != nullptr) {
    lo = tile_lo[blockIdx.x];
    hi = tile_lo[blockIdx.x + 1];
  } else {
    lo = (long long)blockIdx.x * kTileRows;
    hi = lo + kTileRows < n ? lo + kTileRows : n;
  }
  ACC acc = ACC(0);
  for (long long i = lo + threadIdx.x; i < hi; i += kTileThreads) {
    if (SQ) {
      const ACC v = static_cast<ACC>(x[i]);
      acc = add_rn(acc, mul_rn(v, v));
    } else {
      acc = add_rn(acc, mul_rn(static_cast<ACC>(x[i]), static_cast<ACC>(y[i])));
    }
  }
  const ACC tot = block_tree<kTileThreads>(acc, ws);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

template <typename ACC>
__global__ void __launch_bounds__(kFinThreads) k_fin(const ACC *part, long long nparts, ACC *out) {
  __shared__ ACC ws[32];
  ACC acc = ACC(0);
  for (long long i = threadIdx.x; i < nparts; i += kFinThreads) acc = add_rn(acc, part[i]);
  const ACC tot = block_tree<kFinThreads>(acc, ws);
  if (threadIdx.x == 0) *out = tot;
}

// RN-even narrowing with overflow count / first index (sparse.py:202-214)
__global__ void k_narrow(long long n, const double *src, float *dst, unsigned long long *cnt, long long *first) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = src[i];
    const float f = __double2float_rn(v);
    dst[i] = f;
    if (isinf(f) && isfinite(v)) {
      atomicAdd(cnt, 1ull);
      atomicMin(first, i);
    }
  }
}
__global__ void k_widen(long long n, const float *src, double *dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = static_cast<double>(src[i]);
}

// stored diagonal per row (bjac.py:171-185); missing / zero reported by row
template <typename T>
__global__ void k_setup_diag(long long n, const int *rp, const int *ci, const T *val, T *diag, long long *missing,
                             long long *zero) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    bool have = false;
    T dd = T(0);
    for (int e = rp[i]; e < rp[i + 1]; e++)
      if (ci[e] == i) {
        have = true;
        dd = val[e];
      }
    diag[i] = dd;
    if (!have) atomicMin(missing, i);
    else if (dd == T(0)) atomicMin(zero, i);
  }
}

}  // namespace mpb
