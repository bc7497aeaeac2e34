// mpbjac_kernels.cuh — the sm_100a kernels of the mixed-precision BJAC-PCG
// hot path.
//
// Matrix layout on the hot path: SELL-32 (sliced ELLPACK, slice height 32 =
// one warp, no row sorting).  Row r lives in slice r/32, lane r%32; its j-th
// stored entry (CSR order, i.e. ascending column) is at
// slice_ptr[r/32] + 32*j + r%32.  A warp therefore loads 32 rows' j-th entries
// with one coalesced 128/256-byte access, while every thread still owns one
// row and accumulates it sequentially in ascending column order without FMA —
// which is what makes the kernels bit-identical to the reference's
// row-sequential numba kernels (pkg/src/mpcg/kernels_numba.py:37-70).
// Padding (slice width = longest row of the slice) carries column -1 and is
// skipped, so the hot kernels need no row_ptr at all.  Each CTA owns one tile
// (whole BJAC blocks, <= 512 rows) with one thread per row.
//
// Dot products follow the fixed tile-tree order of include/mpbjac_order.h.
// The scalar steps of the recurrence (rho, alpha, beta, relres, the aMP
// branch, error flags, trace) are executed by the last CTA of the kernel that
// produces the corresponding partials (ticket in SolverState), so an
// iteration is 4 kernels (k = 2: BJAC first pass, BJAC last pass, fused
// p-update+SpMV, x/r update).
#pragma once
#include "mpbjac_device.cuh"

namespace mpb {

constexpr int kChunk = 8;  // row entries held in registers (stencils: all of them)

// SELL-32 access: slice s = r / 32 spans sp[s] .. sp[s+1] (width * 32
// entries); padding slots carry column -1 and value 0.
struct SellRow {
  int base;   // sp[s] + r % 32
  int width;  // slots of the slice
};

// ---------------------------------------------------------------------------
// scalar steps of the recurrence (solver.py:128-177, policies.py:102-116)
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

// Executed by one thread once the global sum `tot` of a step is known.
__device__ __noinline__ void scalar_step(int step, double tot, SolverState *st) {
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
      st->tr_relres[it - 1] = relres;
      st->tr_branch[it - 1] = st->branch;
      st->tr_time[it - 1] = 1e-9 * static_cast<double>(globaltimer_ns() - st->t0_ns);
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
      st->tr_true[st->last_it - 1] = sqrt(tot) / st->r0;
      st->true_pending = 0;
      break;
    }
    case kStepFinal: {
      const double v = sqrt(tot) / st->r0;
      st->final_true = v;
      if (st->converged && st->last_it > 0 && isnan(st->tr_true[st->last_it - 1])) st->tr_true[st->last_it - 1] = v;
      break;
    }
    case kStepStart: {
      st->t0_ns = globaltimer_ns();
      break;
    }
  }
}

// Tile sum in the fixed order with one thread per row (kCtaThreads = 512):
// lane j < 256 adds its rows j and j + 256 in that order (rows past `count`
// skipped), then the 256 lanes are reduced by block_tree.  Called by all
// threads; result valid in thread 0.
__device__ __forceinline__ double tile_sum(double v, int count, double *s_hi, double *ws) {
  const int tid = threadIdx.x;
  if (tid >= kTileThreads) s_hi[tid - kTileThreads] = v;
  __syncthreads();
  double acc = 0.0;
  if (tid < kTileThreads) {
    if (tid < count) acc = __dadd_rn(acc, v);
    if (tid + kTileThreads < count) acc = __dadd_rn(acc, s_hi[tid]);
  }
  return block_tree<kTileThreads>(acc, ws);
}

// Publish the tile partial; the CTA that finishes last reduces all partials
// in the fixed order and runs the scalar step (solve mode: st != null).
__device__ __forceinline__ void publish_and_finish(double tile_total, double *part, int tile, unsigned ntiles,
                                                   SolverState *st, int ticket, int step, double *ws) {
  if (!publish_last(tile_total, part, tile, st ? &st->ticket[ticket] : nullptr, ntiles)) return;
  const double tot = fin_sum(part, ntiles, ws);
  if (threadIdx.x == 0) {
    scalar_step(step, tot, st);
    st->ticket[ticket] = 0u;
  }
}

// ---------------------------------------------------------------------------
// fused block-Jacobi pass: z_out = z_in + D_b^{-1}(r - A z_in)
// (bjac.py:127-149 one outer pass; kernels_numba.py:48-70 the t inner sweeps)
// ---------------------------------------------------------------------------
template <typename T>
struct PassArgs {
  const int *sp;       // SELL slice_ptr
  const int *scol;     // SELL columns (-1 = padding)
  const T *sval;       // SELL values in storage precision
  const int *tile_lo;  // ntiles+1 row offsets
  const int *tile_bf;  // first block overlapping each tile
  const int *tile_bl;  // last block overlapping each tile
  const int *boff;     // nb+1 block offsets
  int t;
  int ntiles;
  const double *r64;   // fp64 residual, narrowed on load for T=float ...
  const T *rT;         // ... or a residual already in T (when r64 == null)
  const T *zin;        // previous pass output (null on the first pass)
  T *zout;             // storage-precision output (may be null)
  double *zout64;      // widened output (may be null)
  double *part;        // r.z tile partials (last pass, needs r64)
  unsigned long long *ovf_count;  // narrowing overflow (first pass, T=float)
  long long *ovf_first;
  T *resbuf;           // large-block path
  T *dbuf;
  SolverState *st;     // solve mode: gate + fused scalar step
  int want_branch;
};

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

// Shared tile prologue: slice pointers of the tile (s_sp) and block offsets
// (s_boff) into shared memory.
__device__ __forceinline__ void load_tile_tables(const int *sp, int lo, int hi, int *s_sp, const int *boff, int bf,
                                                 int nbk, int *s_boff) {
  const int s0 = lo >> 5, s1 = (hi + 31) >> 5;
  for (int j = threadIdx.x; j <= s1 - s0; j += blockDim.x) s_sp[j] = sp[s0 + j];
  if (s_boff != nullptr)
    for (int j = threadIdx.x; j <= nbk; j += blockDim.x) s_boff[j] = boff[bf + j] - lo;
}

__device__ __forceinline__ SellRow sell_row(const int *s_sp, int lo, int row) {
  const int s = (row >> 5) - (lo >> 5);
  SellRow r;
  r.base = s_sp[s] + (row & 31);
  r.width = (s_sp[s + 1] - s_sp[s]) >> 5;
  return r;
}

// fused pass, one tile (whole blocks) per CTA, one row per thread
template <typename T, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kCtaThreads) k_bjac_tile(const PassArgs<T> a) {
  if (gated_off(a)) return;
  __shared__ T s_w[kTileRows];
  __shared__ int s_boff[kTileRows + 2];
  __shared__ int s_sp[kTileRows / 32 + 2];
  __shared__ double s_hi[kTileThreads];
  __shared__ double ws[32];
  const int tid = threadIdx.x, tile = blockIdx.x;
  const int lo = a.tile_lo[tile], hi = a.tile_lo[tile + 1];
  const int bf = a.tile_bf[tile], nbk = a.tile_bl[tile] - bf + 1;
  const int row = lo + tid;
  const bool valid = row < hi;
  const T rv = valid ? load_residual(a, row, FIRST) : T(0);
  const T zown = (!FIRST && valid) ? __ldg(a.zin + row) : T(0);
  load_tile_tables(a.sp, lo, hi, s_sp, a.boff, bf, nbk, s_boff);
  __syncthreads();
  // (1) row scan in ascending column order: az = A z_in, the diagonal and
  //     the in-block slots (registers); rows wider than kChunk re-read
  int c[kChunk];
  T v[kChunk];
  T res = T(0), d = T(1), w = T(0);
  int blo = 0, bhi = 0;
  SellRow sr{0, 0};
  if (valid) {
    sr = sell_row(s_sp, lo, row);
    find_block(s_boff, nbk, tid, blo, bhi);
    blo += lo;
    bhi += lo;
#pragma unroll
    for (int u = 0; u < kChunk; u++) {
      const bool ok = u < sr.width;
      c[u] = ok ? __ldg(a.scol + sr.base + 32 * u) : -1;
      v[u] = ok ? __ldg(a.sval + sr.base + 32 * u) : T(0);
    }
    T g[kChunk];
    if (!FIRST) {
#pragma unroll
      for (int u = 0; u < kChunk; u++) g[u] = c[u] >= 0 ? __ldg(a.zin + c[u]) : T(0);
    }
    T az = T(0), dd = T(0);
#pragma unroll
    for (int u = 0; u < kChunk; u++) {
      if (c[u] >= 0) {
        if (!FIRST) az = add_rn(az, mul_rn(v[u], g[u]));
        if (c[u] == row) dd = v[u];
      }
    }
    for (int j = kChunk; j < sr.width; j++) {  // long rows
      const int cj = __ldg(a.scol + sr.base + 32 * j);
      if (cj < 0) continue;
      const T vj = __ldg(a.sval + sr.base + 32 * j);
      if (!FIRST) az = add_rn(az, mul_rn(vj, __ldg(a.zin + cj)));
      if (cj == row) dd = vj;
    }
    res = FIRST ? rv : sub_rn(rv, az);
    d = dd;
    w = div_rn(res, dd);
    s_w[tid] = w;
  }
  // (2) inner sweeps on the tile's blocks, w in shared memory
  for (int s = 1; s < a.t; s++) {
    __syncthreads();
    T acc = T(0);
    if (valid) {
#pragma unroll
      for (int u = 0; u < kChunk; u++)
        if (c[u] >= blo && c[u] < bhi) acc = add_rn(acc, mul_rn(v[u], s_w[c[u] - lo]));
      for (int j = kChunk; j < sr.width; j++) {
        const int cj = __ldg(a.scol + sr.base + 32 * j);
        if (cj >= blo && cj < bhi) acc = add_rn(acc, mul_rn(__ldg(a.sval + sr.base + 32 * j), s_w[cj - lo]));
      }
    }
    __syncthreads();
    if (valid) {
      w = add_rn(w, div_rn(sub_rn(res, acc), d));
      s_w[tid] = w;
    }
  }
  // (3) z_out = z_in + w (or w); r.z partial and the fused rho step
  double prod = 0.0;
  if (valid) {
    const T zo = FIRST ? w : add_rn(zown, w);
    if (a.zout != nullptr) a.zout[row] = zo;
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
    if (LAST && a.part != nullptr) prod = __dmul_rn(a.r64[row], static_cast<double>(zo));
  }
  if (LAST && a.part != nullptr) {
    const double tot = tile_sum(prod, hi - lo, s_hi, ws);
    publish_and_finish(tot, a.part, tile, a.ntiles, a.st, 0, kStepRho, ws);
  }
}

// ---- large blocks (> kTileRows rows): one launch per inner sweep ----------
// pass prologue: res = r - A z_in, d = diag, w0 = res / d
template <typename T, bool FIRST>
__global__ void __launch_bounds__(kCtaThreads) k_big_resid(const PassArgs<T> a, T *w0) {
  if (gated_off(a)) return;
  __shared__ int s_sp[kTileRows / 32 + 2];
  const int lo = a.tile_lo[blockIdx.x], hi = a.tile_lo[blockIdx.x + 1];
  load_tile_tables(a.sp, lo, hi, s_sp, nullptr, 0, 0, nullptr);
  __syncthreads();
  const int row = lo + threadIdx.x;
  if (row >= hi) return;
  const T rv = load_residual(a, row, FIRST);
  const SellRow sr = sell_row(s_sp, lo, row);
  T az = T(0), dd = T(0);
  for (int j = 0; j < sr.width; j++) {
    const int cj = __ldg(a.scol + sr.base + 32 * j);
    if (cj < 0) continue;
    const T vj = __ldg(a.sval + sr.base + 32 * j);
    if (!FIRST) az = add_rn(az, mul_rn(vj, __ldg(a.zin + cj)));
    if (cj == row) dd = vj;
  }
  const T res = FIRST ? rv : sub_rn(rv, az);
  a.resbuf[row] = res;
  a.dbuf[row] = dd;
  w0[row] = div_rn(res, dd);
}

// one inner sweep: w_new = w + (res - A_b w) / d  (A_b: in-block entries)
template <typename T>
__global__ void __launch_bounds__(kCtaThreads) k_big_sweep(const PassArgs<T> a, const T *wsrc, T *wdst) {
  if (gated_off(a)) return;
  __shared__ int s_sp[kTileRows / 32 + 2];
  const int tile = blockIdx.x;
  const int lo = a.tile_lo[tile], hi = a.tile_lo[tile + 1];
  const int bf = a.tile_bf[tile], bl = a.tile_bl[tile];
  load_tile_tables(a.sp, lo, hi, s_sp, nullptr, 0, 0, nullptr);
  __syncthreads();
  const int row = lo + threadIdx.x;
  if (row >= hi) return;
  int L = bf, H = bl + 1;
  while (H - L > 1) {
    const int M = (L + H) >> 1;
    if (a.boff[M] <= row) L = M; else H = M;
  }
  const int blo = a.boff[L], bhi = a.boff[L + 1];
  const SellRow sr = sell_row(s_sp, lo, row);
  T acc = T(0);
  for (int j = 0; j < sr.width; j++) {
    const int cj = __ldg(a.scol + sr.base + 32 * j);
    if (cj >= blo && cj < bhi) acc = add_rn(acc, mul_rn(__ldg(a.sval + sr.base + 32 * j), wsrc[cj]));
  }
  wdst[row] = add_rn(wsrc[row], div_rn(sub_rn(a.resbuf[row], acc), a.dbuf[row]));
}

template <typename T, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kCtaThreads) k_big_finish(const PassArgs<T> a, const T *w) {
  if (gated_off(a)) return;
  __shared__ double s_hi[kTileThreads];
  __shared__ double ws[32];
  const int tile = blockIdx.x;
  const int lo = a.tile_lo[tile], hi = a.tile_lo[tile + 1];
  const int row = lo + threadIdx.x;
  double prod = 0.0;
  if (row < hi) {
    const T zo = FIRST ? w[row] : add_rn(a.zin[row], w[row]);
    if (a.zout != nullptr) a.zout[row] = zo;
    if (a.zout64 != nullptr) a.zout64[row] = static_cast<double>(zo);
    if (LAST && a.part != nullptr) prod = __dmul_rn(a.r64[row], static_cast<double>(zo));
  }
  if (LAST && a.part != nullptr) {
    const double tot = tile_sum(prod, hi - lo, s_hi, ws);
    publish_and_finish(tot, a.part, tile, a.ntiles, a.st, 0, kStepRho, ws);
  }
}

// ---------------------------------------------------------------------------
// fused p-update + fp64 SpMV + p.q partial (solver.py:150-159)
//   p = z (first iteration) | z + beta * p_old ;  q = A p
// Gathered p_j are recomputed from z_j and p_old_j: bitwise the value the
// owning thread stores, so p never makes a separate HBM round trip.
// ---------------------------------------------------------------------------
struct SpmvArgs {
  const int *sp;
  const int *scol;
  const double *sval;
  const int *tile_lo;
  int ntiles;
  const float *z32;   // low-branch z (fp32; widening is exact)
  const double *z64;  // high-branch z
  double *p0, *p1;    // p ping-pong: new = p[it & 1]
  double *q;
  double *part;
  SolverState *st;
};

template <bool LOW>
__device__ __forceinline__ double spmv_row(const SpmvArgs &a, const SellRow &sr, int row, bool first, double beta,
                                           const double *pold, double *pnew) {
  auto ZJ = [&](int j) -> double {
    return LOW ? static_cast<double>(__ldg(a.z32 + j)) : __ldg(a.z64 + j);
  };
  const double zi = ZJ(row);
  const double pi = first ? zi : __dadd_rn(zi, __dmul_rn(beta, __ldg(pold + row)));
  double acc = 0.0;
  for (int j0 = 0; j0 < sr.width; j0 += kChunk) {
    int c[kChunk];
    double v[kChunk], pj[kChunk];
#pragma unroll
    for (int u = 0; u < kChunk; u++) {
      const bool ok = j0 + u < sr.width;
      c[u] = ok ? __ldg(a.scol + sr.base + 32 * (j0 + u)) : -1;
      v[u] = ok ? __ldg(a.sval + sr.base + 32 * (j0 + u)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kChunk; u++) {
      const double zg = c[u] >= 0 ? ZJ(c[u]) : 0.0;
      const double pg = (c[u] >= 0 && !first) ? __ldg(pold + c[u]) : 0.0;
      pj[u] = first ? zg : __dadd_rn(zg, __dmul_rn(beta, pg));
    }
#pragma unroll
    for (int u = 0; u < kChunk; u++)
      if (c[u] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[u], pj[u]));
  }
  pnew[row] = pi;
  a.q[row] = acc;
  return __dmul_rn(pi, acc);
}

__global__ void __launch_bounds__(kCtaThreads) k_spmv_pq(const SpmvArgs a) {
  if (a.st->done) return;
  __shared__ int s_sp[kTileRows / 32 + 2];
  __shared__ double s_hi[kTileThreads];
  __shared__ double ws[32];
  const bool low = a.st->branch == 1;
  const bool first = a.st->first != 0;
  const double beta = a.st->beta;
  const bool odd = (a.st->it & 1) != 0;
  const double *pold = odd ? a.p0 : a.p1;
  double *pnew = odd ? a.p1 : a.p0;
  const int tile = blockIdx.x;
  const int lo = a.tile_lo[tile], hi = a.tile_lo[tile + 1];
  load_tile_tables(a.sp, lo, hi, s_sp, nullptr, 0, 0, nullptr);
  __syncthreads();
  const int row = lo + threadIdx.x;
  double prod = 0.0;
  if (row < hi) {
    const SellRow sr = sell_row(s_sp, lo, row);
    prod = low ? spmv_row<true>(a, sr, row, first, beta, pold, pnew)
               : spmv_row<false>(a, sr, row, first, beta, pold, pnew);
  }
  const double tot = tile_sum(prod, hi - lo, s_hi, ws);
  publish_and_finish(tot, a.part, tile, a.ntiles, a.st, 1, kStepPq, ws);
}

// x += alpha p ; r -= alpha q ; r.r partial   (solver.py:160-165)
__global__ void __launch_bounds__(kCtaThreads)
    k_update(const int *tile_lo, int ntiles, double *x, const double *p0, const double *p1, const double *q,
             double *r, double *part, SolverState *st) {
  if (st->done) return;
  __shared__ double s_hi[kTileThreads];
  __shared__ double ws[32];
  const double alpha = st->alpha;
  const double *p = (st->it & 1) ? p1 : p0;
  const int lo = tile_lo[blockIdx.x], hi = tile_lo[blockIdx.x + 1];
  const int row = lo + threadIdx.x;
  double sq = 0.0;
  if (row < hi) {
    x[row] = __dadd_rn(x[row], __dmul_rn(alpha, p[row]));
    const double rn = __dsub_rn(r[row], __dmul_rn(alpha, q[row]));
    r[row] = rn;
    sq = __dmul_rn(rn, rn);
  }
  const double tot = tile_sum(sq, hi - lo, s_hi, ws);
  publish_and_finish(tot, part, blockIdx.x, ntiles, st, 2, kStepRr, ws);
}

// res = b - A x (or b), optionally stored; res.res partial; the last CTA runs
// `step` (R0 / True / Final) when st != null.
// gate: 0 always, 1 only when st->true_pending (strided true residual)
template <bool HAS_X>
__global__ void __launch_bounds__(kCtaThreads)
    k_resid(const int *sp, const int *scol, const double *sval, const int *tile_lo, int ntiles, const double *b,
            const double *x, double *rout, double *part, SolverState *st, int gate, int step) {
  if (gate == 1 && (st == nullptr || !st->true_pending)) return;
  __shared__ int s_sp[kTileRows / 32 + 2];
  __shared__ double s_hi[kTileThreads];
  __shared__ double ws[32];
  const int lo = tile_lo[blockIdx.x], hi = tile_lo[blockIdx.x + 1];
  if (HAS_X) {
    load_tile_tables(sp, lo, hi, s_sp, nullptr, 0, 0, nullptr);
    __syncthreads();
  }
  const int row = lo + threadIdx.x;
  double sq = 0.0;
  if (row < hi) {
    double res = b[row];
    if (HAS_X) {
      const SellRow sr = sell_row(s_sp, lo, row);
      double ax = 0.0;
      for (int j0 = 0; j0 < sr.width; j0 += kChunk) {
        int c[kChunk];
        double v[kChunk], g[kChunk];
#pragma unroll
        for (int u = 0; u < kChunk; u++) {
          const bool ok = j0 + u < sr.width;
          c[u] = ok ? __ldg(scol + sr.base + 32 * (j0 + u)) : -1;
          v[u] = ok ? __ldg(sval + sr.base + 32 * (j0 + u)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kChunk; u++) g[u] = c[u] >= 0 ? __ldg(x + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kChunk; u++)
          if (c[u] >= 0) ax = __dadd_rn(ax, __dmul_rn(v[u], g[u]));
      }
      res = __dsub_rn(res, ax);
    }
    if (rout != nullptr) rout[row] = res;
    sq = __dmul_rn(res, res);
  }
  const double tot = tile_sum(sq, hi - lo, s_hi, ws);
  publish_and_finish(tot, part, blockIdx.x, ntiles, st, 3, step, ws);
}

// one-thread scalar step (solve start: wall-clock origin of the trace)
__global__ void k_scalar_start(SolverState *st) {
  if (threadIdx.x == 0) scalar_step(kStepStart, 0.0, st);
}

__global__ void k_fill(double *p, long long n, double v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

// ---------------------------------------------------------------------------
// SELL-32 construction: slice s of rows [32s, 32s+32), entry j of row r at
// sp[s] + 32 j + r % 32 (padding: column -1 / value 0, set by memset)
// ---------------------------------------------------------------------------
template <typename E>
__global__ void k_sell_pack(long long n, const int *rp, const int *sp, const E *csr, E *sell) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const int base = sp[r >> 5] + static_cast<int>(r & 31);
    const int s = rp[r], len = rp[r + 1] - s;
    for (int j = 0; j < len; j++) sell[base + 32 * j] = csr[s + j];
  }
}

// ---------------------------------------------------------------------------
// reference backend kernels (plugin level; CSR; kernels_numba.py)
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
