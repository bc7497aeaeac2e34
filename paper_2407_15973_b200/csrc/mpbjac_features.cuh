// mpbjac_features.cuh — row-wise structural features of a CSR matrix on the
// device (pkg/src/mpcg/features.py:41-211 restated): multiscale strength
// tau_i = max|a_ij| / min|a_ij| over stored nonzero off-diagonals, diagonal
// dominance |a_ii| / sum_{j!=i} |a_ij|, signed and absolute row sums, the
// tau histogram, vector statistics (min / median / max / count above), and
// the first k violations of the M-matrix sign checks in index order.
//
// Row sums follow numpy's ufunc.reduceat order exactly (features.py:31-38
// sums with np.add.reduceat): a segment a[0..m) sums to a[0] + pairwise(a[1..m)),
// pairwise(p, n) = (-0.0 + p0) + p1 ... for n < 8; eight strided accumulators
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail for
// n <= 128; else split at n/2 rounded down to a multiple of 8.  So every
// per-row value is bit-identical to the reference's.
#pragma once
#include <cstdint>

#include "mpbjac_device.cuh"

namespace mpb {

// numpy pairwise_sum for n <= 128 (no recursion; inlined)
template <typename F>
__device__ __forceinline__ double np_pairwise_small(const F &f, long long i0, long long n) {
  if (n < 8) {
    double r = -0.0;
    for (long long i = 0; i < n; i++) r = __dadd_rn(r, f(i0 + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = f(i0 + j);
  long long i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], f(i0 + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; i++) res = __dadd_rn(res, f(i0 + i));
  return res;
}
// the recursive split for longer segments (rare: rows of more than 129 entries)
template <typename F>
__device__ __noinline__ double np_pairwise_big(const F &f, long long i0, long long n) {
  long long n2 = n / 2;
  n2 -= n2 % 8;
  const double a = n2 <= 128 ? np_pairwise_small(f, i0, n2) : np_pairwise_big(f, i0, n2);
  const double b = n - n2 <= 128 ? np_pairwise_small(f, i0 + n2, n - n2) : np_pairwise_big(f, i0 + n2, n - n2);
  return __dadd_rn(a, b);
}
// np.add.reduceat of one nonempty segment [lo, lo + m)
template <typename F>
__device__ __forceinline__ double np_segment_sum(const F &f, long long lo, long long m) {
  const double rest = m - 1 <= 128 ? np_pairwise_small(f, lo + 1, m - 1) : np_pairwise_big(f, lo + 1, m - 1);
  return __dadd_rn(f(lo), rest);
}

// One thread per row (features.py:41-55 multiscale_profile, :127-152
// dominance_stats, :171-211 m_matrix_sign_check's sums).  V: the stored
// value type; every quantity is computed from the value widened to fp64.
template <typename V>
__global__ void k_row_features(long long n, const int32_t *rp, const int32_t *ci, const V *val, double *tau,
                               double *dom, double *rsum, double *asum, double *diag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long lo = rp[i], hi = rp[i + 1], m = hi - lo;
    double mx = -INFINITY, mn = INFINITY, dg = 0.0;
    bool nan = false;
    for (long long e = lo; e < hi; e++) {
      const double v = static_cast<double>(val[e]);
      if (ci[e] == i) {
        dg = v;
      } else if (val[e] != V(0)) {  // qualifying: off-diagonal, stored nonzero
        const double a = fabs(v);
        if (isnan(a)) nan = true;
        mx = fmax(mx, a);
        mn = fmin(mn, a);
      }
    }
    // np.maximum / np.minimum propagate NaN; defined = isfinite(row max)
    const bool defined = !nan && isfinite(mx);
    if (tau) tau[i] = defined ? __ddiv_rn(mx, mn) : NAN;
    if (diag) diag[i] = dg;
    if (dom) {
      const double off = m == 0 ? 0.0
                                : np_segment_sum([&](long long e) { return ci[e] != i ? fabs(static_cast<double>(val[e])) : 0.0; },
                                                 lo, m);
      dom[i] = off == 0.0 ? INFINITY : __ddiv_rn(fabs(dg), off);
    }
    if (rsum) rsum[i] = m == 0 ? 0.0 : np_segment_sum([&](long long e) { return static_cast<double>(val[e]); }, lo, m);
    if (asum) asum[i] = m == 0 ? 0.0 : np_segment_sum([&](long long e) { return fabs(static_cast<double>(val[e])); }, lo, m);
  }
}

// Lower-inclusive bins (features.py:94-113): bin = #{edges <= tau} - 1 for
// defined rows (tau not NaN; tau >= 1 >= edges[0]); NaN counts as undefined.
constexpr int kMaxEdges = 64;
__global__ void k_tau_histogram(long long n, const double *tau, const double *edges, int nedges,
                                unsigned long long *counts /* nedges + 1: last = undefined */) {
  __shared__ unsigned long long s_cnt[kMaxEdges + 1];
  __shared__ double s_edges[kMaxEdges];
  for (int j = threadIdx.x; j <= nedges; j += blockDim.x) s_cnt[j] = 0ull;
  for (int j = threadIdx.x; j < nedges; j += blockDim.x) s_edges[j] = edges[j];
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double t = tau[i];
    if (isnan(t)) {
      atomicAdd(&s_cnt[nedges], 1ull);
      continue;
    }
    int lo = 0, hi = nedges;  // first edge > t
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s_edges[mid] <= t) lo = mid + 1; else hi = mid;
    }
    atomicAdd(&s_cnt[lo - 1], 1ull);
  }
  __syncthreads();
  for (int j = threadIdx.x; j <= nedges; j += blockDim.x)
    if (s_cnt[j]) atomicAdd(&counts[j], s_cnt[j]);
}

// order-preserving map of doubles to unsigned 64-bit keys (for atomic min/max)
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double dkey_inv(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double d;
  static_assert(sizeof(d) == sizeof(b), "double bits");
  __builtin_memcpy(&d, &b, sizeof(d));
  return d;
#endif
}
// acc[0] min key, acc[1] max key, acc[2] NaN seen, acc[3] count of x > thresh
__global__ void k_vector_stats(long long n, const double *x, double thresh, unsigned long long *acc) {
  unsigned long long kmin = ~0ull, kmax = 0ull, nan = 0ull, cnt = 0ull;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = x[i];
    if (isnan(v)) {
      nan = 1ull;
      continue;
    }
    const unsigned long long k = dkey(v);
    kmin = k < kmin ? k : kmin;
    kmax = k > kmax ? k : kmax;
    if (v > thresh) cnt++;
  }
  for (int o = 16; o >= 1; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
    kmin = a < kmin ? a : kmin;
    kmax = b > kmax ? b : kmax;
    nan |= __shfl_xor_sync(0xffffffffu, nan, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&acc[0], kmin);
    atomicMax(&acc[1], kmax);
    if (nan) atomicOr(&acc[2], 1ull);
    if (cnt) atomicAdd(&acc[3], cnt);
  }
}

// First k flagged items in index order, per block of kFlagBlock items:
// block b stores the first min(k, count_b) of its flagged indices at
// out[b*k..] and its count at cnt[b] (items base + b*kFlagBlock + ...).
// kind 0: !(a[i] > 0); 1: a[i] < -(tol * b[i]); 2: entry i is off-diagonal
// with value > 0 (row from a binary search of row_ptr).
constexpr int kFlagBlock = 1024;
template <typename V>
__device__ __forceinline__ bool violation(int kind, long long i, const double *a, const double *b, double tol,
                                          const int32_t *rp, long long nrows, const int32_t *ci, const V *val) {
  if (kind == 0) return !(a[i] > 0.0);
  if (kind == 1) return a[i] < -(tol * b[i]);
  if (!(val[i] > V(0))) return false;
  long long L = 0, H = nrows;  // row r with rp[r] <= i < rp[r+1]
  while (H - L > 1) {
    const long long M = (L + H) >> 1;
    if (rp[M] <= i) L = M; else H = M;
  }
  return ci[i] != L;
}
template <typename V>
__global__ void __launch_bounds__(256) k_first_flags(int kind, long long n, long long base, const double *a,
                                                     const double *b, double tol, const int32_t *rp, long long nrows,
                                                     const int32_t *ci, const V *val, int k, long long *out,
                                                     int *cnt) {
  __shared__ int s_total;
  __shared__ int s_warp[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_total = 0;
  __syncthreads();
  const long long start = base + (long long)blockIdx.x * kFlagBlock;
  for (int j = 0; j < kFlagBlock / 256; j++) {
    const long long i = start + j * 256 + threadIdx.x;
    const bool f = i < n && violation<V>(kind, i, a, b, tol, rp, nrows, ci, val);
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int before = s_total;
    for (int w = 0; w < warp; w++) before += s_warp[w];
    const int pos = before + __popc(m & ((1u << lane) - 1u));
    if (f && pos < k) out[(long long)blockIdx.x * k + pos] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = 0;
      for (int w = 0; w < 8; w++) s += s_warp[w];
      s_total += s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) cnt[blockIdx.x] = s_total;
}

}  // namespace mpb
