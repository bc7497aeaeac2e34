// Micro-benchmark: the x/r update (x += a p; r -= a q; r.r tile partials)
// over 2^21 rows in several launch shapes, to see what bounds k_update.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream stream.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

constexpr int T = 256;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double block_sum(double v, double *ws) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = threadIdx.x < T / 32 ? ws[threadIdx.x] : 0.0;
  if (threadIdx.x < 32) t = warp_sum(t);
  __syncthreads();
  return t;
}

// 1: persistent, U tiles per batch, all loads up front
template <int U>
__global__ void __launch_bounds__(T) k_persist(int ntiles, double *x, const double *p, const double *q, double *r,
                                               double *part, double a) {
  __shared__ double ws[32];
  for (int t0 = blockIdx.x; t0 < ntiles; t0 += U * gridDim.x) {
    double xv[U], pv[U], qv[U], rv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int tile = t0 + u * gridDim.x;
      const int row = tile * T + threadIdx.x;
      const bool ok = tile < ntiles;
      xv[u] = ok ? x[row] : 0;
      pv[u] = ok ? p[row] : 0;
      qv[u] = ok ? q[row] : 0;
      rv[u] = ok ? r[row] : 0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int tile = t0 + u * gridDim.x;
      if (tile >= ntiles) break;
      const int row = tile * T + threadIdx.x;
      x[row] = xv[u] + a * pv[u];
      const double rn = rv[u] - a * qv[u];
      r[row] = rn;
      const double s = block_sum(rn * rn, ws);
      if (threadIdx.x == 0) part[tile] = s;
    }
  }
}

// 2: one tile per CTA, non-persistent
__global__ void __launch_bounds__(T) k_tile(int ntiles, double *x, const double *p, const double *q, double *r,
                                            double *part, double a) {
  __shared__ double ws[32];
  const int tile = blockIdx.x, row = tile * T + threadIdx.x;
  const double xv = x[row], pv = p[row], qv = q[row], rv = r[row];
  x[row] = xv + a * pv;
  const double rn = rv - a * qv;
  r[row] = rn;
  const double s = block_sum(rn * rn, ws);
  if (threadIdx.x == 0) part[tile] = s;
}

// 3: plain streaming, no reduction, grid-stride, 2 rows per thread (double2)
__global__ void __launch_bounds__(T) k_plain(long long n2, double2 *x, const double2 *p, const double2 *q,
                                             double2 *r, double a) {
  for (long long i = blockIdx.x * (long long)T + threadIdx.x; i < n2; i += (long long)gridDim.x * T) {
    double2 xv = x[i], pv = p[i], qv = q[i], rv = r[i];
    xv.x += a * pv.x; xv.y += a * pv.y;
    rv.x -= a * qv.x; rv.y -= a * qv.y;
    x[i] = xv; r[i] = rv;
  }
}

// 4: read-only (4 streams), reduction per tile (isolates write cost)
__global__ void __launch_bounds__(T) k_readonly(int ntiles, const double *x, const double *p, const double *q,
                                                const double *r, double *part) {
  __shared__ double ws[32];
  const int tile = blockIdx.x, row = tile * T + threadIdx.x;
  const double s = block_sum(x[row] + p[row] + q[row] + r[row], ws);
  if (threadIdx.x == 0) part[tile] = s;
}

// 5: plain copy a -> b (the peak reference)
__global__ void __launch_bounds__(T) k_copy(long long n2, const double2 *a, double2 *b) {
  for (long long i = blockIdx.x * (long long)T + threadIdx.x; i < n2; i += (long long)gridDim.x * T) b[i] = a[i];
}

int main() {
  const int n = 1 << 21, ntiles = n / T;
  double *x, *p, *q, *r, *part, *flush;
  cudaMalloc(&x, 8LL * n); cudaMalloc(&p, 8LL * n); cudaMalloc(&q, 8LL * n); cudaMalloc(&r, 8LL * n);
  cudaMalloc(&part, 8LL * ntiles);
  const size_t fl = 512ull << 20;
  cudaMalloc(&flush, fl);
  cudaMemset(x, 0, 8LL * n); cudaMemset(p, 0, 8LL * n); cudaMemset(q, 0, 8LL * n); cudaMemset(r, 0, 8LL * n);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char *name, double bytes, auto launch) {
    float best = 1e9, sum = 0;
    const int reps = 50;
    for (int i = 0; i < reps + 3; i++) {
      cudaMemsetAsync(flush, i, fl);  // evict L2
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (i >= 3) { best = ms < best ? ms : best; sum += ms; }
    }
    printf("%-34s best %7.2f us  mean %7.2f us  %7.1f GB/s (best)\n", name, best * 1e3, sum / reps * 1e3,
           bytes / (best * 1e-3) / 1e9);
  };
  const double B = 48.0 * n;
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_persist<4>, T, 0);
  timeit("persistent U=4 (as k_update)", B, [&] { k_persist<4><<<per * sms, T>>>(ntiles, x, p, q, r, part, 1e-3); });
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_persist<2>, T, 0);
  timeit("persistent U=2", B, [&] { k_persist<2><<<per * sms, T>>>(ntiles, x, p, q, r, part, 1e-3); });
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_persist<8>, T, 0);
  timeit("persistent U=8", B, [&] { k_persist<8><<<per * sms, T>>>(ntiles, x, p, q, r, part, 1e-3); });
  timeit("one tile per CTA", B, [&] { k_tile<<<ntiles, T>>>(ntiles, x, p, q, r, part, 1e-3); });
  timeit("plain double2 grid-stride 4xSM", B, [&] {
    k_plain<<<sms * 8, T>>>(n / 2, (double2 *)x, (const double2 *)p, (const double2 *)q, (double2 *)r, 1e-3); });
  timeit("plain double2 one pass", B, [&] {
    k_plain<<<n / 2 / T, T>>>(n / 2, (double2 *)x, (const double2 *)p, (const double2 *)q, (double2 *)r, 1e-3); });
  timeit("read-only 4 streams + tile sums", 32.0 * n, [&] { k_readonly<<<ntiles, T>>>(ntiles, x, p, q, r, part); });
  timeit("copy 16 MB (a->b)", 16.0 * n, [&] { k_copy<<<n / 2 / T, T>>>(n / 2, (const double2 *)x, (double2 *)p); });
  double *big_a, *big_b;
  const long long nb = 1LL << 27;  // 1 GiB each
  cudaMalloc(&big_a, 8 * nb); cudaMalloc(&big_b, 8 * nb);
  timeit("copy 1 GiB (peak ref)", 16.0 * nb, [&] { k_copy<<<nb / 2 / T, T>>>(nb / 2, (const double2 *)big_a, (double2 *)big_b); });
  printf("sms %d\n", sms);
  return 0;
}
