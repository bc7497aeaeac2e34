// Micro-benchmark: the last CTA's global sum of tile partials (fin_sum) --
// the serial tail of every kernel with a fused scalar step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o fin fin.cu
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ double warp_bfly(double v) {
  for (int o = 16; o >= 1; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int B>
__global__ void k_fin(const double *part, long long count, int reps, double *out) {
  __shared__ double ws[32];
  double keep = 0.0;
  for (int r = 0; r < reps; r++) {
    double acc = 0.0;
    for (long long i0 = threadIdx.x; i0 < count; i0 += (long long)B * 256) {
      double v[B];
#pragma unroll
      for (int u = 0; u < B; u++) {
        const long long i = i0 + (long long)u * 256;
        v[u] = i < count ? __ldcg(part + i + r) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < B; u++)
        if (i0 + (long long)u * 256 < count) acc = __dadd_rn(acc, v[u]);
    }
    acc = warp_bfly(acc);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) keep += warp_bfly(threadIdx.x < 8 ? ws[threadIdx.x] : 0.0);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = keep;
}

int main() {
  const long long n = 8192;
  double *part, *out;
  cudaMalloc(&part, 8 * (n + 1024));
  cudaMalloc(&out, 8);
  cudaMemset(part, 0, 8 * (n + 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char *name, auto kern) {
    for (int reps : {1, 101}) {
      float best = 1e9;
      for (int i = 0; i < 20; i++) {
        cudaEventRecord(e0);
        kern<<<1, 256>>>(part, n, reps, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("%-12s reps %3d: %8.2f us\n", name, reps, best * 1e3);
    }
  };
  run("batch 8", k_fin<8>);
  run("batch 16", k_fin<16>);
  run("batch 32", k_fin<32>);
  return 0;
}
