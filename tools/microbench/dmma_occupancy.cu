// DMMA (mma.sync m8n8k4 f64) and DFMA throughput versus resident warps per SM and
// independent accumulators per warp: how much parallelism the FP64 pipe needs on a
// B200 (sm_100a). Informs the M2L GEMM tiling.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}
template <int ILP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 1234.5) out[0] = s;
}

template <typename K>
double run(K kern, int warps_per_sm, int sms, int iters, double flop_per_warp_iter, bool fma_args) {
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 32 * (warps_per_sm <= 8 ? warps_per_sm : 8);
  const int blocks = sms * (warps_per_sm * 32 / threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    if (fma_args) ((void (*)(double*, int, double, double))kern)<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    else ((void (*)(double*, int))kern)<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  return double(blocks) * (threads / 32) * iters * flop_per_warp_iter / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int iters = 20000;
  printf("DMMA m8n8k4 f64 TFLOP/s (rows: warps/SM, cols: independent accumulators per warp 1 2 4 8 16)\n");
  for (int w : {4, 8, 12, 16, 24, 32}) {
    printf("w=%2d:", w);
    printf(" %6.2f", run((void*)dmma_kernel<1>, w, sms, iters, 512.0 * 1, false));
    printf(" %6.2f", run((void*)dmma_kernel<2>, w, sms, iters, 512.0 * 2, false));
    printf(" %6.2f", run((void*)dmma_kernel<4>, w, sms, iters / 2, 512.0 * 4, false));
    printf(" %6.2f", run((void*)dmma_kernel<8>, w, sms, iters / 4, 512.0 * 8, false));
    printf(" %6.2f\n", run((void*)dmma_kernel<16>, w, sms, iters / 8, 512.0 * 16, false));
  }
  printf("DFMA TFLOP/s (cols: independent chains per thread 1 2 4 8)\n");
  for (int w : {4, 8, 12, 16, 24, 32}) {
    printf("w=%2d:", w);
    printf(" %6.2f", run((void*)dfma_kernel<1>, w, sms, iters, 64.0 * 1, true));
    printf(" %6.2f", run((void*)dfma_kernel<2>, w, sms, iters, 64.0 * 2, true));
    printf(" %6.2f", run((void*)dfma_kernel<4>, w, sms, iters / 2, 64.0 * 4, true));
    printf(" %6.2f\n", run((void*)dfma_kernel<8>, w, sms, iters / 4, 64.0 * 8, true));
  }
  return 0;
}
