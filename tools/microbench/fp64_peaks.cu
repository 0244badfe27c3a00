// FP64 peak microbenchmarks for B200 (sm_100a): DFMA chains, DMMA m8n8k4, rsqrt.
// Used to fix the FP64 roofline denominator (not in MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

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

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void rsqrt_kernel(double* out, int iters) {
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = 1.0 + threadIdx.x * 1e-3 + i;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) { double r = rsqrt(x[i]); s += r; x[i] += 1e-9; }
  }
  if (s == 1234.5) out[0] = s;
}

__global__ void sqrtdiv_kernel(double* out, int iters) {
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = 1.0 + threadIdx.x * 1e-3 + i;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) { double r = 1.0 / sqrt(x[i]); s += r; x[i] += 1e-9; }
  }
  if (s == 1234.5) out[0] = s;
}

__global__ void rsq64h_kernel(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = 1.0 + threadIdx.x * 1e-3 + i;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[i])); x[i] = y; }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

__global__ void rsqnr_kernel(double* out, int iters) {
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = 1.0 + threadIdx.x * 1e-3 + i;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[i]));
      const double t = x[i] * y; const double e = fma(-t, y, 1.0); const double p = fma(e, 0.375, 0.5);
      s += fma(y, e * p, y); x[i] += 1e-9; }
  }
  if (s == 1234.5) out[0] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  for (int bpsm : {4, 8}) {
    int blocks = sms * bpsm, threads = 256, iters = 20000;
    dfma_kernel<8><<<blocks, threads>>>(d, 100, 0.999, 1e-3);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, fl / ms / 1e9, ms);
  }
  for (int bpsm : {4, 8}) {
    int blocks = sms * bpsm, threads = 256, iters = 5000;
    dmma_kernel<<<blocks, threads>>>(d, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("DMMA m8n8k4 blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, fl / ms / 1e9, ms);
  }
  {
    int blocks = sms * 8, threads = 256, iters = 20000;
    rsqrt_kernel<<<blocks, threads>>>(d, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    rsqrt_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rsqrt(double): %.2f G/s\n", 4.0 * iters * blocks * threads / ms / 1e6);
    sqrtdiv_kernel<<<blocks, threads>>>(d, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    sqrtdiv_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("1/sqrt(double): %.2f G/s\n", 4.0 * iters * blocks * threads / ms / 1e6);
  }
  {
    int blocks = sms * 8, threads = 256, iters = 20000;
    float ms;
    rsq64h_kernel<<<blocks, threads>>>(d, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    rsq64h_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("MUFU.RSQ64H: %.2f G/s = %.2f per SM per clk at 1965 MHz\n", 8.0 * iters * blocks * threads / ms / 1e6,
           8.0 * iters * blocks * threads / (ms * 1e-3) / sms / 1.965e9);
    rsqnr_kernel<<<blocks, threads>>>(d, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    rsqnr_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("rsqrt_nr (MUFU + 5 DP + add): %.2f G/s\n", 4.0 * iters * blocks * threads / ms / 1e6);
  }
  return 0;
}
