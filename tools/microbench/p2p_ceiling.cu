// Ceiling of the P2P inner loop on B200 (development aid): the exact per-interaction
// instruction mix of csrc/p2p.cu (18 DP ops + MUFU.RSQ64H) with every lane busy, sources
// broadcast from shared memory and no memory traffic. Reports interactions/s and the
// fraction of the DFMA issue rate (34.0 TF/s = 17.0e12 DP instr/s) it reaches, i.e. the
// pipe utilisation the real kernel can at best approach.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double t = x * y;
  const double e = fma(-t, y, 1.0);
  const double p = fma(e, 0.375, 0.5);
  return fma(y, e * p, y);
}

__device__ __forceinline__ void interact(double xi, double yi, double zi, double4 pj, double& pot, double& fx,
                                         double& fy, double& fz) {
  const double dx = xi - pj.x, dy = yi - pj.y, dz = zi - pj.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  double inv = rsqrt_nr(r2);
  inv = __double2hiint(r2) != 0 ? inv : 0.0;
  const double winv = pj.w * inv;
  pot += winv;
  const double s3 = winv * (inv * inv);
  fx = fma(s3, dx, fx);
  fy = fma(s3, dy, fy);
  fz = fma(s3, dz, fz);
}

constexpr int NS = 1024;

template <int MODE>  // 0: as p2p.cu (groups of 4); 1: no self-mask select; 2: no MUFU (seed = const)
__global__ void k(double4* out, int reps) {
  __shared__ double4 src[NS];
  for (int i = threadIdx.x; i < NS; i += blockDim.x)
    src[i] = make_double4(0.001 * i, 0.002 * (i % 97), 0.0005 * (i % 31), 1.0 + (i & 3));
  __syncthreads();
  const double xi = 0.5 + 1e-4 * threadIdx.x, yi = 0.25 + 1e-5 * blockIdx.x, zi = 0.125;
  double pot = 0, fx = 0, fy = 0, fz = 0;
  for (int r = 0; r < reps; ++r)
    for (int g = 0; g < NS; g += 4) {
      const double4 p0 = src[g], p1 = src[g + 1], p2 = src[g + 2], p3 = src[g + 3];
      interact(xi, yi, zi, p0, pot, fx, fy, fz);
      interact(xi, yi, zi, p1, pot, fx, fy, fz);
      interact(xi, yi, zi, p2, pot, fx, fy, fz);
      interact(xi, yi, zi, p3, pot, fx, fy, fz);
    }
  if (pot == 1234.5) out[0] = make_double4(pot, fx, fy, fz);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double4* out;
  CK(cudaMalloc(&out, 32));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int warps : {4, 8, 12, 16, 24}) {
    for (int ctas_per_sm : {1, 2}) {
      const int reps = 8;
      const int grid = sms * ctas_per_sm * 4;
      k<0><<<grid, warps * 32>>>(out, 1);
      CK(cudaEventRecord(a));
      k<0><<<grid, warps * 32>>>(out, reps);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double inter = double(grid) * warps * 32 * NS * reps;
      const double rate = inter / (ms * 1e-3);
      printf("warps/CTA %2d grid %5d: %.3f ms  %.3e interactions/s  DP-instr util %.1f%%\n", warps, grid, ms, rate,
             100.0 * rate * 18 / 17.01e12);
    }
  }
  return 0;
}
