// Ceiling of mutual (symmetric) P2P inner loops on B200 vs the one-sided loop of
// csrc/p2p.cu (development aid; no memory traffic, every lane busy).
//
// One-sided: 18 DP ops per DIRECTIONAL interaction, sources broadcast from shared memory.
// Mutual (p2p_block(mutual=true), direct.cpp:151-184): one pair evaluation serves both
// directions: 24 DP ops + MUFU per PAIR (= 2 directional interactions), but the j-side sums
// must travel. Variants (T targets per lane, sources rotating around the warp):
//   ring<T, 0>: source {x,y,z,w} and its 4 j-side sums rotate by one lane per step via
//               __shfl_sync (16 SHFL.32 per step, T pairs per lane per step);
//   ring<T, 1>: source position read from shared memory at lane (l + s) % 32 (2 LDS.128,
//               conflict-free), only the 4 j-side sums rotate (8 SHFL.32).
// Reports directional interactions/s and the implied time for config B's 9.98e9.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ double rsqrt_nr(double x, double c375) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double t = x * y;
  const double e = fma(-t, y, 1.0);
  return fma(y, e * fma(e, c375, 0.5), y);
}

__device__ __forceinline__ void one_sided(double xi, double yi, double zi, double4 pj, double c375, double& pot,
                                          double& fx, double& fy, double& fz) {
  const double dx = xi - pj.x, dy = yi - pj.y, dz = zi - pj.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double inv = rsqrt_nr(r2, c375);
  const double winv = pj.w * inv;
  pot += winv;
  const double s3 = winv * (inv * inv);
  fx = fma(s3, dx, fx);
  fy = fma(s3, dy, fy);
  fz = fma(s3, dz, fz);
}

// one pair, both sides: i gets +w_j (inv, inv^3 d), j gets +w_i inv and -w_i inv^3 d
__device__ __forceinline__ void mutual(const double4 pi, const double4 pj, double c375, double4& ai, double4& aj) {
  const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double inv = rsqrt_nr(r2, c375);
  const double inv2 = inv * inv;
  const double wj = pj.w * inv, wi = pi.w * inv;
  ai.x += wj;
  aj.x += wi;
  const double sj = wj * inv2, si = wi * inv2;
  ai.y = fma(sj, dx, ai.y);
  ai.z = fma(sj, dy, ai.z);
  ai.w = fma(sj, dz, ai.w);
  aj.y = fma(-si, dx, aj.y);
  aj.z = fma(-si, dy, aj.z);
  aj.w = fma(-si, dz, aj.w);
}

__device__ __forceinline__ double rot(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

constexpr int NS = 1024;

__global__ void k_one_sided(double4* out, int reps) {
  __shared__ double4 src[NS];
  for (int i = threadIdx.x; i < NS; i += blockDim.x)
    src[i] = make_double4(0.001 * i, 0.002 * (i % 97), 0.0005 * (i % 31), 1.0 + (i & 3));
  __syncthreads();
  double c375 = 0.375;
  asm volatile("" : "+d"(c375));
  const double xi = 0.5 + 1e-4 * threadIdx.x, yi = 0.25 + 1e-5 * blockIdx.x, zi = 0.125;
  double pot = 0, fx = 0, fy = 0, fz = 0;
  for (int r = 0; r < reps; ++r)
    for (int g = 0; g < NS; g += 4) {
      const double4 p0 = src[g], p1 = src[g + 1], p2 = src[g + 2], p3 = src[g + 3];
      one_sided(xi, yi, zi, p0, c375, pot, fx, fy, fz);
      one_sided(xi, yi, zi, p1, c375, pot, fx, fy, fz);
      one_sided(xi, yi, zi, p2, c375, pot, fx, fy, fz);
      one_sided(xi, yi, zi, p3, c375, pot, fx, fy, fz);
    }
  if (pot == 1234.5) out[0] = make_double4(pot, fx, fy, fz);
}

// T targets per lane; NS/32 source tiles of 32, each rotated through the whole warp
template <int T, int MODE>
__global__ void k_ring(double4* out, int reps) {
  __shared__ double4 src[NS];
  for (int i = threadIdx.x; i < NS; i += blockDim.x)
    src[i] = make_double4(0.001 * i + 7.0, 0.002 * (i % 97), 0.0005 * (i % 31), 1.0 + (i & 3));
  __syncthreads();
  double c375 = 0.375;
  asm volatile("" : "+d"(c375));
  const int lane = threadIdx.x & 31;
  const int next = (lane + 1) & 31;
  double4 pi[T], ai[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    pi[t] = make_double4(0.5 + 1e-4 * threadIdx.x + 0.01 * t, 0.25 + 1e-5 * blockIdx.x, 0.125, 1.0);
    ai[t] = make_double4(0, 0, 0, 0);
  }
  double jsum = 0;
  for (int r = 0; r < reps; ++r)
    for (int g = 0; g < NS; g += 32) {
      double4 pj = src[g + lane];
      double4 aj = make_double4(0, 0, 0, 0);
#pragma unroll 4
      for (int s = 0; s < 32; ++s) {
        if (MODE == 1) pj = src[g + ((lane + s) & 31)];
#pragma unroll
        for (int t = 0; t < T; ++t) mutual(pi[t], pj, c375, ai[t], aj);
        if (MODE == 0) {
          pj.x = rot(pj.x, next);
          pj.y = rot(pj.y, next);
          pj.z = rot(pj.z, next);
          pj.w = rot(pj.w, next);
        }
        aj.x = rot(aj.x, next);
        aj.y = rot(aj.y, next);
        aj.z = rot(aj.z, next);
        aj.w = rot(aj.w, next);
      }
      jsum += aj.x + aj.y + aj.z + aj.w;
    }
  double acc = jsum;
#pragma unroll
  for (int t = 0; t < T; ++t) acc += ai[t].x + ai[t].y + ai[t].z + ai[t].w;
  if (acc == 1234.5) out[0] = make_double4(acc, 0, 0, 0);
}


// sub-ring design of csrc/p2p.cu's mutual kernel: 4 sub-rings of 8 lanes; each lane holds
// TS sources (fixed, j-side sums in registers); a tile of 8 targets rotates around each
// sub-ring (positions re-read from shared memory, accumulators moved by SHFL); the 4
// sub-rings' partial target sums are combined by a 2-level butterfly after 8 steps.
template <int TS>
__global__ void k_subring(double4* out, int reps) {
  __shared__ double4 tgt[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x)
    tgt[i] = make_double4(0.5 + 1e-3 * i, 0.25 + 1e-5 * blockIdx.x, 0.125 + 1e-4 * (i % 7), 1.0);
  __syncthreads();
  double c375 = 0.375;
  asm volatile("" : "+d"(c375));
  const int lane = threadIdx.x & 31, l8 = lane & 7, base8 = lane & ~7;
  double4 ps[TS], as[TS];
#pragma unroll
  for (int t = 0; t < TS; ++t) {
    ps[t] = make_double4(7.0 + 0.001 * lane + 0.01 * t, 0.002 * (lane % 5), 0.0005 * t, 1.0 + (lane & 3));
    as[t] = make_double4(0, 0, 0, 0);
  }
  double isum = 0;
  for (int r = 0; r < reps; ++r)
    for (int tile = 0; tile < 64; tile += 8) {
      double4 at = make_double4(0, 0, 0, 0);
#pragma unroll 2
      for (int s = 0; s < 8; ++s) {
        const double4 pt = tgt[tile + ((l8 + s) & 7)];
#pragma unroll
        for (int t = 0; t < TS; ++t) mutual(pt, ps[t], c375, at, as[t]);
        const int src = base8 | ((l8 + 1) & 7);
        at.x = rot(at.x, src);
        at.y = rot(at.y, src);
        at.z = rot(at.z, src);
        at.w = rot(at.w, src);
      }
#pragma unroll
      for (int o = 8; o < 32; o <<= 1) {
        at.x += __shfl_xor_sync(0xffffffffu, at.x, o);
        at.y += __shfl_xor_sync(0xffffffffu, at.y, o);
        at.z += __shfl_xor_sync(0xffffffffu, at.z, o);
        at.w += __shfl_xor_sync(0xffffffffu, at.w, o);
      }
      isum += at.x + at.y + at.z + at.w;
    }
  double acc = isum;
#pragma unroll
  for (int t = 0; t < TS; ++t) acc += as[t].x + as[t].y + as[t].z + as[t].w;
  if (acc == 1234.5) out[0] = make_double4(acc, 0, 0, 0);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double4* out;
  CK(cudaMalloc(&out, 32));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](auto launch, double directional, const char* name, int warps, int grid) {
    launch(1);
    cudaEventRecord(a);
    launch(4);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double rate = directional * 4 / (ms * 1e-3);
    printf("%-22s warps/CTA %2d grid %5d: %8.3f ms  %.3e directional/s  config-B P2P at this rate %.2f ms\n", name,
           warps, grid, ms, rate, 9.98e9 / rate * 1e3);
  };
  for (int warps : {8, 12, 16}) {
    const int grid = sms * 2 * 4;
    const double thr = double(grid) * warps * 32;
    time([&](int reps) { k_one_sided<<<grid, warps * 32>>>(out, reps); }, thr * NS, "one-sided", warps, grid);
    time([&](int reps) { k_ring<1, 0><<<grid, warps * 32>>>(out, reps); }, thr * NS * 2 * 1, "ring T=1 shfl-src", warps, grid);
    time([&](int reps) { k_ring<2, 0><<<grid, warps * 32>>>(out, reps); }, thr * NS * 2 * 2, "ring T=2 shfl-src", warps, grid);
    time([&](int reps) { k_ring<4, 0><<<grid, warps * 32>>>(out, reps); }, thr * NS * 2 * 4, "ring T=4 shfl-src", warps, grid);
    time([&](int reps) { k_ring<1, 1><<<grid, warps * 32>>>(out, reps); }, thr * NS * 2 * 1, "ring T=1 lds-src", warps, grid);
    time([&](int reps) { k_ring<2, 1><<<grid, warps * 32>>>(out, reps); }, thr * NS * 2 * 2, "ring T=2 lds-src", warps, grid);
    time([&](int reps) { k_ring<4, 1><<<grid, warps * 32>>>(out, reps); }, thr * NS * 2 * 4, "ring T=4 lds-src", warps, grid);
    for (int ts : {2, 3, 4, 6}) {
      const double pairs = thr * 64 * ts * 2;  // directional per rep
      char nm[32];
      snprintf(nm, sizeof nm, "subring TS=%d", ts);
      auto go = [&](int reps) {
        if (ts == 2) k_subring<2><<<grid, warps * 32>>>(out, reps);
        if (ts == 3) k_subring<3><<<grid, warps * 32>>>(out, reps);
        if (ts == 4) k_subring<4><<<grid, warps * 32>>>(out, reps);
        if (ts == 6) k_subring<6><<<grid, warps * 32>>>(out, reps);
      };
      time(go, pairs, nm, warps, grid);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
