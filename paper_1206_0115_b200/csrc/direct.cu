// GPU direct-sum checker: direct_oracle (direct.cpp:202-226) on the device, the
// accuracy check of run_fmm (bench.cpp:366-398) at sizes where the O(k N) CPU loop takes
// minutes. Every sampled target sums over all N input particles
// except itself, with the reference's per-term arithmetic (1/sqrt(r^2) correctly
// rounded, s = ((w inv) inv) inv; this file is compiled without FMA contraction) and a
// fixed-order reduction (chunk partials, then chunk order), so results are
// deterministic and agree with the reference loop to summation-order rounding.
#include "common.cuh"

namespace fmmgpu {

namespace {

constexpr int DIRECT_THREADS = 256;

__global__ void __launch_bounds__(DIRECT_THREADS) k_direct(const double4* __restrict__ in, uint64_t n,
                                                           const uint32_t* __restrict__ targets, uint64_t chunk,
                                                           double4* __restrict__ partial) {
  const uint32_t t = blockIdx.y;
  const uint32_t ti = targets[t];
  const double4 a = in[ti];
  const uint64_t j0 = blockIdx.x * chunk, j1 = min(n, j0 + chunk);
  double pot = 0, fx = 0, fy = 0, fz = 0;
  for (uint64_t j = j0 + threadIdx.x; j < j1; j += DIRECT_THREADS) {
    if (j == ti) continue;
    const double4 b = in[j];
    const double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
    const double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
    const double s = b.w * inv * inv * inv;
    pot += b.w * inv;
    fx += s * dx;
    fy += s * dy;
    fz += s * dz;
  }
  __shared__ double red[4][DIRECT_THREADS];
  red[0][threadIdx.x] = pot;
  red[1][threadIdx.x] = fx;
  red[2][threadIdx.x] = fy;
  red[3][threadIdx.x] = fz;
  __syncthreads();
  for (int w = DIRECT_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    partial[uint64_t(t) * gridDim.x + blockIdx.x] = make_double4(red[0][0], red[1][0], red[2][0], red[3][0]);
}

__global__ void k_direct_sum(const double4* __restrict__ partial, uint32_t k, uint32_t nchunks,
                             double* __restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  double4 s = make_double4(0, 0, 0, 0);
  for (uint32_t c = 0; c < nchunks; ++c) {
    const double4 p = partial[uint64_t(t) * nchunks + c];
    s.x += p.x;
    s.y += p.y;
    s.z += p.z;
    s.w += p.w;
  }
  out[t] = s.x;
  out[k + t] = s.y;
  out[2 * k + t] = s.z;
  out[3 * k + t] = s.w;
}

}  // namespace

}  // namespace fmmgpu

using namespace fmmgpu;

extern "C" int fmmgpu_direct(fmmgpu_ctx* c, const uint32_t* targets, uint64_t k, double* pot, double* fx,
                             double* fy, double* fz) {
  try {
    if (!c || !c->have_tree) throw Error(FMMGPU_LOGIC_ERROR, "no tree: call fmmgpu_build_tree first");
    if (k == 0) return FMMGPU_OK;
    if (!targets || k > 65535u * 1024u) throw Error(FMMGPU_INVALID_ARGUMENT, "direct: bad target list");
    for (uint64_t t = 0; t < k; ++t)
      if (targets[t] >= c->n) throw Error(FMMGPU_OUT_OF_RANGE, "direct: target index out of range");
    FMM_CUDA(cudaSetDevice(c->device));
    cudaStream_t s = c->s_far;
    const uint32_t nchunks = static_cast<uint32_t>(std::min<uint64_t>(64, (c->n + 4095) / 4096));
    const uint64_t chunk = (c->n + nchunks - 1) / nchunks;
    uint32_t* dt = nullptr;
    double4* part = nullptr;
    double* dout = nullptr;
    FMM_CUDA(cudaMallocAsync(&dt, k * sizeof(uint32_t), s));
    FMM_CUDA(cudaMallocAsync(&part, k * nchunks * sizeof(double4), s));
    FMM_CUDA(cudaMallocAsync(&dout, 4 * k * sizeof(double), s));
    FMM_CUDA(cudaMemcpyAsync(dt, targets, k * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    // the input particles in input order are still resident from fmmgpu_build_tree
    k_direct<<<dim3(nchunks, static_cast<unsigned>(k)), DIRECT_THREADS, 0, s>>>(c->d_in, c->n, dt, chunk, part);
    FMM_CUDA(cudaGetLastError());
    k_direct_sum<<<static_cast<unsigned>((k + 255) / 256), 256, 0, s>>>(part, static_cast<uint32_t>(k), nchunks,
                                                                        dout);
    FMM_CUDA(cudaGetLastError());
    double* dst[4] = {pot, fx, fy, fz};
    for (int q = 0; q < 4; ++q)
      if (dst[q]) FMM_CUDA(cudaMemcpyAsync(dst[q], dout + q * k, k * sizeof(double), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(dt, s);
    cudaFreeAsync(part, s);
    cudaFreeAsync(dout, s);
    FMM_CUDA(cudaStreamSynchronize(s));
    return FMMGPU_OK;
  } catch (const Error& e) {
    if (c) c->err = e.what();
    return e.code;
  }
}
