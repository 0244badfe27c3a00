// Near field (P2P) on the device: the leaf-level 1/r potential and force of
// p2p_block / p2p_reduce (direct.cpp:111-200), evaluated one-sided per target so
// every accumulator has exactly one writer (deterministic, no atomics).
//
// Mapping: one warp = 32 consecutive Morton-ordered targets (usually 1-2 leaf
// cells). The warp walks the union of its target cells' 27-neighbourhoods
// (self included) once, each source cell in a warp-uniform loop; every source
// particle is a broadcast load and each lane masks the interaction to zero when
// the source cell is not adjacent to its own cell or when it is the lane's own
// particle (r^2 == 0; coincident distinct particles are rejected at tree build,
// geometry.cpp:126-136). Per interaction: 3 DADD + 3 DMUL/DFMA (r^2) + 5 DP ops and
// one MUFU for 1/sqrt (rsqrt_nr) + 7 DP ops of accumulation.
#include "common.cuh"

namespace fmmgpu {

namespace {

struct P2PArgs {
  LevelView leaf;
  const uint32_t* first;
  const uint32_t* count;
  const uint32_t* pcell;
  const double4* pw;
  double* near;  // [4][n]
  uint64_t n;
};

__device__ __forceinline__ bool adjacent(const int a[3], const int b[3]) {
  return abs(a[0] - b[0]) <= 1 && abs(a[1] - b[1]) <= 1 && abs(a[2] - b[2]) <= 1;
}

__global__ void __launch_bounds__(256) k_p2p(const P2PArgs a) {
  const uint64_t wid = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t base = wid * 32;
  if (base >= a.n) return;
  const uint64_t s = base + lane;
  const bool valid = s < a.n;
  const uint64_t sc = valid ? s : a.n - 1;
  const uint32_t my_cell = a.pcell[sc];
  int my[3];
  demorton(a.leaf.code[my_cell], my);
  const double4 xi = a.pw[sc];
  const uint32_t c_first = a.pcell[base];
  const uint32_t c_last = a.pcell[(base + 31 < a.n) ? base + 31 : a.n - 1];

  double pot = 0, fx = 0, fy = 0, fz = 0;
  for (uint32_t tc = c_first; tc <= c_last; ++tc) {
    int t[3];
    demorton(a.leaf.code[tc], t);
    for (int o = 0; o < 27; ++o) {
      const int sx = t[0] + o / 9 - 1, sy = t[1] + (o / 3) % 3 - 1, sz = t[2] + o % 3 - 1;
      const uint32_t scell = find_ijk(a.leaf, sx, sy, sz);
      if (scell == NPOS) continue;
      const int sijk[3] = {sx, sy, sz};
      bool dup = false;  // already visited through an earlier target cell of this warp
      for (uint32_t pc = c_first; pc < tc && !dup; ++pc) {
        int p[3];
        demorton(a.leaf.code[pc], p);
        dup = adjacent(p, sijk);
      }
      if (dup) continue;
      const bool use = valid && adjacent(my, sijk);
      const uint32_t j0 = a.first[scell], j1 = j0 + a.count[scell];
#pragma unroll 4
      for (uint32_t j = j0; j < j1; ++j) {
        const double4 pj = a.pw[j];
        const double dx = xi.x - pj.x, dy = xi.y - pj.y, dz = xi.z - pj.z;
        const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
        double inv = rsqrt_nr(r2);
        inv = (use && r2 > 0.0) ? inv : 0.0;
        const double winv = pj.w * inv;
        pot += winv;
        const double s3 = winv * inv * inv;
        fx = fma(s3, dx, fx);
        fy = fma(s3, dy, fy);
        fz = fma(s3, dz, fz);
      }
    }
  }
  if (valid) {
    a.near[s] += pot;
    a.near[a.n + s] += fx;
    a.near[2 * a.n + s] += fy;
    a.near[3 * a.n + s] += fz;
  }
}

}  // namespace

void launch_p2p(fmmgpu_ctx* c, cudaStream_t s) {
  const int leaf = c->height - 1;
  const Level& L = c->lv[leaf];
  P2PArgs a{L.view(leaf), L.first_particle, L.particle_count, c->d_pcell, c->d_pw, c->d_near, c->n};
  const uint64_t warps = (c->n + 31) / 32;
  const unsigned blocks = static_cast<unsigned>((warps * 32 + 255) / 256);
  k_p2p<<<blocks, 256, 0, s>>>(a);
  FMM_CUDA(cudaGetLastError());
  ++c->launches;
}

}  // namespace fmmgpu
