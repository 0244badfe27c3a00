// Near field (P2P) on the device: the leaf-level 1/r potential and force of
// p2p_block / p2p_reduce (direct.cpp:111-200; pair kernels direct.cpp:9-20),
// evaluated one-sided per target so every accumulator has exactly one writer
// (deterministic, no atomics, no P2PBuffers slots).
//
// Mapping: one CTA per non-empty parent cell (level leaf-1).
// Its 2x2x2 children are the target cells; the union of their 27-neighbourhoods
// is the 4x4x4 block of leaf positions around the parent, whose particles are
// staged ONCE into shared memory as {x,y,z,w} (8 loads per particle per
// evaluation instead of 27). Warp w owns child octant w: its targets sit in
// registers, 32 at a time, and every source is a broadcast LDS.128 pair. When
// fewer than 32 targets remain, the lanes split the sources of each neighbour
// cell S ways (S = 32 / remaining) and the S partial sums are combined in a fixed
// order through shared memory, so a 38-particle leaf costs 1.2 passes, not 2.
// Neighbourhoods larger than the staging capacity (non-uniform clouds) are
// streamed through shared memory in chunks; targets then accumulate into HBM per
// chunk, still single-writer.
//
// Per interaction: 3 DADD (d) + 3 DP (r^2) + MUFU.RSQ64H and 4 DP (rsqrt_nr)
// + 1 DMUL (w/r) + 1 DADD (pot) + 2 DMUL (w/r^3) + 3 DFMA (force) = 18 DP ops.
#include <cstdlib>

#include "common.cuh"

namespace fmmgpu {

namespace {

constexpr int P2P_CAP = 3072;            // staged particles per chunk (96 KB), multiple of 4

struct P2PArgs {
  LevelView leaf;
  const uint64_t* parent_code;  // level leaf-1
  uint32_t p0;                  // first parent of the launch (partitioned runs: owned range)
  uint32_t usplit;              // CTAs per parent: CTA y takes the units u = y (mod usplit)
  const uint32_t* first;        // leaf first_particle
  const uint32_t* count;        // leaf particle_count
  const double4* pw;
  double4* near;  // [n] x {pot, fx, fy, fz}, Morton order
  uint64_t n;
};

template <int WARPS>
struct P2PSmem {
  double4 src[P2P_CAP + 4];  // + one group of zero-weight sources (tail of a 2-group step)
  double red[WARPS][4][32];
  uint32_t first[64];
  uint32_t cnt[64];
  uint32_t voff[65];  // virtual offsets of the 64 positions (prefix sum of counts padded to 4)
  uint32_t full_off[9];  // prefix over the 8 children of their full 32-target passes
  uint32_t next_unit;    // work-unit queue head (per chunk)
};

// A staged source that contributes exactly zero: w = 0 far away (finite r^2, so
// w/r and w/r^3 are +0 and the accumulators are unchanged bit for bit).
__device__ __forceinline__ double4 dummy_source() { return make_double4(1e100, 1e100, 1e100, 0.0); }

__device__ __forceinline__ void interact(const double xi, const double yi, const double zi, const double4 pj,
                                         double& pot, double& fx, double& fy, double& fz) {
  const double dx = xi - pj.x, dy = yi - pj.y, dz = zi - pj.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  double inv = rsqrt_nr(r2);
  // i == j gives r^2 = +0 exactly (coincident distinct particles are rejected at
  // build): an integer test on the high word keeps the select off the FP64 pipe.
  inv = __double2hiint(r2) != 0 ? inv : 0.0;
  const double winv = pj.w * inv;
  pot += winv;
  const double s3 = winv * (inv * inv);
  fx = fma(s3, dx, fx);
  fy = fma(s3, dy, fy);
  fz = fma(s3, dz, fz);
}

// WARPS warps per CTA pull the work units; G groups of 4 sources per inner iteration.
template <int WARPS, int G>
__global__ void __launch_bounds__(WARPS * 32, 2) k_p2p(const P2PArgs a) {
  constexpr int P2P_THREADS = WARPS * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  P2PSmem<WARPS>& sm = *reinterpret_cast<P2PSmem<WARPS>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  int pc[3];
  demorton(a.parent_code[a.p0 + blockIdx.x / a.usplit], pc);
  const uint32_t ysplit = blockIdx.x % a.usplit;
  if (tid < 64) {
    const int qa = tid >> 4, qb = (tid >> 2) & 3, qc = tid & 3;
    const uint32_t cell = find_ijk(a.leaf, 2 * pc[0] - 1 + qa, 2 * pc[1] - 1 + qb, 2 * pc[2] - 1 + qc);
    const uint32_t cnt = cell == NPOS ? 0u : a.count[cell];
    sm.first[tid] = cell == NPOS ? 0u : a.first[cell];
    sm.cnt[tid] = cnt;
    // inclusive warp scan over the 64 padded counts (two warps), then fix up
    // runs start at qc = 0 or 1 and end at qc = 3 or the row end, so only those
    // boundaries must sit on groups of 4: position qc = 1 is not padded and qc = 2
    // pads the pair (qc = 1, qc = 2) to a whole number of groups
    const uint32_t cnt_prev = __shfl_up_sync(0xffffffffu, cnt, 1);
    uint32_t x = qc == 1 ? cnt : qc == 2 ? ((cnt_prev + cnt + 3u) & ~3u) - cnt_prev : (cnt + 3u) & ~3u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((tid & 31) >= o) x += y;
    }
    sm.voff[tid + 1] = x;
    if (tid == 0) sm.voff[0] = 0;
  }
  __syncthreads();
  if (tid >= 33 && tid <= 64) sm.voff[tid] += sm.voff[32];
  __syncthreads();
  const uint32_t total = sm.voff[64];

  // Work units: every full 32-target pass of every child, then every child's partial
  // last pass (cost ~ m/32 of a full one). Warps pull units from a shared queue, so a
  // CTA whose children differ in size still keeps all 8 warps busy to the end (a
  // static warp-per-child mapping idles ~20% at ~38 particles per leaf). Each unit
  // owns distinct targets, so results do not depend on which warp takes it.
  if (tid < 4) sm.src[P2P_CAP + tid] = dummy_source();
  if (tid == 0) {
    uint32_t acc = 0;
    for (int w = 0; w < 8; ++w) {
      sm.full_off[w] = acc;
      const int tp = ((1 + ((w >> 2) & 1)) << 4) | ((1 + ((w >> 1) & 1)) << 2) | (1 + (w & 1));
      acc += sm.cnt[tp] / 32u;
    }
    sm.full_off[8] = acc;
  }
  __syncthreads();
  const uint32_t nfull = sm.full_off[8];
  uint32_t npart = 0;
  for (int w = 0; w < 8; ++w) {
    const int tp = ((1 + ((w >> 2) & 1)) << 4) | ((1 + ((w >> 1) & 1)) << 2) | (1 + (w & 1));
    npart += (sm.cnt[tp] % 32u) != 0;
  }
  const uint32_t nunits = nfull + npart;

  for (uint32_t base = 0; base < total; base += P2P_CAP) {
    const uint32_t clen = min(static_cast<uint32_t>(P2P_CAP), total - base);
    if (base) __syncthreads();
    if (tid == 0) sm.next_unit = 0;
    for (uint32_t i = tid; i < clen; i += P2P_THREADS) {
      const uint32_t v = base + i;
      int lo = 0, hi = 63;  // last position with voff[pos] <= v
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sm.voff[mid] <= v) lo = mid; else hi = mid - 1;
      }
      const uint32_t k = v - sm.voff[lo];
      sm.src[i] = k < sm.cnt[lo] ? a.pw[sm.first[lo] + k] : dummy_source();
    }
    __syncthreads();

    for (;;) {
      uint32_t u = 0;
      if (lane == 0) u = atomicAdd(&sm.next_unit, 1u);
      u = __shfl_sync(0xffffffffu, u, 0) * a.usplit + ysplit;
      if (u >= nunits) break;
      // decode unit -> (child octant w, first target t0)
      int w = 0;
      uint32_t t0 = 0;
      if (u < nfull) {
        while (sm.full_off[w + 1] <= u) ++w;
        t0 = 32u * (u - sm.full_off[w]);
      } else {
        uint32_t k = u - nfull;
        for (w = 0; w < 8; ++w) {
          const int tp = ((1 + ((w >> 2) & 1)) << 4) | ((1 + ((w >> 1) & 1)) << 2) | (1 + (w & 1));
          if (sm.cnt[tp] % 32u == 0) continue;
          if (k == 0) break;
          --k;
        }
        t0 = 32u * (sm.full_off[w + 1] - sm.full_off[w]);
      }
      const int ca = (w >> 2) & 1, cb = (w >> 1) & 1, cc = w & 1;
      const int tpos = ((1 + ca) << 4) | ((1 + cb) << 2) | (1 + cc);
      const uint32_t nT = sm.cnt[tpos];
      const uint32_t tfirst = sm.first[tpos];
      const uint32_t m = min(32u, nT - t0);
      const uint32_t S = 32u / m;
      const uint32_t lt = lane % m, split = lane / m;
      const bool active = split < S;
      const uint64_t tg = uint64_t(tfirst) + t0 + lt;
      const double4 xi = a.pw[tg];
      double pot = 0, fx = 0, fy = 0, fz = 0;
      if (active) {
        // the 27 neighbour positions as 9 runs of 3 consecutive positions (qc = cc..cc+2),
        // whose padded segments are contiguous in shared memory
#pragma unroll 1
        for (int q = 0; q < 9; ++q) {
          const int pos = ((ca + q / 3) << 4) | ((cb + q % 3) << 2) | cc;
          // intersection of the run's virtual range with this chunk, chunk-relative
          // (segments are padded to groups of 4 and chunks are multiples of 4)
          const uint32_t v0 = max(sm.voff[pos], base), v1 = min(sm.voff[pos + 3], base + clen);
          const int g1 = static_cast<int>(v1 - base) >> 2;
          const int gs = static_cast<int>(S);
          for (int g = (static_cast<int>(v0 - base) >> 2) + static_cast<int>(split); g < g1; g += G * gs) {
            const double4* sj = sm.src + 4 * g;
            const double4 p0 = sj[0], p1 = sj[1], p2 = sj[2], p3 = sj[3];
            if constexpr (G == 2) {
              const double4* sk = (g + gs < g1) ? sm.src + 4 * (g + gs) : sm.src + P2P_CAP;
              const double4 p4 = sk[0], p5 = sk[1], p6 = sk[2], p7 = sk[3];
              interact(xi.x, xi.y, xi.z, p0, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p1, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p2, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p3, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p4, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p5, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p6, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p7, pot, fx, fy, fz);
            } else {
              interact(xi.x, xi.y, xi.z, p0, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p1, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p2, pot, fx, fy, fz);
              interact(xi.x, xi.y, xi.z, p3, pot, fx, fy, fz);
            }
          }
        }
      }
      if (S > 1) {  // combine the S source splits of each target in a fixed order
        sm.red[warp][0][lane] = pot;
        sm.red[warp][1][lane] = fx;
        sm.red[warp][2][lane] = fy;
        sm.red[warp][3][lane] = fz;
        __syncwarp();
        if (lane < m) {
          for (uint32_t s = 1; s < S; ++s) {
            pot += sm.red[warp][0][lane + s * m];
            fx += sm.red[warp][1][lane + s * m];
            fy += sm.red[warp][2][lane + s * m];
            fz += sm.red[warp][3][lane + s * m];
          }
        }
        __syncwarp();
      }
      if (lane < m) {
        double4 r = a.near[tg];
        r.x += pot;
        r.y += fx;
        r.z += fy;
        r.w += fz;
        a.near[tg] = r;
      }
    }
  }
}

}  // namespace

void launch_p2p(fmmgpu_ctx* c, cudaStream_t s) {
  const int leaf = c->height - 1;
  const Level& L = c->lv[leaf];
  const Level& P = c->lv[leaf - 1];
  const uint32_t np = P.own1 - P.own0;
  if (np == 0) return;
  // few parents (shallow trees, big leaves): several CTAs per parent share its units
  // (each re-stages the neighbourhood) so the grid still covers 2 CTAs per SM
  uint32_t usplit = 1;
  while (np * usplit < 2u * 148u && usplit < 16u) usplit *= 2;
  P2PArgs a{L.view(leaf), P.code, P.own0, usplit, L.first_particle, L.particle_count, c->d_pw,
             reinterpret_cast<double4*>(c->d_near), c->n};
  auto run = [&](auto kern, int warps, int smem) {
    FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<np * usplit, warps * 32, smem, s>>>(a);
  };
  // FMMGPU_P2P_VARIANT (tuning experiments): 0 = 12 warps x 1 group, 1 = 8 x 2, 2 = 16 x 1, 3 = 8 x 1
  static const int variant = [] {
    const char* e = std::getenv("FMMGPU_P2P_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  switch (variant) {
    case 1: run(k_p2p<8, 2>, 8, static_cast<int>(sizeof(P2PSmem<8>))); break;
    case 2: run(k_p2p<16, 1>, 16, static_cast<int>(sizeof(P2PSmem<16>))); break;
    case 3: run(k_p2p<8, 1>, 8, static_cast<int>(sizeof(P2PSmem<8>))); break;
    default: run(k_p2p<12, 1>, 12, static_cast<int>(sizeof(P2PSmem<12>))); break;
  }
  FMM_CUDA(cudaGetLastError());
  ++c->launches;
}

}  // namespace fmmgpu
