// Near field (P2P) on the device: the leaf-level 1/r potential and force of
// p2p_block / p2p_reduce (direct.cpp:111-200; pair kernels direct.cpp:9-20),
// evaluated one-sided per target so every accumulator has exactly one writer
// (deterministic, no atomics, no P2PBuffers slots).
//
// Unit of staging: one parent cell (level leaf-1). Its 2x2x2
// children are the target cells; the union of their 27-neighbourhoods is the 4x4x4
// block of leaf positions around the parent, whose particles are staged ONCE into
// shared memory as {x,y,z,w} (8 loads per particle per evaluation instead of 27),
// each position's segment padded so a child's 27 neighbours read as 9 contiguous runs
// of whole groups of 4. Work units: every full 32-target pass of every child, then
// each child's partial last pass cut into chunks of 16, 8, 4, 2, 1 targets (largest
// first); targets sit in registers (one per lane) and every source is a broadcast
// LDS.128 pair. A chunk of m = 2^b targets splits the sources of each run S = 32 / m
// ways, so every lane works, and combines the S partial sums in a fixed order through
// shared memory. The evaluation writes near (first staging chunk) instead of adding.
//
// k_p2p runs one CTA (12 warps, 2 CTAs per SM) per parent. Neighbourhoods larger than
// one staging buffer (non-uniform clouds) stream through shared memory in chunks
// (targets then accumulate into HBM per chunk, still single-writer), and shallow trees
// with too few parents for the GPU split a parent's units over several CTAs.
//
// Per interaction: 3 DADD (d) + 3 DP (r^2) + MUFU.RSQ64H and 5 DP (Newton)
// + 1 DMUL (w/r) + 1 DADD (pot) + 2 DMUL (w/r^3) + 3 DFMA (force) = 18 DP ops.
#include <cstdlib>

#include "common.cuh"

namespace fmmgpu {

namespace {

constexpr int P2P_CAP = 3072;  // staged particles per chunk (96 KB), multiple of 4

struct P2PArgs {
  LevelView leaf;
  const uint64_t* parent_code;  // level leaf-1
  uint32_t p0;                  // first parent of the launch (partitioned runs: owned range)
  uint32_t np;                  // parents in the launch
  uint32_t usplit;              // CTAs per parent (CTA y takes the units u = y (mod usplit))
  const uint32_t* first;        // leaf first_particle
  const uint32_t* count;        // leaf particle_count
  const double4* pw;
  double4* near;  // [n] x {pot, fx, fy, fz}, Morton order
  uint64_t n;
  int ow;         // overwrite (evaluation): the first staging chunk writes near instead of adding
};

// A staged source that contributes exactly zero: w = 0 far away (finite r^2, so
// w/r and w/r^3 are +0 and the accumulators are unchanged bit for bit).
__device__ __forceinline__ double4 dummy_source() { return make_double4(1e100, 1e100, 1e100, 0.0); }

// One interaction; SELF: the source run may hold the target itself. i == j gives
// r^2 = +0 exactly (coincident distinct particles are rejected at build), and an
// integer test on r^2's high word keeps that select off the FP64 pipe; the other 8
// of a target's 9 runs skip it. 1/sqrt is the MUFU.RSQ64H seed and one third-order
// Newton step (rsqrt_nr, common.cuh) with the 0.375 coefficient held in a register.
template <bool SELF>
__device__ __forceinline__ void interact(const double xi, const double yi, const double zi, const double4 pj,
                                         const double c375, double& pot, double& fx, double& fy, double& fz) {
  const double dx = xi - pj.x, dy = yi - pj.y, dz = zi - pj.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  const double t = r2 * y;
  const double e = fma(-t, y, 1.0);
  double inv = fma(y, e * fma(e, c375, 0.5), y);
  if constexpr (SELF) inv = __double2hiint(r2) != 0 ? inv : 0.0;
  const double winv = pj.w * inv;
  pot += winv;
  const double s3 = winv * (inv * inv);
  fx = fma(s3, dx, fx);
  fy = fma(s3, dy, fy);
  fz = fma(s3, dz, fz);
}

// The sources of one run from sj to se, a group of 4 per step. ROT (chunks with S > 1
// source splits): the S splits read groups 128 B apart, i.e. the same four banks, so
// split s reads its group in the order k ^ (s & 3): the four element positions of a
// group sit in disjoint banks, which cuts the wavefronts of each LDS.128 by 4 (an S-way
// conflict becomes S/4-way). Full passes (S = 1, broadcast) keep the plain order.
// Measured at config B: P2P 12.78 -> 12.54 ms, evaluation 26.60 -> 26.36 ms (the
// chunks' sums change order, so their fields differ from the plain order by rounding).
template <bool SELF, bool ROT>
__device__ __forceinline__ void run_sources(const double4* sj, const double4* se, const int step, const int rot,
                                            const double4 xi, const double c375, double& pot, double& fx,
                                            double& fy, double& fz) {
  for (; sj < se; sj += step) {
    const double4 p0 = sj[ROT ? rot : 0], p1 = sj[ROT ? rot ^ 1 : 1], p2 = sj[ROT ? rot ^ 2 : 2],
                  p3 = sj[ROT ? rot ^ 3 : 3];
    interact<SELF>(xi.x, xi.y, xi.z, p0, c375, pot, fx, fy, fz);
    interact<SELF>(xi.x, xi.y, xi.z, p1, c375, pot, fx, fy, fz);
    interact<SELF>(xi.x, xi.y, xi.z, p2, c375, pot, fx, fy, fz);
    interact<SELF>(xi.x, xi.y, xi.z, p3, c375, pot, fx, fy, fz);
  }
}

// leaf position (0..63) of child octant w inside the 4x4x4 block
__device__ __forceinline__ int child_pos(int w) {
  return ((1 + ((w >> 2) & 1)) << 4) | ((1 + ((w >> 1) & 1)) << 2) | (1 + (w & 1));
}

// Metadata of one staged neighbourhood.
struct Neigh {
  uint32_t first[64];
  uint32_t cnt[64];
  uint32_t voff[65];     // virtual offsets of the 64 positions (prefix sum of padded counts)
  uint32_t full_off[9];  // prefix over the 8 children of their full 32-target passes
  uint32_t nunits;
  // the partial last pass of child w (m = count % 32 targets) is cut into chunks of
  // 16, 8, 4, 2, 1 targets (the binary digits of m); a chunk of 2^b targets splits the
  // sources 32 / 2^b ways, so every lane works. Entries (w << 8) | b, largest first.
  uint16_t part[40];
};

// Counts and padded offsets of the 64 leaf positions around parent pc, by one warp
// (lane handles positions lane and lane + 32). Runs start at qc = 0 or 1 and end at
// qc = 3 or the row end, so only those boundaries must sit on groups of 4: position
// qc = 1 is not padded and qc = 2 pads the pair (qc = 1, qc = 2) to whole groups.
__device__ void neigh_meta(const P2PArgs& a, const int pc[3], Neigh& nb, int lane) {
  uint32_t x[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int pos = lane + 32 * h;
    const int qa = pos >> 4, qb = (pos >> 2) & 3, qc = pos & 3;
    const uint32_t cell = find_ijk(a.leaf, 2 * pc[0] - 1 + qa, 2 * pc[1] - 1 + qb, 2 * pc[2] - 1 + qc);
    const uint32_t cnt = cell == NPOS ? 0u : a.count[cell];
    nb.first[pos] = cell == NPOS ? 0u : a.first[cell];
    nb.cnt[pos] = cnt;
    const uint32_t cnt_prev = __shfl_up_sync(0xffffffffu, cnt, 1);
    uint32_t v = qc == 1 ? cnt : qc == 2 ? ((cnt_prev + cnt + 3u) & ~3u) - cnt_prev : (cnt + 3u) & ~3u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    x[h] = v;
  }
  const uint32_t tot0 = __shfl_sync(0xffffffffu, x[0], 31);
  nb.voff[lane + 1] = x[0];
  nb.voff[lane + 33] = x[1] + tot0;
  if (lane == 0) nb.voff[0] = 0;
  __syncwarp();
  if (lane == 0) {
    uint32_t acc = 0, npart = 0;
    for (int w = 0; w < 8; ++w) {
      nb.full_off[w] = acc;
      acc += nb.cnt[child_pos(w)] / 32u;
    }
    nb.full_off[8] = acc;
    for (int b = 4; b >= 0; --b)
      for (int w = 0; w < 8; ++w)
        if ((nb.cnt[child_pos(w)] >> b) & 1u) nb.part[npart++] = static_cast<uint16_t>((w << 8) | b);
    nb.nunits = acc + npart;
  }
  __syncwarp();
}

// Virtual slot v (< voff[64]) -> staged source (a particle or a zero-weight pad).
__device__ __forceinline__ void locate(const Neigh& nb, uint32_t v, uint32_t& pos, uint32_t& k) {
  int lo = 0, hi = 63;  // last position with voff[pos] <= v
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (nb.voff[mid] <= v) lo = mid; else hi = mid - 1;
  }
  pos = static_cast<uint32_t>(lo);
  k = v - nb.voff[lo];
}

// One work unit u over the staged sources [base, base + clen) of the virtual range;
// src[0..clen) are the staged sources, src[P2P_CAP..+4) a group of zero sources.
__device__ void p2p_unit(const P2PArgs& a, const Neigh& nb, const double4* src, uint32_t base, uint32_t clen,
                         uint32_t u, double (*red)[32], int lane) {
  const uint32_t nfull = nb.full_off[8];
  // decode unit -> (child octant w, first target t0, m targets)
  int w = 0;
  uint32_t t0 = 0, m = 32;
  if (u < nfull) {
    while (nb.full_off[w + 1] <= u) ++w;
    t0 = 32u * (u - nb.full_off[w]);
  } else {
    const uint32_t e = nb.part[u - nfull];
    w = static_cast<int>(e >> 8);
    const int b = static_cast<int>(e & 0xff);
    const uint32_t rem = nb.cnt[child_pos(w)] % 32u;
    t0 = 32u * (nb.full_off[w + 1] - nb.full_off[w]) + ((rem >> (b + 1)) << (b + 1));
    m = 1u << b;
  }
  const int ca = (w >> 2) & 1, cb = (w >> 1) & 1, cc = w & 1;
  const int tpos = child_pos(w);
  const uint32_t tfirst = nb.first[tpos];
  const uint32_t S = 32u / m;  // source splits: lanes split * m + lt, split < S
  const uint32_t lt = lane % m, split = lane / m;
  const uint64_t tg = uint64_t(tfirst) + t0 + lt;
  const int rot = static_cast<int>(split & 3u);
  const double4 xi = a.pw[tg];
  double c375 = 0.375;
  asm volatile("" : "+d"(c375));  // opaque: stays in a register instead of being rebuilt per group
  double pot = 0, fx = 0, fy = 0, fz = 0;
  // the 27 neighbour positions as 9 runs of 3 consecutive positions (qc = cc..cc+2),
  // whose padded segments are contiguous in shared memory; run 4 holds the target's
  // own leaf
#pragma unroll 1
  for (int q = 0; q < 9; ++q) {
    const int pos = ((ca + q / 3) << 4) | ((cb + q % 3) << 2) | cc;
    // intersection of the run's virtual range with this chunk, chunk-relative
    // (segments are padded to groups of 4 and chunks are multiples of 4)
    const uint32_t v0 = max(nb.voff[pos], base), v1 = min(nb.voff[pos + 3], base + clen);
    const double4* sj = src + 4 * ((static_cast<int>(v0 - base) >> 2) + static_cast<int>(split));
    const double4* se = src + 4 * (static_cast<int>(v1 - base) >> 2);
    const int step = 4 * static_cast<int>(S);
    if (S == 1) {
      if (q == 4) run_sources<true, false>(sj, se, step, 0, xi, c375, pot, fx, fy, fz);
      else run_sources<false, false>(sj, se, step, 0, xi, c375, pot, fx, fy, fz);
    } else {
      if (q == 4) run_sources<true, true>(sj, se, step, rot, xi, c375, pot, fx, fy, fz);
      else run_sources<false, true>(sj, se, step, rot, xi, c375, pot, fx, fy, fz);
    }
  }
  if (S > 1) {  // combine the S source splits of each target in a fixed order
    red[0][lane] = pot;
    red[1][lane] = fx;
    red[2][lane] = fy;
    red[3][lane] = fz;
    __syncwarp();
    if (lane < m) {
      for (uint32_t s = 1; s < S; ++s) {
        pot += red[0][lane + s * m];
        fx += red[1][lane + s * m];
        fy += red[2][lane + s * m];
        fz += red[3][lane + s * m];
      }
    }
    __syncwarp();
  }
  if (lane < m) {
    double4 r = a.ow && base == 0 ? make_double4(0, 0, 0, 0) : a.near[tg];
    r.x += pot;
    r.y += fx;
    r.z += fy;
    r.w += fz;
    a.near[tg] = r;
  }
}

// ------------------------------------------------------------------ k_p2p
template <int WARPS>
struct P2PSmem {
  double4 src[P2P_CAP + 4];  // + one group of zero-weight sources (tail of a 2-group step)
  double red[WARPS][4][32];
  Neigh nb;
  uint32_t next_unit;  // work-unit queue head (per chunk)
};

// WARPS warps per CTA pull the work units.
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 2) k_p2p(const P2PArgs a) {
  constexpr int P2P_THREADS = WARPS * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  P2PSmem<WARPS>& sm = *reinterpret_cast<P2PSmem<WARPS>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  int pc[3];
  demorton(a.parent_code[a.p0 + blockIdx.x / a.usplit], pc);
  const uint32_t ysplit = blockIdx.x % a.usplit;
  if (warp == 0) neigh_meta(a, pc, sm.nb, lane);
  if (tid < 4) sm.src[P2P_CAP + tid] = dummy_source();
  __syncthreads();
  const uint32_t total = sm.nb.voff[64];
  const uint32_t nunits = sm.nb.nunits;

  for (uint32_t base = 0; base < total; base += P2P_CAP) {
    const uint32_t clen = min(static_cast<uint32_t>(P2P_CAP), total - base);
    if (base) __syncthreads();
    if (tid == 0) sm.next_unit = 0;
    for (uint32_t i = tid; i < clen; i += P2P_THREADS) {
      uint32_t pos, k;
      locate(sm.nb, base + i, pos, k);
      sm.src[i] = k < sm.nb.cnt[pos] ? a.pw[sm.nb.first[pos] + k] : dummy_source();
    }
    __syncthreads();
    for (;;) {
      uint32_t u = 0;
      if (lane == 0) u = atomicAdd(&sm.next_unit, 1u);
      u = __shfl_sync(0xffffffffu, u, 0) * a.usplit + ysplit;
      if (u >= nunits) break;
      p2p_unit(a, sm.nb, sm.src, base, clen, u, sm.red[warp], lane);
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
  P2PArgs a{L.view(leaf), P.code, P.own0, np, 1, L.first_particle, L.particle_count, c->d_pw,
             reinterpret_cast<double4*>(c->d_near), c->n, c->ow ? 1 : 0};
  auto run = [&](auto kern, int warps, int smem, unsigned grid) {
    FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, warps * 32, smem, s>>>(a);
    FMM_CUDA(cudaGetLastError());
    ++c->launches;
  };
  // FMMGPU_P2P_VARIANT (tuning experiments): 0 = 12 warps per CTA (default), 2 = 16, 3 = 8.
  // Config B before the chunked partial passes: 13.7 / 13.9 / 13.8 ms; with the chunks
  // and the rotated split reads: 12.60 / 12.92 / 12.58 ms. Staging 4 particles per thread
  // with their loads in flight together: 12.59 vs 12.56 ms (the other CTA of the SM
  // already hides the staging latency). Also measured
  // slower and removed: 8 sources per inner iteration, split accumulators (14.0 ms), two
  // targets per lane sharing each source load (12.9 / 13.0 ms with 8 / 12 warps vs 12.86
  // after the chunked partial passes), and
  // a persistent one-CTA-per-SM kernel walking its parents through two staging slots
  // without CTA barriers (15.0 / 16.8 ms with 16 / 24 warps: with one parent of
  // look-ahead its warps idle at the same unit-granularity tails).
  static const int variant = [] {
    const char* e = std::getenv("FMMGPU_P2P_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  int sms = 148;
  FMM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  // few parents (shallow trees, big leaves): several CTAs per parent share its units
  // (each re-stages the neighbourhood) so the grid still covers 2 CTAs per SM
  uint32_t usplit = 1;
  while (np * usplit < 2u * static_cast<uint32_t>(sms) && usplit < 16u) usplit *= 2;
  a.usplit = usplit;
  const unsigned grid = np * usplit;
  switch (variant) {
    case 2: run(k_p2p<16>, 16, static_cast<int>(sizeof(P2PSmem<16>)), grid); break;
    case 3: run(k_p2p<8>, 8, static_cast<int>(sizeof(P2PSmem<8>)), grid); break;
    default: run(k_p2p<12>, 12, static_cast<int>(sizeof(P2PSmem<12>)), grid); break;
  }
}

}  // namespace fmmgpu
