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
#include <cub/cub.cuh>

#include <algorithm>
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

// ================================================================== mutual P2P
// p2p_block(mutual=true) (direct.cpp:151-184) with the reference's P2PBuffers slots and
// ordered p2p_reduce (direct.cpp:63-92, 187-200) restated for the GPU: each pair of a
// leaf c and one of its 13 upper half-shell neighbours q = c + d (d > 0 in (x, y, z)
// lexicographic order, MU_UP) is evaluated ONCE; c's side accumulates in the warp that
// owns c, q's side is written to slot s(d) of q's particles ([13][n] double4, single
// writer) and drained into near[] by k_p2p_drain in the fixed slot order. A leaf's own
// pairs are evaluated one-sided (i != j), like every pair with a neighbour this rank
// does not own (partitioned runs), so no slot ever crosses a rank.
//
// Warp layout (tools/microbench/p2p_mutual_ceiling.cu "subring"): 4 sub-rings of 8
// lanes. Each lane holds TS <= 4 SOURCES of c's stream (own leaf, then the half-shell
// leaves, then non-owned lower neighbours) in registers with their j-side sums; a tile
// of 8 TARGETS of c rotates around each sub-ring (positions re-read from shared memory,
// the 4 accumulators moved by SHFL one lane per step), so after 8 steps every lane's
// sources met all 8 targets and each target's sums are back in their home lane; the
// 4 sub-rings' partial target sums are then combined by a fixed 2-level butterfly.
// Per pair: 24 DP instructions + 1 MUFU.RSQ64H for both directions (12 per directional
// interaction against 18 one-sided).
//
// One warp owns a leaf from start to end (targets in chunks of TCAP, every chunk
// streams all sources; later chunks add into the slots the first one wrote), leaves are
// pulled from a global counter: results do not depend on which warp ran a leaf, so
// evaluations stay bitwise reproducible.
#ifndef FMMGPU_MU_WARPS
#define FMMGPU_MU_WARPS 12
#endif
constexpr int MU_WARPS = FMMGPU_MU_WARPS;
#ifndef FMMGPU_MU_TS
#define FMMGPU_MU_TS 4
#endif
#ifndef FMMGPU_MU_MINB
#define FMMGPU_MU_MINB 1
#endif
constexpr int MU_TS = FMMGPU_MU_TS;  // sources per lane per pass
constexpr int MU_NUP = 13;
constexpr int MU_MAXSEG = 27;

// slot s -> upper direction d (s = 0: (0,0,1); 1..3: (0,1,-1..1); 4..12: (1,-1..1,-1..1))
__device__ __forceinline__ void mu_up(int s, int d[3]) {
  d[0] = s >= 4 ? 1 : 0;
  d[1] = s >= 4 ? (s - 4) / 3 - 1 : (s >= 1 ? 1 : 0);
  d[2] = s >= 4 ? (s - 4) % 3 - 1 : (s >= 1 ? s - 2 : 1);
}

struct MuArgs {
  LevelView leaf;
  const uint32_t* first;
  const uint32_t* count;
  const double4* pw;
  double4* near;
  double4* slot;      // [13][n]
  uint64_t n;
  uint32_t c0, c1;    // leaves this launch processes / drains (the owned range)
  uint32_t* ctr;      // leaf counter (zeroed before the launch)
  const uint32_t* order;  // leaves by decreasing work (non-uniform trees), nullptr = c0 ..
  int ow;             // evaluation: write near instead of adding
};

// per-warp shared memory; TCAP = targets per chunk (64 on full leaf levels, 256 else:
// config D 192 -> 163 ms with 128 and the largest-first order, 162.5 with 256). Measured alternative for
// big leaves (config D, ~570 particles): the full 32-lane ring with 4 targets per lane
// in registers and sources rotating (no combine; tools/microbench "ring T=4 lds-src"):
// 79% of the FP64 pipe under ncu but 161.5 ms + 2.9 ms for the small leaves, no faster
// than this kernel alone (163 ms).
template <int TCAP>
struct MuWarp {
  double4 tpos[TCAP];
  double4 iacc[TCAP];
  uint32_t seg_off[MU_MAXSEG + 1];
  uint32_t seg_first[MU_MAXSEG];
  int32_t seg_slot[MU_MAXSEG];  // slot index (mutual) or -1 (one-sided)
};

__device__ __forceinline__ double4 mu_dummy_target() { return make_double4(-1e100, -1e100, -1e100, 0.0); }

// One pair, both directions (direct.cpp:156-169): d = x_t - x_s; the target gets
// +w_s (inv, inv^3 d), the source +w_t inv and -w_t inv^3 d. The target side is formed
// exactly as interact() forms it. SELF: i == j (r^2 = +0) contributes nothing.
// Measured alternatives (tools/gpu/gpu_r02t.sh, P2P ms at config B / D): the Newton step
// at dependency depth 4 (11.01 / 162.7 vs 10.90 / 159.5), and 23 DP instructions per pair
// (potentials fused into the accumulations, inv^3 shared; 12.04 / 163.0 with the tail
// tiles below): the kernel is latency-bound, a longer chain costs more than an
// instruction saves.
template <bool SELF>
__device__ __forceinline__ void mu_pair(const double4 pt, const double4 ps, const double c375, double4& at,
                                        double4& as) {
  const double dx = pt.x - ps.x, dy = pt.y - ps.y, dz = pt.z - ps.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  const double t = r2 * y;
  const double e = fma(-t, y, 1.0);
  double inv = fma(y, e * fma(e, c375, 0.5), y);
  if constexpr (SELF) inv = __double2hiint(r2) != 0 ? inv : 0.0;
  const double inv2 = inv * inv;
  const double ws = ps.w * inv, wt = pt.w * inv;
  at.x += ws;
  as.x += wt;
  const double st = ws * inv2, ss = wt * inv2;
  at.y = fma(st, dx, at.y);
  at.z = fma(st, dy, at.z);
  at.w = fma(st, dz, at.w);
  as.y = fma(-ss, dx, as.y);
  as.z = fma(-ss, dy, as.z);
  as.w = fma(-ss, dz, as.w);
}

__device__ __forceinline__ void add4(double4& a, const double4 b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// One target tile of RING (8, or 4 for a leaf's last 1..4 targets) at targets
// tpos[t0 .. t0+RING) against the lane's TS sources: each step every lane meets one target
// (TS pairs), then the target accumulators move one lane on around the lane's sub-ring;
// after RING steps lane l of every sub-ring holds its partial sums of target t0 + l, and
// the 32 / RING sub-rings are combined by a fixed butterfly (commutative pairs: every
// lane forms the bitwise same total).
// (Loading the next step's target a step ahead, against the short-scoreboard waits ncu's
// source view shows on the first subtraction: 166 registers, P2P 10.75 vs 10.50 ms at B,
// D 159.0 vs 156.0 ms; tools/gpu/gpu_r02bf.sh. Not adopted.)
template <int TS, int RING, bool SELF, class W>
__device__ __forceinline__ void mu_tile(W& w, const int t0, const double4 (&ps)[TS], double4 (&as)[TS],
                                        const int lane, const double c375) {
  const int lr = lane & (RING - 1);
  const int nxt = (lane & ~(RING - 1)) | ((lr + 1) & (RING - 1));
  const double4* tp = w.tpos + t0;
  double4 at = make_double4(0, 0, 0, 0);
#pragma unroll 2
  for (int s = 0; s < RING; ++s) {
    const double4 pt = tp[(lr + s) & (RING - 1)];
#pragma unroll
    for (int m = 0; m < TS; ++m) mu_pair<SELF>(pt, ps[m], c375, at, as[m]);
    at.x = __shfl_sync(0xffffffffu, at.x, nxt);
    at.y = __shfl_sync(0xffffffffu, at.y, nxt);
    at.z = __shfl_sync(0xffffffffu, at.z, nxt);
    at.w = __shfl_sync(0xffffffffu, at.w, nxt);
  }
#pragma unroll
  for (int o = RING; o < 32; o <<= 1) {
    at.x += __shfl_xor_sync(0xffffffffu, at.x, o);
    at.y += __shfl_xor_sync(0xffffffffu, at.y, o);
    at.z += __shfl_xor_sync(0xffffffffu, at.z, o);
    at.w += __shfl_xor_sync(0xffffffffu, at.w, o);
  }
  if (lane < RING) add4(w.iacc[t0 + lane], at);
}

// stream entry v -> (global particle index, slot index or -1). A lane's entries only grow
// (v = base + lane + 32 m, passes in increasing base), so its segment cursor only moves
// forward: 0-1 shared loads per entry (segments hold ~40 entries at config B) instead of a
// binary search over the 27 segments (6% of the kernel's stall samples in ncu's source view).
template <class W>
__device__ __forceinline__ uint64_t mu_locate(const W& w, int& cur, const uint32_t v, int& sl) {
  while (w.seg_off[cur + 1] <= v) ++cur;
  sl = w.seg_slot[cur];
  return uint64_t(w.seg_first[cur]) + (v - w.seg_off[cur]);
}

// One pass: TS sources per lane (stream entries base + lane + 32 m) against the tcn staged
// targets; then the sources' j-side sums go to their slots (the first target chunk
// writes them, later chunks of a large leaf add).
template <int TS, bool SELF, class W>
__device__ __forceinline__ void mu_pass(const MuArgs& a, W& w, int& cur, const uint32_t base,
                                        const uint32_t total, const int tcn, const bool first_chunk, const int lane,
                                        const double c375) {
  double4 ps[TS], as[TS];
  uint64_t dst[TS];
#pragma unroll
  for (int m = 0; m < TS; ++m) {
    const uint32_t v = base + static_cast<uint32_t>(lane + 32 * m);
    as[m] = make_double4(0, 0, 0, 0);
    dst[m] = ~0ull;
    if (v < total) {
      int sl;
      const uint64_t j = mu_locate(w, cur, v, sl);
      ps[m] = a.pw[j];
      if (sl >= 0) dst[m] = uint64_t(sl) * a.n + j;
    } else {
      ps[m] = dummy_source();
    }
  }
  // 8-target tiles, and a last tile of 4 when only 1..4 targets remain. (Tails of 4 + 2
  // targets, at most one dummy per chunk instead of up to 3, measured slower: P2P 12.49 vs
  // 10.90 ms at B -- the extra tile instantiation costs the main loop its schedule.)
  const int n8 = (tcn & 7) > 4 ? (tcn + 7) & ~7 : tcn & ~7;
#pragma unroll 1
  for (int t0 = 0; t0 < n8; t0 += 8) mu_tile<TS, 8, SELF>(w, t0, ps, as, lane, c375);
  if (tcn > n8) mu_tile<TS, 4, SELF>(w, n8, ps, as, lane, c375);
#pragma unroll
  for (int m = 0; m < TS; ++m) {
    if (dst[m] != ~0ull) {
      double4 r = as[m];
      if (!first_chunk) {
        const double4 o = a.slot[dst[m]];
        r = make_double4(o.x + r.x, o.y + r.y, o.z + r.z, o.w + r.w);
      }
      a.slot[dst[m]] = r;
    }
  }
}

template <bool SELF, class W>
__device__ __forceinline__ void mu_pass_ts(const int ts, const MuArgs& a, W& w, int& cur,
                                           const uint32_t base, const uint32_t total, const int tcn,
                                           const bool first_chunk, const int lane, const double c375) {
  switch (ts) {
    case 1: mu_pass<1, SELF>(a, w, cur, base, total, tcn, first_chunk, lane, c375); break;
    case 2: mu_pass<2, SELF>(a, w, cur, base, total, tcn, first_chunk, lane, c375); break;
    case 3: mu_pass<3, SELF>(a, w, cur, base, total, tcn, first_chunk, lane, c375); break;
#if FMMGPU_MU_TS > 4
    case 4: mu_pass<4, SELF>(a, w, cur, base, total, tcn, first_chunk, lane, c375); break;
    case 5: case 6: mu_pass<6, SELF>(a, w, cur, base, total, tcn, first_chunk, lane, c375); break;
#endif
    default: mu_pass<MU_TS, SELF>(a, w, cur, base, total, tcn, first_chunk, lane, c375); break;
  }
}

template <int TCAP>
__global__ void __launch_bounds__(MU_WARPS * 32, FMMGPU_MU_MINB) k_p2p_mutual(const MuArgs a) {
  extern __shared__ __align__(16) unsigned char mu_smem[];
  const int lane = threadIdx.x & 31;
  MuWarp<TCAP>& w = reinterpret_cast<MuWarp<TCAP>*>(mu_smem)[threadIdx.x >> 5];
  double c375 = 0.375;
  asm volatile("" : "+d"(c375));
  const uint32_t nl = a.c1 - a.c0;
  for (;;) {
    uint32_t u = 0;
    if (lane == 0) u = atomicAdd(a.ctr, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= nl) break;
    const uint32_t c = a.order ? a.order[u] : a.c0 + u;
    int ijk[3];
    demorton(a.leaf.code[c], ijk);
    const uint32_t cf = a.first[c], cn = a.count[c];
    // segments after the own leaf: lanes 0..12 the upper neighbours (mutual when owned,
    // else one-sided), lanes 13..25 the lower neighbours this rank does not own
    bool use = false;
    int sl = -1;
    uint32_t q = NPOS;
    if (lane < 2 * MU_NUP) {
      const int s = lane < MU_NUP ? lane : lane - MU_NUP;
      const int sg = lane < MU_NUP ? 1 : -1;
      int d[3];
      mu_up(s, d);
      q = find_ijk(a.leaf, ijk[0] + sg * d[0], ijk[1] + sg * d[1], ijk[2] + sg * d[2]);
      const bool owned = q != NPOS && q >= a.c0 && q < a.c1;
      use = lane < MU_NUP ? q != NPOS : (q != NPOS && !owned);
      sl = (lane < MU_NUP && owned) ? s : -1;
    }
    const uint32_t mask = __ballot_sync(0xffffffffu, use);
    const uint32_t cnt = use ? a.count[q] : 0u;
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t total = cn + __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t nseg = 1u + __popc(mask);
    if (use) {
      const int k = 1 + __popc(mask & ((1u << lane) - 1u));
      w.seg_off[k] = cn + incl - cnt;
      w.seg_first[k] = a.first[q];
      w.seg_slot[k] = sl;
    }
    if (lane == 0) {
      w.seg_off[0] = 0;
      w.seg_first[0] = cf;
      w.seg_slot[0] = -1;
      w.seg_off[nseg] = total;
    }
    for (uint32_t tc0 = 0; tc0 < cn; tc0 += TCAP) {
      const int tcn = static_cast<int>(min(static_cast<uint32_t>(TCAP), cn - tc0));
      __syncwarp();
      for (int i = lane; i < ((tcn + 7) & ~7); i += 32) {
        w.tpos[i] = i < tcn ? a.pw[cf + tc0 + i] : mu_dummy_target();
        w.iacc[i] = make_double4(0, 0, 0, 0);
      }
      __syncwarp();
      int cur = 0;  // this lane's segment cursor (mu_locate)
      for (uint32_t base = 0; base < total; base += 32 * MU_TS) {
        const int ts = static_cast<int>(min(static_cast<uint32_t>(MU_TS), (total - base + 31) / 32));
        if (base < cn) mu_pass_ts<true>(ts, a, w, cur, base, total, tcn, tc0 == 0, lane, c375);
        else mu_pass_ts<false>(ts, a, w, cur, base, total, tcn, tc0 == 0, lane, c375);
        __syncwarp();
      }
      for (int i = lane; i < tcn; i += 32) {
        const uint64_t tg = uint64_t(cf) + tc0 + i;
        double4 r = w.iacc[i];
        if (!a.ow) {
          const double4 o = a.near[tg];
          r = make_double4(o.x + r.x, o.y + r.y, o.z + r.z, o.w + r.w);
        }
        a.near[tg] = r;
      }
    }
    __syncwarp();
  }
}

// p2p_reduce (direct.cpp:187-200): near[j] += slot[s][j] in slot order, for every slot
// whose writer (the leaf q - d(s)) exists and is owned. One warp per leaf. A separate
// HBM-bound pass (0.77 ms at config B, 6 TB/s): draining inside k_p2p_mutual by the warp
// that completes a leaf's writer count (release atomics, L2 reads) measured slower
// (config B P2P 10.93 -> 14.07 ms, D 163 -> 177 ms).
__global__ void __launch_bounds__(256) k_p2p_drain(const MuArgs a) {
  const uint64_t wid = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= a.c1 - a.c0) return;
  const uint32_t q = a.c0 + static_cast<uint32_t>(wid);
  int ijk[3];
  demorton(a.leaf.code[q], ijk);
  bool has = false;
  if (lane < MU_NUP) {
    int d[3];
    mu_up(lane, d);
    const uint32_t c = find_ijk(a.leaf, ijk[0] - d[0], ijk[1] - d[1], ijk[2] - d[2]);
    has = c != NPOS && c >= a.c0 && c < a.c1;
  }
  const uint32_t mask = __ballot_sync(0xffffffffu, has);
  if (!mask) return;
  const uint32_t qf = a.first[q], qn = a.count[q];
  for (uint32_t i = lane; i < qn; i += 32) {
    const uint64_t j = uint64_t(qf) + i;
    double4 r = a.near[j];
#pragma unroll
    for (int s = 0; s < MU_NUP; ++s)
      if ((mask >> s) & 1u) add4(r, a.slot[uint64_t(s) * a.n + j]);
    a.near[j] = r;
  }
}

}  // namespace

namespace {
// work estimate of a leaf (its targets x its stream), complemented so an ascending radix
// sort puts the heaviest leaves first
__global__ void k_mu_work(const LevelView leaf, const uint32_t* __restrict__ count, const uint32_t c0,
                          const uint32_t nl, uint64_t* __restrict__ key, uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nl) return;
  const uint32_t c = c0 + i;
  int ijk[3];
  demorton(leaf.code[c], ijk);
  uint64_t tot = count[c];
  for (int s = 0; s < MU_NUP; ++s) {
    int d[3];
    mu_up(s, d);
    const uint32_t q = find_ijk(leaf, ijk[0] + d[0], ijk[1] + d[1], ijk[2] + d[2]);
    if (q != NPOS) tot += count[q];
  }
  key[i] = ~(uint64_t(count[c]) * tot);
  idx[i] = c;
}
}  // namespace

// The slot array of the current tree and, for trees with a non-full leaf level (clustered
// clouds, config D), the buffers of the largest-first leaf order: allocated with the tree
// on s_far (ordered before any evaluation's fork).
// Mode 2 (auto, the default) runs the mutual kernel when the (owned) leaf level has at
// least 8 leaves per resident warp: each warp owns a leaf from start to end, so a few
// large leaves leave most warps idle (config A, 512 leaves of ~195 particles: mutual 1.78
// ms, one-sided 0.6 ms), while the one-sided kernel splits a parent's work units over
// several CTAs.
bool p2p_use_mutual(const fmmgpu_ctx* c, uint32_t leaves) {
  if (c->p2p_mode != 2) return c->p2p_mode == 1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  return uint64_t(leaves) >= 8ull * static_cast<uint64_t>(sms) * MU_WARPS;
}

void ensure_p2p_slots(fmmgpu_ctx* c) {
  if (!c->have_tree || c->d_slot || !p2p_use_mutual(c, c->lv[c->height - 1].n)) return;
  c->d_slot = static_cast<double*>(cache_alloc(c, size_t(MU_NUP) * 32 * c->n, c->s_far));
  c->p2p_order_range[0] = c->p2p_order_range[1] = 0;
  const Level& L = c->lv[c->height - 1];
  if (L.full) return;
  size_t tmp = 0;
  FMM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, static_cast<const uint64_t*>(nullptr),
                                           static_cast<uint64_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                           static_cast<uint32_t*>(nullptr), static_cast<int>(L.n)));
  c->p2p_order_tmp = tmp;
  c->d_p2p_order = static_cast<uint32_t*>(cache_alloc(c, (24 + 1) * size_t(L.n) + tmp + 256, c->s_far));
}

namespace {
// the largest-first order of the owned leaves (recomputed when the owned range changed)
const uint32_t* p2p_order(fmmgpu_ctx* c, const Level& L, cudaStream_t s) {
  if (!c->d_p2p_order) return nullptr;
  if (c->p2p_order_range[0] == L.own0 && c->p2p_order_range[1] == L.own1 + 1) return c->d_p2p_order;
  const uint32_t nl = L.own1 - L.own0;
  auto* base = reinterpret_cast<unsigned char*>(c->d_p2p_order);
  uint32_t* out = c->d_p2p_order;                                   // [n] sorted leaves
  auto* idx = reinterpret_cast<uint32_t*>(base + 4 * size_t(L.n));  // [n]
  auto* key = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(base + 8 * size_t(L.n)) + 7) & ~uintptr_t(7));
  uint64_t* key2 = key + L.n;
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(key2 + L.n) + 255) & ~uintptr_t(255));
  k_mu_work<<<(nl + 255) / 256, 256, 0, s>>>(L.view(c->height - 1), L.particle_count, L.own0, nl, key, idx);
  FMM_CUDA(cudaGetLastError());
  size_t tb = c->p2p_order_tmp;
  FMM_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, idx, out, static_cast<int>(nl), 0, 64, s));
  c->launches += 2;
  c->p2p_order_range[0] = L.own0;
  c->p2p_order_range[1] = L.own1 + 1;
  return out;
}
}  // namespace

void launch_p2p(fmmgpu_ctx* c, cudaStream_t s, bool fuse_drain) {
  const int leaf = c->height - 1;
  const Level& L = c->lv[leaf];
  const Level& P = c->lv[leaf - 1];
  if (p2p_use_mutual(c, L.own1 - L.own0)) {
    if (!c->d_slot) throw Error(FMMGPU_LOGIC_ERROR, "mutual P2P: slot array not allocated");
    const uint32_t nl = L.own1 - L.own0;
    if (nl == 0) return;
    MuArgs a{L.view(leaf), L.first_particle, L.particle_count, c->d_pw, reinterpret_cast<double4*>(c->d_near),
             reinterpret_cast<double4*>(c->d_slot), c->n, L.own0, L.own1, c->d_ctr, p2p_order(c, L, s), c->ow ? 1 : 0};
    // 12-warp CTAs, one per SM at <= 168 registers (164 used): config B P2P 10.97 -> 10.89
    // ms, config D 163.4 -> 160.0 ms against 8-warp CTAs, 2 per SM at 128 registers. Also
    // measured (tools/gpu/gpu_r02g.sh, gpu_r02ax.sh): 11 warps at 164 registers (11.10 / 160.3 ms),
    // 13 warps at 128 (11.79 / 173.0), the next leaf claimed one leaf ahead (10.59 / 157.4 vs
    // 10.52 / 155.9: a warp holding a claimed leaf delays it), 10 warps at 164 registers
    // (11.36 / 165.2 ms), 8 warps
    // at up to 255 registers (11.97 / 171.7), 6 sources per lane with 8 or 12 warps (12.16 /
    // 162.2, 12.45 / 169.0), the pairs of a step written stage by stage (ptxas schedules
    // them the same way: no change). Loop ceiling of this sub-ring layout without memory
    // traffic or padding (tools/microbench/p2p_mutual_ceiling.cu): 8.0 ms at config B's
    // interaction count. Earlier measurements at config B (P2P 11.07 ms with 4 sources per
    // lane, the rotation unrolled twice, 8-warp CTAs, 2 per SM at 128 registers): 2 or 3 sources per lane with
    // two target tiles interleaved per step (11.72 / 12.23 ms), 3 CTAs per SM at 80
    // registers (11.77 ms, spills), 4-warp CTAs with 20 warps per SM (11.5 ms), the rotation
    // unrolled 4 / 8 times (12.3 / 17.8 ms, register pressure), the slot addresses
    // recomputed instead of held (11.36 ms).
    int sms = 148;
    FMM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    auto go = [&](auto kern, int smem) {
      int b = 0;
      FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, MU_WARPS * 32, smem) != cudaSuccess || b < 1) b = 1;
      // one CTA per SM: the kernel holds every SM for its ~10 ms and the far chain follows
      // (per-launch trace at config B: P2M starts at 10.45 ms); leaving 4-32 SMs to the far
      // chain measured 24.62-24.55 vs 24.65 ms per evaluation (the sum of the kernels is
      // the evaluation either way). Sharing each SM instead (8- or 6-warp near-field CTAs,
      // one per SM, every evaluation kernel at the maximum shared-memory carveout so the
      // far chain's CTAs co-reside; tools/gpu/gpu_r02ar.sh): 26.85 / 27.70 ms, the M2L
      // GEMMs and the pair loop compete for the one FP64 pipe
      const uint32_t grid = std::min<uint32_t>(static_cast<uint32_t>(sms * b), (nl + MU_WARPS - 1) / MU_WARPS);
      FMM_CUDA(cudaMemsetAsync(c->d_ctr, 0, sizeof(uint32_t), s));
      kern<<<grid, MU_WARPS * 32, smem, s>>>(a);
    };
    if (L.full) go(k_p2p_mutual<64>, static_cast<int>(MU_WARPS * sizeof(MuWarp<64>)));
    // non-full leaf levels: 256-target chunks (12 x 16.4 KB of shared memory): config D
    // 164.5 -> 162.5 ms per evaluation against 128 (192: 163.2), fewer passes over each
    // large leaf's source stream and fewer read-modify-writes of its slots
    else go(k_p2p_mutual<256>, static_cast<int>(MU_WARPS * sizeof(MuWarp<256>)));
    FMM_CUDA(cudaGetLastError());
    if (fuse_drain) {  // the drain happens in L2P (transfer.cu), after this event
      FMM_CUDA(cudaEventRecord(c->ev_p2p_main, s));
      c->launches += 1;
      return;
    }
    const uint64_t dthreads = uint64_t(nl) * 32;
    k_p2p_drain<<<static_cast<unsigned>((dthreads + 255) / 256), 256, 0, s>>>(a);
    FMM_CUDA(cudaGetLastError());
    c->launches += 2;
    return;
  }
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
