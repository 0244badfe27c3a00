// Chebyshev transfers on the device (InterpolationEngine, chebyshev.cpp:57-229),
// one launch per operator per level over all cells of that level:
//   P2M  warp per leaf cell; particles staged through shared memory in chunks of 32
//        as their three 1-D interpolation vectors (particle-minor), then lane p owns
//        the l coefficients of the pair p = (n1, n2) (chebyshev.cpp:116-136).
//   M2M  CTA per parent, warp per child: the three l x l passes of tensor_step in
//        shared memory (chebyshev.cpp:181-220), children summed in child order.
//   L2L  CTA per parent: own+down staged once, pushed into each child
//        (chebyshev.cpp:222-229, bench.cpp:300-316).
//   In an evaluation every operator writes its output (P2M and M2M also the zero
//   padding of the ldE stride) instead of accumulating into cleared arrays.
//   L2P  thread per particle, the n3 reduction factored as
//        sum_{n1,n2} (Sx Sy) * sum_{n3} L Sz (and the three gradient variants)
//        (chebyshev.cpp:138-179, bench.cpp:317-336); above order 5 the n2 sums are
//        factored as well.
// Templated on the order so every loop is unrolled with compile-time bounds.
#include <cstdlib>

#include "common.cuh"

namespace fmmgpu {

namespace {

struct Geo {  // root geometry for cell_cube (geometry.cpp:165-175)
  double lo[3];
  double cw;    // cell width at the operator's level
  double inv;   // 2 / cw
};

// cell centre exactly as geometry.cpp:173: (center - width/2) + (ijk + 0.5) * cw
__device__ __forceinline__ void cell_center(const Geo& g, uint64_t code, double c[3]) {
  int ijk[3];
  demorton(code, ijk);
  for (int a = 0; a < 3; ++a) c[a] = __dadd_rn(g.lo[a], __dmul_rn(static_cast<double>(ijk[a]) + 0.5, g.cw));
}

// eval_all / grad_all (chebyshev.cpp:78-114)
template <int L>
__device__ __forceinline__ void eval_all(const double* tn, double x, double* out) {
  double t[L > 1 ? L - 1 : 1];
  double tp = 1.0, tc = x;
#pragma unroll
  for (int n = 1; n < L; ++n) {
    t[n - 1] = tc;
    const double nx = 2.0 * x * tc - tp;
    tp = tc;
    tc = nx;
  }
#pragma unroll
  for (int m = 0; m < L; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int n = 0; n < L - 1; ++n) acc += tn[m * (L - 1) + n] * t[n];
    out[m] = 1.0 / L + 2.0 / L * acc;
  }
}
template <int L>
__device__ __forceinline__ void grad_all(const double* tn, double x, double* out) {
  double dt[L > 1 ? L - 1 : 1];
  double up = 1.0, uc = 2.0 * x;
#pragma unroll
  for (int n = 1; n < L; ++n) {
    dt[n - 1] = n * up;
    const double nx = 2.0 * x * uc - up;
    up = uc;
    uc = nx;
  }
#pragma unroll
  for (int m = 0; m < L; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int n = 0; n < L - 1; ++n) acc += tn[m * (L - 1) + n] * dt[n];
    out[m] = 2.0 / L * acc;
  }
}

struct LeafArgs {
  const uint64_t* code;
  const uint32_t* first;
  const uint32_t* count;
  const double4* pw;
  const uint32_t* pcell;
  const double* tn;
  double* expansion;       // multipole (P2M) or local_own (L2P)
  const double* down;      // local_down (L2P)
  double* far;             // [n] x {pot, fx, fy, fz} (L2P), Morton order
  uint64_t n;
  uint32_t cell0;   // first leaf cell of the launch (partitioned runs: the owned range)
  uint32_t ncells;  // one past the last leaf cell of the launch
  int ldE;
  Geo geo;
  int ow;  // overwrite (evaluation): P2M writes the multipole incl. zero padding, L2P writes far
  // L2P with the mutual near field's slot drain fused (evaluations): near[j] += slot[s][j]
  // in slot order for the slots whose writer leaf exists and is owned (k_p2p_drain)
  const double4* slot;  // [13][n], nullptr = no drain
  double4* near;
  LevelView leafv;
};

// upper half-shell direction of slot s (p2p.cu mu_up)
__device__ __forceinline__ void drain_dir(int s, int d[3]) {
  d[0] = s >= 4 ? 1 : 0;
  d[1] = s >= 4 ? (s - 4) / 3 - 1 : (s >= 1 ? 1 : 0);
  d[2] = s >= 4 ? (s - 4) % 3 - 1 : (s >= 1 ? s - 2 : 1);
}

constexpr int P2M_THREADS = 128;
constexpr int P2M_WARPS = P2M_THREADS / 32;

// P2M, warp per leaf cell, interpolation vectors stored particle-minor
// (sv[component][particle]) so one LDS.128 returns a component for two particles:
// per particle pair a lane reads a[n1], b[n2] (one LDS.128 each) and the l values
// c[0..l) (l LDS.128, broadcast) for 2 (l + 1) DP ops -- half the shared-memory
// instructions per FMA of a row-major layout, which is MIO-throttle bound. The
// reference's particle order and product order (wx, wxy, out += wxy sz). Chunks of 32
// particles; a chunk's odd tail is zero-padded. (The row-major layout, one LDS.64 per
// value, measured 1.00 vs 0.76 ms at config B.) Rows are padded to SVS = 34 doubles:
// with 32 the l rows a[n1] (and b[n2]) the lanes read at one column sit 256 B apart,
// in the same four banks, and each LDS.128 replays l times; at 34 they fall in disjoint
// banks (0.80 -> 0.56 ms at config B; with <= 128 registers, 4 CTAs per SM, 0.50 ms;
// 80 registers spill and measured 0.58; orders above 5 would spill at 128).
constexpr int P2M_SVS = 34;
template <int L>
__global__ void __launch_bounds__(P2M_THREADS, L <= 5 ? 4 : 1) k_p2m_warp2(LeafArgs a) {
  constexpr int PP = (L * L + 31) / 32;  // (n1, n2) pairs per lane
  __shared__ double tn[L * (L - 1) + 1];
  __shared__ __align__(16) double SV[P2M_WARPS][3 * L][P2M_SVS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < L * (L - 1); i += P2M_THREADS) tn[i] = a.tn[i];
  __syncthreads();
  const uint32_t c = a.cell0 + blockIdx.x * P2M_WARPS + warp;
  if (c >= a.ncells) return;
  double ctr[3];
  cell_center(a.geo, a.code[c], ctr);
  const uint32_t first = a.first[c], cnt = a.count[c];
  double* out = a.expansion + size_t(c) * a.ldE;
  const double4 zero4 = make_double4(0, 0, 0, 0);
  const double4 q0 = lane < cnt ? a.pw[first + lane] : zero4;
  const double4 q1 = lane + 32 < cnt ? a.pw[first + 32 + lane] : zero4;
  double acc[PP][L];
#pragma unroll
  for (int i = 0; i < PP; ++i)
#pragma unroll
    for (int n = 0; n < L; ++n) acc[i][n] = (!a.ow && lane + 32 * i < L * L) ? out[(lane + 32 * i) * L + n] : 0.0;
  if (a.ow)
    for (int i = L * L * L + lane; i < a.ldE; i += 32) out[i] = 0.0;  // padding read by M2L phase A (K = ldE)
  double(*sv)[P2M_SVS] = SV[warp];
  for (uint32_t base = 0; base < cnt; base += 32) {
    double s[L];
    if (base + lane < cnt) {
      const double4 p = base == 0 ? q0 : base == 32 ? q1 : a.pw[first + base + lane];
      eval_all<L>(tn, (p.x - ctr[0]) * a.geo.inv, s);
#pragma unroll
      for (int m = 0; m < L; ++m) sv[m][lane] = p.w * s[m];
      eval_all<L>(tn, (p.y - ctr[1]) * a.geo.inv, s);
#pragma unroll
      for (int m = 0; m < L; ++m) sv[L + m][lane] = s[m];
      eval_all<L>(tn, (p.z - ctr[2]) * a.geo.inv, s);
#pragma unroll
      for (int m = 0; m < L; ++m) sv[2 * L + m][lane] = s[m];
    } else {
#pragma unroll
      for (int m = 0; m < 3 * L; ++m) sv[m][lane] = 0.0;
    }
    __syncwarp();
    const int m2 = static_cast<int>(min(32u, cnt - base) + 1) & ~1;  // particle pairs
#pragma unroll
    for (int i = 0; i < PP; ++i) {
      const int pr = lane + 32 * i;
      if (pr < L * L) {
        const int n1 = pr / L, n2 = pr % L;
        for (int j = 0; j < m2; j += 2) {
          const double2 av = *reinterpret_cast<const double2*>(&sv[n1][j]);
          const double2 bv = *reinterpret_cast<const double2*>(&sv[L + n2][j]);
          double2 cv[L];
#pragma unroll
          for (int n = 0; n < L; ++n) cv[n] = *reinterpret_cast<const double2*>(&sv[2 * L + n][j]);
          const double ab0 = av.x * bv.x;
#pragma unroll
          for (int n = 0; n < L; ++n) acc[i][n] = fma(ab0, cv[n].x, acc[i][n]);
          const double ab1 = av.y * bv.y;
#pragma unroll
          for (int n = 0; n < L; ++n) acc[i][n] = fma(ab1, cv[n].y, acc[i][n]);
        }
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int i = 0; i < PP; ++i) {
    const int pr = lane + 32 * i;
    if (pr < L * L)
#pragma unroll
      for (int n = 0; n < L; ++n) out[pr * L + n] = acc[i][n];
  }
}

// L2P, CTA per run of L2P_CELLS consecutive leaf cells: total = own + down is formed
// once per cell in shared memory (bench.cpp:320-325), then thread per particle of
// those cells (contiguous in Morton order) reads it as (near-)broadcast LDS.
constexpr int L2P_CELLS = 8, L2P_THREADS = 128;

template <int L, bool L2P_FACTORED, int MINB>
__global__ void __launch_bounds__(L2P_THREADS, MINB > 0 ? MINB : 0) k_l2p_block(LeafArgs a) {
  constexpr int L3 = L * L * L;
  extern __shared__ __align__(16) double tot[];  // [L2P_CELLS][L3]
  __shared__ double tn[L * (L - 1) + 1];
  __shared__ uint32_t cfirst[L2P_CELLS + 1];
  __shared__ double cctr[L2P_CELLS][3];
  __shared__ uint32_t cmask[L2P_CELLS];  // fused drain: slots present per cell
  const uint32_t c0 = a.cell0 + blockIdx.x * L2P_CELLS;
  const uint32_t nc = min(static_cast<uint32_t>(L2P_CELLS), a.ncells - c0);
  const uint64_t p0 = a.first[c0], p1 = uint64_t(a.first[c0 + nc - 1]) + a.count[c0 + nc - 1];
  // the first particle of each thread: position and accumulated fields in flight
  // while the cells' totals are staged
  const uint64_t s_first = p0 + threadIdx.x;
  const double4 zero4 = make_double4(0, 0, 0, 0);
  const double4 pf = s_first < p1 ? a.pw[s_first] : zero4;
  double4* far4 = reinterpret_cast<double4*>(a.far);
  const double4 ff = s_first < p1 && !a.ow ? far4[s_first] : zero4;
  if (threadIdx.x < nc) {
    const uint32_t c = c0 + threadIdx.x;
    cfirst[threadIdx.x] = a.first[c];
    cell_center(a.geo, a.code[c], cctr[threadIdx.x]);
  }
  if (threadIdx.x == 0) cfirst[nc] = static_cast<uint32_t>(p1);
  if (a.slot) {
    if (threadIdx.x < L2P_CELLS) cmask[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < nc * 13; e += L2P_THREADS) {
      const uint32_t lc = e / 13, sl = e % 13, q = c0 + lc;
      int ijk[3], d[3];
      demorton(a.code[q], ijk);
      drain_dir(static_cast<int>(sl), d);
      const uint32_t w = find_ijk(a.leafv, ijk[0] - d[0], ijk[1] - d[1], ijk[2] - d[2]);
      if (w != NPOS && w >= a.cell0 && w < a.ncells) atomicOr(&cmask[lc], 1u << sl);
    }
  }
  for (int i = threadIdx.x; i < L * (L - 1); i += L2P_THREADS) tn[i] = a.tn[i];
  // staged 4 elements at a time so the loads of a thread are in flight together
  for (uint32_t i0 = threadIdx.x; i0 < nc * L3; i0 += 4 * L2P_THREADS) {
    double e[4], d[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = i0 + u * L2P_THREADS;
      if (i < nc * L3) {
        const size_t g = size_t(c0 + i / L3) * a.ldE + i % L3;
        e[u] = a.expansion[g];
        d[u] = a.down[g];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = i0 + u * L2P_THREADS;
      if (i < nc * L3) tot[i] = e[u] + d[u];
    }
  }
  __syncthreads();
  const double inv = a.geo.inv;
  double4 pnext = pf, fnext = ff;
  for (uint64_t s = s_first; s < p1; s += L2P_THREADS) {
    uint32_t lc = 0;  // local cell of slot s (cells are contiguous in Morton order)
    while (lc + 1 < nc && cfirst[lc + 1] <= s) ++lc;
    const uint32_t c = c0 + lc;
    const double* ctr = cctr[lc];
    const double4 p = pnext;
    const double4 fprev = fnext;
    if (s + L2P_THREADS < p1) {  // next particle's loads overlap this one's arithmetic
      pnext = a.pw[s + L2P_THREADS];
      fnext = a.ow ? zero4 : far4[s + L2P_THREADS];
    }
    const double rx = (p.x - ctr[0]) * inv, ry = (p.y - ctr[1]) * inv, rz = (p.z - ctr[2]) * inv;
    double sx[L], sy[L], sz[L], gx[L], gy[L], gz[L];
    eval_all<L>(tn, rx, sx);
    eval_all<L>(tn, ry, sy);
    eval_all<L>(tn, rz, sz);
    grad_all<L>(tn, rx, gx);
    grad_all<L>(tn, ry, gy);
    grad_all<L>(tn, rz, gz);
    const double* t = tot + (c - c0) * L3;
    double pot = 0, dx = 0, dy = 0, dz = 0;
    constexpr int UNROLL_N1 = L <= 7 ? L : 1;  // keep sx/gx in registers
#pragma unroll UNROLL_N1
    for (int n1 = 0; n1 < L; ++n1) {
      if constexpr (L2P_FACTORED) {
        // the n2 sums factored too: a1 = sum sy u, a2 = sum gy u, a3 = sum sy w, then
        // pot += sx a1, dx += gx a1, dy += sx a2, dz += sx a3 (3 instead of 7 DP per (n1, n2))
        double a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
        for (int n2 = 0; n2 < L; ++n2) {
          double u = 0, w = 0;
#pragma unroll
          for (int n3 = 0; n3 < L; ++n3) {
            const double v = t[(n1 * L + n2) * L + n3];
            u = fma(v, sz[n3], u);
            w = fma(v, gz[n3], w);
          }
          a1 = fma(sy[n2], u, a1);
          a2 = fma(gy[n2], u, a2);
          a3 = fma(sy[n2], w, a3);
        }
        pot = fma(sx[n1], a1, pot);
        dx = fma(gx[n1], a1, dx);
        dy = fma(sx[n1], a2, dy);
        dz = fma(sx[n1], a3, dz);
      } else {
#pragma unroll
      for (int n2 = 0; n2 < L; ++n2) {
        double u = 0, w = 0;
#pragma unroll
        for (int n3 = 0; n3 < L; ++n3) {
          const double v = t[(n1 * L + n2) * L + n3];
          u = fma(v, sz[n3], u);
          w = fma(v, gz[n3], w);
        }
        const double ss = sx[n1] * sy[n2];
        pot = fma(ss, u, pot);
        dx = fma(gx[n1] * sy[n2], u, dx);
        dy = fma(sx[n1] * gy[n2], u, dy);
        dz = fma(ss, w, dz);
      }
      }
    }
    double4 r = fprev;
    r.x += pot;
    r.y -= inv * dx;
    r.z -= inv * dy;
    r.w -= inv * dz;
    far4[s] = r;
    if (a.slot) {  // p2p_reduce of this particle (the k_p2p_drain order)
      const uint32_t m = cmask[lc];
      double4 nr = a.near[s];
#pragma unroll
      for (int sl = 0; sl < 13; ++sl)
        if ((m >> sl) & 1u) {
          const double4 v = a.slot[uint64_t(sl) * a.n + s];
          nr.x += v.x;
          nr.y += v.y;
          nr.z += v.z;
          nr.w += v.w;
        }
      a.near[s] = nr;
    }
  }
}

struct TransArgs {
  const uint64_t* child_code;
  const uint32_t* first_child;
  const uint32_t* child_count;
  const double* mats;      // [2][L*L]: child_t (M2M) or child (L2L)
  const double* parent_a;  // M2M: unused; L2L: local_own of parents
  const double* parent_b;  // L2L: local_down of parents
  const double* child_in;  // M2M: child multipoles
  double* out;             // M2M: parent multipole; L2L: child local_down
  uint32_t p0;             // first parent of the launch (partitioned runs: the owned range)
  uint32_t nparents;
  int ldE;
  int ow;  // overwrite (evaluation): M2M writes the parent incl. zero padding, L2L writes local_down
};

// dst[r*L + n] = sum_k mt[k*L + n] * src[k*L*L + r]  (tensor_step, chebyshev.cpp:186-199)
template <int L>
__device__ __forceinline__ double step_one(const double* mt, const double* src, int idx) {
  const int r = idx / L, n = idx % L;
  double acc = 0;
#pragma unroll
  for (int k = 0; k < L; ++k) acc += mt[k * L + n] * src[k * L * L + r];
  return acc;
}

// M2M / L2L, CTA per parent with one warp per child (<= 8): each warp runs the three
// l x l passes of tensor_step (chebyshev.cpp:181-211) on its own shared buffers with
// __syncwarp only. M2M sums the children's contributions into the parent in child
// order (the reference's order, bench.cpp:280-284); L2L stages own+down of the parent
// once (bench.cpp:308-309) and each warp accumulates into its child's local_down.
// One output row of tensor_step: dst[r*L + n] = sum_k mt[k*L + n] * src[k*L*L + r] for
// all n -- the L source values are loaded once per row instead of once per output.
template <int L>
__device__ __forceinline__ void step_row(const double* mt, const double* src, int r, double* out) {
  double s[L];
#pragma unroll
  for (int k = 0; k < L; ++k) s[k] = src[k * L * L + r];
#pragma unroll
  for (int n = 0; n < L; ++n) {
    double acc = 0;
#pragma unroll
    for (int k = 0; k < L; ++k) acc += mt[k * L + n] * s[k];
    out[n] = acc;
  }
}

template <int L, bool IS_M2M>
__global__ void __launch_bounds__(256) k_transfer_warp(TransArgs a) {
  constexpr int L3 = L * L * L;
  __shared__ double mats[2 * L * L];
  __shared__ double par[L3];
  __shared__ double buf[8][2][L3];
  const uint32_t p = a.p0 + blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 2 * L * L; i += 256) mats[i] = a.mats[i];
  if (!IS_M2M) {  // own + down of the parent, every load of a thread in flight together
    constexpr int NP = (L3 + 255) / 256;
    const double* pa = a.parent_a + size_t(p) * a.ldE;
    const double* pb = a.parent_b + size_t(p) * a.ldE;
    double va[NP], vb[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int i = tid + 256 * j;
      va[j] = i < L3 ? pa[i] : 0.0;
      vb[j] = i < L3 ? pb[i] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NP; ++j)
      if (tid + 256 * j < L3) par[tid + 256 * j] = va[j] + vb[j];
  }
  __syncthreads();
  const uint32_t f = a.first_child[p], nch = a.child_count[p];
  if (warp < static_cast<int>(nch)) {
    const uint32_t ch = f + warp;
    const int oct = static_cast<int>(a.child_code[ch] & 7);
    const double* m0 = mats + ((oct >> 2) & 1) * L * L;
    const double* m1 = mats + ((oct >> 1) & 1) * L * L;
    const double* m2 = mats + (oct & 1) * L * L;
    double* b0 = buf[warp][0];
    double* b1 = buf[warp][1];
    const double* src = par;
    if (IS_M2M) {
      // all of a lane's loads in flight together (one DRAM round trip, not L3/32)
      constexpr int NL = (L3 + 31) / 32;
      const double* cin = a.child_in + size_t(ch) * a.ldE;
      double v[NL];
#pragma unroll
      for (int j = 0; j < NL; ++j) v[j] = lane + 32 * j < L3 ? cin[lane + 32 * j] : 0.0;
#pragma unroll
      for (int j = 0; j < NL; ++j)
        if (lane + 32 * j < L3) b1[lane + 32 * j] = v[j];
      __syncwarp();
      src = b1;
    }
    double o[L];
    for (int r = lane; r < L * L; r += 32) {
      step_row<L>(m0, src, r, o);
#pragma unroll
      for (int n = 0; n < L; ++n) b0[r * L + n] = o[n];
    }
    __syncwarp();
    for (int r = lane; r < L * L; r += 32) {
      step_row<L>(m1, b0, r, o);
#pragma unroll
      for (int n = 0; n < L; ++n) b1[r * L + n] = o[n];
    }
    __syncwarp();
    if (IS_M2M) {
      for (int r = lane; r < L * L; r += 32) {
        step_row<L>(m2, b1, r, o);
#pragma unroll
        for (int n = 0; n < L; ++n) b0[r * L + n] = o[n];  // b0 is free again after pass 2
      }
    } else {
      // the last pass goes to shared memory (b0 is free again), then out is written
      // coalesced: a row-strided store touches a sector per lane (with the unrolled
      // staging loads: config-C evaluation 90.4 -> 89.7 ms; order 5 unchanged)
      for (int r = lane; r < L * L; r += 32) {
        step_row<L>(m2, b1, r, o);
#pragma unroll
        for (int n = 0; n < L; ++n) b0[r * L + n] = o[n];
      }
      __syncwarp();
      double* out = a.out + size_t(ch) * a.ldE;
      constexpr int NL = (L3 + 31) / 32;
      if (a.ow) {
#pragma unroll
        for (int j = 0; j < NL; ++j)
          if (lane + 32 * j < L3) out[lane + 32 * j] = b0[lane + 32 * j];
      } else {
        double v[NL];
#pragma unroll
        for (int j = 0; j < NL; ++j) v[j] = lane + 32 * j < L3 ? out[lane + 32 * j] : 0.0;
#pragma unroll
        for (int j = 0; j < NL; ++j)
          if (lane + 32 * j < L3) out[lane + 32 * j] = v[j] + b0[lane + 32 * j];
      }
    }
  }
  if (IS_M2M) {
    __syncthreads();
    double* out = a.out + size_t(p) * a.ldE;
    for (int i = tid; i < L3; i += 256) {
      double acc = a.ow ? 0.0 : out[i];
      for (uint32_t c = 0; c < nch; ++c) acc += buf[c][0][i];
      out[i] = acc;
    }
    if (a.ow)
      for (int i = L3 + tid; i < a.ldE; i += 256) out[i] = 0.0;
  }
}

template <int L, bool IS_M2M>
__global__ void __launch_bounds__(128) k_transfer(TransArgs a) {
  constexpr int L3 = L * L * L;
  constexpr int OPT = (L3 + 127) / 128;
  __shared__ double mats[2 * L * L];
  __shared__ double buf0[L3], buf1[L3], par[IS_M2M ? 1 : L3];
  const uint32_t p = a.p0 + blockIdx.x;
  const int tid = threadIdx.x;
  for (int i = tid; i < 2 * L * L; i += 128) mats[i] = a.mats[i];
  if (!IS_M2M)
    for (int i = tid; i < L3; i += 128) par[i] = a.parent_a[size_t(p) * a.ldE + i] + a.parent_b[size_t(p) * a.ldE + i];
  const uint32_t f = a.first_child[p], e = f + a.child_count[p];
  double acc[OPT];
#pragma unroll
  for (int o = 0; o < OPT; ++o) acc[o] = 0;
  for (uint32_t ch = f; ch < e; ++ch) {
    const int oct = static_cast<int>(a.child_code[ch] & 7);
    const double* m0 = mats + ((oct >> 2) & 1) * L * L;
    const double* m1 = mats + ((oct >> 1) & 1) * L * L;
    const double* m2 = mats + (oct & 1) * L * L;
    __syncthreads();
    const double* src0 = par;
    if (IS_M2M) {
      for (int i = tid; i < L3; i += 128) buf1[i] = a.child_in[size_t(ch) * a.ldE + i];
      __syncthreads();
      src0 = buf1;
    }
    for (int i = tid; i < L3; i += 128) buf0[i] = step_one<L>(m0, src0, i);
    __syncthreads();
    for (int i = tid; i < L3; i += 128) buf1[i] = step_one<L>(m1, buf0, i);
    __syncthreads();
    if (IS_M2M) {
#pragma unroll
      for (int o = 0; o < OPT; ++o) {
        const int i = tid + o * 128;
        if (i < L3) acc[o] += step_one<L>(m2, buf1, i);
      }
    } else {
      double* out = a.out + size_t(ch) * a.ldE;
      for (int i = tid; i < L3; i += 128) {
        const double v = step_one<L>(m2, buf1, i);
        out[i] = a.ow ? v : out[i] + v;
      }
    }
  }
  if (IS_M2M) {
    double* out = a.out + size_t(p) * a.ldE;
#pragma unroll
    for (int o = 0; o < OPT; ++o) {
      const int i = tid + o * 128;
      if (i < L3) out[i] = a.ow ? acc[o] : out[i] + acc[o];
    }
    if (a.ow)
      for (int i = L3 + tid; i < a.ldE; i += 128) out[i] = 0.0;
  }
}

// FmmContext::gather (bench.cpp:350-365): input slot o reads its Morton slot
// inv[o] (one 32-byte sector per field array) and writes the four fields coalesced.
// Partitioned runs own the Morton slots [s0, s1); other slots are written as zero.
__global__ void k_gather(const double4* __restrict__ far, const double4* __restrict__ near,
                         const uint32_t* __restrict__ inv, uint64_t n, uint64_t s0, uint64_t s1,
                         double* __restrict__ out) {
  const uint64_t o = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (o >= n) return;
  const uint32_t s = inv[o];
  const bool own = s >= s0 && s < s1;
  const double4 z = make_double4(0, 0, 0, 0);
  const double4 f = own ? far[s] : z, e = own ? near[s] : z;
  out[o] = f.x + e.x;
  out[n + o] = f.y + e.y;
  out[2 * n + o] = f.z + e.z;
  out[3 * n + o] = f.w + e.w;
}

Geo make_geo(const fmmgpu_ctx* c, int level) {
  Geo g;
  for (int a = 0; a < 3; ++a) g.lo[a] = c->lo[a];
  g.cw = c->root[3] / static_cast<double>(uint64_t{1} << level);  // geometry.cpp:163-165
  g.inv = 2.0 / g.cw;                                               // chebyshev.cpp:120
  return g;
}

template <template <int> class F, typename... Args>
void dispatch_order(int order, Args&&... args) {
  switch (order) {
    case 2: F<2>::run(args...); break;
    case 3: F<3>::run(args...); break;
    case 4: F<4>::run(args...); break;
    case 5: F<5>::run(args...); break;
    case 6: F<6>::run(args...); break;
    case 7: F<7>::run(args...); break;
    case 8: F<8>::run(args...); break;
    case 9: F<9>::run(args...); break;
    case 10: F<10>::run(args...); break;
    default: throw Error(FMMGPU_INVALID_ARGUMENT, "order must be in [2, 10]");
  }
}

template <int L>
struct RunP2M {
  static void run(const LeafArgs& a, cudaStream_t s) {
    const uint32_t nc = a.ncells - a.cell0;
    if (!nc) return;
    k_p2m_warp2<L><<<(nc + P2M_WARPS - 1) / P2M_WARPS, P2M_THREADS, 0, s>>>(a);
  }
};
template <int L>
struct RunL2P {
  static void run(const LeafArgs& a, cudaStream_t s) {
    const uint32_t nc = a.ncells - a.cell0;
    if (!nc) return;
    const int smem = static_cast<int>(sizeof(double) * L2P_CELLS * L * L * L);
    // orders <= 5: the (n1, n2) loop as written, <= 128 registers (4 CTAs per SM);
    // higher orders: the n2 sums factored as well (config-C leaf 1.65 -> 1.22 ms; at
    // order 5 the factored loop needs 162-188 registers and measured 0.59-0.79 vs 0.56 ms)
    constexpr bool factored = L > 5;
    // (5 / 6 CTAs per SM at 96 / 80 registers with small spills: B 24.25 / 24.41-24.58 vs
    // 24.28-24.46 ms, E 234.2 / 235.4 vs 233.6 ms; tools/gpu/gpu_r02be.sh: kept at 4)
    auto kern = k_l2p_block<L, factored, factored ? 0 : 4>;
    FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<(nc + L2P_CELLS - 1) / L2P_CELLS, L2P_THREADS, smem, s>>>(a);
  }
};
template <int L>
struct RunM2M {
  static void run(const TransArgs& a, cudaStream_t s) {
    if (!a.nparents) return;
    if constexpr (L <= 7) k_transfer_warp<L, true><<<a.nparents, 256, 0, s>>>(a);  // 48 KB static smem
    else k_transfer<L, true><<<a.nparents, 128, 0, s>>>(a);
  }
};
template <int L>
struct RunL2L {
  static void run(const TransArgs& a, cudaStream_t s) {
    if (!a.nparents) return;
    if constexpr (L <= 7) k_transfer_warp<L, false><<<a.nparents, 256, 0, s>>>(a);
    else k_transfer<L, false><<<a.nparents, 128, 0, s>>>(a);
  }
};

LeafArgs leaf_args(fmmgpu_ctx* c) {
  const int leaf = c->height - 1;
  const Level& L = c->lv[leaf];
  LeafArgs a{};
  a.code = L.code;
  a.first = L.first_particle;
  a.count = L.particle_count;
  a.pw = c->d_pw;
  a.pcell = c->d_pcell;
  a.tn = c->d_interp;
  a.n = c->n;
  a.cell0 = L.own0;  // partitioned runs: this rank's leaves only
  a.ncells = L.own1;
  a.ldE = c->ldE;
  a.geo = make_geo(c, leaf);
  return a;
}

}  // namespace

void interp_setup(fmmgpu_ctx* c) {
  // InterpolationEngine ctor (chebyshev.cpp:57-76), host arithmetic
  const int l = c->order;
  auto cheb_t = [](int n, double x) {
    double tp = 1.0, t = x;
    if (n == 0) return tp;
    for (int i = 1; i < n; ++i) {
      const double nx = 2.0 * x * t - tp;
      tp = t;
      t = nx;
    }
    return t;
  };
  c->h_roots.resize(l);
  for (int m = 0; m < l; ++m) c->h_roots[m] = std::cos((2 * m + 1) * 3.14159265358979323846 / (2 * l));
  c->h_tn.assign(size_t(l) * (l - 1), 0.0);
  for (int m = 0; m < l; ++m)
    for (int n = 1; n < l; ++n) c->h_tn[m * (l - 1) + n - 1] = cheb_t(n, c->h_roots[m]);
  auto s_eval = [&](double root, double x) {
    double acc = 1.0 / l;
    for (int n = 1; n < l; ++n) acc += (2.0 / l) * cheb_t(n, root) * cheb_t(n, x);
    return acc;
  };
  for (int side = 0; side < 2; ++side) {
    c->h_child[side].assign(l * l, 0.0);
    c->h_child_t[side].assign(l * l, 0.0);
    const double shift = side == 0 ? -0.5 : 0.5;
    for (int m = 0; m < l; ++m)
      for (int k = 0; k < l; ++k) {
        const double v = s_eval(c->h_roots[m], 0.5 * c->h_roots[k] + shift);
        c->h_child[side][m * l + k] = v;
        c->h_child_t[side][k * l + m] = v;
      }
  }
  // device layout: [tn (l*(l-1)) padded to l*l][child0][child1][child_t0][child_t1]
  std::vector<double> h(5 * l * l, 0.0);
  std::copy(c->h_tn.begin(), c->h_tn.end(), h.begin());
  std::copy(c->h_child[0].begin(), c->h_child[0].end(), h.begin() + l * l);
  std::copy(c->h_child[1].begin(), c->h_child[1].end(), h.begin() + 2 * l * l);
  std::copy(c->h_child_t[0].begin(), c->h_child_t[0].end(), h.begin() + 3 * l * l);
  std::copy(c->h_child_t[1].begin(), c->h_child_t[1].end(), h.begin() + 4 * l * l);
  FMM_CUDA(cudaMalloc(&c->d_interp, h.size() * sizeof(double)));
  FMM_CUDA(cudaMemcpy(c->d_interp, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
}

void launch_p2m(fmmgpu_ctx* c, cudaStream_t s) {
  LeafArgs a = leaf_args(c);
  a.expansion = c->lv[c->height - 1].multipole;
  a.ow = c->ow;
  dispatch_order<RunP2M>(c->order, a, s);
  FMM_CUDA(cudaGetLastError());
  ++c->launches;
}

void launch_l2p(fmmgpu_ctx* c, cudaStream_t s, bool drain) {
  LeafArgs a = leaf_args(c);
  a.expansion = c->lv[c->height - 1].local_own;
  a.down = c->lv[c->height - 1].local_down;
  a.far = c->d_far;
  a.ow = c->ow;
  if (drain) {
    a.slot = reinterpret_cast<const double4*>(c->d_slot);
    a.near = reinterpret_cast<double4*>(c->d_near);
    a.leafv = c->lv[c->height - 1].view(c->height - 1);
  }
  dispatch_order<RunL2P>(c->order, a, s);
  FMM_CUDA(cudaGetLastError());
  ++c->launches;
}

void launch_m2m(fmmgpu_ctx* c, int v, cudaStream_t s) {
  const int l = c->order;
  TransArgs a{};
  a.child_code = c->lv[v + 1].code;
  a.first_child = c->lv[v].first_child;
  a.child_count = c->lv[v].child_count;
  a.mats = c->d_interp + 3 * l * l;  // child_t
  a.child_in = c->lv[v + 1].multipole;
  a.out = c->lv[v].multipole;
  a.ow = c->ow;
  a.p0 = c->lv[v].own0;
  a.nparents = c->lv[v].own1 - c->lv[v].own0;
  a.ldE = c->ldE;
  dispatch_order<RunM2M>(l, a, s);
  FMM_CUDA(cudaGetLastError());
  ++c->launches;
}

void launch_l2l(fmmgpu_ctx* c, int v, cudaStream_t s) {
  const int l = c->order;
  TransArgs a{};
  a.child_code = c->lv[v + 1].code;
  a.first_child = c->lv[v].first_child;
  a.child_count = c->lv[v].child_count;
  a.mats = c->d_interp + l * l;  // child
  a.parent_a = c->lv[v].local_own;
  a.parent_b = c->lv[v].local_down;
  a.out = c->lv[v + 1].local_down;
  a.ow = c->ow;
  a.p0 = c->lv[v].own0;
  a.nparents = c->lv[v].own1 - c->lv[v].own0;
  a.ldE = c->ldE;
  dispatch_order<RunL2L>(l, a, s);
  FMM_CUDA(cudaGetLastError());
  ++c->launches;
}

void launch_gather(fmmgpu_ctx* c, cudaStream_t s) {
  k_gather<<<static_cast<unsigned>((c->n + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<const double4*>(c->d_far), reinterpret_cast<const double4*>(c->d_near), c->d_inv, c->n,
      c->own_s0, c->own_s1, c->d_out);
  FMM_CUDA(cudaGetLastError());
  ++c->launches;
}

}  // namespace fmmgpu
