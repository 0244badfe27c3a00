// Octree construction on the device: GroupTree::build (geometry.cpp:73-161) as
// reductions, a stable LSD radix sort of (Morton key, input index) and run-length
// encodes. Bit-exact with the reference: keys come from the same IEEE FP64 ops
// (explicit _rn intrinsics, no FMA contraction), the sort is stable so ties keep
// input order exactly like std::sort on (key, index) pairs (geometry.cpp:95).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace fmmgpu {

namespace {

template <typename T>
T* dalloc(fmmgpu_ctx* c, size_t count, cudaStream_t s) {
  return static_cast<T*>(cache_alloc(c, (count ? count : 1) * sizeof(T), s));
}
template <typename T>
void dfree(fmmgpu_ctx* c, T*& p, cudaStream_t s) {
  if (p) cache_free(c, p, s);
  p = nullptr;
}

// FMMGPU_TRACE=1: host wall time of the tree-build phases on stderr (development aid)
struct PhaseTrace {
  bool on = std::getenv("FMMGPU_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void operator()(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tree] %-24s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// bounding_cube (geometry.cpp:18-36): per-axis min / max. Exact (order-free).
__global__ void k_minmax_partial(const double4* __restrict__ p, uint64_t n, double* __restrict__ part) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const double4 q = p[i];
    mn[0] = fmin(mn[0], q.x); mx[0] = fmax(mx[0], q.x);
    mn[1] = fmin(mn[1], q.y); mx[1] = fmax(mx[1], q.y);
    mn[2] = fmin(mn[2], q.z); mx[2] = fmax(mx[2], q.z);
  }
  __shared__ double sm[6][32];
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = fmin(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = fmax(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int a = 0; a < 3; ++a) { sm[a][w] = mn[a]; sm[3 + a][w] = mx[a]; }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int nw = blockDim.x >> 5;
    double r = sm[threadIdx.x][0];
    for (int i = 1; i < nw; ++i) r = threadIdx.x < 3 ? fmin(r, sm[threadIdx.x][i]) : fmax(r, sm[threadIdx.x][i]);
    part[threadIdx.x * gridDim.x + blockIdx.x] = r;
  }
}

// Morton key per particle (geometry.cpp:76-94): u = floor((c - lo) / cw), clamped.
template <typename K>  // uint32_t when 3 * leaf <= 32 (height <= 11): half the sort traffic
__global__ void k_keys(const double4* __restrict__ p, uint64_t n, double lo0, double lo1, double lo2,
                       double hi0, double hi1, double hi2, double cw, uint32_t grid,
                       K* __restrict__ keys, uint32_t* __restrict__ idx, int* __restrict__ flag) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double4 q = p[i];
  const double c[3] = {q.x, q.y, q.z}, lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
  uint32_t ijk[3];
  for (int a = 0; a < 3; ++a) {
    if (c[a] < lo[a] || c[a] > hi[a]) atomicOr(flag, 1);  // domain_error
    double u = floor(__ddiv_rn(__dsub_rn(c[a], lo[a]), cw));
    if (u < 0) u = 0;
    if (u >= grid) u = grid - 1;
    ijk[a] = static_cast<uint32_t>(u);
  }
  keys[i] = static_cast<K>(morton(ijk[0], ijk[1], ijk[2]));
  idx[i] = static_cast<uint32_t>(i);
}

// Root cube and key geometry on the device, so the keys need no host round trip: the
// reduction of the min / max partials and bounding_cube's arithmetic (geometry.cpp:28-34)
// in explicit round-to-nearest operations, bit-identical to root_from_bounds on the host;
// the host reads the result back together with the leaf count.
struct TreeGeo {
  double root[4];
  double lo[3], hi[3];
  double cw;
  uint32_t runs, pad;
};
__global__ void k_root_geo(const double* __restrict__ part, int nb, int given, double r0, double r1, double r2,
                           double r3, uint32_t grid, TreeGeo* __restrict__ g) {
  __shared__ double red[6][32];
  const int a6 = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp a6 < 6 reduces one bound
  if (!given && a6 < 6) {
    double v = a6 < 3 ? INFINITY : -INFINITY;
    for (int b = lane; b < nb; b += 32) v = a6 < 3 ? fmin(v, part[a6 * nb + b]) : fmax(v, part[a6 * nb + b]);
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = a6 < 3 ? fmin(v, w) : fmax(v, w);
    }
    red[a6][lane] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double root[4];
  if (given) {
    root[0] = r0; root[1] = r1; root[2] = r2; root[3] = r3;
  } else {
    double extent = 0;
    for (int a = 0; a < 3; ++a) {
      const double lo = red[a][0], hi = red[3 + a][0];
      root[a] = __dmul_rn(0.5, __dadd_rn(lo, hi));
      extent = fmax(extent, __dsub_rn(hi, lo));
    }
    root[3] = extent > 0 ? __dmul_rn(extent, 1.0 + 1e-6) : 1.0;
  }
  for (int a = 0; a < 4; ++a) g->root[a] = root[a];
  for (int a = 0; a < 3; ++a) {
    g->lo[a] = __dsub_rn(root[a], __dmul_rn(0.5, root[3]));
    g->hi[a] = __dadd_rn(g->lo[a], root[3]);
  }
  g->cw = __ddiv_rn(root[3], static_cast<double>(grid));
}
template <typename K>
__global__ void k_keys_geo(const double4* __restrict__ p, uint64_t n, const TreeGeo* __restrict__ g, uint32_t grid,
                           K* __restrict__ keys, uint32_t* __restrict__ idx, int* __restrict__ flag) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double4 q = p[i];
  const double c[3] = {q.x, q.y, q.z};
  const double cw = g->cw;
  uint32_t ijk[3];
  for (int a = 0; a < 3; ++a) {
    const double lo = g->lo[a], hi = g->hi[a];
    if (c[a] < lo || c[a] > hi) atomicOr(flag, 1);  // domain_error
    double u = floor(__ddiv_rn(__dsub_rn(c[a], lo), cw));
    if (u < 0) u = 0;
    if (u >= grid) u = grid - 1;
    ijk[a] = static_cast<uint32_t>(u);
  }
  keys[i] = static_cast<K>(morton(ijk[0], ijk[1], ijk[2]));
  idx[i] = static_cast<uint32_t>(i);
}

__global__ void k_permute(const double4* __restrict__ in, const uint32_t* __restrict__ idx, uint64_t n,
                          double4* __restrict__ out, uint32_t* __restrict__ inv) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) {
    const uint32_t o = idx[i];
    out[i] = in[o];
    inv[o] = static_cast<uint32_t>(i);
  }
}

// distributed builds: input index per slot is the sorted iota, its inverse is all that
// the permute pass produced besides the positions (which arrive by the particle exchange)
__global__ void k_iota(uint32_t* __restrict__ idx, uint64_t n) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) idx[i] = static_cast<uint32_t>(i);
}
__global__ void k_inverse(const uint32_t* __restrict__ id, uint64_t n, uint32_t* __restrict__ inv) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) inv[id[i]] = static_cast<uint32_t>(i);
}

// leaf cell of every Morton slot, and the coincident-particle check
// (geometry.cpp:126-136: equal positions inside one leaf -> domain_error).
__global__ void k_leaf_scan(const uint32_t* __restrict__ first, const uint32_t* __restrict__ count, uint32_t ncells,
                            const double4* __restrict__ pw, uint32_t* __restrict__ pcell, int* __restrict__ flag,
                            uint32_t cell0, uint32_t* __restrict__ big, uint32_t big_cap) {
  __shared__ double xs[8][64];  // x of the leaf's particles (leaves of <= 64), per warp
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  if (warp >= ncells) return;
  const uint32_t f = first[warp], m = count[warp];
  const double* px = reinterpret_cast<const double*>(pw + f);
  if (pcell)
    for (uint32_t a = lane; a < m; a += 32) pcell[f + a] = cell0 + warp;
  if (m <= 64) {
    // x staged once; the pair loop reads it as a shared-memory broadcast (one wavefront
    // per source instead of a strided L1 read per pair), y and z only for equal x
    // (config B: 261 -> 166 us)
    const double nan = __longlong_as_double(0x7ff8000000000000ll);  // equal to nothing
    const double xa0 = lane < m ? px[4 * lane] : nan, xa1 = lane + 32 < m ? px[4 * (lane + 32)] : nan;
    xs[wl][lane] = xa0;
    xs[wl][lane + 32] = xa1;
    __syncwarp();
    for (uint32_t b = 1; b < m; ++b) {
      const double xb = xs[wl][b];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t a = lane + 32 * h;
        if (xb == (h ? xa1 : xa0) && a < b) {
          const double4 pa = pw[f + a], pb = pw[f + b];
          if (pa.y == pb.y && pa.z == pb.z) atomicOr(flag, 2);
        }
      }
    }
    return;
  }
  // a leaf of more than 64 particles: listed for k_leaf_scan_big (one CTA per leaf); the
  // list order does not matter (the check is an OR). Overflow -> the sorted fine-key pass.
  if (lane == 0) {
    const uint32_t k = atomicAdd(big, 1u);
    if (k < big_cap) big[1 + k] = warp;
    else atomicOr(flag, 4);
  }
}

// The listed leaves of 65..LS_BIG particles, one CTA (256 threads) per leaf: x staged in
// shared memory, thread a compares its particle with every later one (x by broadcast-ish
// reads, y and z only for equal x). At config B a uniform cloud has ~20 such leaves (a
// Poisson tail above 64 around a mean of 38), which used to send all 10M particles
// through the sorted fine-key check (1.1 ms); leaves above LS_BIG still take that path.
constexpr uint32_t LS_BIG = 4096;
__global__ void __launch_bounds__(256) k_leaf_scan_big(const uint32_t* __restrict__ first,
                                                       const uint32_t* __restrict__ count,
                                                       const uint32_t* __restrict__ big, uint32_t big_cap,
                                                       const double4* __restrict__ pw, int* __restrict__ flag) {
  __shared__ double xs[LS_BIG];
  const uint32_t nbig = min(big[0], big_cap);
  for (uint32_t e = blockIdx.x; e < nbig; e += gridDim.x) {
    const uint32_t c = big[1 + e], f = first[c], m = count[c];
    if (m > LS_BIG) {
      if (threadIdx.x == 0) atomicOr(flag, 4);
      continue;
    }
    __syncthreads();
    for (uint32_t a = threadIdx.x; a < m; a += blockDim.x) xs[a] = pw[f + a].x;
    __syncthreads();
    for (uint32_t a = threadIdx.x; a < m; a += blockDim.x) {
      const double xa = xs[a];
      for (uint32_t b = a + 1; b < m; ++b)
        if (xs[b] == xa) {
          const double4 pa = pw[f + a], pb = pw[f + b];
          if (pa.y == pb.y && pa.z == pb.z) atomicOr(flag, 2);
        }
    }
  }
}

// Large leaves (mean > 64 particles, e.g. config D's surface cloud, or any leaf above 64
// particles found by k_leaf_scan): the pairwise per-leaf scan is O(m^2). Instead every particle gets its Morton key at level 21
// (equal positions => equal keys), the keys are sorted, and runs of equal keys (tiny:
// distinct positions share a key only within 2^-21 of the root width) are compared
// pairwise on the exact positions. Same answer as geometry.cpp:126-136 (equal
// positions always share a leaf).
__global__ void k_leaf_cells(const uint32_t* __restrict__ first, const uint32_t* __restrict__ count, uint32_t ncells,
                             uint32_t* __restrict__ pcell) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= ncells) return;
  const uint32_t f = first[warp], m = count[warp];
  for (uint32_t a = lane; a < m; a += 32) pcell[f + a] = warp;
}
__global__ void k_fine_keys(const double4* __restrict__ pw, uint64_t n, double lo0, double lo1, double lo2, double cw,
                            uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double4 q = pw[i];
  const double c[3] = {q.x, q.y, q.z}, lo[3] = {lo0, lo1, lo2};
  uint32_t ijk[3];
  for (int a = 0; a < 3; ++a) {
    double u = floor(__ddiv_rn(__dsub_rn(c[a], lo[a]), cw));
    u = u < 0 ? 0 : (u > 2097151.0 ? 2097151.0 : u);
    ijk[a] = static_cast<uint32_t>(u);
  }
  keys[i] = morton(ijk[0], ijk[1], ijk[2]);
  idx[i] = static_cast<uint32_t>(i);
}
__global__ void k_equal_key_runs(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx, uint64_t n,
                                 const double4* __restrict__ pw, int* __restrict__ flag) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n || (i > 0 && keys[i] == keys[i - 1])) return;  // one thread per run of equal keys
  for (uint64_t a = i; a + 1 < n && keys[a + 1] == keys[i]; ++a) {
    const double4 pa = pw[idx[a]];
    for (uint64_t b = a + 1; b < n && keys[b] == keys[i]; ++b) {
      const double4 pb = pw[idx[b]];
      if (pa.x == pb.x && pa.y == pb.y && pa.z == pb.z) atomicOr(flag, 2);
    }
  }
}

// Parent levels without host round trips (geometry.cpp:138-153 semantics): level v's
// cells are the runs of leaf_code >> 3 (leaf - v) over the R sorted leaf codes; idx_v[i]
// (inclusive scan of the run-start flags) is the 1-based level-v cell of leaf i, so
// parent / first_child / child_count follow from the leaf ranges of the cells. Arrays
// are sized R (an upper bound); the cell counts come back in one readback at the end.
__global__ void k_level_flags(const uint64_t* __restrict__ lc, uint32_t R, int shift, uint32_t* __restrict__ flag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < R) flag[i] = (i == 0 || (lc[i] >> shift) != (lc[i - 1] >> shift)) ? 1u : 0u;
}
__global__ void k_level_cells(const uint64_t* __restrict__ lc, uint32_t R, int shift, const uint32_t* __restrict__ idx,
                              uint64_t* __restrict__ code, uint32_t* __restrict__ leafstart, uint32_t* __restrict__ n_out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R) return;
  if (i == 0 || idx[i] != idx[i - 1]) {
    code[idx[i] - 1] = lc[i] >> shift;
    leafstart[idx[i] - 1] = i;
  }
  if (i == R - 1) *n_out = idx[i];
}
// idx_c == nullptr: the children are the leaves themselves (idx = i + 1)
__global__ void k_level_children(const uint32_t* __restrict__ leafstart, const uint32_t* __restrict__ n_v, uint32_t R,
                                 const uint32_t* __restrict__ idx_c, uint32_t* __restrict__ first_child,
                                 uint32_t* __restrict__ child_count) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t n = *n_v;
  if (p >= n) return;
  const uint32_t ls = leafstart[p], le = (p + 1 < n ? leafstart[p + 1] : R) - 1;
  const uint32_t a = idx_c ? idx_c[ls] : ls + 1, b = idx_c ? idx_c[le] : le + 1;
  first_child[p] = a - 1;
  child_count[p] = b - a + 1;
}
// leafstart_c == nullptr: the child level is the leaf level (cell j = leaf j, R cells)
__global__ void k_level_parent(const uint32_t* __restrict__ leafstart_c, const uint32_t* __restrict__ n_c, uint32_t R,
                               const uint32_t* __restrict__ idx_v, uint32_t* __restrict__ parent_c) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= (n_c ? *n_c : R)) return;
  parent_c[j] = idx_v[leafstart_c ? leafstart_c[j] : j] - 1;
}

// Full trees (every leaf position occupied, e.g. uniform clouds: configs B, C, E): every
// level is full, cell i of a level has code i, children 8i..8i+7 and parent i / 8, and the
// parity class q of a level of n cells is the cells 8j + q. One launch fills all of it
// (the general path above takes ~80 small launches: level flags, scans, class sorts).
struct FullLevels {
  uint64_t* code[22];
  uint32_t* first_child[22];
  uint32_t* child_count[22];
  uint32_t* parent[22];
  uint32_t* cls_cells[22];
  uint32_t* first_particle[22];  // parent levels: zero (the reference keeps them 0)
  uint32_t* particle_count[22];
  uint64_t start[23];  // first flattened index of level v
  int leaf;
};
__global__ void k_full_levels(const FullLevels f) {
  const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (t >= f.start[f.leaf + 1]) return;
  int v = 0;
  while (t >= f.start[v + 1]) ++v;
  const uint64_t i = t - f.start[v], n = f.start[v + 1] - f.start[v];
  if (v < f.leaf) {  // the leaf level's code / first_child / child_count come from the build
    f.code[v][i] = i;
    f.first_child[v][i] = static_cast<uint32_t>(8 * i);
    f.child_count[v][i] = 8;
    f.first_particle[v][i] = 0;
    f.particle_count[v][i] = 0;
  }
  f.parent[v][i] = static_cast<uint32_t>(i >> 3);  // level 0: 0, as the general path
  if (v >= 2) f.cls_cells[v][(i & 7) * (n >> 3) + (i >> 3)] = static_cast<uint32_t>(i);
}

__global__ void k_fill_u32(uint32_t* p, uint64_t n, uint32_t v) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = v;
}
__global__ void k_scatter_map(const uint64_t* __restrict__ code, uint32_t n, uint32_t* __restrict__ map) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) map[code[i]] = i;
}
__global__ void k_octant(const uint64_t* __restrict__ code, uint32_t n, uint8_t* __restrict__ oct,
                         uint32_t* __restrict__ iota) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { oct[i] = static_cast<uint8_t>(code[i] & 7); iota[i] = i; }
}

__global__ void k_copy_words(const uint32_t* __restrict__ src, uint32_t nwords, uint32_t* __restrict__ dst) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
// lower_bound of q = 0..8 in the sorted octants (parity class offsets)
__global__ void k_class_offsets(const uint8_t* __restrict__ oct_sorted, uint32_t n, uint32_t* __restrict__ off) {
  const int q = threadIdx.x;
  if (q > 8) return;
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (oct_sorted[mid] < q) lo = mid + 1; else hi = mid;
  }
  off[q] = lo;
}

inline unsigned blocks(uint64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

void free_level(fmmgpu_ctx* c, fmmgpu::Level& L, cudaStream_t s) {
  dfree(c, L.code, s); dfree(c, L.first_particle, s); dfree(c, L.particle_count, s); dfree(c, L.parent, s);
  dfree(c, L.first_child, s); dfree(c, L.child_count, s); dfree(c, L.map, s); dfree(c, L.cls_cells, s);
  dfree(c, L.multipole, s); dfree(c, L.local_own, s); dfree(c, L.local_down, s); dfree(c, L.yt, s);
  dfree(c, L.far_target, s); dfree(c, L.far_source, s); dfree(c, L.far_vec, s); dfree(c, L.far_group_off, s);
  dfree(c, L.srcA, s); dfree(c, L.tgtB, s);
  L.far_pairs = 0;
}

}  // namespace

const void* readback(fmmgpu_ctx* c, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes > READBACK_CAP || bytes % 4) throw Error(FMMGPU_LOGIC_ERROR, "readback: bad size");
  if (!c->h_rb) FMM_CUDA(cudaHostAlloc(&c->h_rb, READBACK_CAP, cudaHostAllocMapped));
  uint32_t* d = nullptr;
  FMM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), c->h_rb, 0));
  const uint32_t nw = static_cast<uint32_t>(bytes / 4);
  k_copy_words<<<std::max(1u, std::min(64u, (nw + 255) / 256)), 256, 0, s>>>(static_cast<const uint32_t*>(src), nw, d);
  FMM_CUDA(cudaGetLastError());
  static const bool tr = std::getenv("FMMGPU_TRACE") != nullptr;
  static std::chrono::steady_clock::time_point last{};
  const auto t0 = std::chrono::steady_clock::now();
  FMM_CUDA(cudaStreamSynchronize(s));
  if (tr) {
    const auto t1 = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    const double host = std::chrono::duration<double, std::milli>(t0 - last).count();
    std::fprintf(stderr, "[readback] %zu B: sync %.3f ms, host work since the previous readback %.3f ms\n", bytes, ms,
                 host < 1e4 ? host : -1.0);
    last = t1;
  }
  return c->h_rb;
}

void yt_keep_free(fmmgpu_ctx* c) {
  for (auto& p : c->yt_keep) dfree(c, p, c->s_far);
}

void* cache_alloc(fmmgpu_ctx* c, size_t bytes, cudaStream_t s) {
  bytes = (bytes + 255) & ~size_t(255);
  auto& C = c->cache;
  auto it = C.idle.lower_bound(bytes);
  if (it != C.idle.end() && it->first <= bytes + bytes / 4 + (size_t(1) << 20)) {
    void* p = it->second.first;
    C.live[p] = it->first;
    C.idle.erase(it);
    return p;
  }
  void* p = nullptr;
  static const bool tr = std::getenv("FMMGPU_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  FMM_CUDA(cudaMallocAsync(&p, bytes, s));
  if (tr)
    std::fprintf(stderr, "[alloc] cache miss %zu bytes: %.3f ms\n", bytes,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  C.live[p] = bytes;
  return p;
}

void cache_free(fmmgpu_ctx* c, void* p, cudaStream_t s) {
  auto& C = c->cache;
  auto it = C.live.find(p);
  if (it == C.live.end()) {
    cudaFreeAsync(p, s);
    return;
  }
  C.idle.emplace(it->second, std::make_pair(p, C.epoch));
  C.live.erase(it);
}

void cache_trim(fmmgpu_ctx* c, cudaStream_t s) {
  for (auto& kv : c->cache.idle) cudaFreeAsync(kv.second.first, s);
  c->cache.idle.clear();
}

void cache_trim_old(fmmgpu_ctx* c, cudaStream_t s) {
  auto& C = c->cache;
  for (auto it = C.idle.begin(); it != C.idle.end();) {
    if (it->second.second < C.epoch) {
      cudaFreeAsync(it->second.first, s);
      it = C.idle.erase(it);
    } else {
      ++it;
    }
  }
}

void* scratch(fmmgpu_ctx* c, size_t bytes) {
  if (bytes > c->d_tmp_cap) {
    if (c->d_tmp) FMM_CUDA(cudaFreeAsync(c->d_tmp, c->s_far));
    c->d_tmp_cap = std::max(bytes, c->d_tmp_cap * 3 / 2);
    FMM_CUDA(cudaMallocAsync(&c->d_tmp, c->d_tmp_cap, c->s_far));
  }
  return c->d_tmp;
}

void tree_free(fmmgpu_ctx* c) {
  cudaStream_t s = c->s_far;
  for (size_t v = 0; v < c->lv.size(); ++v) {
    auto& L = c->lv[v];
    if (L.yt && L.full && v < 22) {
      dfree(c, c->yt_keep[v], s);
      c->yt_keep[v] = L.yt;
      c->yt_keep_n[v] = L.n;
      L.yt = nullptr;
    }
  }
  for (auto& L : c->lv) free_level(c, L, s);
  c->lv.clear();
  dfree(c, c->d_pw, s); dfree(c, c->d_id, s); dfree(c, c->d_inv, s); dfree(c, c->d_pcell, s);
  dfree(c, c->d_near, s); dfree(c, c->d_far, s); dfree(c, c->d_out, s);
  dfree(c, c->d_slot, s);
  dfree(c, c->d_p2p_order, s);
  dist_free(c);
  c->have_tree = false;
}

// bounding_cube (geometry.cpp:28-34) from per-axis bounds, host arithmetic without
// contraction; shared by the single-device build and the distributed one
void root_from_bounds(const double lo[3], const double hi[3], double root[4]) {
  double extent = 0;
  for (int a = 0; a < 3; ++a) {
    root[a] = 0.5 * (lo[a] + hi[a]);
    extent = std::max(extent, hi[a] - lo[a]);
  }
  root[3] = extent > 0 ? extent * (1.0 + 1e-6) : 1.0;
}

// per-axis min / max of n device particles -> lohi = {lo[3], hi[3]} (+-inf when n = 0)
void device_bounds(fmmgpu_ctx* c, const double4* d, uint64_t n, double lohi[6], cudaStream_t s) {
  for (int a = 0; a < 3; ++a) {
    lohi[a] = INFINITY;
    lohi[3 + a] = -INFINITY;
  }
  if (n == 0) return;
  const int nb = static_cast<int>(std::min<uint64_t>(1184, blocks(n, 256)));
  double* part = static_cast<double*>(scratch(c, sizeof(double) * 6 * nb));
  k_minmax_partial<<<nb, 256, 0, s>>>(d, n, part);
  FMM_CUDA(cudaGetLastError());
  std::vector<double> h(6 * nb);
  std::memcpy(h.data(), readback(c, part, sizeof(double) * 6 * nb, s), sizeof(double) * 6 * nb);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < nb; ++b) {
      lohi[a] = std::min(lohi[a], h[a * nb + b]);
      lohi[3 + a] = std::max(lohi[3 + a], h[(3 + a) * nb + b]);
    }
}

// Morton leaf keys of n device particles against root (geometry.cpp:76-94), as u64, and
// the outside-the-root flag (bit 1 of *flag, device) -- the per-rank step of a
// distributed build
void device_keys(const double4* d, uint64_t n, const double root[4], int height, uint64_t* keys, uint32_t* idx,
                 int* flag, cudaStream_t s) {
  if (n == 0) return;
  const int leaf = height - 1;
  const uint32_t grid = 1u << leaf;
  const double cw = root[3] / static_cast<double>(grid);
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = root[a] - 0.5 * root[3];
    hi[a] = lo[a] + root[3];
  }
  k_keys<<<blocks(n, 256), 256, 0, s>>>(d, n, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], cw, grid, keys, idx, flag);
  FMM_CUDA(cudaGetLastError());
}

// Distributed builds (dist != nullptr, csrc/dist.cu): the keys of all n particles were
// computed by the ranks from their input slices and all-gathered (device, input order);
// the positions are NOT here: d_pw stays zero until the particle exchange places this
// rank's owned and halo leaves, and the coincident-particle check runs after it on the
// owned leaves. Everything else (sort, levels, classes, expansions) is the same code, so
// the tree is bit-identical to the single-device build of the whole set.
void tree_build(fmmgpu_ctx* c, const double* xyzw, uint64_t n, bool on_device, int height, int group,
                const double* root4, const DistKeys* dist) {
  // argument validation, geometry.cpp:65-69 and bounding_cube's empty check
  if (height < 3 || height > 21) throw Error(FMMGPU_INVALID_ARGUMENT, "GroupTree: height must be in [3, 21]");
  if (group < 1) throw Error(FMMGPU_INVALID_ARGUMENT, "GroupTree: group size must be positive");
  if (n == 0) throw Error(FMMGPU_INVALID_ARGUMENT, "GroupTree: empty particle set");
  if (n >= 0xffffffffull) throw Error(FMMGPU_INVALID_ARGUMENT, "GroupTree: particle count exceeds 32-bit ids");
  if (root4 && !(root4[3] > 0)) throw Error(FMMGPU_INVALID_ARGUMENT, "GroupTree: root cube width must be positive");
  cudaStream_t s = c->s_far;
  PhaseTrace trace;
  fmmgpu_invalidate_graph(c);
  partition_free(c);
  tree_free(c);
  ++c->cache.epoch;
  lists_free(c);  // after the epoch bump: the next lists build reuses these blocks
  trace("free");

  // input -> device (input order); a pipelined run (fmmgpu_run_async) has already
  // copied it into d_in on its H2D stream
  if (dist && !root4) throw Error(FMMGPU_LOGIC_ERROR, "distributed build without a root cube");
  const bool in_place = dist || (on_device && xyzw == reinterpret_cast<const double*>(c->d_in) && c->d_in_cap >= n);
  if (!in_place && c->d_in_cap < n) {
    if (c->d_in) FMM_CUDA(cudaFreeAsync(c->d_in, s));
    FMM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c->d_in), n * sizeof(double4), s));
    c->d_in_cap = n;
  }
  if (!in_place)
    FMM_CUDA(cudaMemcpyAsync(c->d_in, xyzw, n * sizeof(double4), on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  FMM_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));

  // root cube and key geometry, on the device (read back with the leaf count below)
  c->n = n;
  c->height = height;
  c->group = group;
  const int leaf = height - 1;
  const uint32_t grid = 1u << leaf;
  double* geo_mem = dalloc<double>(c, sizeof(TreeGeo) / sizeof(double), s);
  FMM_CUDA(cudaMemsetAsync(geo_mem, 0, sizeof(TreeGeo), s));
  TreeGeo* geo = reinterpret_cast<TreeGeo*>(geo_mem);
  {
    const int nb = root4 ? 1 : static_cast<int>(std::min<uint64_t>(1184, blocks(n, 256)));
    double* part = static_cast<double*>(scratch(c, sizeof(double) * 6 * nb));
    if (!root4) {
      k_minmax_partial<<<nb, 256, 0, s>>>(c->d_in, n, part);
      FMM_CUDA(cudaGetLastError());
    }
    k_root_geo<<<1, 256, 0, s>>>(part, nb, root4 ? 1 : 0, root4 ? root4[0] : 0, root4 ? root4[1] : 0,
                                 root4 ? root4[2] : 0, root4 ? root4[3] : 0, grid, geo);
    FMM_CUDA(cudaGetLastError());
  }
  trace("root cube");

  // keys + stable radix sort of (key, input index); leaf cells = runs of equal keys
  // (geometry.cpp:113-122)
  c->d_id = dalloc<uint32_t>(c, n, s);
  uint32_t* idx = dalloc<uint32_t>(c, n, s);
  c->lv.resize(height);
  Level& L = c->lv[leaf];
  uint32_t* d_runs = &geo->runs;
  L.code = dalloc<uint64_t>(c, n, s);
  L.particle_count = dalloc<uint32_t>(c, n, s);
  size_t tb = 0;
  auto sort_and_encode = [&](auto* keys, auto* keys_sorted) {
    if (dist) {
      k_iota<<<blocks(n, 256), 256, 0, s>>>(idx, n);
    } else {
      k_keys_geo<<<blocks(n, 256), 256, 0, s>>>(c->d_in, n, geo, grid, keys, idx, c->d_flag);
    }
    FMM_CUDA(cudaGetLastError());
    trace("keys");
    FMM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys_sorted, idx, c->d_id, static_cast<int>(n), 0,
                                             std::max(1, 3 * leaf), s));
    FMM_CUDA(cub::DeviceRadixSort::SortPairs(scratch(c, tb), tb, keys, keys_sorted, idx, c->d_id, static_cast<int>(n),
                                             0, std::max(1, 3 * leaf), s));
    trace("sort");
    c->d_pw = dalloc<double4>(c, n, s);
    c->d_inv = dalloc<uint32_t>(c, n, s);
    if (dist) {
      k_inverse<<<blocks(n, 256), 256, 0, s>>>(c->d_id, n, c->d_inv);
      FMM_CUDA(cudaMemsetAsync(c->d_pw, 0, n * sizeof(double4), s));
    } else {
      k_permute<<<blocks(n, 256), 256, 0, s>>>(c->d_in, c->d_id, n, c->d_pw, c->d_inv);
    }
    FMM_CUDA(cudaGetLastError());
    trace("keys+sort+permute");
    FMM_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb, keys_sorted, L.code, L.particle_count, d_runs,
                                                static_cast<int>(n), s));
    FMM_CUDA(cub::DeviceRunLengthEncode::Encode(scratch(c, tb), tb, keys_sorted, L.code, L.particle_count, d_runs,
                                                static_cast<int>(n), s));
  };
  if (dist) {  // the all-gathered u64 keys are sorted in place of computed ones
    uint64_t* k64s = dalloc<uint64_t>(c, n, s);
    sort_and_encode(const_cast<uint64_t*>(dist->keys), k64s);
    dfree(c, k64s, s);
  } else if (3 * leaf <= 32) {
    uint32_t* k32 = dalloc<uint32_t>(c, n, s);
    uint32_t* k32s = dalloc<uint32_t>(c, n, s);
    sort_and_encode(k32, k32s);
    dfree(c, k32, s);
    dfree(c, k32s, s);
  } else {
    uint64_t* k64 = dalloc<uint64_t>(c, n, s);
    uint64_t* k64s = dalloc<uint64_t>(c, n, s);
    sort_and_encode(k64, k64s);
    dfree(c, k64, s);
    dfree(c, k64s, s);
  }
  uint32_t runs = 0;
  {  // the one readback before the level arrays: leaf count, root cube, key geometry
    TreeGeo hg;
    std::memcpy(&hg, readback(c, geo, sizeof(TreeGeo), s), sizeof(TreeGeo));
    runs = hg.runs;
    std::copy(hg.root, hg.root + 4, c->root);
    std::copy(hg.lo, hg.lo + 3, c->lo);
  }
  L.n = runs;
  L.first_particle = dalloc<uint32_t>(c, runs, s);
  FMM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, L.particle_count, L.first_particle, static_cast<int>(runs), s));
  FMM_CUDA(cub::DeviceScan::ExclusiveSum(scratch(c, tb), tb, L.particle_count, L.first_particle, static_cast<int>(runs), s));
  L.first_child = dalloc<uint32_t>(c, runs, s);
  L.child_count = dalloc<uint32_t>(c, runs, s);
  L.parent = dalloc<uint32_t>(c, runs, s);
  FMM_CUDA(cudaMemsetAsync(L.first_child, 0, 4ull * runs, s));
  FMM_CUDA(cudaMemsetAsync(L.child_count, 0, 4ull * runs, s));
  FMM_CUDA(cudaMemsetAsync(L.parent, 0, 4ull * runs, s));
  c->d_pcell = dalloc<uint32_t>(c, n, s);
  // exact duplicates via level-21 keys: sort, then compare runs of equal keys
  auto fine_key_check = [&] {
    uint64_t* fk = dalloc<uint64_t>(c, n, s);
    uint64_t* fks = dalloc<uint64_t>(c, n, s);
    uint32_t* fi = dalloc<uint32_t>(c, n, s);
    uint32_t* fis = dalloc<uint32_t>(c, n, s);
    k_fine_keys<<<blocks(n, 256), 256, 0, s>>>(c->d_pw, n, c->lo[0], c->lo[1], c->lo[2], c->root[3] / 2097152.0, fk,
                                                fi);
    FMM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, fk, fks, fi, fis, static_cast<int>(n), 0, 63, s));
    FMM_CUDA(cub::DeviceRadixSort::SortPairs(scratch(c, tb), tb, fk, fks, fi, fis, static_cast<int>(n), 0, 63, s));
    k_equal_key_runs<<<blocks(n, 256), 256, 0, s>>>(fks, fis, n, c->d_pw, c->d_flag);
    FMM_CUDA(cudaGetLastError());
    dfree(c, fk, s);
    dfree(c, fks, s);
    dfree(c, fi, s);
    dfree(c, fis, s);
  };
  if (dist) {  // positions arrive later: the coincident check runs in fmmgpu_dist_check
    k_leaf_cells<<<blocks(uint64_t(runs) * 32, 256), 256, 0, s>>>(L.first_particle, L.particle_count, runs,
                                                                  c->d_pcell);
  } else if (n <= 64ull * runs) {
    // small leaves on average; a leaf above 64 raises flag bit 4 and the sorted check
    // runs after the readback below (clustered inputs)
    uint32_t* big = dalloc<uint32_t>(c, 1 + 65536, s);
    FMM_CUDA(cudaMemsetAsync(big, 0, 4, s));
    k_leaf_scan<<<blocks(uint64_t(runs) * 32, 256), 256, 0, s>>>(L.first_particle, L.particle_count, runs, c->d_pw,
                                                                 c->d_pcell, c->d_flag, 0, big, 65536);
    FMM_CUDA(cudaGetLastError());
    k_leaf_scan_big<<<296, 256, 0, s>>>(L.first_particle, L.particle_count, big, 65536, c->d_pw, c->d_flag);
    dfree(c, big, s);
    FMM_CUDA(cudaGetLastError());
  } else {
    k_leaf_cells<<<blocks(uint64_t(runs) * 32, 256), 256, 0, s>>>(L.first_particle, L.particle_count, runs,
                                                                  c->d_pcell);
    fine_key_check();
  }

  trace("leaf level");
  const bool full_tree = leaf <= 10 && uint64_t(runs) == (uint64_t{1} << (3 * leaf));
  if (full_tree) {  // every level full: one launch (k_full_levels) instead of the general path
    FullLevels f{};
    f.leaf = leaf;
    f.start[0] = 0;
    for (int v = 0; v <= leaf; ++v) {
      const uint64_t nv = uint64_t{1} << (3 * v);
      f.start[v + 1] = f.start[v] + nv;
      Level& V = c->lv[v];
      V.n = static_cast<uint32_t>(nv);
      if (v < leaf) {
        V.code = dalloc<uint64_t>(c, nv, s);
        V.first_child = dalloc<uint32_t>(c, nv, s);
        V.child_count = dalloc<uint32_t>(c, nv, s);
        V.parent = dalloc<uint32_t>(c, nv, s);
        V.first_particle = dalloc<uint32_t>(c, nv, s);
        V.particle_count = dalloc<uint32_t>(c, nv, s);
      }
      if (v >= 2) {
        V.cls_cells = dalloc<uint32_t>(c, nv, s);
        for (int q = 0; q <= 8; ++q) V.cls_off[q] = static_cast<uint32_t>(q * (nv >> 3));
      }
      f.code[v] = V.code;
      f.first_child[v] = V.first_child;
      f.child_count[v] = V.child_count;
      f.parent[v] = V.parent;
      f.cls_cells[v] = V.cls_cells;
      f.first_particle[v] = v < leaf ? V.first_particle : nullptr;
      f.particle_count[v] = v < leaf ? V.particle_count : nullptr;
    }
    k_full_levels<<<blocks(f.start[leaf + 1], 256), 256, 0, s>>>(f);
    FMM_CUDA(cudaGetLastError());
    dfree(c, idx, s);
    dfree(c, geo_mem, s);
  } else {
  // parent levels (geometry.cpp:138-153), on the device only
  const uint32_t R = runs;
  uint32_t* d_counts = dalloc<uint32_t>(c, 22, s);
  uint32_t* runflag = dalloc<uint32_t>(c, R, s);
  uint32_t* idx_c = nullptr;        // level v + 1 (nullptr: the leaf level)
  uint32_t* leafstart_c = nullptr;
  for (int v = leaf - 1; v >= 0; --v) {
    Level& C = c->lv[v + 1];
    Level& P = c->lv[v];
    const int shift = 3 * (leaf - v);
    uint32_t* idx_v = dalloc<uint32_t>(c, R, s);
    uint32_t* leafstart_v = dalloc<uint32_t>(c, R, s);
    k_level_flags<<<blocks(R, 256), 256, 0, s>>>(L.code, R, shift, runflag);
    FMM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, runflag, idx_v, static_cast<int>(R), s));
    FMM_CUDA(cub::DeviceScan::InclusiveSum(scratch(c, tb), tb, runflag, idx_v, static_cast<int>(R), s));
    P.code = dalloc<uint64_t>(c, R, s);
    k_level_cells<<<blocks(R, 256), 256, 0, s>>>(L.code, R, shift, idx_v, P.code, leafstart_v, d_counts + v);
    P.first_child = dalloc<uint32_t>(c, R, s);
    P.child_count = dalloc<uint32_t>(c, R, s);
    k_level_children<<<blocks(R, 256), 256, 0, s>>>(leafstart_v, d_counts + v, R, idx_c, P.first_child,
                                                    P.child_count);
    k_level_parent<<<blocks(R, 256), 256, 0, s>>>(leafstart_c, idx_c ? d_counts + v + 1 : nullptr, R, idx_v,
                                                  C.parent);
    P.first_particle = dalloc<uint32_t>(c, R, s);
    P.particle_count = dalloc<uint32_t>(c, R, s);
    P.parent = dalloc<uint32_t>(c, R, s);
    FMM_CUDA(cudaMemsetAsync(P.first_particle, 0, 4ull * R, s));
    FMM_CUDA(cudaMemsetAsync(P.particle_count, 0, 4ull * R, s));
    FMM_CUDA(cudaMemsetAsync(P.parent, 0, 4ull * R, s));
    FMM_CUDA(cudaGetLastError());
    if (idx_c) dfree(c, idx_c, s);
    if (leafstart_c) dfree(c, leafstart_c, s);
    idx_c = idx_v;
    leafstart_c = leafstart_v;
  }
  if (idx_c) dfree(c, idx_c, s);
  if (leafstart_c) dfree(c, leafstart_c, s);
  dfree(c, runflag, s);
  if (leaf > 0) {
    const uint32_t* hc = static_cast<const uint32_t*>(readback(c, d_counts, leaf * sizeof(uint32_t), s));
    for (int v = 0; v < leaf; ++v) c->lv[v].n = hc[v];
  }
  dfree(c, d_counts, s);
  dfree(c, idx, s);
  dfree(c, geo_mem, s);
  }  // general (not full) tree

  trace("parent levels");
  // blocks of group_size cells (geometry.cpp:155-160); lookup maps; parity classes;
  // expansions (cell-major, stride ldE, zero padding). The class offsets of every level
  // and the error flag come back in one readback at the end.
  uint32_t* d_offs = dalloc<uint32_t>(c, 9 * height + 1, s);
  FMM_CUDA(cudaMemsetAsync(d_offs, 0, sizeof(uint32_t) * (9 * height + 1), s));  // levels 0, 1 stay 0
  for (int v = 0; v < height; ++v) {
    Level& V = c->lv[v];
    V.block_offsets.clear();
    for (uint64_t b = 0; b < V.n; b += static_cast<uint64_t>(group)) V.block_offsets.push_back(static_cast<uint32_t>(b));
    V.block_offsets.push_back(V.n);
    V.full = static_cast<uint64_t>(V.n) == (uint64_t{1} << (3 * v));
    if (!V.full && v <= DENSE_MAP_MAX_LEVEL) {
      const uint64_t cap = uint64_t{1} << (3 * v);
      V.map = dalloc<uint32_t>(c, cap, s);
      k_fill_u32<<<blocks(cap, 256), 256, 0, s>>>(V.map, cap, NPOS);
      k_scatter_map<<<blocks(V.n, 256), 256, 0, s>>>(V.code, V.n, V.map);
    }
    if (v >= 2 && !full_tree) {
      uint8_t* oct = dalloc<uint8_t>(c, V.n, s);
      uint8_t* oct_sorted = dalloc<uint8_t>(c, V.n, s);
      uint32_t* iota = dalloc<uint32_t>(c, V.n, s);
      V.cls_cells = dalloc<uint32_t>(c, V.n, s);
      k_octant<<<blocks(V.n, 256), 256, 0, s>>>(V.code, V.n, oct, iota);
      FMM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, oct, oct_sorted, iota, V.cls_cells, static_cast<int>(V.n), 0, 3, s));
      FMM_CUDA(cub::DeviceRadixSort::SortPairs(scratch(c, tb), tb, oct, oct_sorted, iota, V.cls_cells, static_cast<int>(V.n), 0, 3, s));
      k_class_offsets<<<1, 32, 0, s>>>(oct_sorted, V.n, d_offs + 9 * v);
      dfree(c, oct, s);
      dfree(c, oct_sorted, s);
      dfree(c, iota, s);
    }
    V.own0 = 0;  // unpartitioned: every cell is owned
    V.own1 = V.n;
    const size_t e = size_t(V.n) * c->ldE;
    V.multipole = dalloc<double>(c, e, s);
    V.local_own = dalloc<double>(c, e, s);
    V.local_down = dalloc<double>(c, e, s);
  }
  trace("blocks+classes+expansions");
  c->part_rank = 0;
  c->part_n = 1;
  c->part_align = 0;
  c->own_s0 = 0;
  c->own_s1 = n;
  c->d_near = dalloc<double>(c, 4 * n, s);
  c->d_far = dalloc<double>(c, 4 * n, s);
  c->d_out = dalloc<double>(c, 4 * n, s);
  // cleared by the first entry point that uses them (an evaluation clears them anyway)
  c->zero_pending = true;

  k_copy_words<<<1, 32, 0, s>>>(reinterpret_cast<const uint32_t*>(c->d_flag), 1, d_offs + 9 * height);
  const uint32_t* h_offs = static_cast<const uint32_t*>(readback(c, d_offs, (9 * height + 1) * sizeof(uint32_t), s));
  if (!full_tree)
    for (int v = 2; v < height; ++v) std::memcpy(c->lv[v].cls_off, h_offs + 9 * v, 9 * sizeof(uint32_t));
  int flag = static_cast<int>(h_offs[9 * height]);
  if (dist) flag = dist->flag & 1;  // every rank's key step, OR-ed by the caller
  if ((flag & 4) && !(flag & 3)) {  // a leaf above 64 particles: the sorted fine-key check
    fine_key_check();
    flag = *static_cast<const int*>(readback(c, c->d_flag, sizeof(int), s));
  }
  dfree(c, d_offs, s);
  trace("fields+flag sync");
  if (flag & 1) {
    tree_free(c);
    throw Error(FMMGPU_DOMAIN_ERROR, "GroupTree: particle outside the root cube");
  }
  if (flag & 2) {
    tree_free(c);
    throw Error(FMMGPU_DOMAIN_ERROR, "GroupTree: coincident particles");
  }
  c->have_tree = true;
  c->dist = dist != nullptr;
  c->dist_ready = !c->dist;
  ensure_p2p_slots(c);
  cache_trim_old(c, s);  // blocks of the previous tree this one did not reuse
}


// Coincident-particle check (geometry.cpp:126-136) of the leaves [c0, c1) of the current
// tree, positions in d_pw: the distributed build runs it on each rank's owned leaves
// after the particle exchange. Returns the flag bits (2 = coincident particles).
int coincident_check(fmmgpu_ctx* c, uint32_t c0, uint32_t c1, cudaStream_t s) {
  const Level& L = c->lv[c->height - 1];
  if (c1 <= c0) return 0;
  const uint32_t runs = c1 - c0;
  const uint32_t f0 = *static_cast<const uint32_t*>(readback(c, L.first_particle + c0, 4, s));
  const uint64_t s0 = f0, s1 = c1 < L.n ? *static_cast<const uint32_t*>(readback(c, L.first_particle + c1, 4, s))
                                        : c->n;
  const uint64_t m = s1 - s0;
  FMM_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
  bool fine = m > 64ull * runs;
  if (!fine) {
    uint32_t* big = dalloc<uint32_t>(c, 1 + 65536, s);
    FMM_CUDA(cudaMemsetAsync(big, 0, 4, s));
    k_leaf_scan<<<blocks(uint64_t(runs) * 32, 256), 256, 0, s>>>(L.first_particle + c0, L.particle_count + c0, runs,
                                                                 c->d_pw, nullptr, c->d_flag, 0, big, 65536);
    FMM_CUDA(cudaGetLastError());
    k_leaf_scan_big<<<296, 256, 0, s>>>(L.first_particle + c0, L.particle_count + c0, big, 65536, c->d_pw,
                                        c->d_flag);
    dfree(c, big, s);
    FMM_CUDA(cudaGetLastError());
    const int f = *static_cast<const int*>(readback(c, c->d_flag, sizeof(int), s));
    if (f & 2) return f;
    fine = (f & 4) != 0;
  }
  if (!fine) return 0;
  size_t tb = 0;
  uint64_t* fk = dalloc<uint64_t>(c, m, s);
  uint64_t* fks = dalloc<uint64_t>(c, m, s);
  uint32_t* fi = dalloc<uint32_t>(c, m, s);
  uint32_t* fis = dalloc<uint32_t>(c, m, s);
  const double4* pw = c->d_pw + s0;
  k_fine_keys<<<blocks(m, 256), 256, 0, s>>>(pw, m, c->lo[0], c->lo[1], c->lo[2], c->root[3] / 2097152.0, fk, fi);
  FMM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, fk, fks, fi, fis, static_cast<int>(m), 0, 63, s));
  FMM_CUDA(cub::DeviceRadixSort::SortPairs(scratch(c, tb), tb, fk, fks, fi, fis, static_cast<int>(m), 0, 63, s));
  FMM_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
  k_equal_key_runs<<<blocks(m, 256), 256, 0, s>>>(fks, fis, m, pw, c->d_flag);
  FMM_CUDA(cudaGetLastError());
  dfree(c, fk, s);
  dfree(c, fks, s);
  dfree(c, fi, s);
  dfree(c, fis, s);
  return *static_cast<const int*>(readback(c, c->d_flag, sizeof(int), s)) & 2;
}

}  // namespace fmmgpu
