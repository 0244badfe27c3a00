// Interaction lists on the device, bit-exact with the reference plan:
//   near CSR   = build_near_field_plan (direct.cpp:22-61) over near_field_list
//                (geometry.cpp:222-242): per leaf cell, existing cells at Chebyshev
//                distance 1, ascending index;
//   far pairs  = build_interaction_plan (taskflow.cpp:67-105) over far_field_list
//                (geometry.cpp:244-280): per level, grouped by (block*16+canonical),
//                within a group target ascending then source ascending.
// Both are count -> exclusive scan -> fill passes; the fill writes each cell's
// entries straight into their final CSR slot (no sort of the pair array).
#include <cub/cub.cuh>

#include "common.cuh"

namespace fmmgpu {

namespace {

inline unsigned blocks(uint64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

// list arrays come from the context's stream-ordered block cache, so rebuilds reuse the
// previous lists' blocks (config E's far lists are 4.4 GB: a fresh cudaMallocAsync of them
// cost tens of ms)
template <typename T>
T* dalloc(fmmgpu_ctx* c, size_t count, cudaStream_t s) {
  return static_cast<T*>(cache_alloc(c, (count ? count : 1) * sizeof(T), s));
}
void dfree(fmmgpu_ctx* c, void* p, cudaStream_t s) {
  if (p) cache_free(c, p, s);
}

// ---- near field -----------------------------------------------------------------
__device__ int near_cells_of(const LevelView& L, uint64_t code, uint32_t out[26]) {
  int ijk[3];
  demorton(code, ijk);
  int m = 0;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj)
      for (int dk = -1; dk <= 1; ++dk) {
        if (!di && !dj && !dk) continue;
        const uint32_t f = find_ijk(L, ijk[0] + di, ijk[1] + dj, ijk[2] + dk);
        if (f != NPOS) out[m++] = f;
      }
  // ascending (direct.cpp:22-34 via std::sort in near_field_list)
  for (int a = 1; a < m; ++a) {
    const uint32_t x = out[a];
    int b = a - 1;
    while (b >= 0 && out[b] > x) { out[b + 1] = out[b]; --b; }
    out[b + 1] = x;
  }
  return m;
}

__global__ void k_near_count(LevelView L, const uint32_t* __restrict__ pcount, uint32_t* __restrict__ cnt,
                             unsigned long long* __restrict__ work) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L.n) return;
  uint32_t nb[26];
  const int m = near_cells_of(L, L.code[c], nb);
  cnt[c] = static_cast<uint32_t>(m);
  // count_interactions near term (taskflow.cpp:116-122): nc(nc-1) + sum nc*n_nbr
  const unsigned long long nc = pcount[c];
  unsigned long long w = nc * (nc - 1);
  for (int a = 0; a < m; ++a) w += nc * pcount[nb[a]];
  work[c] = w;
}

__global__ void k_near_fill(LevelView L, const uint32_t* __restrict__ off, uint32_t* __restrict__ cells) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L.n) return;
  uint32_t nb[26];
  const int m = near_cells_of(L, L.code[c], nb);
  for (int a = 0; a < m; ++a) cells[off[c] + a] = nb[a];
}

// ---- far field ------------------------------------------------------------------
// Sorted parent-neighbour indices; their children are disjoint ascending index
// ranges, so visiting them in this order yields sources in ascending order
// (the std::sort by source of geometry.cpp:277-278).
__device__ int parent_neighbours(const LevelView& P, uint64_t pcode, uint32_t out[27]) {
  int ijk[3];
  demorton(pcode, ijk);
  int m = 0;
  for (int di = -1; di <= 1; ++di)
    for (int dj = -1; dj <= 1; ++dj)
      for (int dk = -1; dk <= 1; ++dk) {
        const uint32_t f = find_ijk(P, ijk[0] + di, ijk[1] + dj, ijk[2] + dk);
        if (f != NPOS) out[m++] = f;
      }
  for (int a = 1; a < m; ++a) {
    const uint32_t x = out[a];
    int b = a - 1;
    while (b >= 0 && out[b] > x) { out[b + 1] = out[b]; --b; }
    out[b + 1] = x;
  }
  return m;
}

struct FarArgs {
  LevelView L, P;
  const uint32_t* parent;
  const uint32_t* p_first_child;
  const uint32_t* p_child_count;
  const int* canon;  // 343
  uint32_t group;
};

// counts per (block, class, cell) of the far pairs (the fill is k_far_fill_warp)
__global__ void k_far_count(FarArgs a, uint32_t* __restrict__ cnt) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.L.n) return;
  const uint64_t code = a.L.code[c];
  int ijk[3];
  demorton(code, ijk);
  uint32_t pn[27];
  const int m = parent_neighbours(a.P, code >> 3, pn);
  const uint32_t b = c / a.group, cl = c % a.group;
  uint32_t k16[16];
  for (int q = 0; q < 16; ++q) k16[q] = 0;
  for (int t = 0; t < m; ++t) {
    const uint32_t np = pn[t];
    const uint32_t f = a.p_first_child[np], e = f + a.p_child_count[np];
    for (uint32_t ch = f; ch < e; ++ch) {
      int cijk[3];
      demorton(a.L.code[ch], cijk);
      const int ti = cijk[0] - ijk[0], tj = cijk[1] - ijk[1], tk = cijk[2] - ijk[2];
      const int d = max(abs(ti), max(abs(tj), abs(tk)));
      if (d <= 1) continue;
      const int slot = (ti + 3) * 49 + (tj + 3) * 7 + (tk + 3);
      ++k16[a.canon[slot]];
    }
  }
  for (int q = 0; q < 16; ++q) cnt[(size_t(b) * 16 + q) * a.group + cl] = k16[q];
}

// The fill as one warp per target cell: the candidate sources (children of the sorted
// parent neighbours, ascending) are spread over the lanes in order; each 32-candidate step
// groups the lanes by canonical class (__match_any_sync), so a class's entries of the step
// are written to consecutive slots (a few segments per store instead of 32 scattered
// ones). Positions: within a (block, class) group the cells in order,
// within a cell the sources ascending.
__global__ void __launch_bounds__(256) k_far_fill_warp(FarArgs a, const unsigned long long* __restrict__ pos,
                                                       uint32_t* __restrict__ tgt, uint32_t* __restrict__ src,
                                                       uint16_t* __restrict__ vec) {
  __shared__ uint32_t s_first[8][28], s_off[8][28];
  __shared__ uint32_t s_cnt[8][16];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= a.L.n) return;
  const uint64_t code = a.L.code[c];
  int ijk[3];
  demorton(code, ijk);
  // parent neighbours, ascending (every lane forms the same list), children per neighbour
  uint32_t pn[27];
  const int m = parent_neighbours(a.P, code >> 3, pn);
  uint32_t cntn = 0, firstn = 0;
  if (lane < m) {
    firstn = a.p_first_child[pn[lane]];
    cntn = a.p_child_count[pn[lane]];
  }
  uint32_t incl = cntn;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  if (lane < m) {
    s_first[wl][lane] = firstn;
    s_off[wl][lane] = incl - cntn;
  }
  if (lane < 16) s_cnt[wl][lane] = 0;
  __syncwarp();
  const uint32_t b = c / a.group, cl = c % a.group;
  for (uint32_t base = 0; base < total; base += 32) {
    const uint32_t e = base + lane;
    int q = -1, slot = 0;
    uint32_t ch = 0;
    if (e < total) {
      int t = 0;
      while (t + 1 < m && s_off[wl][t + 1] <= e) ++t;
      ch = s_first[wl][t] + (e - s_off[wl][t]);
      int cijk[3];
      demorton(a.L.code[ch], cijk);
      const int ti = cijk[0] - ijk[0], tj = cijk[1] - ijk[1], tk = cijk[2] - ijk[2];
      if (max(abs(ti), max(abs(tj), abs(tk))) > 1) {
        slot = (ti + 3) * 49 + (tj + 3) * 7 + (tk + 3);
        q = a.canon[slot];
      }
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, q);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    if (q >= 0) {
      const unsigned long long p = pos[(size_t(b) * 16 + q) * a.group + cl] + s_cnt[wl][q] + rank;
      tgt[p] = c;
      src[p] = ch;
      vec[p] = static_cast<uint16_t>(slot);
    }
    __syncwarp();
    if (q >= 0 && rank == 0) s_cnt[wl][q] += __popc(peers);
    __syncwarp();
  }
}

// NearFieldPlan block arrays (build_near_field_plan, direct.cpp:36-58): per leaf cell c of
// block b, its near cells o owned by b's side (ob > b, or ob == b and o > c) add
// 2 n_c n_o directional interactions to b's task, and every ob != b is a partner above b;
// n_c (n_c - 1) for the cell itself. Integer atomics: the sums are order-free.
__global__ void k_near_blocks(LevelView L, const uint32_t* __restrict__ count, const uint32_t* __restrict__ off,
                              const uint32_t* __restrict__ cells, uint32_t group,
                              unsigned long long* __restrict__ task, unsigned long long* __restrict__ keys,
                              unsigned int* __restrict__ nkeys) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L.n) return;
  const uint32_t b = c / group;
  const unsigned long long nc = count[c];
  unsigned long long owned = nc * (nc - 1);
  for (uint32_t k = off[c]; k < off[c + 1]; ++k) {
    const uint32_t o = cells[k], ob = o / group;
    if (ob < b || (ob == b && o < c)) continue;
    if (ob != b) keys[atomicAdd(nkeys, 1u)] = (static_cast<unsigned long long>(b) << 32) | ob;
    owned += 2 * nc * count[o];
  }
  atomicAdd(&task[b], owned);
}
// sorted (hi << 32 | lo) keys -> lo list, counts per hi, optionally the swapped keys
__global__ void k_split_keys(const unsigned long long* __restrict__ keys, uint32_t n,
                             uint32_t* __restrict__ lo_out, unsigned long long* __restrict__ swapped,
                             uint32_t* __restrict__ cnt) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t hi = static_cast<uint32_t>(keys[i] >> 32), lo = static_cast<uint32_t>(keys[i]);
  lo_out[i] = lo;
  atomicAdd(&cnt[hi], 1u);
  if (swapped) swapped[i] = (static_cast<unsigned long long>(lo) << 32) | hi;
}

// far pairs of level v -> (target block << 32 | source block) keys
__global__ void k_far_block_keys(const uint32_t* __restrict__ tgt, const uint32_t* __restrict__ src, uint64_t n,
                                 uint32_t group, unsigned long long* __restrict__ keys) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) keys[i] = (static_cast<unsigned long long>(tgt[i] / group) << 32) | (src[i] / group);
}

__global__ void k_group_off(const unsigned long long* __restrict__ pos, uint64_t ngroups, uint32_t group,
                            uint64_t total, uint64_t* __restrict__ goff) {
  const uint64_t g = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (g < ngroups) goff[g] = pos[g * group];
  if (g == ngroups) goff[g] = total;
}

}  // namespace

void lists_free(fmmgpu_ctx* c) {
  cudaStream_t s = c->s_far;
  dfree(c, c->d_near_off, s);
  dfree(c, c->d_near_cells, s);
  c->d_near_off = nullptr;
  c->d_near_cells = nullptr;
  for (auto& L : c->lv) {
    dfree(c, L.far_target, s);
    dfree(c, L.far_source, s);
    dfree(c, L.far_vec, s);
    dfree(c, L.far_group_off, s);
    L.far_target = L.far_source = nullptr;
    L.far_vec = nullptr;
    L.far_group_off = nullptr;
    L.far_pairs = 0;
  }
  c->have_lists = false;
}

uint64_t near_directional_count(fmmgpu_ctx* c) {
  cudaStream_t s = c->s_far;
  const int leaf = c->height - 1;
  const Level& L = c->lv[leaf];
  uint32_t* cnt = dalloc<uint32_t>(c, L.n, s);
  unsigned long long* work = dalloc<unsigned long long>(c, L.n + 1, s);
  k_near_count<<<blocks(L.n, 128), 128, 0, s>>>(L.view(leaf), L.particle_count, cnt, work);
  FMM_CUDA(cudaGetLastError());
  size_t tb = 0;
  FMM_CUDA(cub::DeviceReduce::Sum(nullptr, tb, work, work + L.n, static_cast<int>(L.n), s));
  FMM_CUDA(cub::DeviceReduce::Sum(scratch(c, tb), tb, work, work + L.n, static_cast<int>(L.n), s));
  unsigned long long total = 0;
  FMM_CUDA(cudaMemcpyAsync(&total, work + L.n, 8, cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  dfree(c, cnt, s);
  dfree(c, work, s);
  return total;
}

void lists_build(fmmgpu_ctx* c) {
  if (!c->have_tree) throw Error(FMMGPU_LOGIC_ERROR, "build_lists: no tree");
  lists_free(c);
  cudaStream_t s = c->s_far;
  const int leaf = c->height - 1;
  // near CSR
  {
    const Level& L = c->lv[leaf];
    uint32_t* cnt = dalloc<uint32_t>(c, L.n + 1, s);
    unsigned long long* work = dalloc<unsigned long long>(c, L.n + 1, s);
    FMM_CUDA(cudaMemsetAsync(cnt + L.n, 0, 4, s));
    k_near_count<<<blocks(L.n, 128), 128, 0, s>>>(L.view(leaf), L.particle_count, cnt, work);
    FMM_CUDA(cudaGetLastError());
    c->d_near_off = dalloc<uint32_t>(c, L.n + 1, s);
    size_t tb = 0;
    FMM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, c->d_near_off, static_cast<int>(L.n + 1), s));
    FMM_CUDA(cub::DeviceScan::ExclusiveSum(scratch(c, tb), tb, cnt, c->d_near_off, static_cast<int>(L.n + 1), s));
    FMM_CUDA(cub::DeviceReduce::Sum(nullptr, tb, work, work + L.n, static_cast<int>(L.n), s));
    FMM_CUDA(cub::DeviceReduce::Sum(scratch(c, tb), tb, work, work + L.n, static_cast<int>(L.n), s));
    uint32_t entries = 0;
    unsigned long long total = 0;
    FMM_CUDA(cudaMemcpyAsync(&entries, c->d_near_off + L.n, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(&total, work + L.n, 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    c->near_entries = entries;
    c->near_directional = total;
    c->d_near_cells = dalloc<uint32_t>(c, entries, s);
    k_near_fill<<<blocks(L.n, 128), 128, 0, s>>>(L.view(leaf), c->d_near_off, c->d_near_cells);
    FMM_CUDA(cudaGetLastError());
    dfree(c, cnt, s);
    dfree(c, work, s);
  }
  // far pairs per level
  for (int v = 2; v <= leaf; ++v) {
    Level& L = c->lv[v];
    const Level& P = c->lv[v - 1];
    const uint64_t nb = L.block_offsets.size() - 1;
    const uint64_t ng = nb * 16;
    const uint64_t slots = ng * c->group;
    uint32_t* cnt = dalloc<uint32_t>(c, slots, s);
    unsigned long long* pos = dalloc<unsigned long long>(c, slots + 1, s);
    FMM_CUDA(cudaMemsetAsync(cnt, 0, 4 * slots, s));
    FarArgs a{L.view(v), P.view(v - 1), L.parent, P.first_child, P.child_count, c->d_canon,
              static_cast<uint32_t>(c->group)};
    k_far_count<<<blocks(L.n, 128), 128, 0, s>>>(a, cnt);
    FMM_CUDA(cudaGetLastError());
    size_t tb = 0;
    FMM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, pos, static_cast<int>(slots), s));
    FMM_CUDA(cub::DeviceScan::ExclusiveSum(scratch(c, tb), tb, cnt, pos, static_cast<int>(slots), s));
    unsigned long long last_pos = 0;
    uint32_t last_cnt = 0;
    FMM_CUDA(cudaMemcpyAsync(&last_pos, pos + slots - 1, 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaMemcpyAsync(&last_cnt, cnt + slots - 1, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    const uint64_t total = last_pos + last_cnt;
    L.far_pairs = total;
    L.far_target = dalloc<uint32_t>(c, total, s);
    L.far_source = dalloc<uint32_t>(c, total, s);
    L.far_vec = dalloc<uint16_t>(c, total, s);
    L.far_group_off = dalloc<uint64_t>(c, ng + 1, s);
    k_group_off<<<blocks(ng + 1, 256), 256, 0, s>>>(pos, ng, c->group, total, L.far_group_off);
    k_far_fill_warp<<<blocks(uint64_t(L.n) * 32, 256), 256, 0, s>>>(a, pos, L.far_target, L.far_source, L.far_vec);
    FMM_CUDA(cudaGetLastError());
    dfree(c, cnt, s);
    dfree(c, pos, s);
  }
  FMM_CUDA(cudaStreamSynchronize(s));
  c->have_lists = true;
}


// The block-level near plan (partners_above / contributors_below as CSR, task_interactions)
// from the near CSR; host arrays, NULL = skip. Returns the two list lengths.
void near_blocks(fmmgpu_ctx* c, uint64_t* task_out, uint32_t* above_off, uint32_t* above, uint32_t* below_off,
                 uint32_t* below, uint64_t* n_above, uint64_t* n_below) {
  if (!c->have_lists) throw Error(FMMGPU_LOGIC_ERROR, "no lists: call fmmgpu_build_lists first");
  cudaStream_t s = c->s_far;
  const int leaf = c->height - 1;
  const Level& L = c->lv[leaf];
  const uint32_t nb = static_cast<uint32_t>(L.block_offsets.size() - 1);
  const uint32_t group = static_cast<uint32_t>(c->group);
  unsigned long long* task = dalloc<unsigned long long>(c, nb, s);
  unsigned long long* keys = dalloc<unsigned long long>(c, c->near_entries + 1, s);
  unsigned long long* keys2 = dalloc<unsigned long long>(c, c->near_entries + 1, s);
  uint32_t* nkeys = dalloc<uint32_t>(c, 2, s);
  FMM_CUDA(cudaMemsetAsync(task, 0, 8ull * nb, s));
  FMM_CUDA(cudaMemsetAsync(nkeys, 0, 8, s));
  k_near_blocks<<<blocks(L.n, 128), 128, 0, s>>>(L.view(leaf), L.particle_count, c->d_near_off, c->d_near_cells,
                                                 group, task, keys, nkeys);
  FMM_CUDA(cudaGetLastError());
  uint32_t nk = 0;
  FMM_CUDA(cudaMemcpyAsync(&nk, nkeys, 4, cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  size_t tb = 0;
  // unique sorted (b, b') pairs: partners_above in order
  uint32_t nu = 0;
  if (nk) {
    FMM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys2, static_cast<int>(nk), 0, 64, s));
    FMM_CUDA(cub::DeviceRadixSort::SortKeys(scratch(c, tb), tb, keys, keys2, static_cast<int>(nk), 0, 64, s));
    FMM_CUDA(cub::DeviceSelect::Unique(nullptr, tb, keys2, keys, nkeys + 1, static_cast<int>(nk), s));
    FMM_CUDA(cub::DeviceSelect::Unique(scratch(c, tb), tb, keys2, keys, nkeys + 1, static_cast<int>(nk), s));
    FMM_CUDA(cudaMemcpyAsync(&nu, nkeys + 1, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  uint32_t* lo = dalloc<uint32_t>(c, nu + 1, s);
  uint32_t* cnt = dalloc<uint32_t>(c, nb + 1, s);
  uint32_t* offs = dalloc<uint32_t>(c, nb + 1, s);
  auto csr = [&](const unsigned long long* k, unsigned long long* swapped, uint32_t* off_out, uint32_t* list_out) {
    FMM_CUDA(cudaMemsetAsync(cnt, 0, 4ull * (nb + 1), s));
    if (nu) {
      k_split_keys<<<blocks(nu, 256), 256, 0, s>>>(k, nu, lo, swapped, cnt);
      FMM_CUDA(cudaGetLastError());
    }
    FMM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, offs, static_cast<int>(nb + 1), s));
    FMM_CUDA(cub::DeviceScan::ExclusiveSum(scratch(c, tb), tb, cnt, offs, static_cast<int>(nb + 1), s));
    if (off_out) FMM_CUDA(cudaMemcpyAsync(off_out, offs, 4ull * (nb + 1), cudaMemcpyDeviceToHost, s));
    if (list_out && nu) FMM_CUDA(cudaMemcpyAsync(list_out, lo, 4ull * nu, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  };
  csr(keys, keys2, above_off, above);  // keys2 <- (b', b): the transposed pairs
  if (nu) {  // contributors_below: the transposed pairs sorted
    FMM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys2, keys, static_cast<int>(nu), 0, 64, s));
    FMM_CUDA(cub::DeviceRadixSort::SortKeys(scratch(c, tb), tb, keys2, keys, static_cast<int>(nu), 0, 64, s));
  }
  csr(keys, nullptr, below_off, below);
  if (task_out) FMM_CUDA(cudaMemcpyAsync(task_out, task, 8ull * nb, cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  if (n_above) *n_above = nu;
  if (n_below) *n_below = nu;
  dfree(c, task, s);
  dfree(c, keys, s);
  dfree(c, keys2, s);
  dfree(c, nkeys, s);
  dfree(c, lo, s);
  dfree(c, cnt, s);
  dfree(c, offs, s);
}


// LevelM2L::source_blocks (taskflow.cpp:96-102): per target block of level v, its far
// sources' blocks, ascending and unique, as CSR (host arrays, NULL = skip).
void far_source_blocks(fmmgpu_ctx* c, int v, uint32_t* off_out, uint32_t* list_out, uint64_t* n_out) {
  if (!c->have_lists) throw Error(FMMGPU_LOGIC_ERROR, "no lists: call fmmgpu_build_lists first");
  if (v < 2 || v >= c->height) throw Error(FMMGPU_OUT_OF_RANGE, "far_source_blocks: level out of range");
  cudaStream_t s = c->s_far;
  const Level& L = c->lv[v];
  const uint32_t nb = static_cast<uint32_t>(L.block_offsets.size() - 1);
  const uint64_t np = L.far_pairs;
  unsigned long long* keys = dalloc<unsigned long long>(c, np + 1, s);
  unsigned long long* keys2 = dalloc<unsigned long long>(c, np + 1, s);
  uint32_t* nu_d = dalloc<uint32_t>(c, 1, s);
  uint32_t nu = 0;
  size_t tb = 0;
  if (np) {
    k_far_block_keys<<<static_cast<unsigned>((np + 255) / 256), 256, 0, s>>>(L.far_target, L.far_source, np,
                                                                             static_cast<uint32_t>(c->group), keys);
    FMM_CUDA(cudaGetLastError());
    FMM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys2, static_cast<int>(np), 0, 64, s));
    FMM_CUDA(cub::DeviceRadixSort::SortKeys(scratch(c, tb), tb, keys, keys2, static_cast<int>(np), 0, 64, s));
    FMM_CUDA(cub::DeviceSelect::Unique(nullptr, tb, keys2, keys, nu_d, static_cast<int>(np), s));
    FMM_CUDA(cub::DeviceSelect::Unique(scratch(c, tb), tb, keys2, keys, nu_d, static_cast<int>(np), s));
    FMM_CUDA(cudaMemcpyAsync(&nu, nu_d, 4, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
  }
  uint32_t* lo = dalloc<uint32_t>(c, nu + 1, s);
  uint32_t* cnt = dalloc<uint32_t>(c, nb + 1, s);
  uint32_t* offs = dalloc<uint32_t>(c, nb + 1, s);
  FMM_CUDA(cudaMemsetAsync(cnt, 0, 4ull * (nb + 1), s));
  if (nu) {
    k_split_keys<<<blocks(nu, 256), 256, 0, s>>>(keys, nu, lo, nullptr, cnt);
    FMM_CUDA(cudaGetLastError());
  }
  FMM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, offs, static_cast<int>(nb + 1), s));
  FMM_CUDA(cub::DeviceScan::ExclusiveSum(scratch(c, tb), tb, cnt, offs, static_cast<int>(nb + 1), s));
  if (off_out) FMM_CUDA(cudaMemcpyAsync(off_out, offs, 4ull * (nb + 1), cudaMemcpyDeviceToHost, s));
  if (list_out && nu) FMM_CUDA(cudaMemcpyAsync(list_out, lo, 4ull * nu, cudaMemcpyDeviceToHost, s));
  FMM_CUDA(cudaStreamSynchronize(s));
  if (n_out) *n_out = nu;
  dfree(c, keys, s);
  dfree(c, keys2, s);
  dfree(c, nu_d, s);
  dfree(c, lo, s);
  dfree(c, cnt, s);
  dfree(c, offs, s);
}

}  // namespace fmmgpu
