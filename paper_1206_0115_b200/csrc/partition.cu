// Multi-GPU evaluation by contiguous Morton ranges of leaves.
//
// Every rank holds the whole particle set and builds the whole tree (bit-identical by
// construction), then owns a contiguous Morton range of leaf cells aligned to the cells
// of an alignment level a, balanced by an estimate of near + far work. Per level:
//   levels >= a : cells are owned by exactly one rank; P2M / M2M / M2L / L2L / L2P / P2P
//                 run on owned cells (M2L phase A on the sources that have an owned
//                 target: owned cells plus a halo of the far stencil);
//   levels <  a : replicated (every rank computes every cell: a handful of cells).
// One exchange step per upward level >= a, after that level's multipoles are formed:
//   level a (when M2M(a-1) >= 2 runs on the replicated levels): an all-gather (in-place
//           allgatherv = one ncclBroadcast per rank inside a group) -- every rank needs
//           all of level a for its replicated parents;
//   levels > a: a HALO exchange -- each rank receives exactly the multipoles of the
//           non-owned cells its M2L phase A reads (children of the parents adjacent to
//           the parents of its owned targets) from their owners, ncclSend / ncclRecv per
//           peer inside one group, packed / unpacked by two small kernels.
// The downward pass, P2P and L2P need no communication (replicated particles, owner
// computes; P2P pairs across a rank boundary are evaluated one-sided on the owner's
// side), so results are deterministic and identical to the single-device evaluation up
// to rounding order.
//
// NCCL is loaded lazily (dlopen) only when a communicator is attached; the stepped API
// (fmmgpu_upward_level / fmmgpu_downward + fmmgpu_exchange_plan) lets a host drive the
// same exchange itself (tests: N contexts on one device, or processes over gloo).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <numeric>

#include <cstdlib>

#include "common.cuh"

namespace fmmgpu {

namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

}  // namespace

// The NCCL the process already has (torch's, when torch.distributed is up) wins; else
// FMMGPU_NCCL_LIB (the Python binding points it at torch's bundled libnccl, so a later
// `import torch` finds the NCCL it was built against under the same soname); else the
// system libnccl.so.2.
void* open_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  const char* env = std::getenv("FMMGPU_NCCL_LIB");
  if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw Error(FMMGPU_RUNTIME_ERROR, "NCCL not available (dlopen libnccl.so.2 failed)");
  return h;
}

namespace {

NcclApi& nccl() {
  static NcclApi api;
  if (!api.handle) {
    void* h = open_nccl();
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    if (!api.getUniqueId || !api.commInitRank || !api.commDestroy || !api.groupStart || !api.groupEnd ||
        !api.broadcast || !api.errorString || !api.send || !api.recv)
      throw Error(FMMGPU_RUNTIME_ERROR, "NCCL library lacks required symbols");
    api.handle = h;
  }
  return api;
}

#define NCCL_CHECK(x)                                                                                    \
  do {                                                                                                   \
    ncclResult_t r_ = (x);                                                                               \
    if (r_ != ncclSuccess) throw Error(FMMGPU_RUNTIME_ERROR, std::string("NCCL: ") + nccl().errorString(r_)); \
  } while (0)

template <typename T>
std::vector<T> download(const T* d, size_t n) {
  std::vector<T> h(n);
  if (n) FMM_CUDA(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
  return h;
}

void free_lists(Level& L) {
  if (L.srcA) cudaFree(L.srcA);
  if (L.tgtB) cudaFree(L.tgtB);
  if (L.halo_idx) cudaFree(L.halo_idx);
  L.srcA = L.tgtB = nullptr;
  L.halo_idx = nullptr;
  L.xkind = 0;
  L.halo_send_off.clear();
  L.halo_recv_off.clear();
  L.halo_send.clear();
  L.halo_recv.clear();
}

// rows idx[0..cnt) of the multipole array <-> a contiguous buffer (ld doubles per row)
__global__ void k_pack_rows(const double* __restrict__ src, const uint32_t* __restrict__ idx, uint32_t cnt, int ld,
                            double* __restrict__ dst) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= uint64_t(cnt) * ld) return;
  const uint64_t r = i / ld, k = i % ld;
  dst[i] = src[uint64_t(idx[r]) * ld + k];
}
__global__ void k_unpack_rows(const double* __restrict__ src, const uint32_t* __restrict__ idx, uint32_t cnt, int ld,
                              double* __restrict__ dst) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= uint64_t(cnt) * ld) return;
  const uint64_t r = i / ld, k = i % ld;
  dst[uint64_t(idx[r]) * ld + k] = src[i];
}

// cells grouped by parity class (code & 7), ascending index inside a class
void upload_class_list(const std::vector<uint64_t>& code, const std::vector<uint32_t>& cells, uint32_t** dst,
                       uint32_t off[9]) {
  std::vector<uint32_t> sorted;
  sorted.reserve(cells.size());
  for (int q = 0; q < 8; ++q) {
    off[q] = static_cast<uint32_t>(sorted.size());
    for (uint32_t c : cells)
      if (static_cast<int>(code[c] & 7) == q) sorted.push_back(c);
  }
  off[8] = static_cast<uint32_t>(sorted.size());
  FMM_CUDA(cudaMalloc(dst, std::max<size_t>(1, sorted.size()) * sizeof(uint32_t)));
  if (!sorted.empty())
    FMM_CUDA(cudaMemcpy(*dst, sorted.data(), sorted.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
}

}  // namespace

void partition_free(fmmgpu_ctx* c) {
  for (auto& L : c->lv) free_lists(L);
  c->part_begin.clear();
  if (c->d_halo_buf) cudaFree(c->d_halo_buf);
  c->d_halo_buf = nullptr;
  c->halo_buf_cap = 0;
}

void exchange_level(fmmgpu_ctx* c, int v, cudaStream_t s) {
  if (c->part_n <= 1 || v >= c->height || c->lv[v].xkind == 0) return;
  if (c->skip_exchange) return;  // fmmgpu_set_measurement: one rank's work timed alone
  if (!c->nccl) throw Error(FMMGPU_LOGIC_ERROR, "partitioned evaluate needs a communicator (fmmgpu_comm_init) "
                                                "or the stepped API with a host exchange");
  auto& api = nccl();
  Level& L = c->lv[v];
  const int ld = c->ldE;
  auto* comm = static_cast<ncclComm_t>(c->nccl);
  if (L.xkind == 1) {  // all-gather: every rank broadcasts its owned rows in place
    const auto& b = c->part_begin[v];
    NCCL_CHECK(api.groupStart());
    for (int r = 0; r < c->part_n; ++r) {
      const size_t cnt = size_t(b[r + 1] - b[r]) * ld;
      if (!cnt) continue;
      double* p = L.multipole + size_t(b[r]) * ld;
      NCCL_CHECK(api.broadcast(p, p, cnt, ncclDouble, r, comm, s));
    }
    NCCL_CHECK(api.groupEnd());
    return;
  }
  // halo: pack the rows every peer needs, send / receive per peer, unpack
  const uint32_t nsend = L.halo_send_off.back(), nrecv = L.halo_recv_off.back();
  double* sbuf = c->d_halo_buf;
  double* rbuf = c->d_halo_buf + size_t(nsend) * ld;
  if (nsend) {
    const uint64_t tot = uint64_t(nsend) * ld;
    k_pack_rows<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(L.multipole, L.halo_idx, nsend, ld, sbuf);
    FMM_CUDA(cudaGetLastError());
    ++c->launches;
  }
  NCCL_CHECK(api.groupStart());
  for (int p = 0; p < c->part_n; ++p) {
    if (p == c->part_rank) continue;
    const uint32_t so = L.halo_send_off[p], sc = L.halo_send_off[p + 1] - so;
    const uint32_t ro = L.halo_recv_off[p], rc = L.halo_recv_off[p + 1] - ro;
    if (sc) NCCL_CHECK(api.send(sbuf + size_t(so) * ld, size_t(sc) * ld, ncclDouble, p, comm, s));
    if (rc) NCCL_CHECK(api.recv(rbuf + size_t(ro) * ld, size_t(rc) * ld, ncclDouble, p, comm, s));
  }
  NCCL_CHECK(api.groupEnd());
  if (nrecv) {
    const uint64_t tot = uint64_t(nrecv) * ld;
    k_unpack_rows<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(rbuf, L.halo_idx + nsend, nrecv, ld,
                                                                           L.multipole);
    FMM_CUDA(cudaGetLastError());
    ++c->launches;
  }
}

}  // namespace fmmgpu

using namespace fmmgpu;

extern "C" {

// Balanced contiguous split of weighted items (host only, no device needed):
// begins[r] = first item of rank r, begins[nranks] = n; rank r takes the items whose
// weight prefix midpoint falls in [r/nranks, (r+1)/nranks) of the total.
int fmmgpu_plan_partition(const uint64_t* weights, uint32_t n, int nranks, uint32_t* begins) {
  if (nranks < 1 || (!weights && n) || !begins) return FMMGPU_INVALID_ARGUMENT;
  long double total = 0;
  for (uint32_t i = 0; i < n; ++i) total += static_cast<long double>(weights[i]);
  std::fill(begins, begins + nranks + 1, n);
  begins[0] = 0;
  long double acc = 0;
  int r = 1;
  for (uint32_t i = 0; i < n && r < nranks; ++i) {
    const long double mid = acc + 0.5L * weights[i];
    while (r < nranks && total > 0 && mid >= total * r / nranks) begins[r++] = i;
    acc += weights[i];
  }
  for (int k = 1; k <= nranks; ++k) begins[k] = std::max(begins[k], begins[k - 1]);
  return FMMGPU_OK;
}

int fmmgpu_partition(fmmgpu_ctx* c, int rank, int nranks) {
  try {
    if (!c || !c->have_tree) throw Error(FMMGPU_LOGIC_ERROR, "no tree: call fmmgpu_build_tree first");
    if (nranks < 1 || rank < 0 || rank >= nranks || nranks > 64)
      throw Error(FMMGPU_INVALID_ARGUMENT, "bad rank / nranks (1 <= nranks <= 64)");
    if (c->dist && !c->dsend_off.empty() && (rank != c->part_rank || nranks != c->part_n))
      throw Error(FMMGPU_LOGIC_ERROR, "distributed tree: its particles were placed for rank " +
                                          std::to_string(c->part_rank) + " of " + std::to_string(c->part_n));
    if (c->dist && !c->dsend_off.empty()) return FMMGPU_OK;  // already partitioned this way
    FMM_CUDA(cudaSetDevice(c->device));
    FMM_CUDA(cudaStreamSynchronize(c->s_near));
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
    partition_free(c);
    fmmgpu_invalidate_graph(c);
    const int h = c->height, leaf = h - 1;
    c->part_rank = rank;
    c->part_n = nranks;
    c->part_begin.assign(h, {});
    if (nranks == 1) {
      c->part_align = 0;
      for (int v = 0; v < h; ++v) {
        c->lv[v].own0 = 0;
        c->lv[v].own1 = c->lv[v].n;
        c->part_begin[v] = {0, c->lv[v].n};
      }
      c->own_s0 = 0;
      c->own_s1 = c->n;
      return FMMGPU_OK;
    }
    // alignment level: the first level with enough cells to balance nranks
    int a = leaf - 1;
    for (int v = 1; v <= leaf - 1; ++v)
      if (c->lv[v].n >= 4u * static_cast<uint32_t>(nranks)) {
        a = v;
        break;
      }
    c->part_align = a;
    std::vector<std::vector<uint64_t>> code(h);
    for (int v = std::max(0, a - 1); v < h; ++v) code[v] = download(c->lv[v].code, c->lv[v].n);
    const auto lcnt = download(c->lv[leaf].particle_count, c->lv[leaf].n);
    const auto lfirst = download(c->lv[leaf].first_particle, c->lv[leaf].n);
    // work estimate per level-a cell: near field 15 * 27 n^2 + far field 8 l^3 R per leaf
    const uint64_t far_leaf = 8ull * c->l3 * static_cast<uint64_t>(c->m2l.R);
    std::vector<uint64_t> wa(c->lv[a].n, 0);
    {
      const int sh = 3 * (leaf - a);
      uint32_t ia = 0;
      for (uint32_t i = 0; i < c->lv[leaf].n; ++i) {
        const uint64_t anc = code[leaf][i] >> sh;
        while (code[a][ia] != anc) ++ia;
        wa[ia] += 405ull * lcnt[i] * lcnt[i] + far_leaf;
      }
    }
    std::vector<uint32_t> ba(nranks + 1);
    fmmgpu_plan_partition(wa.data(), c->lv[a].n, nranks, ba.data());
    for (int v = 0; v < h; ++v) {
      auto& pb = c->part_begin[v];
      if (v < a) {
        pb.assign(nranks + 1, c->lv[v].n);
        pb[0] = 0;
        c->lv[v].own0 = 0;
        c->lv[v].own1 = c->lv[v].n;
        continue;
      }
      pb.resize(nranks + 1);
      const int sh = 3 * (v - a);
      for (int r = 0; r <= nranks; ++r) {
        if (ba[r] >= c->lv[a].n) {
          pb[r] = c->lv[v].n;
          continue;
        }
        const uint64_t first = code[a][ba[r]] << sh;  // first possible descendant code
        pb[r] = static_cast<uint32_t>(std::lower_bound(code[v].begin(), code[v].end(), first) - code[v].begin());
      }
      c->lv[v].own0 = pb[rank];
      c->lv[v].own1 = pb[rank + 1];
    }
    const Level& LL = c->lv[leaf];
    c->own_s0 = LL.own0 < LL.n ? lfirst[LL.own0] : c->n;
    c->own_s1 = LL.own1 < LL.n ? lfirst[LL.own1] : c->n;
    // M2L lists of the partitioned levels: phase B targets = owned cells; phase A
    // sources = children of parents adjacent to (or equal to) an owned target's parent.
    // The same rule for every rank gives the halo plan: cell s is needed by the ranks
    // owning a target below a parent adjacent to parent(s) (bit mask over ranks).
    size_t halo_rows = 0;
    for (int v = std::max(2, a); v <= leaf; ++v) {
      Level& L = c->lv[v];
      const auto par = download(L.parent, L.n);
      const Level& P = c->lv[v - 1];
      const auto& pb = c->part_begin[v];
      const int gp = 1 << (v - 1);
      // owner rank of every cell of this level
      std::vector<uint16_t> owner(L.n);
      for (int r = 0; r < nranks; ++r)
        for (uint32_t t = pb[r]; t < pb[r + 1]; ++t) owner[t] = static_cast<uint16_t>(r);
      // ranks owning a child of each parent, then the ranks needing each parent's children
      std::vector<uint64_t> kids(P.n, 0), need(P.n, 0);
      for (uint32_t t = 0; t < L.n; ++t) kids[par[t]] |= 1ull << (owner[t] & 63);
      const bool pfull = P.full;
      for (uint32_t p = 0; p < P.n; ++p) {
        int ijk[3];
        demorton(code[v - 1][p], ijk);
        uint64_t m = 0;
        for (int di = -1; di <= 1; ++di)
          for (int dj = -1; dj <= 1; ++dj)
            for (int dk = -1; dk <= 1; ++dk) {
              const int x = ijk[0] + di, y = ijk[1] + dj, z = ijk[2] + dk;
              if (x < 0 || y < 0 || z < 0 || x >= gp || y >= gp || z >= gp) continue;
              const uint64_t cd = morton(x, y, z);
              if (pfull) {
                m |= kids[cd];
              } else {
                auto it = std::lower_bound(code[v - 1].begin(), code[v - 1].end(), cd);
                if (it != code[v - 1].end() && *it == cd) m |= kids[it - code[v - 1].begin()];
              }
            }
        need[p] = m;
      }
      std::vector<uint32_t> src, tgt;
      for (uint32_t s2 = 0; s2 < L.n; ++s2)
        if ((need[par[s2]] >> rank) & 1u) src.push_back(s2);
      for (uint32_t t = L.own0; t < L.own1; ++t) tgt.push_back(t);
      upload_class_list(code[v], src, &L.srcA, L.srcA_off);
      upload_class_list(code[v], tgt, &L.tgtB, L.tgtB_off);
      // exchange kind: the alignment level is all-gathered when the replicated levels
      // above it run M2M (parent level a-1 >= 2); deeper levels exchange the halo only
      L.xkind = (v == a && a - 1 >= 2) ? 1 : 2;
      if (L.xkind == 2) {
        std::vector<std::vector<uint32_t>> snd(nranks), rcv(nranks);
        for (uint32_t s2 = 0; s2 < L.n; ++s2) {
          const uint64_t m = need[par[s2]];
          const int o = owner[s2];
          if (o == rank) {
            for (int p = 0; p < nranks; ++p)
              if (p != rank && ((m >> p) & 1u)) snd[p].push_back(s2);
          } else if ((m >> rank) & 1u) {
            rcv[o].push_back(s2);
          }
        }
        L.halo_send_off.assign(1, 0);
        L.halo_recv_off.assign(1, 0);
        for (int p = 0; p < nranks; ++p) {
          L.halo_send.insert(L.halo_send.end(), snd[p].begin(), snd[p].end());
          L.halo_recv.insert(L.halo_recv.end(), rcv[p].begin(), rcv[p].end());
          L.halo_send_off.push_back(static_cast<uint32_t>(L.halo_send.size()));
          L.halo_recv_off.push_back(static_cast<uint32_t>(L.halo_recv.size()));
        }
        const size_t tot = L.halo_send.size() + L.halo_recv.size();
        FMM_CUDA(cudaMalloc(&L.halo_idx, std::max<size_t>(1, tot) * sizeof(uint32_t)));
        if (!L.halo_send.empty())
          FMM_CUDA(cudaMemcpy(L.halo_idx, L.halo_send.data(), L.halo_send.size() * 4, cudaMemcpyHostToDevice));
        if (!L.halo_recv.empty())
          FMM_CUDA(cudaMemcpy(L.halo_idx + L.halo_send.size(), L.halo_recv.data(), L.halo_recv.size() * 4,
                              cudaMemcpyHostToDevice));
        halo_rows = std::max(halo_rows, tot);
      }
    }
    if (halo_rows) {
      FMM_CUDA(cudaMalloc(&c->d_halo_buf, halo_rows * c->ldE * sizeof(double)));
      c->halo_buf_cap = halo_rows;
    }
    return FMMGPU_OK;
  } catch (const Error& e) {
    if (c) c->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return FMMGPU_RUNTIME_ERROR;
  }
}

int fmmgpu_partition_ranges(const fmmgpu_ctx* c, int level, uint32_t* begins) {
  if (!c || !c->have_tree || level < 0 || level >= c->height || !begins) return FMMGPU_INVALID_ARGUMENT;
  if (c->part_begin.empty()) {
    begins[0] = 0;
    begins[1] = c->lv[level].n;
    return FMMGPU_OK;
  }
  std::copy(c->part_begin[level].begin(), c->part_begin[level].end(), begins);
  return FMMGPU_OK;
}

int fmmgpu_partition_info(const fmmgpu_ctx* c, int* rank, int* nranks, int* align_level, uint64_t* slot_begin,
                          uint64_t* slot_end) {
  if (!c || !c->have_tree) return FMMGPU_LOGIC_ERROR;
  if (rank) *rank = c->part_rank;
  if (nranks) *nranks = c->part_n;
  if (align_level) *align_level = c->part_align;
  if (slot_begin) *slot_begin = c->own_s0;
  if (slot_end) *slot_end = c->own_s1;
  return FMMGPU_OK;
}

int fmmgpu_exchange_plan(const fmmgpu_ctx* c, int level, int peer, int* kind, uint32_t* send_cells,
                         uint32_t* send_count, uint32_t* recv_cells, uint32_t* recv_count) {
  if (!c || !c->have_tree || level < 0 || level >= c->height) return FMMGPU_INVALID_ARGUMENT;
  const Level& L = c->lv[level];
  const int k = c->part_n > 1 ? L.xkind : 0;
  if (kind) *kind = k;
  uint32_t sc = 0, rc = 0;
  if (k == 2) {
    if (peer < 0 || peer >= c->part_n) return FMMGPU_INVALID_ARGUMENT;
    const uint32_t so = L.halo_send_off[peer], ro = L.halo_recv_off[peer];
    sc = L.halo_send_off[peer + 1] - so;
    rc = L.halo_recv_off[peer + 1] - ro;
    if (send_cells) std::copy(L.halo_send.begin() + so, L.halo_send.begin() + so + sc, send_cells);
    if (recv_cells) std::copy(L.halo_recv.begin() + ro, L.halo_recv.begin() + ro + rc, recv_cells);
  }
  if (send_count) *send_count = sc;
  if (recv_count) *recv_count = rc;
  return FMMGPU_OK;
}

int fmmgpu_set_measurement(fmmgpu_ctx* c, int skip_exchange) {
  if (!c) return FMMGPU_INVALID_ARGUMENT;
  c->skip_exchange = skip_exchange != 0;
  c->out_valid = false;
  return FMMGPU_OK;
}

int fmmgpu_comm_unique_id(char* out128) {
  try {
    ncclUniqueId id;
    NCCL_CHECK(nccl().getUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return FMMGPU_OK;
  } catch (const std::exception&) {
    return FMMGPU_RUNTIME_ERROR;
  }
}

int fmmgpu_comm_destroy(fmmgpu_ctx* c) {
  if (!c) return FMMGPU_INVALID_ARGUMENT;
  if (c->nccl) {
    try {
      nccl().commDestroy(static_cast<ncclComm_t>(c->nccl));
    } catch (...) {
    }
    c->nccl = nullptr;
  }
  return FMMGPU_OK;
}

int fmmgpu_comm_init(fmmgpu_ctx* c, const char* id128, int nranks, int rank) {
  try {
    if (!c || !id128 || nranks < 1 || rank < 0 || rank >= nranks)
      throw Error(FMMGPU_INVALID_ARGUMENT, "bad communicator arguments");
    FMM_CUDA(cudaSetDevice(c->device));
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    NCCL_CHECK(nccl().commInitRank(&comm, nranks, id, rank));
    if (c->nccl) nccl().commDestroy(static_cast<ncclComm_t>(c->nccl));
    c->nccl = comm;
    c->comm_rank = rank;
    c->comm_n = nranks;
    return FMMGPU_OK;
  } catch (const Error& e) {
    if (c) c->err = e.what();
    return e.code;
  }
}

}  // extern "C"
