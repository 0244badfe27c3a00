// Distributed input for the multi-GPU path ("leaves partitioned by
// contiguous Morton ranges, with halo particles ... exchanged"). Rank r holds only the
// input slice [off[r], off[r + 1]) of the n particles (input order, slices in rank
// order). Nothing but Morton keys and the particles a rank actually reads cross the
// ranks:
//
//   1. local bounds      each rank's per-axis min / max (device reduction); the ranks'
//                        bounds are combined (min / max, exact) and the root cube follows
//                        from the same arithmetic as the single-device build
//                        (geometry.cpp:28-34, root_from_bounds);
//   2. local keys        leaf Morton keys of the slice (geometry.cpp:76-94), u64;
//   3. all-gather keys   8 B per particle instead of the 32 B particle record;
//   4. tree from keys    the stable radix sort of (key, input index) and every level
//                        array exactly as tree_build computes them from positions, so
//                        the tree, Morton order and ids are bit-identical to the
//                        single-device build of the whole set; then the partition
//                        (partition.cu) of the leaves into contiguous Morton ranges;
//   5. particle plan     a leaf is needed by the rank that owns it and by the owners of
//                        its 26 neighbours (P2P reads the 27-neighbourhood of an owned
//                        leaf; P2M / L2P read owned leaves only). Slot j goes from the
//                        rank holding input index id[j] to every rank that needs its
//                        leaf: one compaction per peer over the Morton slots, computed
//                        identically on both sides, so sender and receiver agree on the
//                        order without exchanging the lists;
//   6. particle exchange records of owned + halo leaves only (per-peer send / receive);
//   7. coincident check  on each rank's owned leaves (geometry.cpp:126-136: equal
//                        positions always share a leaf), flags OR-ed over the ranks.
//
// The stepped entry points (fmmgpu_dist_*) let a host drive steps 1-7 with its own
// collectives (tests: processes over gloo); fmmgpu_build_tree_distributed runs them with
// the attached NCCL communicator.
#include <dlfcn.h>
#include <nccl.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace fmmgpu {

namespace {

template <typename T>
T* dev_alloc(size_t count) {
  T* p = nullptr;
  FMM_CUDA(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
  return p;
}

// ranks (bit mask) needing each leaf: its owner and the owners of its 26 neighbours
__global__ void k_leaf_need(const LevelView leaf, const uint32_t* __restrict__ pb, int nranks,
                            uint64_t* __restrict__ need) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= leaf.n) return;
  auto owner = [&](uint32_t q) {
    int lo = 0, hi = nranks - 1;  // last rank with pb[r] <= q
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pb[mid] <= q) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  int ijk[3];
  demorton(leaf.code[c], ijk);
  uint64_t m = 1ull << owner(c);
  for (int d = 0; d < 27; ++d) {
    if (d == 13) continue;
    const uint32_t q = find_ijk(leaf, ijk[0] + d / 9 - 1, ijk[1] + (d / 3) % 3 - 1, ijk[2] + d % 3 - 1);
    if (q != NPOS) m |= 1ull << owner(q);
  }
  need[c] = m;
}

// slot j is moved from the rank holding input index id[j] (input slice [s0, s1)) to rank
// `to` when `to` needs its leaf
struct SlotPred {
  const uint64_t* need;
  const uint32_t* pcell;
  const uint32_t* id;
  uint64_t s0, s1;
  int to;
  __device__ __forceinline__ bool operator()(const uint32_t j) const {
    const uint64_t i = id[j];
    return i >= s0 && i < s1 && ((need[pcell[j]] >> to) & 1ull);
  }
};

__global__ void k_pack_particles(const double4* __restrict__ loc, uint64_t offset, const uint32_t* __restrict__ id,
                                 const uint32_t* __restrict__ slots, uint32_t cnt, double4* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) out[i] = loc[id[slots[i]] - offset];
}
__global__ void k_unpack_particles(const double4* __restrict__ in, const uint32_t* __restrict__ slots, uint32_t cnt,
                                   double4* __restrict__ pw) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) pw[slots[i]] = in[i];
}
__global__ void k_self_particles(const double4* __restrict__ loc, uint64_t offset, const uint32_t* __restrict__ id,
                                 const uint32_t* __restrict__ slots, uint32_t cnt, double4* __restrict__ pw) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) {
    const uint32_t j = slots[i];
    pw[j] = loc[id[j] - offset];
  }
}

unsigned grid_of(uint64_t n) { return static_cast<unsigned>((n + 255) / 256); }

void need_dist(const fmmgpu_ctx* c) {
  if (!c->have_tree || !c->dist) throw Error(FMMGPU_LOGIC_ERROR, "no distributed tree: call fmmgpu_dist_build first");
}

// step 5: the per-peer slot lists (device) and their offsets (host)
void particle_plan(fmmgpu_ctx* c) {
  cudaStream_t s = c->s_far;
  const int nr = c->part_n, me = c->part_rank;
  const Level& L = c->lv[c->height - 1];
  const auto& pb = c->part_begin[c->height - 1];
  uint32_t* d_pb = dev_alloc<uint32_t>(nr + 1);
  FMM_CUDA(cudaMemcpyAsync(d_pb, pb.data(), (nr + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  uint64_t* need = dev_alloc<uint64_t>(L.n);
  k_leaf_need<<<grid_of(L.n), 256, 0, s>>>(L.view(c->height - 1), d_pb, nr, need);
  FMM_CUDA(cudaGetLastError());
  ++c->launches;
  // per peer p: send = {slots with id in my slice, leaf needed by p} (p == me: the local
  // copy), recv = {slots with id in p's slice, leaf needed by me} (p != me)
  uint32_t* tmp_out = dev_alloc<uint32_t>(c->n);
  uint32_t* d_cnt = dev_alloc<uint32_t>(1);
  size_t tb = 0;
  cub::CountingInputIterator<uint32_t> it(0);
  auto select = [&](const SlotPred& pr, std::vector<uint32_t>& dst_counts, std::vector<uint32_t*>& dst_lists) {
    FMM_CUDA(cub::DeviceSelect::If(nullptr, tb, it, tmp_out, d_cnt, static_cast<int>(c->n), pr, s));
    FMM_CUDA(cub::DeviceSelect::If(scratch(c, tb), tb, it, tmp_out, d_cnt, static_cast<int>(c->n), pr, s));
    const uint32_t k = *static_cast<const uint32_t*>(readback(c, d_cnt, 4, s));
    uint32_t* lst = dev_alloc<uint32_t>(k);
    if (k) FMM_CUDA(cudaMemcpyAsync(lst, tmp_out, k * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    dst_counts.push_back(k);
    dst_lists.push_back(lst);
  };
  std::vector<uint32_t> scnt, rcnt;
  std::vector<uint32_t*> slst, rlst;
  for (int p = 0; p < nr; ++p) {
    select(SlotPred{need, c->d_pcell, c->d_id, c->dist_off[me], c->dist_off[me + 1], p}, scnt, slst);
    if (p == me) {
      rcnt.push_back(0);
      rlst.push_back(nullptr);
    } else {
      select(SlotPred{need, c->d_pcell, c->d_id, c->dist_off[p], c->dist_off[p + 1], me}, rcnt, rlst);
    }
  }
  // concatenate per peer
  c->dsend_off.assign(1, 0);
  c->drecv_off.assign(1, 0);
  for (int p = 0; p < nr; ++p) {
    c->dsend_off.push_back(c->dsend_off.back() + scnt[p]);
    c->drecv_off.push_back(c->drecv_off.back() + rcnt[p]);
  }
  c->d_dsend = dev_alloc<uint32_t>(c->dsend_off.back());
  c->d_drecv = dev_alloc<uint32_t>(c->drecv_off.back());
  for (int p = 0; p < nr; ++p) {
    if (scnt[p])
      FMM_CUDA(cudaMemcpyAsync(c->d_dsend + c->dsend_off[p], slst[p], scnt[p] * 4, cudaMemcpyDeviceToDevice, s));
    if (rcnt[p])
      FMM_CUDA(cudaMemcpyAsync(c->d_drecv + c->drecv_off[p], rlst[p], rcnt[p] * 4, cudaMemcpyDeviceToDevice, s));
  }
  FMM_CUDA(cudaStreamSynchronize(s));
  for (auto* q : slst) cudaFree(q);
  for (auto* q : rlst)
    if (q) cudaFree(q);
  cudaFree(tmp_out);
  cudaFree(d_cnt);
  cudaFree(need);
  cudaFree(d_pb);
  // this rank's own records go straight into place
  const uint32_t so = c->dsend_off[me], sc = c->dsend_off[me + 1] - so;
  if (sc) {
    k_self_particles<<<grid_of(sc), 256, 0, s>>>(c->d_loc, c->dist_offset, c->d_id, c->d_dsend + so, sc, c->d_pw);
    FMM_CUDA(cudaGetLastError());
    ++c->launches;
  }
}

// NCCL (dlopen'ed by partition.cu) for fmmgpu_build_tree_distributed
struct NcclDist {
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};
NcclDist& ncd() {
  static NcclDist api;
  if (!api.groupStart) {
    void* h = open_nccl();  // partition.cu
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    if (!api.groupStart || !api.groupEnd || !api.broadcast || !api.send || !api.recv)
      throw Error(FMMGPU_RUNTIME_ERROR, "NCCL library lacks required symbols");
  }
  return api;
}
#define NCCLD(x)                                                                          \
  do {                                                                                    \
    if ((x) != ncclSuccess) throw Error(FMMGPU_RUNTIME_ERROR, "NCCL call failed: " #x);   \
  } while (0)

// in-place all-gather of per-rank segments [off[r], off[r + 1]) (elements of `bytes_each`
// bytes) of a device buffer: one broadcast per rank inside a group
void nccl_allgatherv(fmmgpu_ctx* c, void* buf, const std::vector<uint64_t>& off, size_t bytes_each) {
  auto& api = ncd();
  auto* comm = static_cast<ncclComm_t>(c->nccl);
  NCCLD(api.groupStart());
  for (int r = 0; r + 1 < static_cast<int>(off.size()); ++r) {
    const size_t cnt = (off[r + 1] - off[r]) * bytes_each;
    if (!cnt) continue;
    char* p = static_cast<char*>(buf) + off[r] * bytes_each;
    NCCLD(api.broadcast(p, p, cnt, ncclChar, r, comm, c->s_far));
  }
  NCCLD(api.groupEnd());
}

}  // namespace

void dist_free(fmmgpu_ctx* c) {
  if (c->d_dsend) cudaFree(c->d_dsend);
  if (c->d_drecv) cudaFree(c->d_drecv);
  c->d_dsend = c->d_drecv = nullptr;
  c->dsend_off.clear();
  c->drecv_off.clear();
  c->dist = false;
  c->dist_ready = true;
}

}  // namespace fmmgpu

using namespace fmmgpu;

namespace {
template <class F>
int guard(fmmgpu_ctx* c, F&& f) {
  try {
    if (!c) return FMMGPU_INVALID_ARGUMENT;
    FMM_CUDA(cudaSetDevice(c->device));
    f();
    return FMMGPU_OK;
  } catch (const Error& e) {
    c->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    c->err = e.what();
    return FMMGPU_RUNTIME_ERROR;
  }
}
}  // namespace

extern "C" {

int fmmgpu_root_from_bounds(const double* lohi6, double* root4) {
  if (!lohi6 || !root4) return FMMGPU_INVALID_ARGUMENT;
  for (int a = 0; a < 3; ++a)
    if (!(lohi6[a] <= lohi6[3 + a])) return FMMGPU_INVALID_ARGUMENT;  // empty set / NaN
  root_from_bounds(lohi6, lohi6 + 3, root4);
  return FMMGPU_OK;
}

int fmmgpu_dist_local(fmmgpu_ctx* c, const double* xyzw_local, uint64_t n_local, int on_device, double* lohi6) {
  return guard(c, [&] {
    if (n_local && !xyzw_local) throw Error(FMMGPU_INVALID_ARGUMENT, "dist_local: null particles");
    cudaStream_t s = c->s_far;
    if (c->d_loc_cap < n_local) {
      if (c->d_loc) FMM_CUDA(cudaFree(c->d_loc));
      FMM_CUDA(cudaMalloc(&c->d_loc, n_local * sizeof(double4)));
      c->d_loc_cap = n_local;
    }
    if (n_local)
      FMM_CUDA(cudaMemcpyAsync(c->d_loc, xyzw_local, n_local * sizeof(double4),
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    c->dist_nloc = n_local;
    double b[6];
    device_bounds(c, c->d_loc, n_local, b, s);
    if (lohi6) std::copy(b, b + 6, lohi6);
  });
}

int fmmgpu_dist_keys(fmmgpu_ctx* c, const double* root4, int height, uint64_t* keys_out, int out_on_device,
                     int* flag_out) {
  return guard(c, [&] {
    if (!root4 || !(root4[3] > 0)) throw Error(FMMGPU_INVALID_ARGUMENT, "dist_keys: root cube width must be positive");
    if (height < 3 || height > 21) throw Error(FMMGPU_INVALID_ARGUMENT, "GroupTree: height must be in [3, 21]");
    cudaStream_t s = c->s_far;
    const uint64_t n = c->dist_nloc;
    FMM_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), s));
    uint64_t* k = out_on_device ? keys_out : dev_alloc<uint64_t>(n);
    uint32_t* idx = dev_alloc<uint32_t>(n);
    device_keys(c->d_loc, n, root4, height, k, idx, c->d_flag, s);
    if (!out_on_device && n) FMM_CUDA(cudaMemcpyAsync(keys_out, k, n * 8, cudaMemcpyDeviceToHost, s));
    const int f = *static_cast<const int*>(readback(c, c->d_flag, sizeof(int), s));
    if (flag_out) *flag_out = f & 1;
    FMM_CUDA(cudaStreamSynchronize(s));
    if (!out_on_device) cudaFree(k);
    cudaFree(idx);
  });
}

int fmmgpu_dist_build(fmmgpu_ctx* c, const uint64_t* keys_all, int keys_on_device, const uint64_t* offsets,
                      int rank, int nranks, int height, int group, const double* root4, int flag) {
  return guard(c, [&] {
    if (!keys_all || !offsets || !root4) throw Error(FMMGPU_INVALID_ARGUMENT, "dist_build: null argument");
    if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks)
      throw Error(FMMGPU_INVALID_ARGUMENT, "bad rank / nranks (1 <= nranks <= 64)");
    const uint64_t n = offsets[nranks];
    if (offsets[0] != 0) throw Error(FMMGPU_INVALID_ARGUMENT, "dist_build: offsets must start at 0");
    for (int r = 0; r < nranks; ++r)
      if (offsets[r + 1] < offsets[r]) throw Error(FMMGPU_INVALID_ARGUMENT, "dist_build: offsets not ascending");
    if (offsets[rank + 1] - offsets[rank] != c->dist_nloc)
      throw Error(FMMGPU_INVALID_ARGUMENT, "dist_build: this rank's slice size differs from fmmgpu_dist_local");
    cudaStream_t s = c->s_far;
    const uint64_t* dk = keys_all;
    uint64_t* tmp = nullptr;
    if (!keys_on_device) {
      tmp = dev_alloc<uint64_t>(n);
      FMM_CUDA(cudaMemcpyAsync(tmp, keys_all, n * 8, cudaMemcpyHostToDevice, s));
      dk = tmp;
    }
    DistKeys dkeys{dk, flag};
    try {
      tree_build(c, nullptr, n, true, height, group, root4, &dkeys);
    } catch (...) {
      if (tmp) cudaFree(tmp);
      throw;
    }
    if (tmp) {
      FMM_CUDA(cudaStreamSynchronize(s));
      cudaFree(tmp);
    }
    c->dist_off.assign(offsets, offsets + nranks + 1);
    c->dist_offset = offsets[rank];
    c->dist_ntot = n;
    // the partition of the leaves (partition.cu) decides which particles this rank needs
    const int rc = fmmgpu_partition(c, rank, nranks);
    if (rc != FMMGPU_OK) throw Error(rc, c->err);
    particle_plan(c);
  });
}

int fmmgpu_dist_plan(fmmgpu_ctx* c, int peer, uint32_t* send_slots, uint32_t* send_count, uint32_t* recv_slots,
                     uint32_t* recv_count) {
  return guard(c, [&] {
    need_dist(c);
    if (peer < 0 || peer >= c->part_n || c->dsend_off.empty()) throw Error(FMMGPU_INVALID_ARGUMENT, "dist_plan: bad peer");
    const uint32_t so = c->dsend_off[peer], sc = c->dsend_off[peer + 1] - so;
    const uint32_t ro = c->drecv_off[peer], rc = c->drecv_off[peer + 1] - ro;
    if (send_count) *send_count = sc;
    if (recv_count) *recv_count = rc;
    if (send_slots && sc) FMM_CUDA(cudaMemcpy(send_slots, c->d_dsend + so, sc * 4, cudaMemcpyDeviceToHost));
    if (recv_slots && rc) FMM_CUDA(cudaMemcpy(recv_slots, c->d_drecv + ro, rc * 4, cudaMemcpyDeviceToHost));
  });
}

int fmmgpu_dist_pack(fmmgpu_ctx* c, int peer, double* out, int out_on_device) {
  return guard(c, [&] {
    need_dist(c);
    if (peer < 0 || peer >= c->part_n || peer == c->part_rank) throw Error(FMMGPU_INVALID_ARGUMENT, "dist_pack: bad peer");
    const uint32_t so = c->dsend_off[peer], sc = c->dsend_off[peer + 1] - so;
    if (!sc) return;
    cudaStream_t s = c->s_far;
    double4* d = out_on_device ? reinterpret_cast<double4*>(out) : dev_alloc<double4>(sc);
    k_pack_particles<<<grid_of(sc), 256, 0, s>>>(c->d_loc, c->dist_offset, c->d_id, c->d_dsend + so, sc, d);
    FMM_CUDA(cudaGetLastError());
    if (!out_on_device) {
      FMM_CUDA(cudaMemcpyAsync(out, d, sc * sizeof(double4), cudaMemcpyDeviceToHost, s));
      FMM_CUDA(cudaStreamSynchronize(s));
      cudaFree(d);
    }
  });
}

int fmmgpu_dist_unpack(fmmgpu_ctx* c, int peer, const double* in, int in_on_device) {
  return guard(c, [&] {
    need_dist(c);
    if (peer < 0 || peer >= c->part_n || peer == c->part_rank) throw Error(FMMGPU_INVALID_ARGUMENT, "dist_unpack: bad peer");
    const uint32_t ro = c->drecv_off[peer], rc = c->drecv_off[peer + 1] - ro;
    if (!rc) return;
    cudaStream_t s = c->s_far;
    const double4* d = reinterpret_cast<const double4*>(in);
    double4* tmp = nullptr;
    if (!in_on_device) {
      tmp = dev_alloc<double4>(rc);
      FMM_CUDA(cudaMemcpyAsync(tmp, in, rc * sizeof(double4), cudaMemcpyHostToDevice, s));
      d = tmp;
    }
    k_unpack_particles<<<grid_of(rc), 256, 0, s>>>(d, c->d_drecv + ro, rc, c->d_pw);
    FMM_CUDA(cudaGetLastError());
    if (tmp) {
      FMM_CUDA(cudaStreamSynchronize(s));
      cudaFree(tmp);
    }
  });
}

int fmmgpu_dist_check(fmmgpu_ctx* c, int* flag_out) {
  return guard(c, [&] {
    need_dist(c);
    const Level& L = c->lv[c->height - 1];
    const int f = coincident_check(c, L.own0, L.own1, c->s_far);
    if (flag_out) *flag_out = f & 2;
  });
}

int fmmgpu_dist_commit(fmmgpu_ctx* c, int flag) {
  return guard(c, [&] {
    need_dist(c);
    if (flag & 2) {
      tree_free(c);
      throw Error(FMMGPU_DOMAIN_ERROR, "GroupTree: coincident particles");
    }
    c->dist_ready = true;
  });
}

// Steps 1-7 with the attached NCCL communicator (fmmgpu_comm_init): every rank calls it
// with its own slice; slices are in rank order.
int fmmgpu_build_tree_distributed(fmmgpu_ctx* c, const double* xyzw_local, uint64_t n_local, int on_device,
                                  int height, int group, const double* root4) {
  return guard(c, [&] {
    if (!c->nccl) throw Error(FMMGPU_LOGIC_ERROR, "distributed build needs a communicator (fmmgpu_comm_init)");
    const int nr = c->comm_n, me = c->comm_rank;
    cudaStream_t s = c->s_far;
    // slice sizes and bounds of every rank (one all-gather of 8 doubles per rank)
    double lohi[6];
    int rc = fmmgpu_dist_local(c, xyzw_local, n_local, on_device, lohi);
    if (rc != FMMGPU_OK) throw Error(rc, c->err);
    double* d_meta = dev_alloc<double>(8 * nr);
    std::vector<double> meta(8 * nr, 0.0);
    std::copy(lohi, lohi + 6, meta.begin() + 8 * me);
    meta[8 * me + 6] = static_cast<double>(n_local);  // exact below 2^53
    FMM_CUDA(cudaMemcpyAsync(d_meta, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice, s));
    std::vector<uint64_t> roff(nr + 1);
    for (int r = 0; r <= nr; ++r) roff[r] = uint64_t(8) * r;
    nccl_allgatherv(c, d_meta, roff, sizeof(double));
    FMM_CUDA(cudaMemcpyAsync(meta.data(), d_meta, meta.size() * 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_meta);
    std::vector<uint64_t> off(nr + 1, 0);
    double g[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int r = 0; r < nr; ++r) {
      off[r + 1] = off[r] + static_cast<uint64_t>(meta[8 * r + 6]);
      for (int a = 0; a < 3; ++a) {
        g[a] = std::min(g[a], meta[8 * r + a]);
        g[3 + a] = std::max(g[3 + a], meta[8 * r + 3 + a]);
      }
    }
    if (off[nr] == 0) throw Error(FMMGPU_INVALID_ARGUMENT, "GroupTree: empty particle set");
    double root[4];
    if (root4) std::copy(root4, root4 + 4, root);
    else root_from_bounds(g, g + 3, root);
    // keys of every rank's slice, all-gathered in place (plus each rank's outside flag)
    uint64_t* keys = dev_alloc<uint64_t>(off[nr] + nr);
    int flag = 0;
    rc = fmmgpu_dist_keys(c, root, height, keys + off[me], 1, &flag);
    if (rc != FMMGPU_OK) throw Error(rc, c->err);
    nccl_allgatherv(c, keys, off, sizeof(uint64_t));
    // flags: one u64 per rank after the keys
    uint64_t fl = static_cast<uint64_t>(flag);
    FMM_CUDA(cudaMemcpyAsync(keys + off[nr] + me, &fl, 8, cudaMemcpyHostToDevice, s));
    std::vector<uint64_t> foff(nr + 1);
    for (int r = 0; r <= nr; ++r) foff[r] = off[nr] + r;
    nccl_allgatherv(c, keys, foff, sizeof(uint64_t));
    std::vector<uint64_t> flags(nr);
    FMM_CUDA(cudaMemcpyAsync(flags.data(), keys + off[nr], nr * 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    for (uint64_t f : flags) flag |= static_cast<int>(f);
    rc = fmmgpu_dist_build(c, keys, 1, off.data(), me, nr, height, group, root, flag);
    FMM_CUDA(cudaStreamSynchronize(s));
    cudaFree(keys);
    if (rc != FMMGPU_OK) throw Error(rc, c->err);
    // particle records of the owned + halo leaves, per peer
    const uint64_t nv = c->drecv_off.back();
    double4* sbuf = dev_alloc<double4>(c->dsend_off.back());
    double4* rbuf = dev_alloc<double4>(nv);
    for (int p = 0; p < nr; ++p) {
      const uint32_t so = c->dsend_off[p], sc = c->dsend_off[p + 1] - so;
      if (p == me || !sc) continue;
      k_pack_particles<<<grid_of(sc), 256, 0, s>>>(c->d_loc, c->dist_offset, c->d_id, c->d_dsend + so, sc, sbuf + so);
      FMM_CUDA(cudaGetLastError());
      ++c->launches;
    }
    auto& api = ncd();
    auto* comm = static_cast<ncclComm_t>(c->nccl);
    NCCLD(api.groupStart());
    for (int p = 0; p < nr; ++p) {
      if (p == me) continue;
      const uint32_t so = c->dsend_off[p], sc = c->dsend_off[p + 1] - so;
      const uint32_t ro = c->drecv_off[p], rcn = c->drecv_off[p + 1] - ro;
      if (sc) NCCLD(api.send(sbuf + so, size_t(sc) * 32, ncclChar, p, comm, s));
      if (rcn) NCCLD(api.recv(rbuf + ro, size_t(rcn) * 32, ncclChar, p, comm, s));
    }
    NCCLD(api.groupEnd());
    if (nv) {
      k_unpack_particles<<<grid_of(nv), 256, 0, s>>>(rbuf, c->d_drecv, static_cast<uint32_t>(nv), c->d_pw);
      FMM_CUDA(cudaGetLastError());
      ++c->launches;
    }
    FMM_CUDA(cudaStreamSynchronize(s));
    cudaFree(sbuf);
    cudaFree(rbuf);
    // coincident particles anywhere -> every rank raises
    int cf = 0;
    rc = fmmgpu_dist_check(c, &cf);
    if (rc != FMMGPU_OK) throw Error(rc, c->err);
    uint64_t* d_cf = dev_alloc<uint64_t>(nr);
    const uint64_t mine = static_cast<uint64_t>(cf);
    FMM_CUDA(cudaMemcpyAsync(d_cf + me, &mine, 8, cudaMemcpyHostToDevice, s));
    std::vector<uint64_t> one(nr + 1);
    for (int r = 0; r <= nr; ++r) one[r] = r;
    nccl_allgatherv(c, d_cf, one, sizeof(uint64_t));
    std::vector<uint64_t> cfs(nr);
    FMM_CUDA(cudaMemcpyAsync(cfs.data(), d_cf, nr * 8, cudaMemcpyDeviceToHost, s));
    FMM_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_cf);
    int all = 0;
    for (uint64_t f : cfs) all |= static_cast<int>(f);
    rc = fmmgpu_dist_commit(c, all);
    if (rc != FMMGPU_OK) throw Error(rc, c->err);
  });
}

}  // extern "C"
