// C ABI (include/fmmgpu.h): context lifetime, operator dispatch, the evaluation
// schedule, downloads for parity, timings and the flop ledger.
//
// The schedule replaces the reference's task DAG + worker pool (taskflow.cpp:143-289,
// runtime.cpp:91-216) by a fixed level-synchronous order on two CUDA streams:
//   s_far : P2M -> M2M(leaf-1..2) -> M2L(2..leaf) -> L2L(2..leaf-1) -> L2P
//   s_near: P2P (concurrent with the whole far chain; the paper's pipelining of
//           near and far field)
// joined before the gather that sums both and returns input order. Every output
// array has one writer per phase, so results are run-to-run bitwise reproducible
// (the reference's single-writer property, README.md:84-92).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

using namespace fmmgpu;

namespace {

thread_local std::string g_global_err;

template <typename F>
int guarded(fmmgpu_ctx* c, F&& f) {
  try {
    f();
    return FMMGPU_OK;
  } catch (const Error& e) {
    if (c) c->err = e.what();
    g_global_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    g_global_err = e.what();
    return FMMGPU_RUNTIME_ERROR;
  }
}

void reset_arrays(fmmgpu_ctx* c, cudaStream_t s);

// Every entry point that reads or accumulates into a tree's arrays: the arrays of a
// new tree start zeroed (GroupTree::allocate_*, geometry.cpp:199-214).
void need_tree(fmmgpu_ctx* c) {
  if (!c->have_tree) throw Error(FMMGPU_LOGIC_ERROR, "no tree: call fmmgpu_build_tree first");
  if (!c->dist_ready)
    throw Error(FMMGPU_LOGIC_ERROR, "distributed tree: particle exchange not committed (fmmgpu_dist_commit)");
  if (c->zero_pending) {
    reset_arrays(c, c->s_far);
    c->zero_pending = false;
  }
}
void need_level(fmmgpu_ctx* c, int v, int lo, int hi, const char* what) {
  need_tree(c);
  if (v < lo || v > hi) throw Error(FMMGPU_OUT_OF_RANGE, std::string(what) + ": level out of range");
}

__global__ void k_pad_copy(const double* __restrict__ src, int l3, int ldE, uint64_t cells, double* __restrict__ dst,
                           int to_padded) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= cells * l3) return;
  const uint64_t c = i / l3, k = i % l3;
  if (to_padded) dst[c * ldE + k] = src[i];
  else dst[i] = src[c * ldE + k];
}

__global__ void k_cells_aos(const uint64_t* code, const uint32_t* fp, const uint32_t* pc, const uint32_t* par,
                            const uint32_t* fc, const uint32_t* cc, uint32_t n, uint32_t* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t* o = out + 8ull * i;
  const uint64_t cd = code[i];
  o[0] = static_cast<uint32_t>(cd);
  o[1] = static_cast<uint32_t>(cd >> 32);
  o[2] = fp[i];
  o[3] = pc[i];
  o[4] = par[i];
  o[5] = fc[i];
  o[6] = cc[i];
  o[7] = 0;
}

__global__ void k_soa(const double4* pw, uint64_t n, double* x, double* y, double* z, double* w) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double4 p = pw[i];
  x[i] = p.x; y[i] = p.y; z[i] = p.z; w[i] = p.w;
}

// Morton-order AoS near + far -> SoA [4][n]
__global__ void k_sum4(const double4* a, const double4* b, uint64_t n, double* out) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double4 x = a[i], y = b[i];
  out[i] = x.x + y.x;
  out[n + i] = x.y + y.y;
  out[2 * n + i] = x.z + y.z;
  out[3 * n + i] = x.w + y.w;
}

void reset_arrays(fmmgpu_ctx* c, cudaStream_t s) {
  for (auto& L : c->lv) {
    const size_t e = size_t(L.n) * c->ldE * sizeof(double);
    FMM_CUDA(cudaMemsetAsync(L.multipole, 0, e, s));
    FMM_CUDA(cudaMemsetAsync(L.local_own, 0, e, s));
    FMM_CUDA(cudaMemsetAsync(L.local_down, 0, e, s));
  }
  FMM_CUDA(cudaMemsetAsync(c->d_near, 0, 32 * c->n, s));
  FMM_CUDA(cudaMemsetAsync(c->d_far, 0, 32 * c->n, s));
}

// Event pair -> ms; 0 for a pair that was never recorded (e.g. evaluation timings read
// before the first evaluation). The failed query's error is consumed here so it cannot
// surface at an unrelated cudaGetLastError later.
float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0.0f;
  }
  return ms;
}

// M2LOperatorSet::load_cache (m2l.cpp:247-288): the factors of the binary cache of
// (order, eps) into the context's operator set (its transport tables are rebuilt by
// m2l_setup).
void read_m2l_cache(fmmgpu_ctx* c, const char* path) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) throw Error(FMMGPU_RUNTIME_ERROR, std::string("cannot open M2L cache ") + path);
  uint64_t magic = 0;
  int32_t order = 0;
  double eps = 0;
  bool ok = std::fread(&magic, 8, 1, f) == 1 && std::fread(&order, 4, 1, f) == 1 && std::fread(&eps, 8, 1, f) == 1;
  if (!ok || magic != 0x4c324d4d4d465400ull || order != c->order || eps != c->eps) {
    std::fclose(f);
    throw Error(FMMGPU_INVALID_ARGUMENT, "M2L cache does not match (magic, order, eps)");
  }
  int32_t ranks[16];
  ok = std::fread(ranks, 4, 16, f) == 16;
  std::vector<double> u[16], sg[16], v[16];  // committed only when the whole file reads
  for (int cl = 0; cl < 16 && ok; ++cl) {
    if (ranks[cl] < 1 || ranks[cl] > c->l3) { ok = false; break; }
    u[cl].resize(size_t(c->l3) * ranks[cl]);
    sg[cl].resize(ranks[cl]);
    v[cl].resize(size_t(c->l3) * ranks[cl]);
    ok = ok && std::fread(u[cl].data(), 8, u[cl].size(), f) == u[cl].size();
    ok = ok && std::fread(sg[cl].data(), 8, sg[cl].size(), f) == sg[cl].size();
    ok = ok && std::fread(v[cl].data(), 8, v[cl].size(), f) == v[cl].size();
  }
  std::fclose(f);
  if (!ok) throw Error(FMMGPU_RUNTIME_ERROR, "truncated or corrupt M2L cache");
  auto& T = c->m2l;
  for (int cl = 0; cl < 16; ++cl) {
    T.rank[cl] = ranks[cl];
    T.u[cl] = std::move(u[cl]);
    T.sigma[cl] = std::move(sg[cl]);
    T.v[cl] = std::move(v[cl]);
  }
}

// InterpolationEngine + M2LOperatorSet of a new context (fmmgpu_create); `factors`
// (optional) supplies the compressed M2L operators instead of a new device SVD.
void ctx_init(fmmgpu_ctx* c, int device, int order, double eps, const fmmgpu_ctx* factors,
              const char* cache = nullptr) {
  if (order < 2 || order > MAX_ORDER) throw Error(FMMGPU_INVALID_ARGUMENT, "InterpolationEngine: order must be in [2, 10]");
  if (!(eps > 0)) throw Error(FMMGPU_INVALID_ARGUMENT, "M2LOperatorSet: eps must be positive");
  int ndev = 0;
  FMM_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) throw Error(FMMGPU_INVALID_ARGUMENT, "no such CUDA device");
  c->device = device;
  c->order = order;
  c->eps = eps;
  c->l3 = order * order * order;
  const char* ge = std::getenv("FMMGPU_GRAPH");
  c->use_graph = ge && std::atoi(ge) == 1;
  c->ldE = round_up(c->l3, 32);  // multiple of the GEMM k-slice (32)
  FMM_CUDA(cudaSetDevice(device));
  cudaMemPool_t pool;
  FMM_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  FMM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  // The far-field chain gets the higher priority: its coarse levels cannot fill the
  // GPU, so P2P CTAs (lower priority, concurrent stream) fill the idle SMs instead of
  // the chain queueing behind 32k P2P CTAs.
  int prio_lo = 0, prio_hi = 0;
  FMM_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  FMM_CUDA(cudaStreamCreateWithPriority(&c->s_far, cudaStreamNonBlocking, prio_hi));
  FMM_CUDA(cudaStreamCreateWithPriority(&c->s_near, cudaStreamNonBlocking, prio_lo));
  FMM_CUDA(cudaStreamCreateWithPriority(&c->s_aux, cudaStreamNonBlocking, prio_hi));
  FMM_CUDA(cudaEventCreateWithFlags(&c->ev_up, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&c->ev_aux, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&c->ev_p2p_main, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  FMM_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  for (auto& e : c->ev_t) FMM_CUDA(cudaEventCreate(&e));
  FMM_CUDA(cudaMalloc(&c->d_flag, sizeof(int)));
  FMM_CUDA(cudaMalloc(&c->d_ctr, 256));
  {  // FMMGPU_P2P_ONESIDED=1: new contexts start with the one-sided kernel (fmmgpu_set_p2p_mode)
    const char* pe = std::getenv("FMMGPU_P2P_ONESIDED");
    c->p2p_mode = (pe && std::atoi(pe) == 1) ? 0 : 2;
  }
  interp_setup(c);
  if (factors) {  // share the operators of an existing context (no second SVD)
    auto& T = c->m2l;
    const auto& F = factors->m2l;
    for (int cl = 0; cl < 16; ++cl) {
      T.rank[cl] = F.rank[cl];
      T.u[cl] = F.u[cl];
      T.v[cl] = F.v[cl];
      T.sigma[cl] = F.sigma[cl];
    }
    m2l_setup(c, false);
  } else if (cache) {  // the factors of a saved operator set: no SVD
    read_m2l_cache(c, cache);
    m2l_setup(c, false);
  } else {
    m2l_setup(c, true);
  }
}

}  // namespace

extern "C" {

const char* fmmgpu_global_error(void) { return g_global_err.c_str(); }
const char* fmmgpu_last_error(const fmmgpu_ctx* c) { return c ? c->err.c_str() : g_global_err.c_str(); }

int fmmgpu_create(int device, int order, double eps, fmmgpu_ctx** out) {
  if (!out) return FMMGPU_INVALID_ARGUMENT;
  *out = nullptr;
  auto* c = new fmmgpu_ctx;
  const int rc = guarded(c, [&] { ctx_init(c, device, order, eps, nullptr); });
  if (rc != FMMGPU_OK) {
    g_global_err = c->err;
    fmmgpu_destroy(c);
    return rc;
  }
  *out = c;
  return FMMGPU_OK;
}

int fmmgpu_create_from_cache(int device, int order, double eps, const char* path, fmmgpu_ctx** out) {
  if (!out || !path) return FMMGPU_INVALID_ARGUMENT;
  *out = nullptr;
  auto* c = new fmmgpu_ctx;
  const int rc = guarded(c, [&] { ctx_init(c, device, order, eps, nullptr, path); });
  if (rc != FMMGPU_OK) {
    g_global_err = c->err;
    fmmgpu_destroy(c);
    return rc;
  }
  *out = c;
  return FMMGPU_OK;
}

void fmmgpu_destroy(fmmgpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->s_h2d) {  // pipelined runs
    cudaStreamSynchronize(c->s_h2d);
    cudaStreamSynchronize(c->s_d2h);
    for (auto p : c->pipe_out)
      if (p) cudaFree(p);
    cudaEventDestroy(c->ev_in_free);
    cudaEventDestroy(c->ev_in_ready);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(c->ev_out_ready[i]);
      cudaEventDestroy(c->ev_d2h_done[i]);
    }
    cudaStreamDestroy(c->s_h2d);
    cudaStreamDestroy(c->s_d2h);
  }
  if (c->s_far) {
    cudaStreamSynchronize(c->s_far);
    cudaStreamSynchronize(c->s_near);
    try {
      partition_free(c);
      lists_free(c);
      tree_free(c);
      yt_keep_free(c);
      cache_trim(c, c->s_far);
    } catch (...) {
    }
    if (c->d_in) cudaFreeAsync(c->d_in, c->s_far);
    if (c->d_tmp) cudaFreeAsync(c->d_tmp, c->s_far);
    if (c->d_loc) cudaFree(c->d_loc);  // distributed input slice (dist.cu)
    cudaStreamSynchronize(c->s_far);
  }
  m2l_free(c);
  fmmgpu_invalidate_graph(c);
  for (auto* p : c->d_splitk)
    if (p) cudaFree(p);
  if (c->nccl) fmmgpu_comm_destroy(c);
  if (c->d_interp) cudaFree(c->d_interp);
  if (c->d_flag) cudaFree(c->d_flag);
  if (c->d_ctr) cudaFree(c->d_ctr);
  if (c->d_canon) cudaFree(c->d_canon);
  if (c->h_rb) cudaFreeHost(c->h_rb);
  for (auto e : c->tr_ev) cudaEventDestroy(e);
  for (auto& e : c->ev_t)
    if (e) cudaEventDestroy(e);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->s_far) cudaStreamDestroy(c->s_far);
  if (c->s_near) cudaStreamDestroy(c->s_near);
  if (c->s_aux) cudaStreamDestroy(c->s_aux);
  if (c->ev_up) cudaEventDestroy(c->ev_up);
  if (c->ev_aux) cudaEventDestroy(c->ev_aux);
  if (c->ev_p2p_main) cudaEventDestroy(c->ev_p2p_main);
  delete c;
}

int fmmgpu_load_m2l_cache(fmmgpu_ctx* c, const char* path) {
  return guarded(c, [&] {
    read_m2l_cache(c, path);
    m2l_setup(c, false);
  });
}

int fmmgpu_save_m2l_cache(const fmmgpu_ctx* cc, const char* path) {
  auto* c = const_cast<fmmgpu_ctx*>(cc);
  return guarded(c, [&] {
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw Error(FMMGPU_RUNTIME_ERROR, std::string("cannot write ") + path);
    const uint64_t magic = 0x4c324d4d4d465400ull;
    const int32_t order = c->order;
    bool ok = std::fwrite(&magic, 8, 1, f) == 1 && std::fwrite(&order, 4, 1, f) == 1 && std::fwrite(&c->eps, 8, 1, f) == 1;
    const auto& T = c->m2l;
    for (int cl = 0; cl < 16; ++cl) {
      const int32_t r = T.rank[cl];
      ok = ok && std::fwrite(&r, 4, 1, f) == 1;
    }
    for (int cl = 0; cl < 16; ++cl) {
      ok = ok && std::fwrite(T.u[cl].data(), 8, T.u[cl].size(), f) == T.u[cl].size();
      ok = ok && std::fwrite(T.sigma[cl].data(), 8, T.sigma[cl].size(), f) == T.sigma[cl].size();
      ok = ok && std::fwrite(T.v[cl].data(), 8, T.v[cl].size(), f) == T.v[cl].size();
    }
    std::fclose(f);
    if (!ok) throw Error(FMMGPU_RUNTIME_ERROR, "write failed");
  });
}

int fmmgpu_m2l_report(const fmmgpu_ctx* c, int32_t* ranks16, int32_t* mult16, double* wmean) {
  if (!c) return FMMGPU_INVALID_ARGUMENT;
  double acc = 0;
  for (int cl = 0; cl < 16; ++cl) {
    if (ranks16) ranks16[cl] = c->m2l.rank[cl];
    if (mult16) mult16[cl] = c->m2l.mult[cl];
    acc += double(c->m2l.mult[cl]) * c->m2l.rank[cl];
  }
  if (wmean) *wmean = acc / 316.0;  // m2l.cpp:159-162
  return FMMGPU_OK;
}

int fmmgpu_build_tree(fmmgpu_ctx* c, const double* xyzw, uint64_t n, int on_device, int height, int group,
                      const double* root4) {
  return guarded(c, [&] {
    FMM_CUDA(cudaSetDevice(c->device));
    FMM_CUDA(cudaEventRecord(c->ev_t[14], c->s_far));
    c->out_valid = false;
    tree_build(c, xyzw, n, on_device != 0, height, group, root4);
    FMM_CUDA(cudaEventRecord(c->ev_t[15], c->s_far));
    FMM_CUDA(cudaEventSynchronize(c->ev_t[15]));
    c->timings[8] = elapsed(c->ev_t[14], c->ev_t[15]);
  });
}

int fmmgpu_build_lists(fmmgpu_ctx* c) {
  return guarded(c, [&] {
    need_tree(c);
    FMM_CUDA(cudaEventRecord(c->ev_t[14], c->s_far));
    lists_build(c);
    FMM_CUDA(cudaEventRecord(c->ev_t[15], c->s_far));
    FMM_CUDA(cudaEventSynchronize(c->ev_t[15]));
    c->timings[9] = elapsed(c->ev_t[14], c->ev_t[15]);
  });
}

int fmmgpu_reset(fmmgpu_ctx* c) {
  return guarded(c, [&] {
    need_tree(c);
    c->out_valid = false;
    reset_arrays(c, c->s_far);
  });
}
int fmmgpu_p2m(fmmgpu_ctx* c) {
  return guarded(c, [&] {
    need_tree(c);
    c->out_valid = false;
    launch_p2m(c, c->s_far);
  });
}
int fmmgpu_m2m(fmmgpu_ctx* c, int v) {
  return guarded(c, [&] {
    need_level(c, v, 2, c->height - 2, "m2m");  // parent levels 2..leaf-1 (taskflow.cpp:190-199)
    launch_m2m(c, v, c->s_far);
  });
}
int fmmgpu_m2l(fmmgpu_ctx* c, int v) {
  return guarded(c, [&] {
    need_level(c, v, 2, c->height - 1, "m2l");
    launch_m2l(c, v, c->s_far);
  });
}
int fmmgpu_l2l(fmmgpu_ctx* c, int v) {
  return guarded(c, [&] {
    need_level(c, v, 2, c->height - 2, "l2l");
    launch_l2l(c, v, c->s_far);
  });
}
int fmmgpu_l2p(fmmgpu_ctx* c) {
  return guarded(c, [&] {
    need_tree(c);
    c->out_valid = false;
    launch_l2p(c, c->s_far);
  });
}
int fmmgpu_p2p(fmmgpu_ctx* c) {
  return guarded(c, [&] {
    need_tree(c);
    c->out_valid = false;
    launch_p2p(c, c->s_far);
  });
}

}  // extern "C"

namespace {

// Timing events must stay visible outside a captured graph (cudaEventRecordExternal).
void record(fmmgpu_ctx* c, cudaEvent_t e, cudaStream_t s) {
  if (c->capturing) FMM_CUDA(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
  else FMM_CUDA(cudaEventRecord(e, s));
}

// One evaluation: the DAG as a level-synchronous two-stream schedule (unpartitioned:
// every operator writes its output once; partitioned: clear, then accumulate).
// trace span around one launch (eager evaluations with tracing on)
struct Span {
  fmmgpu_ctx* c;
  size_t i = 0;
  Span(fmmgpu_ctx* cc, int kind, int level, cudaStream_t st, int stream_id) : c(cc) {
    if (!c->trace) return;
    i = c->tr_ev.size();
    for (int k = 0; k < 2; ++k) {
      cudaEvent_t e;
      FMM_CUDA(cudaEventCreate(&e));
      c->tr_ev.push_back(e);
    }
    c->tr_meta.insert(c->tr_meta.end(), {kind, level, stream_id});
    FMM_CUDA(cudaEventRecord(c->tr_ev[i], st));
    this->st = st;
  }
  ~Span() {
    if (c->trace) cudaEventRecord(c->tr_ev[i + 1], st);
  }
  cudaStream_t st = nullptr;
};

void trace_clear(fmmgpu_ctx* c) {
  for (auto e : c->tr_ev) cudaEventDestroy(e);
  c->tr_ev.clear();
  c->tr_meta.clear();
}

void enqueue_evaluation(fmmgpu_ctx* c) {
  const int leaf = c->height - 1;
  cudaStream_t s = c->s_far;
  c->launches = 0;
  if (c->trace) trace_clear(c);
  cudaEvent_t* e = c->ev_t;
  record(c, e[0], s);
  struct OwReset {  // per-operator calls after this evaluation (or after an error) accumulate
    fmmgpu_ctx* c;
    ~OwReset() { c->ow = false; }
  } ow_reset{c};
  c->ow = c->part_n == 1;
  if (c->ow) {  // only level 2's local_down is read without being written (L2L's first parent
    // level); levels 0 and 1 (<= 9 cells) are never touched by an evaluation and read as zero
    // like the reference's (GroupTree::allocate_expansions, geometry.cpp:199-206)
    for (int v = 0; v <= std::min(2, c->height - 1); ++v) {
      const Level& L = c->lv[v];
      const size_t e = size_t(L.n) * c->ldE * sizeof(double);
      if (v < 2) {
        FMM_CUDA(cudaMemsetAsync(L.multipole, 0, e, s));
        FMM_CUDA(cudaMemsetAsync(L.local_own, 0, e, s));
      }
      FMM_CUDA(cudaMemsetAsync(L.local_down, 0, e, s));
    }
  } else {
    reset_arrays(c, s);
  }
  FMM_CUDA(cudaEventRecord(c->ev_fork, s));
  FMM_CUDA(cudaStreamWaitEvent(c->s_near, c->ev_fork, 0));
  // mutual near field: its ordered slot drain (p2p_reduce) is fused into L2P, which waits
  // for the near-field kernel (the drain's HBM pass then overlaps L2P's arithmetic)
  static const int fuse_env = [] {  // FMMGPU_FUSE_DRAIN=0: separate drain kernel (A/B aid)
    const char* v = std::getenv("FMMGPU_FUSE_DRAIN");
    return v ? std::atoi(v) : 1;
  }();
  const Level& LL = c->lv[leaf];
  const bool fuse = fuse_env != 0 && p2p_use_mutual(c, LL.own1 - LL.own0);
  record(c, e[6], c->s_near);
  {
    Span sp(c, FMMGPU_P2P, leaf, c->s_near, 1);
    launch_p2p(c, c->s_near, fuse);
  }
  record(c, e[7], c->s_near);
  record(c, e[1], s);
  {
    Span sp(c, FMMGPU_P2M, leaf, s, 0);
    launch_p2m(c, s);
  }
  exchange_level(c, leaf, s);  // partitioned runs: all-gather this level's multipoles
  record(c, e[2], s);
  for (int v = leaf - 1; v >= 2; --v) {
    {
      Span sp(c, FMMGPU_M2M, v, s, 0);
      launch_m2m(c, v, s);
    }
    exchange_level(c, v, s);
  }
  record(c, e[3], s);
  // Measured (tools/gpu/gpu_r02af.sh, ms per evaluation single stream / aux stream): A 0.97 /
  // 0.99, B 24.54 / 24.62, C 80.18 / 79.61, E 240.54 / 240.73; a config-B rank of 8
  // (partitioned, tools/gpu/gpu_r02ak.sh) 4.28 / 3.94 -- used above order 5 and for
  // partitioned evaluations, whose small per-rank levels are latency-bound.
  static const int aux_env = [] {  // FMMGPU_AUX=0/1 forces it (A/B aid)
    const char* v = std::getenv("FMMGPU_AUX");
    return v ? std::atoi(v) : -1;
  }();
  const bool aux = aux_env >= 0 ? aux_env != 0 : (c->ldE > 128 || c->part_n > 1);
  if (aux && leaf > 2) {
    // M2L of every level reads only that level's multipoles, complete after the upward
    // pass, so the coarse levels' M2L and the L2L chain (which needs local(v) = own + down
    // of the coarse levels only) run on a second high-priority stream beside the leaf M2L;
    // L2P waits for both. The small, latency-bound coarse launches then overlap the leaf
    // M2L instead of running alone.
    FMM_CUDA(cudaEventRecord(c->ev_up, s));
    FMM_CUDA(cudaStreamWaitEvent(c->s_aux, c->ev_up, 0));
    {
      Span sp(c, FMMGPU_M2L, leaf, s, 0);
      launch_m2l(c, leaf, s);
    }
    for (int v = 2; v < leaf; ++v) {
      Span sp(c, FMMGPU_M2L, v, c->s_aux, 2);
      launch_m2l(c, v, c->s_aux);
    }
    for (int v = 2; v < leaf; ++v) {
      Span sp(c, FMMGPU_L2L, v, c->s_aux, 2);
      launch_l2l(c, v, c->s_aux);
    }
    record(c, e[4], s);
    FMM_CUDA(cudaEventRecord(c->ev_aux, c->s_aux));
    FMM_CUDA(cudaStreamWaitEvent(s, c->ev_aux, 0));
  } else {
    for (int v = 2; v <= leaf; ++v) {
      Span sp(c, FMMGPU_M2L, v, s, 0);
      launch_m2l(c, v, s);
    }
    record(c, e[4], s);
    for (int v = 2; v < leaf; ++v) {
      Span sp(c, FMMGPU_L2L, v, s, 0);
      launch_l2l(c, v, s);
    }
  }
  record(c, e[5], s);
  if (fuse) FMM_CUDA(cudaStreamWaitEvent(s, c->ev_p2p_main, 0));
  {
    Span sp(c, FMMGPU_L2P, leaf, s, 0);
    launch_l2p(c, s, fuse);
  }
  record(c, e[8], s);
  FMM_CUDA(cudaEventRecord(c->ev_join, c->s_near));
  FMM_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
  record(c, e[9], s);
  {
    Span sp(c, FMMGPU_P2PREDUCE, leaf, s, 0);  // the gather of near + far (P2PReduce's role)
    launch_gather(c, s);
  }
  record(c, e[10], s);
}

}  // namespace

extern "C" {

// With fmmgpu_set_graph(ctx, 1) (or FMMGPU_GRAPH=1 for new contexts) the evaluation's ~25 launches are captured once into a CUDA graph
// (after one eager run, so every lazy allocation has happened) and replayed while the
// tree, partition and operators are unchanged (the stream/event
// schedule as a graph). Off by default: at config B the replayed graph measured 27.20
// ms per evaluation against 26.89 ms for eager launches on the two prioritised streams
// (setting the kernel nodes' priorities after capture did not close the gap), and the
// host launch cost of ~25 kernels hides under a 27 ms evaluation anyway. Partitioned
// runs with an NCCL communicator are always eager.
int fmmgpu_evaluate(fmmgpu_ctx* c) {
  return guarded(c, [&] {
    c->zero_pending = false;  // the evaluation clears its arrays itself
    need_tree(c);
    FMM_CUDA(cudaSetDevice(c->device));
    const bool graphable = c->use_graph && !(c->part_n > 1 && c->nccl) && !c->trace;
    if (graphable && c->graph_exec) {
      FMM_CUDA(cudaGraphLaunch(c->graph_exec, c->s_far));
      c->launches = c->graph_launches;
      c->out_valid = true;
      return;
    }
    enqueue_evaluation(c);
    c->out_valid = true;
    if (!graphable || !c->graph_warm) {  // first run eager: lazy allocations happen here
      c->graph_warm = graphable;
      return;
    }
    cudaGraph_t g = nullptr;
    FMM_CUDA(cudaStreamBeginCapture(c->s_far, cudaStreamCaptureModeRelaxed));
    c->capturing = true;
    try {
      enqueue_evaluation(c);
    } catch (...) {
      c->capturing = false;
      cudaStreamEndCapture(c->s_far, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    c->capturing = false;
    FMM_CUDA(cudaStreamEndCapture(c->s_far, &g));
    FMM_CUDA(cudaGraphInstantiate(&c->graph_exec, g, 0));
    FMM_CUDA(cudaGraphDestroy(g));
    c->graph_launches = c->launches;
  });
}

void fmmgpu_invalidate_graph(fmmgpu_ctx* c) {
  if (!c) return;
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  c->graph_exec = nullptr;
  c->graph_warm = false;
}

// Stepped evaluation for a host-driven exchange (partitioned runs without an attached
// communicator): fmmgpu_reset, then fmmgpu_upward_level(leaf .. 2) with the host
// all-gathering each level >= the alignment level between calls, then fmmgpu_downward.
int fmmgpu_upward_level(fmmgpu_ctx* c, int v) {
  return guarded(c, [&] {
    need_level(c, v, 2, c->height - 1, "upward_level");
    c->out_valid = false;
    if (v == c->height - 1) launch_p2m(c, c->s_far);
    else launch_m2m(c, v, c->s_far);
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

int fmmgpu_downward(fmmgpu_ctx* c) {
  return guarded(c, [&] {
    need_tree(c);
    const int leaf = c->height - 1;
    cudaStream_t s = c->s_far;
    FMM_CUDA(cudaEventRecord(c->ev_fork, s));
    FMM_CUDA(cudaStreamWaitEvent(c->s_near, c->ev_fork, 0));
    launch_p2p(c, c->s_near);
    for (int v = 2; v <= leaf; ++v) launch_m2l(c, v, s);
    for (int v = 2; v < leaf; ++v) launch_l2l(c, v, s);
    launch_l2p(c, s);
    FMM_CUDA(cudaEventRecord(c->ev_join, c->s_near));
    FMM_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
    launch_gather(c, s);
    c->out_valid = true;
    FMM_CUDA(cudaStreamSynchronize(s));
  });
}

int fmmgpu_synchronize(fmmgpu_ctx* c) {
  return guarded(c, [&] {
    FMM_CUDA(cudaStreamSynchronize(c->s_near));
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

int fmmgpu_timings(const fmmgpu_ctx* cc, double* ms) {
  auto* c = const_cast<fmmgpu_ctx*>(cc);
  return guarded(c, [&] {
    if (cudaEventSynchronize(c->ev_t[10]) != cudaSuccess) (void)cudaGetLastError();  // no evaluation yet
    cudaEvent_t* e = c->ev_t;
    ms[FMMGPU_P2M] = elapsed(e[1], e[2]);
    ms[FMMGPU_M2M] = elapsed(e[2], e[3]);
    ms[FMMGPU_M2L] = elapsed(e[3], e[4]);
    ms[FMMGPU_L2L] = elapsed(e[4], e[5]);
    ms[FMMGPU_L2P] = elapsed(e[5], e[8]);
    ms[FMMGPU_P2P] = elapsed(e[6], e[7]);
    ms[FMMGPU_P2PREDUCE] = elapsed(e[9], e[10]);
    ms[7] = elapsed(e[0], e[10]);
    ms[8] = c->timings[8];
    ms[9] = c->timings[9];
  });
}

uint64_t fmmgpu_last_launch_count(const fmmgpu_ctx* c) { return c ? c->launches : 0; }

int fmmgpu_set_graph(fmmgpu_ctx* c, int on) {
  return guarded(c, [&] {
    c->use_graph = on != 0;
    fmmgpu_invalidate_graph(c);
  });
}

int fmmgpu_set_p2p_mode(fmmgpu_ctx* c, int mutual) {
  return guarded(c, [&] {
    if (mutual < 0 || mutual > 2) throw Error(FMMGPU_INVALID_ARGUMENT, "set_p2p_mode: mode must be 0, 1 or 2");
    c->p2p_mode = mutual;
    fmmgpu_invalidate_graph(c);
    ensure_p2p_slots(c);
  });
}

int fmmgpu_p2p_kernel(const fmmgpu_ctx* c) {
  if (!c || !c->have_tree) return -1;
  const Level& L = c->lv[c->height - 1];
  return p2p_use_mutual(c, L.own1 - L.own0) ? 1 : 0;
}

int fmmgpu_set_trace(fmmgpu_ctx* c, int on) {
  return guarded(c, [&] {
    c->trace = on != 0;
    fmmgpu_invalidate_graph(c);
    if (!c->trace) trace_clear(c);
  });
}

int fmmgpu_trace_spans(fmmgpu_ctx* c, int cap, int* count, int* meta3, double* start_end_ms) {
  return guarded(c, [&] {
    const int nsp = static_cast<int>(c->tr_ev.size() / 2);
    if (count) *count = nsp;
    if (nsp == 0 || cap <= 0) return;
    FMM_CUDA(cudaEventSynchronize(c->tr_ev.back()));
    for (int i = 0; i < std::min(nsp, cap); ++i) {
      if (meta3) std::copy(c->tr_meta.begin() + 3 * i, c->tr_meta.begin() + 3 * i + 3, meta3 + 3 * i);
      if (start_end_ms) {
        start_end_ms[2 * i] = elapsed(c->tr_ev[0], c->tr_ev[2 * i]);
        start_end_ms[2 * i + 1] = elapsed(c->tr_ev[0], c->tr_ev[2 * i + 1]);
      }
    }
  });
}

int fmmgpu_time_evaluations(fmmgpu_ctx* c, int steps, double* total_ms, double* kind_ms10, uint64_t* launches) {
  return guarded(c, [&] {
    need_tree(c);
    if (steps < 1) throw Error(FMMGPU_INVALID_ARGUMENT, "steps must be >= 1");
    double acc[10] = {};
    uint64_t nl = 0;
    FMM_CUDA(cudaStreamSynchronize(c->s_near));
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
    FMM_CUDA(cudaEventRecord(c->ev_t[12], c->s_far));
    for (int i = 0; i < steps; ++i) {
      if (fmmgpu_evaluate(c) != FMMGPU_OK) throw Error(FMMGPU_RUNTIME_ERROR, c->err);
      nl += c->launches;
      double ms[10];
      if (fmmgpu_timings(c, ms) != FMMGPU_OK) throw Error(FMMGPU_RUNTIME_ERROR, c->err);
      for (int k = 0; k < 8; ++k) acc[k] += ms[k];
    }
    FMM_CUDA(cudaEventRecord(c->ev_t[13], c->s_far));
    FMM_CUDA(cudaEventSynchronize(c->ev_t[13]));
    if (total_ms) *total_ms = elapsed(c->ev_t[12], c->ev_t[13]);
    if (kind_ms10) {
      for (int k = 0; k < 8; ++k) kind_ms10[k] = acc[k];
      kind_ms10[8] = c->timings[8];
      kind_ms10[9] = c->timings[9];
    }
    if (launches) *launches = nl;
  });
}

int fmmgpu_time_operator(fmmgpu_ctx* c, int kind, int level, int reps, double* ms) {
  return guarded(c, [&] {
    need_tree(c);
    if (reps < 1 || !ms) throw Error(FMMGPU_INVALID_ARGUMENT, "reps must be >= 1 and ms non-null");
    const int leaf = c->height - 1;
    auto levels = [&](int lo, int hi) {
      if (level >= 0) {
        need_level(c, level, lo, hi, "time_operator");
        return std::vector<int>{level};
      }
      std::vector<int> v;
      for (int i = lo; i <= hi; ++i) v.push_back(i);
      return v;
    };
    std::vector<int> lv;
    switch (kind) {
      case FMMGPU_M2M: case FMMGPU_L2L: lv = levels(2, leaf - 1); break;
      case FMMGPU_M2L: lv = levels(2, leaf); break;
      case FMMGPU_P2M: case FMMGPU_L2P: case FMMGPU_P2P: lv = {leaf}; break;
      default: throw Error(FMMGPU_INVALID_ARGUMENT, "time_operator: kind must be P2M..P2P");
    }
    cudaStream_t s = c->s_far;
    FMM_CUDA(cudaStreamSynchronize(c->s_near));
    FMM_CUDA(cudaStreamSynchronize(s));
    c->out_valid = false;
    FMM_CUDA(cudaEventRecord(c->ev_t[12], s));
    for (int r = 0; r < reps; ++r)
      for (int v : lv) {
        switch (kind) {
          case FMMGPU_P2M: launch_p2m(c, s); break;
          case FMMGPU_M2M: launch_m2m(c, v, s); break;
          case FMMGPU_M2L: launch_m2l(c, v, s); break;
          case FMMGPU_L2L: launch_l2l(c, v, s); break;
          case FMMGPU_L2P: launch_l2p(c, s); break;
          case FMMGPU_P2P: launch_p2p(c, s); break;
        }
      }
    FMM_CUDA(cudaEventRecord(c->ev_t[13], s));
    FMM_CUDA(cudaEventSynchronize(c->ev_t[13]));
    *ms = elapsed(c->ev_t[12], c->ev_t[13]) / reps;
  });
}

int fmmgpu_download_fields(fmmgpu_ctx* c, double* pot, double* fx, double* fy, double* fz, int dst_on_device) {
  return guarded(c, [&] {
    need_tree(c);
    if (c->skip_exchange && c->part_n > 1)
      throw Error(FMMGPU_LOGIC_ERROR, "measurement mode (fmmgpu_set_measurement): partitioned evaluations skip the "
                                      "exchange and their fields are not valid");
    if (!c->out_valid) {  // per-operator use: gather near + far now
      FMM_CUDA(cudaEventRecord(c->ev_join, c->s_near));
      FMM_CUDA(cudaStreamWaitEvent(c->s_far, c->ev_join, 0));
      launch_gather(c, c->s_far);
      c->out_valid = true;
    }
    const cudaMemcpyKind k = dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    double* dst[4] = {pot, fx, fy, fz};
    for (int i = 0; i < 4; ++i)
      if (dst[i]) FMM_CUDA(cudaMemcpyAsync(dst[i], c->d_out + i * c->n, 8 * c->n, k, c->s_far));
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

int fmmgpu_run(fmmgpu_ctx* c, const double* xyzw, uint64_t n, int height, int group, double* pot, double* fx,
               double* fy, double* fz) {
  int rc = fmmgpu_build_tree(c, xyzw, n, 0, height, group, nullptr);
  if (rc) return rc;
  rc = fmmgpu_evaluate(c);
  if (rc) return rc;
  return fmmgpu_download_fields(c, pot, fx, fy, fz, 0);
}

namespace {
// FMMGPU_TRACE=1: timeline of pipelined runs (events per step, printed by run_wait)
std::vector<std::pair<std::string, cudaEvent_t>> g_pipe_trace;
void pipe_mark(const char* what, uint64_t k, cudaStream_t s) {
  static const bool on = std::getenv("FMMGPU_TRACE") != nullptr;
  if (!on) return;
  cudaEvent_t e;
  FMM_CUDA(cudaEventCreate(&e));
  FMM_CUDA(cudaEventRecord(e, s));
  g_pipe_trace.emplace_back(std::string(what) + " " + std::to_string(k), e);
}
void pipe_trace_dump() {
  if (g_pipe_trace.empty()) return;
  for (auto& [what, e] : g_pipe_trace) {
    float ms = 0;
    cudaEventElapsedTime(&ms, g_pipe_trace.front().second, e);
    std::fprintf(stderr, "[pipe] %9.3f ms  %s\n", ms, what.c_str());
  }
  for (auto& pe : g_pipe_trace) cudaEventDestroy(pe.second);
  g_pipe_trace.clear();
}
}  // namespace

// Pipelined run_fmm over a stream of particle sets. Step k's H2D runs on its own copy
// stream as soon as tree build k-1 has finished reading the input buffer, i.e. under
// evaluation k-1; step k's fields are gathered into one of two pipeline buffers and
// copied back on a second copy stream under tree build + evaluation k+1. The device
// work of one step is unchanged (tree build, evaluate, gather); only the PCIe copies
// leave the critical path.
namespace {
// Issue the deferred D2H of the last enqueued step (if any).
void pipe_issue_d2h(fmmgpu_ctx* c) {
  if (!c->pipe_pend) return;
  const int slot = c->pend_slot;
  FMM_CUDA(cudaStreamWaitEvent(c->s_d2h, c->ev_out_ready[slot], 0));
  pipe_mark("d2h start", c->pend_k, c->s_d2h);
  for (int i = 0; i < 4; ++i)
    if (c->pend_dst[i])
      FMM_CUDA(cudaMemcpyAsync(c->pend_dst[i], c->pipe_out[slot] + i * c->pend_n, 8 * c->pend_n,
                               cudaMemcpyDeviceToHost, c->s_d2h));
  FMM_CUDA(cudaEventRecord(c->ev_d2h_done[slot], c->s_d2h));
  pipe_mark("d2h end", c->pend_k, c->s_d2h);
  c->pipe_pend = false;
}

// One pipelined step on context c (its own copy streams, events and output slots).
void pipe_step(fmmgpu_ctx* c, const double* xyzw, uint64_t n, int height, int group, double* pot, double* fx,
               double* fy, double* fz) {
  if (!c->s_h2d) {
    FMM_CUDA(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    FMM_CUDA(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    FMM_CUDA(cudaEventCreateWithFlags(&c->ev_in_free, cudaEventDisableTiming));
    FMM_CUDA(cudaEventCreateWithFlags(&c->ev_in_ready, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      FMM_CUDA(cudaEventCreateWithFlags(&c->ev_out_ready[i], cudaEventDisableTiming));
      FMM_CUDA(cudaEventCreateWithFlags(&c->ev_d2h_done[i], cudaEventDisableTiming));
      FMM_CUDA(cudaEventRecord(c->ev_d2h_done[i], c->s_d2h));
    }
    FMM_CUDA(cudaEventRecord(c->ev_in_free, c->s_far));
  }
  if (c->d_in_cap < n || c->pipe_cap < n) {  // grow: drain the pipeline first
    pipe_issue_d2h(c);
    FMM_CUDA(cudaStreamSynchronize(c->s_h2d));
    FMM_CUDA(cudaStreamSynchronize(c->s_d2h));
    FMM_CUDA(cudaStreamSynchronize(c->s_near));
    if (c->d_in_cap < n) {
      if (c->d_in) FMM_CUDA(cudaFreeAsync(c->d_in, c->s_far));
      FMM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&c->d_in), n * sizeof(double4), c->s_far));
      c->d_in_cap = n;
    }
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
    if (c->pipe_cap < n) {
      for (auto& p : c->pipe_out) {
        if (p) FMM_CUDA(cudaFree(p));
        p = nullptr;
        FMM_CUDA(cudaMalloc(&p, 32 * n));
      }
      c->pipe_cap = n;
    }
    FMM_CUDA(cudaEventRecord(c->ev_in_free, c->s_far));
  }
  FMM_CUDA(cudaStreamWaitEvent(c->s_h2d, c->ev_in_free, 0));
  pipe_mark("h2d start", c->pipe_k, c->s_h2d);
  FMM_CUDA(cudaMemcpyAsync(c->d_in, xyzw, n * sizeof(double4), cudaMemcpyHostToDevice, c->s_h2d));
  FMM_CUDA(cudaEventRecord(c->ev_in_ready, c->s_h2d));
  pipe_mark("h2d end", c->pipe_k, c->s_h2d);
  FMM_CUDA(cudaStreamWaitEvent(c->s_far, c->ev_in_ready, 0));
  c->out_valid = false;
  pipe_mark("tree start", c->pipe_k, c->s_far);
  tree_build(c, reinterpret_cast<const double*>(c->d_in), n, true, height, group, nullptr);
  FMM_CUDA(cudaEventRecord(c->ev_in_free, c->s_far));
  pipe_mark("tree end", c->pipe_k, c->s_far);
  pipe_issue_d2h(c);  // the previous step's fields, under this step's evaluation
  const int slot = static_cast<int>(c->pipe_k & 1);
  FMM_CUDA(cudaStreamWaitEvent(c->s_far, c->ev_d2h_done[slot], 0));
  double* own_out = c->d_out;
  c->d_out = c->pipe_out[slot];
  const int rc = fmmgpu_evaluate(c);
  c->d_out = own_out;
  c->out_valid = false;
  if (rc != FMMGPU_OK) throw Error(rc, c->err);
  FMM_CUDA(cudaEventRecord(c->ev_out_ready[slot], c->s_far));
  pipe_mark("eval end", c->pipe_k, c->s_far);
  c->pipe_pend = true;
  c->pend_slot = slot;
  c->pend_n = n;
  c->pend_k = c->pipe_k;
  c->pend_dst[0] = pot;
  c->pend_dst[1] = fx;
  c->pend_dst[2] = fy;
  c->pend_dst[3] = fz;
  ++c->pipe_k;
}

}  // namespace

int fmmgpu_run_async(fmmgpu_ctx* c, const double* xyzw, uint64_t n, int height, int group, double* pot,
                     double* fx, double* fy, double* fz) {
  return guarded(c, [&] {
    FMM_CUDA(cudaSetDevice(c->device));
    if (!xyzw) throw Error(FMMGPU_INVALID_ARGUMENT, "run_async: null particle buffer");
    if (n == 0) throw Error(FMMGPU_INVALID_ARGUMENT, "GroupTree: empty particle set");
    pipe_step(c, xyzw, n, height, group, pot, fx, fy, fz);
  });
}

int fmmgpu_run_wait(fmmgpu_ctx* c) {
  return guarded(c, [&] {
    FMM_CUDA(cudaSetDevice(c->device));
    pipe_issue_d2h(c);
    if (c->s_d2h) FMM_CUDA(cudaStreamSynchronize(c->s_d2h));
    if (c->s_h2d) FMM_CUDA(cudaStreamSynchronize(c->s_h2d));
    FMM_CUDA(cudaStreamSynchronize(c->s_near));
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
    pipe_trace_dump();
  });
}

int fmmgpu_tree_info(const fmmgpu_ctx* c, uint64_t* n, int* height, int* group, double* root4) {
  if (!c || !c->have_tree) return FMMGPU_LOGIC_ERROR;
  if (n) *n = c->n;
  if (height) *height = c->height;
  if (group) *group = c->group;
  if (root4) std::copy(c->root, c->root + 4, root4);
  return FMMGPU_OK;
}

uint64_t fmmgpu_level_cells(const fmmgpu_ctx* c, int v) {
  if (!c || !c->have_tree || v < 0 || v >= c->height) return 0;
  return c->lv[v].n;
}

int fmmgpu_download_level(fmmgpu_ctx* c, int v, void* cells32, uint32_t* bo) {
  return guarded(c, [&] {
    need_level(c, v, 0, c->height - 1, "download_level");
    const Level& L = c->lv[v];
    if (cells32 && L.n) {
      uint32_t* d = static_cast<uint32_t*>(scratch(c, 32ull * L.n));
      k_cells_aos<<<(L.n + 255) / 256, 256, 0, c->s_far>>>(L.code, L.first_particle, L.particle_count, L.parent,
                                                          L.first_child, L.child_count, L.n, d);
      FMM_CUDA(cudaGetLastError());
      FMM_CUDA(cudaMemcpyAsync(cells32, d, 32ull * L.n, cudaMemcpyDeviceToHost, c->s_far));
    }
    if (bo) std::copy(L.block_offsets.begin(), L.block_offsets.end(), bo);
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

int fmmgpu_download_particles(fmmgpu_ctx* c, double* x, double* y, double* z, double* w, uint32_t* id) {
  return guarded(c, [&] {
    need_tree(c);
    double* d = static_cast<double*>(scratch(c, 32 * c->n));
    k_soa<<<(c->n + 255) / 256, 256, 0, c->s_far>>>(c->d_pw, c->n, d, d + c->n, d + 2 * c->n, d + 3 * c->n);
    FMM_CUDA(cudaGetLastError());
    double* dst[4] = {x, y, z, w};
    for (int i = 0; i < 4; ++i)
      if (dst[i]) FMM_CUDA(cudaMemcpyAsync(dst[i], d + i * c->n, 8 * c->n, cudaMemcpyDeviceToHost, c->s_far));
    if (id) FMM_CUDA(cudaMemcpyAsync(id, c->d_id, 4 * c->n, cudaMemcpyDeviceToHost, c->s_far));
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

int fmmgpu_download_sorted_fields(fmmgpu_ctx* c, double* pot, double* fx, double* fy, double* fz) {
  return guarded(c, [&] {
    need_tree(c);
    FMM_CUDA(cudaStreamSynchronize(c->s_near));
    double* d = static_cast<double*>(scratch(c, 32 * c->n));
    k_sum4<<<(c->n + 255) / 256, 256, 0, c->s_far>>>(reinterpret_cast<const double4*>(c->d_far),
                                                      reinterpret_cast<const double4*>(c->d_near), c->n, d);
    FMM_CUDA(cudaGetLastError());
    double* dst[4] = {pot, fx, fy, fz};
    for (int i = 0; i < 4; ++i)
      if (dst[i]) FMM_CUDA(cudaMemcpyAsync(dst[i], d + i * c->n, 8 * c->n, cudaMemcpyDeviceToHost, c->s_far));
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

int fmmgpu_download_expansion(fmmgpu_ctx* c, int v, int which, double* out) {
  return guarded(c, [&] {
    need_level(c, v, 0, c->height - 1, "download_expansion");
    if (which < 0 || which > 2) throw Error(FMMGPU_INVALID_ARGUMENT, "which must be 0, 1 or 2");
    const Level& L = c->lv[v];
    if (L.n == 0) return;
    const double* src = which == 0 ? L.multipole : which == 1 ? L.local_own : L.local_down;
    double* d = static_cast<double*>(scratch(c, 8ull * L.n * c->l3));
    const uint64_t tot = uint64_t(L.n) * c->l3;
    FMM_CUDA(cudaStreamSynchronize(c->s_near));
    k_pad_copy<<<(tot + 255) / 256, 256, 0, c->s_far>>>(src, c->l3, c->ldE, L.n, d, 0);
    FMM_CUDA(cudaGetLastError());
    FMM_CUDA(cudaMemcpyAsync(out, d, 8 * tot, cudaMemcpyDeviceToHost, c->s_far));
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

int fmmgpu_upload_expansion(fmmgpu_ctx* c, int v, int which, const double* in) {
  return guarded(c, [&] {
    need_level(c, v, 0, c->height - 1, "upload_expansion");
    if (which < 0 || which > 2) throw Error(FMMGPU_INVALID_ARGUMENT, "which must be 0, 1 or 2");
    const Level& L = c->lv[v];
    if (L.n == 0) return;
    double* dst = which == 0 ? L.multipole : which == 1 ? L.local_own : L.local_down;
    double* d = static_cast<double*>(scratch(c, 8ull * L.n * c->l3));
    const uint64_t tot = uint64_t(L.n) * c->l3;
    FMM_CUDA(cudaMemcpyAsync(d, in, 8 * tot, cudaMemcpyHostToDevice, c->s_far));
    k_pad_copy<<<(tot + 255) / 256, 256, 0, c->s_far>>>(d, c->l3, c->ldE, L.n, dst, 1);
    FMM_CUDA(cudaGetLastError());
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

uint64_t fmmgpu_near_entries(const fmmgpu_ctx* c) { return (c && c->have_lists) ? c->near_entries : 0; }

int fmmgpu_download_near(fmmgpu_ctx* c, uint32_t* off, uint32_t* cells, uint64_t* total) {
  return guarded(c, [&] {
    if (!c->have_lists) throw Error(FMMGPU_LOGIC_ERROR, "no lists: call fmmgpu_build_lists first");
    const Level& L = c->lv[c->height - 1];
    if (off) FMM_CUDA(cudaMemcpyAsync(off, c->d_near_off, 4ull * (L.n + 1), cudaMemcpyDeviceToHost, c->s_far));
    if (cells && c->near_entries)
      FMM_CUDA(cudaMemcpyAsync(cells, c->d_near_cells, 4ull * c->near_entries, cudaMemcpyDeviceToHost, c->s_far));
    if (total) *total = c->near_directional;
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

int fmmgpu_download_near_blocks(fmmgpu_ctx* c, uint64_t* task_interactions, uint32_t* above_off, uint32_t* above,
                                uint32_t* below_off, uint32_t* below, uint64_t* n_above, uint64_t* n_below) {
  return guarded(c, [&] {
    FMM_CUDA(cudaSetDevice(c->device));
    near_blocks(c, task_interactions, above_off, above, below_off, below, n_above, n_below);
  });
}

int fmmgpu_download_far_source_blocks(fmmgpu_ctx* c, int level, uint32_t* offsets, uint32_t* blocks,
                                      uint64_t* count) {
  return guarded(c, [&] {
    FMM_CUDA(cudaSetDevice(c->device));
    far_source_blocks(c, level, offsets, blocks, count);
  });
}

uint64_t fmmgpu_far_pairs(const fmmgpu_ctx* c, int v) {
  if (!c || !c->have_lists || v < 2 || v >= c->height) return 0;
  return c->lv[v].far_pairs;
}

int fmmgpu_download_far(fmmgpu_ctx* c, int v, uint32_t* target, uint32_t* source, uint16_t* vec, uint64_t* goff) {
  return guarded(c, [&] {
    if (!c->have_lists) throw Error(FMMGPU_LOGIC_ERROR, "no lists: call fmmgpu_build_lists first");
    need_level(c, v, 2, c->height - 1, "download_far");
    const Level& L = c->lv[v];
    const uint64_t np = L.far_pairs;
    if (np) {
      if (target) FMM_CUDA(cudaMemcpyAsync(target, L.far_target, 4 * np, cudaMemcpyDeviceToHost, c->s_far));
      if (source) FMM_CUDA(cudaMemcpyAsync(source, L.far_source, 4 * np, cudaMemcpyDeviceToHost, c->s_far));
      if (vec) FMM_CUDA(cudaMemcpyAsync(vec, L.far_vec, 2 * np, cudaMemcpyDeviceToHost, c->s_far));
    }
    const uint64_t ng = (L.block_offsets.size() - 1) * 16 + 1;
    if (goff) FMM_CUDA(cudaMemcpyAsync(goff, L.far_group_off, 8 * ng, cudaMemcpyDeviceToHost, c->s_far));
    FMM_CUDA(cudaStreamSynchronize(c->s_far));
  });
}

// count_interactions + build_ledger (taskflow.cpp:107-135, bench.cpp:151-181) from the
// device lists: per (kind, level) work and flops, kind-major [7][height], and the M2L
// pairs per (level, canonical class) [height][16].
int fmmgpu_ledger_rows(fmmgpu_ctx* c, uint64_t* work, uint64_t* flops, uint64_t* m2l_pairs16) {
  return guarded(c, [&] {
    need_tree(c);
    if (!c->have_lists) lists_build(c);
    const uint64_t l = c->order, n = c->n;
    const int h = c->height, leaf = h - 1;
    std::vector<uint64_t> W(size_t(7) * h, 0), F(size_t(7) * h, 0), P(size_t(16) * h, 0);
    auto at = [&](int k, int v) { return size_t(k) * h + v; };
    W[at(FMMGPU_P2M, leaf)] = n;
    F[at(FMMGPU_P2M, leaf)] = n * (4 * l * l * l + 15 * l);  // bench.cpp:104-122
    W[at(FMMGPU_L2P, leaf)] = n;
    F[at(FMMGPU_L2P, leaf)] = n * (16 * l * l * l + 30 * l);
    W[at(FMMGPU_P2P, leaf)] = c->near_directional;
    F[at(FMMGPU_P2P, leaf)] = c->near_directional * 15;
    W[at(FMMGPU_P2PREDUCE, leaf)] = n;
    for (int v = 2; v < leaf; ++v) {  // transfers[v] = children at v + 1 (taskflow.cpp:131-133)
      const uint64_t t = c->lv[v + 1].n;
      W[at(FMMGPU_M2M, v)] = W[at(FMMGPU_L2L, v)] = t;
      F[at(FMMGPU_M2M, v)] = F[at(FMMGPU_L2L, v)] = t * 6 * l * l * l * l;
    }
    for (int v = 2; v <= leaf; ++v) {
      const Level& L = c->lv[v];
      const uint64_t ng = (L.block_offsets.size() - 1) * 16;
      std::vector<uint64_t> go(ng + 1);
      FMM_CUDA(cudaMemcpy(go.data(), L.far_group_off, 8 * (ng + 1), cudaMemcpyDeviceToHost));
      for (uint64_t g = 0; g < ng; ++g) P[size_t(v) * 16 + g % 16] += go[g + 1] - go[g];
      for (int cl = 0; cl < 16; ++cl) {
        const uint64_t cnt = P[size_t(v) * 16 + cl], r = c->m2l.rank[cl];
        W[at(FMMGPU_M2L, v)] += cnt;
        F[at(FMMGPU_M2L, v)] += cnt * (4 * l * l * l * r + r * r);
      }
    }
    if (work) std::copy(W.begin(), W.end(), work);
    if (flops) std::copy(F.begin(), F.end(), flops);
    if (m2l_pairs16) std::copy(P.begin(), P.end(), m2l_pairs16);
  });
}

int fmmgpu_ledger(fmmgpu_ctx* c, uint64_t* flops7, uint64_t* near_dir, uint64_t* m2l_pairs) {
  return guarded(c, [&] {
    need_tree(c);
    const int h = c->height;
    std::vector<uint64_t> W(size_t(7) * h), F(size_t(7) * h);
    const int rc = fmmgpu_ledger_rows(c, W.data(), F.data(), nullptr);
    if (rc != FMMGPU_OK) throw Error(rc, c->err);
    for (int k = 0; k < 7; ++k) {
      uint64_t f = 0;
      for (int v = 0; v < h; ++v) f += F[size_t(k) * h + v];
      if (flops7) flops7[k] = f;
    }
    uint64_t pairs = 0;
    for (int v = 0; v < h; ++v) pairs += W[size_t(FMMGPU_M2L) * h + v];
    if (near_dir) *near_dir = c->near_directional;
    if (m2l_pairs) *m2l_pairs = pairs;
  });
}

void fmmgpu_generate_particles(uint64_t n, int dist, uint64_t seed, double* xyzw) {
  // bench.cpp:19-61
  std::mt19937_64 rng(seed);
  auto u01 = [&] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
  if (dist == 0) {
    for (uint64_t i = 0; i < n; ++i) {
      const double x = u01(), y = u01(), z = u01();
      xyzw[4 * i] = x;
      xyzw[4 * i + 1] = y;
      xyzw[4 * i + 2] = z;
      xyzw[4 * i + 3] = 1.0;
    }
    return;
  }
  constexpr double two_pi = 6.283185307179586476925286766559;
  auto normal_pair = [&](double& a, double& b) {
    const double u1 = static_cast<double>((rng() >> 11) + 1) * 0x1.0p-53;
    const double u2 = u01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    a = r * std::cos(two_pi * u2);
    b = r * std::sin(two_pi * u2);
  };
  for (uint64_t i = 0; i < n; ++i) {
    double gx, gy, gz, spare, norm = 0;
    do {
      normal_pair(gx, gy);
      normal_pair(gz, spare);
      norm = std::sqrt(gx * gx + gy * gy + gz * gz);
    } while (norm < 1e-12);
    // dist 2: config D's ellipsoid surface, semi-axes (0.5, 0.35, 0.2)
    const double ax = 0.5, ay = dist == 2 ? 0.35 : 0.5, az = dist == 2 ? 0.2 : 0.5;
    xyzw[4 * i] = 0.5 + ax * gx / norm;
    xyzw[4 * i + 1] = 0.5 + ay * gy / norm;
    xyzw[4 * i + 2] = 0.5 + az * gz / norm;
    xyzw[4 * i + 3] = 1.0;
  }
}

}  // extern "C"
