// Shared definitions of the B200 FMM path: context layout in HBM, Morton helpers,
// cell lookup, FP64 reciprocal square root. See DESIGN.md "Data layout in HBM".
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <vector>

#include "fmmgpu.h"

namespace fmmgpu {

constexpr uint32_t NPOS = 0xffffffffu;
constexpr int MAX_ORDER = 10;
constexpr int DENSE_MAP_MAX_LEVEL = 9;  // 8^9 x 4 B = 512 MB worst case

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FMM_CUDA(x)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      throw ::fmmgpu::Error(FMMGPU_RUNTIME_ERROR, std::string("CUDA: ") +                 \
                                                      cudaGetErrorString(e_) + " at " +   \
                                                      __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// dlopen of NCCL shared by the partitioned evaluation and the distributed build (partition.cu)
void* open_nccl();

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------- Morton codes
// geometry.cpp:38-57: bit b of i -> 3b+2, j -> 3b+1, k -> 3b.
__host__ __device__ inline uint64_t spread3(uint32_t x) {
  uint64_t v = x & 0x1fffffu;
  v = (v | (v << 32)) & 0x1f00000000ffffULL;
  v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
  v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
  v = (v | (v << 2)) & 0x1249249249249249ULL;
  return v;
}
__host__ __device__ inline uint32_t compact3(uint64_t v) {
  v &= 0x1249249249249249ULL;
  v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ULL;
  v = (v ^ (v >> 4)) & 0x100f00f00f00f00fULL;
  v = (v ^ (v >> 8)) & 0x1f0000ff0000ffULL;
  v = (v ^ (v >> 16)) & 0x1f00000000ffffULL;
  v = (v ^ (v >> 32)) & 0x1fffffULL;
  return static_cast<uint32_t>(v);
}
__host__ __device__ inline uint64_t morton(uint32_t i, uint32_t j, uint32_t k) {
  return (spread3(i) << 2) | (spread3(j) << 1) | spread3(k);
}
__host__ __device__ inline void demorton(uint64_t c, int* ijk) {
  ijk[0] = static_cast<int>(compact3(c >> 2));
  ijk[1] = static_cast<int>(compact3(c >> 1));
  ijk[2] = static_cast<int>(compact3(c));
}

// Cell lookup on one level (GroupTree::find_cell, geometry.cpp:177-186): O(1) on a
// full level, a dense code->index map up to DENSE_MAP_MAX_LEVEL, else binary search.
struct LevelView {
  const uint64_t* code;
  const uint32_t* map;
  uint32_t n;
  int level;
  int full;
};
__device__ inline uint32_t find_cell(const LevelView& L, uint64_t code) {
  if (L.full) return static_cast<uint32_t>(code);
  if (L.map) return L.map[code];
  uint32_t lo = 0, hi = L.n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (L.code[mid] < code) lo = mid + 1; else hi = mid;
  }
  return (lo < L.n && L.code[lo] == code) ? lo : NPOS;
}
// grid coords -> cell index or NPOS (out of range / absent)
__device__ inline uint32_t find_ijk(const LevelView& L, int i, int j, int k) {
  const int g = 1 << L.level;
  if (i < 0 || j < 0 || k < 0 || i >= g || j >= g || k >= g) return NPOS;
  return find_cell(L, morton(static_cast<uint32_t>(i), static_cast<uint32_t>(j), static_cast<uint32_t>(k)));
}

// FP64 1/sqrt(x), x > 0: MUFU.RSQ64H seed (rsqrt.approx.ftz.f64) and one
// third-order Newton step: e = 1 - x y^2, y *= 1 + e/2 + 3e^2/8. With the seed's
// ~2^-22 relative error the residual is ~2^-65, i.e. rounding-level (checked by
// tests/test_gpu_kernels.py against 1/sqrt). 5 DP ops + 1 MUFU versus ~12 DP-op
// equivalents for the libdevice rsqrt (profiles/r01_fp64_peaks.txt).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double t = x * y;
  const double e = fma(-t, y, 1.0);
  const double p = fma(e, 0.375, 0.5);
  return fma(y, e * p, y);
}

// ---------------------------------------------------------------- context
struct Level {
  uint32_t n = 0;
  bool full = false;
  uint64_t* code = nullptr;
  uint32_t *first_particle = nullptr, *particle_count = nullptr, *parent = nullptr,
           *first_child = nullptr, *child_count = nullptr;
  uint32_t* map = nullptr;         // dense code -> index (sparse levels <= DENSE_MAP_MAX_LEVEL)
  uint32_t* cls_cells = nullptr;   // cell indices grouped by parity class (code & 7)
  uint32_t cls_off[9] = {};        // class offsets into cls_cells (host copy)
  // partitioned runs (fmmgpu_partition): owned cells [own0, own1) -- every cell when the
  // level is replicated -- and the M2L phase A source / phase B target lists per parity
  // class (nullptr = cls_cells)
  uint32_t own0 = 0, own1 = 0;
  uint32_t* srcA = nullptr;
  uint32_t srcA_off[9] = {};
  uint32_t* tgtB = nullptr;
  uint32_t tgtB_off[9] = {};
  // exchange after this level's upward step (partitioned runs): 0 none, 1 all-gather of
  // the owned rows, 2 halo -- rows sent to / received from every peer (host lists with
  // per-peer offsets, device indices: sends then receives)
  int xkind = 0;
  std::vector<uint32_t> halo_send, halo_recv, halo_send_off, halo_recv_off;
  uint32_t* halo_idx = nullptr;
  double *multipole = nullptr, *local_own = nullptr, *local_down = nullptr;  // n x ldE
  double* yt = nullptr;  // M2L compressed intermediates, n x ldY (zero where no source)
  std::vector<uint32_t> block_offsets;
  // far plan (LevelM2L), built by fmmgpu_build_lists
  uint64_t far_pairs = 0;
  uint32_t *far_target = nullptr, *far_source = nullptr;
  uint16_t* far_vec = nullptr;
  uint64_t* far_group_off = nullptr;
  LevelView view(int v) const { return LevelView{code, map, n, v, full ? 1 : 0}; }
};

struct M2LTables {
  // host-side operator factors (cache format): per class row-major U, sigma, V
  int rank[16] = {};
  int mult[16] = {};
  std::vector<double> u[16], sigma[16], v[16];
  int canonical[343];
  std::vector<uint32_t> perm[343];  // grid permutation per vector slot
  // stacked operators
  int R = 0;        // rows of the source-side stack = columns of the target-side stack
  int ldY = 0;      // round_up(R, 32): stride of one target's compressed vector
  int rowsA = 0;    // round_up(R, bmA): padded M of phase A
  int bmA = 64;     // phase A M-tile rows (64 for l <= 5, 128 above)
  int rowsB = 0;    // round_up(l^3, 64)... padded M of phase B
  double* dM1 = nullptr;    // [8][rowsA][ldE]
  double* dM2 = nullptr;    // [8][rowsB][ldY]
  int4* dRowA = nullptr;    // [8][rowsA]: {slot or -1, destination column in Yt, vector index in its M-tile, 0}
  int* dTileVec = nullptr;  // [8][rowsA/64][vtMax]: vector slots of each 64-row M-tile (-1 = none)
  int vtMax = 0;            // max distinct vectors in one 64-row M-tile
  int* dTileVec2 = nullptr; // the same for the 128-row tiles of the streamed phase A (rowA.w)
  int vtMax2 = 0;
  int* dKslot = nullptr;    // [8][ldY]: vector slot of column kk of the target stack, -1 = pad
};

// Device blocks of a context recycled across tree builds (cudaMallocAsync of the
// 80-320 MB tree arrays costs 0.2-2 ms per call, occasionally far more)
struct DevCache {
  std::unordered_map<void*, size_t> live;                  // block -> capacity
  std::multimap<size_t, std::pair<void*, uint64_t>> idle;  // capacity -> {free block, epoch freed}
  uint64_t epoch = 0;                                      // one per tree build
};

struct Timing {
  cudaEvent_t ev[32];
  int used = 0;
};

}  // namespace fmmgpu

struct fmmgpu_ctx {
  int device = 0;
  int order = 0;
  double eps = 0;
  int l3 = 0;
  int ldE = 0;  // padded expansion stride (multiple of 32 doubles: whole GEMM k-slices)
  std::string err;
  cudaStream_t s_far = nullptr, s_near = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // coarse M2L levels and the L2L chain run on s_aux beside the leaf M2L (evaluation)
  cudaStream_t s_aux = nullptr;
  cudaEvent_t ev_up = nullptr, ev_aux = nullptr;
  cudaEvent_t ev_p2p_main = nullptr;  // the mutual near-field kernel done (slots written)
  cudaEvent_t ev_t[16] = {};
  double timings[10] = {};
  uint64_t launches = 0;
  // interpolation tables (device): tn[l][l-1], child[2][l*l], child_t[2][l*l]
  double* d_interp = nullptr;
  std::vector<double> h_roots, h_tn, h_child[2], h_child_t[2];
  fmmgpu::M2LTables m2l;
  // tree
  bool have_tree = false;
  uint64_t n = 0;
  int height = 0, group = 0;
  double root[4] = {};
  double lo[3] = {};
  std::vector<fmmgpu::Level> lv;
  double4* d_in = nullptr;       // input particles, input order
  size_t d_in_cap = 0;
  double4* d_pw = nullptr;       // Morton-ordered {x,y,z,w}
  uint32_t* d_id = nullptr;      // original index per Morton slot
  uint32_t* d_pcell = nullptr;   // leaf cell per Morton slot
  uint32_t* d_inv = nullptr;     // Morton slot per input index (inverse of d_id)
  double* d_near = nullptr;      // near-field fields [n] x {pot,fx,fy,fz} (Morton order)
  // mutual P2P (p2p.cu): the j-side sums of each leaf's 13 upper half-shell neighbours,
  // [13][n] x {pot,fx,fy,fz} (the reference's P2PBuffers slots), and the leaf counter
  int p2p_mode = 2;  // 0 one-sided, 1 mutual, 2 auto (mutual when there are enough leaves)
  double* d_slot = nullptr;
  uint32_t* d_ctr = nullptr;
  // non-full leaf levels: leaves by decreasing work (+ sort buffers), valid for the owned
  // leaf range p2p_order_range = {own0, own1 + 1} (0, 0 = not computed)
  uint32_t* d_p2p_order = nullptr;
  size_t p2p_order_tmp = 0;
  uint32_t p2p_order_range[2] = {0, 0};
  double* d_far = nullptr;       // far-field fields [n] x {pot,fx,fy,fz} (Morton order)
  double* d_out = nullptr;       // gathered fields [4][n] (input order)
  // partition: this context is rank part_rank of part_n; levels below
  // part_align are replicated; own_s0..own_s1 = owned Morton particle slots
  int part_rank = 0, part_n = 1, part_align = 0;
  uint64_t own_s0 = 0, own_s1 = 0;
  void* nccl = nullptr;          // ncclComm_t when fmmgpu_comm_init attached one
  double* d_halo_buf = nullptr;  // halo exchange staging (send rows, then received rows)
  size_t halo_buf_cap = 0;
  bool skip_exchange = false;    // fmmgpu_set_measurement: partitioned work timed without peers
  std::vector<std::vector<uint32_t>> part_begin;  // per level: first owned cell of every rank (+ end)
  // distributed input (dist.cu, SURVEY §8e halo particles): this rank holds the input slice
  // [dist_off[rank], dist_off[rank + 1]) in d_loc; the tree comes from all-gathered keys,
  // d_pw holds only the owned and halo leaves once the particle exchange is committed
  bool dist = false, dist_ready = true;
  double4* d_loc = nullptr;
  size_t d_loc_cap = 0;
  uint64_t dist_nloc = 0, dist_ntot = 0, dist_offset = 0;
  std::vector<uint64_t> dist_off;                 // nranks + 1 slice offsets (input order)
  uint32_t* d_dsend = nullptr;                    // slots to send, grouped by peer
  uint32_t* d_drecv = nullptr;                    // slots to receive, grouped by peer
  std::vector<uint32_t> dsend_off, drecv_off;     // nranks + 1 offsets into the two lists
  int comm_rank = 0, comm_n = 1;                  // of the attached NCCL communicator
  // captured evaluation (fmmgpu_evaluate): replayed while tree / partition / operators hold
  cudaGraphExec_t graph_exec = nullptr;
  bool graph_warm = false;   // one eager evaluation done since the last invalidation
  bool use_graph = false;    // replay evaluations as a captured graph (fmmgpu_set_graph)
  bool capturing = false;
  uint64_t graph_launches = 0;
  // M2L phase B split-K partials: [0] coarse levels, [1] the leaf level (the two can run
  // concurrently on s_aux and s_far)
  double* d_splitk[2] = {};
  size_t splitk_cap[2] = {};
  bool out_valid = false;        // d_out holds near + far of the current arrays
  bool zero_pending = false;     // expansions / field accumulators of a new tree not yet cleared
  // set while an unpartitioned evaluation is enqueued: every operator writes its output
  // (sums formed in the same order as accumulating into zero) instead of accumulating,
  // so the evaluation needs no clearing pass and no read of the old values
  bool ow = false;
  // per-launch device trace of evaluations (fmmgpu_set_trace): one event pair per
  // operator launch, {kind, level, stream} beside it; evaluations run eagerly while on
  bool trace = false;
  std::vector<cudaEvent_t> tr_ev;
  std::vector<int> tr_meta;  // 3 per span: kind, level, stream (0 far field, 1 near field)
  int* d_flag = nullptr;         // error flags
  // near plan
  bool have_lists = false;
  uint32_t* d_near_off = nullptr;
  uint32_t* d_near_cells = nullptr;
  uint64_t near_entries = 0;
  uint64_t near_directional = 0;
  // scratch
  void* d_tmp = nullptr;
  size_t d_tmp_cap = 0;
  int* d_canon = nullptr;  // canonical class per vector slot (343)
  // pipelined runs (fmmgpu_run_async): copy streams, double-buffered gathered fields
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in_free = nullptr, ev_in_ready = nullptr, ev_out_ready[2] = {}, ev_d2h_done[2] = {};
  double* pipe_out[2] = {};
  // small device -> host readbacks (counts, flags) through mapped pinned memory written
  // by a kernel, so they never queue behind bulk transfers on the copy engines
  void* h_rb = nullptr;
  fmmgpu::DevCache cache;
  // M2L intermediates of full levels kept across tree rebuilds: on a full level the
  // blocks without a source are the same for every tree, so they are still zero and
  // the 5 GB (config B leaf) clear is skipped; index = level
  double* yt_keep[22] = {};
  uint32_t yt_keep_n[22] = {};
  uint64_t pipe_cap = 0;
  uint64_t pipe_k = 0;
  // the D2H of the last enqueued step is issued after the NEXT step's tree build, so the
  // build's small readbacks do not share the device->host PCIe direction with it
  bool pipe_pend = false;
  int pend_slot = 0;
  uint64_t pend_n = 0, pend_k = 0;
  double* pend_dst[4] = {};
};

namespace fmmgpu {
// implemented in the .cu files
void interp_setup(fmmgpu_ctx* c);
void m2l_setup(fmmgpu_ctx* c, bool compute_factors);
void m2l_free(fmmgpu_ctx* c);
struct DistKeys {            // distributed build (dist.cu): all-gathered keys, no positions
  const uint64_t* keys;      // [n] leaf Morton keys in input order (device)
  int flag;                  // OR of the ranks' outside-the-root flags (bit 0)
};
void tree_build(fmmgpu_ctx* c, const double* xyzw, uint64_t n, bool on_device, int height, int group,
                const double* root4, const DistKeys* dist = nullptr);
void root_from_bounds(const double lo[3], const double hi[3], double root[4]);
void device_bounds(fmmgpu_ctx* c, const double4* d, uint64_t n, double lohi[6], cudaStream_t s);
void device_keys(const double4* d, uint64_t n, const double root[4], int height, uint64_t* keys, uint32_t* idx,
                 int* flag, cudaStream_t s);
void dist_free(fmmgpu_ctx* c);
int coincident_check(fmmgpu_ctx* c, uint32_t leaf0, uint32_t leaf1, cudaStream_t s);
void tree_free(fmmgpu_ctx* c);
void yt_keep_free(fmmgpu_ctx* c);
void lists_build(fmmgpu_ctx* c);
void lists_free(fmmgpu_ctx* c);
void near_blocks(fmmgpu_ctx* c, uint64_t* task, uint32_t* above_off, uint32_t* above, uint32_t* below_off,
                 uint32_t* below, uint64_t* n_above, uint64_t* n_below);
void far_source_blocks(fmmgpu_ctx* c, int v, uint32_t* off, uint32_t* list, uint64_t* n);
void launch_p2m(fmmgpu_ctx* c, cudaStream_t s);
void launch_m2m(fmmgpu_ctx* c, int parent_level, cudaStream_t s);
void launch_l2l(fmmgpu_ctx* c, int parent_level, cudaStream_t s);
void launch_l2p(fmmgpu_ctx* c, cudaStream_t s, bool drain = false);
void launch_m2l(fmmgpu_ctx* c, int level, cudaStream_t s);
// fuse_drain (evaluations): the mutual kernel only; its slot drain runs inside L2P
// (launch_l2p(..., true)) after the event ev_p2p_main this records
void launch_p2p(fmmgpu_ctx* c, cudaStream_t s, bool fuse_drain = false);
void ensure_p2p_slots(fmmgpu_ctx* c);  // allocates the mutual P2P slots of the current tree (s_far)
bool p2p_use_mutual(const fmmgpu_ctx* c, uint32_t leaves);  // the kernel launch_p2p picks
void launch_gather(fmmgpu_ctx* c, cudaStream_t s);
void partition_free(fmmgpu_ctx* c);
}  // namespace fmmgpu
extern "C" void fmmgpu_invalidate_graph(fmmgpu_ctx* c);
namespace fmmgpu {
void exchange_level(fmmgpu_ctx* c, int v, cudaStream_t s);
void* scratch(fmmgpu_ctx* c, size_t bytes);
// stream-ordered block cache: blocks freed on s are reused by later allocations on s
void* cache_alloc(fmmgpu_ctx* c, size_t bytes, cudaStream_t s);
void cache_free(fmmgpu_ctx* c, void* p, cudaStream_t s);  // blocks it did not allocate: cudaFreeAsync
void cache_trim(fmmgpu_ctx* c, cudaStream_t s);            // release the idle blocks
// release the idle blocks freed before the current epoch (the previous tree's arrays
// this build did not reuse); the build's own temporaries stay for the next build
void cache_trim_old(fmmgpu_ctx* c, cudaStream_t s);
constexpr size_t READBACK_CAP = 64 * 1024;
// copies `bytes` (multiple of 4, <= READBACK_CAP) of device memory to host through the
// mapped buffer, synchronizing s; the returned host pointer is valid until the next call
const void* readback(fmmgpu_ctx* c, const void* src, size_t bytes, cudaStream_t s);
uint64_t near_directional_count(fmmgpu_ctx* c);
int canonicalize_host(const int v[3], int perm[3], int sign[3]);
inline int vec_slot(int i, int j, int k) { return (i + 3) * 49 + (j + 3) * 7 + (k + 3); }
}  // namespace fmmgpu
