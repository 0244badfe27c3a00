/* fmmgpu.h — C ABI of the B200-native black-box Chebyshev FMM evaluation path.
 *
 * Drop-in boundary for the reference ("taskfmm", /root/reference/proj) operator
 * seam: FmmContext::run_task (bench.cpp:255-344) dispatching P2M / M2M / M2L /
 * L2L / L2P / P2P payloads over a GroupTree (geometry.hpp:70-112) with an
 * InteractionPlan (taskflow.hpp:60-70). Plain pointers and sizes only; no C++ or
 * torch types cross this boundary. One context owns all device memory of one
 * device and is driven by one host thread.
 *
 * Semantics follow the reference:
 *   - operators ACCUMULATE into arrays zeroed by fmmgpu_reset (FmmContext::reset,
 *     bench.cpp:240-253); M2L writes only local_own, L2L writes the child's
 *     local_down, L2L and L2P read own+down (bench.cpp:300-336);
 *   - fields are returned in INPUT order (FmmContext::gather, bench.cpp:350-365);
 *   - errors are status codes, one per reference exception class, with the text in
 *     fmmgpu_last_error (bench.hpp / geometry.cpp:65-69, 86-87, 134; m2l.cpp:60-61).
 *
 * Every entry point replaces the reference interface cited beside it.
 */
#ifndef FMMGPU_H_
#define FMMGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fmmgpu_ctx fmmgpu_ctx;

enum fmmgpu_status {
  FMMGPU_OK = 0,
  FMMGPU_INVALID_ARGUMENT = 1, /* std::invalid_argument (geometry.cpp:65-69, chebyshev.cpp:58-59) */
  FMMGPU_DOMAIN_ERROR = 2,     /* std::domain_error (geometry.cpp:86-87, 134) */
  FMMGPU_OUT_OF_RANGE = 3,     /* std::out_of_range (direct.cpp:79-80) */
  FMMGPU_LOGIC_ERROR = 4,      /* std::logic_error (m2l.cpp:69, taskflow.cpp:271) */
  FMMGPU_RUNTIME_ERROR = 5     /* std::runtime_error, CUDA / cuSOLVER failures */
};

/* Task kinds, same numbering as taskfmm::TaskKind (taskflow.hpp:15). */
enum fmmgpu_kind {
  FMMGPU_P2M = 0, FMMGPU_M2M = 1, FMMGPU_M2L = 2, FMMGPU_L2L = 3,
  FMMGPU_L2P = 4, FMMGPU_P2P = 5, FMMGPU_P2PREDUCE = 6
};

/* ---- context: InterpolationEngine(order) + M2LOperatorSet(order, eps) ----------
 * chebyshev.cpp:57-76, m2l.cpp:136-163. The 16 canonical operators are assembled
 * (m2l.cpp:90-111) and compressed with a truncated SVD on the device (cuSOLVER),
 * rank rule of m2l.cpp:116-122. order in [2,10]; eps > 0 (reference: 10^-order). */
int fmmgpu_create(int device, int order, double eps, fmmgpu_ctx** out);
void fmmgpu_destroy(fmmgpu_ctx* ctx);
const char* fmmgpu_last_error(const fmmgpu_ctx* ctx); /* never NULL */
/* Process-wide error text for failures before a context exists. */
const char* fmmgpu_global_error(void);

/* M2LOperatorSet::load_cache / save_cache binary format (m2l.cpp:212-288):
 * magic 0x4c324d4d4d465400, int32 order, f64 eps, 16 x int32 ranks, then per class
 * row-major U (l^3 x r), sigma (r), V (l^3 x r). load replaces the operators. */
int fmmgpu_load_m2l_cache(fmmgpu_ctx* ctx, const char* path);
int fmmgpu_save_m2l_cache(const fmmgpu_ctx* ctx, const char* path);
/* fmmgpu_create with the operators of a saved cache instead of a new device SVD
 * (M2LOperatorSet::load_cache(path, order, eps), m2l.cpp:247-288: a cache of another
 * order or eps, or an unreadable file, is an error). */
int fmmgpu_create_from_cache(int device, int order, double eps, const char* path, fmmgpu_ctx** out);
/* CompressionReport (m2l.hpp:56-62): ranks and multiplicities per canonical class. */
int fmmgpu_m2l_report(const fmmgpu_ctx* ctx, int32_t* ranks16, int32_t* multiplicity16,
                      double* weighted_mean_rank);

/* ---- tree: GroupTree(particles, height, group_size[, root]) ---------------------
 * geometry.cpp:59-161. xyzw: n particles as {x, y, z, w} doubles (Particle,
 * geometry.hpp:16-19), in HOST memory (copied to the device inside the call) or
 * DEVICE memory when xyzw_on_device != 0. root4 = {cx, cy, cz, width} or NULL for
 * bounding_cube (geometry.cpp:18-36). height in [3,21], group_size >= 1. */
int fmmgpu_build_tree(fmmgpu_ctx* ctx, const double* xyzw, uint64_t n, int xyzw_on_device,
                      int height, int group_size, const double* root4);

/* ---- interaction plan: build_interaction_plan (taskflow.cpp:67-105) -------------
 * near CSR (direct.cpp:22-61: near_offsets / near_cells, plus total_directional) and
 * per level v >= 2 the LevelM2L far pairs grouped by (block, canonical)
 * (taskflow.cpp:78-94). The evaluation itself enumerates interactions implicitly;
 * the explicit lists exist for parity, ledgers and reference tooling. */
int fmmgpu_build_lists(fmmgpu_ctx* ctx);

/* ---- evaluation: the payloads of FmmContext::run_task, level granular ----------
 * Each call enqueues device work on the context's streams and returns; errors of
 * asynchronous work surface at the next fmmgpu_synchronize / download. */
int fmmgpu_reset(fmmgpu_ctx* ctx);                  /* bench.cpp:240-253 */
int fmmgpu_p2m(fmmgpu_ctx* ctx);                    /* bench.cpp:259-273 (all leaf blocks) */
int fmmgpu_m2m(fmmgpu_ctx* ctx, int parent_level);  /* bench.cpp:274-287, level 2..leaf-1 */
int fmmgpu_m2l(fmmgpu_ctx* ctx, int level);         /* bench.cpp:288-299, level 2..leaf */
int fmmgpu_l2l(fmmgpu_ctx* ctx, int parent_level);  /* bench.cpp:300-316, level 2..leaf-1 */
int fmmgpu_l2p(fmmgpu_ctx* ctx);                    /* bench.cpp:317-336 */
int fmmgpu_p2p(fmmgpu_ctx* ctx);                    /* bench.cpp:337-342: P2P + P2PREDUCE */
/* The whole DAG (execute over the task graph, runtime.cpp:91-216) as a level-synchronous
 * two-stream schedule: far field on one stream, near field concurrently on another. The
 * result equals fmmgpu_reset followed by every operator; unpartitioned evaluations write
 * each output once (same sums) instead of clearing and accumulating. */
int fmmgpu_evaluate(fmmgpu_ctx* ctx);
int fmmgpu_synchronize(fmmgpu_ctx* ctx);
/* Replay evaluations from a captured CUDA graph (captured after one eager run; rebuilt
 * after tree, partition or operator changes). Off by default (FMMGPU_GRAPH=1 turns it on
 * for new contexts): eager launches on the two prioritised streams measured faster. */
int fmmgpu_set_graph(fmmgpu_ctx* ctx, int on);
/* Near-field kernel: mutual = 1 evaluates each pair of neighbouring leaves once,
 * p2p_block(mutual=true) with P2PBuffers slots and the ordered p2p_reduce
 * (direct.cpp:63-92, 151-200); mutual = 0 evaluates every directional interaction on the
 * target's side (p2p_block(mutual=false), direct.cpp:111-150); mutual = 2 (default) picks
 * the mutual kernel when the owned leaf level has >= 8 leaves per resident warp of it,
 * else the one-sided one. Both are deterministic and agree to rounding;
 * FMMGPU_P2P_ONESIDED=1 makes 0 the default of new contexts. */
int fmmgpu_set_p2p_mode(fmmgpu_ctx* ctx, int mutual);
/* the kernel the current tree / partition runs: 1 mutual, 0 one-sided, -1 no tree */
int fmmgpu_p2p_kernel(const fmmgpu_ctx* ctx);

/* FmmContext::gather (bench.cpp:350-365): fields in input order into HOST or DEVICE
 * arrays of n doubles each (any may be NULL). Synchronizes. */
int fmmgpu_download_fields(fmmgpu_ctx* ctx, double* potential, double* fx, double* fy,
                           double* fz, int dst_on_device);

/* Whole run with host buffers: build_tree + evaluate + download_fields
 * (run_fmm minus the oracle check, bench.cpp:415-469). */
int fmmgpu_run(fmmgpu_ctx* ctx, const double* xyzw, uint64_t n, int height, int group_size,
               double* potential, double* fx, double* fy, double* fz);

/* Pipelined fmmgpu_run over a stream of particle sets (run_fmm called repeatedly,
 * bench.cpp:415-469, with the copies off the critical path). Returns once step k's tree
 * is built and its evaluation is enqueued: the H2D of step k+1 overlaps evaluation k,
 * the D2H of step k overlaps step k+1. xyzw and the four outputs should be PINNED host
 * memory; xyzw may be reused once the next fmmgpu_run_async returns, outputs are valid
 * after fmmgpu_run_wait. Errors of the tree build are reported synchronously (same
 * codes as fmmgpu_build_tree). */
int fmmgpu_run_async(fmmgpu_ctx* ctx, const double* xyzw, uint64_t n, int height, int group_size,
                     double* potential, double* fx, double* fy, double* fz);
int fmmgpu_run_wait(fmmgpu_ctx* ctx);

/* ---- tree / plan / expansion access (parity dumps) ---------------------------- */
int fmmgpu_tree_info(const fmmgpu_ctx* ctx, uint64_t* n, int* height, int* group_size,
                     double* root4);
uint64_t fmmgpu_level_cells(const fmmgpu_ctx* ctx, int level);
/* cells as taskfmm::Cell AoS (geometry.hpp:34-41, 32 bytes each) and block_offsets
 * (cells/group_size rounded up, plus one). */
int fmmgpu_download_level(fmmgpu_ctx* ctx, int level, void* cells32, uint32_t* block_offsets);
/* ParticleStore in Morton order (geometry.hpp:59-65). */
int fmmgpu_download_particles(fmmgpu_ctx* ctx, double* x, double* y, double* z, double* w,
                              uint32_t* id);
/* Morton-order accumulators (potential/fx/fy/fz of ParticleStore). */
int fmmgpu_download_sorted_fields(fmmgpu_ctx* ctx, double* potential, double* fx, double* fy,
                                  double* fz);
/* which: 0 multipole, 1 local_own, 2 local_down; cells x l^3 doubles, cell-major
 * (GroupTree::allocate_expansions, geometry.cpp:199-206). */
int fmmgpu_download_expansion(fmmgpu_ctx* ctx, int level, int which, double* out);
int fmmgpu_upload_expansion(fmmgpu_ctx* ctx, int level, int which, const double* in);

uint64_t fmmgpu_near_entries(const fmmgpu_ctx* ctx);
int fmmgpu_download_near(fmmgpu_ctx* ctx, uint32_t* near_offsets, uint32_t* near_cells,
                         uint64_t* total_directional);
/* NearFieldPlan's block arrays (direct.cpp:36-58): task_interactions (one per leaf block),
 * partners_above and contributors_below as CSR (offsets: blocks + 1 entries). Any array
 * may be NULL; *n_above / *n_below = the list lengths (query with NULL lists first).
 * Needs fmmgpu_build_lists. */
int fmmgpu_download_near_blocks(fmmgpu_ctx* ctx, uint64_t* task_interactions, uint32_t* above_off,
                                uint32_t* above, uint32_t* below_off, uint32_t* below, uint64_t* n_above,
                                uint64_t* n_below);
/* LevelM2L::source_blocks (taskflow.cpp:96-102): per block of `level` the blocks of its
 * far sources, ascending, as CSR (offsets: blocks + 1); NULL arrays = query *count. */
int fmmgpu_download_far_source_blocks(fmmgpu_ctx* ctx, int level, uint32_t* offsets, uint32_t* blocks,
                                      uint64_t* count);
uint64_t fmmgpu_far_pairs(const fmmgpu_ctx* ctx, int level);
/* M2LPairRef (m2l.hpp:66-70) as three arrays, and group_offsets (blocks*16+1). */
int fmmgpu_download_far(fmmgpu_ctx* ctx, int level, uint32_t* target, uint32_t* source,
                        uint16_t* vec, uint64_t* group_offsets);

/* ---- measurement --------------------------------------------------------------- */
/* Device time (ms, CUDA events) of the last fmmgpu_evaluate per kind (index =
 * fmmgpu_kind; P2PREDUCE slot = field gather), plus [7] = whole evaluation,
 * [8] = last build_tree, [9] = last build_lists. */
int fmmgpu_timings(const fmmgpu_ctx* ctx, double* ms10);
/* Analytic work of the current tree (flop_cost, bench.cpp:102-122; ledger,
 * bench.cpp:151-181): flops per kind (7), near directional interactions, M2L pairs. */
int fmmgpu_ledger(fmmgpu_ctx* ctx, uint64_t* flops7, uint64_t* near_directional,
                  uint64_t* m2l_pairs);
/* FlopLedger rows (build_ledger, bench.cpp:151-181, over count_interactions,
 * taskflow.cpp:107-135): work[k * height + v] and flops[k * height + v] per task kind k
 * (fmmgpu_kind) and level v; m2l_pairs16[v * 16 + c] = M2L pairs of canonical class c at
 * level v (InteractionStats::m2l_pairs). Any pointer may be NULL. */
int fmmgpu_ledger_rows(fmmgpu_ctx* ctx, uint64_t* work, uint64_t* flops, uint64_t* m2l_pairs16);
/* Number of kernels launched by the last fmmgpu_evaluate. */
uint64_t fmmgpu_last_launch_count(const fmmgpu_ctx* ctx);
/* Per-launch device trace of evaluations (runtime.cpp:157-171 TraceEvent, written by
 * write_chrome_trace, runtime.cpp:277-292): while on, fmmgpu_evaluate runs eagerly and
 * brackets every operator launch with events. fmmgpu_trace_spans returns, for the last
 * evaluation, `count` spans: meta3[3 i..] = {fmmgpu_kind, level, stream (0 far field,
 * 1 near field)} and start/end in ms from the first span's start (P2PREDUCE = the
 * gather of near + far). Arrays hold `cap` spans; NULL pointers only query the count. */
int fmmgpu_set_trace(fmmgpu_ctx* ctx, int on);
int fmmgpu_trace_spans(fmmgpu_ctx* ctx, int cap, int* count, int* meta3, double* start_end_ms);
/* Runs `steps` back-to-back evaluations bracketed by CUDA events on the launching
 * stream: total_ms = device time of all steps; kind_ms10 (optional) = per-kind sums
 * as in fmmgpu_timings; launches (optional) = kernels launched in the region. */
int fmmgpu_time_evaluations(fmmgpu_ctx* ctx, int steps, double* total_ms, double* kind_ms10,
                            uint64_t* launches);

/* Isolated device time of one operator (CUDA events on the launching stream, the
 * operator alone on the device): `reps` back-to-back launches of kind (fmmgpu_kind,
 * P2M..P2P) at `level` (ignored for P2M / L2P / P2P; -1 = all levels of that kind),
 * average ms per repetition in *ms. Accumulators are left dirty: call fmmgpu_reset
 * (or fmmgpu_evaluate) before reading fields. */
int fmmgpu_time_operator(fmmgpu_ctx* ctx, int kind, int level, int reps, double* ms);

/* ---- accuracy check: direct_oracle (direct.cpp:202-226) on the device ------------
 * Exact sums over all n input particles (self excluded) for the k sampled input indices
 * `targets` (host array), as run_fmm's check (bench.cpp:366-398) uses them; outputs
 * are host arrays of k doubles (any may be NULL). Deterministic. */
int fmmgpu_direct(fmmgpu_ctx* ctx, const uint32_t* targets, uint64_t k, double* potential,
                  double* fx, double* fy, double* fz);

/* ---- multi-GPU: contiguous Morton ranges of leaves -------------
 * No reference counterpart (the reference is single-process); added by
 * the north star. Every rank builds the whole tree from the whole particle set, then
 * fmmgpu_partition makes this context rank `rank` of `nranks`: leaves are split into
 * contiguous Morton ranges aligned to the cells of an alignment level and balanced by
 * estimated work; levels below it are replicated. Evaluations then compute only the
 * owned targets (gathered fields are zero for other particles), with one exchange per
 * upward level >= the alignment level (fmmgpu_exchange_plan): the alignment level's
 * multipoles are all-gathered when the replicated levels above it need them, deeper
 * levels exchange only the halo the M2L of each rank reads (per-peer send / receive).
 * An attached NCCL communicator does it inside fmmgpu_evaluate; without one the host
 * does it between fmmgpu_upward_level calls (stepped API). nranks = 1 restores the full
 * evaluation; 1 <= nranks <= 64. */
int fmmgpu_partition(fmmgpu_ctx* ctx, int rank, int nranks);
/* Exchange after the upward step of `level`: *kind = 0 none, 1 all-gather of every rank's
 * owned rows (fmmgpu_partition_ranges), 2 halo. For kind 2: the cells (ascending row
 * indices of the level) this rank sends to `peer` and receives from `peer`; arrays may be
 * NULL to query the counts. A rank's receive list from p equals p's send list to it. */
int fmmgpu_exchange_plan(const fmmgpu_ctx* ctx, int level, int peer, int* kind, uint32_t* send_cells,
                         uint32_t* send_count, uint32_t* recv_cells, uint32_t* recv_count);
/* Measurement aid (tools/scaling_projection.py): skip_exchange = 1 times one rank's
 * partitioned work on a single device without its peers; fields downloaded while it is
 * set are refused (FMMGPU_LOGIC_ERROR). */
int fmmgpu_set_measurement(fmmgpu_ctx* ctx, int skip_exchange);
/* first owned cell of every rank at `level` (nranks + 1 entries, last = cell count) */
int fmmgpu_partition_ranges(const fmmgpu_ctx* ctx, int level, uint32_t* begins);
int fmmgpu_partition_info(const fmmgpu_ctx* ctx, int* rank, int* nranks, int* align_level,
                          uint64_t* slot_begin, uint64_t* slot_end);
/* host-only balanced contiguous split of n weighted items: begins[nranks + 1] */
int fmmgpu_plan_partition(const uint64_t* weights, uint32_t n, int nranks, uint32_t* begins);
/* NCCL communicator (libnccl.so.2 loaded on first use): rank 0 creates the 128-byte
 * id, every rank passes it to fmmgpu_comm_init. */
int fmmgpu_comm_unique_id(char* out128);
int fmmgpu_comm_init(fmmgpu_ctx* ctx, const char* id128, int nranks, int rank);
int fmmgpu_comm_destroy(fmmgpu_ctx* ctx);
/* stepped evaluation: fmmgpu_reset; fmmgpu_upward_level(leaf), (leaf-1), ..., (2)
 * (P2M at the leaf, M2M above; owned or replicated cells), the caller exchanging each
 * level >= the alignment level in between; then fmmgpu_downward (M2L, L2L, L2P, P2P,
 * gather). Synchronous. */
int fmmgpu_upward_level(fmmgpu_ctx* ctx, int level);
int fmmgpu_downward(fmmgpu_ctx* ctx);

/* Distributed input (halo particles; csrc/dist.cu). Rank r holds only
 * the input slice [offsets[r], offsets[r+1]) of the n particles (input order, slices in
 * rank order). Replaces GroupTree::build (geometry.cpp:73-161) for a partitioned run:
 * only Morton keys (8 B per particle) are all-gathered; the tree is bit-identical to the
 * single-device build of the whole set; each rank then receives the particle records of
 * its owned leaves and their 26-neighbour halo, nothing else.
 *
 * With an attached NCCL communicator, one call does all of it: */
int fmmgpu_build_tree_distributed(fmmgpu_ctx* ctx, const double* xyzw_local, uint64_t n_local, int on_device,
                                  int height, int group, const double* root4 /* NULL: bounding cube */);
/* Stepped form (the caller supplies the collectives):
 *   fmmgpu_dist_local   upload the slice, *lohi6 = its per-axis {min[3], max[3]};
 *   (caller: min / max over ranks) fmmgpu_root_from_bounds -> root cube (geometry.cpp:28-34);
 *   fmmgpu_dist_keys    the slice's leaf keys (u64) and its outside-the-root flag;
 *   (caller: all-gather keys in rank order, OR the flags)
 *   fmmgpu_dist_build   tree from the keys, fmmgpu_partition(rank, nranks), particle plan,
 *                       own records placed;
 *   fmmgpu_dist_plan    per peer: Morton slots sent to / received from it (NULL = counts);
 *   fmmgpu_dist_pack / fmmgpu_dist_unpack   records {x,y,z,w} of those slots, in that order;
 *   fmmgpu_dist_check   coincident particles among the owned leaves (*flag bit 2);
 *   (caller: OR the flags) fmmgpu_dist_commit   FMMGPU_DOMAIN_ERROR if set, else the tree
 *                       is ready for evaluations. */
int fmmgpu_root_from_bounds(const double* lohi6, double* root4);
int fmmgpu_dist_local(fmmgpu_ctx* ctx, const double* xyzw_local, uint64_t n_local, int on_device, double* lohi6);
int fmmgpu_dist_keys(fmmgpu_ctx* ctx, const double* root4, int height, uint64_t* keys_out, int out_on_device,
                     int* flag);
int fmmgpu_dist_build(fmmgpu_ctx* ctx, const uint64_t* keys_all, int keys_on_device, const uint64_t* offsets,
                      int rank, int nranks, int height, int group, const double* root4, int flag);
int fmmgpu_dist_plan(fmmgpu_ctx* ctx, int peer, uint32_t* send_slots, uint32_t* send_count, uint32_t* recv_slots,
                     uint32_t* recv_count);
int fmmgpu_dist_pack(fmmgpu_ctx* ctx, int peer, double* records_out, int out_on_device);
int fmmgpu_dist_unpack(fmmgpu_ctx* ctx, int peer, const double* records_in, int in_on_device);
int fmmgpu_dist_check(fmmgpu_ctx* ctx, int* flag);
int fmmgpu_dist_commit(fmmgpu_ctx* ctx, int flag);

/* bench.cpp:19-61 generate_particles (mt19937_64, explicit scaling); dist 0 uniform,
 * 1 sphere, 2 ellipsoid surface (config D: the sphere's directions on semi-axes
 * 0.5, 0.35, 0.2). Host-side input generator so both sides see identical doubles. */
void fmmgpu_generate_particles(uint64_t n, int dist, uint64_t seed, double* xyzw);

#ifdef __cplusplus
}
#endif
#endif /* FMMGPU_H_ */
