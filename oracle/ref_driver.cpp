// oracle/_ref driver — TEST INFRASTRUCTURE ONLY.
//
// A C ABI around the UNMODIFIED reference sources (/root/reference/proj/src/*.cpp,
// compiled in place by oracle/build_ref.sh against oracle/eigen_shim). Only tests/,
// __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs load the
// resulting oracle/_ref/libtaskfmm_ref.so, and only as the checker or the timed CPU
// reference — never as the product path.
//
// Entry points mirror the reference seams:
//   FmmContext ctor / run_task / gather      bench.cpp:220-365
//   execute(graph, workers, policy, body)    runtime.cpp:91-216
//   GroupTree levels, ParticleStore          geometry.hpp:34-65
//   NearFieldPlan, LevelM2L                  direct.hpp:22-33, taskflow.hpp:46-66
//   M2LOperatorSet::save_cache               m2l.cpp:212-245
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "taskfmm/bench.hpp"

using namespace taskfmm;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::domain_error*>(&e)) return 2;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 3;
  if (dynamic_cast<const std::logic_error*>(&e)) return 4;
  return 5;
}
std::vector<Particle> to_particles(const double* xyzw, std::uint64_t n) {
  std::vector<Particle> ps(n);
  for (std::uint64_t i = 0; i < n; ++i)
    ps[i] = {{xyzw[4 * i], xyzw[4 * i + 1], xyzw[4 * i + 2]}, xyzw[4 * i + 3]};
  return ps;
}
struct Ctx {
  std::unique_ptr<FmmContext> fmm;
  int acc = 0;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// bench.cpp:29-61 (mt19937_64, explicit scaling). dist 0 = uniform, 1 = sphere.
void ref_generate_particles(std::uint64_t n, int dist, std::uint64_t seed, double* xyzw) {
  const auto ps = generate_particles(n, dist == 0 ? Distribution::Uniform : Distribution::Sphere, seed);
  for (std::uint64_t i = 0; i < n; ++i) {
    xyzw[4 * i] = ps[i].position[0];
    xyzw[4 * i + 1] = ps[i].position[1];
    xyzw[4 * i + 2] = ps[i].position[2];
    xyzw[4 * i + 3] = ps[i].weight;
  }
}

int ref_create(const double* xyzw, std::uint64_t n, int height, int acc, int group_size, void** out) {
  try {
    RunConfig cfg;
    cfg.height = height;
    cfg.acc = acc;
    cfg.group_size = group_size;
    auto c = std::make_unique<Ctx>();
    c->fmm = std::make_unique<FmmContext>(to_particles(xyzw, n), cfg);
    c->acc = acc;
    *out = c.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_destroy(void* h) { delete static_cast<Ctx*>(h); }

double ref_setup_seconds(void* h) { return static_cast<Ctx*>(h)->fmm->setup_seconds(); }

// reset + execute(graph, workers, policy) (runtime.cpp:91); returns wall seconds or -1.
double ref_execute(void* h, int workers, int policy) {
  auto* c = static_cast<Ctx*>(h);
  try {
    c->fmm->reset();
    const auto pol = policy == 0 ? SchedulePolicy::Fifo
                     : policy == 1 ? SchedulePolicy::Priority
                                   : SchedulePolicy::CostModel;
    return execute(c->fmm->graph(), workers, pol, c->fmm->body()).wall_seconds;
  } catch (const std::exception& e) {
    fail(e);
    return -1.0;
  }
}

// reset, then run_task serially in task-id order (a topological order by
// construction, taskflow.cpp:172-209) for the kinds in kind_mask (bit = TaskKind).
int ref_run_serial(void* h, unsigned kind_mask) {
  auto* c = static_cast<Ctx*>(h);
  try {
    c->fmm->reset();
    for (const Task& t : c->fmm->graph().tasks)
      if (kind_mask & (1u << static_cast<int>(t.kind))) c->fmm->run_task(t);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Run a bounded sample: the first `max_tasks` tasks of each selected kind, serially.
int ref_run_tasks(void* h, const std::uint32_t* ids, std::uint64_t count) {
  auto* c = static_cast<Ctx*>(h);
  try {
    for (std::uint64_t i = 0; i < count; ++i) c->fmm->run_task(c->fmm->graph().tasks[ids[i]]);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_reset(void* h) { static_cast<Ctx*>(h)->fmm->reset(); }

std::uint64_t ref_task_count(void* h) { return static_cast<Ctx*>(h)->fmm->graph().size(); }
// per task: kind, level, block, work
void ref_task_info(void* h, std::uint8_t* kind, std::int16_t* level, std::uint32_t* block,
                   std::uint64_t* work) {
  const auto& g = static_cast<Ctx*>(h)->fmm->graph();
  for (std::size_t i = 0; i < g.size(); ++i) {
    kind[i] = static_cast<std::uint8_t>(g.tasks[i].kind);
    level[i] = g.tasks[i].level;
    block[i] = g.tasks[i].block;
    work[i] = g.tasks[i].work;
  }
}

void ref_fields(void* h, double* pot, double* fx, double* fy, double* fz) {
  const auto f = static_cast<Ctx*>(h)->fmm->gather();
  std::memcpy(pot, f.potential.data(), 8 * f.potential.size());
  std::memcpy(fx, f.fx.data(), 8 * f.fx.size());
  std::memcpy(fy, f.fy.data(), 8 * f.fy.size());
  std::memcpy(fz, f.fz.data(), 8 * f.fz.size());
}

void ref_root_cube(void* h, double* out4) {
  const Cube& r = static_cast<Ctx*>(h)->fmm->tree().root_cube();
  out4[0] = r.center[0];
  out4[1] = r.center[1];
  out4[2] = r.center[2];
  out4[3] = r.width;
}

// Morton-ordered ParticleStore (geometry.hpp:59-65): x,y,z,w and id.
void ref_sorted_particles(void* h, double* x, double* y, double* z, double* w, std::uint32_t* id) {
  const ParticleStore& st = static_cast<Ctx*>(h)->fmm->tree().particles();
  const std::size_t n = st.size();
  std::memcpy(x, st.x.data(), 8 * n);
  std::memcpy(y, st.y.data(), 8 * n);
  std::memcpy(z, st.z.data(), 8 * n);
  std::memcpy(w, st.w.data(), 8 * n);
  std::memcpy(id, st.id.data(), 4 * n);
}

std::uint64_t ref_level_cells(void* h, int v) {
  return static_cast<Ctx*>(h)->fmm->tree().level(v).cells.size();
}
// Cell = {u64 code, u32 first_particle, particle_count, parent, first_child, child_count} (32 B)
void ref_level_dump(void* h, int v, void* cells_out, std::uint32_t* block_offsets_out) {
  const TreeLevel& lv = static_cast<Ctx*>(h)->fmm->tree().level(v);
  static_assert(sizeof(Cell) == 32);
  std::memcpy(cells_out, lv.cells.data(), sizeof(Cell) * lv.cells.size());
  std::memcpy(block_offsets_out, lv.block_offsets.data(), 4 * lv.block_offsets.size());
}
std::uint64_t ref_level_blocks(void* h, int v) {
  return static_cast<Ctx*>(h)->fmm->tree().level(v).block_count();
}
// which: 0 multipole, 1 local_own, 2 local_down
void ref_level_expansion(void* h, int v, int which, double* out) {
  const TreeLevel& lv = static_cast<Ctx*>(h)->fmm->tree().level(v);
  const auto& a = which == 0 ? lv.multipole : which == 1 ? lv.local_own : lv.local_down;
  std::memcpy(out, a.data(), 8 * a.size());
}
// Morton-order accumulators (before gather)
void ref_sorted_fields(void* h, double* pot, double* fx, double* fy, double* fz) {
  const ParticleStore& st = static_cast<Ctx*>(h)->fmm->tree().particles();
  const std::size_t n = st.size();
  std::memcpy(pot, st.potential.data(), 8 * n);
  std::memcpy(fx, st.fx.data(), 8 * n);
  std::memcpy(fy, st.fy.data(), 8 * n);
  std::memcpy(fz, st.fz.data(), 8 * n);
}

// NearFieldPlan (direct.hpp:22-33)
std::uint64_t ref_near_entries(void* h) { return static_cast<Ctx*>(h)->fmm->plan().near.near_cells.size(); }
void ref_near_dump(void* h, std::uint32_t* offsets, std::uint32_t* cells) {
  const NearFieldPlan& p = static_cast<Ctx*>(h)->fmm->plan().near;
  std::memcpy(offsets, p.near_offsets.data(), 4 * p.near_offsets.size());
  std::memcpy(cells, p.near_cells.data(), 4 * p.near_cells.size());
}
std::uint64_t ref_near_total_directional(void* h) {
  return static_cast<Ctx*>(h)->fmm->plan().near.total_directional;
}
// per block: task_interactions, and CSR of partners_above / contributors_below
void ref_near_blocks(void* h, std::uint64_t* task_interactions, std::uint32_t* above_off,
                     std::uint32_t* above, std::uint32_t* below_off, std::uint32_t* below) {
  const NearFieldPlan& p = static_cast<Ctx*>(h)->fmm->plan().near;
  const std::size_t nb = p.partners_above.size();
  above_off[0] = below_off[0] = 0;
  for (std::size_t b = 0; b < nb; ++b) {
    task_interactions[b] = p.task_interactions[b];
    above_off[b + 1] = above_off[b] + static_cast<std::uint32_t>(p.partners_above[b].size());
    below_off[b + 1] = below_off[b] + static_cast<std::uint32_t>(p.contributors_below[b].size());
    std::memcpy(above + above_off[b], p.partners_above[b].data(), 4 * p.partners_above[b].size());
    std::memcpy(below + below_off[b], p.contributors_below[b].data(), 4 * p.contributors_below[b].size());
  }
}
std::uint64_t ref_near_block_list_sizes(void* h, std::uint64_t* below_total) {
  const NearFieldPlan& p = static_cast<Ctx*>(h)->fmm->plan().near;
  std::uint64_t a = 0, b = 0;
  for (const auto& v : p.partners_above) a += v.size();
  for (const auto& v : p.contributors_below) b += v.size();
  *below_total = b;
  return a;
}

// LevelM2L (taskflow.hpp:46-66): pairs as (target, source, vec) triples
std::uint64_t ref_far_pairs(void* h, int v) { return static_cast<Ctx*>(h)->fmm->plan().far[v].pairs.size(); }
void ref_far_dump(void* h, int v, std::uint32_t* target, std::uint32_t* source, std::uint16_t* vec,
                  std::uint64_t* group_offsets) {
  const LevelM2L& f = static_cast<Ctx*>(h)->fmm->plan().far[v];
  for (std::size_t i = 0; i < f.pairs.size(); ++i) {
    target[i] = f.pairs[i].target;
    source[i] = f.pairs[i].source;
    vec[i] = f.pairs[i].vec;
  }
  std::memcpy(group_offsets, f.group_offsets.data(), 8 * f.group_offsets.size());
}
std::uint64_t ref_far_source_blocks_total(void* h, int v) {
  std::uint64_t t = 0;
  for (const auto& s : static_cast<Ctx*>(h)->fmm->plan().far[v].source_blocks) t += s.size();
  return t;
}
void ref_far_source_blocks(void* h, int v, std::uint32_t* off, std::uint32_t* blocks) {
  const auto& sb = static_cast<Ctx*>(h)->fmm->plan().far[v].source_blocks;
  off[0] = 0;
  for (std::size_t b = 0; b < sb.size(); ++b) {
    off[b + 1] = off[b] + static_cast<std::uint32_t>(sb[b].size());
    std::memcpy(blocks + off[b], sb[b].data(), 4 * sb[b].size());
  }
}

int ref_save_m2l_cache(void* h, const char* path) {
  return static_cast<Ctx*>(h)->fmm->ops().save_cache(path) ? 0 : 5;
}
void ref_m2l_ranks(void* h, int* ranks16) {
  const auto& r = static_cast<Ctx*>(h)->fmm->ops().report();
  for (int c = 0; c < 16; ++c) ranks16[c] = r.ranks[c];
}

// Standalone operator set (m2l.cpp:136-144) -> cache file; returns weighted mean rank.
double ref_build_m2l_cache(int order, double eps, const char* path, int* ranks16) {
  try {
    M2LOperatorSet ops(order, eps);
    for (int c = 0; c < 16; ++c) ranks16[c] = ops.report().ranks[c];
    if (path && *path && !ops.save_cache(path)) return -1;
    return ops.report().weighted_mean_rank;
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

// assemble_m2l (m2l.cpp:90-111) column-major n3 x n3
void ref_assemble_m2l(int i, int j, int k, int order, double width, double* out) {
  const auto m = assemble_m2l({i, j, k}, order, width);
  std::memcpy(out, m.data(), 8 * m.size());
}
void ref_canonicalize(int i, int j, int k, int* index, int* perm3, int* sign3) {
  const auto c = canonicalize_m2l_vector({i, j, k});
  *index = c.index;
  for (int a = 0; a < 3; ++a) {
    perm3[a] = c.op.perm[a];
    sign3[a] = c.op.sign[a];
  }
}

// InterpolationEngine single-cell operators (chebyshev.hpp:45-63)
void ref_p2m(int order, const double* cube4, const double* px, const double* py, const double* pz,
             const double* pw, std::uint64_t n, double* multipole) {
  InterpolationEngine e(order);
  Cube c{{cube4[0], cube4[1], cube4[2]}, cube4[3]};
  const std::size_t l3 = static_cast<std::size_t>(order) * order * order;
  e.p2m(c, {px, n}, {py, n}, {pz, n}, {pw, n}, {multipole, l3});
}
void ref_l2p(int order, const double* cube4, const double* local, const double* px,
             const double* py, const double* pz, std::uint64_t n, double* pot, double* fx,
             double* fy, double* fz) {
  InterpolationEngine e(order);
  Cube c{{cube4[0], cube4[1], cube4[2]}, cube4[3]};
  const std::size_t l3 = static_cast<std::size_t>(order) * order * order;
  e.l2p(c, {local, l3}, {px, n}, {py, n}, {pz, n}, {pot, n}, {fx, n}, {fy, n}, {fz, n});
}
void ref_m2m(int order, int octant, const double* child, double* parent) {
  InterpolationEngine e(order);
  const std::size_t l3 = static_cast<std::size_t>(order) * order * order;
  e.m2m(octant, {child, l3}, {parent, l3});
}
void ref_l2l(int order, int octant, const double* parent, double* child) {
  InterpolationEngine e(order);
  const std::size_t l3 = static_cast<std::size_t>(order) * order * order;
  e.l2l(octant, {parent, l3}, {child, l3});
}
void ref_child_matrix(int order, int side, double* out) {
  InterpolationEngine e(order);
  std::memcpy(out, e.child_matrix(side).data(), 8 * order * order);
}
void ref_roots(int order, double* out) {
  const auto r = chebyshev_roots(order);
  std::memcpy(out, r.data(), 8 * order);
}

// direct_oracle (direct.cpp:202-226)
void ref_direct_oracle(const double* xyzw, std::uint64_t n, const std::uint32_t* targets,
                       std::uint64_t nt, double* pot, double* fx, double* fy, double* fz) {
  const auto ps = to_particles(xyzw, n);
  const auto r = direct_oracle(ps, {targets, nt});
  std::memcpy(pot, r.potential.data(), 8 * nt);
  std::memcpy(fx, r.fx.data(), 8 * nt);
  std::memcpy(fy, r.fy.data(), 8 * nt);
  std::memcpy(fz, r.fz.data(), 8 * nt);
}

// Morton helpers (geometry.cpp:38-57) and bounding_cube (geometry.cpp:18-36)
std::uint64_t ref_morton_encode(std::uint32_t i, std::uint32_t j, std::uint32_t k, int level) {
  return morton_encode(i, j, k, level);
}
int ref_bounding_cube(const double* xyzw, std::uint64_t n, double* out4) {
  try {
    const Cube c = bounding_cube(to_particles(xyzw, n));
    out4[0] = c.center[0];
    out4[1] = c.center[1];
    out4[2] = c.center[2];
    out4[3] = c.width;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
// GroupTree validation only (error behaviour, geometry.cpp:59-71, 82-94, 126-136)
int ref_tree_check(const double* xyzw, std::uint64_t n, int height, int group_size) {
  try {
    GroupTree t(to_particles(xyzw, n), height, group_size);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// count_interactions + build_ledger (taskflow.cpp:113-135, bench.cpp:151-181):
// out[kind*height + level] = flops, work likewise
int ref_ledger(const double* xyzw, std::uint64_t n, int height, int acc, int group_size,
               std::uint64_t* flops, std::uint64_t* work) {
  try {
    const auto ps = to_particles(xyzw, n);
    GroupTree tree(ps, height, group_size);
    const auto stats = count_interactions(tree);
    M2LOperatorSet ops(acc, std::pow(10.0, -acc));
    const auto ledger = build_ledger(stats, ops.report(), acc, n, height);
    for (int k = 0; k < TASK_KIND_COUNT; ++k)
      for (int v = 0; v < height; ++v) {
        flops[k * height + v] = ledger.rows[k][v].flops;
        work[k * height + v] = ledger.rows[k][v].work;
      }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"

extern "C" {

// count_interactions + build_ledger over an existing context's tree and operators
// (bench.cpp:440-442): flops / work [kind * height + level], m2l_pairs [level * 16 + c].
int ref_ctx_ledger(void* h, std::uint64_t* flops, std::uint64_t* work, std::uint64_t* pairs16) {
  auto* c = static_cast<Ctx*>(h);
  try {
    const GroupTree& tree = c->fmm->tree();
    const int height = tree.height();
    const auto stats = count_interactions(tree);
    const auto ledger = build_ledger(stats, c->fmm->ops().report(), c->acc, tree.particles().size(), height);
    for (int k = 0; k < TASK_KIND_COUNT; ++k)
      for (int v = 0; v < height; ++v) {
        flops[k * height + v] = ledger.rows[k][v].flops;
        work[k * height + v] = ledger.rows[k][v].work;
      }
    for (int v = 0; v < height; ++v)
      for (int cl = 0; cl < 16; ++cl)
        pairs16[v * 16 + cl] = v < static_cast<int>(stats.m2l_pairs.size()) ? stats.m2l_pairs[v][cl] : 0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// run_fmm (bench.cpp:415-469) with out_dir: the reference's own writers produce
// results.csv and summary.json (bench.cpp:400-411, 504-584). dist 0 uniform, 1 sphere.
int ref_run_fmm(std::uint64_t n, int dist, std::uint64_t seed, int height, int acc, int group_size,
                int workers, std::uint64_t check, const char* out_dir, double* eps2) {
  try {
    RunConfig cfg;
    cfg.n = n;
    cfg.dist = dist == 0 ? Distribution::Uniform : Distribution::Sphere;
    cfg.seed = seed;
    cfg.height = height;
    cfg.acc = acc;
    cfg.group_size = group_size;
    cfg.workers = workers;
    cfg.check = check;
    cfg.out_dir = out_dir ? out_dir : "";
    const RunResult r = run_fmm(cfg);
    if (eps2) {
      eps2[0] = r.eps_l2_potential;
      eps2[1] = r.eps_l2_force;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"

extern "C" {
// The task graph's edges (TaskGraph, taskflow.hpp:34-42): successors of task i are
// succ[off[i] .. off[i+1]); returns the edge count (call with null arrays to size).
std::uint64_t ref_task_edges(void* h, std::uint32_t* off, std::uint32_t* succ) {
  const auto& g = static_cast<Ctx*>(h)->fmm->graph();
  std::uint64_t e = 0;
  for (std::size_t i = 0; i < g.size(); ++i) {
    if (off) off[i] = static_cast<std::uint32_t>(e);
    for (std::uint32_t s : g.tasks[i].successors) {
      if (succ) succ[e] = s;
      ++e;
    }
  }
  if (off) off[g.size()] = static_cast<std::uint32_t>(e);
  return e;
}
}  // extern "C"
