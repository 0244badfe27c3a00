// taskfmm_b200.hpp — header-only C++ mirror of the reference's operator API over the
// C ABI of fmmgpu.h (libfmmgpu.so, CUDA sm_100a). A C++ caller of the reference
// ("taskfmm", /root/reference/proj/include/taskfmm/*.hpp) switches its FMM evaluation
// path by replacing `taskfmm::` with `taskfmm_b200::` for the names below; the
// semantics (accumulate contract, input-order fields, exception classes) are the
// reference's. See INTEGRATION.md.
//
//   Particle, Cube                     geometry.hpp:16-24
//   TaskKind, Task                     taskflow.hpp:15-31
//   RunConfig, Distribution            bench.hpp:19-35
//   generate_particles                 bench.cpp:29-61 (same mt19937_64 stream)
//   relative_l2_error                  bench.cpp:91-100
//   FmmContext (ctor, reset, run_task, gather, setup_seconds)   bench.hpp:86-121
//   run_fmm (oracle check on the device, no writers)            bench.cpp:415-469
//
// Granularity: the device runs one launch per (operator, level), in the fixed far-field
// chain P2M -> M2M(leaf-1 .. 2) -> M2L(2 .. leaf) -> L2L(2 .. leaf-1) -> L2P, with P2P
// independent of it. run_task(task) launches, since the last reset(), every chain
// element up to and including (task.kind, task.level) that has not run yet (each level
// launch reads only inputs complete at that point: particles, or levels earlier in the
// chain), and P2P on the first P2P / P2PReduce task; the remaining tasks of a level are
// no-ops. So executing a reference TaskGraph in ANY topological order -- including the
// graphs whose elided zero-pair M2L blocks leave L2L(2, b) without predecessors
// (taskflow.cpp:179-186) -- reproduces one evaluation. run_task may be called from the
// reference's worker threads (execute, runtime.cpp:165): calls are serialised by a
// mutex. The first P2P / P2PReduce task runs the mutual near field and its ordered slot
// drain (p2p_block(mutual=true) + p2p_reduce, direct.cpp:151-200).
#pragma once

#include <array>
#include <chrono>
#include <cmath>
#include <algorithm>
#include <cstdint>
#include <limits>
#include <mutex>
#include <utility>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fmmgpu.h"

namespace taskfmm_b200 {

struct Particle {
  std::array<double, 3> position;
  double weight;
};

struct Cube {
  std::array<double, 3> center{0.5, 0.5, 0.5};
  double width = 1.0;
};

enum class TaskKind : std::uint8_t { P2M, M2M, M2L, L2L, L2P, P2P, P2PReduce };
inline constexpr int TASK_KIND_COUNT = 7;

struct Task {
  std::uint32_t id = 0;
  TaskKind kind = TaskKind::P2M;
  std::int16_t level = 0;
  std::uint32_t block = 0;
  std::uint64_t work = 0;
};

enum class Distribution { Uniform, Sphere };

struct RunConfig {
  std::uint64_t n = 10000;
  Distribution dist = Distribution::Uniform;
  int height = 4;
  int acc = 5;  // interpolation order l = acc, svd eps = 10^-acc
  int group_size = 250;
  std::uint64_t seed = 42;
  std::uint64_t check = 1000;  // oracle sample size, 0 disables (exact sums on the device)
  int device = 0;
};

// status code -> the reference's exception class
inline void check(int rc, const char* msg) {
  switch (rc) {
    case FMMGPU_OK: return;
    case FMMGPU_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case FMMGPU_DOMAIN_ERROR: throw std::domain_error(msg);
    case FMMGPU_OUT_OF_RANGE: throw std::out_of_range(msg);
    case FMMGPU_LOGIC_ERROR: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline std::vector<Particle> generate_particles(std::uint64_t n, Distribution dist, std::uint64_t seed) {
  std::vector<double> xyzw(4 * n);
  fmmgpu_generate_particles(n, dist == Distribution::Uniform ? 0 : 1, seed, xyzw.data());
  std::vector<Particle> out(n);
  for (std::uint64_t i = 0; i < n; ++i)
    out[i] = Particle{{xyzw[4 * i], xyzw[4 * i + 1], xyzw[4 * i + 2]}, xyzw[4 * i + 3]};
  return out;
}

inline double relative_l2_error(std::span<const double> estimate, std::span<const double> reference) {
  if (estimate.size() != reference.size()) throw std::invalid_argument("relative_l2_error: size mismatch");
  double num = 0, den = 0;
  for (std::size_t i = 0; i < estimate.size(); ++i) {
    const double d = estimate[i] - reference[i];
    num += d * d;
    den += reference[i] * reference[i];
  }
  if (den == 0) return num == 0 ? 0.0 : std::numeric_limits<double>::infinity();  // bench.cpp:97-98
  return std::sqrt(num / den);
}

class FmmContext {
 public:
  struct Fields {
    std::vector<double> potential, fx, fy, fz;  // original input order
  };

  FmmContext(std::vector<Particle> particles, const RunConfig& cfg) : input_(std::move(particles)), cfg_(cfg) {
    const auto t0 = std::chrono::steady_clock::now();
    if (cfg.acc < 2) throw std::invalid_argument("accuracy parameter must be at least 2");  // bench.cpp:223
    check(fmmgpu_create(cfg.device, cfg.acc, std::pow(10.0, -cfg.acc), &ctx_), fmmgpu_global_error());
    std::vector<double> xyzw(4 * input_.size());
    for (std::size_t i = 0; i < input_.size(); ++i) {
      xyzw[4 * i] = input_[i].position[0];
      xyzw[4 * i + 1] = input_[i].position[1];
      xyzw[4 * i + 2] = input_[i].position[2];
      xyzw[4 * i + 3] = input_[i].weight;
    }
    try {
      call(fmmgpu_build_tree(ctx_, xyzw.empty() ? nullptr : xyzw.data(), input_.size(), 0, cfg.height,
                             cfg.group_size, nullptr));
      call(fmmgpu_reset(ctx_));
    } catch (...) {
      fmmgpu_destroy(ctx_);
      throw;
    }
    setup_seconds_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  ~FmmContext() { fmmgpu_destroy(ctx_); }
  FmmContext(const FmmContext&) = delete;
  FmmContext& operator=(const FmmContext&) = delete;

  const std::vector<Particle>& input() const { return input_; }
  double setup_seconds() const { return setup_seconds_; }
  int height() const { return cfg_.height; }
  fmmgpu_ctx* handle() const { return ctx_; }

  //! FmmContext::reset (bench.cpp:240-253): zero every accumulator.
  void reset() {
    std::lock_guard<std::mutex> lock(mu_);
    call(fmmgpu_reset(ctx_));
    next_ = 0;
    p2p_done_ = false;
  }

  //! FmmContext::run_task (bench.cpp:255-344) at level granularity (see header).
  void run_task(const Task& task) {
    const int k = static_cast<int>(task.kind);
    if (k < 0 || k >= TASK_KIND_COUNT) throw std::invalid_argument("run_task: unknown task kind");
    if (task.level < 0 || task.level >= cfg_.height) throw std::out_of_range("run_task: level out of range");
    std::lock_guard<std::mutex> lock(mu_);
    if (task.kind == TaskKind::P2P || task.kind == TaskKind::P2PReduce) {
      if (task.level != cfg_.height - 1) throw std::out_of_range("run_task: P2P tasks live on the leaf level");
      if (!p2p_done_) call(fmmgpu_p2p(ctx_));
      p2p_done_ = true;
      return;
    }
    const auto it = std::find(chain_.begin(), chain_.end(), std::make_pair(task.kind, int(task.level)));
    if (it == chain_.end()) throw std::out_of_range("run_task: no such (kind, level) in the task graph");
    const std::size_t pos = static_cast<std::size_t>(it - chain_.begin());
    for (; next_ <= pos; ++next_) {
      const auto [kind, level] = chain_[next_];
      switch (kind) {
        case TaskKind::P2M: call(fmmgpu_p2m(ctx_)); break;
        case TaskKind::M2M: call(fmmgpu_m2m(ctx_, level)); break;
        case TaskKind::M2L: call(fmmgpu_m2l(ctx_, level)); break;
        case TaskKind::L2L: call(fmmgpu_l2l(ctx_, level)); break;
        case TaskKind::L2P: call(fmmgpu_l2p(ctx_)); break;
        default: break;
      }
    }
  }

  //! The whole task graph at once (reset + all payloads, near/far on two streams).
  void evaluate() { call(fmmgpu_evaluate(ctx_)); }

  //! FmmContext::gather (bench.cpp:350-365): fields in input order.
  Fields gather() const {
    Fields f;
    const std::size_t n = input_.size();
    f.potential.resize(n);
    f.fx.resize(n);
    f.fy.resize(n);
    f.fz.resize(n);
    call(fmmgpu_download_fields(ctx_, f.potential.data(), f.fx.data(), f.fy.data(), f.fz.data(), 0));
    return f;
  }

 private:
  void call(int rc) const { check(rc, fmmgpu_last_error(ctx_)); }

  std::vector<Particle> input_;
  RunConfig cfg_;
  fmmgpu_ctx* ctx_ = nullptr;
  double setup_seconds_ = 0;
  // the far-field chain in launch order (taskflow.cpp:143-289 dependencies, level granular)
  std::vector<std::pair<TaskKind, int>> chain_ = far_chain(cfg_.height);
  std::size_t next_ = 0;  // first chain element not launched since reset()
  bool p2p_done_ = false;
  std::mutex mu_;

  static std::vector<std::pair<TaskKind, int>> far_chain(int height) {
    const int leaf = height - 1;
    std::vector<std::pair<TaskKind, int>> c{{TaskKind::P2M, leaf}};
    for (int v = leaf - 1; v >= 2; --v) c.emplace_back(TaskKind::M2M, v);
    for (int v = 2; v <= leaf; ++v) c.emplace_back(TaskKind::M2L, v);
    for (int v = 2; v < leaf; ++v) c.emplace_back(TaskKind::L2L, v);
    c.emplace_back(TaskKind::L2P, leaf);
    return c;
  }
};

struct RunResult {
  RunConfig config;
  double setup_seconds = 0;
  double exec_seconds = 0;
  double wall_seconds = 0;
  double eps_l2_potential = -1;  // -1 when not checked
  double eps_l2_force = -1;
  FmmContext::Fields fields;
  std::vector<Particle> input;
};

//! bench.cpp:368-376
inline std::vector<std::uint32_t> check_targets(std::uint64_t n, std::uint64_t check) {
  std::vector<std::uint32_t> t;
  for (std::uint64_t k = 0; k < check; ++k) t.push_back(static_cast<std::uint32_t>(k * n / check));
  std::sort(t.begin(), t.end());
  t.erase(std::unique(t.begin(), t.end()), t.end());
  return t;
}

//! run_fmm (bench.cpp:415-469) without the ledger or writers; the oracle check
//! (bench.cpp:378-398) runs on the device (fmmgpu_direct).
inline RunResult run_fmm(const RunConfig& cfg) {
  const auto w0 = std::chrono::steady_clock::now();
  RunResult r;
  r.config = cfg;
  r.input = generate_particles(cfg.n, cfg.dist, cfg.seed);
  FmmContext ctx(r.input, cfg);
  r.setup_seconds = ctx.setup_seconds();
  const auto e0 = std::chrono::steady_clock::now();
  ctx.evaluate();
  r.fields = ctx.gather();
  r.exec_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - e0).count();
  if (cfg.check > 0 && !r.input.empty()) {
    const auto t = check_targets(r.input.size(), std::min<std::uint64_t>(cfg.check, r.input.size()));
    std::vector<double> pot(t.size()), fx(t.size()), fy(t.size()), fz(t.size());
    check(fmmgpu_direct(ctx.handle(), t.data(), t.size(), pot.data(), fx.data(), fy.data(), fz.data()),
          fmmgpu_last_error(ctx.handle()));
    std::vector<double> ep(t.size()), ef, rf;
    for (std::size_t i = 0; i < t.size(); ++i) {
      ep[i] = r.fields.potential[t[i]];
      ef.insert(ef.end(), {r.fields.fx[t[i]], r.fields.fy[t[i]], r.fields.fz[t[i]]});
      rf.insert(rf.end(), {fx[i], fy[i], fz[i]});
    }
    r.eps_l2_potential = relative_l2_error(ep, pot);
    r.eps_l2_force = relative_l2_error(ef, rf);
  }
  r.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
  return r;
}

}  // namespace taskfmm_b200
