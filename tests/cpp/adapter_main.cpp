// C++ drop-in check of include/taskfmm_b200.hpp (the reference-API mirror over the
// C ABI). Built and run by tests/test_cpp_adapter.py on a GPU box:
//   adapter_main <n> <height> <acc> <seed> <out.bin> [<group> <dist> <order.bin>]
// Runs the evaluation task by task in a valid reference DAG order (run_task,
// bench.cpp:255-344) and as evaluate(); with an order file (the reference's own task
// graph for these particles, int32 {kind, level, block} per task, in a topological
// order that runs the most downstream ready task first) also that order on one thread
// and the same task list pulled by 8 threads at once (the reference's execute() calls
// run_task from its workers, runtime.cpp:165). Writes every field set, and checks the
// reference exception classes.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <stdexcept>
#include <vector>

#include "taskfmm_b200.hpp"

using namespace taskfmm_b200;

static int expect_throw(const char* what, auto&& f, auto tag) {
  try {
    f();
  } catch (const decltype(tag)&) {
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s: wrong exception %s\n", what, e.what());
    return 1;
  }
  std::fprintf(stderr, "%s: no exception\n", what);
  return 1;
}

int main(int argc, char** argv) {
  if (argc != 6 && argc != 9) return 2;
  RunConfig cfg;
  cfg.n = std::strtoull(argv[1], nullptr, 10);
  cfg.height = std::atoi(argv[2]);
  cfg.acc = std::atoi(argv[3]);
  cfg.seed = std::strtoull(argv[4], nullptr, 10);
  if (argc == 9) {
    cfg.group_size = std::atoi(argv[6]);
    cfg.dist = std::atoi(argv[7]) ? Distribution::Sphere : Distribution::Uniform;
  }
  auto particles = generate_particles(cfg.n, cfg.dist, cfg.seed);
  FmmContext ctx(particles, cfg);
  const int leaf = cfg.height - 1;
  // a valid topological order of the reference task graph (taskflow.cpp:215-247),
  // three blocks per (kind, level): P2P first, then the far-field chain
  ctx.reset();
  std::uint32_t id = 0;
  auto run = [&](TaskKind k, int level) {
    for (std::uint32_t b = 0; b < 3; ++b) ctx.run_task(Task{id++, k, static_cast<std::int16_t>(level), b, 0});
  };
  run(TaskKind::P2P, leaf);
  run(TaskKind::P2M, leaf);
  for (int v = leaf - 1; v >= 2; --v) run(TaskKind::M2M, v);
  for (int v = 2; v <= leaf; ++v) run(TaskKind::M2L, v);
  for (int v = 2; v < leaf; ++v) run(TaskKind::L2L, v);
  run(TaskKind::L2P, leaf);
  run(TaskKind::P2PReduce, leaf);
  const auto a = ctx.gather();
  ctx.evaluate();
  const auto b = ctx.gather();
  std::vector<FmmContext::Fields> sets{a, b};
  if (argc == 9) {
    std::vector<Task> tasks;
    std::FILE* o = std::fopen(argv[8], "rb");
    if (!o) return 4;
    std::int32_t t[3];
    while (std::fread(t, 4, 3, o) == 3)
      tasks.push_back(Task{static_cast<std::uint32_t>(tasks.size()), static_cast<TaskKind>(t[0]),
                           static_cast<std::int16_t>(t[1]), static_cast<std::uint32_t>(t[2]), 0});
    std::fclose(o);
    ctx.reset();
    for (const Task& task : tasks) ctx.run_task(task);
    sets.push_back(ctx.gather());
    ctx.reset();
    std::atomic<std::size_t> next{0};
    std::vector<std::thread> workers;
    for (int w = 0; w < 8; ++w)
      workers.emplace_back([&] {
        for (std::size_t i; (i = next.fetch_add(1)) < tasks.size();) ctx.run_task(tasks[i]);
      });
    for (auto& th : workers) th.join();
    sets.push_back(ctx.gather());
  }
  std::FILE* f = std::fopen(argv[5], "wb");
  if (!f) return 3;
  for (const auto& fs : sets)
    for (const auto* v : {&fs.potential, &fs.fx, &fs.fy, &fs.fz}) std::fwrite(v->data(), 8, v->size(), f);
  std::fclose(f);

  int bad = 0;
  RunConfig bad_h = cfg;
  bad_h.height = 2;
  bad += expect_throw("height 2", [&] { FmmContext c(particles, bad_h); }, std::invalid_argument(""));
  RunConfig bad_acc = cfg;
  bad_acc.acc = 11;
  bad += expect_throw("acc 11", [&] { FmmContext c(particles, bad_acc); }, std::invalid_argument(""));
  std::vector<Particle> dup = {{{0.1, 0.1, 0.1}, 1.0}, {{0.1, 0.1, 0.1}, 1.0}, {{0.9, 0.9, 0.9}, 1.0}};
  bad += expect_throw("coincident", [&] { FmmContext c(dup, cfg); }, std::domain_error(""));
  bad += expect_throw("level", [&] { ctx.run_task(Task{0, TaskKind::M2L, 99, 0, 0}); }, std::out_of_range(""));
  const auto r = run_fmm(cfg);  // includes the device-side oracle check (cfg.check = 1000)
  if (!(r.eps_l2_potential > 0 && r.eps_l2_potential < 1e-4 && r.eps_l2_force > 0 && r.eps_l2_force < 1e-2)) {
    std::fprintf(stderr, "run_fmm accuracy out of range: %g %g\n", r.eps_l2_potential, r.eps_l2_force);
    ++bad;
  }
  if (relative_l2_error(r.fields.potential, b.potential) != 0.0) {
    std::fprintf(stderr, "run_fmm differs from evaluate\n");
    ++bad;
  }
  std::printf("adapter: n=%llu setup %.3f s exec %.3f s eps_l2 %.3e / %.3e, %d failures\n",
              static_cast<unsigned long long>(cfg.n), r.setup_seconds, r.exec_seconds, r.eps_l2_potential,
              r.eps_l2_force, bad);
  return bad;
}
