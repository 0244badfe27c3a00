"""Benchmark of the B200 FMM evaluation path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config B]

A "step" is one FMM evaluation (all payloads of the reference task graph: P2M, M2M,
M2L, L2L, L2P, P2P + reduce, fields gathered to input order) over the resident
octree of config B: 10M uniform particles (bench.cpp:29-39, seed 42), height 7,
Chebyshev order 5, eps 1e-5, group size 250 -- BASELINE.json configs[1].

ours:       value = Mparticles/s from CUDA events on the launching stream (max over
            ranks), inputs resident in HBM; e2e = the same metric through the C ABI with
            pinned host buffers: H2D of the particles, tree build, evaluation, D2H of the
            four fields, every step (N = 1: fmmgpu_run_async pipelined, the serial
            fmmgpu_run beside it; N > 1: each rank's slice through
            fmmgpu_build_tree_distributed + evaluate + download).
reference:  the reference's own CPU implementation (oracle/_ref: the unmodified
            reference sources, FmmContext + execute with all host threads) on the same
            configuration (--cpu-sample: the labelled 1/8 sample), rank 0 only; setup,
            exec and the 1-worker time reported separately.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, dist, height, order, description)
    "A": (100_000, "uniform", 4, 5, "uniform cube N=100k, height 4, order 5"),
    "B": (10_000_000, "uniform", 7, 5, "uniform cube N=10M, height 7, order 5"),
    "C": (10_000_000, "uniform", 7, 7, "uniform cube N=10M, height 7, order 7"),
    "D": (20_000_000, "ellipsoid", 8, 5, "ellipsoid surface (semi-axes 0.5, 0.35, 0.2) N=20M, height 8, order 5"),
    "E": (100_000_000, "uniform", 8, 5, "uniform cube N=100M, height 8, order 5"),
}
# Labelled fallback (--cpu-sample): a bounded sample at the same particles per leaf (~38) and
# order, one level shallower (1/8 of the particles): the reference's per-particle work is
# the same.
CPU_SAMPLE = {"B": (1_250_000, "uniform", 6, 5), "C": (1_250_000, "uniform", 6, 7), "A": (100_000, "uniform", 4, 5),
              "D": (1_250_000, "ellipsoid", 6, 5), "E": (1_562_500, "uniform", 6, 5)}
# (volume clouds keep N / 8^h, the surface cloud N / 4^h: same particles per leaf as the
# full configuration, so the reference's per-particle work is the same)

METRIC = "FMM eval time (s) and Mparticles/s at N=10M, order 5; scaling 1/2/4/8 B200"
UNIT = "Mparticles/s"
# FP64 peaks measured on this pool's B200 by tools/microbench/fp64_peaks.cu
# (profiles/r01_fp64_peaks.txt); MEASURED_PEAKS.json carries HBM and bf16 only.
FP64_DMMA_TFLOPS = 37.15  # mma.sync m8n8k4 f64 (the M2L GEMMs)
FP64_DFMA_TFLOPS = 34.02  # DFMA chains (the P2P kernel)
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            for k in ("hbm_gbs", "hbm_GBs", "hbm"):
                if k in d:
                    return float(d[k]), "MEASURED_PEAKS.json"
        except Exception:  # pragma: no cover
            pass
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def config_dict(name, world=1):
    """The workload description shared by both arms' JSON lines."""
    n, dist, h, order, desc = CONFIGS[name]
    return {"workload": desc, "n": n, "height": h, "order": order, "eps": 10.0 ** -order, "group_size": 250,
            "parallelism": f"morton-range partition x{world}; distributed input (each rank holds 1/{world} of the "
                           "particles: keys all-gathered, owned + halo particle records exchanged over NCCL); "
                           "multipole exchange per upward level: all-gather at the alignment level, per-peer halo "
                           "send/recv below"
                           if world > 1 else "single",
            "l2": "inputs (32 B/particle + 1 KB per leaf expansion array) exceed the 126 MB L2"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- CPU legs
def reference_context(cfg_name, sample=False):
    """The reference's FmmContext (oracle/_ref: the unmodified reference sources) on the
    workload's own particles (or, with sample=True, the labelled 1/8 sample); returns
    (RefContext, n, description) or (None, ...) when oracle/_ref was never built."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"  # the reference's GEMMs run inside its own workers
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracles import Oracle, RefContext, RefLib
    n, dist, h, order = CPU_SAMPLE[cfg_name] if sample else CONFIGS[cfg_name][:4]
    xyzw = Oracle.generate_particles(n, dist, 42)
    desc = (f"N={n} {dist}, height {h}, order {order}" +
            (f" (labelled fallback: 1/{CONFIGS[cfg_name][0] // n} of config {cfg_name}'s particles at the same "
             f"particles per leaf)" if sample else f" (config {cfg_name} itself)"))
    if not RefLib.available():
        return None, n, desc, xyzw
    return RefContext(xyzw, h, order), n, desc, xyzw


def reference_run(cfg_name, workers, warmup, steps, sample=False, t1=False):
    """Times the reference's execute() of the whole task graph (runtime.cpp:91-216, the
    exec_seconds of run_fmm, bench.cpp:458-459) with `workers` threads and the priority
    policy; setup (tree, plan, graph, SVD: bench.cpp:220-236) is reported separately.
    Returns (exec seconds per step, info dict, ref context)."""
    ref, n, desc, xyzw = reference_context(cfg_name, sample)
    if ref is None:  # the CPU restatement (single thread), when the reference was never built here
        from oracles import OracleOps, OracleTree
        _, _, h, order = CPU_SAMPLE[cfg_name] if sample else CONFIGS[cfg_name][:4]
        t = OracleTree(xyzw, h)
        ops = OracleOps.cached(order)
        times = []
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            t.evaluate(ops)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
        return times, {"kind": "port", "cores": 1, "n": n, "sample": desc + "; the CPU restatement, 1 thread"}, None
    for _ in range(warmup):
        ref.execute(workers=workers)
    times = [ref.execute(workers=workers) for _ in range(steps)]
    info = {"kind": "reference", "cores": workers, "n": n, "same_config": not sample,
            "setup_seconds": ref.setup_seconds(), "exec_seconds": float(np.mean(times)),
            "exec_seconds_min": float(np.min(times)), "policy": "priority", "group_size": 250,
            "sample": desc + f"; timed = the reference's execute() of the whole task graph with {workers} "
                             f"workers, {steps} steps after {warmup} warm-up; setup reported separately"}
    if t1:  # t_1 and the parallel efficiency e_n = t_1 / (n t_n)
        t1s = ref.execute(workers=1)
        info["exec_seconds_1_worker"] = t1s
        info["parallel_efficiency"] = t1s / (workers * info["exec_seconds"])
    return times, info, ref


def run_reference(args, world, rank):
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    times, info, _ = reference_run(args.config, workers, args.warmup, args.steps, sample=args.cpu_sample,
                                   t1=not args.no_t1)
    n = info["n"]
    v = n / float(np.mean(times)) / 1e6
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(np.mean(times)) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, seed 42)", "impl": "reference",
            "config": dict(config_dict(args.config), **({"sample_n": n} if args.cpu_sample else {})),
            "cpu_baseline": dict(info, value=v, unit=UNIT),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def parity_vs_reference(ctx, ref, fields, h):
    """The same run's parity with the reference (cpu_baseline leg only): tree and lists
    bit-exact, fields of our fmmgpu_run (input order) vs the reference's gather."""
    import config_parity
    rf = ref.fields()
    ep, ef = config_parity.field_errors([f.numpy() for f in fields], rf)
    tree = config_parity.compare_tree(ctx, ref, h)
    lists = config_parity.compare_lists(ctx, ref, h)
    return {"tree_bit_exact": tree["bit_exact"], "lists_bit_exact": lists["bit_exact"],
            "rel_l2_potential": ep, "rel_l2_force": ef, "tolerance": 1e-12,
            "what": "this run's fmmgpu_run fields (own device-SVD factors) vs the reference's FmmContext "
                    "gather after execute(); tree, Morton order, near CSR and far lists compared element-wise"}


# ----------------------------------------------------------------------------- our arm
def run_ours(args, world, rank, local):
    import paper_1206_0115_b200 as P
    n, dist, h, order, desc = CONFIGS[args.config]
    xyzw = P.generate_particles(n, dist, 42)
    ctx = P.FmmContext(None, order=order, device=local)
    import torch
    # N > 1: rank r holds only the input slice [r n / N, (r + 1) n / N): the
    # distributed build all-gathers Morton keys and moves the particles of each rank's
    # owned leaves and their halo over NCCL (csrc/dist.cu); the tree is the same as the
    # single-device build and each rank owns a contiguous Morton range of leaves
    sl = slice(rank * n // world, (rank + 1) * n // world)
    if world > 1:
        import torch.distributed as dist
        uid = [P.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(uid[0], world, rank)

    def build(dev_ptr=None):
        if world == 1:
            if dev_ptr is None:
                ctx.build_tree(xyzw, h, 250)
            else:
                ctx.build_tree(n, h, 250, on_device_ptr=dev_ptr)
        elif dev_ptr is None:
            ctx.build_tree_distributed(xyzw[sl], h, 250)
        else:
            ctx.build_tree_distributed(None, h, 250, on_device_ptr=dev_ptr, n_local=sl.stop - sl.start)

    t0 = time.perf_counter()
    build()
    tree_cold_ms = ctx.timings()["TREE"] if world == 1 else (time.perf_counter() - t0) * 1e3
    ledger = ctx.ledger()

    # tree + lists, warm: rebuilds from device-resident input,
    # CUDA events around fmmgpu_build_tree / fmmgpu_build_lists, best of 5 (N > 1: the
    # distributed build, host clock around the call, max over ranks)
    dev_in = torch.from_numpy(np.ascontiguousarray(xyzw[sl] if world > 1 else xyzw)).to(f"cuda:{local}")
    tree_ms, lists_ms = [], []
    for _ in range(6):
        barrier(world)
        t0 = time.perf_counter()
        build(dev_in.data_ptr())
        host_ms = (time.perf_counter() - t0) * 1e3
        ctx.build_lists()
        t = ctx.timings()
        tree_ms.append(t["TREE"] if world == 1 else max_over_ranks(host_ms, world))
        lists_ms.append(t["LISTS"])
    del dev_in
    torch.cuda.empty_cache()

    def attach_partition():
        """N > 1: the distributed build already partitioned the leaves for this rank."""
        if world > 1:
            ctx.partition(rank, world)

    attach_partition()
    for _ in range(args.warmup):
        ctx.evaluate()
    ctx.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(world)
    total_ms, kinds, launches = ctx.time_evaluations(args.steps)
    barrier(world)
    clk = clocks.stop()
    ms_step = max_over_ranks(total_ms / args.steps, world)
    value = n / (ms_step / 1e3) / 1e6  # the whole job: N particles evaluated across all ranks

    # isolated per-operator device times (each operator alone, CUDA events on its
    # stream, 5 repetitions), taken right after the timed evaluations: the roofline
    # numerators' denominators. The P2P kernel is the largest single kernel; its share of
    # the step is reported beside it.
    iso = {k: ctx.time_operator(k, -1, 5) for k in ("P2M", "M2M", "M2L", "L2L", "L2P", "P2P")}
    iso_m2l_leaf = ctx.time_operator("M2L", h - 1, 5)
    ctx.evaluate()
    ctx.synchronize()

    # e2e through the C ABI with pinned host buffers, every step: H2D + tree + eval + D2H.
    # N = 1: the pipelined entry point (fmmgpu_run_async), two pinned input sets and two
    # pinned output sets used alternately, so step k's H2D and step k-1's D2H run on the
    # copy engines under step k-1's / step k's device work; the serial fmmgpu_run is
    # timed beside it.
    pins = [torch.from_numpy(np.ascontiguousarray(xyzw[sl] if world > 1 else xyzw)).pin_memory()
            for _ in range(2 if world == 1 else 1)]
    outsets = [[torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)] for _ in range(len(pins))]
    pin_in, outs = pins[0], outsets[0]
    lib = P.lib()
    from ctypes import c_void_p

    def e2e_step():
        if world == 1:
            rc = lib.fmmgpu_run(ctx.h, c_void_p(pin_in.data_ptr()), n, h, 250, *[c_void_p(o.data_ptr()) for o in outs])
            ctx._check(rc)
            return
        # N > 1: pinned H2D of this rank's slice, distributed build (keys all-gathered,
        # owned + halo particles exchanged over NCCL), evaluate with the multipole
        # exchange, D2H of the gathered fields (zero outside the owned particles)
        rc = lib.fmmgpu_build_tree_distributed(ctx.h, c_void_p(pin_in.data_ptr()), sl.stop - sl.start, 0, h, 250,
                                               None)
        ctx._check(rc)
        ctx.evaluate()
        ctx._check(lib.fmmgpu_download_fields(ctx.h, *[c_void_p(o.data_ptr()) for o in outs], 0))

    e2e_step()
    ksteps = max(1, min(args.steps, 5))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(ksteps):
        e2e_step()
    barrier(world)
    e2e_serial_s = max_over_ranks((time.perf_counter() - t0) / ksteps, world)
    e2e_s, path = e2e_serial_s, "fmmgpu_run (C ABI): pinned H2D, build_tree, evaluate, D2H"
    if world == 1:
        serial_ref = [o.clone() for o in outs]

        def submit(k):
            ctx.run_async(pins[k % 2].data_ptr(), n, h, 250, [o.data_ptr() for o in outsets[k % 2]])

        submit(0)
        ctx.run_wait()
        ksteps = max(2, args.steps)
        t0 = time.perf_counter()
        for k in range(ksteps):
            submit(k)
        ctx.run_wait()
        e2e_s = (time.perf_counter() - t0) / ksteps
        path = ("fmmgpu_run_async + fmmgpu_run_wait (C ABI), double-buffered pinned host sets: per step "
                "H2D, build_tree, evaluate, gather, D2H; the copies of neighbouring steps overlap the device work")
        for k in range(2):  # every step's result really came back: compare with the serial run
            if not all(torch.equal(a, b) for a, b in zip(outsets[k], serial_ref)):
                raise RuntimeError("pipelined run returned different fields than fmmgpu_run")
    e2e = {"value": n / e2e_s / 1e6, "unit": UNIT, "h2d_bytes_per_step": 32 * n,
           "d2h_bytes_per_step": 32 * n * world,
           "ms_per_step": e2e_s * 1e3, "steps": ksteps, "path": path,
           "serial_fmmgpu_run": {"value": n / e2e_serial_s / 1e6, "ms_per_step": e2e_serial_s * 1e3}}

    flops = ledger["flops"]
    leaf = h - 1
    peaks = {"P2M": FP64_DFMA_TFLOPS, "M2M": FP64_DFMA_TFLOPS, "M2L": FP64_DMMA_TFLOPS, "L2L": FP64_DFMA_TFLOPS,
             "L2P": FP64_DFMA_TFLOPS, "P2P": FP64_DFMA_TFLOPS}
    per_op = {}
    for k, ms in iso.items():
        tf = flops[k] / (ms / 1e3) / 1e12
        per_op[k] = {"ms_isolated": ms, "ms_in_step": kinds[k] / args.steps, "ledger_flops": flops[k],
                     "tflops": tf, "peak_tflops": peaks[k], "frac": tf / peaks[k]}
    hbm, hbm_src = hbm_peak()
    for k in ("M2M", "L2L"):  # HBM-bound transfers: algorithmic bytes 8 l^3 (children + 2 parents)
        cells = [ctx.level(v)[0].shape[0] for v in range(h)]
        l3 = order ** 3
        byts = sum(8 * l3 * (cells[v + 1] + 2 * cells[v]) for v in range(2, leaf))
        per_op[k]["hbm_gbs"] = byts / (iso[k] / 1e3) / 1e9
        per_op[k]["hbm_frac"] = per_op[k]["hbm_gbs"] / hbm
    # executed FP64 flops per operator (ncu DFMA / DADD / DMUL / DMMA counters of one
    # evaluation, tools/fp64_ops.py -> profiles/fp64_ops.json): the utilisation beside the
    # ledger fraction (the factored P2M / L2P kernels execute fewer flops than the ledger
    # counts, M2L's DMMA executes padding rows)
    fo = os.path.join(ROOT, "profiles", "fp64_ops.json")
    if os.path.exists(fo):
        ops = json.load(open(fo)).get(args.config, {})
        for k, v in per_op.items():
            if k in ops and ops[k].get("exec_flops"):
                ef = ops[k]["exec_flops"]
                v["exec_flops"] = ef
                v["exec_frac"] = ef / (v["ms_isolated"] / 1e3) / 1e12 / v["peak_tflops"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{args.config}:P2P")
    p2p_tf = flops["P2P"] / (iso["P2P"] / 1e3) / 1e12
    mutual = ctx.p2p_kernel() == "mutual"
    # DP instructions per directional interaction: 12 for the mutual kernel (24 per pair,
    # both directions), 18 for the one-sided kernel; the ledger counts 15 flop per
    # directional interaction and the peak 2 flop per DFMA
    dp_per_dir = 12 if mutual else 18
    roof = {"bound": "fp64",
            "kernel": ("k_p2p_mutual + k_p2p_drain (P2P with P2PBuffers slots and ordered reduce, FP64 pipe)"
                       if mutual else "k_p2p (one-sided P2P, FP64 pipe)"),
            "achieved": p2p_tf,
            "peak": FP64_DFMA_TFLOPS, "unit": "TFLOP/s", "frac": p2p_tf / FP64_DFMA_TFLOPS, "traffic": traffic,
            "flops_per_launch": flops["P2P"], "ms_per_launch": iso["P2P"],
            "share_of_step": iso["P2P"] / ms_step,
            "peak_source": "FP64 DFMA measured by tools/microbench/fp64_peaks.cu (profiles/r01_fp64_peaks.txt); "
                           "MEASURED_PEAKS.json has no FP64 figure",
            "traffic_note": "ncu DRAM bytes of the mutual kernel + its drain per evaluation: 0.64 GB of particles and "
                            "near fields plus the [13][n] P2PBuffers-style slot array (4.16 GB written, read back by "
                            "the ordered drain); the kernel stays FP64-bound (DRAM ~6% busy during it)",
            "flop_convention": "reference ledger (bench.hpp:49-53): 15 flop per directional interaction; the "
                               f"kernel issues {dp_per_dir} FP64 instructions per directional interaction and the "
                               f"peak counts 2 flop per DFMA, so frac <= 15/{2 * dp_per_dir} = "
                               f"{15 / (2 * dp_per_dir):.3f} at a saturated FP64 pipe",
            # the same launch against the FP64 instruction issue rate (DFMA peak / 2 flop):
            # useful interactions x DP instructions per interaction / duration
            "fp64_instr_frac": (ledger["near_directional"] * dp_per_dir / (iso["P2P"] / 1e3))
                               / (FP64_DFMA_TFLOPS * 1e12 / 2),
            "m2l": {"bound": "tensor (FP64 DMMA)", "ms_all_levels": iso["M2L"], "ms_leaf": iso_m2l_leaf,
                    "achieved": per_op["M2L"]["tflops"], "peak": FP64_DMMA_TFLOPS,
                    "frac": per_op["M2L"]["frac"]},
            "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "eval_seconds": ms_step / 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (reference generator bench.cpp:29-39, seed 42, unit weights)",
            "config": config_dict(args.config, world),
            "gpu_launches": launches, "e2e": e2e, "roofline": roof, "per_operator": per_op,
            "tree_build_ms": min(tree_ms[1:]), "lists_build_ms": min(lists_ms[1:]),
            "tree_build_cold_ms": tree_cold_ms,
            "tree_note": "tree_build_ms / lists_build_ms: best of 5 warm rebuilds from device-resident particles "
                         "(CUDA events around fmmgpu_build_tree / fmmgpu_build_lists); the evaluation does not "
                         "read the explicit lists. tree_build_cold_ms: the first build (H2D + allocations)",
            "clocks": clk,
            "note": "P2P runs on its own stream concurrently with the far-field chain; per-operator times "
                    "of the far chain include waiting for SMs the P2P kernel holds"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            times, info, ref = reference_run(args.config, os.cpu_count() or 1, 1, 2, sample=args.cpu_sample)
            line["cpu_baseline"] = dict(info, value=info["n"] / float(np.mean(times)) / 1e6, unit=UNIT)
            if ref is not None and not args.cpu_sample:
                line["parity"] = parity_vs_reference(ctx, ref, serial_ref, h)
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="B", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", action="store_true",
                    help="time the reference on the labelled 1/8 sample instead of the configuration itself")
    ap.add_argument("--no-t1", action="store_true", help="reference arm: skip the 1-worker run (t_1)")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
