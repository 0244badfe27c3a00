"""B200-native black-box Chebyshev FMM evaluation path (arXiv 1206.0115, "taskfmm").

Host-side mirror of the reference's operator interface, over the C ABI of
``include/fmmgpu.h`` (``libfmmgpu.so``, CUDA sm_100a). Names follow the reference:

* ``RunConfig``            bench.hpp:21-35
* ``generate_particles``   bench.cpp:29-61 (same mt19937_64 stream, host side)
* ``FmmContext``           bench.hpp:86-121 -- tree + operators + evaluation; the
  reference's ``run_task(Task)`` seam is exposed per operator and level
  (``p2m``, ``m2m(v)``, ``m2l(v)``, ``l2l(v)``, ``l2p``, ``p2p``) and as the whole
  schedule (``evaluate``); ``gather`` returns fields in input order.
* ``run_fmm``              bench.cpp:415-469 (without the oracle check)

There is no CPU fallback: if the CUDA library is missing or no GPU is present the
calls raise. The reference's exception classes map to Python exceptions of the
same meaning (ValueError = invalid_argument, DomainError = domain_error, ...).
"""
from __future__ import annotations

import ctypes
import importlib.util
import os
from ctypes import c_double, c_int, c_uint64, c_void_p, byref
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FMMGPU_LIB: another in-tree build of the library (compile-time variants for A/B timing)
LIB_PATH = os.path.join(_HERE, os.path.basename(os.environ.get("FMMGPU_LIB", "libfmmgpu.so")))

KINDS = ("P2M", "M2M", "M2L", "L2L", "L2P", "P2P", "P2PREDUCE")
DISTS = {"uniform": 0, "sphere": 1, "ellipsoid": 2}
CELL_DTYPE = np.dtype(
    [("code", "<u8"), ("first_particle", "<u4"), ("particle_count", "<u4"), ("parent", "<u4"),
     ("first_child", "<u4"), ("child_count", "<u4"), ("_pad", "<u4")])


class FmmError(RuntimeError):
    code = 5


class DomainError(FmmError, ValueError):      # std::domain_error
    code = 2


class InvalidArgument(FmmError, ValueError):  # std::invalid_argument
    code = 1


class OutOfRange(FmmError, IndexError):       # std::out_of_range
    code = 3


class LogicError(FmmError):                   # std::logic_error
    code = 4


_ERRORS = {1: InvalidArgument, 2: DomainError, 3: OutOfRange, 4: LogicError, 5: FmmError}

_lib = None


def lib():
    """Loads libfmmgpu.so (built by ``__graft_entry__.build()`` / ``make -C paper_1206_0115_b200``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FmmError(f"{LIB_PATH} missing: build it with `make -C {_HERE}` (no CPU fallback)")
        if "FMMGPU_NCCL_LIB" not in os.environ:
            # the library dlopens NCCL only when a communicator is used; point it at torch's
            # bundled copy so both share one libnccl.so.2 (a system NCCL loaded first would
            # shadow it and break a later `import torch`)
            spec = importlib.util.find_spec("nvidia.nccl")
            for d in (spec.submodule_search_locations or []) if spec else []:
                cand = os.path.join(d, "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["FMMGPU_NCCL_LIB"] = cand
                    break
        L = ctypes.CDLL(LIB_PATH)
        L.fmmgpu_last_error.restype = ctypes.c_char_p
        L.fmmgpu_last_error.argtypes = [c_void_p]
        L.fmmgpu_global_error.restype = ctypes.c_char_p
        L.fmmgpu_create.argtypes = [c_int, c_int, c_double, ctypes.POINTER(c_void_p)]
        L.fmmgpu_create_from_cache.argtypes = [c_int, c_int, c_double, ctypes.c_char_p, ctypes.POINTER(c_void_p)]
        L.fmmgpu_destroy.argtypes = [c_void_p]
        L.fmmgpu_build_tree.argtypes = [c_void_p, c_void_p, c_uint64, c_int, c_int, c_int, c_void_p]
        L.fmmgpu_level_cells.restype = c_uint64
        L.fmmgpu_level_cells.argtypes = [c_void_p, c_int]
        L.fmmgpu_near_entries.restype = c_uint64
        L.fmmgpu_near_entries.argtypes = [c_void_p]
        L.fmmgpu_far_pairs.restype = c_uint64
        L.fmmgpu_far_pairs.argtypes = [c_void_p, c_int]
        L.fmmgpu_last_launch_count.restype = c_uint64
        L.fmmgpu_last_launch_count.argtypes = [c_void_p]
        L.fmmgpu_generate_particles.argtypes = [c_uint64, c_int, c_uint64, c_void_p]
        L.fmmgpu_run.argtypes = [c_void_p, c_void_p, c_uint64, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p]
        L.fmmgpu_run_async.argtypes = L.fmmgpu_run.argtypes
        L.fmmgpu_run_wait.argtypes = [c_void_p]
        L.fmmgpu_set_trace.argtypes = [c_void_p, c_int]
        L.fmmgpu_set_graph.argtypes = [c_void_p, c_int]
        L.fmmgpu_set_p2p_mode.argtypes = [c_void_p, c_int]
        L.fmmgpu_p2p_kernel.argtypes = [c_void_p]
        L.fmmgpu_trace_spans.argtypes = [c_void_p, c_int, c_void_p, c_void_p, c_void_p]
        for name in ("fmmgpu_reset", "fmmgpu_p2m", "fmmgpu_l2p", "fmmgpu_p2p", "fmmgpu_evaluate",
                     "fmmgpu_synchronize", "fmmgpu_build_lists"):
            getattr(L, name).argtypes = [c_void_p]
        for name in ("fmmgpu_m2m", "fmmgpu_m2l", "fmmgpu_l2l", "fmmgpu_upward_level"):
            getattr(L, name).argtypes = [c_void_p, c_int]
        L.fmmgpu_downward.argtypes = [c_void_p]
        L.fmmgpu_partition.argtypes = [c_void_p, c_int, c_int]
        L.fmmgpu_direct.argtypes = [c_void_p, c_void_p, c_uint64, c_void_p, c_void_p, c_void_p, c_void_p]
        L.fmmgpu_partition_ranges.argtypes = [c_void_p, c_int, c_void_p]
        L.fmmgpu_plan_partition.argtypes = [c_void_p, ctypes.c_uint32, c_int, c_void_p]
        L.fmmgpu_comm_init.argtypes = [c_void_p, ctypes.c_char_p, c_int, c_int]
        L.fmmgpu_comm_destroy.argtypes = [c_void_p]
        L.fmmgpu_comm_unique_id.argtypes = [ctypes.c_char_p]
        L.fmmgpu_exchange_plan.argtypes = [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        L.fmmgpu_download_near_blocks.argtypes = [c_void_p] + [c_void_p] * 7
        L.fmmgpu_download_far_source_blocks.argtypes = [c_void_p, c_int, c_void_p, c_void_p, c_void_p]
        L.fmmgpu_set_measurement.argtypes = [c_void_p, c_int]
        L.fmmgpu_root_from_bounds.argtypes = [c_void_p, c_void_p]
        L.fmmgpu_dist_local.argtypes = [c_void_p, c_void_p, c_uint64, c_int, c_void_p]
        L.fmmgpu_dist_keys.argtypes = [c_void_p, c_void_p, c_int, c_void_p, c_int, c_void_p]
        L.fmmgpu_dist_build.argtypes = [c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int, c_void_p,
                                        c_int]
        L.fmmgpu_dist_plan.argtypes = [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]
        L.fmmgpu_dist_pack.argtypes = [c_void_p, c_int, c_void_p, c_int]
        L.fmmgpu_dist_unpack.argtypes = [c_void_p, c_int, c_void_p, c_int]
        L.fmmgpu_dist_check.argtypes = [c_void_p, c_void_p]
        L.fmmgpu_dist_commit.argtypes = [c_void_p, c_int]
        L.fmmgpu_build_tree_distributed.argtypes = [c_void_p, c_void_p, c_uint64, c_int, c_int, c_int, c_void_p]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(c_void_p)


@dataclass
class RunConfig:
    """bench.hpp:21-35 (the fields this path uses)."""
    n: int = 10000
    dist: str = "uniform"
    height: int = 4
    acc: int = 5          # interpolation order l = acc, SVD eps = 10^-acc
    group_size: int = 250
    seed: int = 42
    device: int = 0


def plan_partition(weights, nranks: int) -> np.ndarray:
    """Balanced contiguous split of weighted items (host only): first item of each rank + end."""
    w = np.ascontiguousarray(weights, dtype=np.uint64)
    out = np.zeros(nranks + 1, dtype=np.uint32)
    rc = lib().fmmgpu_plan_partition(_p(w) if len(w) else None, len(w), nranks, _p(out))
    if rc:
        raise _ERRORS.get(rc, FmmError)("plan_partition failed")
    return out


def root_from_bounds(lohi) -> np.ndarray:
    """Root cube {cx, cy, cz, width} of per-axis bounds {min[3], max[3]} (geometry.cpp:28-34)."""
    b = np.ascontiguousarray(lohi, dtype=np.float64)
    out = np.zeros(4)
    rc = lib().fmmgpu_root_from_bounds(_p(b), _p(out))
    if rc != 0:
        raise InvalidArgument("root_from_bounds: empty or invalid bounds")
    return out


def comm_unique_id() -> bytes:
    """NCCL unique id (128 bytes) for fmmgpu_comm_init; create on rank 0 and broadcast."""
    buf = ctypes.create_string_buffer(128)
    rc = lib().fmmgpu_comm_unique_id(buf)
    if rc:
        raise FmmError("ncclGetUniqueId failed")
    return buf.raw


def generate_particles(n: int, dist: str = "uniform", seed: int = 42) -> np.ndarray:
    """bench.cpp:29-61: (n, 4) array of x, y, z, w (unit weights); dist uniform, sphere or
    ellipsoid (config D: the sphere's directions on semi-axes 0.5, 0.35, 0.2)."""
    out = np.zeros((n, 4), dtype=np.float64)
    lib().fmmgpu_generate_particles(n, DISTS[dist], seed, _p(out))
    return out


class FmmContext:
    """FmmContext (bench.hpp:86-121) on one B200.

    ``FmmContext(particles, cfg)`` builds the operators (InterpolationEngine +
    M2LOperatorSet, device SVD, or the factors of ``m2l_cache``) and the tree on the GPU; ``evaluate()`` runs the
    whole evaluation; ``gather()`` returns (potential, fx, fy, fz) in input order.
    """

    def __init__(self, particles=None, cfg: RunConfig | None = None, *, order=None, eps=None, device=0,
                 m2l_cache: str | None = None):
        self.cfg = cfg or RunConfig()
        self.order = order if order is not None else self.cfg.acc
        if self.order < 2:
            raise InvalidArgument("accuracy parameter must be at least 2")  # bench.cpp:223
        self.eps = eps if eps is not None else 10.0 ** (-self.order)
        self._lib = lib()
        h = c_void_p()
        dev = device if cfg is None else cfg.device
        if m2l_cache is not None:  # M2LOperatorSet::load_cache(path, order, eps): no device SVD
            rc = self._lib.fmmgpu_create_from_cache(dev, self.order, self.eps, m2l_cache.encode(), byref(h))
        else:
            rc = self._lib.fmmgpu_create(dev, self.order, self.eps, byref(h))
        if rc:
            raise _ERRORS.get(rc, FmmError)(self._lib.fmmgpu_global_error().decode())
        self.h = h
        self.n = 0
        if particles is not None:
            self.build_tree(particles, self.cfg.height, self.cfg.group_size)

    # -- plumbing
    def _check(self, rc):
        if rc:
            raise _ERRORS.get(rc, FmmError)(self._lib.fmmgpu_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self._lib.fmmgpu_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- M2LOperatorSet
    def load_m2l_cache(self, path: str):
        self._check(self._lib.fmmgpu_load_m2l_cache(self.h, path.encode()))

    def save_m2l_cache(self, path: str):
        self._check(self._lib.fmmgpu_save_m2l_cache(self.h, path.encode()))

    def compression_report(self):
        r = np.zeros(16, dtype=np.int32)
        m = np.zeros(16, dtype=np.int32)
        w = c_double()
        self._check(self._lib.fmmgpu_m2l_report(self.h, _p(r), _p(m), byref(w)))
        return {"ranks": r, "multiplicity": m, "weighted_mean_rank": w.value}

    # -- GroupTree
    def build_tree(self, particles, height: int, group_size: int = 250, root=None, on_device_ptr=None):
        """GroupTree(particles, height, group_size[, root]); particles (n,4) float64."""
        if on_device_ptr is not None:
            n = int(particles)
            self._check(self._lib.fmmgpu_build_tree(self.h, c_void_p(on_device_ptr), n, 1, height, group_size,
                                                    _p(None if root is None else np.asarray(root, np.float64))))
        else:
            xyzw = np.ascontiguousarray(particles, dtype=np.float64)
            if xyzw.ndim != 2 or (len(xyzw) and xyzw.shape[1] != 4):
                raise InvalidArgument("particles must be an (n, 4) array of x, y, z, w")
            n = len(xyzw)
            r = None if root is None else np.ascontiguousarray(root, dtype=np.float64)
            self._check(self._lib.fmmgpu_build_tree(self.h, _p(xyzw) if n else None, n, 0, height, group_size, _p(r)))
        self.n, self.height, self.group_size = n, height, group_size

    def build_lists(self):
        self._check(self._lib.fmmgpu_build_lists(self.h))

    def root_cube(self):
        out = np.zeros(4)
        n = c_uint64()
        self._check(self._lib.fmmgpu_tree_info(self.h, byref(n), None, None, _p(out)))
        return out

    def level(self, v: int):
        n = self._lib.fmmgpu_level_cells(self.h, v)
        cells = np.zeros(n, dtype=CELL_DTYPE)
        nb = (n + self.group_size - 1) // self.group_size
        bo = np.zeros(nb + 1, dtype=np.uint32)
        self._check(self._lib.fmmgpu_download_level(self.h, v, _p(cells), _p(bo)))
        return cells, bo

    def particles(self):
        x, y, z, w = (np.zeros(self.n) for _ in range(4))
        ids = np.zeros(self.n, dtype=np.uint32)
        self._check(self._lib.fmmgpu_download_particles(self.h, _p(x), _p(y), _p(z), _p(w), _p(ids)))
        return x, y, z, w, ids

    def near(self):
        ne = self._lib.fmmgpu_near_entries(self.h)
        nc = self._lib.fmmgpu_level_cells(self.h, self.height - 1)
        off = np.zeros(nc + 1, dtype=np.uint32)
        cells = np.zeros(max(ne, 1), dtype=np.uint32)
        tot = c_uint64()
        self._check(self._lib.fmmgpu_download_near(self.h, _p(off), _p(cells), byref(tot)))
        return off, cells[:ne], tot.value

    def near_blocks(self):
        """NearFieldPlan block arrays (direct.cpp:36-58): (task_interactions, partners_above
        offsets, partners_above, contributors_below offsets, contributors_below)."""
        na, nb_ = c_uint64(), c_uint64()
        self._check(self._lib.fmmgpu_download_near_blocks(self.h, None, None, None, None, None, byref(na),
                                                          byref(nb_)))
        nc = self._lib.fmmgpu_level_cells(self.h, self.height - 1)
        nblk = (nc + self.group_size - 1) // self.group_size
        ti = np.zeros(nblk, dtype=np.uint64)
        ao = np.zeros(nblk + 1, dtype=np.uint32)
        bo = np.zeros(nblk + 1, dtype=np.uint32)
        a = np.zeros(max(na.value, 1), dtype=np.uint32)
        b = np.zeros(max(nb_.value, 1), dtype=np.uint32)
        self._check(self._lib.fmmgpu_download_near_blocks(self.h, _p(ti), _p(ao), _p(a), _p(bo), _p(b), byref(na),
                                                          byref(nb_)))
        return ti, ao, a[:na.value], bo, b[:nb_.value]

    def far_source_blocks(self, v: int):
        """LevelM2L::source_blocks of level v as (offsets, blocks)."""
        n = c_uint64()
        self._check(self._lib.fmmgpu_download_far_source_blocks(self.h, v, None, None, byref(n)))
        nc = self._lib.fmmgpu_level_cells(self.h, v)
        nblk = (nc + self.group_size - 1) // self.group_size
        off = np.zeros(nblk + 1, dtype=np.uint32)
        blk = np.zeros(max(n.value, 1), dtype=np.uint32)
        self._check(self._lib.fmmgpu_download_far_source_blocks(self.h, v, _p(off), _p(blk), byref(n)))
        return off, blk[:n.value]

    def far(self, v: int):
        npairs = self._lib.fmmgpu_far_pairs(self.h, v)
        nc = self._lib.fmmgpu_level_cells(self.h, v)
        nb = (nc + self.group_size - 1) // self.group_size
        t = np.zeros(max(npairs, 1), dtype=np.uint32)
        s = np.zeros(max(npairs, 1), dtype=np.uint32)
        vec = np.zeros(max(npairs, 1), dtype=np.uint16)
        go = np.zeros(nb * 16 + 1, dtype=np.uint64)
        self._check(self._lib.fmmgpu_download_far(self.h, v, _p(t), _p(s), _p(vec), _p(go)))
        return t[:npairs], s[:npairs], vec[:npairs], go

    def expansion(self, v: int, which: int):
        """which: 0 multipole, 1 local_own, 2 local_down; (cells, l^3)."""
        n = self._lib.fmmgpu_level_cells(self.h, v)
        out = np.zeros((n, self.order ** 3))
        self._check(self._lib.fmmgpu_download_expansion(self.h, v, which, _p(out)))
        return out

    def set_expansion(self, v: int, which: int, values):
        a = np.ascontiguousarray(values, dtype=np.float64)
        self._check(self._lib.fmmgpu_upload_expansion(self.h, v, which, _p(a)))

    # -- the run_task seam, level granular (bench.cpp:255-344)
    def reset(self):
        self._check(self._lib.fmmgpu_reset(self.h))

    def p2m(self):
        self._check(self._lib.fmmgpu_p2m(self.h))

    def m2m(self, parent_level: int):
        self._check(self._lib.fmmgpu_m2m(self.h, parent_level))

    def m2l(self, level: int):
        self._check(self._lib.fmmgpu_m2l(self.h, level))

    def l2l(self, parent_level: int):
        self._check(self._lib.fmmgpu_l2l(self.h, parent_level))

    def l2p(self):
        self._check(self._lib.fmmgpu_l2p(self.h))

    def p2p(self):
        self._check(self._lib.fmmgpu_p2p(self.h))

    def run_kinds(self, kinds):
        """reset + the selected payload kinds in DAG order (cf. oracle ref_run_serial)."""
        self.reset()
        leaf = self.height - 1
        if "P2M" in kinds:
            self.p2m()
        if "M2M" in kinds:
            for v in range(leaf - 1, 1, -1):
                self.m2m(v)
        if "M2L" in kinds:
            for v in range(2, leaf + 1):
                self.m2l(v)
        if "L2L" in kinds:
            for v in range(2, leaf):
                self.l2l(v)
        if "L2P" in kinds:
            self.l2p()
        if "P2P" in kinds:
            self.p2p()
        self.synchronize()

    def evaluate(self):
        """The whole evaluation (all payloads of the task graph), asynchronous."""
        self._check(self._lib.fmmgpu_evaluate(self.h))

    def synchronize(self):
        self._check(self._lib.fmmgpu_synchronize(self.h))

    def gather(self):
        """FmmContext::gather (bench.cpp:350-365): potential, fx, fy, fz in input order."""
        out = [np.zeros(self.n) for _ in range(4)]
        self._check(self._lib.fmmgpu_download_fields(self.h, *[_p(a) for a in out], 0))
        return out

    def gather_device(self, ptrs):
        self._check(self._lib.fmmgpu_download_fields(self.h, *[c_void_p(p) for p in ptrs], 1))

    def sorted_fields(self):
        out = [np.zeros(self.n) for _ in range(4)]
        self._check(self._lib.fmmgpu_download_sorted_fields(self.h, *[_p(a) for a in out]))
        return out

    def timings(self):
        ms = np.zeros(10)
        self._check(self._lib.fmmgpu_timings(self.h, _p(ms)))
        keys = list(KINDS[:6]) + ["GATHER", "EVAL", "TREE", "LISTS"]
        return dict(zip(keys, ms.tolist()))

    def ledger(self):
        flops = np.zeros(7, dtype=np.uint64)
        near = c_uint64()
        pairs = c_uint64()
        self._check(self._lib.fmmgpu_ledger(self.h, _p(flops), byref(near), byref(pairs)))
        return {"flops": dict(zip(KINDS, flops.tolist())), "near_directional": near.value, "m2l_pairs": pairs.value}

    def ledger_rows(self):
        """FlopLedger rows (build_ledger, bench.cpp:151-181): work and flops as
        (7 kinds, height) arrays, and M2L pairs per (level, canonical class)."""
        h = self.height
        work = np.zeros((7, h), dtype=np.uint64)
        flops = np.zeros((7, h), dtype=np.uint64)
        pairs = np.zeros((h, 16), dtype=np.uint64)
        self._check(self._lib.fmmgpu_ledger_rows(self.h, _p(work), _p(flops), _p(pairs)))
        return {"work": work, "flops": flops, "m2l_pairs": pairs}

    def launch_count(self):
        return int(self._lib.fmmgpu_last_launch_count(self.h))

    def time_evaluations(self, steps: int):
        """K back-to-back evaluations timed with CUDA events on the launching stream.
        Returns (total_ms, per-kind ms sums, kernel launches)."""
        total = c_double()
        ms = np.zeros(10)
        nl = c_uint64()
        self._check(self._lib.fmmgpu_time_evaluations(self.h, steps, byref(total), _p(ms), byref(nl)))
        keys = list(KINDS[:6]) + ["GATHER", "EVAL", "TREE", "LISTS"]
        return total.value, dict(zip(keys, ms.tolist())), nl.value

    # -- accuracy check (direct.cpp:202-226 on the device)
    def direct(self, targets):
        """Exact potential / force at the given input indices (sum over all particles)."""
        t = np.ascontiguousarray(targets, dtype=np.uint32)
        out = [np.zeros(len(t)) for _ in range(4)]
        self._check(self._lib.fmmgpu_direct(self.h, _p(t), len(t), *[_p(a) for a in out]))
        return out

    # -- multi-GPU partition
    def partition(self, rank: int, nranks: int):
        """Own a contiguous Morton range of leaves (rank of nranks); nranks=1 undoes it."""
        self._check(self._lib.fmmgpu_partition(self.h, rank, nranks))

    def partition_info(self):
        r, n, a = c_int(), c_int(), c_int()
        s0, s1 = c_uint64(), c_uint64()
        self._check(self._lib.fmmgpu_partition_info(self.h, byref(r), byref(n), byref(a), byref(s0), byref(s1)))
        return {"rank": r.value, "nranks": n.value, "align_level": a.value, "slots": (s0.value, s1.value)}

    def partition_ranges(self, level: int):
        n = self.partition_info()["nranks"]
        out = np.zeros(n + 1, dtype=np.uint32)
        self._check(self._lib.fmmgpu_partition_ranges(self.h, level, _p(out)))
        return out

    def exchange_plan(self, level: int, peer: int = 0):
        """(kind, send_cells, recv_cells) of the exchange after the upward step of `level`
        with `peer`: kind 0 none, 1 all-gather of the owned rows, 2 halo (fmmgpu_exchange_plan)."""
        kind = c_int()
        sc, rc = ctypes.c_uint32(), ctypes.c_uint32()
        self._check(self._lib.fmmgpu_exchange_plan(self.h, level, peer, byref(kind), None, byref(sc), None, byref(rc)))
        snd = np.zeros(sc.value, dtype=np.uint32)
        rcv = np.zeros(rc.value, dtype=np.uint32)
        if kind.value == 2:
            self._check(self._lib.fmmgpu_exchange_plan(self.h, level, peer, byref(kind), _p(snd), byref(sc), _p(rcv),
                                                       byref(rc)))
        return kind.value, snd, rcv

    def set_measurement(self, skip_exchange: bool = True):
        """Measurement aid: partitioned evaluations skip the exchange (fields then refused)."""
        self._check(self._lib.fmmgpu_set_measurement(self.h, 1 if skip_exchange else 0))

    def comm_init(self, uid: bytes, nranks: int, rank: int):
        self._check(self._lib.fmmgpu_comm_init(self.h, uid, nranks, rank))

    # ---- distributed input (fmmgpu_dist_*, csrc/dist.cu): this rank holds one input slice
    def dist_local(self, xyzw_local) -> np.ndarray:
        """Upload this rank's input slice; returns its per-axis bounds {min[3], max[3]}."""
        a = np.ascontiguousarray(xyzw_local, dtype=np.float64).reshape(-1, 4)
        self._dist_n = a.shape[0]
        lohi = np.zeros(6)
        self._check(self._lib.fmmgpu_dist_local(self.h, _p(a), a.shape[0], 0, _p(lohi)))
        return lohi

    def dist_keys(self, root, height: int):
        """Leaf Morton keys (u64) of the uploaded slice and its outside-the-root flag."""
        r = np.ascontiguousarray(root, dtype=np.float64)
        keys = np.zeros(self._dist_n, dtype=np.uint64)
        flag = c_int()
        self._check(self._lib.fmmgpu_dist_keys(self.h, _p(r), height, _p(keys), 0, byref(flag)))
        return keys, flag.value

    def dist_build(self, keys_all, offsets, rank: int, nranks: int, height: int, group_size: int, root, flag: int):
        """Tree from the all-gathered keys, partition, particle plan (own records placed)."""
        k = np.ascontiguousarray(keys_all, dtype=np.uint64)
        o = np.ascontiguousarray(offsets, dtype=np.uint64)
        r = np.ascontiguousarray(root, dtype=np.float64)
        self._check(self._lib.fmmgpu_dist_build(self.h, _p(k), 0, _p(o), rank, nranks, height, group_size, _p(r),
                                                int(flag)))
        self.n, self.height, self.group_size = int(o[-1]), height, group_size

    def dist_plan(self, peer: int):
        """(send_slots, recv_slots): Morton slots whose records go to / come from `peer`."""
        sc, rc = ctypes.c_uint32(), ctypes.c_uint32()
        self._check(self._lib.fmmgpu_dist_plan(self.h, peer, None, byref(sc), None, byref(rc)))
        snd = np.zeros(sc.value, dtype=np.uint32)
        rcv = np.zeros(rc.value, dtype=np.uint32)
        self._check(self._lib.fmmgpu_dist_plan(self.h, peer, _p(snd), byref(sc), _p(rcv), byref(rc)))
        return snd, rcv

    def dist_pack(self, peer: int) -> np.ndarray:
        n = len(self.dist_plan(peer)[0])
        out = np.zeros((n, 4))
        self._check(self._lib.fmmgpu_dist_pack(self.h, peer, _p(out), 0))
        return out

    def dist_unpack(self, peer: int, records):
        a = np.ascontiguousarray(records, dtype=np.float64).reshape(-1, 4)
        self._check(self._lib.fmmgpu_dist_unpack(self.h, peer, _p(a), 0))

    def dist_check(self) -> int:
        f = c_int()
        self._check(self._lib.fmmgpu_dist_check(self.h, byref(f)))
        return f.value

    def dist_commit(self, flag: int):
        self._check(self._lib.fmmgpu_dist_commit(self.h, int(flag)))

    def build_tree_distributed(self, xyzw_local, height: int, group_size: int = 250, root=None, on_device_ptr=None,
                               n_local=None):
        """All of the distributed build over the attached NCCL communicator."""
        if on_device_ptr is not None:
            ptr, n, dev = c_void_p(on_device_ptr), int(n_local), 1
        else:
            a = np.ascontiguousarray(xyzw_local, dtype=np.float64).reshape(-1, 4)
            ptr, n, dev = _p(a), a.shape[0], 0
        r = None if root is None else np.ascontiguousarray(root, dtype=np.float64)
        self._check(self._lib.fmmgpu_build_tree_distributed(self.h, ptr, n, dev, height, group_size, _p(r)))
        ntot = c_uint64()
        self._check(self._lib.fmmgpu_tree_info(self.h, byref(ntot), None, None, None))
        self.n, self.height, self.group_size = ntot.value, height, group_size

    def upward_level(self, level: int):
        self._check(self._lib.fmmgpu_upward_level(self.h, level))

    def downward(self):
        self._check(self._lib.fmmgpu_downward(self.h))

    def time_operator(self, kind: str, level: int = -1, reps: int = 5):
        """Isolated device time (ms per repetition) of one operator; leaves accumulators dirty."""
        ms = c_double()
        self._check(self._lib.fmmgpu_time_operator(self.h, KINDS.index(kind), level, reps, byref(ms)))
        return ms.value

    def run(self, particles, height, group_size=250):
        """Whole run through the C ABI with host buffers (fmmgpu_run)."""
        xyzw = np.ascontiguousarray(particles, dtype=np.float64)
        n = len(xyzw)
        out = [np.zeros(n) for _ in range(4)]
        self._check(self._lib.fmmgpu_run(self.h, _p(xyzw), n, height, group_size, *[_p(a) for a in out]))
        self.n, self.height, self.group_size = n, height, group_size
        return out

    def run_async(self, xyzw_ptr: int, n: int, height: int, group_size: int, out_ptrs):
        """Pipelined run (fmmgpu_run_async) on caller-owned, preferably pinned, host
        buffers given as raw addresses: the {x,y,z,w} input and four n-double outputs.
        Returns once the step's tree is built; outputs are valid after run_wait()."""
        self._check(self._lib.fmmgpu_run_async(self.h, c_void_p(xyzw_ptr), n, height, group_size,
                                               *[c_void_p(a) for a in out_ptrs]))
        self.n, self.height, self.group_size = n, height, group_size

    def run_wait(self):
        self._check(self._lib.fmmgpu_run_wait(self.h))

    def set_graph(self, on: bool = True):
        """Replay evaluations from a captured CUDA graph (fmmgpu_set_graph)."""
        self._check(self._lib.fmmgpu_set_graph(self.h, 1 if on else 0))

    def set_p2p_mode(self, mutual: bool = True):
        """Near field kernel: mutual (p2p_block(mutual=true) + slots + ordered reduce,
        direct.cpp:63-92, 151-200) or one-sided (fmmgpu_set_p2p_mode)."""
        mode = mutual if (isinstance(mutual, int) and not isinstance(mutual, bool)) else (1 if mutual else 0)
        self._check(self._lib.fmmgpu_set_p2p_mode(self.h, mode))

    def p2p_kernel(self) -> str:
        """'mutual' or 'onesided': the near-field kernel the current tree runs (mode 2 = auto)."""
        return "mutual" if self._lib.fmmgpu_p2p_kernel(self.h) == 1 else "onesided"

    def set_trace(self, on: bool = True):
        """Per-launch device trace of the following evaluations (fmmgpu_set_trace)."""
        self._check(self._lib.fmmgpu_set_trace(self.h, 1 if on else 0))

    def trace_spans(self):
        """Spans of the last traced evaluation: [(kind, level, stream, start_ms, end_ms)],
        stream 0 = far field, 1 = near field (runtime.hpp TraceEvent analogue)."""
        cnt = c_int()
        self._check(self._lib.fmmgpu_trace_spans(self.h, 0, byref(cnt), None, None))
        n = cnt.value
        meta = np.zeros(3 * max(n, 1), dtype=np.int32)
        t = np.zeros(2 * max(n, 1))
        self._check(self._lib.fmmgpu_trace_spans(self.h, n, byref(cnt), _p(meta), _p(t)))
        return [(KINDS[meta[3 * i]], int(meta[3 * i + 1]), int(meta[3 * i + 2]), float(t[2 * i]), float(t[2 * i + 1]))
                for i in range(n)]


def check_targets(n: int, check: int) -> np.ndarray:
    """bench.cpp:368-376: k * n / check for k < check, sorted, unique."""
    k = np.arange(check, dtype=np.uint64)
    return np.unique((k * np.uint64(n) // np.uint64(check)).astype(np.uint32))


def relative_l2_error(estimate, reference) -> float:
    """bench.cpp:91-100: sqrt(sum (est-ref)^2 / sum ref^2); 0 or inf when the reference is 0."""
    e, r = np.asarray(estimate, dtype=np.float64), np.asarray(reference, dtype=np.float64)
    num, den = float(np.sum((e - r) ** 2)), float(np.sum(r * r))
    if den == 0:
        return 0.0 if num == 0 else float("inf")
    return float(np.sqrt(num / den))


def run_fmm(cfg: RunConfig, particles=None, check: int = 0):
    """run_fmm (bench.cpp:415-469): fields in input order; with check > 0 also the
    accuracy against the exact sum at `check` sampled targets (bench.cpp:378-398),
    computed on the device. Returns (fields, eps_potential, eps_force)."""
    xyzw = generate_particles(cfg.n, cfg.dist, cfg.seed) if particles is None else particles
    with FmmContext(None, cfg) as ctx:
        fields = ctx.run(xyzw, cfg.height, cfg.group_size)
        if check <= 0:
            return fields, -1.0, -1.0
        t = check_targets(len(xyzw), min(check, len(xyzw)))
        ref = ctx.direct(t)
    est_f = np.stack([fields[1][t], fields[2][t], fields[3][t]], axis=1).ravel()
    ref_f = np.stack(ref[1:], axis=1).ravel()
    return fields, relative_l2_error(fields[0][t], ref[0]), relative_l2_error(est_f, ref_f)
