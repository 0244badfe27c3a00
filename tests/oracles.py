"""ctypes bindings to the two CPU checkers (test infrastructure only).

* ``Oracle``  -> oracle/_build/liboracle.so, our CPU restatement of the reference
  algorithm (oracle/restate/fmm_oracle.cpp).
* ``RefLib``  -> oracle/_ref/libtaskfmm_ref.so, the UNMODIFIED reference sources
  compiled by oracle/build_ref.sh (optional: absent if /root/reference was never
  present where the repo was built).

Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline legs
import this module.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_uint, c_uint64, c_void_p, byref

import numpy as np

# the reference's Eigen-shim GEMMs call OpenBLAS inside its own worker threads: one BLAS
# thread each (read when the library loads), as bench.py's reference arm runs it
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtaskfmm_ref.so")

CELL_DTYPE = np.dtype(
    [("code", "<u8"), ("first_particle", "<u4"), ("particle_count", "<u4"), ("parent", "<u4"),
     ("first_child", "<u4"), ("child_count", "<u4"), ("_pad", "<u4")])

KIND = {"P2M": 0, "M2M": 1, "M2L": 2, "L2L": 3, "L2P": 4, "P2P": 5, "P2PREDUCE": 6}


def _p(a):
    return a.ctypes.data_as(c_void_p)


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


# ------------------------------------------------------------------ restatement
class Oracle:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                import subprocess
                subprocess.check_call([os.path.join(ROOT, "oracle", "build_oracle.sh")])
            L = ctypes.CDLL(ORACLE_SO)
            L.orc_last_error.restype = ctypes.c_char_p
            L.orc_morton_encode.restype = c_uint64
            L.orc_level_cells.restype = c_uint64
            L.orc_near_entries.restype = c_uint64
            L.orc_near_dump.restype = c_uint64
            L.orc_far_pairs.restype = c_uint64
            L.orc_s_eval.restype = c_double
            L.orc_s_eval.argtypes = [c_double, c_double, c_int]
            L.orc_count.restype = c_uint64
            cls._lib = L
        return cls._lib

    @classmethod
    def check(cls, rc):
        if rc != 0:
            raise CheckerError(rc, cls.lib().orc_last_error().decode())

    @classmethod
    def generate_particles(cls, n, dist="uniform", seed=42):
        out = np.zeros((n, 4))
        cls.lib().orc_generate_particles(c_uint64(n), {"uniform": 0, "sphere": 1, "ellipsoid": 2}[dist], c_uint64(seed), _p(out))
        return out


class OracleTree:
    """GroupTree restatement handle (geometry.cpp:59-161)."""

    def __init__(self, xyzw, height, group_size=250, root=None):
        self.L = Oracle.lib()
        self.xyzw = np.ascontiguousarray(xyzw, dtype=np.float64)
        self.n = len(self.xyzw)
        self.height = height
        self.group_size = group_size
        h = c_void_p()
        r = None if root is None else np.ascontiguousarray(root, dtype=np.float64)
        Oracle.check(self.L.orc_tree_create(_p(self.xyzw), c_uint64(self.n), height, group_size,
                                            None if r is None else _p(r), byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_tree_destroy(self.h)
            self.h = None

    def root_cube(self):
        out = np.zeros(4)
        self.L.orc_root_cube(self.h, _p(out))
        return out

    def level(self, v):
        n = self.L.orc_level_cells(self.h, v)
        cells = np.zeros(n, dtype=CELL_DTYPE)
        nb = (n + self.group_size - 1) // self.group_size
        bo = np.zeros(nb + 1, dtype=np.uint32)
        self.L.orc_level_dump(self.h, v, _p(cells), _p(bo))
        return cells, bo

    def particles(self):
        x, y, z, w = (np.zeros(self.n) for _ in range(4))
        ids = np.zeros(self.n, dtype=np.uint32)
        self.L.orc_sorted_particles(self.h, _p(x), _p(y), _p(z), _p(w), _p(ids))
        return x, y, z, w, ids

    def near(self):
        ne = self.L.orc_near_entries(self.h)
        nc = self.L.orc_level_cells(self.h, self.height - 1)
        off = np.zeros(nc + 1, dtype=np.uint32)
        cells = np.zeros(ne, dtype=np.uint32)
        nb = (nc + self.group_size - 1) // self.group_size
        ti = np.zeros(nb, dtype=np.uint64)
        total = self.L.orc_near_dump(self.h, _p(off), _p(cells), _p(ti))
        return off, cells, ti, int(total)

    def far(self, v):
        npairs = self.L.orc_far_pairs(self.h, v)
        nc = self.L.orc_level_cells(self.h, v)
        nb = (nc + self.group_size - 1) // self.group_size
        t = np.zeros(npairs, dtype=np.uint32)
        s = np.zeros(npairs, dtype=np.uint32)
        vec = np.zeros(npairs, dtype=np.uint16)
        go = np.zeros(nb * 16 + 1, dtype=np.uint64)
        self.L.orc_far_dump(self.h, v, _p(t), _p(s), _p(vec), _p(go))
        return t, s, vec, go

    def evaluate(self, ops, mask=63, mutual=True):
        out = [np.zeros(self.n) for _ in range(4)]
        Oracle.check(self.L.orc_evaluate(self.h, ops.h, c_uint(mask), 1 if mutual else 0, *[_p(a) for a in out]))
        return out

    def expansion(self, v, which, order):
        n = self.L.orc_level_cells(self.h, v)
        out = np.zeros(n * order ** 3)
        self.L.orc_level_expansion(self.h, v, which, _p(out))
        return out.reshape(n, order ** 3)

    def count(self, ops):
        pairs = np.zeros(self.height, dtype=np.uint64)
        flops = np.zeros(7, dtype=np.uint64)
        near = self.L.orc_count(self.h, ops.h, _p(pairs), _p(flops))
        return int(near), pairs, flops


class OracleOps:
    """M2LOperatorSet restatement (m2l.cpp:136-163); cache_path loads reference factors."""

    _memo = {}

    @classmethod
    def cached(cls, order):
        """Own-SVD operator set per order, computed once per process (Jacobi at l=7 takes seconds)."""
        if order not in cls._memo:
            cls._memo[order] = cls(order)
        return cls._memo[order]

    def __init__(self, order, eps=None, cache_path=None):
        self.L = Oracle.lib()
        self.order = order
        self.eps = 10.0 ** (-order) if eps is None else eps
        h = c_void_p()
        Oracle.check(self.L.orc_ops_create(order, c_double(self.eps),
                                           cache_path.encode() if cache_path else None, byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.orc_ops_destroy(self.h)
            self.h = None

    def ranks(self):
        r = np.zeros(16, dtype=np.int32)
        m = np.zeros(16, dtype=np.int32)
        self.L.orc_ops_ranks(self.h, _p(r), _p(m))
        return r, m

    def dense(self, c):
        n3 = self.order ** 3
        out = np.zeros((n3, n3))
        self.L.orc_ops_dense(self.h, c, _p(out))
        return out


# ------------------------------------------------------------------ reference itself
class RefLib:
    _lib = None

    @classmethod
    def available(cls):
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = ctypes.CDLL(REF_SO)
            L.ref_last_error.restype = ctypes.c_char_p
            for name in ("ref_setup_seconds", "ref_execute", "ref_build_m2l_cache"):
                getattr(L, name).restype = c_double
            L.ref_build_m2l_cache.argtypes = [c_int, c_double, ctypes.c_char_p, c_void_p]
            for name in ("ref_level_cells", "ref_level_blocks", "ref_near_entries", "ref_near_total_directional",
                         "ref_far_pairs", "ref_task_count", "ref_morton_encode", "ref_far_source_blocks_total",
                         "ref_near_block_list_sizes"):
                getattr(L, name).restype = c_uint64
            cls._lib = L
        return cls._lib

    @classmethod
    def check(cls, rc):
        if rc != 0:
            raise CheckerError(rc, cls.lib().ref_last_error().decode())


class RefContext:
    """FmmContext of the reference (bench.cpp:220-365) through oracle/_ref."""

    def __init__(self, xyzw, height, order, group_size=250):
        self.L = RefLib.lib()
        self.xyzw = np.ascontiguousarray(xyzw, dtype=np.float64)
        self.n = len(self.xyzw)
        self.height, self.order, self.group_size = height, order, group_size
        h = c_void_p()
        RefLib.check(self.L.ref_create(_p(self.xyzw), c_uint64(self.n), height, order, group_size, byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_destroy(self.h)
            self.h = None

    def setup_seconds(self):
        return self.L.ref_setup_seconds(self.h)

    def execute(self, workers=1, policy=1):
        t = self.L.ref_execute(self.h, workers, policy)
        if t < 0:
            raise CheckerError(5, self.L.ref_last_error().decode())
        return t

    def run_serial(self, kinds):
        mask = 0
        for k in kinds:
            mask |= 1 << KIND[k]
        RefLib.check(self.L.ref_run_serial(self.h, c_uint(mask)))

    def fields(self):
        out = [np.zeros(self.n) for _ in range(4)]
        self.L.ref_fields(self.h, *[_p(a) for a in out])
        return out

    def sorted_fields(self):
        out = [np.zeros(self.n) for _ in range(4)]
        self.L.ref_sorted_fields(self.h, *[_p(a) for a in out])
        return out

    def root_cube(self):
        out = np.zeros(4)
        self.L.ref_root_cube(self.h, _p(out))
        return out

    def level(self, v):
        n = self.L.ref_level_cells(self.h, v)
        nb = self.L.ref_level_blocks(self.h, v)
        cells = np.zeros(n, dtype=CELL_DTYPE)
        bo = np.zeros(nb + 1, dtype=np.uint32)
        self.L.ref_level_dump(self.h, v, _p(cells), _p(bo))
        return cells, bo

    def particles(self):
        x, y, z, w = (np.zeros(self.n) for _ in range(4))
        ids = np.zeros(self.n, dtype=np.uint32)
        self.L.ref_sorted_particles(self.h, _p(x), _p(y), _p(z), _p(w), _p(ids))
        return x, y, z, w, ids

    def expansion(self, v, which):
        n = self.L.ref_level_cells(self.h, v)
        out = np.zeros(n * self.order ** 3)
        self.L.ref_level_expansion(self.h, v, which, _p(out))
        return out.reshape(n, self.order ** 3)

    def near(self):
        ne = self.L.ref_near_entries(self.h)
        nc = self.L.ref_level_cells(self.h, self.height - 1)
        off = np.zeros(nc + 1, dtype=np.uint32)
        cells = np.zeros(ne, dtype=np.uint32)
        self.L.ref_near_dump(self.h, _p(off), _p(cells))
        nb = self.L.ref_level_blocks(self.h, self.height - 1)
        below_total = c_uint64()
        na = self.L.ref_near_block_list_sizes(self.h, byref(below_total))
        ti = np.zeros(nb, dtype=np.uint64)
        ao = np.zeros(nb + 1, dtype=np.uint32)
        a = np.zeros(max(na, 1), dtype=np.uint32)
        bo = np.zeros(nb + 1, dtype=np.uint32)
        b = np.zeros(max(below_total.value, 1), dtype=np.uint32)
        self.L.ref_near_blocks(self.h, _p(ti), _p(ao), _p(a), _p(bo), _p(b))
        self._blocks = (ti, ao, a[:na], bo, b[:below_total.value])
        return off, cells, ti, int(self.L.ref_near_total_directional(self.h))

    def near_blocks(self):
        """NearFieldPlan block arrays: (task_interactions, above_off, above, below_off, below)."""
        self.near()
        return self._blocks

    def far_source_blocks(self, v):
        """LevelM2L::source_blocks of level v as (offsets, blocks)."""
        total = self.L.ref_far_source_blocks_total(self.h, v)
        nb = self.L.ref_level_blocks(self.h, v)
        off = np.zeros(nb + 1, dtype=np.uint32)
        blk = np.zeros(max(total, 1), dtype=np.uint32)
        self.L.ref_far_source_blocks(self.h, v, _p(off), _p(blk))
        return off, blk[:total]

    def far(self, v):
        npairs = self.L.ref_far_pairs(self.h, v)
        nb = self.L.ref_level_blocks(self.h, v)
        t = np.zeros(npairs, dtype=np.uint32)
        s = np.zeros(npairs, dtype=np.uint32)
        vec = np.zeros(npairs, dtype=np.uint16)
        go = np.zeros(nb * 16 + 1, dtype=np.uint64)
        self.L.ref_far_dump(self.h, v, _p(t), _p(s), _p(vec), _p(go))
        return t, s, vec, go

    def save_m2l_cache(self, path):
        RefLib.check(self.L.ref_save_m2l_cache(self.h, path.encode()))

    def ranks(self):
        r = np.zeros(16, dtype=np.int32)
        self.L.ref_m2l_ranks(self.h, _p(r))
        return r

    def task_graph(self):
        """TaskGraph (taskflow.hpp:34-42): kind, level, block per task and the successor
        CSR (off, succ)."""
        L = self.L
        L.ref_task_edges.restype = c_uint64
        nt = L.ref_task_count(self.h)
        kind = np.zeros(nt, np.uint8)
        lev = np.zeros(nt, np.int16)
        blk = np.zeros(nt, np.uint32)
        work = np.zeros(nt, np.uint64)
        L.ref_task_info(self.h, _p(kind), _p(lev), _p(blk), _p(work))
        ne = L.ref_task_edges(self.h, None, None)
        off = np.zeros(nt + 1, np.uint32)
        succ = np.zeros(max(ne, 1), np.uint32)
        L.ref_task_edges(self.h, _p(off), _p(succ))
        return kind, lev, blk, off, succ[:ne]

    def ledger_rows(self):
        """count_interactions + build_ledger of this context (bench.cpp:440-442)."""
        h = self.height
        work = np.zeros((7, h), dtype=np.uint64)
        flops = np.zeros((7, h), dtype=np.uint64)
        pairs = np.zeros((h, 16), dtype=np.uint64)
        RefLib.check(self.L.ref_ctx_ledger(self.h, _p(flops), _p(work), _p(pairs)))
        return {"work": work, "flops": flops, "m2l_pairs": pairs}


def ref_run_fmm(n, dist, seed, height, acc, out_dir, group_size=250, workers=1, check=1000):
    """The reference's run_fmm with out_dir (its own results.csv / summary.json writers);
    returns (eps_potential, eps_force)."""
    L = RefLib.lib()
    eps = np.zeros(2)
    RefLib.check(L.ref_run_fmm(c_uint64(n), {"uniform": 0, "sphere": 1}[dist], c_uint64(seed), height, acc,
                               group_size, workers, c_uint64(check), out_dir.encode(), _p(eps)))
    return float(eps[0]), float(eps[1])


def relative_l2_error(est, ref):
    """bench.cpp:91-100"""
    est = np.asarray(est, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    den = float(np.sum(ref * ref))
    num = float(np.sum((est - ref) ** 2))
    if den == 0:
        return 0.0 if num == 0 else float("inf")
    return float(np.sqrt(num / den))


def force_error(fx, fy, fz, rx, ry, rz):
    return relative_l2_error(np.stack([fx, fy, fz], 1), np.stack([rx, ry, rz], 1))
