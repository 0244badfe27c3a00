"""The C++ reference-API mirror (include/taskfmm_b200.hpp) as a C++ caller uses it:
compiled with g++ against libfmmgpu.so, run task by task and as evaluate(), checked
against the oracle (<= 1e-12 relative L2) and for the reference's exception classes."""
import os
import subprocess

import numpy as np
import pytest

from oracles import Oracle, OracleOps, OracleTree, RefContext, RefLib, force_error, relative_l2_error

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1206_0115_b200")


def build(tmp_path):
    exe = str(tmp_path / "adapter_main")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "adapter_main.cpp"), "-L", PKG, "-lfmmgpu",
                           f"-Wl,-rpath,{PKG}", "-o", exe])
    return exe


def test_adapter_compiles(tmp_path):
    """CPU-side: the header compiles and links against the exported C ABI."""
    if not os.path.exists(os.path.join(PKG, "libfmmgpu.so")):
        pytest.skip("libfmmgpu.so not built")
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_adapter_matches_oracle(tmp_path):
    exe = build(tmp_path)
    n, h, acc, seed = 20000, 5, 5, 42
    out = str(tmp_path / "fields.bin")
    r = subprocess.run([exe, str(n), str(h), str(acc), str(seed), out], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    data = np.fromfile(out).reshape(2, 4, n)
    xyzw = Oracle.generate_particles(n, "uniform", seed)
    ref = OracleTree(xyzw, h).evaluate(OracleOps.cached(acc))
    for fields in data:  # task-by-task and evaluate()
        assert relative_l2_error(fields[0], ref[0]) <= 1e-12
        assert force_error(*fields[1:], *ref[1:]) <= 1e-12


def downstream_first_order(kind, off, succ):
    """A topological order of the reference graph that always runs the most downstream
    ready task (L2P, then L2L, M2L, M2M, P2M, P2P, P2PReduce): L2L(v, b) runs as soon as
    its own M2L(v, b) and parent L2L have, before the M2L tasks of the other blocks."""
    import heapq
    nt = len(kind)
    npred = np.bincount(succ, minlength=nt).astype(np.int64)
    rank = {4: 0, 3: 1, 2: 2, 1: 3, 0: 4, 5: 5, 6: 6}
    ready = [(rank[int(kind[i])], i) for i in range(nt) if npred[i] == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        _, i = heapq.heappop(ready)
        order.append(i)
        for s in succ[off[i]:off[i + 1]]:
            npred[s] -= 1
            if npred[s] == 0:
                heapq.heappush(ready, (rank[int(kind[s])], int(s)))
    assert len(order) == nt
    return order


@pytest.mark.gpu
def test_adapter_runs_reference_graph_in_any_order(tmp_path):
    """the reference's own task graph for a ragged sphere cloud (group size 3,
    zero-pair M2L blocks elided, taskflow.cpp:179-186) executed through run_task in a
    downstream-first topological order, and by 8 threads at once, gives the evaluation."""
    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    exe = build(tmp_path)
    n, h, acc, seed, group = 4000, 5, 4, 3, 3
    xyzw = Oracle.generate_particles(n, "sphere", seed)
    kind, lev, blk, off, succ = RefContext(xyzw, h, acc, group_size=group).task_graph()
    order = downstream_first_order(kind, off, succ)
    tri = np.stack([kind[order].astype(np.int32), lev[order].astype(np.int32), blk[order].astype(np.int32)], 1)
    order_file = str(tmp_path / "order.bin")
    tri.astype(np.int32).tofile(order_file)
    out = str(tmp_path / "fields.bin")
    r = subprocess.run([exe, str(n), str(h), str(acc), str(seed), out, str(group), "1", order_file],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    data = np.fromfile(out).reshape(4, 4, n)
    ref = OracleTree(xyzw, h, group).evaluate(OracleOps.cached(acc))
    for fields in data:  # fixed order, evaluate(), downstream-first order, 8 threads
        assert relative_l2_error(fields[0], ref[0]) <= 1e-12
        assert force_error(*fields[1:], *ref[1:]) <= 1e-12
