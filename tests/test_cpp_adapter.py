"""The C++ reference-API mirror (include/taskfmm_b200.hpp) as a C++ caller uses it:
compiled with g++ against libfmmgpu.so, run task by task and as evaluate(), checked
against the oracle (<= 1e-12 relative L2) and for the reference's exception classes."""
import os
import subprocess

import numpy as np
import pytest

from oracles import Oracle, OracleOps, OracleTree, force_error, relative_l2_error

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
