"""Mutation tests of the product's guards: the library is
rebuilt with -DTM_MUTATE=n (tc_gemm.cuh), each build breaking one guard on
purpose, and the checks the parity suite relies on must catch it:

  1  partial-tile predicate ignored (every 4-column group stored as a full
     vector) -> the guard band beside C (ldc > n) is overwritten
     (full/partial tile separation);
  2  the B_lo split term dropped -> the 1e-5 normalized error bound is missed
     (3xTF32 without one correction term is ~2^-11 accurate).

The shipped library passes both checks (same script, same inputs).  The mutant
builds go to a temporary directory and are loaded by a subprocess through
TM_LIB_PATH; the product library is never replaced."""
import json
import os
import subprocess
import sys
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHECK = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["TM_ROOT"])
sys.path.insert(0, os.path.join(os.environ["TM_ROOT"], "tests"))
import seeded_inputs as si
from gpu_util import run, max_err, SENTINEL
m, n, k, ldc = 300, 70, 45, 80
A, B, C0 = si.matrices(m, n, k, 5, lda=48, ldb=72)
C, buf = run(A, B, C0, si.ALPHA, si.BETA, 1, lda=48, ldb=72, ldc=ldc, guard_rows=9, config="2,64")
print(json.dumps({"sentinel_ok": bool(np.all(buf[:m, n:] == SENTINEL) and np.all(buf[m:, :] == SENTINEL)),
                  "max_err": max_err(C, A, B, C0, si.ALPHA, si.BETA)}))
'''


def _check(lib=None):
    env = dict(os.environ, TM_ROOT=ROOT)
    if lib:
        env["TM_LIB_PATH"] = lib
    r = subprocess.run([sys.executable, "-c", CHECK], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_product_passes_the_checks():
    res = _check()
    assert res["sentinel_ok"] and res["max_err"] <= 1e-5, res


@pytest.mark.parametrize("mutant", [1, 2])
def test_mutant_is_caught(mutant):
    sys.path.insert(0, ROOT)
    import importlib.util
    spec = importlib.util.spec_from_file_location("_tm_build", os.path.join(ROOT, "paper_1804_10694_b200", "_build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    with tempfile.TemporaryDirectory(prefix="tm_mutant_") as d:
        lib = b.build(extra=[f"-DTM_MUTATE={mutant}"], out=os.path.join(d, f"libtm_mut{mutant}.so"))
        res = _check(lib)
    if mutant == 1:
        assert not res["sentinel_ok"], res          # the guard band caught the missing predicate
    else:
        assert res["sentinel_ok"] and res["max_err"] > 1e-5, res  # the tolerance caught the dropped term
