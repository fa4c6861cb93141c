"""The oracle's pins are load-bearing: real mutants of oracle/oracle.c fail them.

Each mutant is oracle.c compiled with -DORACLE_MUTANT=n (one step broken on
purpose: a dropped term, a wrong sign or index, a transposed operand, flipped
filter taps, a padding slip, the partition remainder on the wrong ranks, C0 read
when beta == 0; the list is in oracle.c's header).  The pin suites
(tests/test_oracle.py, tests/test_conv_oracle.py, tests/test_blur_oracle.py) are run against each mutant in
a subprocess through TM_ORACLE_LIB and must FAIL; the same harness on the
unmutated source (n = 0) must PASS, so a failure is the mutant's doing.
"""
import concurrent.futures as cf
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PINS = ["tests/test_oracle.py", "tests/test_conv_oracle.py", "tests/test_blur_oracle.py"]
MUTANTS = {
    1: "beta term dropped", 2: "last product dropped (k-1)", 3: "op(B) transposed",
    4: "lda ignored for A", 5: "fabs dropped from D", 6: "beta term subtracted",
    7: "alpha dropped", 8: "conv filter taps flipped", 9: "conv padding not subtracted",
    10: "partition remainder to the last ranks", 11: "beta == 0 reads C0",
    12: "blur bx reads j+1 for j+2", 13: "blur by misses its /3",
}


def _run_pins(n, tmp):
    lib = oracle.build_mutant(n, os.path.join(tmp, f"liboracle_mut{n}.so"))
    env = dict(os.environ, TM_ORACLE_LIB=lib, OMP_NUM_THREADS="2")
    r = subprocess.run([sys.executable, "-m", "pytest", *PINS, "-x", "-q", "-p", "no:cacheprovider"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    return n, r.returncode, r.stdout[-600:]


def test_oracle_mutants_fail_the_pins(tmp_path):
    with cf.ThreadPoolExecutor(max_workers=min(6, os.cpu_count() or 2)) as ex:
        results = list(ex.map(lambda n: _run_pins(n, str(tmp_path)), [0, *MUTANTS]))
    by = {n: (rc, out) for n, rc, out in results}
    assert by[0][0] == 0, "unmutated oracle must pass its pins:\n" + by[0][1]
    survivors = [f"{n} ({MUTANTS[n]})" for n in MUTANTS if by[n][0] == 0]
    assert not survivors, f"mutants not caught by any pin: {survivors}"
