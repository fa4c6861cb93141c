"""Every stream-K schedule against the oracle: TM_SK_HYBRID=0 (pure stream-K:
the whole tiles x K-blocks space split evenly), 1 (only the partial wave's
tiles split, whole tiles after) and 2 (partial wave + one full wave split).
The mode is read once per process, so each runs in its own subprocess.  Shapes
have more tiles than clusters (so modes 1 and 2 differ from 0), ragged edges,
K tails, and both short (< 64 K-blocks, default mode 2) and long K (default 1),
plus partial waves too small to give every cluster two iterations (which must
fall back to pure stream-K: an empty cluster range would never publish the
partial its tile's finalizer waits for).
Each result must meet the 1e-5 bound (north_star tolerance) and
repeat bit for bit (fixed-order reduction)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHECK = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.environ["TM_ROOT"])
sys.path.insert(0, os.path.join(os.environ["TM_ROOT"], "tests"))
import seeded_inputs as si
from gpu_util import run, max_err
out = []
for (m, n, k, cfg) in ((2500, 2100, 700, "2,64,1"), (4100, 1000, 1200, "1,128,1"), (20000, 64, 580, "2,32,1"),
                       (1300, 1500, 2500, "2,128,1"),
                       # a partial wave too small to give every cluster two iterations
                       # (80 tiles of 2 / 1 K-blocks): falls back to pure stream-K
                       (2560, 2048, 64, "2,128,1"), (2560, 2048, 20, "2,128,1")):
    pad = lambda x: (x + 3) // 4 * 4
    A, B, C0 = si.matrices(m, n, k, seed=m + k, lda=pad(k), ldb=pad(n), ldc=pad(n))
    C1, _ = run(A, B, C0, si.ALPHA, si.BETA, 1, lda=pad(k), ldb=pad(n), ldc=pad(n), config=cfg)
    C2, _ = run(A, B, C0, si.ALPHA, si.BETA, 1, lda=pad(k), ldb=pad(n), ldc=pad(n), config=cfg)
    out.append({"shape": [m, n, k, cfg], "repeat": bool(np.array_equal(C1, C2)),
                "max_err": max_err(C1, A, B, C0, si.ALPHA, si.BETA)})
print(json.dumps(out))
'''


@pytest.mark.parametrize("mode", ["0", "1", "2"])
def test_streamk_mode_parity(mode):
    env = dict(os.environ, TM_ROOT=ROOT, TM_SK_HYBRID=mode)
    r = subprocess.run([sys.executable, "-c", CHECK], capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    for res in json.loads(r.stdout.strip().splitlines()[-1]):
        assert res["repeat"] and res["max_err"] <= 1e-5, (mode, res)
