"""bench.py's driver contract on the box: the N = 1 line (C2, short) and the
N > 1 path (torchrun, two ranks time-slicing the one GPU via
TM_BENCH_SHARED_GPU=1, copy-engine transport) print one JSON line with the
required keys; the N = 2 line's world, transport and launch count are right."""
import json
import os
import signal
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks"}


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_n1_line():
    r = subprocess.run([sys.executable, "bench.py", "--config", "C2", "--steps", "5", "--warmup", "3", "--no-cpu",
                        "--no-e2e"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 5
    assert d["roofline"]["frac"] > 0 and d["clocks"]["samples"] >= 1


def test_bench_n2_shared_gpu_ce_transport():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, TM_BENCH_SHARED_GPU="1")
    # own session: on a timeout the whole process group (torchrun and its
    # ranks) is killed, so a hang cannot leave ranks running on the GPU
    p = subprocess.Popen([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                          "--config", "C3", "--transport", "ce", "--steps", "3", "--warmup", "3", "--no-cpu"],
                         cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, env=env,
                         start_new_session=True)
    try:
        out, err = p.communicate(timeout=600)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        p.communicate()
        raise
    assert p.returncode == 0, err[-3000:]
    d = _last_json(out)
    assert KEYS <= set(d)
    assert d["n_gpus"] == 2 and d["config"]["transport"] == "ce" and d["config"]["rows_per_rank"] == 2048
    assert d["gpu_launches"] == 3 * 3  # geometric chunks of K = 4096 at P = 2: 512, 1024, 2560
    assert "e2e" in d and d["e2e"]["value"] > 0
    assert "note" in d  # flagged as a code-path check, not a measurement
