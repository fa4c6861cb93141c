#!/usr/bin/env python
"""bench.py -- sgemm throughput on B200 (driver contract: one JSON line on rank 0).

Default workload (BASELINE.json configs[4], the config the metric is quoted on
"at 1/2/4/8 B200"): C = alpha*A*B + beta*C, M = N = K = 16384, fp32, alpha=1.5,
beta=0.5, row-block sharded over the N GPUs with B broadcast from rank 0 via
NCCL (strong scaling: total work fixed).  At N = 1 it is one tm_sgemm call.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C1|C2|C3|C3b|C4|C5] [--algo auto|tf32x3|simt]

A "step" is one pass of the whole hot path (one sgemm over the workload) with
inputs resident in HBM; `e2e` repeats the metric through tm_sgemm_host (host
buffers, copies inside the timed region).  `--impl reference` times the CPU
oracle (the tier's reference arm) on a bounded row sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sgemm GFLOP/s and % of TF32/FP32 roofline at 1/2/4/8 B200 vs CPU oracle"
ALGOS = {"auto": 0, "tf32x3": 1, "simt": 2, "tf32x1": 3, "bf16x9": 4}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0,
            "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(config, path, world):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed `ncu --set full` capture of this workload (profiles/ncu_traffic_*.json),
    or None when no capture matches (e.g. per-rank shards at N > 1)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_traffic_r*.json")))
    if not files or world != 1:
        return None, None
    with open(files[-1]) as f:
        d = json.load(f)
    key = config if path != "simt" else f"{config}:simt"
    if key not in d:
        return None, None
    e = d[key]
    return e["dram_read_bytes"] + e["dram_write_bytes"], os.path.relpath(files[-1], ROOT)


def roofline_peak(path, peaks):
    """(bound, peak, unit, note).  3xTF32: measured bf16 dense peak x nominal
    tf32/bf16 ratio (1.1/2.25) / 3 MMAs per fp32 product.  SIMT: FFMA peak from
    unit counts (148 SMs x 128 FP32 lanes x 2 flop x max SM clock)."""
    if path == "simt":
        return "alu", 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12, "TFLOP/s", "148 SM x 128 FFMA/clk x 2 x sm_max_mhz"
    if path == "bf16x9":  # nine bf16 MMAs per fp32 product
        return "tensor", peaks["bf16_tflops"] / 9.0, "TFLOP/s", f"{peaks['source']} bf16 {peaks['bf16_tflops']} / 9 (BF16x9)"
    tf32 = peaks["bf16_tflops"] * (1.1 / 2.25)
    if path == "tf32x1":  # one MMA per product: the TF32 dense peak itself
        return "tensor", tf32, "TFLOP/s", f"{peaks['source']} bf16 {peaks['bf16_tflops']} x 1.1/2.25 (tf32, 1xTF32)"
    return "tensor", tf32 / 3.0, "TFLOP/s", f"{peaks['source']} bf16 {peaks['bf16_tflops']} x 1.1/2.25 (tf32) / 3 (3xTF32)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []      # (host time of arrival, csv line)
        self.window = None   # (t0, t1) host times of the timed region

    def mark_region(self, t0, t1):
        """Host wall-clock bounds of the timed region: samples arriving inside it
        are the in-region ones."""
        self.window = (t0, t1)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *a):
        self.late = False
        if self.proc and not self.lines and not self.window:
            # timed region shorter than nvidia-smi's start-up: take the first
            # sample just after it (flagged in the summary) rather than none
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.02)
            self.late = bool(self.lines)
            del self.lines[1:]
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = [ln for _, ln in self.lines]
        where = "timed region"
        if self.window:
            # nvidia-smi prints a sample ~at its query time; allow one period of lag
            inside = [ln for t, ln in self.lines if self.window[0] <= t <= self.window[1] + 0.1]
            if inside:
                lines = inside
            else:
                where = "soak before the timed region (same kernel, back to back)"
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
               "sampled_during": where}
        if getattr(self, "late", False):
            out["note"] = "timed region shorter than the sampler start-up; one sample taken right after it"
        return out


# Test-only: TM_BENCH_SHARED_GPU=1 puts every rank on cuda:0 with a gloo
# process group, so the N > 1 code path (barriers, max over ranks, the
# copy-engine transport) can be exercised on a one-GPU box.  Its timings are
# meaningless (the ranks time-slice one GPU) and say so in the JSON line.
SHARED_GPU = os.environ.get("TM_BENCH_SHARED_GPU") == "1"


def init_dist(torch, dist, world, local):
    """Binds this rank's GPU and, for N > 1, the process group; returns the GPU index."""
    dev = 0 if SHARED_GPU else local
    torch.cuda.set_device(dev)
    if world > 1:
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    return dev


def max_over_ranks(torch, dist, world, values):
    """Element-wise max over ranks of a list of floats (CUDA events' ms)."""
    t = torch.tensor(values, dtype=torch.float64, device="cpu" if SHARED_GPU else "cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def soak_more(torch, dist, world, t_soak):
    """True while the >= 1 s soak before the timed steps should go on, agreed by
    every rank: each N > 1 step is a collective (the B broadcast / border
    exchange), so all ranks must run the same number of steps -- a per-rank
    wall-clock decision would leave one rank in a collective the others never
    join."""
    want = time.time() - t_soak < 1.0
    if world == 1:
        return want
    cpu = SHARED_GPU or dist.get_backend() == "gloo"
    t = torch.tensor([1.0 if want else 0.0], dtype=torch.float64, device="cpu" if cpu else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) > 0.0


def workload(name):
    import seeded_inputs as si
    m, n, k = si.CONFIGS[name]
    desc = {
        "C1": "sgemm 64^3 alpha=1.5 beta=0.5",
        "C2": "sgemm 1060^3 (partial tiles)",
        "C3": "sgemm 4096^3",
        "C3b": "sgemm 8192^3 (north_star target size)",
        "C4": "conv-shaped im2col sgemm 50176x64x576",
        "C5": "sgemm 16384^3 row-block sharded, B broadcast via NCCL",
    }[name]
    return m, n, k, desc


def make_inputs(name, m, n, k, rank_rows=None, device="cuda"):
    """Seeded synthetic inputs generated on the device (torch Philox, U[-1,1))
    for the big configs -- the parity tests use the numpy generator at the
    same shapes; throughput does not depend on the values."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(1804)
    r0, rows = rank_rows if rank_rows else (0, m)
    A = torch.rand((rows, k), generator=g, device=device, dtype=torch.float32) * 2 - 1
    B = torch.rand((k, n), generator=g, device=device, dtype=torch.float32) * 2 - 1
    C = torch.rand((rows, n), generator=g, device=device, dtype=torch.float32) * 2 - 1
    return A, B, C


def cpu_oracle_sample(m, n, k, alpha, beta, budget_s=15.0, extra_rows=()):
    """Times the CPU oracle (as it stands) on a row sample of the workload;
    returns (GFLOP/s extrapolated, cores, sample description)."""
    import numpy as np
    import oracle
    import seeded_inputs as si
    g = si.rng(99)
    B = si.uniform(g, (k, n))
    cores = oracle.get_threads()
    # calibrate on `cores` rows, then size the sample to ~budget_s
    rows = np.arange(min(m, cores), dtype=np.int64)
    A = si.uniform(g, (m if m <= 4 * cores else len(rows), k))
    C0 = si.uniform(g, (A.shape[0], n))
    t0 = time.perf_counter()
    oracle.sgemm(alpha, A, B, beta, C0, rows=rows, m=A.shape[0])
    t1 = time.perf_counter() - t0
    target = int(max(len(rows), min(m, len(rows) * budget_s / max(t1, 1e-3))))
    target = max(cores, target - target % cores) if target > cores else target
    A = si.uniform(g, (target, k))
    C0 = si.uniform(g, (target, n))
    t0 = time.perf_counter()
    oracle.sgemm(alpha, A, B, beta, C0)
    dt = time.perf_counter() - t0
    gflops = 2.0 * target * n * k / dt / 1e9
    return gflops, cores, f"{target} rows x {n} cols x K={k} of the {m}x{n}x{k} workload ({dt:.1f} s)"


def parity_sample(tm, torch, A, B, C0, alpha, beta, algo, path):
    """The timed launch configuration checked against the oracle on sampled
    rows of THIS run's inputs (part of the cpu_baseline leg): one more call on
    a fresh copy of C0, then max |C - R| / D over every column of the rows
    (tile and row-block boundaries plus seeded random rows)."""
    import numpy as np
    import oracle
    m = A.shape[0]
    Cc = C0.clone()
    tm.sgemm_ex(A, B, Cc, alpha, beta, algo)
    torch.cuda.synchronize()
    rows = {0, 1, m // 2, m - 2, m - 1} | {r for b in range(128, m, 128) for r in (b - 1, b)}  # every 128-row band
    rows |= set(np.random.default_rng(7).integers(0, m, size=48).tolist())
    rows = sorted(r for r in rows if 0 <= r < m)
    idx = torch.tensor(rows, device=A.device)
    R, D = oracle.sgemm(alpha, A.index_select(0, idx).cpu().numpy(), B.cpu().numpy(), beta,
                        C0.index_select(0, idx).cpu().numpy())
    err = float(np.max(oracle.normalized_error(Cc.index_select(0, idx).cpu().numpy(), R, D)))
    tol = 2.0 ** -9 + 2.0 ** -14 if path == "tf32x1" else 1e-5
    return {"rows": len(rows), "cols": int(B.shape[1]), "max_normalized_error": err, "tolerance": tol,
            "pass": err <= tol}


def run_reference_blur(args):
    """--impl reference --config BLUR: the blur oracle on a bounded row sample per
    step of the paper's 2112x3520 image; GB/s of the algorithmic bytes, scaled."""
    import numpy as np
    import oracle
    import seeded_inputs as si
    N, M = si.BLUR_IMAGE
    img = si.image(N, M)
    vals = []
    rows = np.arange(0, N - 2, 8, dtype=np.int64)  # every 8th output row: ~264 rows
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.blur(img, rows=rows)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(12 * len(rows) * (2 * M - 2) / dt / 1e9)
    value = statistics.median(vals)
    full = 12 * (N * M + (N - 2) * (M - 2))
    line = {"impl": "reference", "metric": "blur GB/s (PAPER.md:216-219 Blur on the 2112x3520 RGB image of PAPER.md:842)",
            "value": round(value, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(full / (value * 1e9) * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded U[0,1) RGB image, numpy PCG64)",
            "config": {"workload": f"blur {N}x{M}x3 (PAPER.md:842)"},
            "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": oracle.get_threads(), "kind": "oracle",
                             "sample": f"{len(rows)} of {N - 2} output rows per step; ms_per_step extrapolated"},
            "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import seeded_inputs as si
    if args.config == "BLUR":
        return run_reference_blur(args)
    if args.config == "CONV":
        print(json.dumps({"impl": "reference", "unavailable": "the CONV line is a SURVEY 8(f) extension; its oracle "
                                                              "parity runs in tests/test_conv.py (no reference arm)"}))
        return 0
    m, n, k, desc = workload(args.config)
    budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    vals = []
    sample = cores = None
    for i in range(args.warmup + args.steps):
        v, cores, sample = cpu_oracle_sample(m, n, k, si.ALPHA, si.BETA, budget_s=budget)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    flops = 2.0 * m * n * k
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(flops / (value * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded U[-1,1) fp32 inputs)",
        "config": {"workload": desc, "m": m, "n": n, "k": k, "alpha": si.ALPHA, "beta": si.BETA},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": sample + "; ms_per_step extrapolated to the full workload"},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C3b", "C4", "C5", "CONV", "BLUR"])
    ap.add_argument("--algo", default="auto", choices=list(ALGOS))
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ce"],
                    help="N > 1: B broadcast by NCCL (tm_sgemm_dist) or the copy-engine chain (tm_sgemm_dist_ce)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--conv-beta", type=float, default=0.0)
    ap.add_argument("--conv-r", type=int, default=3, help="filter size R = S (PAPER.md:835: 3..11)")
    ap.add_argument("--conv-valid", action="store_true", help="valid padding (PAPER.md:826 exact shape)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "CONV":
        return run_conv(args)
    if args.config == "BLUR":
        return run_blur(args)

    import torch
    import torch.distributed as dist

    import paper_1804_10694_b200 as tm
    import seeded_inputs as si

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    local = init_dist(torch, dist, world, local)
    peaks = load_peaks()
    m, n, k, desc = workload(args.config)
    alpha, beta = si.ALPHA, si.BETA
    algo = ALGOS[args.algo]
    stream = torch.cuda.current_stream()

    if args.config == "C4":
        A_np, B_np, C_np = si.im2col_conv()
        A, B, C = (torch.from_numpy(x).cuda() for x in (A_np, B_np, C_np))
        r0, rows = 0, m
    else:
        r0, rows = tm.dist_rows(m, world, rank)
        A, B, C = make_inputs(args.config, m, n, k, (r0, rows))
    comm = (tm.CeComm(rank, world) if args.transport == "ce" else tm.Comm(rank, world)) if world > 1 else None
    ce_handles = comm.exchange(B) if args.transport == "ce" and comm is not None else None
    in_bytes = 4 * (m * k + k * n + m * n)
    small = in_bytes < 2 * 126 * 2 ** 20  # inputs fit in L2: flush between iterations
    # L2 flush by READING 512 MiB (a write-flush would leave ~126 MB of dirty
    # lines whose write-back competes with the next GEMM's DRAM reads)
    flush = torch.ones(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda") if small else None
    flush_out = torch.empty(1, dtype=torch.float32, device="cuda")

    def step():
        if comm is None:
            tm.sgemm_ex(A, B, C, alpha, beta, algo)
        else:
            if ce_handles is not None:
                comm.sgemm(m, n, k, A, B, C, alpha, beta, root=0, handles=ce_handles)
            else:
                comm.sgemm(m, n, k, A, B, C, alpha, beta, root=0)

    path = tm.plan_name(rows, n, k, alpha, beta, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                        C.data_ptr(), C.stride(0), algo)
    check = rank == 0 and not args.no_cpu and world == 1
    C0 = C.clone() if check else None  # the steps update C in place; the parity sample needs the input

    def one(i=None):
        if flush is not None:
            torch.sum(flush, dim=0, out=flush_out[0])
        if i is not None:
            ev[i][0].record(stream)
        step()
        if i is not None:
            ev[i][1].record(stream)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        # The sampler starts before the warm-up, which then soaks the GPU with
        # the same step for >= 1 s, so short timed regions still have clock
        # samples under this load (in-region ones preferred, see summary()).
        t_soak = time.time()
        for _ in range(args.warmup):
            one()
        torch.cuda.synchronize()
        while soak_more(torch, dist, world, t_soak):
            for _ in range(8):
                one()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0_host = time.time()
        for i in range(args.steps):
            one(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks.mark_region(t0_host, time.time())
    per_step = [a.elapsed_time(b) for a, b in ev]  # ms, device time of each step's hot path
    total_ms = sum(per_step)
    med_ms = statistics.median(per_step)
    total_ms, med_ms = max_over_ranks(torch, dist, world, [total_ms, med_ms])
    ms_per_step = total_ms / args.steps
    flops = 2.0 * m * n * k
    value = flops * args.steps / (total_ms * 1e-3) / 1e9  # GFLOP/s, whole job

    # roofline of the dominant kernel (the GEMM), from this rank's live event times
    kernel = "simt" if path in ("simt", "simt_small") else path if path in ("tf32x1", "bf16x9") else "tf32x3"
    bound, peak, unit, peak_note = roofline_peak(kernel, peaks)
    my_flops = 2.0 * rows * n * k
    my_ms = statistics.median(per_step)  # the paper reports medians
    if args.config == "C4":
        bound, unit = "hbm", "GB/s"
        peak = peaks["hbm_gbs"]
        algo_bytes = 4 * (m * k + k * n + (2 if beta != 0 else 1) * m * n)
        achieved = algo_bytes / (my_ms * 1e-3) / 1e9
        peak_note = peaks["source"] + " hbm_gbs"
    else:
        achieved = my_flops / (my_ms * 1e-3) / 1e12
    traffic, traffic_src = ncu_traffic(args.config, path, world)
    roof = {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": unit,
            "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_unit": "bytes per launch",
            "traffic_source": traffic_src, "kernel": f"k_sgemm_tc ({path})" if kernel != "simt"
            else ("k_sgemm_small" if path == "simt_small" else "k_sgemm_simt"), "peak_source": peak_note}
    if path == "simt_small":
        roof["note"] = ("launch-latency bound (SURVEY.md 8(d): C1's roofline fraction is not meaningful; "
                        "step_ms.median is the figure)")
    if bound == "tensor":
        per_product = {"tf32x1": 1.0, "bf16x9": 9.0}.get(kernel, 3.0)  # tensor MMAs per fp32 product
        ratio = 1.0 if kernel == "bf16x9" else 1.1 / 2.25                  # bf16 -> tf32 nominal
        sus = peaks["bf16_tflops_sustained"] * ratio / per_product
        roof["frac_of_sustained_peak"] = round(achieved / sus, 4)
        # clock-normalised: against the tf32 rate measured by scripts/mma_rate.py
        # (4096 flop/clk/SM, kind::tf32; bf16 twice that) at the median SM clock sampled under load
        f_sm = clocks.summary().get("sm_mhz")
        if f_sm:
            clk_peak = 148 * (8192 if kernel == "bf16x9" else 4096) * f_sm * 1e6 / 1e12 / per_product
            roof["frac_clock_normalized"] = round(achieved / clk_peak, 4)
            roof["clock_normalized_peak"] = round(clk_peak, 2)
    launches = args.steps * (1 if comm is None else len(tm.dist_chunks(k, world)))

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "step_ms": {"median": round(med_ms, 4), "min": round(min(per_step), 4), "max": round(max(per_step), 4)},
        "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": {"simt": "f32", "tf32x1": "tf32 (1xTF32 tensor-core, fp32 accumulate)",
                                                          "bf16x9": "f32 (BF16x9 tensor-core, fp32 accumulate)"}.get(
            kernel, "f32 (3xTF32 tensor-core, fp32 accumulate)"), "data": "synthetic (seeded U[-1,1) fp32, device-generated)",
        "config": {"workload": desc, "m": m, "n": n, "k": k, "alpha": alpha, "beta": beta, "path": path,
                   "rows_per_rank": rows, "parallelism": f"row-shard x{world}" if world > 1 else "single GPU",
                   "transport": (args.transport if world > 1 else None),
                   "l2": "inputs larger than L2, no flush" if not small else "L2 flushed (512 MiB read) between steps"},
        "roofline": roof, "gpu_launches": launches, "clocks": clocks.summary(),
    }
    if SHARED_GPU and world > 1:
        line["note"] = "TM_BENCH_SHARED_GPU: all ranks time-slice cuda:0 -- a code-path check, not a measurement"

    # e2e through the public API with host buffers (copies inside the timed region)
    if not args.no_e2e:
        line["e2e"] = measure_e2e(tm, torch, dist, world, rank, m, n, k, rows, alpha, beta, algo, comm, args)

    if rank == 0 and not args.no_cpu and world == 1:
        v, cores, sample = cpu_oracle_sample(m, n, k, alpha, beta, budget_s=15.0)
        line["cpu_baseline"] = {"value": round(v, 3), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                                "sample": sample}
        line["cpu_baseline"]["parity_sample"] = parity_sample(tm, torch, A, B, C0, alpha, beta, algo, path)
    if comm is not None:
        comm.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_conv(args):
    """The paper's Conv benchmark shape (512x512 input, 16 input/output
    features, batch 32, 3x3 filter, here with 'same' padding; a convolution
    layer, so Y = conv(X, W): alpha 1, beta 0 unless --conv-beta) through the
    implicit-GEMM tensor-core convolution (not a
    BASELINE.json config).  Roofline: HBM (X read once, Y written [and read])."""
    import torch
    import paper_1804_10694_b200 as tm
    R = S = args.conv_r
    pad = 0 if args.conv_valid else R // 2
    Nb, H, W, C, F = 32, 512, 512, 16, 16
    Ho, Wo = H + 2 * pad - R + 1, W + 2 * pad - S + 1
    g = torch.Generator(device="cuda")
    g.manual_seed(1804)
    X = torch.rand((Nb, H, W, C), generator=g, device="cuda") * 2 - 1
    Wt = torch.rand((F, R, S, C), generator=g, device="cuda") * 2 - 1
    Y = torch.rand((Nb, Ho, Wo, F), generator=g, device="cuda") * 2 - 1
    algo = ALGOS[args.algo]
    alpha, beta = (1.0, 0.0) if args.conv_beta == 0.0 else (1.5, args.conv_beta)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(0) as clocks:
        t_soak = time.time()
        for _ in range(args.warmup):
            tm.conv2d_nhwc(X, Wt, Y, alpha, beta, pad, algo=algo)
        torch.cuda.synchronize()
        while time.time() - t_soak < 1.0:
            for _ in range(8):
                tm.conv2d_nhwc(X, Wt, Y, alpha, beta, pad, algo=algo)
            torch.cuda.synchronize()
        t0_host = time.time()
        for i in range(args.steps):
            ev[i][0].record()
            tm.conv2d_nhwc(X, Wt, Y, alpha, beta, pad, algo=algo)
            ev[i][1].record()
        torch.cuda.synchronize()
        clocks.mark_region(t0_host, time.time())
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)  # median
    flops = 2.0 * Nb * Ho * Wo * F * R * S * C
    algo_bytes = 4 * (X.numel() + Wt.numel() + (2 if beta != 0.0 else 1) * Y.numel())
    peaks = load_peaks()
    gbs = algo_bytes / (ms * 1e-3) / 1e9
    paper_default = R == 3 and not args.conv_valid
    traffic, traffic_src = (ncu_traffic("CONV", "tf32x3", 1) if (beta == 0.0 and algo != 2 and paper_default)
                            else (None, None))
    plan = tm.conv2d_plan_name(Nb, H, W, C, F, R, S, pad, alpha, algo, X.data_ptr(), Wt.data_ptr(), Y.data_ptr())
    # Dominant bound: HBM (X, W, Y once) for the 3x3 / 5x5 shapes, the tensor
    # cores for the large filters (K = R*S*C grows with the filter, the bytes do not)
    _, tpeak, _, tnote = roofline_peak("tf32x3" if algo != 2 else "simt", peaks)
    t_hbm, t_tc = algo_bytes / (peaks["hbm_gbs"] * 1e9), flops / (tpeak * 1e12)
    tensor_bound = t_tc > t_hbm
    line = {"metric": "conv2d GB/s (PAPER.md:826 Conv shape, 3xTF32 tensor cores)", "value": round(gbs, 2), "unit": "GB/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "dtype": "f32 (3xTF32 tensor-core)" if algo != 2 else "f32",
            "gflops": round(flops / (ms * 1e-3) / 1e9, 1), "data": "synthetic (device-generated U[-1,1))",
            "config": {"workload": f"PAPER.md:826 Conv: NHWC 32x512x512x16, KRSC 16x{R}x{S}x16, pad {pad}"
                                   f"{' (valid)' if args.conv_valid else ''}, alpha {alpha} beta {beta}",
                       "gemm_view": {"m": Nb * Ho * Wo, "n": F, "k": R * S * C},
                       "l2": "inputs larger than L2, no flush"},
            "roofline": {"bound": "tensor" if tensor_bound else "hbm",
                         "achieved": round(flops / (ms * 1e-3) / 1e12, 2) if tensor_bound else round(gbs, 1),
                         "peak": round(tpeak, 2) if tensor_bound else peaks["hbm_gbs"],
                         "unit": "TFLOP/s" if tensor_bound else "GB/s",
                         "frac": round((flops / (ms * 1e-3) / 1e12) / tpeak if tensor_bound else gbs / peaks["hbm_gbs"], 4),
                         "peak_source": tnote if tensor_bound else peaks["source"] + " hbm_gbs",
                         "hbm_frac": round(gbs / peaks["hbm_gbs"], 4), "traffic": traffic,
                         "traffic_unit": "bytes per launch", "traffic_source": traffic_src,
                         "algorithmic_bytes": algo_bytes,
                         "kernel": {"direct": "k_conv_direct", "direct_split": "k_conv_direct (2 launches)",
                                    "implicit_gemm": "k_sgemm_tc<CONV> (implicit GEMM)", "simt": "k_conv_simt"}.get(
                             plan, "?")},
            "gpu_launches": args.steps * (2 if plan == "direct_split" else 1),
            "clocks": clocks.summary()}
    print(json.dumps(line), flush=True)
    return 0


def run_blur(args):
    """The paper's Blur on its 2112x3520 RGB image
     through tm_blur (N = 1) or the row-distributed tm_blur_dist
    (N > 1: the Fig. 5 schedule, border rows over NCCL; strong scaling, the image
    is fixed).  SURVEY.md 8(f) item 3's second distributed workload, not a
    BASELINE.json config.  Roofline: HBM; algorithmic bytes = the image read once
    + the output written once, 12 (N M + (N-2)(M-2)) bytes.  The 89 MB image fits
    in L2, so L2 is flushed (512 MiB read) between steps."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1804_10694_b200 as tm
    import seeded_inputs as si
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = init_dist(torch, dist, world, local)
    N, M = si.BLUR_IMAGE
    img = si.image(N, M)
    r0, rows = tm.dist_rows(N - 2, world, rank)
    lin = torch.from_numpy(np.ascontiguousarray(img[r0:r0 + rows + 2])).cuda()  # chunk + border region
    if world > 1 and rank < world - 1:
        lin[rows:] = float("nan")  # received from rank + 1 every step
    lout = torch.empty((rows, M - 2, 3), dtype=torch.float32, device="cuda")
    if world > 1 and args.transport == "ce":
        raise SystemExit("--config BLUR: the border exchange runs over NCCL (--transport nccl)")
    comm = tm.Comm(rank, world) if world > 1 else None
    flush = torch.ones(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
    flush_out = torch.empty(1, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        if comm is None:
            tm.blur(lin, lout)
        else:
            comm.blur(N, M, lin, lout)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        t_soak = time.time()
        for _ in range(args.warmup):
            torch.sum(flush, dim=0, out=flush_out[0])
            step()
        torch.cuda.synchronize()
        while soak_more(torch, dist, world, t_soak):
            for _ in range(8):
                torch.sum(flush, dim=0, out=flush_out[0])
                step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0_host = time.time()
        for i in range(args.steps):
            torch.sum(flush, dim=0, out=flush_out[0])
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks.mark_region(t0_host, time.time())
    per_step = [a.elapsed_time(b) for a, b in ev]
    total_ms, med_ms = max_over_ranks(torch, dist, world, [sum(per_step), statistics.median(per_step)])
    algo_bytes = 12 * (N * M + (N - 2) * (M - 2))
    value = algo_bytes * args.steps / (total_ms * 1e-3) / 1e9
    my_bytes = 12 * ((rows + 2) * M + rows * (M - 2))
    my_gbs = my_bytes / (statistics.median(per_step) * 1e-3) / 1e9
    peaks = load_peaks()
    traffic, traffic_src = ncu_traffic("BLUR", "blur", world)
    line = {"metric": "blur GB/s (PAPER.md:216-219 Blur on the 2112x3520 RGB image of PAPER.md:842)",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_ms / args.steps, 5),
            "step_ms": {"median": round(med_ms, 5), "min": round(min(per_step), 5), "max": round(max(per_step), 5)},
            "mpixels_per_s": round((N - 2) * (M - 2) * args.steps / (total_ms * 1e-3) / 1e6, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded U[0,1) RGB image, numpy PCG64)",
            "config": {"workload": f"blur {N}x{M}x3 (PAPER.md:842)", "rows_per_rank": rows,
                       "parallelism": f"row-shard x{world} (Fig. 5 border exchange)" if world > 1 else "single GPU",
                       "l2": "L2 flushed (512 MiB read) between steps"},
            "roofline": {"bound": "hbm", "achieved": round(my_gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(my_gbs / peaks["hbm_gbs"], 4), "traffic": traffic,
                         "traffic_unit": "bytes per launch", "traffic_source": traffic_src,
                         "algorithmic_bytes": my_bytes, "kernel": "k_blur"},
            "gpu_launches": args.steps * (1 if world == 1 else 2), "clocks": clocks.summary()}
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        # parity of this run's output on sampled rows, and the oracle's rate on them
        rows_s = np.unique(np.concatenate([[0, 1, N - 4, N - 3], np.arange(31, N - 2, 32),
                                           np.random.default_rng(7).integers(0, N - 2, 64)])).astype(np.int64)
        t0 = time.perf_counter()
        R, D = oracle.blur(img, rows=rows_s)
        dt = time.perf_counter() - t0
        got = lout.cpu().numpy()[rows_s].astype(np.float64)
        err = float(np.max(np.abs(got - R) / np.where(D == 0, 1.0, D)))
        line["cpu_baseline"] = {"value": round(12 * len(rows_s) * (2 * M - 2) / dt / 1e9, 3), "unit": "GB/s",
                                "cores": oracle.get_threads(), "kind": "oracle",
                                "sample": f"{len(rows_s)} output rows x {M - 2} x 3 ({dt:.2f} s)",
                                "parity_sample": {"rows": int(len(rows_s)), "max_normalized_error": err,
                                                  "tolerance": 1e-6, "pass": err <= 1e-6}}
    if comm is not None:
        comm.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_e2e(tm, torch, dist, world, rank, m, n, k, rows, alpha, beta, algo, comm, args):
    steps = max(1, min(args.steps, 3))
    hA = torch.empty((rows, k), dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
    hB = torch.empty((k, n), dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
    hC = torch.empty((rows, n), dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
    if comm is None:
        def step():
            tm.sgemm_host(hA, hB, hC, alpha, beta, algo)
        h2d = 4 * (rows * k + k * n + rows * n)
    else:
        dA = torch.empty((rows, k), dtype=torch.float32, device="cuda")
        dB = torch.empty((k, n), dtype=torch.float32, device="cuda")
        dC = torch.empty((rows, n), dtype=torch.float32, device="cuda")

        def step():
            dA.copy_(hA, non_blocking=True)
            if rank == 0:
                dB.copy_(hB, non_blocking=True)
            dC.copy_(hC, non_blocking=True)
            comm.sgemm(m, n, k, dA, dB, dC, alpha, beta, root=0)
            hC.copy_(dC, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        h2d = 4 * (rows * k + (k * n if rank == 0 else 0) + rows * n)
    step()  # warm-up (workspace allocation)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    dt = max_over_ranks(torch, dist, world, [dt])[0]
    return {"value": round(2.0 * m * n * k * steps / dt / 1e9, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": 4 * rows * n, "steps": steps,
            "note": "tm_sgemm_host: pinned host A,B,C -> device, GEMM, C -> host, per step (host wall clock, synchronised)"
            if comm is None else "pinned H2D of shards + tm_sgemm_dist + D2H of C shard (host wall clock, max over ranks)"}


if __name__ == "__main__":
    sys.exit(main())
