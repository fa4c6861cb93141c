"""Summarise an ncu report (or a launch-list csv) into a short text file for profiles/.

  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt
  python scripts/ncu_summary.py --launches gpurun_out/launches.csv > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__cluster_dim_x",
    "smsp__inst_executed.sum",
]


def summarise_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    header, units = rows[0], rows[1]
    out = [f"# ncu --set full summary of {path}"]
    for vals in rows[2:]:
        d = dict(zip(header, vals))
        u = dict(zip(header, units))
        out.append(f"\n## kernel: {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                out.append(f"{k:80s} {d[k]:>20s} {u.get(k, '')}")
        rb = float(d.get("dram__bytes_read.sum", "0") or 0)
        wb = float(d.get("dram__bytes_write.sum", "0") or 0)
        out.append(f"{'traffic = dram read + write (units as above)':80s} {rb + wb:>20.4f}")
    return "\n".join(out)


def summarise_launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    out = [f"# ncu launch list ({path}); gpu__time_duration per launch (cold-cache, serialised)"]
    tot = {}
    for r in rows:
        name = r["Kernel Name"]
        v = float(r["Metric Value"])
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(r["Metric Unit"], 1.0)
        ms = v * scale
        out.append(f"{r['ID']:>4s}  {ms:12.4f} ms  {name[:110]}")
        key = name.split("(")[0]
        tot[key] = tot.get(key, 0.0) + ms
    all_ms = sum(tot.values())
    out.append("\n# share of device time by kernel")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"{100 * v / all_ms:6.2f}%  {v:12.4f} ms  {k[:110]}")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(summarise_launches(sys.argv[2]))
    else:
        print(summarise_report(sys.argv[1]))
