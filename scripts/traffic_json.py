"""Write profiles/ncu_traffic_<tag>.json (DRAM bytes per launch of the dominant
kernel per bench config) from the committed ncu summaries, for bench.py's
roofline.traffic.   python scripts/traffic_json.py r01"""
import json, os, re, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
if tag == "r01":
    files = {"C5": f"ncu_c5_k_sgemm_tc_{tag}.txt", "C4": f"ncu_c4_k_sgemm_tc_{tag}.txt",
             "C3:simt": f"ncu_c3_k_sgemm_simt_{tag}.txt", "CONV": f"ncu_conv_k_conv_direct_{tag}.txt"}
else:  # round 2 names (scripts/gpu_full_r02.sh)
    files = {"C5": f"ncu_C5_{tag}.txt", "C4": f"ncu_C4_{tag}.txt", "C3": f"ncu_C3_{tag}.txt", "C2": f"ncu_C2_{tag}.txt",
             "C1": f"ncu_C1_{tag}.txt", "C3:simt": f"ncu_simt_c3_{tag}.txt", "CONV": f"ncu_conv_{tag}.txt",
             "BLUR": f"ncu_blur_{tag}.txt"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TUNIT = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
out = {}
for key, name in files.items():
    path = os.path.join(ROOT, "profiles", name)
    if not os.path.exists(path):
        continue
    txt = open(path).read()
    kern = re.search(r"^## kernel: (.*)$", txt, re.M).group(1)
    def val(metric, table):
        m = re.search(rf"^{re.escape(metric)}\s+([\d.]+)\s+(\S+)", txt, re.M)
        return float(m.group(1)) * table[m.group(2)]
    out[key] = {"kernel": kern, "dram_read_bytes": val("dram__bytes_read.sum", UNIT),
                "dram_write_bytes": val("dram__bytes_write.sum", UNIT),
                "duration_s": val("gpu__time_duration.sum", TUNIT), "source": f"profiles/{name}"}
with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{tag}.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
