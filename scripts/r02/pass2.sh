set -u
timeout 1500 python -m pytest tests/ -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -4
python scripts/r02/rank_probe.py 2>&1 | grep auto
python scripts/scaling_projection.py > gpurun_out/proj.log 2>&1; tail -1 gpurun_out/proj.log > gpurun_out/scaling_projection_r02.json
python - <<'PY'
import json
d = json.load(open("gpurun_out/scaling_projection_r02.json"))
print("T1", d["T1_ms"])
for P, r in d["P"].items():
    print(P, r["rank_gemm_full_k_ms"], round(sum(r["gemm_ms_all_sms"]), 3), {k: v["projected_efficiency"] for k, v in r.items() if isinstance(v, dict)})
PY
