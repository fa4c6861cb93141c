set -u
timeout 900 python -m pytest tests/test_dist_loopback.py -q -p no:cacheprovider --timeout 600 -x 2>&1 | tail -3
timeout 1500 python scripts/scaling_projection.py > gpurun_out/proj.log 2>&1
tail -1 gpurun_out/proj.log > gpurun_out/scaling_projection_r02.json
python - <<'PY'
import json
d = json.load(open("gpurun_out/scaling_projection_r02.json"))
print("T1", d["T1_ms"])
for P, res in d["P"].items():
    print(P, {k: v.get("projected_efficiency", v.get("error")) for k, v in res.items()})
PY
