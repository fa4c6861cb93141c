"""Print the direct-conv kernel's CTA-0 timeline (TM_TRACE_PATH output), us relative to the first event."""
import json, sys
import numpy as np
names = ["halo_issued", "split_saw_halo", "mma_first_ready", "mma_last_commit", "epi_saw_last_part",
         "epi_stored", "split_last_ready", "mma_saw_last_ready"]
for line in open(sys.argv[1]):
    d = json.loads(line)
    if d.get("kernel") != "conv_direct":
        continue
    t = np.array(d["t"], dtype=np.float64).reshape(-1, d["ev"])
    t0 = t[t > 0].min()
    r = np.where(t > 0, (t - t0) / 1e3, np.nan)
    order = [0, 1, 2, 6, 7, 3, 4, 5]
    print("tile " + " ".join(f"{names[i][:16]:>16s}" for i in order))
    for i in range(r.shape[0]):
        print(f"{i:4d} " + " ".join(f"{r[i, j]:16.2f}" for j in order))
