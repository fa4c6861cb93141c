"""Print the clock64 event log of the direct conv kernel (TM_DC_CLK build): per tile, per pair."""
import json, sys
import numpy as np
for line in open(sys.argv[1]):
    d = json.loads(line)
    if d.get("kernel") != "conv_direct":
        continue
    t = np.array(d["t"], dtype=np.float64).reshape(16, 6, 8)
    t0 = t[t > 0].min()
    r = np.where(t > 0, t - t0, np.nan)
    for i in range(4, 10):
        tl = r[i, 5]
        print(f"tile {i}: halo_issue {tl[0]:.0f} split_halo_wait {tl[1]:.0f}->{tl[2]:.0f} "
              f"epi_wait {tl[3]:.0f}->{tl[4]:.0f} epi_store_end {tl[5]:.0f}  mma part_empty {r[i,0,6]:.0f}->{r[i,0,7]:.0f}")
        for j in range(5):
            e = r[i, j]
            print(f"   pair {j}: split wait {e[0]:.0f}->{e[1]:.0f} (+{e[1]-e[0]:.0f}) arrive {e[2]:.0f} (+{e[2]-e[1]:.0f}) | "
                  f"mma wait {e[3]:.0f}->{e[4]:.0f} (+{e[4]-e[3]:.0f}) commit {e[5]:.0f} (+{e[5]-e[4]:.0f})")
