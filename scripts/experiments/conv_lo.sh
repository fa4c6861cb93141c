# NOTE: TM_DC_LO_TRUNC was a temporary knob; the truncated A_lo is now the kernel default (reading 4)
python - <<'PY'
# accuracy of the paper-shape conv against the oracle on sampled pixels (max normalized error)
import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, torch, oracle, seeded_inputs as si, paper_1804_10694_b200 as tm
g = si.rng(3)
nb, h, w, c, f, r, s, pad = 4, 96, 100, 16, 16, 3, 3, 1
X = si.uniform(g, (nb, h, w, c)); W = si.uniform(g, (f, r, s, c)); Y0 = si.uniform(g, (nb, h, w, f))
for kind in ("uniform", "positive"):
    if kind == "positive":
        X = np.abs(X); W = np.abs(W); Y0 = np.abs(Y0)
    dY = torch.from_numpy(Y0.copy()).cuda()
    tm.conv2d_nhwc(torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda(), dY, 1.5, 0.5, pad)
    torch.cuda.synchronize()
    R, D = oracle.conv2d_nhwc(1.5, X, W, 0.5, Y0, pad)
    e = float(np.max(oracle.normalized_error(dY.cpu().numpy().reshape(R.shape), R, D)))
    print("conv", kind, "max normalized error", e)
PY
