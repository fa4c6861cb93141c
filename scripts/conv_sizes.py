"""Run the convolution at a list of shapes (argv: 'nb,h,w,c,f,r,s,pad' ...), check vs torch fp64 on a few pixels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1804_10694_b200 as tm
for spec in sys.argv[1:]:
    nb, h, w, c, f, r, s, pad = (int(v) for v in spec.split(","))
    X = torch.rand(nb, h, w, c, device="cuda"); Wt = torch.rand(f, r, s, c, device="cuda")
    ho, wo = h + 2 * pad - r + 1, w + 2 * pad - s + 1
    Y = torch.rand(nb, ho, wo, f, device="cuda")
    tm.conv2d_nhwc(X, Wt, Y, 1.0, 0.0, pad)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(X[:1].permute(0, 3, 1, 2).double(), Wt.permute(0, 3, 1, 2).double(), padding=pad)
    err = (Y[:1].permute(0, 3, 1, 2).double() - ref).abs().max().item() / ref.abs().max().item()
    print(spec, "ok, rel err image 0:", f"{err:.2e}", flush=True)
