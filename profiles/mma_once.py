"""A few device MMA steps at cfg 2 / cfg 3 design sizes (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 120000
rng = np.random.default_rng(0)
w = torch.ones(n, dtype=torch.float64, device="cuda")
opt = tb.MmaOptimizer(torch.zeros_like(w), torch.ones_like(w), w, 0.4 * n)
x = torch.full((n,), 0.4, dtype=torch.float64, device="cuda")
for k in range(4):
    g = torch.as_tensor(-np.abs(rng.standard_normal(n)) - 0.01, device="cuda")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    x = opt.step(x, 0.0, g)
    b.record()
    torch.cuda.synchronize()
    print(f"mma step {k}: {a.elapsed_time(b):.3f} ms, volume {float(w @ x):.6f}")
