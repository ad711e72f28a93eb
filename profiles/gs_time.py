"""Time tb_gram_schmidt on device-resident vectors: cfg 5's basis build (n = 12.8M dofs, k = 64
columns) and a trust-region-sized window (n = 241,602, 20 snapshots)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_05756_b200 import rom  # noqa: E402

for n, m in ((241_602, 20), (12_830_211, 64)):
    g = torch.Generator(device="cuda").manual_seed(0)
    cols = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
    rom._gs_device(cols, 1e-10)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        q = rom._gs_device(cols, 1e-10)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    e = (q.T @ q - torch.eye(q.shape[1], dtype=torch.float64, device="cuda")).abs().max().item()
    print(f"gram_schmidt n={n} m={m}: {dt * 1e3:.2f} ms  kept={q.shape[1]}  max|Q^T Q - I|={e:.2e}")
