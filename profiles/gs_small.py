import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2004_05756_b200 import rom
n, m = int(os.environ.get("GSN", "241602")), int(os.environ.get("GSM", "20"))
cols = torch.randn((m, n), dtype=torch.float64, device="cuda")
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    q = rom._gs_device(cols, 1e-10)
    torch.cuda.synchronize(); print(f"{(time.perf_counter() - t0) * 1e3:.2f} ms")
