import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2004_05756_b200 import _lib
n_e, n_u = 1769472, 5447811
psi = np.random.rand(n_e)
u_d = torch.randn(n_u, dtype=torch.float64, device="cuda")
def t(fn, reps=10):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): out = fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
print("to_dev psi (pageable)", t(lambda: _lib.to_dev(psi, torch.device("cuda"))))
print("np.array copy psi", t(lambda: np.array(psi, dtype=float, copy=True)))
print("array_equal psi", t(lambda: np.array_equal(psi.view(np.uint64), psi.copy().view(np.uint64))))
print("u to_user pinned", t(lambda: _lib.to_user(u_d, False)))
print("u .cpu() pageable", t(lambda: u_d.cpu().numpy()))
keep = []
print("u to_user pinned, results kept", t(lambda: keep.append(_lib.to_user(u_d, False))))
