"""Time tb_rom_reconstruct (U = Phi Uhat, 16 designs) at cfg 5 size with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402

import torch  # noqa: E402

from paper_2004_05756_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
n, k, nd = int(os.environ.get("N", 12830211)), 64, 16
phi = torch.randn(n, k, dtype=torch.float64, device=dev)
uhat = torch.randn(nd, k, dtype=torch.float64, device=dev)
u = torch.empty(nd, n, dtype=torch.float64, device=dev)
lib = _lib.lib()
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(lib.tb_rom_reconstruct(ctypes.c_int64(n), _lib.ptr(phi), k, _lib.ptr(uhat), nd, _lib.ptr(u),
                                      _lib.stream_ptr(dev)), "reconstruct")
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
ref = (phi[:100000] @ uhat.T).T
err = (u[:, :100000] - ref).abs().max().item() / ref.abs().max().item()
print(f"reconstruct {n} x {k} x {nd}: {ms:.3f} ms, {(n * k * 8 + nd * n * 8) / ms / 1e6:.0f} GB/s, rel err {err:.2e}")
