"""Time tb_rom_project (Phi^T V) and tb_rom_gram-type passes over a cfg 5 size basis."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402

import torch  # noqa: E402

from paper_2004_05756_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
n, k = int(os.environ.get("N", 12830211)), 64
phi = torch.randn(n, k, dtype=torch.float64, device=dev)
lib = _lib.lib()
for nvec in (1, 16):
    vec = torch.randn(nvec, n, dtype=torch.float64, device=dev)
    out = torch.empty(nvec, k, dtype=torch.float64, device=dev)
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.tb_rom_project(ctypes.c_int64(n), _lib.ptr(phi), k, _lib.ptr(vec), nvec, _lib.ptr(out),
                                      _lib.stream_ptr(dev)), "project")
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
    ref = vec[:, :200000] @ phi[:200000]
    print(f"project {n} x {k}, {nvec} vectors: {ms:.3f} ms, {(n * k * 8 + nvec * n * 8) / ms / 1e6:.0f} GB/s")
