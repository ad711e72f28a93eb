"""Reproduce the bench step loop (L2 flush, NVML sampler thread, events) and time each phase
of every step on the host to locate occasional ~20-45 ms outliers."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

prob = configs.cfg2()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
obj = tb.ComplianceObjective(s.f)
psi = torch.as_tensor(prob.psi, device="cuda")
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
use_nvml = len(sys.argv) > 1 and sys.argv[1] == "nvml"
stop = threading.Event()
if use_nvml:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)

    def run():
        while not stop.is_set():
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            stop.wait(0.1)
    threading.Thread(target=run, daemon=True).start()
for _ in range(3):
    sol = s.solve(psi, obj)
    s.gradient(psi, sol, obj)
torch.cuda.synchronize()
for k in range(8):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = [time.perf_counter()]
    a.record()
    rho, _ = s.filtered_density_device(psi)
    t.append(time.perf_counter())
    u = s.pcg_device(rho, s._f_d)
    t.append(time.perf_counter())
    sol = s.solve(psi, obj)
    t.append(time.perf_counter())
    g = s.gradient(psi, sol, obj)
    t.append(time.perf_counter())
    b.record()
    torch.cuda.synchronize()
    d = [round((t[i + 1] - t[i]) * 1e3, 2) for i in range(len(t) - 1)]
    print(f"step {k}: gpu {a.elapsed_time(b):7.2f} ms  host filter/pcg/solve/grad {d}")
stop.set()
