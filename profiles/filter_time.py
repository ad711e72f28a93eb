"""Time the Helmholtz filter solve and its adjoint (device-resident) on a BASELINE config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

for name in sys.argv[1:] or ["cfg2", "cfg3"]:
    prob = getattr(configs, name)()
    filt = tb.HelmholtzFilter(prob.mesh, prob.radius)
    psi = torch.as_tensor(prob.psi, device="cuda")
    v = torch.rand(prob.mesh.n_elems, dtype=torch.float64, device="cuda")
    for fn, arg, label in ((filt.apply_device, psi, "apply"), (filt.apply_adjoint_device, v, "adjoint")):
        for _ in range(3):
            fn(arg)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn(arg)
        b.record()
        torch.cuda.synchronize()
        print(f"{name} filter {label}: {a.elapsed_time(b) / 10:.3f} ms, iterations {filt.last_iterations if hasattr(filt, 'last_iterations') else '?'}")
