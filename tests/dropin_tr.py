"""The reference's TrustRegionDriver.run (trustregion.py:383-513) on its built-in ``mbb-small``
problem for a few major iterations, either pure reference (``ref``: romtopt on the CPU) or with
the B200 drop-in classes swapped in (``gpu``).  Prints the iteration records
as one JSON line.  Test infrastructure (tests/test_gpu_dropin.py compares the two)."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
os.environ["TB_DROPIN_PLUGIN"] = "0"  # import only; patch() below decides
import dropin_plugin  # noqa: E402  (puts baseline/_ref and the repo on sys.path)

mode, iters, method = sys.argv[1], int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "rom-tr-res"
if mode == "gpu":
    dropin_plugin.patch()
import romtopt.problems as P  # noqa: E402
import romtopt.trustregion as T  # noqa: E402
from romtopt.runner import RunConfig  # noqa: E402

spec = P.builtin_problem("mbb-small")
prob = P.assemble_problem(spec)
cfg = RunConfig()
driver = T.TrustRegionDriver(solver=prob.solver, rom=prob.rom, objective=prob.objective,
                             volume_weights=prob.volume_weights, volume_cap=prob.volume_cap,
                             config=cfg.tr_config("dist" if method == "rom-tr-dist" else "res", True),
                             stats=prob.stats)
recs = driver.run(prob.psi0, max_iters=iters)
out = [{"k": r.k, "j_center": r.j_center, "j_candidate": r.j_candidate, "accepted": bool(r.accepted),
        "rho_ratio": r.rho_ratio, "delta": r.delta, "basis_size": r.basis_size, "inner_steps": r.inner_steps,
        "theta": r.theta_candidate} for r in recs]
print(json.dumps({"mode": mode, "solver": type(prob.solver).__module__, "records": out,
                  "hdm_solves": prob.stats.hdm_solves, "rom_solves": prob.stats.rom_solves}))
