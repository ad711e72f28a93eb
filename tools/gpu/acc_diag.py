"""Diagnostic: one ROM-TR run of the reference's runner (romtopt.runner.run) on a built-in
benchmark, pure reference (ACC_DROPIN=0) or with the B200 drop-in classes (ACC_DROPIN=1,
optionally TB_DROPIN_PRECOND / TB_DROPIN_RTOL); prints the cutoff costs criterion 7 reads."""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [os.path.join(REPO, "tests"), os.path.join(REPO, "baseline", "_ref"), REPO]
if os.environ.get("ACC_DROPIN", "1") == "1":
    import dropin_plugin

    dropin_plugin.patch()
import romtopt.runner as rt  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ssbeam"
method = sys.argv[2] if len(sys.argv) > 2 else "rom-tr-res"
j_star = float(sys.argv[3]) if len(sys.argv) > 3 else None
cfg = rt.RunConfig().with_overrides({"max_iters": 160, "stop_eps": 0.0005})
t0 = time.time()
cache = rt.ReferenceCache(os.path.join(REPO, "baseline", "_ref", ".ref_cache"))
ref = rt.build_reference(rt.builtin_problem(name), rt.RunConfig(), cache=cache)
j_star = j_star if j_star is not None else ref["j_star"]


def cutoff_iteration(hist, js, eps):
    for k, j in enumerate(hist):
        if abs(j - js) < eps * abs(js):
            return k
    return None


mma = {str(e): cutoff_iteration(ref["j_history"], ref["j_star"], e) for e in (0.01, 0.001)}
rep = rt.run(name, method, config=cfg, j_star=j_star)
out = {"name": name, "method": method, "dropin": os.environ.get("ACC_DROPIN", "1"),
       "precond": os.environ.get("TB_DROPIN_PRECOND"), "rtol": os.environ.get("TB_DROPIN_RTOL"),
       "secs": round(time.time() - t0, 1), "j_star": j_star, "mma_cut": mma}
for eps in (0.01, 0.001):
    c = rep.cutoff(eps)
    out[str(eps)] = {"reached": c.reached, "n_hdm": c.n_hdm, "n_rom": c.n_rom, "c_eps": c.c_eps}
print(json.dumps(out))
