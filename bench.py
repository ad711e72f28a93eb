#!/usr/bin/env python
"""Benchmark of the FE-evaluation hot path (BASELINE.json metric) on B200.

Headline (default ``--config cfg3``): "FE solve+sensitivity s/eval" on BASELINE cfg 3, the
largest single-GPU configuration (192x96x96 Hex8 cantilever, 5,447,811 DOF): psi -> Helmholtz
filter (R = 2.5) -> clamp -> matrix-free Jacobi-pCG K(rho)u = f to a TRUE relative residual of
1e-8 -> compliance -> element sensitivities -> filter adjoint (the gradient).  One step = one
design evaluation with psi resident in HBM.  ``e2e`` repeats it through the reference-facing API
(HdmSolver.solve(numpy) + gradient -> numpy): H2D of psi, D2H of rho, u, g and the scalars.

Every other BASELINE config is measured in the same run under ``extra`` (cfg 1 and cfg 2 2D
evaluations, cfg 3 with the multigrid preconditioner, the cfg 4 43M-DOF evaluation sharded over
all ranks, the cfg 5 16-design ROM step), each with its roofline and its CPU baseline.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config cfg3]

Multi-GPU: cfg 1-3 do not shard (SURVEY §8e "replicas only"): N ranks run N independent
replicas, value = total step time (max over ranks) / (K * N).  The cfg 4 extra is one
evaluation slab-sharded over all N ranks (strong scaling).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
REF_PATH = os.path.join(REPO, "baseline", "_ref")  # romtopt installed from /root/reference (git-ignored)

METRIC = "FE solve+sensitivity s/eval"
UNIT = "s/eval"
# Jacobi-pCG iterations of the cfg 3 evaluation (seed 0) measured on B200; the standalone CPU
# reference arm extrapolates its fixed-budget CG sample to this count.
CFG3_JACOBI_ITERS = 2513


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"],
                    help="cfg1-3: HDM evaluation (headline cfg3); cfg4: slab-sharded 3D evaluation; cfg5: ROM step")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--precond", default="jacobi", choices=["mg", "jacobi"],
                    help="pCG preconditioner of the cfg1-3 evaluation (both stop on the same true residual)")
    ap.add_argument("--halo", default="peer", choices=["peer", "nccl"],
                    help="cfg4 halo exchange: NVLink peer stores fused into the update kernel, or NCCL send/recv")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--extras", default="cfg1,cfg2,cfg3mg,cfg4,cfg5", help="comma list of extras to run")
    ap.add_argument("--no-flush", action="store_true", help="diagnostic: skip the L2 flush between steps")
    return ap.parse_args()


def rank_info():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def peaks():
    try:
        return json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


def peak_source(pk):
    return "fallback (B200_PROFILING.md)" if pk.get("fallback") else "MEASURED_PEAKS.json hbm_gbs (burst copy)"


PC_DESC = {"mg": "multigrid-preconditioned CG (geometric MG, Galerkin coarse levels; 2D V(1,1), 3D V(2,2))",
           "jacobi": "matrix-free Jacobi-pCG"}


def workload_desc(prob, precond):
    m = prob.mesh
    dims = f"{m.nx}x{m.ny}" + (f"x{m.nz}" if m.dim == 3 else "")
    el = "Hex8" if m.dim == 3 else "Q4"
    return (f"{prob.name}: {dims} {el}, {m.n_dofs} DOF ({prob.n_free} free); Helmholtz filter R={prob.radius:g} + "
            f"{PC_DESC[precond]} to true-residual rtol {prob.rtol:g} + compliance + sensitivity + filter adjoint; fp64")


# --------------------------------------------------------------------------------------
# problems (cfg 3's design is pre-filtered with R = 2: on the GPU for our arm, on the CPU
# -- same restated Helmholtz operator, CG to 1e-13 -- for the standalone reference arm)
# --------------------------------------------------------------------------------------
def problem(name, seed, dev=None):
    from paper_2004_05756_b200 import configs

    if name != "cfg3":
        return getattr(configs, name)(seed=seed)
    if dev is not None:
        import torch

        import paper_2004_05756_b200 as tb

        def prefilter(mesh, psi0):
            return tb.HelmholtzFilter(mesh, 2.0).apply(torch.as_tensor(psi0, device=dev)).rho.cpu().numpy()
    else:
        from oracle import iterative as it
        from oracle.fem import build_grid

        def prefilter(mesh, psi0):
            g = build_grid(mesh.nx, mesh.ny, mesh.h, nz=mesh.nz)
            return it.Helmholtz(g, 2.0).filter_apply(psi0, rtol=1e-13)[1]
    return configs.cfg3(seed=seed, prefilter=prefilter)


# --------------------------------------------------------------------------------------
# CPU legs (cpu_baseline and --impl reference): the reference's own code where it can run,
# else the oracle restatement -- test/measurement infrastructure, never the product path
# --------------------------------------------------------------------------------------
def _romtopt():
    """The unmodified reference package, installed into baseline/_ref (pure Python)."""
    if os.path.isdir(os.path.join(REF_PATH, "romtopt")):
        if REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        try:
            import romtopt

            return romtopt
        except Exception:  # noqa: BLE001
            return None
    return None


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:  # noqa: BLE001
        return cores()


class Cpu2d:
    """cfg 1/2: the reference's HdmSolver.solve + gradient (SuperLU per design), romtopt itself
    when installed in baseline/_ref ("reference"), else the oracle port ("port")."""

    def __init__(self, prob):
        from paper_2004_05756_b200 import configs

        rt = _romtopt()
        m = prob.mesh
        if rt is not None:
            mesh = rt.build_mesh(m.nx, m.ny, m.h)
            filt = rt.HelmholtzFilter(mesh, prob.radius)
            self.solver = rt.HdmSolver(mesh, rt.elasticity_element_matrix(1.0, 0.3), filt, prob.f, prob.fixed,
                                       rt.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP))
            self.obj = rt.ComplianceObjective(self.solver.f)
            self.kind, self.what = "reference", "romtopt (baseline/_ref, unmodified) HdmSolver.solve + gradient"
        else:
            from oracle.fem import build_grid
            from oracle.hdm import Filter, Hdm, Material

            g = build_grid(m.nx, m.ny, m.h)
            self.hdm = Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed,
                           Material(configs.RHO_L, configs.P_SIMP))
            self.solver = None
            self.kind, self.what = "port", "oracle port of romtopt HdmSolver.solve + gradient"

    def eval(self, psi):
        if self.solver is not None:
            sol = self.solver.solve(psi, self.obj)
            self.solver.gradient(psi, sol, self.obj)
            return sol.j
        sol = self.hdm.solve(psi)
        self.hdm.gradient(sol)
        return sol["j"]

    def sample(self, psi, budget_s=60.0, max_n=20):
        t0 = time.perf_counter()
        self.eval(psi)
        n = 1
        per = time.perf_counter() - t0
        while n < max_n and (n + 1) * per <= budget_s:
            self.eval(psi)
            n += 1
        return (time.perf_counter() - t0) / n, n


class Cpu3d:
    """cfg 3/4: the reference cannot run in 3D, so the restated path on the
    host cores -- the reference's element-by-element K(rho)v (hdm.py:224-233) inside a
    Jacobi-PCG for a fixed iteration budget extrapolated to the GPU's iteration count, the
    Helmholtz filter and its adjoint by CG (filtering.py:73-114; the same budget rule when
    ``filter_its`` is given), and element_sensitivity (hdm.py:211-222)."""

    def __init__(self, prob):
        from oracle import iterative as it
        from oracle.fem import build_grid
        from paper_2004_05756_b200 import configs

        m = prob.mesh
        self.it, self.prob = it, prob
        self.grid = build_grid(m.nx, m.ny, m.h, nz=m.nz)
        self.hz = it.Helmholtz(self.grid, prob.radius)
        self.free = np.ones(m.n_dofs, bool)
        self.free[prob.fixed] = False
        self.rho_l, self.p = configs.RHO_L, configs.P_SIMP

    def step(self, psi, cg_iters, gpu_iters, filter_its=None, filter_sample=None):
        """Seconds per extrapolated evaluation and the sample description."""
        it, g, prob = self.it, self.grid, self.prob
        t = {}
        t0 = time.perf_counter()
        if filter_its is None:
            _, rho_raw = self.hz.filter_apply(psi, rtol=1e-13)
            t["filter"] = time.perf_counter() - t0
        else:  # sampled Helmholtz CG, extrapolated to the GPU's filter iterations
            b = self.hz.load_vector(psi)
            phi, _ = it.pcg(self.hz.apply, 1.0 / self.hz.diag, b, 1e-13, filter_sample, iters_only=filter_sample)
            rho_raw = self.hz.average(phi)
            t["filter"] = (time.perf_counter() - t0) * filter_its[0] / filter_sample
        rho = np.clip(rho_raw, self.rho_l, 1.0)
        a = it.alpha(rho, self.rho_l, self.p)
        kapply = lambda v: it.apply_stiffness(g, prob.k_e, a, v)  # noqa: E731
        dinv = np.where(self.free, 1.0 / np.where(self.free, it.stiffness_diagonal(g, prob.k_e, a, self.free), 1.0), 0.0)
        t1 = time.perf_counter()
        u, _ = it.pcg(kapply, dinv, prob.f, prob.rtol, cg_iters, iters_only=cg_iters)
        t["pcg_sample"] = time.perf_counter() - t1
        t["pcg"] = t["pcg_sample"] / cg_iters * gpu_iters
        t2 = time.perf_counter()
        float(prob.f @ u)
        s = it.element_sensitivity(g, prob.k_e, rho, u, u, self.rho_l, self.p)
        t["sensitivity"] = time.perf_counter() - t2
        t3 = time.perf_counter()
        if filter_its is None:
            self.hz.filter_adjoint(s, rtol=1e-13)
            t["adjoint"] = time.perf_counter() - t3
        else:
            q = self.hz.load_vector(s) / (g.elem_volume)  # same transfer cost as filtering.py:107-109
            it.pcg(self.hz.apply, 1.0 / self.hz.diag, q, 1e-13, filter_sample, iters_only=filter_sample)
            t["adjoint"] = (time.perf_counter() - t3) * filter_its[1] / filter_sample
        total = t["filter"] + t["pcg"] + t["sensitivity"] + t["adjoint"]
        return total, t


def cpu_cfg3(prob, gpu_iters, cg_iters=10):
    c = Cpu3d(prob)
    v, t = c.step(prob.psi, cg_iters, gpu_iters)
    return {"value": v, "unit": UNIT, "cores": _blas_threads(), "kind": "port",
            "sample": (f"restated cfg3 evaluation on the host (oracle/iterative.py, BASELINE.md §4.3): Helmholtz "
                       f"filter + adjoint by CG to 1e-13 (full), reference element formulas for K(rho)v and the "
                       f"sensitivities; Jacobi-PCG timed for {cg_iters} iterations ({t['pcg_sample']:.2f} s) and "
                       f"extrapolated to the GPU's {gpu_iters}; numpy, BLAS threads = cores"),
            "parts_s": t}


def cpu_cfg4(prob, gpu_iters, filter_its, cg_iters=2, filter_sample=2):
    c = Cpu3d(prob)
    v, t = c.step(prob.psi, cg_iters, gpu_iters, filter_its=filter_its, filter_sample=filter_sample)
    return {"value": v, "unit": UNIT, "cores": _blas_threads(), "kind": "port",
            "sample": (f"restated cfg4 evaluation on the host: {cg_iters} Jacobi-PCG iterations of the reference "
                       f"element formulas extrapolated to the GPU's {gpu_iters}, {filter_sample} Helmholtz CG "
                       f"iterations per filter solve extrapolated to {filter_its}; sensitivities in full"),
            "parts_s": t}


def cpu_cfg5(prob, chunk=8192):
    """16-design ROM step: the reference's reduced_stiffness (rom.py:254-262: one GEMM over the
    stacked element caches) and residual scatter (rom.py:309-325) on an element chunk with k = 64
    caches, scaled linearly to N_e (the full caches would need 103 GB)."""
    from paper_2004_05756_b200 import configs

    k, n_e, nd = prob.rom_k, prob.mesh.n_elems, len(prob.rom_designs)
    rng = np.random.default_rng(1)
    ephi = rng.standard_normal((chunk, 24, k))
    ekphi = np.matmul(prob.k_e, ephi)
    rho = prob.rom_designs[0][:chunk]
    rt = _romtopt()
    if rt is not None:
        rom = object.__new__(rt.RomModel)
        rom.material = rt.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)
        basis = rt.ReducedBasis(phi=np.zeros((1, k)), elem_phi=ephi, elem_k_phi=ekphi, f_hat=np.zeros(k))
        kind, who = "reference", "romtopt RomModel.reduced_stiffness (baseline/_ref, unmodified)"
        khat = lambda: rom.reduced_stiffness(basis, rho)  # noqa: E731
    else:
        kind, who = "port", "oracle restatement of rom.py:254-262"

        def khat():
            a = configs.RHO_L + (1 - configs.RHO_L) * rho**3
            return (ephi * a[:, None, None]).reshape(-1, k).T @ ekphi.reshape(-1, k)
    khat()
    reps, t0 = 0, time.perf_counter()
    while reps < 3 or time.perf_counter() - t0 < 2.0:
        khat()
        reps += 1
    t_k = (time.perf_counter() - t0) / reps
    uhat = rng.standard_normal(k)
    t1 = time.perf_counter()
    contrib = (ekphi @ uhat) * rho[:, None]
    np.bincount(np.arange(chunk * 24) % (chunk * 3), weights=contrib.ravel())
    t_r = time.perf_counter() - t1
    scale = n_e / chunk
    v = nd * (t_k + t_r) * scale
    return {"value": v, "unit": "s/step", "cores": _blas_threads(), "kind": kind,
            "sample": (f"{who} on a {chunk}-element chunk with k={k} caches ({t_k * 1e3:.1f} ms) + residual scatter "
                       f"({t_r * 1e3:.1f} ms), scaled x{scale:.0f} to N_e and x{nd} designs")}


# --------------------------------------------------------------------------------------
# clocks sampled during the timed region
# --------------------------------------------------------------------------------------
class Clocks:
    """SM clocks and throttle reasons sampled every 10 ms DURING the timed region (in-process
    NVML on a thread; the nvidia-smi CLI is the fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.stop_flag = None
        self.thread = None
        self.smi = None

    def start(self):
        if os.environ.get("TB_BENCH_CLOCKS", "nvml") == "off":  # diagnostic only
            return
        try:
            import threading

            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.stop_flag = threading.Event()

            def run():
                while not self.stop_flag.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        self.rows.append((sm, mx, rs))
                    except Exception:  # noqa: BLE001
                        pass
                    self.stop_flag.wait(0.01)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001 - no pynvml: nvidia-smi CLI
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            try:
                self.smi = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                             "--format=csv,noheader,nounits", "-lms", "10"], stdout=self.f,
                                            stderr=subprocess.DEVNULL)
            except OSError:
                self.smi = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join()
            sm = [r[0] for r in self.rows]
            mx = [r[1] for r in self.rows]
            reasons = sorted({n for r in self.rows for n, bit in self.REASONS.items() if r[2] & bit})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                    "reasons": reasons, "samples": len(self.rows), "source": "nvml"}
        if self.smi is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        time.sleep(0.25)
        self.smi.terminate()
        self.smi.wait()
        self.f.flush()
        rows = [[x.strip() for x in line.split(",")] for line in open(self.f.name)]
        rows = [r for r in rows if len(r) >= 6]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi"}


# --------------------------------------------------------------------------------------
# GPU legs
# --------------------------------------------------------------------------------------
import numpy as np  # noqa: E402


def make_solver(tb, configs, prob, precond):
    return tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                        tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol,
                        preconditioner=precond)


def time_steps(solver, obj, psi_d, torch, steps, warmup, flush=None):
    """Device-resident evaluations (solve + gradient): per-step CUDA-event ms, iterations."""
    sol = g = None
    for _ in range(max(warmup, 1)):  # results kept alive as in the timed loop (caching allocator)
        sol = solver.solve(psi_d, obj)
        g = solver.gradient(psi_d, sol, obj)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    iters = []
    for k in range(steps):
        if flush is not None:
            flush.zero_()  # L2 flush between steps, outside the step events
        ev[k][0].record()
        sol = solver.solve(psi_d, obj)
        g = solver.gradient(psi_d, sol, obj)
        ev[k][1].record()
        iters.append(sol.iterations)
    torch.cuda.synchronize()
    del g
    return [a.elapsed_time(b) for a, b in ev], iters, sol


def time_e2e(solver, obj, psi_host, steps, torch):
    """Seconds per evaluation through the reference-facing numpy API, and the bytes copied."""
    for _ in range(2):
        s_ = solver.solve(psi_host, obj)
        g_h = solver.gradient(psi_host, s_, obj)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        s_ = solver.solve(psi_host, obj)
        g_h = solver.gradient(psi_host, s_, obj)
        assert isinstance(g_h, np.ndarray) and np.isfinite(s_.j)
    torch.cuda.synchronize()
    m = solver.mesh
    # H2D: psi; D2H: rho, u, g (+ J and the clamp width); gradient reuses the solve's device
    # copies of rho and u (HdmSolution._dev), nothing else crosses
    return (time.perf_counter() - t0) / steps, 8 * m.n_elems, 8 * (2 * m.n_elems + m.n_dofs) + 16


def pcg_path(_lib, plan):
    """Which 3D Jacobi-pCG the plan runs: "sweep" (one single-reduction kernel per iteration)
    or "two-kernel" (operator + update)."""
    fn = getattr(_lib.lib(), "tb_pcg_path", None)
    if fn is None:
        return "two-kernel"
    import ctypes

    fn.argtypes, fn.restype = [ctypes.c_void_p], ctypes.c_int
    return "sweep" if fn(plan) == 1 else "two-kernel"


def rom_profile(_lib, rom, basis, rhos, pk, torch):
    """Dominant kernel of the ROM step: Phi^T K(rho_d) Phi for all designs of the batch
    (tb_rom_reduced_stiffness -> k_rom_fused on Hex8 plans), CUDA events around the call on the
    current stream.  Fused path: tensor-bound, executed DMMA flops from tb_rom_fused_info against
    the cuBLAS DGEMM throughput measured in this run; else: Phi streamed once, against HBM."""
    import ctypes

    m = rom.mesh
    k = basis.size
    nd = rhos.shape[0]
    for _ in range(2):
        rom.reduced_stiffness_device(basis, rhos)
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rom.reduced_stiffness_device(basis, rhos)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    t = statistics.median(ts)
    fl = ctypes.c_double(0.0)
    fused = _lib.lib().tb_rom_fused_info(rom._plan, k, nd, ctypes.byref(fl)) == 1
    if fused:
        tf = fl.value / t / 1e12
        return {"kernel": "k_rom_fused<64> (element form: S_e = C_e^T C_e on DMMA m8n8k4 f64, weighted into all designs "
                          "by DMMA; warp-specialised producers stream Phi with cp.async.bulk)",
                "bound": "tensor", "achieved": tf, "peak": pk.get("fp64_tflops"), "unit": "TFLOP/s", "us": t * 1e6,
                "flops": fl.value, "launches_per_step": 1,
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (MEASURED_PEAKS.json has no FP64 figure)",
                "note": (f"one call = K_hat for all {nd} designs (+ a 2 us partial reduction); executed tensor flops per "
                         f"element and 8x8 tile: 5 DMMA (S) + ceil(nd/8) * 8 / 4 DMMA (weighting)")}
    by = 8 * (m.n_dofs * k + nd * m.n_elems)
    return {"kernel": "tb_rom_reduced_stiffness (all designs of the step)",
            "bound": "hbm", "achieved": by / t / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s", "us": t * 1e6,
            "bytes": by, "launches_per_step": 1, "peak_source": peak_source(pk),
            "note": f"one call = Phi^T K(rho_d) Phi for all {nd} designs; algorithmic bytes = Phi once + rho_d"}


def roofline_3d(tb, _lib, solver, rho_d, pk, torch, live=None):
    """Dominant kernel of the 3D Jacobi-pCG iteration.  Sweep path: timed live inside the timed
    steps (``live`` = tb_pcg_iter_time: CUDA events on the solve's stream around every
    iteration-graph launch, divided by the sweeps they ran); tb_pcg_profile (an event pair
    around each single launch, outside the timed region) is reported beside it.  Bytes: the
    algorithmic traffic of that kernel per SURVEY §8(d)."""
    import ctypes

    m = solver.mesh
    n_u, n_e = m.n_dofs, m.n_elems
    msf, msu = ctypes.c_double(0.0), ctypes.c_double(0.0)
    _lib.check(_lib.lib().tb_pcg_profile(solver._plan, _lib.ptr(rho_d), _lib.ptr(solver._f_d), 50, ctypes.byref(msf),
                                         ctypes.byref(msu), _lib.stream_ptr(rho_d.device)), "profile")
    path = pcg_path(_lib, solver._plan)
    if path == "sweep":  # one single-reduction sweep per iteration: the whole pCG iteration
        by = 8 * (9 * n_u + n_e)
        t = msf.value * 1e-3
        kern = ("k_hex8_cg (Chronopoulos-Gear Jacobi-pCG iteration in ONE z-sweep: TMA node planes, WHT-block Hex8 "
                "operator, x/r/p/s/w updates, 3 dot products; x update lagged on every other sweep; sweeps alternate z direction "
                "and store with an L2 evict_last policy so each starts on L2-resident planes)")
        note = "bytes = one Jacobi-pCG iteration, 8(9 N_u + N_e) (SURVEY §8(d)); the kernel IS the iteration"
        upd = None
        if live is not None and live[1] > 0:
            t = live[0] / live[1] * 1e-3
            note += (f"; time = {live[0]:.1f} ms of iteration-graph launches over {live[1]} sweeps inside the timed "
                     f"steps (events on the solve stream); isolated per-launch events: {msf.value * 1e3:.1f} us")
    else:
        by = 8 * (4 * n_u + n_e)
        t = msf.value * 1e-3
        kern = "k_hex8<true> (WHT-block Hex8 operator fused with p = z + beta p_old and p.q)"
        note = "bytes = z, p_old, alpha in; p, q out: 8(4 N_u + N_e)"
        by_u = 8 * 8 * n_u
        upd = {"us_per_launch": msu.value * 1e3, "bytes_per_launch": by_u,
               "achieved_gbs": by_u / (msu.value * 1e-3) / 1e9,
               "frac": by_u / (msu.value * 1e-3) / 1e9 / pk["hbm_gbs"]}
    ach = by / t / 1e9
    out = {"kernel": kern, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
           "frac": ach / pk["hbm_gbs"], "traffic": None, "bytes_per_launch": by, "us_per_launch": t * 1e6,
           "peak_source": peak_source(pk), "note": note}
    if upd is not None:
        out["update_kernel"] = upd
        out["us_per_iteration"] = (msf.value + msu.value) * 1e3
    else:
        out["us_per_iteration"] = msf.value * 1e3
    out["iteration_gbs_s8d"] = 8 * (9 * n_u + n_e) / (out["us_per_iteration"] * 1e-6) / 1e9
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath) and (m.nx, m.ny, m.nz) == (192, 96, 96):  # captured at cfg 3
        out["traffic"] = json.load(open(tpath)).get("cfg3_" + path)
    return out


def apply_roofline(solver, rho_d, pk, torch):
    """K(rho)u GDOF/s (HdmSolver.apply_stiffness, hdm.py:224-233, alpha(rho) included):
    20 calls captured in a CUDA graph, median of 5 replays; bytes 8(2 N_u + N_e).  Reported
    twice: back-to-back on one (rho, v) -- at cfg 3 the ~100 MB of operands can stay in the
    126 MB L2 -- and cold, the calls cycling through 4 distinct (rho, v) pairs (~230 MB of
    inputs), so every call streams its operands from HBM."""
    m = solver.mesh
    n_u = m.n_dofs
    by = 8 * (2 * n_u + m.n_elems)

    def timed(pairs):
        for r, v in pairs:
            solver.apply_device(r, v)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(20):
                r, v = pairs[i % len(pairs)]
                solver.apply_device(r, v)
        graph.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            graph.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 20 * 1e-3)
        del graph
        return statistics.median(ts)

    v = torch.randn(n_u, dtype=torch.float64, device=rho_d.device)
    t = timed([(rho_d, v)])
    cold = [(rho_d.clone(), torch.randn(n_u, dtype=torch.float64, device=rho_d.device)) for _ in range(4)]
    tc = timed(cold)
    del cold
    return {"us_per_call": t * 1e6, "gdofs": n_u / t / 1e9, "bytes_per_launch": by, "achieved_gbs": by / t / 1e9,
            "frac": by / t / 1e9 / pk["hbm_gbs"],
            "note": "back-to-back calls: v and rho may be L2-resident between calls when they fit in 126 MB",
            "bound_note": ("3D Hex8: the WHT-block operator is FP64-pipe bound, not HBM bound (~165 FP64 "
                           "instructions per element, ncu FP64 pipe 48% busy, arithmetic floor ~24 us at cfg 3; "
                           "DESIGN.md 4.1); frac is against HBM as SURVEY 8(d) asks") if m.dim == 3 else None,
            "cold": {"us_per_call": tc * 1e6, "gdofs": n_u / tc / 1e9, "achieved_gbs": by / tc / 1e9,
                     "frac": by / tc / 1e9 / pk["hbm_gbs"],
                     "note": "calls cycle through 4 distinct (rho, v) pairs: operands streamed from HBM"}}


def mg_bytes_per_iteration(nx, ny, min_dofs=1200):
    """Algorithmic bytes of one MG-preconditioned CG iteration of the persistent 2D kernel
    (k_mgpcg2d, V(1,1) cycle), each vector read or written once per phase."""
    levels = [(nx, ny)]
    while 2 * (levels[-1][0] + 1) * (levels[-1][1] + 1) > min_dofs:
        a, b = levels[-1]
        c = ((a + 1) // 2, (b + 1) // 2)
        if c == (a, b):
            break
        levels.append(c)
    n = [2 * (a + 1) * (b + 1) for a, b in levels]
    ne = nx * ny
    L = len(n)
    d = (4 * n[0] + ne) + 8 * n[0]
    d += 4 * n[0] + ne
    d += 2 * n[0] + n[1]
    d += 4 * n[0] + ne + 2 * n[0]
    for l in range(1, L - 1):
        d += n[l - 1] + 3 * n[l]
        d += 14 * n[l]
        d += 2 * n[l] + n[l + 1]
        d += 14 * n[l]
    d += n[L - 2] + 2 * n[L - 1]
    d += n[L - 1] ** 2 + 2 * n[L - 1]
    return 8 * d, n


def roofline_2d(solver, rho_d, pk, torch, precond):
    """2D: the whole solve is ONE persistent cooperative launch (Jacobi: k_pcg2d_treg; MG:
    k_mgpcg2d), timed with events around it; bytes = per-iteration model x iterations."""
    m = solver.mesh
    if precond == "mg":
        solver.pcg_device(rho_d, solver._f_d)
        solver.pcg_device(rho_d, solver._f_d)
        ms, launches = solver.last_kernel_time()
        t = ms * 1e-3
        per_it, _ = mg_bytes_per_iteration(m.nx, m.ny)
        kern = "k_mgpcg2d (persistent multigrid-preconditioned CG, one cooperative launch per solve)"
        note = ("hierarchy L2-resident; ~20 grid-barrier phases per V(1,1) iteration (latency-bound); the coarsest "
                "inverse (k_mg_gj_inverse) is set-up, not timed here")
    else:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        solver.pcg_device(rho_d, solver._f_d)
        a.record()
        solver.pcg_device(rho_d, solver._f_d)
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) * 1e-3
        per_it = 8 * (9 * m.n_dofs + m.n_elems)
        kern = "k_pcg2d_treg (persistent single-reduction Jacobi-pCG on node tiles, one launch per solve)"
        note = "working set L2/SMEM-resident; one grid barrier + partial exchange per iteration"
    its = solver.last_iterations
    ach = per_it * its / t / 1e9 if t > 0 else 0.0
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath) and m.nx == 600:  # captured at cfg 2
        traffic = json.load(open(tpath)).get("cfg2_mg" if precond == "mg" else "cfg2")
    return {"kernel": kern, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": ach / pk["hbm_gbs"], "traffic": traffic, "bytes_per_launch": per_it * its, "us_per_launch": t * 1e6,
            "iterations_per_launch": its, "us_per_iteration": t * 1e6 / max(its, 1), "bytes_per_iteration": per_it,
            "peak_source": peak_source(pk), "note": note}


def eval_extra(tb, configs, _lib, name, precond, dev, pk, torch, cpu, steps=5, prob=None):
    """One BASELINE evaluation config measured end to end: s/eval (device-resident), e2e through
    the numpy API, the dominant kernel's roofline and the CPU baseline."""
    prob = prob or problem(name, 0, dev)
    s = make_solver(tb, configs, prob, precond)
    obj = tb.ComplianceObjective(s.f)
    psi_d = torch.as_tensor(prob.psi, device=dev)
    ms, iters, sol = time_steps(s, obj, psi_d, torch, steps, 2)
    pin = torch.empty(prob.mesh.n_elems, dtype=torch.float64, pin_memory=True)
    pin.copy_(torch.from_numpy(prob.psi))
    e2e_t, h2d, d2h = time_e2e(s, obj, pin.numpy(), max(2, steps // 2), torch)
    rho_d, _ = s.filtered_density_device(psi_d)
    roof = roofline_3d(tb, _lib, s, rho_d, pk, torch) if prob.mesh.dim == 3 else roofline_2d(s, rho_d, pk, torch,
                                                                                              precond)
    out = {"workload": workload_desc(prob, precond), "value": statistics.median(ms) * 1e-3, "unit": UNIT,
           "pcg_iterations": int(statistics.median(iters)), "J": sol.j,
           "e2e": {"value": e2e_t, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
           "roofline": roof, "apply": apply_roofline(s, rho_d, pk, torch)}
    if cpu is not None:
        out["cpu_baseline"] = cpu(prob, out)
    del s, sol
    torch.cuda.empty_cache()
    return out


def cpu_2d_leg(prob, _out):
    c = Cpu2d(prob)
    v, n = c.sample(prob.psi, budget_s=30.0, max_n=5)
    return {"value": v, "unit": UNIT, "cores": _blas_threads(), "kind": c.kind,
            "sample": f"{n} full evaluations of {prob.name}: {c.what} (SuperLU single-threaded, BLAS on all cores)"}


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------
def run_ours(args):
    import torch

    import paper_2004_05756_b200 as tb
    from paper_2004_05756_b200 import _lib, configs

    rank, local, world = rank_info()
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pk = peaks()

    prob = problem(args.config, args.seed, dev)
    mesh = prob.mesh
    solver = make_solver(tb, configs, prob, args.precond)
    obj = tb.ComplianceObjective(solver.f)
    psi_d = torch.as_tensor(prob.psi, device=dev)
    flush = None if args.no_flush else torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev)  # 256 MiB

    clocks = Clocks(dev.index)
    clocks.start()  # before the warm-up: NVML start-up once stalled the first timed steps
    for _ in range(max(args.warmup, 3)):
        sol = solver.solve(psi_d, obj)
        g = solver.gradient(psi_d, sol, obj)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    live = None  # in-situ sweep timing over the timed steps (events around the iteration graphs)
    if mesh.dim == 3 and args.precond == "jacobi" and pcg_path(_lib, solver._plan) == "sweep":
        live = [ctypes.c_double(0.0), ctypes.c_int64(0)]
        _lib.check(_lib.lib().tb_pcg_iter_time(solver._plan, 1, ctypes.byref(live[0]), ctypes.byref(live[1])), "timer")
    launches0 = _lib.lib().tb_launch_count()
    step_ms, iters, sol = time_steps(solver, obj, psi_d, torch, args.steps, 0, flush)
    clk = clocks.stop()
    if live is not None:
        _lib.check(_lib.lib().tb_pcg_iter_time(solver._plan, 0, ctypes.byref(live[0]), ctypes.byref(live[1])), "timer")
        live = (live[0].value, live[1].value)
    launches = _lib.lib().tb_launch_count() - launches0
    if dist:
        dist.barrier()
    print("step ms:", [round(x, 3) for x in step_ms], file=sys.stderr)
    t = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = total_ms / 1e3 / (args.steps * world)

    pin = torch.empty(mesh.n_elems, dtype=torch.float64, pin_memory=True)
    pin.copy_(torch.from_numpy(prob.psi))
    e2e_t, h2d, d2h = time_e2e(solver, obj, pin.numpy(), args.steps, torch)
    e2e_d = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(e2e_d, op=dist.ReduceOp.MAX)
    e2e = {"value": float(e2e_d.item()) / world, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "api": "HdmSolver.solve(psi: numpy) + HdmSolver.gradient -> numpy (reference signatures)"}

    rho_d, _ = solver.filtered_density_device(psi_d)
    if mesh.dim == 3:
        roof = roofline_3d(tb, _lib, solver, rho_d, pk, torch, live) if args.precond == "jacobi" else None
    else:
        roof = roofline_2d(solver, rho_d, pk, torch, args.precond)
    apply = apply_roofline(solver, rho_d, pk, torch)
    its = int(statistics.median(iters))
    del solver, sol, g, rho_d
    torch.cuda.empty_cache()

    cpu = None
    want_cpu = rank == 0 and world == 1 and not args.no_cpu_baseline
    if want_cpu:
        cpu = cpu_cfg3(prob, its) if args.config == "cfg3" else cpu_2d_leg(prob, None)

    extras = {}
    if not args.no_extras:
        names = [x for x in args.extras.split(",") if x]
        leg2d = cpu_2d_leg if want_cpu else None
        if "cfg1" in names and args.config != "cfg1":
            extras["cfg1"] = {"mg": eval_extra(tb, configs, _lib, "cfg1", "mg", dev, pk, torch, leg2d),
                              "jacobi": eval_extra(tb, configs, _lib, "cfg1", "jacobi", dev, pk, torch, None)}
        if "cfg2" in names and args.config != "cfg2":
            p2 = problem("cfg2", 0)
            extras["cfg2"] = {"mg": eval_extra(tb, configs, _lib, "cfg2", "mg", dev, pk, torch, leg2d, prob=p2),
                              "jacobi": eval_extra(tb, configs, _lib, "cfg2", "jacobi", dev, pk, torch, None, prob=p2)}
            extras["cfg2"]["rom_khat_ms"] = rom_khat_ms(tb, configs, p2, dev, torch)
        if "cfg3mg" in names and args.config == "cfg3" and args.precond == "jacobi":
            extras["cfg3_mg"] = eval_extra(tb, configs, _lib, "cfg3", "mg", dev, pk, torch, None, prob=prob)
        if "cfg4" in names and os.environ.get("TB_BENCH_CFG4", "1") != "0":
            extras["cfg4_sharded"] = cfg4_extra(args, dev, dist, world, rank, pk, want_cpu)
        if "cfg5" in names and world == 1:
            extras["cfg5"] = cfg5_extra(args, dev, pk, want_cpu)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE cfg recipe, SURVEY App. B.1 / §8(d))",
            "config": {"workload": workload_desc(prob, args.precond), "preconditioner": args.precond,
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": ("256 MiB buffer written between steps (outside the step events); the cfg3 working set "
                              "(~350 MB of pCG vectors) also exceeds the 126 MB L2") if flush is not None else "no flush",
                       "pcg_iterations": its, "seed": args.seed,
                       "filter_solver": "direct (tensor-product cosine basis, DMMA mode products; spectral.cu)"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk, "apply": apply, "extra": extras,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def rom_khat_ms(tb, configs, prob, dev, torch):
    s = make_solver(tb, configs, prob, "jacobi")
    k = prob.rom_k
    phi = torch.linalg.qr(torch.randn(prob.mesh.n_dofs, k, dtype=torch.float64, device=dev))[0].contiguous()
    rom = tb.RomModel(s)
    basis = tb.ReducedBasis(phi, None, None, torch.zeros(k, dtype=torch.float64, device=dev))
    rho_d = torch.as_tensor(prob.psi, device=dev)
    for _ in range(2):
        rom.reduced_stiffness_device(basis, rho_d)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        rom.reduced_stiffness_device(basis, rho_d)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 10


def cfg4_extra(args, dev, dist, world, rank, pk, want_cpu):
    """BASELINE cfg 4 (43M DOF Hex8), one design evaluation.  N = 1: the single-GPU HdmSolver
    (Jacobi: the single-sweep TMA pCG; also the multigrid-preconditioned solve).
    N > 1: slab-sharded over ALL ranks of this run (slab_evaluate; strong scaling)."""
    import torch

    import paper_2004_05756_b200 as tb
    from paper_2004_05756_b200 import _lib, configs
    from paper_2004_05756_b200.slab import SlabFilter, SlabSolver, TorchComm, partition, slab_evaluate

    prob = configs.cfg4(seed=args.seed)
    m = prob.mesh
    by_it = 8 * (9 * m.n_dofs + m.n_elems)
    if world == 1:
        s = make_solver(tb, configs, prob, "jacobi")
        obj = tb.ComplianceObjective(s.f)
        psi_d = torch.as_tensor(prob.psi, device=dev)
        ms, iters, sol = time_steps(s, obj, psi_d, torch, 1, 1)
        rho_d, _ = s.filtered_density_device(psi_d)
        roof = roofline_3d(tb, _lib, s, rho_d, pk, torch)
        out = {"workload": workload_desc(prob, "jacobi"), "value": ms[0] * 1e-3, "unit": UNIT, "n_gpus": 1,
               "scaling": "strong", "pcg_iterations": iters[0], "J": sol.j, "roofline": roof,
               "path": "single-GPU HdmSolver (no slabs at N = 1)"}
        del s, sol, rho_d
        torch.cuda.empty_cache()
        smg = make_solver(tb, configs, prob, "mg")
        objm = tb.ComplianceObjective(smg.f)
        msm, itm, solm = time_steps(smg, objm, psi_d, torch, 2, 1)
        out["mg"] = {"workload": workload_desc(prob, "mg"), "value": statistics.median(msm) * 1e-3, "unit": UNIT,
                     "pcg_iterations": itm[-1], "J": solm.j,
                     "J_rel_vs_jacobi": abs(solm.j - out["J"]) / abs(out["J"])}
        del smg, solm
        torch.cuda.empty_cache()
        if want_cpu:
            out["cpu_baseline"] = cpu_cfg4(prob, out["pcg_iterations"], [21, 20])
        return out
    mat = tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)
    slab = partition(m.nz, world)[rank]
    sv = SlabSolver(m, prob.k_e, prob.f, prob.fixed, mat, slab, device=dev)
    fl = SlabFilter(m, prob.radius, slab, device=dev)
    psi = torch.as_tensor(sv.local_elems(prob.psi).copy(), device=dev)
    comm = TorchComm(peer=True)
    ev = slab_evaluate([sv], [fl], comm, [psi], rtol=prob.rtol)  # warm-up
    del ev
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ev = slab_evaluate([sv], [fl], comm, [psi], rtol=prob.rtol)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_eval = float(t.item())
    per_it = t_eval / max(ev.iterations, 1)
    out = {"workload": f"cfg4 {m.nx}x{m.ny}x{m.nz} Hex8, {m.n_dofs} DOF: filter R={prob.radius:g} + Jacobi-pCG "
                       f"{prob.rtol:g} + compliance + sensitivities + adjoint, z-slabs x{world}",
           "value": t_eval, "unit": UNIT, "n_gpus": world, "scaling": "strong", "pcg_iterations": ev.iterations,
           "filter_iterations": list(ev.filter_iterations), "J": ev.j,
           "halo": "NVLink peer stores (CUDA IPC)" if comm.peer_active else "nccl send/recv",
           "allreduces_per_iteration": getattr(comm, "allreduces", 0) / max(ev.iterations, 1),
           "roofline": {"kernel": "whole Jacobi-pCG iteration (upper bound: evaluation time / iterations)",
                        "bound": "hbm", "achieved": by_it / world / per_it / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": by_it / world / per_it / 1e9 / pk["hbm_gbs"], "traffic": None,
                        "bytes_per_iteration_per_rank": by_it / world, "us_per_iteration_upper_bound": per_it * 1e6,
                        "peak_source": peak_source(pk),
                        "note": "SURVEY §8(d) bytes 8(9 N_u + N_e) per iteration / N; filter and sensitivities included"}}
    del ev, sv, fl, psi
    torch.cuda.empty_cache()
    return out


def fp64_peak_tflops(torch, dev):
    """Measured FP64 GEMM throughput (cuBLAS DGEMM 8192^3, best of 5) as the FP64 roofline
    denominator; MEASURED_PEAKS.json carries no FP64 figure."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    del a, b
    return 2 * n**3 / best / 1e12


def cfg5_setup(tb, configs, dev, torch, seed=0):
    prob = configs.cfg5(seed=seed)
    m = prob.mesh
    s = make_solver(tb, configs, prob, "jacobi")
    k = prob.rom_k
    cols = configs.phi_columns(m, k, seed=seed, xp=torch, device=dev)
    cols[:, torch.as_tensor(~s.free_mask, device=dev)] = 0.0
    phi = tb.gram_schmidt(list(cols))
    del cols
    basis = tb.ReducedBasis(phi, None, None, phi.T @ s._f_d)
    rom = tb.RomModel(s)
    rhos = torch.as_tensor(np.stack(prob.rom_designs), device=dev)
    return prob, s, basis, rom, rhos


def cfg5_measure(tb, _lib, prob, basis, rom, rhos, dev, pk, torch, steps, warmup):
    """16-design ROM step timing + the dominant kernel's roofline (tb_rom_reduced_stiffness's
    kernel times, read back with tb_rom_profile when the library provides it)."""
    for _ in range(max(warmup, 1)):
        khat, uhat, norms = rom.solve_batch(basis, rhos)
    torch.cuda.synchronize()
    launches0 = _lib.lib().tb_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        ev[i][0].record()
        khat, uhat, norms = rom.solve_batch(basis, rhos)
        ev[i][1].record()
    torch.cuda.synchronize()
    launches = _lib.lib().tb_launch_count() - launches0
    t_step = statistics.median(a.elapsed_time(b) for a, b in ev) * 1e-3
    m = prob.mesh
    n_u, n_e, k, nd = m.n_dofs, m.n_elems, prob.rom_k, rhos.shape[0]
    prof = rom_profile(_lib, rom, basis, rhos, pk, torch)
    canonical = n_e * (2 * k * 24**2 + 2 * k**2 * 24)  # PAPER.md:664 element form, per design
    roof = {"kernel": prof["kernel"], "bound": prof["bound"], "achieved": prof["achieved"], "peak": prof["peak"],
            "unit": prof["unit"], "frac": prof["achieved"] / prof["peak"], "traffic": None,
            "us_per_launch": prof["us"], "bytes_per_launch": prof.get("bytes"), "flops_per_launch": prof.get("flops"),
            "peak_source": prof["peak_source"], "share_of_step": prof["us"] * prof.get("launches_per_step", 1) * 1e-6 / t_step,
            "note": prof.get("note", "")}
    out = {"workload": f"cfg5 {m.nx}x{m.ny}x{m.nz} Hex8, {n_u} DOF, k={k}, {nd} designs: Phi^T K(rho_d) Phi + batched "
                       "Cholesky + residual norms ||K Phi uhat - f||",
           "value": t_step, "unit": "s/step", "gpu_launches_per_step": launches / steps, "roofline": roof,
           "canonical_elementform_tflops_equiv": canonical * nd / t_step / 1e12,
           "residual_norms": norms[:4]}
    return out


def cfg5_extra(args, dev, pk, want_cpu):
    import torch

    import paper_2004_05756_b200 as tb
    from paper_2004_05756_b200 import _lib, configs

    prob, s, basis, rom, rhos = cfg5_setup(tb, configs, dev, torch, args.seed)
    pk = dict(pk)
    pk["fp64_tflops"] = fp64_peak_tflops(torch, dev)
    out = cfg5_measure(tb, _lib, prob, basis, rom, rhos, dev, pk, torch, 3, 1)
    del s, basis, rom, rhos
    torch.cuda.empty_cache()
    if want_cpu:
        out["cpu_baseline"] = cpu_cfg5(prob)
    return out


def run_cfg5(args):
    """BASELINE cfg 5 standalone line: per trust-region step, 16 designs x (Phi^T K(rho_d) Phi,
    reduced solve, ||K(rho_d) Phi uhat_d - f||), k = 64, 256x128x128 Hex8 (12.8M DOF)."""
    import torch

    import paper_2004_05756_b200 as tb
    from paper_2004_05756_b200 import _lib, configs

    rank, local, world = rank_info()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pk = dict(peaks())
    pk["fp64_tflops"] = fp64_peak_tflops(torch, dev)
    prob, s, basis, rom, rhos = cfg5_setup(tb, configs, dev, torch, args.seed)
    clocks = Clocks(dev.index)
    clocks.start()
    out = cfg5_measure(tb, _lib, prob, basis, rom, rhos, dev, pk, torch, args.steps, args.warmup)
    clk = clocks.stop()
    cpu = cpu_cfg5(prob) if (rank == 0 and not args.no_cpu_baseline) else None
    if rank == 0:
        print(json.dumps({
            "metric": "PhiT K Phi time (16-design ROM step)", "value": out["value"], "unit": "s/step", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 1), "ms_per_step": out["value"] * 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded cfg 5 recipe)", "config": {"workload": out["workload"], "parallelism": "single"},
            "roofline": out["roofline"], "cpu_baseline": cpu, "gpu_launches": int(out["gpu_launches_per_step"] * args.steps),
            "clocks": clk, "extra": {"residual_norms": out["residual_norms"]}}), flush=True)


def run_cfg4(args):
    """BASELINE cfg 4 standalone line: one evaluation on 384x192x192 Hex8 (43M DOF),
    slab-sharded along z over the ranks of the run."""
    import torch
    import torch.distributed as dist

    from paper_2004_05756_b200 import _lib

    rank, local, world = rank_info()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    pk = peaks()
    clocks = Clocks(dev.index)
    clocks.start()
    launches0 = _lib.lib().tb_launch_count()
    out = cfg4_extra(args, dev, dist if world > 1 else None, world, rank, pk,
                     rank == 0 and world == 1 and not args.no_cpu_baseline)
    launches = _lib.lib().tb_launch_count() - launches0
    clk = clocks.stop()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": out["value"], "unit": UNIT, "n_gpus": world, "steps": 1, "warmup": 1,
            "ms_per_step": out["value"] * 1e3, "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded cfg 4 recipe)",
            "config": {"workload": out["workload"], "parallelism": f"slab{world}", "halo": args.halo,
                       "pcg_iterations": out["pcg_iterations"], "filter_iterations": out.get("filter_iterations"),
                       "J": out["J"], "seed": args.seed},
            "roofline": out["roofline"], "cpu_baseline": out.get("cpu_baseline"),
            "gpu_launches": int(launches), "clocks": clk}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation on the host cores
# --------------------------------------------------------------------------------------
def run_reference(args):
    rank, _, world = rank_info()
    if rank != 0:
        return
    name = args.config
    budget = 150.0
    if name in ("cfg1", "cfg2"):
        prob = problem(name, args.seed)
        c = Cpu2d(prob)  # one-time set-up (filter factorisation, pattern) as the reference constructors
        for _ in range(min(args.warmup, 1)):
            c.eval(prob.psi)
        v, n = c.sample(prob.psi, budget_s=budget, max_n=args.steps)
        kind, sample = c.kind, f"{n} full evaluations: {c.what} (SuperLU single-threaded, BLAS on all cores)"
        unit, metric = UNIT, METRIC
        workload = workload_desc(prob, "jacobi").replace(PC_DESC["jacobi"], "SuperLU direct solve (fem.py:270-349)")
    elif name == "cfg5":
        prob = problem(name, args.seed)
        cb = cpu_cfg5(prob)
        v, n, kind, sample, unit = cb["value"], 1, cb["kind"], cb["sample"], "s/step"
        metric, workload = "PhiT K Phi time (16-design ROM step)", "cfg5 16-design ROM step on the host"
    else:
        prob = problem(name, args.seed)  # cfg3: CPU pre-filter (not timed)
        c = Cpu3d(prob)
        gpu_iters = CFG3_JACOBI_ITERS if name == "cfg3" else 7503
        vals, t0, n = [], time.perf_counter(), 0
        while n < max(args.steps, 1) and (n == 0 or time.perf_counter() - t0 < budget):
            if name == "cfg3":
                v1, _ = c.step(prob.psi, 10, gpu_iters)
            else:
                v1, _ = c.step(prob.psi, 2, gpu_iters, filter_its=(21, 20), filter_sample=2)
            vals.append(v1)
            n += 1
        v = statistics.median(vals)
        kind = "port"
        sample = (f"{n} restated {name} evaluations on the host (oracle/iterative.py, BASELINE.md §4.3): reference "
                  f"element formulas, Jacobi-PCG sampled for a fixed budget and extrapolated to {gpu_iters} iterations "
                  f"(the B200 run's count), Helmholtz filter/adjoint by CG")
        unit, metric = UNIT, METRIC
        workload = workload_desc(prob, "jacobi")
    line = {
        "impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": world, "steps": n,
        "warmup": min(args.warmup, 1), "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE recipe)",
        "config": {"workload": workload, "parallelism": "cpu", "seed": args.seed},
        "cpu_baseline": {"value": v, "unit": unit, "cores": _blas_threads(), "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "cfg5":
        run_cfg5(args)
    elif args.config == "cfg4":
        run_cfg4(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
