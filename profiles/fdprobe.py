import sys, os, numpy as np, json
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '/root/repo')); sys.path.insert(0, os.path.join(os.environ.get('GRAFT_REPO_ROOT', '/root/repo'), 'baseline/_ref')); sys.path.insert(0,os.path.join(os.environ.get('GRAFT_REPO_ROOT', '/root/repo'), 'baseline/_ref/romtopt_tests'))
os.chdir(os.environ.get('GRAFT_REPO_ROOT', '/root/repo'))
import paper_2004_05756_b200 as tb
import romtopt
from romtopt.fem import build_mesh, elasticity_element_matrix
from romtopt.hdm import ComplianceObjective, MaterialModel
def make(cls_s, cls_f, nx=12, ny=4, **kw):
    mesh = build_mesh(nx, ny, 1.0); k_e = elasticity_element_matrix(1.0, 0.3, 1.0)
    filt = cls_f(mesh, 1.5, **({} if cls_f is romtopt.HelmholtzFilter else kw.get('fkw', {})))
    f = np.zeros(mesh.n_dofs); tip = mesh.node_id(nx, ny // 2); f[2 * tip + 1] = -1.0
    left = mesh.boundary_nodes("left"); fixed = np.concatenate([2 * left, 2 * left + 1])
    return cls_s(mesh, k_e, filt, f, fixed, material=MaterialModel(), **kw.get('skw', {}))
rng = np.random.default_rng(12)
ref = make(romtopt.HdmSolver, romtopt.HelmholtzFilter)
psi = 0.25 + 0.5 * rng.random(ref.mesh.n_elems)
obj = ComplianceObjective(ref.f)
sr = ref.solve(psi, obj); gr = ref.gradient(psi, sr, obj)
out = {}
for name, kw in [("default", {}), ("tight", dict(fkw=dict(rtol=1e-15), skw=dict(rtol=1e-13)))]:
    s = make(tb.HdmSolver, tb.HelmholtzFilter, **kw)
    so = s.solve(psi, obj); g = s.gradient(psi, so, obj)
    out[name] = dict(J_rel=abs(so.j - sr.j) / sr.j, rho_rel=float(np.abs(so.rho - sr.rho).max()),
                     u_rel=float(np.abs(so.u - sr.u).max() / np.abs(sr.u).max()),
                     g_rel=float(np.abs(g - gr).max() / np.abs(gr).max()), iters=so.iterations)
    e = int(np.argmax(np.abs(gr)))
    d = 1e-6; up, dn = psi.copy(), psi.copy(); up[e] += d; dn[e] -= d
    fd = (s.solve(up, obj).j - s.solve(dn, obj).j) / (2 * d)
    fdr = (ref.solve(up, obj).j - ref.solve(dn, obj).j) / (2 * d)
    out[name].update(fd=fd, fd_ref=fdr, g=float(g[e]), g_ref=float(gr[e]))
print(json.dumps(out, indent=1))
