"""CPU: the C-ABI library loads and exports every declared symbol; host-side mesh numbering,
element matrices, BC masks and config generators are bit-exact against the oracle/golden."""

import os
import re

import numpy as np
import pytest

from conftest import REPO, golden
from oracle.fem import build_grid, elasticity_element_matrix as ke_oracle, helmholtz_element_matrices as he_oracle
from paper_2004_05756_b200 import _lib, configs
from paper_2004_05756_b200.fem import (
    build_mesh,
    build_mesh_3d,
    elasticity_element_matrix,
    helmholtz_element_matrices,
    hex8_element_matrix,
)


def declared_symbols():
    src = open(os.path.join(REPO, "include", "topo_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(tb_\w+)\s*\(", src, flags=re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    lib = _lib.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.tb_version() >= 100
    nm = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", nm), name


def test_invalid_arguments_fail_loudly_without_gpu():
    import ctypes

    h = ctypes.c_void_p()
    ke = np.zeros(64)
    fixed = np.zeros(2, np.uint8)
    rc = _lib.lib().tb_plan_create(4, 1, 1, 1, 1.0, ke.ctypes.data_as(ctypes.c_void_p), 1e-3, 3.0,
                                   fixed.ctypes.data_as(ctypes.c_void_p), 0, ctypes.byref(h))
    assert rc == _lib.TB_ERR_INVALID and "dim" in _lib.last_error()
    with pytest.raises(ValueError):
        _lib.check(rc, "plan")


@pytest.mark.parametrize("nx,ny,h", [(3, 2, 0.5), (7, 5, 0.3), (120, 40, 1.0)])
def test_mesh_numbering_bit_exact(nx, ny, h):
    m = build_mesh(nx, ny, h)
    g = build_grid(nx, ny, h)
    assert np.array_equal(m.elem_nodes, g.elem_nodes)
    assert np.array_equal(m.elem_dofs, g.elem_dofs)
    for side in ("left", "right", "top", "bottom"):
        assert np.array_equal(m.boundary_nodes(side), g.boundary_nodes(side))


def test_mesh_numbering_3d_bit_exact():
    m = build_mesh_3d(4, 3, 2, 1.0)
    g = build_grid(4, 3, 1.0, nz=2)
    assert np.array_equal(m.elem_dofs, g.elem_dofs)
    for side in ("left", "right", "top", "bottom", "front", "back"):
        assert np.array_equal(m.boundary_nodes(side), g.boundary_nodes(side))
    assert m.n_dofs == 3 * 5 * 4 * 3


def test_reference_hand_enumeration():
    # reference tests/test_fem.py:35-56
    m = build_mesh(3, 2, 0.5)
    assert set(m.elem_nodes[4]) == {5, 6, 9, 10}
    assert list(m.boundary_nodes("left")) == [0, 4, 8]
    assert list(m.boundary_nodes("top")) == [8, 9, 10, 11]


def test_element_matrices_bit_exact():
    for nu in (0.0, 0.2, 0.3, 0.45):
        assert np.array_equal(elasticity_element_matrix(1.3, nu), ke_oracle(1.3, nu))
    for r, h in ((0.7, 0.3), (0.0, 0.5), (2.0, 0.1)):
        a, b = helmholtz_element_matrices(r, h), he_oracle(r, h)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.abs(hex8_element_matrix(1.0, 0.3) - ke_oracle(1.0, 0.3, 1.0, dim=3)).max() < 1e-15


def test_cfg1_inputs_and_bc_mask_match_golden():
    G = golden("golden_cfg1.npz")
    p = configs.cfg1()
    assert np.array_equal(p.psi, G["psi"])
    assert np.array_equal(p.fixed, G["fixed"])
    assert p.mesh.n_dofs == 9922


def test_config_sizes_and_loads():
    # DOF counts from d * prod(n_i + 1)
    assert configs.cfg2(nx=600, ny=200).mesh.n_dofs == 241602
    assert build_mesh_3d(192, 96, 96, 1.0).n_dofs == 5447811
    assert build_mesh_3d(384, 192, 192, 1.0).n_dofs == 43022595
    assert build_mesh_3d(256, 128, 128, 1.0).n_dofs == 12830211
    p3 = configs.cfg3(nx=8, ny=4, nz=4)
    assert abs(p3.f.sum() + 1.0) < 1e-15 and np.all(p3.f[0::3] == 0) and np.all(p3.f[1::3] == 0)
    assert p3.fixed.size == 3 * 5 * 5
    p4 = configs.cfg4(nx=8, ny=4, nz=4)
    assert abs(p4.f.sum() + 1.0) < 1e-15
    assert 0.01 <= p4.psi.min() and p4.psi.max() <= 1.0
    frac = np.mean(p4.psi >= 0.5)
    assert 0.25 <= frac <= 0.35
    p5 = configs.cfg5(nx=8, ny=4, nz=4, n_designs=3, k=5)
    assert len(p5.rom_designs) == 3 and all(d.min() >= 0.01 for d in p5.rom_designs)
    cols = configs.phi_columns(p5.mesh, 5, seed=0)
    assert cols.shape == (5, p5.mesh.n_dofs)
    # clamped face x = 0 carries no basis motion
    left = p5.mesh.boundary_nodes("left")
    assert np.abs(cols[:, 3 * left]).max() < 1e-15


def test_psi_digest_matches_reference_definition():
    import hashlib

    from paper_2004_05756_b200.hdm import psi_digest

    x = np.random.default_rng(0).random(17)
    assert psi_digest(x) == hashlib.sha256(x.astype(float).tobytes()).hexdigest()
