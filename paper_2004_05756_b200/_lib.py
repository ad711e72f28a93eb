"""ctypes binding of libtopo_b200.so (the C ABI declared in include/topo_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``.  There is no
CPU fallback: if the library or a CUDA device is missing, every compute entry
point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TB_LIB_PATH") or os.path.join(_HERE, "libtopo_b200.so")

TB_OK = 0
TB_ERR_INVALID = 1
TB_ERR_CUDA = 2
TB_ERR_INDEFINITE = 3
TB_ERR_NOT_CONVERGED = 4
TB_ERR_DEGENERATE = 5
TB_ERR_DENSITY = 6
TB_ERR_RUNTIME = 7

# every symbol include/topo_b200.h declares
EXPORTS = (
    "tb_version", "tb_last_error", "tb_plan_create", "tb_plan_destroy", "tb_plan_sizes",
    "tb_material", "tb_clamp_density", "tb_apply_stiffness", "tb_element_sensitivity",
    "tb_pcg_solve", "tb_plan_set_preconditioner", "tb_pcg_profile", "tb_launch_count", "tb_plan_set_owned_planes", "tb_pcg_dist_phase",
    "tb_pcg_dist_buffers", "tb_pcg_dist_state", "tb_plan_set_halo_peers", "tb_ipc_get_handle", "tb_ipc_open",
    "tb_ipc_close", "tb_dot", "tb_filter_create", "tb_filter_destroy", "tb_filter_load_vector",
    "tb_filter_apply", "tb_filter_adjoint", "tb_rom_project", "tb_rom_reduced_stiffness",
    "tb_rom_gram_colmajor", "tb_rom_cholesky_solve", "tb_rom_reconstruct", "tb_rom_residual_norms", "tb_gram_schmidt",
    "tb_mma_workspace_bytes", "tb_mma_step", "tb_cone_create", "tb_cone_destroy", "tb_cone_apply",
    "tb_cone_adjoint", "tb_filter_set_owned_planes", "tb_filter_dist_phase", "tb_filter_dist_buffers",
    "tb_filter_dist_state", "tb_filter_set_halo_peers", "tb_filter_transfer", "tb_mgp_prof_read", "tb_pcg_kernel_time", "tb_pcg_iter_time", "tb_pcg_path", "tb_rom_fused_info",
)


class NotConvergedError(RuntimeError):
    """The matrix-free pCG did not reach its tolerance within maxit iterations."""


_lib = None

P = ctypes.c_void_p
I = ctypes.c_int
I64 = ctypes.c_int64
D = ctypes.c_double
PI = ctypes.POINTER(ctypes.c_int)
PD = ctypes.POINTER(ctypes.c_double)
PI64 = ctypes.POINTER(ctypes.c_int64)

class MmaConfigC(ctypes.Structure):
    """tb_mma_config (include/topo_b200.h) = MmaConfig (mma.py:25-38)."""

    _fields_ = [(f, ctypes.c_double) for f in ("asy_init", "asy_incr", "asy_decr", "asy_min_frac", "asy_max_frac",
                                                "move", "albefa", "raa0", "bisect_rtol")] + [
        ("bisect_max_iter", ctypes.c_int)]


_SIGS = {
    "tb_version": ([], I),
    "tb_last_error": ([], ctypes.c_char_p),
    "tb_plan_create": ([I, I, I, I, D, P, D, D, P, I, ctypes.POINTER(P)], I),
    "tb_plan_destroy": ([P], I),
    "tb_plan_sizes": ([P, PI64, PI64, PI64], I),
    "tb_material": ([P, P, P, P, P], I),
    "tb_clamp_density": ([P, P, P, PD, P], I),
    "tb_apply_stiffness": ([P, P, P, P, I, P], I),
    "tb_element_sensitivity": ([P, P, P, P, P, P, P], I),
    "tb_pcg_solve": ([P, P, P, P, D, I, PI, PD, P], I),
    "tb_plan_set_preconditioner": ([P, I], I),
    "tb_pcg_profile": ([P, P, P, I, PD, PD, P], I),
    "tb_launch_count": ([], I64),
    "tb_plan_set_owned_planes": ([P, I, I], I),
    "tb_pcg_dist_phase": ([P, I, P, P, D, I, I, P], I),
    "tb_pcg_dist_buffers": ([P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P)], I),
    "tb_pcg_dist_state": ([P, PI, PI, PD, PD, P], I),
    "tb_plan_set_halo_peers": ([P, P, P], I),
    "tb_ipc_get_handle": ([P, P], I),
    "tb_ipc_open": ([P, I, ctypes.POINTER(P)], I),
    "tb_ipc_close": ([P], I),
    "tb_dot": ([P, P, P, I64, PD, P], I),
    "tb_filter_create": ([I, I, I, I, D, D, I, ctypes.POINTER(P)], I),
    "tb_filter_destroy": ([P], I),
    "tb_filter_load_vector": ([P, P, P, P], I),
    "tb_filter_apply": ([P, P, P, P, D, PI, P], I),
    "tb_filter_adjoint": ([P, P, P, D, PI, P], I),
    "tb_filter_set_owned_planes": ([P, I, I], I),
    "tb_filter_dist_phase": ([P, I, P, D, I, I, P], I),
    "tb_filter_dist_buffers": ([P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P)], I),
    "tb_filter_dist_state": ([P, PI, PI, PD, PD, P], I),
    "tb_filter_set_halo_peers": ([P, P, P], I),
    "tb_filter_transfer": ([P, I, P, D, P, P], I),
    "tb_mgp_prof_read": ([ctypes.POINTER(ctypes.c_ulonglong)], I),
    "tb_pcg_kernel_time": ([P, ctypes.POINTER(ctypes.c_float), PI], I),
    "tb_pcg_path": ([P], I),
    "tb_pcg_iter_time": ([P, I, PD, ctypes.POINTER(ctypes.c_int64)], I),
    "tb_rom_fused_info": ([P, I, I, PD], I),
    "tb_rom_project": ([I64, P, I, P, I, P, P], I),
    "tb_rom_reduced_stiffness": ([P, P, I, P, I, P, P], I),
    "tb_rom_gram_colmajor": ([I64, I, P, P, I64, I, P, P], I),
    "tb_rom_cholesky_solve": ([I, I, I, P, P, P, PI, P], I),
    "tb_rom_reconstruct": ([I64, P, I, P, I, P, P], I),
    "tb_rom_residual_norms": ([P, P, I, P, P, I, P, I64, PD, P], I),
    "tb_gram_schmidt": ([I64, I, P, D, P, PI, P], I),
    "tb_mma_workspace_bytes": ([I64], ctypes.c_size_t),
    "tb_cone_create": ([I, I, I, I, D, D, I, ctypes.POINTER(P)], I),
    "tb_cone_destroy": ([P], I),
    "tb_cone_apply": ([P, P, P, P], I),
    "tb_cone_adjoint": ([P, P, P, P], I),
    "tb_mma_step": ([I64, P, P, P, P, P, D, D, I, I, I, ctypes.POINTER(MmaConfigC), P, P, P, P, P, P, P], I),
}


def lib():
    """Load the shared library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        handle = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = res
        _lib = handle
    return _lib


def last_error() -> str:
    return lib().tb_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Map a C status code to the reference's exception classes."""
    if rc == TB_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc in (TB_ERR_INVALID, TB_ERR_DENSITY):
        raise ValueError(msg)
    if rc == TB_ERR_INDEFINITE:
        from .fem import IndefiniteMatrixError

        raise IndefiniteMatrixError(msg)
    if rc == TB_ERR_DEGENERATE:
        from .rom import DegenerateBasisError

        raise DegenerateBasisError(msg)
    if rc == TB_ERR_NOT_CONVERGED:
        raise NotConvergedError(msg)
    raise RuntimeError(msg)


# --------------------------------------------------------------------------------------
# torch plumbing (device memory and streams only)
# --------------------------------------------------------------------------------------
def torch():
    import torch as _t

    return _t


def require_cuda(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2004_05756_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    lib()
    if isinstance(device, t.device):
        if device.type != "cuda":
            raise ValueError(f"device must be a CUDA device, got {device}")
        return t.device("cuda", t.cuda.current_device() if device.index is None else device.index)
    if isinstance(device, str):
        return require_cuda(t.device(device))
    return t.device("cuda", t.cuda.current_device() if device is None else int(device))


def mesh_dims(mesh):
    """(dim, nz) of a mesh: this package's StructuredMesh carries both; the reference's 2D
    romtopt.fem.StructuredMesh (fem.py:154-212) has neither (dim 2, nz 0) -- so the drop-in
    classes accept the reference's own meshes."""
    return int(getattr(mesh, "dim", 2)), int(getattr(mesh, "nz", 0) or 0)


def stream_ptr(device) -> P:
    t = torch()
    return P(t.cuda.current_stream(device).cuda_stream)


def ptr(t) -> P:
    return P(t.data_ptr()) if t is not None else P(0)


def is_torch(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor)


def to_dev(x, device, shape=None, dtype=None):
    """Contiguous fp64 (or ``dtype``) device tensor view/copy of a numpy array or tensor."""
    t = torch()
    dtype = dtype or t.float64
    if isinstance(x, t.Tensor):
        out = x.to(device=device, dtype=dtype)
    else:
        arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64 if dtype == t.float64 else None))
        out = t.from_numpy(arr).to(device=device, dtype=dtype, non_blocking=False)
    out = out.contiguous()
    if shape is not None and tuple(out.shape) != tuple(shape):
        out = out.reshape(shape)
    return out


def to_host_async(t_out):
    """Start a D2H copy of a device tensor into fresh pinned host memory (stream-ordered)."""
    t = torch()
    host = t.empty(tuple(t_out.shape), dtype=t_out.dtype, pin_memory=True)
    host.copy_(t_out.detach(), non_blocking=True)
    ev = t.cuda.Event()
    ev.record()
    return host, ev


def finish_host(pending):
    """numpy view of a finished to_host_async copy (the array keeps its pinned buffer alive)."""
    host, ev = pending
    ev.synchronize()
    return host.numpy()


def to_user(t_out, like_torch: bool):
    """Return a device tensor as-is (native mode) or as a numpy array (compat mode, through
    pinned memory: ~3x the pageable D2H rate)."""
    if like_torch:
        return t_out
    return finish_host(to_host_async(t_out))
