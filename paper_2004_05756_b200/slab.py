"""z-slab domain decomposition of the 3D HDM solve across GPUs (BASELINE cfg 4).

Rank r owns the global node planes [k0, k1) and holds the element planes [e0, e1) that touch
them, i.e. its own slab plus one ghost element layer per interior side.  Its local grid is an
ordinary structured Hex8 grid with node planes [e0, e1].  Because nodes are numbered plane by
plane, every local vector is a contiguous slice of the global one, and ghost node planes are
contiguous too.

Ghost node planes are Dirichlet-masked in the local plan, so the unmodified kernels
(operator, update, Jacobi diagonal) run on the slab.  Their rows are never updated, and every
reduction and the operator's p.q are restricted to the owned planes
(tb_plan_set_owned_planes).  One iteration of the distributed Jacobi-pCG:

    phase 2  operator + local p.q   ->  allreduce(red)  ->  phase 3  alpha
    phase 4  update + local r.z, r.r ->  allreduce(red)  ->  phase 5  beta / convergence
    halo     ghost planes of z <- neighbours' first / last owned planes

With ``peer=True`` the halo step disappears: phases 0 and 4 store the boundary planes of z
straight into the neighbours' ghost planes while computing them (tb_plan_set_halo_peers; CUDA
IPC mappings over NVLink between processes).  The allreduce that already follows those phases
orders the stores against the neighbours' reads, so no flag, copy or extra collective is
added.

The direction p = z + beta p_old is formed inside the operator for owned and ghost nodes
alike from identical z and p_old, so ghost p needs no exchange.  All ranks receive bitwise
identical allreduce results, so every rank takes the same convergence decision.

The phase driver takes a list of local solvers and a communicator: one solver per process
with ``TorchComm`` (NCCL on GPUs; gloo for the CPU tests), or several solvers in one process
on one GPU with ``LocalComm``.  ``LocalComm`` emulates the exchange step by step on the host;
no kernel ever waits on another rank.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .fem import StructuredMesh, build_mesh_3d

__all__ = ["Slab", "partition", "SlabSolver", "SlabFilter", "LocalComm", "TorchComm", "dist_pcg_solve",
           "slab_evaluate", "SlabEvaluation"]


@dataclass(frozen=True)
class Slab:
    rank: int
    nranks: int
    k0: int  # owned global node planes [k0, k1)
    k1: int
    e0: int  # local element planes [e0, e1) (global ids); local node planes [e0, e1]
    e1: int

    @property
    def local_nz(self) -> int:
        return self.e1 - self.e0

    @property
    def ghost_lo(self) -> bool:
        return self.k0 > self.e0

    @property
    def ghost_hi(self) -> bool:
        return self.e1 >= self.k1

    @property
    def own_local(self):
        return self.k0 - self.e0, self.k1 - self.e0


def partition(nz: int, nranks: int) -> list:
    """Split the nz+1 node planes into nranks contiguous owned ranges (sizes differ by <= 1)."""
    nnz = nz + 1
    if nranks < 1 or nranks > nnz // 2:
        raise ValueError(f"cannot split {nnz} node planes over {nranks} ranks (need >= 2 planes each)")
    base, extra = divmod(nnz, nranks)
    out, k = [], 0
    for r in range(nranks):
        k1 = k + base + (1 if r < extra else 0)
        out.append(Slab(r, nranks, k, k1, max(0, k - 1), min(nz, k1)))
        k = k1
    return out


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory (torch.as_tensor aliases it)."""

    def __init__(self, ptr, n, device):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}
        self.device = device


class SlabSolver:
    """Rank-local part of the distributed HDM solve (one z-slab of a 3D Hex8 problem)."""

    def __init__(self, mesh: StructuredMesh, k_e, f, fixed_dofs, material, slab: Slab, device=None):
        t = _lib.torch()
        if not mesh.nz:
            raise ValueError("slab decomposition is for 3D meshes")
        self.mesh, self.slab = mesh, slab
        self.device = _lib.require_cuda(device)
        self.local = build_mesh_3d(mesh.nx, mesh.ny, slab.local_nz, mesh.h)
        self.plane_nodes = (mesh.nx + 1) * (mesh.ny + 1)
        self.plane_dofs = 3 * self.plane_nodes
        self.plane_elems = mesh.nx * mesh.ny
        d0 = slab.e0 * self.plane_dofs
        nl = self.local.n_dofs
        fixed = np.zeros(mesh.n_dofs, dtype=np.uint8)
        fixed[np.asarray(fixed_dofs, dtype=np.int64)] = 1
        fixed_l = fixed[d0:d0 + nl].copy()
        if slab.ghost_lo:
            fixed_l[:self.plane_dofs] = 1
        if slab.ghost_hi:
            fixed_l[-self.plane_dofs:] = 1
        f_l = np.asarray(f, dtype=float)[d0:d0 + nl].copy()
        f_l[fixed_l != 0] = 0.0
        self.fixed_local = fixed_l
        ke = np.ascontiguousarray(np.asarray(k_e, dtype=float))
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().tb_plan_create(3, mesh.nx, mesh.ny, slab.local_nz, mesh.h,
                                             ke.ctypes.data_as(ctypes.c_void_p), material.rho_l, material.p,
                                             np.ascontiguousarray(fixed_l).ctypes.data_as(ctypes.c_void_p),
                                             self.device.index, ctypes.byref(h)), "slab plan")
        self._plan = h
        k0, k1 = slab.own_local
        _lib.check(_lib.lib().tb_plan_set_owned_planes(h, k0, k1), "owned planes")
        self.f = _lib.to_dev(f_l, self.device)
        px, pz, pr = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.lib().tb_pcg_dist_buffers(h, ctypes.byref(px), ctypes.byref(pz), ctypes.byref(pr)), "bufs")
        self.x = t.as_tensor(_CudaArray(px.value, nl, self.device), device=self.device)
        self.z = t.as_tensor(_CudaArray(pz.value, nl, self.device), device=self.device)
        self.red = t.as_tensor(_CudaArray(pr.value, 4, self.device), device=self.device)
        self.rho = None
        self.rtol, self.maxit = 1e-8, 200000
        # Chronopoulos-Gear phases 10-13: ONE allreduce per iteration (Hex8 plans)
        self.single_reduction = True

    def __del__(self):
        h = getattr(self, "_plan", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.tb_plan_destroy(h)
            self._plan = None

    # -- element / node slices of global fields
    def local_elems(self, global_elem_field):
        s = self.slab
        return global_elem_field[s.e0 * self.plane_elems:s.e1 * self.plane_elems]

    def owned_dofs(self):
        """(local slice, global slice) of this rank's owned dofs."""
        k0, k1 = self.slab.own_local
        return (slice(k0 * self.plane_dofs, k1 * self.plane_dofs),
                slice(self.slab.k0 * self.plane_dofs, self.slab.k1 * self.plane_dofs))

    def plane(self, vec, local_plane):
        return vec[local_plane * self.plane_dofs:(local_plane + 1) * self.plane_dofs]

    # -- phases (see module docstring)
    def phase(self, p, parity=0):
        rho = _lib.ptr(self.rho) if p in (0, 10) else _lib.P(0)
        b = _lib.ptr(self.f) if p in (0, 10) else _lib.P(0)
        _lib.check(_lib.lib().tb_pcg_dist_phase(self._plan, p, rho, b, self.rtol, self.maxit, parity,
                                                _lib.stream_ptr(self.device)), f"dist phase {p}")

    def set_halo_peers(self, lo_dst: int, hi_dst: int):
        """Device addresses that receive this rank's first / last owned plane of z (0: none)."""
        _lib.check(_lib.lib().tb_plan_set_halo_peers(self._plan, _lib.P(lo_dst or None), _lib.P(hi_dst or None)),
                   "halo peers")

    def ghost_addresses(self, z_base: int):
        """(ghost-below, ghost-above) plane addresses for a z allocation at ``z_base``."""
        k0, k1 = self.slab.own_local
        lo = z_base if self.slab.ghost_lo else 0
        hi = z_base + 8 * k1 * self.plane_dofs if self.slab.ghost_hi else 0
        return lo, hi

    def z_ipc_handle(self) -> bytes:
        h = ctypes.create_string_buffer(64)
        _lib.check(_lib.lib().tb_ipc_get_handle(_lib.P(self.z.data_ptr()), h), "ipc handle")
        return h.raw

    # -- element-level steps of the evaluation (slab_evaluate)
    def clamp(self, rho_raw):
        """(rho, local clamp width) of tb_clamp_density (hdm.py:144-154) on the local elements."""
        t = _lib.torch()
        rho = t.empty_like(rho_raw)
        cw = ctypes.c_double(0.0)
        _lib.check(_lib.lib().tb_clamp_density(self._plan, _lib.ptr(rho_raw), _lib.ptr(rho), ctypes.byref(cw),
                                               _lib.stream_ptr(self.device)), "slab clamp")
        return rho, float(cw.value)

    def sensitivity(self, rho, u):
        """Compliance sensitivities of every local element (hdm.py:211-222); u must hold the
        ghost planes (halo of x)."""
        t = _lib.torch()
        out = t.empty(self.local.n_elems, dtype=t.float64, device=self.device)
        _lib.check(_lib.lib().tb_element_sensitivity(self._plan, _lib.ptr(rho), _lib.ptr(u), _lib.ptr(u), _lib.P(0),
                                                     _lib.ptr(out), _lib.stream_ptr(self.device)), "slab sensitivity")
        return out

    def owned_compliance(self, u):
        """f . u over the owned dofs (f is zero on the ghost planes)."""
        out = ctypes.c_double(0.0)
        _lib.check(_lib.lib().tb_dot(self._plan, _lib.ptr(self.f), _lib.ptr(u), self.local.n_dofs, ctypes.byref(out),
                                     _lib.stream_ptr(self.device)), "slab compliance")
        return float(out.value)

    def owned_elems(self):
        """(local slice, global slice) of the element planes this rank owns: [k0, min(k1, nz))."""
        s = self.slab
        top = min(s.k1, self.mesh.nz)
        pe = self.plane_elems
        return slice((s.k0 - s.e0) * pe, (top - s.e0) * pe), slice(s.k0 * pe, top * pe)

    def state(self):
        it, done, rr, bb = ctypes.c_int(), ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.lib().tb_pcg_dist_state(self._plan, ctypes.byref(it), ctypes.byref(done), ctypes.byref(rr),
                                                ctypes.byref(bb), _lib.stream_ptr(self.device)), "dist state")
        return it.value, done.value, rr.value, bb.value


class SlabFilter:
    """Rank-local part of the distributed Helmholtz filter (HelmholtzFilter, filtering.py:47-114)
    on one z-slab: the same local grid and owned planes as the rank's SlabSolver, a scalar
    field (one value per node), solved with the phases of dist_pcg_solve."""

    def __init__(self, mesh: StructuredMesh, radius: float, slab: Slab, device=None, rtol: float = 1e-13):
        t = _lib.torch()
        if not mesh.nz:
            raise ValueError("slab decomposition is for 3D meshes")
        self.mesh, self.slab = mesh, slab
        self.device = _lib.require_cuda(device)
        self.local = build_mesh_3d(mesh.nx, mesh.ny, slab.local_nz, mesh.h)
        self.plane_nodes = (mesh.nx + 1) * (mesh.ny + 1)
        self.plane_dofs = self.plane_nodes  # one unknown per node
        self.plane_elems = mesh.nx * mesh.ny
        self.vol_share = mesh.h**3 / 8.0  # b_e entries (filtering.py:75-76), 3D
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().tb_filter_create(3, mesh.nx, mesh.ny, slab.local_nz, mesh.h, float(radius),
                                               self.device.index, ctypes.byref(h)), "slab filter")
        self._h = h
        k0, k1 = slab.own_local
        _lib.check(_lib.lib().tb_filter_set_owned_planes(h, k0, k1), "filter owned planes")
        nl = self.local.n_nodes
        px, pz, pr = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.lib().tb_filter_dist_buffers(h, ctypes.byref(px), ctypes.byref(pz), ctypes.byref(pr)), "bufs")
        self.x = t.as_tensor(_CudaArray(px.value, nl, self.device), device=self.device)
        self.z = t.as_tensor(_CudaArray(pz.value, nl, self.device), device=self.device)
        self.red = t.as_tensor(_CudaArray(pr.value, 4, self.device), device=self.device)
        self.b = t.zeros(nl, dtype=t.float64, device=self.device)
        self.rtol, self.maxit = float(rtol), 200000

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.tb_filter_destroy(h)
            self._h = None

    def plane(self, vec, local_plane):
        return vec[local_plane * self.plane_dofs:(local_plane + 1) * self.plane_dofs]

    def set_load(self, elem_values, scale):
        """b_n = scale * sum_{e∋n} v_e over the local elements (filtering.py:73-76, 106-108)."""
        _lib.check(_lib.lib().tb_filter_transfer(self._h, 0, _lib.ptr(elem_values), float(scale), _lib.ptr(self.b),
                                                 _lib.stream_ptr(self.device)), "filter load")

    def to_elems(self, scale):
        """out_e = scale * sum_{n∈e} x_n for every local element (filtering.py:95-97, 112-114);
        x must hold the ghost planes (halo of x)."""
        t = _lib.torch()
        out = t.empty(self.local.n_elems, dtype=t.float64, device=self.device)
        _lib.check(_lib.lib().tb_filter_transfer(self._h, 1, _lib.ptr(self.x), float(scale), _lib.ptr(out),
                                                 _lib.stream_ptr(self.device)), "filter average")
        return out

    def phase(self, p, parity=0):
        b = _lib.ptr(self.b) if p == 0 else _lib.P(0)
        _lib.check(_lib.lib().tb_filter_dist_phase(self._h, p, b, self.rtol, self.maxit, parity,
                                                   _lib.stream_ptr(self.device)), f"filter dist phase {p}")

    def set_halo_peers(self, lo_dst: int, hi_dst: int):
        _lib.check(_lib.lib().tb_filter_set_halo_peers(self._h, _lib.P(lo_dst or None), _lib.P(hi_dst or None)),
                   "filter halo peers")

    def ghost_addresses(self, z_base: int):
        k0, k1 = self.slab.own_local
        lo = z_base if self.slab.ghost_lo else 0
        hi = z_base + 8 * k1 * self.plane_dofs if self.slab.ghost_hi else 0
        return lo, hi

    def z_ipc_handle(self) -> bytes:
        h = ctypes.create_string_buffer(64)
        _lib.check(_lib.lib().tb_ipc_get_handle(_lib.P(self.z.data_ptr()), h), "ipc handle")
        return h.raw

    def state(self):
        it, done, rr, bb = ctypes.c_int(), ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.lib().tb_filter_dist_state(self._h, ctypes.byref(it), ctypes.byref(done), ctypes.byref(rr),
                                                   ctypes.byref(bb), _lib.stream_ptr(self.device)), "filter state")
        return it.value, done.value, rr.value, bb.value


class LocalComm:
    """All ranks in one process: allreduce = fixed-order sum, halo = device copies (or, with
    ``peer=True``, the update kernels' direct stores into the neighbours' ghost planes)."""

    def __init__(self, peer: bool = False):
        self.peer = peer
        self.allreduces = 0  # allreduce steps executed (graph replays counted per captured call)
        self.capturable = True  # every step is a device op on the current stream

    def setup(self, solvers):
        if not self.peer:
            return
        for i, s in enumerate(solvers):
            lo = solvers[i - 1].ghost_addresses(solvers[i - 1].z.data_ptr())[1] if i > 0 else 0
            hi = solvers[i + 1].ghost_addresses(solvers[i + 1].z.data_ptr())[0] if i + 1 < len(solvers) else 0
            s.set_halo_peers(lo, hi)

    def allreduce(self, solvers):
        self.allreduces += 1
        total = solvers[0].red.clone()
        for s in solvers[1:]:
            total = total + s.red
        for s in solvers:
            s.red.copy_(total)

    def reduce_scalars(self, values, op="sum"):
        """values: one list of floats per local solver -> the element-wise sum / max over them."""
        out = list(values[0])
        for v in values[1:]:
            out = [a + b if op == "sum" else max(a, b) for a, b in zip(out, v)]
        return out

    def halo(self, solvers, name="z"):
        if self.peer and name == "z":
            return
        for lo, hi in zip(solvers[:-1], solvers[1:]):
            vlo, vhi = getattr(lo, name), getattr(hi, name)
            k0_hi, _ = hi.slab.own_local
            _, k1_lo = lo.slab.own_local
            # hi's ghost-below plane <- lo's last owned plane; lo's ghost-above <- hi's first owned
            hi.plane(vhi, 0).copy_(lo.plane(vlo, k1_lo - 1))
            lo.plane(vlo, k1_lo).copy_(hi.plane(vhi, k0_hi))


class TorchComm:
    """One solver per process; collectives through torch.distributed (NCCL or gloo).

    ``peer=True`` (CUDA solvers): the z allocations are exchanged once as CUDA IPC handles and
    mapped into the neighbours' address spaces; the halo then travels as NVLink peer stores from
    inside the update kernel and ``halo`` is a no-op.  Call ``close()`` before the solvers go."""

    def __init__(self, group=None, peer: bool = False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.peer = peer
        self._mapped = []
        self._ready = set()   # solvers whose z halo travels as peer stores
        self._failed = set()  # solvers that fell back to NCCL send/recv
        self.allreduces = 0   # allreduce steps executed (graph replays counted per captured call)

    # The single-reduction iteration has no collective between the update that pushes u into the
    # neighbours' ghost planes and the operator that reads them (neighbor_sync orders them with a
    # one-double P2P token per neighbour), so it runs as an eager host loop here.
    capturable = False

    def setup(self, solvers):
        if not self.peer or id(solvers[0]) in self._ready or id(solvers[0]) in self._failed:
            return
        s = solvers[0]
        r, n = s.slab.rank, s.slab.nranks
        handles = [None] * n
        self.dist.all_gather_object(handles, s.z_ipc_handle(), group=self.group)
        addr, ok, mine = {}, True, []
        try:
            for nb in (r - 1, r + 1):
                if 0 <= nb < n:
                    base = _lib.P()
                    _lib.check(_lib.lib().tb_ipc_open(handles[nb], s.device.index, ctypes.byref(base)), "ipc open")
                    mine.append(base.value)
                    addr[nb] = base.value
        except Exception:  # e.g. no peer access between the two devices
            ok = False
        # every rank takes the same decision: peer stores only if all ranks mapped their neighbours;
        # otherwise this solver's z halo goes through NCCL send/recv
        flags = [None] * n
        self.dist.all_gather_object(flags, ok, group=self.group)
        if not all(flags):
            for base in mine:
                _lib.lib().tb_ipc_close(_lib.P(base))
            self._failed.add(id(s))
            return
        self._mapped += mine
        # the neighbours' ghost planes: below-neighbour's ghost-above, above-neighbour's ghost-below
        lo = addr[r - 1] + 8 * self._ghost_hi_plane(s, r - 1) * s.plane_dofs if r > 0 else 0
        hi = addr[r + 1] if r + 1 < n else 0
        s.set_halo_peers(lo, hi)
        self._ready.add(id(s))
        self.dist.barrier(group=self.group)

    @staticmethod
    def _ghost_hi_plane(s, rank):
        """Local index of rank ``rank``'s ghost-above plane (its owned range ends there)."""
        other = partition(s.mesh.nz, s.slab.nranks)[rank]
        return other.own_local[1]

    @property
    def peer_active(self) -> bool:
        return bool(self._ready)

    def close(self):
        for base in self._mapped:
            _lib.lib().tb_ipc_close(_lib.P(base))
        self._mapped, self._ready, self._failed = [], set(), set()

    def allreduce(self, solvers):
        self.allreduces += 1
        red = solvers[0].red
        if red.is_cuda and self.dist.get_backend(self.group) == "gloo":
            host = red.cpu()  # waits for the phase on the current stream
            self.dist.all_reduce(host, group=self.group)
            red.copy_(host)
        else:
            self.dist.all_reduce(red, group=self.group)

    def neighbor_sync(self, solvers):
        """Order this rank's peer stores (issued by the kernels before this call on its stream)
        before the neighbours' next kernels: a one-double send/recv with each neighbour.  NCCL:
        stream-ordered on both sides.  gloo: the host waits for the stream first.  A no-op unless
        the z halo travels as peer stores (otherwise halo() moves the planes, which orders them)."""
        s = solvers[0]
        if id(s) not in self._ready:
            return
        d = self.dist
        t = _lib.torch()
        r, n = s.slab.rank, s.slab.nranks
        gloo = d.get_backend(self.group) == "gloo"
        if gloo and s.red.is_cuda:
            t.cuda.current_stream(s.device).synchronize()
        dev = "cpu" if gloo else s.device
        send = t.zeros(1, dtype=t.float64, device=dev)
        recv = [t.empty(1, dtype=t.float64, device=dev) for _ in range(2)]
        ops = []
        for k, nb in enumerate((r - 1, r + 1)):
            if 0 <= nb < n:
                ops.append(d.P2POp(d.isend, send, nb, self.group))
                ops.append(d.P2POp(d.irecv, recv[k], nb, self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()

    def reduce_scalars(self, values, op="sum"):
        """values: [floats of this rank's solver] -> the element-wise sum / max over the ranks."""
        t = _lib.torch()
        dev = "cpu" if self.dist.get_backend(self.group) == "gloo" else t.device("cuda", t.cuda.current_device())
        v = t.tensor(list(values[0]), dtype=t.float64, device=dev)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX,
                             group=self.group)
        return [float(a) for a in v.cpu()]

    def halo(self, solvers, name="z"):
        if name == "z" and id(solvers[0]) in self._ready:
            return
        d = self.dist
        s = solvers[0]
        v = getattr(s, name)
        r, n = s.slab.rank, s.slab.nranks
        k0, k1 = s.slab.own_local
        ops = []
        if r > 0:
            ops.append(d.P2POp(d.isend, s.plane(v, k0).contiguous(), r - 1, self.group))
            ops.append(d.P2POp(d.irecv, s.plane(v, 0), r - 1, self.group))
        if r < n - 1:
            ops.append(d.P2POp(d.isend, s.plane(v, k1 - 1).contiguous(), r + 1, self.group))
            ops.append(d.P2POp(d.irecv, s.plane(v, k1), r + 1, self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()


def dist_pcg_solve(solvers, comm, rtol=1e-8, maxit=200000, check_every=32, graph=None):
    """Jacobi-pCG over the slabs of ``solvers`` (this process's share).  Returns
    (iterations, recursive relative residual, converged flag).  The host reads the device state
    every ``check_every`` iterations (a pipeline drain each time); phases issued after
    convergence are no-ops on the device (their kernels return on st->done).

    Solvers with ``single_reduction`` (SlabSolver) run the Chronopoulos-Gear phases 10-13: ONE
    allreduce of (w.u, r.u, r.r) per iteration.  When every step is a device operation on the
    current stream (``comm.capturable``: LocalComm, or NCCL with the halo as peer stores) and
    ``graph`` is not False, ``check_every`` iterations are captured once in a CUDA graph --
    kernels, collectives and halo -- and the host loop only replays it and reads the state."""
    setup = getattr(comm, "setup", None)
    if setup is not None:
        setup(solvers)
    for s in solvers:
        s.rtol, s.maxit = rtol, maxit
    if getattr(solvers[0], "single_reduction", False):
        return _dist_cg1(solvers, comm, maxit, check_every, graph)
    for s in solvers:
        s.phase(0)
    comm.allreduce(solvers)
    for s in solvers:
        s.phase(1)
    comm.halo(solvers)
    it = 0
    while True:
        for s in solvers:
            s.phase(2, parity=it)
        comm.allreduce(solvers)
        for s in solvers:
            s.phase(3)
            s.phase(4, parity=it)
        comm.allreduce(solvers)
        for s in solvers:
            s.phase(5)
        comm.halo(solvers)
        it += 1
        if it % check_every == 0 or it >= maxit:
            r = _dist_state(solvers)
            if r is not None:
                return r


def _dist_state(solvers):
    iters, done, rr, bb = solvers[0].state()
    if done == 0:
        return None
    if done == 3:
        from .fem import IndefiniteMatrixError

        raise IndefiniteMatrixError("distributed pCG breakdown")
    return iters, (rr / bb) ** 0.5 if bb > 0 else 0.0, done == 1


def _dist_cg1(solvers, comm, maxit, check_every, graph):
    """Single-reduction iteration: 13 update -> z halo -> 11 operator -> allreduce -> 12."""

    sync = getattr(comm, "neighbor_sync", None)

    def step():
        for s in solvers:
            s.phase(13)
        comm.halo(solvers)
        if sync is not None:
            sync(solvers)  # peer stores of u before the neighbours' operator (no collective)
        for s in solvers:
            s.phase(11)
        comm.allreduce(solvers)
        for s in solvers:
            s.phase(12)

    for s in solvers:
        s.phase(10)
    comm.halo(solvers)
    if sync is not None:
        sync(solvers)
    for s in solvers:
        s.phase(11)
    comm.allreduce(solvers)
    for s in solvers:
        s.phase(12)
    use_graph = graph is not False and getattr(comm, "capturable", False) and solvers[0].red.is_cuda
    if use_graph:
        t = _lib.torch()
        g = t.cuda.CUDAGraph()
        side = t.cuda.Stream(device=solvers[0].device)
        side.wait_stream(t.cuda.current_stream(solvers[0].device))
        before = comm.allreduces
        with t.cuda.stream(side):
            with t.cuda.graph(g, stream=side):
                for _ in range(check_every):
                    step()
        captured = comm.allreduces - before
        comm.allreduces = before  # capture issued nothing; replays are counted below
    it = 0
    while True:
        if use_graph:
            g.replay()
            comm.allreduces += captured
            it += check_every
        else:
            for _ in range(check_every):
                step()
            it += check_every
        r = _dist_state(solvers)
        if r is not None:
            return r
        if it >= maxit:
            return solvers[0].state()[0], 0.0, False


@dataclass
class SlabEvaluation:
    """Result of slab_evaluate for this process's slabs: global scalars plus, per slab, the
    local (owned + ghost layer) element fields and node vectors."""

    j: float
    clamp_width: float
    iterations: int
    filter_iterations: tuple
    rho: list
    u: list
    s: list
    g: list


def slab_evaluate(solvers, filters, comm, psi_locals, rtol=None, filter_rtol=None) -> SlabEvaluation:
    """One compliance design evaluation, HdmSolver.solve + gradient (hdm.py:170-209), over
    z-slabs (BASELINE cfg 4: "full HDM solve, sensitivities and filter"):

        psi -> b = (h^3/8) sum_e psi_e -> H phi = b (distributed pCG) -> x halo -> rho_raw = mean phi
            -> clamp (max width over ranks) -> K(rho) u = f (distributed pCG) -> u halo
            -> J = sum_ranks f.u (owned rows) ; s_e on every local element (ghost layer too)
            -> b = (1/8) sum_e s_e -> H mu = b -> x halo -> g_e = (h^3/8) sum mu

    ``psi_locals`` are the local element slices (owned planes plus the ghost layer, as
    SlabSolver.local_elems).  Collectives: the two 4-double allreduces per pCG iteration, one
    plane halo of x after each of the three solves, two scalar allreduces (clamp width, J)."""
    for f, psi in zip(filters, psi_locals):
        f.set_load(psi, f.vol_share)
    fit1, _, ok1 = dist_pcg_solve(filters, comm, rtol=filter_rtol or filters[0].rtol)
    if not ok1:
        raise _lib.NotConvergedError(f"distributed Helmholtz filter did not converge in {fit1} iterations")
    comm.halo(filters, "x")
    rhos, widths = [], []
    for s, f in zip(solvers, filters):
        r, w = s.clamp(f.to_elems(0.125))
        rhos.append(r)
        widths.append([w])
    cw = comm.reduce_scalars(widths, "max")[0]
    for s, r in zip(solvers, rhos):
        s.rho = r
    it, _, ok = dist_pcg_solve(solvers, comm, rtol=rtol or solvers[0].rtol)
    if not ok:
        raise _lib.NotConvergedError(f"distributed pCG did not converge in {it} iterations")
    comm.halo(solvers, "x")
    us = [s.x.clone() for s in solvers]
    j = comm.reduce_scalars([[s.owned_compliance(u)] for s, u in zip(solvers, us)], "sum")[0]
    sens = [s.sensitivity(r, u) for s, r, u in zip(solvers, rhos, us)]
    for f, v in zip(filters, sens):
        f.set_load(v, 0.125)
    fit2, _, ok2 = dist_pcg_solve(filters, comm, rtol=filter_rtol or filters[0].rtol)
    if not ok2:
        raise _lib.NotConvergedError(f"distributed filter adjoint did not converge in {fit2} iterations")
    comm.halo(filters, "x")
    grads = [f.to_elems(f.vol_share) for f in filters]
    return SlabEvaluation(j, cw, it, (fit1, fit2), rhos, us, sens, grads)


class SlabRom:
    """Element-sharded ROM evaluation (BASELINE cfg 5): each rank holds the slab rows of Phi
    (owned + ghost planes), contracts only its owned rows, and the k x k operators, Phi^T f and
    squared residual norms are allreduced.  The k x k Cholesky runs redundantly on
    every rank."""

    def __init__(self, solver: SlabSolver, phi_local, comm):
        t = _lib.torch()
        self.s, self.comm = solver, comm
        self.phi = phi_local.to(device=solver.device, dtype=t.float64).contiguous()
        self.k = self.phi.shape[1]
        sl, _ = solver.owned_dofs()
        own_f = t.zeros_like(solver.f)
        own_f[sl] = solver.f[sl]
        self._fhat_part = self._project(own_f)

    def _project(self, v):
        from .rom import _project

        return _project(self.phi, v[None, :])[0]

    @staticmethod
    def allreduce_tensors(slab_roms, comm, name):
        """Sum ``getattr(rom, name)`` over ranks in place (LocalComm: fixed rank order)."""
        if isinstance(comm, LocalComm):
            total = getattr(slab_roms[0], name).clone()
            for r in slab_roms[1:]:
                total = total + getattr(r, name)
            for r in slab_roms:
                getattr(r, name).copy_(total)
        else:
            v = getattr(slab_roms[0], name)
            comm.allreduces += 1
            if v.is_cuda and comm.dist.get_backend(comm.group) == "gloo":
                host = v.cpu()  # gloo reduces host tensors; waits for the producing kernels
                comm.dist.all_reduce(host, group=comm.group)
                v.copy_(host)
            else:
                comm.dist.all_reduce(v, group=comm.group)

    def local_khat(self, rho_batch_local):
        t = _lib.torch()
        rho2 = rho_batch_local.reshape(-1, self.s.local.n_elems).contiguous()
        nd = rho2.shape[0]
        khat = t.empty((nd, self.k, self.k), dtype=t.float64, device=self.s.device)
        _lib.check(_lib.lib().tb_rom_reduced_stiffness(self.s._plan, _lib.ptr(self.phi), self.k, _lib.ptr(rho2), nd,
                                                       _lib.ptr(khat), _lib.stream_ptr(self.s.device)), "slab khat")
        return khat


def slab_rom_solve_batch(roms, comm, rho_batches_local):
    """Reduced stiffness, reduced solve and full-space residual norms for nd designs across the
    slabs of ``roms`` (this process's share).  Returns (khat, uhat, residual norms)."""
    t = _lib.torch()
    for r, rho in zip(roms, rho_batches_local):
        r.khat = r.local_khat(rho)
        r.fhat = r._fhat_part.clone()
    SlabRom.allreduce_tensors(roms, comm, "khat")
    SlabRom.allreduce_tensors(roms, comm, "fhat")
    for r, rho in zip(roms, rho_batches_local):
        nd, k = r.khat.shape[0], r.k
        rhs = r.fhat[None, None, :].expand(nd, 1, k).contiguous()
        x = t.empty((nd, 1, k), dtype=t.float64, device=r.s.device)
        status = (ctypes.c_int * nd)()
        _lib.check(_lib.lib().tb_rom_cholesky_solve(k, nd, 1, _lib.ptr(r.khat), _lib.ptr(rhs), _lib.ptr(x), status,
                                                    _lib.stream_ptr(r.s.device)), "slab cholesky")
        r.uhat = x[:, 0, :].contiguous()
        rho2 = rho.reshape(nd, -1).contiguous()
        norms = []
        for s0 in range(0, nd, 16):
            e = min(nd, s0 + 16)
            out = (ctypes.c_double * (e - s0))()
            _lib.check(_lib.lib().tb_rom_residual_norms(r.s._plan, _lib.ptr(r.phi), k, _lib.ptr(rho2[s0:e]),
                                                        _lib.ptr(r.uhat[s0:e]), e - s0, _lib.ptr(r.s.f), 0, out,
                                                        _lib.stream_ptr(r.s.device)), "slab residual")
            norms += [v * v for v in out]  # squared partials over this rank's owned free rows
        r.res2 = t.tensor(norms, dtype=t.float64, device=r.s.device)
    SlabRom.allreduce_tensors(roms, comm, "res2")
    return roms[0].khat, roms[0].uhat, [float(v) ** 0.5 for v in roms[0].res2.cpu()]
