"""Diffusion-decay solver and cell exchange on the GPU.

Mirrors /root/reference/pkg/src/cellbench/diffusion.py: ``lod_step``
(:127-192), ``apply_cell_exchange`` (:201-234), ``refresh_nonempty_list``
(:195-198) and ``TraversalMode`` (:31-33) keep their signatures, return types
and errors.  The work runs in libcellgpu.so (csrc/diffusion.cu); the
traversal mode and pool only shape the returned ``RegionRecord``s, exactly as
they only shape scheduling (never results) in the reference.

Keyword-only extensions (default off = the reference's behaviour, bit-for-bit):
  * ``lod_step(..., bc="dirichlet", dirichlet=[...])`` -- G1, every outer-face
    voxel pinned to the substrate's value before the x sweep and after each
    sweep (BioFVM's apply_dirichlet_conditions);
  * ``apply_cell_exchange`` with per-cell arrays -- G4: ``secretion`` /
    ``uptake`` of shape (n,) apply to ``substrate``; shape (S, n) apply to
    every substrate (``saturation`` scalar or (S,)).
"""

from __future__ import annotations

import ctypes
import enum
import time

import numpy as np

from . import _lib
from .core import CartesianMesh, CellContainer, Microenvironment
from .errors import DomainError
from .parallel import RegionRecord, gpu_record


class TraversalMode(enum.Enum):
    OUTER_LOOP = "outer"
    COLLAPSED = "collapsed"


def _bc_code(bc: str) -> int:
    if bc in ("neumann", "no-flux", None):
        return _lib.BC_NEUMANN
    if bc == "dirichlet":
        return _lib.BC_DIRICHLET
    raise DomainError(f"unknown boundary condition {bc!r}")


def lod_step(micro: Microenvironment, mesh: CartesianMesh, dt: float,
             mode: TraversalMode, pool, container: CellContainer | None = None, *,
             bc: str = "neumann", dirichlet=None) -> list[RegionRecord]:
    """One operator-split step: implicit x, y, z sweeps, decay split lambda/3.

    With a container, its non-empty voxel list is refreshed (diffusion.py:
    188-191); on the GPU the list is a by-product of the last rebin.
    Returns one record per sweep per substrate.
    """
    if dt <= 0.0:
        raise DomainError("diffusion step needs dt > 0")
    bcc = _bc_code(bc)
    S = micro.substrate_count
    dirv = None
    if bcc == _lib.BC_DIRICHLET:
        if dirichlet is None:
            raise DomainError("dirichlet boundary needs one value per substrate")
        dirv = np.ascontiguousarray(np.broadcast_to(np.asarray(dirichlet, np.float64), (S,)))
    t0 = time.perf_counter()
    if S:
        dens = micro.device_densities()
        ctx = _lib.context_for(mesh, S, 0)
        D = np.ascontiguousarray(micro.diffusion, dtype=np.float64)
        K = np.ascontiguousarray(micro.decay, dtype=np.float64)
        vp = ctypes.c_void_p
        code = _lib.load().cg_lod_step(
            ctx.handle, _lib.ptr(dens), D.ctypes.data_as(vp), K.ctypes.data_as(vp), float(dt),
            bcc, None if dirv is None else dirv.ctypes.data_as(vp))
        _lib.raise_for(code, "lod_step")
        ctx.sync("lod_step")
        micro.pull()
    elapsed = time.perf_counter() - t0
    if container is not None:
        container._nonempty_override = None
    nx, ny, nz = mesh.nx, mesh.ny, mesh.nz
    if mode is TraversalMode.OUTER_LOOP:
        chunks = (nz, nz, ny)
    else:
        chunks = (nz * ny, nz * nx, ny * nx)
    per = elapsed / max(3 * S, 1)
    return [gpu_record(c, c, per) for _ in range(S) for c in chunks]


def refresh_nonempty_list(container: CellContainer, mesh: CartesianMesh | None = None) -> list[int]:
    """Standalone recompute of the non-empty voxel list from the agent index."""
    container.nonempty_voxels = sorted(v for v, ids in container.agent.items() if ids)
    return container.nonempty_voxels


def apply_cell_exchange(micro: Microenvironment, container: CellContainer, dt: float,
                        secretion, uptake, saturation, substrate: int = 0,
                        pool=None) -> RegionRecord | None:
    """Implicit per-cell secretion/uptake against each cell's voxel density;
    cells of a voxel apply in ascending id order (diffusion.py:201-234)."""
    if dt <= 0.0:
        raise DomainError("exchange needs dt > 0")
    S = micro.substrate_count
    t0 = time.perf_counter()
    d = container.device_cells()
    n = d.n
    b = container._bins
    if b is None or b.n != n:
        # Never rebinned at this size: the reference would see an empty agent.
        nne = 0
    else:
        nne = None
    per_cell = np.ndim(secretion) > 0 or np.ndim(uptake) > 0
    if nne == 0 or n == 0:
        if pool is None:
            return None
        return gpu_record(0, 0, time.perf_counter() - t0)
    dens = micro.device_densities()
    ctx = _lib.context_for(micro.mesh, S, n)
    L = _lib.load()
    P = _lib.ptr
    vp = ctypes.c_void_p
    if not per_cell:
        code = L.cg_exchange(ctx.handle, P(dens), int(substrate), float(dt), float(secretion),
                             float(uptake), float(saturation), n, P(d.volume), P(b.bin_start),
                             P(b.bin_cells_by_id), P(b.nonempty), P(b.n_nonempty))
    else:
        torch = _lib.require_cuda()
        sec = np.asarray(secretion, dtype=np.float64)
        upt = np.asarray(uptake, dtype=np.float64)
        if sec.ndim <= 1 and upt.ndim <= 1:
            full_s = np.zeros((S, n))
            full_u = np.zeros((S, n))
            full_s[substrate] = np.broadcast_to(sec, (n,))
            full_u[substrate] = np.broadcast_to(upt, (n,))
        else:
            full_s = np.ascontiguousarray(np.broadcast_to(sec, (S, n)))
            full_u = np.ascontiguousarray(np.broadcast_to(upt, (S, n)))
        sat = np.ascontiguousarray(np.broadcast_to(np.asarray(saturation, np.float64), (S,)))
        ts = torch.tensor(full_s, dtype=torch.float64, device="cuda")
        tu = torch.tensor(full_u, dtype=torch.float64, device="cuda")
        code = L.cg_exchange_cells(ctx.handle, P(dens), float(dt), P(ts), P(tu),
                                   sat.ctypes.data_as(vp), n, P(d.volume), P(b.bin_start),
                                   P(b.bin_cells_by_id), P(b.nonempty), P(b.n_nonempty))
    _lib.raise_for(code, "apply_cell_exchange")
    ctx.sync("apply_cell_exchange")
    micro.pull()
    if pool is None:
        return None
    nvox = int(b.n_nonempty.cpu().item())
    return gpu_record(nvox, nvox, time.perf_counter() - t0)


def compute_gradients(micro: Microenvironment, mesh: CartesianMesh, mode: TraversalMode,
                      pool) -> list[RegionRecord]:
    """Central-difference gradients, boundary-face components zero
    (diffusion.py:237-278), written into ``micro.gradients`` in place.
    One record per substrate with the reference's chunk count for ``mode``."""
    S = micro.substrate_count
    t0 = time.perf_counter()
    if S:
        torch = _lib.require_cuda()
        dens = micro.device_densities()
        if micro._grad_dev is None:
            micro._grad_dev = torch.empty(micro.gradients.shape, dtype=torch.float64,
                                          device="cuda")
        ctx = _lib.context_for(mesh, S, 0)
        _lib.raise_for(_lib.load().cg_gradients(ctx.handle, _lib.ptr(dens),
                                                _lib.ptr(micro._grad_dev)), "compute_gradients")
        ctx.sync("compute_gradients")
        np.copyto(micro.gradients, micro._grad_dev.cpu().numpy())
    elapsed = time.perf_counter() - t0
    chunks = mesh.nz if mode is TraversalMode.OUTER_LOOP else mesh.nz * mesh.ny
    return [gpu_record(chunks, chunks, elapsed / max(S, 1)) for _ in range(S)]

