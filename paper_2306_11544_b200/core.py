"""Simulation domain with device-resident state behind the reference API.

Mirrors /root/reference/pkg/src/cellbench/core.py: ``CartesianMesh`` (:35-102),
``Microenvironment`` (:109-145), ``Cell`` (:148-163), ``CellContainer``
(:166-215) and ``rebin_cells`` (:218-240) keep their names, constructor
arguments, attributes and error behaviour.  What changes is where the state
lives during a call: every hot-path call runs in libcellgpu.so on torch
device buffers.

Synchronisation follows the reference's object semantics exactly: the host
objects (``micro.densities``, the ``Cell`` objects) stay authoritative; each
API call uploads what it reads, runs on the GPU and writes its results back
IN PLACE (same numpy array, same Cell objects), so references a caller holds
see the update as with the reference.  Derived indexes (``agent``,
``nonempty_voxels``, ``storage_index``) are materialised lazily from the
device bins.  Containers built with ``CellContainer.from_arrays`` have no Cell
objects and stay device-resident until ``cells`` is read; the step engine
(engine.py) never touches the host.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DomainError, NumericError

Vec3 = list

#: Positions are clamped this far (um) inside the mesh when pushed past a face.
POSITION_EPS = 1e-6


def vec3(x: float = 0.0, y: float = 0.0, z: float = 0.0) -> Vec3:
    return [float(x), float(y), float(z)]


def vec3_finite(v) -> bool:
    return math.isfinite(v[0]) and math.isfinite(v[1]) and math.isfinite(v[2])


@dataclass(frozen=True)
class CartesianMesh:
    """Uniform axis-aligned voxel grid, half-open voxels, x-fastest flattening
    (core.py:35-102).  Scalar host helpers; the batched versions run in
    ``rebin_cells`` on the GPU with the same CPython float semantics."""

    nx: int
    ny: int
    nz: int
    dx: float = 20.0
    dy: float = 20.0
    dz: float = 20.0
    origin: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise DomainError("voxel counts must be >= 1")
        if min(self.dx, self.dy, self.dz) <= 0:
            raise DomainError("voxel edge lengths must be > 0")

    @property
    def voxel_count(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def voxel_volume(self) -> float:
        return self.dx * self.dy * self.dz

    @property
    def upper(self) -> tuple:
        ox, oy, oz = self.origin
        return (ox + self.nx * self.dx, oy + self.ny * self.dy, oz + self.nz * self.dz)

    def flatten(self, ix: int, iy: int, iz: int) -> int:
        return ix + self.nx * (iy + self.ny * iz)

    def unflatten(self, v: int) -> tuple:
        ix = v % self.nx
        rest = v // self.nx
        return (ix, rest % self.ny, rest // self.ny)

    def voxel_of(self, position) -> int:
        ox, oy, oz = self.origin
        try:
            ix = int((position[0] - ox) // self.dx)
            iy = int((position[1] - oy) // self.dy)
            iz = int((position[2] - oz) // self.dz)
        except (ValueError, OverflowError):
            raise DomainError(f"position {tuple(position)} outside mesh bounds") from None
        if not (0 <= ix < self.nx and 0 <= iy < self.ny and 0 <= iz < self.nz):
            raise DomainError(f"position {tuple(position)} outside mesh bounds")
        return self.flatten(ix, iy, iz)

    def contains(self, position) -> bool:
        ox, oy, oz = self.origin
        ux, uy, uz = self.upper
        return ox <= position[0] < ux and oy <= position[1] < uy and oz <= position[2] < uz

    def clamp_inside(self, position) -> None:
        ox, oy, oz = self.origin
        ux, uy, uz = self.upper
        position[0] = min(max(position[0], ox + POSITION_EPS), ux - POSITION_EPS)
        position[1] = min(max(position[1], oy + POSITION_EPS), uy - POSITION_EPS)
        position[2] = min(max(position[2], oz + POSITION_EPS), uz - POSITION_EPS)


def voxel_of(position, mesh: CartesianMesh) -> int:
    return mesh.voxel_of(position)


class Microenvironment:
    """Substrate fields (S, nvox) float64 (core.py:109-145).  ``densities`` is
    the authoritative host array; device calls upload it and write back into
    the same array."""

    def __init__(self, mesh: CartesianMesh, diffusion, decay, initial=None):
        self.mesh = mesh
        self.diffusion = np.asarray(diffusion, dtype=np.float64).reshape(-1)
        self.decay = np.asarray(decay, dtype=np.float64).reshape(-1)
        if self.diffusion.shape != self.decay.shape:
            raise DomainError("diffusion and decay must list one value per substrate")
        if np.any(self.diffusion < 0) or np.any(self.decay < 0):
            raise DomainError("diffusion and decay rates must be >= 0")
        s = self.diffusion.shape[0]
        n = mesh.voxel_count
        self._host = np.zeros((s, n), dtype=np.float64)
        if initial is not None:
            init = np.asarray(initial, dtype=np.float64).reshape(-1)
            if init.shape[0] != s:
                raise DomainError("one initial density per substrate required")
            self._host += init[:, None]
        self._dev = None
        # (S, nvox, 3), written in place by compute_gradients (diffusion.py:237-278)
        self.gradients = np.zeros((s, n, 3), dtype=np.float64)
        self._grad_dev = None

    @property
    def substrate_count(self) -> int:
        return self._host.shape[0]

    @property
    def densities(self) -> np.ndarray:
        return self._host

    @densities.setter
    def densities(self, value) -> None:
        self._host[...] = np.asarray(value, dtype=np.float64).reshape(self._host.shape)

    def device_densities(self):
        """Upload the field; returns the CUDA float64 tensor (S, nvox)."""
        torch = _lib.require_cuda()
        if self._dev is None:
            self._dev = torch.empty(self._host.shape, dtype=torch.float64, device="cuda")
        self._dev.copy_(torch.from_numpy(self._host))
        return self._dev

    def pull(self) -> None:
        """Write the device field back into the host array (in place)."""
        np.copyto(self._host, self._dev.cpu().numpy())

    def grid_view(self, s: int) -> np.ndarray:
        m = self.mesh
        return self._host[s].reshape(m.nz, m.ny, m.nx)

    def check_state(self) -> None:
        d = self._host
        if not np.isfinite(d).all() or (d < 0.0).any():
            raise NumericError("substrate field left finite/non-negative range")


@dataclass
class Cell:
    """One agent (core.py:148-163)."""

    id: int
    position: Vec3
    velocity: Vec3
    radius: float = 8.0
    repulsion: float = 10.0
    adhesion: float = 0.4
    adhesion_multiplier: float = 1.25
    division_rate: float = 0.0
    voxel_index: int = -1

    @property
    def volume(self) -> float:
        return (4.0 / 3.0) * math.pi * self.radius**3


class _DeviceCells:
    """Structure-of-arrays cell state in storage order (torch, cuda)."""

    def __init__(self, torch, n: int):
        dev = "cuda"
        self.n = n
        self.pos = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.vel = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.prev_vel = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.radius = torch.zeros(n, dtype=torch.float64, device=dev)
        self.volume = torch.zeros(n, dtype=torch.float64, device=dev)
        self.ids = torch.zeros(n, dtype=torch.int64, device=dev)


class _DeviceBins:
    """CSR voxel bins produced by cg_rebin (see include/cellgpu.h)."""

    def __init__(self, torch, n: int, nvox: int):
        dev = "cuda"
        i32 = torch.int32
        self.n, self.nvox = n, nvox
        self.voxel = torch.zeros(max(n, 1), dtype=i32, device=dev)
        self.bin_start = torch.zeros(nvox + 1, dtype=i32, device=dev)
        self.bin_cells = torch.zeros(max(n, 1), dtype=i32, device=dev)
        self.bin_cells_by_id = torch.zeros(max(n, 1), dtype=i32, device=dev)
        self.nonempty = torch.zeros(nvox, dtype=i32, device=dev)
        self.n_nonempty = torch.zeros(1, dtype=i32, device=dev)


class CellContainer:
    """Ordered cell storage plus the per-voxel spatial index (core.py:166-215).

    Storage order is the order of ``cells``; bins hold storage indices in
    storage order within each voxel, exactly like the reference's ``agent``.

    Two modes.  Object mode (``Cell`` objects exist): the objects are
    authoritative, every device call uploads them and writes its results back
    into the same objects.  Array mode (``from_arrays``): the state lives on
    the device only; reading ``cells`` or ``by_id`` materialises the objects
    once and switches the container to object mode.
    """

    def __init__(self, mesh: CartesianMesh):
        self.mesh = mesh
        self._cells: list | None = []
        self._by_id: dict | None = {}
        self._dev: _DeviceCells | None = None
        self._bins: _DeviceBins | None = None
        self._bins_mesh: CartesianMesh | None = None
        self._bins_ids = None   # device ids snapshot of the last rebin
        self._n = 0
        self._agent_override = None
        self._nonempty_override = None
        self._derived = None  # cached host agent/storage_index after a rebin
        self._prev_vel_host = None
        self._div_rate = None  # array mode: per-cell division rates (from_arrays)
        self.next_id = 0
        self.positions_dirty = False

    # ---- construction from arrays (large populations: no Cell objects)
    @classmethod
    def from_arrays(cls, mesh: CartesianMesh, positions, radius, ids=None,
                    velocities=None, division_rate=None) -> "CellContainer":
        """Container whose cells exist only on the device until ``cells`` is read.

        ``positions``: (n, 3); ``radius`` and ``division_rate``: scalar or
        (n,); ``ids`` default 0..n-1 in storage order.  Marked dirty, like
        ``new_cell``.
        """
        torch = _lib.require_cuda()
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        n = pos.shape[0]
        rad = np.ascontiguousarray(np.broadcast_to(np.asarray(radius, np.float64), (n,)))
        idv = np.arange(n, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        if len(np.unique(idv)) != n:
            raise DomainError("duplicate cell id")
        self = cls(mesh)
        self._cells = None
        self._by_id = None
        dc = _DeviceCells(torch, n)
        dc.pos.copy_(torch.from_numpy(pos))
        if velocities is not None:
            dc.vel.copy_(torch.from_numpy(np.ascontiguousarray(velocities, np.float64).reshape(n, 3)))
        dc.radius.copy_(torch.from_numpy(rad))
        dc.volume.copy_(torch.from_numpy(_lib.cell_volumes(rad)))
        dc.ids.copy_(torch.from_numpy(idv))
        self._dev = dc
        self._n = n
        self.next_id = int(idv.max()) + 1 if n else 0
        # per-cell division rates (population.attempt_divisions); daughters inherit
        self._div_rate = (None if division_rate is None else
                          np.ascontiguousarray(np.broadcast_to(
                              np.asarray(division_rate, np.float64), (n,))))
        self.positions_dirty = True
        return self

    @property
    def object_mode(self) -> bool:
        return self._cells is not None

    # ---- host views
    def __len__(self) -> int:
        return len(self._cells) if self._cells is not None else self._n

    def _materialize(self) -> None:
        """Array mode -> object mode: build the Cell objects from the device."""
        if self._cells is not None:
            return
        d = self._dev
        pos = d.pos.cpu().numpy()
        vel = d.vel.cpu().numpy()
        rad = d.radius.cpu().numpy()
        ids = d.ids.cpu().numpy()
        rate = self._div_rate
        self._cells = [Cell(id=int(ids[i]), position=pos[i].tolist(),
                            velocity=vel[i].tolist(), radius=float(rad[i]),
                            division_rate=0.0 if rate is None else float(rate[i]))
                       for i in range(d.n)]
        self._by_id = {c.id: c for c in self._cells}
        b = self._bins
        if b is not None and b.n == d.n and d.n:
            vox = b.voxel[: d.n].cpu().numpy()
            for i, c in enumerate(self._cells):
                c.voxel_index = int(vox[i])
        self._prev_vel_host = d.prev_vel.cpu().numpy()

    def _sync_back(self, *, pos: bool = False, vel: bool = False, voxel: bool = False,
                   prev: bool = False) -> None:
        """Object mode: write a device call's results into the held objects,
        in place (the reference mutates ``position``/``velocity`` lists and
        ``voxel_index`` of the same Cell objects)."""
        if self._cells is None:
            return
        d = self._dev
        n = d.n
        if n == 0:
            return
        cells = self._cells
        if pos:
            hp = d.pos.cpu().numpy().tolist()
            for c, p in zip(cells, hp):
                c.position[:] = p
        if vel:
            hv = d.vel.cpu().numpy().tolist()
            for c, v in zip(cells, hv):
                c.velocity[:] = v
        if voxel:
            vox = self._bins.voxel[:n].cpu().numpy().tolist()
            for c, v in zip(cells, vox):
                c.voxel_index = v
        if prev:
            self._prev_vel_host = d.prev_vel.cpu().numpy()

    @property
    def cells(self) -> list:
        self._materialize()
        return self._cells

    @cells.setter
    def cells(self, value) -> None:
        self._materialize()
        self._cells = value

    @property
    def by_id(self) -> dict:
        self._materialize()
        return self._by_id

    @by_id.setter
    def by_id(self, value) -> None:
        self._materialize()
        self._by_id = value

    @property
    def previous_velocities(self) -> np.ndarray:
        """G2 (AB2) state: velocity of the previous mechanics step, (n, 3)."""
        self._materialize()
        if self._prev_vel_host is None or self._prev_vel_host.shape[0] != len(self._cells):
            self._prev_vel_host = np.zeros((len(self._cells), 3))
        return self._prev_vel_host

    def _derive(self):
        if self._derived is None:
            if self._bins is None or self._bins_ids is None:
                self._derived = ({}, {}, [])
            else:
                b = self._bins
                n = b.n
                ids = self._bins_ids.cpu().numpy()
                bs = b.bin_start.cpu().numpy()
                bc = b.bin_cells[:n].cpu().numpy()
                nne = int(b.n_nonempty.cpu().item())
                ne = b.nonempty[:nne].cpu().numpy()
                agent = {int(v): [int(ids[c]) for c in bc[bs[v]:bs[v + 1]]] for v in ne.tolist()}
                storage_index = {int(ids[i]): i for i in range(n)}
                self._derived = (agent, storage_index, ne.tolist())
        return self._derived

    @property
    def agent(self) -> dict:
        if self._agent_override is not None:
            return self._agent_override
        return self._derive()[0]

    @agent.setter
    def agent(self, value) -> None:
        self._agent_override = value

    @property
    def storage_index(self) -> dict:
        return self._derive()[1]

    @property
    def nonempty_voxels(self) -> list:
        if self._nonempty_override is not None:
            return self._nonempty_override
        return list(self._derive()[2])

    @nonempty_voxels.setter
    def nonempty_voxels(self, value) -> None:
        self._nonempty_override = list(value)

    def max_radius(self) -> float:
        if self._cells is not None:
            return max((c.radius for c in self._cells), default=0.0)
        d = self._dev
        return float(d.radius.max().item()) if d.n else 0.0

    # ---- mutation (host)
    def new_cell(self, position, **kwargs) -> Cell:
        self._materialize()
        cell = Cell(id=self.next_id, position=list(position), velocity=vec3(), **kwargs)
        self.next_id += 1
        self._cells.append(cell)
        self._by_id[cell.id] = cell
        self.positions_dirty = True
        return cell

    def append_cell(self, cell: Cell) -> None:
        self._materialize()
        if cell.id in self._by_id:
            raise DomainError(f"duplicate cell id {cell.id}")
        self.next_id = max(self.next_id, cell.id + 1)
        self._cells.append(cell)
        self._by_id[cell.id] = cell
        self.positions_dirty = True

    def check_consistent(self) -> None:
        """Verify the container invariants; AssertionError on violation (core.py:204-215)."""
        seen = 0
        for v, ids in self.agent.items():
            assert ids, f"agent list for voxel {v} is empty but present"
            for cid in ids:
                cell = self.by_id[cid]
                assert cell.voxel_index == v
                assert self.mesh.voxel_of(cell.position) == v
                seen += 1
        assert seen == len(self.cells)
        assert self.nonempty_voxels == sorted(self.agent)

    # ---- device views
    def device_cells(self) -> _DeviceCells:
        """SoA tensors in storage order.  Object mode uploads the objects on
        every call (they are authoritative); array mode returns the resident
        tensors."""
        torch = _lib.require_cuda()
        cells = self._cells
        if cells is not None:
            n = len(cells)
            if self._dev is None or self._dev.n != n:
                self._dev = _DeviceCells(torch, n)
            d = self._dev
            pv = self._prev_vel_host
            if pv is not None and pv.shape[0] == n:
                d.prev_vel.copy_(torch.from_numpy(np.ascontiguousarray(pv, np.float64)))
            else:
                d.prev_vel.zero_()
            if n:
                pos = np.array([c.position for c in cells], dtype=np.float64).reshape(n, 3)
                vel = np.array([c.velocity for c in cells], dtype=np.float64).reshape(n, 3)
                rad = np.array([c.radius for c in cells], dtype=np.float64)
                ids = np.array([c.id for c in cells], dtype=np.int64)
                d.pos.copy_(torch.from_numpy(pos))
                d.vel.copy_(torch.from_numpy(vel))
                d.radius.copy_(torch.from_numpy(rad))
                d.volume.copy_(torch.from_numpy(_lib.cell_volumes(rad)))
                d.ids.copy_(torch.from_numpy(ids))
        self._n = self._dev.n
        return self._dev

    def device_bins(self, mesh: CartesianMesh | None = None) -> _DeviceBins:
        torch = _lib.require_cuda()
        mesh = mesh or self.mesh
        n = self._dev.n if self._dev is not None else len(self)
        if (self._bins is None or self._bins.n != n or self._bins_mesh != mesh):
            self._bins = _DeviceBins(torch, n, mesh.voxel_count)
            self._bins_mesh = mesh
        return self._bins


def rebin_cells(container: CellContainer, mesh: CartesianMesh | None = None) -> CellContainer:
    """Rebuild the per-voxel bins, storage index and non-empty list on the GPU
    (core.py:218-240) as a counting sort; raises DomainError for a cell
    outside the mesh.  Object mode: every cell's ``voxel_index`` is updated."""
    mesh = mesh or container.mesh
    t0 = time.perf_counter()
    d = container.device_cells()
    b = container.device_bins(mesh)
    ctx = _lib.context_for(mesh, 0, d.n)
    L = _lib.load()
    P = _lib.ptr
    code = L.cg_rebin(ctx.handle, d.n, P(d.pos), P(d.ids), P(b.voxel), P(b.bin_start),
                      P(b.bin_cells), P(b.bin_cells_by_id), P(b.nonempty), P(b.n_nonempty))
    _lib.raise_for(code, "rebin_cells")
    ctx.sync("rebin_cells")
    container._bins_ids = d.ids.clone()
    container._derived = None
    container._agent_override = None
    container._nonempty_override = None
    container._sync_back(voxel=True)
    container.positions_dirty = False
    container._last_elapsed = time.perf_counter() - t0
    return container


def sort_cells_by_voxel(container: CellContainer) -> CellContainer:
    """Reorder storage by (voxel index, id) and rebuild the spatial index
    (population.py:132-135).  The key is each cell's voxel_index from the last
    rebin, as in the reference.  Device-resident containers whose bins match
    their cells are permuted on the GPU: the id-sorted bins, read in voxel
    order, are exactly that order."""
    b = container._bins
    d = container._dev
    if (container._cells is None and d is not None and b is not None and b.n == d.n
            and container._bins_ids is not None):
        order = b.bin_cells_by_id[:d.n].long()
        for name in ("pos", "vel", "prev_vel", "radius", "volume", "ids"):
            t = getattr(d, name)
            t.copy_(t[order])
        if container._div_rate is not None:  # division rates move with their cell
            container._div_rate = container._div_rate[order.cpu().numpy()]
        return rebin_cells(container)
    cells = container.cells
    order = sorted(range(len(cells)), key=lambda i: (cells[i].voxel_index, cells[i].id))
    cells[:] = [cells[i] for i in order]
    pv = container._prev_vel_host
    if pv is not None and pv.shape[0] == len(order):
        container._prev_vel_host = pv[order]  # the AB2 state moves with its cell
    return rebin_cells(container)
