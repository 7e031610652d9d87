"""Neighbour-interaction velocities and position integration on the GPU.

Mirrors /root/reference/pkg/src/cellbench/mechanics.py: ``InteractionParams``
(:74-84), ``MechanicsSchedule`` / ``ScheduleKind`` (:41-71),
``check_binning_exact`` (:87-96), ``pair_velocity_contribution`` (:99-115, a
scalar host helper), ``update_velocities`` (:175-225) and
``integrate_positions`` (:228-245).  Schedules and allocation modes are
accepted and only shape the returned record: on the GPU every schedule is the
same warp-per-non-empty-voxel kernel, and the reference guarantees all of them
are bit-identical anyway (mechanics.py:1-8).

Keyword-only extension (G2): ``integrate_positions(..., integrator="ab2")``
applies PhysiCell's Adams-Bashforth 2 update ``x += 1.5 dt v - 0.5 dt v_prev``
with ``v_prev`` kept per cell in the container (``previous_velocities``).
"""

from __future__ import annotations


import enum
import math
import time

import numpy as np
from dataclasses import dataclass

from . import _lib
from .core import CartesianMesh, Cell, CellContainer, Vec3
from .errors import ContainerStateError, DomainError
from .parallel import RegionRecord, gpu_record

#: Pairs closer than this (um) are skipped; the direction is numerically void.
EPS_SKIP = 1e-8


class AllocationMode(enum.Enum):
    """Accepted for signature compatibility (smallvec.py:25-27); the kernels
    allocate nothing per interaction in either mode."""

    TEMPORARY_ALLOCATING = "temporary_allocating"
    IN_PLACE = "in_place"


class ScheduleKind(enum.Enum):
    CELL_STATIC = "cell_static"
    CELL_DYNAMIC = "cell_dynamic"
    VOXEL = "voxel"
    NONEMPTY_VOXEL = "nonempty_voxel"


@dataclass(frozen=True)
class MechanicsSchedule:
    kind: ScheduleKind
    grain: int = 16

    def __post_init__(self):
        if self.grain < 1:
            raise DomainError("schedule grain must be >= 1")

    @staticmethod
    def cell_static() -> "MechanicsSchedule":
        return MechanicsSchedule(ScheduleKind.CELL_STATIC)

    @staticmethod
    def cell_dynamic(grain: int = 16) -> "MechanicsSchedule":
        return MechanicsSchedule(ScheduleKind.CELL_DYNAMIC, grain)

    @staticmethod
    def voxel(grain: int = 16) -> "MechanicsSchedule":
        return MechanicsSchedule(ScheduleKind.VOXEL, grain)

    @staticmethod
    def nonempty_voxel(grain: int = 16) -> "MechanicsSchedule":
        return MechanicsSchedule(ScheduleKind.NONEMPTY_VOXEL, grain)


@dataclass(frozen=True)
class InteractionParams:
    repulsion: float = 10.0
    adhesion: float = 0.4
    adhesion_multiplier: float = 1.25

    def __post_init__(self):
        if self.repulsion < 0.0 or self.adhesion < 0.0:
            raise DomainError("interaction strengths must be >= 0")
        if self.adhesion_multiplier < 1.0:
            raise DomainError("adhesion range multiplier must be >= 1")


def binning_report(positions, radius, mesh: CartesianMesh, params: InteractionParams) -> dict:
    """What the truncated 3x3x3 neighbourhood drops (the pairs
    check_binning_exact guards against, mechanics.py:87-96): every pair of
    cells closer than its adhesion reach m_a * (R_i + R_j) (and farther than
    EPS_SKIP, mechanics.py:110) whose voxels are more than one voxel apart on
    some axis, so _voxel_candidates (mechanics.py:118-133) never offers it.
    Host diagnostic (scipy k-d tree over the positions); returns the counts
    and the missed fraction of all in-range pairs."""
    from scipy.spatial import cKDTree

    pos = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    rad = np.ascontiguousarray(np.broadcast_to(np.asarray(radius, np.float64), (len(pos),)))
    m_a = float(params.adhesion_multiplier)
    r_max = float(rad.max()) if len(rad) else 0.0
    reach_max = m_a * 2.0 * r_max
    out = {"reach_max": reach_max, "voxel_edge_min": min(mesh.dx, mesh.dy, mesh.dz),
           "binning_exact": min(mesh.dx, mesh.dy, mesh.dz) >= reach_max}
    if len(pos) < 2:
        out.update(in_range_pairs=0, missed_pairs=0, missed_fraction=0.0)
        return out
    pairs = cKDTree(pos).query_pairs(reach_max, output_type="ndarray")
    i, j = pairs[:, 0], pairs[:, 1]
    d = np.sqrt(np.sum((pos[j] - pos[i]) ** 2, axis=1))
    keep = (d >= 1e-8) & (d < m_a * (rad[i] + rad[j]))
    i, j = i[keep], j[keep]
    org = np.asarray(mesh.origin, np.float64)
    sp = np.array([mesh.dx, mesh.dy, mesh.dz])
    idx = np.floor((pos - org) / sp).astype(np.int64)
    far = np.any(np.abs(idx[i] - idx[j]) > 1, axis=1)
    n_in, n_miss = int(len(i)), int(far.sum())
    out.update(in_range_pairs=n_in, missed_pairs=n_miss,
               missed_fraction=(n_miss / n_in) if n_in else 0.0)
    return out


def check_binning_exact(container: CellContainer, mesh: CartesianMesh,
                        params: InteractionParams) -> None:
    """Voxel binning covers every interaction iff edge >= m_a * 2 * R_max.

    The BASELINE configs violate this (R = 8.4127 um, 20 um voxels; SURVEY.md
    G3): like the reference's update_velocities, this package then uses the
    truncated 3x3x3 neighbourhood; the guard is only enforced when called."""
    r_max = container.max_radius()
    reach = params.adhesion_multiplier * 2.0 * r_max
    if min(mesh.dx, mesh.dy, mesh.dz) < reach:
        raise DomainError(
            f"voxel edge {min(mesh.dx, mesh.dy, mesh.dz)} shorter than the "
            f"interaction reach {reach}; neighbor binning would miss pairs")


def pair_velocity_contribution(ci: Cell, cj: Cell, params: InteractionParams) -> Vec3:
    """Scalar host helper: velocity contribution of cj on ci (mechanics.py:99-115)."""
    if ci.id == cj.id:
        raise DomainError("pair contribution needs two distinct cells")
    pi, pj = ci.position, cj.position
    dx = pj[0] - pi[0]
    dy = pj[1] - pi[1]
    dz = pj[2] - pi[2]
    d = math.sqrt(dx * dx + dy * dy + dz * dz)
    contact = ci.radius + cj.radius
    reach = params.adhesion_multiplier * contact
    if d < EPS_SKIP or d >= reach:
        return [0.0, 0.0, 0.0]
    rep = -params.repulsion * (1.0 - d / contact) ** 2 if d < contact else 0.0
    adh = params.adhesion * (1.0 - d / reach) ** 2
    coef = (rep + adh) / d
    return [coef * dx, coef * dy, coef * dz]


def update_velocities(container: CellContainer, mesh: CartesianMesh,
                      params: InteractionParams, schedule: MechanicsSchedule, pool,
                      alloc_mode: AllocationMode = AllocationMode.IN_PLACE) -> RegionRecord:
    """Recompute every cell's velocity from its in-range neighbours."""
    if container.positions_dirty:
        raise ContainerStateError("velocity update requires a rebinned container")
    if schedule.kind not in ScheduleKind:
        raise DomainError(f"unknown schedule kind {schedule.kind!r}")
    t0 = time.perf_counter()
    d = container.device_cells()
    n = d.n
    b = container._bins
    nne = 0
    if n:
        if b is None or b.n != n:
            raise ContainerStateError("velocity update requires a rebinned container")
        ctx = _lib.context_for(container._bins_mesh or mesh, 0, n)
        P = _lib.ptr
        code = _lib.load().cg_velocities(
            ctx.handle, n, P(d.pos), P(d.radius), P(d.ids), P(b.bin_start),
            P(b.bin_cells_by_id), P(b.nonempty), P(b.n_nonempty), float(params.repulsion),
            float(params.adhesion), float(params.adhesion_multiplier), P(d.vel))
        _lib.raise_for(code, "update_velocities")
        ctx.sync("update_velocities")
        container._sync_back(vel=True)
        nne = int(b.n_nonempty.cpu().item())
    elapsed = time.perf_counter() - t0
    kind = schedule.kind
    if kind is ScheduleKind.CELL_STATIC:
        return gpu_record(n, n, elapsed)
    if kind is ScheduleKind.CELL_DYNAMIC:
        return gpu_record(n, -(-n // schedule.grain), elapsed, claims=-(-n // schedule.grain))
    if kind is ScheduleKind.VOXEL:
        nv = mesh.voxel_count
        return gpu_record(nv, -(-nv // schedule.grain), elapsed, claims=-(-nv // schedule.grain))
    return gpu_record(nne, -(-nne // schedule.grain), elapsed, claims=-(-nne // schedule.grain))


def integrate_positions(container: CellContainer, mesh: CartesianMesh, dt: float, pool, *,
                        integrator: str = "euler") -> RegionRecord:
    """x += dt*v (or G2 AB2), clamped strictly inside the mesh; marks dirty."""
    if dt <= 0.0:
        raise DomainError("integration needs dt > 0")
    if integrator not in ("euler", "ab2"):
        raise DomainError(f"unknown integrator {integrator!r}")
    t0 = time.perf_counter()
    d = container.device_cells()
    if d.n:
        ctx = _lib.context_for(mesh, 0, d.n)
        P = _lib.ptr
        code = _lib.load().cg_integrate(ctx.handle, d.n, P(d.pos), P(d.vel), P(d.prev_vel),
                                        float(dt),
                                        _lib.AB2 if integrator == "ab2" else _lib.EULER)
        _lib.raise_for(code, "integrate_positions")
        ctx.sync("integrate_positions")
        container._sync_back(pos=True, prev=True)
    container.positions_dirty = True
    return gpu_record(d.n, d.n, time.perf_counter() - t0)
