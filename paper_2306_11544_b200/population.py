"""Cell divisions on the GPU (reference: cellbench/population.py).

``division_draws`` and ``attempt_divisions`` keep the reference's signatures
and semantics (population.py:44-129): the counter-based draws keyed by
(seed, cell id, step), the hazard rule u0 < 1 - exp(-rate*dt), daughters in
ascending parent id with fresh ids, placed R/2 away along the drawn
direction and clamped inside, velocity copied from the parent, the cap
checked before anything is appended, then a rebin.

The draws, the decisions and the placement run in libcellgpu.so
(cg_division_draws / cg_divisions_count / cg_divisions_place).  The
threshold 1 - exp(-rate*dt) is evaluated once per distinct rate on the host
with the same libm ``exp`` CPython uses, so which cells divide is bit-exact;
the device cos/sin place daughters within a few ulp of the reference (~1e-15
relative, inside the 1e-12 position bar).  ``sort_cells_by_voxel`` lives in
core (population.py:132-135).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .core import Cell, CartesianMesh, CellContainer, _DeviceCells, rebin_cells, sort_cells_by_voxel
from .errors import CapacityError, DomainError

#: population.py:28-29 desk-scale guard.
DEFAULT_CELL_CAP = 200000

_MASK = (1 << 64) - 1


def _as_i64(v: int) -> int:
    """Python's `v & _MASK` (population.py:46) as a two's-complement int64."""
    v = int(v) & _MASK
    return v - (1 << 64) if v >= 1 << 63 else v


def division_draws(seed: int, cell_id: int, step: int) -> tuple[float, float, float]:
    """Three uniforms in [0, 1) that depend only on (seed, cell id, step)
    (population.py:44-51), computed on the device."""
    torch = _lib.require_cuda()
    ctx = _lib.context_for(CartesianMesh(1, 1, 1), 0, 1)
    ids = torch.tensor([_as_i64(cell_id)], dtype=torch.int64, device="cuda")
    out = torch.empty(3, dtype=torch.float64, device="cuda")
    _lib.raise_for(_lib.load().cg_division_draws(ctx.handle, 1, int(seed) & _MASK, _as_i64(step),
                                                  _lib.ptr(ids), _lib.ptr(out)), "division_draws")
    return tuple(float(x) for x in out.cpu().tolist())


def _thresholds(rates: np.ndarray, dt: float) -> np.ndarray:
    """1 - exp(-rate*dt) per cell (CPython's math.exp per distinct rate), -1
    where rate <= 0 (never divides)."""
    thr = np.full(len(rates), -1.0)
    for r in np.unique(rates):
        if r > 0.0:
            thr[rates == r] = 1.0 - math.exp(-float(r) * dt)
    return thr


def _rates(container: CellContainer) -> np.ndarray:
    if container.object_mode:
        return np.array([c.division_rate for c in container.cells], dtype=np.float64)
    r = container._div_rate
    return np.zeros(len(container)) if r is None else r


def attempt_divisions(container: CellContainer, seed: int, dt: float, mesh: CartesianMesh,
                      step: int, cap: int = DEFAULT_CELL_CAP):
    """Division pass (population.py:77-129).  Object mode returns the
    daughters (``Cell`` objects, appended in parent-id order); a
    device-resident container (``from_arrays``) grows on the device and the
    daughters' ids are returned as an int64 array."""
    if not dt > 0.0:
        raise DomainError("division step needs dt > 0")
    n = len(container)
    rates = _rates(container)
    if n == 0 or not (rates > 0.0).any():
        return [] if container.object_mode else np.zeros(0, np.int64)
    torch = _lib.require_cuda()
    d = container.device_cells()
    ctx = _lib.context_for(mesh, 0, n)
    L = _lib.load()
    P = _lib.ptr
    thr = torch.from_numpy(_thresholds(rates, float(dt))).cuda()
    step64 = _as_i64(step)
    seed64 = int(seed) & _MASK
    cnt = _lib.I(0)
    _lib.raise_for(L.cg_divisions_count(ctx.handle, n, seed64, step64, P(d.ids), P(thr),
                                        ctypes.byref(cnt)), "attempt_divisions")
    m = int(cnt.value)
    if m == 0:
        return [] if container.object_mode else np.zeros(0, np.int64)
    if n + m > cap:
        raise CapacityError(f"division would exceed the {cap}-cell cap ({n} + {m})")
    parent = torch.empty(m, dtype=torch.int32, device="cuda")
    dpos = torch.empty((m, 3), dtype=torch.float64, device="cuda")
    _lib.raise_for(L.cg_divisions_place(ctx.handle, n, m, seed64, step64, P(d.ids), P(d.pos),
                                        P(d.radius), P(parent), P(dpos)), "attempt_divisions")
    ctx.sync("attempt_divisions")
    new_ids = np.arange(container.next_id, container.next_id + m, dtype=np.int64)
    if container.object_mode:
        cells = container.cells
        par = parent.cpu().numpy()
        hp = dpos.cpu().numpy().tolist()
        prev = container._prev_vel_host
        daughters = []
        for r in range(m):
            p = cells[int(par[r])]
            dcell = container.new_cell(hp[r], radius=p.radius, repulsion=p.repulsion,
                                       adhesion=p.adhesion,
                                       adhesion_multiplier=p.adhesion_multiplier,
                                       division_rate=p.division_rate)
            dcell.velocity[0] = p.velocity[0]
            dcell.velocity[1] = p.velocity[1]
            dcell.velocity[2] = p.velocity[2]
            daughters.append(dcell)
        if prev is not None and prev.shape[0] == n:  # G2 AB2 state follows the parent
            container._prev_vel_host = np.concatenate([prev, prev[par]])
        rebin_cells(container, mesh)
        return daughters
    # device-resident: grow the arrays; daughters copy the parent's state
    pl = parent.long()
    nd = _DeviceCells(torch, n + m)
    for name in ("pos", "vel", "prev_vel", "radius", "volume", "ids"):
        getattr(nd, name)[:n] = getattr(d, name)
    nd.pos[n:] = dpos
    nd.vel[n:] = d.vel[pl]
    nd.prev_vel[n:] = d.prev_vel[pl]
    nd.radius[n:] = d.radius[pl]
    nd.volume[n:] = d.volume[pl]
    nd.ids[n:] = torch.from_numpy(new_ids).cuda()
    container._dev = nd
    container._n = n + m
    container._div_rate = np.concatenate([rates, rates[parent.cpu().numpy()]])
    container.next_id += m
    container.positions_dirty = True
    rebin_cells(container, mesh)
    return new_ids


__all__ = ["DEFAULT_CELL_CAP", "attempt_divisions", "division_draws", "sort_cells_by_voxel",
           "Cell"]
