"""ctypes wrapper over liboracle.so -- the CPU ORACLE (test infrastructure).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module, and only as the checker or the
CPU baseline; the product package never does.  See cellref.h for what each
function restates (reference file:line) and how the oracle is pinned.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OK, DOMAIN, NUMERIC, STATE, CAPACITY = 0, 1, 2, 3, 4
BC_NEUMANN, BC_DIRICHLET = 0, 1
EULER, AB2 = 0, 1
SQUARE_POW, SQUARE_MUL = 0, 1


class OracleError(Exception):
    def __init__(self, code, what):
        super().__init__(f"oracle {what} returned status {code}")
        self.code = code


class RefMesh(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
        ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double),
        ("ox", ctypes.c_double), ("oy", ctypes.c_double), ("oz", ctypes.c_double),
    ]


def build() -> str:
    """Compile liboracle.so with the oracle's Makefile (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I, D, LG = ctypes.c_int, ctypes.c_double, ctypes.c_long
        M = ctypes.POINTER(RefMesh)
        L.ref_voxel_of.argtypes = [M, P, P]
        L.ref_line_factors.argtypes = [I, D, D, P, P]
        L.ref_line_factors.restype = None
        L.ref_lod_step.argtypes = [M, I, P, P, P, D, I, P, I]
        L.ref_exchange.argtypes = [M, P, I, I, D, P, P, LG, LG, P, LG, I, P, P, P, P, P, I, I]
        L.ref_rebin.argtypes = [M, I, P, P, P, P, P, P]
        L.ref_velocities.argtypes = [M, I, P, P, P, P, P, P, D, D, D, I, P, I]
        L.ref_integrate.argtypes = [M, I, P, P, P, D, I, I]
        L.ref_cell_volumes.argtypes = [I, P, P]
        L.ref_cell_volumes.restype = None
        L.ref_mech_step.argtypes = (
            [M, I, P, P, P, D, I, I, P, P, P, P, I, P, P, P, P, P, P, P, P, P, P, P,
             D, D, D, D, I, I, I])
        L.ref_max_threads.argtypes = []
        U64, I64 = ctypes.c_uint64, ctypes.c_int64
        L.ref_division_draws.argtypes = [U64, I64, I64, P]
        L.ref_division_draws.restype = None
        L.ref_divisions.argtypes = [M, I, P, P, P, P, D, U64, I64, I, P, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(code, what):
    if code != OK:
        raise OracleError(code, what)


def mesh_struct(nx, ny, nz, dx=20.0, dy=20.0, dz=20.0, origin=(0.0, 0.0, 0.0)):
    return RefMesh(nx, ny, nz, dx, dy, dz, *[float(o) for o in origin])


def mesh_from(mesh) -> RefMesh:
    """RefMesh from any object with nx..nz, dx..dz, origin (reference or ours)."""
    return mesh_struct(mesh.nx, mesh.ny, mesh.nz, mesh.dx, mesh.dy, mesh.dz, mesh.origin)


def max_threads() -> int:
    return lib().ref_max_threads()


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def line_factors(n, r, lam3):
    inv = np.empty(max(n, 1))
    gam = np.empty(max(n, 1))
    lib().ref_line_factors(n, r, lam3, _p(inv), _p(gam))
    return inv[:n].copy(), (gam[:n].copy() if n > 1 else np.zeros(0))


def voxel_of(m: RefMesh, p) -> int:
    p = f64(p)
    out = np.zeros(1, np.int32)
    _check(lib().ref_voxel_of(ctypes.byref(m), _p(p), _p(out)), "voxel_of")
    return int(out[0])


def lod_step(m: RefMesh, dens, diffusion, decay, dt, bc=BC_NEUMANN, dirichlet=None, threads=1):
    """In place on dens (S, nvox) float64 C-contiguous."""
    assert dens.dtype == np.float64 and dens.flags.c_contiguous
    S = dens.shape[0]
    D = f64(diffusion).reshape(S)
    K = f64(decay).reshape(S)
    dv = None if dirichlet is None else f64(dirichlet).reshape(S)
    _check(lib().ref_lod_step(ctypes.byref(m), S, _p(dens), _p(D), _p(K), float(dt), bc,
                              _p(dv), threads), "lod_step")


class Bins:
    """Output of rebin: voxel per cell, CSR bins (storage order), non-empty list."""

    def __init__(self, voxel, bin_start, bin_cells, nonempty):
        self.voxel = voxel
        self.bin_start = bin_start
        self.bin_cells = bin_cells
        self.nonempty = nonempty

    def agent(self):
        """The reference's container.agent dict: voxel -> [ids in storage order]."""
        out = {}
        for v in self.nonempty.tolist():
            out[v] = self.bin_cells[self.bin_start[v]:self.bin_start[v + 1]].tolist()
        return out


def rebin(m: RefMesh, pos) -> Bins:
    pos = f64(pos).reshape(-1, 3)
    n = pos.shape[0]
    nvox = m.nx * m.ny * m.nz
    voxel = np.zeros(n, np.int32)
    bin_start = np.zeros(nvox + 1, np.int32)
    bin_cells = np.zeros(max(n, 1), np.int32)
    nonempty = np.zeros(nvox, np.int32)
    nne = np.zeros(1, np.int32)
    _check(lib().ref_rebin(ctypes.byref(m), n, _p(pos), _p(voxel), _p(bin_start),
                           _p(bin_cells), _p(nonempty), _p(nne)), "rebin")
    return Bins(voxel, bin_start, bin_cells[:n], nonempty[: int(nne[0])].copy())


def exchange(m: RefMesh, dens, bins: Bins, ids, volume, dt, secretion, uptake, saturation,
             substrates=None, threads=1):
    """apply_cell_exchange.  secretion/uptake: scalar, (S,) or (S, n) arrays;
    saturation: scalar or (S,).  substrates: (s0, s1) range, default all."""
    S, _ = dens.shape
    n = len(ids)
    s0, s1 = substrates if substrates is not None else (0, S)
    sec = np.asarray(secretion, dtype=np.float64)
    upt = np.asarray(uptake, dtype=np.float64)
    if sec.ndim == 0:
        sec = np.full((S, 1), float(sec))
        upt = np.full((S, 1), float(upt))
        strides = (1, 0)
    else:
        sec = np.ascontiguousarray(np.broadcast_to(sec.reshape(S, -1), (S, n)))
        upt = np.ascontiguousarray(np.broadcast_to(upt.reshape(S, -1), (S, n)))
        strides = (n, 1)
    sat = np.ascontiguousarray(np.broadcast_to(f64(saturation).reshape(-1), (S,)))
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    volume = f64(volume)
    _check(lib().ref_exchange(ctypes.byref(m), _p(dens), s0, s1, float(dt), _p(sec), _p(upt),
                              strides[0], strides[1], _p(sat), 1, n, _p(volume), _p(ids),
                              _p(bins.bin_start), _p(bins.bin_cells), _p(bins.nonempty),
                              len(bins.nonempty), threads), "exchange")


def velocities(m: RefMesh, pos, radius, ids, bins: Bins, repulsion=10.0, adhesion=0.4,
               adhesion_multiplier=1.25, square_mode=SQUARE_POW, threads=1):
    pos = f64(pos).reshape(-1, 3)
    n = pos.shape[0]
    vel = np.zeros((n, 3))
    _check(lib().ref_velocities(ctypes.byref(m), n, _p(pos), _p(f64(radius)),
                                _p(np.ascontiguousarray(ids, dtype=np.int64)), _p(bins.voxel),
                                _p(bins.bin_start), _p(bins.bin_cells), float(repulsion),
                                float(adhesion), float(adhesion_multiplier), square_mode,
                                _p(vel), threads), "velocities")
    return vel


def integrate(m: RefMesh, pos, vel, dt, prev_vel=None, integrator=EULER, threads=1):
    """In place on pos (and prev_vel for AB2)."""
    assert pos.dtype == np.float64 and pos.flags.c_contiguous
    n = pos.shape[0]
    v = f64(vel)
    _check(lib().ref_integrate(ctypes.byref(m), n, _p(pos), _p(v), _p(prev_vel), float(dt),
                               integrator, threads), "integrate")


def division_draws(seed, cell_id, step):
    """population.py:44-51: three uniforms for (seed, cell id, step)."""
    out = np.empty(3)
    lib().ref_division_draws(int(seed) & ((1 << 64) - 1), int(cell_id), int(step), _p(out))
    return tuple(float(x) for x in out)


def divisions(m: RefMesh, ids, pos, radius, rate, dt, seed, step, cap):
    """population.py:77-129 minus the container bookkeeping: (parent indices in
    ascending parent id, daughter positions); None when n + count > cap."""
    ids = np.ascontiguousarray(ids, np.int64)
    pos, rad, rate = f64(pos), f64(radius), f64(rate)
    n = len(ids)
    parent = np.empty(max(n, 1), np.int32)
    out = np.empty((max(n, 1), 3))
    k = lib().ref_divisions(ctypes.byref(m), n, _p(ids), _p(pos), _p(rad), _p(rate), float(dt),
                            int(seed) & ((1 << 64) - 1), int(step), int(cap), _p(parent), _p(out))
    if k < 0:
        return None
    return parent[:k].copy(), out[:k].copy()


def cell_volumes(radius):
    r = f64(radius)
    out = np.empty_like(r)
    lib().ref_cell_volumes(len(r), _p(r), _p(out))
    return out


class OracleState:
    """Host-side state of one simulation, advanced by ref_mech_step."""

    def __init__(self, m: RefMesh, dens, pos, radius, ids, diffusion, decay, *,
                 secretion=None, uptake=None, saturation=None, bc=BC_NEUMANN,
                 dirichlet=None, repulsion=10.0, adhesion=0.4, adhesion_multiplier=1.25,
                 dt_diff=0.01, dt_mech=0.1, substeps=10, integrator=EULER,
                 square_mode=SQUARE_POW, vel=None, prev_vel=None):
        self.m = m
        self.dens = np.array(dens, dtype=np.float64, order="C")
        self.S = self.dens.shape[0]
        self.pos = np.array(pos, dtype=np.float64, order="C").reshape(-1, 3)
        self.n = self.pos.shape[0]
        self.radius = f64(radius)
        self.volume = cell_volumes(self.radius)
        self.ids = np.ascontiguousarray(ids, dtype=np.int64)
        self.vel = np.zeros((self.n, 3)) if vel is None else np.array(vel, np.float64)
        self.prev_vel = (np.zeros((self.n, 3)) if prev_vel is None
                         else np.array(prev_vel, np.float64))
        self.diffusion = f64(diffusion).reshape(self.S)
        self.decay = f64(decay).reshape(self.S)
        self.secretion = None if secretion is None else np.ascontiguousarray(
            np.broadcast_to(f64(secretion).reshape(self.S, -1), (self.S, self.n)))
        self.uptake = None if uptake is None else np.ascontiguousarray(
            np.broadcast_to(f64(uptake).reshape(self.S, -1), (self.S, self.n)))
        self.saturation = (np.full(self.S, 38.0) if saturation is None
                           else np.ascontiguousarray(np.broadcast_to(
                               f64(saturation).reshape(-1), (self.S,))))
        self.bc = bc
        self.dirichlet = None if dirichlet is None else f64(dirichlet).reshape(self.S)
        self.params = (float(repulsion), float(adhesion), float(adhesion_multiplier))
        self.dt_diff, self.dt_mech, self.substeps = float(dt_diff), float(dt_mech), int(substeps)
        self.integrator, self.square_mode = integrator, square_mode
        self.bins = rebin(m, self.pos)
        nvox = m.nx * m.ny * m.nz
        self._nonempty_buf = np.zeros(nvox, np.int32)
        self._nonempty_buf[: len(self.bins.nonempty)] = self.bins.nonempty
        self._nne = np.array([len(self.bins.nonempty)], np.int32)
        self._bin_cells = np.zeros(max(self.n, 1), np.int32)
        self._bin_cells[: self.n] = self.bins.bin_cells

    def step(self, threads=1):
        b = self.bins
        _check(lib().ref_mech_step(
            ctypes.byref(self.m), self.S, _p(self.dens), _p(self.diffusion), _p(self.decay),
            self.dt_diff, self.substeps, self.bc, _p(self.dirichlet), _p(self.secretion),
            _p(self.uptake), _p(self.saturation), self.n, _p(self.pos), _p(self.vel),
            _p(self.prev_vel), _p(self.radius), _p(self.volume), _p(self.ids), _p(b.voxel),
            _p(b.bin_start), _p(self._bin_cells), _p(self._nonempty_buf), _p(self._nne),
            self.params[0], self.params[1], self.params[2], self.dt_mech, self.integrator,
            self.square_mode, threads), "mech_step")
        b.bin_cells = self._bin_cells[: self.n]
        b.nonempty = self._nonempty_buf[: int(self._nne[0])].copy()
