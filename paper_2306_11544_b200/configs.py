"""The five BASELINE.json configurations and their seeded synthetic inputs.

Every input is generated once on the host from ``numpy.random.default_rng``
with the config's seed; the GPU path, the CPU oracle and the reference all
consume the same arrays, so the RNG choice cannot affect parity.  Draw order
is fixed: positions (rejection sampling in the bounding cube, or the radial
inverse CDF for config 2), then radii when they are random, then uptake on
substrate 0, then secretion on substrates 1..S-1.

Resolutions of the BASELINE/reference gaps:
  G1 Dirichlet 38/0/0(/0) on every outer-face voxel; initial value = the
     Dirichlet value.          G2 Adams-Bashforth 2 position update.
  G3 R = 8.4127 um with 20 um voxels: the 3x3x3 neighbourhood is kept (as the
     reference's update_velocities computes it) and the guard is bypassed.
  G4 per-cell rates: uptake U[5,15] on s0, secretion U[0,1] on s1..S-1;
     config 0: uptake 10 on s0, no secretion.
  G5 cube [-L, L]^3 via the mesh origin; sphere seeding by rejection.
  G6 saturation (secretion target) 38 for every substrate.
  G7 config 2 keeps the stated exp(-r/150 um) profile truncated at 700 um
     (core overlap accepted; it stresses dense voxels).
  G8 config 2 runs 30 sim-min like config 1; config 4's global box is
     [-2560, 2560]^2 x [-320 P, 320 P] um for P ranks.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import CartesianMesh


@dataclass(frozen=True)
class SimConfig:
    name: str
    nx: int
    ny: int
    nz: int
    dx: float
    origin: tuple
    diffusion: tuple
    decay: tuple
    dirichlet: tuple
    n_cells: int
    seed: int
    seeding: str  # "sphere" | "radial" | "box"
    seed_radius: float = 0.0
    radial_scale: float = 150.0
    radial_cutoff: float = 700.0
    radius: float = 8.4127
    radius_sd: float = 0.0
    radius_clip: tuple = ()
    uptake: tuple = (5.0, 15.0)     # U[lo, hi] on substrate 0 (lo == hi: constant)
    secretion: tuple = (0.0, 1.0)   # U[lo, hi] on substrates 1..S-1
    saturation: float = 38.0
    repulsion: float = 10.0
    adhesion: float = 0.4
    adhesion_multiplier: float = 1.25
    dt_diffusion: float = 0.01
    dt_mechanics: float = 0.1
    sim_minutes: float = 6.0
    bc: str = "dirichlet"
    integrator: str = "ab2"

    @property
    def n_substrates(self) -> int:
        return len(self.diffusion)

    @property
    def substeps(self) -> int:
        return int(round(self.dt_mechanics / self.dt_diffusion))

    @property
    def mech_steps(self) -> int:
        return int(round(self.sim_minutes / self.dt_mechanics))

    @property
    def voxel_count(self) -> int:
        return self.nx * self.ny * self.nz

    def mesh(self) -> CartesianMesh:
        return CartesianMesh(self.nx, self.ny, self.nz, self.dx, self.dx, self.dx, self.origin)

    def field_bytes(self) -> int:
        """All substrates' fields, float64."""
        return 8 * self.voxel_count * self.n_substrates


D3 = (1.0e5, 1.0e3, 6.4e4)
K3 = (0.1, 0.01, 0.0256)
D4 = D3 + (5.0e4,)
K4 = K3 + (0.05,)

CONFIGS = {
    0: SimConfig("c0-cpu-ref", 20, 20, 20, 20.0, (-200.0, -200.0, -200.0), (1.0e5,), (0.1,),
                 (38.0,), 2000, 0, "sphere", seed_radius=150.0, uptake=(10.0, 10.0),
                 secretion=(0.0, 0.0), sim_minutes=6.0),
    1: SimConfig("c1-1gpu-mid", 80, 80, 80, 20.0, (-800.0,) * 3, D3, K3, (38.0, 0.0, 0.0),
                 100_000, 1, "sphere", seed_radius=600.0, sim_minutes=30.0),
    2: SimConfig("c2-spheroid", 80, 80, 80, 20.0, (-800.0,) * 3, D3, K3, (38.0, 0.0, 0.0),
                 200_000, 2, "radial", radial_scale=150.0, radial_cutoff=700.0, radius=8.41,
                 radius_sd=0.5, radius_clip=(7.0, 10.0), sim_minutes=30.0),
    3: SimConfig("c3-strong", 160, 160, 160, 20.0, (-1600.0,) * 3, D4, K4,
                 (38.0, 0.0, 0.0, 0.0), 1_000_000, 3, "sphere", seed_radius=1400.0,
                 sim_minutes=10.0),
    4: SimConfig("c4-weak-slab", 256, 256, 32, 20.0, (-2560.0, -2560.0, -320.0), D4, K4,
                 (38.0, 0.0, 0.0, 0.0), 1_000_000, 4, "box", sim_minutes=5.0),
}


def slab_config(cfg: SimConfig, rank: int, world: int) -> SimConfig:
    """Config 4 per-rank slab: global nz = 32 * world, rank owns planes
    [32 rank, 32 rank + 32); seed 4 + rank."""
    from dataclasses import replace

    oz = -320.0 * world + 640.0 * rank
    return replace(cfg, origin=(cfg.origin[0], cfg.origin[1], oz), seed=cfg.seed + rank)


@dataclass
class Inputs:
    """Host arrays of one configuration (storage order = id order)."""

    positions: np.ndarray   # (n, 3)
    radius: np.ndarray      # (n,)
    ids: np.ndarray         # (n,) int64
    secretion: np.ndarray   # (S, n)
    uptake: np.ndarray      # (S, n)
    densities: np.ndarray   # (S, nvox)
    extra: dict = field(default_factory=dict)


def _sphere(rng, n, r, center=(0.0, 0.0, 0.0)):
    out = np.empty((0, 3))
    while out.shape[0] < n:
        batch = rng.uniform(-r, r, size=(2 * (n - out.shape[0]) + 16, 3))
        keep = batch[(batch * batch).sum(axis=1) < r * r]
        out = np.concatenate([out, keep])
    return out[:n] + np.asarray(center)


def _radial(rng, n, scale, cutoff):
    # density ~ exp(-r/a) in 3D: radial pdf ~ r^2 exp(-r/a) on [0, cutoff]
    grid = np.linspace(0.0, cutoff, 200_001)
    pdf = grid * grid * np.exp(-grid / scale)
    cdf = np.concatenate([[0.0], np.cumsum(0.5 * (pdf[1:] + pdf[:-1]) * np.diff(grid))])
    cdf /= cdf[-1]
    u = rng.uniform(0.0, 1.0, n)
    r = np.interp(u, cdf, grid)
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1)[:, None]
    return v * r[:, None]


def _clamp_inside(mesh: CartesianMesh, pos):
    lo = np.asarray(mesh.origin) + 1e-6
    hi = np.asarray(mesh.upper) - 1e-6
    return np.minimum(np.maximum(pos, lo), hi)


def make_inputs(cfg: SimConfig, n_cells: int | None = None) -> Inputs:
    """Seeded synthetic inputs; ``n_cells`` overrides the count (smaller parity cases)."""
    rng = np.random.default_rng(cfg.seed)
    n = cfg.n_cells if n_cells is None else n_cells
    mesh = cfg.mesh()
    if cfg.seeding == "sphere":
        pos = _sphere(rng, n, cfg.seed_radius)
    elif cfg.seeding == "radial":
        pos = _radial(rng, n, cfg.radial_scale, cfg.radial_cutoff)
    elif cfg.seeding == "box":
        lo, hi = np.asarray(mesh.origin), np.asarray(mesh.upper)
        pos = lo + rng.uniform(0.0, 1.0, size=(n, 3)) * (hi - lo)
    else:
        raise ValueError(cfg.seeding)
    pos = _clamp_inside(mesh, np.ascontiguousarray(pos, dtype=np.float64))
    if cfg.radius_sd > 0:
        rad = rng.normal(cfg.radius, cfg.radius_sd, n)
        if cfg.radius_clip:
            rad = np.clip(rad, *cfg.radius_clip)
    else:
        rad = np.full(n, cfg.radius)
    S = cfg.n_substrates
    sec = np.zeros((S, n))
    upt = np.zeros((S, n))
    lo, hi = cfg.uptake
    upt[0] = rng.uniform(lo, hi, n) if hi > lo else lo
    lo, hi = cfg.secretion
    for s in range(1, S):
        sec[s] = rng.uniform(lo, hi, n) if hi > lo else lo
    dens = np.repeat(np.asarray(cfg.dirichlet, np.float64)[:, None], cfg.voxel_count, axis=1)
    return Inputs(positions=np.ascontiguousarray(pos), radius=np.ascontiguousarray(rad),
                  ids=np.arange(n, dtype=np.int64), secretion=sec, uptake=upt,
                  densities=np.ascontiguousarray(dens))


def sorted_storage(cfg: SimConfig, inp: Inputs) -> Inputs:
    """The same cells in voxel-sorted storage: (voxel, id) order, as
    sort_cells_by_voxel leaves them (population.py:132-135; run_simulation
    sorts before its loop with the voxel_sorted strategy,
    simulate.py:156-158).  Ids travel with their cells."""
    mesh = cfg.mesh()
    o = np.asarray(mesh.origin)
    d = np.array([mesh.dx, mesh.dy, mesh.dz])
    ijk = np.floor((inp.positions - o) / d).astype(np.int64)
    vox = ijk[:, 0] + mesh.nx * (ijk[:, 1] + mesh.ny * ijk[:, 2])
    order = np.lexsort((inp.ids, vox))
    return Inputs(positions=np.ascontiguousarray(inp.positions[order]),
                  radius=np.ascontiguousarray(inp.radius[order]), ids=inp.ids[order].copy(),
                  secretion=np.ascontiguousarray(inp.secretion[:, order]),
                  uptake=np.ascontiguousarray(inp.uptake[:, order]), densities=inp.densities,
                  extra=dict(inp.extra))
