"""Generate tests/golden/*.npz by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py          # golden.npz
    python tests/golden/make_golden.py traj60   # traj60.npz (config 0, 60 steps)

It imports the reference package read-only from /root/reference/pkg/src and
calls its hot-path functions directly (lod_step, apply_cell_exchange,
rebin_cells, update_velocities, integrate_positions, compute_gradients,
_line_factors, CartesianMesh.voxel_of) on seeded inputs, and stores inputs +
outputs.  The
committed fixtures pin both the CPU oracle (tests/test_oracle_golden.py,
bit-for-bit) and the GPU path (tests/test_gpu_parity.py).

The G1/G2/G4 extensions have no reference implementation; the ``ext_*``
fixtures come from the small Python restatement below (``Ext``), which reuses
the reference's own _line_factors/_solve_rows and loop bodies and only adds
the extension.  Those fixtures are labelled "ext" and are "parity unpinned"
with respect to the reference.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True

import cellbench as cb  # noqa: E402  (the reference, read-only)
from cellbench.diffusion import _line_factors, _solve_rows  # noqa: E402

from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402


def mesh_arr(m):
    return np.array([m.nx, m.ny, m.nz, m.dx, m.dy, m.dz, *m.origin], dtype=np.float64)


def container_from(mesh, positions, radius, order=None):
    """Reference container with ids 0..n-1; `order` permutes storage."""
    cont = cb.CellContainer(mesh)
    for i, p in enumerate(positions):
        cont.new_cell([float(p[0]), float(p[1]), float(p[2])], radius=float(radius[i]))
    if order is not None:
        cont.cells = [cont.cells[k] for k in order]
    cb.rebin_cells(cont)
    return cont


def bins_of(cont):
    """agent as CSR over storage indices (storage order within each voxel)."""
    mesh = cont.mesh
    sidx = cont.storage_index
    counts = np.zeros(mesh.voxel_count + 1, np.int64)
    for v, ids in cont.agent.items():
        counts[v + 1] = len(ids)
    start = np.cumsum(counts).astype(np.int32)
    cells = np.zeros(len(cont.cells), np.int32)
    for v in sorted(cont.agent):
        for k, cid in enumerate(cont.agent[v]):
            cells[start[v] + k] = sidx[cid]
    voxel = np.array([c.voxel_index for c in cont.cells], np.int32)
    return start, cells, np.array(cont.nonempty_voxels, np.int32), voxel


def storage_arrays(cont):
    pos = np.array([c.position for c in cont.cells], np.float64).reshape(-1, 3)
    vel = np.array([c.velocity for c in cont.cells], np.float64).reshape(-1, 3)
    rad = np.array([c.radius for c in cont.cells], np.float64)
    ids = np.array([c.id for c in cont.cells], np.int64)
    return pos, vel, rad, ids


class Ext:
    """Extensions G1/G2/G4 restated on top of the reference's own pieces."""

    @staticmethod
    def dirichlet(micro, values):
        m = micro.mesh
        for s in range(micro.substrate_count):
            g = micro.grid_view(s)
            g[0, :, :] = values[s]
            g[-1, :, :] = values[s]
            g[:, 0, :] = values[s]
            g[:, -1, :] = values[s]
            g[:, :, 0] = values[s]
            g[:, :, -1] = values[s]

    @staticmethod
    def lod_step_dirichlet(micro, mesh, dt, values):
        """diffusion.py:127-192 with BioFVM Dirichlet pins around every sweep."""
        nx, ny, nz = mesh.nx, mesh.ny, mesh.nz
        for s in range(micro.substrate_count):
            lam3 = dt * micro.decay[s] / 3.0
            grid = micro.grid_view(s)
            one = [values[s]]

            def pin():
                grid[0, :, :] = one[0]
                grid[-1, :, :] = one[0]
                grid[:, 0, :] = one[0]
                grid[:, -1, :] = one[0]
                grid[:, :, 0] = one[0]
                grid[:, :, -1] = one[0]

            pin()
            rows = micro.densities[s].reshape(nz * ny, nx)
            r = dt * micro.diffusion[s] / (mesh.dx * mesh.dx)
            inv, gamma = _line_factors(nx, r, lam3)
            _solve_rows(rows, 0, nz * ny, inv, gamma, r)
            pin()
            r = dt * micro.diffusion[s] / (mesh.dy * mesh.dy)
            inv, gamma = _line_factors(ny, r, lam3)
            scratch = grid.transpose(0, 2, 1).copy().reshape(nz * nx, ny)
            _solve_rows(scratch, 0, nz * nx, inv, gamma, r)
            grid[:] = scratch.reshape(nz, nx, ny).transpose(0, 2, 1)
            pin()
            r = dt * micro.diffusion[s] / (mesh.dz * mesh.dz)
            inv, gamma = _line_factors(nz, r, lam3)
            scratch = grid.transpose(1, 2, 0).copy().reshape(ny * nx, nz)
            _solve_rows(scratch, 0, ny * nx, inv, gamma, r)
            grid[:] = scratch.reshape(ny, nx, nz).transpose(2, 0, 1)
            pin()

    @staticmethod
    def exchange_cells(micro, cont, dt, sec, upt, sat):
        """diffusion.py:219-229 with per-cell rates sec[s][id], upt[s][id]."""
        inv_vol = 1.0 / micro.mesh.voxel_volume
        for s in range(micro.substrate_count):
            dens = micro.densities[s]
            for v in cont.nonempty_voxels:
                rho = dens[v]
                for cid in sorted(cont.agent[v]):
                    f = dt * cont.by_id[cid].volume * inv_vol
                    se, up = float(sec[s][cid]), float(upt[s][cid])
                    den = 1.0 + f * (se + up)
                    rho = (rho + f * se * float(sat[s])) / den
                dens[v] = rho

    @staticmethod
    def integrate_ab2(cont, mesh, dt, prev):
        """PhysiCell Cell::update_position: x += 1.5dt v - 0.5dt v_prev."""
        d1 = dt * 1.5
        d2 = dt * -0.5
        for c in cont.cells:
            p, v, pv = c.position, c.velocity, prev[c.id]
            for k in range(3):
                p[k] += d1 * v[k] + d2 * pv[k]
                pv[k] = v[k]
            if not mesh.contains(p):
                mesh.clamp_inside(p)
        cont.positions_dirty = True


def gen_line_factors(out):
    cases = [(1, 0.0, 0.0), (1, 2.5, 0.01), (2, 2.5, 0.003), (5, 0.25, 0.0333),
             (20, 2.5, 3.3333333333333335e-4), (80, 2.5, 3.3333333333333335e-4),
             (80, 0.025, 3.333e-5), (160, 1.6, 8.53e-05), (7, 1e5, 0.7)]
    for k, (n, r, lam3) in enumerate(cases):
        inv, gam = _line_factors(n, r, lam3)
        out[f"lf{k}_args"] = np.array([n, r, lam3])
        out[f"lf{k}_inv"] = inv
        out[f"lf{k}_gamma"] = gam


def gen_voxel_of(out):
    rng = np.random.default_rng(11)
    meshes = [cb.CartesianMesh(75, 75, 75), cb.CartesianMesh(20, 20, 20, origin=(-200.0,) * 3),
              cb.CartesianMesh(7, 5, 3, dx=0.1, dy=0.3, dz=0.7),
              cb.CartesianMesh(6, 5, 4, 10.0, 20.0, 30.0, origin=(-30.0, 10.0, -50.0))]
    for k, m in enumerate(meshes):
        lo, hi = np.array(m.origin), np.array(m.upper)
        pts = [lo + rng.uniform(0, 1, 3) * (hi - lo) for _ in range(300)]
        d = np.array([m.dx, m.dy, m.dz])
        for _ in range(300):  # exact and near faces
            i = rng.integers(-1, np.array([m.nx, m.ny, m.nz]) + 2)
            p = lo + i * d
            p = p + rng.choice([0.0, 1e-12, -1e-12, 1e-9, -1e-9, 5e-324], 3) * np.maximum(1, np.abs(p))
            pts.append(p)
        pts.append(np.array([30.0, 30.0, 30.0]))
        pts = np.array(pts)
        res = []
        for p in pts:
            try:
                res.append(m.voxel_of(tuple(float(x) for x in p)))
            except cb.DomainError:
                res.append(-1)
        out[f"vo{k}_mesh"] = mesh_arr(m)
        out[f"vo{k}_pts"] = pts
        out[f"vo{k}_voxel"] = np.array(res, np.int64)


def random_field(mesh, S, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 50.0, (S, mesh.voxel_count))


def gen_lod(out):
    pool = cb.WorkerPool(2)
    cases = [
        (cb.CartesianMesh(3, 4, 5), [1000.0], [0.1], 0.1, 5),
        (cb.CartesianMesh(1, 4, 4), [70000.0], [0.0], 0.1, 20),
        (cb.CartesianMesh(6, 5, 4), [90000.0], [0.4], 0.1, 5),
        (cb.CartesianMesh(8, 8, 8), [1e5, 1e3], [0.1, 0.01], 0.01, 10),
        (cb.CartesianMesh(20, 20, 20, origin=(-200.0,) * 3), [1e5], [0.1], 0.01, 10),
        (cb.CartesianMesh(33, 17, 9, 10.0, 20.0, 30.0), [6.4e4, 5e4, 0.0], [0.0256, 0.05, 2.0], 0.01, 3),
    ]
    for k, (m, D, K, dt, steps) in enumerate(cases):
        micro = cb.Microenvironment(m, D, K)
        micro.densities[:] = random_field(m, len(D), 100 + k)
        out[f"lod{k}_mesh"] = mesh_arr(m)
        out[f"lod{k}_in"] = micro.densities.copy()
        out[f"lod{k}_D"] = np.array(D)
        out[f"lod{k}_K"] = np.array(K)
        out[f"lod{k}_dt_steps"] = np.array([dt, steps])
        mode = cb.TraversalMode.OUTER_LOOP if k % 2 else cb.TraversalMode.COLLAPSED
        for _ in range(steps):
            cb.lod_step(micro, m, dt, mode, pool)
        out[f"lod{k}_out"] = micro.densities.copy()
        # G1 extension fixture (restated): same inputs, Dirichlet pins.
        micro2 = cb.Microenvironment(m, D, K)
        micro2.densities[:] = out[f"lod{k}_in"]
        vals = [38.0] + [0.0] * (len(D) - 1)
        for _ in range(steps):
            Ext.lod_step_dirichlet(micro2, m, dt, vals)
        out[f"ext_lod{k}_dirichlet"] = np.array(vals)
        out[f"ext_lod{k}_out"] = micro2.densities.copy()
    pool.shutdown()


def gen_gradients(out):
    """compute_gradients (diffusion.py:237-278) on meshes with degenerate axes,
    anisotropic spacing and several substrates, both traversal modes."""
    pool = cb.WorkerPool(2)
    cases = [
        (cb.CartesianMesh(3, 4, 5), 1),
        (cb.CartesianMesh(1, 4, 4), 1),
        (cb.CartesianMesh(2, 3, 4), 2),
        (cb.CartesianMesh(20, 20, 20, origin=(-200.0,) * 3), 2),
        (cb.CartesianMesh(33, 17, 9, 10.0, 20.0, 30.0), 3),
    ]
    for k, (m, S) in enumerate(cases):
        micro = cb.Microenvironment(m, [1e3] * S, [0.1] * S)
        micro.densities[:] = random_field(m, S, 500 + k)
        mode = cb.TraversalMode.OUTER_LOOP if k % 2 else cb.TraversalMode.COLLAPSED
        cb.compute_gradients(micro, m, mode, pool)
        out[f"grad{k}_mesh"] = mesh_arr(m)
        out[f"grad{k}_in"] = micro.densities.copy()
        out[f"grad{k}_out"] = micro.gradients.copy()
    pool.shutdown()


def gen_rebin(out):
    rng = np.random.default_rng(21)
    cases = [
        (cb.CartesianMesh(6, 5, 4, 10.0, 20.0, 30.0, origin=(-30.0, 10.0, -50.0)), 300),
        (cb.CartesianMesh(4, 4, 4), 40),
        (cb.CartesianMesh(20, 20, 20, origin=(-200.0,) * 3), 2000),
    ]
    for k, (m, n) in enumerate(cases):
        lo, hi = np.array(m.origin), np.array(m.upper)
        pos = lo + rng.uniform(0, 1, (n, 3)) * (hi - lo)
        pos[: n // 10] = np.round(pos[: n // 10] / 10.0) * 10.0  # on voxel faces
        pos = np.minimum(np.maximum(pos, lo + 1e-6), hi - 1e-6)
        order = rng.permutation(n)
        cont = container_from(m, pos, np.full(n, 8.0), order)
        start, cells, ne, voxel = bins_of(cont)
        p, _, _, ids = storage_arrays(cont)
        out[f"rb{k}_mesh"] = mesh_arr(m)
        out[f"rb{k}_pos"] = p
        out[f"rb{k}_ids"] = ids
        out[f"rb{k}_bin_start"] = start
        out[f"rb{k}_bin_cells"] = cells
        out[f"rb{k}_nonempty"] = ne
        out[f"rb{k}_voxel"] = voxel


def gen_exchange(out):
    rng = np.random.default_rng(31)
    m = cb.CartesianMesh(20, 20, 20, origin=(-200.0,) * 3)
    inp = make_inputs(CONFIGS[0], 600)
    rad = rng.uniform(6.0, 10.0, 600)
    order = rng.permutation(600)
    cont = container_from(m, inp.positions, rad, order)
    micro = cb.Microenvironment(m, [1e5, 1e3], [0.1, 0.01])
    micro.densities[:] = random_field(m, 2, 41)
    p, _, r, ids = storage_arrays(cont)
    out["ex_mesh"] = mesh_arr(m)
    out["ex_pos"] = p
    out["ex_radius"] = r
    out["ex_ids"] = ids
    out["ex_in"] = micro.densities.copy()
    for k, (dt, sec, upt, sat, s) in enumerate([(0.02, 2.0, 3.0, 38.0, 0), (0.01, 0.0, 10.0, 38.0, 1),
                                                (0.05, 4.2, 0.0, 38.0, 0)]):
        cb.apply_cell_exchange(micro, cont, dt, sec, upt, sat, substrate=s)
        out[f"ex{k}_args"] = np.array([dt, sec, upt, sat, s])
        out[f"ex{k}_out"] = micro.densities.copy()
    # G4 extension (restated): per-cell rates on both substrates.
    micro2 = cb.Microenvironment(m, [1e5, 1e3], [0.1, 0.01])
    micro2.densities[:] = out["ex_in"]
    sec = np.stack([np.zeros(600), rng.uniform(0, 1, 600)])
    upt = np.stack([rng.uniform(5, 15, 600), np.zeros(600)])
    Ext.exchange_cells(micro2, cont, 0.01, sec, upt, [38.0, 38.0])
    out["ext_ex_sec"] = sec  # indexed by id
    out["ext_ex_upt"] = upt
    out["ext_ex_out"] = micro2.densities.copy()


def gen_velocities(out):
    params = cb.InteractionParams()
    pool = cb.WorkerPool(1)
    sched = cb.MechanicsSchedule.cell_static()
    rng = np.random.default_rng(51)
    # (a) the reference test's clustered blob (test_mechanics.py:111-117)
    m4 = cb.CartesianMesh(4, 4, 4)
    posa = []
    for i in range(40):
        u1, u2, u3 = cb.division_draws(2, i, 0)
        posa.append((10.0 + 50.0 * u1, 10.0 + 50.0 * u2, 10.0 + 50.0 * u3))
    # (b) config 0 seeding; (c) dense, random radii, shuffled storage
    m0 = cb.CartesianMesh(20, 20, 20, origin=(-200.0,) * 3)
    inp = make_inputs(CONFIGS[0])
    m6 = cb.CartesianMesh(6, 6, 6)
    posc = rng.uniform(1.0, 119.0, (700, 3))
    cases = [(m4, np.array(posa), np.full(40, 8.0), None),
             (m0, inp.positions, inp.radius, None),
             (m6, posc, rng.uniform(7.0, 10.0, 700), rng.permutation(700))]
    for k, (m, pos, rad, order) in enumerate(cases):
        cont = container_from(m, pos, rad, order)
        cb.update_velocities(cont, m, params, sched, pool)
        p, v, r, ids = storage_arrays(cont)
        out[f"ve{k}_mesh"] = mesh_arr(m)
        out[f"ve{k}_pos"] = p
        out[f"ve{k}_radius"] = r
        out[f"ve{k}_ids"] = ids
        out[f"ve{k}_vel"] = v
    pool.shutdown()


def gen_integrate(out):
    rng = np.random.default_rng(61)
    m = cb.CartesianMesh(6, 5, 4, 10.0, 20.0, 30.0, origin=(-30.0, 10.0, -50.0))
    lo, hi = np.array(m.origin), np.array(m.upper)
    n = 400
    pos = lo + rng.uniform(0, 1, (n, 3)) * (hi - lo)
    vel = rng.normal(0, 3.0, (n, 3))
    vel[:40] *= 1e4  # pushed through faces -> all-axis clamp
    pv = rng.normal(0, 3.0, (n, 3))
    pool = cb.WorkerPool(1)
    for k, dt in enumerate([0.1, 1.0]):
        cont = container_from(m, pos, np.full(n, 8.0))
        for c in cont.cells:
            c.velocity[:] = vel[c.id].tolist()
        cb.integrate_positions(cont, m, dt, pool)
        p, _, _, _ = storage_arrays(cont)
        out[f"in{k}_mesh"] = mesh_arr(m)
        out[f"in{k}_pos0"] = pos
        out[f"in{k}_vel"] = vel
        out[f"in{k}_dt"] = np.array([dt])
        out[f"in{k}_pos"] = p
        # G2 (restated)
        cont2 = container_from(m, pos, np.full(n, 8.0))
        for c in cont2.cells:
            c.velocity[:] = vel[c.id].tolist()
        prev = {i: list(pv[i]) for i in range(n)}
        Ext.integrate_ab2(cont2, m, dt, prev)
        p2, _, _, _ = storage_arrays(cont2)
        out[f"ext_in{k}_prev"] = pv
        out[f"ext_in{k}_pos"] = p2
        out[f"ext_in{k}_prev_out"] = np.array([prev[i] for i in range(n)])
    pool.shutdown()


def gen_trajectory(out, steps=5):
    """Config 0 run with the reference's functions in run_simulation order.

    "ref": Neumann, Euler, scalar uptake 10 on s0 (what the reference does).
    "ext": config 0 as BASELINE.json states it (Dirichlet 38, AB2, per-cell
    rates) through the Ext restatement."""
    cfg = CONFIGS[0]
    inp = make_inputs(cfg)
    m = cfg.mesh()
    params = cb.InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier)
    pool = cb.WorkerPool(1)
    sched = cb.MechanicsSchedule.nonempty_voxel(16)
    for tag in ("ref", "ext"):
        micro = cb.Microenvironment(m, list(cfg.diffusion), list(cfg.decay), list(cfg.dirichlet))
        cont = container_from(m, inp.positions, inp.radius)
        prev = {i: [0.0, 0.0, 0.0] for i in range(cfg.n_cells)}
        sums, dsum = [], []
        for step in range(steps):
            for _ in range(cfg.substeps):
                if tag == "ref":
                    cb.apply_cell_exchange(micro, cont, cfg.dt_diffusion, 0.0, 10.0,
                                           cfg.saturation, pool=pool)
                    cb.lod_step(micro, m, cfg.dt_diffusion, cb.TraversalMode.OUTER_LOOP, pool,
                                container=cont)
                else:
                    Ext.exchange_cells(micro, cont, cfg.dt_diffusion, inp.secretion, inp.uptake,
                                       [cfg.saturation])
                    Ext.lod_step_dirichlet(micro, m, cfg.dt_diffusion, list(cfg.dirichlet))
            cb.update_velocities(cont, m, params, sched, pool)
            if tag == "ref":
                cb.integrate_positions(cont, m, cfg.dt_mechanics, pool)
            else:
                Ext.integrate_ab2(cont, m, cfg.dt_mechanics, prev)
            cb.rebin_cells(cont)
            sums.append(cb.state_checksum(cont))
            dsum.append(hashlib.sha256(micro.densities.tobytes()).hexdigest())
        p, v, _, _ = storage_arrays(cont)
        out[f"{tag}_traj_dens"] = micro.densities.copy()
        out[f"{tag}_traj_pos"] = p
        out[f"{tag}_traj_vel"] = v
        out[f"{tag}_traj_checksums"] = np.array(sums)
        out[f"{tag}_traj_dens_sha"] = np.array(dsum)
    pool.shutdown()


def gen_trajectory_long(path, steps=60):
    """Config 0's whole run (60 mechanics steps = 6 sim-min) with the
    reference's functions in run_simulation order, for both the reference's
    own semantics ("ref": Neumann, Euler, scalar uptake 10 on s0) and config 0
    as BASELINE.json states it ("ext": Dirichlet 38, AB2, per-cell rates via
    Ext).  Stored per step: every cell's voxel (storage order = id order),
    the state_checksum and a SHA-256 of the field; every 10 steps positions
    and velocities; at the end the field.  Written to its own file
    (tests/golden/traj60.npz)."""
    cfg = CONFIGS[0]
    inp = make_inputs(cfg)
    m = cfg.mesh()
    params = cb.InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier)
    pool = cb.WorkerPool(1)
    sched = cb.MechanicsSchedule.nonempty_voxel(16)
    out = {}
    for tag in ("ref", "ext"):
        micro = cb.Microenvironment(m, list(cfg.diffusion), list(cfg.decay), list(cfg.dirichlet))
        cont = container_from(m, inp.positions, inp.radius)
        prev = {i: [0.0, 0.0, 0.0] for i in range(cfg.n_cells)}
        vox, sums, dsha, pos_k, vel_k = [], [], [], [], []
        for step in range(steps):
            for _ in range(cfg.substeps):
                if tag == "ref":
                    cb.apply_cell_exchange(micro, cont, cfg.dt_diffusion, 0.0, 10.0,
                                           cfg.saturation, pool=pool)
                    cb.lod_step(micro, m, cfg.dt_diffusion, cb.TraversalMode.OUTER_LOOP, pool,
                                container=cont)
                else:
                    Ext.exchange_cells(micro, cont, cfg.dt_diffusion, inp.secretion, inp.uptake,
                                       [cfg.saturation])
                    Ext.lod_step_dirichlet(micro, m, cfg.dt_diffusion, list(cfg.dirichlet))
            cb.update_velocities(cont, m, params, sched, pool)
            if tag == "ref":
                cb.integrate_positions(cont, m, cfg.dt_mechanics, pool)
            else:
                Ext.integrate_ab2(cont, m, cfg.dt_mechanics, prev)
            cb.rebin_cells(cont)
            micro.check_state()
            vox.append(np.array([c.voxel_index for c in cont.cells], np.int16))
            sums.append(cb.state_checksum(cont))
            dsha.append(hashlib.sha256(micro.densities.tobytes()).hexdigest())
            if (step + 1) % 10 == 0:
                p, v, _, _ = storage_arrays(cont)
                pos_k.append(p)
                vel_k.append(v)
        out[f"{tag}_voxel"] = np.array(vox)
        out[f"{tag}_checksums"] = np.array(sums)
        out[f"{tag}_dens_sha"] = np.array(dsha)
        out[f"{tag}_pos10"] = np.array(pos_k)
        out[f"{tag}_vel10"] = np.array(vel_k)
        out[f"{tag}_dens"] = micro.densities.copy()
    pool.shutdown()
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


def gen_divisions(out):
    """division_draws (population.py:41-48) on a spread of (seed, id, step), and
    attempt_divisions (population.py:72-128) on containers with per-cell
    rates, several steps (daughters divide again), shuffled storage order and
    cells near the faces (clamping).  Stores, per case and step, the cells'
    (id, position, radius, rate) before the call and the daughters' ids,
    parent ids and positions after it."""
    rng = np.random.default_rng(77)
    seeds = np.array([0, 1, 42, 123, 2**63, 2**64 - 1, 987654321987], dtype=np.uint64)
    trip = []
    for sd in seeds:
        for cid in (0, 1, 7, 999, 10**6):
            for st in (0, 3, 17, 10**6):
                trip.append((int(sd), cid, st, *cb.division_draws(int(sd), cid, st)))
    out["div_draws"] = np.array([t[3:] for t in trip])
    out["div_draws_seed"] = np.array([t[0] for t in trip], dtype=np.uint64)
    out["div_draws_id_step"] = np.array([t[1:3] for t in trip], dtype=np.int64)
    cases = [
        # mesh, n cells, rate range, dt, seed, steps, near-face
        (cb.CartesianMesh(4, 4, 4), 6, (50.0, 50.0), 1.0, 1, 1, False),
        (cb.CartesianMesh(4, 4, 4), 6, (0.2, 0.2), 0.5, 123, 1, False),
        (cb.CartesianMesh(6, 5, 4, 20.0, 20.0, 20.0, (-60.0, -50.0, -40.0)), 120, (0.0, 3.0), 0.4,
         7, 4, False),
        (cb.CartesianMesh(4, 4, 4), 40, (2.0, 6.0), 0.5, 3, 3, True),
    ]
    for k, (mesh, n, (r0, r1), dt, seed, steps, near) in enumerate(cases):
        lo = np.array(mesh.origin)
        hi = lo + np.array([mesh.nx * mesh.dx, mesh.ny * mesh.dy, mesh.nz * mesh.dz])
        if near:
            pos = hi - rng.uniform(0.0, 3.0, (n, 3))
            pos[::2] = lo + rng.uniform(0.0, 3.0, (len(pos[::2]), 3))
        else:
            pos = rng.uniform(lo + 5.0, hi - 5.0, (n, 3))
        rad = rng.uniform(6.0, 9.0, n)
        rates = rng.uniform(r0, r1, n) if r1 > r0 else np.full(n, r0)
        cont = cb.CellContainer(mesh)
        for i in range(n):
            c = cont.new_cell([float(x) for x in pos[i]], radius=float(rad[i]),
                              division_rate=float(rates[i]))
            c.velocity[:] = [float(x) for x in rng.normal(0.0, 1.0, 3)]
        order = rng.permutation(n)
        cont.cells = [cont.cells[j] for j in order]
        cb.rebin_cells(cont)
        out[f"div{k}_mesh"] = mesh_arr(mesh)
        out[f"div{k}_args"] = np.array([dt, seed, steps], dtype=np.float64)
        for st in range(steps):
            cells = cont.cells
            out[f"div{k}_s{st}_ids"] = np.array([c.id for c in cells], np.int64)
            out[f"div{k}_s{st}_pos"] = np.array([c.position for c in cells])
            out[f"div{k}_s{st}_radius"] = np.array([c.radius for c in cells])
            out[f"div{k}_s{st}_rate"] = np.array([c.division_rate for c in cells])
            before = {c.id for c in cells}
            daughters = cb.attempt_divisions(cont, seed=seed, dt=dt, mesh=mesh, step=st, cap=10**6)
            out[f"div{k}_s{st}_d_ids"] = np.array([d.id for d in daughters], np.int64)
            out[f"div{k}_s{st}_d_pos"] = np.array([d.position for d in daughters]).reshape(-1, 3)
            # parents: the dividers in ascending id (population.py:91)
            par = sorted(c.id for c in cells[: len(before)]
                         if c.division_rate > 0.0 and cb.division_draws(seed, c.id, st)[0]
                         < 1.0 - math.exp(-c.division_rate * dt))
            out[f"div{k}_s{st}_parents"] = np.array(par, np.int64)


def main():
    out = {}
    gen_line_factors(out)
    gen_voxel_of(out)
    gen_lod(out)
    gen_gradients(out)
    gen_rebin(out)
    gen_exchange(out)
    gen_velocities(out)
    gen_integrate(out)
    gen_trajectory(out)
    gen_divisions(out)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "traj60":
        gen_trajectory_long(os.path.join(HERE, "traj60.npz"))
    else:
        main()
