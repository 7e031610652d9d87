"""The z-slab decomposition on the GPU: P ranks (processes) share cuda:0 and
talk through gloo with host staging -- no kernel waits on another rank's
kernel.  Against the single-GPU engine on the same inputs: cells (ids,
positions, velocities) bit-for-bit, fields within 1e-12 normwise (the
partitioned z sweep rounds differently; the bar is 1e-10)."""

import numpy as np
import pytest

import _dist_util

pytestmark = pytest.mark.gpu


def _slab_run(rank, world, cfg_key, n_cells, steps, bounds=None, numerics="exact"):
    import torch
    import torch.distributed as dist

    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.distributed import Comm, build

    torch.cuda.set_device(0)
    cfg = CONFIGS[cfg_key]
    inp = make_inputs(cfg, n_cells)
    sim = build(cfg, Comm(dist, "cuda:0"), inp, bounds, numerics=numerics)
    assert sim.fast == (numerics == "fast")
    for _ in range(steps):
        sim.step()
    ids, pos, vel = sim.owned_state()
    return sim.z0, sim.z1, ids, pos, vel, sim.densities()


def _single(cfg_key, n_cells, steps, numerics="exact"):
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[cfg_key]
    sim = Simulation.from_config(cfg, make_inputs(cfg, n_cells), numerics=numerics)
    sim.run(steps, graph=False)
    sim.sync()
    out = sim.positions(), sim.velocities(), sim.densities()
    sim.close()
    return cfg, out


@pytest.mark.parametrize("world", [1, 2, 3])
def test_slabs_match_single_gpu(tmp_path, world):
    cfg_key, n_cells, steps = 0, 2000, 3
    cfg, (pos1, vel1, dens1) = _single(cfg_key, n_cells, steps)
    if world == 1:
        import torch  # noqa: F401

        from paper_2306_11544_b200.configs import make_inputs
        from paper_2306_11544_b200.distributed import Comm, build

        sim = build(cfg, Comm(None, "cuda:0"), make_inputs(cfg, n_cells))
        for _ in range(steps):
            sim.step()
        ids, pos, vel = sim.owned_state()
        assert np.array_equal(ids, np.arange(n_cells))
        assert np.array_equal(pos, pos1) and np.array_equal(vel, vel1)
        assert np.array_equal(sim.densities(), dens1)
        return
    res = _dist_util.run(world, _slab_run, (cfg_key, n_cells, steps), tmp_path)
    ids = np.concatenate([r[2] for r in res])
    pos = np.concatenate([r[3] for r in res])
    vel = np.concatenate([r[4] for r in res])
    o = np.argsort(ids)
    assert np.array_equal(ids[o], np.arange(n_cells)), "every cell owned exactly once"
    assert np.array_equal(pos[o], pos1)
    assert np.array_equal(vel[o], vel1)
    S, plane = cfg.n_substrates, cfg.nx * cfg.ny
    dens = np.concatenate([r[5].reshape(S, -1, plane) for r in res], axis=1).reshape(S, -1)
    err = np.max(np.abs(dens - dens1)) / np.max(np.abs(dens1))
    assert err <= 1e-12, err


@pytest.mark.parametrize("bounds", [[(0, 7), (7, 20)], [(0, 9), (9, 10), (10, 20)], "balanced"])
def test_uneven_slabs_match_single_gpu(tmp_path, bounds):
    """Non-uniform (load-balanced) slabs, a 1-plane slab included: same bar."""
    cfg_key, n_cells, steps = 0, 2000, 3
    cfg, (pos1, vel1, dens1) = _single(cfg_key, n_cells, steps)
    if bounds == "balanced":
        from paper_2306_11544_b200.configs import make_inputs
        from paper_2306_11544_b200.distributed import load_balanced_bounds

        bounds = load_balanced_bounds(cfg, make_inputs(cfg, n_cells), 3)
        assert bounds != [(0, 7), (7, 14), (14, 20)], "cells concentrate mid-box"
    world = len(bounds)
    res = _dist_util.run(world, _slab_run, (cfg_key, n_cells, steps, bounds), tmp_path)
    ids = np.concatenate([r[2] for r in res])
    o = np.argsort(ids)
    assert np.array_equal(ids[o], np.arange(n_cells))
    assert np.array_equal(np.concatenate([r[3] for r in res])[o], pos1)
    assert np.array_equal(np.concatenate([r[4] for r in res])[o], vel1)
    S, plane = cfg.n_substrates, cfg.nx * cfg.ny
    dens = np.concatenate([r[5].reshape(S, -1, plane) for r in res], axis=1).reshape(S, -1)
    assert np.max(np.abs(dens - dens1)) / np.max(np.abs(dens1)) <= 1e-12


def _slab_gradients(rank, world, cfg_key, n_cells, steps):
    import torch
    import torch.distributed as dist

    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.distributed import Comm, build

    torch.cuda.set_device(0)
    cfg = CONFIGS[cfg_key]
    sim = build(cfg, Comm(dist, "cuda:0"), make_inputs(cfg, n_cells))
    for _ in range(steps):
        sim.step()
    g = sim.gradients()
    sim.sync()
    return sim.z0, sim.z1, sim.densities(), g.cpu().numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_gradients_with_halo(tmp_path, world):
    """diffusion.py:237-278 on z-slabs: the one-plane halo makes every slab's
    gradients equal, bit for bit, to those of the gathered field computed on
    one GPU (zero normal component on the global faces only)."""
    import torch

    from paper_2306_11544_b200 import _lib
    from paper_2306_11544_b200.configs import CONFIGS

    cfg_key, n_cells, steps = 0, 2000, 2
    cfg = CONFIGS[cfg_key]
    res = _dist_util.run(world, _slab_gradients, (cfg_key, n_cells, steps), tmp_path)
    S, plane = cfg.n_substrates, cfg.nx * cfg.ny
    dens = np.concatenate([r[2].reshape(S, -1, plane) for r in res], axis=1).reshape(S, -1)
    grads = np.concatenate([r[3].reshape(S, -1, plane, 3) for r in res], axis=1)
    ctx = _lib.Context(cfg.mesh(), S, 1, 0)
    d = torch.from_numpy(dens).cuda()
    g = torch.empty((S, dens.shape[1], 3), dtype=torch.float64, device="cuda")
    _lib.raise_for(_lib.load().cg_gradients(ctx.handle, _lib.ptr(d), _lib.ptr(g)), "gradients")
    ctx.sync("gradients")
    want = g.cpu().numpy().reshape(S, -1, plane, 3)
    assert np.array_equal(grads, want)
    ctx.close()


# ---- the kernel combinations the scaling bench runs

FIELD_TOL = 1e-10  # BASELINE.json: fp64 fields within 1e-10 per step


def _field_err(got, want, S):
    g, w = got.reshape(S, -1), want.reshape(S, -1)
    return max(float(np.max(np.abs(g[s] - w[s])) / max(np.max(np.abs(w[s])), 1e-300)) for s in range(S))


def _c4_rank_inputs(rank, world, n_cells):
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs, slab_config

    cfg = CONFIGS[4]
    return cfg, make_inputs(slab_config(cfg, rank, world), n_cells)


def _c4_global_mesh(cfg, world):
    from dataclasses import replace

    return replace(cfg.mesh(), nz=cfg.nz * world, origin=(cfg.origin[0], cfg.origin[1], -320.0 * world))


def _c4_slab_run(rank, world, n_cells, steps, numerics="exact"):
    import torch
    import torch.distributed as dist

    from paper_2306_11544_b200.distributed import Comm, SlabSimulation
    from paper_2306_11544_b200.mechanics import InteractionParams

    torch.cuda.set_device(0)
    cfg, inp = _c4_rank_inputs(rank, world, n_cells)
    sim = SlabSimulation(
        _c4_global_mesh(cfg, world), Comm(dist, "cuda:0"), diffusion=cfg.diffusion,
        decay=cfg.decay, densities=inp.densities, positions=inp.positions, radius=inp.radius,
        ids=inp.ids + rank * n_cells, secretion=inp.secretion, uptake=inp.uptake,
        saturation=cfg.saturation, bc=cfg.bc, dirichlet=cfg.dirichlet,
        params=InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier),
        dt_diffusion=cfg.dt_diffusion, dt_mechanics=cfg.dt_mechanics, integrator=cfg.integrator,
        numerics=numerics)
    assert sim.fast == (numerics == "fast")
    for _ in range(steps):
        sim.step()
    ids, pos, vel = sim.owned_state()
    return sim.z0, sim.z1, ids, pos, vel, sim.densities()


@pytest.mark.parametrize("world,numerics", [(2, "exact"), (4, "exact"), (2, "fast"), (4, "fast")])
def test_config4_weak_scaling_slabs_match_single_gpu(tmp_path, world, numerics):
    """BASELINE config 4's geometry as the weak-scaling bench runs it: every
    rank a 256 x 256 x 32 slab x 4 substrates (x rows + streaming y columns +
    the 32-plane register z kernel in slab mode + the interface correction;
    ghosts and migration every step), its own cells (seed 4 + rank, 60k per
    rank to keep the test short).  Against one GPU running the gathered
    256 x 256 x 32P box: cells bit for bit, fields within 1e-10.  Fast
    numerics: the slabs' fast x rows (affine exchange fused), y columns and
    velocities (cg_*_fast) against the single-GPU engine's fast kernels."""
    from paper_2306_11544_b200.engine import Simulation
    from paper_2306_11544_b200.mechanics import InteractionParams

    n_cells, steps = 60000, 2
    res = _dist_util.run(world, _c4_slab_run, (n_cells, steps, numerics), tmp_path)
    parts = [_c4_rank_inputs(r, world, n_cells) for r in range(world)]
    cfg = parts[0][0]
    S, plane = cfg.n_substrates, cfg.nx * cfg.ny
    dens0 = np.concatenate([p.densities.reshape(S, -1, plane) for _, p in parts], axis=1).reshape(S, -1)
    sim = Simulation(
        _c4_global_mesh(cfg, world), diffusion=cfg.diffusion, decay=cfg.decay, densities=dens0,
        positions=np.concatenate([p.positions for _, p in parts]),
        radius=np.concatenate([p.radius for _, p in parts]),
        ids=np.concatenate([p.ids + r * n_cells for r, (_, p) in enumerate(parts)]),
        secretion=np.concatenate([p.secretion for _, p in parts], axis=1),
        uptake=np.concatenate([p.uptake for _, p in parts], axis=1), saturation=cfg.saturation,
        bc=cfg.bc, dirichlet=cfg.dirichlet,
        params=InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier),
        dt_diffusion=cfg.dt_diffusion, dt_mechanics=cfg.dt_mechanics, integrator=cfg.integrator,
        numerics=numerics)
    sim.run(steps, graph=False)
    sim.sync()
    pos1, vel1, dens1 = sim.positions(), sim.velocities(), sim.densities()
    sim.close()
    ids = np.concatenate([r[2] for r in res])
    o = np.argsort(ids)
    assert np.array_equal(ids[o], np.arange(world * n_cells)), "every cell owned exactly once"
    assert np.array_equal(np.concatenate([r[3] for r in res])[o], pos1)
    assert np.array_equal(np.concatenate([r[4] for r in res])[o], vel1)
    dens = np.concatenate([r[5].reshape(S, -1, plane) for r in res], axis=1).reshape(S, -1)
    assert _field_err(dens, dens1, S) <= FIELD_TOL


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_config2_load_balanced_three_slabs_match_single_gpu(tmp_path, monkeypatch, numerics):
    """Config 2's dense spheroid (200k cells, the over-capacity voxel kernels)
    split over 3 ranks with load_balanced_bounds (middle rank gets fewer
    planes): same bar as the balanced split.  Fast numerics: the segmented
    80 x 80 plane kernel (affine exchange fused) on every slab, the exact
    slab z block solve + interface correction, the fast velocities."""
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.distributed import load_balanced_bounds

    cfg_key, n_cells, steps = 2, None, 2
    # the slabs' velocities are the per-cell kernel's (cg_velocities_fast); the
    # engine would pick four lanes per cell for this dense spheroid
    monkeypatch.setenv("CELLGPU_VEL_KERNEL", "cell")
    cfg, (pos1, vel1, dens1) = _single(cfg_key, n_cells, steps, numerics)
    bounds = load_balanced_bounds(cfg, make_inputs(cfg), 3)
    sizes = [b - a for a, b in bounds]
    assert sizes[1] < sizes[0] and sizes[1] < sizes[2], bounds
    res = _dist_util.run(3, _slab_run, (cfg_key, n_cells, steps, bounds, numerics), tmp_path)
    ids = np.concatenate([r[2] for r in res])
    o = np.argsort(ids)
    assert np.array_equal(ids[o], np.arange(cfg.n_cells))
    assert np.array_equal(np.concatenate([r[3] for r in res])[o], pos1)
    assert np.array_equal(np.concatenate([r[4] for r in res])[o], vel1)
    S, plane = cfg.n_substrates, cfg.nx * cfg.ny
    dens = np.concatenate([r[5].reshape(S, -1, plane) for r in res], axis=1).reshape(S, -1)
    assert _field_err(dens, dens1, S) <= FIELD_TOL


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_config3_strong_split_two_slabs_match_single_gpu(tmp_path, numerics):
    """Config 3 (160^3 x 4 substrates, 1M cells) strong-split over 2 ranks:
    80-plane slabs of 160 x 160 (exact: the streaming plane kernel with the
    whole plane in shared memory, streaming z columns in slab mode; fast: the
    segmented 160 x 160 plane kernel with the affine exchange fused and the
    same slab z solve) against the single-GPU engine in the same numerics:
    cells bit for bit, fields within 1e-10."""
    cfg_key, n_cells, steps = 3, None, 2
    cfg, (pos1, vel1, dens1) = _single(cfg_key, n_cells, steps, numerics)
    res = _dist_util.run(2, _slab_run, (cfg_key, n_cells, steps, None, numerics), tmp_path)
    ids = np.concatenate([r[2] for r in res])
    o = np.argsort(ids)
    assert np.array_equal(ids[o], np.arange(cfg.n_cells))
    assert np.array_equal(np.concatenate([r[3] for r in res])[o], pos1)
    assert np.array_equal(np.concatenate([r[4] for r in res])[o], vel1)
    S, plane = cfg.n_substrates, cfg.nx * cfg.ny
    dens = np.concatenate([r[5].reshape(S, -1, plane) for r in res], axis=1).reshape(S, -1)
    assert _field_err(dens, dens1, S) <= FIELD_TOL


def _slab_iface_run(rank, world, cfg_key, n_cells, steps, mode):
    import os

    os.environ["CELLGPU_SLAB_IFACE"] = mode
    return _slab_run(rank, world, cfg_key, n_cells, steps)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_interface_blocks_match_all_gather(tmp_path, world):
    """The interface system by line blocks (two all-to-alls, each rank
    solving the reduced systems of its own nx*ny / P lines) against the
    all-gather + redundant solve: fields and cells bit for bit (config 0
    split 2, 3 and 4 ways; 400 lines do not divide by 3: a short last
    block)."""
    cfg_key, n_cells, steps = 0, 2000, 3
    got = {}
    for mode in ("gather", "blocks"):
        (tmp_path / mode).mkdir()
        res = _dist_util.run(world, _slab_iface_run, (cfg_key, n_cells, steps, mode),
                             tmp_path / mode)
        got[mode] = res
    for a, b in zip(got["gather"], got["blocks"]):
        for x, y in zip(a[2:], b[2:]):
            assert np.array_equal(x, y)


def _c4_pipe_run(rank, world, n_cells, steps, pipe, iface):
    import os

    os.environ["CELLGPU_SLAB_PIPE"] = pipe  # (default off)
    os.environ["CELLGPU_SLAB_IFACE"] = iface
    return _c4_slab_run(rank, world, n_cells, steps, "fast")


@pytest.mark.parametrize("world,iface", [(2, "gather"), (3, "blocks"), (4, "blocks")])
def test_substrate_pipeline_matches_unpipelined(tmp_path, world, iface):
    """The per-substrate pipeline of the slab step (substrate windows on the
    context; one substrate's interface exchange in flight while the next
    substrate's sweeps run) against all substrates per call: config 4's
    fast slabs, fields and cells bit for bit, with the all-gather and with
    the block interface solve."""
    n_cells, steps = 30000, 2
    got = {}
    for pipe in ("0", "1"):
        (tmp_path / pipe).mkdir()
        got[pipe] = _dist_util.run(world, _c4_pipe_run, (n_cells, steps, pipe, iface), tmp_path / pipe)
    for a, b in zip(got["0"], got["1"]):
        for x, y in zip(a[2:], b[2:]):
            assert np.array_equal(x, y)


def _defer_run(rank, world, cfg_key, n_cells, steps, defer):
    import os

    os.environ["CELLGPU_SLAB_DEFER"] = defer
    if cfg_key == 4:
        return _c4_slab_run(rank, world, n_cells, steps, "fast")
    return _slab_run(rank, world, cfg_key, n_cells, steps, None, "fast")


@pytest.mark.parametrize("cfg_key,world", [(4, 2), (4, 4), (2, 3), (3, 2)])
def test_deferred_correction_matches_separate_pass(tmp_path, cfg_key, world):
    """The interface correction of substeps 1..n-1 applied by the next
    substep's x-row (config 4's 256 x 256 slabs) or plane kernel (80 x 80
    and 160 x 160 slabs) while it stages the field, against the separate
    correction pass: fields and cells bit for bit, with the all-gather
    (P = 2) and the line-block interface solve (P = 3, 4)."""
    n_cells = 30000 if cfg_key == 4 else None
    got = {}
    for defer in ("0", "1"):
        (tmp_path / defer).mkdir()
        got[defer] = _dist_util.run(world, _defer_run, (cfg_key, n_cells, 2, defer), tmp_path / defer)
    for a, b in zip(got["0"], got["1"]):
        for x, y in zip(a[2:], b[2:]):
            assert np.array_equal(x, y)


def test_config4_slabs_ten_steps_match_single_gpu(tmp_path):
    """Ten mechanics steps (cells migrating across the slab faces every step)
    of config 4's fast slabs at P = 4 with every default on -- overlapped
    mechanics, line-block interface solve, deferred corrections -- against
    one GPU on the gathered box: cells bit for bit, fields within 1e-10."""
    from paper_2306_11544_b200.engine import Simulation
    from paper_2306_11544_b200.mechanics import InteractionParams

    world, n_cells, steps = 4, 200000, 10
    res = _dist_util.run(world, _c4_slab_run, (n_cells, steps, "fast"), tmp_path)
    parts = [_c4_rank_inputs(r, world, n_cells) for r in range(world)]
    cfg = parts[0][0]
    S, plane = cfg.n_substrates, cfg.nx * cfg.ny
    dens0 = np.concatenate([p.densities.reshape(S, -1, plane) for _, p in parts], axis=1).reshape(S, -1)
    sim = Simulation(
        _c4_global_mesh(cfg, world), diffusion=cfg.diffusion, decay=cfg.decay, densities=dens0,
        positions=np.concatenate([p.positions for _, p in parts]),
        radius=np.concatenate([p.radius for _, p in parts]),
        ids=np.concatenate([p.ids + r * n_cells for r, (_, p) in enumerate(parts)]),
        secretion=np.concatenate([p.secretion for _, p in parts], axis=1),
        uptake=np.concatenate([p.uptake for _, p in parts], axis=1), saturation=cfg.saturation,
        bc=cfg.bc, dirichlet=cfg.dirichlet,
        params=InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier),
        dt_diffusion=cfg.dt_diffusion, dt_mechanics=cfg.dt_mechanics, integrator=cfg.integrator,
        numerics="fast")
    sim.run(steps, graph=False)
    sim.sync()
    pos1, vel1, dens1 = sim.positions(), sim.velocities(), sim.densities()
    sim.close()
    ids = np.concatenate([r[2] for r in res])
    o = np.argsort(ids)
    assert np.array_equal(ids[o], np.arange(world * n_cells))
    assert np.array_equal(np.concatenate([r[3] for r in res])[o], pos1)
    assert np.array_equal(np.concatenate([r[4] for r in res])[o], vel1)
    dens = np.concatenate([r[5].reshape(S, -1, plane) for r in res], axis=1).reshape(S, -1)
    assert _field_err(dens, dens1, S) <= FIELD_TOL
    # cells did cross the slab faces
    moved = sum(int(np.sum((r[2] // n_cells) != k)) for k, r in enumerate(res))
    assert moved > 0, moved
