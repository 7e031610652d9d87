"""The z-slab decomposition on the GPU: P ranks (processes) share cuda:0 and
talk through gloo with host staging -- no kernel waits on another rank's
kernel.  Against the single-GPU engine on the same inputs: cells (ids,
positions, velocities) bit-for-bit, fields within 1e-12 normwise (the
partitioned z sweep rounds differently; the bar is 1e-10)."""

import numpy as np
import pytest

import _dist_util

pytestmark = pytest.mark.gpu


def _slab_run(rank, world, cfg_key, n_cells, steps, bounds=None):
    import torch
    import torch.distributed as dist

    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.distributed import Comm, build

    torch.cuda.set_device(0)
    cfg = CONFIGS[cfg_key]
    inp = make_inputs(cfg, n_cells)
    sim = build(cfg, Comm(dist, "cuda:0"), inp, bounds)
    for _ in range(steps):
        sim.step()
    ids, pos, vel = sim.owned_state()
    return sim.z0, sim.z1, ids, pos, vel, sim.densities()


def _single(cfg_key, n_cells, steps):
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[cfg_key]
    sim = Simulation.from_config(cfg, make_inputs(cfg, n_cells))
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
