"""Host-side logic that needs no GPU: mesh semantics (the reference's own
core tests, run against this package), validation and error behaviour,
record shapes, and the seeded config generators."""

import math

import numpy as np
import pytest

import paper_2306_11544_b200 as cg
from paper_2306_11544_b200 import DomainError, NumericError
from paper_2306_11544_b200.configs import CONFIGS, make_inputs, slab_config


def test_flatten_reference_voxel():
    mesh = cg.CartesianMesh(75, 75, 75)
    assert mesh.voxel_of((30.0, 30.0, 30.0)) == 5701
    assert mesh.flatten(1, 1, 1) == 5701
    assert mesh.unflatten(5701) == (1, 1, 1)


def test_voxel_of_half_open_and_bounds():
    mesh = cg.CartesianMesh(3, 3, 3)
    assert mesh.voxel_of((0.0, 0.0, 0.0)) == 0
    assert mesh.voxel_of((19.999, 0.0, 0.0)) == 0
    assert mesh.voxel_of((20.0, 0.0, 0.0)) == 1
    with pytest.raises(DomainError):
        mesh.voxel_of((-0.1, 10.0, 10.0))
    with pytest.raises(DomainError):
        mesh.voxel_of((10.0, 10.0, 60.0))
    with pytest.raises(DomainError):
        mesh.voxel_of((float("nan"), 10.0, 10.0))


def test_voxel_of_matches_golden(golden):
    from conftest import cases, mesh_from_arr

    for k in cases(golden, "vo"):
        m = mesh_from_arr(golden[f"{k}_mesh"])
        for p, want in zip(golden[f"{k}_pts"], golden[f"{k}_voxel"]):
            try:
                got = m.voxel_of(tuple(float(x) for x in p))
            except DomainError:
                got = -1
            assert got == want


def test_clamp_and_bounds():
    mesh = cg.CartesianMesh(3, 3, 3)
    p = [-5.0, 30.0, 1e9]
    mesh.clamp_inside(p)
    assert mesh.contains(p)
    assert p[0] == pytest.approx(1e-6) and p[1] == 30.0 and p[2] == pytest.approx(60.0 - 1e-6)
    m2 = cg.CartesianMesh(5, 4, 3, dx=10.0, dy=20.0, dz=30.0)
    assert m2.voxel_count == 60 and m2.upper == (50.0, 80.0, 90.0)
    with pytest.raises(DomainError):
        cg.CartesianMesh(0, 4, 4)
    with pytest.raises(DomainError):
        cg.CartesianMesh(4, 4, 4, dx=-1.0)


def test_microenvironment_host_side(small_mesh=None):
    mesh = cg.CartesianMesh(4, 4, 4)
    micro = cg.Microenvironment(mesh, [100.0, 10.0], [0.1, 0.0], [38.0, 1.0])
    assert micro.substrate_count == 2
    assert micro.densities.shape == (2, 64)
    assert np.all(micro.densities[0] == 38.0)
    micro.grid_view(1)[2, 1, 3] = 7.0
    assert micro.densities[1, mesh.flatten(3, 1, 2)] == 7.0
    micro.check_state()
    micro.densities[0, 5] = -1e-9
    with pytest.raises(NumericError):
        micro.check_state()
    with pytest.raises(DomainError):
        cg.Microenvironment(mesh, [-1.0], [0.0])
    with pytest.raises(DomainError):
        cg.Microenvironment(mesh, [1.0, 1.0], [0.0])


def test_cell_volume_and_container_ids():
    c = cg.Cell(id=0, position=[0.0, 0.0, 0.0], velocity=[0.0, 0.0, 0.0], radius=8.0)
    assert c.volume == (4.0 / 3.0) * math.pi * 8.0**3
    cont = cg.CellContainer(cg.CartesianMesh(4, 4, 4))
    a = cont.new_cell([10.0, 10.0, 10.0])
    b = cont.new_cell([30.0, 10.0, 10.0])
    assert (a.id, b.id) == (0, 1) and cont.by_id[1] is b and cont.positions_dirty
    with pytest.raises(DomainError):
        cont.append_cell(cg.Cell(id=1, position=[1.0, 1.0, 1.0], velocity=[0.0] * 3))


def test_argument_errors_raise_before_touching_the_device():
    mesh = cg.CartesianMesh(3, 3, 3)
    micro = cg.Microenvironment(mesh, [100.0], [0.0])
    with pytest.raises(DomainError):
        cg.lod_step(micro, mesh, 0.0, cg.TraversalMode.OUTER_LOOP, cg.WorkerPool(2))
    cont = cg.CellContainer(mesh)
    with pytest.raises(DomainError):
        cg.apply_cell_exchange(micro, cont, 0.0, 1.0, 0.0, 38.0)
    with pytest.raises(DomainError):
        cg.integrate_positions(cont, mesh, -0.1, cg.WorkerPool(1))
    cont.new_cell([10.0, 10.0, 10.0])
    with pytest.raises(cg.ContainerStateError):  # appended but not rebinned
        cg.update_velocities(cont, mesh, cg.InteractionParams(),
                             cg.MechanicsSchedule.cell_static(), cg.WorkerPool(1))
    with pytest.raises(DomainError):
        cg.lod_step(micro, mesh, 0.1, cg.TraversalMode.OUTER_LOOP, None, bc="robin")


def test_no_cpu_fallback_without_a_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    mesh = cg.CartesianMesh(3, 3, 3)
    micro = cg.Microenvironment(mesh, [100.0], [0.0], [1.0])
    with pytest.raises(cg.DeviceError):
        cg.lod_step(micro, mesh, 0.1, cg.TraversalMode.OUTER_LOOP, cg.WorkerPool(1))


def test_pair_contribution_host_helper():
    p = cg.InteractionParams(repulsion=10.0, adhesion=0.0, adhesion_multiplier=1.25)
    ci = cg.Cell(id=0, position=[0.0, 0.0, 0.0], velocity=[0.0] * 3, radius=8.4)
    cj = cg.Cell(id=1, position=[8.4, 0.0, 0.0], velocity=[0.0] * 3, radius=8.4)
    v = cg.pair_velocity_contribution(ci, cj, p)
    assert v[0] == pytest.approx(-2.5, rel=1e-15) and v[1] == 0.0 and v[2] == 0.0
    with pytest.raises(DomainError):
        cg.InteractionParams(adhesion_multiplier=0.9)
    with pytest.raises(DomainError):
        cg.MechanicsSchedule.voxel(0)


def test_static_ranges_and_records():
    assert cg.static_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    from paper_2306_11544_b200.parallel import gpu_record

    r = gpu_record(5, 5, 0.1)
    assert r.total_iterations == 5 and r.total_claims == 5 and r.total_alloc_events == 0


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_config_inputs_are_deterministic_and_in_bounds(k):
    cfg = CONFIGS[k]
    n = min(cfg.n_cells, 5000)
    a, b = make_inputs(cfg, n), make_inputs(cfg, n)
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.uptake, b.uptake)
    mesh = cfg.mesh()
    lo, hi = np.array(mesh.origin), np.array(mesh.upper)
    assert np.all(a.positions >= lo) and np.all(a.positions < hi)
    assert a.densities.shape == (cfg.n_substrates, cfg.voxel_count)
    assert a.secretion.shape == (cfg.n_substrates, n)
    assert cfg.substeps == 10
    if cfg.seeding == "sphere":
        assert np.all((a.positions ** 2).sum(1) < cfg.seed_radius ** 2 + 1e-6)


def test_slab_configs_tile_the_global_box():
    base = CONFIGS[4]
    world = 4
    zs = [slab_config(base, r, world).mesh() for r in range(world)]
    for r in range(world - 1):
        assert zs[r].upper[2] == zs[r + 1].origin[2]
    assert zs[0].origin[2] == -320.0 * world and zs[-1].upper[2] == 320.0 * world


def test_check_binning_exact_guard():
    """mechanics.py:87-96: the guard passes iff min(dx) >= m_a * 2 * R_max;
    the BASELINE radius (8.4127 um, reach 21.03 um) violates it on 20 um
    voxels, R = 8 (reach exactly 20 um) does not."""
    import paper_2306_11544_b200 as cg

    mesh = cg.CartesianMesh(4, 4, 4)
    params = cg.InteractionParams()
    ok = cg.CellContainer(mesh)
    ok.new_cell([10.0, 10.0, 10.0], radius=8.0)
    cg.check_binning_exact(ok, mesh, params)
    bad = cg.CellContainer(mesh)
    bad.new_cell([10.0, 10.0, 10.0], radius=8.4127)
    with pytest.raises(cg.DomainError):
        cg.check_binning_exact(bad, mesh, params)


def test_binning_report_counts_missed_pairs():
    """Two cells 20.2 um apart along x in voxels 0 and 2 are in range (reach
    21.03 um) but outside each other's 3x3x3 block: one missed pair of two;
    the other pair (same voxel) is seen."""
    import paper_2306_11544_b200 as cg
    from paper_2306_11544_b200.mechanics import binning_report

    mesh = cg.CartesianMesh(4, 4, 4)
    pos = np.array([[19.9, 30.0, 30.0], [40.1, 30.0, 30.0], [45.0, 30.0, 30.0]])
    rep = binning_report(pos, 8.4127, mesh, cg.InteractionParams())
    assert not rep["binning_exact"]
    # pairs in range: (0,1) d=20.2 missed; (1,2) d=4.9 same voxel; (0,2) d=25.1 out of reach
    assert rep["in_range_pairs"] == 2 and rep["missed_pairs"] == 1
    assert rep["missed_fraction"] == 0.5


def test_binning_report_config0():
    """The missed-pair fraction of BASELINE config 0's seeding (G3 bookkeeping):
    small but non-zero."""
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.mechanics import InteractionParams, binning_report

    cfg = CONFIGS[0]
    inp = make_inputs(cfg)
    rep = binning_report(inp.positions, inp.radius, cfg.mesh(),
                         InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier))
    assert rep["in_range_pairs"] > 1000
    assert 0.0 < rep["missed_fraction"] < 0.05, rep


def test_sorted_storage_orders_by_voxel_then_id():
    """configs.sorted_storage (the voxel_sorted strategy's initial sort,
    population.py:132-135): cells in (voxel, id) order, every per-cell array
    permuted with its cell, fields untouched."""
    from paper_2306_11544_b200.configs import sorted_storage

    cfg = CONFIGS[0]
    inp = make_inputs(cfg)
    srt = sorted_storage(cfg, inp)
    mesh = cfg.mesh()
    vox = np.array([mesh.voxel_of(tuple(p)) for p in srt.positions])
    key = vox * 10**7 + srt.ids
    assert np.all(np.diff(key) > 0)
    o = np.argsort(srt.ids)
    assert np.array_equal(srt.ids[o], inp.ids)
    assert np.array_equal(srt.positions[o], inp.positions)
    assert np.array_equal(srt.radius[o], inp.radius)
    assert np.array_equal(srt.secretion[:, o], inp.secretion)
    assert np.array_equal(srt.uptake[:, o], inp.uptake)
    assert srt.densities is inp.densities
