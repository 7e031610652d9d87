"""The reference's own hot-path tests, run against this package on the GPU.

Each test restates one in /root/reference/pkg/tests (file:line in the
docstring) with ``cb`` = paper_2306_11544_b200 instead of cellbench: same
calls, same assertions.  This is the drop-in check -- a user of the reference
switching imports sees the same behaviour."""

import math

import numpy as np
import pytest

import paper_2306_11544_b200 as cb
from paper_2306_11544_b200 import (DomainError, InteractionParams, MechanicsSchedule,
                                   TraversalMode, WorkerPool, apply_cell_exchange,
                                   integrate_positions, lod_step, refresh_nonempty_list,
                                   update_velocities)

pytestmark = pytest.mark.gpu


@pytest.fixture
def pool2():
    pool = WorkerPool(2)
    yield pool
    pool.shutdown()


@pytest.fixture
def small_mesh():
    return cb.CartesianMesh(4, 4, 4)


def make_container(mesh, positions, **cell_kwargs):
    cont = cb.CellContainer(mesh)
    for p in positions:
        cont.new_cell(list(p), **cell_kwargs)
    cb.rebin_cells(cont)
    return cont


def uniform_micro(mesh, diffusion, decay, value=38.0):
    return cb.Microenvironment(mesh, [diffusion], [decay], [value])


def random_micro(mesh, diffusion, decay, seed=3):
    micro = cb.Microenvironment(mesh, [diffusion], [decay])
    rng = np.random.default_rng(seed)
    micro.densities[0] = rng.uniform(0.0, 50.0, mesh.voxel_count)
    return micro


# ---------------------------------------------------------------- lod (test_diffusion.py)

def test_decay_only_matches_closed_form(pool2):
    """test_diffusion.py:87-94"""
    mesh = cb.CartesianMesh(4, 4, 4)
    micro = uniform_micro(mesh, diffusion=0.0, decay=0.7, value=38.0)
    dt, steps = 0.05, 10
    for _ in range(steps):
        lod_step(micro, mesh, dt, TraversalMode.OUTER_LOOP, pool2)
    expected = 38.0 / (1.0 + dt * 0.7 / 3.0) ** (3 * steps)
    np.testing.assert_allclose(micro.densities[0], expected, rtol=1e-14)


def test_no_decay_conserves_mass(pool2):
    """test_diffusion.py:97-104"""
    mesh = cb.CartesianMesh(8, 8, 8)
    micro = random_micro(mesh, diffusion=100000.0, decay=0.0)
    mass0 = micro.densities[0].sum()
    for _ in range(100):
        lod_step(micro, mesh, 0.1, TraversalMode.COLLAPSED, pool2)
    assert micro.densities[0].sum() == pytest.approx(mass0, rel=1e-10)
    micro.check_state()


def test_uniform_field_is_steady_to_roundoff(pool2):
    """test_diffusion.py:107-114"""
    mesh = cb.CartesianMesh(5, 4, 3)
    micro = uniform_micro(mesh, diffusion=80000.0, decay=0.0)
    for _ in range(3):
        lod_step(micro, mesh, 0.1, TraversalMode.OUTER_LOOP, pool2)
    np.testing.assert_allclose(micro.densities[0], 38.0, rtol=0.0, atol=1e-11)


def test_field_stays_nonnegative(pool2):
    """test_diffusion.py:117-124"""
    mesh = cb.CartesianMesh(6, 6, 6)
    micro = random_micro(mesh, diffusion=50000.0, decay=2.0, seed=11)
    micro.densities[0, ::7] = 0.0
    for _ in range(50):
        lod_step(micro, mesh, 0.2, TraversalMode.OUTER_LOOP, pool2)
    micro.check_state()
    assert micro.densities[0].min() >= 0.0


def test_traversal_and_worker_count_do_not_change_the_field():
    """test_diffusion.py:134-149"""
    mesh = cb.CartesianMesh(6, 5, 4)
    runs = []
    for mode, workers in [(TraversalMode.OUTER_LOOP, 1), (TraversalMode.OUTER_LOOP, 4),
                          (TraversalMode.COLLAPSED, 1), (TraversalMode.COLLAPSED, 3)]:
        micro = random_micro(mesh, diffusion=90000.0, decay=0.4)
        with WorkerPool(workers) as pool:
            for _ in range(5):
                lod_step(micro, mesh, 0.1, mode, pool)
        runs.append(micro.densities.copy())
    for other in runs[1:]:
        assert np.array_equal(runs[0], other)


def test_sweep_chunk_granularity_contract(pool2):
    """test_diffusion.py:152-162"""
    mesh = cb.CartesianMesh(3, 4, 5)
    micro = uniform_micro(mesh, 1000.0, 0.1)
    outer = lod_step(micro, mesh, 0.1, TraversalMode.OUTER_LOOP, pool2)
    assert [r.schedulable_chunks for r in outer] == [5, 5, 4]
    collapsed = lod_step(micro, mesh, 0.1, TraversalMode.COLLAPSED, pool2)
    assert [r.schedulable_chunks for r in collapsed] == [20, 15, 12]
    assert [r.total_iterations for r in outer] == [5, 5, 4]
    assert [r.total_iterations for r in collapsed] == [20, 15, 12]


def test_degenerate_single_voxel_axis(pool2):
    """test_diffusion.py:165-171"""
    mesh = cb.CartesianMesh(1, 4, 4)
    micro = random_micro(mesh, diffusion=70000.0, decay=0.0)
    mass0 = micro.densities[0].sum()
    for _ in range(20):
        lod_step(micro, mesh, 0.1, TraversalMode.COLLAPSED, pool2)
    assert micro.densities[0].sum() == pytest.approx(mass0, rel=1e-12)


def test_fused_refresh_matches_standalone(pool2):
    """test_diffusion.py:176-188"""
    mesh = cb.CartesianMesh(4, 4, 4)
    micro = uniform_micro(mesh, 1000.0, 0.1)
    cont = make_container(mesh, [(10.0, 10.0, 10.0), (70.0, 70.0, 70.0), (30.0, 50.0, 10.0)])
    cont.nonempty_voxels = []
    lod_step(micro, mesh, 0.1, TraversalMode.OUTER_LOOP, pool2, container=cont)
    oracle = sorted(v for v, ids in cont.agent.items() if ids)
    assert cont.nonempty_voxels == oracle
    cont.nonempty_voxels = [999]
    assert refresh_nonempty_list(cont) == oracle
    assert cont.nonempty_voxels == oracle


# ---------------------------------------------------------------- gradients

def test_gradient_of_uniform_field_is_zero(pool2):
    """test_diffusion.py:300-304"""
    mesh = cb.CartesianMesh(5, 5, 5)
    micro = uniform_micro(mesh, 1000.0, 0.0)
    cb.compute_gradients(micro, mesh, TraversalMode.OUTER_LOOP, pool2)
    assert np.all(micro.gradients == 0.0)


def test_gradient_of_linear_field_is_exact_interior(pool2):
    """test_diffusion.py:307-322"""
    mesh = cb.CartesianMesh(5, 4, 3)
    micro = cb.Microenvironment(mesh, [1000.0], [0.0])
    ix = np.arange(5)
    micro.grid_view(0)[...] = (2.0 * (10.0 + 20.0 * ix))[None, None, :]
    cb.compute_gradients(micro, mesh, TraversalMode.COLLAPSED, pool2)
    g = micro.gradients[0].reshape(3, 4, 5, 3)
    assert np.all(g[:, :, 1:-1, 0] == 2.0)
    assert np.all(g[:, :, [0, -1], 0] == 0.0)
    assert np.all(g[..., 1:] == 0.0)


def test_gradient_modes_and_workers_agree_bitwise():
    """test_diffusion.py:325-341"""
    mesh = cb.CartesianMesh(6, 5, 4)
    results = []
    for mode, workers in [(TraversalMode.OUTER_LOOP, 1), (TraversalMode.OUTER_LOOP, 3),
                          (TraversalMode.COLLAPSED, 1), (TraversalMode.COLLAPSED, 4)]:
        micro = random_micro(mesh, 1000.0, 0.0, seed=9)
        with WorkerPool(workers) as pool:
            recs = cb.compute_gradients(micro, mesh, mode, pool)
        results.append(micro.gradients.copy())
    assert all(np.array_equal(results[0], r) for r in results[1:])
    assert recs[0].schedulable_chunks == 5 * 4


def test_gradient_chunk_granularity(pool2):
    """test_diffusion.py:344-350"""
    mesh = cb.CartesianMesh(3, 4, 5)
    micro = uniform_micro(mesh, 1000.0, 0.0)
    assert cb.compute_gradients(micro, mesh, TraversalMode.OUTER_LOOP, pool2)[0].schedulable_chunks == 5
    assert cb.compute_gradients(micro, mesh, TraversalMode.COLLAPSED, pool2)[0].schedulable_chunks == 20


# ---------------------------------------------------------------- exchange

def exchange_fixture(value=38.0):
    mesh = cb.CartesianMesh(4, 4, 4)
    micro = uniform_micro(mesh, 1000.0, 0.0, value)
    cont = make_container(mesh, [(10.0, 10.0, 10.0), (12.0, 10.0, 10.0), (50.0, 30.0, 10.0)],
                          radius=8.0)
    return mesh, micro, cont


def test_exchange_noop_without_rates():
    """test_diffusion.py:208-213"""
    _, micro, cont = exchange_fixture()
    before = micro.densities.copy()
    apply_cell_exchange(micro, cont, 0.01, secretion=0.0, uptake=0.0, saturation=38.0)
    assert np.array_equal(micro.densities, before)


def test_exchange_saturated_secretion_is_a_fixed_point():
    """test_diffusion.py:216-220"""
    _, micro, cont = exchange_fixture(value=38.0)
    apply_cell_exchange(micro, cont, 0.01, secretion=4.2, uptake=0.0, saturation=38.0)
    np.testing.assert_allclose(micro.densities[0], 38.0, rtol=1e-14)


def test_exchange_uptake_decreases_and_stays_nonnegative():
    """test_diffusion.py:223-232"""
    _, micro, cont = exchange_fixture(value=38.0)
    occupied = sorted(cont.nonempty_voxels)
    for _ in range(500):
        apply_cell_exchange(micro, cont, 0.05, secretion=0.0, uptake=40.0, saturation=38.0)
    assert micro.densities[0][occupied].max() < 38.0
    assert micro.densities[0].min() >= 0.0
    untouched = np.setdiff1d(np.arange(64), occupied)
    assert np.all(micro.densities[0][untouched] == 38.0)


def test_exchange_secretion_moves_toward_saturation():
    """test_diffusion.py:235-240"""
    _, micro, cont = exchange_fixture(value=1.0)
    v = cont.nonempty_voxels[0]
    apply_cell_exchange(micro, cont, 0.1, secretion=5.0, uptake=0.0, saturation=38.0)
    assert 1.0 < micro.densities[0][v] < 38.0


def test_exchange_is_storage_order_independent():
    """test_diffusion.py:243-259"""
    mesh = cb.CartesianMesh(4, 4, 4)
    results = []
    for reverse in (False, True):
        micro = uniform_micro(mesh, 1000.0, 0.0, 20.0)
        cont = cb.CellContainer(mesh)
        cont.new_cell([10.0, 10.0, 10.0], radius=8.0)
        cont.new_cell([12.0, 11.0, 10.0], radius=6.0)
        if reverse:
            cont.cells.reverse()
        cb.rebin_cells(cont)
        apply_cell_exchange(micro, cont, 0.05, secretion=3.0, uptake=7.0, saturation=38.0)
        results.append(micro.densities.copy())
    assert np.array_equal(results[0], results[1])


def test_exchange_parallel_matches_serial(pool2):
    """test_diffusion.py:262-275"""
    mesh = cb.CartesianMesh(4, 4, 4)
    fields = []
    for pool in (None, pool2):
        micro = uniform_micro(mesh, 1000.0, 0.0, 25.0)
        cont = make_container(mesh, [(10.0, 10.0, 10.0), (30.0, 30.0, 30.0), (50.0, 50.0, 50.0),
                                     (70.0, 10.0, 50.0)])
        record = apply_cell_exchange(micro, cont, 0.02, secretion=2.0, uptake=3.0,
                                     saturation=38.0, pool=pool)
        fields.append(micro.densities.copy())
    assert np.array_equal(fields[0], fields[1])
    assert record is not None and record.items == 4


def test_exchange_rejects_nonpositive_denominator():
    """test_diffusion.py:278-285"""
    _, micro, cont = exchange_fixture()
    with pytest.raises(DomainError):
        apply_cell_exchange(micro, cont, 1.0, secretion=0.0, uptake=-8.0, saturation=38.0)
    with pytest.raises(DomainError):
        apply_cell_exchange(micro, cont, 0.0, secretion=1.0, uptake=0.0, saturation=38.0)


# ---------------------------------------------------------------- container (test_core.py)

def test_rebin_matches_bruteforce_oracle(small_mesh):
    """test_core.py:145-158"""
    cont = make_container(small_mesh, [(10.0, 10.0, 10.0), (11.0, 10.0, 10.0),
                                       (70.0, 70.0, 70.0), (35.0, 50.0, 10.0)])
    oracle = {}
    for c in cont.cells:
        oracle.setdefault(small_mesh.voxel_of(c.position), []).append(c.id)
    got = {v: ids for v, ids in cont.agent.items() if ids}
    assert got == oracle
    assert cont.nonempty_voxels == sorted(oracle)
    for c in cont.cells:
        assert c.voxel_index == small_mesh.voxel_of(c.position)
    cont.check_consistent()


def test_rebin_preserves_storage_order_within_voxel(small_mesh):
    """test_core.py:161-169"""
    cont = cb.CellContainer(small_mesh)
    a = cont.new_cell([10.0, 10.0, 10.0])
    b = cont.new_cell([11.0, 10.0, 10.0])
    cont.cells.reverse()
    cb.rebin_cells(cont)
    assert cont.agent[a.voxel_index] == [b.id, a.id]
    assert cont.storage_index == {b.id: 0, a.id: 1}


def test_new_cell_assigns_sequential_ids(small_mesh):
    """test_core.py:133-142"""
    cont = cb.CellContainer(small_mesh)
    a = cont.new_cell([10.0, 10.0, 10.0])
    b = cont.new_cell([30.0, 10.0, 10.0])
    assert (a.id, b.id) == (0, 1) and cont.by_id[a.id] is a and cont.positions_dirty
    cb.rebin_cells(cont)
    assert cont.storage_index[b.id] == 1 and not cont.positions_dirty


def test_check_consistent_detects_stale_bin(small_mesh):
    """test_core.py:172-176"""
    cont = make_container(small_mesh, [(10.0, 10.0, 10.0)])
    cont.cells[0].position[0] = 50.0
    with pytest.raises(AssertionError):
        cont.check_consistent()


# ---------------------------------------------------------------- mechanics (test_mechanics.py)

def clustered_container(mesh, n=40, seed=2):
    """test_mechanics.py:111-117 (division_draws restated: population.py:32-51)"""
    MASK = (1 << 64) - 1

    def mix(x):
        x = (x + 0x9E3779B97F4A7C15) & MASK
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
        return x ^ (x >> 31)

    def draws(s, cid, step):
        base = mix(mix(mix(s & MASK) ^ (cid & MASK)) ^ (step & MASK))
        return tuple((mix(base ^ k) >> 11) * (1.0 / (1 << 53)) for k in (1, 2, 3))

    positions = []
    for i in range(n):
        u1, u2, u3 = draws(seed, i, 0)
        positions.append((10.0 + 50.0 * u1, 10.0 + 50.0 * u2, 10.0 + 50.0 * u3))
    return make_container(mesh, positions, radius=8.0)


ALL_SCHEDULES = [MechanicsSchedule.cell_static(), MechanicsSchedule.cell_dynamic(4),
                 MechanicsSchedule.voxel(8), MechanicsSchedule.nonempty_voxel(2)]


def test_every_schedule_worker_count_and_mode_agrees_bitwise(small_mesh):
    """test_mechanics.py:136-144"""
    def velocities_under(schedule, workers, mode):
        cont = clustered_container(small_mesh)
        with WorkerPool(workers) as pool:
            update_velocities(cont, small_mesh, InteractionParams(), schedule, pool,
                              alloc_mode=mode)
        return [tuple(c.velocity) for c in cont.cells]

    reference = velocities_under(MechanicsSchedule.cell_static(), 1, cb.AllocationMode.IN_PLACE)
    assert any(v != (0.0, 0.0, 0.0) for v in reference)
    for schedule in ALL_SCHEDULES:
        for workers in (1, 2, 4):
            for mode in cb.AllocationMode:
                assert velocities_under(schedule, workers, mode) == reference


def test_voxel_schedule_iterates_empty_voxels_too(small_mesh):
    """test_mechanics.py:147-159"""
    cont = clustered_container(small_mesh)
    with WorkerPool(2) as pool:
        r_voxel = update_velocities(cont, small_mesh, InteractionParams(),
                                    MechanicsSchedule.voxel(8), pool)
        r_nonempty = update_velocities(cont, small_mesh, InteractionParams(),
                                       MechanicsSchedule.nonempty_voxel(2), pool)
        r_cells = update_velocities(cont, small_mesh, InteractionParams(),
                                    MechanicsSchedule.cell_static(), pool)
    assert r_voxel.total_iterations == small_mesh.voxel_count
    assert r_nonempty.total_iterations == len(cont.nonempty_voxels)
    assert r_nonempty.total_iterations < r_voxel.total_iterations
    assert r_cells.total_iterations == len(cont.cells)


def test_update_requires_consistent_binning(small_mesh):
    """test_mechanics.py:162-168"""
    cont = clustered_container(small_mesh)
    cont.new_cell([33.0, 33.0, 33.0])
    with WorkerPool(1) as pool:
        with pytest.raises(cb.ContainerStateError):
            update_velocities(cont, small_mesh, InteractionParams(),
                              MechanicsSchedule.cell_static(), pool)


def test_empty_container_is_fine(small_mesh):
    """test_mechanics.py:171-177"""
    cont = cb.CellContainer(small_mesh)
    with WorkerPool(2) as pool:
        for schedule in ALL_SCHEDULES:
            record = update_velocities(cont, small_mesh, InteractionParams(), schedule, pool)
    assert record.total_claims == 0


def test_integration_moves_cells_exactly(small_mesh):
    """test_mechanics.py:235-244"""
    cont = make_container(small_mesh, [(10.0, 10.0, 10.0), (30.0, 30.0, 30.0)])
    cont.cells[0].velocity[:] = [1.0, 2.0, 3.0]
    with WorkerPool(1) as pool:
        record = integrate_positions(cont, small_mesh, 0.1, pool)
    assert cont.cells[0].position == [10.0 + 0.1 * 1.0, 10.0 + 0.1 * 2.0, 10.0 + 0.1 * 3.0]
    assert cont.cells[1].position == [30.0, 30.0, 30.0]
    assert cont.positions_dirty
    assert record.items == 2


def test_integration_clamps_at_the_boundary(small_mesh):
    """test_mechanics.py:247-255"""
    cont = make_container(small_mesh, [(79.0, 40.0, 40.0)])
    cont.cells[0].velocity[:] = [1000.0, 0.0, -1e9]
    with WorkerPool(1) as pool:
        integrate_positions(cont, small_mesh, 1.0, pool)
    p = cont.cells[0].position
    assert small_mesh.contains(p)
    assert p[0] == pytest.approx(80.0 - 1e-6)
    assert p[2] == pytest.approx(1e-6)


def test_state_checksum_matches_a_host_recomputation(small_mesh):
    """simulate.py:79-90 digest over (id, position, velocity)"""
    cont = clustered_container(small_mesh)
    update_velocities(cont, small_mesh, InteractionParams(), MechanicsSchedule.cell_static(),
                      WorkerPool(1))
    a = cb.state_checksum(cont)
    cont.cells.reverse()  # order-independent
    assert cb.state_checksum(cont) == a
    assert a != cb.state_checksum(clustered_container(small_mesh))  # velocities differ
    assert math.isfinite(cont.cells[0].velocity[0])


# ---------------------------------------------------------------- storage order (test_population.py)

def test_sort_cells_by_voxel_orders_storage(small_mesh):
    """test_population.py:154-166"""
    cont = cb.CellContainer(small_mesh)
    a = cont.new_cell([70.0, 70.0, 70.0])  # high voxel, low id
    b = cont.new_cell([10.0, 10.0, 10.0])
    c = cont.new_cell([11.0, 10.0, 10.0])
    cb.rebin_cells(cont)
    cb.sort_cells_by_voxel(cont)
    assert [x.id for x in cont.cells] == [b.id, c.id, a.id]
    assert cont.storage_index[a.id] == 2
    cont.check_consistent()
    cb.sort_cells_by_voxel(cont)  # idempotent
    assert [x.id for x in cont.cells] == [b.id, c.id, a.id]


def test_sorting_never_changes_velocities(small_mesh):
    """test_population.py:169-179: accumulation order is id-based."""
    cont = make_container(small_mesh, [(15.0 + 8.0 * i, 40.0, 40.0) for i in range(8)],
                          radius=8.0)  # a touching row: every cell interacts
    with WorkerPool(2) as pool:
        update_velocities(cont, small_mesh, InteractionParams(), MechanicsSchedule.cell_static(),
                          pool)
        before = {c.id: tuple(c.velocity) for c in cont.cells}
        cb.sort_cells_by_voxel(cont)
        update_velocities(cont, small_mesh, InteractionParams(), MechanicsSchedule.cell_static(),
                          pool)
    assert {c.id: tuple(c.velocity) for c in cont.cells} == before


def test_sort_cells_by_voxel_on_device_resident_container(small_mesh):
    """from_arrays containers are permuted on the GPU; same order as the host path."""
    rng = np.random.default_rng(12)
    pos = rng.uniform(1.0, 79.0, (40, 3))
    ids = rng.permutation(40) + 100
    dev = cb.CellContainer.from_arrays(small_mesh, pos, 8.0, ids=ids)
    cb.rebin_cells(dev)
    cb.sort_cells_by_voxel(dev)
    host = cb.CellContainer(small_mesh)
    for p, i in zip(pos, ids):
        host.append_cell(cb.Cell(id=int(i), position=list(p), velocity=[0.0, 0.0, 0.0]))
    cb.rebin_cells(host)
    cb.sort_cells_by_voxel(host)
    assert [c.id for c in dev.cells] == [c.id for c in host.cells]
    assert [c.position for c in dev.cells] == [c.position for c in host.cells]
    dev.check_consistent()


# ---------------------------------------------------------------- divisions
# pkg/tests/test_population.py:29-146 with cb = paper_2306_11544_b200.

def test_draws_are_deterministic():
    """test_population.py:29-34"""
    assert cb.division_draws(42, 7, 3) == cb.division_draws(42, 7, 3)
    assert cb.division_draws(42, 7, 3) != cb.division_draws(42, 7, 4)
    assert cb.division_draws(42, 7, 3) != cb.division_draws(42, 8, 3)
    assert cb.division_draws(41, 7, 3) != cb.division_draws(42, 7, 3)


@pytest.mark.parametrize("seed,cid,step", [(0, 0, 0), (2**63, 10**6, 10**6), (5, 17, 3)])
def test_draws_are_unit_interval(seed, cid, step):
    """test_population.py:37-41"""
    triple = cb.division_draws(seed, cid, step)
    assert len(triple) == 3
    for u in triple:
        assert 0.0 <= u < 1.0


def populated(mesh, n=6, rate=0.0, radius=8.0):
    positions = [(15.0 + 8.0 * i, 40.0, 40.0) for i in range(n)]
    return make_container(mesh, positions, radius=radius, division_rate=rate)


def test_no_rate_means_no_divisions(small_mesh):
    """test_population.py:57-62"""
    cont = populated(small_mesh, rate=0.0)
    daughters = cb.attempt_divisions(cont, seed=1, dt=1.0, mesh=small_mesh, step=0)
    assert daughters == []
    assert len(cont) == 6
    assert not cont.positions_dirty


def test_certain_division_doubles_the_population(small_mesh):
    """test_population.py:65-76"""
    cont = populated(small_mesh, rate=50.0)
    daughters = cb.attempt_divisions(cont, seed=1, dt=1.0, mesh=small_mesh, step=0)
    assert len(daughters) == 6
    assert len(cont) == 12
    assert not cont.positions_dirty
    cont.check_consistent()
    assert [d.id for d in daughters] == list(range(6, 12))
    assert [cont.storage_index[d.id] for d in daughters] == list(range(6, 12))


def test_daughter_copies_parent_and_sits_half_radius_away(small_mesh):
    """test_population.py:79-90"""
    cont = populated(small_mesh, n=1, rate=50.0, radius=7.0)
    parent = cont.cells[0]
    parent.velocity[:] = [0.5, -0.25, 1.0]
    daughter = cb.attempt_divisions(cont, seed=9, dt=1.0, mesh=small_mesh, step=4)[0]
    assert daughter.radius == parent.radius
    assert daughter.division_rate == parent.division_rate
    assert daughter.velocity == parent.velocity
    assert daughter.velocity is not parent.velocity
    d = math.dist(daughter.position, parent.position)
    assert d == pytest.approx(3.5, rel=1e-12)


def test_probability_matches_the_draw_rule(small_mesh):
    """test_population.py:93-105"""
    rate, dt, seed, step = 0.2, 0.5, 123, 17
    cont = populated(small_mesh, rate=rate)
    p = 1.0 - math.exp(-rate * dt)
    expected = sorted(c.id for c in cont.cells if cb.division_draws(seed, c.id, step)[0] < p)
    daughters = cb.attempt_divisions(cont, seed=seed, dt=dt, mesh=small_mesh, step=step)
    assert [d.id for d in daughters] == list(range(6, 6 + len(expected)))
    assert len(daughters) == len(expected)


def test_divisions_ignore_storage_order(small_mesh):
    """test_population.py:108-119"""
    outcomes = []
    for reverse in (False, True):
        cont = populated(small_mesh, rate=1.5)
        if reverse:
            cont.cells.reverse()
            cb.rebin_cells(cont)
        daughters = cb.attempt_divisions(cont, seed=5, dt=1.0, mesh=small_mesh, step=2)
        outcomes.append([(d.id, tuple(d.position)) for d in daughters])
    assert outcomes[0] == outcomes[1]
    assert outcomes[0]


def test_capacity_error_fires_before_any_append(small_mesh):
    """test_population.py:122-127"""
    cont = populated(small_mesh, rate=50.0)
    with pytest.raises(cb.CapacityError):
        cb.attempt_divisions(cont, seed=1, dt=1.0, mesh=small_mesh, step=0, cap=8)
    assert len(cont) == 6
    cont.check_consistent()


def test_division_rejects_bad_dt(small_mesh):
    """test_population.py:130-133"""
    cont = populated(small_mesh, rate=1.0)
    with pytest.raises(DomainError):
        cb.attempt_divisions(cont, seed=1, dt=0.0, mesh=small_mesh, step=0)


def test_daughters_are_clamped_inside(small_mesh):
    """test_population.py:136-144"""
    cont = make_container(small_mesh, [(79.9, 79.9, 79.9)], radius=8.0, division_rate=50.0)
    for step in range(6):
        cb.attempt_divisions(cont, seed=3, dt=1.0, mesh=small_mesh, step=step, cap=100)
    assert all(small_mesh.contains(c.position) for c in cont.cells)
