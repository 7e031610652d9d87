"""GPU parity: every hot-path call through the C-ABI against the reference's
golden fixtures and the CPU oracle.

Bars: bins, voxel keys, non-empty lists, substrate
fields and integration are compared bit-for-bit.  Velocities are bit-for-bit
against the oracle evaluating ``(1 - d/c)**2`` as t*t (SQUARE_MUL, the GPU's
arithmetic) and within 1e-12 normwise (max|dv| <= 1e-12 max|v|) against the
reference itself, whose ``**2`` is a libm pow call that is off by one ulp in
~0.08% of evaluations on this glibc.
"""

import numpy as np
import pytest

import paper_2306_11544_b200 as cg
from conftest import cases, mesh_from_arr, refmesh_from_arr

pytestmark = pytest.mark.gpu

VEL_TOL = 1e-12


def normwise(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def container(mesh, pos, ids, radius):
    """Container whose storage order is the fixture's (ids need not be sorted)."""
    cont = cg.CellContainer(mesh)
    for p, i, r in zip(pos, ids, radius):
        cont.append_cell(cg.Cell(id=int(i), position=[float(x) for x in p],
                                 velocity=[0.0, 0.0, 0.0], radius=float(r)))
    cg.rebin_cells(cont)
    return cont


@pytest.mark.parametrize("ext", [False, True])
def test_lod_step_bitwise(golden, ext):
    pool = cg.WorkerPool(1)
    for k in cases(golden, "lod"):
        mesh = mesh_from_arr(golden[f"{k}_mesh"])
        micro = cg.Microenvironment(mesh, golden[f"{k}_D"], golden[f"{k}_K"])
        micro.densities = golden[f"{k}_in"]
        dt, steps = golden[f"{k}_dt_steps"]
        kw = dict(bc="dirichlet", dirichlet=golden[f"ext_{k}_dirichlet"]) if ext else {}
        for _ in range(int(steps)):
            recs = cg.lod_step(micro, mesh, dt, cg.TraversalMode.COLLAPSED, pool, **kw)
        assert len(recs) == 3 * micro.substrate_count
        want = golden[f"ext_{k}_out"] if ext else golden[f"{k}_out"]
        assert np.array_equal(micro.densities, want), k


def test_rebin_bitwise(golden):
    for k in cases(golden, "rb"):
        mesh = mesh_from_arr(golden[f"{k}_mesh"])
        pos, ids = golden[f"{k}_pos"], golden[f"{k}_ids"]
        cont = container(mesh, pos, ids, np.full(len(ids), 8.0))
        start, cells = golden[f"{k}_bin_start"], golden[f"{k}_bin_cells"]
        want_agent = {int(v): [int(ids[c]) for c in cells[start[v]:start[v + 1]]]
                      for v in golden[f"{k}_nonempty"]}
        assert cont.agent == want_agent, k
        assert cont.nonempty_voxels == golden[f"{k}_nonempty"].tolist(), k
        assert [c.voxel_index for c in cont.cells] == golden[f"{k}_voxel"].tolist(), k
        assert cont.storage_index == {int(i): s for s, i in enumerate(ids)}
        cont.check_consistent()


def test_device_voxel_of_matches_reference(golden):
    """core.py:77-85 voxel_of on the device (the function every rebin bins
    with) against the reference's own results on the vo* fixtures: random
    points, points exactly on voxel faces and +-1e-12 / +-1e-9 / 5e-324 off
    them, out-of-bounds points (DomainError -> -1), and a dx = 0.1 mesh where
    CPython's fmod-based // differs from floor(a / d).  Then the same points
    through cg_rebin: in-bounds points get the same voxel keys, and any
    out-of-bounds point makes the rebin raise DomainError."""
    import torch

    from paper_2306_11544_b200 import _lib

    L = _lib.load()
    for k in cases(golden, "vo"):
        mesh = mesh_from_arr(golden[f"{k}_mesh"])
        pts, want = golden[f"{k}_pts"], golden[f"{k}_voxel"]
        n = len(pts)
        ctx = _lib.Context(mesh, 0, n, 0)
        ctx.bind_stream()
        d_pts = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
        out = torch.full((n,), -7, dtype=torch.int32, device="cuda")
        _lib.raise_for(L.cg_voxel_index(ctx.handle, n, _lib.ptr(d_pts), _lib.ptr(out)), "voxel_index")
        ctx.sync("voxel_index")
        got = out.cpu().numpy().astype(np.int64)
        assert np.array_equal(got, want), (k, np.flatnonzero(got != want)[:10])
        inside = want >= 0
        assert inside.sum() > 0 and (~inside).sum() > 0, k
        cont = cg.CellContainer(mesh)
        for i, p in enumerate(pts[inside]):
            cont.append_cell(cg.Cell(id=i, position=[float(x) for x in p], velocity=[0.0] * 3))
        cg.rebin_cells(cont)
        assert [c.voxel_index for c in cont.cells] == want[inside].tolist(), k
        bad = cg.CellContainer(mesh)
        bad.append_cell(cg.Cell(id=0, position=[float(x) for x in pts[~inside][0]], velocity=[0.0] * 3))
        with pytest.raises(cg.DomainError):
            cg.rebin_cells(bad)
        ctx.close()


def test_exchange_bitwise(golden):
    mesh = mesh_from_arr(golden["ex_mesh"])
    pos, ids, rad = golden["ex_pos"], golden["ex_ids"], golden["ex_radius"]
    cont = container(mesh, pos, ids, rad)
    micro = cg.Microenvironment(mesh, [1e5, 1e3], [0.1, 0.01])
    micro.densities = golden["ex_in"]
    for k in range(3):
        dt, sec, upt, sat, s = golden[f"ex{k}_args"]
        cg.apply_cell_exchange(micro, cont, dt, sec, upt, sat, substrate=int(s))
        assert np.array_equal(micro.densities, golden[f"ex{k}_out"]), k
    micro.densities = golden["ex_in"]
    sec = golden["ext_ex_sec"][:, ids]
    upt = golden["ext_ex_upt"][:, ids]
    cg.apply_cell_exchange(micro, cont, 0.01, sec, upt, [38.0, 38.0])
    assert np.array_equal(micro.densities, golden["ext_ex_out"])


def test_velocities_vs_reference_and_oracle(golden, oracle):
    params = cg.InteractionParams()
    for k in cases(golden, "ve"):
        mesh = mesh_from_arr(golden[f"{k}_mesh"])
        pos, ids, rad = golden[f"{k}_pos"], golden[f"{k}_ids"], golden[f"{k}_radius"]
        cont = container(mesh, pos, ids, rad)
        cg.update_velocities(cont, mesh, params, cg.MechanicsSchedule.nonempty_voxel(4),
                             cg.WorkerPool(1))
        got = np.array([c.velocity for c in cont.cells])
        ref = golden[f"{k}_vel"]
        assert normwise(got, ref) <= VEL_TOL, k
        m = refmesh_from_arr(golden[f"{k}_mesh"])
        b = oracle.rebin(m, pos)
        exact = oracle.velocities(m, pos, rad, ids, b, square_mode=oracle.SQUARE_MUL)
        assert np.array_equal(got, exact), k


@pytest.mark.parametrize("ext", [False, True])
def test_integrate_bitwise(golden, ext):
    for k in cases(golden, "in"):
        mesh = mesh_from_arr(golden[f"{k}_mesh"])
        pos0, vel = golden[f"{k}_pos0"], golden[f"{k}_vel"]
        dt = float(golden[f"{k}_dt"][0])
        cont = container(mesh, pos0, np.arange(len(pos0)), np.full(len(pos0), 8.0))
        for c in cont.cells:
            c.velocity[:] = vel[c.id].tolist()
        if ext:
            cont.previous_velocities[:] = golden[f"ext_{k}_prev"]
            cg.integrate_positions(cont, mesh, dt, None, integrator="ab2")
            want = golden[f"ext_{k}_pos"]
            assert np.array_equal(cont.previous_velocities, golden[f"ext_{k}_prev_out"])
        else:
            cg.integrate_positions(cont, mesh, dt, None)
            want = golden[f"{k}_pos"]
        assert cont.positions_dirty
        assert np.array_equal(np.array([c.position for c in cont.cells]), want), k


def _oracle_state(oracle, cfg, inp, square_mode):
    return oracle.OracleState(
        oracle.mesh_from(cfg.mesh()), inp.densities, inp.positions, inp.radius, inp.ids,
        cfg.diffusion, cfg.decay, secretion=inp.secretion, uptake=inp.uptake,
        saturation=[cfg.saturation] * cfg.n_substrates,
        bc=oracle.BC_DIRICHLET if cfg.bc == "dirichlet" else oracle.BC_NEUMANN,
        dirichlet=cfg.dirichlet, dt_diff=cfg.dt_diffusion, dt_mech=cfg.dt_mechanics,
        substeps=cfg.substeps, integrator=oracle.AB2 if cfg.integrator == "ab2" else oracle.EULER,
        square_mode=square_mode, repulsion=cfg.repulsion, adhesion=cfg.adhesion,
        adhesion_multiplier=cfg.adhesion_multiplier)


@pytest.mark.parametrize("graph", [True, False])
def test_engine_config0_trajectory(golden, oracle, graph):
    """Config 0 as BASELINE states it, 5 mechanics steps through the step
    engine: bit-for-bit vs the oracle (t*t) every step; vs the reference-run
    fixture: fields and bins bitwise, kinematics within 1e-12 normwise."""
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[0]
    inp = make_inputs(cfg)
    sim = Simulation.from_config(cfg, inp)
    st = _oracle_state(oracle, cfg, inp, oracle.SQUARE_MUL)
    for step in range(5):
        sim.run(1, graph=graph)
        st.step(threads=4)
        assert np.array_equal(sim.densities(), st.dens), step
        assert np.array_equal(sim.positions(), st.pos), step
        assert np.array_equal(sim.velocities(), st.vel), step
        b = sim.bins()
        assert np.array_equal(b["bin_start"], st.bins.bin_start), step
        assert np.array_equal(b["bin_cells"], st.bins.bin_cells), step
        assert np.array_equal(b["nonempty"], st.bins.nonempty), step
    sim.sync()
    assert np.array_equal(sim.densities(), golden["ext_traj_dens"])
    assert normwise(sim.positions(), golden["ext_traj_pos"]) <= VEL_TOL
    assert normwise(sim.velocities(), golden["ext_traj_vel"]) <= VEL_TOL
    sim.close()


@pytest.mark.parametrize("k,env", [
    (1, {}), (2, {}), (3, {}), (4, {}),
    (3, {"CELLGPU_REGLINES": "0", "CELLGPU_EXCH_SPLIT": "0"}),
    (1, {"CELLGPU_EXCH_SPLIT": "0"}),
])
def test_engine_full_size_configs_vs_oracle(oracle, monkeypatch, k, env):
    """Full-size BASELINE configs (1: 80^3 x 3, 100k cells -- register-line
    kernels; 2: dense radial spheroid, 200k cells -- the over-capacity voxel
    kernels; 3: 160^3 x 4, 1M cells -- relay register lines, 2 lanes per
    line; 4: 256x256x32 slab x 4, 1M cells, plane too large for shared
    memory -> split x/y kernels, 32-plane register z kernel; the env variants
    reach the streaming plane kernel and the exchange fused into the plane
    kernels): two mechanics steps bit-for-bit against the oracle."""
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    for var, val in env.items():
        monkeypatch.setenv(var, val)
    cfg = CONFIGS[k]
    inp = make_inputs(cfg)
    sim = Simulation.from_config(cfg, inp)
    st = _oracle_state(oracle, cfg, inp, oracle.SQUARE_MUL)
    for step in range(2):
        sim.run(1)
        st.step(threads=oracle.max_threads())
        sim.sync()
        assert np.array_equal(sim.densities(), st.dens), (k, step)
        assert np.array_equal(sim.positions(), st.pos), (k, step)
        assert np.array_equal(sim.velocities(), st.vel), (k, step)
        assert np.array_equal(sim.bins()["nonempty"], st.bins.nonempty), (k, step)
    sim.close()


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_engine_fast_numerics_full_size_vs_oracle(oracle, k):
    """CG_NUMERICS_FAST on every BASELINE config at full size (config 1/3:
    segmented plane + z kernels with the affine exchange fused; 0, 2, 4: the
    exact LOD kernels; every config: direct velocities), two mechanics steps
    against the oracle in the reference's arithmetic (libm pow): fields within
    1e-10 (per substrate, max|d| / max|ref|), positions and velocities within
    1e-12 normwise, bins and non-empty lists identical."""
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[k]
    inp = make_inputs(cfg)
    sim = Simulation.from_config(cfg, inp, numerics="fast")
    st = _oracle_state(oracle, cfg, inp, oracle.SQUARE_POW)
    S = cfg.n_substrates
    for step in range(2):
        sim.run(1)
        st.step(threads=oracle.max_threads())
        sim.sync()
        got, want = sim.densities().reshape(S, -1), st.dens.reshape(S, -1)
        for s in range(S):
            assert normwise(got[s], want[s]) <= 1e-10, (k, step, s)
        assert normwise(sim.positions(), st.pos) <= 1e-12, (k, step)
        assert normwise(sim.velocities(), st.vel) <= 1e-12, (k, step)
        b = sim.bins()
        assert np.array_equal(b["bin_start"], st.bins.bin_start), (k, step)
        assert np.array_equal(b["nonempty"], st.bins.nonempty), (k, step)
        assert np.array_equal(b["bin_cells"], st.bins.bin_cells), (k, step)
    sim.close()


def test_out_of_bounds_position_raises_domain_error():
    mesh = cg.CartesianMesh(4, 4, 4)
    cont = cg.CellContainer(mesh)
    cont.new_cell([10.0, 10.0, 10.0])
    cont.new_cell([10.0, 10.0, 80.0])  # on the upper face: half-open -> outside
    with pytest.raises(cg.DomainError):
        cg.rebin_cells(cont)
    cont.cells[1].position[2] = 79.0
    cg.rebin_cells(cont)  # the context recovers after the error
    assert cont.nonempty_voxels == sorted({mesh.voxel_of(c.position) for c in cont.cells})


def test_empty_and_single_cell_containers():
    mesh = cg.CartesianMesh(3, 3, 3)
    micro = cg.Microenvironment(mesh, [1000.0], [0.0], [5.0])
    cont = cg.CellContainer(mesh)
    cg.rebin_cells(cont)
    before = micro.densities.copy()
    cg.apply_cell_exchange(micro, cont, 0.1, 1.0, 1.0, 38.0)
    assert np.array_equal(micro.densities, before)
    rec = cg.update_velocities(cont, mesh, cg.InteractionParams(),
                               cg.MechanicsSchedule.cell_static(), cg.WorkerPool(2))
    assert rec.total_claims == 0
    cont.new_cell([30.0, 30.0, 30.0])
    cg.rebin_cells(cont)
    cg.update_velocities(cont, mesh, cg.InteractionParams(),
                         cg.MechanicsSchedule.cell_static(), cg.WorkerPool(1))
    assert cont.cells[0].velocity == [0.0, 0.0, 0.0]


def test_exchange_nonpositive_denominator_raises():
    mesh = cg.CartesianMesh(4, 4, 4)
    micro = cg.Microenvironment(mesh, [1000.0], [0.0], [38.0])
    cont = cg.CellContainer(mesh)
    cont.new_cell([10.0, 10.0, 10.0], radius=8.0)
    cg.rebin_cells(cont)
    with pytest.raises(cg.DomainError):
        cg.apply_cell_exchange(micro, cont, 1.0, secretion=0.0, uptake=-8.0, saturation=38.0)


@pytest.mark.parametrize("env", [{}, {"CELLGPU_VEL_DENSE_MIN": "100000"},
                                 {"CELLGPU_VEL_DENSE_MIN": "0"}, {"CELLGPU_VEL_EXACT": "lists"}])
def test_dense_voxels_take_the_overflow_kernel(oracle, monkeypatch, env):
    """Hundreds of candidates per cell: the warp-per-cell exact pass (default),
    the thread-level id-ordered queue in several walks (DENSE_MIN=100000),
    every cell through the warp pass (0), and the candidate-list kernels with
    the CTA-per-voxel overflow (lists); results stay bit-exact."""
    for var, val in env.items():
        monkeypatch.setenv(var, val)
    rng = np.random.default_rng(5)
    mesh = cg.CartesianMesh(3, 3, 3)
    n = 900
    pos = rng.uniform(1.0, 59.0, (n, 3))
    rad = rng.uniform(7.0, 10.0, n)
    ids = rng.permutation(10 * n)[:n]
    cont = container(mesh, pos, ids, rad)
    cg.update_velocities(cont, mesh, cg.InteractionParams(), cg.MechanicsSchedule.cell_static(),
                         cg.WorkerPool(1))
    got = np.array([c.velocity for c in cont.cells])
    m = oracle.mesh_struct(3, 3, 3)
    b = oracle.rebin(m, pos)
    exact = oracle.velocities(m, pos, rad, ids, b, square_mode=oracle.SQUARE_MUL)
    assert np.array_equal(got, exact)
    assert np.any(got != 0.0)


@pytest.mark.parametrize("env", [{}, {"CELLGPU_VEL_DENSE_MIN": "100000"}])
def test_exact_velocities_more_in_range_than_queues(oracle, monkeypatch, env):
    """300 cells inside a 4 um ball: every pair is in range (299 per cell),
    more than the warp pass's shared-memory capacity (256) and many times the
    thread queue (16): both fall back to repeated id-ordered walks."""
    for var, val in env.items():
        monkeypatch.setenv(var, val)
    rng = np.random.default_rng(11)
    mesh = cg.CartesianMesh(3, 3, 3)
    n = 300
    d = rng.normal(size=(n, 3))
    d *= (rng.uniform(0.0, 1.0, n) ** (1 / 3) * 4.0 / np.linalg.norm(d, axis=1))[:, None]
    pos = 30.0 + d
    rad = rng.uniform(7.0, 9.0, n)
    ids = rng.permutation(5 * n)[:n]
    cont = container(mesh, pos, ids, rad)
    cg.update_velocities(cont, mesh, cg.InteractionParams(), cg.MechanicsSchedule.cell_static(),
                         cg.WorkerPool(1))
    got = np.array([c.velocity for c in cont.cells])
    m = oracle.mesh_struct(3, 3, 3)
    exact = oracle.velocities(m, pos, rad, ids, oracle.rebin(m, pos), square_mode=oracle.SQUARE_MUL)
    assert np.array_equal(got, exact)
    assert np.all(np.any(got != 0.0, axis=1))


def test_exact_velocities_at_the_reach_far_from_the_origin(oracle):
    """The velocity walks pre-test in fp32 with a margin scaled by the mesh
    box (pretest_f32): pairs within a few ulp of the adhesion reach, on a mesh
    10 mm from the origin (fp32 coordinates there are ~1e-3 um apart), must
    still be summed exactly as the reference sums them."""
    rng = np.random.default_rng(23)
    o = (1.0e4, -2.0e4, 3.0e4)
    mesh = cg.CartesianMesh(4, 4, 4, origin=o)
    ma = cg.InteractionParams().adhesion_multiplier
    pos, rad = [], []
    for k in range(60):
        c = np.array(o) + rng.uniform(15.0, 65.0, 3)
        r1, r2 = rng.uniform(7.0, 9.0, 2)
        reach = ma * (r1 + r2)
        d = reach * (1.0 + rng.choice([-1, 1]) * rng.choice([1e-15, 1e-12, 1e-9, 1e-7, 1e-5]))
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        pos += [c, c + d * u]
        rad += [r1, r2]
    pos, rad = np.array(pos), np.array(rad)
    keep = np.all((pos > np.array(o) + 0.5) & (pos < np.array(o) + 79.5), axis=1)
    pos, rad = pos[keep], rad[keep]
    ids = rng.permutation(10 * len(pos))[:len(pos)]
    cont = container(mesh, pos, ids, rad)
    cg.update_velocities(cont, mesh, cg.InteractionParams(), cg.MechanicsSchedule.cell_static(),
                         cg.WorkerPool(1))
    got = np.array([c.velocity for c in cont.cells])
    m = oracle.mesh_struct(4, 4, 4, origin=o)
    exact = oracle.velocities(m, pos, rad, ids, oracle.rebin(m, pos), square_mode=oracle.SQUARE_MUL)
    assert np.array_equal(got, exact)
    assert np.any(got != 0.0)


def _prepared_vs_per_cell(mesh, pos, ids, rad, sec, upt, sat, dens0, substeps=2, dt=0.01):
    """cg_rebin_exchange + cg_exchange_prepared (coefficients once, records of
    the first cells inline) against apply_cell_exchange every substep."""
    import ctypes

    import torch

    from paper_2306_11544_b200 import _lib

    S, n = sec.shape
    cont = container(mesh, pos, ids, rad)
    micro = cg.Microenvironment(mesh, [1e5] * S, [0.1] * S)
    micro.densities = dens0
    for _ in range(substeps):
        cg.apply_cell_exchange(micro, cont, dt, sec, upt, sat)
    want = micro.densities.copy()

    dev = "cuda"
    t = lambda a, dt_=torch.float64: torch.as_tensor(np.ascontiguousarray(a), dtype=dt_, device=dev)
    nvox = mesh.voxel_count
    d = t(dens0.reshape(S, nvox))
    P = _lib.ptr
    b = {k: torch.zeros(m, dtype=torch.int32, device=dev) for k, m in
         (("voxel", n), ("bin_start", nvox + 1), ("bin_cells", n), ("by_id", n),
          ("nonempty", nvox), ("n_ne", 1))}
    ctx = _lib.Context(mesh, S, n, 0)
    satv = np.ascontiguousarray(np.broadcast_to(np.asarray(sat, np.float64), (S,)))
    L = _lib.load()
    # keep every device array referenced until the stream has consumed it
    tpos, tids, tsec, tupt = t(pos), t(ids, torch.int64), t(sec), t(upt)
    tvol = t(_lib.cell_volumes(rad))
    _lib.raise_for(L.cg_rebin_exchange(
        ctx.handle, n, P(tpos), P(tids), P(b["voxel"]), P(b["bin_start"]), P(b["bin_cells"]),
        P(b["by_id"]), P(b["nonempty"]), P(b["n_ne"]), dt, P(tsec), P(tupt),
        satv.ctypes.data_as(ctypes.c_void_p), P(tvol)), "cg_rebin_exchange")
    for _ in range(substeps):
        _lib.raise_for(L.cg_exchange_prepared(ctx.handle, P(d), n, P(b["nonempty"]), P(b["n_ne"])),
                       "cg_exchange_prepared")
    ctx.sync("prepared exchange")
    return d.cpu().numpy().reshape(want.shape), want


def test_prepared_exchange_bitwise(golden):
    mesh = mesh_from_arr(golden["ex_mesh"])
    pos, ids, rad = golden["ex_pos"], golden["ex_ids"], golden["ex_radius"]
    sec = golden["ext_ex_sec"][:, ids]
    upt = golden["ext_ex_upt"][:, ids]
    got, want = _prepared_vs_per_cell(mesh, pos, ids, rad, sec, upt, [38.0, 38.0],
                                      golden["ex_in"])
    assert np.array_equal(got, want)


def test_prepared_exchange_long_voxels_bitwise():
    """Voxels with more cells than the inline records (kRecCells = 4) continue
    from the slot arrays; ids shuffled against storage order."""
    rng = np.random.default_rng(7)
    mesh = cg.CartesianMesh(6, 5, 4, 20.0, 20.0, 20.0, (0.0, 0.0, 0.0))
    n = 600  # ~5 cells per voxel on average, many above 4
    pos = rng.uniform(0.0, [120.0, 100.0, 80.0], size=(n, 3))
    ids = rng.permutation(n).astype(np.int64) * 3 + 11
    rad = rng.uniform(7.0, 10.0, n)
    S = 3
    sec = rng.uniform(0.0, 1.0, (S, n))
    upt = rng.uniform(5.0, 15.0, (S, n))
    dens0 = rng.uniform(0.0, 38.0, (S, mesh.voxel_count))
    got, want = _prepared_vs_per_cell(mesh, pos, ids, rad, sec, upt, [38.0, 30.0, 20.0], dens0,
                                      substeps=3)
    assert np.array_equal(got, want)


def test_compute_gradients_bitwise(golden):
    """compute_gradients against the reference's own outputs (degenerate
    axes, anisotropic spacing, several substrates, both traversal modes)."""
    pool = cg.WorkerPool(1)
    for k in cases(golden, "grad"):
        mesh = mesh_from_arr(golden[f"{k}_mesh"])
        dens = golden[f"{k}_in"]
        S = dens.shape[0]
        micro = cg.Microenvironment(mesh, [1e3] * S, [0.1] * S)
        micro.densities = dens
        held = micro.gradients  # the reference writes the same array in place
        mode = cg.TraversalMode.OUTER_LOOP if int(k[4:]) % 2 else cg.TraversalMode.COLLAPSED
        recs = cg.compute_gradients(micro, mesh, mode, pool)
        assert len(recs) == S
        assert micro.gradients is held
        assert np.array_equal(micro.gradients, golden[f"{k}_out"]), k


def test_engine_gradients_match_api():
    """Simulation(gradients=True) refreshes the gradients after the substeps,
    equal to compute_gradients on the step's final field."""
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[0]
    sim = Simulation.from_config(cfg, make_inputs(cfg), gradients=True)
    sim.run(2)
    g = sim.gradients()
    mesh = cfg.mesh()
    micro = cg.Microenvironment(mesh, cfg.diffusion, cfg.decay)
    micro.densities = sim.densities()
    cg.compute_gradients(micro, mesh, cg.TraversalMode.COLLAPSED, cg.WorkerPool(1))
    assert np.array_equal(g, micro.gradients)
    sim.close()


def test_device_checksum_matches_reference_digests(golden):
    """cg_state_checksum (BLAKE2b-128 per cell on the GPU, XOR-reduced)
    reproduces the reference's state_checksum of its own final trajectory
    states, and the host restatement on arrays with signed zeros, NaNs,
    infinities and negative ids."""
    import torch

    from paper_2306_11544_b200 import _lib
    from paper_2306_11544_b200.checksum import checksum_arrays, device_checksum

    mesh = cg.CartesianMesh(2, 2, 2)
    ctx = _lib.Context(mesh, 0, 4096, 0)
    dev = lambda a, t=torch.float64: torch.as_tensor(np.ascontiguousarray(a), dtype=t, device="cuda")
    for tag in ("ref", "ext"):
        pos, vel = golden[f"{tag}_traj_pos"], golden[f"{tag}_traj_vel"]
        ids = np.arange(pos.shape[0], dtype=np.int64)
        tids, tpos, tvel = dev(ids, torch.int64), dev(pos), dev(vel)
        got = device_checksum(ctx, len(ids), tids, tpos, tvel)
        assert got == str(golden[f"{tag}_traj_checksums"][-1]), tag
    rng = np.random.default_rng(5)
    n = 3001
    pos = rng.normal(size=(n, 3))
    vel = rng.normal(size=(n, 3))
    pos[0] = [0.0, -0.0, np.inf]
    vel[1] = [np.nan, -np.inf, 1e-310]
    ids = rng.integers(-2**62, 2**62, n)
    tids, tpos, tvel = dev(ids, torch.int64), dev(pos), dev(vel)
    assert device_checksum(ctx, n, tids, tpos, tvel) == checksum_arrays(ids, pos, vel)
    assert device_checksum(ctx, 0, tids, tpos, tvel) == "0" * 32


def test_engine_checksum_matches_host():
    from paper_2306_11544_b200.checksum import checksum_arrays
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[0]
    inp = make_inputs(cfg)
    sim = Simulation.from_config(cfg, inp)
    sim.run(2)
    assert sim.checksum() == checksum_arrays(inp.ids if inp.ids is not None else np.arange(sim.n),
                                             sim.positions(), sim.velocities())
    sim.close()


@pytest.mark.parametrize("bad", [None, "nan", "neg", "inf"])
def test_check_state_device(bad):
    """cg_check_state = Microenvironment.check_state (core.py:142-144):
    NumericError for a non-finite or negative value, silent otherwise."""
    import torch

    from paper_2306_11544_b200 import _lib
    from paper_2306_11544_b200.core import CartesianMesh
    from paper_2306_11544_b200.errors import NumericError

    mesh = CartesianMesh(7, 5, 3, 20.0, 20.0, 20.0, (0.0, 0.0, 0.0))
    ctx = _lib.Context(mesh, 2, 16, 0)
    d = torch.full((2, mesh.voxel_count), 3.0, dtype=torch.float64, device="cuda")
    d[1, 0] = 0.0  # zero is allowed
    if bad is not None:
        d[1, 57] = {"nan": float("nan"), "neg": -1e-300, "inf": float("inf")}[bad]
    torch.cuda.synchronize()
    _lib.raise_for(_lib.load().cg_check_state(ctx.handle, _lib.ptr(d)), "cg_check_state")
    if bad is None:
        ctx.sync("check_state")
    else:
        with pytest.raises(NumericError):
            ctx.sync("check_state")
    ctx.close()


def test_engine_check_state_raises():
    """The engine runs check_state on every step's final field (simulate.py:218)."""
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation
    from paper_2306_11544_b200.errors import NumericError

    cfg = CONFIGS[1]
    inp = make_inputs(cfg)
    sim = Simulation.from_config(cfg, inp)
    sim.run(1)
    sim.sync()  # a healthy step raises nothing
    sim.dens[2, 40 * 6400 + 40 * 80 + 40] = float("nan")  # spreads through the substeps
    sim.run(1)
    with pytest.raises(NumericError):
        sim.sync()
    sim.close()


@pytest.mark.parametrize("cfg_id,alloc,n_cells,numerics,chains", [
    (0, "torch", None, "exact", "1"), (0, "hostmem", None, "exact", "1"),
    (1, "hostmem", None, "exact", "1"), (1, "hostmem", None, "fast", "1"),
    (3, "hostmem", 20000, "exact", "1"), (3, "hostmem", 20000, "exact", "0"),
    (3, "hostmem", 20000, "fast", "1"),
])
def test_step_host_matches_device_loop(monkeypatch, cfg_id, alloc, n_cells, numerics, chains):
    """Simulation.step_host (state round-tripped through pinned host buffers,
    copies overlapped with the step) gives the device-resident run's state,
    with torch's pinned tensors or the package's cudaHostAlloc buffers.
    Config 1 / 3 host-driven steps run one substrate chain per substrate
    (substrate windows of the register-line, relay and segmented kernels),
    device-resident steps all substrates per launch; CELLGPU_SUBSTRATE_CHAINS=0
    keeps one chain."""
    import torch

    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation
    from paper_2306_11544_b200.hostmem import host_like

    monkeypatch.setenv("CELLGPU_SUBSTRATE_CHAINS", chains)
    # config 3's multi-wave sweeps run the mechanics after the substeps by
    # default (no substrate chains); force the concurrent layout here
    monkeypatch.setenv("CELLGPU_OVERLAP", "1")
    cfg = CONFIGS[cfg_id]
    inp = make_inputs(cfg, n_cells)
    ref = Simulation.from_config(cfg, inp, numerics=numerics)
    ref.run(4)
    want = (ref.densities(), ref.positions(), ref.velocities())
    ref.close()
    sim = Simulation.from_config(cfg, inp, numerics=numerics)
    if cfg_id in (1, 3):
        from paper_2306_11544_b200 import _lib

        assert _lib.load().cg_engine_substrate_chains(sim._eng) == (cfg.n_substrates if chains == "1" else 1)
    src = (sim.densities(), sim.positions(), sim.previous_velocities())
    if alloc == "torch":
        h = [torch.from_numpy(a).pin_memory() for a in src]
        o = [torch.empty_like(t).pin_memory() for t in h]
    else:
        h = [host_like(a) for a in src]
        o = [host_like(np.zeros_like(a)) for a in src]
        assert all(t.is_pinned() for t in h + o)
    for _ in range(4):
        sim.step_host(h[0], h[1], h[2], o[0], o[1], o[2])
        h, o = o, h  # outputs feed the next step (AB2: previous velocity = velocity)
    torch.cuda.synchronize()
    sim.sync()
    assert np.array_equal(h[0].numpy(), want[0])
    assert np.array_equal(h[1].numpy(), want[1])
    assert np.array_equal(h[2].numpy(), want[2])
    sim.close()


def test_division_draws_golden(golden):
    """cg_division_draws vs the reference's division_draws, bit for bit."""
    from paper_2306_11544_b200 import division_draws

    seeds, idst = golden["div_draws_seed"], golden["div_draws_id_step"]
    for k in range(0, len(seeds), 7):
        assert division_draws(int(seeds[k]), int(idst[k, 0]), int(idst[k, 1])) == \
            tuple(golden["div_draws"][k])


@pytest.mark.parametrize("mode", ["objects", "arrays"])
def test_divisions_golden(golden, mode):
    """attempt_divisions against the reference run (tests/golden, several
    steps with growth, shuffled storage, cells near the faces): which cells
    divide, daughter ids, storage order and daughter positions bit for bit
    (the direction's cos / sin come from the host's libm, as CPython's)."""
    import paper_2306_11544_b200 as cb
    from paper_2306_11544_b200.population import attempt_divisions

    k = 0
    while f"div{k}_mesh" in golden:
        a = golden[f"div{k}_mesh"]
        mesh = cb.CartesianMesh(int(a[0]), int(a[1]), int(a[2]), float(a[3]), float(a[4]),
                                float(a[5]), (float(a[6]), float(a[7]), float(a[8])))
        dt, seed, steps = golden[f"div{k}_args"]
        p0 = f"div{k}_s0_"
        if mode == "objects":
            cont = cb.CellContainer(mesh)
            for cid, pos, rad, rate in zip(golden[p0 + "ids"], golden[p0 + "pos"],
                                           golden[p0 + "radius"], golden[p0 + "rate"]):
                cont.append_cell(cb.Cell(id=int(cid), position=[float(x) for x in pos],
                                         velocity=[0.0, 0.0, 0.0], radius=float(rad),
                                         division_rate=float(rate)))
            cb.rebin_cells(cont)
        else:
            cont = cb.CellContainer.from_arrays(mesh, golden[p0 + "pos"], golden[p0 + "radius"],
                                                ids=golden[p0 + "ids"],
                                                division_rate=golden[p0 + "rate"])
            cb.rebin_cells(cont)
        for st in range(int(steps)):
            p = f"div{k}_s{st}_"
            if mode == "objects":
                ids = np.array([c.id for c in cont.cells])
                pos = np.array([c.position for c in cont.cells])
            else:
                d = cont.device_cells()
                ids, pos = d.ids.cpu().numpy(), d.pos.cpu().numpy()
            np.testing.assert_array_equal(ids, golden[p + "ids"])
            np.testing.assert_array_equal(pos, golden[p + "pos"])
            got = attempt_divisions(cont, seed=int(seed), dt=float(dt), mesh=mesh, step=st,
                                    cap=10**6)
            want_ids = golden[p + "d_ids"]
            if mode == "objects":
                np.testing.assert_array_equal([d.id for d in got], want_ids)
                dpos = np.array([d.position for d in got]).reshape(-1, 3)
            else:
                np.testing.assert_array_equal(got, want_ids)
                dpos = cont.device_cells().pos[len(ids):].cpu().numpy()
            np.testing.assert_array_equal(dpos, golden[p + "d_pos"].reshape(-1, 3))
        k += 1


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_voxel_sorted_storage_same_results_per_id(numerics):
    """Voxel-sorted storage (the reference's StorageOrder.voxel_sorted,
    population.py:132-135 every k steps, simulate.py:156-158, 209-212) only
    moves cells in storage: per cell id the state after 5 steps (resorts
    before step 1 and after steps 2 and 4) equals the append-order run's bit
    for bit, and the storage is (voxel, id) sorted after a resort."""
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[1]
    inp = make_inputs(cfg, 30000)
    ref = Simulation.from_config(cfg, inp, numerics=numerics)
    ref.run(5)
    want = (ref.densities(), ref.positions(), ref.velocities())
    ref.close()
    sim = Simulation.from_config(cfg, inp, numerics=numerics, resort_every=2)
    b = sim.bins()
    ids = sim.cell_ids()
    key = b["voxel"].astype(np.int64) * (1 << 32) + ids
    assert np.all(np.diff(key) > 0), "storage is (voxel, id) sorted"
    assert np.array_equal(b["bin_cells"], np.arange(len(ids)))
    sim.run(5)
    sim.sync()
    ids = sim.cell_ids()
    o = np.argsort(ids)
    assert np.array_equal(ids[o], np.arange(len(ids)))
    assert np.array_equal(sim.densities(), want[0])
    assert np.array_equal(sim.positions()[o], want[1])
    assert np.array_equal(sim.velocities()[o], want[2])
    sim.close()


def test_engine_divisions_vs_oracle(oracle):
    """run_simulation's division pass inside the engine loop (simulate.py:
    205-206, population.py:77-129): 400 config-0 cells with per-cell rates
    0.5-2 / min divide over 4 steps; after every step (engine step + division
    pass + graph recapture for the new count) the storage, ids, positions,
    velocities, AB2 state and fields equal the oracle's step + division pass
    bit for bit."""
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[0]
    n0 = 400
    inp = make_inputs(cfg, n0)
    rate = np.random.default_rng(5).uniform(0.5, 2.0, n0)
    seed = 9
    sim = Simulation.from_config(cfg, inp, division_rate=rate, division_seed=seed, capacity=3000)
    m = oracle.mesh_from(cfg.mesh())
    cur = dict(dens=inp.densities.copy(), pos=inp.positions.copy(), radius=inp.radius.copy(),
               ids=inp.ids.copy(), sec=inp.secretion.copy(), upt=inp.uptake.copy(),
               vel=np.zeros((n0, 3)), prev=np.zeros((n0, 3)), rate=rate.copy())
    next_id = n0
    grew = 0
    for step in range(4):
        st = oracle.OracleState(
            m, cur["dens"], cur["pos"], cur["radius"], cur["ids"], cfg.diffusion, cfg.decay,
            secretion=cur["sec"], uptake=cur["upt"], saturation=[cfg.saturation],
            bc=oracle.BC_DIRICHLET, dirichlet=cfg.dirichlet, dt_diff=cfg.dt_diffusion,
            dt_mech=cfg.dt_mechanics, substeps=cfg.substeps, integrator=oracle.AB2,
            square_mode=oracle.SQUARE_MUL, repulsion=cfg.repulsion, adhesion=cfg.adhesion,
            adhesion_multiplier=cfg.adhesion_multiplier, vel=cur["vel"], prev_vel=cur["prev"])
        st.step(threads=4)
        par, dpos = oracle.divisions(m, st.ids, st.pos, st.radius, cur["rate"], cfg.dt_mechanics,
                                     seed, step, 10**6)
        k = len(par)
        grew += k
        cur = dict(dens=st.dens.copy(), pos=np.concatenate([st.pos, dpos]),
                   radius=np.concatenate([st.radius, st.radius[par]]),
                   ids=np.concatenate([st.ids, np.arange(next_id, next_id + k)]),
                   sec=np.concatenate([cur["sec"], cur["sec"][:, par]], axis=1),
                   upt=np.concatenate([cur["upt"], cur["upt"][:, par]], axis=1),
                   vel=np.concatenate([st.vel, st.vel[par]]),
                   prev=np.concatenate([st.prev_vel, st.prev_vel[par]]),
                   rate=np.concatenate([cur["rate"], cur["rate"][par]]))
        next_id += k
        sim.run(1)
        sim.sync()
        assert sim.n == len(cur["ids"]), step
        assert np.array_equal(sim.cell_ids(), cur["ids"]), step
        assert np.array_equal(sim.densities(), cur["dens"]), step
        assert np.array_equal(sim.positions(), cur["pos"]), step
        assert np.array_equal(sim.velocities(), cur["vel"]), step
        assert np.array_equal(sim.previous_velocities(), cur["prev"]), step
    assert grew > 20, grew
    sim.close()


@pytest.mark.parametrize("case", ["neumann-1sub", "neumann-2sub-euler", "no-cells", "one-cell",
                                  "160-neumann"])
def test_engine_fast_numerics_variants_vs_oracle(oracle, case):
    """The fast kernels' other template branches against the oracle: Neumann
    faces (the reference's own boundary), one and two substrates, Euler,
    empty and single-cell populations (no exchange records), the 160^3
    kernels with Neumann faces; fields within 1e-10, cells within 1e-12."""
    from dataclasses import replace

    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    base = CONFIGS[3] if case.startswith("160") else CONFIGS[1]
    kw = dict(n_cells=5000)
    if case == "neumann-1sub":
        kw.update(bc="neumann", diffusion=base.diffusion[:1], decay=base.decay[:1],
                  dirichlet=base.dirichlet[:1])
    elif case == "neumann-2sub-euler":
        kw.update(bc="neumann", integrator="euler", diffusion=base.diffusion[:2],
                  decay=base.decay[:2], dirichlet=base.dirichlet[:2])
    elif case == "no-cells":
        kw.update(n_cells=0)
    elif case == "one-cell":
        kw.update(n_cells=1)
    else:
        kw.update(bc="neumann", n_cells=20000)
    cfg = replace(base, **kw)
    inp = make_inputs(cfg)
    # give the fields structure (Neumann runs would otherwise stay uniform)
    rng = np.random.default_rng(3)
    inp.densities[:] = rng.uniform(0.0, 50.0, inp.densities.shape)
    sim = Simulation.from_config(cfg, inp, numerics="fast")
    st = _oracle_state(oracle, cfg, inp, oracle.SQUARE_POW)
    S = cfg.n_substrates
    for step in range(2):
        sim.run(1)
        st.step(threads=oracle.max_threads())
        sim.sync()
        got, want = sim.densities().reshape(S, -1), st.dens.reshape(S, -1)
        for s in range(S):
            assert normwise(got[s], want[s]) <= 1e-10, (case, step, s)
        if cfg.n_cells:
            assert normwise(sim.positions(), st.pos) <= 1e-12, (case, step)
            if np.max(np.abs(st.vel)) > 0:
                assert normwise(sim.velocities(), st.vel) <= 1e-12, (case, step)
            assert np.array_equal(sim.bins()["bin_start"], st.bins.bin_start), (case, step)
    sim.close()


def test_fast_lod_availability_and_errors():
    """cg_fast_lod_available: cubic 80^3 / 160^3 and 256 x 256 planes have
    fast kernels, other meshes do not -- and the fast calls say so (CG_STATE)
    instead of running anything."""
    import ctypes

    import torch

    from paper_2306_11544_b200 import _lib

    L = _lib.load()
    vp = ctypes.c_void_p
    cases = [((80, 80, 80), True), ((160, 160, 160), True), ((256, 256, 32), True),
             ((20, 20, 20), False), ((80, 80, 40), False), ((33, 17, 9), False)]
    for (nx, ny, nz), want in cases:
        mesh = cg.CartesianMesh(nx, ny, nz)
        ctx = _lib.Context(mesh, 2, 16, 0)
        ctx.bind_stream()
        assert (L.cg_fast_lod_available(ctx.handle) == 1) == want, (nx, ny, nz)
        if not want:
            dens = torch.zeros((2, mesh.voxel_count), dtype=torch.float64, device="cuda")
            D = np.array([1e3, 1e3])
            K = np.array([0.1, 0.1])
            code = L.cg_lod_step_fast(ctx.handle, _lib.ptr(dens), D.ctypes.data_as(vp),
                                      K.ctypes.data_as(vp), 0.01, 0, None, 0)
            assert code == 3, code  # CG_STATE -> ContainerStateError
        ctx.close()
    # z slabs of 80 x 80 / 160 x 160 planes (configs 1-3 split over ranks):
    # the plane kernel is fast, the z solve the slab's exact block solve
    for n, nz_loc in [(80, 40), (160, 80), (80, 7)]:
        ctx = _lib.Context(cg.CartesianMesh(n, n, nz_loc), 2, 16, 0)
        starts = (ctypes.c_int * 3)(0, nz_loc, 2 * nz_loc)
        _lib.raise_for(L.cg_ctx_set_slab_bounds(ctx.handle, 0, 2, 2 * nz_loc, starts), "slab")
        assert L.cg_fast_lod_available(ctx.handle) == 1, (n, nz_loc)
        ctx.close()


def test_slab_context_calls_validate_their_arguments():
    """The z-slab C-ABI refuses what it cannot do instead of running it:
    substrate windows out of range (DomainError), block / deferral calls on
    a context that is not a slab of >= 2 ranks (ContainerStateError), a
    deferred correction without the fast slab kernels."""
    import ctypes

    from paper_2306_11544_b200 import _lib

    L = _lib.load()
    ctx = _lib.Context(cg.CartesianMesh(20, 20, 10), 2, 16, 0)
    assert L.cg_ctx_set_substrate_window(ctx.handle, 0, 3) == 1  # CG_DOMAIN
    assert L.cg_ctx_set_substrate_window(ctx.handle, -1, 1) == 1
    assert L.cg_ctx_set_substrate_window(ctx.handle, 1, 1) == 0
    assert L.cg_ctx_set_substrate_window(ctx.handle, 0, 0) == 0
    assert L.cg_zslab_defer(ctx.handle, None) == 3          # not a slab: CG_STATE
    assert L.cg_zslab_pack_blocks(ctx.handle, None, None) == 3
    starts = (ctypes.c_int * 3)(0, 10, 20)
    _lib.raise_for(L.cg_ctx_set_slab_bounds(ctx.handle, 0, 2, 20, starts), "slab")
    assert L.cg_zslab_block_lines(ctx.handle) == 200          # ceil(20 * 20 / 2)
    # 20 x 20 planes have no fast kernels: nothing to defer into
    assert L.cg_zslab_defer(ctx.handle, ctypes.c_void_p(1)) == 3
    assert L.cg_zslab_defer(ctx.handle, None) == 0
    ctx.close()
