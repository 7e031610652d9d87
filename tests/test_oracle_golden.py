"""The CPU oracle (oracle/cellref.c) against fixtures produced by the
reference itself (tests/golden/make_golden.py): every check is bit-for-bit.
This is what pins the oracle before it is trusted as the GPU's checker."""

import numpy as np
import pytest

from conftest import cases, refmesh_from_arr


def test_line_factors(golden, oracle):
    for k in cases(golden, "lf"):
        n, r, lam3 = golden[f"{k}_args"]
        inv, gam = oracle.line_factors(int(n), r, lam3)
        assert np.array_equal(inv, golden[f"{k}_inv"]), k
        assert np.array_equal(gam, golden[f"{k}_gamma"]), k


def test_voxel_of(golden, oracle):
    for k in cases(golden, "vo"):
        m = refmesh_from_arr(golden[f"{k}_mesh"])
        for p, want in zip(golden[f"{k}_pts"], golden[f"{k}_voxel"]):
            try:
                got = oracle.voxel_of(m, p)
            except oracle.OracleError:
                got = -1
            assert got == want, (k, p)


@pytest.mark.parametrize("ext", [False, True])
def test_lod_step(golden, oracle, ext):
    for k in cases(golden, "lod"):
        m = refmesh_from_arr(golden[f"{k}_mesh"])
        dens = golden[f"{k}_in"].copy()
        dt, steps = golden[f"{k}_dt_steps"]
        for _ in range(int(steps)):
            if ext:
                oracle.lod_step(m, dens, golden[f"{k}_D"], golden[f"{k}_K"], dt,
                                oracle.BC_DIRICHLET, golden[f"ext_{k}_dirichlet"], threads=2)
            else:
                oracle.lod_step(m, dens, golden[f"{k}_D"], golden[f"{k}_K"], dt, threads=2)
        want = golden[f"ext_{k}_out"] if ext else golden[f"{k}_out"]
        assert np.array_equal(dens, want), k


def test_rebin(golden, oracle):
    for k in cases(golden, "rb"):
        m = refmesh_from_arr(golden[f"{k}_mesh"])
        b = oracle.rebin(m, golden[f"{k}_pos"])
        assert np.array_equal(b.bin_start, golden[f"{k}_bin_start"]), k
        assert np.array_equal(b.bin_cells, golden[f"{k}_bin_cells"]), k
        assert np.array_equal(b.nonempty, golden[f"{k}_nonempty"]), k
        assert np.array_equal(b.voxel, golden[f"{k}_voxel"]), k


def test_exchange_scalar_and_per_cell(golden, oracle):
    m = refmesh_from_arr(golden["ex_mesh"])
    pos, ids, rad = golden["ex_pos"], golden["ex_ids"], golden["ex_radius"]
    vol = oracle.cell_volumes(rad)
    b = oracle.rebin(m, pos)
    dens = golden["ex_in"].copy()
    for k in range(3):
        dt, sec, upt, sat, s = golden[f"ex{k}_args"]
        oracle.exchange(m, dens, b, ids, vol, dt, sec, upt, sat, substrates=(int(s), int(s) + 1))
        assert np.array_equal(dens, golden[f"ex{k}_out"]), k
    # G4 restated extension: rates are indexed by id, the oracle by storage
    dens = golden["ex_in"].copy()
    sec = golden["ext_ex_sec"][:, ids]
    upt = golden["ext_ex_upt"][:, ids]
    oracle.exchange(m, dens, b, ids, vol, 0.01, sec, upt, [38.0, 38.0], threads=3)
    assert np.array_equal(dens, golden["ext_ex_out"])


def test_velocities(golden, oracle):
    for k in cases(golden, "ve"):
        m = refmesh_from_arr(golden[f"{k}_mesh"])
        pos = golden[f"{k}_pos"]
        b = oracle.rebin(m, pos)
        vel = oracle.velocities(m, pos, golden[f"{k}_radius"], golden[f"{k}_ids"], b, threads=2)
        assert np.array_equal(vel, golden[f"{k}_vel"]), k


def test_velocities_square_modes_agree_to_an_ulp(golden, oracle):
    """SQUARE_MUL (the GPU's t*t) differs from libm pow by at most an ulp per
    pair term; the accumulated velocities stay within 1e-12 normwise."""
    for k in cases(golden, "ve"):
        m = refmesh_from_arr(golden[f"{k}_mesh"])
        pos = golden[f"{k}_pos"]
        b = oracle.rebin(m, pos)
        v = oracle.velocities(m, pos, golden[f"{k}_radius"], golden[f"{k}_ids"], b,
                              square_mode=oracle.SQUARE_MUL)
        ref = golden[f"{k}_vel"]
        assert np.max(np.abs(v - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1e-300)


@pytest.mark.parametrize("ext", [False, True])
def test_integrate(golden, oracle, ext):
    for k in cases(golden, "in"):
        m = refmesh_from_arr(golden[f"{k}_mesh"])
        pos = golden[f"{k}_pos0"].copy()
        dt = float(golden[f"{k}_dt"][0])
        if ext:
            prev = golden[f"ext_{k}_prev"].copy()
            oracle.integrate(m, pos, golden[f"{k}_vel"], dt, prev_vel=prev,
                             integrator=oracle.AB2)
            assert np.array_equal(pos, golden[f"ext_{k}_pos"]), k
            assert np.array_equal(prev, golden[f"ext_{k}_prev_out"]), k
        else:
            oracle.integrate(m, pos, golden[f"{k}_vel"], dt)
            assert np.array_equal(pos, golden[f"{k}_pos"]), k


def _config0_state(oracle, ext):
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs

    cfg = CONFIGS[0]
    inp = make_inputs(cfg)
    m = oracle.mesh_from(cfg.mesh())
    kw = dict(dt_diff=cfg.dt_diffusion, dt_mech=cfg.dt_mechanics, substeps=cfg.substeps,
              saturation=[cfg.saturation])
    if ext:
        kw.update(secretion=inp.secretion, uptake=inp.uptake, bc=oracle.BC_DIRICHLET,
                  dirichlet=cfg.dirichlet, integrator=oracle.AB2)
    else:
        kw.update(secretion=np.zeros((1, cfg.n_cells)), uptake=np.full((1, cfg.n_cells), 10.0))
    return oracle.OracleState(m, inp.densities, inp.positions, inp.radius, inp.ids,
                              cfg.diffusion, cfg.decay, **kw)


@pytest.mark.parametrize("tag", ["ref", "ext"])
def test_config0_trajectory(golden, oracle, tag):
    """Five mechanics steps of config 0 through ref_mech_step: per-step
    state_checksum and density digest equal the reference run's."""
    import hashlib

    from paper_2306_11544_b200.checksum import checksum_arrays

    st = _config0_state(oracle, tag == "ext")
    sums = golden[f"{tag}_traj_checksums"]
    dsha = golden[f"{tag}_traj_dens_sha"]
    for step in range(len(sums)):
        st.step(threads=4)
        assert checksum_arrays(st.ids, st.pos, st.vel) == sums[step], step
        assert hashlib.sha256(st.dens.tobytes()).hexdigest() == dsha[step], step
    assert np.array_equal(st.dens, golden[f"{tag}_traj_dens"])
    assert np.array_equal(st.pos, golden[f"{tag}_traj_pos"])
    assert np.array_equal(st.vel, golden[f"{tag}_traj_vel"])


@pytest.fixture(scope="module")
def traj60():
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traj60.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("tag", ["ref", "ext"])
def test_config0_full_run(traj60, oracle, tag):
    """Config 0's whole run (60 mechanics steps, 6 sim-min) against the
    reference's own run (tests/golden/traj60.npz): every step's bins, state
    checksum and field digest bit for bit."""
    import hashlib

    from paper_2306_11544_b200.checksum import checksum_arrays

    st = _config0_state(oracle, tag == "ext")
    vox = traj60[f"{tag}_voxel"]
    for step in range(len(vox)):
        st.step(threads=4)
        assert np.array_equal(st.bins.voxel, vox[step]), step
        assert checksum_arrays(st.ids, st.pos, st.vel) == traj60[f"{tag}_checksums"][step], step
        assert hashlib.sha256(st.dens.tobytes()).hexdigest() == traj60[f"{tag}_dens_sha"][step], step
        if (step + 1) % 10 == 0:
            k = (step + 1) // 10 - 1
            assert np.array_equal(st.pos, traj60[f"{tag}_pos10"][k]), step
            assert np.array_equal(st.vel, traj60[f"{tag}_vel10"][k]), step
    assert np.array_equal(st.dens, traj60[f"{tag}_dens"])


def test_division_draws(golden, oracle):
    """population.py:44-51 counter RNG, bit for bit."""
    seeds = golden["div_draws_seed"]
    idst = golden["div_draws_id_step"]
    for k in range(len(seeds)):
        got = oracle.division_draws(int(seeds[k]), int(idst[k, 0]), int(idst[k, 1]))
        assert got == tuple(golden["div_draws"][k])


def _division_cases(golden):
    k = 0
    while f"div{k}_mesh" in golden:
        dt, seed, steps = golden[f"div{k}_args"]
        for st in range(int(steps)):
            yield k, st, float(dt), int(seed)
        k += 1


def test_divisions(golden, oracle):
    """population.py:77-129: which cells divide, in which order, and where the
    daughters land (libm cos/sin as CPython), bit for bit."""
    n_cases = 0
    for k, st, dt, seed in _division_cases(golden):
        m = refmesh_from_arr(golden[f"div{k}_mesh"])
        p = f"div{k}_s{st}_"
        ids = golden[p + "ids"]
        res = oracle.divisions(m, ids, golden[p + "pos"], golden[p + "radius"], golden[p + "rate"],
                               dt, seed, st, cap=10**6)
        parent, pos = res
        np.testing.assert_array_equal(ids[parent], golden[p + "parents"])
        np.testing.assert_array_equal(pos, golden[p + "d_pos"].reshape(-1, 3))
        # daughters take fresh ids in parent-id order (population.py:116-123)
        d_ids = golden[p + "d_ids"]
        np.testing.assert_array_equal(d_ids, ids.max() + 1 + np.arange(len(d_ids)))
        n_cases += 1
    assert n_cases >= 8


def test_divisions_capacity(golden, oracle):
    """population.py:98-102: the cap is checked before anything is appended."""
    m = refmesh_from_arr(golden["div0_mesh"])
    p = "div0_s0_"
    assert oracle.divisions(m, golden[p + "ids"], golden[p + "pos"], golden[p + "radius"],
                            golden[p + "rate"], 1.0, 1, 0, cap=8) is None
