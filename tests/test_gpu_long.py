"""Long-horizon parity: config 0's whole run (60 mechanics steps = 6 sim-min)
through the step engine against the reference's own run
(tests/golden/traj60.npz, made by tests/golden/make_golden.py traj60).

Exact numerics: every step's voxel keys bit for bit, so the exchange sees the
reference's bins and the fields stay bit-identical to the reference's (every
step's digest); positions / velocities within 1e-12 normwise (the GPU squares
with t*t where CPython calls libm pow).  Fast numerics: the same bins every
step, fields within 1e-10, positions / velocities within 1e-12 normwise."""

import hashlib
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def traj60():
    with np.load(os.path.join(HERE, "golden", "traj60.npz")) as z:
        return {k: z[k] for k in z.files}


def normwise(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def _sim(tag, numerics):
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[0]
    inp = make_inputs(cfg)
    if tag == "ext":
        return Simulation.from_config(cfg, inp, numerics=numerics)
    # the reference's own semantics: Neumann faces, Euler, scalar uptake 10 on s0
    from paper_2306_11544_b200.mechanics import InteractionParams

    n = cfg.n_cells
    return Simulation(
        cfg.mesh(), diffusion=cfg.diffusion, decay=cfg.decay, densities=inp.densities,
        positions=inp.positions, radius=inp.radius, ids=inp.ids,
        secretion=np.zeros((1, n)), uptake=np.full((1, n), 10.0), saturation=cfg.saturation,
        bc="neumann", params=InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier),
        dt_diffusion=cfg.dt_diffusion, dt_mechanics=cfg.dt_mechanics, integrator="euler",
        numerics=numerics)


@pytest.mark.parametrize("numerics", ["exact", "fast"])
@pytest.mark.parametrize("tag", ["ref", "ext"])
def test_config0_full_run_vs_reference(traj60, tag, numerics):
    sim = _sim(tag, numerics)
    vox = traj60[f"{tag}_voxel"]
    for step in range(len(vox)):
        sim.run(1)
        sim.sync()
        b = sim.bins()
        assert np.array_equal(b["voxel"], vox[step].astype(np.int32)), (tag, numerics, step)
        dens = sim.densities()
        if numerics == "exact":
            assert hashlib.sha256(dens.tobytes()).hexdigest() == traj60[f"{tag}_dens_sha"][step], step
        if (step + 1) % 10 == 0:
            k = (step + 1) // 10 - 1
            assert normwise(sim.positions(), traj60[f"{tag}_pos10"][k]) <= 1e-12, (tag, step)
            assert normwise(sim.velocities(), traj60[f"{tag}_vel10"][k]) <= 1e-12, (tag, step)
    want = traj60[f"{tag}_dens"]
    if numerics == "exact":
        assert np.array_equal(sim.densities(), want)
    else:
        S = want.shape[0]
        got = sim.densities().reshape(S, -1)
        for s in range(S):
            assert normwise(got[s], want[s]) <= 1e-10, s
    sim.close()


@pytest.mark.parametrize("k,steps", [(1, 30), (2, 20), (3, 20), (4, 20)])
@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_config_steps_vs_oracle(numerics, k, steps):
    """The headline workload (BASELINE config 1: 80^3 x 3 substrates, 100k
    cells, Dirichlet + AB2 + per-cell rates) for 30 mechanics steps (3
    sim-min), and configs 2 (the dense spheroid, 200k cells), 3 (160^3 x 4,
    1M cells) and 4 (256 x 256 x 32 x 4, 1M cells) for 20 (2 sim-min),
    through the graph-replayed engine beside the oracle, compared after
    every step.  Exact numerics: fields, positions, velocities and bins
    bit for bit (oracle squaring with t*t, as the GPU).  Fast numerics (the
    bench's mode): bins identical every step, fields within 1e-10 per
    substrate, positions and velocities within 1e-12 normwise of the oracle
    in the reference's arithmetic (libm pow) -- no drift over the run."""
    from oracle import oracle as o
    from paper_2306_11544_b200.configs import CONFIGS, make_inputs
    from paper_2306_11544_b200.engine import Simulation

    cfg = CONFIGS[k]
    inp = make_inputs(cfg)
    sim = Simulation.from_config(cfg, inp, numerics=numerics)
    st = o.OracleState(
        o.mesh_from(cfg.mesh()), inp.densities, inp.positions, inp.radius, inp.ids,
        cfg.diffusion, cfg.decay, secretion=inp.secretion, uptake=inp.uptake,
        saturation=[cfg.saturation] * cfg.n_substrates, bc=o.BC_DIRICHLET,
        dirichlet=cfg.dirichlet, dt_diff=cfg.dt_diffusion, dt_mech=cfg.dt_mechanics,
        substeps=cfg.substeps, integrator=o.AB2,
        square_mode=o.SQUARE_MUL if numerics == "exact" else o.SQUARE_POW,
        repulsion=cfg.repulsion, adhesion=cfg.adhesion,
        adhesion_multiplier=cfg.adhesion_multiplier)
    S = cfg.n_substrates
    worst = 0.0
    for step in range(steps):
        sim.run(1)
        st.step(threads=o.max_threads())
        sim.sync()
        b = sim.bins()
        assert np.array_equal(b["voxel"], st.bins.voxel), step
        assert np.array_equal(b["bin_cells"], st.bins.bin_cells), step
        if numerics == "exact":
            assert np.array_equal(sim.densities(), st.dens), step
            assert np.array_equal(sim.positions(), st.pos), step
            assert np.array_equal(sim.velocities(), st.vel), step
        else:
            got, want = sim.densities().reshape(S, -1), st.dens.reshape(S, -1)
            for s in range(S):
                err = normwise(got[s], want[s])
                worst = max(worst, err)
                assert err <= 1e-10, (step, s, err)
            assert normwise(sim.positions(), st.pos) <= 1e-12, step
            assert normwise(sim.velocities(), st.vel) <= 1e-12, step
    sim.close()
