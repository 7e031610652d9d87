"""GPU <-> CPU equivalence report (the reference's verify_equivalence idea,
harness.py:292-333, for this path): run a BASELINE config for a few
mechanics steps through the step engine and through the CPU oracle side by
side, and print per step how far apart fields, positions, velocities, bins
and the state checksum are.

    python tools/verify_equivalence.py [--config 1] [--steps 3] [--threads N]

The oracle (oracle/cellref.c) is test infrastructure; this tool is a checker
like tests/ and never part of the product path.  Exit status 1 when a step
leaves the parity bars (fields, bins, non-empty lists bitwise; positions /
velocities bitwise against the oracle's t*t mode).
"""
import argparse
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as o  # noqa: E402
from paper_2306_11544_b200.checksum import checksum_arrays  # noqa: E402
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402


def rel(a, b):
    d = np.abs(a - b).max() if a.size else 0.0
    s = np.abs(b).max() if b.size else 0.0
    return float(d / s) if s > 0 else float(d)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    o.build()
    cfg = CONFIGS[args.config]
    inp = make_inputs(cfg)
    sim = Simulation.from_config(cfg, inp)
    st = o.OracleState(
        o.mesh_from(cfg.mesh()), inp.densities, inp.positions, inp.radius, inp.ids,
        cfg.diffusion, cfg.decay, secretion=inp.secretion, uptake=inp.uptake,
        saturation=[cfg.saturation] * cfg.n_substrates,
        bc=o.BC_DIRICHLET if cfg.bc == "dirichlet" else o.BC_NEUMANN,
        dirichlet=cfg.dirichlet, dt_diff=cfg.dt_diffusion, dt_mech=cfg.dt_mechanics,
        substeps=cfg.substeps, integrator=o.AB2 if cfg.integrator == "ab2" else o.EULER,
        square_mode=o.SQUARE_MUL, repulsion=cfg.repulsion, adhesion=cfg.adhesion,
        adhesion_multiplier=cfg.adhesion_multiplier)
    threads = args.threads or o.max_threads()
    ids = inp.ids if inp.ids is not None else np.arange(sim.n)
    print(f"config {args.config} ({cfg.name}): {cfg.voxel_count} voxels x {cfg.n_substrates}, "
          f"{sim.n} cells, oracle on {threads} threads")
    print(f"{'step':>4} {'fields max rel':>15} {'fields ==':>9} {'pos ==':>7} {'vel ==':>7} "
          f"{'pos max rel':>12} {'bins ==':>7} {'checksum ==':>11}")
    ok = True
    for step in range(args.steps):
        sim.run(1)
        st.step(threads=threads)
        sim.sync()
        d, p, v = sim.densities(), sim.positions(), sim.velocities()
        b = sim.bins()
        f_eq = np.array_equal(d, st.dens)
        p_eq, v_eq = np.array_equal(p, st.pos), np.array_equal(v, st.vel)
        b_eq = (np.array_equal(b["bin_start"], st.bins.bin_start)
                and np.array_equal(b["bin_cells"], st.bins.bin_cells)
                and np.array_equal(b["nonempty"], st.bins.nonempty))
        c_eq = sim.checksum() == checksum_arrays(ids, st.pos, st.vel)
        print(f"{step:4d} {max(rel(d[s], st.dens[s]) for s in range(d.shape[0])):15.3e} "
              f"{str(f_eq):>9} {str(p_eq):>7} {str(v_eq):>7} {rel(p, st.pos):12.3e} "
              f"{str(b_eq):>7} {str(c_eq):>11}")
        ok = ok and f_eq and p_eq and v_eq and b_eq and c_eq
    sim.close()
    print("equivalent" if ok else "NOT equivalent")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
