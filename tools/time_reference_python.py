"""Time the reference's OWN Python CPU path (cellbench, read-only import from
/root/reference) on BASELINE config 1's shape, in run_simulation's order
(simulate.py:169-202): per substep apply_cell_exchange for each substrate +
lod_step, then update_velocities, integrate_positions, rebin_cells.  The
reference has no Dirichlet faces, AB2 or per-cell rates,
so this is its native semantics on the same mesh, substrates and cells
(scalar uptake/secretion).  Build-container only (the reference does not
travel to the GPU box); the result is committed as
profiles/r6_reference_python.json and reported by bench.py as a probe.

    python tools/time_reference_python.py [WORKERS ...]
"""
import json
import os
import platform
import sys
import time

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True

import cellbench as cb  # noqa: E402

from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402


def cpu_model():
    for ln in open("/proc/cpuinfo"):
        if ln.startswith("model name"):
            return ln.split(":", 1)[1].strip()
    return platform.processor()


def main():
    cfg = CONFIGS[1]
    inp = make_inputs(cfg)
    m = cfg.mesh()
    mesh = cb.CartesianMesh(m.nx, m.ny, m.nz, m.dx, m.dy, m.dz, m.origin)
    params = cb.InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier)
    out = {"config": "BASELINE config 1 shape (80^3 x 3 substrates, 100k cells, 10 substeps)",
           "semantics": "the reference's own (Neumann, Euler, scalar rates per substrate)",
           "host": cpu_model(), "cores": os.cpu_count(), "runs": []}
    for workers in [int(w) for w in (sys.argv[1:] or ["1", str(os.cpu_count())])]:
        micro = cb.Microenvironment(mesh, list(cfg.diffusion), list(cfg.decay), list(cfg.dirichlet))
        cont = cb.CellContainer(mesh)
        for i, p in enumerate(inp.positions):
            cont.new_cell([float(x) for x in p], radius=float(inp.radius[i]))
        cb.rebin_cells(cont)
        pool = cb.WorkerPool(workers)
        sched = cb.MechanicsSchedule.nonempty_voxel(16)
        t = {"exchange": 0.0, "lod": 0.0, "velocity": 0.0, "integrate": 0.0, "rebin": 0.0}
        t0 = time.perf_counter()
        for _ in range(cfg.substeps):
            a = time.perf_counter()
            for s in range(cfg.n_substrates):
                cb.apply_cell_exchange(micro, cont, cfg.dt_diffusion, 0.5, 10.0 if s == 0 else 0.0,
                                       cfg.saturation, substrate=s, pool=pool)
            b = time.perf_counter()
            cb.lod_step(micro, mesh, cfg.dt_diffusion, cb.TraversalMode.OUTER_LOOP, pool,
                        container=cont)
            c = time.perf_counter()
            t["exchange"] += b - a
            t["lod"] += c - b
        a = time.perf_counter()
        cb.update_velocities(cont, mesh, params, sched, pool)
        b = time.perf_counter()
        cb.integrate_positions(cont, mesh, cfg.dt_mechanics, pool)
        c = time.perf_counter()
        cb.rebin_cells(cont)
        d = time.perf_counter()
        t["velocity"], t["integrate"], t["rebin"] = b - a, c - b, d - c
        total = time.perf_counter() - t0
        pool.shutdown()
        units = cfg.voxel_count * cfg.n_substrates * cfg.substeps
        run = {"workers": workers, "s_per_step": total,
               "voxel_substrate_updates_per_s": units / total,
               "cell_updates_per_s": cfg.n_cells / total,
               "seconds": {k: round(v, 3) for k, v in t.items()}}
        print(json.dumps(run), flush=True)
        out["runs"].append(run)
    best = min(out["runs"], key=lambda r: r["s_per_step"])
    out["best"] = best
    path = os.path.join(ROOT, "profiles", "r6_reference_python.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
