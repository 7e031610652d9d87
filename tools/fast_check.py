"""Fast vs exact engine numerics on one config: per-step field / kinematics
errors and bins, then device ms per step and per-stage times of each mode.

    python tools/fast_check.py [CONFIG] [STEPS]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402


def normwise(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def timed(sim, steps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sim.run(1)
    sim.sync()
    a.record(sim.stream)
    sim.run(steps)
    b.record(sim.stream)
    b.synchronize()
    return a.elapsed_time(b) / steps


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = CONFIGS[k]
    inp = make_inputs(cfg)
    ex = Simulation.from_config(cfg, inp, numerics="exact")
    fa = Simulation.from_config(cfg, inp, numerics="fast")
    S = cfg.n_substrates
    for st in range(steps):
        ex.run(1)
        fa.run(1)
        ex.sync()
        fa.sync()
        de, df = ex.densities().reshape(S, -1), fa.densities().reshape(S, -1)
        ferr = max(normwise(df[s], de[s]) for s in range(S))
        perr = normwise(fa.positions(), ex.positions())
        verr = normwise(fa.velocities(), ex.velocities())
        be, bf = ex.bins(), fa.bins()
        same = all(np.array_equal(be[x], bf[x]) for x in ("voxel", "bin_start", "bin_cells", "nonempty"))
        print(f"cfg {k} step {st}: field {ferr:.2e} pos {perr:.2e} vel {verr:.2e} bins_equal {same}",
              flush=True)
    for name, sim in (("exact", ex), ("fast", fa)):
        ms = timed(sim, 20)
        print(f"{name}: {ms:.4f} ms/step, launches/step {sim.launches_per_step}", flush=True)
    for name, sim in (("exact", ex), ("fast", fa)):
        st = sim.time_stages(20)
        print(name, "stages us:", {kk: round(v * 1e3, 1) for kk, v in st.items()}, flush=True)
    ex.close()
    fa.close()


if __name__ == "__main__":
    main()
