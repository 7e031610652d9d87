"""Per-CTA phase cycles of the last k_plane_xy launch (probe build, config 1)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
os.environ["CELLGPU_LIB"] = os.path.abspath("paper_2306_11544_b200/libcellgpu_probe.so")
from paper_2306_11544_b200 import _lib
from paper_2306_11544_b200.configs import CONFIGS, make_inputs
from paper_2306_11544_b200.engine import Simulation

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
for reg in ("0", "1"):
    os.environ["CELLGPU_REGLINES"] = reg
    sim = Simulation.from_config(cfg, make_inputs(cfg))
    sim.run(2, graph=False)
    sim.sync()
    buf = (ctypes.c_longlong * (8 * 1024))()
    _lib.load().cg_probe_read(buf, 8 * 1024)
    a = np.frombuffer(buf, dtype=np.int64).reshape(-1, 8)[: cfg.mesh().nz * len(cfg.diffusion)]
    d = np.diff(a[:, :7], axis=1)
    names = ["issue", "wait", "exch", "x", "y", "store"]
    c0 = a[:, 7] - a[:, 2]
    nq = None
    print(f"   first exchange chunk (mark7 - mark2): mean {c0.mean():.0f} max {c0.max():.0f}")
    print(f"reglines={reg}: mean cycles " + ", ".join(f"{n} {v:.0f}" for n, v in zip(names, d.mean(0))) +
          f" | max total {d.sum(1).max():.0f}, start spread {a[:,0].max()-a[:,0].min()}")
