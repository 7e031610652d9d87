"""Phase timeline of the last k_plane_seg launch (probe build): per CTA the
%globaltimer at kernel entry, after the PDL wait, plane staged, exchange
applied, x sweep, y sweep + store.  python tools/seg_phases.py [CONFIG]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ["CELLGPU_LIB"] = os.path.abspath("paper_2306_11544_b200/libcellgpu_probe.so")
from paper_2306_11544_b200 import _lib  # noqa: E402
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
sim = Simulation.from_config(cfg, make_inputs(cfg), numerics="fast")
for graph in (False, True):
    sim.run(2, graph=graph)
    sim.sync()
    buf = (ctypes.c_ulonglong * (8 * 2048))()
    _lib.load().cg_seg_probe_read(buf, 8 * 2048)
    n = cfg.mesh().nz * len(cfg.diffusion)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 8)[:n, :6].astype(np.int64)
    t0 = a[:, 0].min()
    a = a - t0
    names = ["entry", "pdl_wait", "staged", "exchange", "x", "y+store"]
    print(f"graph={graph}: {n} CTAs; ns from the first CTA entry")
    for k, nm in enumerate(names):
        print(f"  {nm:9s} min {a[:, k].min():7d} median {int(np.median(a[:, k])):7d} max {a[:, k].max():7d}")
    d = np.diff(a, axis=1)
    for k, nm in enumerate(names[1:]):
        print(f"  phase {nm:9s} median {int(np.median(d[:, k])):6d} ns  p90 {int(np.percentile(d[:, k], 90)):6d}")
    d = np.diff(a, axis=1)
    print("  durations (median ns): " + ", ".join(f"{names[k+1]} {int(np.median(d[:, k]))}" for k in range(5)))
