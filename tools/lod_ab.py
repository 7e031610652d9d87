"""A/B: register-line LOD kernels vs streaming (CELLGPU_REGLINES), bitwise + timing."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs
from paper_2306_11544_b200.engine import Simulation

for ci in [int(a) for a in sys.argv[1:]] or [0, 1]:
    cfg = CONFIGS[ci]
    inp = make_inputs(cfg)
    sims = {}
    for k in ("0", "1"):
        os.environ["CELLGPU_REGLINES"] = k
        sims[k] = Simulation.from_config(cfg, inp)
    for s in sims.values():
        s.run(2, graph=False); s.run(1, graph=True); s.sync()
    d0, d1 = sims["0"].densities(), sims["1"].densities()
    p0, p1 = sims["0"].positions(), sims["1"].positions()
    print(f"config {ci}: densities bitwise equal {np.array_equal(d0, d1)}, positions {np.array_equal(p0, p1)}")
    for k, s in sims.items():
        s.run(3); s.sync()
        st = s.stream
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st); s.run(20); b.record(st); s.sync()
        print(f"   reglines={k}: {a.elapsed_time(b)/20*1e3:.1f} us/step  stages {{{', '.join(f'{n}: {v*1e3:.1f}' for n, v in s.time_stages(20).items())}}}")
