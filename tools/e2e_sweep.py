"""e2e (Simulation.step_host) time per step vs the density chunk count, with
the host-side enqueue time per step (a host-bound loop shows equal numbers)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402
from paper_2306_11544_b200.hostmem import host_like  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
inp = make_inputs(cfg)
for chunks in (1, 2, 4, 8, 16):
    sim = Simulation.from_config(cfg, inp)
    h = [host_like(a) for a in (sim.densities(), sim.positions(), sim.previous_velocities())]
    o = [host_like(np.zeros_like(t.numpy())) for t in h]
    for _ in range(3):
        sim.step_host(*h, *o, chunks=chunks)
        h, o = o, h
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(sim.stream)
    t0 = time.perf_counter()
    for _ in range(20):
        sim.step_host(*h, *o, chunks=chunks)
        h, o = o, h
    t1 = time.perf_counter()
    b.record(sim.stream)
    torch.cuda.synchronize()
    print("chunks", chunks, round(a.elapsed_time(b) / 20, 4), "ms/step;",
          round((t1 - t0) / 20 * 1e3, 4), "ms/step host enqueue")
    sim.close()
