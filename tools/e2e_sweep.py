"""e2e (Simulation.step_host) time per step vs the density chunk count, with
the host-side enqueue time per step (a host-bound loop shows equal numbers).
    python tools/e2e_sweep.py [CONFIG] [fast|exact]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402
from paper_2306_11544_b200.hostmem import host_like  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
numerics = sys.argv[2] if len(sys.argv) > 2 else "fast"
inp = make_inputs(cfg)
for chunks in [int(c) for c in (sys.argv[3].split(',') if len(sys.argv) > 3 else '1,2,4,8,16'.split(','))]:
    sim = Simulation.from_config(cfg, inp, numerics=numerics, resort_every=50)
    h = [host_like(a) for a in (sim.densities(), sim.positions(), sim.previous_velocities())]
    o = [host_like(np.zeros_like(t.numpy())) for t in h]
    for _ in range(3):
        sim.step_host(*h, *o, chunks=chunks)
        h, o = o, h
    torch.cuda.synchronize()
    best = None
    for rep in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(sim.stream)
        t0 = time.perf_counter()
        for _ in range(50):
            sim.step_host(*h, *o, chunks=chunks)
            h, o = o, h
        t1 = time.perf_counter()
        b.record(sim.stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 50
        best = ms if best is None else min(best, ms)
    print("chunks", chunks, round(best, 4), "ms/step (best of 3 x 50);",
          round((t1 - t0) / 50 * 1e3, 4), "ms/step host enqueue")
    sim.close()
