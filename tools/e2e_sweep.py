import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs
from paper_2306_11544_b200.engine import Simulation
cfg = CONFIGS[1]; inp = make_inputs(cfg)
for chunks in (1, 2, 4, 8, 16):
    sim = Simulation.from_config(cfg, inp)
    h = [torch.from_numpy(a).pin_memory() for a in (sim.densities(), sim.positions(), sim.prev_vel.cpu().numpy())]
    o = [torch.empty_like(t).pin_memory() for t in h]
    for _ in range(3):
        sim.step_host(*h, *o, chunks=chunks); h, o = o, h
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(sim.stream)
    for _ in range(20):
        sim.step_host(*h, *o, chunks=chunks); h, o = o, h
    for s_ in (sim._cin, sim._cout): sim.stream.wait_stream(s_)
    b.record(sim.stream); torch.cuda.synchronize()
    print("chunks", chunks, round(a.elapsed_time(b) / 20, 4), "ms/step")
    sim.close()
