"""A/B any engine env switches: python tools/ab_env.py CONFIG[:fast] 'A=1 B=0' 'A=0' ...
Checks that every variant's densities/positions equal the first variant's bit for bit."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs
from paper_2306_11544_b200.engine import Simulation

key, _, numerics = sys.argv[1].partition(":")
cfg = CONFIGS[int(key)]
inp = make_inputs(cfg)
ref = None
for variant in sys.argv[2:]:
    env = dict(kv.split("=") for kv in variant.split())
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    s = Simulation.from_config(cfg, inp, numerics=numerics or "exact", resort_every=50)
    for k, v in saved.items():
        if v is None: os.environ.pop(k)
        else: os.environ[k] = v
    s.run(2, graph=False); s.run(1, graph=True); s.sync()
    d, p = s.densities(), s.positions()
    same = "" if ref is None else f" bitwise={np.array_equal(d, ref[0]) and np.array_equal(p, ref[1])}"
    if ref is None: ref = (d, p)
    s.run(3); s.sync()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s.stream); s.run(20); b.record(s.stream); s.sync()
    st = s.time_stages(20)
    print(f"[{variant}] {a.elapsed_time(b)/20*1e3:.1f} us/step{same}  " + ", ".join(f"{n} {v*1e3:.1f}" for n, v in st.items()))
    del s
