"""A/B of the fast-numerics kernel variants (env CELLGPU_SEG_KP / _KZ /
_TMA_STORE) on one config: device ms per step (graph replays, 20 steps after
warm-up) and per-stage times.  Each variant runs in its own process.

    python tools/seg_ab.py CONFIG 'KP=4 KZ=4' 'KP=8 KZ=8 TS=1' ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2306_11544_b200.configs import CONFIGS, make_inputs
from paper_2306_11544_b200.engine import Simulation
cfg = CONFIGS[%d]
import os
sim = Simulation.from_config(cfg, make_inputs(cfg), numerics=os.environ.get("AB_NUMERICS", "fast"),
                             resort_every=int(os.environ.get("AB_RESORT", "0")))
sim.run(3); sim.sync()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for rep in range(3):
    a.record(sim.stream); sim.run(20); b.record(sim.stream); b.synchronize()
    ms.append(a.elapsed_time(b) / 20)
st = sim.time_stages(20)
print("ms/step", round(min(ms), 4), {k: round(v * 1e3, 1) for k, v in st.items()})
'''

cfg = int(sys.argv[1])
for var in sys.argv[2:]:
    env = dict(os.environ)
    for kv in var.split():
        k, v = kv.split("=")
        env[{"KP": "CELLGPU_SEG_KP", "KZ": "CELLGPU_SEG_KZ", "TS": "CELLGPU_SEG_TMA_STORE"}.get(k, k)] = v
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env, capture_output=True,
                         text=True)
    print(var, "->", out.stdout.strip() or out.stderr.strip()[-400:], flush=True)
