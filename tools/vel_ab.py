"""A/B fast-velocity kernel variants: python tools/vel_ab.py CONFIG 'A=1' 'A=0 B=1' ...
Each variant runs with its env set throughout (capture and stage timing);
prints the stage times and the velocity difference to the first variant."""
import os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs
from paper_2306_11544_b200.engine import Simulation

cfg = CONFIGS[int(sys.argv[1])]
inp = make_inputs(cfg)
ref = None
for variant in sys.argv[2:]:
    env = dict(kv.split("=") for kv in variant.split())
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    s = Simulation.from_config(cfg, inp, numerics=os.environ.get("VEL_AB_NUMERICS", "fast"), resort_every=50)
    s.run(1, graph=False); s.sync()
    v = s.velocities()
    dn = s.densities()
    st = s.time_stages(20)
    s.run(3); s.sync()
    import torch
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s.stream); s.run(20); b.record(s.stream); s.sync()
    diff = "" if ref is None else (f" dv={np.max(np.abs(v - ref)) / np.max(np.abs(ref)):.2e}"
                                   f" fields_bitwise={np.array_equal(dn, refd)}")
    if ref is None: ref, refd = v, dn
    print(f"[{variant}] step {a.elapsed_time(b)/20*1e3:.1f} us{diff}  " + ", ".join(f"{n} {x*1e3:.1f}" for n, x in st.items()), flush=True)
    s.close()
    for k, x in saved.items():
        if x is None: os.environ.pop(k)
        else: os.environ[k] = x
