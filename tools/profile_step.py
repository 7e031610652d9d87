"""Small driver for ncu --set full captures: one config's engine, two
mechanics steps without graphs (every kernel is a separate launch ncu can
replay).  python tools/profile_step.py [CONFIG] [exact|fast] [RESORT_EVERY]"""
import sys

sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
numerics = sys.argv[2] if len(sys.argv) > 2 else "exact"
resort = int(sys.argv[3]) if len(sys.argv) > 3 else 0
sim = Simulation.from_config(cfg, make_inputs(cfg), numerics=numerics, resort_every=resort)
sim.run(2, graph=False)
sim.sync()
