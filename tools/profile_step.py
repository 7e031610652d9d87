"""Small driver for ncu --set full captures: config 1 engine, two mechanics
steps without graphs (every kernel is a separate launch ncu can replay)."""
import sys

sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
sim = Simulation.from_config(cfg, make_inputs(cfg))
sim.run(2, graph=False)
sim.sync()
