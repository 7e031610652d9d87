"""Config-1 velocity branch for ncu: a few engine steps, then the velocity
stage alone (time_stages enqueues it back to back).  Run under
  ncu --kernel-name regex:'k_velocity_cells|k_cand_lists' -c 4 --metrics ... \
      python tools/velocity_profile.py
Also prints the pair statistics of the configuration (candidates and in-range
pairs per cell) from the positions, for the FP64 op count."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402

cfg = CONFIGS[1]
inp = make_inputs(cfg)
sim = Simulation.from_config(cfg, inp)
sim.run(2)
sim.sync()
pos = sim.positions()
print("pairs:", __import__("json").dumps(__import__("bench").pair_stats(cfg, pos, inp)))
sim.time_stages(2)
sim.sync()
