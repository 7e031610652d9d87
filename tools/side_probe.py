"""What the mechanics branch costs the step (probe build): ms per step with
the velocities and / or the integration + rebin skipped
(CELLGPU_PROBE_SKIP; results are wrong while skipping).
    python tools/side_probe.py CONFIG"""
import os
import subprocess
import sys

cfg = sys.argv[1] if len(sys.argv) > 1 else "1"
lib = os.path.abspath("paper_2306_11544_b200/libcellgpu_probe.so")
for skip in ("0", "1", "2", "3"):
    env = dict(os.environ, CELLGPU_LIB=lib, CELLGPU_PROBE_SKIP=skip)
    out = subprocess.run([sys.executable, "tools/seg_ab.py", cfg, "AB_RESORT=50"], env=env,
                         capture_output=True, text=True)
    print("skip", skip, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:],
          flush=True)
