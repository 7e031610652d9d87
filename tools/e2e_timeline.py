"""Timeline of host-driven steps (Simulation.step_host): every kernel and
every host<->device copy of the last of N steps with its stream and device
timestamps (torch.profiler / CUPTI; the image has no nsys), plus per-link busy
time -- where the PCIe links idle.  python tools/e2e_timeline.py [CONFIG] [chunks]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402
from paper_2306_11544_b200.hostmem import host_empty, host_like  # noqa: E402

key = int(sys.argv[1]) if len(sys.argv) > 1 else 1
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = CONFIGS[key]
sim = Simulation.from_config(cfg, make_inputs(cfg), numerics="fast", resort_every=50)
n = sim.n
h = [host_like(sim.densities()), host_like(sim.positions()), host_like(sim.previous_velocities())]
o = [host_empty(tuple(h[0].shape)), host_empty(tuple(h[1].shape)), host_empty((n, 3))]


def step():
    global h, o
    sim.step_host(h[0], h[1], h[2], o[0], o[1], o[2], chunks=chunks)
    h, o = [o[0], o[1], o[2]], [h[0], h[1], h[2]]


for _ in range(10):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

N = 6
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    a.record(sim.stream)
    for _ in range(N):
        step()
    b.record(sim.stream)
    torch.cuda.synchronize()
print(f"config {key}, chunks {chunks}: {a.elapsed_time(b) / N * 1e3:.1f} us per host-driven step")
out = f"gpurun_out/e2e_timeline_c{key}.json"
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
t_end = max(e["ts"] + e["dur"] for e in ev)
span = t_end - ev[0]["ts"]
t0 = t_end - 2 * span / N  # the last two steps
win = [e for e in ev if e["ts"] + e["dur"] > t0]
busy = {"HtoD": 0.0, "DtoH": 0.0, "kernel": 0.0}
for e in win:
    kind = "kernel" if e["cat"] == "kernel" else ("HtoD" if "HtoD" in e["name"] else "DtoH")
    s, t = max(e["ts"], t0), e["ts"] + e["dur"]
    busy[kind] += t - s
    nm = e["name"] if kind == "kernel" else f"{kind} {e['args'].get('bytes', 0) / 1e6:.2f} MB"
    print(f"  {kind:6s} stream {e['args'].get('stream', '?'):>4} {s - t0:8.1f} .. {t - t0:8.1f}  {nm[:60]}")
print(f"window {t_end - t0:.1f} us (2 steps): busy HtoD {busy['HtoD']:.1f}  DtoH {busy['DtoH']:.1f}"
      f"  kernels (sum over streams) {busy['kernel']:.1f}")
