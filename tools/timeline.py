"""Kernel timeline of graph-replayed mechanics steps (an nsys stand-in: the
image has no nsys).  torch.profiler (CUPTI) records every kernel of the
replayed step graphs with its stream and device timestamps; this prints the
last step's kernels in start order relative to the step's first kernel, the
per-stream busy time and the overlap of the two streams, and writes the
chrome trace.  python tools/timeline.py CONFIG [fast|exact] [out.json]"""
import collections
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402

key = int(sys.argv[1]) if len(sys.argv) > 1 else 1
numerics = sys.argv[2] if len(sys.argv) > 2 else "fast"
out = sys.argv[3] if len(sys.argv) > 3 else f"gpurun_out/timeline_c{key}_{numerics}.json"
cfg = CONFIGS[key]
sim = Simulation.from_config(cfg, make_inputs(cfg), numerics=numerics, resort_every=50)
sim.run(5, graph=True)
sim.sync()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sim.run(4, graph=True)
    sim.sync()
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"]
      if e.get("cat") == "kernel" and e.get("ph") == "X"]
ev.sort(key=lambda e: e["ts"])
# split into steps at the first plane kernel after a gap of the side branch: use
# the graph-launch correlation -- simpler: the last quarter of the kernels
# belongs to the last step (4 identical steps)
n = len(ev) // 4
step = ev[-n:]
t0 = step[0]["ts"]
t1 = max(e["ts"] + e["dur"] for e in step)
print(f"config {key} {numerics}: last of 4 replayed steps, {n} kernels, span {t1 - t0:.1f} us")
busy = collections.defaultdict(float)
intervals = collections.defaultdict(list)
for e in step:
    s = e["args"].get("stream", e.get("tid"))
    busy[s] += e["dur"]
    intervals[s].append((e["ts"] - t0, e["ts"] - t0 + e["dur"]))
    print(f"  stream {s:>4} {e['ts'] - t0:8.1f} .. {e['ts'] - t0 + e['dur']:8.1f}  {e['name'][:70]}")
for s, b in busy.items():
    print(f"stream {s}: {len(intervals[s])} kernels, busy {b:.1f} us")
