"""Where the bench's per-step time goes beyond back-to-back replay: config 1,
fast numerics, graph replays timed (a) back to back, (b) one event pair per
step, (c) + 256 MiB write flush before each step, (d) + a 256 MiB read pass
after the write."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2306_11544_b200.configs import CONFIGS, make_inputs
from paper_2306_11544_b200.engine import Simulation

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
sim = Simulation.from_config(cfg, make_inputs(cfg), numerics="fast", resort_every=50)
st = sim.stream
buf = torch.empty(256 << 20 >> 2, dtype=torch.int32, device="cuda")
rd = torch.ones(256 << 20 >> 2, dtype=torch.int32, device="cuda")
out = torch.empty((), dtype=torch.int64, device="cuda")
with torch.cuda.stream(st):
    sim.run(10, graph=True)
torch.cuda.synchronize()
N = 30


def per_step(pre):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
    with torch.cuda.stream(st):
        for i in range(N):
            pre(i)
            ev[i][0].record(st)
            sim.run(1, graph=True)
            ev[i][1].record(st)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return f"median {t[N // 2]:.1f} min {t[0]:.1f} max {t[-1]:.1f}"


a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    a.record(st); sim.run(N, graph=True); b.record(st)
torch.cuda.synchronize()
print(f"(a) back to back: {a.elapsed_time(b) / N * 1e3:.1f} us/step")
print("(b) events per step:", per_step(lambda i: None))
print("(c) write flush:", per_step(lambda i: buf.fill_(i)))
print("(d) write + read flush:", per_step(lambda i: (buf.fill_(i), torch.sum(rd, dim=0, out=out))))
print("(e) sleep kernel gap:", per_step(lambda i: torch.cuda._sleep(100000)))
# (f) events per step, but the span of all steps / N
ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
with torch.cuda.stream(st):
    for i in range(N):
        ev[i].record(st)
        sim.run(1, graph=True)
    ev[N].record(st)
torch.cuda.synchronize()
print(f"(f) events per step, span / N: {ev[0].elapsed_time(ev[N]) / N * 1e3:.1f}")
# (g) non-timing events between the graphs, span timed
nt = [torch.cuda.Event() for _ in range(N)]
with torch.cuda.stream(st):
    a.record(st)
    for i in range(N):
        nt[i].record(st)
        sim.run(1, graph=True)
    b.record(st)
torch.cuda.synchronize()
print(f"(g) non-timing events between steps, span / N: {a.elapsed_time(b) / N * 1e3:.1f}")
# (h) a tiny kernel between graphs, span timed
with torch.cuda.stream(st):
    a.record(st)
    for i in range(N):
        out.zero_()
        sim.run(1, graph=True)
    b.record(st)
torch.cuda.synchronize()
print(f"(h) tiny kernel between steps, span / N: {a.elapsed_time(b) / N * 1e3:.1f}")
