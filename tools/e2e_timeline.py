"""Timeline of pipelined host-driven steps (Simulation.step_host's sequence
with substrate chains, timing events on the copy streams), config 1, steady
state: per substrate when its upload ends (chain may start), when its chain
ends (download may start) and when its download ends; the cell state likewise.
Pass 'nocopy' to drop the transfers (events only)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_11544_b200 import _lib  # noqa: E402
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402
from paper_2306_11544_b200.hostmem import host_like  # noqa: E402

nocopy = "nocopy" in sys.argv
cfg = CONFIGS[1]
inp = make_inputs(cfg)
sim = Simulation.from_config(cfg, inp)
L = _lib.load()
h = [host_like(a) for a in (sim.densities(), sim.positions(), sim.prev_vel.cpu().numpy())]
o = [host_like(np.zeros_like(t.numpy())) for t in h]
sim.step_host(*h, *o)  # sets up streams / events / graphs
h, o = o, h
torch.cuda.synchronize()
S = sim.S
assert sim._chains > 1
cin, cout, ccell, main = sim._cin, sim._cout, sim._ccell, sim.stream
T0 = torch.cuda.Event(enable_timing=True)
T0.record(main)
cin.wait_stream(main)
sim._cpos.wait_stream(main)


def ev(stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def cp(dst, src):
    if not nocopy:
        dst.copy_(src, non_blocking=True)


rows = []
for step in range(8):
    h_dens, h_pos, h_prev, o_dens, o_pos, o_vel = *h, *o
    r = {}
    for s in range(S):  # fields first
        with torch.cuda.stream(cin):
            cin.wait_event(sim._dens_out[s])
            cp(sim.dens[s], h_dens[s])
            r[f"up{s}"] = ev(cin)
        L.cg_engine_io_substrate_ready(sim._eng, s, _lib.P(cin.cuda_stream))
    cpos = sim._cpos  # cells on their own upload stream ("split")
    with torch.cuda.stream(cpos):
        cpos.wait_event(sim._cells_out)
        cp(sim.pos, h_pos)
        cp(sim.prev_vel, h_prev)
        r["upC"] = ev(cpos)
    L.cg_engine_io_inputs_ready(sim._eng, _lib.P(cpos.cuda_stream))
    L.cg_engine_step_io(sim._eng)
    L.cg_engine_io_wait_cells(sim._eng, _lib.P(ccell.cuda_stream))
    with torch.cuda.stream(ccell):
        r["mechEnd"] = ev(ccell)
        cp(o_pos, sim.pos)
        cp(o_vel, sim.vel)
        r["downC"] = ev(ccell)
        sim._cells_out.record(ccell)
    for s in range(S):
        L.cg_engine_io_wait_substrate(sim._eng, s, _lib.P(cout.cuda_stream))
        with torch.cuda.stream(cout):
            r[f"chain{s}End"] = ev(cout)
            cp(o_dens[s], sim.dens[s])
            r[f"down{s}"] = ev(cout)
            sim._dens_out[s].record(cout)
    rows.append(r)
    h, o = o, h
L.cg_engine_io_join(sim._eng, _lib.P(main.cuda_stream))
torch.cuda.synchronize()
prev = None
for st, r in enumerate(rows):
    t = {n: T0.elapsed_time(e) * 1e3 for n, e in r.items()}
    base = t["up0"]
    print(f"step {st} (+{base - prev if prev else 0:.0f}): " +
          "  ".join(f"{n}={v - base:.0f}" for n, v in sorted(t.items(), key=lambda kv: kv[1])))
    prev = base
