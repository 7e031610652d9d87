"""Timeline of the host-driven step (Simulation.step_host's copy pattern with
timing events on every stream), steady state, config 1: when the substeps end,
when the cell state is final, when each density piece is down / up again."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_11544_b200 import _lib  # noqa: E402
from paper_2306_11544_b200.configs import CONFIGS, make_inputs  # noqa: E402
from paper_2306_11544_b200.engine import Simulation  # noqa: E402
from paper_2306_11544_b200.hostmem import host_like  # noqa: E402

nocopy = "nocopy" in sys.argv  # events only: the step graph with no transfers in flight
cfg = CONFIGS[1]
inp = make_inputs(cfg)
sim = Simulation.from_config(cfg, inp)
L = _lib.load()
h = [host_like(a) for a in (sim.densities(), sim.positions(), sim.prev_vel.cpu().numpy())]
o = [host_like(np.zeros_like(t.numpy())) for t in h]
k = 4
sim.step_host(*h, *o, chunks=k)  # sets up the streams / events
h, o = o, h
torch.cuda.synchronize()
cin, cout, ccell, main = sim._cin, sim._cout, sim._ccell, sim.stream
T0 = torch.cuda.Event(enable_timing=True)
T0.record(main)
cin.wait_stream(main)


def ev(stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


rows = []
for step in range(6):
    h_dens, h_pos, h_prev, o_dens, o_pos, o_vel = *h, *o
    dflat, hflat, oflat = sim.dens.view(-1), h_dens.view(-1), o_dens.view(-1)
    b = [dflat.numel() * i // k for i in range(k + 1)]
    r = {}
    with torch.cuda.stream(cin):
        cin.wait_event(sim._cells_out)
        r["pos_up_start"] = ev(cin)
        if not nocopy:
            sim.pos.copy_(h_pos, non_blocking=True)
            sim.prev_vel.copy_(h_prev, non_blocking=True)
        r["pos_up_end"] = ev(cin)
    L.cg_engine_io_inputs_ready(sim._eng, _lib.P(cin.cuda_stream))
    with torch.cuda.stream(cin):
        for i in range(k):
            cin.wait_event(sim._dens_out[i])
            r[f"up{i}_start"] = ev(cin)
            if not nocopy:
                dflat[b[i]:b[i + 1]].copy_(hflat[b[i]:b[i + 1]], non_blocking=True)
            r[f"up{i}_end"] = ev(cin)
    L.cg_engine_io_fields_ready(sim._eng, _lib.P(cin.cuda_stream))
    r["graph_enq"] = ev(main)
    sim.run(1, graph=True)
    r["graph_end"] = ev(main)
    L.cg_engine_io_wait_cells(sim._eng, _lib.P(ccell.cuda_stream))
    with torch.cuda.stream(ccell):
        r["cells_final"] = ev(ccell)
        if not nocopy:
            o_pos.copy_(sim.pos, non_blocking=True)
            o_vel.copy_(sim.vel, non_blocking=True)
        r["cells_down_end"] = ev(ccell)
        sim._cells_out.record(ccell)
    L.cg_engine_io_wait_fields(sim._eng, _lib.P(cout.cuda_stream))
    with torch.cuda.stream(cout):
        r["substeps_end"] = ev(cout)
        for i in range(k):
            if not nocopy:
                oflat[b[i]:b[i + 1]].copy_(dflat[b[i]:b[i + 1]], non_blocking=True)
            r[f"down{i}_end"] = ev(cout)
            sim._dens_out[i].record(cout)
    rows.append(r)
    h, o = o, h
torch.cuda.synchronize()
for s, r in enumerate(rows):
    t = {n: T0.elapsed_time(e) * 1e3 for n, e in r.items()}
    print(f"step {s}: " + "  ".join(f"{n}={v:.0f}" for n, v in sorted(t.items(), key=lambda kv: kv[1])))
