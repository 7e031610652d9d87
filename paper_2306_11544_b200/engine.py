"""Device-resident step loop: the reference's run_simulation body on one GPU.

``Simulation`` owns every array of one run as torch tensors on the GPU and
drives libcellgpu.so's step engine (cg_engine_*): per mechanics step,
``substeps`` x [G4 exchange fused into the x/y sweep kernel -> z sweep], then
velocities, integration and the counting-sort rebin -- the order of
simulate.py:169-202 with gradients, divisions and resorting left out (out of
scope).  After the first step the whole mechanics step
is replayed as one CUDA graph; nothing synchronises with the host until a
result is read.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .configs import Inputs, SimConfig, make_inputs
from .core import CartesianMesh
from .mechanics import InteractionParams


class Simulation:
    def __init__(self, mesh: CartesianMesh, *, diffusion, decay, densities, positions, radius,
                 ids=None, secretion=None, uptake=None, saturation=38.0, bc="dirichlet",
                 dirichlet=None, params: InteractionParams = InteractionParams(),
                 dt_diffusion=0.01, dt_mechanics=0.1, integrator="ab2", device=None,
                 gradients: bool = False):
        torch = _lib.require_cuda()
        self.torch = torch
        self.mesh = mesh
        dev = torch.cuda.current_device() if device is None else device
        self.device = dev
        D = np.ascontiguousarray(diffusion, np.float64).reshape(-1)
        S = D.shape[0]
        self.S = S
        self.diffusion = D
        self.decay = np.ascontiguousarray(decay, np.float64).reshape(S)
        pos = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
        n = pos.shape[0]
        self.n = n
        rad = np.ascontiguousarray(np.broadcast_to(np.asarray(radius, np.float64), (n,)))
        idv = np.arange(n, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        self.dirichlet = (np.zeros(S) if dirichlet is None
                          else np.ascontiguousarray(np.broadcast_to(np.asarray(dirichlet, np.float64), (S,))))
        self.saturation = np.ascontiguousarray(np.broadcast_to(np.asarray(saturation, np.float64), (S,)))
        self.substeps = int(round(dt_mechanics / dt_diffusion))
        self.params = params
        self.bc = bc
        self.integrator = integrator
        self.dt_diffusion, self.dt_mechanics = float(dt_diffusion), float(dt_mechanics)

        cuda = torch.device("cuda", dev)
        f64, i32 = torch.float64, torch.int32
        nvox = mesh.voxel_count
        t = lambda a: torch.from_numpy(np.array(a, copy=True, order="C")).to(cuda)
        self.dens = t(np.asarray(densities, np.float64).reshape(S, nvox))
        self.pos = t(pos)
        self.vel = torch.zeros((n, 3), dtype=f64, device=cuda)
        self.prev_vel = torch.zeros((n, 3), dtype=f64, device=cuda)
        self.radius = t(rad)
        self.volume = t(_lib.cell_volumes(rad))
        self.ids = t(idv)
        self.secretion = None if secretion is None else t(np.asarray(secretion, np.float64).reshape(S, n))
        self.uptake = None if uptake is None else t(np.asarray(uptake, np.float64).reshape(S, n))
        self.voxel = torch.zeros(max(n, 1), dtype=i32, device=cuda)
        self.bin_start = torch.zeros(nvox + 1, dtype=i32, device=cuda)
        self.bin_cells = torch.zeros(max(n, 1), dtype=i32, device=cuda)
        self.bin_cells_by_id = torch.zeros(max(n, 1), dtype=i32, device=cuda)
        self.nonempty = torch.zeros(nvox, dtype=i32, device=cuda)
        self.n_nonempty = torch.zeros(1, dtype=i32, device=cuda)
        # compute_gradients after the substeps (simulate.py:184-187), on request
        self.grad = torch.zeros((S, nvox, 3), dtype=f64, device=cuda) if gradients else None
        torch.cuda.synchronize(dev)

        # CELLGPU_MAIN_PRIORITY: stream priority of the step (torch: lower is higher)
        self.stream = torch.cuda.Stream(device=dev,
                                        priority=int(os.environ.get("CELLGPU_MAIN_PRIORITY", "0")))
        self.ctx = _lib.Context(mesh, S, max(n, 1), dev)
        self.ctx.bind_stream(self.stream)
        P = _lib.ptr
        self._ptrs = _lib.StatePtrs(
            P(self.dens), P(self.pos), P(self.vel), P(self.prev_vel), P(self.radius),
            P(self.volume), P(self.ids), P(self.secretion), P(self.uptake), P(self.voxel),
            P(self.bin_start), P(self.bin_cells), P(self.bin_cells_by_id), P(self.nonempty),
            P(self.n_nonempty), P(self.grad))
        vp = ctypes.c_void_p
        self._params = _lib.StepParams(
            n, self.substeps, self.dt_diffusion, self.dt_mechanics,
            _lib.BC_DIRICHLET if bc == "dirichlet" else _lib.BC_NEUMANN,
            _lib.AB2 if integrator == "ab2" else _lib.EULER,
            float(params.repulsion), float(params.adhesion), float(params.adhesion_multiplier),
            self.diffusion.ctypes.data_as(vp), self.decay.ctypes.data_as(vp),
            self.dirichlet.ctypes.data_as(vp), self.saturation.ctypes.data_as(vp),
            1 if gradients else 0)
        eng = ctypes.c_void_p()
        L = _lib.load()
        _lib.raise_for(L.cg_engine_create(self.ctx.handle, ctypes.byref(self._ptrs),
                                          ctypes.byref(self._params), ctypes.byref(eng)),
                       "cg_engine_create")
        self._eng = eng
        self.ctx.sync("initial rebin")
        self.steps_done = 0

    @classmethod
    def from_config(cls, cfg: SimConfig, inputs: Inputs | None = None, n_cells=None, **kw):
        inp = inputs if inputs is not None else make_inputs(cfg, n_cells)
        return cls(cfg.mesh(), diffusion=cfg.diffusion, decay=cfg.decay,
                   densities=inp.densities, positions=inp.positions, radius=inp.radius,
                   ids=inp.ids, secretion=inp.secretion, uptake=inp.uptake,
                   saturation=cfg.saturation, bc=cfg.bc, dirichlet=cfg.dirichlet,
                   params=InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier),
                   dt_diffusion=cfg.dt_diffusion, dt_mechanics=cfg.dt_mechanics,
                   integrator=cfg.integrator, **kw)

    # ---- stepping
    def run(self, steps: int = 1, graph: bool = True) -> None:
        """Enqueue ``steps`` mechanics steps on ``self.stream`` (asynchronous)."""
        code = _lib.load().cg_engine_run(self._eng, int(steps), 1 if graph else 0)
        _lib.raise_for(code, "cg_engine_run")
        self.steps_done += steps

    # upload order of the host-driven step: "cells_first", "fields_first",
    # "first_field" (field piece 0, cells, the other pieces; one upload
    # stream) or "split" (cells and fields on two streams)
    io_order = "auto"  # split with substrate chains, else cells_first (measured)

    def step_host(self, h_dens, h_pos, h_prev, o_dens, o_pos, o_vel, chunks: int = 4) -> None:
        """One mechanics step from host state to host state (pinned torch CPU
        tensors): the step consumes h_dens (S, nvox), h_pos (n, 3) and h_prev
        (n, 3, the AB2 state) and leaves densities, positions and velocities
        in o_dens, o_pos, o_vel.  Asynchronous: synchronise the device (the
        copies run on the simulation's own copy streams) before reading the
        outputs; o_* may be passed as the next step's h_* (ordering is handled
        here).

        Copies overlap the step.  The cell state and the densities have their
        own dependency chains: the mechanics (velocities, integration, rebin)
        wait only for the position / AB2 upload and their results go out as
        soon as the rebin is done, while the substeps still run; the substeps
        wait only for the density upload, and the density download starts when
        they end.  The densities move in `chunks` pieces so the next step's
        upload of a piece starts as soon as that piece has come down (PCIe is
        full duplex).  With substrate chains (cg_engine_substrate_chains > 1)
        the pieces are the substrates and each substrate's substeps wait only
        for its own upload and release only its own download, so the transfers
        of one substrate run under the substeps of the others."""
        torch = self.torch
        L = _lib.load()
        if not getattr(self, "_io", False):
            _lib.raise_for(L.cg_engine_io_enable(self._eng), "cg_engine_io_enable")
            self._cin = torch.cuda.Stream(device=self.device)     # uploads
            self._cout = torch.cuda.Stream(device=self.device)    # density download
            self._ccell = torch.cuda.Stream(device=self.device)   # cell state download
            self._cpos = torch.cuda.Stream(device=self.device)    # cell state upload ("split")
            # substrate chains: the fields move substrate by substrate
            self._chains = int(L.cg_engine_substrate_chains(self._eng))
            if self._chains > 1:
                chunks = self._chains
            self._dens_out = [torch.cuda.Event() for _ in range(chunks)]
            self._cells_out = torch.cuda.Event()
            for e in self._dens_out:
                e.record(self._cout)
            self._cells_out.record(self._ccell)
            self._io = True
        k = len(self._dens_out)
        cin, cout, ccell = self._cin, self._cout, self._ccell
        dflat, hflat, oflat = self.dens.view(-1), h_dens.view(-1), o_dens.view(-1)
        bounds = [dflat.numel() * i // k for i in range(k + 1)]

        def up_cells(st):
            with torch.cuda.stream(st):
                st.wait_event(self._cells_out)  # the previous step's cell state is out
                self.pos.copy_(h_pos, non_blocking=True)
                self.prev_vel.copy_(h_prev, non_blocking=True)
            _lib.raise_for(L.cg_engine_io_inputs_ready(self._eng, _lib.P(st.cuda_stream)),
                           "cg_engine_io_inputs_ready")

        chains = self._chains > 1  # then piece i is substrate i
        if chains:
            bounds = [self.dens.shape[1] * i for i in range(k + 1)]

        def up_fields(st, i0=0, i1=k):
            for i in range(i0, i1):  # piece i is overwritten once its download is done
                with torch.cuda.stream(st):
                    st.wait_event(self._dens_out[i])
                    sl = slice(bounds[i], bounds[i + 1])
                    dflat[sl].copy_(hflat[sl], non_blocking=True)
                if chains:
                    _lib.raise_for(L.cg_engine_io_substrate_ready(self._eng, i, _lib.P(st.cuda_stream)),
                                   "cg_engine_io_substrate_ready")
            if not chains and i1 == k:
                _lib.raise_for(L.cg_engine_io_fields_ready(self._eng, _lib.P(st.cuda_stream)),
                               "cg_engine_io_fields_ready")

        order = self.io_order
        if order == "auto":
            order = "split" if chains else "cells_first"
        if order == "fields_first":
            up_fields(cin)
            up_cells(cin)
        elif order == "first_field":  # piece 0, cells, other pieces
            up_fields(cin, 0, 1)
            up_cells(cin)
            up_fields(cin, 1, k)
        elif order == "split":
            up_cells(self._cpos)
            up_fields(cin)
        else:
            up_cells(cin)
            up_fields(cin)
        if chains:  # pipelined across steps (cg_engine_step_io)
            _lib.raise_for(L.cg_engine_step_io(self._eng), "cg_engine_step_io")
            self.steps_done += 1
        else:
            self.run(1, graph=True)
        _lib.raise_for(L.cg_engine_io_wait_cells(self._eng, _lib.P(ccell.cuda_stream)),
                       "cg_engine_io_wait_cells")
        with torch.cuda.stream(ccell):
            o_pos.copy_(self.pos, non_blocking=True)
            o_vel.copy_(self.vel, non_blocking=True)
            self._cells_out.record(ccell)
        if not chains:
            _lib.raise_for(L.cg_engine_io_wait_fields(self._eng, _lib.P(cout.cuda_stream)),
                           "cg_engine_io_wait_fields")
        for i in range(k):
            if chains:
                _lib.raise_for(L.cg_engine_io_wait_substrate(self._eng, i, _lib.P(cout.cuda_stream)),
                               "cg_engine_io_wait_substrate")
            with torch.cuda.stream(cout):
                sl = slice(bounds[i], bounds[i + 1])
                oflat[sl].copy_(dflat[sl], non_blocking=True)
                self._dens_out[i].record(cout)
        if chains:  # the simulation stream sees the step (reads, sync)
            _lib.raise_for(L.cg_engine_io_join(self._eng, _lib.P(self.stream.cuda_stream)),
                           "cg_engine_io_join")

    def sync(self) -> None:
        """Wait for the stream and raise the first device-side error, if any."""
        self.ctx.sync("simulation step")

    @property
    def launches_per_step(self) -> int:
        return int(_lib.load().cg_engine_launches_per_step(self._eng))

    def time_stages(self, reps: int = 20) -> dict:
        """Per-stage device ms (each stage `reps`x back to back; perturbs state)."""
        maxk = 16
        names = ctypes.create_string_buffer(32 * maxk)
        ms = (ctypes.c_double * maxk)()
        k = _lib.load().cg_engine_time_stages(self._eng, int(reps), maxk, names,
                                              ctypes.cast(ms, ctypes.c_void_p))
        if k < 0:
            _lib.raise_for(k, "cg_engine_time_stages")
        return {names.raw[32 * i:32 * (i + 1)].split(b"\0", 1)[0].decode(): ms[i] for i in range(k)}

    # ---- results (host copies)
    def densities(self) -> np.ndarray:
        self.stream.synchronize()
        return self.dens.cpu().numpy()

    def positions(self) -> np.ndarray:
        self.stream.synchronize()
        return self.pos.cpu().numpy()

    def velocities(self) -> np.ndarray:
        self.stream.synchronize()
        return self.vel.cpu().numpy()

    def gradients(self) -> np.ndarray:
        """(S, nvox, 3) gradients of the last step (Simulation(gradients=True))."""
        if self.grad is None:
            raise ValueError("Simulation was created without gradients=True")
        self.stream.synchronize()
        return self.grad.cpu().numpy()

    def checksum(self) -> str:
        """state_checksum (simulate.py:79-90) of the current cells, on the GPU."""
        from .checksum import device_checksum

        self.stream.synchronize()
        return device_checksum(self.ctx, self.n, self.ids, self.pos, self.vel)

    def nonempty_count(self) -> int:
        self.stream.synchronize()
        return int(self.n_nonempty.cpu().item())

    def bins(self) -> dict:
        self.stream.synchronize()
        n = self.n
        nne = int(self.n_nonempty.cpu().item())
        return {
            "voxel": self.voxel[:n].cpu().numpy(),
            "bin_start": self.bin_start.cpu().numpy(),
            "bin_cells": self.bin_cells[:n].cpu().numpy(),
            "bin_cells_by_id": self.bin_cells_by_id[:n].cpu().numpy(),
            "nonempty": self.nonempty[:nne].cpu().numpy(),
        }

    def close(self) -> None:
        if getattr(self, "_eng", None):
            self.stream.synchronize()
            _lib.load().cg_engine_destroy(self._eng)
            self._eng = None
        if getattr(self, "ctx", None):
            self.ctx.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
