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
                 gradients: bool = False, numerics: str = "exact", resort_every: int = 0,
                 division_rate=None, division_seed: int = 0, capacity: int | None = None):
        """``numerics``: "exact" (default) -- every operation in the
        reference's order, results bit-identical to it; "fast" --
        BASELINE.json's tolerances instead (fields within 1e-10, velocities
        and positions within 1e-12 normwise per step, bins identical):
        segmented line solves, affine per-voxel exchange fused into the plane
        kernel, velocities summed per cell over its neighbour rows
        (include/cellgpu.h CG_NUMERICS_FAST).

        ``resort_every`` > 0: voxel-sorted storage, the reference's
        StorageOrder.voxel_sorted(every) strategy -- cells are sorted by
        (voxel, id) before the first step and after every ``resort_every``
        steps (simulate.py:156-158, 209-212; population.py:132-135).  Results
        per cell id are unchanged; positions() etc. come back in the current
        storage order (cell_ids() gives it).

        ``division_rate`` (scalar or per cell, default none): cells divide
        after every step as in run_simulation (simulate.py:205-206,
        population.py:77-129, seed ``division_seed``, step index = steps
        done), daughters appended at the end of every per-cell array within
        ``capacity`` cells (default: 2n when any rate is positive, else n;
        CapacityError beyond it); the next step recaptures its graphs for the
        new count."""
        if numerics not in ("exact", "fast"):
            raise ValueError("numerics must be 'exact' or 'fast'")
        self.numerics = numerics
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
        rates = (None if division_rate is None else
                 np.ascontiguousarray(np.broadcast_to(np.asarray(division_rate, np.float64), (n,))))
        self.division_seed = int(division_seed)
        dividing = rates is not None and bool((rates > 0.0).any())
        cap = max(n, int(capacity) if capacity is not None else (2 * n if dividing else n), 1)
        self.capacity = cap
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

        def cells(a, dtype=f64, width=None):
            """A per-cell array in a capacity-sized buffer (rows [0, n) live)."""
            shape = (cap,) if width is None else (cap, width)
            buf = torch.zeros(shape, dtype=dtype, device=cuda)
            if a is not None:
                buf[:n] = torch.from_numpy(np.array(a, copy=True, order="C")).to(cuda)
            return buf

        self.dens = t(np.asarray(densities, np.float64).reshape(S, nvox))
        self.pos = cells(pos, width=3)
        self.vel = cells(None, width=3)
        self.prev_vel = cells(None, width=3)
        self.radius = cells(rad)
        self.volume = cells(_lib.cell_volumes(rad))
        self.ids = cells(idv, dtype=torch.int64)
        self.next_id = int(idv.max()) + 1 if n else 0
        self.div_rate = cells(rates) if rates is not None else None

        def rows(a):
            """(S, n) rates with stride n inside an (S * capacity) buffer."""
            if a is None:
                return None
            buf = torch.zeros(S * cap, dtype=f64, device=cuda)
            buf[:S * n] = torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.float64).reshape(S * n))).to(cuda)
            return buf

        self._sec_buf, self._upt_buf = rows(secretion), rows(uptake)
        self.voxel = torch.zeros(cap, dtype=i32, device=cuda)
        self.bin_start = torch.zeros(nvox + 1, dtype=i32, device=cuda)
        self.bin_cells = torch.zeros(cap, dtype=i32, device=cuda)
        self.bin_cells_by_id = torch.zeros(cap, dtype=i32, device=cuda)
        self.nonempty = torch.zeros(nvox, dtype=i32, device=cuda)
        self.n_nonempty = torch.zeros(1, dtype=i32, device=cuda)
        # compute_gradients after the substeps (simulate.py:184-187), on request
        self.grad = torch.zeros((S, nvox, 3), dtype=f64, device=cuda) if gradients else None
        torch.cuda.synchronize(dev)

        # CELLGPU_MAIN_PRIORITY: stream priority of the step (torch: lower is higher)
        self.stream = torch.cuda.Stream(device=dev,
                                        priority=int(os.environ.get("CELLGPU_MAIN_PRIORITY", "0")))
        self.ctx = _lib.Context(mesh, S, cap, dev)
        self.ctx.bind_stream(self.stream)
        P = _lib.ptr
        self._ptrs = _lib.StatePtrs(
            P(self.dens), P(self.pos), P(self.vel), P(self.prev_vel), P(self.radius),
            P(self.volume), P(self.ids), P(self._sec_buf), P(self._upt_buf), P(self.voxel),
            P(self.bin_start), P(self.bin_cells), P(self.bin_cells_by_id), P(self.nonempty),
            P(self.n_nonempty), P(self.grad), P(self.div_rate))
        vp = ctypes.c_void_p
        self._params = _lib.StepParams(
            n, self.substeps, self.dt_diffusion, self.dt_mechanics,
            _lib.BC_DIRICHLET if bc == "dirichlet" else _lib.BC_NEUMANN,
            _lib.AB2 if integrator == "ab2" else _lib.EULER,
            float(params.repulsion), float(params.adhesion), float(params.adhesion_multiplier),
            self.diffusion.ctypes.data_as(vp), self.decay.ctypes.data_as(vp),
            self.dirichlet.ctypes.data_as(vp), self.saturation.ctypes.data_as(vp),
            1 if gradients else 0, 1 if numerics == "fast" else 0)
        eng = ctypes.c_void_p()
        L = _lib.load()
        _lib.raise_for(L.cg_engine_create(self.ctx.handle, ctypes.byref(self._ptrs),
                                          ctypes.byref(self._params), ctypes.byref(eng)),
                       "cg_engine_create")
        self._eng = eng
        self.ctx.sync("initial rebin")
        self.steps_done = 0
        self.resort_every = int(resort_every)
        if self.resort_every > 0:
            self.sort_cells_by_voxel()

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
    @property
    def dividing(self) -> bool:
        return self.div_rate is not None and bool((self.div_rate[:self.n] > 0.0).any().item())

    def run(self, steps: int = 1, graph: bool = True) -> None:
        """Enqueue ``steps`` mechanics steps on ``self.stream`` (asynchronous);
        with voxel-sorted storage the resorts fall between them; with dividing
        cells every step is followed by the division pass (synchronising: the
        daughter count sizes the append), in run_simulation's order
        (simulate.py:201-212: rebin, divisions, resort)."""
        L = _lib.load()
        left = int(steps)
        divide = self.dividing
        while left > 0:
            k = 1 if divide else left
            if self.resort_every > 0:
                k = min(k, self.resort_every - self.steps_done % self.resort_every)
            _lib.raise_for(L.cg_engine_run(self._eng, k, 1 if graph else 0), "cg_engine_run")
            self.steps_done += k
            left -= k
            if divide:
                self.divide(self.steps_done - 1)
            if self.resort_every > 0 and self.steps_done % self.resort_every == 0:
                self.sort_cells_by_voxel()

    def divide(self, step: int) -> np.ndarray:
        """population.py:77-129 on the engine's cells (division pass of
        mechanics step ``step``): draws and decisions on the device, daughters
        in ascending parent id with fresh ids, placed R/2 along the drawn
        direction (the direction's cos / sin from the host's libm) and clamped;
        each daughter copies its parent's radius, volume, velocity, AB2 state,
        rates and division rate.  Returns the daughters' ids."""
        import math

        from .errors import CapacityError, DomainError

        torch = self.torch
        if not self.dt_mechanics > 0.0:
            raise DomainError("division step needs dt > 0")
        n = self.n
        if self.div_rate is None or n == 0:
            return np.zeros(0, np.int64)
        L = _lib.load()
        P = _lib.ptr
        self.stream.synchronize()
        rates = self.div_rate[:n].cpu().numpy()
        thr = np.full(n, -1.0)
        for r in np.unique(rates[rates > 0.0]):  # population.py:94 as CPython evaluates it
            thr[rates == r] = 1.0 - math.exp(-float(r) * self.dt_mechanics)
        d_thr = torch.from_numpy(thr).to(self.pos.device)
        seed = self.division_seed & ((1 << 64) - 1)
        step64 = int(step)
        cnt = _lib.I(0)
        _lib.raise_for(L.cg_divisions_count(self.ctx.handle, n, seed, step64, P(self.ids),
                                            P(d_thr), ctypes.byref(cnt)), "divide")
        m = int(cnt.value)
        if m == 0:
            return np.zeros(0, np.int64)
        if n + m > self.capacity:
            raise CapacityError(f"division would exceed the engine's capacity ({n} + {m} > "
                                f"{self.capacity} cells)")
        parent = torch.empty(m, dtype=torch.int32, device=self.pos.device)
        dpos = torch.empty((m, 3), dtype=torch.float64, device=self.pos.device)
        _lib.raise_for(L.cg_divisions_place(self.ctx.handle, n, m, seed, step64, P(self.ids),
                                            P(self.pos), P(self.radius), P(parent), P(dpos)),
                       "divide")
        self.ctx.sync("divide")
        pl = parent.long()
        new_ids = np.arange(self.next_id, self.next_id + m, dtype=np.int64)
        with torch.cuda.stream(self.stream):
            self.pos[n:n + m] = dpos
            for t in (self.vel, self.prev_vel, self.radius, self.volume, self.div_rate):
                t[n:n + m] = t[pl]
            self.ids[n:n + m] = torch.from_numpy(new_ids).to(self.pos.device)
            S = self.S
            for buf in (self._sec_buf, self._upt_buf):
                if buf is None:
                    continue
                old = buf[:S * n].view(S, n).clone()  # (S, n) -> (S, n + m), stride changes
                new = buf[:S * (n + m)].view(S, n + m)
                new[:, :n] = old
                new[:, n:] = old[:, pl]
        self.stream.synchronize()
        self.n = n + m
        self.next_id += m
        _lib.raise_for(L.cg_engine_set_cell_count(self._eng, self.n), "divide")
        return new_ids

    def sort_cells_by_voxel(self) -> None:
        """population.py:132-135 on the device: storage order (voxel, id)."""
        _lib.raise_for(_lib.load().cg_engine_sort_cells(self._eng), "cg_engine_sort_cells")

    def cell_ids(self) -> np.ndarray:
        """Cell ids in the current storage order."""
        self.stream.synchronize()
        return self.ids[:self.n].cpu().numpy()

    @property
    def secretion(self):
        """(S, n) per-cell secretion rates (device view), or None."""
        return None if self._sec_buf is None else self._sec_buf[:self.S * self.n].view(self.S, self.n)

    @property
    def uptake(self):
        return None if self._upt_buf is None else self._upt_buf[:self.S * self.n].view(self.S, self.n)

    def step_host(self, h_dens, h_pos, h_prev, o_dens, o_pos, o_vel, chunks: int = 2) -> None:
        """One mechanics step from host state to host state through the C-ABI
        (cg_engine_step_host): the step consumes h_dens (S, nvox), h_pos
        (n, 3) and h_prev (n, 3, the AB2 state) and leaves densities,
        positions and velocities in o_dens, o_pos, o_vel -- contiguous
        float64 CPU tensors, page-locked for the copies to overlap
        (hostmem.host_empty / Tensor.pin_memory).  Asynchronous; o_* may be
        passed as the next step's h_* (the library orders the copies).
        ``self.stream`` waits for the step and its copies (sync() then
        raises device errors).

        The copies overlap the step: the mechanics wait only for the cell
        upload and their results go out right after integration; with
        substrate chains every substrate's field moves in `chunks` pieces,
        its substeps wait only for its own upload and release only its own
        download (one substrate's transfers run under the others' substeps),
        and a piece goes back up as soon as it has come down (PCIe is full
        duplex)."""
        L = _lib.load()
        for t in (h_dens, h_pos, h_prev, o_dens, o_pos, o_vel):
            if t.device.type != "cpu" or t.dtype != self.torch.float64 or not t.is_contiguous():
                raise ValueError("step_host takes contiguous float64 CPU tensors")
        P = _lib.P
        _lib.raise_for(L.cg_engine_step_host(
            self._eng, P(h_dens.data_ptr()), P(h_pos.data_ptr()), P(h_prev.data_ptr()),
            P(o_dens.data_ptr()), P(o_pos.data_ptr()), P(o_vel.data_ptr()), int(chunks)),
            "cg_engine_step_host")
        self.steps_done += 1
        _lib.raise_for(L.cg_engine_host_join(self._eng, P(self.stream.cuda_stream)),
                       "cg_engine_host_join")

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
        return self.pos[:self.n].cpu().numpy()

    def velocities(self) -> np.ndarray:
        self.stream.synchronize()
        return self.vel[:self.n].cpu().numpy()

    def previous_velocities(self) -> np.ndarray:
        """The AB2 state (the previous step's velocities)."""
        self.stream.synchronize()
        return self.prev_vel[:self.n].cpu().numpy()

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
