"""z-slab domain decomposition across GPUs.

One process per GPU; rank r owns the global planes ``slab_bounds(nz, P)[r]``
and the cells whose voxel lies in them.  Per mechanics step (the order of
simulate.py:169-202):

* diffusion substeps: per-cell exchange and the x/y sweeps are slab-local;
  the z sweep is a partitioned Thomas solve -- local block solve
  (cg_lod_step in slab mode), one all-gather of each line's two end values
  (2 doubles per line per rank), and the per-line 2x2 block-tridiagonal
  interface solve + correction (cg_zslab_correct); see slab.py;
* ghost cells: the cells of the first / last owned plane (positions, radii,
  global ids) go to the neighbour below / above; velocities are computed on an
  extended mesh (one ghost plane each side) and kept for owned cells only.
  Candidates are accumulated in global-id order, so velocities and positions
  equal the single-GPU ones bit for bit;
* integration (global box clamp), then migration of cells whose voxel left
  the slab to the neighbouring rank (cg_voxel_z decides, CPython-exact), and
  the local rebin.

Communication uses torch.distributed: NCCL on device tensors, or gloo with
host staging (used by the tests, including 2 ranks sharing one GPU -- no
kernel ever waits on another rank's kernel; the host does the waiting).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .configs import SimConfig
from .core import CartesianMesh
from .errors import CapacityError
from .mechanics import InteractionParams
from .slab import plane_costs, slab_bounds, weighted_bounds


def slab_mesh(mesh: CartesianMesh, z0: int, z1: int, ghost: int = 0) -> CartesianMesh:
    ox, oy, oz = mesh.origin
    return CartesianMesh(mesh.nx, mesh.ny, z1 - z0 + 2 * ghost, mesh.dx, mesh.dy, mesh.dz,
                         (ox, oy, oz + (z0 - ghost) * mesh.dz))


class _Done:
    """Handle of a collective that has completed already."""

    def wait(self):
        return None


class Comm:
    """Thin torch.distributed wrapper: device tensors for NCCL, host staging
    for gloo (and plain CPU tensors in the CPU tests).  ``dist=None`` is the
    single-rank case."""

    def __init__(self, dist=None, device="cpu", group=None):
        self.dist = dist
        self.device = device
        self.group = group
        self.rank = dist.get_rank() if dist is not None else 0
        self.world = dist.get_world_size() if dist is not None else 1
        self.host = dist is None or dist.get_backend() != "nccl"

    def split(self) -> "Comm":
        """The same ranks on a communicator of their own (collective: every
        rank calls it).  The slab step's mechanics exchanges run on it, on
        their own stream, beside the substeps' interface all-gathers."""
        if self.world == 1:
            return Comm(self.dist, self.device)
        return Comm(self.dist, self.device, self.dist.new_group(list(range(self.world))))

    def all_gather(self, out, inp):
        """out: (world, *inp.shape)."""
        if self.world == 1:
            out.copy_(inp.reshape(out.shape))
            return
        if self.host:
            parts = [p for p in out.cpu().unbind(0)]
            self.dist.all_gather(parts, inp.cpu().contiguous(), group=self.group)
            out.copy_(__import__("torch").stack(parts))
        else:
            self.dist.all_gather_into_tensor(out, inp.contiguous(), group=self.group)

    def all_to_all(self, out, inp):
        """out[k] = rank k's inp[self.rank] (inp, out: (world, ...) with equal
        blocks)."""
        if self.world == 1:
            out.copy_(inp)
            return
        if self.host:
            o = out.cpu()
            self.dist.all_to_all_single(o, inp.cpu().contiguous(), group=self.group)
            out.copy_(o)
        else:
            self.dist.all_to_all_single(out, inp.contiguous(), group=self.group)

    def all_to_all_async(self, out, inp):
        """all_to_all without waiting: the returned handle's wait() makes the
        current stream wait for it (NCCL); host-staged backends complete it
        here."""
        if self.world == 1 or self.host:
            self.all_to_all(out, inp)
            return _Done()
        return self.dist.all_to_all_single(out, inp, group=self.group, async_op=True)

    def all_gather_async(self, out, inp):
        """all_gather (out: (world, *inp.shape)) without waiting, as all_to_all_async."""
        if self.world == 1 or self.host:
            self.all_gather(out, inp)
            return _Done()
        return self.dist.all_gather_into_tensor(out, inp, group=self.group, async_op=True)

    def exchange_rows(self, send_lo, send_hi, width):
        """Variable-length row exchange with the neighbours r-1 (lo) and r+1
        (hi): returns (from_lo, from_hi), float64 (k, width) tensors."""
        import torch

        dist = self.dist
        r, P = self.rank, self.world
        empty = torch.empty((0, width), dtype=torch.float64, device=self.device)
        if P == 1:
            return empty, empty
        dev = "cpu" if self.host else self.device
        peers = []
        if r > 0:
            peers.append(("lo", r - 1, send_lo))
        if r < P - 1:
            peers.append(("hi", r + 1, send_hi))
        ops, cnt_recv, cnt_send = [], {}, {}
        for name, peer, t in peers:
            cnt_send[name] = torch.tensor([t.shape[0]], dtype=torch.int64, device=dev)
            cnt_recv[name] = torch.zeros(1, dtype=torch.int64, device=dev)
            ops.append(dist.P2POp(dist.isend, cnt_send[name], peer, self.group))
            ops.append(dist.P2POp(dist.irecv, cnt_recv[name], peer, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        ops, bufs, keep = [], {}, []
        for name, peer, t in peers:
            k = int(cnt_recv[name].item())
            bufs[name] = torch.empty((k, width), dtype=torch.float64, device=dev)
            payload = t.to(dev).contiguous()
            keep.append(payload)
            if payload.shape[0]:
                ops.append(dist.P2POp(dist.isend, payload, peer, self.group))
            if k:
                ops.append(dist.P2POp(dist.irecv, bufs[name], peer, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        lo = bufs.get("lo", empty).to(self.device)
        hi = bufs.get("hi", empty).to(self.device)
        return lo, hi

    def max(self, x: float) -> float:
        import torch

        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if self.host else self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def sum(self, x: int) -> int:
        import torch

        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.int64, device="cpu" if self.host else self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return int(t.item())


class SlabSimulation:
    """This rank's slab of a z-decomposed run of the step loop."""

    def __init__(self, mesh: CartesianMesh, comm: Comm, *, diffusion, decay, densities, positions,
                 radius, ids, secretion, uptake, saturation=38.0, bc="dirichlet", dirichlet=None,
                 params: InteractionParams = InteractionParams(), dt_diffusion=0.01,
                 dt_mechanics=0.1, integrator="ab2", bounds=None, numerics="exact",
                 resort_every=0):
        """``densities``: this rank's (S, nvox_local) field; cell arrays: the
        cells this rank owns (their voxel lies in the slab).  ``bounds``: every
        rank's [z0, z1) (default: the balanced split; see load_balanced_bounds).

        One rank (P = 1) owns the whole box: no ghosts, no migration, no
        interface system -- the step is the single-GPU graph engine's
        (engine.Simulation, ``numerics`` as there), so the weak-scaling curve's
        N = 1 point is the engine itself.  P > 1 with numerics="fast" (and a
        mesh with fast kernels, e.g. config 4's 256 x 256 slabs) runs the fast
        x/y kernels with the affine exchange fused, the partitioned z sweep
        and the fast velocities (cg_*_fast)."""
        torch = _lib.require_cuda()
        self.torch = torch
        self.comm = comm
        self.mesh = mesh
        P, r = comm.world, comm.rank
        self.engine = None
        if P == 1:
            from .engine import Simulation

            self.bounds = [(0, mesh.nz)]
            self.z0, self.z1 = 0, mesh.nz
            self.local = mesh
            self.S = len(np.atleast_1d(diffusion))
            self.engine = Simulation(
                mesh, diffusion=diffusion, decay=decay, densities=densities, positions=positions,
                radius=radius, ids=ids, secretion=secretion, uptake=uptake, saturation=saturation,
                bc=bc, dirichlet=dirichlet, params=params, dt_diffusion=dt_diffusion,
                dt_mechanics=dt_mechanics, integrator=integrator, numerics=numerics,
                resort_every=resort_every)
            self.stream = self.engine.stream
            self.dens = self.engine.dens
            self.dev = self.dens.device
            self._n = self.engine.n
            return
        self.bounds = list(bounds) if bounds is not None else slab_bounds(mesh.nz, P)
        if len(self.bounds) != P:
            raise ValueError("one (z0, z1) range per rank")
        self.z0, self.z1 = self.bounds[r]
        self.local = slab_mesh(mesh, self.z0, self.z1)
        self.ext = slab_mesh(mesh, self.z0, self.z1, ghost=1)
        self.D = np.ascontiguousarray(diffusion, np.float64).reshape(-1)
        self.S = S = self.D.shape[0]
        self.K = np.ascontiguousarray(decay, np.float64).reshape(S)
        self.diri = (np.zeros(S) if dirichlet is None else
                     np.ascontiguousarray(np.broadcast_to(np.asarray(dirichlet, np.float64), (S,))))
        self.sat = np.ascontiguousarray(np.broadcast_to(np.asarray(saturation, np.float64), (S,)))
        self.bc = _lib.BC_DIRICHLET if bc == "dirichlet" else _lib.BC_NEUMANN
        self.integrator = _lib.AB2 if integrator == "ab2" else _lib.EULER
        self.params = params
        self.numerics = numerics
        self.dt_d, self.dt_m = float(dt_diffusion), float(dt_mechanics)
        self.substeps = int(round(dt_mechanics / dt_diffusion))
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.stream = torch.cuda.current_stream(dev)
        f64 = torch.float64
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        self.dens = t(np.asarray(densities, np.float64).reshape(S, self.local.voxel_count))
        n = len(ids)
        self.cap = max(4 * n, 4096)
        # Overlapped step (default; env CELLGPU_SLAB_OVERLAP=0: one stream):
        # the mechanics (ghosts, velocities, integration, migration, rebin)
        # run on a side stream with a communicator of their own, beside the
        # substeps and their interface all-gathers on the main stream.  The
        # rebin of step k writes the exchange maps and bins step k + 1's
        # substeps read, so there are two sets (one context + bins each):
        # step k's substeps read set k % 2 while its mechanics write the other.
        self.overlap = os.environ.get("CELLGPU_SLAB_OVERLAP", "1") != "0"
        starts = (ctypes.c_int * (P + 1))(*([b[0] for b in self.bounds] + [mesh.nz]))
        self.ctxs = []
        for _ in range(2 if self.overlap else 1):
            cx = _lib.Context(self.local, S, self.cap, dev.index)
            cx.bind_stream(self.stream)
            _lib.raise_for(_lib.load().cg_ctx_set_slab_bounds(cx.handle, r, P, mesh.nz, starts),
                           "cg_ctx_set_slab_bounds")
            self.ctxs.append(cx)
        self.ctx = self.ctxs[0]
        self.side = torch.cuda.Stream(dev) if self.overlap else self.stream
        self.mcomm = comm.split() if self.overlap else comm
        self._k = 0  # steps taken: set k % 2 is the current one
        self._ev_main = torch.cuda.Event()
        self._ev_side = torch.cuda.Event()
        self.ctx_ext = _lib.Context(self.ext, 0, self.cap, dev.index)
        self.ctx_ext.bind_stream(self.side)
        self.ctx_glob = _lib.Context(mesh, 0, self.cap, dev.index)
        self.ctx_glob.bind_stream(self.side)
        # The interface system: by line blocks with two all-to-alls (P >= 3:
        # 2 (P - 1) / P instead of P - 1 times S 2 L doubles received per rank;
        # bit-identical) or all-gathered and solved redundantly (P = 2: the
        # same volume, one exchange); env CELLGPU_SLAB_IFACE=gather|blocks.
        mode = os.environ.get("CELLGPU_SLAB_IFACE", "")
        self.blocks = mode == "blocks" or (mode != "gather" and P >= 3)
        # owned cells (storage order) in capacity buffers; self.cells holds
        # views of the first n rows (migration edits the buffers in place)
        pos = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
        rad = np.ascontiguousarray(radius, np.float64).reshape(-1)
        init = {
            "pos": t(pos), "vel": torch.zeros((n, 3), dtype=f64, device=dev),
            "prev": torch.zeros((n, 3), dtype=f64, device=dev), "radius": t(rad),
            "volume": t(_lib.cell_volumes(rad)), "ids": t(np.asarray(ids, np.int64)),
            "sec": t(np.asarray(secretion, np.float64).reshape(S, n).T.copy()),
            "upt": t(np.asarray(uptake, np.float64).reshape(S, n).T.copy()),
        }
        self.buf = {}
        for k, v in init.items():
            b = torch.zeros((self.cap,) + tuple(v.shape[1:]), dtype=v.dtype, device=dev)
            b[:n] = v
            self.buf[k] = b
        self._set_n(n)
        self.bin_sets = [self._bins_for(n, self.local.voxel_count) for _ in self.ctxs]
        self.fast = (numerics == "fast" and S > 0 and
                     _lib.load().cg_fast_lod_available(self.ctx.handle) != 0)
        self._alloc_interface()
        self._sec_sn = [None] * len(self.ctxs)
        self._upt_sn = [None] * len(self.ctxs)
        self._rebin_local(0)
        self.sync()

    def _alloc_interface(self):
        """Exchange buffers of the interface system.  Per-substrate pipeline
        (fast kernels, S > 1; env CELLGPU_SLAB_PIPE=1): substrate s's
        interface exchange is in flight while substrate s + 1's sweeps run
        (substrate windows on the context, one buffer set per substrate);
        the same kernels per substrate, so the fields are bit-identical.  Off
        by default: it multiplies the host calls per substep by S (config 4:
        ~29 library calls and 8 collectives per substep, ~0.3 ms of Python
        against ~0.1 ms of device time), so without the substeps captured in
        a graph the step would become host-bound."""
        torch = self.torch
        f64, dev, P, S = torch.float64, self.dev, self.comm.world, self.S
        L = self.mesh.nx * self.mesh.ny
        self.pipe = (self.fast and S > 1 and os.environ.get("CELLGPU_SLAB_PIPE", "0") != "0")
        G = S if self.pipe else 1   # buffer sets
        W = 1 if self.pipe else S   # substrates per set
        # Deferred correction (fast kernels, not pipelined; env
        # CELLGPU_SLAB_DEFER=0 off): substeps 1..n-1 hand their interface
        # correction to the next substep's x-row / plane kernel, which applies
        # it while staging the field (cg_zslab_defer) -- one full read + write
        # pass of the field saved per substep; bit-identical.
        self.defer = (self.fast and not self.pipe and
                      os.environ.get("CELLGPU_SLAB_DEFER", "1") != "0")
        Lb = int(_lib.load().cg_zslab_block_lines(self.ctxs[0].handle))
        self.lrg = (torch.empty((P, S, 2, Lb), dtype=f64, device=dev)
                    if self.defer and not self.blocks else None)
        if self.blocks:
            shape = (G, P, W, 2, Lb)
            self.send = torch.empty(shape, dtype=f64, device=dev)
            self.recv = torch.empty(shape, dtype=f64, device=dev)
            self.red = torch.empty(shape, dtype=f64, device=dev)
            self.lr = torch.empty(shape, dtype=f64, device=dev)
        else:
            self.send = torch.empty((G, W, 2, L), dtype=f64, device=dev)
            self.recv = torch.empty((G, P, W, 2, L), dtype=f64, device=dev)

    # ---- helpers
    @property
    def n(self) -> int:
        return self._n

    def _set_n(self, n: int) -> None:
        self._n = n
        self.cells = {k: b[:n] for k, b in self.buf.items()}

    def _bins_for(self, n, nvox):
        torch = self.torch
        i32 = torch.int32
        d = self.dev
        return {"voxel": torch.zeros(max(n, 1), dtype=i32, device=d),
                "bin_start": torch.zeros(nvox + 1, dtype=i32, device=d),
                "bin_cells": torch.zeros(max(n, 1), dtype=i32, device=d),
                "by_id": torch.zeros(max(n, 1), dtype=i32, device=d),
                "nonempty": torch.zeros(nvox, dtype=i32, device=d),
                "n_ne": torch.zeros(1, dtype=i32, device=d)}

    @property
    def bins(self):
        """Bins of the owned cells (the set the next step reads)."""
        return self.bin_sets[self._k % len(self.bin_sets)]

    def _ensure_cap(self, n):
        if n > self.cap:
            raise CapacityError(f"rank {self.comm.rank}: {n} cells exceed the slab capacity {self.cap}")

    def _rebin(self, ctx, n, pos, ids, b):
        P = _lib.ptr
        _lib.raise_for(_lib.load().cg_rebin(ctx.handle, n, P(pos), P(ids), P(b["voxel"]),
                                            P(b["bin_start"]), P(b["bin_cells"]), P(b["by_id"]),
                                            P(b["nonempty"]), P(b["n_ne"])), "cg_rebin (slab)")

    def _rebin_local(self, k):
        """Re-bin the owned cells into set k; the same pass computes the
        exchange coefficients the next step's substeps reuse
        (cg_rebin_exchange), in set k's context.  Runs on that context's
        stream (the side stream inside a step)."""
        c = self.cells
        n = self.n
        if self.bin_sets[k]["voxel"].shape[0] < max(n, 1):
            self.bin_sets[k] = self._bins_for(n, self.local.voxel_count)
        b = self.bin_sets[k]
        ctx = self.ctxs[k]
        if n == 0:
            self._rebin(ctx, n, c["pos"], c["ids"], b)
            return
        P = _lib.ptr
        # (S, n) for the C-ABI, kept alive until set k is rebinned again
        self._sec_sn[k] = c["sec"].T.contiguous()
        self._upt_sn[k] = c["upt"].T.contiguous()
        L_ = _lib.load()
        fn = L_.cg_rebin_exchange_affine if self.fast else L_.cg_rebin_exchange
        _lib.raise_for(fn(
            ctx.handle, n, P(c["pos"]), P(c["ids"]), P(b["voxel"]), P(b["bin_start"]),
            P(b["bin_cells"]), P(b["by_id"]), P(b["nonempty"]), P(b["n_ne"]), self.dt_d,
            P(self._sec_sn[k]), P(self._upt_sn[k]), self.sat.ctypes.data_as(ctypes.c_void_p),
            P(c["volume"])), "cg_rebin_exchange (slab)")

    def join(self):
        """Make the main stream wait for the last step's mechanics."""
        if self.engine is None and self.overlap:
            self.stream.wait_event(self._ev_side)

    def sync(self):
        if self.engine is not None:
            self.engine.sync()
            return
        self.join()
        for cx in self.ctxs:
            cx.sync("slab step")
        self.ctx_ext.sync("slab velocities")
        self.ctx_glob.sync("slab integrate")
        self.side.synchronize()

    # ---- one mechanics step
    def step(self):
        if self.engine is not None:
            self.engine.run(1)
            return
        torch = self.torch
        cur = self._k % len(self.ctxs)
        nxt = (self._k + 1) % len(self.ctxs)
        if self.overlap:
            # the side stream may overwrite set nxt once the previous step's
            # substeps (which read it) are done; this step's substeps need
            # the previous step's mechanics (set cur, the cell table)
            self.side.wait_event(self._ev_main)
            self.stream.wait_event(self._ev_side)
        n = self.n
        self._substeps(cur, n)
        if self.overlap:
            self._ev_main.record(self.stream)
        with torch.cuda.stream(self.side):
            self._mechanics(cur, n)
            self._migrate()
            self.ctxs[nxt].bind_stream(self.side)
            self._rebin_local(nxt)
        if self.overlap:
            self._ev_side.record(self.side)
        self._k += 1

    def _substeps(self, cur, n):
        """The diffusion substeps on the main stream: slab-local exchange and
        x/y sweeps, the local z block solve, the interface exchange (one
        all-gather, or two all-to-alls by line blocks), the correction.  No
        host synchronisation.  Pipelined (self.pipe): per substrate, so one
        substrate's exchange is in flight under the next one's sweeps."""
        torch = self.torch
        L_ = _lib.load()
        P = _lib.ptr
        vp = ctypes.c_void_p
        ctx = self.ctxs[cur]
        ctx.bind_stream(self.stream)
        b = self.bin_sets[cur]
        h = ctx.handle
        diri = self.diri.ctypes.data_as(vp)

        def sweeps():
            if self.fast:
                # affine exchange fused into the fast x-row / plane kernel
                _lib.raise_for(L_.cg_lod_step_fast(
                    h, P(self.dens), self.D.ctypes.data_as(vp), self.K.ctypes.data_as(vp),
                    self.dt_d, self.bc, diri, 1 if n else 0), "lod_step_fast (slab)")
            else:
                if n:
                    _lib.raise_for(L_.cg_exchange_prepared(
                        h, P(self.dens), n, P(b["nonempty"]), P(b["n_ne"])), "exchange (slab)")
                _lib.raise_for(L_.cg_lod_step(
                    h, P(self.dens), self.D.ctypes.data_as(vp), self.K.ctypes.data_as(vp),
                    self.dt_d, self.bc, diri), "lod_step (slab)")

        def window(s0, ns):
            _lib.raise_for(L_.cg_ctx_set_substrate_window(h, s0, ns), "substrate window")

        parts = list(range(self.S)) if self.pipe else [None]
        with torch.cuda.stream(self.stream):
            for k in range(self.substeps):
                # all but the last substep leave their correction to the next
                defer = self.defer and k + 1 < self.substeps
                first = []
                for g, s in enumerate(parts):
                    if s is not None:
                        window(s, 1)
                    sweeps()
                    if self.blocks:
                        _lib.raise_for(L_.cg_zslab_pack_blocks(h, P(self.dens), P(self.send[g])),
                                       "zslab_pack_blocks")
                        first.append(self.comm.all_to_all_async(self.recv[g], self.send[g]))
                    else:
                        _lib.raise_for(L_.cg_zslab_pack(h, P(self.dens), P(self.send[g])),
                                       "zslab_pack")
                        first.append(self.comm.all_gather_async(self.recv[g], self.send[g]))
                second = []
                for g, s in enumerate(parts):
                    first[g].wait()
                    if s is not None:
                        window(s, 1)
                    if self.blocks:
                        _lib.raise_for(L_.cg_zslab_reduce_blocks(h, P(self.recv[g]), P(self.red[g])),
                                       "zslab_reduce_blocks")
                        second.append(self.comm.all_to_all_async(self.lr[g], self.red[g]))
                    elif defer:
                        _lib.raise_for(L_.cg_zslab_lr_gather(h, P(self.recv[g]), P(self.lrg)),
                                       "zslab_lr_gather")
                        _lib.raise_for(L_.cg_zslab_defer(h, P(self.lrg)), "zslab_defer")
                    else:
                        _lib.raise_for(L_.cg_zslab_correct(h, P(self.dens), P(self.recv[g]), self.bc,
                                                           diri), "zslab_correct")
                if self.blocks:
                    for g, s in enumerate(parts):
                        second[g].wait()
                        if s is not None:
                            window(s, 1)
                        if defer:
                            _lib.raise_for(L_.cg_zslab_defer(h, P(self.lr[g])), "zslab_defer")
                            continue
                        _lib.raise_for(L_.cg_zslab_correct_blocks(h, P(self.dens), P(self.lr[g]),
                                                                  self.bc, diri),
                                       "zslab_correct_blocks")
                if self.pipe:
                    window(0, 0)

    def _mechanics(self, cur, n):
        """Velocities of the owned cells (ghost cells of the neighbours'
        boundary planes included in the candidate sets) and integration, on
        the current (side) stream, from the bins of set cur."""
        torch = self.torch
        L_ = _lib.load()
        P = _lib.ptr
        c = self.cells
        b = self.bin_sets[cur]
        vel_args = (float(self.params.repulsion), float(self.params.adhesion),
                    float(self.params.adhesion_multiplier))
        # ghosts: owned cells of the first / last plane go to the neighbours
        plane = self.local.nx * self.local.ny
        bs = b["bin_start"]
        # one host read for both ghost ranges (cells of the first / last plane)
        idx = torch.tensor([plane, self.local.voxel_count - plane], device=self.dev)
        lo_end, hi_beg = (int(v) for v in bs.index_select(0, idx).cpu().tolist())
        by_id = b["by_id"][:n].long()

        def rows(idx):
            return torch.cat([c["pos"][idx], c["radius"][idx, None],
                              c["ids"][idx, None].double()], dim=1)

        g_lo, g_hi = self.mcomm.exchange_rows(rows(by_id[:lo_end]), rows(by_id[hi_beg:]), 5)
        ghosts = torch.cat([g_lo, g_hi])
        n_all = n + ghosts.shape[0]
        self._ensure_cap(n_all)
        pos_all = torch.cat([c["pos"], ghosts[:, 0:3]]).contiguous()
        rad_all = torch.cat([c["radius"], ghosts[:, 3]]).contiguous()
        ids_all = torch.cat([c["ids"], ghosts[:, 4].round().long()]).contiguous()
        vel_all = torch.zeros((n_all, 3), dtype=torch.float64, device=self.dev)
        eb = self._bins_for(n_all, self.ext.voxel_count)
        if n_all:
            self._rebin(self.ctx_ext, n_all, pos_all, ids_all, eb)
            if self.fast:
                _lib.raise_for(L_.cg_velocities_fast(
                    self.ctx_ext.handle, n_all, P(pos_all), P(rad_all), P(eb["voxel"]),
                    P(eb["bin_start"]), P(eb["by_id"]), *vel_args, P(vel_all)),
                    "velocities_fast (slab)")
            else:
                _lib.raise_for(L_.cg_velocities(
                    self.ctx_ext.handle, n_all, P(pos_all), P(rad_all), P(ids_all),
                    P(eb["bin_start"]), P(eb["by_id"]), P(eb["nonempty"]), P(eb["n_ne"]),
                    *vel_args, P(vel_all)), "velocities (slab)")
        self.buf["vel"][:n] = vel_all[:n]
        if n:
            _lib.raise_for(L_.cg_integrate(self.ctx_glob.handle, n, P(c["pos"]), P(c["vel"]),
                                           P(c["prev"]), self.dt_m, self.integrator),
                           "integrate (slab)")

    def _migrate(self):
        """Cells whose voxel left the slab go to the neighbour rank with their
        whole state.  One host read per step sizes everything (how many cells
        go down / up, and whether any moved further than one slab): a stable
        sort by destination puts the leavers at the two ends and the stayers
        in their storage order in between, the stayers are compacted to the
        front and arrivals appended (storage order within a rank does not
        affect any result: exchange and velocities run in id order)."""
        torch = self.torch
        c = self.cells
        n = self.n
        S = self.S
        z = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        if n:
            _lib.raise_for(_lib.load().cg_voxel_z(self.ctx_glob.handle, n, _lib.ptr(c["pos"]),
                                                  _lib.ptr(z)), "voxel_z")
        order, n_lo, n_hi, n_far = migration_plan(z[:n], self.z0, self.z1)
        if n_far and self.comm.world > 1:
            raise RuntimeError("a cell moved further than one slab in one step")
        width = 12 + 2 * S
        cols = ("pos", "vel", "prev", "radius", "volume", "ids", "sec", "upt")

        def pack(idx):
            return torch.cat([c["pos"][idx], c["vel"][idx], c["prev"][idx],
                              c["radius"][idx, None], c["volume"][idx, None],
                              c["ids"][idx, None].double(), c["sec"][idx], c["upt"][idx]], dim=1)

        empty = torch.empty(0, dtype=torch.long, device=self.dev)
        lo_idx = order[:n_lo] if n_lo else empty
        hi_idx = order[n - n_hi:] if n_hi else empty
        in_lo, in_hi = self.mcomm.exchange_rows(pack(lo_idx), pack(hi_idx), width)
        incoming = torch.cat([in_lo, in_hi])
        k_out = n_lo + n_hi
        if k_out == 0 and incoming.shape[0] == 0:
            return  # the cell table is unchanged
        n_keep = n - k_out
        self._ensure_cap(n_keep + incoming.shape[0])
        if k_out:
            stay = order[n_lo:n - n_hi]
            for k in cols:
                self.buf[k][:n_keep] = self.buf[k][stay]
        m = incoming.shape[0]
        if m:
            sl = slice(n_keep, n_keep + m)
            self.buf["pos"][sl] = incoming[:, 0:3]
            self.buf["vel"][sl] = incoming[:, 3:6]
            self.buf["prev"][sl] = incoming[:, 6:9]
            self.buf["radius"][sl] = incoming[:, 9]
            self.buf["volume"][sl] = incoming[:, 10]
            self.buf["ids"][sl] = incoming[:, 11].round().long()
            self.buf["sec"][sl] = incoming[:, 12:12 + S]
            self.buf["upt"][sl] = incoming[:, 12 + S:12 + 2 * S]
        self._set_n(n_keep + m)

    # ---- gradients (diffusion.py:237-278) with a one-plane halo
    def gradients(self):
        """(S, local voxels, 3) central-difference gradients of this slab's
        field, boundary-face components zero on the global box only: the
        neighbours' adjacent planes come in as a halo (one plane per
        substrate each way) and the kernel runs on the slab extended by them,
        so the slab's end planes are interior exactly where the global mesh
        has a neighbour.  Equal bit for bit to the gradients of the gathered
        field on one GPU."""
        torch = self.torch
        S, plane = self.S, self.local.nx * self.local.ny
        nz = self.local.nz
        d = self.dens.view(S, nz, plane)
        lo_halo, hi_halo = self.comm.exchange_rows(d[:, 0, :], d[:, nz - 1, :], plane)
        has_lo, has_hi = self.comm.rank > 0, self.comm.rank < self.comm.world - 1
        parts = ([lo_halo.view(S, 1, plane)] if has_lo else []) + [d] + \
                ([hi_halo.view(S, 1, plane)] if has_hi else [])
        ext_field = torch.cat(parts, dim=1).contiguous()
        z0 = self.z0 - (1 if has_lo else 0)
        mesh = slab_mesh(self.mesh, z0, z0 + ext_field.shape[1])
        key = (mesh.nz, mesh.origin)
        if getattr(self, "_grad_ctx_key", None) != key:
            self._grad_ctx = _lib.Context(mesh, S, 1, self.dev.index)
            self._grad_ctx_key = key
        ctx = self._grad_ctx
        ctx.bind_stream(self.stream)
        g = torch.empty((S, ext_field.shape[1] * plane, 3), dtype=torch.float64, device=self.dev)
        _lib.raise_for(_lib.load().cg_gradients(ctx.handle, _lib.ptr(ext_field), _lib.ptr(g)),
                       "gradients (slab)")
        first = plane if has_lo else 0
        return g[:, first:first + nz * plane, :].contiguous()

    # ---- results
    def owned_state(self):
        """(ids, pos, vel) of the owned cells, sorted by id (host numpy)."""
        self.sync()
        if self.engine is not None:
            ids = self.engine.cell_ids()
            o = np.argsort(ids)
            return ids[o], self.engine.positions()[o], self.engine.velocities()[o]
        ids = self.cells["ids"].cpu().numpy()
        o = np.argsort(ids)
        return (ids[o], self.cells["pos"].cpu().numpy()[o], self.cells["vel"].cpu().numpy()[o])

    def densities(self):
        self.sync()
        return self.dens.cpu().numpy()

    def close(self):
        if self.engine is not None:
            self.engine.close()
            self.engine = None


def migration_plan(z, z0: int, z1: int):
    """Where each owned cell goes after a move, from its global voxel plane z
    (cg_voxel_z): (order, n_lo, n_hi, n_far) with order a stable permutation
    putting the n_lo cells bound for rank r - 1 (z < z0) first, the stayers in
    storage order next and the n_hi cells bound for rank r + 1 (z >= z1) last;
    n_far counts cells more than one plane outside (an error).  One host read
    (the three counts)."""
    import torch

    dest = (z >= z1).to(torch.int32) - (z < z0).to(torch.int32)  # -1 / 0 / +1
    far = (z < z0 - 1) | (z > z1)
    counts = torch.stack([(dest < 0).sum(), (dest > 0).sum(), far.sum()]).cpu().tolist()
    n_lo, n_hi, n_far = (int(v) for v in counts)
    order = torch.sort(dest, stable=True).indices if n_lo + n_hi else None
    return order, n_lo, n_hi, n_far


def cell_planes(mesh: CartesianMesh, positions) -> np.ndarray:
    """Voxel z of every cell (host CPython-semantics voxel_of, as the device)."""
    plane = mesh.nx * mesh.ny
    return np.array([mesh.voxel_of(p) // plane for p in np.asarray(positions).tolist()],
                    dtype=np.int64)


def load_balanced_bounds(cfg: SimConfig, inp, world: int, alpha: float = 1.0,
                         beta: float = 10.0) -> list:
    """Slab bounds balancing alpha * voxels + beta * cells per rank (SURVEY.md
    section 8f row 1): for config 2's spheroid the central planes hold most
    cells, so equal plane counts leave the middle ranks doing most work."""
    mesh = cfg.mesh()
    costs = plane_costs(mesh.nz, mesh.nx * mesh.ny, cell_planes(mesh, inp.positions), alpha, beta)
    return weighted_bounds(costs, world)


def split_inputs(cfg: SimConfig, inp, rank: int, world: int, bounds=None):
    """This rank's share of globally generated inputs (strong scaling): its
    slab of the field and the cells whose voxel z lies in the slab."""
    mesh = cfg.mesh()
    z0, z1 = (bounds if bounds is not None else slab_bounds(mesh.nz, world))[rank]
    S = cfg.n_substrates
    plane = mesh.nx * mesh.ny
    dens = inp.densities.reshape(S, mesh.nz, plane)[:, z0:z1].reshape(S, -1)
    zs = cell_planes(mesh, inp.positions)
    own = (zs >= z0) & (zs < z1)
    return dict(densities=dens, positions=inp.positions[own], radius=inp.radius[own],
                ids=inp.ids[own], secretion=inp.secretion[:, own], uptake=inp.uptake[:, own])


def build(cfg: SimConfig, comm: Comm, inp, bounds=None, **kw) -> SlabSimulation:
    """This rank's SlabSimulation of globally generated inputs (``kw``:
    numerics, resort_every)."""
    part = split_inputs(cfg, inp, comm.rank, comm.world, bounds)
    return SlabSimulation(
        cfg.mesh(), comm, diffusion=cfg.diffusion, decay=cfg.decay,
        saturation=cfg.saturation, bc=cfg.bc, dirichlet=cfg.dirichlet,
        params=InteractionParams(cfg.repulsion, cfg.adhesion, cfg.adhesion_multiplier),
        dt_diffusion=cfg.dt_diffusion, dt_mechanics=cfg.dt_mechanics, integrator=cfg.integrator,
        bounds=bounds, **part, **kw)


def timed_steps(sim: SlabSimulation, steps: int) -> float:
    """Device time of `steps` mechanics steps, max over ranks (ms per step);
    one rank with voxel-sorted storage: the window starts after a resort and
    the amortised share of one resort is added."""
    torch = sim.torch
    eng = sim.engine
    R = eng.resort_every if eng is not None else 0
    if R > 0 and eng.steps_done % R:  # start right after a resort (see bench.py)
        eng.run(R - eng.steps_done % R)
    sim.sync()
    if sim.comm.world > 1:
        sim.comm.dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(sim.stream)
    for _ in range(steps):
        sim.step()
    sim.join()
    b.record(sim.stream)
    b.synchronize()
    total = a.elapsed_time(b)
    frac = steps / R - steps // R if R > 0 else 0.0
    if frac > 0:  # the amortised share of the resorts the window did not hold
        a.record(sim.stream)
        eng.sort_cells_by_voxel()
        b.record(sim.stream)
        b.synchronize()
        total += frac * a.elapsed_time(b)
    ms = total / max(steps, 1)
    if sim.comm.world > 1:
        sim.comm.dist.barrier()
    return sim.comm.max(ms)


__all__ = ["Comm", "SlabSimulation", "build", "migration_plan", "split_inputs", "slab_mesh",
           "timed_steps"]
