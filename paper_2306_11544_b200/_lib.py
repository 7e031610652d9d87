"""ctypes binding of libcellgpu.so (include/cellgpu.h).

This is the only path to the compute: there is no CPU fallback.  If the
library is missing or no CUDA device is visible, every device call raises
``DeviceError`` -- loudly, by design.
"""

from __future__ import annotations

import ctypes
import os

from .errors import CapacityError, ContainerStateError, DeviceError, DomainError, NumericError

_HERE = os.path.dirname(os.path.abspath(__file__))
# CELLGPU_LIB: alternative build of the same library (e.g. the phase-probe build).
LIB_PATH = os.environ.get("CELLGPU_LIB") or os.path.join(_HERE, "libcellgpu.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "cellgpu.h")

CG_OK, CG_DOMAIN, CG_NUMERIC, CG_STATE, CG_CAPACITY, CG_CUDA = 0, 1, 2, 3, 4, 100
BC_NEUMANN, BC_DIRICHLET = 0, 1
EULER, AB2 = 0, 1

# Every symbol include/cellgpu.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "cg_version", "cg_last_error", "cg_ctx_create", "cg_ctx_destroy", "cg_ctx_set_stream",
    "cg_sync", "cg_lod_step", "cg_exchange", "cg_exchange_cells", "cg_rebin", "cg_velocities",
    "cg_integrate", "cg_engine_create", "cg_engine_destroy", "cg_engine_run",
    "cg_engine_io_enable", "cg_engine_io_inputs_ready", "cg_engine_io_wait_fields",
    "cg_engine_io_fields_ready", "cg_engine_io_wait_cells", "cg_host_alloc", "cg_host_free",
    "cg_engine_io_substrate_ready", "cg_engine_io_wait_substrate", "cg_engine_substrate_chains",
    "cg_engine_step_io", "cg_engine_io_join", "cg_check_state",
    "cg_division_draws", "cg_divisions_count", "cg_divisions_place",
    "cg_engine_step_host", "cg_engine_host_join",
    "cg_engine_launches_per_step", "cg_engine_sort_cells", "cg_engine_set_cell_count", "cg_engine_time_stages", "cg_prof_enable", "cg_prof_read", "cg_launch_count",
    "cg_cell_volumes", "cg_state_checksum", "cg_gradients", "cg_rebin_exchange", "cg_exchange_prepared", "cg_ctx_set_slab", "cg_ctx_set_slab_bounds", "cg_zslab_pack", "cg_zslab_correct", "cg_zslab_block_lines", "cg_zslab_lr_gather", "cg_zslab_defer", "cg_ctx_set_substrate_window", "cg_zslab_pack_blocks", "cg_zslab_reduce_blocks", "cg_zslab_correct_blocks", "cg_voxel_z", "cg_voxel_index",
    "cg_rebin_exchange_affine", "cg_lod_step_fast", "cg_velocities_fast", "cg_fast_lod_available",
)

P = ctypes.c_void_p
I = ctypes.c_int
D = ctypes.c_double


class StatePtrs(ctypes.Structure):
    """cg_state_ptrs"""
    _fields_ = [(name, P) for name in (
        "dens", "pos", "vel", "prev_vel", "radius", "volume", "ids", "secretion", "uptake",
        "voxel", "bin_start", "bin_cells", "bin_cells_by_id", "nonempty", "n_nonempty", "grad",
        "division_rate")]


class StepParams(ctypes.Structure):
    """cg_step_params"""
    _fields_ = [
        ("n_cells", I), ("substeps", I), ("dt_diffusion", D), ("dt_mechanics", D),
        ("bc", I), ("integrator", I), ("repulsion", D), ("adhesion", D),
        ("adhesion_multiplier", D), ("diffusion", P), ("decay", P), ("dirichlet", P),
        ("saturation", P), ("gradients", I), ("numerics", I),
    ]


_lib = None


def load():
    """Load and declare libcellgpu.so (no GPU needed just to load)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    L.cg_version.restype = ctypes.c_char_p
    L.cg_last_error.restype = ctypes.c_char_p
    L.cg_ctx_create.argtypes = [I, I, I, I, D, D, D, D, D, D, I, I, ctypes.POINTER(P)]
    L.cg_ctx_destroy.argtypes = [P]
    L.cg_ctx_destroy.restype = None
    L.cg_ctx_set_stream.argtypes = [P, P]
    L.cg_sync.argtypes = [P]
    L.cg_lod_step.argtypes = [P, P, P, P, D, I, P]
    L.cg_exchange.argtypes = [P, P, I, D, D, D, D, I, P, P, P, P, P]
    L.cg_exchange_cells.argtypes = [P, P, D, P, P, P, I, P, P, P, P, P]
    L.cg_rebin.argtypes = [P, I, P, P, P, P, P, P, P, P]
    L.cg_velocities.argtypes = [P, I, P, P, P, P, P, P, P, D, D, D, P]
    L.cg_integrate.argtypes = [P, I, P, P, P, D, I]
    L.cg_engine_create.argtypes = [P, ctypes.POINTER(StatePtrs), ctypes.POINTER(StepParams),
                                   ctypes.POINTER(P)]
    L.cg_engine_destroy.argtypes = [P]
    L.cg_engine_destroy.restype = None
    L.cg_engine_run.argtypes = [P, I, I]
    L.cg_engine_launches_per_step.argtypes = [P]
    L.cg_engine_time_stages.argtypes = [P, I, I, ctypes.c_char_p, P]
    L.cg_prof_enable.argtypes = [P, I]
    L.cg_prof_read.argtypes = [P, I, ctypes.c_char_p, P, P]
    L.cg_launch_count.argtypes = [P]
    L.cg_launch_count.restype = ctypes.c_longlong
    L.cg_ctx_set_slab.argtypes = [P, I, I, I, I]
    L.cg_engine_io_enable.argtypes = [P]
    L.cg_engine_io_inputs_ready.argtypes = [P, P]
    L.cg_engine_io_fields_ready.argtypes = [P, P]
    L.cg_engine_io_substrate_ready.argtypes = [P, I, P]
    L.cg_engine_io_wait_substrate.argtypes = [P, I, P]
    L.cg_engine_substrate_chains.argtypes = [P]
    L.cg_engine_step_io.argtypes = [P]
    L.cg_engine_sort_cells.argtypes = [P]
    L.cg_engine_set_cell_count.argtypes = [P, I]
    L.cg_check_state.argtypes = [P, P]
    L.cg_engine_step_host.argtypes = [P, P, P, P, P, P, P, I]
    L.cg_engine_host_join.argtypes = [P, P]
    U64, I64 = ctypes.c_uint64, ctypes.c_int64
    L.cg_division_draws.argtypes = [P, I, U64, I64, P, P]
    L.cg_divisions_count.argtypes = [P, I, U64, I64, P, P, ctypes.POINTER(I)]
    L.cg_divisions_place.argtypes = [P, I, I, U64, I64, P, P, P, P, P]
    L.cg_engine_io_join.argtypes = [P, P]
    L.cg_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
    L.cg_host_free.argtypes = [P]
    L.cg_host_free.restype = None
    L.cg_engine_io_wait_cells.argtypes = [P, P]
    L.cg_engine_io_wait_fields.argtypes = [P, P]
    L.cg_ctx_set_slab_bounds.argtypes = [P, I, I, I, ctypes.POINTER(I)]
    L.cg_gradients.argtypes = [P, P, P]
    L.cg_state_checksum.argtypes = [P, I, P, P, P, ctypes.POINTER(ctypes.c_uint64)]
    L.cg_rebin_exchange.argtypes = [P, I, P, P, P, P, P, P, P, P, D, P, P, P, P]
    L.cg_rebin_exchange_affine.argtypes = [P, I, P, P, P, P, P, P, P, P, D, P, P, P, P]
    L.cg_lod_step_fast.argtypes = [P, P, P, P, D, I, P, I]
    L.cg_velocities_fast.argtypes = [P, I, P, P, P, P, P, D, D, D, P]
    L.cg_fast_lod_available.argtypes = [P]
    L.cg_exchange_prepared.argtypes = [P, P, I, P, P]
    L.cg_zslab_pack.argtypes = [P, P, P]
    L.cg_zslab_correct.argtypes = [P, P, P, I, P]
    L.cg_ctx_set_substrate_window.argtypes = [P, I, I]
    L.cg_zslab_lr_gather.argtypes = [P, P, P]
    L.cg_zslab_defer.argtypes = [P, P]
    L.cg_zslab_block_lines.argtypes = [P]
    L.cg_zslab_block_lines.restype = ctypes.c_long
    L.cg_zslab_pack_blocks.argtypes = [P, P, P]
    L.cg_zslab_reduce_blocks.argtypes = [P, P, P]
    L.cg_zslab_correct_blocks.argtypes = [P, P, P, I, P]
    L.cg_voxel_z.argtypes = [P, I, P, P]
    L.cg_voxel_index.argtypes = [P, I, P, P]
    L.cg_cell_volumes.argtypes = [I, P, P]
    L.cg_cell_volumes.restype = None
    _lib = L
    return L


def raise_for(code: int, what: str = "") -> None:
    """Map a C-ABI status onto the reference's exception classes."""
    if code == CG_OK:
        return
    msg = (load().cg_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if code == CG_DOMAIN:
        raise DomainError(text)
    if code == CG_NUMERIC:
        raise NumericError(text)
    if code == CG_STATE:
        raise ContainerStateError(text)
    if code == CG_CAPACITY:
        raise CapacityError(text)
    raise DeviceError(text)


def require_cuda():
    """torch with a visible CUDA device, or DeviceError."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device is visible; the cellgpu path has no CPU fallback")
    load()
    return torch


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (or None)."""
    return None if t is None else t.data_ptr()


class Context:
    """Owns one cg_ctx (mesh + substrate count + per-cell scratch capacity)."""

    def __init__(self, mesh, n_substrates: int, capacity: int, device: int):
        L = load()
        self._L = L
        out = P()
        code = L.cg_ctx_create(device, mesh.nx, mesh.ny, mesh.nz, float(mesh.dx),
                               float(mesh.dy), float(mesh.dz), float(mesh.origin[0]),
                               float(mesh.origin[1]), float(mesh.origin[2]), n_substrates,
                               max(int(capacity), 1), ctypes.byref(out))
        raise_for(code, "cg_ctx_create")
        self.handle = out
        self.capacity = max(int(capacity), 1)
        self.n_substrates = n_substrates
        self.device = device

    def bind_stream(self, stream=None):
        import torch

        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._L.cg_ctx_set_stream(self.handle, P(s.cuda_stream))
        return s

    def sync(self, what=""):
        raise_for(self._L.cg_sync(self.handle), what)

    def prof_enable(self, on: bool):
        self._L.cg_prof_enable(self.handle, 1 if on else 0)

    def prof_read(self) -> dict:
        maxk = 32
        names = ctypes.create_string_buffer(32 * maxk)
        tot = (ctypes.c_double * maxk)()
        cnt = (ctypes.c_int * maxk)()
        k = self._L.cg_prof_read(self.handle, maxk, names, ctypes.cast(tot, P),
                                 ctypes.cast(cnt, P))
        if k < 0:
            raise_for(k, "cg_prof_read")
        out = {}
        for i in range(k):
            name = names.raw[32 * i:32 * (i + 1)].split(b"\0", 1)[0].decode()
            out[name] = (tot[i], cnt[i])
        return out

    def launch_count(self) -> int:
        return int(self._L.cg_launch_count(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            self._L.cg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_contexts: dict = {}


def context_for(mesh, n_substrates: int, n_cells: int, device: int | None = None) -> Context:
    """Shared context per (mesh, S, device); grows its cell capacity on demand."""
    torch = require_cuda()
    dev = torch.cuda.current_device() if device is None else device
    key = (mesh.nx, mesh.ny, mesh.nz, float(mesh.dx), float(mesh.dy), float(mesh.dz),
           tuple(float(o) for o in mesh.origin), int(n_substrates), dev)
    ctx = _contexts.get(key)
    if ctx is None or ctx.capacity < n_cells:
        if ctx is not None:
            ctx.close()
        cap = max(n_cells, 1024)
        if ctx is not None:
            cap = max(cap, 2 * ctx.capacity)
        ctx = Context(mesh, n_substrates, cap, dev)
        _contexts[key] = ctx
    ctx.bind_stream()
    return ctx


def cell_volumes(radius):
    """core.py:161-163 Cell.volume = (4/3)*pi*R**3 with libm pow, like CPython,
    evaluated in libcellgpu.so's host code (no GPU needed)."""
    import numpy as np

    r = np.ascontiguousarray(radius, dtype=np.float64)
    out = np.empty_like(r)
    load().cg_cell_volumes(len(r), r.ctypes.data_as(P), out.ctypes.data_as(P))
    return out
