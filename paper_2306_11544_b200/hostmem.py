"""Page-locked host buffers for the host-driven step (Simulation.step_host).

``host_empty(shape)`` returns a CPU torch tensor backed by ``cg_host_alloc``
(cudaHostAlloc in libcellgpu.so), freed when the last view of it goes away.
Copies from it move at the copy engines' full rate: 225 us per 12.3 MB
host-to-device against 350 us from ``Tensor.pin_memory()`` on the B200 boxes
(tools/pcie_probe.py).  torch sees it as pinned, so ``copy_(...,
non_blocking=True)`` stays asynchronous.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


class _HostBlock:
    """Owns one cg_host_alloc block; frees it on collection."""

    def __init__(self, nbytes: int):
        L = _lib.load()
        ptr = ctypes.c_void_p()
        _lib.raise_for(L.cg_host_alloc(max(int(nbytes), 1), ctypes.byref(ptr)), "cg_host_alloc")
        self.ptr = ptr.value
        self._free = L.cg_host_free

    def __del__(self):
        if getattr(self, "ptr", None):
            self._free(self.ptr)
            self.ptr = None


def host_empty(shape, dtype=np.float64):
    """Uninitialised page-locked CPU tensor of `shape` / numpy `dtype`."""
    import torch

    dtype = np.dtype(dtype)
    shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
    count = int(np.prod(shape)) if shape else 1
    block = _HostBlock(count * dtype.itemsize)
    buf = (ctypes.c_char * max(count * dtype.itemsize, 1)).from_address(block.ptr)
    buf.owner = block  # the numpy array's base keeps the block alive
    arr = np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)
    return torch.from_numpy(arr)


def host_like(t):
    """Page-locked copy of CPU tensor / array `t`."""
    import torch

    src = t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t))
    out = host_empty(tuple(src.shape), src.numpy().dtype)
    out.copy_(src)
    return out
