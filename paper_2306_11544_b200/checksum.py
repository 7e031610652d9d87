"""Order-independent state digest (simulate.py:79-90 state_checksum).

XOR of blake2b-128 over ``<q6d`` (id, position, velocity) per cell -- the
reference's parity tool, usable on a container or on raw arrays."""

from __future__ import annotations

import hashlib
import struct


def checksum_arrays(ids, positions, velocities) -> str:
    acc = 0
    for cid, p, v in zip(ids, positions, velocities):
        blob = struct.pack("<q6d", int(cid), float(p[0]), float(p[1]), float(p[2]),
                           float(v[0]), float(v[1]), float(v[2]))
        acc ^= int.from_bytes(hashlib.blake2b(blob, digest_size=16).digest(), "little")
    return f"{acc:032x}"


def device_checksum(ctx, n: int, ids, positions, velocities) -> str:
    """The same digest computed on the GPU (cg_state_checksum) from device
    tensors: ids (n,) int64, positions / velocities (n, 3) float64."""
    import ctypes

    from . import _lib

    out = (ctypes.c_uint64 * 2)()
    _lib.raise_for(_lib.load().cg_state_checksum(ctx.handle, int(n), _lib.ptr(ids),
                                                 _lib.ptr(positions), _lib.ptr(velocities), out),
                   "state_checksum")
    return f"{(int(out[1]) << 64) | int(out[0]):032x}"


def state_checksum(container) -> str:
    """Host digest of a container's cells (the reference's own computation);
    containers still on the device (from_arrays) are digested there."""
    if container._cells is None and container._dev is not None:
        from . import _lib

        d = container._dev
        ctx = _lib.context_for(container.mesh, 0, max(d.n, 1))
        return device_checksum(ctx, d.n, d.ids, d.pos, d.vel)
    cells = container.cells
    return checksum_arrays([c.id for c in cells], [c.position for c in cells],
                           [c.velocity for c in cells])
