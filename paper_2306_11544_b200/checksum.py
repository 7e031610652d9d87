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


def state_checksum(container) -> str:
    cells = container.cells
    return checksum_arrays([c.id for c in cells], [c.position for c in cells],
                           [c.velocity for c in cells])
