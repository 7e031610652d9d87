"""Dispatch records of the reference's worker pool (parallel.py:26-67).

On the GPU there is no fork-join pool: every hot-path call is one or a few
kernel launches on a CUDA stream.  The reference's signatures still take a
``pool`` and return ``RegionRecord``s, so this module keeps those types:
``WorkerPool`` is accepted (any object with ``.workers`` works, including the
reference's own pool) and ignored for results, and each call returns one
record whose single worker slot carries the GPU wall time.
"""

from __future__ import annotations

from dataclasses import dataclass, field


def static_ranges(n_items: int, workers: int) -> list[tuple[int, int]]:
    """Contiguous [lo, hi) per worker; sizes differ by at most one (parallel.py:26-35)."""
    base, rem = divmod(n_items, workers)
    ranges, lo = [], 0
    for w in range(workers):
        hi = lo + base + (1 if w < rem else 0)
        ranges.append((lo, hi))
        lo = hi
    return ranges


@dataclass
class WorkerStats:
    busy: float = 0.0
    iterations: int = 0
    claims: int = 0
    alloc_events: int = 0
    dealloc_events: int = 0


@dataclass
class RegionRecord:
    """One dispatch: iteration space, schedulable chunks, per-worker stats."""

    items: int
    schedulable_chunks: int
    elapsed: float
    workers: list = field(default_factory=list)
    claim_log: list | None = None

    @property
    def total_alloc_events(self) -> int:
        return sum(w.alloc_events for w in self.workers)

    @property
    def total_iterations(self) -> int:
        return sum(w.iterations for w in self.workers)

    @property
    def total_claims(self) -> int:
        return sum(w.claims for w in self.workers)


def gpu_record(items: int, chunks: int, elapsed: float, claims: int | None = None) -> RegionRecord:
    """A record for one GPU dispatch: the device is the single 'worker'."""
    stats = WorkerStats(busy=elapsed, iterations=items,
                        claims=items if claims is None else claims)
    return RegionRecord(items=items, schedulable_chunks=chunks, elapsed=elapsed, workers=[stats])


class WorkerPool:
    """Stand-in for the reference's fork-join pool (parallel.py:89-216).

    Accepted by every hot-path call for signature compatibility; the GPU does
    the work, so no threads are spawned and results never depend on it.
    """

    def __init__(self, workers: int = 1):
        if workers < 1:
            raise ValueError("worker count must be >= 1")
        self.workers = workers

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.shutdown()
        return False

    def shutdown(self) -> None:
        pass
