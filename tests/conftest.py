"""Shared fixtures.  Markers: ``gpu`` = needs a CUDA device (run on the B200
box with ``-m gpu``); everything else runs on the CPU-only build container."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.lib()
    return o


def mesh_from_arr(a):
    """(nx, ny, nz, dx, dy, dz, ox, oy, oz) fixture array -> our CartesianMesh."""
    from paper_2306_11544_b200 import CartesianMesh

    return CartesianMesh(int(a[0]), int(a[1]), int(a[2]), float(a[3]), float(a[4]), float(a[5]),
                         (float(a[6]), float(a[7]), float(a[8])))


def refmesh_from_arr(a):
    from oracle import oracle as o

    return o.mesh_struct(int(a[0]), int(a[1]), int(a[2]), float(a[3]), float(a[4]), float(a[5]),
                         (float(a[6]), float(a[7]), float(a[8])))


def cases(golden, prefix):
    ks = sorted({k.split("_")[0] for k in golden if k.startswith(prefix) and k.split("_")[0][len(prefix):].isdigit()})
    return ks
