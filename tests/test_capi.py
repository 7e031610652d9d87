"""The C-ABI library loads and exports every symbol include/cellgpu.h declares
(no GPU needed), and the product package never routes through the oracle."""

import math
import os
import re

import numpy as np

from paper_2306_11544_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(_lib.HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cg_[a-z_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.load()
    names = declared_symbols()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(_lib.EXPORTS)
    assert L.cg_version().startswith(b"cellgpu")


def test_library_is_built_for_sm_100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_cell_volumes_match_cpython_bitwise():
    rng = np.random.default_rng(0)
    r = np.concatenate([rng.uniform(5.0, 12.0, 20000), [8.0, 8.4127, 7.0, 10.0]])
    got = _lib.cell_volumes(r)
    want = np.array([(4.0 / 3.0) * math.pi * float(x) ** 3 for x in r])
    assert np.array_equal(got, want)


def test_error_codes_map_to_reference_exceptions():
    import pytest

    from paper_2306_11544_b200 import errors

    for code, cls in [(1, errors.DomainError), (2, errors.NumericError),
                      (3, errors.ContainerStateError), (4, errors.CapacityError),
                      (101, errors.DeviceError)]:
        with pytest.raises(cls):
            _lib.raise_for(code, "t")
    assert issubclass(errors.DomainError, ValueError)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2306_11544_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "liboracle" not in src and "cellref" not in src, f
