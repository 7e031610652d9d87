"""Partitioned z sweep (paper_2306_11544_b200/slab.py): the reduced 2x2
block-tridiagonal interface system reproduces the serial Thomas solve of the
reference (diffusion.py:80-112) to rounding, for every split."""

import numpy as np
import pytest

from paper_2306_11544_b200.slab import (block_factors, distributed_line_solve, make_plan,
                                        slab_bounds, thomas)


def serial(d, nz, r, lam3):
    inv, gam = block_factors(nz, r, lam3, True, True)
    return thomas(d, inv, gam, r)


def test_slab_bounds_partition():
    assert slab_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert slab_bounds(256, 8)[-1] == (224, 256)
    with pytest.raises(ValueError):
        slab_bounds(3, 4)


def test_block_factors_reduce_to_reference():
    from oracle import oracle as o

    for n, r, lam3 in [(1, 2.5, 1e-3), (2, 2.5, 1e-3), (80, 2.5, 3.3e-4), (7, 0.025, 0.1)]:
        inv, gam = block_factors(n, r, lam3, True, True)
        ri, rg = o.line_factors(n, r, lam3)
        assert np.array_equal(inv, ri)
        if n > 1:
            assert np.array_equal(gam, rg)


@pytest.mark.parametrize("nz,world", [(20, 1), (20, 2), (32, 4), (80, 3), (256, 8), (9, 8), (16, 16)])
@pytest.mark.parametrize("r", [2.5, 0.025, 1.6])
def test_partitioned_matches_serial(nz, world, r):
    rng = np.random.default_rng(nz * 100 + world)
    d = rng.uniform(0.0, 50.0, (64, nz))
    lam3 = 0.01 * 0.1 / 3.0
    want = serial(d, nz, r, lam3)
    got = distributed_line_solve(d, nz, world, r, lam3)
    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert err <= 1e-13, err
    if world == 1:
        assert np.array_equal(got, want)


def test_spikes_vanish_at_the_global_ends():
    plan = make_plan(32, 4, 2.5, 1e-3)
    assert np.all(plan.v[0] == 0.0) and np.all(plan.w[-1] == 0.0)
    assert np.all(plan.v[1] > 0.0) and np.all(plan.w[0] > 0.0)


@pytest.mark.parametrize("bounds", [[(0, 1), (1, 20)], [(0, 13), (13, 14), (14, 20)],
                                    [(0, 5), (5, 6), (6, 7), (7, 20)]])
@pytest.mark.parametrize("r", [2.5, 0.025])
def test_partitioned_uneven_slabs_match_serial(bounds, r):
    """Non-uniform slabs (load-balanced splits, 1-plane slabs included)."""
    nz, world = 20, len(bounds)
    rng = np.random.default_rng(world)
    d = rng.uniform(0.0, 50.0, (16, nz))
    lam3 = 0.01 * 0.1 / 3.0
    want = serial(d, nz, r, lam3)
    got = distributed_line_solve(d, nz, world, r, lam3, bounds)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) <= 1e-13


def test_weighted_bounds_balance_and_partition():
    from paper_2306_11544_b200.slab import plane_costs, weighted_bounds

    # a spheroid-like profile: cells concentrated in the middle planes
    z = np.concatenate([np.full(500, 40), np.full(300, 39), np.full(300, 41),
                        np.arange(80).repeat(2)])
    costs = plane_costs(80, 6400, z, alpha=1.0, beta=100.0)
    for world in (1, 2, 3, 4, 8):
        b = weighted_bounds(costs, world)
        assert b[0][0] == 0 and b[-1][1] == 80
        assert all(b[k][1] == b[k + 1][0] for k in range(world - 1))
        assert all(z1 > z0 for z0, z1 in b)
        loads = [costs[z0:z1].sum() for z0, z1 in b]
        even = [costs[z0:z1].sum() for z0, z1 in slab_bounds(80, world)]
        assert max(loads) <= max(even) + 1e-9
    # the middle ranks get narrower slabs than the balanced plane split
    b4 = weighted_bounds(costs, 4)
    assert (b4[1][1] - b4[1][0]) < 20 and (b4[2][1] - b4[2][0]) < 20
    with pytest.raises(ValueError):
        weighted_bounds(np.ones(3), 4)
    # every rank keeps a plane even with all cost in one plane
    spike = np.zeros(10)
    spike[0] = 1.0
    b = weighted_bounds(spike, 5)
    assert all(z1 - z0 >= 1 for z0, z1 in b) and b[-1][1] == 10
