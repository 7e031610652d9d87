"""The z-slab decomposition's communication and math on CPU with gloo
(world_size 2 and 3): neighbour row exchange with variable counts, the
all-gather, and the partitioned z sweep vs the serial Thomas solve."""

import numpy as np
import pytest

import _dist_util


def _comm_case(rank, world, split=False):
    import torch
    import torch.distributed as dist

    from paper_2306_11544_b200.distributed import Comm

    comm = Comm(dist, "cpu")
    if split:  # the mechanics' own communicator (SlabSimulation's overlapped step)
        comm.all_gather(torch.empty((world, 1), dtype=torch.float64),
                        torch.zeros(1, dtype=torch.float64))
        comm = comm.split()
        assert comm.group is not None and comm.world == world and comm.rank == rank
    lo = torch.full((rank + 1, 4), float(rank), dtype=torch.float64)      # rows to rank-1
    hi = torch.full((2 * rank + 3, 4), 10.0 + rank, dtype=torch.float64)  # rows to rank+1
    got_lo, got_hi = comm.exchange_rows(lo, hi, 4)
    ends = torch.full((2, 3), float(rank), dtype=torch.float64)
    out = torch.empty((world, 2, 3), dtype=torch.float64)
    comm.all_gather(out, ends)
    # block k of rank r's input goes to rank k: out[q] = 100 q + 10 rank + k...
    blocks = torch.stack([torch.full((2, 3), 100.0 * rank + k, dtype=torch.float64)
                          for k in range(world)])
    a2a = torch.empty_like(blocks)
    comm.all_to_all(a2a, blocks)
    return (got_lo.numpy(), got_hi.numpy(), out.numpy(), comm.max(float(rank)), comm.sum(rank),
            a2a.numpy())


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_neighbour_exchange_and_all_gather(tmp_path, world, split):
    res = _dist_util.run(world, _comm_case, (split,), tmp_path)
    for r, (got_lo, got_hi, out, mx, sm, a2a) in enumerate(res):
        # all-to-all: block q came from rank q, which sent its block r
        assert np.array_equal(a2a[:, 0, 0], 100.0 * np.arange(world) + r)
        if r > 0:  # from rank r-1: its "hi" rows
            assert got_lo.shape == (2 * (r - 1) + 3, 4) and np.all(got_lo == 10.0 + r - 1)
        else:
            assert got_lo.shape == (0, 4)
        if r < world - 1:  # from rank r+1: its "lo" rows
            assert got_hi.shape == (r + 2, 4) and np.all(got_hi == r + 1)
        else:
            assert got_hi.shape == (0, 4)
        assert np.array_equal(out[:, 0, 0], np.arange(world, dtype=float))
        assert mx == world - 1 and sm == world * (world - 1) // 2


def _zsolve_case(rank, world, nz, r, lam3):
    import torch
    import torch.distributed as dist

    from paper_2306_11544_b200.distributed import Comm
    from paper_2306_11544_b200.slab import correct, make_plan, solve_interfaces, thomas

    comm = Comm(dist, "cpu")
    rng = np.random.default_rng(5)
    d = rng.uniform(0.0, 50.0, (40, nz))           # every rank builds the same global lines
    plan = make_plan(nz, world, r, lam3)
    z0, z1 = plan.bounds[rank]
    y = thomas(d[:, z0:z1], plan.inv[rank], plan.gam[rank], r)      # local block solve
    ends = torch.from_numpy(np.stack([y[:, 0], y[:, -1]]))          # (2, L)
    allends = torch.empty((world, 2, 40), dtype=torch.float64)
    comm.all_gather(allends, ends)                                  # the only collective
    Z = solve_interfaces(allends.numpy(), plan.ends())
    return z0, z1, correct(y, rank, Z, plan), d


@pytest.mark.parametrize("world,nz", [(2, 20), (3, 32)])
def test_partitioned_z_sweep_over_gloo(tmp_path, world, nz):
    from paper_2306_11544_b200.slab import block_factors, thomas

    r, lam3 = 2.5, 1e-3 / 3
    res = _dist_util.run(world, _zsolve_case, (nz, r, lam3), tmp_path)
    d = res[0][3]
    inv, gam = block_factors(nz, r, lam3, True, True)
    want = thomas(d, inv, gam, r)
    got = np.concatenate([x for _, _, x, _ in res], axis=1)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


def test_migration_plan_orders_leavers_to_the_ends():
    import torch

    from paper_2306_11544_b200.distributed import migration_plan

    z = torch.tensor([5, 3, 9, 4, 10, 2, 6, 9], dtype=torch.int32)  # slab [4, 10)
    order, n_lo, n_hi, n_far = migration_plan(z, 4, 10)
    assert (n_lo, n_hi, n_far) == (2, 1, 1)  # 3, 2 go down (2 is far), 10 up
    o = order.tolist()
    assert o[:2] == [1, 5] and o[-1:] == [4] and o[2:-1] == [0, 2, 3, 6, 7]
    order, n_lo, n_hi, n_far = migration_plan(torch.tensor([4, 5], dtype=torch.int32), 4, 10)
    assert order is None and (n_lo, n_hi, n_far) == (0, 0, 0)


def _migration_case(rank, world):
    """Every rank owns cells with global plane z; after one migration round
    (plan + Comm.exchange_rows + compaction as SlabSimulation._migrate) each
    cell lives on the rank whose slab holds its plane, exactly once."""
    import torch
    import torch.distributed as dist

    from paper_2306_11544_b200.distributed import Comm, migration_plan

    comm = Comm(dist, "cpu")
    z0, z1 = 10 * rank, 10 * rank + 10
    g = torch.Generator().manual_seed(rank)
    n = 50
    z = torch.randint(max(z0 - 1, 0), min(z1 + 1, 10 * world), (n,), generator=g, dtype=torch.int32)
    ids = torch.arange(n, dtype=torch.float64) + 1000 * rank
    rows = torch.stack([ids, z.double()], dim=1)
    order, n_lo, n_hi, _ = migration_plan(z, z0, z1)
    if order is None:
        order = torch.arange(n)
    in_lo, in_hi = comm.exchange_rows(rows[order[:n_lo]], rows[order[n - n_hi:]], 2)
    kept = rows[order[n_lo:n - n_hi]]
    mine = torch.cat([kept, in_lo, in_hi])
    return z0, z1, mine.numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_migration_round_conserves_cells(tmp_path, world):
    res = _dist_util.run(world, _migration_case, (), tmp_path)
    all_ids = np.concatenate([r[2][:, 0] for r in res])
    assert len(all_ids) == 50 * world and len(np.unique(all_ids)) == 50 * world
    for z0, z1, mine in res:
        assert np.all((mine[:, 1] >= z0) & (mine[:, 1] < z1))
