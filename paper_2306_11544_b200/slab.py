"""z-slab domain decomposition: host-side planning and the reduced system of
the partitioned z sweep.

Rank r of P owns global planes [z0_r, z1_r).  The x and y sweeps, the cell
exchange and the velocity kernel are slab-local; the z sweep is a tridiagonal
solve along lines that cross every slab.  With the line matrix
A = tridiag(-r, b_i, -r) (b_i = 1 + lam3 + 2r inside, 1 + lam3 + r at the two
global ends, diffusion.py:80-99), rank r's block A_r satisfies

    A_r x_r = d_r + r x_{a-1} e_0 + r x_b e_{m-1}

so x_r = y_r + x_{a-1} v_r + x_b w_r with y_r = A_r^{-1} d_r (a local Thomas
solve) and the spikes v_r = r A_r^{-1} e_0, w_r = r A_r^{-1} e_{m-1}, which
depend only on the matrix and are precomputed here.  The interface values
z_r = (x_r[0], x_r[m-1]) satisfy a 2x2 block-tridiagonal system

    z_r - v_r(ends) * l_{r-1} - w_r(ends) * f_{r+1} = (y_r[0], y_r[m-1])

(f = first, l = last component) which every rank solves redundantly per line
after an all-gather of the (y_r[0], y_r[m-1]) pairs: 2 doubles per line per
rank -- or, for P >= 3, rank r solves it for its block of lines only after an
all-to-all and returns each rank its (l_{k-1}, f_{k+1}) with a second one
(distributed.SlabSimulation, cg_zslab_*_blocks; same operations).  Rounding differs from the single-GPU serial Thomas (the bar for
multi-GPU fields is 1e-10 relative, BASELINE.json); with P = 1 the correction
vanishes and the result is the single-GPU one bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def slab_bounds(nz: int, world: int) -> list[tuple[int, int]]:
    """Contiguous plane ranges, sizes differing by at most one (parallel.py:26-35 rule)."""
    if world < 1 or nz < world:
        raise ValueError(f"cannot split {nz} planes over {world} ranks")
    base, rem = divmod(nz, world)
    out, z = [], 0
    for r in range(world):
        z1 = z + base + (1 if r < rem else 0)
        out.append((z, z1))
        z = z1
    return out


def weighted_bounds(weights, world: int) -> list[tuple[int, int]]:
    """Contiguous plane ranges minimising the largest per-rank cost (SURVEY.md
    section 8f row 1: the paper's load-imbalance lesson; cost = alpha voxels +
    beta cells per plane, metrics.py:201-218).  Binary search on the bottleneck
    with a greedy feasibility check (the classic linear-partition bound), then
    parts are split until there is exactly one per rank (splitting never
    raises the bottleneck); every rank keeps at least one plane."""
    w = np.asarray(weights, dtype=np.float64)
    nz = w.shape[0]
    if world < 1 or nz < world:
        raise ValueError(f"cannot split {nz} planes over {world} ranks")
    if np.any(w < 0):
        raise ValueError("plane costs must be >= 0")

    def greedy(limit):
        cuts, cur = [0], 0.0
        for z in range(nz):
            if z > cuts[-1] and cur + w[z] > limit:
                cuts.append(z)
                cur = 0.0
            cur += w[z]
        return cuts + [nz]

    lo, hi = float(w.max(initial=0.0)), float(w.sum())
    for _ in range(200):
        if hi - lo <= 1e-12 * max(hi, 1.0):
            break
        mid = 0.5 * (lo + hi)
        if len(greedy(mid)) - 1 <= world:
            hi = mid
        else:
            lo = mid
    cuts = greedy(hi)
    while len(cuts) - 1 < world:  # split the widest part
        k = max(range(len(cuts) - 1), key=lambda i: cuts[i + 1] - cuts[i])
        cuts.insert(k + 1, cuts[k + 1] - 1)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def plane_costs(nz: int, plane_voxels: int, cell_z, alpha: float = 1.0,
                beta: float = 10.0) -> np.ndarray:
    """alpha * voxels + beta * cells per z plane (cell_z: voxel z of each cell)."""
    counts = np.bincount(np.asarray(cell_z, dtype=np.int64), minlength=nz)[:nz]
    return alpha * plane_voxels + beta * counts.astype(np.float64)


def block_factors(n: int, r: float, lam3: float, top_end: bool, bottom_end: bool):
    """Thomas factors (inv, gamma) of a block of the line matrix: the
    reference's _line_factors (diffusion.py:80-99) with the boundary diagonal
    only where the block touches a global end of the line."""
    interior = 1.0 + lam3 + 2.0 * r
    boundary = 1.0 + lam3 + r
    if n == 1 and top_end and bottom_end:
        return np.array([1.0 / (1.0 + lam3)]), np.zeros(1)
    diag = np.full(n, interior)
    if top_end:
        diag[0] = boundary
    if bottom_end:
        diag[-1] = boundary
    if n == 1 and (top_end ^ bottom_end):
        diag[0] = boundary
    inv = np.empty(n)
    gam = np.empty(n)
    inv[0] = 1.0 / diag[0]
    gam[0] = r * inv[0]
    for i in range(1, n):
        inv[i] = 1.0 / (diag[i] - r * gam[i - 1])
        gam[i] = r * inv[i]
    return inv, gam


def thomas(d: np.ndarray, inv: np.ndarray, gam: np.ndarray, r: float) -> np.ndarray:
    """diffusion.py:102-112 on the last axis (rows = lines), in the reference's op order."""
    d = np.array(d, dtype=np.float64, copy=True)
    n = d.shape[-1]
    d[..., 0] *= inv[0]
    for i in range(1, n):
        d[..., i] += r * d[..., i - 1]
        d[..., i] *= inv[i]
    for i in range(n - 2, -1, -1):
        d[..., i] += gam[i] * d[..., i + 1]
    return d


@dataclass
class SlabPlan:
    """Per-substrate z-sweep data of one decomposition (all ranks)."""

    bounds: list            # [(z0, z1)] per rank
    r: float                # dt * D / dz^2
    inv: list               # per rank: local Thomas factors
    gam: list
    v: list                 # per rank: spike r A_r^{-1} e_0 (length m_r)
    w: list                 # per rank: spike r A_r^{-1} e_{m-1}

    @property
    def world(self) -> int:
        return len(self.bounds)

    def ends(self) -> np.ndarray:
        """(P, 4): v[0], v[m-1], w[0], w[m-1] of every rank (the reduced system's coefficients)."""
        return np.array([[v[0], v[-1], w[0], w[-1]] for v, w in zip(self.v, self.w)])


def make_plan(nz: int, world: int, r: float, lam3: float, bounds=None) -> SlabPlan:
    bounds = slab_bounds(nz, world) if bounds is None else list(bounds)
    inv, gam, vs, ws = [], [], [], []
    for k, (z0, z1) in enumerate(bounds):
        m = z1 - z0
        top, bottom = z0 == 0, z1 == nz
        iv, g = block_factors(m, r, lam3, top, bottom)
        e0 = np.zeros(m)
        e0[0] = r
        e1 = np.zeros(m)
        e1[-1] = r
        vs.append(thomas(e0, iv, g, r) if k > 0 else np.zeros(m))
        ws.append(thomas(e1, iv, g, r) if k < world - 1 else np.zeros(m))
        inv.append(iv)
        gam.append(g)
    return SlabPlan(bounds, r, inv, gam, vs, ws)


def solve_interfaces(yends: np.ndarray, coef: np.ndarray) -> np.ndarray:
    """Reduced system for every line.

    yends: (P, 2, L) = (y_r[0], y_r[m-1]) per rank and line; coef: (P, 4) from
    SlabPlan.ends().  Returns (P, 2, L): the exact first/last values
    (f_r, l_r).  Block Thomas with 2x2 blocks, z_r + L_r z_{r-1} + U_r z_{r+1}
    = Y_r, L_r = -[v0; v1] [0 1], U_r = -[w0; w1] [1 0].  Restated by the
    device kernel k_zslab_correct (same operation order)."""
    P, _, L = yends.shape
    G = np.zeros((P, 2, L))   # first column of G_r (second column is zero)
    H = np.zeros((P, 2, L))
    for r in range(P):
        v0, v1, w0, w1 = coef[r]
        y0, y1 = yends[r, 0], yends[r, 1]
        if r == 0:
            # D = I; G = -w; H = y
            a00, a01, a10, a11 = 1.0, 0.0, 0.0, 1.0
            b0, b1 = y0, y1
        else:
            g1 = G[r - 1, 1]      # l-component of G_{r-1}'s first column
            h1 = H[r - 1, 1]
            # D_r = I - L_r G_{r-1} = I + [v0; v1] [g1 0]
            a00 = 1.0 + v0 * g1
            a01 = 0.0
            a10 = v1 * g1
            a11 = 1.0
            # rhs = Y_r - L_r H_{r-1} = y + [v0; v1] h1
            b0 = y0 + v0 * h1
            b1 = y1 + v1 * h1
        # D is lower triangular: solve D x = b and D g = -w
        det0 = a00
        H[r, 0] = b0 / det0
        H[r, 1] = (b1 - a10 * H[r, 0]) / a11
        G[r, 0] = (-w0) / det0
        G[r, 1] = ((-w1) - a10 * G[r, 0]) / a11
    Z = np.zeros((P, 2, L))
    Z[P - 1] = H[P - 1]
    for r in range(P - 2, -1, -1):
        f_next = Z[r + 1, 0]
        Z[r, 0] = H[r, 0] - G[r, 0] * f_next
        Z[r, 1] = H[r, 1] - G[r, 1] * f_next
    return Z


def correct(y: np.ndarray, k: int, Z: np.ndarray, plan: SlabPlan) -> np.ndarray:
    """x_k = y_k + l_{k-1} v_k + f_{k+1} w_k (y: (..., m_k) lines on the last axis)."""
    P = plan.world
    left = Z[k - 1, 1] if k > 0 else 0.0
    right = Z[k + 1, 0] if k < P - 1 else 0.0
    left = np.asarray(left)[..., None]
    right = np.asarray(right)[..., None]
    return y + left * plan.v[k] + right * plan.w[k]


def distributed_line_solve(d_global: np.ndarray, nz: int, world: int, r: float,
                           lam3: float, bounds=None) -> np.ndarray:
    """Reference restatement of the whole partitioned z solve on one host
    (lines on the last axis).  Used by the CPU tests; the GPU path does the
    same per rank with one all-gather.  ``bounds``: any contiguous split."""
    plan = make_plan(nz, world, r, lam3, bounds)
    ys = [thomas(d_global[..., z0:z1], plan.inv[k], plan.gam[k], r)
          for k, (z0, z1) in enumerate(plan.bounds)]
    yends = np.stack([np.stack([y[..., 0], y[..., -1]]) for y in ys])
    L = yends.shape[-1] if yends.ndim == 3 else 1
    Z = solve_interfaces(yends.reshape(world, 2, -1), plan.ends())
    out = [correct(y.reshape(-1, y.shape[-1]), k, Z, plan).reshape(y.shape)
           for k, y in enumerate(ys)]
    del L
    return np.concatenate(out, axis=-1)
