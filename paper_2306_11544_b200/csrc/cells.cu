// Cell container rebuild, neighbour velocities and position integration.
//
// Reference: /root/reference/pkg/src/cellbench
//   core.py:77-85   voxel_of          -> py_floordiv / voxel_of_dev (CPython-exact)
//   core.py:218-240   rebin_cells       -> launch_rebin (counting sort)
//   mechanics.py:118-133 _voxel_candidates + :145-172 _cell_velocity
//                                       -> k_velocity_fast/_mid/_big (warp per non-empty voxel)
//   mechanics.py:228-245 integrate_positions -> k_integrate
//
// Rebin is a counting sort: voxel keys + histogram (atomics), one packed
// 64-bit scan that yields both the CSR offsets and the compacted non-empty
// list, an atomic scatter, and a per-bin fix-up that restores storage order
// (the reference's agent lists) and builds the id-sorted order used by the
// exchange and the velocity kernels.  The velocity kernel gives each non-
// empty voxel one warp: the 27-bin candidate union (9 contiguous slot ranges
// in bin order) is staged in shared memory and rank-sorted by id; then lanes
// compute pair terms for 32 candidates at a time and one lane per (resident,
// component) adds them in ascending id order, which reproduces the
// reference's accumulation order exactly.
#include <algorithm>
#include <climits>
#include <cstring>
#include <cstdlib>

#include "common.cuh"
#include "lod_common.cuh"

#define EPS_SKIP 1e-8

// CPython Objects/floatobject.c _float_div_mod (floor-division part).
__device__ __forceinline__ double py_floordiv(double vx, double wx) {
    double mod = fmod(vx, wx);
    double div = (vx - mod) / wx;
    if (mod != 0.0) {
        if ((wx < 0) != (mod < 0)) {
            mod += wx;
            div -= 1.0;
        }
    }
    double fl;
    if (div != 0.0) {
        fl = floor(div);
        if (div - fl > 0.5) fl += 1.0;
    } else {
        fl = copysign(0.0, vx / wx);
    }
    return fl;
}

__device__ __forceinline__ int voxel_of_dev(const MeshDev& m, double px, double py, double pz) {
    const double fx = py_floordiv(px - m.ox, m.dx);
    const double fy = py_floordiv(py - m.oy, m.dy);
    const double fz = py_floordiv(pz - m.oz, m.dz);
    if (!(fx >= 0.0 && fx < (double)m.nx && fy >= 0.0 && fy < (double)m.ny && fz >= 0.0 &&
          fz < (double)m.nz))
        return -1;
    return (int)fx + m.nx * ((int)fy + m.ny * (int)fz);
}

// ---------------------------------------------------------------- rebin

// Single-pass scan state: per tile one aggregate word and one inclusive-prefix
// word (bit 63 = published, the rest the packed value, so a reader needs one
// load and no fence), plus the tile ticket.
struct ScanState {
    unsigned long long* agg;
    unsigned long long* incl;
    int* ticket;
    int nb;
};
constexpr unsigned long long SCAN_READY = 1ull << 63;

static ScanState scan_state(cg_ctx* c) {
    const int nb = (int)((c->nvox + SCAN_TILE - 1) / SCAN_TILE);
    return ScanState{c->d_part, c->d_scan_incl, c->d_scan_flag + nb, nb};
}

// Zero the scan state for the next scan (the scan kernel runs after this one
// in stream order).
__device__ __forceinline__ void reset_scan_state(const ScanState& st) {
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < st.nb; i += blockDim.x) {
            st.agg[i] = 0;
            st.incl[i] = 0;
        }
        if (threadIdx.x == 0) *st.ticket = 0;
    }
}

__global__ void k_voxel_count(int n, const double* __restrict__ pos, MeshDev m,
                              int32_t* __restrict__ voxel, int* __restrict__ counts,
                              int* __restrict__ flags, ScanState scan) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    reset_scan_state(scan);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int v = voxel_of_dev(m, pos[3L * i], pos[3L * i + 1], pos[3L * i + 2]);
    voxel[i] = v;
    if (v < 0) {
        atomicOr(&flags[FLAG_DOMAIN], 1);
        return;
    }
    atomicAdd(&counts[v], 1);
    pdl_trigger();  // dependents launch as this grid finishes
}

// Packed scan element: high 32 bits = non-empty flag count, low = cell count.

__device__ __forceinline__ unsigned long long pack_count(int c) {
    return ((unsigned long long)(c > 0) << 32) | (unsigned)c;
}

// Block-wide exclusive scan of one u64 per thread; returns the block total.
__device__ __forceinline__ unsigned long long block_exscan(unsigned long long x,
                                                           unsigned long long* ws,
                                                           unsigned long long* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        unsigned long long w = lane < nw ? ws[lane] : 0ull;
        unsigned long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < nw) ws[lane] = wi - w;
        if (lane == nw - 1) ws[32] = wi;
    }
    __syncthreads();
    const unsigned long long r = ws[wid] + inc - x;
    *total = ws[32];
    __syncthreads();
    return r;
}

// Single-pass scan (decoupled look-back): tiles are taken in launch order
// from a ticket, so every predecessor is resident or done and publishes its
// aggregate without waiting.  Warp 0 then reads 32 predecessors per round,
// one status word each, and stops at the nearest published inclusive prefix.
// One launch produces the CSR offsets, the compacted non-empty list, row_ne
// and ne_start.  Each thread owns SCAN_ITEMS consecutive voxels (two 16-byte
// loads and stores).
__global__ void __launch_bounds__(SCAN_T) k_scan_lookback(
    const int* __restrict__ counts, long nvox, int nx, ScanState scan,
    int32_t* __restrict__ bin_start, int32_t* __restrict__ nonempty,
    int32_t* __restrict__ n_nonempty, int32_t* __restrict__ row_ne, int32_t* __restrict__ ne_start) {
    static_assert(SCAN_ITEMS == 8, "two int4 per thread");
    pdl_wait();
    __shared__ unsigned long long ws[33];
    __shared__ int s_tile;
    __shared__ unsigned long long s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(scan.ticket, 1);
    __syncthreads();
    const int tile = s_tile;
    const long base = (long)tile * SCAN_TILE + (long)threadIdx.x * SCAN_ITEMS;
    const bool full = base + SCAN_ITEMS <= nvox;
    int c[SCAN_ITEMS];
    if (full) {
        const int4 a = *reinterpret_cast<const int4*>(counts + base);
        const int4 b = *reinterpret_cast<const int4*>(counts + base + 4);
        c[0] = a.x, c[1] = a.y, c[2] = a.z, c[3] = a.w;
        c[4] = b.x, c[5] = b.y, c[6] = b.z, c[7] = b.w;
    } else {
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; j++) c[j] = base + j < nvox ? counts[base + j] : 0;
    }
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) sum += pack_count(c[j]);
    unsigned long long total;
    const unsigned long long local = block_exscan(sum, ws, &total);
    volatile unsigned long long* vagg = scan.agg;
    volatile unsigned long long* vincl = scan.incl;
    if (threadIdx.x == 0) {
        if (tile == 0) {
            vincl[0] = total | SCAN_READY;
            s_excl = 0;
        } else {
            vagg[tile] = total | SCAN_READY;
        }
    }
    if (tile > 0 && threadIdx.x < 32) {
        const int lane = threadIdx.x;
        unsigned long long acc = 0;
        for (int end = tile;; end -= 32) {
            const int j = end - 1 - lane;
            unsigned long long w = 0;
            bool inc = j < 0;
            if (j >= 0) {
                for (;;) {
                    w = vincl[j];
                    if (w & SCAN_READY) {
                        inc = true;
                        break;
                    }
                    w = vagg[j];
                    if (w & SCAN_READY) break;
                }
            }
            const unsigned stops = __ballot_sync(0xffffffffu, inc);
            const int stop = stops ? __ffs(stops) - 1 : 32;
            unsigned long long v = (lane <= stop && j >= 0) ? (w & ~SCAN_READY) : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc += v;
            if (stops) break;
        }
        if (lane == 0) {
            vincl[tile] = (acc + total) | SCAN_READY;
            s_excl = acc;
        }
    }
    __syncthreads();
    unsigned long long run = s_excl + local;
    int32_t out[SCAN_ITEMS];
    int r = (int)(base % nx);  // x of the first voxel: one division per thread
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; j++) {
        const long v = base + j;
        out[j] = (int32_t)(run & 0xffffffffull);
        if (v < nvox) {
            if (c[j] > 0) {
                nonempty[run >> 32] = (int32_t)v;
                ne_start[run >> 32] = out[j];
            }
            if (r == 0) row_ne[v / nx] = (int32_t)(run >> 32);
        }
        r = r + 1 == nx ? 0 : r + 1;
        run += pack_count(c[j]);
    }
    if (full && (reinterpret_cast<uintptr_t>(bin_start) & 15) == 0) {
        *reinterpret_cast<int4*>(bin_start + base) = make_int4(out[0], out[1], out[2], out[3]);
        *reinterpret_cast<int4*>(bin_start + base + 4) = make_int4(out[4], out[5], out[6], out[7]);
    } else {
#pragma unroll
        for (int j = 0; j < SCAN_ITEMS; j++)
            if (base + j < nvox) bin_start[base + j] = out[j];
    }
    if (tile == scan.nb - 1 && threadIdx.x == blockDim.x - 1) {
        const unsigned long long g = run;  // inclusive total after this thread's items
        bin_start[nvox] = (int32_t)(g & 0xffffffffull);
        *n_nonempty = (int32_t)(g >> 32);
        row_ne[nvox / nx] = (int32_t)(g >> 32);
        ne_start[g >> 32] = (int32_t)(g & 0xffffffffull);
    }
    pdl_trigger();  // dependents launch as this grid finishes
}

// Slots are filled from the top of each bin down; counts return to zero.
__global__ void k_scatter(int n, const int32_t* __restrict__ voxel,
                          const int32_t* __restrict__ bin_start, int* __restrict__ counts,
                          int32_t* __restrict__ bin_cells, int* __restrict__ n_big) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) *n_big = 0;  // the bin fix-up's queue of large bins
    if (i >= n) return;
    const int v = voxel[i];
    if (v < 0) return;
    const int slot = bin_start[v] + atomicSub(&counts[v], 1) - 1;
    bin_cells[slot] = i;
    pdl_trigger();  // dependents launch as this grid finishes
}

// Per non-empty voxel: storage order within the bin (core.py:226-235 appends
// in storage order) and the ascending-id copy (diffusion.py:223,
// mechanics.py:132).
struct CoefArgs {  // G4 exchange coefficients (k_exchange_coef), fused into the bin fix-up
    int S;
    double dt, inv_vol;
    const double* secretion;  // (S, n) by storage index
    const double* uptake;
    const double* sat;        // (S)
    const double* volume;     // (n)
    double* A;                // (S, n) by id-sorted slot
    double* D;
    double* R;                // (S, rq, 2 kRecCells) per non-empty voxel: {A, D} of its first cells
    int rq;
    int32_t* xv;              // optional (engine exchange set): non-empty list copy,
    int32_t* xs;              //   slot offsets (+1 sentinel)
    int32_t* xn;              //   and count
    // optional (fast numerics, S <= kLineMaxS): each voxel's exchange as one
    // affine map per substrate, {alpha, beta} = the composition of its cells'
    // rho -> (rho + A) / D in ascending id, and the first list index of every
    // x row (ny * nz + 1): units of `plane` (= nx) voxels, `nz` (= ny * nz) of them
    double* aff;              // (S, rq, 2)
    int32_t* pz;
    int plane, nz;
    // optional (fast numerics): (x, y, z, R) and the voxel of every slot for
    // the next step's velocities (positions do not change until then)
    const double* pos;
    const double* radius;
    double4* sp;
    int* svox;
    float4* spf;
};

// Compare-exchange of a register sorting network on (primary key, payload).
template <typename K, typename V>
__device__ __forceinline__ void cswap(K& ka, V& va, K& kb, V& vb) {
    if (kb < ka) {
        const K tk = ka;
        ka = kb;
        kb = tk;
        const V tv = va;
        va = vb;
        vb = tv;
    }
}

// Odd-even transposition network on BF_K entries (unused entries carry the
// largest key and stay at the end).
constexpr int BF_K = 8;
template <typename K, typename V>
__device__ __forceinline__ void sort_net(K (&k)[BF_K], V (&v)[BF_K]) {
#pragma unroll
    for (int r = 0; r < BF_K; r++)
#pragma unroll
        for (int i = r & 1; i + 1 < BF_K; i += 2) cswap(k[i], v[i], k[i + 1], v[i + 1]);
}

// Exchange coefficients of substrate s for the cells of one bin (slots
// [b0, b0 + nc), id order): diffusion.py:224-228's subexpressions per
// (slot, substrate), as k_exchange_coef, or the affine map folded in the
// bin's id order.
template <bool COEF>
__device__ __forceinline__ void bin_coef_s(const CoefArgs& ca, int n, int q, int v, int b0, int nc,
                                           const int32_t* __restrict__ by_id, int s,
                                           int* __restrict__ flags) {
    double alpha = 1.0, beta = 0.0;
#pragma unroll 1
    for (int u = 0; u < nc; u++) {
        const int k = b0 + u, cidx = by_id[k];
        const double f = ca.dt * ca.volume[cidx] * ca.inv_vol;
        const double sec = ca.secretion[(long)s * n + cidx];
        const double upt = ca.uptake[(long)s * n + cidx];
        const double den = 1.0 + f * (sec + upt);
        if (den <= 0.0) atomicOr(&flags[FLAG_DOMAIN], 1);
        const double a = f * sec * ca.sat[s];
        if (!ca.aff) {
            ca.A[(long)s * n + k] = a;
            ca.D[(long)s * n + k] = den;
            if (u < kRecCells) {
                double* r = ca.R + ((long)s * ca.rq + q) * (2 * kRecCells) + 2 * u;
                r[0] = a;
                r[1] = den;
            }
        } else {
            beta = (beta + a) / den;
            alpha = alpha / den;
        }
        if (s == 0 && ca.sp) {
            const double4 p = make_double4(ca.pos[3L * cidx], ca.pos[3L * cidx + 1],
                                           ca.pos[3L * cidx + 2], ca.radius[cidx]);
            ca.sp[k] = p;
            ca.spf[k] = make_float4((float)p.x, (float)p.y, (float)p.z, (float)p.w);
            ca.svox[k] = v;
        }
    }
    if (ca.aff && s < kLineMaxS)
        reinterpret_cast<double2*>(ca.aff)[(long)s * ca.rq + q] = make_double2(alpha, beta);
}

// The bin fix-up with the exchange coefficients, G lanes per non-empty voxel
// (adjacent lanes of one warp): lane 0 sorts the bin (registers for bins of
// up to BF_K cells, global memory beyond) and writes the storage- and
// id-ordered slots; lane g then computes the exchange coefficients / affine
// maps of substrates g, g + G, ... (each substrate's fold over the bin in id
// order, bin_coef_s).  Substrate-outer loops: config 1 0.159 vs 0.164 ms per
// step against one thread per voxel looping cells outer, substrates inner.
template <bool COEF, int G>
__global__ void k_bin_fix_g(const int32_t* __restrict__ nonempty,
                            const int32_t* __restrict__ n_nonempty,
                            const int32_t* __restrict__ bin_start, const long long* __restrict__ ids,
                            int32_t* __restrict__ bin_cells, int32_t* __restrict__ by_id, int n,
                            int maxq, CoefArgs ca, int* __restrict__ flags, int* __restrict__ big,
                            int* __restrict__ n_big) {
    pdl_wait();
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int q = (int)(t / G), g = (int)(t % G);
    const int nne = *n_nonempty;
    if (q == 0 && g == 0) {
        if (COEF && ca.xv) *ca.xn = nne;
        if (COEF && ca.aff && nne == 0)
            for (int z = 0; z <= ca.nz; z++) ca.pz[z] = 0;
    }
    const bool live = q < maxq && q < nne;
    int v = 0, b0 = 0, b1 = 0;
    if (live) {
        v = nonempty[q];
        b0 = bin_start[v];
        b1 = bin_start[v + 1];
    }
    const int nc = b1 - b0;
    if (live && g == 0) {
        if (COEF && ca.aff) {
            const int z = v / ca.plane;
            const int zp = q > 0 ? nonempty[q - 1] / ca.plane : -1;
            for (int zz = zp + 1; zz <= z; zz++) ca.pz[zz] = q;
            if (q == nne - 1)
                for (int zz = z + 1; zz <= ca.nz; zz++) ca.pz[zz] = nne;
        }
        if (COEF && ca.xv) {
            ca.xv[q] = v;
            ca.xs[q] = b0;
            if (q == nne - 1) ca.xs[nne] = b1;
        }
    }
    if (live && nc <= 2) {
        // most bins (one or two cells) need no network
        if (g == 0) {
            const int a = bin_cells[b0];
            if (nc == 1) {
                by_id[b0] = a;
            } else {
                const int b = bin_cells[b0 + 1];
                const long long ka = ids[a], kb = ids[b];
                bin_cells[b0] = min(a, b);
                bin_cells[b0 + 1] = max(a, b);
                by_id[b0] = kb < ka ? b : a;
                by_id[b0 + 1] = kb < ka ? a : b;
            }
        }
    } else if (live && nc <= BF_K) {
        if (g == 0) {
            int st[BF_K], sv[BF_K];
            long long key[BF_K];
#pragma unroll
            for (int u = 0; u < BF_K; u++) st[u] = u < nc ? bin_cells[b0 + u] : 0x7fffffff;
#pragma unroll
            for (int u = 0; u < BF_K; u++) key[u] = u < nc ? ids[st[u]] : 0x7fffffffffffffffll;
            // storage order within the bin (core.py:226-235 appends in storage order)
#pragma unroll
            for (int u = 0; u < BF_K; u++) sv[u] = st[u];
            int dummy[BF_K];
#pragma unroll
            for (int u = 0; u < BF_K; u++) dummy[u] = 0;
            sort_net(sv, dummy);
#pragma unroll
            for (int u = 0; u < BF_K; u++)
                if (u < nc) bin_cells[b0 + u] = sv[u];
            // ascending id (diffusion.py:223, mechanics.py:132)
            sort_net(key, st);
#pragma unroll
            for (int u = 0; u < BF_K; u++)
                if (u < nc) by_id[b0 + u] = st[u];
        }
    } else if (live && g == 0 && big) {
        big[atomicAdd(n_big, 1)] = q;  // k_bin_fix_big: a warp per large bin
    } else if (live && g == 0) {
        for (int i = b0 + 1; i < b1; i++) {
            const int c0 = bin_cells[i];
            int j = i - 1;
            while (j >= b0 && bin_cells[j] > c0) {
                bin_cells[j + 1] = bin_cells[j];
                j--;
            }
            bin_cells[j + 1] = c0;
        }
        for (int i = b0; i < b1; i++) {
            const int c0 = bin_cells[i];
            const long long key = ids[c0];
            int j = i - 1;
            while (j >= b0 && ids[by_id[j]] > key) {
                by_id[j + 1] = by_id[j];
                j--;
            }
            by_id[j + 1] = c0;
        }
    }
    if (COEF) {
        if (G > 1) __syncwarp();  // lane 0's id order is visible to the group
        if (live && !(big && nc > BF_K))
            for (int s = g; s < ca.S; s += G) bin_coef_s<COEF>(ca, n, q, v, b0, nc, by_id, s, flags);
    }
    pdl_trigger();
}

// Bins of more than BF_K cells (queued by k_bin_fix_g), a warp each: the
// bin's cells and ids staged in shared memory, both orders by rank (ids are
// unique, cell indices too), then lane s folds substrate s's coefficients
// in id order.  Bins beyond BIG_BIN cells: lane 0's insertion sorts.
constexpr int BIG_W = 4, BIG_BIN = 256, BIG_FOLD = 64;
template <bool COEF>
__global__ void __launch_bounds__(BIG_W * 32) k_bin_fix_big(
    const int32_t* __restrict__ nonempty, const int32_t* __restrict__ bin_start,
    const long long* __restrict__ ids, int32_t* __restrict__ bin_cells, int32_t* __restrict__ by_id,
    int n, CoefArgs ca, int* __restrict__ flags, const int* __restrict__ big,
    const int* __restrict__ n_big) {
    pdl_wait();
    __shared__ int s_cell[BIG_W][BIG_BIN];
    __shared__ long long s_key[BIG_W][BIG_BIN];
    // affine folds of bins up to BIG_FOLD cells: every (cell, substrate)'s
    // (a, den) computed by the lanes in parallel, then lane s folds them
    __shared__ int s_ord[BIG_W][BIG_FOLD];
    __shared__ double s_a[BIG_W][kLineMaxS][BIG_FOLD], s_d[BIG_W][kLineMaxS][BIG_FOLD];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nb = *n_big;
    for (int w = blockIdx.x * BIG_W + wid; w < nb; w += gridDim.x * BIG_W) {
        const int q = big[w], v = nonempty[q];
        const int b0 = bin_start[v], nc = bin_start[v + 1] - b0;
        if (nc <= BIG_BIN) {
            int* cell = s_cell[wid];
            long long* key = s_key[wid];
            for (int e = lane; e < nc; e += 32) {
                const int c0 = bin_cells[b0 + e];
                cell[e] = c0;
                key[e] = ids[c0];
            }
            __syncwarp();
            for (int e = lane; e < nc; e += 32) {
                const int ce = cell[e];
                const long long ke = key[e];
                int rc = 0, rk = 0;
                for (int f = 0; f < nc; f++) {
                    rc += cell[f] < ce;
                    rk += key[f] < ke;
                }
                bin_cells[b0 + rc] = ce;  // storage order
                by_id[b0 + rk] = ce;      // ascending id
                if (rk < BIG_FOLD) s_ord[wid][rk] = ce;
            }
        } else if (lane == 0) {
            for (int i = b0 + 1; i < b0 + nc; i++) {
                const int c0 = bin_cells[i];
                int j = i - 1;
                while (j >= b0 && bin_cells[j] > c0) {
                    bin_cells[j + 1] = bin_cells[j];
                    j--;
                }
                bin_cells[j + 1] = c0;
            }
            for (int i = b0; i < b0 + nc; i++) {
                const int c0 = bin_cells[i];
                const long long k0 = ids[c0];
                int j = i - 1;
                while (j >= b0 && ids[by_id[j]] > k0) {
                    by_id[j + 1] = by_id[j];
                    j--;
                }
                by_id[j + 1] = c0;
            }
        }
        __syncwarp();  // the id order is visible to the warp
        if (COEF && ca.aff && !ca.sp && nc <= BIG_FOLD && ca.S <= kLineMaxS) {
            // bin_coef_s's operations, the loads of all cells at once
            for (int it = lane; it < nc * ca.S; it += 32) {
                const int s = it / nc, u = it - s * nc, cidx = s_ord[wid][u];
                const double f = ca.dt * ca.volume[cidx] * ca.inv_vol;
                const double sec = ca.secretion[(long)s * n + cidx];
                const double upt = ca.uptake[(long)s * n + cidx];
                const double den = 1.0 + f * (sec + upt);
                if (den <= 0.0) atomicOr(&flags[FLAG_DOMAIN], 1);
                s_a[wid][s][u] = f * sec * ca.sat[s];
                s_d[wid][s][u] = den;
            }
            __syncwarp();
            if (lane < ca.S) {
                double alpha = 1.0, beta = 0.0;
                for (int u = 0; u < nc; u++) {
                    beta = (beta + s_a[wid][lane][u]) / s_d[wid][lane][u];
                    alpha = alpha / s_d[wid][lane][u];
                }
                reinterpret_cast<double2*>(ca.aff)[(long)lane * ca.rq + q] = make_double2(alpha, beta);
            }
        } else if (COEF) {
            for (int s = lane; s < ca.S; s += 32) bin_coef_s<COEF>(ca, n, q, v, b0, nc, by_id, s, flags);
        }
        __syncwarp();
    }
    pdl_trigger();
}

int launch_rebin(cg_ctx* c, int n, const double* pos, const int64_t* ids, int32_t* voxel,
                 int32_t* bin_start, int32_t* bin_cells, int32_t* bin_cells_by_id,
                 int32_t* nonempty, int32_t* n_nonempty, bool counted, const CoefLaunch* coef) {
    const int T = 256;
    const long nvox = c->nvox;
    const ScanState scan = scan_state(c);
    if (!counted)
        CG_LAUNCH(c, K_VOXEL_COUNT, k_voxel_count, std::max(1, (n + T - 1) / T), T, 0, n, pos, c->m,
                  voxel, c->d_counts, c->d_flags, scan);
    CG_LAUNCH(c, K_SCAN_BLOCK, k_scan_lookback, scan.nb, SCAN_T, 0, c->d_counts, nvox, c->m.nx,
              scan, bin_start, nonempty, n_nonempty, c->d_row_ne, c->d_ne_start);
    if (n > 0) {
        CG_LAUNCH(c, K_SCATTER, k_scatter, (n + T - 1) / T, T, 0, n, voxel, bin_start, c->d_counts,
                  bin_cells, c->d_n_big);
        const int maxq = (int)std::min<long>(nvox, n);
        // bins of more than BF_K cells: a warp each in k_bin_fix_big (env
        // CELLGPU_BINFIX_BIG=0: one thread's insertion sorts in k_bin_fix_g)
        const char* env_big = std::getenv("CELLGPU_BINFIX_BIG");
        int* big = env_big && std::atoi(env_big) == 0 ? nullptr : c->d_big;
        CoefArgs ca{};
        if (coef) {
            const ExchSet* o = coef->out;
            ca = CoefArgs{c->S, coef->dt, 1.0 / (c->m.dx * c->m.dy * c->m.dz), coef->secretion,
                          coef->uptake, c->d_sat, coef->volume, o ? o->A : c->d_exA,
                          o ? o->D : c->d_exD, o ? o->R : c->d_exR,
                          (int)std::min<long>(c->nvox, c->cap_cells), o ? o->vox : nullptr,
                          o ? o->start : nullptr, o ? o->n : nullptr,
                          coef->affine && o ? o->aff : nullptr, coef->affine && o ? o->pz : nullptr,
                          c->m.nx, c->m.ny * c->m.nz, coef->pos, coef->radius,
                          coef->pos ? (double4*)c->d_sp : nullptr, coef->pos ? c->d_svox : nullptr,
                          c->d_spf};
            // lanes per voxel (env CELLGPU_BINFIX_LANES = 2 / 4: the substrates'
            // coefficient folds side by side).  Measured: one lane per voxel
            // is fastest (config 1 0.159 vs 0.166 ms per step with 4 lanes,
            // config 3 1.807 vs 1.883, config 2 0.259 vs 0.273).
            const char* env = std::getenv("CELLGPU_BINFIX_LANES");
            int G = env ? std::atoi(env) : 1;
            G = G >= 4 ? 4 : G >= 2 ? 2 : 1;
            const long threads = (long)maxq * G;
            const int blocks = (int)((threads + T - 1) / T);
            if (G == 4)
                CG_LAUNCH(c, K_BIN_FIX, (k_bin_fix_g<true, 4>), blocks, T, 0, nonempty, n_nonempty,
                          bin_start, (const long long*)ids, bin_cells, bin_cells_by_id, n, maxq, ca,
                          c->d_flags, big, c->d_n_big);
            else if (G == 2)
                CG_LAUNCH(c, K_BIN_FIX, (k_bin_fix_g<true, 2>), blocks, T, 0, nonempty, n_nonempty,
                          bin_start, (const long long*)ids, bin_cells, bin_cells_by_id, n, maxq, ca,
                          c->d_flags, big, c->d_n_big);
            else
                CG_LAUNCH(c, K_BIN_FIX, (k_bin_fix_g<true, 1>), blocks, T, 0, nonempty, n_nonempty,
                          bin_start, (const long long*)ids, bin_cells, bin_cells_by_id, n, maxq, ca,
                          c->d_flags, big, c->d_n_big);
            if (big)
                CG_LAUNCH(c, K_BIN_FIX, k_bin_fix_big<true>, c->num_sms * 2, BIG_W * 32, 0, nonempty,
                          bin_start, (const long long*)ids, bin_cells, bin_cells_by_id, n, ca,
                          c->d_flags, big, c->d_n_big);
        } else {
            CG_LAUNCH(c, K_BIN_FIX, (k_bin_fix_g<false, 1>), (maxq + T - 1) / T, T, 0, nonempty,
                      n_nonempty, bin_start, (const long long*)ids, bin_cells, bin_cells_by_id, n,
                      maxq, ca, c->d_flags, big, c->d_n_big);
            if (big)
                CG_LAUNCH(c, K_BIN_FIX, k_bin_fix_big<false>, c->num_sms * 2, BIG_W * 32, 0, nonempty,
                          bin_start, (const long long*)ids, bin_cells, bin_cells_by_id, n, ca,
                          c->d_flags, big, c->d_n_big);
        }
    }
    return CG_OK;
}

// ---------------------------------------------------------------- velocities

// Gather (x, y, z, R) and id into id-sorted bin order: candidate reads in the
// velocity kernel then walk 9 contiguous slot ranges.
__global__ void k_gather(int n, const int32_t* __restrict__ by_id, const double* __restrict__ pos,
                         const double* __restrict__ radius, const long long* __restrict__ ids,
                         double4* __restrict__ sp, long long* __restrict__ sid,
                         int* __restrict__ sid32, int* __restrict__ wide,
                         int* __restrict__ n_queues, const int32_t* __restrict__ voxel,
                         int* __restrict__ svox, float4* __restrict__ spf) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int i = by_id[k];
    const double4 p = make_double4(pos[3L * i], pos[3L * i + 1], pos[3L * i + 2], radius[i]);
    sp[k] = p;
    spf[k] = make_float4((float)p.x, (float)p.y, (float)p.z, (float)p.w);
    if (voxel) svox[k] = voxel[i];
    if (k == 0) {  // mid / overflow queues (read by the previous call's last kernels)
        n_queues[0] = 0;
        n_queues[1] = 0;
    }
    const long long id = ids[i];
    sid[k] = id;
    sid32[k] = (int)id;
    if (id < 0 || id > 0x7fffffffll) *wide = 1;  // 32-bit rank keys would be wrong
    pdl_trigger();  // dependents launch as this grid finishes
}

struct PairParams {
    double c_r, c_a, m_a;
};

// mechanics.py:160-170 for one (resident i, candidate j) pair.  Returns the
// contribution, or zeros when the reference would `continue` (self, too close,
// out of reach).  Adding +0.0 to an accumulator that starts at +0.0 never
// changes its bits (IEEE RN never produces -0.0 from x + y unless both are
// -0.0), so skipped pairs may be summed as zeros.
// In-range test and contribution of pair (i, j) in the order of
// mechanics.py:99-115 (callers handle i == j).  d2 > reach^2 (1 + 2^-48)
// proves RN(sqrt(d2)) >= reach (sqrt and RN are monotone and the bound
// exceeds the exact reach^2 despite the two roundings), so most
// out-of-range pairs skip the square root.
__device__ __forceinline__ bool pair_in_range(const double4& pi, const double4& pj,
                                              const PairParams& pp, double& cx, double& cy,
                                              double& cz) {
    const double dx = pj.x - pi.x, dy = pj.y - pi.y, dz = pj.z - pi.z;
    const double d2 = dx * dx + dy * dy + dz * dz;
    const double contact = pi.w + pj.w;
    const double reach = pp.m_a * contact;
    if (d2 > (reach * reach) * 0x1.0000000000010p+0) return false;
    const double d = sqrt(d2);
    if (d < EPS_SKIP || d >= reach) return false;
    double rep = 0.0;
    if (d < contact) {
        const double t = 1.0 - d / contact;
        rep = -pp.c_r * (t * t);  // Python `(..)**2` is libm pow; see DESIGN.md (1e-12 bar)
    }
    const double t2 = 1.0 - d / reach;
    const double adh = pp.c_a * (t2 * t2);
    const double coef = (rep + adh) / d;
    cx = coef * dx;
    cy = coef * dy;
    cz = coef * dz;
    return true;
}

// Fast numerics: the same in-range test, then one division instead of three
// (q = 1/(d contact): d/contact = d2 q, d/reach = d2 q / m_a, 1/d = contact q);
// a few ulp from the reference's terms, well inside the 1e-12 bar.
struct PairParamsFast {
    double c_r, c_a, m_a, inv_ma;
};
// Conservative fp32 pre-test over (x, y, z, R) rounded to fp32: a pair is
// kept when d~^2 <= thr^2, thr = m_a (Ri + Rj) (1 + 2^-12) + 2^-21 Xmax
// (Xmax: the largest |coordinate| of the mesh box).  The coordinates' fp32
// rounding moves each difference by at most 2u Xmax (u = 2^-24) and the fp32
// arithmetic by a few u relative, so every pair the fp64 pre-test keeps
// (d^2 <= reach^2 (1 + 2^-48)) is kept here too; the kept pairs' fp64 terms
// still decide (out of range: +0.0).  Half the bytes of the walk's loads.
struct PreTest {
    float m_a, rel, abs;
};
__device__ __forceinline__ bool pretest_f32(const float4& pi, const float4& pj, const PreTest& t) {
    const float dx = pj.x - pi.x, dy = pj.y - pi.y, dz = pj.z - pi.z;
    const float d2 = dx * dx + dy * dy + dz * dz;
    const float thr = t.m_a * (pi.w + pj.w) * t.rel + t.abs;
    return d2 <= thr * thr;
}
static PreTest pretest_params(const MeshDev& m, double m_a) {
    const double lo[3] = {m.ox, m.oy, m.oz};
    const double hi[3] = {m.ox + m.nx * m.dx, m.oy + m.ny * m.dy, m.oz + m.nz * m.dz};
    double xmax = 0.0;
    for (int k = 0; k < 3; k++) xmax = std::max(xmax, std::max(std::fabs(lo[k]), std::fabs(hi[k])));
    return PreTest{(float)m_a, 1.0f + 0x1p-12f, (float)(xmax * 0x1p-21) + 1e-30f};
}

__device__ __forceinline__ bool pair_in_range_fast(const double4& pi, const double4& pj,
                                                   const PairParamsFast& pp, double& cx,
                                                   double& cy, double& cz) {
    const double dx = pj.x - pi.x, dy = pj.y - pi.y, dz = pj.z - pi.z;
    const double d2 = dx * dx + dy * dy + dz * dz;
    const double contact = pi.w + pj.w;
    const double reach = pp.m_a * contact;
    if (d2 > (reach * reach) * 0x1.0000000000010p+0) return false;
    const double d = sqrt(d2);
    if (d < EPS_SKIP || d >= reach) return false;
    const double q = 1.0 / (d * contact);
    const double dc = d2 * q;  // d / contact
    double rep = 0.0;
    if (d < contact) {
        const double t = 1.0 - dc;
        rep = -pp.c_r * (t * t);
    }
    const double t2 = 1.0 - dc * pp.inv_ma;
    const double coef = (rep + pp.c_a * (t2 * t2)) * (contact * q);
    cx = coef * dx;
    cy = coef * dy;
    cz = coef * dz;
    return true;
}

// The terms of a pre-test survivor without branches: the operations of
// pair_in_range / pair_in_range_fast on an in-range pair, +0.0 otherwise (a
// survivor out of range has d >= reach or d < EPS_SKIP; the discarded
// quotients may be inf/NaN).  Straight-line code lets two pairs' division
// and square-root chains overlap.
__device__ __forceinline__ void pair_term_sel(const double4& pi, const double4& pj,
                                              const PairParams& pp, double& cx, double& cy,
                                              double& cz) {
    const double dx = pj.x - pi.x, dy = pj.y - pi.y, dz = pj.z - pi.z;
    const double d2 = dx * dx + dy * dy + dz * dz;
    const double contact = pi.w + pj.w;
    const double reach = pp.m_a * contact;
    const double d = sqrt(d2);
    const bool in = d >= EPS_SKIP && d < reach;
    const double t = 1.0 - d / contact;
    const double rep = d < contact ? -pp.c_r * (t * t) : 0.0;
    const double t2 = 1.0 - d / reach;
    const double adh = pp.c_a * (t2 * t2);
    const double coef = (rep + adh) / d;
    cx = in ? coef * dx : 0.0;
    cy = in ? coef * dy : 0.0;
    cz = in ? coef * dz : 0.0;
}
__device__ __forceinline__ void pair_term_sel_fast(const double4& pi, const double4& pj,
                                                   const PairParamsFast& pp, double& cx,
                                                   double& cy, double& cz) {
    const double dx = pj.x - pi.x, dy = pj.y - pi.y, dz = pj.z - pi.z;
    const double d2 = dx * dx + dy * dy + dz * dz;
    const double contact = pi.w + pj.w;
    const double reach = pp.m_a * contact;
    const double d = sqrt(d2);
    const bool in = d >= EPS_SKIP && d < reach;
    const double q = 1.0 / (d * contact);
    const double dc = d2 * q;
    const double t = 1.0 - dc;
    const double rep = d < contact ? -pp.c_r * (t * t) : 0.0;
    const double t2 = 1.0 - dc * pp.inv_ma;
    const double coef = (rep + pp.c_a * (t2 * t2)) * (contact * q);
    cx = in ? coef * dx : 0.0;
    cy = in ? coef * dy : 0.0;
    cz = in ? coef * dz : 0.0;
}

__device__ __forceinline__ void pair_term(const double4& pi, long long idi, const double4& pj,
                                          long long idj, const PairParams& pp, double& cx,
                                          double& cy, double& cz) {
    if (idi == idj || !pair_in_range(pi, pj, pp, cx, cy, cz)) cx = cy = cz = 0.0;
}

constexpr int VEL_WARPS = 4;
constexpr int VEL_CAP = 256;  // candidates per warp in shared memory
constexpr int VEL_G = 10;     // residents summed concurrently (3 lanes each)
constexpr int VEL_BUF = 32 * 3 + 1;  // padded per-resident stride (doubles)

struct VelWarpSmem {
    long long cid[VEL_CAP];
    int cslot[VEL_CAP];
    int order[VEL_CAP];
    double buf[VEL_G * VEL_BUF];
};

// Candidate ranges of voxel (ix,iy,iz): lanes 0..8 each own one (dz, dy) row
// of the 3x3x3 block, clamped to the mesh (mechanics.py:124-131).
__device__ __forceinline__ void row_range(const MeshDev& m, const int32_t* __restrict__ bin_start,
                                          int ix, int iy, int iz, int lane, int& s0, int& cnt) {
    s0 = 0;
    cnt = 0;
    if (lane < 9) {
        const int z = iz + lane / 3 - 1, y = iy + lane % 3 - 1;
        if (z >= 0 && z < m.nz && y >= 0 && y < m.ny) {
            const long row = ((long)z * m.ny + y) * m.nx;
            const int xlo = ix > 0 ? ix - 1 : 0, xhi = ix + 1 < m.nx ? ix + 1 : m.nx - 1;
            s0 = bin_start[row + xlo];
            cnt = bin_start[row + xhi + 1] - s0;
        }
    }
}

// Accumulate velocities of residents [r0, r1) of a voxel whose id-sorted
// candidate slots are order[0, n).  Executed by one warp.
__device__ __forceinline__ void warp_accumulate(const int* order, int n, int b0, int r0, int r1,
                                                const double4* __restrict__ sp,
                                                const long long* __restrict__ sid,
                                                const int32_t* __restrict__ by_id,
                                                const PairParams& pp, double* buf,
                                                double* __restrict__ vel, int lane, int rstep) {
    for (int g0 = r0; g0 < r1; g0 += VEL_G * rstep) {
        // residents g0, g0+rstep, ... (at most VEL_G)
        int gn = 0;
        for (int r = g0; r < r1 && gn < VEL_G; r += rstep) gn++;
        double acc = 0.0;
        const int my_r = lane / 3, my_c = lane - 3 * (lane / 3);
        for (int j0 = 0; j0 < n; j0 += 32) {
            const int jn = min(32, n - j0);
            double4 pj = make_double4(0.0, 0.0, 0.0, 0.0);
            long long idj = -1;
            if (lane < jn) {
                const int sj = order[j0 + lane];
                pj = sp[sj];
                idj = sid[sj];
            }
            for (int r = 0; r < gn; r++) {
                const int si = b0 + g0 + r * rstep;
                const double4 pi = sp[si];
                const long long idi = sid[si];
                double cx = 0.0, cy = 0.0, cz = 0.0;
                if (lane < jn) pair_term(pi, idi, pj, idj, pp, cx, cy, cz);
                double* b = buf + r * VEL_BUF + lane * 3;
                b[0] = cx;
                b[1] = cy;
                b[2] = cz;
            }
            __syncwarp();
            if (lane < 3 * gn) {
                const double* b = buf + my_r * VEL_BUF + my_c;
                for (int jj = 0; jj < jn; jj++) acc = acc + b[jj * 3];
            }
            __syncwarp();
        }
        if (lane < 3 * gn) {
            const int cell = by_id[b0 + g0 + my_r * rstep];
            vel[3L * cell + my_c] = acc;
        }
    }
}

// Velocities in two passes.
//
// Pass 1, k_cand_lists (one warp per non-empty voxel): gathers the 3x3x3
// candidate union (9 contiguous slot ranges; lane j's slot comes from a
// per-warp table written by the 9 row owners), ranks the candidates by id with
// 32-bit keys over warp shuffles (two candidates per lane, at most 64), and
// writes the id-sorted slot list of the voxel -- the reference's
// _voxel_candidates (mechanics.py:118-133) -- to cand[q*64 + rank].  Each
// resident slot records its voxel's list index.  Voxels with more than 64
// candidates, or ids that do not fit 32-bit keys, go to k_velocity_mid.
//
// Pass 2, k_velocity_cells (one thread per cell in id-sorted bin order): walks
// its voxel's list in order and accumulates the pair terms in registers --
// exactly _cell_velocity's loop (mechanics.py:145-172).  Consecutive threads
// belong to the same or adjacent voxels, so their candidate loads share L1.
constexpr int LIST_WARPS = 8;
constexpr int LIST_CAP = 64;

__global__ void __launch_bounds__(LIST_WARPS * 32) k_cand_lists(
    MeshDev m, const int32_t* __restrict__ bin_start, const int32_t* __restrict__ nonempty,
    const int32_t* __restrict__ n_nonempty, const int* __restrict__ sid32,
    const int* __restrict__ wide, int* __restrict__ cand, int* __restrict__ slot_list,
    int* __restrict__ mid, int* __restrict__ n_mid) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    __shared__ int sdslot[LIST_WARPS][LIST_CAP];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int* dslot = sdslot[wid];
    const int nne = *n_nonempty;
    const bool ids32 = *wide == 0;
    for (int q = blockIdx.x * LIST_WARPS + wid; q < nne; q += gridDim.x * LIST_WARPS) {
        const int v = nonempty[q];
        const int rest = (int)fdiv((unsigned)v, m.fnx), ix = v - rest * m.nx;
        const int iz = (int)fdiv((unsigned)rest, m.fny), iy = rest - iz * m.ny;
        int s0, cnt;
        row_range(m, bin_start, ix, iy, iz, lane, s0, cnt);
        int bb = 0;
        if (lane == 9) bb = bin_start[v];
        if (lane == 10) bb = bin_start[v + 1];
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const int n = __shfl_sync(0xffffffffu, inc, 8);
        const int b0 = __shfl_sync(0xffffffffu, bb, 9);
        const int nres = __shfl_sync(0xffffffffu, bb, 10) - b0;
        const bool listed = n <= LIST_CAP && ids32;
        for (int r = lane; r < nres; r += 32) slot_list[b0 + r] = listed ? q : -1;
        if (!listed) {
            if (lane == 0) mid[atomicAdd(n_mid, 1)] = v;
            continue;
        }
        {
            const int off = inc - cnt;
            for (int j = 0; j < cnt; j++) dslot[off + j] = s0 - off;
        }
        __syncwarp();
        const bool has0 = lane < n, has1 = lane + 32 < n;
        const int slot0 = has0 ? lane + dslot[lane] : 0;
        const int slot1 = has1 ? lane + 32 + dslot[lane + 32] : 0;
        const int k0 = has0 ? sid32[slot0] : 0x7fffffff;
        const int k1 = has1 ? sid32[slot1] : 0x7fffffff;
        int* out = cand + (long)q * LIST_CAP;
        if (n <= 32) {
            // Bitonic sort of (id key, slot) across the warp: lane k ends up
            // holding the k-th smallest id; one coalesced 128 B list write.
            int key = k0, val = slot0;
#pragma unroll
            for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    const int ok = __shfl_xor_sync(0xffffffffu, key, stride);
                    const int ov = __shfl_xor_sync(0xffffffffu, val, stride);
                    const bool up = (lane & size) == 0;           // ascending segment
                    const bool lower = (lane & stride) == 0;      // partner is above
                    const bool take_other = (lower == up) ? (ok < key) : (ok > key);
                    if (take_other) {
                        key = ok;
                        val = ov;
                    }
                }
            }
            out[lane] = lane < n ? val : -1;
            if (n == 32 && lane < 4) out[32 + lane] = -1;  // terminate the last int4
        } else {
            int rank0 = 0, rank1 = 0;
            for (int k = 0; k < 32; k++) {
                const int x = __shfl_sync(0xffffffffu, k0, k);
                rank0 += x < k0;
                rank1 += x < k1;
            }
            for (int k = 0; k < n - 32; k++) {
                const int x = __shfl_sync(0xffffffffu, k1, k);
                rank0 += x < k0;
                rank1 += x < k1;
            }
            out[rank0] = slot0;
            if (has1) out[rank1] = slot1;
            // -1 from n to the end of its int4 (the per-cell loop reads 4 at a time)
            const int pad_end = min(LIST_CAP, (n / 4 + 1) * 4);
            if (n + lane < pad_end) out[n + lane] = -1;
        }
        __syncwarp();
    }
    pdl_trigger();  // dependents launch as this grid finishes
}

__global__ void __launch_bounds__(256) k_velocity_cells(
    int n_cells, const int* __restrict__ slot_list, const int* __restrict__ cand,
    const int32_t* __restrict__ by_id, const double4* __restrict__ sp,
    const int* __restrict__ sid32, PairParams pp, double* __restrict__ vel) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    // Grid-stride: the engine may cap the grid so the velocity branch leaves
    // room on every SM for the concurrent diffusion kernels.
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_cells; k += gridDim.x * blockDim.x) {
    const int q = slot_list[k];
    if (q < 0) continue;  // voxel handled by k_velocity_mid / k_velocity_big
    const double4 pi = sp[k];
    const int idi = sid32[k];
    const int* list = cand + (long)q * LIST_CAP;
    double ax = 0.0, ay = 0.0, az = 0.0;
    // Software pipeline: candidate j + 1's position and id are in flight
    // while candidate j's term is computed (the list is read one further).
    int sj = list[0];
    double4 pj = make_double4(0.0, 0.0, 0.0, 0.0);
    int idj = 0;
    if (sj >= 0) {
        pj = sp[sj];
        idj = sid32[sj];
    }
    int j = 1;
    int s_next = LIST_CAP > 1 ? list[1] : -1;
    while (sj >= 0) {
        double4 pn = pj;
        int idn = idj;
        const int sn = s_next;
        if (sn >= 0) {
            pn = sp[sn];
            idn = sid32[sn];
        }
        j++;
        s_next = (sn >= 0 && j < LIST_CAP) ? list[j] : -1;
        double cx, cy, cz;
        pair_term(pi, idi, pj, idj, pp, cx, cy, cz);
        ax = ax + cx;
        ay = ay + cy;
        az = az + cz;
        sj = sn;
        pj = pn;
        idj = idn;
    }
    const int cell = by_id[k];
    vel[3L * cell] = ax;
    vel[3L * cell + 1] = ay;
    vel[3L * cell + 2] = az;
    }
    pdl_trigger();  // dependents launch as this grid finishes
}

// General path: candidate unions of 33..VEL_CAP cells staged in shared memory
// and rank-sorted there; larger ones go on to k_velocity_big.
__global__ void __launch_bounds__(VEL_WARPS * 32) k_velocity_mid(
    MeshDev m, const int32_t* __restrict__ bin_start, const int* __restrict__ mid,
    const int* __restrict__ n_mid, const int32_t* __restrict__ by_id,
    const double4* __restrict__ sp, const long long* __restrict__ sid, PairParams pp,
    double* __restrict__ vel, int* __restrict__ overflow, int* __restrict__ n_overflow) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    __shared__ VelWarpSmem smem[VEL_WARPS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    VelWarpSmem& ws = smem[wid];
    const int nq = *n_mid;
    for (int q = blockIdx.x * VEL_WARPS + wid; q < nq; q += gridDim.x * VEL_WARPS) {
        const int v = mid[q];
        const int rest = (int)fdiv((unsigned)v, m.fnx), ix = v - rest * m.nx;
        const int iz = (int)fdiv((unsigned)rest, m.fny), iy = rest - iz * m.ny;
        int s0, cnt;
        row_range(m, bin_start, ix, iy, iz, lane, s0, cnt);
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const int n = __shfl_sync(0xffffffffu, inc, 8);
        const int off = inc - cnt;
        if (n > VEL_CAP) {
            if (lane == 0) overflow[atomicAdd(n_overflow, 1)] = v;
            continue;
        }
        for (int r = 0; r < 9; r++) {
            const int rs = __shfl_sync(0xffffffffu, s0, r);
            const int rc = __shfl_sync(0xffffffffu, cnt, r);
            const int ro = __shfl_sync(0xffffffffu, off, r);
            for (int j = lane; j < rc; j += 32) {
                ws.cslot[ro + j] = rs + j;
                ws.cid[ro + j] = sid[rs + j];
            }
        }
        __syncwarp();
        for (int j = lane; j < n; j += 32) {  // rank sort by id (ids are unique)
            const long long id = ws.cid[j];
            int rank = 0;
            for (int k = 0; k < n; k++) rank += ws.cid[k] < id;
            ws.order[rank] = ws.cslot[j];
        }
        __syncwarp();
        const int b0 = bin_start[v], nres = bin_start[v + 1] - b0;
        warp_accumulate(ws.order, n, b0, 0, nres, sp, sid, by_id, pp, ws.buf, vel, lane, 1);
        __syncwarp();
    }
    pdl_trigger();  // dependents launch as this grid finishes
}

// Voxels whose candidate union exceeds VEL_CAP: one CTA each, candidates in
// dynamic shared memory, residents split across the CTA's warps.
constexpr int BIG_T = 256;
__global__ void __launch_bounds__(BIG_T) k_velocity_big(
    MeshDev m, const int32_t* __restrict__ bin_start, const int* __restrict__ overflow,
    const int* __restrict__ n_overflow, const int32_t* __restrict__ by_id,
    const double4* __restrict__ sp, const long long* __restrict__ sid, PairParams pp,
    double* __restrict__ vel, int big_cap, int* __restrict__ flags) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    extern __shared__ double bsm[];
    double* bufs = bsm;                                        // (BIG_T/32) * VEL_G * VEL_BUF
    long long* cid = (long long*)(bufs + (BIG_T / 32) * VEL_G * VEL_BUF);  // big_cap
    int* cslot = (int*)(cid + big_cap);                        // big_cap
    int* order = cslot + big_cap;                              // big_cap
    __shared__ int rs[9], rc[9], ro[10];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nov = *n_overflow;
    // Last velocity kernel: reset the ids-not-32-bit flag k_gather raises
    // (k_cand_lists, its only reader, has completed).
    if (blockIdx.x == 0 && threadIdx.x == 0) const_cast<int*>(n_overflow)[2] = 0;
    for (int o = blockIdx.x; o < nov; o += gridDim.x) {
        const int v = overflow[o];
        const int rest = (int)fdiv((unsigned)v, m.fnx), ix = v - rest * m.nx;
        const int iz = (int)fdiv((unsigned)rest, m.fny), iy = rest - iz * m.ny;
        if (wid == 0) {
            int s0, cnt;
            row_range(m, bin_start, ix, iy, iz, lane, s0, cnt);
            int inc = cnt;
            for (int k = 1; k < 16; k <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, k);
                if (lane >= k) inc += y;
            }
            if (lane < 9) {
                rs[lane] = s0;
                rc[lane] = cnt;
                ro[lane] = inc - cnt;
            }
            if (lane == 8) ro[9] = inc;
        }
        __syncthreads();
        const int n = ro[9];
        if (n > big_cap) {
            if (threadIdx.x == 0) atomicOr(&flags[FLAG_CAPACITY], 1);
            __syncthreads();
            continue;
        }
        for (int r = 0; r < 9; r++)
            for (int j = threadIdx.x; j < rc[r]; j += BIG_T) {
                cslot[ro[r] + j] = rs[r] + j;
                cid[ro[r] + j] = sid[rs[r] + j];
            }
        __syncthreads();
        for (int j = threadIdx.x; j < n; j += BIG_T) {
            const long long id = cid[j];
            int rank = 0;
            for (int k = 0; k < n; k++) rank += cid[k] < id;
            order[rank] = cslot[j];
        }
        __syncthreads();
        const int b0 = bin_start[v], nres = bin_start[v + 1] - b0;
        warp_accumulate(order, n, b0, wid, nres, sp, sid, by_id, pp,
                        bufs + wid * VEL_G * VEL_BUF, vel, lane, BIG_T / 32);
        __syncthreads();
    }
    pdl_trigger();  // dependents launch as this grid finishes
}

// Exact numerics without candidate lists.  A skipped pair adds +0.0, which
// never changes an accumulator that starts at +0.0, so the reference's sum
// over the id-sorted candidate union (mechanics.py:145-172) equals the sum
// over its in-range pairs alone in ascending id.
//
// Thread per cell (id-sorted bin order): walk the 9 row ranges with the
// squared-distance pre-test, insert the survivors into a small id-sorted
// queue, then add the exact pair terms in queue order.  More than XQ
// survivors: the XQ smallest ids are summed, and the walk repeats for the ids
// above the last one summed.  Cells with more than dense_min candidates go
// to k_velocity_exact_dense (warp per cell).
constexpr int XQ = 16;

// Row ranges of the 3x3x3 block around voxel v (mechanics.py:124-131).
__device__ __forceinline__ void block_rows(const MeshDev& m, const int32_t* __restrict__ bin_start,
                                           int v, int (&r0)[9], int (&r1)[9]) {
    const int rest = (int)fdiv((unsigned)v, m.fnx), ix = v - rest * m.nx;
    const int iz = (int)fdiv((unsigned)rest, m.fny), iy = rest - iz * m.ny;
    const int xlo = ix > 0 ? ix - 1 : 0, xhi = ix + 1 < m.nx ? ix + 1 : m.nx - 1;
#pragma unroll
    for (int r = 0; r < 9; r++) {
        const int z = iz + r / 3 - 1, y = iy + r % 3 - 1;
        r0[r] = r1[r] = 0;
        if (z >= 0 && z < m.nz && y >= 0 && y < m.ny) {
            const long row = ((long)z * m.ny + y) * m.nx;
            r0[r] = bin_start[row + xlo];
            r1[r] = bin_start[row + xhi + 1];
        }
    }
}

__device__ __forceinline__ void exact_cell_queue(int k, const int (&r0)[9], const int (&r1)[9],
                                                 const double4* __restrict__ sp,
                                                 const long long* __restrict__ sid,
                                                 const PairParams& pp, double& ax, double& ay,
                                                 double& az) {
    const double4 pi = sp[k];
    ax = ay = az = 0.0;
    long long qid[XQ];
    int qs[XQ];
    long long lo = LLONG_MIN;  // ids up to lo are summed
    for (;;) {
        int nq = 0;
        bool more = false;
#pragma unroll 1
        for (int r = 0; r < 9; r++) {
#pragma unroll 2
            for (int j = r0[r]; j < r1[r]; j++) {
                const double4 pj = sp[j];
                const double dx = pj.x - pi.x, dy = pj.y - pi.y, dz = pj.z - pi.z;
                const double d2 = dx * dx + dy * dy + dz * dz;
                const double reach = pp.m_a * (pi.w + pj.w);
                if (j == k || d2 > (reach * reach) * 0x1.0000000000010p+0) continue;
                const long long id = sid[j];
                if (id <= lo) continue;
                if (nq == XQ) {
                    more = true;
                    if (id > qid[XQ - 1]) continue;
                    nq--;  // the largest waits for the next walk
                }
                int t = nq++;
                for (; t > 0 && qid[t - 1] > id; t--) {
                    qid[t] = qid[t - 1];
                    qs[t] = qs[t - 1];
                }
                qid[t] = id;
                qs[t] = j;
            }
        }
        int t = 0;
        for (; t + 1 < nq; t += 2) {  // two terms in flight, added in queue order
            double c0x, c0y, c0z, c1x, c1y, c1z;
            pair_term_sel(pi, sp[qs[t]], pp, c0x, c0y, c0z);
            pair_term_sel(pi, sp[qs[t + 1]], pp, c1x, c1y, c1z);
            ax = ax + c0x;
            ay = ay + c0y;
            az = az + c0z;
            ax = ax + c1x;
            ay = ay + c1y;
            az = az + c1z;
        }
        if (t < nq) {
            double cx, cy, cz;
            pair_term_sel(pi, sp[qs[t]], pp, cx, cy, cz);
            ax = ax + cx;
            ay = ay + cy;
            az = az + cz;
        }
        if (!more) break;
        lo = qid[nq - 1];
    }
}

template <bool DENSE>
__global__ void __launch_bounds__(256) k_velocity_exact(int n, MeshDev m,
                                                        const int32_t* __restrict__ bin_start,
                                                        const int32_t* __restrict__ by_id,
                                                        const double4* __restrict__ sp,
                                                        const long long* __restrict__ sid,
                                                        const int* __restrict__ svox, PairParams pp,
                                                        double* __restrict__ vel,
                                                        int* __restrict__ dense,
                                                        int* __restrict__ n_dense, int dense_min,
                                                        const float4* __restrict__ spf, PreTest pt) {
    pdl_wait();
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        int r0[9], r1[9];
        block_rows(m, bin_start, svox[k], r0, r1);
        if (DENSE) {
            int nc = 0;
#pragma unroll
            for (int r = 0; r < 9; r++) nc += r1[r] - r0[r];
            if (nc > dense_min) {
                dense[atomicAdd(n_dense, 1)] = k;
                continue;
            }
        }
        // Common case: the survivors' slots are queued during the walk (no
        // dependent id load in the walk), their ids loaded together after
        // it and the queue sorted; more than XQ survivors: exact_cell_queue.
        const double4 pi = sp[k];
        const float4 pif = spf[k];
        int qs[XQ];
        int nq = 0;
        bool over = false;
#pragma unroll 1
        for (int r = 0; r < 9 && !over; r++) {
#pragma unroll 2
            for (int j = r0[r]; j < r1[r]; j++) {
                if (j == k || !pretest_f32(pif, spf[j], pt)) continue;
                if (nq == XQ) {
                    over = true;
                    break;
                }
                qs[nq++] = j;
            }
        }
        double ax = 0.0, ay = 0.0, az = 0.0;
        if (over) {
            exact_cell_queue(k, r0, r1, sp, sid, pp, ax, ay, az);
        } else {
            long long qid[XQ];
            for (int t = 0; t < nq; t++) qid[t] = sid[qs[t]];
            for (int t = 1; t < nq; t++) {  // insertion sort by id
                const long long id = qid[t];
                const int sl = qs[t];
                int u = t;
                for (; u > 0 && qid[u - 1] > id; u--) {
                    qid[u] = qid[u - 1];
                    qs[u] = qs[u - 1];
                }
                qid[u] = id;
                qs[u] = sl;
            }
            int t = 0;
            for (; t + 1 < nq; t += 2) {
                double c0x, c0y, c0z, c1x, c1y, c1z;
                pair_term_sel(pi, sp[qs[t]], pp, c0x, c0y, c0z);
                pair_term_sel(pi, sp[qs[t + 1]], pp, c1x, c1y, c1z);
                ax = ax + c0x;
                ay = ay + c0y;
                az = az + c0z;
                ax = ax + c1x;
                ay = ay + c1y;
                az = az + c1z;
            }
            if (t < nq) {
                double cx, cy, cz;
                pair_term_sel(pi, sp[qs[t]], pp, cx, cy, cz);
                ax = ax + cx;
                ay = ay + cy;
                az = az + cz;
            }
        }
        const int cell = by_id[k];
        vel[3L * cell] = ax;
        vel[3L * cell + 1] = ay;
        vel[3L * cell + 2] = az;
    }
    pdl_trigger();
}

// Warp per dense cell: the lanes run the exact pair terms over the candidate
// union in parallel and append the in-range ones (id, term) to shared memory;
// a rank sort by id orders them, and lanes 0..2 sum one component each in that
// order.  More than DCAP in-range pairs: the thread-level queue walk.
constexpr int DW = 4;
constexpr int DCAP = 256;
__global__ void __launch_bounds__(DW * 32) k_velocity_exact_dense(
    const int* __restrict__ dense, const int* __restrict__ n_dense, MeshDev m,
    const int32_t* __restrict__ bin_start, const int32_t* __restrict__ by_id,
    const double4* __restrict__ sp, const long long* __restrict__ sid,
    const int* __restrict__ svox, PairParams pp, double* __restrict__ vel,
    int* __restrict__ wide) {
    pdl_wait();
    __shared__ long long s_id[DW][DCAP];
    __shared__ double s_c[DW][3][DCAP];
    __shared__ short s_ord[DW][DCAP];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // Last exact velocity kernel: reset k_gather's ids-not-32-bit flag (read
    // only by the candidate-list path).
    if (blockIdx.x == 0 && threadIdx.x == 0) *wide = 0;
    const int nd = *n_dense;
    for (int q = blockIdx.x * DW + wid; q < nd; q += gridDim.x * DW) {
        const int k = dense[q];
        int r0[9], r1[9];
        block_rows(m, bin_start, svox[k], r0, r1);
        int off[10];
        off[0] = 0;
#pragma unroll
        for (int r = 0; r < 9; r++) off[r + 1] = off[r] + (r1[r] - r0[r]);
        const int nc = off[9];
        const double4 pi = sp[k];
        int cnt = 0;
        for (int b = 0; b < nc; b += 32) {
            const int i = b + lane;
            bool in = false;
            double cx = 0.0, cy = 0.0, cz = 0.0;
            long long id = 0;
            if (i < nc) {
                int r = 0;
#pragma unroll
                for (int u = 1; u < 9; u++) r += i >= off[u];
                const int j = r0[r] + (i - off[r]);
                if (j != k) {
                    in = pair_in_range(pi, sp[j], pp, cx, cy, cz);
                    if (in) id = sid[j];
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            const int pos = cnt + __popc(bal & ((1u << lane) - 1));
            if (in && pos < DCAP) {
                s_id[wid][pos] = id;
                s_c[wid][0][pos] = cx;
                s_c[wid][1][pos] = cy;
                s_c[wid][2][pos] = cz;
            }
            cnt += __popc(bal);
        }
        double acc = 0.0;
        if (cnt <= DCAP) {
            __syncwarp();
            for (int e = lane; e < cnt; e += 32) {
                const long long id = s_id[wid][e];
                int rank = 0;
                for (int f = 0; f < cnt; f++) rank += s_id[wid][f] < id;
                s_ord[wid][rank] = (short)e;
            }
            __syncwarp();
            if (lane < 3)
                for (int r = 0; r < cnt; r++) acc = acc + s_c[wid][lane][s_ord[wid][r]];
        } else if (lane == 0) {
            double ax, ay, az;
            exact_cell_queue(k, r0, r1, sp, sid, pp, ax, ay, az);
            vel[3L * by_id[k]] = ax;
            vel[3L * by_id[k] + 1] = ay;
            vel[3L * by_id[k] + 2] = az;
        }
        if (cnt <= DCAP && lane < 3) vel[3L * by_id[k] + lane] = acc;
        __syncwarp();
    }
    pdl_trigger();
}

// Voxel of every bin slot (cg_velocities without the rebin's per-cell voxel
// keys): thread per non-empty voxel.
__global__ void k_slot_voxel(const int32_t* __restrict__ nonempty,
                             const int32_t* __restrict__ n_nonempty,
                             const int32_t* __restrict__ bin_start, int maxq, int* __restrict__ svox) {
    pdl_wait();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < maxq && q < *n_nonempty) {
        const int v = nonempty[q];
        for (int k = bin_start[v], e = bin_start[v + 1]; k < e; k++) svox[k] = v;
    }
    pdl_trigger();
}

// ---- fast numerics (CG_NUMERICS_FAST)
// Gather (x, y, z, R) and the voxel into id-sorted bin order.
__global__ void k_gather_fast(int n, const int32_t* __restrict__ by_id, const double* __restrict__ pos,
                              const double* __restrict__ radius, const int32_t* __restrict__ voxel,
                              double4* __restrict__ sp, int* __restrict__ svox,
                              float4* __restrict__ spf) {
    pdl_wait();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) {
        const int i = by_id[k];
        const double4 p = make_double4(pos[3L * i], pos[3L * i + 1], pos[3L * i + 2], radius[i]);
        sp[k] = p;
        spf[k] = make_float4((float)p.x, (float)p.y, (float)p.z, (float)p.w);
        svox[k] = voxel[i];
    }
    pdl_trigger();
}

// Thread per cell (id-sorted bin order, so a warp's cells share their
// neighbourhood in L1): the pair terms of mechanics.py:99-115 over the 3x3x3
// block (mechanics.py:118-133), row by row -- 9 contiguous slot ranges, x
// then id within a row -- instead of the reference's global ascending-id
// order (mechanics.py:145-172).  Same terms, summed in another order: within
// 1e-12 of the reference (normwise), and no candidate-list pass, no capacity
// limit on dense voxels.
__global__ void __launch_bounds__(256) k_velocity_direct(int n, MeshDev m,
                                                         const int32_t* __restrict__ bin_start,
                                                         const int32_t* __restrict__ by_id,
                                                         const double4* __restrict__ sp,
                                                         const int* __restrict__ svox, PairParamsFast pp,
                                                         double* __restrict__ vel) {
    pdl_wait();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) {
        const int v = svox[k];
        const int rest = (int)fdiv((unsigned)v, m.fnx), ix = v - rest * m.nx;
        const int iz = (int)fdiv((unsigned)rest, m.fny), iy = rest - iz * m.ny;
        const int xlo = ix > 0 ? ix - 1 : 0, xhi = ix + 1 < m.nx ? ix + 1 : m.nx - 1;
        int r0[9], r1[9];
#pragma unroll
        for (int r = 0; r < 9; r++) {
            const int z = iz + r / 3 - 1, y = iy + r % 3 - 1;
            r0[r] = r1[r] = 0;
            if (z >= 0 && z < m.nz && y >= 0 && y < m.ny) {
                const long row = ((long)z * m.ny + y) * m.nx;
                r0[r] = bin_start[row + xlo];
                r1[r] = bin_start[row + xhi + 1];
            }
        }
        const double4 pi = sp[k];
        double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll 1
        for (int r = 0; r < 9; r++) {
            int j = r0[r];
            const int j1 = r1[r];
            // two candidates in flight
            for (; j + 1 < j1; j += 2) {
                const double4 pa = sp[j], pb = sp[j + 1];
                double cx, cy, cz;
                if (j != k && pair_in_range_fast(pi, pa, pp, cx, cy, cz)) {
                    ax = ax + cx;
                    ay = ay + cy;
                    az = az + cz;
                }
                if (j + 1 != k && pair_in_range_fast(pi, pb, pp, cx, cy, cz)) {
                    ax = ax + cx;
                    ay = ay + cy;
                    az = az + cz;
                }
            }
            if (j < j1 && j != k) {
                double cx, cy, cz;
                if (pair_in_range_fast(pi, sp[j], pp, cx, cy, cz)) {
                    ax = ax + cx;
                    ay = ay + cy;
                    az = az + cz;
                }
            }
        }
        const int cell = by_id[k];
        vel[3L * cell] = ax;
        vel[3L * cell + 1] = ay;
        vel[3L * cell + 2] = az;
    }
    pdl_trigger();
}

// Per-cell velocities with the in-range pairs compacted (fast numerics): the
// walk over the 9 row ranges only runs the cheap squared-distance pre-test
// and queues the survivors' slots (local memory, encounter order); the full
// pair terms then run over the queue.  A warp executes the expensive branch
// (square root, division) max-queue-length times instead of once per
// candidate index at which any lane is in range.  Summation order unchanged
// (rows, x, id).
constexpr int VQ = 32;
__global__ void __launch_bounds__(256) k_velocity_compact(int n, MeshDev m,
                                                          const int32_t* __restrict__ bin_start,
                                                          const int32_t* __restrict__ by_id,
                                                          const double4* __restrict__ sp,
                                                          const int* __restrict__ svox,
                                                          PairParamsFast pp, double* __restrict__ vel,
                                                          const float4* __restrict__ spf, PreTest pt) {
    pdl_wait();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) {
        const int v = svox[k];
        const int rest = (int)fdiv((unsigned)v, m.fnx), ix = v - rest * m.nx;
        const int iz = (int)fdiv((unsigned)rest, m.fny), iy = rest - iz * m.ny;
        const int xlo = ix > 0 ? ix - 1 : 0, xhi = ix + 1 < m.nx ? ix + 1 : m.nx - 1;
        int r0[9], r1[9];
#pragma unroll
        for (int r = 0; r < 9; r++) {
            const int z = iz + r / 3 - 1, y = iy + r % 3 - 1;
            r0[r] = r1[r] = 0;
            if (z >= 0 && z < m.nz && y >= 0 && y < m.ny) {
                const long row = ((long)z * m.ny + y) * m.nx;
                r0[r] = bin_start[row + xlo];
                r1[r] = bin_start[row + xhi + 1];
            }
        }
        const double4 pi = sp[k];
        const float4 pif = spf[k];
        double ax = 0.0, ay = 0.0, az = 0.0;
        int q[VQ];
        int nq = 0;
        auto flush = [&]() {
            int t = 0;
            for (; t + 1 < nq; t += 2) {  // two terms in flight
                double c0x, c0y, c0z, c1x, c1y, c1z;
                pair_term_sel_fast(pi, sp[q[t]], pp, c0x, c0y, c0z);
                pair_term_sel_fast(pi, sp[q[t + 1]], pp, c1x, c1y, c1z);
                ax = ax + c0x;
                ay = ay + c0y;
                az = az + c0z;
                ax = ax + c1x;
                ay = ay + c1y;
                az = az + c1z;
            }
            if (t < nq) {
                double cx, cy, cz;
                pair_term_sel_fast(pi, sp[q[t]], pp, cx, cy, cz);
                ax = ax + cx;
                ay = ay + cy;
                az = az + cz;
            }
            nq = 0;
        };
#pragma unroll 1
        for (int r = 0; r < 9; r++) {
#pragma unroll 2
            for (int j = r0[r]; j < r1[r]; j++) {
                if (j != k && pretest_f32(pif, spf[j], pt)) {
                    q[nq++] = j;
                    if (nq == VQ) flush();
                }
            }
        }
        flush();
        const int cell = by_id[k];
        vel[3L * cell] = ax;
        vel[3L * cell + 1] = ay;
        vel[3L * cell + 2] = az;
    }
    pdl_trigger();
}

// Four lanes per cell (fast numerics): lane `sub` of a quad walks rows
// sub, sub + 4, sub + 8 of the cell's 3x3x3 block, the quad adds its partial
// sums with two butterflies.  4x the threads and a quarter of the dependent
// candidate walk of k_velocity_direct.
__global__ void __launch_bounds__(256) k_velocity_quad(int n, MeshDev m,
                                                       const int32_t* __restrict__ bin_start,
                                                       const int32_t* __restrict__ by_id,
                                                       const double4* __restrict__ sp,
                                                       const int* __restrict__ svox,
                                                       PairParamsFast pp, double* __restrict__ vel) {
    pdl_wait();
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int k = (int)(t >> 2), sub = (int)(t & 3);
    double ax = 0.0, ay = 0.0, az = 0.0;
    if (k < n) {  // quad-uniform
        const int v = svox[k];
        const int rest = (int)fdiv((unsigned)v, m.fnx), ix = v - rest * m.nx;
        const int iz = (int)fdiv((unsigned)rest, m.fny), iy = rest - iz * m.ny;
        const int xlo = ix > 0 ? ix - 1 : 0, xhi = ix + 1 < m.nx ? ix + 1 : m.nx - 1;
        int r0[3], r1[3];
#pragma unroll
        for (int u = 0; u < 3; u++) {
            const int r = sub + 4 * u;
            const int z = iz + r / 3 - 1, y = iy + r % 3 - 1;
            r0[u] = r1[u] = 0;
            if (r < 9 && z >= 0 && z < m.nz && y >= 0 && y < m.ny) {
                const long row = ((long)z * m.ny + y) * m.nx;
                r0[u] = bin_start[row + xlo];
                r1[u] = bin_start[row + xhi + 1];
            }
        }
        const double4 pi = sp[k];
#pragma unroll
        for (int u = 0; u < 3; u++) {
            int j = r0[u];
            const int j1 = r1[u];
            for (; j + 1 < j1; j += 2) {
                const double4 pa = sp[j], pb = sp[j + 1];
                double cx, cy, cz;
                if (j != k && pair_in_range_fast(pi, pa, pp, cx, cy, cz)) {
                    ax = ax + cx;
                    ay = ay + cy;
                    az = az + cz;
                }
                if (j + 1 != k && pair_in_range_fast(pi, pb, pp, cx, cy, cz)) {
                    ax = ax + cx;
                    ay = ay + cy;
                    az = az + cz;
                }
            }
            if (j < j1 && j != k) {
                double cx, cy, cz;
                if (pair_in_range_fast(pi, sp[j], pp, cx, cy, cz)) {
                    ax = ax + cx;
                    ay = ay + cy;
                    az = az + cz;
                }
            }
        }
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
        ax = ax + __shfl_xor_sync(0xffffffffu, ax, o);
        ay = ay + __shfl_xor_sync(0xffffffffu, ay, o);
        az = az + __shfl_xor_sync(0xffffffffu, az, o);
    }
    if (k < n && sub < 3) vel[3L * by_id[k] + sub] = sub == 0 ? ax : sub == 1 ? ay : az;
    pdl_trigger();
}

int launch_velocities_fast(cg_ctx* c, int n, const double* pos, const double* radius,
                           const int32_t* voxel, const int32_t* bin_start,
                           const int32_t* bin_cells_by_id, bool gathered, bool quad, double c_r,
                           double c_a, double m_a, double* vel) {
    if (n <= 0) return CG_OK;
    const int T = 256;
    double4* sp = (double4*)c->d_sp;
    if (!gathered)
        CG_LAUNCH(c, K_GATHER, k_gather_fast, (n + T - 1) / T, T, 0, n, bin_cells_by_id, pos, radius,
                  voxel, sp, c->d_svox, c->d_spf);
    const PairParamsFast pp{c_r, c_a, m_a, 1.0 / m_a};
    if (!quad) {
        static const bool compact = [] {
            // measured: config 1 25.3 vs 27.5 us, config 3 175 vs 189 us
            const char* e = std::getenv("CELLGPU_VEL_COMPACT");
            return e ? std::atoi(e) != 0 : true;
        }();
        if (compact)
            CG_LAUNCH(c, K_VELOCITY_DIRECT, k_velocity_compact, (n + T - 1) / T, T, 0, n, c->m,
                      bin_start, bin_cells_by_id, sp, c->d_svox, pp, vel, c->d_spf,
                      pretest_params(c->m, m_a));
        else
            CG_LAUNCH(c, K_VELOCITY_DIRECT, k_velocity_direct, (n + T - 1) / T, T, 0, n, c->m,
                      bin_start, bin_cells_by_id, sp, c->d_svox, pp, vel);
        return CG_OK;
    }
    CG_LAUNCH(c, K_VELOCITY_DIRECT, k_velocity_quad, (int)((4L * n + T - 1) / T), T, 0, n, c->m,
              bin_start, bin_cells_by_id, sp, c->d_svox, pp, vel);
    return CG_OK;
}

int init_cells_kernels(cg_ctx* c) {
    CG_CUDA_CHECK(cudaFuncSetAttribute(k_velocity_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       c->big_smem));
    return CG_OK;
}

int launch_velocities(cg_ctx* c, int n, const double* pos, const double* radius,
                      const int64_t* ids, const int32_t* voxel, const int32_t* bin_start,
                      const int32_t* bin_cells_by_id, const int32_t* nonempty,
                      const int32_t* n_nonempty, double c_r, double c_a, double m_a,
                      double* vel, bool dense) {
    if (n <= 0) return CG_OK;
    const int T = 256;
    double4* sp = (double4*)c->d_sp;
    // Exact velocities: the pre-tested in-range pairs of each cell in id
    // order (k_velocity_exact), or (env CELLGPU_VEL_EXACT=lists) per-voxel
    // id-sorted candidate lists.
    const char* env_lists = std::getenv("CELLGPU_VEL_EXACT");
    const bool lists = env_lists && std::strcmp(env_lists, "lists") == 0;
    // candidates above which a cell is summed by a warp (k_velocity_exact_dense)
    const char* env_dense = std::getenv("CELLGPU_VEL_DENSE_MIN");
    const int dense_min = env_dense ? std::atoi(env_dense) : 64;
    CG_LAUNCH(c, K_GATHER, k_gather, (n + T - 1) / T, T, 0, n, bin_cells_by_id, pos, radius,
              (const long long*)ids, sp, c->d_sid, c->d_sid32, c->d_n_overflow + 2,
              c->d_n_overflow, lists ? nullptr : voxel, c->d_svox, c->d_spf);
    const PairParams pp{c_r, c_a, m_a};
    const int maxq = (int)std::min<long>(c->nvox, n);
    // vel_ctas_per_sm > 0 caps the grids (grid-stride kernels; see cg_ctx).
    const int cap = c->vel_ctas_per_sm > 0 ? c->vel_ctas_per_sm * c->num_sms : 1 << 30;
    if (!lists) {
        if (!voxel)
            CG_LAUNCH(c, K_GATHER, k_slot_voxel, (maxq + T - 1) / T, T, 0, nonempty, n_nonempty,
                      bin_start, maxq, c->d_svox);
        if (!dense) {
            CG_LAUNCH(c, K_VELOCITY, k_velocity_exact<false>, std::min((n + T - 1) / T, cap), T, 0, n,
                      c->m, bin_start, bin_cells_by_id, sp, c->d_sid, c->d_svox, pp, vel,
                      c->d_slot_list, c->d_n_overflow + 1, dense_min, c->d_spf,
                      pretest_params(c->m, m_a));
            return CG_OK;
        }
        CG_LAUNCH(c, K_VELOCITY, k_velocity_exact<true>, std::min((n + T - 1) / T, cap), T, 0, n,
                  c->m, bin_start, bin_cells_by_id, sp, c->d_sid, c->d_svox, pp, vel,
                  c->d_slot_list, c->d_n_overflow + 1, dense_min, c->d_spf,
                  pretest_params(c->m, m_a));
        CG_LAUNCH(c, K_VELOCITY_MID, k_velocity_exact_dense, std::min(c->num_sms * 8, cap), DW * 32,
                  0, c->d_slot_list, c->d_n_overflow + 1, c->m, bin_start, bin_cells_by_id, sp,
                  c->d_sid, c->d_svox, pp, vel, c->d_n_overflow + 2);
        return CG_OK;
    }

    const int lblocks = std::max(1, std::min(std::min((maxq + LIST_WARPS - 1) / LIST_WARPS, c->num_sms * 8), cap));
    CG_LAUNCH(c, K_VELOCITY_LISTS, k_cand_lists, lblocks, LIST_WARPS * 32, 0, c->m, bin_start,
              nonempty, n_nonempty, c->d_sid32, c->d_n_overflow + 2, c->d_cand, c->d_slot_list,
              c->d_mid, c->d_n_overflow + 1);
    CG_LAUNCH(c, K_VELOCITY, k_velocity_cells, std::min((n + 255) / 256, cap), 256, 0, n, c->d_slot_list,
              c->d_cand, bin_cells_by_id, sp, c->d_sid32, pp, vel);
    CG_LAUNCH(c, K_VELOCITY_MID, k_velocity_mid, c->num_sms * 4, VEL_WARPS * 32, 0, c->m,
              bin_start, c->d_mid, c->d_n_overflow + 1, bin_cells_by_id, sp, c->d_sid, pp, vel,
              c->d_overflow, c->d_n_overflow);
    const int big_cap = (c->big_smem - (BIG_T / 32) * VEL_G * VEL_BUF * (int)sizeof(double)) / 16;
    CG_LAUNCH(c, K_VELOCITY_BIG, k_velocity_big, c->num_sms, BIG_T, c->big_smem, c->m, bin_start,
              c->d_overflow, c->d_n_overflow, bin_cells_by_id, sp, c->d_sid, pp, vel, big_cap,
              c->d_flags);
    return CG_OK;
}

// Global voxel z index of each cell (CPython-exact, core.py:77-85) on the
// context's mesh, -1 outside: decides slab ownership for migration.  full:
// the flat voxel index itself (cg_voxel_index).
__global__ void k_voxel_z(int n, const double* __restrict__ pos, MeshDev m, int32_t* __restrict__ out,
                          int full) {
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int v = voxel_of_dev(m, pos[3L * i], pos[3L * i + 1], pos[3L * i + 2]);
    out[i] = v < 0 ? -1 : full ? v : (int)fdiv(fdiv((unsigned)v, m.fnx), m.fny);
    pdl_trigger();  // dependents launch as this grid finishes
}

int launch_voxel_index(cg_ctx* c, int n, const double* pos, int32_t* out, bool full) {
    if (n <= 0) return CG_OK;
    CG_LAUNCH(c, K_VOXEL_Z, k_voxel_z, (n + 255) / 256, 256, 0, n, pos, c->m, out, full ? 1 : 0);
    return CG_OK;
}

int launch_voxel_z(cg_ctx* c, int n, const double* pos, int32_t* out) {
    return launch_voxel_index(c, n, pos, out, false);
}

// ---------------------------------------------------------------- integrate

struct Box {
    double lo[3], hi[3], up[3], org[3];
};

// mechanics.py:236-242 (+ G2 AB2: PhysiCell Cell::update_position).
// mechanics.py:236-242 (+ G2 AB2: PhysiCell Cell::update_position) for cell i;
// the new position is stored and returned in p.
__device__ __forceinline__ void integrate_one(int i, double* __restrict__ pos,
                                              const double* __restrict__ vel,
                                              double* __restrict__ prev_vel, double dt,
                                              int integrator, const Box& b, double* p) {
    p[0] = pos[3L * i];
    p[1] = pos[3L * i + 1];
    p[2] = pos[3L * i + 2];
    const double v[3] = {vel[3L * i], vel[3L * i + 1], vel[3L * i + 2]};
    if (integrator == CG_AB2) {
        const double d1 = dt * 1.5, d2 = dt * -0.5;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const double pv = prev_vel[3L * i + k];
            p[k] = p[k] + (d1 * v[k] + d2 * pv);
            prev_vel[3L * i + k] = v[k];
        }
    } else {
#pragma unroll
        for (int k = 0; k < 3; k++) p[k] = p[k] + dt * v[k];
    }
    // core.py:87-102: contains() half-open; clamp_inside on all axes.
    const bool inside = b.org[0] <= p[0] && p[0] < b.up[0] && b.org[1] <= p[1] &&
                        p[1] < b.up[1] && b.org[2] <= p[2] && p[2] < b.up[2];
    if (!inside) {
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const double t = b.lo[k] > p[k] ? b.lo[k] : p[k];  // max(p, lo)
            p[k] = b.hi[k] < t ? b.hi[k] : t;                  // min(., hi)
        }
    }
    pos[3L * i] = p[0];
    pos[3L * i + 1] = p[1];
    pos[3L * i + 2] = p[2];
}

__global__ void k_integrate(int n, double* __restrict__ pos, const double* __restrict__ vel,
                            double* __restrict__ prev_vel, double dt, int integrator, Box b) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double p[3];
    integrate_one(i, pos, vel, prev_vel, dt, integrator, b, p);
    pdl_trigger();  // dependents launch as this grid finishes
}

// Engine: integration fused with the rebin's voxel keys and histogram
// (mechanics.py:236-242 then core.py:77-85), one pass over the cells.
__global__ void k_integrate_count(int n, double* __restrict__ pos, const double* __restrict__ vel,
                                  double* __restrict__ prev_vel, double dt, int integrator, Box b,
                                  MeshDev m, int32_t* __restrict__ voxel, int* __restrict__ counts,
                                  int* __restrict__ flags, ScanState scan) {
    pdl_wait();
    reset_scan_state(scan);
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double p[3];
    integrate_one(i, pos, vel, prev_vel, dt, integrator, b, p);
    const int v = voxel_of_dev(m, p[0], p[1], p[2]);
    voxel[i] = v;
    if (v < 0) {
        atomicOr(&flags[FLAG_DOMAIN], 1);
        return;
    }
    atomicAdd(&counts[v], 1);
    pdl_trigger();  // dependents launch as this grid finishes
}

int launch_integrate(cg_ctx* c, int n, double* pos, const double* vel, double* prev_vel,
                     double dt, int integrator, int32_t* voxel_for_rebin) {
    if (n <= 0) return CG_OK;
    const MeshDev& m = c->m;
    Box b;
    const double org[3] = {m.ox, m.oy, m.oz};
    const int ns[3] = {m.nx, m.ny, m.nz};
    const double ds[3] = {m.dx, m.dy, m.dz};
    for (int k = 0; k < 3; k++) {
        b.org[k] = org[k];
        b.up[k] = org[k] + ns[k] * ds[k];  // core.py:64-66 upper
        b.lo[k] = org[k] + POSITION_EPS;
        b.hi[k] = b.up[k] - POSITION_EPS;
    }
    const int T = 256;
    if (voxel_for_rebin) {
        CG_LAUNCH(c, K_INTEGRATE, k_integrate_count, (n + T - 1) / T, T, 0, n, pos, vel, prev_vel,
                  dt, integrator, b, c->m, voxel_for_rebin, c->d_counts, c->d_flags,
                  scan_state(c));
    } else {
        CG_LAUNCH(c, K_INTEGRATE, k_integrate, (n + T - 1) / T, T, 0, n, pos, vel, prev_vel, dt,
                  integrator, b);
    }
    return CG_OK;
}
