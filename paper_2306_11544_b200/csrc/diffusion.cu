// LOD diffusion-decay sweeps and the cell secretion/uptake exchange.
//
// Reference: /root/reference/pkg/src/cellbench/diffusion.py
//   _line_factors  :80-99    -> host_line_factors (host, cached per (dt, D, decay))
//   _solve_rows    :102-112  -> solve_line (one line per thread, same op order)
//   lod_step       :127-192  -> launch_lod: per substrate x, y, z sweeps
//   apply_cell_exchange :201-234 -> k_exchange_scalar / fused G4 exchange
//
// Kernel plan (HBM/L2-bound fp64 streaming; one line per thread keeps the
// reference's sequential Thomas recurrence, so results are bit-identical):
//   k_plane_xy : one CTA per (z-plane, substrate).  The whole plane is staged
//                in shared memory with an odd row pitch (conflict-free both
//                along rows and along columns), the fused exchange and the
//                Dirichlet pins are applied in smem, then the x sweep (thread
//                per row) and the y sweep (thread per column) run back to back.
//                16 B of global traffic per voxel-substrate for two sweeps.
//   k_z_cols   : one thread per (x, y) column, 64 consecutive columns per CTA
//                so every z-row access is one coalesced 512 B segment; the
//                column is staged in smem for the back substitution.
//   k_x_rows / k_y_cols : fallback pair when a plane exceeds shared memory
//                (e.g. 256 x 256 x 8 B = 512 KB).

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "lod_common.cuh"


// ---------------------------------------------------------------- host side

void host_line_factors(int n, double r, double lam3, double* inv, double* gamma) {
    if (n == 1) {  // diffusion.py:88-89
        inv[0] = 1.0 / (1.0 + lam3);
        gamma[0] = 0.0;
        return;
    }
    double interior = 1.0 + lam3 + 2.0 * r;  // diffusion.py:90
    double boundary = 1.0 + lam3 + r;        // diffusion.py:91
    inv[0] = 1.0 / boundary;
    gamma[0] = r * inv[0];
    for (int i = 1; i < n; i++) {
        double diag = (i == n - 1) ? boundary : interior;
        inv[i] = 1.0 / (diag - r * gamma[i - 1]);
        gamma[i] = r * inv[i];
    }
}

// Factors of a block of the line matrix (paper_2306_11544_b200/slab.py
// block_factors): the boundary diagonal only where the block touches a
// global end of the line.
void host_block_factors(int n, double r, double lam3, bool top, bool bottom, double* inv,
                        double* gam) {
    if (top && bottom) {
        host_line_factors(n, r, lam3, inv, gam);
        return;
    }
    const double interior = 1.0 + lam3 + 2.0 * r, boundary = 1.0 + lam3 + r;
    std::vector<double> diag(n, interior);
    if (top) diag[0] = boundary;
    if (bottom) diag[n - 1] = boundary;
    inv[0] = 1.0 / diag[0];
    gam[0] = r * inv[0];
    for (int i = 1; i < n; i++) {
        inv[i] = 1.0 / (diag[i] - r * gam[i - 1]);
        gam[i] = r * inv[i];
    }
}

void host_thomas(double* d, int n, const double* inv, const double* gam, double r) {
    d[0] *= inv[0];
    for (int i = 1; i < n; i++) {
        d[i] += r * d[i - 1];
        d[i] *= inv[i];
    }
    for (int i = n - 2; i >= 0; i--) d[i] += gam[i] * d[i + 1];
}

// Spikes of every rank's block (slab.py make_plan): this rank's full v, w
// and the four end values of every rank's v, w.
static int upload_slab_plan(cg_ctx* c, double dt, const double* diffusion, const double* decay) {
    const int P = c->slab_world, S = c->S, nzl = c->m.nz;
    std::vector<double> spk((size_t)S * 2 * nzl, 0.0), ends((size_t)S * P * 4, 0.0);
    for (int s = 0; s < S; s++) {
        const double lam3 = dt * decay[s] / 3.0;
        const double r = dt * diffusion[s] / (c->m.dz * c->m.dz);
        for (int k = 0; k < P; k++) {
            const int z0 = c->slab_starts[k];
            const int m = c->slab_starts[k + 1] - z0;
            const bool top = z0 == 0, bottom = z0 + m == c->nz_global;
            std::vector<double> inv(m), gam(m), v(m, 0.0), w(m, 0.0);
            host_block_factors(m, r, lam3, top, bottom, inv.data(), gam.data());
            if (k > 0) {
                v[0] = r;
                host_thomas(v.data(), m, inv.data(), gam.data(), r);
            }
            if (k < P - 1) {
                w[m - 1] = r;
                host_thomas(w.data(), m, inv.data(), gam.data(), r);
            }
            double* e = &ends[((size_t)s * P + k) * 4];
            e[0] = v[0];
            e[1] = v[m - 1];
            e[2] = w[0];
            e[3] = w[m - 1];
            if (k == c->slab_rank) {
                if (m != nzl) return set_error(CG_DOMAIN, "slab plane count does not match the split");
                std::copy(v.begin(), v.end(), spk.begin() + (size_t)s * 2 * nzl);
                std::copy(w.begin(), w.end(), spk.begin() + (size_t)s * 2 * nzl + nzl);
            }
        }
    }
    CG_CUDA_CHECK(cudaMemcpyAsync(c->d_spk, spk.data(), spk.size() * sizeof(double),
                                  cudaMemcpyHostToDevice, c->stream));
    CG_CUDA_CHECK(cudaMemcpyAsync(c->d_ends, ends.data(), ends.size() * sizeof(double),
                                  cudaMemcpyHostToDevice, c->stream));
    return CG_OK;
}

int ensure_factors(cg_ctx* c, double dt, const double* diffusion, const double* decay) {
    std::vector<double> key;
    key.push_back(dt);
    for (int s = 0; s < c->S; s++) key.push_back(diffusion[s]);
    for (int s = 0; s < c->S; s++) key.push_back(decay[s]);
    if (key == c->fac_key) return CG_OK;
    const int nmax = c->nmax;
    std::vector<double> fac((size_t)c->S * 3 * 2 * nmax, 0.0), rr((size_t)c->S * 3);
    const int ns[3] = {c->m.nx, c->m.ny, c->m.nz};
    const double ds[3] = {c->m.dx, c->m.dy, c->m.dz};
    for (int s = 0; s < c->S; s++) {
        double lam3 = dt * decay[s] / 3.0;  // diffusion.py:144
        for (int a = 0; a < 3; a++) {
            double r = dt * diffusion[s] / (ds[a] * ds[a]);  // diffusion.py:149,157,168
            rr[s * 3 + a] = r;
            double* inv = &fac[((size_t)(s * 3 + a) * 2 + 0) * nmax];
            double* gam = &fac[((size_t)(s * 3 + a) * 2 + 1) * nmax];
            if (a == 2 && c->slab_world > 1)
                host_block_factors(ns[a], r, lam3, c->m.zlo, c->m.zhi, inv, gam);
            else
                host_line_factors(ns[a], r, lam3, inv, gam);
        }
    }
    if (c->slab_world > 1) {
        int st = upload_slab_plan(c, dt, diffusion, decay);
        if (st) return st;
    }
    // Synchronous upload on the context stream: these are tiny and only change
    // when (dt, D, decay) change, never inside a captured step.
    CG_CUDA_CHECK(cudaMemcpyAsync(c->d_fac, fac.data(), fac.size() * sizeof(double),
                                  cudaMemcpyHostToDevice, c->stream));
    CG_CUDA_CHECK(cudaMemcpyAsync(c->d_r, rr.data(), rr.size() * sizeof(double),
                                  cudaMemcpyHostToDevice, c->stream));
    CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    c->h_fac = fac;
    c->h_r = rr;
    c->fac_key = key;
    return CG_OK;
}

static int upload_small(cg_ctx* c, double* dst, const double* src, std::vector<double>& key) {
    std::vector<double> k(src, src + c->S);
    if (k == key) return CG_OK;
    CG_CUDA_CHECK(cudaMemcpyAsync(dst, src, c->S * sizeof(double), cudaMemcpyHostToDevice,
                                  c->stream));
    CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    key = k;
    return CG_OK;
}

int ensure_dirichlet(cg_ctx* c, const double* dirichlet) {
    return upload_small(c, c->d_diri, dirichlet, c->diri_key);
}
int ensure_saturation(cg_ctx* c, const double* saturation) {
    return upload_small(c, c->d_sat, saturation, c->sat_key);
}


// One (z-plane, substrate) item: stage, exchange, Dirichlet, x sweep, y sweep,
// store.  Used by k_plane_xy (one item per CTA).
// Staging uses one TMA bulk copy per row when rows are 16B aligned; the fused
// exchange's index and coefficient loads are issued while the plane is in
// flight, so its global round trips overlap the staging.
// Optional phase probe (tools/plane_probe.cu builds with -DCG_PROBE):
// thread 0 of every CTA records clock64 at phase boundaries.

#ifdef CG_PROBE
__device__ long long g_probe[8 * 1024];
extern "C" int cg_probe_read(long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, g_probe, sizeof(long long) * (size_t)std::min(n, 8 * 1024));
}
#define PROBE_MARK(k) \
    if (threadIdx.x == 0) g_probe[8 * (blockIdx.y * gridDim.x + blockIdx.x) + (k)] = clock64()
#else
#define PROBE_MARK(k)
#endif

// One thread's batch of the fused exchange: XB voxels q = q_first + j *
// blockDim.x.  One round trip loads each voxel's id, slot range and the
// inline {A, D} of its first two cells (ExchArgs::R, written by the bin
// fix-up); voxels with more cells read the rest from the slot arrays.
template <int XB_>
struct XBatch {
    static constexpr int XB = XB_;
    int v[XB], k0[XB], k1[XB];
    double2 r0[XB], r1[XB];
    __device__ __forceinline__ void issue(const ExchArgs& ex, const double* __restrict__ R,
                                          int q_first, int q_end) {
#pragma unroll
        for (int j = 0; j < XB; j++) {
            const int q = q_first + j * (int)blockDim.x;
            v[j] = -1;
            if (q < q_end) {
                v[j] = ex.nonempty[q];
                k0[j] = ex.ne_start[q];
                k1[j] = ex.ne_start[q + 1];
                const double2* rq = reinterpret_cast<const double2*>(R + 2L * kRecCells * q);
                r0[j] = rq[0];
                r1[j] = rq[1];
            }
        }
    }
    template <typename At>
    __device__ __forceinline__ void apply(const double* __restrict__ A,
                                          const double* __restrict__ D, At at) const {
#pragma unroll
        for (int j = 0; j < XB; j++) {
            if (v[j] >= 0) {
                double* cell = at(v[j]);
                double rho = (*cell + r0[j].x) / r0[j].y;
                if (k1[j] - k0[j] > 1) {
                    rho = (rho + r1[j].x) / r1[j].y;
                    for (int k = k0[j] + 2; k < k1[j]; k++) rho = (rho + A[k]) / D[k];
                }
                *cell = rho;
            }
        }
    }
};

// Branch-free select (a plain ?: over a register line compiles to one
// branch per element).
__device__ __forceinline__ double selp(bool p, double a, double b) {
    double r;
    asm("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\nselp.f64 %0, %1, %2, q;\n}"
        : "=d"(r) : "d"(a), "d"(b), "r"((int)p));
    return r;
}

// G1 pins of a register line: both ends, or every element when the whole
// line lies on an outer face.
template <int N>
__device__ __forceinline__ void pin_line(double (&w)[N], bool full, double dv) {
    w[0] = dv;
    w[N - 1] = dv;
#pragma unroll
    for (int i = 1; i < N - 1; i++) w[i] = selp(full, dv, w[i]);
}

// Register-line plane kernel block: one thread per line, at least four warps
// so the staging and exchange phases have enough threads.
template <int N>
__host__ __device__ constexpr int reg_threads() {
    return (N + 31) / 32 * 32 > 128 ? (N + 31) / 32 * 32 : 128;
}

// x then y sweep of one staged N x N plane with register lines, a thread
// per line.  Rows are read and written as 16 B pairs (conflict-free with the
// pitch == 2 mod 4 staging); the y sweep writes its results straight to
// global memory (coalesced along x), so the kernel has no store phase.
template <bool DIRI, int N>
__device__ __forceinline__ void plane_sweeps_reg(double* __restrict__ plane,
                                                 double* __restrict__ g, bool zface, double dv,
                                                 const double* __restrict__ fx,
                                                 const double* __restrict__ fy, double rx,
                                                 double ry) {
    constexpr int P = ((N + 2) & ~1) | 2;
    static_assert(N % 2 == 0, "rows are read in pairs");
    const int t = threadIdx.x;
    if (t < N) {
        double* row = plane + t * P;
        const bool full = zface || t == 0 || t == N - 1;
        double w[N];
#pragma unroll
        for (int i = 0; i < N; i += 2) {
            const double2 v = *reinterpret_cast<const double2*>(row + i);
            w[i] = v.x;
            w[i + 1] = v.y;
        }
        if (DIRI) pin_line<N>(w, full, dv);
        solve_regs_smem<N>(w, fx, fx + N, rx);
        if (DIRI) pin_line<N>(w, full, dv);
#pragma unroll
        for (int i = 0; i < N; i += 2) *reinterpret_cast<double2*>(row + i) = make_double2(w[i], w[i + 1]);
    }
    __syncthreads();
    PROBE_MARK(4);
    if (t < N) {
        const bool full = zface || t == 0 || t == N - 1;
        double w[N];
#pragma unroll
        for (int i = 0; i < N; i++) w[i] = plane[i * P + t];
        solve_regs_smem<N>(w, fy, fy + N, ry);
        if (DIRI) pin_line<N>(w, full, dv);
#pragma unroll
        for (int i = 0; i < N; i++) g[(long)i * N + t] = w[i];
    }
}

// x then y sweep of one staged N x N plane with relay register lines
// (solve_relay): K lanes per line, M = N / K elements each; lanes l and
// l + 32/K hold adjacent segments of line warp * 32/K + l % (32/K).  Same
// staging, pins and direct y store as plane_sweeps_reg.
template <bool DIRI, int M, int K>
__device__ __forceinline__ void plane_sweeps_relay(double* __restrict__ plane,
                                                   double* __restrict__ g, bool zface, double dv,
                                                   const double* __restrict__ fx,
                                                   const double* __restrict__ fy, double rx,
                                                   double ry) {
    constexpr int N = M * K, LPW = 32 / K;
    constexpr int P = ((N + 2) & ~1) | 2;
    static_assert(M % 2 == 0 && N % LPW == 0, "segments are read in pairs; whole warps");
    const int lane = threadIdx.x & 31, seg = lane / LPW, ls = lane % LPW;
    const int line = (threadIdx.x >> 5) * LPW + ls;
    const bool full = zface || line == 0 || line == N - 1;
    const bool first = seg == 0, last = seg == K - 1;
    {
        double* row = plane + line * P + seg * M;
        double w[M];
#pragma unroll
        for (int i = 0; i < M; i += 2) {
            const double2 v = *reinterpret_cast<const double2*>(row + i);
            w[i] = v.x;
            w[i + 1] = v.y;
        }
        if (DIRI) pin_seg<M>(w, full, first, last, dv);
        const double *ix = fx, *gx = fx + N;
        solve_relay<M, K>(w, ix, gx, rx, seg, ls);
        if (DIRI) pin_seg<M>(w, full, first, last, dv);
#pragma unroll
        for (int i = 0; i < M; i += 2) *reinterpret_cast<double2*>(row + i) = make_double2(w[i], w[i + 1]);
    }
    __syncthreads();
    PROBE_MARK(4);
    {
        const double* col = plane + seg * M * P + line;
        double w[M];
#pragma unroll
        for (int i = 0; i < M; i++) w[i] = col[i * P];
        const double *iy = fy, *gy = fy + N;
        solve_relay<M, K>(w, iy, gy, ry, seg, ls);
        if (DIRI) pin_seg<M>(w, full, first, last, dv);
        double* gc = g + (long)seg * M * N + line;
#pragma unroll
        for (int i = 0; i < M; i++) gc[(long)i * N] = w[i];
    }
}

// NL > 0: register lines (nx == ny == NL); NL == 0: streaming line solves.
// Line factors of the x and y sweeps into smem behind the plane (cp.async).
__device__ __forceinline__ void stage_plane_factors(double* __restrict__ sm, const MeshDev& m,
                                                    const double* __restrict__ fac, int nmax,
                                                    int s) {
    const int nx = m.nx, ny = m.ny;
    double* fx = sm + (long)ny * plane_pitch(nx);
    double* fy = fx + 2 * nx;
    const double* facx = fac + (long)(s * 3 + 0) * 2 * nmax;
    const double* facy = fac + (long)(s * 3 + 1) * 2 * nmax;
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
        cp_async8(fx + i, facx + i);
        cp_async8(fx + nx + i, facx + nmax + i);
    }
    for (int i = threadIdx.x; i < ny; i += blockDim.x) {
        cp_async8(fy + i, facy + i);
        cp_async8(fy + ny + i, facy + nmax + i);
    }
}

template <bool EXCH, bool DIRI, int NL = 0, int KR = 1>
__device__ __forceinline__ void plane_body(double* __restrict__ sm, unsigned long long* bar,
                                           unsigned& phase, double* __restrict__ dens,
                                           const MeshDev& m, const double* __restrict__ fac,
                                           const double* __restrict__ rr, int nmax,
                                           const double* __restrict__ diri, const ExchArgs& ex,
                                           int z, int s) {
    const int nx = m.nx, ny = m.ny, P = plane_pitch(nx);
    const long plane_sz = (long)nx * ny;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
    double* plane = sm;
    double* fx = plane + (long)ny * P;  // inv_x[nx], gam_x[nx]
    double* fy = fx + 2 * nx;           // inv_y[ny], gam_y[ny]
    double* g = dens + ((long)s * m.nz + z) * plane_sz;
    PROBE_MARK(0);
    const bool bulk = ((nx * 8) % 16 == 0) && (((unsigned long long)g) % 16 == 0);
    if (bulk) {
        // One bulk copy per row; lane 0 of every warp issues its share (the
        // copies of one warp serialise on the uniform datapath).
        if (t == 0) mbar_expect_tx(bar, (unsigned)(ny * nx * 8));
        __syncthreads();
        if (lane == 0)
            for (int y = wid; y < ny; y += nw) bulk_g2s(plane + y * P, g + (long)y * nx, nx * 8, bar);
    } else {
        for (int y = wid; y < ny; y += nw)
            for (int x = lane; x < nx; x += 32) cp_async8(plane + y * P + x, g + (long)y * nx + x);
    }
    stage_plane_factors(sm, m, fac, nmax, s);
    // Fused exchange, in batches of XB voxels per thread (XBatch); the first
    // batch is issued while the plane is in flight.
    int q0 = 0, q1 = 0;
    const double* A = ex.A + (long)s * ex.n_cells;
    const double* D = ex.D + (long)s * ex.n_cells;
    const double* R = ex.R + 2L * kRecCells * s * ex.rq;
    XBatch<4> xb;
    if (EXCH) {
        q0 = ex.row_ne[z * ny];
        q1 = ex.row_ne[(z + 1) * ny];
        xb.issue(ex, R, q0 + t, q1);
    }
    PROBE_MARK(1);
    cp_async_wait_all();
    if (bulk) {
        mbar_wait(bar, phase);
        phase ^= 1u;
    }
    __syncthreads();
    PROBE_MARK(2);
    if (EXCH) {
        // rho = (rho + A_k) / D_k over the voxel's cells in ascending id
        // (diffusion.py:219-229); cells occupy id-sorted slots [k0, k1).
        const long base = (long)z * plane_sz;
        auto at = [&](int v) {
            const int local = (int)(v - base);
            const int y = local / nx;
            return plane + y * P + (local - y * nx);
        };
        const int step = decltype(xb)::XB * (int)blockDim.x;
        for (int qb = q0 + t;;) {
            xb.apply(A, D, at);
            qb += step;
            if (qb >= q1) break;
            xb.issue(ex, R, qb, q1);
        }
        __syncthreads();
    }
    PROBE_MARK(3);
    // G1 pins (before the x sweep, after x, after y) are applied by the thread
    // that owns each row / column: the union of the rows' (columns') outer-face
    // voxels is the plane's whole outer face, so this equals pinning the plane
    // between the sweeps without extra passes or barriers.
    const double dv = DIRI ? diri[s] : 0.0;
    const bool zface = is_zface(z, m);
    const double rx = rr[s * 3 + 0], ry = rr[s * 3 + 1];
    if constexpr (NL > 0) {
        // (shared-memory factors measured faster than parameter-space ones
        // here: 2 CTAs of different substrates share an SM's constant cache)
        if constexpr (KR > 1)
            plane_sweeps_relay<DIRI, NL / KR, KR>(plane, g, zface, dv, fx, fy, rx, ry);
        else
            plane_sweeps_reg<DIRI, NL>(plane, g, zface, dv, fx, fy, rx, ry);
    } else {
        for (int y = t; y < ny; y += blockDim.x) {
            double* row = plane + y * P;
            const bool full = zface || y == 0 || y == ny - 1;
            if (DIRI) {
                if (full) for (int x = 0; x < nx; x++) row[x] = dv;
                else { row[0] = dv; row[nx - 1] = dv; }
            }
            solve_line(row, 1, nx, fx, fx + nx, rx);
            if (DIRI) {
                if (full) for (int x = 0; x < nx; x++) row[x] = dv;
                else { row[0] = dv; row[nx - 1] = dv; }
            }
        }
        __syncthreads();
        PROBE_MARK(4);
        for (int x = t; x < nx; x += blockDim.x) {
            double* col = plane + x;
            solve_line(col, P, ny, fy, fy + ny, ry);
            if (DIRI) {
                if (zface || x == 0 || x == nx - 1) for (int y = 0; y < ny; y++) col[y * P] = dv;
                else { col[0] = dv; col[(ny - 1) * P] = dv; }
            }
        }
        __syncthreads();
    }
    PROBE_MARK(5);
    if constexpr (NL > 0) {
        // stored by the y sweep
    } else if (bulk) {
        fence_proxy_async_smem();
        __syncthreads();
        if (lane == 0) {
            for (int y = wid; y < ny; y += nw) bulk_s2g(g + (long)y * nx, plane + y * P, nx * 8);
            bulk_commit_wait_read();
        }
    } else {
        for (int y = wid; y < ny; y += nw)
            for (int x = lane; x < nx; x += 32) g[(long)y * nx + x] = plane[y * P + x];
    }
    __syncthreads();  // the staging buffer is reused by the next item
    PROBE_MARK(6);
}

template <bool EXCH, bool DIRI>
__global__ void __launch_bounds__(256) k_plane_xy(double* __restrict__ dens, MeshDev m,
                                                  const double* __restrict__ fac,
                                                  const double* __restrict__ rr, int nmax,
                                                  const double* __restrict__ diri, ExchArgs ex) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    pdl_trigger();
    extern __shared__ double sm[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    unsigned phase = 0;
    plane_body<EXCH, DIRI>(sm, &bar, phase, dens, m, fac, rr, nmax, diri, ex, blockIdx.x,
                           blockIdx.y);
}

// Register-line variant (exact; nx == ny == NL).
template <bool EXCH, bool DIRI, int NL>
__global__ void __launch_bounds__(reg_threads<NL>(), 2) k_plane_xy_reg(
    double* __restrict__ dens, MeshDev m, const double* __restrict__ fac,
    const double* __restrict__ rr, int nmax, const double* __restrict__ diri, ExchArgs ex) {
    extern __shared__ double sm[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    // (staging the factors before the PDL wait measured slower: 8.3 vs 7.8 us)
    __syncthreads();
    pdl_wait();
    unsigned phase = 0;
    plane_body<EXCH, DIRI, NL>(
        sm, &bar, phase, dens, m, fac, rr, nmax, diri, ex, blockIdx.x, blockIdx.y);
    pdl_trigger();  // the z kernel may launch while the last planes finish
}

// Relay variant for lines longer than a thread's registers (nx == ny == NL,
// KR lanes per line; exchange as its own kernel).
template <bool DIRI, int NL, int KR>
__global__ void __launch_bounds__(NL * KR, 1) k_plane_xy_relay(
    double* __restrict__ dens, MeshDev m, const double* __restrict__ fac,
    const double* __restrict__ rr, int nmax, const double* __restrict__ diri, ExchArgs ex) {
    extern __shared__ double sm[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    pdl_wait();
    unsigned phase = 0;
    plane_body<false, DIRI, NL, KR>(
        sm, &bar, phase, dens, m, fac, rr, nmax, diri, ex, blockIdx.x, blockIdx.y);
    pdl_trigger();
}

// Fallback x sweep: RX consecutive rows (z*ny + y) per CTA, thread per row.
template <bool EXCH, bool DIRI>
__global__ void __launch_bounds__(128) k_x_rows(double* __restrict__ dens, MeshDev m,
                                                const double* __restrict__ fac,
                                                const double* __restrict__ rr, int nmax,
                                                const double* __restrict__ diri, ExchArgs ex) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    pdl_trigger();
    extern __shared__ double sm[];
    const int nx = m.nx, P = nx | 1, RX = blockDim.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const long nrows = (long)m.ny * m.nz;
    const long row0 = (long)blockIdx.x * RX;
    const int rows = (int)min((long)RX, nrows - row0);
    const int s = blockIdx.y;
    double* tile = sm;
    double* fx = tile + (long)RX * P;
    double* g = dens + (long)s * nrows * nx + row0 * nx;
    for (int r = wid; r < rows; r += nw)
        for (int x = lane; x < nx; x += 32) cp_async8(tile + r * P + x, g + (long)r * nx + x);
    const double* facx = fac + (long)(s * 3 + 0) * 2 * nmax;
    for (int i = threadIdx.x; i < nx; i += RX) {
        cp_async8(fx + i, facx + i);
        cp_async8(fx + nx + i, facx + nmax + i);
    }
    cp_async_wait_all();
    __syncthreads();
    if (EXCH) {
        const long lo = row0 * nx;
        exchange_tile(ex.row_ne[row0], ex.row_ne[row0 + rows], ex.nonempty, ex.ne_start,
                      ex.A + (long)s * ex.n_cells, ex.D + (long)s * ex.n_cells, [&](int v) {
                          const int local = (int)(v - lo);
                          const int r = local / nx;
                          return tile + r * P + (local - r * nx);
                      });
        __syncthreads();
    }
    const int r = threadIdx.x;
    if (r < rows) {
        double* row = tile + r * P;
        const long grow = row0 + r;
        const int y = (int)(grow % m.ny), z = (int)(grow / m.ny);
        const bool full = DIRI && (y == 0 || y == m.ny - 1 || is_zface(z, m));
        if (DIRI) {
            const double dv = diri[s];
            if (full) for (int x = 0; x < nx; x++) row[x] = dv;
            else { row[0] = dv; row[nx - 1] = dv; }
        }
        solve_line(row, 1, nx, fx, fx + nx, rr[s * 3 + 0]);
        if (DIRI) {
            const double dv = diri[s];
            if (full) for (int x = 0; x < nx; x++) row[x] = dv;
            else { row[0] = dv; row[nx - 1] = dv; }
        }
    }
    __syncthreads();
    for (int rr2 = wid; rr2 < rows; rr2 += nw)
        for (int x = lane; x < nx; x += 32) g[(long)rr2 * nx + x] = tile[rr2 * P + x];
}

// y sweep (fallback) and z sweep: one thread per line, TC consecutive lines
// per tile whose elements are contiguous in memory for a fixed position along
// the sweep axis.  Column tile staged as col[i][TC] (conflict-free).
//   AXIS 1 (y): lines indexed by (z, x); element i at z*nx*ny + i*nx + x.
//   AXIS 2 (z): lines indexed by p = y*nx + x; element i at i*nx*ny + p.
// Threads >= TC only help with staging.  Used by k_cols.
template <int AXIS, bool DIRI>
__device__ __forceinline__ void cols_body(double* __restrict__ sm, unsigned long long* bar,
                                          unsigned& phase, double* __restrict__ dens,
                                          const MeshDev& m, const double* __restrict__ fac,
                                          const double* __restrict__ rr, int nmax,
                                          const double* __restrict__ diri, int tile, int s,
                                          int TC) {
    const int n = AXIS == 1 ? m.ny : m.nz;
    const long plane_sz = (long)m.nx * m.ny;
    double* inv = sm + (long)n * TC;
    double* gam = inv + n;
    const double* f = fac + (long)(s * 3 + AXIS) * 2 * nmax;
    const int t = threadIdx.x;
    long base0;  // first line of the tile
    long st;
    int valid_lines;
    if (AXIS == 1) {
        const int tiles_x = (m.nx + TC - 1) / TC;
        const int z = tile / tiles_x;
        const int x0 = (tile - z * tiles_x) * TC;
        valid_lines = min(TC, m.nx - x0);
        base0 = (long)z * plane_sz + x0;
        st = m.nx;
    } else {
        const long p0 = (long)tile * TC;
        valid_lines = (int)min((long)TC, plane_sz - p0);
        base0 = p0;
        st = plane_sz;
    }
    double* g0 = dens + (long)s * plane_sz * m.nz + base0;
    // Whole tile in bounds and every row segment 16B aligned: each of the n
    // rows (TC contiguous doubles) is one TMA bulk copy, issued by warp 0.
    const bool bulk = valid_lines == TC && ((st * 8) % 16 == 0) && (((unsigned long long)g0) % 16 == 0) &&
                      ((TC * 8) % 16 == 0);
    const int lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
    if (bulk) {
        if (t == 0) mbar_expect_tx(bar, (unsigned)(n * TC * 8));
        __syncthreads();
        if (lane == 0)
            for (int i = wid; i < n; i += nw) bulk_g2s(sm + i * TC, g0 + i * st, TC * 8, bar);
    } else {
        for (int i = t >> 5; i < n; i += blockDim.x >> 5)
            for (int l = t & 31; l < valid_lines; l += 32) cp_async8(sm + i * TC + l, g0 + i * st + l);
    }
    for (int i = t; i < n; i += blockDim.x) {
        cp_async8(inv + i, f + i);
        cp_async8(gam + i, f + nmax + i);
    }
    cp_async_wait_all();
    if (bulk) {
        mbar_wait(bar, phase);
        phase ^= 1u;
    }
    __syncthreads();
    if (t < valid_lines) {
        double* col = sm + t;
        solve_line(col, TC, n, inv, gam, rr[s * 3 + AXIS]);
        // Partitioned z sweep: pins follow the interface correction instead.
        if (DIRI && !(AXIS == 2 && m.slab)) {
            const double dv = diri[s];
            // Element i of this line sits at (x, i, z) for AXIS 1, (x, y, i) for AXIS 2.
            bool full;
            if (AXIS == 1) {
                const int z = (int)(base0 / plane_sz);
                const int x = (int)(base0 - (long)z * plane_sz) + t;
                full = x == 0 || x == m.nx - 1 || is_zface(z, m);
            } else {
                const long p = base0 + t;
                const int y = (int)(p / m.nx), x = (int)(p - (long)y * m.nx);
                full = x == 0 || x == m.nx - 1 || y == 0 || y == m.ny - 1;
            }
            if (full) {
                for (int i = 0; i < n; i++) col[i * TC] = dv;
            } else {
                col[0] = dv;
                col[(n - 1) * TC] = dv;
            }
        }
    }
    if (bulk) {
        fence_proxy_async_smem();  // generic-proxy smem writes -> async-proxy reads
        __syncthreads();
        if (lane == 0) {
            for (int i = wid; i < n; i += nw) bulk_s2g(g0 + i * st, sm + i * TC, TC * 8);
            bulk_commit_wait_read();
        }
    } else {
        __syncthreads();
        for (int i = t >> 5; i < n; i += blockDim.x >> 5)
            for (int l = t & 31; l < valid_lines; l += 32) g0[i * st + l] = sm[i * TC + l];
    }
    __syncthreads();  // the staging buffer is reused by the next item
}

template <int AXIS, bool DIRI>
__global__ void __launch_bounds__(256) k_cols(double* __restrict__ dens, MeshDev m,
                                              const double* __restrict__ fac,
                                              const double* __restrict__ rr, int nmax,
                                              const double* __restrict__ diri, int TC) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    pdl_trigger();
    extern __shared__ double sm[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    unsigned phase = 0;
    cols_body<AXIS, DIRI>(sm, &bar, phase, dens, m, fac, rr, nmax, diri, blockIdx.x, blockIdx.y, TC);
}

// z sweep with register lines on an N^3 mesh: thread per (x, y) column, read
// straight from global (lanes = consecutive columns: every z step is one
// coalesced 256 B warp access), solved in registers, written back.  Slab
// contexts skip the pins (the interface correction applies them).
// check_state's test: finite and non-negative (NaN fails both compares).
__device__ __forceinline__ bool field_value_ok(double v) { return v >= 0.0 && v <= 0x1.fffffffffffffp+1023; }

template <int N>
__device__ __forceinline__ void check_values(const double (&w)[N], int* __restrict__ flags) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < N; i++) ok = ok && field_value_ok(w[i]);
    if (!ok) atomicOr(&flags[FLAG_NUMERIC], 1);
}

// Standalone check_state over n values (cg_check_state; the engine's
// streaming-kernel path).
__global__ void k_check_field(const double* __restrict__ d, long n, int* __restrict__ flags) {
    pdl_wait();
    bool ok = true;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        ok = ok && field_value_ok(d[i]);
    if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) atomicOr(&flags[FLAG_NUMERIC], 1);
    pdl_trigger();
}

int launch_check_field(cg_ctx* c, const double* d, long n) {
    if (n <= 0) return CG_OK;
    const int T = 256;
    const int G = (int)std::min<long>((n + T - 1) / T, (long)c->num_sms * 8);
    CG_LAUNCH(c, K_CHECK_STATE, k_check_field, G, T, 0, d, n, c->d_flags);
    return CG_OK;
}

template <bool DIRI, int N, int SI>
__device__ __forceinline__ void zcol_reg(double* __restrict__ dens, const MeshDev& m,
                                         const double* __restrict__ diri,
                                         const LineFactors<N>& lf, int p, int* __restrict__ chk) {
    constexpr long PS = (long)N * N;
    double* col = dens + (long)SI * N * PS + p;
    double w[N];
#pragma unroll
    for (int i = 0; i < N; i++) w[i] = col[i * PS];
    solve_regs<N>(w, lf.inv[SI][2], lf.gam[SI][2], lf.r[SI][2]);
    if (DIRI && !m.slab) {
        const int y = p / N, x = p - y * N;
        pin_line<N>(w, x == 0 || x == N - 1 || y == 0 || y == N - 1, diri[SI]);
    }
    if (chk) check_values<N>(w, chk);
#pragma unroll
    for (int i = 0; i < N; i++) col[i * PS] = w[i];
}

// chk != nullptr (last substep of a step): also Microenvironment.check_state
// on the final values (core.py:142-144) -> FLAG_NUMERIC.
template <bool DIRI, int N>
__global__ void __launch_bounds__(64, 1) k_zcols_reg(double* __restrict__ dens, MeshDev m,
                                                     const double* __restrict__ diri,
                                                     const __grid_constant__ LineFactors<N> lf,
                                                     int* __restrict__ chk) {
    pdl_wait();
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < N * N) {
        switch (blockIdx.y) {
            case 0: zcol_reg<DIRI, N, 0>(dens, m, diri, lf, p, chk); break;
            case 1: zcol_reg<DIRI, N, 1>(dens, m, diri, lf, p, chk); break;
            case 2: zcol_reg<DIRI, N, 2>(dens, m, diri, lf, p, chk); break;
            default: zcol_reg<DIRI, N, 3>(dens, m, diri, lf, p, chk); break;
        }
    }
    pdl_trigger();  // the next kernel may launch while the last columns finish
}

// z sweep with relay register lines on an NL^3 mesh (NL too long for one
// thread): KR lanes per (x, y) column, lanes l and l + 32/KR holding adjacent
// z segments of column warp * 32/KR + l % (32/KR); every z step of a segment
// is a coalesced 128 B half-warp access (KR = 2).
template <bool DIRI, int NL, int KR, int SI>
__device__ __forceinline__ void zcol_relay(double* __restrict__ dens, const MeshDev& m,
                                           const double* __restrict__ diri,
                                           const LineFactors<NL>& lf, int p, int seg, int ls,
                                           int* __restrict__ chk) {
    constexpr int M = NL / KR;
    constexpr long PS = (long)NL * NL;
    double* col = dens + (long)SI * NL * PS + (long)seg * M * PS + p;
    double w[M];
#pragma unroll
    for (int i = 0; i < M; i++) w[i] = col[i * PS];
    solve_relay<M, KR>(w, lf.inv[SI][2], lf.gam[SI][2], lf.r[SI][2], seg, ls);
    if (DIRI && !m.slab) {
        const int y = p / NL, x = p - y * NL;
        pin_seg<M>(w, x == 0 || x == NL - 1 || y == 0 || y == NL - 1, seg == 0, seg == KR - 1, diri[SI]);
    }
    if (chk) check_values<M>(w, chk);
#pragma unroll
    for (int i = 0; i < M; i++) col[i * PS] = w[i];
}

template <bool DIRI, int NL, int KR>
__global__ void __launch_bounds__(128) k_zcols_relay(double* __restrict__ dens, MeshDev m,
                                                     const double* __restrict__ diri,
                                                     const __grid_constant__ LineFactors<NL> lf,
                                                     int* __restrict__ chk) {
    pdl_wait();
    constexpr int LPW = 32 / KR;
    const int lane = threadIdx.x & 31, seg = lane / LPW, ls = lane % LPW;
    const int p = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * LPW + ls;
    if (p - ls < NL * NL) {  // warp-uniform: NL * NL is a multiple of LPW
        switch (blockIdx.y) {
            case 0: zcol_relay<DIRI, NL, KR, 0>(dens, m, diri, lf, p, seg, ls, chk); break;
            case 1: zcol_relay<DIRI, NL, KR, 1>(dens, m, diri, lf, p, seg, ls, chk); break;
            case 2: zcol_relay<DIRI, NL, KR, 2>(dens, m, diri, lf, p, seg, ls, chk); break;
            default: zcol_relay<DIRI, NL, KR, 3>(dens, m, diri, lf, p, seg, ls, chk); break;
        }
    }
    pdl_trigger();
}

// z sweep with register lines for a compile-time line length NZ and any
// plane size (e.g. config 4's 256 x 256 x 32 slabs): thread per column,
// loads and stores coalesced across lanes, factors as a kernel parameter.
template <int NZ>
struct ZFactors {
    double inv[kLineMaxS][NZ];
    double gam[kLineMaxS][NZ];
    double r[kLineMaxS];
};

template <bool DIRI, int NZ, int SI>
__device__ __forceinline__ void zcol_nz(double* __restrict__ dens, const MeshDev& m,
                                        const double* __restrict__ diri, const ZFactors<NZ>& zf,
                                        long p, long ps) {
    double* col = dens + (long)SI * NZ * ps + p;
    double w[NZ];
#pragma unroll
    for (int i = 0; i < NZ; i++) w[i] = col[i * ps];
    solve_regs<NZ>(w, zf.inv[SI], zf.gam[SI], zf.r[SI]);
    if (DIRI && !m.slab) {
        const int y = (int)(p / m.nx), x = (int)(p - (long)y * m.nx);
        pin_line<NZ>(w, x == 0 || x == m.nx - 1 || y == 0 || y == m.ny - 1, diri[SI]);
    }
#pragma unroll
    for (int i = 0; i < NZ; i++) col[i * ps] = w[i];
}

template <bool DIRI, int NZ>
__global__ void __launch_bounds__(128) k_zcols_nz(double* __restrict__ dens, MeshDev m,
                                                  const double* __restrict__ diri,
                                                  const __grid_constant__ ZFactors<NZ> zf) {
    pdl_wait();
    pdl_trigger();
    const long ps = (long)m.nx * m.ny;
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= ps) return;
    switch (blockIdx.y) {
        case 0: zcol_nz<DIRI, NZ, 0>(dens, m, diri, zf, p, ps); break;
        case 1: zcol_nz<DIRI, NZ, 1>(dens, m, diri, zf, p, ps); break;
        case 2: zcol_nz<DIRI, NZ, 2>(dens, m, diri, zf, p, ps); break;
        default: zcol_nz<DIRI, NZ, 3>(dens, m, diri, zf, p, ps); break;
    }
}


static size_t plane_smem_bytes(const MeshDev& m) {
    const int P = plane_pitch(m.nx);
    return ((size_t)m.ny * P + 2 * (size_t)m.nx + 2 * (size_t)m.ny) * sizeof(double);
}
static size_t cols_smem_bytes(int n, int TC) { return ((size_t)n * TC + 2 * (size_t)n) * sizeof(double); }
static const size_t kSmemLimit = 227 * 1024 - 1024;

template <typename Kern>
static int set_max_smem(Kern kernel) {
    CG_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kSmemLimit));
    return CG_OK;
}

template <int N>
static void fill_line_factors(const cg_ctx* c, LineFactors<N>& f, int s0, int ns) {
    std::memset(&f, 0, sizeof f);
    for (int j = 0; j < ns && j < kLineMaxS; j++)
        for (int a = 0; a < 3; a++) {
            const int s = s0 + j;
            const double* inv = &c->h_fac[((size_t)(s * 3 + a) * 2 + 0) * c->nmax];
            const double* gam = &c->h_fac[((size_t)(s * 3 + a) * 2 + 1) * c->nmax];
            for (int i = 0; i < N; i++) {
                f.inv[j][a][i] = inv[i];
                f.gam[j][a][i] = gam[i];
            }
            f.r[j][a] = c->h_r[s * 3 + a];
        }
}

// parts: bit 0 = x/y sweeps (+ fused exchange), bit 1 = z sweep.  NL > 0:
// register-line kernels (cubic NL^3 mesh), else the streaming kernels.
template <bool EXCH, bool DIRI, int NL = 0>
static int launch_lod_t(cg_ctx* c, double* dens, const ExchArgs& ex, int parts, bool check) {
    const MeshDev& m = c->m;
    const int P = m.nx | 1;
    const size_t plane_smem = plane_smem_bytes(m);
    const int S = c->S;
    static DeviceFlags attrs;  // per instantiation and device
    if (!attrs.test_and_set(c->device)) {
        int st;
        if ((st = set_max_smem(k_plane_xy<EXCH, DIRI>)) || (st = set_max_smem(k_x_rows<EXCH, DIRI>)) ||
            (st = set_max_smem(k_cols<1, DIRI>)) || (st = set_max_smem(k_cols<2, DIRI>)))
            return st;
        if constexpr (NL > 0)
            if ((st = set_max_smem(k_plane_xy_reg<EXCH, DIRI, NL>))) return st;
    }
    const long plane_sz = (long)m.nx * m.ny;
    if constexpr (NL > 0) {
        // substrate window [s0, s0 + ns) (c->sub_n > 0: one engine chain per substrate)
        const int s0 = c->sub_n > 0 ? c->sub0 : 0, ns = c->sub_n > 0 ? c->sub_n : S;
        if (EXCH && s0 != 0) return set_error(CG_STATE, "substrate window with the fused exchange");
        static thread_local LineFactors<NL> lf;  // host staging of the kernel parameter
        fill_line_factors(c, lf, s0, ns);
        double* d = dens + (long)s0 * c->nvox;
        if (parts & 1)
            CG_LAUNCH(c, K_PLANE_XY, (k_plane_xy_reg<EXCH, DIRI, NL>), dim3(m.nz, ns),
                      reg_threads<NL>(), plane_smem, d, m, c->d_fac + (size_t)s0 * 6 * c->nmax,
                      c->d_r + 3 * s0, c->nmax, c->d_diri + s0, ex);
        if (parts & 2)
            CG_LAUNCH(c, K_Z_COLS, (k_zcols_reg<DIRI, NL>), dim3((unsigned)((plane_sz + 63) / 64), ns),
                      64, 0, d, m, c->d_diri + s0, lf, check ? c->d_flags : nullptr);
        return CG_OK;
    }
    // substrate windows: the register-line kernels above, and the z sweep
    // alone (parts == 2: the slab driver's per-substrate pipeline)
    const bool window = c->sub_n > 0 && (c->sub0 != 0 || c->sub_n != S);
    if (window && (parts & 1))
        return set_error(CG_STATE, "substrate windows need the register-line kernels");
    const int w0 = window ? c->sub0 : 0, wn = window ? c->sub_n : S;
    if (!(parts & 1)) {
    } else if (plane_smem <= kSmemLimit) {
        // The sweeps use max(nx, ny) threads; staging and Dirichlet use all
        // of plane_threads.
        CG_LAUNCH(c, K_PLANE_XY, (k_plane_xy<EXCH, DIRI>), dim3(m.nz, S), c->plane_threads,
                  plane_smem, dens, m, c->d_fac, c->d_r, c->nmax, c->d_diri, ex);
    } else {
        const int RX = 32;
        const size_t xs = ((size_t)RX * P + 2 * (size_t)m.nx) * sizeof(double);
        const long nrows = (long)m.ny * m.nz;
        CG_LAUNCH(c, K_X_ROWS, (k_x_rows<EXCH, DIRI>), dim3((unsigned)((nrows + RX - 1) / RX), S),
                  RX, xs, dens, m, c->d_fac, c->d_r, c->nmax, c->d_diri, ex);
        const int TC = 64;
        const int tiles_x = (m.nx + TC - 1) / TC;
        CG_LAUNCH(c, K_Y_COLS, (k_cols<1, DIRI>), dim3(tiles_x * m.nz, S), 256,
                  cols_smem_bytes(m.ny, TC), dens, m, c->d_fac, c->d_r, c->nmax, c->d_diri, TC);
    }
    if (!(parts & 2)) return CG_OK;
    double* dz = dens + (long)w0 * c->nvox;
    if (c->reg_lines && m.nz == 32 && S <= kLineMaxS) {
        static thread_local ZFactors<32> zf;  // host staging of the kernel parameter
        std::memset(&zf, 0, sizeof zf);
        for (int j = 0; j < wn; j++) {
            const int s = w0 + j;
            for (int i = 0; i < 32; i++) {
                zf.inv[j][i] = c->h_fac[((size_t)(s * 3 + 2) * 2 + 0) * c->nmax + i];
                zf.gam[j][i] = c->h_fac[((size_t)(s * 3 + 2) * 2 + 1) * c->nmax + i];
            }
            zf.r[j] = c->h_r[s * 3 + 2];
        }
        CG_LAUNCH(c, K_Z_COLS, (k_zcols_nz<DIRI, 32>), dim3((unsigned)((plane_sz + 127) / 128), wn),
                  128, 0, dz, m, c->d_diri + w0, zf);
        return check ? launch_check_field(c, dz, (long)wn * c->nvox) : CG_OK;
    }
    const int TC = 64;
    // 64 lines per tile, 256 threads: the extra warps only stage (measured
    // 8.4 vs 10.2 us per launch at config 1, tools/launch_probe.cu)
    CG_LAUNCH(c, K_Z_COLS, (k_cols<2, DIRI>), dim3((unsigned)((plane_sz + TC - 1) / TC), wn), 256,
              cols_smem_bytes(m.nz, TC), dz, m, c->d_fac + (size_t)w0 * 6 * c->nmax, c->d_r + 3 * w0,
              c->nmax, c->d_diri + w0, TC);
    return check ? launch_check_field(c, dz, (long)wn * c->nvox) : CG_OK;
}

// Relay register lines (NL^3 mesh, no fused exchange): KP lanes per line in
// the plane kernel, KR in the z kernel.  Registers are split over the four
// SM sub-partitions: a CTA of W warps puts ceil(W / 4) on one, so a thread
// may hold at most 16384 / (32 ceil(W / 4)) registers -- 160 lines x 2 lanes
// (10 warps) would cap it at 168 and spill 200-280 B of the 80-element
// segments; 4 lanes of 40 (20 warps, cap 96) still spill 64 B
// (<0, 160, 4>) / 80 B (<1, 160, 4>) at 96 registers (ptxas -v) -- the
// least of the layouts tried.  The z kernel (4 warps per CTA) keeps 2 x 80
// at 246 registers, i.e. 2 CTAs of 128 threads per SM.
template <bool DIRI, int NL, int KP, int KR>
static int launch_lod_relay(cg_ctx* c, double* dens, int parts, bool check) {
    static_assert((NL * NL) % (32 / KR) == 0, "whole warps of columns");
    const MeshDev& m = c->m;
    static DeviceFlags attrs;  // per instantiation and device
    if (!attrs.test_and_set(c->device)) {
        int st;
        if ((st = set_max_smem(k_plane_xy_relay<DIRI, NL, KP>))) return st;
    }
    const int s0 = c->sub_n > 0 ? c->sub0 : 0, ns = c->sub_n > 0 ? c->sub_n : c->S;
    static thread_local LineFactors<NL> lf;  // host staging of the kernel parameter
    fill_line_factors(c, lf, s0, ns);
    double* d = dens + (long)s0 * c->nvox;
    const ExchArgs ex{};
    if (parts & 1)
        CG_LAUNCH(c, K_PLANE_XY, (k_plane_xy_relay<DIRI, NL, KP>), dim3(m.nz, ns), NL * KP,
                  plane_smem_bytes(m), d, m, c->d_fac + (size_t)s0 * 6 * c->nmax, c->d_r + 3 * s0,
                  c->nmax, c->d_diri + s0, ex);
    if (parts & 2) {
        const long threads = (long)NL * NL * KR;
        CG_LAUNCH(c, K_Z_COLS, (k_zcols_relay<DIRI, NL, KR>), dim3((unsigned)((threads + 127) / 128), ns),
                  128, 0, d, m, c->d_diri + s0, lf, check ? c->d_flags : nullptr);
    }
    return CG_OK;
}

template <int NL = 0>
static int launch_lod_k(cg_ctx* c, double* dens, bool e, bool di, const ExchArgs& ex, int parts,
                        bool check) {
    if (e && di) return launch_lod_t<true, true, NL>(c, dens, ex, parts, check);
    if (e) return launch_lod_t<true, false, NL>(c, dens, ex, parts, check);
    if (di) return launch_lod_t<false, true, NL>(c, dens, ex, parts, check);
    return launch_lod_t<false, false, NL>(c, dens, ex, parts, check);
}

// Register lines for the cubic meshes of the BASELINE configs (160: relay
// lines, 2 lanes per line; every line
// length a compile-time constant); other meshes stream through smem.
int reg_line_length(const cg_ctx* c) {
    const MeshDev& m = c->m;
    if (!c->reg_lines || c->S > kLineMaxS || m.nx != m.ny || m.ny != m.nz) return 0;
    return (m.nx == 20 || m.nx == 80 || m.nx == 160) ? m.nx : 0;
}

// Own kernel by default (S <= 4): with one CTA per plane the fused exchange
// serialises its divisions on 8 warps per SM (config 3: 53.6k of 100k cycles
// per plane, tools/plane_phases.py), while k_exchange_rec spreads them over
// the whole GPU (config 3 step 4.07 -> 3.77 ms).  The streaming meshes gain
// most: config 4 (256 x 256 x 32, x-row kernel) 2.94 vs 7.68 ms per step
// exact, 2.35 vs 7.21 fast (the fused row kernel spends 679 us per substep
// on divisions); config 1 8.4 + 5.8 vs 20-22 us per substep.
// The price is memory: the rotating exchange sets hold 2 more copies of the
// per-slot A/D (S x cells doubles each) and records.
bool lod_exchange_split(const cg_ctx* c) {
    return c->exch_split >= 0 ? c->exch_split != 0 : c->S <= kLineMaxS;
}

int launch_lod(cg_ctx* c, double* dens, int bc, const int32_t* nonempty, const double* exA,
               const double* exD, int n_cells, int parts, bool check) {
    const ExchArgs ex{nonempty, c->d_ne_start, c->d_row_ne, exA, exD, n_cells, c->d_exR,
                      (int)std::min<long>(c->nvox, c->cap_cells)};
    const bool e = exA != nullptr;
    const bool di = bc == CG_BC_DIRICHLET;
    switch (reg_line_length(c)) {
        case 20: return launch_lod_k<20>(c, dens, e, di, ex, parts, check);
        case 80: return launch_lod_k<80>(c, dens, e, di, ex, parts, check);
        case 160:  // relay lines (the fused exchange streams)
            if (e) return launch_lod_k<0>(c, dens, e, di, ex, parts, check);
            return di ? launch_lod_relay<true, 160, 4, 2>(c, dens, parts, check)
                      : launch_lod_relay<false, 160, 4, 2>(c, dens, parts, check);
        default: return launch_lod_k<0>(c, dens, e, di, ex, parts, check);
    }
}



// ---------------------------------------------------------------- z slabs

// Per (substrate, line): this rank's local solution y at its first and last
// plane -> send[s][2][L], the payload of the all-gather.
__global__ void k_zslab_pack(const double* __restrict__ dens, MeshDev m, int S,
                             double* __restrict__ send) {
    pdl_wait();
    pdl_trigger();
    const long L = (long)m.nx * m.ny;
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= L) return;
    const double* g = dens + (long)s * L * m.nz + p;
    send[((long)s * 2 + 0) * L + p] = g[0];
    send[((long)s * 2 + 1) * L + p] = g[(long)(m.nz - 1) * L];
}

// Reduced 2x2 block-tridiagonal interface system over the ranks (slab.py
// solve_interfaces, same operation order), then x = y + l_{k-1} v + f_{k+1} w
// along the local line and the line's Dirichlet pins.
template <bool DIRI>
__global__ void k_zslab_correct(double* __restrict__ dens, MeshDev m, int S, int world, int rank,
                                const double* __restrict__ recv, const double* __restrict__ ends,
                                const double* __restrict__ spk, const double* __restrict__ diri) {
    pdl_wait();
    pdl_trigger();
    const long L = (long)m.nx * m.ny;
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= L) return;
    double G0[32], G1[32], H0[32], H1[32];
    for (int k = 0; k < world; k++) {
        const double* e = ends + ((long)s * world + k) * 4;
        const double v0 = e[0], v1 = e[1], w0 = e[2], w1 = e[3];
        const double y0 = recv[(((long)k * S + s) * 2 + 0) * L + p];
        const double y1 = recv[(((long)k * S + s) * 2 + 1) * L + p];
        double a00, a10, b0, b1;
        if (k == 0) {
            a00 = 1.0;
            a10 = 0.0;
            b0 = y0;
            b1 = y1;
        } else {
            const double g1 = G1[k - 1], h1 = H1[k - 1];
            a00 = 1.0 + v0 * g1;
            a10 = v1 * g1;
            b0 = y0 + v0 * h1;
            b1 = y1 + v1 * h1;
        }
        H0[k] = b0 / a00;
        H1[k] = b1 - a10 * H0[k];  // / a11 with a11 == 1
        G0[k] = (-w0) / a00;
        G1[k] = (-w1) - a10 * G0[k];
    }
    double zf = H0[world - 1], zl = H1[world - 1];
    double left = 0.0, right = 0.0;
    if (rank == world - 2) right = zf;
    for (int k = world - 2; k >= 0; k--) {
        const double f = H0[k] - G0[k] * zf;
        const double l = H1[k] - G1[k] * zf;
        if (k == rank - 1) left = l;
        if (k == rank + 1) right = f;
        zf = f;
        zl = l;
    }
    (void)zl;
    double* g = dens + (long)s * L * m.nz + p;
    const double* v = spk + (long)s * 2 * m.nz;
    const double* w = v + m.nz;
    const int x = (int)(p % m.nx), y = (int)(p / m.nx);
    const bool full = DIRI && (x == 0 || x == m.nx - 1 || y == 0 || y == m.ny - 1);
    const double dv = DIRI ? diri[s] : 0.0;
    for (int i = 0; i < m.nz; i++) {
        double t = g[(long)i * L];
        t = t + left * v[i];
        t = t + right * w[i];
        if (DIRI && (full || (i == 0 && m.zlo) || (i == m.nz - 1 && m.zhi))) t = dv;
        g[(long)i * L] = t;
    }
}

// ---- the interface system by line blocks (all-to-all variant)
//
// Instead of every rank gathering every rank's end values for every line
// (all-gather: (P - 1) S 2 L doubles received per rank) and solving all L
// reduced systems redundantly, rank r owns the line block
// [r Lb, (r + 1) Lb) (Lb = ceil(L / P)): one all-to-all brings it every
// rank's end values for its block, it solves those Lb systems (the same
// operations as k_zslab_correct) and a second all-to-all returns to each rank
// k its two correction coefficients (l_{k-1}, f_{k+1}) for the block's lines
// -- 2 (P - 1) / P S 2 L doubles received per rank instead of (P - 1) S 2 L,
// 4x less at P = 8, bit-identical fields.

// send[r][s][2][Lb]: this rank's (y[0], y[m-1]) of line r Lb + j.
__global__ void k_zslab_pack_blocks(const double* __restrict__ dens, MeshDev m, int S, int world,
                                    long Lb, double* __restrict__ send) {
    pdl_wait();
    pdl_trigger();
    const long L = (long)m.nx * m.ny;
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= L) return;
    const long r = p / Lb, j = p - r * Lb;
    const double* g = dens + (long)s * L * m.nz + p;
    double* o = send + ((r * S + s) * 2) * Lb + j;
    o[0] = g[0];
    o[Lb] = g[(long)(m.nz - 1) * L];
}

// recv[k][s][2][Lb]: rank k's end values for this rank's block; out[k][s][2][Lb]:
// (left, right) = (l_{k-1}, f_{k+1}) of rank k for the block's lines.
__global__ void k_zslab_reduce_blocks(MeshDev m, int S, int world, int rank, long Lb,
                                      const double* __restrict__ recv,
                                      const double* __restrict__ ends, double* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const long L = (long)m.nx * m.ny;
    const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (j >= Lb || (long)rank * Lb + j >= L) return;
    double G0[32], G1[32], H0[32], H1[32];
    for (int k = 0; k < world; k++) {
        const double* e = ends + ((long)s * world + k) * 4;
        const double v0 = e[0], v1 = e[1], w0 = e[2], w1 = e[3];
        const double y0 = recv[(((long)k * S + s) * 2 + 0) * Lb + j];
        const double y1 = recv[(((long)k * S + s) * 2 + 1) * Lb + j];
        double a00, a10, b0, b1;
        if (k == 0) {
            a00 = 1.0;
            a10 = 0.0;
            b0 = y0;
            b1 = y1;
        } else {
            const double g1 = G1[k - 1], h1 = H1[k - 1];
            a00 = 1.0 + v0 * g1;
            a10 = v1 * g1;
            b0 = y0 + v0 * h1;
            b1 = y1 + v1 * h1;
        }
        H0[k] = b0 / a00;
        H1[k] = b1 - a10 * H0[k];
        G0[k] = (-w0) / a00;
        G1[k] = (-w1) - a10 * G0[k];
    }
    // Z_k = (f_k, l_k) backward; rank k's left = l_{k-1}, right = f_{k+1}
    double f = H0[world - 1], l = H1[world - 1];
    double* o = out + (((long)(world - 1) * S + s) * 2) * Lb + j;
    o[Lb] = 0.0;  // the last rank has no right neighbour
    double fn = f;  // f_{k+1} for rank k
    for (int k = world - 2; k >= 0; k--) {
        const double fk = H0[k] - G0[k] * fn;
        const double lk = H1[k] - G1[k] * fn;
        // rank k + 1's left is l_k; rank k's right is f_{k+1}
        out[(((long)(k + 1) * S + s) * 2 + 0) * Lb + j] = lk;
        out[(((long)k * S + s) * 2 + 1) * Lb + j] = fn;
        fn = fk;
    }
    out[(((long)0 * S + s) * 2 + 0) * Lb + j] = 0.0;  // the first rank has no left neighbour
    (void)l;
}

// The all-gather variant's reduced solve to per-line (left, right) of this
// rank in the line-block layout (world, S, 2, Lb) -- what the deferred
// correction (cg_zslab_defer) reads.  Same operations as k_zslab_correct.
__global__ void k_zslab_lr_gather(MeshDev m, int S, int world, int rank, long Lb,
                                  const double* __restrict__ recv, const double* __restrict__ ends,
                                  double* __restrict__ lr) {
    pdl_wait();
    pdl_trigger();
    const long L = (long)m.nx * m.ny;
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= L) return;
    double G0[32], G1[32], H0[32], H1[32];
    for (int k = 0; k < world; k++) {
        const double* e = ends + ((long)s * world + k) * 4;
        const double v0 = e[0], v1 = e[1], w0 = e[2], w1 = e[3];
        const double y0 = recv[(((long)k * S + s) * 2 + 0) * L + p];
        const double y1 = recv[(((long)k * S + s) * 2 + 1) * L + p];
        double a00, a10, b0, b1;
        if (k == 0) {
            a00 = 1.0;
            a10 = 0.0;
            b0 = y0;
            b1 = y1;
        } else {
            const double g1 = G1[k - 1], h1 = H1[k - 1];
            a00 = 1.0 + v0 * g1;
            a10 = v1 * g1;
            b0 = y0 + v0 * h1;
            b1 = y1 + v1 * h1;
        }
        H0[k] = b0 / a00;
        H1[k] = b1 - a10 * H0[k];
        G0[k] = (-w0) / a00;
        G1[k] = (-w1) - a10 * G0[k];
    }
    double zf = H0[world - 1];
    double left = 0.0, right = 0.0;
    if (rank == world - 2) right = zf;
    for (int k = world - 2; k >= 0; k--) {
        const double f = H0[k] - G0[k] * zf;
        const double l = H1[k] - G1[k] * zf;
        if (k == rank - 1) left = l;
        if (k == rank + 1) right = f;
        zf = f;
    }
    const long r = p / Lb, j = p - r * Lb;
    double* o = lr + ((r * S + s) * 2) * Lb + j;
    o[0] = left;
    o[Lb] = right;
}

// x = y + left v + right w along the local line, with (left, right) of line
// p from lr[p / Lb][s][2][p % Lb], and the line's Dirichlet pins.
template <bool DIRI>
__global__ void k_zslab_correct_lr(double* __restrict__ dens, MeshDev m, int S, long Lb,
                                   const double* __restrict__ lr, const double* __restrict__ spk,
                                   const double* __restrict__ diri) {
    pdl_wait();
    pdl_trigger();
    const long L = (long)m.nx * m.ny;
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    if (p >= L) return;
    const long r = p / Lb, j = p - r * Lb;
    const double* c = lr + ((r * S + s) * 2) * Lb + j;
    const double left = c[0], right = c[Lb];
    double* g = dens + (long)s * L * m.nz + p;
    const double* v = spk + (long)s * 2 * m.nz;
    const double* w = v + m.nz;
    const int x = (int)(p % m.nx), y = (int)(p / m.nx);
    const bool full = DIRI && (x == 0 || x == m.nx - 1 || y == 0 || y == m.ny - 1);
    const double dv = DIRI ? diri[s] : 0.0;
    for (int i = 0; i < m.nz; i++) {
        double t = g[(long)i * L];
        t = t + left * v[i];
        t = t + right * w[i];
        if (DIRI && (full || (i == 0 && m.zlo) || (i == m.nz - 1 && m.zhi))) t = dv;
        g[(long)i * L] = t;
    }
}

// Substrate window of the z-slab calls (c->sub0 / sub_n; all when sub_n == 0):
// the kernels see window-relative substrates, the buffers hold ns substrates.
struct ZWin {
    int s0, ns;
};
static ZWin zwin(const cg_ctx* c) {
    return c->sub_n > 0 ? ZWin{c->sub0, c->sub_n} : ZWin{0, c->S};
}

long zslab_block_lines(const cg_ctx* c) {
    const long L = (long)c->m.nx * c->m.ny;
    return (L + c->slab_world - 1) / c->slab_world;
}

int launch_zslab_pack_blocks(cg_ctx* c, const double* dens, double* send) {
    const long L = (long)c->m.nx * c->m.ny;
    const ZWin w = zwin(c);
    CG_LAUNCH(c, K_ZSLAB_PACK, k_zslab_pack_blocks, dim3((unsigned)((L + 255) / 256), w.ns), 256, 0,
              dens + (long)w.s0 * c->nvox, c->m, w.ns, c->slab_world, zslab_block_lines(c), send);
    return CG_OK;
}

int launch_zslab_lr_gather(cg_ctx* c, const double* recv, double* lr) {
    const long L = (long)c->m.nx * c->m.ny;
    const ZWin w = zwin(c);
    CG_LAUNCH(c, K_ZSLAB_CORRECT, k_zslab_lr_gather, dim3((unsigned)((L + 127) / 128), w.ns), 128, 0,
              c->m, w.ns, c->slab_world, c->slab_rank, zslab_block_lines(c), recv,
              c->d_ends + (size_t)w.s0 * c->slab_world * 4, lr);
    return CG_OK;
}

int launch_zslab_reduce_blocks(cg_ctx* c, const double* recv, double* out) {
    const long Lb = zslab_block_lines(c);
    const ZWin w = zwin(c);
    CG_LAUNCH(c, K_ZSLAB_CORRECT, k_zslab_reduce_blocks, dim3((unsigned)((Lb + 127) / 128), w.ns), 128,
              0, c->m, w.ns, c->slab_world, c->slab_rank, Lb, recv,
              c->d_ends + (size_t)w.s0 * c->slab_world * 4, out);
    return CG_OK;
}

int launch_zslab_correct_lr(cg_ctx* c, double* dens, const double* lr, int bc) {
    const long L = (long)c->m.nx * c->m.ny;
    const ZWin w = zwin(c);
    const dim3 grid((unsigned)((L + 255) / 256), w.ns);
    double* d = dens + (long)w.s0 * c->nvox;
    const double* spk = c->d_spk + (size_t)w.s0 * 2 * c->m.nz;
    if (bc == CG_BC_DIRICHLET)
        CG_LAUNCH(c, K_ZSLAB_CORRECT, k_zslab_correct_lr<true>, grid, 256, 0, d, c->m, w.ns,
                  zslab_block_lines(c), lr, spk, c->d_diri + w.s0);
    else
        CG_LAUNCH(c, K_ZSLAB_CORRECT, k_zslab_correct_lr<false>, grid, 256, 0, d, c->m, w.ns,
                  zslab_block_lines(c), lr, spk, c->d_diri + w.s0);
    return CG_OK;
}

int launch_zslab_pack(cg_ctx* c, const double* dens, double* send) {
    const long L = (long)c->m.nx * c->m.ny;
    const ZWin w = zwin(c);
    CG_LAUNCH(c, K_ZSLAB_PACK, k_zslab_pack, dim3((unsigned)((L + 255) / 256), w.ns), 256, 0,
              dens + (long)w.s0 * c->nvox, c->m, w.ns, send);
    return CG_OK;
}

int launch_zslab_correct(cg_ctx* c, double* dens, const double* recv, int bc) {
    const long L = (long)c->m.nx * c->m.ny;
    const ZWin w = zwin(c);
    const dim3 grid((unsigned)((L + 255) / 256), w.ns);
    double* d = dens + (long)w.s0 * c->nvox;
    const double* ends = c->d_ends + (size_t)w.s0 * c->slab_world * 4;
    const double* spk = c->d_spk + (size_t)w.s0 * 2 * c->m.nz;
    if (bc == CG_BC_DIRICHLET)
        CG_LAUNCH(c, K_ZSLAB_CORRECT, k_zslab_correct<true>, grid, 256, 0, d, c->m, w.ns,
                  c->slab_world, c->slab_rank, recv, ends, spk, c->d_diri + w.s0);
    else
        CG_LAUNCH(c, K_ZSLAB_CORRECT, k_zslab_correct<false>, grid, 256, 0, d, c->m, w.ns,
                  c->slab_world, c->slab_rank, recv, ends, spk, c->d_diri + w.s0);
    return CG_OK;
}

// compute_gradients (diffusion.py:237-278): per substrate and voxel,
// (d[+1] - d[-1]) * (0.5 / spacing) on each axis, zero on the axis's faces
// (the interior ranges of the reference's slices; axes of <= 2 voxels have
// none).  Thread per voxel, x fastest: every neighbour load is coalesced.
__global__ void k_gradients(const double* __restrict__ dens, MeshDev m, long nvox, double sx,
                            double sy, double sz, double* __restrict__ grad) {
    pdl_wait();
    pdl_trigger();
    const long v = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nvox) return;
    const int s = blockIdx.y;
    const int rest = (int)fdiv((unsigned)v, m.fnx), x = (int)v - rest * m.nx;
    const int z = (int)fdiv((unsigned)rest, m.fny), y = rest - z * m.ny;
    const long ps = (long)m.nx * m.ny;
    const double* d = dens + (long)s * nvox + v;
    double gx = 0.0, gy = 0.0, gz = 0.0;
    if (x > 0 && x < m.nx - 1) gx = (d[1] - d[-1]) * sx;
    if (y > 0 && y < m.ny - 1) gy = (d[m.nx] - d[-m.nx]) * sy;
    if (z > 0 && z < m.nz - 1) gz = (d[ps] - d[-ps]) * sz;
    double* g = grad + ((long)s * nvox + v) * 3;
    g[0] = gx;
    g[1] = gy;
    g[2] = gz;
}

int launch_gradients(cg_ctx* c, const double* dens, double* grad) {
    if (c->S == 0 || c->nvox == 0) return CG_OK;
    const MeshDev& m = c->m;
    // the reference's sx = 0.5 / mesh.dx etc. (diffusion.py:246)
    const double sx = 0.5 / m.dx, sy = 0.5 / m.dy, sz = 0.5 / m.dz;
    const int T = 256;
    CG_LAUNCH(c, K_GRADIENTS, k_gradients, dim3((unsigned)((c->nvox + T - 1) / T), c->S), T, 0,
              dens, m, c->nvox, sx, sy, sz, grad);
    return CG_OK;
}

// ---------------------------------------------------------------- exchange

// diffusion.py:219-229 for one substrate with the reference's scalar rates:
//   f = dt*vol*inv_vol; den = 1 + f*(s+u); rho = (rho + f*s*rho_sat)/den.
__global__ void k_exchange_scalar(double* __restrict__ dens_s, const int32_t* __restrict__ nonempty,
                                  const int32_t* __restrict__ n_nonempty,
                                  const int32_t* __restrict__ bin_start,
                                  const int32_t* __restrict__ by_id,
                                  const double* __restrict__ volume, double dt, double inv_vol,
                                  double sec, double upt, double sat, int* __restrict__ flags) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    pdl_trigger();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= *n_nonempty) return;
    const int v = nonempty[q];
    double rho = dens_s[v];
    for (int k = bin_start[v]; k < bin_start[v + 1]; k++) {
        const double f = dt * volume[by_id[k]] * inv_vol;
        const double den = 1.0 + f * (sec + upt);
        if (den <= 0.0) {
            atomicOr(&flags[FLAG_DOMAIN], 1);
            return;
        }
        rho = (rho + f * sec * sat) / den;
    }
    dens_s[v] = rho;
}

int launch_exchange_scalar(cg_ctx* c, double* dens_s, double dt, double sec, double upt,
                           double sat, int n_cells, const double* volume,
                           const int32_t* bin_start, const int32_t* bin_cells_by_id,
                           const int32_t* nonempty, const int32_t* n_nonempty) {
    if (n_cells <= 0) return CG_OK;
    const double inv_vol = 1.0 / (c->m.dx * c->m.dy * c->m.dz);  // diffusion.py:214
    const int maxq = (int)std::min<long>(c->nvox, n_cells);
    const int T = 256;
    CG_LAUNCH(c, K_EXCHANGE, k_exchange_scalar, (maxq + T - 1) / T, T, 0, dens_s, nonempty,
              n_nonempty, bin_start, bin_cells_by_id, volume, dt, inv_vol, sec, upt, sat,
              c->d_flags);
    return CG_OK;
}

// G4 coefficients per cell slot k (id-sorted bin order) and substrate s:
//   A = (f*sec)*sat, D = 1 + f*(sec+upt), f = dt*vol*inv_vol  -- the exact
//   subexpressions of diffusion.py:224-228, hoisted out of the substep loop
//   because cells do not move between mechanics steps.
__global__ void k_exchange_coef(int n, int S, double dt, double inv_vol,
                                const double* __restrict__ secretion,
                                const double* __restrict__ uptake,
                                const double* __restrict__ sat,
                                const double* __restrict__ volume,
                                const int32_t* __restrict__ by_id, double* __restrict__ A,
                                double* __restrict__ D, int* __restrict__ flags) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    pdl_trigger();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int cidx = by_id[k];
    const double f = dt * volume[cidx] * inv_vol;
    for (int s = 0; s < S; s++) {
        const double sec = secretion[(long)s * n + cidx];
        const double upt = uptake[(long)s * n + cidx];
        const double den = 1.0 + f * (sec + upt);
        if (den <= 0.0) atomicOr(&flags[FLAG_DOMAIN], 1);
        A[(long)s * n + k] = f * sec * sat[s];
        D[(long)s * n + k] = den;
    }
}

int launch_exchange_coef(cg_ctx* c, double dt, const double* secretion, const double* uptake,
                         int n_cells, const double* volume, const int32_t* bin_cells_by_id) {
    if (n_cells <= 0) return CG_OK;
    const double inv_vol = 1.0 / (c->m.dx * c->m.dy * c->m.dz);
    const int T = 256;
    CG_LAUNCH(c, K_EXCHANGE_COEF, k_exchange_coef, (n_cells + T - 1) / T, T, 0, n_cells, c->S,
              dt, inv_vol, secretion, uptake, c->d_sat, volume, bin_cells_by_id, c->d_exA,
              c->d_exD, c->d_flags);
    return CG_OK;
}

// Standalone G4 exchange (API call): thread per non-empty voxel, all substrates.
__global__ void k_exchange_apply(double* __restrict__ dens, long nvox, int S, int n,
                                 const int32_t* __restrict__ nonempty,
                                 const int32_t* __restrict__ n_nonempty,
                                 const int32_t* __restrict__ bin_start,
                                 const double* __restrict__ A, const double* __restrict__ D) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    pdl_trigger();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= *n_nonempty) return;
    const int v = nonempty[q];
    const int k0 = bin_start[v], k1 = bin_start[v + 1];
    for (int s = 0; s < S; s++) {
        double rho = dens[(long)s * nvox + v];
        for (int k = k0; k < k1; k++) rho = (rho + A[(long)s * n + k]) / D[(long)s * n + k];
        dens[(long)s * nvox + v] = rho;
    }
}

// Engine variant: the cell range of non-empty voxel q is [ne_start[q],
// ne_start[q+1]) (written by the same rebin), so all of a thread's loads are
// independent of each other and issue in one round trip.
__global__ void __launch_bounds__(256) k_exchange_ne(double* __restrict__ dens, long nvox, int S,
                                                     int n, const int32_t* __restrict__ nonempty,
                                                     const int32_t* __restrict__ n_nonempty,
                                                     const int32_t* __restrict__ ne_start,
                                                     const double* __restrict__ A,
                                                     const double* __restrict__ D) {
    pdl_wait();  // programmatic dependent launch: predecessors complete
    pdl_trigger();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= *n_nonempty) return;
    const int v = nonempty[q];
    const int k0 = ne_start[q], k1 = ne_start[q + 1];
#pragma unroll 4
    for (int s = 0; s < S; s++) {
        const double* As = A + (long)s * n;
        const double* Ds = D + (long)s * n;
        double rho = (dens[(long)s * nvox + v] + As[k0]) / Ds[k0];
        for (int k = k0 + 1; k < k1; k++) rho = (rho + As[k]) / Ds[k];
        dens[(long)s * nvox + v] = rho;
    }
}

// Standalone G4 exchange for the step engine: thread per non-empty voxel,
// every substrate.  Slot range and the inline records of the first
// kRecCells cells load in one round trip (independent of the voxel id), the
// densities in a second; the substrates' division chains are independent.
// Voxels with more cells continue from the slot arrays.
template <int SMAX>
__global__ void __launch_bounds__(256) k_exchange_rec(double* __restrict__ dens, long nvox, int S,
                                                      int n, int rq, int maxq,
                                                      const int32_t* __restrict__ nonempty,
                                                      const int32_t* __restrict__ n_nonempty,
                                                      const int32_t* __restrict__ ne_start,
                                                      const double* __restrict__ R,
                                                      const double* __restrict__ A,
                                                      const double* __restrict__ D,
                                                      int early) {
    // early: the list, offsets and records were written at least two launches
    // back (substeps >= 1), so they load before the wait for the previous
    // kernel and only the densities wait for it.
    if (!early) pdl_wait();
    // The count, the voxel id and its slot range load in one round trip
    // (q < maxq keeps every index inside its array; entries past the count
    // are stale and dropped), the records and densities in a second.
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= maxq) return;
    const int nne = *n_nonempty;
    const int v = nonempty[q];
    const int k0 = ne_start[q], k1 = ne_start[q + 1];
    if (q >= nne) return;
    const int nc = k1 - k0;
    double2 r[SMAX][kRecCells];
    double rho[SMAX];
#pragma unroll
    for (int s = 0; s < SMAX; s++) {
        if (s < S) {
            const double2* rp = reinterpret_cast<const double2*>(R + ((long)s * rq + q) * (2 * kRecCells));
#pragma unroll
            for (int c = 0; c < kRecCells; c++)
                if (c < nc) r[s][c] = rp[c];
        }
    }
    if (early) pdl_wait();
#pragma unroll
    for (int s = 0; s < SMAX; s++)
        if (s < S) rho[s] = dens[(long)s * nvox + v];
#pragma unroll
    for (int s = 0; s < SMAX; s++) {
        if (s < S) {
            double x = rho[s];
#pragma unroll
            for (int c = 0; c < kRecCells; c++)
                if (c < nc) x = (x + r[s][c].x) / r[s][c].y;
            if (nc > kRecCells) {
                const double* As = A + (long)s * n;
                const double* Ds = D + (long)s * n;
                for (int k = k0 + kRecCells; k < k1; k++) x = (x + As[k]) / Ds[k];
            }
            dens[(long)s * nvox + v] = x;
        }
    }
    pdl_trigger();  // (early-returning threads count as exited)
}

int launch_exchange_rec(cg_ctx* c, double* dens, int n_cells, const int32_t* nonempty,
                        const int32_t* n_nonempty, const ExchSet* xs, bool early) {
    if (n_cells <= 0 || c->S == 0) return CG_OK;
    const int maxq = (int)std::min<long>(c->nvox, n_cells);
    const int rq = (int)std::min<long>(c->nvox, c->cap_cells);
    const int T = 256;
    if (xs && c->S > 4) return set_error(CG_STATE, "exchange sets need S <= 4");
    if (c->S <= 4) {
        // substrate window [s0, s0 + ns) (one engine chain per substrate)
        const int s0 = c->sub_n > 0 ? c->sub0 : 0, ns = c->sub_n > 0 ? c->sub_n : c->S;
        const double* R = xs ? xs->R : c->d_exR;
        const double* A = xs ? xs->A : c->d_exA;
        const double* D = xs ? xs->D : c->d_exD;
        CG_LAUNCH(c, K_EXCHANGE_APPLY, k_exchange_rec<4>, (maxq + T - 1) / T, T, 0,
                  dens + (long)s0 * c->nvox, c->nvox, ns, n_cells, rq, maxq,
                  xs ? xs->vox : nonempty, xs ? xs->n : n_nonempty, xs ? xs->start : c->d_ne_start,
                  R + (size_t)s0 * rq * 2 * kRecCells, A + (size_t)s0 * n_cells,
                  D + (size_t)s0 * n_cells, early ? 1 : 0);
        return CG_OK;
    }
    if (c->sub_n > 0 && (c->sub0 != 0 || c->sub_n != c->S))
        return set_error(CG_STATE, "substrate windows need S <= 4");
    return launch_exchange_ne(c, dens, n_cells, nonempty, n_nonempty);
}

int launch_exchange_ne(cg_ctx* c, double* dens, int n_cells, const int32_t* nonempty,
                       const int32_t* n_nonempty) {
    if (n_cells <= 0) return CG_OK;
    const int maxq = (int)std::min<long>(c->nvox, n_cells);
    const int T = 256;
    CG_LAUNCH(c, K_EXCHANGE_APPLY, k_exchange_ne, (maxq + T - 1) / T, T, 0, dens, c->nvox, c->S,
              n_cells, nonempty, n_nonempty, c->d_ne_start, c->d_exA, c->d_exD);
    return CG_OK;
}

int launch_exchange_apply(cg_ctx* c, double* dens, int n_cells, const int32_t* bin_start,
                          const int32_t* nonempty, const int32_t* n_nonempty) {
    if (n_cells <= 0) return CG_OK;
    const int maxq = (int)std::min<long>(c->nvox, n_cells);
    const int T = 256;
    CG_LAUNCH(c, K_EXCHANGE_APPLY, k_exchange_apply, (maxq + T - 1) / T, T, 0, dens, c->nvox,
              c->S, n_cells, nonempty, n_nonempty, bin_start, c->d_exA, c->d_exD);
    return CG_OK;
}
