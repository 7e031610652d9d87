// Fast numerics (CG_NUMERICS_FAST): the LOD sweeps as segmented line solves
// and the cell exchange as one affine map per (voxel, substrate), held to
// BASELINE.json's field tolerance (1e-10 relative per step) instead of the
// reference's bit-exact operation order (diffusion.py:102-112, :219-229).
// The exact kernels (diffusion.cu) stay the default; the engine selects these
// with cg_step_params.numerics = CG_NUMERICS_FAST.
//
// Segmented Thomas solve.  The reference's elimination (diffusion.py:102-112)
//   forward   p_0 = d_0 inv_0,   p_i = (d_i + r p_{i-1}) inv_i
//   backward  x_{n-1} = p_{n-1}, x_i = p_i + gam_i x_{i+1}
// is a pair of first-order linear recurrences whose coefficients (a_i =
// r inv_i and gam_i) depend only on the position along the line.  A line of
// N = K*M elements is held by K lanes of one warp, M consecutive elements
// each.  Every lane runs both recurrences over its own segment with a zero
// carry-in (L_i, U_i); the segments' end values are exchanged with warp
// shuffles and the K-1 carries folded (P_{k+1} = L_end(k) + cf_end(k) P_k,
// X_k = U_start(k+1) + cb_start(k+1) X_{k+1}); then every element is fixed up
// independently,
//   p_i = L_i + cf_i P,   x_i = U_i + cb_i X,
//   cf_i = prod_{j=start(i)}^{i} r inv_j,   cb_i = prod_{j=i}^{end(i)} gam_j
// (host-precomputed in long double).  The dependent chain of a sweep drops
// from ~2N steps to ~2M + 2(K-1); the extra rounding is a few ulp per element
// (|r inv_j| < 1, |gam_j| < 1: the carries contract).  Segment 0's forward
// values and the last segment's backward values are the exact recurrence.
//
// Exchange.  The cells of a voxel do not move during the substeps, so the
// exchange of a voxel, rho -> (...((rho + A_1)/D_1 + A_2)/D_2 ...) over its
// cells in ascending id (diffusion.py:219-229), is one affine map
// rho -> alpha rho + beta, alpha = prod 1/D_k, beta = the same composition
// applied to 0.  The rebin's bin fix-up (cells.cu k_bin_fix_g) builds (alpha,
// beta) per (substrate, non-empty voxel) once per mechanics step, while it
// computes the cells' A/D in ascending id anyway (off the substeps' critical
// path, beside them with the rotating exchange sets); the plane kernel
// applies them to its staged plane before the x sweep -- no exchange launch.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "lod_common.cuh"

// ---------------------------------------------------------------- host side

namespace {

// Factor arrays of the segmented solves per (substrate, axis), kSegArr x
// nmax doubles: inv, gam, cf, cb, then (V_i, cb_i) interleaved (2 nmax) with
// V = U(cf), the backward recurrence of cf within each segment (solve_seg2).
constexpr int kSegArr = 6;

// cf/cb/V of one line for segments of M elements (the last may be shorter).
void seg_products(int n, int M, double r, const double* inv, const double* gam, double* cf,
                  double* cb, double* vc) {
    for (int s0 = 0; s0 < n; s0 += M) {
        const int s1 = std::min(n, s0 + M) - 1;
        std::vector<long double> cfl(n);
        long double acc = 1.0L;
        for (int i = s0; i <= s1; i++) {
            acc *= (long double)r * (long double)inv[i];
            cfl[i] = acc;
            cf[i] = (double)acc;
        }
        acc = 1.0L;
        for (int i = s1; i >= s0; i--) {
            acc *= (long double)gam[i];
            cb[i] = (double)acc;
        }
        long double v = cfl[s1];
        vc[2 * s1] = (double)v;
        for (int i = s1 - 1; i >= s0; i--) {
            v = cfl[i] + (long double)gam[i] * v;
            vc[2 * i] = (double)v;
        }
        for (int i = s0; i <= s1; i++) vc[2 * i + 1] = cb[i];
    }
}

// Segments per line of the plane (x/y) and z kernels for line length N
// (env CELLGPU_SEG_KP / CELLGPU_SEG_KZ for A/B runs).
int seg_k(int N, bool plane) {
    const char* env = std::getenv(plane ? "CELLGPU_SEG_KP" : "CELLGPU_SEG_KZ");
    const int k = env ? std::atoi(env) : 0;
    if (N == 80) return (k == 2 || k == 4 || k == 8) ? k : 4;
    if (N == 160) return plane ? 4 : ((k == 4 || k == 8) ? k : 4);
    return 1;
}

// d_segf[((s * 3 + axis) * kSegArr + {inv, gam, cf, cb, (V, cb) pairs}) * nmax + i]
int ensure_seg_factors(cg_ctx* c, int mp, int mz) {
    std::vector<double> key = c->fac_key;
    key.push_back(mp);
    key.push_back(mz);
    if (key == c->segf_key) return CG_OK;
    const int S = c->S, nmax = c->nmax;
    const int ns[3] = {c->m.nx, c->m.ny, c->m.nz}, ms[3] = {mp, mp, mz};
    std::vector<double> f((size_t)S * 3 * kSegArr * nmax, 0.0);
    for (int s = 0; s < S; s++)
        for (int a = 0; a < 3; a++) {
            const double* inv = &c->h_fac[((size_t)(s * 3 + a) * 2 + 0) * nmax];
            const double* gam = &c->h_fac[((size_t)(s * 3 + a) * 2 + 1) * nmax];
            double* o = &f[(size_t)(s * 3 + a) * kSegArr * nmax];
            std::copy(inv, inv + ns[a], o);
            std::copy(gam, gam + ns[a], o + nmax);
            seg_products(ns[a], ms[a], c->h_r[s * 3 + a], inv, gam, o + 2 * nmax, o + 3 * nmax,
                         o + 4 * nmax);
        }
    if (!c->d_segf) CG_CUDA_CHECK(cudaMalloc((void**)&c->d_segf, f.size() * sizeof(double)));
    CG_CUDA_CHECK(cudaMemcpyAsync(c->d_segf, f.data(), f.size() * sizeof(double),
                                  cudaMemcpyHostToDevice, c->stream));
    CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    c->h_segf = f;
    c->segf_key = key;
    return CG_OK;
}

}  // namespace

int seg_line_length(const cg_ctx* c) {
    const MeshDev& m = c->m;
    if (!c->reg_lines || c->S < 1 || c->S > kLineMaxS || m.slab) return 0;
    if (m.nx != m.ny || m.ny != m.nz || m.dx != m.dy || m.dy != m.dz) return 0;
    return (m.nx == 80 || m.nx == 160) ? m.nx : 0;
}

// Meshes whose planes are too large for shared memory (config 4's
// 256 x 256 x 32 slabs): segmented x rows (row tiles staged by TMA, the
// affine exchange fused) and y columns (straight from global), then the
// exact register z kernel (slab-aware).  Returns the x/y line length.
int seg_stream_length(const cg_ctx* c) {
    const MeshDev& m = c->m;
    if (!c->reg_lines || c->S < 1 || c->S > kLineMaxS) return 0;
    if (m.nx != 256 || m.ny != 256 || m.dx != m.dy) return 0;
    return 256;
}

// z slabs of the cubic meshes' planes (configs 1-3 split over ranks: 80 x 80
// or 160 x 160 planes, any local nz): the segmented plane kernel with the
// affine exchange fused, then the exact z kernel of the mesh in slab mode
// (local block solve; the interface correction follows, cg_zslab_correct).
int seg_slab_plane_length(const cg_ctx* c) {
    const MeshDev& m = c->m;
    if (!c->reg_lines || c->S < 1 || c->S > kLineMaxS || !m.slab) return 0;
    if (m.nx != m.ny || m.dx != m.dy) return 0;
    return (m.nx == 80 || m.nx == 160) ? m.nx : 0;
}

int fast_lod_kind(const cg_ctx* c) {
    if (seg_line_length(c)) return 1;
    if (seg_stream_length(c)) return 2;
    if (seg_slab_plane_length(c)) return 3;
    return 0;
}

// ---------------------------------------------------------------- device side

// The segmented solve of one line (see the header).  w: this lane's M
// elements; fac: the line's inv[N], gam[N], cf[N], cb[N] (stride N, shared
// memory); seg: this lane's segment; lanes seg * (32 / K) + ls hold the line.
template <int M, int K>
__device__ __forceinline__ void solve_seg(double (&w)[M], const double* __restrict__ fac, int N,
                                          double r, int seg, int ls) {
    constexpr int LPW = 32 / K;
    const int o = seg * M;
    const double* inv = fac + o;
    const double* gam = fac + N + o;
    const double* cf = fac + 2 * N;
    const double* cb = fac + 3 * N;
    // forward, zero carry-in
    double prev = w[0] * inv[0];
    w[0] = prev;
#pragma unroll
    for (int i = 1; i < M; i++) {
        prev = (w[i] + r * prev) * inv[i];
        w[i] = prev;
    }
    if constexpr (K > 1) {
        double P = 0.0;
#pragma unroll
        for (int j = 0; j < K - 1; j++) {
            const double le = __shfl_sync(0xffffffffu, prev, j * LPW + ls);
            if (j < seg) P = le + cf[j * M + M - 1] * P;
        }
#pragma unroll
        for (int i = 0; i < M; i++) w[i] = w[i] + cf[o + i] * P;
    }
    // backward, zero carry-in (U_end = p_end)
    double next = w[M - 1];
#pragma unroll
    for (int i = M - 2; i >= 0; i--) {
        next = w[i] + gam[i] * next;
        w[i] = next;
    }
    if constexpr (K > 1) {
        double X = 0.0;
#pragma unroll
        for (int j = K - 1; j > 0; j--) {
            const double us = __shfl_sync(0xffffffffu, next, j * LPW + ls);
            if (j > seg) X = us + cb[j * M] * X;
        }
#pragma unroll
        for (int i = 0; i < M; i++) w[i] = w[i] + cb[o + i] * X;
    }
}

// Phase probe (probe build, -DCG_PROBE; tools/seg_phases.py): %globaltimer
// (ns, one clock for all SMs) at each phase boundary of every plane CTA.
#ifdef CG_PROBE
__device__ unsigned long long g_seg_probe[8 * 2048];
extern "C" int cg_seg_probe_read(unsigned long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, g_seg_probe,
                                     sizeof(unsigned long long) * (size_t)std::min(n, 8 * 2048));
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SEG_MARK(k) \
    if (threadIdx.x == 0) g_seg_probe[8 * (blockIdx.y * gridDim.x + blockIdx.x) + (k)] = gtimer()
#else
#define SEG_MARK(k)
#endif

// Variant with one pass of corrections: the backward recurrence runs on the
// uncorrected forward values L, and by linearity U(p) = U(L) + P V with the
// precomputed V = U(cf), so x_i = U(L)_i + V_i P + cb_i X -- one (V_i, cb_i)
// pair load and two FMAs per element instead of two loads and four roundings;
// the forward carries fold while the backward chain runs.  fac: the kSegArr
// layout with stride N (inv, gam, cf, cb, then (V, cb) pairs).
template <int M, int K>
__device__ __forceinline__ void solve_seg2(double (&w)[M], const double* __restrict__ fac, int N,
                                           double r, int seg, int ls) {
    constexpr int LPW = 32 / K;
    const int o = seg * M;
    const double* inv = fac + o;
    const double* gam = fac + N + o;
    const double* cf = fac + 2 * N;
    const double2* vc = reinterpret_cast<const double2*>(fac + 4 * N) + o;
    const double2* vcall = reinterpret_cast<const double2*>(fac + 4 * N);
    double prev = w[0] * inv[0];
    w[0] = prev;
#pragma unroll
    for (int i = 1; i < M; i++) {
        prev = (w[i] + r * prev) * inv[i];
        w[i] = prev;
    }
    double P = 0.0;
    if constexpr (K > 1) {
#pragma unroll
        for (int j = 0; j < K - 1; j++) {
            const double le = __shfl_sync(0xffffffffu, prev, j * LPW + ls);
            if (j < seg) P = le + cf[j * M + M - 1] * P;
        }
    }
    double next = w[M - 1];
#pragma unroll
    for (int i = M - 2; i >= 0; i--) {
        next = w[i] + gam[i] * next;
        w[i] = next;
    }
    if constexpr (K > 1) {
        double X = 0.0;
        const double ustart = __fma_rn(vc[0].x, P, next);
#pragma unroll
        for (int j = K - 1; j > 0; j--) {
            const double us = __shfl_sync(0xffffffffu, ustart, j * LPW + ls);
            if (j > seg) X = __fma_rn(vcall[j * M].y, X, us);
        }
#pragma unroll
        for (int i = 0; i < M; i++) {
            const double2 f = vc[i];
            w[i] = __fma_rn(f.y, X, __fma_rn(f.x, P, w[i]));
        }
    }
}

template <int M, int K, int V>
__device__ __forceinline__ void solve_segv(double (&w)[M], const double* __restrict__ fac, int N,
                                           double r, int seg, int ls) {
    if constexpr (V == 2) solve_seg2<M, K>(w, fac, N, r, seg, ls);
    else solve_seg<M, K>(w, fac, N, r, seg, ls);
}

struct FastExch {
    const int32_t* vox;  // ascending non-empty voxels
    const int32_t* n;    // their count
    const double* aff;   // (S_window, rq, 2) {alpha, beta}
    const int32_t* pz;   // (ny * nz + 1) first list index of each x row
    int rq;
};

constexpr int kXB = 4;  // exchange records per thread per batch

// Staged plane layout: row pitch P == 2 (mod 4) doubles (16 B aligned rows
// for the TMA copies; the x sweep's 16 B row-segment accesses are conflict-
// free) and a gap of G doubles after every M rows, so the y sweep's K
// segments (same column, M rows apart) fall in the two different half-bank
// groups of a warp's 8-byte access (M * P + G == 8 mod 16 doubles).
template <int N, int K>
struct SegPlane {
    static constexpr int M = N / K;
    static constexpr int P = ((N + 2) & ~1) | 2;
    // segment offset wanted: 32/K doubles (mod 16) -- K/2 segments per half warp
    static constexpr int T = K > 2 ? (32 / K) % 16 : -1;
    static constexpr int gap() {
        if (T < 0) return 0;
        for (int g = 0; g < 16; g += 2)
            if ((M * P + g) % 16 == T) return g;
        return 0;
    }
    static constexpr int G = gap();
    static constexpr int doubles = N * P + (K - 1) * G;
    __device__ __forceinline__ static int row(int r) { return r * P + (r / M) * G; }
};

// CTA per (z plane, substrate): TMA-staged plane, affine exchange, Dirichlet
// pins, segmented x sweep (K lanes per row), segmented y sweep, written
// straight to global memory or (TMA_STORE) back to the staged plane and out
// with one bulk copy per row.  early: the exchange records were written at
// least one launch back on this stream (substeps >= 1) and load before the
// PDL wait.
template <bool DIRI, bool EXCH, int N, int K, bool TMA_STORE, int V>
__global__ void __launch_bounds__(N * K, 1) k_plane_seg(double* __restrict__ dens, MeshDev m,
                                                        const double* __restrict__ segf, int nmax,
                                                        const double* __restrict__ rr,
                                                        const double* __restrict__ diri,
                                                        FastExch fx, int early, PendCorr pc) {
    using L = SegPlane<N, K>;
    constexpr int M = L::M, LPW = 32 / K;
    static_assert(N % K == 0 && M % 2 == 0 && N % LPW == 0, "segments of whole pairs, whole warps");
    extern __shared__ double sm[];
    __shared__ __align__(8) unsigned long long bar;
    double* plane = sm;
    double* fxy = plane + L::doubles;  // [axis x, y][kSegArr][N]
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int z = blockIdx.x, s = blockIdx.y;
    SEG_MARK(0);
    if (t == 0) mbar_init(&bar, 1);
    // factors: constant within the step (written before the graph runs)
    for (int i = t; i < 2 * kSegArr * N; i += blockDim.x) {
        const int a = i / (kSegArr * N), rem = i - a * kSegArr * N, kind = rem / N,
                  j = rem - kind * N;
        // the (V, cb) pairs span two arrays of the global layout
        cp_async8(fxy + i, segf + (long)(s * 3 + a) * kSegArr * nmax +
                               (kind < 4 ? kind * nmax : 4 * nmax + (kind - 4) * N) + j);
    }
    cp_async_commit();
    int q0 = 0, q1 = 0, vb[kXB];
    double2 ab[kXB];
    const double2* aff = reinterpret_cast<const double2*>(fx.aff) + (long)s * fx.rq;
    auto issue = [&](int qb) {
#pragma unroll
        for (int j = 0; j < kXB; j++) {
            const int q = qb + j * (int)blockDim.x;
            vb[j] = q < q1 ? fx.vox[q] : -1;
            if (q < q1) ab[j] = aff[q];
        }
    };
    // V == 3: per-warp pipelined staging -- warp w issues the TMA copies of
    // its own LPW rows on its own mbarrier, applies those rows' exchange maps
    // and runs their x sweep as soon as they land (no CTA-wide wait between
    // staging, exchange and the x sweep).
    constexpr bool PIPE = V == 3;
    __shared__ __align__(8) unsigned long long wbar[PIPE ? N * K / 32 : 1];
    if (PIPE && t < N * K / 32) mbar_init(&wbar[t], 1);
    __syncthreads();  // barrier initialised
    pdl_wait();
    SEG_MARK(1);
    double* g = dens + ((long)s * m.nz + z) * (N * N);
    if constexpr (PIPE) {
        if (lane == 0) {
            mbar_expect_tx(&wbar[wid], (unsigned)(LPW * N * 8));
            for (int y = wid * LPW; y < (wid + 1) * LPW; y++)
                bulk_g2s(plane + L::row(y), g + (long)y * N, N * 8, &wbar[wid]);
        }
        const int ra = z * N + wid * LPW;  // first x row of this warp
        auto issue_w = [&](int qs) {
#pragma unroll
            for (int j = 0; j < kXB; j++) {
                const int qq = qs + j * 32;
                vb[j] = qq < q1 ? fx.vox[qq] : -1;
                if (qq < q1) ab[j] = aff[qq];
            }
        };
        if (EXCH) {
            q0 = fx.pz[ra];
            q1 = fx.pz[ra + LPW];
            issue_w(q0 + lane);
        }
        cp_async_wait_all();
        __syncthreads();  // factors visible to every warp
        mbar_wait(&wbar[wid], 0);
        SEG_MARK(2);
        if (pc.lr) {  // the previous substep's deferred z-slab correction
            const double v = pc.spk[(long)s * 2 * pc.nz + z], w = pc.spk[(long)s * 2 * pc.nz + pc.nz + z];
            for (int i = lane; i < LPW * N; i += 32) {
                const int y = wid * LPW + i / N, x = i - (i / N) * N;
                const long p = (long)y * N + x, r = p / pc.Lb, j = p - r * pc.Lb;
                const double* c = pc.lr + ((r * pc.S + s) * 2) * pc.Lb + j;
                double* cell = plane + L::row(y) + x;
                double u = *cell;
                u = u + c[0] * v;
                u = u + c[pc.Lb] * w;
                *cell = u;
            }
            __syncwarp();
        }
        if (EXCH) {
            const int base = z * N * N;
            for (int qb = q0 + lane; qb < q1;) {
#pragma unroll
                for (int j = 0; j < kXB; j++) {
                    if (vb[j] >= 0) {
                        const int local = vb[j] - base;
                        const int y = local / N;
                        double* cell = plane + L::row(y) + (local - y * N);
                        *cell = *cell * ab[j].x + ab[j].y;
                    }
                }
                qb += kXB * 32;
                if (qb >= q1) break;
                issue_w(qb);
            }
            __syncwarp();
        }
    } else {
    if (t == 0) mbar_expect_tx(&bar, (unsigned)(N * N * 8));
    __syncthreads();
    if (lane == 0)
        for (int y = wid; y < N; y += (int)(blockDim.x >> 5))
            bulk_g2s(plane + L::row(y), g + (long)y * N, N * 8, &bar);
    // the exchange records load while the plane is in flight (early / not:
    // written by the rebin before this step's graph, or by the bin fix-up
    // of an earlier launch on another stream ordered by events)
    if (EXCH) {
        q0 = fx.pz[z * N];
        q1 = fx.pz[(z + 1) * N];
        issue(q0 + t);
    }
    cp_async_wait_all();
    mbar_wait(&bar, 0);
    __syncthreads();
    SEG_MARK(2);
    if (pc.lr) {  // the previous substep's deferred z-slab correction
        const double v = pc.spk[(long)s * 2 * pc.nz + z], w = pc.spk[(long)s * 2 * pc.nz + pc.nz + z];
        for (int i = t; i < N * N; i += (int)blockDim.x) {
            const int y = i / N, x = i - y * N;
            const long p = i, r = p / pc.Lb, j = p - r * pc.Lb;
            const double* c = pc.lr + ((r * pc.S + s) * 2) * pc.Lb + j;
            double* cell = plane + L::row(y) + x;
            double u = *cell;
            u = u + c[0] * v;
            u = u + c[pc.Lb] * w;
            *cell = u;
        }
        __syncthreads();
    }
    if (EXCH) {
        const int base = z * N * N;
        for (int qb = q0 + t;;) {
#pragma unroll
            for (int j = 0; j < kXB; j++) {
                if (vb[j] >= 0) {
                    const int local = vb[j] - base;
                    const int y = local / N;
                    double* cell = plane + L::row(y) + (local - y * N);
                    *cell = *cell * ab[j].x + ab[j].y;
                }
            }
            qb += kXB * (int)blockDim.x;
            if (qb >= q1) break;
            issue(qb);
        }
        __syncthreads();
    }
    }
    SEG_MARK(3);
    const double dv = DIRI ? diri[s] : 0.0;
    const bool zface = is_zface(z, m);
    const int seg = lane / LPW, ls = lane % LPW;
    const int line = wid * LPW + ls;
    const bool full = zface || line == 0 || line == N - 1;
    const bool first = seg == 0, last = seg == K - 1;
    {
        double* row = plane + L::row(line) + seg * M;
        double w[M];
#pragma unroll
        for (int i = 0; i < M; i += 2) {
            const double2 v = *reinterpret_cast<const double2*>(row + i);
            w[i] = v.x;
            w[i + 1] = v.y;
        }
        if (DIRI) pin_seg<M>(w, full, first, last, dv);
        solve_segv<M, K, V>(w, fxy, N, rr[s * 3 + 0], seg, ls);
        if (DIRI) pin_seg<M>(w, full, first, last, dv);
#pragma unroll
        for (int i = 0; i < M; i += 2) *reinterpret_cast<double2*>(row + i) = make_double2(w[i], w[i + 1]);
    }
    __syncthreads();
    SEG_MARK(4);
    {
        double* col = plane + L::row(seg * M) + line;
        double w[M];
#pragma unroll
        for (int i = 0; i < M; i++) w[i] = col[i * L::P];
        solve_segv<M, K, V>(w, fxy + kSegArr * N, N, rr[s * 3 + 1], seg, ls);
        if (DIRI) pin_seg<M>(w, full, first, last, dv);
        if constexpr (TMA_STORE) {
#pragma unroll
            for (int i = 0; i < M; i++) col[i * L::P] = w[i];
        } else {
            double* gc = g + (long)seg * M * N + line;
#pragma unroll
            for (int i = 0; i < M; i++) gc[(long)i * N] = w[i];
        }
    }
    if constexpr (TMA_STORE) {
        fence_proxy_async_smem();
        __syncthreads();
        if (lane == 0) {
            for (int y = wid; y < N; y += (int)(blockDim.x >> 5))
                bulk_s2g(g + (long)y * N, plane + L::row(y), N * 8);
            bulk_commit_wait_read();
        }
    }
    __syncthreads();
    SEG_MARK(5);
    pdl_trigger();  // the z kernel may launch while the last planes finish
}

template <int M>
__device__ __forceinline__ void check_seg(const double (&w)[M], int* __restrict__ flags) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < M; i++) ok = ok && (w[i] >= 0.0 && w[i] <= 0x1.fffffffffffffp+1023);
    if (!ok) atomicOr(&flags[FLAG_NUMERIC], 1);
}

// z sweep: K lanes per (x, y) column (M consecutive planes each) read straight
// from global memory -- every load instruction is K runs of 32/K consecutive
// columns -- solved with the segmented recurrence, pinned, checked (last
// substep: Microenvironment.check_state, core.py:142-145) and written back.
template <bool DIRI, int N, int K, int V>
__global__ void __launch_bounds__(128) k_zcols_seg(double* __restrict__ dens, MeshDev m,
                                                   const double* __restrict__ segf, int nmax,
                                                   const double* __restrict__ rr,
                                                   const double* __restrict__ diri,
                                                   int* __restrict__ chk) {
    constexpr int M = N / K, LPW = 32 / K;
    static_assert(N % K == 0 && (N * N) % LPW == 0, "whole warps of columns");
    __shared__ double fz[kSegArr * N];
    const int s = blockIdx.y;
    for (int i = threadIdx.x; i < kSegArr * N; i += blockDim.x) {
        const int kind = i / N, j = i - kind * N;
        fz[i] = segf[(long)(s * 3 + 2) * kSegArr * nmax +
                     (kind < 4 ? kind * nmax : 4 * nmax + (kind - 4) * N) + j];
    }
    __syncthreads();
    pdl_wait();
    const int lane = threadIdx.x & 31, seg = lane / LPW, ls = lane % LPW;
    const int p = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * LPW + ls;
    if (p - ls < N * N) {  // warp-uniform
        constexpr long PS = (long)N * N;
        double* col = dens + (long)s * N * PS + (long)seg * M * PS + p;
        double w[M];
#pragma unroll
        for (int i = 0; i < M; i++) w[i] = col[i * PS];
        solve_segv<M, K, V>(w, fz, N, rr[s * 3 + 2], seg, ls);
        if (DIRI && !m.slab) {
            const int y = p / N, x = p - y * N;
            pin_seg<M>(w, x == 0 || x == N - 1 || y == 0 || y == N - 1, seg == 0, seg == K - 1,
                       diri[s]);
        }
        if (chk) check_seg<M>(w, chk);
#pragma unroll
        for (int i = 0; i < M; i++) col[i * PS] = w[i];
    }
    pdl_trigger();
}

// ---- streaming meshes (config 4): x rows and y columns

// x sweep over tiles of RT consecutive x rows (row r = (z, y), NX contiguous
// values) of one substrate: TMA bulk rows into smem, the tile's affine
// exchange records (per-row list offsets), Dirichlet pins, K-segment
// solve (solve_seg, shuffled carries), bulk rows back to global.
template <int NX, int K, int RT>
struct RowTile {
    static constexpr int P = ((NX + 2) & ~1) | 2;
    static constexpr int doubles = RT * P;
};

template <bool DIRI, bool EXCH, int NX, int K, int RT>
__global__ void __launch_bounds__(RT * K, 4) k_xrows_seg(double* __restrict__ dens, MeshDev m,
                                                      const double* __restrict__ segf, int nmax,
                                                      const double* __restrict__ rr,
                                                      const double* __restrict__ diri,
                                                      FastExch fx, int early, PendCorr pc) {
    using L = RowTile<NX, K, RT>;
    constexpr int M = NX / K, LPW = 32 / K, P = L::P;
    static_assert(NX % K == 0 && M % 2 == 0 && RT % LPW == 0, "whole pairs and warps");
    extern __shared__ double sm[];
    __shared__ __align__(8) unsigned long long bar;
    double* tile = sm;
    double* fac = tile + L::doubles;  // x-axis inv, gam, cf, cb
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int s = blockIdx.y;
    const long nrows = (long)m.ny * m.nz;
    const long r0 = (long)blockIdx.x * RT;
    const int nr = (int)(nrows - r0 < RT ? nrows - r0 : RT);
    if (t == 0) mbar_init(&bar, 1);
    for (int i = t; i < 4 * NX; i += blockDim.x) {
        const int kind = i / NX, j = i - kind * NX;
        cp_async8(fac + i, segf + (long)(s * 3 + 0) * kSegArr * nmax + kind * nmax + j);
    }
    cp_async_commit();
    int q0 = 0, q1 = 0, vb[kXB];
    double2 ab[kXB];
    const double2* aff = reinterpret_cast<const double2*>(fx.aff) + (long)s * fx.rq;
    auto issue = [&](int qb) {
#pragma unroll
        for (int j = 0; j < kXB; j++) {
            const int q = qb + j * (int)blockDim.x;
            vb[j] = q < q1 ? fx.vox[q] : -1;
            if (q < q1) ab[j] = aff[q];
        }
    };
    __syncthreads();
    pdl_wait();
    const long nvox = nrows * NX;
    double* g = dens + (long)s * nvox + r0 * NX;
    if (t == 0) mbar_expect_tx(&bar, (unsigned)(nr * NX * 8));
    __syncthreads();
    if (lane == 0)
        for (int r = wid; r < nr; r += (int)(blockDim.x >> 5))
            bulk_g2s(tile + r * P, g + (long)r * NX, NX * 8, &bar);
    if (EXCH) {  // records load while the rows are in flight
        q0 = fx.pz[r0];
        q1 = fx.pz[r0 + nr];
        issue(q0 + t);
    }
    cp_async_wait_all();
    mbar_wait(&bar, 0);
    __syncthreads();
    if (pc.lr) {  // the previous substep's deferred z-slab correction
        for (int i = t; i < nr * NX; i += (int)blockDim.x) {
            const int r = i / NX, x = i - r * NX;
            const long row = r0 + r;
            const int y = (int)(row % m.ny), z = (int)(row / m.ny);
            const double v = pc.spk[(long)s * 2 * pc.nz + z], w = pc.spk[(long)s * 2 * pc.nz + pc.nz + z];
            const long p = (long)y * NX + x, rb = p / pc.Lb, j = p - rb * pc.Lb;
            const double* c = pc.lr + ((rb * pc.S + s) * 2) * pc.Lb + j;
            double u = tile[r * P + x];
            u = u + c[0] * v;
            u = u + c[pc.Lb] * w;
            tile[r * P + x] = u;
        }
        __syncthreads();
    }
    if (EXCH) {
        const long base = r0 * NX;
        for (int qb = q0 + t;;) {
#pragma unroll
            for (int j = 0; j < kXB; j++) {
                if (vb[j] >= 0) {
                    const int local = (int)(vb[j] - base);
                    const int r = local / NX;
                    double* cell = tile + r * P + (local - r * NX);
                    *cell = *cell * ab[j].x + ab[j].y;
                }
            }
            qb += kXB * (int)blockDim.x;
            if (qb >= q1) break;
            issue(qb);
        }
        __syncthreads();
    }
    const int seg = lane / LPW, ls = lane % LPW;
    const int lr = wid * LPW + ls;
    if (lr - ls < nr) {  // warp-uniform: nr is a multiple of LPW except at the end
        const int lrc = lr < nr ? lr : nr - 1;
        const long row = r0 + lrc;
        const int y = (int)(row % m.ny), z = (int)(row / m.ny);
        const double dv = DIRI ? diri[s] : 0.0;
        const bool full = is_zface(z, m) || y == 0 || y == m.ny - 1;
        double* rp = tile + lrc * P + seg * M;
        double w[M];
#pragma unroll
        for (int i = 0; i < M; i += 2) {
            const double2 v = *reinterpret_cast<const double2*>(rp + i);
            w[i] = v.x;
            w[i + 1] = v.y;
        }
        if (DIRI) pin_seg<M>(w, full, seg == 0, seg == K - 1, dv);
        solve_seg<M, K>(w, fac, NX, rr[s * 3 + 0], seg, ls);
        if (DIRI) pin_seg<M>(w, full, seg == 0, seg == K - 1, dv);
        if (lr < nr) {
#pragma unroll
            for (int i = 0; i < M; i += 2)
                *reinterpret_cast<double2*>(rp + i) = make_double2(w[i], w[i + 1]);
        }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (lane == 0) {
        for (int r = wid; r < nr; r += (int)(blockDim.x >> 5))
            bulk_s2g(g + (long)r * NX, tile + r * P, NX * 8);
        bulk_commit_wait_read();
    }
    pdl_trigger();
}

// y sweep, warp-uniform segments: CTA = K warps x 32 consecutive x of one z
// plane; warp k holds rows [k M, (k+1) M) of its 32 columns (every load one
// 256 B row), factors in shared memory (uniform, broadcast), carries
// through shared memory.
template <bool DIRI, int NY, int K>
__global__ void __launch_bounds__(32 * K, 2) k_ycols_segw(double* __restrict__ dens, MeshDev m,
                                                       const double* __restrict__ segf, int nmax,
                                                       const double* __restrict__ rr,
                                                       const double* __restrict__ diri) {
    constexpr int M = NY / K;
    __shared__ double fy[4 * NY];
    __shared__ double car[2 * K * 32];
    const int s = blockIdx.y;
    for (int i = threadIdx.x; i < 4 * NY; i += blockDim.x) {
        const int kind = i / NY, j = i - kind * NY;
        fy[i] = segf[(long)(s * 3 + 1) * kSegArr * nmax + kind * nmax + j];
    }
    __syncthreads();
    pdl_wait();
    const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
    const int tiles_x = m.nx / 32;
    const int z = blockIdx.x / tiles_x, x = (blockIdx.x - z * tiles_x) * 32 + lane;
    const long plane = (long)m.nx * NY;
    double* col = dens + (long)s * plane * m.nz + (long)z * plane + (long)seg * M * m.nx + x;
    double w[M];
#pragma unroll
    for (int i = 0; i < M; i++) w[i] = col[(long)i * m.nx];
    const double r = rr[s * 3 + 1];
    const int o = seg * M;
    // forward, zero carry-in
    double prev = w[0] * fy[o];
    w[0] = prev;
#pragma unroll
    for (int i = 1; i < M; i++) {
        prev = (w[i] + r * prev) * fy[o + i];
        w[i] = prev;
    }
    car[seg * 32 + lane] = prev;
    __syncthreads();
    if (seg > 0) {
        double P = 0.0;
        for (int j = 0; j < seg; j++) P = car[j * 32 + lane] + fy[2 * NY + j * M + M - 1] * P;
#pragma unroll
        for (int i = 0; i < M; i++) w[i] = w[i] + fy[2 * NY + o + i] * P;
    }
    double next = w[M - 1];
#pragma unroll
    for (int i = M - 2; i >= 0; i--) {
        next = w[i] + fy[NY + o + i] * next;
        w[i] = next;
    }
    car[(K + seg) * 32 + lane] = next;
    __syncthreads();
    if (seg < K - 1) {
        double X = 0.0;
        for (int j = K - 1; j > seg; j--) X = car[(K + j) * 32 + lane] + fy[3 * NY + j * M] * X;
#pragma unroll
        for (int i = 0; i < M; i++) w[i] = w[i] + fy[3 * NY + o + i] * X;
    }
    if (DIRI) {
        const bool full = is_zface(z, m) || x == 0 || x == m.nx - 1;
        pin_seg<M>(w, full, seg == 0, seg == K - 1, diri[s]);
    }
#pragma unroll
    for (int i = 0; i < M; i++) col[(long)i * m.nx] = w[i];
    pdl_trigger();
}

// ---------------------------------------------------------------- launch

namespace {

// The deferred z-slab correction the next x-row / plane kernel applies
// (cg_zslab_defer), or none.
PendCorr pend_corr(const cg_ctx* c) {
    if (!c->pend_lr) return PendCorr{nullptr, nullptr, 0, 0, 0};
    const long L = (long)c->m.nx * c->m.ny;
    return PendCorr{c->pend_lr, c->d_spk, (L + c->slab_world - 1) / c->slab_world, c->S, c->m.nz};
}

bool seg_tma_store() {
    const char* env = std::getenv("CELLGPU_SEG_TMA_STORE");
    return env ? std::atoi(env) != 0 : false;
}

// Segmented solve variant (env CELLGPU_SEG_SOLVE = 1: two correction
// passes, solve_seg; 2: one FMA correction pass, solve_seg2).
int seg_solve() {
    const char* env = std::getenv("CELLGPU_SEG_SOLVE");
    return env && std::atoi(env) == 2 ? 2 : 1;
}

template <bool DIRI, bool EXCH, int N, int K, bool TS, int V>
int launch_plane_seg_t(cg_ctx* c, double* d, const double* segf, const double* rr,
                       const double* diri, const FastExch& fx, int ns, bool early) {
    const size_t smem = ((size_t)SegPlane<N, K>::doubles + 2 * kSegArr * (size_t)N) * sizeof(double);
    static DeviceFlags attrs;
    if (!attrs.test_and_set(c->device))
        CG_CUDA_CHECK(cudaFuncSetAttribute(k_plane_seg<DIRI, EXCH, N, K, TS, V>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CG_LAUNCH(c, K_PLANE_SEG, (k_plane_seg<DIRI, EXCH, N, K, TS, V>), dim3(c->m.nz, ns), N * K, smem, d,
              c->m, segf, c->nmax, rr, diri, fx, early ? 1 : 0, pend_corr(c));
    return CG_OK;
}

// Per-warp pipelined staging in the plane kernel (env CELLGPU_SEG_PIPE=0:
// one CTA-wide wait for the whole plane).  Bit-identical; config 3 lod_xy
// 88.6 vs 91.0 us per substep (1.773 vs 1.803 ms per step), config 1 8.1
// vs 8.3 us.
bool seg_pipe() {
    const char* env = std::getenv("CELLGPU_SEG_PIPE");
    return env ? std::atoi(env) != 0 : true;
}

template <bool DIRI, bool EXCH, int N, int K>
int launch_plane_seg(cg_ctx* c, double* d, const double* segf, const double* rr,
                     const double* diri, const FastExch& fx, int ns, bool early) {
    if (seg_pipe())
        return launch_plane_seg_t<DIRI, EXCH, N, K, false, 3>(c, d, segf, rr, diri, fx, ns, early);
    if (seg_solve() == 2)
        return launch_plane_seg_t<DIRI, EXCH, N, K, false, 2>(c, d, segf, rr, diri, fx, ns, early);
    return seg_tma_store() ? launch_plane_seg_t<DIRI, EXCH, N, K, true, 1>(c, d, segf, rr, diri, fx, ns, early)
                           : launch_plane_seg_t<DIRI, EXCH, N, K, false, 1>(c, d, segf, rr, diri, fx, ns, early);
}

// ---- warp-uniform segments: factors from the constant bank

// Factors of the segmented solve per substrate as a kernel parameter; the
// meshes with segmented kernels are cubic with equal spacing, so the x, y and
// z lines of a substrate share them.  With the substrate and the segment
// compile-time (warp-uniform dispatch), every factor is a constant-bank
// operand of its FP64 instruction: no shared-memory factor loads.
template <int N>
struct SegConst {
    double inv[kLineMaxS][N], gam[kLineMaxS][N], cf[kLineMaxS][N], cb[kLineMaxS][N];
    double r[kLineMaxS];
};

template <int K, int SEG = 0, typename F>
__device__ __forceinline__ void for_seg(int seg, F&& f) {
    if constexpr (SEG < K) {
        if (seg == SEG) f(std::integral_constant<int, SEG>{});
        else for_seg<K, SEG + 1>(seg, f);
    }
}
template <int SI = 0, typename F>
__device__ __forceinline__ void for_sub(int s, F&& f) {
    if constexpr (SI < kLineMaxS) {
        if (s == SI) f(std::integral_constant<int, SI>{});
        else for_sub<SI + 1>(s, f);
    }
}

// One segmented sweep of 32 lines per warp group: warp `seg` of the group
// holds segment seg (M elements) of each of its lanes' lines; the carries go
// through shared memory (car: [2][K][32] for this group) between the
// group's K warps.  sync(): the barrier shared by the K warps.
template <int N, int K, typename Sync>
__device__ __forceinline__ void sweep_segw(double (&w)[N / K], const SegConst<N>& f, int s,
                                           int seg, int lane, double* car, Sync sync) {
    constexpr int M = N / K;
    for_sub(s, [&](auto si) {
        for_seg<K>(seg, [&](auto sg) {
            constexpr int SI = decltype(si)::value, SEG = decltype(sg)::value, o = SEG * M;
            const double r = f.r[SI];
            double prev = w[0] * f.inv[SI][o];
            w[0] = prev;
#pragma unroll
            for (int i = 1; i < M; i++) {
                prev = (w[i] + r * prev) * f.inv[SI][o + i];
                w[i] = prev;
            }
            car[SEG * 32 + lane] = prev;
        });
    });
    sync();
    for_sub(s, [&](auto si) {
        for_seg<K>(seg, [&](auto sg) {
            constexpr int SI = decltype(si)::value, SEG = decltype(sg)::value, o = SEG * M;
            if constexpr (SEG > 0) {
                double P = 0.0;
#pragma unroll
                for (int j = 0; j < SEG; j++) P = car[j * 32 + lane] + f.cf[SI][j * M + M - 1] * P;
#pragma unroll
                for (int i = 0; i < M; i++) w[i] = w[i] + f.cf[SI][o + i] * P;
            }
            double next = w[M - 1];
#pragma unroll
            for (int i = M - 2; i >= 0; i--) {
                next = w[i] + f.gam[SI][o + i] * next;
                w[i] = next;
            }
            car[(K + SEG) * 32 + lane] = next;
        });
    });
    sync();
    for_sub(s, [&](auto si) {
        for_seg<K>(seg, [&](auto sg) {
            constexpr int SI = decltype(si)::value, SEG = decltype(sg)::value, o = SEG * M;
            if constexpr (SEG < K - 1) {
                double X = 0.0;
#pragma unroll
                for (int j = K - 1; j > SEG; j--) X = car[(K + j) * 32 + lane] + f.cb[SI][j * M] * X;
#pragma unroll
                for (int i = 0; i < M; i++) w[i] = w[i] + f.cb[SI][o + i] * X;
            }
        });
    });
}

// z sweep, warp-uniform segments: CTA = K warps x 32 consecutive (x, y)
// columns; warp k loads planes [k M, (k+1) M) of its 32 columns (every load
// one coalesced 256 B access), the K warps fold their carries through shared
// memory, then pins, check_state (last substep) and the store.
template <bool DIRI, int N, int K>
__global__ void __launch_bounds__(32 * K) k_zcols_segw(double* __restrict__ dens, MeshDev m,
                                                       const double* __restrict__ diri,
                                                       const __grid_constant__ SegConst<N> f,
                                                       int* __restrict__ chk) {
    constexpr int M = N / K;
    constexpr long PS = (long)N * N;
    __shared__ double car[2 * K * 32];
    pdl_wait();
    const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5, s = blockIdx.y;
    const int p = blockIdx.x * 32 + lane;  // N * N is a multiple of 32 (N = 80, 160)
    double* col = dens + (long)s * N * PS + (long)seg * M * PS + p;
    double w[M];
#pragma unroll
    for (int i = 0; i < M; i++) w[i] = col[i * PS];
    sweep_segw<N, K>(w, f, s, seg, lane, car, [] { __syncthreads(); });
    if (DIRI && !m.slab) {
        const int y = p / N, x = p - y * N;
        pin_seg<M>(w, x == 0 || x == N - 1 || y == 0 || y == N - 1, seg == 0, seg == K - 1, diri[s]);
    }
    if (chk) check_seg<M>(w, chk);
#pragma unroll
    for (int i = 0; i < M; i++) col[i * PS] = w[i];
    pdl_trigger();
}

template <int N>
void fill_seg_const(const cg_ctx* c, SegConst<N>& f, int s0, int ns) {
    std::memset(&f, 0, sizeof f);
    const int nmax = c->nmax;
    for (int j = 0; j < ns && j < kLineMaxS; j++) {
        const double* o = &c->h_segf[(size_t)((s0 + j) * 3 + 2) * kSegArr * nmax];
        for (int i = 0; i < N; i++) {
            f.inv[j][i] = o[i];
            f.gam[j][i] = o[nmax + i];
            f.cf[j][i] = o[2 * nmax + i];
            f.cb[j][i] = o[3 * nmax + i];
        }
        f.r[j] = c->h_r[(s0 + j) * 3 + 2];
    }
}

// Warp-uniform segments (constant-bank factors, shared-memory carries) or
// lane segments (shuffled carries, shared-memory factors), per kernel and
// line length (env CELLGPU_SEG_WARP_PLANE / CELLGPU_SEG_WARP_Z = 0 / 1).
// z sweep with warp-uniform segments (k_zcols_segw) or lane segments
// (k_zcols_seg); env CELLGPU_SEG_WARP_Z = 0 / 1.  Measured (in-graph stage
// us): config 1 6.1 lane vs 8.9 warp-uniform, config 3 64.0 vs 54.6 -- the
// 160^3 z sweep gains (coalesced 256 B rows, no factor loads), the 80^3 one
// loses to the barriers and to the constant-cache traffic of three
// substrates' CTAs sharing an SM.  (A warp-uniform plane kernel measured
// slower at both sizes, 12.0 vs 8.8 and 113 vs 90.5 us, and was removed.)
bool seg_warp_uniform(int N) {
    const char* env = std::getenv("CELLGPU_SEG_WARP_Z");
    if (env) return std::atoi(env) != 0;
    return N == 160;
}

template <bool DIRI, int N, int K>
int launch_z_segw(cg_ctx* c, double* d, const double* diri, int s0, int ns, int* chk) {
    static thread_local SegConst<N> f;  // host staging of the kernel parameter
    fill_seg_const<N>(c, f, s0, ns);
    CG_LAUNCH(c, K_Z_SEG, (k_zcols_segw<DIRI, N, K>), dim3((unsigned)(N * N / 32), ns), 32 * K, 0,
              d, c->m, diri, f, chk);
    return CG_OK;
}

template <bool DIRI, int N, int K>
int launch_z_seg(cg_ctx* c, double* d, const double* segf, const double* rr, const double* diri,
                 int ns, int* chk) {
    constexpr int LPW = 32 / K;
    const long warps = ((long)N * N + LPW - 1) / LPW;
    if (seg_solve() == 2)
        CG_LAUNCH(c, K_Z_SEG, (k_zcols_seg<DIRI, N, K, 2>), dim3((unsigned)((warps + 3) / 4), ns),
                  128, 0, d, c->m, segf, c->nmax, rr, diri, chk);
    else
        CG_LAUNCH(c, K_Z_SEG, (k_zcols_seg<DIRI, N, K, 1>), dim3((unsigned)((warps + 3) / 4), ns),
                  128, 0, d, c->m, segf, c->nmax, rr, diri, chk);
    return CG_OK;
}

template <bool DIRI, int N>
int launch_lod_fast_n(cg_ctx* c, double* dens, const FastExch& fx, bool exch, int parts,
                      bool check, bool early) {
    const int kp = seg_k(N, true), kz = seg_k(N, false);
    int st = ensure_seg_factors(c, N / kp, N / kz);
    if (st) return st;
    const int s0 = c->sub_n > 0 ? c->sub0 : 0, ns = c->sub_n > 0 ? c->sub_n : c->S;
    double* d = dens + (long)s0 * c->nvox;
    const double* segf = c->d_segf + (size_t)s0 * 3 * kSegArr * c->nmax;
    const double* rr = c->d_r + 3 * s0;
    const double* diri = c->d_diri + s0;
    FastExch f = fx;
    if (exch) f.aff = fx.aff + (size_t)s0 * fx.rq * 2;
    if (parts & 1) {
        if (kp == 4) {
            st = exch ? launch_plane_seg<DIRI, true, N, 4>(c, d, segf, rr, diri, f, ns, early)
                      : launch_plane_seg<DIRI, false, N, 4>(c, d, segf, rr, diri, f, ns, early);
        } else if constexpr (N == 80) {
            if (kp == 8)
                st = exch ? launch_plane_seg<DIRI, true, N, 8>(c, d, segf, rr, diri, f, ns, early)
                          : launch_plane_seg<DIRI, false, N, 8>(c, d, segf, rr, diri, f, ns, early);
            else
                st = exch ? launch_plane_seg<DIRI, true, N, 2>(c, d, segf, rr, diri, f, ns, early)
                          : launch_plane_seg<DIRI, false, N, 2>(c, d, segf, rr, diri, f, ns, early);
        }
        if (st) return st;
    }
    if (parts & 2) {
        int* chk = check ? c->d_flags : nullptr;
        if (kz == 4 && seg_warp_uniform(N)) return launch_z_segw<DIRI, N, 4>(c, d, diri, s0, ns, chk);
        if (kz == 4) st = launch_z_seg<DIRI, N, 4>(c, d, segf, rr, diri, ns, chk);
        else if (kz == 8) st = launch_z_seg<DIRI, N, 8>(c, d, segf, rr, diri, ns, chk);
        else st = launch_z_seg<DIRI, N, 2>(c, d, segf, rr, diri, ns, chk);
    }
    return st;
}

// The plane kernel alone on a slab of N x N planes (seg_slab_plane_length).
template <bool DIRI, int N>
int launch_slab_planes(cg_ctx* c, double* dens, const FastExch& fx, bool exch, bool early) {
    const int kp = seg_k(N, true);
    int st = ensure_seg_factors(c, N / kp, c->m.nz);
    if (st) return st;
    const int s0 = c->sub_n > 0 ? c->sub0 : 0, ns = c->sub_n > 0 ? c->sub_n : c->S;
    double* d = dens + (long)s0 * c->nvox;
    const double* segf = c->d_segf + (size_t)s0 * 3 * kSegArr * c->nmax;
    const double* rr = c->d_r + 3 * s0;
    const double* diri = c->d_diri + s0;
    FastExch f = fx;
    if (exch) f.aff = fx.aff + (size_t)s0 * fx.rq * 2;
    if (kp == 4)
        return exch ? launch_plane_seg<DIRI, true, N, 4>(c, d, segf, rr, diri, f, ns, early)
                    : launch_plane_seg<DIRI, false, N, 4>(c, d, segf, rr, diri, f, ns, early);
    if constexpr (N == 80) {
        if (kp == 8)
            return exch ? launch_plane_seg<DIRI, true, N, 8>(c, d, segf, rr, diri, f, ns, early)
                        : launch_plane_seg<DIRI, false, N, 8>(c, d, segf, rr, diri, f, ns, early);
        return exch ? launch_plane_seg<DIRI, true, N, 2>(c, d, segf, rr, diri, f, ns, early)
                    : launch_plane_seg<DIRI, false, N, 2>(c, d, segf, rr, diri, f, ns, early);
    }
    return CG_OK;
}

}  // namespace

constexpr int kStreamKX = 8, kStreamKY = 8, kStreamRT = 16;

int prepare_lod_fast(cg_ctx* c) {
    if (seg_stream_length(c)) return ensure_seg_factors(c, 256 / kStreamKX, c->m.nz);
    if (const int N = seg_slab_plane_length(c)) return ensure_seg_factors(c, N / seg_k(N, true), c->m.nz);
    const int N = seg_line_length(c);
    if (N == 0) return CG_OK;
    return ensure_seg_factors(c, N / seg_k(N, true), N / seg_k(N, false));
}

namespace {

template <bool DIRI, bool EXCH>
int launch_xrows_seg(cg_ctx* c, double* d, const double* segf, const double* rr,
                     const double* diri, const FastExch& fx, int ns, bool early) {
    using L = RowTile<256, kStreamKX, kStreamRT>;
    const size_t smem = ((size_t)L::doubles + 4 * 256) * sizeof(double);
    static DeviceFlags attrs;
    if (!attrs.test_and_set(c->device))
        CG_CUDA_CHECK(cudaFuncSetAttribute(k_xrows_seg<DIRI, EXCH, 256, kStreamKX, kStreamRT>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long nrows = (long)c->m.ny * c->m.nz;
    CG_LAUNCH(c, K_PLANE_SEG, (k_xrows_seg<DIRI, EXCH, 256, kStreamKX, kStreamRT>),
              dim3((unsigned)((nrows + kStreamRT - 1) / kStreamRT), ns), kStreamRT * kStreamKX, smem,
              d, c->m, segf, c->nmax, rr, diri, fx, early ? 1 : 0, pend_corr(c));
    return CG_OK;
}

template <bool DIRI>
int launch_ycols_segw(cg_ctx* c, double* d, const double* segf, const double* rr,
                      const double* diri, int ns) {
    CG_LAUNCH(c, K_PLANE_SEG, (k_ycols_segw<DIRI, 256, kStreamKY>),
              dim3((unsigned)(c->m.nx / 32 * c->m.nz), ns), 32 * kStreamKY, 0, d, c->m, segf,
              c->nmax, rr, diri);
    return CG_OK;
}

// Streaming fast LOD: x rows (+ affine exchange), y columns, then the exact
// z kernel of the mesh (launch_lod part 2: register z lines, slab-aware).
int launch_lod_stream(cg_ctx* c, double* dens, int bc, const FastExch& fx, bool exch, int parts,
                      bool check, bool early) {
    int st = ensure_seg_factors(c, 256 / kStreamKX, c->m.nz);
    if (st) return st;
    const int s0 = c->sub_n > 0 ? c->sub0 : 0, ns = c->sub_n > 0 ? c->sub_n : c->S;
    double* d = dens + (long)s0 * c->nvox;
    const double* segf = c->d_segf + (size_t)s0 * 3 * kSegArr * c->nmax;
    const double* rr = c->d_r + 3 * s0;
    const double* diri = c->d_diri + s0;
    FastExch f = fx;
    if (exch) f.aff = fx.aff + (size_t)s0 * fx.rq * 2;
    const bool di = bc == CG_BC_DIRICHLET;
    if (parts & 1) {
        if (di) st = exch ? launch_xrows_seg<true, true>(c, d, segf, rr, diri, f, ns, early)
                          : launch_xrows_seg<true, false>(c, d, segf, rr, diri, f, ns, early);
        else st = exch ? launch_xrows_seg<false, true>(c, d, segf, rr, diri, f, ns, early)
                       : launch_xrows_seg<false, false>(c, d, segf, rr, diri, f, ns, early);
        if (st) return st;
        st = di ? launch_ycols_segw<true>(c, d, segf, rr, diri, ns)
                : launch_ycols_segw<false>(c, d, segf, rr, diri, ns);
        if (st) return st;
    }
    if (parts & 2) return launch_lod(c, dens, bc, nullptr, nullptr, nullptr, 0, 2, check);
    return CG_OK;
}

}  // namespace

int launch_lod_fast(cg_ctx* c, double* dens, int bc, const int32_t* vox, const int32_t* n_ne,
                    const double* aff, const int32_t* pz, int parts, bool check, bool early) {
    const FastExch fx{vox, n_ne, aff, pz, (int)std::min<long>(c->nvox, c->cap_cells)};
    const bool exch = aff != nullptr;
    if (seg_stream_length(c)) return launch_lod_stream(c, dens, bc, fx, exch, parts, check, early);
    if (const int N = seg_slab_plane_length(c)) {
        const bool di = bc == CG_BC_DIRICHLET;
        if (parts & 1) {
            const int st = N == 80 ? (di ? launch_slab_planes<true, 80>(c, dens, fx, exch, early)
                                         : launch_slab_planes<false, 80>(c, dens, fx, exch, early))
                                   : (di ? launch_slab_planes<true, 160>(c, dens, fx, exch, early)
                                         : launch_slab_planes<false, 160>(c, dens, fx, exch, early));
            if (st) return st;
        }
        if (parts & 2) return launch_lod(c, dens, bc, nullptr, nullptr, nullptr, 0, 2, check);
        return CG_OK;
    }
    const int N = seg_line_length(c);
    if (N == 0) return set_error(CG_STATE, "no segmented LOD kernels for this mesh");
    const bool di = bc == CG_BC_DIRICHLET;
    if (N == 80)
        return di ? launch_lod_fast_n<true, 80>(c, dens, fx, exch, parts, check, early)
                  : launch_lod_fast_n<false, 80>(c, dens, fx, exch, parts, check, early);
    return di ? launch_lod_fast_n<true, 160>(c, dens, fx, exch, parts, check, early)
              : launch_lod_fast_n<false, 160>(c, dens, fx, exch, parts, check, early);
}
