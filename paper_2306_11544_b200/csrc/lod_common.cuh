// Device building blocks of the LOD kernels (diffusion.cu): the line solves
// in the reference's operation order (streaming through shared memory, or a
// whole line in registers), async-copy / TMA bulk / mbarrier helpers, the
// Dirichlet plane pin, the fused exchange tile and the staged-plane pitch.
#pragma once

#include "common.cuh"

// Host factor helpers (diffusion.cu).
void host_line_factors(int n, double r, double lam3, double* inv, double* gamma);
void host_block_factors(int n, double r, double lam3, bool top, bool bottom, double* inv,
                        double* gam);
void host_thomas(double* d, int n, const double* inv, const double* gam, double r);


// diffusion.py:102-112 for one line with element stride `st`:
//   d0 *= inv0;  d_i = (d_i + r*d_{i-1}) * inv_i;  d_i += gamma_i * d_{i+1}.
// Each product and sum rounds separately (-fmad=false), as numpy does.
template <int CH = 8>
__device__ __forceinline__ void solve_line(double* __restrict__ d, int st, int n,
                                           const double* __restrict__ inv,
                                           const double* __restrict__ gam, double r) {
    // Chunks of CH elements: bulk-load the chunk's values and factors into
    // registers, run the dependent chain entirely in registers, bulk-store.
    // Measured on B200 (tools/chain_bench.cu): ~28 cycles per forward step,
    // against ~25 for the bare DMUL -> DADD -> DMUL chain and 42-58 when the
    // loads and stores are interleaved with the chain.  CH = 8 measured best
    // for whole 80-element lines (tools/solve_probe.cu: 60-64 cycles per
    // element fwd+bwd vs 69-76 at CH = 16 and 93-102 at CH = 32).
    // Full chunks carry no per-element predicates; only the tail chunk does.
    double prev = d[0] * inv[0];
    d[0] = prev;
    int i0 = 1;
#pragma unroll 1
    for (; i0 + CH <= n; i0 += CH) {
        double w[CH], f[CH];
        const double* p = d + i0 * st;
#pragma unroll
        for (int j = 0; j < CH; j++) {
            w[j] = p[j * st];
            f[j] = inv[i0 + j];
        }
#pragma unroll
        for (int j = 0; j < CH; j++) {
            prev = (w[j] + r * prev) * f[j];
            w[j] = prev;
        }
#pragma unroll
        for (int j = 0; j < CH; j++) d[(i0 + j) * st] = w[j];
    }
    if (i0 < n) {
        double w[CH], f[CH];
#pragma unroll
        for (int j = 0; j < CH; j++) {
            const int i = i0 + j;
            w[j] = i < n ? d[i * st] : 0.0;
            f[j] = i < n ? inv[i] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < CH; j++) {
            if (i0 + j < n) {
                prev = (w[j] + r * prev) * f[j];
                w[j] = prev;
            }
        }
#pragma unroll
        for (int j = 0; j < CH; j++)
            if (i0 + j < n) d[(i0 + j) * st] = w[j];
    }
    double next = prev;
    int i1 = n - 2;
#pragma unroll 1
    for (; i1 - CH + 1 >= 0; i1 -= CH) {
        double w[CH], g[CH];
#pragma unroll
        for (int j = 0; j < CH; j++) {
            w[j] = d[(i1 - j) * st];
            g[j] = gam[i1 - j];
        }
#pragma unroll
        for (int j = 0; j < CH; j++) {
            next = w[j] + g[j] * next;
            w[j] = next;
        }
#pragma unroll
        for (int j = 0; j < CH; j++) d[(i1 - j) * st] = w[j];
    }
    if (i1 >= 0) {
        double w[CH], g[CH];
#pragma unroll
        for (int j = 0; j < CH; j++) {
            const int i = i1 - j;
            w[j] = i >= 0 ? d[i * st] : 0.0;
            g[j] = i >= 0 ? gam[i] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < CH; j++) {
            if (i1 - j >= 0) {
                next = w[j] + g[j] * next;
                w[j] = next;
            }
        }
#pragma unroll
        for (int j = 0; j < CH; j++)
            if (i1 - j >= 0) d[(i1 - j) * st] = w[j];
    }
}

// 8-byte global->shared copies that do not occupy registers: every element of
// a tile is in flight at once (LDGSTS), instead of one load round trip per
// loop iteration.
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// TMA 1D bulk copies (cp.async.bulk): one instruction moves a whole 16B-
// aligned row segment; completion is tracked by an mbarrier transaction count.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// G1: pin every outer-face voxel of plane z (staged with pitch P).
__device__ __forceinline__ void dirichlet_plane(double* plane, int P, int z, const MeshDev& m,
                                                double val) {
    const int nx = m.nx, ny = m.ny;
    if (is_zface(z, m)) {
        for (int y = threadIdx.x >> 5; y < ny; y += blockDim.x >> 5)
            for (int x = threadIdx.x & 31; x < nx; x += 32) plane[y * P + x] = val;
    } else {
        for (int x = threadIdx.x; x < nx; x += blockDim.x) {
            plane[x] = val;
            plane[(ny - 1) * P + x] = val;
        }
        for (int y = threadIdx.x; y < ny; y += blockDim.x) {
            plane[y * P] = val;
            plane[y * P + nx - 1] = val;
        }
    }
}

// Fused G4 exchange for the non-empty voxels q in [q0, q1) (a contiguous run
// of the ascending non-empty list: the voxels of one staged tile).  Their
// cells occupy the contiguous id-sorted slots [ne_start[q], ne_start[q+1]),
// so rho = (rho + A_k) / D_k runs over them in ascending id
// (diffusion.py:219-229).  `at(v)` maps a voxel to its staged smem slot.
template <typename At>
__device__ __forceinline__ void exchange_tile(int q0, int q1, const int32_t* __restrict__ nonempty,
                                              const int32_t* __restrict__ ne_start,
                                              const double* __restrict__ A,
                                              const double* __restrict__ D, At at) {
    for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
        const int v = nonempty[q];
        const int k0 = ne_start[q], k1 = ne_start[q + 1];
        double a = A[k0], d = D[k0];
        double* cell = at(v);
        double rho = (*cell + a) / d;
        for (int k = k0 + 1; k < k1; k++) rho = (rho + A[k]) / D[k];
        *cell = rho;
    }
}

// Exchange records: {A, D} of the first kRecCells cells of every non-empty
// voxel, inline per voxel (written by the bin fix-up), so the exchange needs
// no dependent load for voxels with <= kRecCells cells.
constexpr int kRecCells = 4;

struct ExchArgs {
    const int32_t* nonempty;  // ascending non-empty voxels
    const int32_t* ne_start;  // id-sorted slot offset of each non-empty voxel (+1 sentinel)
    const int32_t* row_ne;    // non-empty voxels before each row start (nz*ny + 1)
    const double* A;          // (S, n) (f*sec)*sat in id-sorted slot order
    const double* D;          // (S, n) 1 + f*(sec+upt)
    int n_cells;
    const double* R;          // (S, rq, 2 kRecCells): per non-empty voxel {A, D} of its first cells
    int rq;
};

// Plane row pitch in doubles: even, so every staged row is 16B aligned for
// the TMA bulk copies, and == 2 (mod 4), so the x sweep's row-per-lane
// accesses are at most 2-way bank conflicted.
__host__ __device__ __forceinline__ int plane_pitch(int nx) { return ((nx + 2) & ~1) | 2; }

// ---------------------------------------------------------------- register lines
// Whole line of exactly N elements held in registers: the sweep reads and
// writes each element once (the streaming solve_line reads and writes it
// twice), in the same operation order as diffusion.py:102-112.  N is a
// compile-time constant so every element address is an immediate offset
// from one base register (no per-element address registers, no spills).
// inv/gam: the line's factors in kernel parameter space (LineFactors, a
// __grid_constant__ argument) at compile-time offsets -- uniform constant
// loads, no vector registers or shared-memory traffic.
template <int N>
__device__ __forceinline__ void solve_regs(double (&w)[N], const double (&inv)[N],
                                           const double (&gam)[N], double r) {
    double prev = w[0] * inv[0];
    w[0] = prev;
#pragma unroll
    for (int i = 1; i < N; i++) {
        prev = (w[i] + r * prev) * inv[i];
        w[i] = prev;
    }
    double next = prev;
#pragma unroll
    for (int i = N - 2; i >= 0; i--) {
        next = w[i] + gam[i] * next;
        w[i] = next;
    }
}

// Same recurrence with the factors in shared memory.  Compiler barriers
// every 8 steps keep the factor loads near their use (hoisting all 2N of
// them would spill the line).
template <int N>
__device__ __forceinline__ void solve_regs_smem(double (&w)[N], const double* __restrict__ inv,
                                                const double* __restrict__ gam, double r) {
    double prev = w[0] * inv[0];
    w[0] = prev;
#pragma unroll
    for (int i = 1; i < N; i++) {
        if (i % 8 == 0) asm volatile("" ::: "memory");
        prev = (w[i] + r * prev) * inv[i];
        w[i] = prev;
    }
    double next = prev;
#pragma unroll
    for (int i = N - 2; i >= 0; i--) {
        if (i % 8 == 7) asm volatile("" ::: "memory");
        next = w[i] + gam[i] * next;
        w[i] = next;
    }
}

// Branch-free select on a register line element.
__device__ __forceinline__ double selp_f64(bool p, double a, double b) {
    double r;
    asm("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\nselp.f64 %0, %1, %2, q;\n}"
        : "=d"(r) : "d"(a), "d"(b), "r"((int)p));
    return r;
}

// Relay register lines: a line of N = K * M elements too long for one
// thread's registers (config 3: 160) is held by K lanes of one warp, M
// consecutive elements each.  Lanes l and l + 32/K hold adjacent segments of
// the same line (seg = lane / (32/K)).  The forward recurrence runs segment
// by segment, the running value handed to the next segment's lane with a
// warp shuffle; the backward one runs back the same way.  Every element sees
// exactly the operations of solve_regs in the same order, so the result is
// bit-identical to the single-thread solve (diffusion.py:102-112); the lanes
// of the other segments idle meanwhile, which costs issue slots but not
// latency, and the chain is what bounds these sweeps.
// inv/gam: the whole line's factors (shared memory or a grid-constant
// parameter array); the segment offsets are compile-time after unrolling.
template <int M, int K, typename F>
__device__ __forceinline__ void solve_relay(double (&w)[M], const F& inv, const F& gam, double r,
                                            int seg, int lane_in_seg) {
    constexpr int LPW = 32 / K;
    double prev = 0.0;
#pragma unroll
    for (int jp = 0; jp < K; jp++) {
        if (seg == jp) {
            if (jp == 0) prev = w[0] * inv[0];
            else prev = (w[0] + r * prev) * inv[jp * M];
            w[0] = prev;
#pragma unroll
            for (int i = 1; i < M; i++) {
                if (i % 8 == 0) asm volatile("" ::: "memory");
                prev = (w[i] + r * prev) * inv[jp * M + i];
                w[i] = prev;
            }
        }
        if (jp + 1 < K) prev = __shfl_sync(0xffffffffu, prev, jp * LPW + lane_in_seg);
    }
    // backward from d[N-1] (the last segment's final forward value)
    double next = prev;
#pragma unroll
    for (int jp = K - 1; jp >= 0; jp--) {
        if (seg == jp) {
            if (jp == K - 1) {
#pragma unroll
                for (int i = M - 2; i >= 0; i--) {
                    if (i % 8 == 7) asm volatile("" ::: "memory");
                    next = w[i] + gam[jp * M + i] * next;
                    w[i] = next;
                }
            } else {
#pragma unroll
                for (int i = M - 1; i >= 0; i--) {
                    if (i % 8 == 7) asm volatile("" ::: "memory");
                    next = w[i] + gam[jp * M + i] * next;
                    w[i] = next;
                }
            }
        }
        if (jp > 0) next = __shfl_sync(0xffffffffu, next, jp * LPW + lane_in_seg);
    }
}

// G1 pins of one segment of a relay line (pin_line restricted to it).
template <int M>
__device__ __forceinline__ void pin_seg(double (&w)[M], bool full, bool first, bool last, double dv) {
    if (first) w[0] = dv;
    if (last) w[M - 1] = dv;
#pragma unroll
    for (int i = 0; i < M; i++) w[i] = selp_f64(full, dv, w[i]);
}

// Factors of the register-line kernels for every (substrate, axis).
constexpr int kLineMaxS = 4;
template <int N>
struct LineFactors {
    double inv[kLineMaxS][3][N];
    double gam[kLineMaxS][3][N];
    double r[kLineMaxS][3];
};

