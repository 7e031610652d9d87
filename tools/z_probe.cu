// Back-to-back timing of z-sweep / plane kernel variants on config 1 sizes
// (80^3 x 3, Dirichlet): streaming vs register lines, factor sources.
#include "../paper_2306_11544_b200/csrc/diffusion.cu"
#include <cstdio>
#include <vector>

// V2: register lines, factors staged in shared memory.
template <int NL>
__global__ void __launch_bounds__(64) kz_smemfac(double* __restrict__ dens, MeshDev m,
                                                 const double* __restrict__ fac,
                                                 const double* __restrict__ rr, int nmax) {
    __shared__ double f[2 * NL];
    const int s = blockIdx.y, nz = m.nz;
    const long plane_sz = (long)m.nx * m.ny;
    const double* fz = fac + (long)(s * 3 + 2) * 2 * nmax;
    for (int i = threadIdx.x; i < nz; i += blockDim.x) { f[i] = fz[i]; f[NL + i] = fz[nmax + i]; }
    __syncthreads();
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= plane_sz) return;
    double* col = dens + (long)s * nz * plane_sz + p;
    double w[NL];
#pragma unroll
    for (int i = 0; i < NL; i++) w[i] = col[i * plane_sz];
    const double r = rr[s * 3 + 2];
    double prev = w[0] * f[0];
    w[0] = prev;
#pragma unroll
    for (int i = 1; i < NL; i++) { prev = (w[i] + r * prev) * f[i]; w[i] = prev; }
    double next = prev;
#pragma unroll
    for (int i = NL - 2; i >= 0; i--) { next = w[i] + f[NL + i] * next; w[i] = next; }
#pragma unroll
    for (int i = 0; i < NL; i++) col[i * plane_sz] = w[i];
}

// V3: same, no launch bounds
template <int NL>
__global__ void kz_smemfac_nb(double* __restrict__ dens, MeshDev m, const double* __restrict__ fac,
                              const double* __restrict__ rr, int nmax) {
    __shared__ double f[2 * NL];
    const int s = blockIdx.y, nz = m.nz;
    const long plane_sz = (long)m.nx * m.ny;
    const double* fz = fac + (long)(s * 3 + 2) * 2 * nmax;
    for (int i = threadIdx.x; i < nz; i += blockDim.x) { f[i] = fz[i]; f[NL + i] = fz[nmax + i]; }
    __syncthreads();
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= plane_sz) return;
    double* col = dens + (long)s * nz * plane_sz + p;
    double w[NL];
#pragma unroll
    for (int i = 0; i < NL; i++) w[i] = col[i * plane_sz];
    const double r = rr[s * 3 + 2];
    double prev = w[0] * f[0];
    w[0] = prev;
#pragma unroll
    for (int i = 1; i < NL; i++) { prev = (w[i] + r * prev) * f[i]; w[i] = prev; }
    double next = prev;
#pragma unroll
    for (int i = NL - 2; i >= 0; i--) { next = w[i] + f[NL + i] * next; w[i] = next; }
#pragma unroll
    for (int i = 0; i < NL; i++) col[i * plane_sz] = w[i];
}

// V4: 2 threads per column (40 elements each), hand-off through shuffles.
template <int NH>
__global__ void __launch_bounds__(128) kz_half(double* __restrict__ dens, MeshDev m,
                                               const double* __restrict__ fac,
                                               const double* __restrict__ rr, int nmax) {
    __shared__ double f[4 * NH];
    const int s = blockIdx.y, nz = m.nz;
    const long plane_sz = (long)m.nx * m.ny;
    const double* fz = fac + (long)(s * 3 + 2) * 2 * nmax;
    for (int i = threadIdx.x; i < nz; i += blockDim.x) { f[i] = fz[i]; f[2 * NH + i] = fz[nmax + i]; }
    __syncthreads();
    const int lane = threadIdx.x & 31, h = lane >> 4;  // half-warp 0: first half of 16 columns
    const long p = ((long)blockIdx.x * blockDim.x + threadIdx.x) / 32 * 16 + (lane & 15);
    const bool ok = p < plane_sz;
    double* col = dens + (long)s * nz * plane_sz + (ok ? p : 0) + (long)h * NH * plane_sz;
    const double* inv = f + h * NH;
    const double* gam = f + 2 * NH + h * NH;
    double w[NH];
#pragma unroll
    for (int i = 0; i < NH; i++) w[i] = ok ? col[i * plane_sz] : 0.0;
    const double r = rr[s * 3 + 2];
    double prev = 0.0;
    // forward: half 0 then half 1
    if (h == 0) {
        prev = w[0] * inv[0];
        w[0] = prev;
#pragma unroll
        for (int i = 1; i < NH; i++) { prev = (w[i] + r * prev) * inv[i]; w[i] = prev; }
    }
    prev = __shfl_sync(0xffffffffu, prev, lane & 15);
    if (h == 1) {
#pragma unroll
        for (int i = 0; i < NH; i++) { prev = (w[i] + r * prev) * inv[i]; w[i] = prev; }
    }
    double next = prev;
    if (h == 1) {
#pragma unroll
        for (int i = NH - 2; i >= 0; i--) { next = w[i] + gam[i] * next; w[i] = next; }
    }
    next = __shfl_sync(0xffffffffu, next, 16 + (lane & 15));
    if (h == 0) {
#pragma unroll
        for (int i = NH - 1; i >= 0; i--) { next = w[i] + gam[i] * next; w[i] = next; }
    }
    if (ok) {
#pragma unroll
        for (int i = 0; i < NH; i++) col[i * plane_sz] = w[i];
    }
}

// Memory pattern only: the z-column read + write with no arithmetic.
__global__ void __launch_bounds__(64) k_touch(double* __restrict__ dens, long plane_sz, int nz) {
    const long p = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= plane_sz) return;
    double* col = dens + (long)blockIdx.y * nz * plane_sz + p;
    double w[80];
#pragma unroll
    for (int i = 0; i < 80; i++) w[i] = col[i * plane_sz];
#pragma unroll
    for (int i = 0; i < 80; i++) col[i * plane_sz] = w[i] * 1.0000001;
}
// Flat streaming copy-in-place (vectorised).
__global__ void k_flat(double2* __restrict__ d, long n2) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
        double2 v = d[i];
        v.x *= 1.0000001; v.y *= 1.0000001;
        d[i] = v;
    }
}
// Arithmetic only: the 80-step chain on registers.
__global__ void __launch_bounds__(64) k_chain(double* __restrict__ out, const double* __restrict__ f, double r) {
    double w[80];
#pragma unroll
    for (int i = 0; i < 80; i++) w[i] = threadIdx.x + i;
    double prev = w[0] * f[0];
    w[0] = prev;
#pragma unroll
    for (int i = 1; i < 80; i++) { prev = (w[i] + r * prev) * f[i]; w[i] = prev; }
    double next = prev;
#pragma unroll
    for (int i = 78; i >= 0; i--) { next = w[i] + f[80 + i] * next; w[i] = next; }
    double acc = 0;
#pragma unroll
    for (int i = 0; i < 80; i++) acc += w[i];
    out[(long)blockIdx.y * gridDim.x * blockDim.x + blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_empty() {}

template <int N>
struct LF { double inv[3][N]; double gam[3][N]; double r[3]; };
template <int N, int SI>
__device__ __forceinline__ void zc_gc(double* __restrict__ dens, const LF<N>& lf, int p) {
    constexpr long PS = (long)N * N;
    double* col = dens + (long)SI * N * PS + p;
    double w[N];
#pragma unroll
    for (int i = 0; i < N; i++) w[i] = col[i * PS];
    const double r = lf.r[SI];
    double prev = w[0] * lf.inv[SI][0];
    w[0] = prev;
#pragma unroll
    for (int i = 1; i < N; i++) { prev = (w[i] + r * prev) * lf.inv[SI][i]; w[i] = prev; }
    double next = prev;
#pragma unroll
    for (int i = N - 2; i >= 0; i--) { next = w[i] + lf.gam[SI][i] * next; w[i] = next; }
#pragma unroll
    for (int i = 0; i < N; i++) col[i * PS] = w[i];
}
template <int N>
__global__ void __launch_bounds__(64, 1) kz_gc(double* __restrict__ dens, const __grid_constant__ LF<N> lf) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N * N) return;
    switch (blockIdx.y) {
        case 0: zc_gc<N, 0>(dens, lf, p); break;
        case 1: zc_gc<N, 1>(dens, lf, p); break;
        default: zc_gc<N, 2>(dens, lf, p); break;
    }
}

// TMA-staged z variant: 80 bulk row copies (512 B) into smem, columns into
// registers, solve with smem factors, direct global stores.
template <int N>
__global__ void __launch_bounds__(64, 1) kz_tma(double* __restrict__ dens, const double* __restrict__ fac,
                                                const double* __restrict__ rr, int nmax) {
    __shared__ __align__(16) double tile[N * 64];
    __shared__ double f[2 * N];
    __shared__ __align__(8) unsigned long long bar;
    constexpr long PS = (long)N * N;
    const int s = blockIdx.y, t = threadIdx.x;
    const long p0 = (long)blockIdx.x * 64;
    double* g = dens + (long)s * N * PS + p0;
    if (t == 0) { mbar_init(&bar, 1); }
    __syncthreads();
    if (t == 0) {
        mbar_expect_tx(&bar, N * 64 * 8);
        for (int i = 0; i < N; i++) bulk_g2s(tile + i * 64, g + i * PS, 512, &bar);
    }
    const double* fz = fac + (long)(s * 3 + 2) * 2 * nmax;
    for (int i = t; i < N; i += 64) { f[i] = fz[i]; f[N + i] = fz[nmax + i]; }
    mbar_wait(&bar, 0);
    __syncthreads();
    double w[N];
#pragma unroll
    for (int i = 0; i < N; i++) w[i] = tile[i * 64 + t];
    solve_regs_smem<N>(w, f, f + N, rr[s * 3 + 2]);
#pragma unroll
    for (int i = 0; i < N; i++) g[i * PS + t] = w[i];
}
// TMA touch: bulk load + direct stores, no math
template <int N>
__global__ void __launch_bounds__(64, 1) kz_tma_touch(double* __restrict__ dens) {
    __shared__ __align__(16) double tile[N * 64];
    __shared__ __align__(8) unsigned long long bar;
    constexpr long PS = (long)N * N;
    const int s = blockIdx.y, t = threadIdx.x;
    double* g = dens + (long)s * N * PS + (long)blockIdx.x * 64;
    if (t == 0) { mbar_init(&bar, 1); }
    __syncthreads();
    if (t == 0) {
        mbar_expect_tx(&bar, N * 64 * 8);
        for (int i = 0; i < N; i++) bulk_g2s(tile + i * 64, g + i * PS, 512, &bar);
    }
    mbar_wait(&bar, 0);
#pragma unroll 8
    for (int i = 0; i < N; i++) g[i * PS + t] = tile[i * 64 + t] * 1.0000001;
}

int main() {
    const int N = 80, S = 3;
    MeshDev m{N, N, N, 20, 20, 20, 0, 0, 0, make_fastdiv(N), make_fastdiv(N)};
    m.zlo = m.zhi = true;
    const long nvox = (long)N * N * N, plane = (long)N * N;
    double *dens, *ref, *fac, *rr, *diri;
    cudaMalloc(&dens, S * nvox * 8); cudaMalloc(&ref, S * nvox * 8);
    cudaMalloc(&fac, S * 3 * 2 * N * 8); cudaMalloc(&rr, S * 3 * 8); cudaMalloc(&diri, S * 8);
    std::vector<double> h(S * nvox), f(S * 3 * 2 * N), r(S * 3);
    for (long i = 0; i < S * nvox; i++) h[i] = 1.0 + (i % 977) * 1e-3;
    for (int s = 0; s < S; s++) for (int a = 0; a < 3; a++) {
        double rv = 2.5 / (1 + s), lam = 1e-4;
        r[s * 3 + a] = rv;
        host_line_factors(N, rv, lam, &f[((s * 3 + a) * 2) * N], &f[((s * 3 + a) * 2 + 1) * N]);
    }
    cudaMemcpy(fac, f.data(), f.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(rr, r.data(), r.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(diri, 0, S * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto reset = [&] { cudaMemcpy(dens, h.data(), S * nvox * 8, cudaMemcpyHostToDevice); };
    auto check = [&](const char* name) {
        std::vector<double> x(S * nvox), y(S * nvox);
        cudaMemcpy(x.data(), dens, S * nvox * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(y.data(), ref, S * nvox * 8, cudaMemcpyDeviceToHost);
        long bad = 0; for (long i = 0; i < S * nvox; i++) bad += x[i] != y[i];
        printf("   %-28s mismatches vs streaming: %ld\n", name, bad);
    };
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    auto timeit = [&](const char* name, auto launch) {
        // 100 launches captured in one graph: in-graph launch gaps (~0.6 us)
        // instead of the stream submit rate.
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        cudaStream_t save = 0;
        (void)save;
        for (int i = 0; i < 100; i++) launch(st);
        cudaGraph_t g; cudaStreamEndCapture(st, &g);
        cudaGraphExec_t ge; cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-40s %8.2f us  %s\n", name, ms * 10, cudaGetErrorString(cudaGetLastError()));
        cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    };
    size_t zs = cols_smem_bytes(N, 64);
    cudaFuncSetAttribute(k_cols<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zs);
    auto stream_z = [&](cudaStream_t s_) { k_cols<2, false><<<dim3(plane / 64, S), 256, zs, s_>>>(dens, m, fac, rr, N, diri, 64); };
    cudaStream_t s_ = 0;
    reset(); stream_z(0); cudaMemcpy(ref, dens, S * nvox * 8, cudaMemcpyDeviceToDevice);
    reset(); kz_smemfac<80><<<dim3(plane / 64, S), 64, 0, s_>>>(dens, m, fac, rr, N); check("smemfac");
    reset(); kz_smemfac_nb<80><<<dim3(plane / 64, S), 64, 0, s_>>>(dens, m, fac, rr, N); check("smemfac_nb");
    reset(); kz_half<40><<<dim3(plane * 2 / 128, S), 128, 0, s_>>>(dens, m, fac, rr, N); check("half");
    timeit("z streaming k_cols<2> TC=64", stream_z);
    timeit("z reg smem factors (lb 64)", [&](cudaStream_t s_) { kz_smemfac<80><<<dim3(plane / 64, S), 64, 0, s_>>>(dens, m, fac, rr, N); });
    timeit("z reg smem factors (no lb) 64", [&](cudaStream_t s_) { kz_smemfac_nb<80><<<dim3(plane / 64, S), 64, 0, s_>>>(dens, m, fac, rr, N); });
    timeit("z reg smem factors (no lb) 128", [&](cudaStream_t s_) { kz_smemfac_nb<80><<<dim3(plane / 128, S), 128, 0, s_>>>(dens, m, fac, rr, N); });
    timeit("z half-lines 2x40", [&](cudaStream_t s_) { kz_half<40><<<dim3(plane * 2 / 128, S), 128, 0, s_>>>(dens, m, fac, rr, N); });
    {
        static LF<80> lf;
        for (int s2 = 0; s2 < S; s2++) { for (int i = 0; i < N; i++) { lf.inv[s2][i] = f[((s2 * 3 + 2) * 2) * N + i]; lf.gam[s2][i] = f[((s2 * 3 + 2) * 2 + 1) * N + i]; } lf.r[s2] = r[s2 * 3 + 2]; }
        reset(); kz_gc<80><<<dim3(plane / 64, S), 64>>>(dens, lf); check("z grid-const compile-time N");
        timeit("z grid-const compile-time N", [&](cudaStream_t s_) { kz_gc<80><<<dim3(plane / 64, S), 64, 0, s_>>>(dens, lf); });
    }
    reset(); kz_tma<80><<<dim3(plane / 64, S), 64>>>(dens, fac, rr, N); check("z tma staged");
    timeit("z tma staged + reg solve", [&](cudaStream_t s_) { kz_tma<80><<<dim3(plane / 64, S), 64, 0, s_>>>(dens, fac, rr, N); });
    timeit("z tma touch", [&](cudaStream_t s_) { kz_tma_touch<80><<<dim3(plane / 64, S), 64, 0, s_>>>(dens); });
    timeit("touch (z pattern, no math)", [&](cudaStream_t s_) { k_touch<<<dim3(plane / 64, S), 64, 0, s_>>>(dens, plane, N); });
    timeit("flat in-place 12.3 MB, 148x4x256", [&](cudaStream_t s_) { k_flat<<<148 * 4, 256, 0, s_>>>((double2*)dens, S * nvox / 2); });
    timeit("flat in-place 12.3 MB, 2400x256", [&](cudaStream_t s_) { k_flat<<<2400, 256, 0, s_>>>((double2*)dens, S * nvox / 2); });
    timeit("chain only (300x64 threads)", [&](cudaStream_t s_) { k_chain<<<dim3(plane / 64, S), 64, 0, s_>>>(ref, fac, 2.5); });
    timeit("empty 300 CTAs", [&](cudaStream_t s_) { k_empty<<<dim3(plane / 64, S), 64, 0, s_>>>(); });
    // plane kernels
    ExchArgs ex{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
    size_t ps = plane_smem_bytes(m);
    cudaFuncSetAttribute(k_plane_xy<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps);
    cudaFuncSetAttribute(k_plane_xy_reg<false, false, 80>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps);
    auto stream_xy = [&](cudaStream_t s_) { k_plane_xy<false, false><<<dim3(N, S), 256, ps, s_>>>(dens, m, fac, rr, N, diri, ex); };
    reset(); stream_xy(0); cudaMemcpy(ref, dens, S * nvox * 8, cudaMemcpyDeviceToDevice);
    reset(); k_plane_xy_reg<false, false, 80><<<dim3(N, S), 128, ps, s_>>>(dens, m, fac, rr, N, diri, ex); check("plane reg");
    timeit("xy streaming k_plane_xy", stream_xy);
    timeit("xy reg k_plane_xy_reg", [&](cudaStream_t s_) { k_plane_xy_reg<false, false, 80><<<dim3(N, S), 128, ps, s_>>>(dens, m, fac, rr, N, diri, ex); });
    cudaFuncSetAttribute(k_plane_xy<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps);
    cudaFuncSetAttribute(k_plane_xy_reg<false, true, 80>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps);
    timeit("xy streaming DIRI", [&](cudaStream_t s_) { k_plane_xy<false, true><<<dim3(N, S), 256, ps, s_>>>(dens, m, fac, rr, N, diri, ex); });
    timeit("xy reg DIRI", [&](cudaStream_t s_) { k_plane_xy_reg<false, true, 80><<<dim3(N, S), 128, ps, s_>>>(dens, m, fac, rr, N, diri, ex); });
    return 0;
}
