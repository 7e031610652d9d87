// Microbenchmark of z-sweep kernel variants on an 80^3 x 3 fp64 field
// (BASELINE config 1), L2-warm, many back-to-back launches timed by events.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

#define N 80
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// chain only: data already in smem, no global traffic
template <int TC>
__global__ void k_chain(double* out, const double* inv, const double* gam, double r, int n) {
    __shared__ double col[N * TC];
    for (int i = 0; i < n; i++) col[i * TC + threadIdx.x] = 1.0 + i;
    double* d = col + threadIdx.x;
    double prev = d[0] * inv[0]; d[0] = prev;
#pragma unroll 8
    for (int i = 1; i < n; i++) { double c = (d[i * TC] + r * prev) * inv[i]; d[i * TC] = c; prev = c; }
    double next = prev;
#pragma unroll 8
    for (int i = n - 2; i >= 0; i--) { double c = d[i * TC] + gam[i] * next; d[i * TC] = c; next = c; }
    out[blockIdx.x * TC + threadIdx.x] = d[0];
}

// load + store only, no compute
template <int TC>
__global__ void k_copy(double* dens, long plane, int n) {
    __shared__ double col[N * TC];
    long p = blockIdx.x * TC + threadIdx.x;
    double* g = dens + blockIdx.y * plane * n + p;
    for (int i = 0; i < n; i++) cp_async8(col + i * TC + threadIdx.x, g + i * plane);
    cp_async_wait_all();
    __syncthreads();
    for (int i = 0; i < n; i++) g[i * plane] = col[i * TC + threadIdx.x] * 1.0000001;
}

// full: load, solve, store (current library design)
template <int TC>
__global__ void k_full(double* dens, long plane, int n, const double* __restrict__ invg,
                       const double* __restrict__ gamg, double r) {
    __shared__ double col[N * TC];
    __shared__ double inv[N], gam[N];
    long p = blockIdx.x * TC + threadIdx.x;
    double* g = dens + blockIdx.y * plane * n + p;
    for (int i = 0; i < n; i++) cp_async8(col + i * TC + threadIdx.x, g + i * plane);
    for (int i = threadIdx.x; i < n; i += TC) { inv[i] = invg[i]; gam[i] = gamg[i]; }
    cp_async_wait_all();
    __syncthreads();
    double* d = col + threadIdx.x;
    double prev = d[0] * inv[0]; d[0] = prev;
#pragma unroll 8
    for (int i = 1; i < n; i++) { double c = (d[i * TC] + r * prev) * inv[i]; d[i * TC] = c; prev = c; }
    double next = prev;
#pragma unroll 8
    for (int i = n - 2; i >= 0; i--) { double c = d[i * TC] + gam[i] * next; d[i * TC] = c; next = c; }
#pragma unroll 8
    for (int i = 0; i < n; i++) g[i * plane] = d[i * TC];
}

// registers: forward pass streams from global with register prefetch and keeps
// intermediates in smem; backward from smem, stores to global.
template <int TC>
__global__ void k_stream(double* dens, long plane, int n, const double* __restrict__ invg,
                         const double* __restrict__ gamg, double r) {
    __shared__ double col[N * TC];
    __shared__ double inv[N], gam[N];
    long p = blockIdx.x * TC + threadIdx.x;
    double* g = dens + blockIdx.y * plane * n + p;
    for (int i = threadIdx.x; i < n; i += TC) { inv[i] = invg[i]; gam[i] = gamg[i]; }
    __syncthreads();
    double* d = col + threadIdx.x;
    double buf[8];
#pragma unroll
    for (int j = 0; j < 8; j++) buf[j] = g[j * plane];
    double prev = 0.0;
    for (int i0 = 0; i0 < n; i0 += 8) {
        double nb[8];
#pragma unroll
        for (int j = 0; j < 8; j++) nb[j] = (i0 + 8 + j < n) ? g[(i0 + 8 + j) * plane] : 0.0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            int i = i0 + j;
            double c = (i == 0) ? buf[j] * inv[0] : (buf[j] + r * prev) * inv[i];
            d[i * TC] = c; prev = c;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) buf[j] = nb[j];
    }
    double next = prev;
    g[(n - 1) * plane] = next;
#pragma unroll 8
    for (int i = n - 2; i >= 0; i--) { double c = d[i * TC] + gam[i] * next; g[i * plane] = c; next = c; }
}


// chain with results written to a separate smem array (no load-after-store hazard)
template <int TC>
__global__ void k_chain2(double* out, const double* inv, const double* gam, double r, int n, long long* clk) {
    __shared__ double col[N * TC];
    __shared__ double res[N * TC];
    for (int i = 0; i < n; i++) col[i * TC + threadIdx.x] = 1.0 + i;
    __syncthreads();
    long long t0 = clock64();
    unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const double* d = col + threadIdx.x;
    double* o = res + threadIdx.x;
    double prev = d[0] * inv[0]; o[0] = prev;
#pragma unroll 8
    for (int i = 1; i < n; i++) { double c = (d[i * TC] + r * prev) * inv[i]; o[i * TC] = c; prev = c; }
    double next = prev;
#pragma unroll 8
    for (int i = n - 2; i >= 0; i--) { double c = o[i * TC] + gam[i] * next; o[i * TC] = c; next = c; }
    long long t1 = clock64();
    unsigned long long g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    out[blockIdx.x * TC + threadIdx.x] = o[0];
    if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = (long long)(g1 - g0); }
}
// chunk-prefetched chain (the library's solve_line)
template <int TC>
__global__ void k_chain3(double* out, const double* inv, const double* gam, double r, int n, long long* clk) {
    __shared__ double col[N * TC];
    for (int i = 0; i < n; i++) col[i * TC + threadIdx.x] = 1.0 + i;
    __syncthreads();
    long long t0 = clock64();
    double* d = col + threadIdx.x;
    const int st = TC;
    constexpr int CH = 8;
    double prev = d[0] * inv[0];
    d[0] = prev;
    double dv[CH], iv[CH];
#pragma unroll
    for (int j = 0; j < CH; j++) { const int i = 1 + j; dv[j] = i < n ? d[i * st] : 0.0; iv[j] = i < n ? inv[i] : 0.0; }
    for (int i0 = 1; i0 < n; i0 += CH) {
        double dn[CH], in[CH];
#pragma unroll
        for (int j = 0; j < CH; j++) { const int i = i0 + CH + j; dn[j] = i < n ? d[i * st] : 0.0; in[j] = i < n ? inv[i] : 0.0; }
#pragma unroll
        for (int j = 0; j < CH; j++) { if (i0 + j < n) { const double cur = (dv[j] + r * prev) * iv[j]; d[(i0 + j) * st] = cur; prev = cur; } }
#pragma unroll
        for (int j = 0; j < CH; j++) { dv[j] = dn[j]; iv[j] = in[j]; }
    }
    double next = prev;
#pragma unroll
    for (int j = 0; j < CH; j++) { const int i = n - 2 - j; dv[j] = i >= 0 ? d[i * st] : 0.0; iv[j] = i >= 0 ? gam[i] : 0.0; }
    for (int i0 = n - 2; i0 >= 0; i0 -= CH) {
        double dn[CH], gn[CH];
#pragma unroll
        for (int j = 0; j < CH; j++) { const int i = i0 - CH - j; dn[j] = i >= 0 ? d[i * st] : 0.0; gn[j] = i >= 0 ? gam[i] : 0.0; }
#pragma unroll
        for (int j = 0; j < CH; j++) { if (i0 - j >= 0) { const double cur = dv[j] + iv[j] * next; d[(i0 - j) * st] = cur; next = cur; } }
#pragma unroll
        for (int j = 0; j < CH; j++) { dv[j] = dn[j]; iv[j] = gn[j]; }
    }
    long long t1 = clock64();
    out[blockIdx.x * TC + threadIdx.x] = d[0];
    if (blockIdx.x == 0 && threadIdx.x == 0) { clk[2] = t1 - t0; }
}
// factors from registers-free constant cache
__constant__ double cinv[256], cgam[256];
template <int TC>
__global__ void k_chain4(double* out, double r, int n, long long* clk) {
    __shared__ double col[N * TC];
    for (int i = 0; i < n; i++) col[i * TC + threadIdx.x] = 1.0 + i;
    __syncthreads();
    long long t0 = clock64();
    double* d = col + threadIdx.x;
    double prev = d[0] * cinv[0]; d[0] = prev;
#pragma unroll 8
    for (int i = 1; i < n; i++) { double c = (d[i * TC] + r * prev) * cinv[i]; d[i * TC] = c; prev = c; }
    double next = prev;
#pragma unroll 8
    for (int i = n - 2; i >= 0; i--) { double c = d[i * TC] + cgam[i] * next; d[i * TC] = c; next = c; }
    long long t1 = clock64();
    out[blockIdx.x * TC + threadIdx.x] = d[0];
    if (blockIdx.x == 0 && threadIdx.x == 0) { clk[3] = t1 - t0; }
}

template <int TC, bool FMA>
__global__ void k_chain5(double* out, double r, int n, long long* clk, int slot) {
    __shared__ double col[N * TC];
    for (int i = 0; i < n; i++) col[i * TC + threadIdx.x] = 1.0 + i;
    __syncthreads();
    long long t0 = clock64();
    double* d = col + threadIdx.x;
    const int st = TC;
    constexpr int CH = 8;
    double prev = d[0] * cinv[0];
    d[0] = prev;
    double dv[CH];
#pragma unroll
    for (int j = 0; j < CH; j++) { const int i = 1 + j; dv[j] = i < n ? d[i * st] : 0.0; }
    for (int i0 = 1; i0 < n; i0 += CH) {
        double dn[CH];
#pragma unroll
        for (int j = 0; j < CH; j++) { const int i = i0 + CH + j; dn[j] = i < n ? d[i * st] : 0.0; }
#pragma unroll
        for (int j = 0; j < CH; j++) { if (i0 + j < n) { const double cur = FMA ? fma(r, prev, dv[j]) * cinv[i0+j] : (dv[j] + r * prev) * cinv[i0 + j]; d[(i0 + j) * st] = cur; prev = cur; } }
#pragma unroll
        for (int j = 0; j < CH; j++) { dv[j] = dn[j]; }
    }
    double next = prev;
#pragma unroll
    for (int j = 0; j < CH; j++) { const int i = n - 2 - j; dv[j] = i >= 0 ? d[i * st] : 0.0; }
    for (int i0 = n - 2; i0 >= 0; i0 -= CH) {
        double dn[CH];
#pragma unroll
        for (int j = 0; j < CH; j++) { const int i = i0 - CH - j; dn[j] = i >= 0 ? d[i * st] : 0.0; }
#pragma unroll
        for (int j = 0; j < CH; j++) { if (i0 - j >= 0) { const double cur = FMA ? fma(cgam[i0-j], next, dv[j]) : dv[j] + cgam[i0 - j] * next; d[(i0 - j) * st] = cur; next = cur; } }
#pragma unroll
        for (int j = 0; j < CH; j++) { dv[j] = dn[j]; }
    }
    long long t1 = clock64();
    out[blockIdx.x * TC + threadIdx.x] = d[0];
    if (blockIdx.x == 0 && threadIdx.x == 0) { clk[slot] = t1 - t0; }
}
// whole line in registers (compile-time n), factors from constant memory
template <int NN, bool FMA>
__global__ void __launch_bounds__(64) k_regs(double* dens, long plane, double r, long long* clk, int slot) {
    long p = blockIdx.x * 64 + threadIdx.x;
    double* g = dens + blockIdx.y * plane * NN + p;
    double v[NN];
#pragma unroll
    for (int i = 0; i < NN; i++) v[i] = g[i * plane];
    long long t0 = clock64();
    v[0] = v[0] * cinv[0];
#pragma unroll
    for (int i = 1; i < NN; i++) v[i] = FMA ? fma(r, v[i-1], v[i]) * cinv[i] : (v[i] + r * v[i - 1]) * cinv[i];
#pragma unroll
    for (int i = NN - 2; i >= 0; i--) v[i] = FMA ? fma(cgam[i], v[i+1], v[i]) : v[i] + cgam[i] * v[i + 1];
    long long t1 = clock64();
#pragma unroll
    for (int i = 0; i < NN; i++) g[i * plane] = v[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) { clk[slot] = t1 - t0; }
}
int main() {
    const int S = 3, n = N;
    const long plane = N * N, nvox = plane * N;
    double *dens, *inv, *gam, *out;
    cudaMalloc(&dens, S * nvox * 8); cudaMalloc(&inv, 256 * 8); cudaMalloc(&gam, 256 * 8);
    cudaMalloc(&out, S * nvox * 8);
    std::vector<double> h(S * nvox, 1.0), f(256, 0.5);
    cudaMemcpy(dens, h.data(), S * nvox * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(inv, f.data(), 256 * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(gam, f.data(), 256 * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        for (int i = 0; i < 5; i++) launch();
        cudaEventRecord(a);
        const int R = 200;
        for (int i = 0; i < R; i++) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %8.2f us/launch   %s\n", name, 1e3 * ms / R, cudaGetErrorString(cudaGetLastError()));
    };
    timeit("empty-ish chain TC=64", [&] { k_chain<64><<<dim3(100 * S), 64>>>(out, inv, gam, 2.5, n); });
    timeit("chain TC=32", [&] { k_chain<32><<<dim3(200 * S), 32>>>(out, inv, gam, 2.5, n); });
    timeit("copy TC=64", [&] { k_copy<64><<<dim3(100, S), 64>>>(dens, plane, n); });
    timeit("copy TC=32", [&] { k_copy<32><<<dim3(200, S), 32>>>(dens, plane, n); });
    timeit("full TC=64", [&] { k_full<64><<<dim3(100, S), 64>>>(dens, plane, n, inv, gam, 2.5); });
    timeit("full TC=32", [&] { k_full<32><<<dim3(200, S), 32>>>(dens, plane, n, inv, gam, 2.5); });

    timeit("stream TC=32", [&] { k_stream<32><<<dim3(200, S), 32>>>(dens, plane, n, inv, gam, 2.5); });
    timeit("stream TC=64", [&] { k_stream<64><<<dim3(100, S), 64>>>(dens, plane, n, inv, gam, 2.5); });
    long long* clk; cudaMalloc(&clk, 8 * 8);
    timeit("chain2 sep arrays TC=32", [&] { k_chain2<32><<<dim3(200 * S), 32>>>(out, inv, gam, 2.5, n, clk); });
    timeit("chain3 chunked TC=64", [&] { k_chain3<64><<<dim3(100 * S), 64>>>(out, inv, gam, 2.5, n, clk); });
    timeit("chain4 const TC=64", [&] { k_chain4<64><<<dim3(100 * S), 64>>>(out, 2.5, n, clk); });
    timeit("chain5 chunk+const", [&] { k_chain5<64,false><<<dim3(100 * S), 64>>>(out, 2.5, n, clk, 4); });
    timeit("chain5 chunk+const FMA", [&] { k_chain5<64,true><<<dim3(100 * S), 64>>>(out, 2.5, n, clk, 5); });
    timeit("regs N=80", [&] { k_regs<80,false><<<dim3(100, S), 64>>>(dens, plane, 2.5, clk, 6); });
    timeit("regs N=80 FMA", [&] { k_regs<80,true><<<dim3(100, S), 64>>>(dens, plane, 2.5, clk, 7); });
    long long hc[8]; cudaMemcpy(hc, clk, 64, cudaMemcpyDeviceToHost);
    printf("chain5 %.1f  chain5fma %.1f  regs %.1f  regsfma %.1f cyc/step\n", hc[4]/160.0, hc[5]/160.0, hc[6]/160.0, hc[7]/160.0);
    printf("chain2 cycles %lld ns %lld (%.2f GHz) cyc/step %.1f | chain3 cycles %lld cyc/step %.1f | chain4 %lld cyc/step %.1f\n", hc[0], hc[1], (double)hc[0]/hc[1], hc[0]/160.0, hc[2], hc[2]/160.0, hc[3], hc[3]/160.0);
    return 0;
}
