// Phase timing (clock64) of the x+y plane kernel on config 1 (80^3 x 3).
#define CG_PROBE 1
#include "../paper_2306_11544_b200/csrc/diffusion.cu"
#include <cstdio>
#include <vector>

__global__ void __launch_bounds__(256) k_probe(double* dens, MeshDev m, const double* fac,
                                               const double* rr, int nmax, long long* clk) {
    extern __shared__ double sm[];
    const int nx = m.nx, ny = m.ny, P = nx | 1;
    const long plane_sz = (long)nx * ny;
    const int z = blockIdx.x, s = blockIdx.y;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* plane = sm;
    double* fx = plane + (long)ny * P;
    double* fy = fx + 2 * nx;
    double* g = dens + ((long)s * m.nz + z) * plane_sz;
    long long t0 = clock64();
    for (int y = wid; y < ny; y += nw)
        for (int x = lane; x < nx; x += 32) cp_async8(plane + y * P + x, g + (long)y * nx + x);
    const double* facx = fac + (long)(s * 3 + 0) * 2 * nmax;
    const double* facy = fac + (long)(s * 3 + 1) * 2 * nmax;
    for (int i = threadIdx.x; i < nx; i += blockDim.x) { cp_async8(fx + i, facx + i); cp_async8(fx + nx + i, facx + nmax + i); }
    for (int i = threadIdx.x; i < ny; i += blockDim.x) { cp_async8(fy + i, facy + i); cp_async8(fy + ny + i, facy + nmax + i); }
    cp_async_wait_all();
    __syncthreads();
    long long t1 = clock64();
    const double rx = rr[s * 3 + 0], ry = rr[s * 3 + 1];
    for (int y = threadIdx.x; y < ny; y += blockDim.x) solve_line(plane + y * P, 1, nx, fx, fx + nx, rx);
    __syncthreads();
    long long t2 = clock64();
    for (int x = threadIdx.x; x < nx; x += blockDim.x) solve_line(plane + x, P, ny, fy, fy + ny, ry);
    __syncthreads();
    long long t3 = clock64();
    for (int y = wid; y < ny; y += nw)
        for (int x = lane; x < nx; x += 32) g[(long)y * nx + x] = plane[y * P + x];
    __syncthreads();
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        long long* c = clk + 5 * (blockIdx.y * gridDim.x + blockIdx.x);
        c[0] = t0; c[1] = t1 - t0; c[2] = t2 - t1; c[3] = t3 - t2; c[4] = t4 - t3;
    }
}

int main() {
    const int N = 80, S = 3;
    MeshDev m{N, N, N, 20, 20, 20, 0, 0, 0, make_fastdiv(N), make_fastdiv(N)};
    const long nvox = (long)N * N * N;
    double *dens, *fac, *rr; long long* clk;
    cudaMalloc(&dens, S * nvox * 8); cudaMalloc(&fac, S * 3 * 2 * N * 8); cudaMalloc(&rr, S * 3 * 8);
    cudaMalloc(&clk, 5 * N * S * 8);
    std::vector<double> h(S * nvox, 1.0), f(S * 3 * 2 * N, 0.4), r(S * 3, 2.5);
    cudaMemcpy(dens, h.data(), S * nvox * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(fac, f.data(), f.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(rr, r.data(), r.size() * 8, cudaMemcpyHostToDevice);
    size_t smem = ((size_t)N * (N | 1) + 4 * N) * 8;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int threads : {96, 256}) {
        for (int it = 0; it < 3; it++) k_probe<<<dim3(N, S), threads, smem>>>(dens, m, fac, rr, N, clk);
        cudaDeviceSynchronize();
        std::vector<long long> c(5 * N * S);
        cudaMemcpy(c.data(), clk, c.size() * 8, cudaMemcpyDeviceToHost);
        double acc[5] = {0}; long long t0min = c[0], t0max = c[0];
        for (int b = 0; b < N * S; b++) { for (int k = 1; k < 5; k++) acc[k] += c[5 * b + k]; t0min = std::min(t0min, c[5*b]); t0max = std::max(t0max, c[5*b]); }
        printf("threads=%d  avg cycles: load %.0f  x-sweep %.0f  y-sweep %.0f  store %.0f   start spread %lld cyc  (%s)\n", threads,
               acc[1] / (N * S), acc[2] / (N * S), acc[3] / (N * S), acc[4] / (N * S), t0max - t0min, cudaGetErrorString(cudaGetLastError()));
    }
    int main2();
    return main2();
}
// (appended) back-to-back timing of the library's k_plane_xy / k_cols<2>
int main2() {
    const int N = 80, S = 3;
    MeshDev m{N, N, N, 20, 20, 20, 0, 0, 0, make_fastdiv(N), make_fastdiv(N)};
    const long nvox = (long)N * N * N;
    double *dens, *fac, *rr, *diri;
    cudaMalloc(&dens, S * nvox * 8); cudaMalloc(&fac, S * 3 * 2 * N * 8); cudaMalloc(&rr, S * 3 * 8);
    cudaMalloc(&diri, S * 8);
    std::vector<double> h(S * nvox, 1.0), f(S * 3 * 2 * N, 0.4), r(S * 3, 2.5);
    cudaMemcpy(dens, h.data(), S * nvox * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(fac, f.data(), f.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(rr, r.data(), r.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(diri, r.data(), S * 8, cudaMemcpyHostToDevice);
    ExchArgs ex{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
    size_t smem = plane_smem_bytes(m);
    cudaFuncSetAttribute(k_plane_xy<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_plane_xy<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        for (int i = 0; i < 5; i++) launch();
        cudaEventRecord(a);
        for (int i = 0; i < 100; i++) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-40s %8.2f us  %s\n", name, ms * 10, cudaGetErrorString(cudaGetLastError()));
    };
    for (int thr : {96, 128, 256})
        { char nm[64]; snprintf(nm, 64, "plane_xy<F,T> thr=%d", thr);
          timeit(nm, [&] { k_plane_xy<false, true><<<dim3(N, S), thr, smem>>>(dens, m, fac, rr, N, diri, ex); }); }
    timeit("plane_xy<F,F> thr=256", [&] { k_plane_xy<false, false><<<dim3(N, S), 256, smem>>>(dens, m, fac, rr, N, diri, ex); });
    timeit("plane_xy<F,F> S=1 thr=256", [&] { k_plane_xy<false, false><<<dim3(N, 1), 256, smem>>>(dens, m, fac, rr, N, diri, ex); });
    size_t zs = cols_smem_bytes(N, 64);
    cudaFuncSetAttribute(k_cols<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zs);
    timeit("cols<2,T> TC=64", [&] { k_cols<2, true><<<dim3(N * N / 64, S), 64, zs>>>(dens, m, fac, rr, N, diri, 64); });
    size_t zs2 = cols_smem_bytes(N, 32);
    timeit("cols<2,T> TC=32", [&] { k_cols<2, true><<<dim3(N * N / 32, S), 32, zs2>>>(dens, m, fac, rr, N, diri, 32); });
    {
        // phase probe of the real k_plane_xy<false,true> (Dirichlet, no exchange)
        for (int it = 0; it < 5; it++) k_plane_xy<false, true><<<dim3(N, S), 256, smem>>>(dens, m, fac, rr, N, diri, ex);
        cudaDeviceSynchronize();
        std::vector<long long> pr(8 * N * S);
        cudaMemcpyFromSymbol(pr.data(), g_probe, pr.size() * 8);
        double acc[7] = {0};
        for (int b = 0; b < N * S; b++) for (int k = 1; k < 7; k++) acc[k] += pr[8 * b + k] - pr[8 * b + k - 1];
        printf("k_plane_xy phases (cycles): issue %.0f  wait %.0f  exch %.0f  x %.0f  y %.0f  store %.0f\n",
               acc[1] / (N*S), acc[2] / (N*S), acc[3] / (N*S), acc[4] / (N*S), acc[5] / (N*S), acc[6] / (N*S));
    }
    return 0;
}
