// Time the persistent LOD kernel's phases (globaltimer, ns) on config-1 sizes.
#define CG_PROBE 1
#include "../paper_2306_11544_b200/csrc/diffusion.cu"
#include <cstdio>
#include <vector>

__device__ unsigned long long g_ts[4096][8];
__device__ __forceinline__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <bool DIRI>
__global__ void __launch_bounds__(256) k_probe_persistent(double* dens, MeshDev m, const double* fac, const double* rr, int nmax,
                                                          const double* diri, ExchArgs ex, int S, int TC) {
    extern __shared__ double sm[];
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    unsigned phase = 0;
    cg::grid_group grid = cg::this_grid();
    const int planes = m.nz * S;
    const long plane_sz = (long)m.nx * m.ny;
    const int tiles = (int)((plane_sz + TC - 1) / TC);
    if (threadIdx.x == 0) g_ts[blockIdx.x][0] = gtime();
    for (int item = blockIdx.x; item < planes; item += gridDim.x)
        plane_body<false, DIRI>(sm, &bar, phase, dens, m, fac, rr, nmax, diri, ex, item % m.nz, item / m.nz);
    if (threadIdx.x == 0) g_ts[blockIdx.x][1] = gtime();
    grid.sync();
    if (threadIdx.x == 0) g_ts[blockIdx.x][2] = gtime();
    for (int item = blockIdx.x; item < tiles * S; item += gridDim.x)
        cols_body<2, DIRI>(sm, &bar, phase, dens, m, fac, rr, nmax, diri, item % tiles, item / tiles, TC);
    if (threadIdx.x == 0) g_ts[blockIdx.x][3] = gtime();
    grid.sync();
    if (threadIdx.x == 0) g_ts[blockIdx.x][4] = gtime();
}

int main() {
    const int N = 80, S = 3;
    MeshDev m{N, N, N, 20, 20, 20, 0, 0, 0, make_fastdiv(N), make_fastdiv(N)};
    const long nvox = (long)N * N * N;
    double *dens, *fac, *rr, *diri;
    cudaMalloc(&dens, S * nvox * 8); cudaMalloc(&fac, S * 3 * 2 * N * 8); cudaMalloc(&rr, S * 3 * 8); cudaMalloc(&diri, S * 8);
    std::vector<double> h(S * nvox, 1.0), f(S * 3 * 2 * N, 0.4), r(S * 3, 2.5);
    cudaMemcpy(dens, h.data(), S * nvox * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(fac, f.data(), f.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(rr, r.data(), r.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(diri, r.data(), S * 8, cudaMemcpyHostToDevice);
    ExchArgs ex{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
    for (int TC : {64, 128}) {
        size_t smem = std::max(plane_smem_bytes(m), cols_smem_bytes(N, TC));
        auto kern = k_probe_persistent<true>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
        int grid = std::min(per_sm * 148, N * S);
        int nmax = N, SS = S;
        void* args[] = {&dens, &m, &fac, &rr, &nmax, &diri, &ex, &SS, &TC};
        for (int it = 0; it < 3; it++) cudaLaunchCooperativeKernel((void*)kern, grid, 256, args, smem, 0);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> ts(4096 * 8);
        cudaMemcpyFromSymbol(ts.data(), g_ts, ts.size() * 8);
        unsigned long long t0 = ~0ull, p1max = 0, s1 = 0, p2max = 0, s2 = 0;
        double p1sum = 0, p2sum = 0;
        for (int b = 0; b < grid; b++) {
            unsigned long long* t = &ts[8 * b];
            t0 = std::min(t0, t[0]);
        }
        for (int b = 0; b < grid; b++) {
            unsigned long long* t = &ts[8 * b];
            p1max = std::max(p1max, t[1] - t0); s1 = std::max(s1, t[2] - t0);
            p2max = std::max(p2max, t[3] - t0); s2 = std::max(s2, t[4] - t0);
            p1sum += t[1] - t[0]; p2sum += t[3] - t[2];
        }
        printf("TC=%d grid=%d per_sm=%d: phase1 end %.2f us (avg CTA %.2f)  sync1 %.2f  phase2 end %.2f (avg CTA %.2f)  sync2 %.2f  (%s)\n",
               TC, grid, per_sm, p1max / 1e3, p1sum / grid / 1e3, s1 / 1e3, p2max / 1e3, p2sum / grid / 1e3, s2 / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
