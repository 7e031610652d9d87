// Cycles per element of the library's solve_line (fwd+bwd) for row (stride 1,
// pitch 82) and column (stride 82) access, 1..8 warps per CTA, 1 CTA per SM.
#include "../paper_2306_11544_b200/csrc/diffusion.cu"
#include <cstdio>
#include <vector>

template <int CH>
__global__ void __launch_bounds__(256) k_solve(int mode, int n, double r, long long* clk) {
    extern __shared__ double sm[];
    const int P = 82;
    double* plane = sm;
    double* inv = plane + n * P;
    double* gam = inv + n;
    for (int i = threadIdx.x; i < n * P; i += blockDim.x) plane[i] = 1.0 + i * 1e-4;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { inv[i] = 0.3 + i * 1e-5; gam[i] = 0.2; }
    __syncthreads();
    long long t0 = clock64();
    for (int l = threadIdx.x; l < n; l += blockDim.x) {
        if (mode == 0) solve_line<CH>(plane + l * P, 1, n, inv, gam, r);
        else solve_line<CH>(plane + l, P, n, inv, gam, r);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
    long long* clk; cudaMalloc(&clk, 1024 * 8);
    const int n = 80;
    size_t smem = (n * 82 + 2 * n) * 8;
    auto run = [&](auto kern, int ch) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode : {0, 1})
        for (int threads : {96}) {
            for (int it = 0; it < 3; it++) kern<<<148, threads, smem>>>(mode, n, 2.5, clk);
            cudaDeviceSynchronize();
            long long h[148]; cudaMemcpy(h, clk, 148 * 8, cudaMemcpyDeviceToHost);
            double a = 0; for (int i = 0; i < 148; i++) a += h[i];
            printf("CH=%d %s threads=%3d: %.0f cycles per sweep, %.1f cycles/element (fwd+bwd)  %s\n", ch, mode ? "col" : "row",
                   threads, a / 148, a / 148 / n, cudaGetErrorString(cudaGetLastError()));
        }
    };
    run(k_solve<4>, 4); run(k_solve<8>, 8); run(k_solve<16>, 16); run(k_solve<32>, 32);
    return 0;
}
