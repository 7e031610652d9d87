// Microbenchmark: dependent-chain latency of fp64 DADD/DMUL/DFMA and of the
// Thomas forward step (d = (d + r*p) * inv) from shared memory, on one warp.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, double a, double b, int n) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-3;
    __syncthreads();
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; i++) { x = x * b; x = x + a; }
    long long t1 = clock64();
    double y = a;
    for (int i = 0; i < n; i++) y = fma(y, b, a);
    long long t2 = clock64();
    double z = a;
    for (int i = 0; i < n; i++) { double c = sm[i & 1023]; z = (c + b * z) * a; }
    long long t3 = clock64();
    double w = a;
    for (int i = 0; i < n; i++) w = w / b + a;
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        out[0] = x + y + z + w;
        out[1] = (t1 - t0) / (2.0 * n);
        out[2] = (t2 - t1) / (1.0 * n);
        out[3] = (t3 - t2) / (1.0 * n);
        out[4] = (t4 - t3) / (1.0 * n);
    }
}

int main() {
    double* d;
    cudaMalloc(&d, 8 * sizeof(double));
    double h[8];
    for (int warps : {1, 4}) {
        lat<<<1, 32 * warps>>>(d, 1.0000001, 0.9999999, 4096);
        cudaMemcpy(h, d, 5 * sizeof(double), cudaMemcpyDeviceToHost);
        printf("warps=%d  dmul/dadd %.2f cyc   dfma %.2f cyc   thomas-fwd step %.2f cyc   div+add %.2f cyc\n",
               warps, h[1], h[2], h[3], h[4]);
    }
    return 0;
}
