// Where do the cycles of one Thomas forward step go?  (one warp, clock64)
#include <cstdio>
#include <cuda_runtime.h>
#define NN 80
__global__ void k(double* out, double r, long long* clk) {
    __shared__ double d[NN * 32], iv[NN], res[NN * 32];
    for (int i = 0; i < NN; i++) { d[i * 32 + threadIdx.x] = 1.0 + i * 1e-3; }
    for (int i = threadIdx.x; i < NN; i += 32) iv[i] = 0.5 + i * 1e-4;
    __syncthreads();
    double reg[16], ivr[16];
#pragma unroll
    for (int j = 0; j < 16; j++) { reg[j] = d[j * 32 + threadIdx.x]; ivr[j] = iv[j]; }
    // (a) pure chain, operands in registers: 5 x 16 steps
    long long t0 = clock64();
    double prev = 1.0;
    for (int rep = 0; rep < 5; rep++) {
#pragma unroll
        for (int j = 0; j < 16; j++) prev = (reg[j] + r * prev) * ivr[j];
    }
    long long t1 = clock64();
    // (b) + STS of each result
    double p2 = 1.0;
    for (int rep = 0; rep < 5; rep++) {
#pragma unroll
        for (int j = 0; j < 16; j++) { p2 = (reg[j] + r * p2) * ivr[j]; res[(rep * 16 + j) * 32 + threadIdx.x] = p2; }
    }
    long long t2 = clock64();
    // (c) operands via LDS (independent of the stores: separate arrays), results stored
    double p3 = 1.0;
#pragma unroll 8
    for (int i = 0; i < NN; i++) { p3 = (d[i * 32 + threadIdx.x] + r * p3) * iv[i]; res[i * 32 + threadIdx.x] = p3; }
    long long t3 = clock64();
    // (d) in place: load d[i], store d[i] (aliasing: loads cannot move above stores)
    double p4 = 1.0;
#pragma unroll 8
    for (int i = 0; i < NN; i++) { p4 = (d[i * 32 + threadIdx.x] + r * p4) * iv[i]; d[i * 32 + threadIdx.x] = p4; }
    long long t4 = clock64();
    // (e) in place with explicit register prefetch distance 8 (loads above stores in program order)
    double p5 = 1.0;
    double* dp = d + threadIdx.x;
    double w[8], fw[8];
#pragma unroll
    for (int j = 0; j < 8; j++) { w[j] = dp[j * 32]; fw[j] = iv[j]; }
    for (int i0 = 0; i0 < NN; i0 += 8) {
        double nw[8], nf[8];
#pragma unroll
        for (int j = 0; j < 8; j++) { int i = i0 + 8 + j; nw[j] = i < NN ? dp[i * 32] : 0.0; nf[j] = i < NN ? iv[i] : 0.0; }
#pragma unroll
        for (int j = 0; j < 8; j++) { p5 = (w[j] + r * p5) * fw[j]; dp[(i0 + j) * 32] = p5; }
#pragma unroll
        for (int j = 0; j < 8; j++) { w[j] = nw[j]; fw[j] = nf[j]; }
    }
    long long t5 = clock64();
    // (f) bulk chunks of 16: loads, then chain from registers, then stores
    double p6 = 1.0;
    for (int i0 = 0; i0 < NN; i0 += 16) {
        double cw[16], cf[16];
#pragma unroll
        for (int j = 0; j < 16; j++) { cw[j] = dp[(i0 + j) * 32]; cf[j] = iv[i0 + j]; }
#pragma unroll
        for (int j = 0; j < 16; j++) { p6 = (cw[j] + r * p6) * cf[j]; cw[j] = p6; }
#pragma unroll
        for (int j = 0; j < 16; j++) dp[(i0 + j) * 32] = cw[j];
    }
    long long t6 = clock64();
    // (g) bulk chunks of 40
    double p7 = 1.0;
    for (int i0 = 0; i0 < NN; i0 += 40) {
        double cw[40], cf[40];
#pragma unroll
        for (int j = 0; j < 40; j++) { cw[j] = dp[(i0 + j) * 32]; cf[j] = iv[i0 + j]; }
#pragma unroll
        for (int j = 0; j < 40; j++) { p7 = (cw[j] + r * p7) * cf[j]; cw[j] = p7; }
#pragma unroll
        for (int j = 0; j < 40; j++) dp[(i0 + j) * 32] = cw[j];
    }
    long long t7 = clock64();
    out[threadIdx.x] = prev + p2 + p3 + p4 + p5 + p6 + p7 + res[threadIdx.x];
    if (threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; clk[3] = t4 - t3; clk[4] = t5 - t4; clk[5] = t6 - t5; clk[6] = t7 - t6; }
}
int main() {
    double* out; long long* clk; cudaMalloc(&out, 64 * 8); cudaMalloc(&clk, 16 * 8);
    for (int it = 0; it < 3; it++) k<<<1, 32>>>(out, 2.5, clk);
    long long h[7]; cudaMemcpy(h, clk, 56, cudaMemcpyDeviceToHost);
    printf("cycles/step: regs %.1f | regs+STS %.1f | LDS+STS sep %.1f | in-place %.1f | in-place prefetch8 %.1f | bulk16 %.1f | bulk40 %.1f\n",
           h[0] / 80.0, h[1] / 80.0, h[2] / 80.0, h[3] / 80.0, h[4] / 80.0, h[5] / 80.0, h[6] / 80.0);
    return 0;
}
