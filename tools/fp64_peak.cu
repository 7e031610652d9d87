// FP64 pipe throughput on this GPU: every SM full of warps running 8
// independent chains of DFMA (2 flop) or DMUL+DADD pairs (1 flop each, the
// -fmad=false instruction mix of the velocity kernel).  Reports instructions
// and flops per second.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_peak.cu -o tools/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

template <bool FMA>
__global__ void k_peak(double* out, double a, double b, int n) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = a + threadIdx.x + k;
    for (int i = 0; i < n; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (FMA) {
                x[k] = fma(x[k], b, a);
            } else {
                x[k] = __dmul_rn(x[k], b);
                x[k] = __dadd_rn(x[k], a);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += x[k];
    if (s == 1.2345) out[0] = s;  // keep the chains alive
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int n = 4096, T = 512, blocks = sms * 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int fma = 1; fma >= 0; fma--) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            if (fma) k_peak<true><<<blocks, T>>>(out, 1e-9, 0.999999, n);
            else k_peak<false><<<blocks, T>>>(out, 1e-9, 0.999999, n);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double thr = (double)blocks * T;
        const double inst = thr * n * 8 * (fma ? 1 : 2);
        const double flop = thr * n * 8 * 2;
        printf("%s: %.2f T thread-instr/s, %.2f TFLOP/s (%.3f ms)\n", fma ? "DFMA" : "DMUL+DADD",
               inst / ms / 1e9, flop / ms / 1e9, ms);
    }
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs %d, max clock %.0f MHz\n", sms, clk / 1e3);
    return 0;
}
