// Host<->device transfer rates for the e2e path (12.3 MB = config-1 fields):
// copy engines on 1 or 4 streams vs SM-driven copies through mapped pinned
// memory (the kernel loads host memory directly), one direction and both.
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/pcie_probe.cu -o /tmp/pcie_probe
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void k_copy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t nb = 12288000;
    char *h_in, *h_out, *d_a, *d_b;
    CK(cudaHostAlloc(&h_in, nb, cudaHostAllocMapped));
    CK(cudaHostAlloc(&h_out, nb, cudaHostAllocMapped));
    CK(cudaMalloc(&d_a, nb));
    CK(cudaMalloc(&d_b, nb));
    cudaStream_t s[4];
    for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto timed = [&](const char* name, auto fn) {
        fn();
        CK(cudaDeviceSynchronize());
        const int reps = 20;
        cudaEvent_t t0, t1;
        cudaEventCreate(&t0);
        cudaEventCreate(&t1);
        cudaEventRecord(t0, s[0]);
        for (int r = 0; r < reps; r++) {
            for (int k = 1; k < 4; k++) cudaStreamWaitEvent(s[k], t0, 0);
            fn();
            cudaEvent_t e[3];
            for (int k = 1; k < 4; k++) {
                cudaEventCreateWithFlags(&e[k - 1], cudaEventDisableTiming);
                cudaEventRecord(e[k - 1], s[k]);
                cudaStreamWaitEvent(s[0], e[k - 1], 0);
            }
        }
        cudaEventRecord(t1, s[0]);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, t0, t1);
        printf("%-28s %7.1f us per 12.3 MB (%.1f GB/s per direction)\n", name, ms * 1e3 / reps,
               nb / (ms / reps) / 1e6);
        return 0;
    };
    timed("CE h2d 1 stream", [&] { cudaMemcpyAsync(d_a, h_in, nb, cudaMemcpyHostToDevice, s[0]); });
    timed("CE d2h 1 stream", [&] { cudaMemcpyAsync(h_out, d_b, nb, cudaMemcpyDeviceToHost, s[0]); });
    timed("CE h2d 4 streams", [&] {
        for (int k = 0; k < 4; k++)
            cudaMemcpyAsync(d_a + k * nb / 4, h_in + k * nb / 4, nb / 4, cudaMemcpyHostToDevice, s[k]);
    });
    timed("CE both 1+1 streams", [&] {
        cudaMemcpyAsync(d_a, h_in, nb, cudaMemcpyHostToDevice, s[0]);
        cudaMemcpyAsync(h_out, d_b, nb, cudaMemcpyDeviceToHost, s[1]);
    });
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (int g : {sms, 2 * sms, 4 * sms, 8 * sms}) {
        char nm[64];
        snprintf(nm, sizeof nm, "SM h2d grid %d", g);
        timed(nm, [&] { k_copy<<<g, 512, 0, s[0]>>>((const int4*)h_in, (int4*)d_a, nb / 16); });
    }
    for (int g : {sms, 4 * sms}) {
        char nm[64];
        snprintf(nm, sizeof nm, "SM d2h grid %d", g);
        timed(nm, [&] { k_copy<<<g, 512, 0, s[0]>>>((const int4*)d_b, (int4*)h_out, nb / 16); });
    }
    timed("SM h2d + CE d2h", [&] {
        k_copy<<<4 * sms, 512, 0, s[0]>>>((const int4*)h_in, (int4*)d_a, nb / 16);
        cudaMemcpyAsync(h_out, d_b, nb, cudaMemcpyDeviceToHost, s[1]);
    });
    timed("SM h2d + SM d2h", [&] {
        k_copy<<<2 * sms, 512, 0, s[0]>>>((const int4*)h_in, (int4*)d_a, nb / 16);
        k_copy<<<2 * sms, 512, 0, s[1]>>>((const int4*)d_b, (int4*)h_out, nb / 16);
    });
    return 0;
}
