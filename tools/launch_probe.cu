// Where does k_plane_xy's stage time go?  Per-CTA start/end (globaltimer)
// of the library kernel body, back-to-back launches.
#define CG_PROBE 1
#include "../paper_2306_11544_b200/csrc/diffusion.cu"
#include <algorithm>
#include <cstdio>
#include <vector>

__device__ unsigned long long g_t[1024][2];
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <bool DIRI>
__global__ void __launch_bounds__(256) k_wrap(double* dens, MeshDev m, const double* fac, const double* rr, int nmax,
                                             const double* diri, ExchArgs ex) {
    extern __shared__ double sm[];
    __shared__ __align__(8) unsigned long long bar;
    const int id = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0) { g_t[id][0] = gt(); mbar_init(&bar, 1); }
    __syncthreads();
    unsigned phase = 0;
    plane_body<false, DIRI>(sm, &bar, phase, dens, m, fac, rr, nmax, diri, ex, blockIdx.x, blockIdx.y);
    if (threadIdx.x == 0) g_t[id][1] = gt();
}

__global__ void k_empty(int* p) { if (threadIdx.x == 1 << 30) p[0] = 1; }

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
    size_t smem = plane_smem_bytes(m);
    cudaFuncSetAttribute(k_wrap<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 5; it++) k_wrap<true><<<dim3(N, S), 256, smem>>>(dens, m, fac, rr, N, diri, ex);
    cudaEventRecord(a);
    k_wrap<true><<<dim3(N, S), 256, smem>>>(dens, m, fac, rr, N, diri, ex);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> t(2 * N * S);
    cudaMemcpyFromSymbol(t.data(), g_t, t.size() * 8);
    unsigned long long s0 = ~0ull, s1 = 0, e1 = 0; double dur = 0, dmax = 0;
    for (int i = 0; i < N * S; i++) { s0 = std::min(s0, t[2*i]); s1 = std::max(s1, t[2*i]); e1 = std::max(e1, t[2*i+1]); double d = (t[2*i+1]-t[2*i])/1e3; dur += d; dmax = std::max(dmax, d); }
    printf("event %.2f us | first start -> last start %.2f us | first start -> last end %.2f us | CTA mean %.2f max %.2f us\n",
           ms * 1e3, (s1 - s0) / 1e3, (e1 - s0) / 1e3, dur / (N * S), dmax);
    auto bb = [&](const char* name, auto launch) {
        for (int i = 0; i < 5; i++) launch();
        cudaEventRecord(a);
        for (int i = 0; i < 100; i++) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float t; cudaEventElapsedTime(&t, a, b);
        printf("%-44s %7.2f us/launch  %s\n", name, t * 10, cudaGetErrorString(cudaGetLastError()));
    };
    int* dummy; cudaMalloc(&dummy, 4);
    bb("empty 1 CTA", [&] { k_empty<<<1, 32>>>(dummy); });
    bb("empty 240 CTAs x 256", [&] { k_empty<<<240, 256>>>(dummy); });
    bb("plane default carveout", [&] { k_wrap<true><<<dim3(N, S), 256, smem>>>(dens, m, fac, rr, N, diri, ex); });
    cudaFuncSetAttribute(k_wrap<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    bb("plane carveout 100", [&] { k_wrap<true><<<dim3(N, S), 256, smem>>>(dens, m, fac, rr, N, diri, ex); });
    size_t zs = cols_smem_bytes(N, 64);
    cudaFuncSetAttribute(k_cols<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zs);
    bb("plane+z alternating (default carveout)", [&] {
        k_wrap<true><<<dim3(N, S), 256, smem>>>(dens, m, fac, rr, N, diri, ex);
        k_cols<2, true><<<dim3(N * N / 64, S), 64, zs>>>(dens, m, fac, rr, N, diri, 64); });
    cudaFuncSetAttribute(k_cols<2, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    bb("plane+z alternating (carveout 100 both)", [&] {
        k_wrap<true><<<dim3(N, S), 256, smem>>>(dens, m, fac, rr, N, diri, ex);
        k_cols<2, true><<<dim3(N * N / 64, S), 64, zs>>>(dens, m, fac, rr, N, diri, 64); });
    // the same sequences captured in a CUDA graph
    auto gb = [&](const char* name, int reps, auto launch) {
        cudaStream_t st; cudaStreamCreate(&st);
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < reps; i++) launch(st);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
        cudaEventRecord(a, st);
        for (int i = 0; i < 10; i++) cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st); cudaEventSynchronize(b);
        float t; cudaEventElapsedTime(&t, a, b);
        printf("graph: %-37s %7.2f us/rep  %s\n", name, t * 1e3 / (10 * reps), cudaGetErrorString(cudaGetLastError()));
    };
    gb("empty 240 CTAs", 100, [&](cudaStream_t st) { k_empty<<<240, 256, 0, st>>>(dummy); });
    gb("plane", 50, [&](cudaStream_t st) { k_wrap<true><<<dim3(N, S), 256, smem, st>>>(dens, m, fac, rr, N, diri, ex); });
    gb("plane+z", 50, [&](cudaStream_t st) {
        k_wrap<true><<<dim3(N, S), 256, smem, st>>>(dens, m, fac, rr, N, diri, ex);
        k_cols<2, true><<<dim3(N * N / 64, S), 64, zs, st>>>(dens, m, fac, rr, N, diri, 64); });
    for (int TC : {32, 64, 128, 256}) {
        size_t zz = cols_smem_bytes(N, TC);
        cudaFuncSetAttribute(k_cols<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)zz);
        char nm[64]; snprintf(nm, 64, "z TC=%d threads=%d", TC, TC);
        gb(nm, 50, [&](cudaStream_t st) { k_cols<2, true><<<dim3(N * N / TC, S), TC, zz, st>>>(dens, m, fac, rr, N, diri, TC); });
        snprintf(nm, 64, "z TC=%d threads=256", TC);
        gb(nm, 50, [&](cudaStream_t st) { k_cols<2, true><<<dim3(N * N / TC, S), 256, zz, st>>>(dens, m, fac, rr, N, diri, TC); });
    }
    return 0;
}
