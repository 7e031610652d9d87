// Cell divisions (population.py:32-129): counter-based draws keyed by
// (seed, cell id, step), the division decision, and daughter placement.
//
// Decisions and draws are integer hashing plus one compare against a
// host-computed threshold 1 - exp(-rate*dt) (the host evaluates it with the
// same libm exp CPython uses), so which cells divide, in which order, and the
// daughters' ids are bit-exact.  Placement uses the device cos/sin (within
// 2 ulp of libm), so daughter positions match the reference to ~1e-15
// relative, not bit for bit.
#include <cmath>
#include <vector>

#include "common.cuh"

namespace {

constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ull;

// population.py:32-37 (_mix64), 64-bit wrap-around arithmetic.
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x = x + kGolden;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// population.py:40-41 (_unit): the top 53 bits as a double in [0, 1).
__device__ __forceinline__ double unit53(unsigned long long h) {
    return (double)(h >> 11) * 0x1p-53;
}

// population.py:44-51 (division_draws).  Python masks negative ids and steps
// to 64 bits (two's complement), which the unsigned conversion reproduces.
__device__ __forceinline__ void draws(unsigned long long seed, long long id, long long step,
                                      double& u0, double& u1, double& u2) {
    const unsigned long long base =
        mix64(mix64(mix64(seed) ^ (unsigned long long)id) ^ (unsigned long long)step);
    u0 = unit53(mix64(base ^ 1ull));
    u1 = unit53(mix64(base ^ 2ull));
    u2 = unit53(mix64(base ^ 3ull));
}

__global__ void k_division_draws(int n, unsigned long long seed, long long step,
                                 const long long* __restrict__ ids, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    draws(seed, ids[i], step, out[3L * i], out[3L * i + 1], out[3L * i + 2]);
}

// population.py:90-95: cell i divides when u0 < 1 - exp(-rate*dt) (thr[i];
// rate <= 0 never divides: thr = -1).  Dividers are compacted (any order).
__global__ void k_division_decide(int n, unsigned long long seed, long long step,
                                  const long long* __restrict__ ids,
                                  const double* __restrict__ thr, int* __restrict__ list,
                                  int* __restrict__ count) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double t = thr[i];
    if (!(t > 0.0)) return;
    double u0, u1, u2;
    draws(seed, ids[i], step, u0, u1, u2);
    if (u0 < t) list[atomicAdd(count, 1)] = i;
}

struct DivBox {
    double lo[3], hi[3];
};

// phi = (2 pi) u_phi of divider j (population.py:108): the host evaluates
// cos / sin of it with libm, as CPython's math.cos / math.sin do.
__global__ void k_division_phi(int m, unsigned long long seed, long long step,
                               const int* __restrict__ list, const long long* __restrict__ ids,
                               double* __restrict__ phi) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    double u0, u_z, u_phi;
    draws(seed, ids[list[j]], step, u0, u_z, u_phi);
    phi[j] = 6.283185307179586 * u_phi;  // (2.0 * math.pi) * u_phi
}

// population.py:104-127: daughters in ascending parent id (rank among the
// dividers), placed R/2 away along the drawn direction, clamped inside
// (core.py:96-102, unconditional).  trig[2 j] = cos, [2 j + 1] = sin of
// divider j's phi (host libm).
__global__ void k_division_place(int m, unsigned long long seed, long long step,
                                 const int* __restrict__ list, const long long* __restrict__ ids,
                                 const double* __restrict__ pos, const double* __restrict__ radius,
                                 const double* __restrict__ trig, DivBox b,
                                 int* __restrict__ parent_out, double* __restrict__ pos_out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int i = list[j];
    const long long id = ids[i];
    int rank = 0;
    for (int k = 0; k < m; k++) rank += ids[list[k]] < id;
    double u0, u_z, u_phi;
    draws(seed, id, step, u0, u_z, u_phi);
    const double z = 2.0 * u_z - 1.0;
    const double t = 1.0 - z * z;
    const double rho = sqrt(t > 0.0 ? t : 0.0);  // max(0.0, 1 - z*z)
    const double c = trig[2L * j], s = trig[2L * j + 1];
    const double half_r = 0.5 * radius[i];
    const double hr = half_r * rho;
    double p[3] = {pos[3L * i] + hr * c, pos[3L * i + 1] + hr * s, pos[3L * i + 2] + half_r * z};
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const double lo = p[k] < b.lo[k] ? b.lo[k] : p[k];  // max(p, lo): p unless p < lo
        p[k] = lo <= b.hi[k] ? lo : b.hi[k];                // min(., hi): . unless . > hi
    }
    parent_out[rank] = i;
    pos_out[3L * rank] = p[0];
    pos_out[3L * rank + 1] = p[1];
    pos_out[3L * rank + 2] = p[2];
}

}  // namespace

extern "C" int cg_division_draws(cg_ctx* c, int n, uint64_t seed, int64_t step,
                                 const int64_t* ids, double* out) {
    if (n < 0) return set_error(CG_DOMAIN, "n must be >= 0");
    if (n == 0) return CG_OK;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    CG_LAUNCH(c, K_DIVISION, k_division_draws, (n + 255) / 256, 256, 0, n, seed, step,
              (const long long*)ids, out);
    return CG_OK;
}

extern "C" int cg_divisions_count(cg_ctx* c, int n, uint64_t seed, int64_t step,
                                  const int64_t* ids, const double* thr, int* count) {
    *count = 0;
    int st = check_cells(c, n);
    if (st) return st;
    if (n == 0) return CG_OK;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    CG_CUDA_CHECK(cudaMemsetAsync(c->d_div_n, 0, sizeof(int), c->stream));
    CG_LAUNCH(c, K_DIVISION, k_division_decide, (n + 255) / 256, 256, 0, n, seed, step,
              (const long long*)ids, thr, c->d_div_list, c->d_div_n);
    CG_CUDA_CHECK(cudaMemcpyAsync(c->h_flags + FLAG_WORDS, c->d_div_n, sizeof(int),
                                  cudaMemcpyDeviceToHost, c->stream));
    CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    *count = c->h_flags[FLAG_WORDS];
    return CG_OK;
}

static int place_with_host_trig(cg_ctx* c, int count, uint64_t seed, int64_t step,
                                const int64_t* ids, const double* pos, const double* radius,
                                const DivBox& b, int32_t* parent_out, double* pos_out,
                                double* d_buf) {
    double* d_trig = d_buf + count;
    CG_LAUNCH(c, K_DIVISION, k_division_phi, (count + 127) / 128, 128, 0, count, seed, step,
              c->d_div_list, (const long long*)ids, d_buf);
    std::vector<double> h((size_t)count * 3);
    CG_CUDA_CHECK(cudaMemcpyAsync(h.data(), d_buf, (size_t)count * sizeof(double),
                                  cudaMemcpyDeviceToHost, c->stream));
    CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    for (int j = 0; j < count; j++) {
        h[count + 2 * j] = cos(h[j]);
        h[count + 2 * j + 1] = sin(h[j]);
    }
    CG_CUDA_CHECK(cudaMemcpyAsync(d_trig, h.data() + count, (size_t)count * 2 * sizeof(double),
                                  cudaMemcpyHostToDevice, c->stream));
    CG_LAUNCH(c, K_DIVISION, k_division_place, (count + 127) / 128, 128, 0, count, seed, step,
              c->d_div_list, (const long long*)ids, pos, radius, d_trig, b, parent_out, pos_out);
    return CG_OK;
}

extern "C" int cg_divisions_place(cg_ctx* c, int n, int count, uint64_t seed,
                                  int64_t step, const int64_t* ids, const double* pos,
                                  const double* radius, int32_t* parent_out, double* pos_out) {
    int st = check_cells(c, n);
    if (st) return st;
    if (count < 0 || count > n) return set_error(CG_DOMAIN, "division count out of range");
    if (count == 0) return CG_OK;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    const MeshDev& m = c->m;
    DivBox b;
    const double org[3] = {m.ox, m.oy, m.oz};
    const int ns[3] = {m.nx, m.ny, m.nz};
    const double ds[3] = {m.dx, m.dy, m.dz};
    for (int k = 0; k < 3; k++) {
        const double up = org[k] + ns[k] * ds[k];  // core.py:64-66 upper
        b.lo[k] = org[k] + POSITION_EPS;
        b.hi[k] = up - POSITION_EPS;
    }
    // cos / sin of every divider's angle with the host's libm (CPython's
    // math.cos / math.sin), so daughter positions are bit-identical
    double* d_buf = nullptr;  // phi (count), then (cos, sin) pairs (2 count)
    CG_CUDA_CHECK(cudaMalloc((void**)&d_buf, (size_t)count * 3 * sizeof(double)));
    const int rc = place_with_host_trig(c, count, seed, step, ids, pos, radius, b, parent_out,
                                        pos_out, d_buf);
    cudaStreamSynchronize(c->stream);
    cudaFree(d_buf);
    return rc;
}
