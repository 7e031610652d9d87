// Device-side state digest: simulate.py:79-90 state_checksum, the XOR over
// cells of BLAKE2b-128 (RFC 7693, unkeyed, digest_size 16) of the 56-byte
// record struct.pack("<q6d", id, x, y, z, vx, vy, vz).  One compression per
// cell (the record fits one 128-byte block); the 128-bit digests are
// XOR-reduced per warp and CTA and folded into two 64-bit words with
// atomicXor.  Cheap per-step parity checking in long runs without copying
// the state to the host.

#include "common.cuh"

namespace {

__constant__ unsigned long long kIV[8] = {
    0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull, 0xa54ff53a5f1d36f1ull,
    0x510e527fade682d1ull, 0x9b05688c2b3e6c1full, 0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};

__constant__ unsigned char kSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

__device__ __forceinline__ unsigned long long rotr(unsigned long long x, int n) {
    return (x >> n) | (x << (64 - n));
}

__device__ __forceinline__ void mix(unsigned long long* v, int a, int b, int c, int d,
                                    unsigned long long x, unsigned long long y) {
    v[a] = v[a] + v[b] + x;
    v[d] = rotr(v[d] ^ v[a], 32);
    v[c] = v[c] + v[d];
    v[b] = rotr(v[b] ^ v[c], 24);
    v[a] = v[a] + v[b] + y;
    v[d] = rotr(v[d] ^ v[a], 16);
    v[c] = v[c] + v[d];
    v[b] = rotr(v[b] ^ v[c], 63);
}

// BLAKE2b-128 of a single block holding `len` bytes (m: 16 little-endian
// words, zero padded); returns the digest's two little-endian words.
__device__ __forceinline__ void blake2b128(const unsigned long long (&m)[16], unsigned len,
                                           unsigned long long& h0, unsigned long long& h1) {
    unsigned long long h[8];
#pragma unroll
    for (int i = 0; i < 8; i++) h[i] = kIV[i];
    h[0] ^= 0x01010000ull ^ 16ull;  // fanout 1, depth 1, no key, 16-byte digest
    unsigned long long v[16];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        v[i] = h[i];
        v[i + 8] = kIV[i];
    }
    v[12] ^= (unsigned long long)len;  // byte counter (low word)
    v[14] = ~v[14];                    // final block
#pragma unroll
    for (int r = 0; r < 12; r++) {
        const unsigned char* s = kSigma[r];
        mix(v, 0, 4, 8, 12, m[s[0]], m[s[1]]);
        mix(v, 1, 5, 9, 13, m[s[2]], m[s[3]]);
        mix(v, 2, 6, 10, 14, m[s[4]], m[s[5]]);
        mix(v, 3, 7, 11, 15, m[s[6]], m[s[7]]);
        mix(v, 0, 5, 10, 15, m[s[8]], m[s[9]]);
        mix(v, 1, 6, 11, 12, m[s[10]], m[s[11]]);
        mix(v, 2, 7, 8, 13, m[s[12]], m[s[13]]);
        mix(v, 3, 4, 9, 14, m[s[14]], m[s[15]]);
    }
    h0 = h[0] ^ v[0] ^ v[8];
    h1 = h[1] ^ v[1] ^ v[9];
}

__global__ void __launch_bounds__(256) k_state_checksum(int n, const long long* __restrict__ ids,
                                                        const double* __restrict__ pos,
                                                        const double* __restrict__ vel,
                                                        unsigned long long* __restrict__ out) {
    __shared__ unsigned long long red[2][8];
    unsigned long long a0 = 0, a1 = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        unsigned long long m[16];
        m[0] = (unsigned long long)ids[i];
#pragma unroll
        for (int k = 0; k < 3; k++) {
            m[1 + k] = (unsigned long long)__double_as_longlong(pos[3L * i + k]);
            m[4 + k] = (unsigned long long)__double_as_longlong(vel[3L * i + k]);
        }
#pragma unroll
        for (int k = 7; k < 16; k++) m[k] = 0;
        unsigned long long d0, d1;
        blake2b128(m, 56, d0, d1);
        a0 ^= d0;
        a1 ^= d1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 ^= __shfl_xor_sync(0xffffffffu, a0, o);
        a1 ^= __shfl_xor_sync(0xffffffffu, a1, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][wid] = a0;
        red[1][wid] = a1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long b0 = 0, b1 = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            b0 ^= red[0][w];
            b1 ^= red[1][w];
        }
        atomicXor(out, b0);
        atomicXor(out + 1, b1);
    }
}

}  // namespace

int launch_state_checksum(cg_ctx* c, int n, const int64_t* ids, const double* pos,
                          const double* vel, unsigned long long* d_out) {
    CG_CUDA_CHECK(cudaMemsetAsync(d_out, 0, 2 * sizeof(unsigned long long), c->stream));
    if (n <= 0) return CG_OK;
    const int T = 256;
    const int blocks = std::min((n + T - 1) / T, c->num_sms * 8);
    CG_LAUNCH(c, K_CHECKSUM, k_state_checksum, blocks, T, 0, n, (const long long*)ids, pos, vel,
              d_out);
    return CG_OK;
}
