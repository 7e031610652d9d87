// Internal declarations shared by the libcellgpu.so translation units.
//
// Numerics contract: this library is compiled with -fmad=false (device) and
// -ffp-contract=off (host), so every a*b+c rounds twice, exactly like the
// numpy ufuncs and CPython float arithmetic of the reference.  Double
// division and sqrt are IEEE round-to-nearest by default on sm_100a.
#pragma once

#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/cellgpu.h"

// Division by a runtime-invariant divisor with one mulhi (Granlund-Montgomery,
// exact for every 32-bit unsigned numerator; tools/fastdiv_test.c).
struct FastDiv {
    unsigned d, m, s;
};
inline FastDiv make_fastdiv(unsigned d) {
    FastDiv f{d, 0u, 0u};
    if (d <= 1) return f;
    unsigned s = 0;
    while ((1ull << s) < d) s++;
    f.s = s;
    f.m = (unsigned)(((1ull << 32) * ((1ull << s) - d)) / d + 1);
    return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ unsigned fdiv(unsigned n, const FastDiv& f) {
    if (f.d <= 1) return n;
    const unsigned t = __umulhi(n, f.m);
    return (t + ((n - t) >> 1)) >> (f.s - 1);
}
#endif

struct MeshDev {
    int nx, ny, nz;
    double dx, dy, dz;
    double ox, oy, oz;
    FastDiv fnx, fny;
    // z-slab decomposition: whether local plane 0 / nz-1 lie
    // on a global z face, and whether the z sweep is partitioned across ranks
    // (then its Dirichlet pins are applied after the interface correction).
    int zlo = 1, zhi = 1, slab = 0;
};
#ifdef __CUDACC__
__device__ __forceinline__ bool is_zface(int z, const MeshDev& m) {
    return (z == 0 && m.zlo) || (z == m.nz - 1 && m.zhi);
}
#endif

enum { FLAG_DOMAIN = 0, FLAG_NUMERIC = 1, FLAG_CAPACITY = 2, FLAG_WORDS = 4 };

// Kernel ids for instrumentation.
enum KernelId {
    K_PLANE_XY = 0,
    K_LOD_PERSISTENT,
    K_X_ROWS,
    K_Y_COLS,
    K_Z_COLS,
    K_EXCHANGE,
    K_EXCHANGE_COEF,
    K_EXCHANGE_APPLY,
    K_VOXEL_COUNT,
    K_SCAN_BLOCK,
    K_SCAN_PARTIALS,
    K_SCAN_FINAL,
    K_SCATTER,
    K_BIN_FIX,
    K_GATHER,
    K_VELOCITY_LISTS,
    K_VELOCITY,
    K_VELOCITY_MID,
    K_VELOCITY_BIG,
    K_INTEGRATE,
    K_ZSLAB_PACK,
    K_ZSLAB_CORRECT,
    K_VOXEL_Z,
    K_GRADIENTS,
    K_CHECKSUM,
    K_CHECK_STATE,
    K_DIVISION,
    K_PLANE_SEG,
    K_Z_SEG,
    K_VELOCITY_DIRECT,
    K_COUNT
};
extern const char* const kKernelNames[K_COUNT];

struct ProfRec {
    int kid;
    cudaEvent_t a, b;
};

// Everything the split exchange kernel reads, written together by the bin
// fix-up (k_bin_fix_g<true>): the non-empty voxel list and its count, the
// id-sorted slot offsets (+1), per-slot {A, D} and the inline records.  The
// engine rotates three so the next step's rebin can run beside this step's
// substeps (one set read, another written) and, in pipelined host-driven
// steps, one step ahead of them.
// core.py:23 POSITION_EPS: clamp_inside keeps positions this far inside the faces.
#define POSITION_EPS 1e-6

constexpr int kExchSets = 3;  // engine exchange sets in rotation

struct ExchSet {
    double* A = nullptr;      // (S, cap)
    double* D = nullptr;
    double* R = nullptr;      // (S, min(nvox, cap), 2 kRecCells)
    int32_t* vox = nullptr;   // (min(nvox, cap))
    int32_t* start = nullptr; // (min(nvox, cap) + 1)
    int32_t* n = nullptr;     // (1)
    // Fast numerics (CG_NUMERICS_FAST): every non-empty voxel's exchange as
    // one affine map per substrate, rho -> alpha rho + beta (the composition
    // of its cells' (rho + A) / D in ascending id), and the first non-empty
    // list index of every z plane (nz + 1), written by the bin fix-up.
    double* aff = nullptr;    // (S, min(nvox, cap), 2)
    int32_t* pz = nullptr;    // (ny * nz + 1): first list index of every x row
};

struct cg_ctx {
    int device = 0;
    MeshDev m{};
    int S = 0;
    long nvox = 0;
    int cap_cells = 0;
    int nmax = 0;  // max(nx, ny, nz)
    cudaStream_t stream = nullptr;
    int num_sms = 148;

    int* d_flags = nullptr;  // FLAG_WORDS
    unsigned long long* d_digest = nullptr;  // (2) cg_state_checksum accumulator
    int* h_flags = nullptr;  // pinned mirror

    // Thomas factors, cached per (dt, diffusion[], decay[]):
    //   d_fac[((s*3 + axis)*2 + {0: inv, 1: gamma}) * nmax + i],  d_r[s*3 + axis]
    double* d_fac = nullptr;
    double* d_r = nullptr;
    double* d_diri = nullptr;  // S
    double* d_sat = nullptr;   // S
    std::vector<double> fac_key;
    std::vector<double> h_fac, h_r;  // host copies of d_fac, d_r
    std::vector<double> diri_key;
    std::vector<double> sat_key;

    // Rebin scratch: per-voxel counts (kept all-zero between rebins), scan partials.
    int* d_counts = nullptr;
    unsigned long long* d_part = nullptr;     // single-pass scan: tile aggregates
    unsigned long long* d_scan_incl = nullptr; // single-pass scan: tile inclusive prefixes
    int* d_scan_flag = nullptr;               // tile flags (nb) + ticket
    // Written by every rebin: non-empty voxels before each row start
    // (nz*ny + 1) and the id-sorted slot offset of each non-empty voxel (+1).
    int* d_row_ne = nullptr;
    int* d_ne_start = nullptr;
    int n_part = 0;

    // Per-cell scratch in id-sorted bin order.
    double* d_sp = nullptr;       // (cap, 4): x, y, z, R
    float4* d_spf = nullptr;      // (cap): the same rounded to fp32 (velocity pre-test)
    long long* d_sid = nullptr;   // (cap)
    int* d_sid32 = nullptr;       // (cap) low 32 bits, rank keys when all ids fit
    int* d_cand = nullptr;        // (min(nvox, cap), 64) id-sorted candidate slots per voxel
    int* d_slot_list = nullptr;   // (cap) list index of each slot's voxel, -1 = slow path
    int* d_svox = nullptr;        // (cap) voxel of each slot (fast velocities)
    double* d_exA = nullptr;      // (S, cap)  (f*sec)*sat
    double* d_exD = nullptr;      // (S, cap)  1 + f*(sec+upt)
    double* d_exR = nullptr;      // (S, min(nvox, cap), 4) first two cells' {A, D} per non-empty voxel
    // xset[0] aliases d_exA/d_exD/d_exR; its list/offset copies and all of
    // xset[1] are allocated by the engine (ensure_exch_sets).
    ExchSet xset[kExchSets];
    bool xset_alloc = false;
    int* d_div_list = nullptr;    // (cap) dividing cells (storage index), cg_divisions_*
    int* d_div_n = nullptr;       // (1) their count
    int* d_mid = nullptr;         // voxels with 33..VEL_CAP candidates
    int* d_overflow = nullptr;    // voxels with more than VEL_CAP candidates
    int* d_big = nullptr;         // bin fix-up: non-empty list indices of bins > BF_K cells
    int* d_n_big = nullptr;       //   and their count (zeroed by the scatter)
    int* d_n_overflow = nullptr;  // [0] overflow count, [1] mid count, [2] ids-not-32-bit
    int big_smem = 0;

    // Programmatic dependent launch: off by default -- faster for back-to-back
    // eager launches but measured slower inside the step graph.
    bool pdl = false;  // env CELLGPU_PDL=1 enables
    // Per-kernel PDL (bit = KernelId; env CELLGPU_PDL_MASK): kernels trigger
    // their dependents at the end of their work, so each launch and CTA ramp
    // overlaps the tail of the kernel before it.  On for the diffusion chain
    // (exchange, plane, z: 290 vs 311 us per step), the rebin chain
    // (integrate, scan, scatter, bin fix-up: -2 us) and, since the velocity
    // branch also carries the rebin, the velocity kernels (0.284 vs 0.286 ms
    // with the L2 flushed).
    unsigned long long pdl_mask =
        (1ull << K_PLANE_XY) | (1ull << K_Z_COLS) | (1ull << K_EXCHANGE_APPLY) |
        (1ull << K_PLANE_SEG) | (1ull << K_Z_SEG) | (1ull << K_VELOCITY_DIRECT) |
        (1ull << K_INTEGRATE) | (1ull << K_SCAN_BLOCK) | (1ull << K_SCATTER) | (1ull << K_BIN_FIX) |
        (1ull << K_GATHER) | (1ull << K_VELOCITY_LISTS) | (1ull << K_VELOCITY) |
        (1ull << K_VELOCITY_MID) | (1ull << K_VELOCITY_BIG);
    int plane_threads = 256;  // env CELLGPU_PLANE_THREADS
    // Grid cap of the per-voxel / per-cell velocity kernels, in CTAs per SM
    // (0: none; env CELLGPU_VEL_CTAS; see cg_engine_create).
    int vel_ctas_per_sm = 0;

    bool reg_lines = true;  // env CELLGPU_REGLINES=0 selects the streaming line solves
    // Substrate window of the diffusion launches (engine substrate chains):
    // sub_n > 0 restricts the LOD and split-exchange kernels to substrates
    // [sub0, sub0 + sub_n); 0 = all.
    int sub0 = 0, sub_n = 0;
    bool exch_ready = false;  // cg_rebin_exchange coefficients valid for exch_n cells
    bool exch_affine = false;  // ... as affine maps only (cg_rebin_exchange_affine)
    int exch_n = 0;
    int exch_split = -1;    // env CELLGPU_EXCH_SPLIT: 1 own kernel, 0 fused, -1 auto

    // Segmented line solves (lod_fast.cu): per (substrate, axis) the four
    // factor arrays inv, gam, cf, cb (nmax each) for segments of seg_len
    // elements; rebuilt when the Thomas factors or the segment lengths change.
    double* d_segf = nullptr;
    std::vector<double> segf_key;
    std::vector<double> h_segf;
    bool fast_sets = false;  // aff / pz of every exchange set allocated

    // z-slab decomposition (cg_ctx_set_slab): this rank's planes
    // [z0, z0 + nz) of nz_global, local block Thomas factors for the z axis,
    // this rank's spikes v, w (S x 2 x nz) and every rank's spike ends
    // (S x world x 4: v[0], v[m-1], w[0], w[m-1]).
    int slab_rank = 0, slab_world = 1, nz_global = 0, slab_z0 = 0;
    std::vector<int> slab_starts;  // (world + 1) first plane of every rank
    double* d_spk = nullptr;
    // z slabs: the interface correction deferred to the next fast LOD call
    // (cg_zslab_defer): per-line (left, right) in the line-block layout
    // (world, S, 2, Lb), applied as the next substep's x-row / plane kernel
    // stages the field; null when none is pending.
    const double* pend_lr = nullptr;
    double* d_ends = nullptr;

    // Instrumentation.
    bool prof = false;
    std::vector<ProfRec> recs;
    std::vector<cudaEvent_t> event_pool;
    long long launches = 0;
};

// Single-pass rebin scan tiles (cells.cu k_scan_lookback).
constexpr int SCAN_T = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_T * SCAN_ITEMS;

// Per-device "done" bits of a one-time setup (e.g. one kernel's dynamic-smem
// opt-in, which is per device; contexts on several devices may share a
// process).  test_and_set is atomic.
struct DeviceFlags {
    unsigned long long bits = 0;
    bool test_and_set(int dev) {
        const unsigned long long b = 1ull << (dev & 63);
        return (__atomic_fetch_or(&bits, b, __ATOMIC_ACQ_REL) & b) != 0;
    }
};

// Error plumbing (capi.cu).
int set_cuda_error(cudaError_t e, const char* where);
int set_error(int code, const std::string& msg);

// Instrumented launch bracket (capi.cu).
void prof_begin(cg_ctx* c, int kid, ProfRec* rec);
void prof_end(cg_ctx* c, ProfRec* rec);

// Programmatic dependent launch: every kernel starts with griddepcontrol.wait
// (a no-op without the attribute) and immediately lets its dependents launch,
// so each kernel's CTA launch and prologue overlap the predecessor's tail
// while data dependences still wait for full completion.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
#endif

#define CG_LAUNCH(ctx, kid, kernel, grid, block, smem, ...)                         \
    do {                                                                            \
        ProfRec _rec;                                                               \
        prof_begin((ctx), (kid), &_rec);                                            \
        cudaLaunchConfig_t _cfg = {};                                               \
        _cfg.gridDim = dim3(grid);                                                  \
        _cfg.blockDim = dim3(block);                                                \
        _cfg.dynamicSmemBytes = (smem);                                             \
        _cfg.stream = (ctx)->stream;                                                \
        cudaLaunchAttribute _at[1];                                                 \
        _at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;             \
        _at[0].val.programmaticStreamSerializationAllowed = 1;                      \
        _cfg.attrs = _at;                                                           \
        _cfg.numAttrs = ((ctx)->pdl || ((ctx)->pdl_mask >> (kid) & 1)) ? 1 : 0;      \
        cudaError_t _e = cudaLaunchKernelEx(&_cfg, kernel, __VA_ARGS__);            \
        if (_e != cudaSuccess) {                                                    \
            char _w[160];                                                           \
            snprintf(_w, sizeof _w, "%s (grid %u x %u, block %u, smem %zu)",        \
                     kKernelNames[kid], _cfg.gridDim.x, _cfg.gridDim.y,             \
                     _cfg.blockDim.x, (size_t)_cfg.dynamicSmemBytes);               \
            return set_cuda_error(_e, _w);                                          \
        }                                                                           \
        prof_end((ctx), &_rec);                                                     \
        (ctx)->launches++;                                                          \
    } while (0)

#define CG_CUDA_CHECK(expr)                                                         \
    do {                                                                            \
        cudaError_t _e = (expr);                                                    \
        if (_e != cudaSuccess) return set_cuda_error(_e, #expr);                    \
    } while (0)

// diffusion.cu
int ensure_factors(cg_ctx* c, double dt, const double* diffusion, const double* decay);
int ensure_dirichlet(cg_ctx* c, const double* dirichlet);
int ensure_saturation(cg_ctx* c, const double* saturation);
// One full LOD step over all substrates; when exA/exD are given the G4
// exchange (precomputed coefficients) is fused ahead of the x sweep.
// Requires the row_ne / ne_start scratch of the rebin that produced `nonempty`.
// parts: bit 0 = x/y sweeps (with the fused exchange), bit 1 = z sweep.
// check: also Microenvironment.check_state on the result (FLAG_NUMERIC).
long zslab_block_lines(const cg_ctx* c);
// A pending z-slab correction as the fast LOD kernels apply it when they
// stage the field: x += left v[z] + right w[z] (k_zslab_correct's operations).
struct PendCorr {
    const double* lr;   // (world, S, 2, Lb) with the substrate window applied by the caller
    const double* spk;  // (S, 2, nz): v then w per substrate
    long Lb;
    int S;              // substrates in lr
    int nz;
};
int launch_zslab_lr_gather(cg_ctx* c, const double* recv, double* lr);
int launch_zslab_pack_blocks(cg_ctx* c, const double* dens, double* send);
int launch_zslab_reduce_blocks(cg_ctx* c, const double* recv, double* out);
int launch_zslab_correct_lr(cg_ctx* c, double* dens, const double* lr, int bc);
int launch_lod(cg_ctx* c, double* dens, int bc, const int32_t* nonempty, const double* exA,
               const double* exD, int n_cells, int parts = 3, bool check = false);
int launch_check_field(cg_ctx* c, const double* d, long n);
// CG_CAPACITY unless 0 <= n <= the context's cell capacity.
int check_cells(cg_ctx* c, int n);
int launch_exchange_scalar(cg_ctx* c, double* dens_s, double dt, double sec, double upt,
                           double sat, int n_cells, const double* volume,
                           const int32_t* bin_start, const int32_t* bin_cells_by_id,
                           const int32_t* nonempty, const int32_t* n_nonempty);
int launch_exchange_coef(cg_ctx* c, double dt, const double* secretion, const double* uptake,
                         int n_cells, const double* volume, const int32_t* bin_cells_by_id);
// Whether the engine runs the G4 exchange as its own kernel before each
// substep's plane kernel (default with register lines) or fused into it.
bool lod_exchange_split(const cg_ctx* c);
// Line length of the register-line kernels for this mesh (0: streaming).
int reg_line_length(const cg_ctx* c);
int launch_gradients(cg_ctx* c, const double* dens, double* grad);
int launch_state_checksum(cg_ctx* c, int n, const int64_t* ids, const double* pos,
                          const double* vel, unsigned long long* d_out);
// xs: read the exchange set instead of the rebin's current list/offsets and
// ctx coefficients (engine, double-buffered).  early: those inputs were
// written at least two launches back on this stream (engine substeps >= 1),
// so the kernel loads them before waiting for its predecessor.
int launch_exchange_rec(cg_ctx* c, double* dens, int n_cells, const int32_t* nonempty,
                        const int32_t* n_nonempty, const ExchSet* xs = nullptr,
                        bool early = false);
int launch_exchange_ne(cg_ctx* c, double* dens, int n_cells, const int32_t* nonempty,
                       const int32_t* n_nonempty);
int launch_exchange_apply(cg_ctx* c, double* dens, int n_cells, const int32_t* bin_start,
                          const int32_t* nonempty, const int32_t* n_nonempty);

// cells.cu
int init_cells_kernels(cg_ctx* c);
struct CoefLaunch {  // fused G4 exchange coefficients (engine)
    double dt;
    const double* secretion;
    const double* uptake;
    const double* volume;
    const ExchSet* out = nullptr;  // also write the exchange set (engine)
    bool affine = false;           // and its affine maps / plane offsets (fast numerics)
    const double* pos = nullptr;   // and (fast numerics) the slots' (x, y, z, R) + voxel for
    const double* radius = nullptr;  //   the next step's velocities (ctx d_sp / d_svox)
};
// counted: voxel keys and histogram already produced (k_integrate_count);
// coef: also compute the exchange coefficients in the bin fix-up.
int launch_rebin(cg_ctx* c, int n, const double* pos, const int64_t* ids, int32_t* voxel,
                 int32_t* bin_start, int32_t* bin_cells, int32_t* bin_cells_by_id,
                 int32_t* nonempty, int32_t* n_nonempty, bool counted = false,
                 const CoefLaunch* coef = nullptr);
int launch_velocities(cg_ctx* c, int n, const double* pos, const double* radius,
                      const int64_t* ids, const int32_t* voxel, const int32_t* bin_start,
                      const int32_t* bin_cells_by_id, const int32_t* nonempty,
                      const int32_t* n_nonempty, double c_r, double c_a, double m_a, double* vel,
                      bool dense);
// voxel_for_rebin: fuse the rebin's voxel keys + histogram (engine).
int launch_integrate(cg_ctx* c, int n, double* pos, const double* vel, double* prev_vel,
                     double dt, int integrator, int32_t* voxel_for_rebin = nullptr);

// Host restatement of diffusion.py:80-99 (bit-identical to the reference).
void host_line_factors(int n, double r, double lam3, double* inv, double* gamma);
// z-slab kernels (diffusion.cu).
int launch_zslab_pack(cg_ctx* c, const double* dens, double* send);
int launch_zslab_correct(cg_ctx* c, double* dens, const double* recv, int bc);
int launch_voxel_z(cg_ctx* c, int n, const double* pos, int32_t* out);
// full: the whole voxel index (-1 outside) instead of its z plane.
int launch_voxel_index(cg_ctx* c, int n, const double* pos, int32_t* out, bool full);

// lod_fast.cu: fast numerics (CG_NUMERICS_FAST, north_star's tolerances:
// fields within 1e-10, bins unchanged).  Line length of the segmented LOD
// kernels for this mesh (0: none -> the exact kernels run).
int seg_line_length(const cg_ctx* c);
// 1: cubic plane + z kernels (seg_line_length); 2: streaming x rows + y
// columns + the exact z kernel (config 4's slabs); 0: none.
int fast_lod_kind(const cg_ctx* c);
int seg_stream_length(const cg_ctx* c);
// One LOD step with the affine exchange (aff/pz/vox/n_ne; null: no exchange)
// fused into the segmented plane kernel; substrate window c->sub0/sub_n.
// Segmented factors for the current Thomas factors (outside graph capture).
int prepare_lod_fast(cg_ctx* c);
// early: the records were written at least one launch back on this stream.
int launch_lod_fast(cg_ctx* c, double* dens, int bc, const int32_t* vox, const int32_t* n_ne,
                    const double* aff, const int32_t* pz, int parts = 3, bool check = false,
                    bool early = false);
// Velocities accumulated per cell over the 9 row ranges of its 3x3x3 block
// (candidate order: rows, then voxel x, then id; not the reference's global
// id order -> within 1e-12 normwise instead of bit-exact).
// gathered: the slots' (x, y, z, R) and voxels are already in the ctx
// scratch (written by the rebin's bin fix-up, CoefLaunch::pos).  quad: four
// lanes per cell (dense voxels) instead of one thread per cell.
int launch_velocities_fast(cg_ctx* c, int n, const double* pos, const double* radius,
                           const int32_t* voxel, const int32_t* bin_start,
                           const int32_t* bin_cells_by_id, bool gathered, bool quad, double c_r,
                           double c_a, double m_a, double* vel);
