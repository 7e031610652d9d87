// C-ABI entry points of libcellgpu.so (declared in include/cellgpu.h): context
// lifecycle, error mapping, instrumentation, the five hot-path calls and the
// graph-replayed step engine.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "lod_common.cuh"

const char* const kKernelNames[K_COUNT] = {
    "plane_xy",  "lod_persistent", "x_rows",      "y_cols",          "z_cols",     "exchange",
    "exchange_coef", "exchange_apply", "voxel_count", "scan", "scan_partials",
    "scan_final", "scatter",    "bin_fix",         "gather",     "cand_lists", "velocity",
    "velocity_mid", "velocity_big", "integrate", "zslab_pack", "zslab_correct", "voxel_z", "gradients", "state_checksum",
    "check_state", "division", "plane_seg", "z_seg", "velocity_direct"};

static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int set_cuda_error(cudaError_t e, const char* where) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return CG_CUDA + (int)e;
}

extern "C" const char* cg_version(void) { return "cellgpu 0.1 sm_100a"; }

// Built with -fno-builtin so pow() stays the libm call CPython makes.
extern "C" void cg_cell_volumes(int n, const double* radius, double* volume) {
    const double pi = 3.141592653589793;  // math.pi
    for (int i = 0; i < n; i++) volume[i] = (4.0 / 3.0) * pi * pow(radius[i], 3.0);
}
extern "C" const char* cg_last_error(void) { return g_last_error.c_str(); }

// ---------------------------------------------------------------- instrumentation

static cudaEvent_t pool_event(cg_ctx* c) {
    if (!c->event_pool.empty()) {
        cudaEvent_t e = c->event_pool.back();
        c->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void prof_begin(cg_ctx* c, int kid, ProfRec* rec) {
    rec->kid = kid;
    rec->a = rec->b = nullptr;
    if (!c->prof) return;
    rec->a = pool_event(c);
    rec->b = pool_event(c);
    cudaEventRecord(rec->a, c->stream);
}

void prof_end(cg_ctx* c, ProfRec* rec) {
    if (!c->prof || !rec->a) return;
    cudaEventRecord(rec->b, c->stream);
    c->recs.push_back(*rec);
}

extern "C" int cg_prof_enable(cg_ctx* c, int on) {
    c->prof = on != 0;
    return CG_OK;
}

extern "C" int cg_prof_read(cg_ctx* c, int max_kernels, char* names, double* total_ms,
                            int* launches) {
    CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    std::vector<double> tot(K_COUNT, 0.0);
    std::vector<int> cnt(K_COUNT, 0);
    for (auto& r : c->recs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        tot[r.kid] += ms;
        cnt[r.kid] += 1;
        c->event_pool.push_back(r.a);
        c->event_pool.push_back(r.b);
    }
    c->recs.clear();
    int k = 0;
    for (int i = 0; i < K_COUNT && k < max_kernels; i++) {
        if (!cnt[i]) continue;
        std::snprintf(names + 32 * k, 32, "%s", kKernelNames[i]);
        total_ms[k] = tot[i];
        launches[k] = cnt[i];
        k++;
    }
    return k;
}

extern "C" long long cg_launch_count(cg_ctx* c) { return c->launches; }

// ---------------------------------------------------------------- context

extern "C" int cg_ctx_create(int device, int nx, int ny, int nz, double dx, double dy, double dz,
                             double ox, double oy, double oz, int n_substrates,
                             int cell_capacity, cg_ctx** out) {
    *out = nullptr;
    if (nx < 1 || ny < 1 || nz < 1) return set_error(CG_DOMAIN, "voxel counts must be >= 1");
    if (!(dx > 0 && dy > 0 && dz > 0)) return set_error(CG_DOMAIN, "voxel edge lengths must be > 0");
    if ((long)nx * ny * nz >= (1L << 31) - 1) return set_error(CG_CAPACITY, "mesh too large for int32 voxel ids");
    if (n_substrates < 0) return set_error(CG_DOMAIN, "substrate count must be >= 0");
    CG_CUDA_CHECK(cudaSetDevice(device));
    cg_ctx* c = new cg_ctx();
    c->device = device;
    c->m = MeshDev{nx, ny, nz, dx, dy, dz, ox, oy, oz, make_fastdiv(nx), make_fastdiv(ny)};
    c->S = n_substrates;
    c->nvox = (long)nx * ny * nz;
    c->cap_cells = std::max(cell_capacity, 1);
    c->nmax = std::max(nx, std::max(ny, nz));
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    const int S = std::max(c->S, 1);
    const size_t cap = (size_t)c->cap_cells;
    const int nb = (int)((c->nvox + SCAN_TILE - 1) / SCAN_TILE);
    c->n_part = nb + 1;
#define ALLOC(ptr, bytes) CG_CUDA_CHECK(cudaMalloc((void**)&(ptr), (bytes)))
    ALLOC(c->d_flags, FLAG_WORDS * sizeof(int));
    ALLOC(c->d_digest, 2 * sizeof(unsigned long long));
    // FLAG_WORDS flags + scalar read-backs (h_flags[FLAG_WORDS]: division count)
    CG_CUDA_CHECK(cudaMallocHost((void**)&c->h_flags, (FLAG_WORDS + 4) * sizeof(int)));
    ALLOC(c->d_fac, (size_t)S * 3 * 2 * c->nmax * sizeof(double));
    ALLOC(c->d_r, (size_t)S * 3 * sizeof(double));
    ALLOC(c->d_diri, (size_t)S * sizeof(double));
    ALLOC(c->d_sat, (size_t)S * sizeof(double));
    ALLOC(c->d_counts, (size_t)c->nvox * sizeof(int));
    ALLOC(c->d_part, (size_t)(c->n_part + 1) * sizeof(unsigned long long));
    ALLOC(c->d_scan_incl, (size_t)(c->n_part + 1) * sizeof(unsigned long long));
    ALLOC(c->d_scan_flag, (size_t)(c->n_part + 2) * sizeof(int));
    ALLOC(c->d_row_ne, ((size_t)ny * nz + 1) * sizeof(int));
    ALLOC(c->d_ne_start, ((size_t)std::min<long>(c->nvox, (long)cap) + 1) * sizeof(int));
    ALLOC(c->d_sp, cap * 4 * sizeof(double));
    ALLOC(c->d_spf, cap * sizeof(float4));
    ALLOC(c->d_sid, cap * sizeof(long long));
    ALLOC(c->d_sid32, cap * sizeof(int));
    ALLOC(c->d_cand, (size_t)std::min<long>(c->nvox, (long)cap) * 64 * sizeof(int));
    ALLOC(c->d_slot_list, cap * sizeof(int));
    ALLOC(c->d_svox, cap * sizeof(int));
    ALLOC(c->d_exA, (size_t)S * cap * sizeof(double));
    ALLOC(c->d_exD, (size_t)S * cap * sizeof(double));
    ALLOC(c->d_exR, (size_t)S * std::min<long>(c->nvox, (long)cap) * 2 * kRecCells * sizeof(double));
    c->xset[0].A = c->d_exA;
    c->xset[0].D = c->d_exD;
    c->xset[0].R = c->d_exR;
    ALLOC(c->d_overflow, (size_t)std::min<long>(c->nvox, (long)cap) * sizeof(int));
    ALLOC(c->d_mid, (size_t)std::min<long>(c->nvox, (long)cap) * sizeof(int));
    ALLOC(c->d_big, (size_t)std::min<long>(c->nvox, (long)cap) * sizeof(int));
    ALLOC(c->d_n_big, sizeof(int));
    ALLOC(c->d_n_overflow, 3 * sizeof(int));
    ALLOC(c->d_div_list, cap * sizeof(int));
    ALLOC(c->d_div_n, sizeof(int));
#undef ALLOC
    CG_CUDA_CHECK(cudaMemset(c->d_flags, 0, FLAG_WORDS * sizeof(int)));
    CG_CUDA_CHECK(cudaMemset(c->d_counts, 0, (size_t)c->nvox * sizeof(int)));
    CG_CUDA_CHECK(cudaMemset(c->d_scan_flag, 0, (size_t)(c->n_part + 2) * sizeof(int)));
    CG_CUDA_CHECK(cudaMemset(c->d_part, 0, (size_t)(c->n_part + 1) * sizeof(unsigned long long)));
    CG_CUDA_CHECK(cudaMemset(c->d_scan_incl, 0, (size_t)(c->n_part + 1) * sizeof(unsigned long long)));
    CG_CUDA_CHECK(cudaMemset(c->d_n_overflow, 0, 3 * sizeof(int)));
    CG_CUDA_CHECK(cudaMemset(c->d_n_big, 0, sizeof(int)));
    std::vector<double> zeros(S, 0.0);
    CG_CUDA_CHECK(cudaMemcpy(c->d_diri, zeros.data(), S * sizeof(double), cudaMemcpyHostToDevice));
    CG_CUDA_CHECK(cudaMemcpy(c->d_sat, zeros.data(), S * sizeof(double), cudaMemcpyHostToDevice));
    c->big_smem = 200 * 1024;
    if (const char* e = std::getenv("CELLGPU_PDL")) c->pdl = std::atoi(e) != 0;
    if (const char* e = std::getenv("CELLGPU_PDL_MASK")) c->pdl_mask = std::strtoull(e, nullptr, 0);
    if (const char* e = std::getenv("CELLGPU_PLANE_THREADS")) c->plane_threads = std::atoi(e);
    if (const char* e = std::getenv("CELLGPU_REGLINES")) c->reg_lines = std::atoi(e) != 0;
    if (const char* e = std::getenv("CELLGPU_VEL_CTAS")) c->vel_ctas_per_sm = std::atoi(e);
    if (const char* e = std::getenv("CELLGPU_EXCH_SPLIT")) c->exch_split = std::atoi(e) != 0;
    int st = init_cells_kernels(c);
    if (st) return st;
    CG_CUDA_CHECK(cudaDeviceSynchronize());
    *out = c;
    return CG_OK;
}

extern "C" void cg_ctx_destroy(cg_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& r : c->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    cudaFree(c->d_flags);
    cudaFree(c->d_digest);
    cudaFreeHost(c->h_flags);
    cudaFree(c->d_fac);
    cudaFree(c->d_r);
    cudaFree(c->d_diri);
    cudaFree(c->d_sat);
    cudaFree(c->d_counts);
    cudaFree(c->d_part);
    cudaFree(c->d_scan_incl);
    cudaFree(c->d_scan_flag);
    cudaFree(c->d_row_ne);
    cudaFree(c->d_ne_start);
    cudaFree(c->d_sp);
    cudaFree(c->d_spf);
    cudaFree(c->d_sid);
    cudaFree(c->d_sid32);
    cudaFree(c->d_cand);
    cudaFree(c->d_slot_list);
    cudaFree(c->d_svox);
    cudaFree(c->d_segf);
    cudaFree(c->d_exA);
    cudaFree(c->d_exD);
    cudaFree(c->d_exR);
    cudaFree(c->d_div_list);
    cudaFree(c->d_div_n);
    if (c->xset_alloc) {
        for (int k = 1; k < kExchSets; k++) {
            cudaFree(c->xset[k].A);
            cudaFree(c->xset[k].D);
            cudaFree(c->xset[k].R);
        }
        for (ExchSet& x : c->xset) {
            cudaFree(x.vox);
            cudaFree(x.start);
            cudaFree(x.n);
        }
    }
    if (c->fast_sets)
        for (ExchSet& x : c->xset) {
            cudaFree(x.aff);
            cudaFree(x.pz);
        }
    cudaFree(c->d_overflow);
    cudaFree(c->d_mid);
    cudaFree(c->d_big);
    cudaFree(c->d_n_big);
    cudaFree(c->d_n_overflow);
    cudaFree(c->d_spk);
    cudaFree(c->d_ends);
    delete c;
}

extern "C" int cg_ctx_set_stream(cg_ctx* c, void* stream) {
    c->stream = (cudaStream_t)stream;
    return CG_OK;
}

extern "C" int cg_sync(cg_ctx* c) {
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    CG_CUDA_CHECK(cudaMemcpyAsync(c->h_flags, c->d_flags, FLAG_WORDS * sizeof(int),
                                  cudaMemcpyDeviceToHost, c->stream));
    CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    int code = CG_OK;
    if (c->h_flags[FLAG_DOMAIN]) code = set_error(CG_DOMAIN, "domain error raised on device");
    else if (c->h_flags[FLAG_NUMERIC])
        code = set_error(CG_NUMERIC, "substrate field left finite/non-negative range");
    else if (c->h_flags[FLAG_CAPACITY])
        code = set_error(CG_CAPACITY, "voxel candidate list exceeds the velocity kernel capacity");
    if (code != CG_OK) {
        // Leave the scratch in a clean state after a failed call.
        CG_CUDA_CHECK(cudaMemsetAsync(c->d_flags, 0, FLAG_WORDS * sizeof(int), c->stream));
        CG_CUDA_CHECK(cudaMemsetAsync(c->d_counts, 0, (size_t)c->nvox * sizeof(int), c->stream));
        CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    }
    return code;
}

int check_cells(cg_ctx* c, int n) {
    if (n < 0) return set_error(CG_DOMAIN, "negative cell count");
    if (n > c->cap_cells) return set_error(CG_CAPACITY, "cell count exceeds the context capacity");
    return CG_OK;
}

// ---------------------------------------------------------------- hot-path calls

extern "C" int cg_lod_step(cg_ctx* c, double* dens, const double* diffusion, const double* decay,
                           double dt, int bc, const double* dirichlet) {
    if (!(dt > 0.0)) return set_error(CG_DOMAIN, "diffusion step needs dt > 0");
    if (c->S == 0) return CG_OK;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    int st = ensure_factors(c, dt, diffusion, decay);
    if (st) return st;
    if (bc == CG_BC_DIRICHLET) {
        if (!dirichlet) return set_error(CG_DOMAIN, "dirichlet boundary needs values");
        if ((st = ensure_dirichlet(c, dirichlet))) return st;
    }
    return launch_lod(c, dens, bc, nullptr, nullptr, nullptr, 0);
}

extern "C" int cg_state_checksum(cg_ctx* c, int n_cells, const int64_t* ids, const double* pos,
                                 const double* vel, uint64_t* digest) {
    if (n_cells < 0) return set_error(CG_DOMAIN, "negative cell count");
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    int st = launch_state_checksum(c, n_cells, ids, pos, vel, c->d_digest);
    if (st) return st;
    unsigned long long h[2];
    CG_CUDA_CHECK(cudaMemcpyAsync(h, c->d_digest, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    digest[0] = h[0];
    digest[1] = h[1];
    return CG_OK;
}

// Microenvironment.check_state (core.py:142-144) on the device: raises
// (at the next cg_sync) CG_NUMERIC when a value is non-finite or negative.
extern "C" int cg_check_state(cg_ctx* c, const double* dens) {
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_check_field(c, dens, (long)c->S * c->nvox);
}

extern "C" int cg_gradients(cg_ctx* c, const double* dens, double* grad) {
    if (c->m.slab) return set_error(CG_STATE, "gradients need the whole z range (not a z-slab context)");
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_gradients(c, dens, grad);
}

extern "C" int cg_exchange(cg_ctx* c, double* dens, int substrate, double dt, double secretion,
                           double uptake, double saturation, int n_cells, const double* volume,
                           const int32_t* bin_start, const int32_t* bin_cells_by_id,
                           const int32_t* nonempty, const int32_t* n_nonempty) {
    if (!(dt > 0.0)) return set_error(CG_DOMAIN, "exchange needs dt > 0");
    if (substrate < 0 || substrate >= c->S) return set_error(CG_DOMAIN, "substrate index out of range");
    int st = check_cells(c, n_cells);
    if (st) return st;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_exchange_scalar(c, dens + (long)substrate * c->nvox, dt, secretion, uptake,
                                  saturation, n_cells, volume, bin_start, bin_cells_by_id,
                                  nonempty, n_nonempty);
}

extern "C" int cg_exchange_cells(cg_ctx* c, double* dens, double dt, const double* secretion,
                                 const double* uptake, const double* saturation, int n_cells,
                                 const double* volume, const int32_t* bin_start,
                                 const int32_t* bin_cells_by_id, const int32_t* nonempty,
                                 const int32_t* n_nonempty) {
    if (!(dt > 0.0)) return set_error(CG_DOMAIN, "exchange needs dt > 0");
    int st = check_cells(c, n_cells);
    if (st) return st;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if ((st = ensure_saturation(c, saturation))) return st;
    if ((st = launch_exchange_coef(c, dt, secretion, uptake, n_cells, volume, bin_cells_by_id)))
        return st;
    return launch_exchange_apply(c, dens, n_cells, bin_start, nonempty, n_nonempty);
}

extern "C" int cg_rebin(cg_ctx* c, int n_cells, const double* pos, const int64_t* ids,
                        int32_t* voxel, int32_t* bin_start, int32_t* bin_cells,
                        int32_t* bin_cells_by_id, int32_t* nonempty, int32_t* n_nonempty) {
    int st = check_cells(c, n_cells);
    if (st) return st;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    c->exch_ready = false;
    return launch_rebin(c, n_cells, pos, ids, voxel, bin_start, bin_cells, bin_cells_by_id,
                        nonempty, n_nonempty);
}

extern "C" int cg_rebin_exchange(cg_ctx* c, int n_cells, const double* pos, const int64_t* ids,
                                 int32_t* voxel, int32_t* bin_start, int32_t* bin_cells,
                                 int32_t* bin_cells_by_id, int32_t* nonempty,
                                 int32_t* n_nonempty, double dt, const double* secretion,
                                 const double* uptake, const double* saturation,
                                 const double* volume) {
    if (!(dt > 0.0)) return set_error(CG_DOMAIN, "exchange needs dt > 0");
    int st = check_cells(c, n_cells);
    if (st) return st;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if ((st = ensure_saturation(c, saturation))) return st;
    const CoefLaunch cl{dt, secretion, uptake, volume};
    c->exch_ready = n_cells > 0;
    c->exch_affine = false;
    c->exch_n = n_cells;
    return launch_rebin(c, n_cells, pos, ids, voxel, bin_start, bin_cells, bin_cells_by_id,
                        nonempty, n_nonempty, false, n_cells > 0 ? &cl : nullptr);
}

static int ensure_exch_sets(cg_ctx* c);
static int ensure_fast_sets(cg_ctx* c);

// Fast numerics for hand-written step loops (the z-slab driver): the rebin
// plus each non-empty voxel's exchange as one affine map per substrate
// (exchange set 0), consumed by cg_lod_step_fast.
extern "C" int cg_rebin_exchange_affine(cg_ctx* c, int n_cells, const double* pos,
                                        const int64_t* ids, int32_t* voxel, int32_t* bin_start,
                                        int32_t* bin_cells, int32_t* bin_cells_by_id,
                                        int32_t* nonempty, int32_t* n_nonempty, double dt,
                                        const double* secretion, const double* uptake,
                                        const double* saturation, const double* volume) {
    if (!(dt > 0.0)) return set_error(CG_DOMAIN, "exchange needs dt > 0");
    int st = check_cells(c, n_cells);
    if (st) return st;
    if (fast_lod_kind(c) == 0) return set_error(CG_STATE, "no fast LOD kernels for this mesh");
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if ((st = ensure_saturation(c, saturation)) || (st = ensure_exch_sets(c)) ||
        (st = ensure_fast_sets(c)))
        return st;
    const CoefLaunch cl{dt, secretion, uptake, volume, &c->xset[0], true};
    c->exch_ready = n_cells > 0;
    c->exch_affine = true;
    c->exch_n = n_cells;
    return launch_rebin(c, n_cells, pos, ids, voxel, bin_start, bin_cells, bin_cells_by_id,
                        nonempty, n_nonempty, false, n_cells > 0 ? &cl : nullptr);
}

// One LOD step with the fast kernels of this mesh (slab-aware: the z sweep
// of a slab context is the local block solve); exchange != 0 applies the
// affine maps of the last cg_rebin_exchange_affine first.
extern "C" int cg_lod_step_fast(cg_ctx* c, double* dens, const double* diffusion,
                                const double* decay, double dt, int bc, const double* dirichlet,
                                int exchange) {
    if (!(dt > 0.0)) return set_error(CG_DOMAIN, "diffusion step needs dt > 0");
    if (c->S == 0) return CG_OK;
    if (fast_lod_kind(c) == 0) return set_error(CG_STATE, "no fast LOD kernels for this mesh");
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    int st = ensure_factors(c, dt, diffusion, decay);
    if (st) return st;
    if (bc == CG_BC_DIRICHLET) {
        if (!dirichlet) return set_error(CG_DOMAIN, "dirichlet boundary needs values");
        if ((st = ensure_dirichlet(c, dirichlet))) return st;
    }
    if ((st = prepare_lod_fast(c))) return st;
    if (exchange && !c->exch_ready) exchange = 0;  // no cells
    if (exchange && (!c->fast_sets || !c->exch_affine))
        return set_error(CG_STATE, "no affine exchange maps (cg_rebin_exchange_affine)");
    const ExchSet& x = c->xset[0];
    st = launch_lod_fast(c, dens, bc, exchange ? x.vox : nullptr, x.n,
                         exchange ? x.aff : nullptr, x.pz, 3, false, false);
    c->pend_lr = nullptr;  // a deferred correction is applied by this step's first kernel
    return st;
}

extern "C" int cg_fast_lod_available(cg_ctx* c) { return fast_lod_kind(c) > 0 ? 1 : 0; }

// Fast-numerics velocities (per cell over its 9 neighbour rows) from a
// rebin's voxel keys, offsets and id-sorted bins.
extern "C" int cg_velocities_fast(cg_ctx* c, int n_cells, const double* pos, const double* radius,
                                  const int32_t* voxel, const int32_t* bin_start,
                                  const int32_t* bin_cells_by_id, double repulsion,
                                  double adhesion, double adhesion_multiplier, double* vel) {
    int st = check_cells(c, n_cells);
    if (st) return st;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_velocities_fast(c, n_cells, pos, radius, voxel, bin_start, bin_cells_by_id,
                                  false, false, repulsion, adhesion, adhesion_multiplier, vel);
}

extern "C" int cg_exchange_prepared(cg_ctx* c, double* dens, int n_cells, const int32_t* nonempty,
                                    const int32_t* n_nonempty) {
    if (n_cells == 0) return CG_OK;
    if (!c->exch_ready || n_cells != c->exch_n || c->exch_affine)
        return set_error(CG_STATE, "no exchange coefficients for these cells (cg_rebin_exchange)");
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_exchange_rec(c, dens, n_cells, nonempty, n_nonempty);
}

extern "C" int cg_velocities(cg_ctx* c, int n_cells, const double* pos, const double* radius,
                             const int64_t* ids, const int32_t* bin_start,
                             const int32_t* bin_cells_by_id, const int32_t* nonempty,
                             const int32_t* n_nonempty, double repulsion, double adhesion,
                             double adhesion_multiplier, double* vel) {
    int st = check_cells(c, n_cells);
    if (st) return st;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_velocities(c, n_cells, pos, radius, ids, nullptr, bin_start, bin_cells_by_id, nonempty,
                             n_nonempty, repulsion, adhesion, adhesion_multiplier, vel, true);
}

extern "C" int cg_integrate(cg_ctx* c, int n_cells, double* pos, const double* vel,
                            double* prev_vel, double dt, int integrator) {
    if (!(dt > 0.0)) return set_error(CG_DOMAIN, "integration needs dt > 0");
    if (integrator == CG_AB2 && !prev_vel) return set_error(CG_DOMAIN, "AB2 needs prev_vel");
    int st = check_cells(c, n_cells);
    if (st) return st;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_integrate(c, n_cells, pos, vel, prev_vel, dt, integrator);
}

// ---------------------------------------------------------------- z slabs

extern "C" int cg_ctx_set_slab_bounds(cg_ctx* c, int rank, int world, int nz_global,
                                      const int* starts) {
    if (world < 1 || rank < 0 || rank >= world || world > 32)
        return set_error(CG_DOMAIN, "slab rank/world out of range (world <= 32)");
    if (starts[0] != 0 || starts[world] != nz_global)
        return set_error(CG_DOMAIN, "slab starts must run from 0 to nz_global");
    for (int k = 0; k < world; k++)
        if (starts[k + 1] <= starts[k]) return set_error(CG_DOMAIN, "every slab needs >= 1 plane");
    const int z0 = starts[rank];
    if (c->m.nz != starts[rank + 1] - z0)
        return set_error(CG_DOMAIN, "context mesh does not match this rank's slab");
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    c->slab_starts.assign(starts, starts + world + 1);
    c->slab_rank = rank;
    c->slab_world = world;
    c->nz_global = nz_global;
    c->slab_z0 = z0;
    c->m.zlo = z0 == 0;
    c->m.zhi = z0 + c->m.nz == nz_global;
    c->m.slab = world > 1;
    const int S = std::max(c->S, 1);
    cudaFree(c->d_spk);
    cudaFree(c->d_ends);
    c->d_spk = nullptr;
    c->d_ends = nullptr;
    CG_CUDA_CHECK(cudaMalloc((void**)&c->d_spk, (size_t)S * 2 * c->m.nz * sizeof(double)));
    CG_CUDA_CHECK(cudaMalloc((void**)&c->d_ends, (size_t)S * world * 4 * sizeof(double)));
    c->fac_key.clear();  // z factors depend on the split
    return CG_OK;
}

extern "C" int cg_ctx_set_slab(cg_ctx* c, int rank, int world, int nz_global, int z0) {
    if (world < 1 || world > 32 || nz_global < world)
        return set_error(CG_DOMAIN, "slab rank/world out of range (world <= 32)");
    std::vector<int> starts(world + 1);
    const int base = nz_global / world, rem = nz_global % world;
    for (int k = 0; k <= world; k++) starts[k] = k * base + std::min(k, rem);
    if (rank >= 0 && rank < world && z0 != starts[rank])
        return set_error(CG_DOMAIN, "slab does not match the balanced split of nz_global");
    return cg_ctx_set_slab_bounds(c, rank, world, nz_global, starts.data());
}

extern "C" int cg_zslab_pack(cg_ctx* c, const double* dens, double* send) {
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_zslab_pack(c, dens, send);
}

extern "C" int cg_zslab_correct(cg_ctx* c, double* dens, const double* recv, int bc,
                                const double* dirichlet) {
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (c->slab_world < 2) return CG_OK;
    if (bc == CG_BC_DIRICHLET) {
        if (!dirichlet) return set_error(CG_DOMAIN, "dirichlet boundary needs values");
        int st = ensure_dirichlet(c, dirichlet);
        if (st) return st;
    }
    return launch_zslab_correct(c, dens, recv, bc);
}

// Substrate window of the following context calls (include/cellgpu.h).
extern "C" int cg_ctx_set_substrate_window(cg_ctx* c, int s0, int ns) {
    if (ns == 0 && s0 == 0) {
        c->sub0 = 0;
        c->sub_n = 0;
        return CG_OK;
    }
    if (s0 < 0 || ns < 1 || s0 + ns > c->S) return set_error(CG_DOMAIN, "substrate window out of range");
    c->sub0 = s0;
    c->sub_n = ns;
    return CG_OK;
}

// The interface system by line blocks (all-to-all variant; include/cellgpu.h).
extern "C" long cg_zslab_block_lines(cg_ctx* c) {
    return c->slab_world >= 2 ? zslab_block_lines(c) : (long)c->m.nx * c->m.ny;
}

extern "C" int cg_zslab_pack_blocks(cg_ctx* c, const double* dens, double* send) {
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (c->slab_world < 2) return set_error(CG_STATE, "not a z-slab context of 2 or more ranks");
    return launch_zslab_pack_blocks(c, dens, send);
}

extern "C" int cg_zslab_reduce_blocks(cg_ctx* c, const double* recv, double* out) {
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (c->slab_world < 2) return set_error(CG_STATE, "not a z-slab context of 2 or more ranks");
    return launch_zslab_reduce_blocks(c, recv, out);
}

extern "C" int cg_zslab_lr_gather(cg_ctx* c, const double* recv, double* lr) {
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (c->slab_world < 2) return set_error(CG_STATE, "not a z-slab context of 2 or more ranks");
    return launch_zslab_lr_gather(c, recv, lr);
}

// Defer this substep's interface correction to the next cg_lod_step_fast on
// the context (all substrates): its x-row / plane kernel applies
// x += left v + right w as it stages the field (the correction's Dirichlet
// pins coincide with the kernel's own).  Saves the correction's full read +
// write pass of the field.  lr: (world, S, 2, Lb), kept alive by the caller.
extern "C" int cg_zslab_defer(cg_ctx* c, const double* lr) {
    if (c->slab_world < 2) return set_error(CG_STATE, "not a z-slab context of 2 or more ranks");
    if (lr && (fast_lod_kind(c) < 2 || c->sub_n > 0))
        return set_error(CG_STATE, "deferred corrections need the fast slab kernels, all substrates");
    c->pend_lr = lr;
    return CG_OK;
}

extern "C" int cg_zslab_correct_blocks(cg_ctx* c, double* dens, const double* lr, int bc,
                                       const double* dirichlet) {
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (c->slab_world < 2) return set_error(CG_STATE, "not a z-slab context of 2 or more ranks");
    if (bc == CG_BC_DIRICHLET) {
        if (!dirichlet) return set_error(CG_DOMAIN, "dirichlet boundary needs values");
        int st = ensure_dirichlet(c, dirichlet);
        if (st) return st;
    }
    return launch_zslab_correct_lr(c, dens, lr, bc);
}

extern "C" int cg_voxel_z(cg_ctx* c, int n_cells, const double* pos, int32_t* out) {
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_voxel_z(c, n_cells, pos, out);
}

extern "C" int cg_voxel_index(cg_ctx* c, int n_cells, const double* pos, int32_t* out) {
    if (n_cells < 0) return set_error(CG_DOMAIN, "negative cell count");
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    return launch_voxel_index(c, n_cells, pos, out, true);
}

// ---------------------------------------------------------------- step engine

struct cg_engine {
    cg_ctx* ctx;
    cg_state_ptrs p;
    cg_step_params q;
    std::vector<double> diffusion, decay, dirichlet, saturation;
    // Step graphs when the exchange sets rotate: graph[k] reads xset[k] and
    // its rebin writes xset[(k + 1) % kExchSets].
    cudaGraph_t graph[kExchSets] = {};
    cudaGraphExec_t exec[kExchSets] = {};
    bool dbl = false;  // rotating exchange sets (rebin beside the substeps)
    bool fast = false;  // CG_NUMERICS_FAST: segmented LOD + affine exchange + direct velocities
    // Substrate chains for device-resident steps too (env CELLGPU_RESIDENT_CHAINS=1).
    bool resident_chains = false;
    // Fast velocities: four lanes per cell when voxels are dense (mean cells
    // per non-empty voxel >= 2 at creation: config 2's spheroid, 2.2, vs
    // 1.3-1.6 for the uniform configs, where one thread per cell is faster);
    // env CELLGPU_VEL_KERNEL=cell|quad overrides.
    bool vel_quad = false;
    // Exact velocities: warp-per-cell pass for cells with many candidates
    // (k_velocity_exact_dense) only when voxels are dense by the same test.
    bool vel_dense = true;
    double* sort_tmp = nullptr;     // cg_engine_sort_cells scratch (n x 3)
    int32_t* sort_order = nullptr;  // (n)
    int cur = 0;       // exchange set the next step reads
    int launches_per_step = 0;
    // Pipelined host-driven steps (cg_engine_step_io): the mechanics branch
    // and every substrate chain as separate graphs on their own streams,
    // ordered by events only, so a substrate's next step starts when its own
    // field is back and the previous step's rebin is done -- not when the
    // whole previous step is.
    cudaGraph_t pg_mech[kExchSets] = {}, pg_chain[kLineMaxS][kExchSets] = {};
    cudaGraphExec_t px_mech[kExchSets] = {}, px_chain[kLineMaxS][kExchSets] = {};
    cudaEvent_t ev_mech = nullptr, ev_chain[kLineMaxS][kExchSets] = {};
    bool pipe_ready = false;
    // cg_engine_step_host: copy streams, per-piece download events, pieces.
    struct HostIo {
        cudaStream_t up_fields = nullptr, up_cells = nullptr, down_fields = nullptr,
                     down_cells = nullptr;
        // per-substrate field copy streams (default with substrate chains;
        // env CELLGPU_IO_STREAMS=shared: one stream per direction): a
        // substrate's pieces queue only behind its own (config 1 e2e 0.446-
        // 0.456 vs 0.491-0.499 ms per step; fields first / cells first: 0.47-0.50)
        cudaStream_t up_sub[kLineMaxS] = {}, down_sub[kLineMaxS] = {};
        bool per_sub = false;
        std::vector<cudaEvent_t> piece_out;  // download of piece i done
        cudaEvent_t cells_out = nullptr;
        std::vector<int> piece_sub;           // substrate of piece i (-1: all)
        std::vector<long> piece_lo, piece_hi;  // element range of piece i
        int chunks = 0;
    } hio;
    bool overlap = true;  // velocities concurrent with the substeps: env CELLGPU_OVERLAP=0 disables
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // Host-driven steps (cg_engine_io_enable): the velocity branch waits for
    // io_in (positions / AB2 state uploaded on the caller's copy stream), and
    // io_fields marks the end of the substeps so the densities can be copied
    // out while the mechanics finish.  Both are external event nodes in the graph.
    // io_dens (optional, recorded by the caller after the density upload)
    // gates only the substeps; io_cells marks positions / velocities final and
    // the rebin done, so they can be copied out (and the next positions in)
    // while the substeps still run.
    cudaEvent_t io_in = nullptr, io_fields = nullptr, io_dens = nullptr, io_cells = nullptr;
    // Per-substrate field events (cg_engine_io_substrate_ready / _wait_substrate).
    cudaEvent_t io_sub_in[kLineMaxS] = {}, io_sub_out[kLineMaxS] = {};
    // Substrate chains: the substeps of substrate s on stream sub[s].
    int chains = 1;
    cudaStream_t sub[kLineMaxS] = {};
    cudaEvent_t ev_sfork = nullptr, ev_sjoin[kLineMaxS] = {};
};

// simulate.py:169-202 minus divisions/resort (out of scope); gradients on request.
// Precondition: bins and exchange coefficients match the current positions.
//
// The velocity update reads only positions, radii, ids and the bins -- never
// the substrate fields -- and the substeps never touch positions, so the two
// are independent: velocities run on a second stream concurrently with the
// 10 diffusion substeps (fork/join by events, captured into the graph), and
// integration joins them.  Results are unchanged (no shared writes).
//
// The rebin that closes the step writes the bins and the next step's exchange
// coefficients.  With double-buffered exchange sets (e->dbl) the substeps read
// only xset[par] and the rebin writes xset[1 - par], so integration and rebin
// follow the velocities on the second stream as well and the step's critical
// path is the longer of the two chains.
// Fast numerics with the segmented LOD kernels (their plane kernel applies
// the affine exchange maps the bin fix-up writes into the exchange sets).
static bool engine_fast_lod(const cg_engine* e) { return e->fast && fast_lod_kind(e->ctx) > 0; }
// The velocities' slot arrays ((x, y, z, R), voxel) can be gathered by the
// rebin's bin fix-up (fast numerics, with the exchange coefficients; env
// CELLGPU_REBIN_GATHER=1) or by the velocity branch (default): the fix-up is
// on the step's serial tail while the velocity branch overlaps the
// diffusion.  Measured with the gather in the branch: config 1 0.164 vs
// 0.166 ms per step, config 2 0.274 vs 0.283, config 3 1.838 vs 1.845
// (exact numerics with the ids too: config 1 0.235 vs 0.249).
// Fast numerics: the bin fix-up also gathers the next step's velocity slot
// arrays (x, y, z, R) and voxels, so the velocity branch starts without
// k_gather_fast.  Default: when the mechanics follow the substeps (no
// overlap: config 3), where the gather launch is on the critical path; with
// the branch beside the substeps the fix-up is its serial tail instead
// (config 1 0.164 vs 0.166 ms without).  env CELLGPU_REBIN_GATHER overrides.
static bool engine_rebin_gathers(const cg_engine* e) {
    const cg_state_ptrs& p = e->p;
    const char* env = std::getenv("CELLGPU_REBIN_GATHER");
    const bool on = env ? std::atoi(env) != 0 : !e->overlap;
    return on && e->fast && p.secretion && p.uptake && e->q.n_cells > 0;
}

static int probe_skip();

static int launch_mechanics_tail(cg_engine* e, int wset) {
    if (probe_skip() & 2) return CG_OK;
    cg_ctx* c = e->ctx;
    const cg_state_ptrs& p = e->p;
    const cg_step_params& q = e->q;
    const bool ex = p.secretion && p.uptake && q.n_cells > 0;
    // integrate + voxel keys/histogram in one pass, then the single-pass scan,
    // scatter, and the bin fix-up that also computes the next step's exchange
    // coefficients (into exchange set wset).
    int st;
    if ((st = launch_integrate(c, q.n_cells, p.pos, p.vel, p.prev_vel, q.dt_mechanics,
                               q.integrator, q.n_cells > 0 ? p.voxel : nullptr)))
        return st;
    // Positions, velocities and the AB2 state are final here and the rest of
    // the rebin does not read them: host-driven steps copy them out now.
    if (e->io_cells)
        CG_CUDA_CHECK(cudaEventRecordWithFlags(e->io_cells, c->stream, cudaEventRecordExternal));
    const bool g = engine_rebin_gathers(e);
    const CoefLaunch cl{q.dt_diffusion, p.secretion, p.uptake, p.volume,
                        (e->dbl || e->fast) ? &c->xset[wset] : nullptr, engine_fast_lod(e),
                        g ? p.pos : nullptr, g ? p.radius : nullptr};
    return launch_rebin(c, q.n_cells, p.pos, p.ids, p.voxel, p.bin_start, p.bin_cells,
                        p.bin_cells_by_id, p.nonempty, p.n_nonempty, q.n_cells > 0,
                        ex ? &cl : nullptr);
}

// The mechanics branch of a step: velocities (they read only positions,
// radii, ids and the bins) and, if the substeps do not read the rebin's
// outputs, integration and rebin, writing exchange set wset.
// Probe build only (-DCG_PROBE, tools/side_probe.py): env CELLGPU_PROBE_SKIP
// bit 0 skips the velocities, bit 1 the integration + rebin -- a timing
// probe of what each part of the mechanics branch costs the step (results
// are wrong while set; the product library has no such switch).
#ifdef CG_PROBE
static int probe_skip() {
    const char* env = std::getenv("CELLGPU_PROBE_SKIP");
    return env ? std::atoi(env) : 0;
}
#else
static int probe_skip() { return 0; }
#endif

static int launch_mechanics(cg_engine* e, bool with_tail, int wset) {
    cg_ctx* c = e->ctx;
    const cg_state_ptrs& p = e->p;
    const cg_step_params& q = e->q;
    if (probe_skip() & 1) return with_tail && !(probe_skip() & 2) ? launch_mechanics_tail(e, wset) : CG_OK;
    int st = e->fast ? launch_velocities_fast(c, q.n_cells, p.pos, p.radius, p.voxel, p.bin_start,
                                              p.bin_cells_by_id, engine_rebin_gathers(e),
                                              e->vel_quad, q.repulsion, q.adhesion,
                                              q.adhesion_multiplier, p.vel)
                     : launch_velocities(c, q.n_cells, p.pos, p.radius, p.ids, p.voxel, p.bin_start,
                                         p.bin_cells_by_id, p.nonempty, p.n_nonempty, q.repulsion,
                                         q.adhesion, q.adhesion_multiplier, p.vel, e->vel_dense);
    if (!st && with_tail) st = launch_mechanics_tail(e, wset);
    return st;
}

// The substeps of substrates [s0, s0 + ns) (ns = 0: all), reading exchange
// set rset.
static int launch_substeps(cg_engine* e, int s0, int ns, int rset) {
    cg_ctx* c = e->ctx;
    const cg_state_ptrs& p = e->p;
    const cg_step_params& q = e->q;
    const bool ex = p.secretion && p.uptake && q.n_cells > 0;
    c->sub0 = s0;
    c->sub_n = ns;
    int st = CG_OK;
    if (engine_fast_lod(e)) {
        // exchange fused into the segmented plane kernel (affine maps of set rset)
        const ExchSet& x = c->xset[rset];
        for (int k = 0; !st && k < q.substeps; k++)
            st = launch_lod_fast(c, p.dens, q.bc, ex ? x.vox : nullptr, x.n, ex ? x.aff : nullptr,
                                 x.pz, 3, k + 1 == q.substeps, k > 0);
        c->sub0 = 0;
        c->sub_n = 0;
        return st;
    }
    for (int k = 0; !st && k < q.substeps; k++) {
        // G4 exchange fused into the x/y plane kernel (or the x-row kernel),
        // or as its own kernel right before it (exch_split).
        const bool fuse = ex && !lod_exchange_split(c);
        if (ex && !fuse)
            st = launch_exchange_rec(c, p.dens, q.n_cells, p.nonempty, p.n_nonempty,
                                     e->dbl ? &c->xset[rset] : nullptr, k > 0);
        // simulate.py:218: micro.check_state() once per step, on the final field
        if (!st)
            st = launch_lod(c, p.dens, q.bc, p.nonempty, fuse ? c->d_exA : nullptr,
                            fuse ? c->d_exD : nullptr, q.n_cells, 3, k + 1 == q.substeps);
    }
    c->sub0 = 0;
    c->sub_n = 0;
    return st;
}

static int engine_step(cg_engine* e) {
    cg_ctx* c = e->ctx;
    const cg_state_ptrs& p = e->p;
    const cg_step_params& q = e->q;
    const bool ex = p.secretion && p.uptake && q.n_cells > 0;
    const int rset = e->dbl ? e->cur : 0, wset = e->dbl ? (e->cur + 1) % kExchSets : 0;
    int st;
    const bool fork = e->overlap && e->side != nullptr;
    // the rebin may run beside the substeps unless they read its outputs
    const bool tail_on_side = fork && (e->dbl || !ex);
    cudaStream_t main = c->stream;
    if (fork) {
        CG_CUDA_CHECK(cudaEventRecord(e->ev_fork, main));
        CG_CUDA_CHECK(cudaStreamWaitEvent(e->side, e->ev_fork, 0));
        if (e->io_in) CG_CUDA_CHECK(cudaStreamWaitEvent(e->side, e->io_in, cudaEventWaitExternal));
        c->stream = e->side;
        st = launch_mechanics(e, tail_on_side, wset);
        c->stream = main;
        if (st) return st;
        CG_CUDA_CHECK(cudaEventRecord(e->ev_join, e->side));
    }
    if (e->io_dens) CG_CUDA_CHECK(cudaStreamWaitEvent(main, e->io_dens, cudaEventWaitExternal));
    // Substrate chains only pay off when fields move per substrate between
    // host and device (host-driven steps: 0.48 vs 0.65 ms per step at config
    // 1); device-resident steps run all substrates per launch (0.285 vs
    // 0.293 ms with the L2 flushed before every step).
    if (e->chains > 1 && (e->io_in || e->resident_chains)) {
        // Substrates are independent through the substeps (per-substrate
        // sweeps and exchange): one chain per substrate on its own stream, each
        // gated by its own field upload and signalling its own completion, so
        // host-driven steps move the fields substrate by substrate.
        CG_CUDA_CHECK(cudaEventRecord(e->ev_sfork, main));
        for (int s = 0; s < e->chains; s++) {
            cudaStream_t ss = e->sub[s];
            CG_CUDA_CHECK(cudaStreamWaitEvent(ss, e->ev_sfork, 0));
            if (e->io_sub_in[s])
                CG_CUDA_CHECK(cudaStreamWaitEvent(ss, e->io_sub_in[s], cudaEventWaitExternal));
            c->stream = ss;
            st = launch_substeps(e, s, 1, rset);
            c->stream = main;
            if (st) return st;
            if (e->io_sub_out[s])
                CG_CUDA_CHECK(cudaEventRecordWithFlags(e->io_sub_out[s], ss, cudaEventRecordExternal));
            CG_CUDA_CHECK(cudaEventRecord(e->ev_sjoin[s], ss));
            CG_CUDA_CHECK(cudaStreamWaitEvent(main, e->ev_sjoin[s], 0));
        }
    } else {
        for (int s = 0; s < kLineMaxS; s++)
            if (e->io_sub_in[s])
                CG_CUDA_CHECK(cudaStreamWaitEvent(main, e->io_sub_in[s], cudaEventWaitExternal));
        if ((st = launch_substeps(e, 0, 0, rset))) return st;
        for (int s = 0; s < kLineMaxS; s++)
            if (e->io_sub_out[s])
                CG_CUDA_CHECK(cudaEventRecordWithFlags(e->io_sub_out[s], main, cudaEventRecordExternal));
    }
    // simulate.py:184-187: the gradient refresh follows the substeps
    if (q.gradients && p.grad && (st = launch_gradients(c, p.dens, p.grad))) return st;
    if (e->io_fields)
        CG_CUDA_CHECK(cudaEventRecordWithFlags(e->io_fields, main, cudaEventRecordExternal));
    if (!fork && e->io_in) CG_CUDA_CHECK(cudaStreamWaitEvent(main, e->io_in, cudaEventWaitExternal));
    if (fork) {
        CG_CUDA_CHECK(cudaStreamWaitEvent(main, e->ev_join, 0));
    } else if ((st = launch_mechanics(e, false, wset))) {
        return st;
    }
    if (!tail_on_side && (st = launch_mechanics_tail(e, wset))) return st;
    return CG_OK;
}

// Exchange sets for the engine: list/offset copies for all, coefficient
// arrays for sets 1.. (set 0 aliases d_exA/d_exD/d_exR).
static int ensure_exch_sets(cg_ctx* c) {
    if (c->xset_alloc) return CG_OK;
    const size_t cap = (size_t)c->cap_cells, S = (size_t)c->S;
    const size_t rq = (size_t)std::min<long>(c->nvox, c->cap_cells);
    for (int k = 1; k < kExchSets; k++) {
        ExchSet& x = c->xset[k];
        CG_CUDA_CHECK(cudaMalloc((void**)&x.A, S * cap * sizeof(double)));
        CG_CUDA_CHECK(cudaMalloc((void**)&x.D, S * cap * sizeof(double)));
        CG_CUDA_CHECK(cudaMalloc((void**)&x.R, S * rq * 2 * kRecCells * sizeof(double)));
    }
    for (ExchSet& x : c->xset) {
        CG_CUDA_CHECK(cudaMalloc((void**)&x.vox, rq * sizeof(int32_t)));
        CG_CUDA_CHECK(cudaMalloc((void**)&x.start, (rq + 1) * sizeof(int32_t)));
        CG_CUDA_CHECK(cudaMalloc((void**)&x.n, sizeof(int32_t)));
        CG_CUDA_CHECK(cudaMemset(x.n, 0, sizeof(int32_t)));
    }
    c->xset_alloc = true;
    return CG_OK;
}

// Affine exchange maps and per-plane offsets of every exchange set (fast numerics).
static int ensure_fast_sets(cg_ctx* c) {
    if (c->fast_sets) return CG_OK;
    const size_t rq = (size_t)std::min<long>(c->nvox, c->cap_cells);
    for (ExchSet& x : c->xset) {
        CG_CUDA_CHECK(cudaMalloc((void**)&x.aff, (size_t)c->S * rq * 2 * sizeof(double)));
        CG_CUDA_CHECK(cudaMalloc((void**)&x.pz, ((size_t)c->m.ny * c->m.nz + 1) * sizeof(int32_t)));
    }
    c->fast_sets = true;
    return CG_OK;
}

extern "C" int cg_engine_create(cg_ctx* c, const cg_state_ptrs* ptrs, const cg_step_params* params,
                                cg_engine** out) {
    *out = nullptr;
    int st = check_cells(c, params->n_cells);
    if (st) return st;
    if (!(params->dt_diffusion > 0.0) || !(params->dt_mechanics > 0.0))
        return set_error(CG_DOMAIN, "time steps must be > 0");
    if (params->substeps < 1) return set_error(CG_DOMAIN, "substeps must be >= 1");
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    cg_engine* e = new cg_engine();
    e->ctx = c;
    e->p = *ptrs;
    e->q = *params;
    const int S = c->S;
    e->diffusion.assign(params->diffusion, params->diffusion + S);
    e->decay.assign(params->decay, params->decay + S);
    if (params->dirichlet) e->dirichlet.assign(params->dirichlet, params->dirichlet + S);
    else e->dirichlet.assign(S, 0.0);
    if (params->saturation) e->saturation.assign(params->saturation, params->saturation + S);
    else e->saturation.assign(S, 0.0);
    e->q.diffusion = e->diffusion.data();
    e->q.decay = e->decay.data();
    e->q.dirichlet = e->dirichlet.data();
    e->q.saturation = e->saturation.data();
    // The mechanics branch runs beside the substeps when their kernels are
    // single-wave (planes x substrates <= 2 per SM: configs 1, 2, 4 -- the
    // latency-bound sweeps leave room; config 2 0.288 vs 0.368 ms, config 1
    // 0.180 vs 0.204); with multi-wave, bandwidth-bound sweeps (config 3)
    // it only steals their bandwidth (1.985 vs 1.938 ms fast, 3.53 vs 3.52
    // exact) and follows them instead.  env CELLGPU_OVERLAP overrides.
    e->overlap = (long)c->m.nz * std::max(S, 1) <= 2L * c->num_sms;
    if (const char* env = std::getenv("CELLGPU_OVERLAP")) e->overlap = std::atoi(env) != 0;
    if (e->overlap) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        // env CELLGPU_SIDE_PRIO: "high" (default) or "low" priority for the
        // velocity branch relative to the diffusion chain.
        int prio = hi;
        if (const char* env = std::getenv("CELLGPU_SIDE_PRIO")) prio = std::strcmp(env, "low") == 0 ? lo : hi;
        if (cudaStreamCreateWithPriority(&e->side, cudaStreamNonBlocking, prio) != cudaSuccess ||
            cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming) != cudaSuccess) {
            e->overlap = false;
            cudaGetLastError();
        }
    }
    if (S > 0) {
        if ((st = ensure_factors(c, params->dt_diffusion, e->q.diffusion, e->q.decay)) ||
            (st = ensure_dirichlet(c, e->q.dirichlet)) ||
            (st = ensure_saturation(c, e->q.saturation))) {
            delete e;
            return st;
        }
    }
    // seed_cells ends with a rebin (simulate.py:116); the bin fix-up also
    // computes the exchange coefficients of the first step.
    const cg_state_ptrs& p = e->p;
    const bool ex = p.secretion && p.uptake && params->n_cells > 0;
    // Double-buffered exchange sets: the split exchange kernel (S <= 4) reads
    // only its set; env CELLGPU_REBIN_OVERLAP=0 keeps the rebin after the substeps.
    e->dbl = ex && e->overlap && lod_exchange_split(c) && S <= 4;
    if (const char* env = std::getenv("CELLGPU_REBIN_OVERLAP"))
        if (std::atoi(env) == 0) e->dbl = false;
    e->fast = params->numerics == CG_NUMERICS_FAST;
    if ((e->dbl || (e->fast && ex)) && (st = ensure_exch_sets(c))) {
        delete e;
        return st;
    }
    if (e->fast && ex && (st = ensure_fast_sets(c))) {
        delete e;
        return st;
    }
    if (e->fast && S > 0 && (st = prepare_lod_fast(c))) {
        delete e;
        return st;
    }
    // The velocity grids stay uncapped (CELLGPU_VEL_CTAS=2 helps back-to-back
    // steps with a warm L2, 272 vs 280 us at config 1, but costs the bench's
    // L2-flushed steps 0.306 vs 0.293 ms: the velocity branch then runs cold
    // and becomes the critical path).
    // One chain per substrate (register-line kernels, split exchange); env
    // CELLGPU_SUBSTRATE_CHAINS=0 keeps all substrates in one chain.
    if (e->dbl && reg_line_length(c) > 0 && S > 1) {
        e->chains = S;
        if (const char* env = std::getenv("CELLGPU_SUBSTRATE_CHAINS"))
            if (std::atoi(env) == 0) e->chains = 1;
    }
    if (const char* env = std::getenv("CELLGPU_RESIDENT_CHAINS")) e->resident_chains = std::atoi(env) != 0;
    if (e->chains > 1) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        // env CELLGPU_CHAIN_PRIO: "low" (default) or "high" for the substrate chains
        int cprio = lo;
        if (const char* env = std::getenv("CELLGPU_CHAIN_PRIO")) cprio = std::strcmp(env, "high") == 0 ? hi : lo;
        bool ok = cudaEventCreateWithFlags(&e->ev_sfork, cudaEventDisableTiming) == cudaSuccess;
        for (int s = 0; ok && s < e->chains; s++)
            ok = cudaStreamCreateWithPriority(&e->sub[s], cudaStreamNonBlocking, cprio) == cudaSuccess &&
                 cudaEventCreateWithFlags(&e->ev_sjoin[s], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) {
            cudaGetLastError();
            e->chains = 1;
        }
    }
    const bool g = engine_rebin_gathers(e);
    const CoefLaunch cl{params->dt_diffusion, p.secretion, p.uptake, p.volume,
                        (e->dbl || e->fast) ? &c->xset[0] : nullptr, engine_fast_lod(e),
                        g ? p.pos : nullptr, g ? p.radius : nullptr};
    if ((st = launch_rebin(c, params->n_cells, p.pos, p.ids, p.voxel, p.bin_start, p.bin_cells,
                           p.bin_cells_by_id, p.nonempty, p.n_nonempty, false,
                           ex ? &cl : nullptr))) {
        delete e;
        return st;
    }
    if (params->n_cells > 0) {
        int nne = 0;
        CG_CUDA_CHECK(cudaMemcpyAsync(&nne, p.n_nonempty, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
        e->vel_dense = nne > 0 && (double)params->n_cells >= 2.0 * nne;
        e->vel_quad = e->fast && e->vel_dense;
        if (const char* env = std::getenv("CELLGPU_VEL_KERNEL")) {
            if (!std::strcmp(env, "quad")) e->vel_quad = true;
            if (!std::strcmp(env, "cell")) e->vel_quad = false;
        }
    }
    *out = e;
    return CG_OK;
}

static void engine_drop_graphs(cg_engine* e) {
    auto drop = [](cudaGraphExec_t& x, cudaGraph_t& g) {
        if (x) cudaGraphExecDestroy(x);
        if (g) cudaGraphDestroy(g);
        x = nullptr;
        g = nullptr;
    };
    for (int k = 0; k < kExchSets; k++) {
        drop(e->exec[k], e->graph[k]);
        drop(e->px_mech[k], e->pg_mech[k]);
        for (int s = 0; s < kLineMaxS; s++) drop(e->px_chain[s][k], e->pg_chain[s][k]);
    }
    e->pipe_ready = false;
}

static int engine_join(cg_engine* e, cudaStream_t stream);
static void hostio_free(cg_engine* e);

// Page-locked host buffers for the host-driven step: cudaHostAlloc memory
// moves at the copy engines' full rate (measured 225 us per 12.3 MB H2D vs
// 350 us from torch's pinned allocation, tools/pcie_probe.py).
extern "C" int cg_host_alloc(size_t bytes, void** out) {
    *out = nullptr;
    CG_CUDA_CHECK(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
    return CG_OK;
}

extern "C" void cg_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

extern "C" int cg_engine_io_enable(cg_engine* e) {
    if (e->io_in) return CG_OK;
    CG_CUDA_CHECK(cudaSetDevice(e->ctx->device));
    CG_CUDA_CHECK(cudaEventCreateWithFlags(&e->io_in, cudaEventDisableTiming));
    CG_CUDA_CHECK(cudaEventCreateWithFlags(&e->io_fields, cudaEventDisableTiming));
    CG_CUDA_CHECK(cudaEventCreateWithFlags(&e->io_dens, cudaEventDisableTiming));
    CG_CUDA_CHECK(cudaEventCreateWithFlags(&e->io_cells, cudaEventDisableTiming));
    for (int s = 0; s < e->ctx->S && s < kLineMaxS; s++) {
        CG_CUDA_CHECK(cudaEventCreateWithFlags(&e->io_sub_in[s], cudaEventDisableTiming));
        CG_CUDA_CHECK(cudaEventCreateWithFlags(&e->io_sub_out[s], cudaEventDisableTiming));
    }
    // the next graph launch recaptures with the two external event nodes
    engine_drop_graphs(e);
    return CG_OK;
}

extern "C" int cg_engine_io_inputs_ready(cg_engine* e, void* stream) {
    if (!e->io_in) return set_error(CG_STATE, "cg_engine_io_enable first");
    CG_CUDA_CHECK(cudaEventRecord(e->io_in, (cudaStream_t)stream));
    return CG_OK;
}

extern "C" int cg_engine_io_fields_ready(cg_engine* e, void* stream) {
    if (!e->io_dens) return set_error(CG_STATE, "cg_engine_io_enable first");
    CG_CUDA_CHECK(cudaEventRecord(e->io_dens, (cudaStream_t)stream));
    return CG_OK;
}

extern "C" int cg_engine_io_substrate_ready(cg_engine* e, int s, void* stream) {
    if (!e->io_dens) return set_error(CG_STATE, "cg_engine_io_enable first");
    if (s < 0 || s >= e->ctx->S || s >= kLineMaxS) return set_error(CG_DOMAIN, "substrate out of range");
    CG_CUDA_CHECK(cudaEventRecord(e->io_sub_in[s], (cudaStream_t)stream));
    return CG_OK;
}

extern "C" int cg_engine_io_wait_substrate(cg_engine* e, int s, void* stream) {
    if (!e->io_dens) return set_error(CG_STATE, "cg_engine_io_enable first");
    if (s < 0 || s >= e->ctx->S || s >= kLineMaxS) return set_error(CG_DOMAIN, "substrate out of range");
    CG_CUDA_CHECK(cudaStreamWaitEvent((cudaStream_t)stream, e->io_sub_out[s], 0));
    return CG_OK;
}

extern "C" int cg_engine_substrate_chains(cg_engine* e) { return e->chains; }

extern "C" int cg_engine_io_wait_cells(cg_engine* e, void* stream) {
    if (!e->io_cells) return set_error(CG_STATE, "cg_engine_io_enable first");
    CG_CUDA_CHECK(cudaStreamWaitEvent((cudaStream_t)stream, e->io_cells, 0));
    return CG_OK;
}

extern "C" int cg_engine_io_wait_fields(cg_engine* e, void* stream) {
    if (!e->io_fields) return set_error(CG_STATE, "cg_engine_io_enable first");
    CG_CUDA_CHECK(cudaStreamWaitEvent((cudaStream_t)stream, e->io_fields, 0));
    return CG_OK;
}

extern "C" void cg_engine_destroy(cg_engine* e) {
    if (!e) return;
    engine_drop_graphs(e);
    hostio_free(e);
    if (e->side) cudaStreamDestroy(e->side);
    if (e->ev_fork) cudaEventDestroy(e->ev_fork);
    if (e->ev_join) cudaEventDestroy(e->ev_join);
    if (e->io_in) cudaEventDestroy(e->io_in);
    if (e->io_fields) cudaEventDestroy(e->io_fields);
    if (e->io_dens) cudaEventDestroy(e->io_dens);
    if (e->io_cells) cudaEventDestroy(e->io_cells);
    for (int s = 0; s < kLineMaxS; s++) {
        if (e->io_sub_in[s]) cudaEventDestroy(e->io_sub_in[s]);
        if (e->io_sub_out[s]) cudaEventDestroy(e->io_sub_out[s]);
        if (e->sub[s]) cudaStreamDestroy(e->sub[s]);
        if (e->ev_sjoin[s]) cudaEventDestroy(e->ev_sjoin[s]);
    }
    if (e->ev_sfork) cudaEventDestroy(e->ev_sfork);
    cudaFree(e->sort_tmp);
    cudaFree(e->sort_order);
    if (e->ev_mech) cudaEventDestroy(e->ev_mech);
    for (int s = 0; s < kLineMaxS; s++)
        for (int k = 0; k < kExchSets; k++)
            if (e->ev_chain[s][k]) cudaEventDestroy(e->ev_chain[s][k]);
    delete e;
}

// Captures the step graphs (one per exchange set when they rotate).
static int engine_capture(cg_engine* e) {
    cg_ctx* c = e->ctx;
    if (c->stream == nullptr)
        return set_error(CG_STATE, "graph capture needs a non-default stream (cg_ctx_set_stream)");
    const bool was_prof = c->prof;
    c->prof = false;
    const int cur0 = e->cur;
    int st = CG_OK;
    for (int k = 0; k < (e->dbl ? kExchSets : 1) && !st; k++) {
        e->cur = k;
        const long long l0 = c->launches;
        CG_CUDA_CHECK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        st = engine_step(e);
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
        e->launches_per_step = (int)(c->launches - l0);
        c->launches = l0;
        if (!st && ce != cudaSuccess) st = set_cuda_error(ce, "cudaStreamEndCapture");
        if (st) {
            if (g) cudaGraphDestroy(g);
            break;
        }
        e->graph[k] = g;
        cudaError_t ie = cudaGraphInstantiate(&e->exec[k], g, 0);
        if (ie != cudaSuccess) st = set_cuda_error(ie, "cudaGraphInstantiate");
    }
    e->cur = cur0;
    c->prof = was_prof;
    if (st) engine_drop_graphs(e);
    return st;
}

extern "C" int cg_engine_run(cg_engine* e, int steps, int use_graph) {
    cg_ctx* c = e->ctx;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (e->pipe_ready) {
        // leaving pipelined I/O steps: the context stream catches up first
        if (int st = engine_join(e, c->stream)) return st;
    }
    if (use_graph && !e->exec[0]) {
        int st = engine_capture(e);
        if (st) return st;
    }
    for (int s = 0; s < steps; s++) {
        if (use_graph) {
            CG_CUDA_CHECK(cudaGraphLaunch(e->exec[e->dbl ? e->cur : 0], c->stream));
            c->launches += e->launches_per_step;
        } else {
            const long long l0 = c->launches;
            int st = engine_step(e);
            if (st) return st;
            e->launches_per_step = (int)(c->launches - l0);
        }
        if (e->dbl) e->cur = (e->cur + 1) % kExchSets;
    }
    return CG_OK;
}

// ---- pipelined host-driven steps

// Captures one component graph: fn() enqueues on `st`.
template <typename F>
static int capture_on(cg_engine* e, cudaStream_t st, F fn, cudaGraph_t* g, cudaGraphExec_t* x,
                      int* launches) {
    cg_ctx* c = e->ctx;
    cudaStream_t keep = c->stream;
    c->stream = st;
    const long long l0 = c->launches;
    CG_CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int rc = fn();
    cudaError_t ce = cudaStreamEndCapture(st, g);
    *launches += (int)(c->launches - l0);
    c->launches = l0;
    c->stream = keep;
    if (!rc && ce != cudaSuccess) rc = set_cuda_error(ce, "cudaStreamEndCapture");
    if (!rc) {
        cudaError_t ie = cudaGraphInstantiate(x, *g, 0);
        if (ie != cudaSuccess) rc = set_cuda_error(ie, "cudaGraphInstantiate");
    }
    return rc;
}

static int pipe_prepare(cg_engine* e) {
    cg_ctx* c = e->ctx;
    const bool was_prof = c->prof;
    c->prof = false;
    int rc = CG_OK, launches = 0;
    if (!e->ev_mech) CG_CUDA_CHECK(cudaEventCreateWithFlags(&e->ev_mech, cudaEventDisableTiming));
    for (int k = 0; k < kExchSets && !rc; k++) {
        const int wset = (k + 1) % kExchSets;
        launches = 0;
        rc = capture_on(e, e->side, [&] { return launch_mechanics(e, true, wset); },
                        &e->pg_mech[k], &e->px_mech[k], &launches);
        for (int s = 0; s < e->chains && !rc; s++) {
            if (!e->ev_chain[s][k])
                CG_CUDA_CHECK(cudaEventCreateWithFlags(&e->ev_chain[s][k], cudaEventDisableTiming));
            rc = capture_on(e, e->sub[s], [&] { return launch_substeps(e, s, 1, k); },
                            &e->pg_chain[s][k], &e->px_chain[s][k], &launches);
        }
    }
    c->prof = was_prof;
    if (rc) return rc;
    e->launches_per_step = launches;
    // the first pipelined step starts after everything on the context stream
    CG_CUDA_CHECK(cudaEventRecord(e->ev_fork, c->stream));
    CG_CUDA_CHECK(cudaStreamWaitEvent(e->side, e->ev_fork, 0));
    for (int s = 0; s < e->chains; s++) CG_CUDA_CHECK(cudaStreamWaitEvent(e->sub[s], e->ev_fork, 0));
    e->pipe_ready = true;
    return CG_OK;
}

// Makes `stream` wait for every pipelined component enqueued so far.
static int engine_join(cg_engine* e, cudaStream_t stream) {
    if (!e->pipe_ready) return CG_OK;
    CG_CUDA_CHECK(cudaEventRecord(e->ev_join, e->side));
    CG_CUDA_CHECK(cudaStreamWaitEvent(stream, e->ev_join, 0));
    for (int s = 0; s < e->chains; s++) {
        CG_CUDA_CHECK(cudaEventRecord(e->ev_sjoin[s], e->sub[s]));
        CG_CUDA_CHECK(cudaStreamWaitEvent(stream, e->ev_sjoin[s], 0));
    }
    return CG_OK;
}

extern "C" int cg_engine_io_join(cg_engine* e, void* stream) {
    CG_CUDA_CHECK(cudaSetDevice(e->ctx->device));
    return engine_join(e, stream ? (cudaStream_t)stream : e->ctx->stream);
}

static void hostio_free(cg_engine* e) {
    auto& h = e->hio;
    for (cudaStream_t* st : {&h.up_fields, &h.up_cells, &h.down_fields, &h.down_cells})
        if (*st) cudaStreamDestroy(*st), *st = nullptr;
    for (int s = 0; s < kLineMaxS; s++) {
        if (h.up_sub[s]) cudaStreamDestroy(h.up_sub[s]), h.up_sub[s] = nullptr;
        if (h.down_sub[s]) cudaStreamDestroy(h.down_sub[s]), h.down_sub[s] = nullptr;
    }
    for (cudaEvent_t ev : h.piece_out) cudaEventDestroy(ev);
    h.piece_out.clear();
    if (h.cells_out) cudaEventDestroy(h.cells_out), h.cells_out = nullptr;
    h.chunks = 0;
}

static int hostio_setup(cg_engine* e, int chunks) {
    auto& h = e->hio;
    if (h.chunks == chunks) return CG_OK;
    cg_ctx* c = e->ctx;
    // no copy of the old layout may be in flight when the pieces change
    if (h.chunks) CG_CUDA_CHECK(cudaDeviceSynchronize());
    hostio_free(e);
    for (cudaStream_t* st : {&h.up_fields, &h.up_cells, &h.down_fields, &h.down_cells})
        CG_CUDA_CHECK(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    const char* env_io = std::getenv("CELLGPU_IO_STREAMS");
    h.per_sub = e->chains > 1 && e->chains <= kLineMaxS && !(env_io && !std::strcmp(env_io, "shared"));
    if (h.per_sub)
        for (int s = 0; s < e->chains; s++) {
            CG_CUDA_CHECK(cudaStreamCreateWithFlags(&h.up_sub[s], cudaStreamNonBlocking));
            CG_CUDA_CHECK(cudaStreamCreateWithFlags(&h.down_sub[s], cudaStreamNonBlocking));
        }
    CG_CUDA_CHECK(cudaEventCreateWithFlags(&h.cells_out, cudaEventDisableTiming));
    const long nv = c->nvox, S = c->S;
    h.piece_sub.clear();
    h.piece_lo.clear();
    h.piece_hi.clear();
    if (e->chains > 1) {
        for (long s = 0; s < S; s++)
            for (long j = 0; j < chunks; j++) {
                h.piece_sub.push_back((int)s);
                h.piece_lo.push_back(s * nv + nv * j / chunks);
                h.piece_hi.push_back(s * nv + nv * (j + 1) / chunks);
            }
    } else {
        for (long j = 0; j < chunks; j++) {
            h.piece_sub.push_back(-1);
            h.piece_lo.push_back(S * nv * j / chunks);
            h.piece_hi.push_back(S * nv * (j + 1) / chunks);
        }
    }
    for (size_t i = 0; i < h.piece_sub.size(); i++) {
        cudaEvent_t ev;
        CG_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        h.piece_out.push_back(ev);
    }
    h.chunks = chunks;
    return CG_OK;
}

// One mechanics step from host state to host state (include/cellgpu.h).
// Cells: up_cells uploads positions / AB2 state once the previous step's
// cell state is out, the mechanics wait for it (io_in), and down_cells copies
// positions / velocities out as soon as integration is done (io_cells).
// Fields: piece i goes up on up_fields once its previous download is done;
// with substrate chains a substrate's substeps start when its last piece is
// up and its pieces go down as soon as its substeps end.
extern "C" int cg_engine_step_host(cg_engine* e, const double* h_dens, const double* h_pos,
                                   const double* h_prev, double* o_dens, double* o_pos,
                                   double* o_vel, int chunks) {
    cg_ctx* c = e->ctx;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (chunks < 1) return set_error(CG_DOMAIN, "chunks must be >= 1");
    int st;
    if ((st = cg_engine_io_enable(e)) || (st = hostio_setup(e, chunks))) return st;
    auto& h = e->hio;
    const cg_state_ptrs& p = e->p;
    const size_t cell_bytes = (size_t)e->q.n_cells * 3 * sizeof(double);
    const bool chains = e->chains > 1;
    // cells up
    CG_CUDA_CHECK(cudaStreamWaitEvent(h.up_cells, h.cells_out, 0));
    if (cell_bytes) {
        CG_CUDA_CHECK(cudaMemcpyAsync(p.pos, h_pos, cell_bytes, cudaMemcpyHostToDevice, h.up_cells));
        if (p.prev_vel)
            CG_CUDA_CHECK(cudaMemcpyAsync(p.prev_vel, h_prev, cell_bytes, cudaMemcpyHostToDevice,
                                          h.up_cells));
    }
    CG_CUDA_CHECK(cudaEventRecord(e->io_in, h.up_cells));
    // fields up
    const int np = (int)h.piece_sub.size();
    for (int i = 0; i < np; i++) {
        cudaStream_t up = h.per_sub ? h.up_sub[h.piece_sub[i]] : h.up_fields;
        CG_CUDA_CHECK(cudaStreamWaitEvent(up, h.piece_out[i], 0));
        const long lo = h.piece_lo[i], n = h.piece_hi[i] - lo;
        CG_CUDA_CHECK(cudaMemcpyAsync(p.dens + lo, h_dens + lo, n * sizeof(double),
                                      cudaMemcpyHostToDevice, up));
        if (chains && (i + 1 == np || h.piece_sub[i + 1] != h.piece_sub[i]))
            CG_CUDA_CHECK(cudaEventRecord(e->io_sub_in[h.piece_sub[i]], up));
    }
    if (!chains) CG_CUDA_CHECK(cudaEventRecord(e->io_dens, h.up_fields));
    // the step
    if ((st = chains ? cg_engine_step_io(e) : cg_engine_run(e, 1, 1))) return st;
    // cells down
    CG_CUDA_CHECK(cudaStreamWaitEvent(h.down_cells, e->io_cells, 0));
    if (cell_bytes) {
        CG_CUDA_CHECK(cudaMemcpyAsync(o_pos, p.pos, cell_bytes, cudaMemcpyDeviceToHost, h.down_cells));
        CG_CUDA_CHECK(cudaMemcpyAsync(o_vel, p.vel, cell_bytes, cudaMemcpyDeviceToHost, h.down_cells));
    }
    CG_CUDA_CHECK(cudaEventRecord(h.cells_out, h.down_cells));
    // fields down
    if (!chains) CG_CUDA_CHECK(cudaStreamWaitEvent(h.down_fields, e->io_fields, 0));
    for (int i = 0; i < np; i++) {
        cudaStream_t down = h.per_sub ? h.down_sub[h.piece_sub[i]] : h.down_fields;
        if (chains && (i == 0 || h.piece_sub[i - 1] != h.piece_sub[i]))
            CG_CUDA_CHECK(cudaStreamWaitEvent(down, e->io_sub_out[h.piece_sub[i]], 0));
        const long lo = h.piece_lo[i], n = h.piece_hi[i] - lo;
        CG_CUDA_CHECK(cudaMemcpyAsync(o_dens + lo, p.dens + lo, n * sizeof(double),
                                      cudaMemcpyDeviceToHost, down));
        CG_CUDA_CHECK(cudaEventRecord(h.piece_out[i], down));
    }
    return CG_OK;
}

// Makes `stream` (NULL: the context stream) wait for the copies of every
// cg_engine_step_host so far (and, through them, the steps).
extern "C" int cg_engine_host_join(cg_engine* e, void* stream) {
    cg_ctx* c = e->ctx;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    cudaStream_t to = stream ? (cudaStream_t)stream : c->stream;
    auto& h = e->hio;
    if (h.chunks) {
        CG_CUDA_CHECK(cudaStreamWaitEvent(to, h.cells_out, 0));
        for (cudaEvent_t ev : h.piece_out) CG_CUDA_CHECK(cudaStreamWaitEvent(to, ev, 0));
    }
    return engine_join(e, to);
}

// One host-driven step, pipelined: step t's chain for substrate s waits for
// its own field upload (io substrate event) and for the rebin of step t - 1
// (the exchange set it reads); the mechanics of step t wait for the cell
// upload and for the chains of step t - 2 (which read the exchange set it
// overwrites).  Falls back to one graph launch per step without substrate
// chains.
extern "C" int cg_engine_step_io(cg_engine* e) {
    cg_ctx* c = e->ctx;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (!e->io_in) return set_error(CG_STATE, "cg_engine_io_enable first");
    if (e->chains < 2 || !e->dbl || e->q.gradients || !e->side) return cg_engine_run(e, 1, 1);
    if (!e->pipe_ready) {
        if (int rc = pipe_prepare(e)) return rc;
    }
    const int k = e->cur, kold = (e->cur + 1) % kExchSets;  // kold: step t - 2's set
    for (int s = 0; s < e->chains; s++) {
        cudaStream_t ss = e->sub[s];
        CG_CUDA_CHECK(cudaStreamWaitEvent(ss, e->ev_mech, 0));  // rebin of step t - 1
        CG_CUDA_CHECK(cudaStreamWaitEvent(ss, e->io_sub_in[s], 0));
        CG_CUDA_CHECK(cudaGraphLaunch(e->px_chain[s][k], ss));
        CG_CUDA_CHECK(cudaEventRecord(e->ev_chain[s][k], ss));
        CG_CUDA_CHECK(cudaEventRecord(e->io_sub_out[s], ss));
    }
    for (int s = 0; s < e->chains; s++)  // chains of step t - 2 (recorded under kold)
        CG_CUDA_CHECK(cudaStreamWaitEvent(e->side, e->ev_chain[s][kold], 0));
    CG_CUDA_CHECK(cudaStreamWaitEvent(e->side, e->io_in, 0));
    CG_CUDA_CHECK(cudaGraphLaunch(e->px_mech[k], e->side));
    CG_CUDA_CHECK(cudaEventRecord(e->ev_mech, e->side));  // (io_cells: recorded inside the graph)
    c->launches += e->launches_per_step;
    e->cur = (e->cur + 1) % kExchSets;
    return CG_OK;
}

extern "C" int cg_engine_launches_per_step(cg_engine* e) { return e->launches_per_step; }

// dst[k * w + j] = src[order[k] * w + j]
__global__ void k_permute_rows(int n, int w, const int32_t* __restrict__ order,
                               const double* __restrict__ src, double* __restrict__ dst) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long)n * w) return;
    const long k = t / w, j = t - k * w;
    dst[t] = src[(long)order[k] * w + j];
}

// sort_cells_by_voxel (population.py:132-135) on the engine's cells: storage
// becomes (voxel, id) order -- exactly the id-sorted bins read in voxel
// order, so the permutation is bin_cells_by_id -- then the rebin (bins,
// exchange coefficients of the set the next step reads) is redone.  Every
// per-cell array moves with its cell (ids included), so results per id are
// unchanged; run_simulation does this before the loop and every `every`
// steps with voxel-sorted storage (simulate.py:156-158, 209-212).  It is the
// memory-locality optimisation of the paper: the rebin's per-cell gathers,
// the scatter and the velocity writes become near-sequential.
static int engine_rebin_current(cg_engine* e);

extern "C" int cg_engine_set_cell_count(cg_engine* e, int n_cells) {
    cg_ctx* c = e->ctx;
    int st = check_cells(c, n_cells);
    if (st) return st;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if ((st = engine_join(e, c->stream))) return st;
    // no graph of the old count may still be running when it is destroyed
    CG_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    engine_drop_graphs(e);
    e->q.n_cells = n_cells;
    cudaFree(e->sort_tmp);
    cudaFree(e->sort_order);
    e->sort_tmp = nullptr;
    e->sort_order = nullptr;
    return engine_rebin_current(e);
}

extern "C" int cg_engine_sort_cells(cg_engine* e) {
    cg_ctx* c = e->ctx;
    const cg_state_ptrs& p = e->p;
    const cg_step_params& q = e->q;
    const int n = q.n_cells;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (n <= 1) return CG_OK;
    if (int st = engine_join(e, c->stream)) return st;
    if (!e->sort_tmp) CG_CUDA_CHECK(cudaMalloc((void**)&e->sort_tmp, (size_t)n * 3 * sizeof(double)));
    if (!e->sort_order) CG_CUDA_CHECK(cudaMalloc((void**)&e->sort_order, (size_t)n * sizeof(int32_t)));
    CG_CUDA_CHECK(cudaMemcpyAsync(e->sort_order, p.bin_cells_by_id, (size_t)n * sizeof(int32_t),
                                  cudaMemcpyDeviceToDevice, c->stream));
    auto permute = [&](double* a, int w) -> int {
        if (!a) return CG_OK;
        const long tot = (long)n * w;
        k_permute_rows<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(n, w, e->sort_order, a,
                                                                           e->sort_tmp);
        CG_CUDA_CHECK(cudaGetLastError());
        c->launches++;
        CG_CUDA_CHECK(cudaMemcpyAsync(a, e->sort_tmp, (size_t)tot * sizeof(double),
                                      cudaMemcpyDeviceToDevice, c->stream));
        return CG_OK;
    };
    int st;
    if ((st = permute(p.pos, 3)) || (st = permute(p.vel, 3)) || (st = permute(p.prev_vel, 3)) ||
        (st = permute(const_cast<double*>(p.radius), 1)) ||
        (st = permute(const_cast<double*>(p.volume), 1)) ||
        (st = permute(reinterpret_cast<double*>(const_cast<int64_t*>(p.ids)), 1)) ||
        (st = permute(p.division_rate, 1)))
        return st;
    for (int s = 0; s < c->S; s++) {
        if (p.secretion && (st = permute(const_cast<double*>(p.secretion) + (size_t)s * n, 1))) return st;
        if (p.uptake && (st = permute(const_cast<double*>(p.uptake) + (size_t)s * n, 1))) return st;
    }
    return engine_rebin_current(e);
}

// Bins and the exchange set the next step reads, for the current cells (on
// the context stream, after everything enqueued so far).
static int engine_rebin_current(cg_engine* e) {
    cg_ctx* c = e->ctx;
    const cg_state_ptrs& p = e->p;
    const cg_step_params& q = e->q;
    const int n = q.n_cells;
    const bool ex = p.secretion && p.uptake && n > 0;
    const int rset = e->dbl ? e->cur : 0;
    const bool g = engine_rebin_gathers(e);
    const CoefLaunch cl{q.dt_diffusion, p.secretion, p.uptake, p.volume,
                        (e->dbl || e->fast) ? &c->xset[rset] : nullptr, engine_fast_lod(e),
                        g ? p.pos : nullptr, g ? p.radius : nullptr};
    int st;
    if ((st = launch_rebin(c, n, p.pos, p.ids, p.voxel, p.bin_start, p.bin_cells,
                           p.bin_cells_by_id, p.nonempty, p.n_nonempty, false, ex ? &cl : nullptr)))
        return st;
    if (e->pipe_ready) {  // pipelined host-driven steps continue after it
        CG_CUDA_CHECK(cudaEventRecord(e->ev_fork, c->stream));
        CG_CUDA_CHECK(cudaStreamWaitEvent(e->side, e->ev_fork, 0));
        for (int s = 0; s < e->chains; s++) CG_CUDA_CHECK(cudaStreamWaitEvent(e->sub[s], e->ev_fork, 0));
    }
    return CG_OK;
}

// Per-stage device time without launch/event overhead: each stage of the
// mechanics step is enqueued `reps` times back to back between two events on
// the context stream.  Used by bench.py for the roofline; it perturbs the
// simulation state (integrate runs `reps` times), so call it last.
extern "C" int cg_engine_time_stages(cg_engine* e, int reps, int max_stages, char* names,
                                     double* ms_per_rep) {
    cg_ctx* c = e->ctx;
    const cg_state_ptrs& p = e->p;
    const cg_step_params& q = e->q;
    const bool ex = p.secretion && p.uptake && q.n_cells > 0;
    CG_CUDA_CHECK(cudaSetDevice(c->device));
    if (int st = engine_join(e, c->stream)) return st;  // after pipelined steps
    struct Stage {
        const char* name;
        int which;
    };
    const Stage stages[] = {{"exchange", 6},  {"lod_xy", 0},    {"lod_z", 1},
                            {"velocity", 2}, {"integrate", 3}, {"rebin", 4},
                            {"exchange_coef", 5}};
    const bool fl = engine_fast_lod(e);
    const bool split = ex && lod_exchange_split(c) && !fl;
    const ExchSet& xs = c->xset[e->dbl ? e->cur : 0];
    const int ns = (int)(sizeof(stages) / sizeof(stages[0]));
    cudaEvent_t a, b;
    CG_CUDA_CHECK(cudaEventCreate(&a));
    CG_CUDA_CHECK(cudaEventCreate(&b));
    const bool was_prof = c->prof;
    c->prof = false;
    int k = 0;
    for (int i = 0; i < ns && k < max_stages; i++) {
        if (stages[i].which == 5 && !ex) continue;
        if (stages[i].which == 6 && !split) continue;
        auto run = [&]() -> int {
            switch (stages[i].which) {
                case 6: return launch_exchange_rec(c, p.dens, q.n_cells, p.nonempty, p.n_nonempty,
                                                   e->dbl ? &c->xset[e->cur] : nullptr);
                case 0:
                    if (fl)
                        return launch_lod_fast(c, p.dens, q.bc, ex ? xs.vox : nullptr, xs.n,
                                               ex ? xs.aff : nullptr, xs.pz, 1, false, true);
                    return launch_lod(c, p.dens, q.bc, p.nonempty,
                                      ex && !split ? c->d_exA : nullptr,
                                      ex && !split ? c->d_exD : nullptr, q.n_cells, 1);
                case 1:
                    if (fl) return launch_lod_fast(c, p.dens, q.bc, nullptr, nullptr, nullptr, nullptr, 2);
                    return launch_lod(c, p.dens, q.bc, p.nonempty, nullptr, nullptr, q.n_cells, 2);
                case 2:
                    if (e->fast)
                        return launch_velocities_fast(c, q.n_cells, p.pos, p.radius, p.voxel,
                                                      p.bin_start, p.bin_cells_by_id,
                                                      engine_rebin_gathers(e), e->vel_quad,
                                                      q.repulsion, q.adhesion,
                                                      q.adhesion_multiplier, p.vel);
                    return launch_velocities(c, q.n_cells, p.pos, p.radius, p.ids, p.voxel, p.bin_start,
                                             p.bin_cells_by_id, p.nonempty, p.n_nonempty,
                                             q.repulsion, q.adhesion, q.adhesion_multiplier, p.vel,
                                             e->vel_dense);
                case 3: return launch_integrate(c, q.n_cells, p.pos, p.vel, p.prev_vel,
                                                q.dt_mechanics, q.integrator);
                case 4: return launch_rebin(c, q.n_cells, p.pos, p.ids, p.voxel, p.bin_start,
                                            p.bin_cells, p.bin_cells_by_id, p.nonempty, p.n_nonempty);
                default: return launch_exchange_coef(c, q.dt_diffusion, p.secretion, p.uptake,
                                                     q.n_cells, p.volume, p.bin_cells_by_id);
            }
        };
        int st = run();  // warm
        if (st) { c->prof = was_prof; return st; }
        // `reps` launches captured in one graph: in-graph launch gaps, as in
        // the step graph, instead of the host submission rate.
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        CG_CUDA_CHECK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        for (int r = 0; r < reps && !st; r++) st = run();
        cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
        if (st || ce != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            c->prof = was_prof;
            return st ? st : set_cuda_error(ce, "stage capture");
        }
        CG_CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
        CG_CUDA_CHECK(cudaGraphLaunch(ge, c->stream));
        CG_CUDA_CHECK(cudaEventRecord(a, c->stream));
        CG_CUDA_CHECK(cudaGraphLaunch(ge, c->stream));
        CG_CUDA_CHECK(cudaEventRecord(b, c->stream));
        CG_CUDA_CHECK(cudaEventSynchronize(b));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        float ms = 0.f;
        CG_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
        std::snprintf(names + 32 * k, 32, "%s", stages[i].name);
        ms_per_rep[k] = ms / reps;
        k++;
    }
    c->prof = was_prof;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return k;
}
