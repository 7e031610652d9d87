/*
 * cellgpu.h -- C-ABI of libcellgpu.so, the B200 (sm_100a) implementation of
 * the cellbench per-step hot path.
 *
 * The reference (/root/reference/pkg/src/cellbench, pure Python + numpy) has
 * no FFI; its "plugin interface" is five Python functions.  Each entry point
 * below replaces one of them and is what a ctypes binding of that function
 * would call (see INTEGRATION.md for the stub):
 *
 *   cg_lod_step        <- diffusion.py:127-192  lod_step
 *   cg_gradients       <- diffusion.py:237-278  compute_gradients
 *   cg_exchange        <- diffusion.py:201-234  apply_cell_exchange
 *   cg_rebin           <- core.py:218-240       rebin_cells
 *   cg_velocities      <- mechanics.py:175-225  update_velocities
 *   cg_integrate       <- mechanics.py:228-245  integrate_positions
 *   cg_engine_*        <- simulate.py:166-202   the run_simulation step loop
 *                         (exchange, lod, velocities, integrate, rebin),
 *                         replayed as one CUDA graph per mechanics step.
 *
 * Conventions
 *  - Every array argument is a DEVICE pointer owned by the caller (the Python
 *    layer allocates them as torch tensors).  Scalars and the small per-
 *    substrate parameter arrays (diffusion, decay, dirichlet, saturation) are
 *    HOST pointers.  No torch types cross this boundary.
 *  - Layouts: densities (S, nz, ny, nx) float64, x fastest (core.py:69-70);
 *    positions/velocities (n, 3) float64 in container storage order; ids
 *    int64; voxel/bin arrays int32.
 *  - Work is enqueued on the context's stream (cg_ctx_set_stream) and is
 *    asynchronous.  Device-side domain checks (position outside the mesh,
 *    exchange denominator <= 0, candidate capacity) raise a flag word that
 *    cg_sync() reads; no entry point synchronises on its own.
 *  - Return codes mirror errors.py:4-37: 0 ok, 1 DomainError, 2 NumericError,
 *    3 ContainerStateError, 4 CapacityError, >=100 CUDA error (message via
 *    cg_last_error()).
 */
#ifndef CELLGPU_H
#define CELLGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CG_OK 0
#define CG_DOMAIN 1
#define CG_NUMERIC 2
#define CG_STATE 3
#define CG_CAPACITY 4
#define CG_CUDA 100

#define CG_BC_NEUMANN 0   /* the reference: no-flux boundaries only        */
#define CG_BC_DIRICHLET 1 /* G1 extension: outer-face voxels pinned         */
#define CG_EULER 0        /* the reference: x += dt*v                       */
#define CG_AB2 1          /* G2 extension: Adams-Bashforth 2 (PhysiCell)    */
/* Engine numerics.  EXACT: every operation in the reference's order, results
 * bit-identical to diffusion.py / mechanics.py.  FAST: BASELINE.json's
 * tolerances instead of bit-exactness -- segmented line solves (K segments
 * per line, carries across segments), each voxel's exchange as one affine
 * map per substrate, velocities summed per cell over its 9 neighbour rows;
 * fields within 1e-10 and velocities / positions within 1e-12 (normwise)
 * of the reference per step, bins and non-empty lists identical. */
#define CG_NUMERICS_EXACT 0
#define CG_NUMERICS_FAST 1

typedef struct cg_ctx cg_ctx;
typedef struct cg_engine cg_engine;

/* Library / context lifecycle ------------------------------------------- */
const char* cg_version(void);
const char* cg_last_error(void);
/* Mesh of core.py:35-102 CartesianMesh (origin = lower corner) with S
 * substrates; cell_capacity sizes the per-cell scratch. */
int cg_ctx_create(int device, int nx, int ny, int nz, double dx, double dy, double dz,
                  double ox, double oy, double oz, int n_substrates, int cell_capacity,
                  cg_ctx** out);
void cg_ctx_destroy(cg_ctx* ctx);
int cg_ctx_set_stream(cg_ctx* ctx, void* cuda_stream);
/* Wait for the stream, then return (and clear) the first raised error. */
int cg_sync(cg_ctx* ctx);

/* Diffusion -------------------------------------------------------------- */
/* diffusion.py:127-192 lod_step: x, y, z implicit sweeps per substrate with
 * decay split lambda/3, constant-coefficient Thomas factors (diffusion.py:80-
 * 99) computed on the host and cached per (dt, D, decay).  dens: (S, nvox).
 * diffusion/decay: S host doubles.  bc/dirichlet: G1 extension. */
int cg_lod_step(cg_ctx* ctx, double* dens, const double* diffusion, const double* decay,
                double dt, int bc, const double* dirichlet);

/* diffusion.py:201-234 apply_cell_exchange with the reference's scalar rates,
 * applied to substrate `substrate` over the non-empty voxels of the bins
 * produced by cg_rebin; cells of a voxel in ascending id order. */
int cg_exchange(cg_ctx* ctx, double* dens, int substrate, double dt, double secretion,
                double uptake, double saturation, int n_cells, const double* volume,
                const int32_t* bin_start, const int32_t* bin_cells_by_id,
                const int32_t* nonempty, const int32_t* n_nonempty);

/* G4 extension: per-cell rates for every substrate.  secretion/uptake: (S, n)
 * device arrays indexed by storage index; saturation: S host doubles. */
int cg_exchange_cells(cg_ctx* ctx, double* dens, double dt, const double* secretion,
                      const double* uptake, const double* saturation, int n_cells,
                      const double* volume, const int32_t* bin_start,
                      const int32_t* bin_cells_by_id, const int32_t* nonempty,
                      const int32_t* n_nonempty);

/* simulate.py:79-90 state_checksum on the device: XOR over cells of the
 * BLAKE2b-128 digest of struct.pack("<q6d", id, x, y, z, vx, vy, vz).
 * ids/pos/vel: device arrays (n), (n, 3), (n, 3); digest: 2 host words, the
 * 128-bit value little-endian (the reference's hex string is
 * f"{digest[1] << 64 | digest[0]:032x}").  Synchronises the stream. */
int cg_state_checksum(cg_ctx* ctx, int n_cells, const int64_t* ids, const double* pos,
                      const double* vel, uint64_t* digest);

/* Divisions (population.py:44-129).  cg_division_draws: the three uniforms
 * of division_draws(seed, ids[i], step) per cell -> out (n, 3).
 * cg_divisions_count: how many cells divide this step (u0 < thr[i], thr =
 * 1 - exp(-rate*dt) computed by the caller, <= 0 for no division); a
 * synchronising call, so the caller can raise CapacityError before anything
 * is appended.  cg_divisions_place: for those `count` cells, in ascending
 * parent id, the parent's storage index and the daughter's clamped position
 * (R/2 along the drawn direction) -> parent_out (count), pos_out (count, 3);
 * the direction's cos / sin are evaluated with the host's libm (as CPython's
 * math.cos / math.sin), so positions are bit-identical to the reference's;
 * synchronising. */
int cg_division_draws(cg_ctx* ctx, int n, uint64_t seed, int64_t step, const int64_t* ids,
                      double* out);
int cg_divisions_count(cg_ctx* ctx, int n, uint64_t seed, int64_t step, const int64_t* ids,
                       const double* thr, int* count);
int cg_divisions_place(cg_ctx* ctx, int n, int count, uint64_t seed, int64_t step,
                       const int64_t* ids, const double* pos, const double* radius,
                       int32_t* parent_out, double* pos_out);

/* Microenvironment.check_state (core.py:142-144) on the device: every value
 * of the (S, nvox) field finite and non-negative, else the next cg_sync
 * returns CG_NUMERIC.  The step engine runs the same test on the final field
 * of every mechanics step (simulate.py:218), fused into the last z sweep. */
int cg_check_state(cg_ctx* ctx, const double* dens);

/* diffusion.py:237-278 compute_gradients: central differences (d[+1] -
 * d[-1]) * (0.5 / spacing) per axis, zero on that axis's two faces (and on
 * axes of <= 2 voxels).  dens: (S, nvox); grad: (S, nvox, 3) device arrays.
 * Not available on z-slab contexts (needs a one-plane halo). */
int cg_gradients(cg_ctx* ctx, const double* dens, double* grad);

/* Cell container ------------------------------------------------------------ */
/* core.py:218-240 rebin_cells as a counting sort.  Outputs:
 *   voxel[n]            flat voxel of each cell (CPython-exact voxel_of)
 *   bin_start[nvox+1]   CSR offsets
 *   bin_cells[n]        storage indices, storage order within a voxel
 *                       (= the reference's agent lists)
 *   bin_cells_by_id[n]  the same bins, ascending id within a voxel
 *   nonempty[nvox]      ascending non-empty voxels (= nonempty_voxels)
 *   n_nonempty[1]       device count
 * A position outside the mesh raises CG_DOMAIN (core.py:83-84). */
int cg_rebin(cg_ctx* ctx, int n_cells, const double* pos, const int64_t* ids,
             int32_t* voxel, int32_t* bin_start, int32_t* bin_cells,
             int32_t* bin_cells_by_id, int32_t* nonempty, int32_t* n_nonempty);

/* cg_rebin followed by the G4 exchange coefficients of the new bins (the
 * exchange of diffusion.py:224-228 split into its cell-constant part):
 * A = (f*sec)*sat, D = 1 + f*(sec+upt) per id-sorted slot and substrate,
 * kept in the context for cg_exchange_prepared until the next rebin.
 * secretion/uptake: (S, n) device arrays by storage index; volume: (n);
 * saturation: S host doubles.  Cells do not move between mechanics steps,
 * so the substeps of one step reuse them (the reference recomputes the same
 * values every substep). */
int cg_rebin_exchange(cg_ctx* ctx, int n_cells, const double* pos, const int64_t* ids,
                      int32_t* voxel, int32_t* bin_start, int32_t* bin_cells,
                      int32_t* bin_cells_by_id, int32_t* nonempty, int32_t* n_nonempty,
                      double dt, const double* secretion, const double* uptake,
                      const double* saturation, const double* volume);
/* The exchange with the coefficients of the last cg_rebin_exchange on this
 * context: every substrate, cells of a voxel in ascending id order
 * (diffusion.py:219-229). */
int cg_exchange_prepared(cg_ctx* ctx, double* dens, int n_cells, const int32_t* nonempty,
                         const int32_t* n_nonempty);

/* Mechanics ----------------------------------------------------------------- */
/* mechanics.py:175-225 update_velocities: each cell's velocity is reset and
 * accumulated over the 3x3x3-voxel candidates (mechanics.py:118-133) in
 * ascending id order with the force law of mechanics.py:145-172. */
int cg_velocities(cg_ctx* ctx, int n_cells, const double* pos, const double* radius,
                  const int64_t* ids, const int32_t* bin_start,
                  const int32_t* bin_cells_by_id, const int32_t* nonempty,
                  const int32_t* n_nonempty, double repulsion, double adhesion,
                  double adhesion_multiplier, double* vel);

/* mechanics.py:228-245 integrate_positions (+ G2 AB2 with prev_vel). */
int cg_integrate(cg_ctx* ctx, int n_cells, double* pos, const double* vel,
                 double* prev_vel, double dt, int integrator);

/* Step engine --------------------------------------------------------------- */
/* simulate.py:166-202: one mechanics step = `substeps` x [G4 exchange on all
 * substrates -> lod_step], then velocities, integrate, rebin.  All arrays are
 * the caller's device buffers (kept alive by the caller).  The first
 * cg_engine_run captures one step as a CUDA graph; later runs replay it. */
typedef struct {
    double* dens;               /* (S, nvox)                                 */
    double* pos;                /* (n, 3)                                    */
    double* vel;                /* (n, 3)                                    */
    double* prev_vel;           /* (n, 3) (AB2) or NULL                      */
    const double* radius;       /* (n)                                       */
    const double* volume;       /* (n) (4/3) pi R**3, host-computed          */
    const int64_t* ids;         /* (n)                                       */
    const double* secretion;    /* (S, n) or NULL                            */
    const double* uptake;       /* (S, n) or NULL                            */
    int32_t* voxel;             /* (n)                                       */
    int32_t* bin_start;         /* (nvox + 1)                                */
    int32_t* bin_cells;         /* (n)                                       */
    int32_t* bin_cells_by_id;   /* (n)                                       */
    int32_t* nonempty;          /* (nvox)                                    */
    int32_t* n_nonempty;        /* (1)                                       */
    double* grad;               /* (S, nvox, 3) or NULL: gradients per step  */
    double* division_rate;      /* (n) or NULL: moves with its cell in sorts */
} cg_state_ptrs;

typedef struct {
    int n_cells;
    int substeps;
    double dt_diffusion;
    double dt_mechanics;
    int bc;
    int integrator;
    double repulsion;
    double adhesion;
    double adhesion_multiplier;
    const double* diffusion;   /* S host doubles */
    const double* decay;       /* S host doubles */
    const double* dirichlet;   /* S host doubles or NULL */
    const double* saturation;  /* S host doubles */
    int gradients;             /* 1: compute_gradients after the substeps   */
    int numerics;              /* CG_NUMERICS_EXACT (0) or CG_NUMERICS_FAST */
} cg_step_params;

int cg_engine_create(cg_ctx* ctx, const cg_state_ptrs* ptrs, const cg_step_params* params,
                     cg_engine** out);
void cg_engine_destroy(cg_engine* eng);
/* Enqueue `steps` mechanics steps (graph replays when use_graph != 0). */
int cg_engine_run(cg_engine* eng, int steps, int use_graph);
/* Host-driven steps (state round-tripping through host memory every step):
 * after cg_engine_io_enable, each step's velocity branch waits for the event
 * the caller records with cg_engine_io_inputs_ready on the stream that
 * uploads positions / AB2 state, and its substeps for the event recorded with
 * cg_engine_io_fields_ready on the stream that uploads the densities (a
 * never-recorded event does not block).  cg_engine_io_wait_cells makes a copy
 * stream wait until positions / velocities are final (integration and rebin
 * done), cg_engine_io_wait_fields until the substeps are done (densities
 * final).  So the mechanics run while the densities come in, and the cell
 * state goes out and comes back while the substeps run.  The caller records
 * inputs_ready (and fields_ready, if used) before every step. */
int cg_engine_io_enable(cg_engine* eng);
/* Page-locked host memory for those copies (cudaHostAlloc, portable). */
int cg_host_alloc(size_t bytes, void** out);
void cg_host_free(void* p);
int cg_engine_io_inputs_ready(cg_engine* eng, void* cuda_stream);
int cg_engine_io_fields_ready(cg_engine* eng, void* cuda_stream);
int cg_engine_io_wait_cells(cg_engine* eng, void* cuda_stream);
int cg_engine_io_wait_fields(cg_engine* eng, void* cuda_stream);
/* Per substrate s: the substeps of s wait for the event recorded with
 * cg_engine_io_substrate_ready (its field upload), and
 * cg_engine_io_wait_substrate makes a copy stream wait until the field of s
 * is final.  With substrate chains (cg_engine_substrate_chains > 1, the
 * substeps of every substrate on their own stream) the fields then move
 * substrate by substrate under the other substrates' substeps. */
int cg_engine_io_substrate_ready(cg_engine* eng, int substrate, void* cuda_stream);
int cg_engine_io_wait_substrate(cg_engine* eng, int substrate, void* cuda_stream);
int cg_engine_substrate_chains(cg_engine* eng);
/* One host-driven step, pipelined across steps (substrate chains only; else
 * the same as cg_engine_run(eng, 1, 1)): the mechanics branch and every
 * substrate chain are separate graphs on their own streams ordered only by
 * events, so substrate s of step t + 1 starts as soon as its field is back
 * and step t's rebin is done.  The caller records the io events as above
 * before the call.  cg_engine_io_join makes `cuda_stream` (NULL: the context
 * stream) wait for everything enqueued so far. */
int cg_engine_step_io(cg_engine* eng);
/* One mechanics step from host state to host state, copies included:
 * consumes h_dens (S, nvox), h_pos / h_prev (n, 3) and leaves the result in
 * o_dens, o_pos, o_vel (host pointers; page-locked memory lets the copies
 * overlap the step: cg_host_alloc).  Asynchronous; the o_ buffers of one call
 * may be the h_ buffers of the next (the library orders the copies).  The
 * fields move in `chunks` pieces (per substrate with substrate chains).  This
 * is the call a host-memory caller (cgo / JNI / ctypes) makes per step;
 * cg_engine_host_join makes `cuda_stream` (NULL: the context stream) wait
 * for every step and copy enqueued so far. */
int cg_engine_step_host(cg_engine* eng, const double* h_dens, const double* h_pos,
                        const double* h_prev, double* o_dens, double* o_pos, double* o_vel,
                        int chunks);
int cg_engine_host_join(cg_engine* eng, void* cuda_stream);
int cg_engine_io_join(cg_engine* eng, void* cuda_stream);
/* population.py:132-135 sort_cells_by_voxel on the engine's cells: storage
 * order becomes (voxel, id), every per-cell array (pos, vel, prev_vel,
 * radius, volume, ids, secretion, uptake) moves with its cell, and the bins /
 * exchange coefficients are rebuilt.  The reference does this before its
 * loop and every `every` steps with voxel-sorted storage
 * (simulate.py:156-158, 209-212).  Asynchronous on the context stream. */
int cg_engine_sort_cells(cg_engine* eng);
/* The engine's cell count changed (population.py:77-129 appended daughters
 * at the end of every per-cell array, within the context's capacity): the
 * next run recaptures its graphs with the new count, and the bins and the
 * exchange coefficients of the set the next step reads are rebuilt now
 * (attempt_divisions ends with a rebin, population.py:128). */
int cg_engine_set_cell_count(cg_engine* eng, int n_cells);
/* Kernels launched by one mechanics step (the graph's kernel nodes). */
int cg_engine_launches_per_step(cg_engine* eng);
/* Device time per stage (lod_xy, lod_z, velocity, integrate, rebin,
 * exchange_coef), each enqueued `reps` times back to back between two events;
 * returns the number of stages written (names: 32 chars each).  Perturbs the
 * state (integration runs `reps` times): a benchmarking aid, call it last. */
int cg_engine_time_stages(cg_engine* eng, int reps, int max_stages, char* names,
                          double* ms_per_rep);

/* z-slab decomposition -------------------------------------- */
/* Declare this context's mesh to be rank `rank`'s slab of a balanced z split
 * of nz_global planes over `world` ranks (its planes [z0, z0 + nz)).  After
 * this, cg_lod_step runs the x/y sweeps and the LOCAL block solve of the z
 * sweep (block Thomas factors: the boundary diagonal only at global ends);
 * the caller then packs each line's end values (cg_zslab_pack: send is
 * (S, 2, nx*ny) doubles), all-gathers them over the ranks into recv
 * (world, S, 2, nx*ny), and calls cg_zslab_correct, which solves the 2x2
 * block-tridiagonal interface system per line and applies
 * x = y + l_{k-1} v + f_{k+1} w plus the z-line Dirichlet pins. */
int cg_ctx_set_slab(cg_ctx* ctx, int rank, int world, int nz_global, int z0);
/* Non-uniform split (load-balanced slabs): starts[k] is
 * rank k's first global plane, starts[0] = 0, starts[world] = nz_global,
 * every slab >= 1 plane; this context's mesh holds rank `rank`'s planes. */
int cg_ctx_set_slab_bounds(cg_ctx* ctx, int rank, int world, int nz_global, const int* starts);
int cg_zslab_pack(cg_ctx* ctx, const double* dens, double* send);
int cg_zslab_correct(cg_ctx* ctx, double* dens, const double* recv, int bc,
                     const double* dirichlet);
/* The same interface system by line blocks, for P >= 3 (replaces the
 * all-gather + redundant solve above; slab.py / DESIGN.md section 6): rank r
 * owns lines [r Lb, (r + 1) Lb), Lb = cg_zslab_block_lines(ctx) =
 * ceil(nx*ny / world).  cg_zslab_pack_blocks writes send (world, S, 2, Lb):
 * block r's end values go to rank r; after an all-to-all, recv (world, S, 2,
 * Lb) holds every rank's end values for this rank's block;
 * cg_zslab_reduce_blocks solves those Lb reduced systems and writes out
 * (world, S, 2, Lb): rank k's (l_{k-1}, f_{k+1}) for the block's lines; after
 * a second all-to-all, lr (world, S, 2, Lb) holds this rank's two
 * coefficients for every line and cg_zslab_correct_blocks applies
 * x = y + l_{k-1} v + f_{k+1} w + pins -- bit-identical to
 * cg_zslab_correct, with 2 (P - 1) / P instead of (P - 1) times S 2 nx*ny
 * doubles received per rank.  Replaces diffusion.py:166-186's z sweep across
 * ranks, as cg_zslab_correct. */
long cg_zslab_block_lines(cg_ctx* ctx);
/* Deferred interface correction (fast numerics on slab contexts with fast
 * kernels, all substrates): cg_zslab_defer(ctx, lr) hands (left, right) per
 * line in the line-block layout (world, S, 2, Lb) -- cg_zslab_reduce_blocks'
 * output after the second all-to-all, or cg_zslab_lr_gather's from the
 * all-gathered end values -- to the next cg_lod_step_fast, whose x-row /
 * plane kernel applies x += left v + right w while it stages the field
 * (bit-identical to cg_zslab_correct*; one read + write pass of the field
 * saved per substep).  lr must stay valid until that call; NULL cancels. */
int cg_zslab_lr_gather(cg_ctx* ctx, const double* recv, double* lr);
int cg_zslab_defer(cg_ctx* ctx, const double* lr);
/* Restrict the following cg_lod_step_fast and cg_zslab_* calls on this
 * context to substrates [s0, s0 + ns) (the slab driver's per-substrate
 * pipeline: one substrate's interface exchange in flight while the next
 * substrate's sweeps run); the zslab buffers then hold ns substrates.
 * (0, 0): every substrate again. */
int cg_ctx_set_substrate_window(cg_ctx* ctx, int s0, int ns);
int cg_zslab_pack_blocks(cg_ctx* ctx, const double* dens, double* send);
int cg_zslab_reduce_blocks(cg_ctx* ctx, const double* recv, double* out);
int cg_zslab_correct_blocks(cg_ctx* ctx, double* dens, const double* lr, int bc,
                            const double* dirichlet);
/* Global voxel z index per cell on this context's mesh (-1 outside), with
 * core.py:77-85 CPython semantics: slab ownership for cell migration. */
int cg_voxel_z(cg_ctx* ctx, int n_cells, const double* pos, int32_t* out);
/* core.py:77-85 CartesianMesh.voxel_of on the device for every position (the
 * function the rebin bins with): the flat voxel index, or -1 where the
 * reference raises DomainError.  No error is raised; device pointers. */
int cg_voxel_index(cg_ctx* ctx, int n_cells, const double* pos, int32_t* out);
/* Fast numerics for hand-written step loops such as the z-slab driver
 * (CG_NUMERICS_FAST's kernels and tolerances): cg_rebin_exchange_affine is
 * cg_rebin_exchange with each non-empty voxel's exchange folded into one
 * affine map per substrate; cg_lod_step_fast runs the mesh's segmented x/y
 * kernels (exchange != 0: those maps applied first, fused) and its z sweep
 * (on a slab context the local block solve, as cg_lod_step);
 * cg_velocities_fast sums each cell's terms over its 9 neighbour rows. */
int cg_rebin_exchange_affine(cg_ctx* ctx, int n_cells, const double* pos, const int64_t* ids,
                             int32_t* voxel, int32_t* bin_start, int32_t* bin_cells,
                             int32_t* bin_cells_by_id, int32_t* nonempty, int32_t* n_nonempty,
                             double dt, const double* secretion, const double* uptake,
                             const double* saturation, const double* volume);
int cg_lod_step_fast(cg_ctx* ctx, double* dens, const double* diffusion, const double* decay,
                     double dt, int bc, const double* dirichlet, int exchange);
/* 1 when this context's mesh has fast LOD kernels (cubic 80^3 / 160^3, or
 * 256 x 256 planes), else 0 (the fast calls then return CG_STATE). */
int cg_fast_lod_available(cg_ctx* ctx);
int cg_velocities_fast(cg_ctx* ctx, int n_cells, const double* pos, const double* radius,
                       const int32_t* voxel, const int32_t* bin_start,
                       const int32_t* bin_cells_by_id, double repulsion, double adhesion,
                       double adhesion_multiplier, double* vel);

/* Host helper ---------------------------------------------------------------- */
/* core.py:161-163 Cell.volume = (4/3)*pi*R**3, evaluated with libm pow exactly
 * as CPython evaluates `R**3`; HOST arrays, no GPU needed.  The exchange uses
 * these volumes, so computing them identically keeps the field bit-exact. */
void cg_cell_volumes(int n, const double* radius, double* volume);

/* Instrumentation ----------------------------------------------------------- */
/* While enabled, every kernel launched eagerly is bracketed by CUDA events on
 * the context stream; cg_prof_read syncs and returns per-kernel totals. */
int cg_prof_enable(cg_ctx* ctx, int on);
int cg_prof_read(cg_ctx* ctx, int max_kernels, char* names /* max_kernels*32 */,
                 double* total_ms, int* launches);
long long cg_launch_count(cg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
