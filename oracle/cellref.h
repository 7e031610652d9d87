/*
 * cellref -- CPU ORACLE for the cellbench hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's per-step compute loop
 * (/root/reference/pkg/src/cellbench, a pure-Python + numpy package), written
 * so that every floating-point operation happens in the same order and with
 * the same rounding as the reference:
 *   - numpy elementwise ufuncs (IEEE binary64, one rounding per op, no FMA);
 *   - CPython float arithmetic (binary64, no FMA), CPython float `//`;
 *   - CPython `x ** k` == libm pow(x, k)  (built with -fno-builtin so gcc does
 *     not fold pow(x, 2.0) into x*x -- the two differ by 1 ulp in ~0.08% of
 *     cases on this glibc).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library, and only as the checker or
 * the CPU baseline.  The product path (paper_2306_11544_b200) never calls it.
 *
 * Pinning: tests/golden/ holds fixtures produced by running the reference
 * itself (tests/golden/make_golden.py imports /root/reference read-only);
 * tests/test_oracle_golden.py checks this oracle bit-for-bit against them.
 * The G1 (Dirichlet), G2 (Adams-Bashforth) and G4 (per-cell multi-substrate
 * exchange) extensions have no reference implementation: with the extension
 * disabled they reduce to the reference bit-for-bit (tested); with it enabled
 * they are pinned only against the Python restatement in make_golden.py
 * ("parity unpinned" w.r.t. the reference).
 */
#ifndef CELLREF_H
#define CELLREF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int nx, ny, nz;
    double dx, dy, dz;
    double ox, oy, oz;
} ref_mesh;

enum { REF_OK = 0, REF_DOMAIN = 1, REF_NUMERIC = 2, REF_STATE = 3, REF_CAPACITY = 4 };
enum { REF_BC_NEUMANN = 0, REF_BC_DIRICHLET = 1 };
enum { REF_EULER = 0, REF_AB2 = 1 };
enum { REF_SQUARE_POW = 0, REF_SQUARE_MUL = 1 };

/* core.py:77-85 CartesianMesh.voxel_of (CPython float // semantics). */
int ref_voxel_of(const ref_mesh* m, const double* p, int32_t* out);

/* diffusion.py:80-99 _line_factors. inv, gamma: n doubles each. */
void ref_line_factors(int n, double r, double lam3, double* inv, double* gamma);

/* diffusion.py:127-192 lod_step over all S substrates; dens is (S, nvox).
 * bc/dirichlet: G1 extension (REF_BC_NEUMANN reproduces the reference). */
int ref_lod_step(const ref_mesh* m, int S, double* dens, const double* diffusion,
                 const double* decay, double dt, int bc, const double* dirichlet,
                 int threads);

/* diffusion.py:201-234 apply_cell_exchange, generalised (G4) to per-cell
 * rates.  secretion/uptake are read as rate[s*rate_stride_s + k*rate_stride_c]
 * for cell storage index k; strides of 0 give the reference's scalar form.
 * Updates substrates [s0, s1). Cells of voxel v are applied in ascending id. */
int ref_exchange(const ref_mesh* m, double* dens, int s0, int s1, double dt,
                 const double* secretion, const double* uptake,
                 long rate_stride_s, long rate_stride_c,
                 const double* saturation, long sat_stride,
                 int n_cells, const double* volume, const int64_t* ids,
                 const int32_t* bin_start, const int32_t* bin_cells,
                 const int32_t* nonempty, int n_nonempty, int threads);

/* core.py:218-240 rebin_cells.  bin_start: nvox+1; bin_cells: n (storage
 * indices, storage order within each voxel = the reference's agent lists);
 * nonempty: ascending voxel list (capacity nvox). */
int ref_rebin(const ref_mesh* m, int n, const double* pos, int32_t* voxel,
              int32_t* bin_start, int32_t* bin_cells, int32_t* nonempty,
              int32_t* n_nonempty);

/* mechanics.py:118-133,145-172,175-225 update_velocities.  Uses the voxel of
 * each cell from the last rebin (cell.voxel_index). square_mode selects how
 * `(1 - d/c)**2` is evaluated: REF_SQUARE_POW = libm pow (the reference),
 * REF_SQUARE_MUL = t*t (used to pin the GPU kernel's op order bit-for-bit). */
int ref_velocities(const ref_mesh* m, int n, const double* pos,
                   const double* radius, const int64_t* ids, const int32_t* voxel,
                   const int32_t* bin_start, const int32_t* bin_cells,
                   double repulsion, double adhesion, double adhesion_multiplier,
                   int square_mode, double* vel, int threads);

/* mechanics.py:228-245 integrate_positions (+ G2 AB2 extension). */
int ref_integrate(const ref_mesh* m, int n, double* pos, const double* vel,
                  double* prev_vel, double dt, int integrator, int threads);

/* core.py:161-163 Cell.volume = (4/3)*pi*R**3 (libm pow, as CPython). */
void ref_cell_volumes(int n, const double* radius, double* volume);

/* One mechanics step in simulate.py:166-202 order (gradients, divisions and
 * resorting are out of scope): substeps x [exchange on every substrate with
 * per-cell rates -> lod_step], update_velocities, integrate, rebin. */
int ref_mech_step(const ref_mesh* m, int S, double* dens, const double* diffusion,
                  const double* decay, double dt_diff, int substeps, int bc,
                  const double* dirichlet, const double* secretion,
                  const double* uptake, const double* saturation, int n,
                  double* pos, double* vel, double* prev_vel,
                  const double* radius, const double* volume, const int64_t* ids,
                  int32_t* voxel, int32_t* bin_start, int32_t* bin_cells,
                  int32_t* nonempty, int32_t* n_nonempty, double repulsion,
                  double adhesion, double adhesion_multiplier, double dt_mech,
                  int integrator, int square_mode, int threads);

int ref_max_threads(void);

/* population.py:44-51, 77-129 (divisions; see cellref.c). */
void ref_division_draws(uint64_t seed, int64_t id, int64_t step, double* out3);
int ref_divisions(const ref_mesh* m, int n, const int64_t* ids, const double* pos,
                  const double* radius, const double* rate, double dt, uint64_t seed,
                  int64_t step, int cap, int32_t* parent_out, double* pos_out);


#ifdef __cplusplus
}
#endif
#endif
