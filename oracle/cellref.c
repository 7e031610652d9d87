/*
 * cellref.c -- CPU ORACLE (test infrastructure, never the product path).
 * See cellref.h for the contract.  Every function cites the reference lines
 * it restates; paths are relative to /root/reference/pkg/src/cellbench/.
 *
 * Build flags matter for parity: -ffp-contract=off (no FMA contraction, as
 * numpy ufuncs and CPython floats) and -fno-builtin (keep pow() a libm call,
 * as CPython's float ** int).
 */
#include "cellref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* core.py:23 POSITION_EPS; mechanics.py:38 EPS_SKIP */
#define POSITION_EPS 1e-6
#define EPS_SKIP 1e-8

int ref_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static int nthreads(int threads) { return threads > 0 ? threads : 1; }

/* CPython Objects/floatobject.c _float_div_mod, floor-division part: the
 * quotient is (vx - fmod(vx, wx)) / wx snapped to the nearest integral value,
 * which is NOT always floor(vx / wx). */
static double py_floordiv(double vx, double wx) {
    double mod = fmod(vx, wx);
    double div = (vx - mod) / wx;
    double fl;
    if (mod) {
        if ((wx < 0) != (mod < 0)) {
            mod += wx;
            div -= 1.0;
        }
    }
    if (div) {
        fl = floor(div);
        if (div - fl > 0.5) fl += 1.0;
    } else {
        fl = copysign(0.0, vx / wx);
    }
    return fl;
}

/* core.py:77-85 voxel_of: int((p - o) // d) per axis, bounds-checked. */
int ref_voxel_of(const ref_mesh* m, const double* p, int32_t* out) {
    double fx = py_floordiv(p[0] - m->ox, m->dx);
    double fy = py_floordiv(p[1] - m->oy, m->dy);
    double fz = py_floordiv(p[2] - m->oz, m->dz);
    if (!(fx >= 0.0 && fx < (double)m->nx && fy >= 0.0 && fy < (double)m->ny &&
          fz >= 0.0 && fz < (double)m->nz))
        return REF_DOMAIN;
    int ix = (int)fx, iy = (int)fy, iz = (int)fz;
    /* core.py:69-70 flatten, x fastest */
    *out = ix + m->nx * (iy + m->ny * iz);
    return REF_OK;
}

/* diffusion.py:80-99 _line_factors */
void ref_line_factors(int n, double r, double lam3, double* inv, double* gamma) {
    if (n == 1) {
        inv[0] = 1.0 / (1.0 + lam3);
        gamma[0] = 0.0;
        return;
    }
    double interior = 1.0 + lam3 + 2.0 * r;
    double boundary = 1.0 + lam3 + r;
    inv[0] = 1.0 / boundary;
    gamma[0] = r * inv[0];
    for (int i = 1; i < n; i++) {
        double diag = (i == n - 1) ? boundary : interior;
        inv[i] = 1.0 / (diag - r * gamma[i - 1]);
        gamma[i] = r * inv[i];
    }
}

/* diffusion.py:102-112 _solve_rows for one line with element stride `st`. */
static void solve_line(double* d, long st, int n, const double* inv,
                       const double* gamma, double r) {
    d[0] *= inv[0];
    for (int i = 1; i < n; i++) {
        d[i * st] += r * d[(i - 1) * st];
        d[i * st] *= inv[i];
    }
    for (int i = n - 2; i >= 0; i--) d[i * st] += gamma[i] * d[(i + 1) * st];
}

/* G1 extension (BioFVM apply_dirichlet_conditions): every voxel on an outer
 * face of the mesh is set to the substrate's Dirichlet value. */
static void apply_dirichlet(const ref_mesh* m, double* g, double value) {
    int nx = m->nx, ny = m->ny, nz = m->nz;
    for (int z = 0; z < nz; z++)
        for (int y = 0; y < ny; y++) {
            double* row = g + ((long)z * ny + y) * nx;
            if (z == 0 || z == nz - 1 || y == 0 || y == ny - 1) {
                for (int x = 0; x < nx; x++) row[x] = value;
            } else {
                row[0] = value;
                row[nx - 1] = value;
            }
        }
}

/* diffusion.py:127-192 lod_step.  The reference solves every line of a sweep
 * independently with elementwise ufuncs, so the order in which lines are
 * visited (and the thread split) cannot change a bit; the y and z sweeps are
 * walked here plane-by-plane so the inner loop runs along contiguous x. */
int ref_lod_step(const ref_mesh* m, int S, double* dens, const double* diffusion,
                 const double* decay, double dt, int bc, const double* dirichlet,
                 int threads) {
    if (!(dt > 0.0)) return REF_DOMAIN; /* diffusion.py:137-138 */
    int nx = m->nx, ny = m->ny, nz = m->nz;
    long plane = (long)nx * ny, nvox = plane * nz;
    int nmax = nx > ny ? (nx > nz ? nx : nz) : (ny > nz ? ny : nz);
    double* inv = malloc(sizeof(double) * nmax);
    double* gam = malloc(sizeof(double) * nmax);
    int nt = nthreads(threads);
    for (int s = 0; s < S; s++) {
        double* g = dens + s * nvox;
        double lam3 = dt * decay[s] / 3.0; /* diffusion.py:144 */
        if (bc == REF_BC_DIRICHLET) apply_dirichlet(m, g, dirichlet[s]);

        /* x sweep: rows are contiguous (diffusion.py:147-154) */
        double r = dt * diffusion[s] / (m->dx * m->dx);
        ref_line_factors(nx, r, lam3, inv, gam);
#pragma omp parallel for num_threads(nt) schedule(static)
        for (long row = 0; row < (long)nz * ny; row++) solve_line(g + row * nx, 1, nx, inv, gam, r);
        if (bc == REF_BC_DIRICHLET) apply_dirichlet(m, g, dirichlet[s]);

        /* y sweep (diffusion.py:156-164): line (z, x) has stride nx */
        r = dt * diffusion[s] / (m->dy * m->dy);
        ref_line_factors(ny, r, lam3, inv, gam);
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int z = 0; z < nz; z++) {
            double* p = g + z * plane;
            for (int x = 0; x < nx; x++) p[x] *= inv[0];
            for (int y = 1; y < ny; y++) {
                double* cur = p + (long)y * nx;
                const double* prev = cur - nx;
                for (int x = 0; x < nx; x++) {
                    cur[x] += r * prev[x];
                    cur[x] *= inv[y];
                }
            }
            for (int y = ny - 2; y >= 0; y--) {
                double* cur = p + (long)y * nx;
                const double* next = cur + nx;
                for (int x = 0; x < nx; x++) cur[x] += gam[y] * next[x];
            }
        }
        if (bc == REF_BC_DIRICHLET) apply_dirichlet(m, g, dirichlet[s]);

        /* z sweep (diffusion.py:166-186): line (y, x) has stride nx*ny */
        r = dt * diffusion[s] / (m->dz * m->dz);
        ref_line_factors(nz, r, lam3, inv, gam);
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int y = 0; y < ny; y++) {
            double* p = g + (long)y * nx;
            for (int x = 0; x < nx; x++) p[x] *= inv[0];
            for (int z = 1; z < nz; z++) {
                double* cur = p + z * plane;
                const double* prev = cur - plane;
                for (int x = 0; x < nx; x++) {
                    cur[x] += r * prev[x];
                    cur[x] *= inv[z];
                }
            }
            for (int z = nz - 2; z >= 0; z--) {
                double* cur = p + z * plane;
                const double* next = cur + plane;
                for (int x = 0; x < nx; x++) cur[x] += gam[z] * next[x];
            }
        }
        if (bc == REF_BC_DIRICHLET) apply_dirichlet(m, g, dirichlet[s]);
    }
    free(inv);
    free(gam);
    return REF_OK;
}

typedef struct {
    int64_t id;
    int32_t idx;
} idpair;

static int cmp_idpair(const void* a, const void* b) {
    int64_t x = ((const idpair*)a)->id, y = ((const idpair*)b)->id;
    return (x > y) - (x < y);
}

static void sort_by_id(idpair* a, int n) {
    if (n < 48) { /* insertion sort: candidate lists are short */
        for (int i = 1; i < n; i++) {
            idpair t = a[i];
            int j = i - 1;
            while (j >= 0 && a[j].id > t.id) {
                a[j + 1] = a[j];
                j--;
            }
            a[j + 1] = t;
        }
    } else {
        qsort(a, n, sizeof(idpair), cmp_idpair);
    }
}

/* diffusion.py:201-234 apply_cell_exchange (per-cell rates: G4). */
int ref_exchange(const ref_mesh* m, double* dens, int s0, int s1, double dt,
                 const double* secretion, const double* uptake,
                 long rate_stride_s, long rate_stride_c,
                 const double* saturation, long sat_stride,
                 int n_cells, const double* volume, const int64_t* ids,
                 const int32_t* bin_start, const int32_t* bin_cells,
                 const int32_t* nonempty, int n_nonempty, int threads) {
    (void)n_cells;
    if (!(dt > 0.0)) return REF_DOMAIN; /* diffusion.py:211-212 */
    long nvox = (long)m->nx * m->ny * m->nz;
    double inv_vol = 1.0 / (m->dx * m->dy * m->dz); /* diffusion.py:214, core.py:60-62 */
    int status = REF_OK;
    int nt = nthreads(threads);
#pragma omp parallel num_threads(nt)
    {
        int cap = 64;
        idpair* buf = malloc(sizeof(idpair) * cap);
#pragma omp for schedule(static)
        for (int q = 0; q < n_nonempty; q++) {
            int v = nonempty[q];
            int b0 = bin_start[v], b1 = bin_start[v + 1];
            int cnt = b1 - b0;
            if (cnt > cap) {
                cap = cnt;
                buf = realloc(buf, sizeof(idpair) * cap);
            }
            for (int k = 0; k < cnt; k++) {
                buf[k].idx = bin_cells[b0 + k];
                buf[k].id = ids[buf[k].idx];
            }
            sort_by_id(buf, cnt); /* diffusion.py:223 sorted(ids) */
            for (int s = s0; s < s1; s++) {
                double rho = dens[s * nvox + v];
                double sat = saturation[s * sat_stride];
                for (int k = 0; k < cnt; k++) {
                    int c = buf[k].idx;
                    double sec = secretion[s * rate_stride_s + c * rate_stride_c];
                    double upt = uptake[s * rate_stride_s + c * rate_stride_c];
                    double f = dt * volume[c] * inv_vol;
                    double den = 1.0 + f * (sec + upt);
                    if (den <= 0.0) {
#pragma omp atomic write
                        status = REF_DOMAIN;
                        break;
                    }
                    rho = (rho + f * sec * sat) / den;
                }
                dens[s * nvox + v] = rho;
            }
        }
        free(buf);
    }
    return status;
}

/* core.py:218-240 rebin_cells: serial pass in storage order. */
int ref_rebin(const ref_mesh* m, int n, const double* pos, int32_t* voxel,
              int32_t* bin_start, int32_t* bin_cells, int32_t* nonempty,
              int32_t* n_nonempty) {
    long nvox = (long)m->nx * m->ny * m->nz;
    memset(bin_start, 0, sizeof(int32_t) * (nvox + 1));
    for (int i = 0; i < n; i++) {
        if (ref_voxel_of(m, pos + 3L * i, &voxel[i]) != REF_OK) return REF_DOMAIN;
        bin_start[voxel[i] + 1]++;
    }
    int ne = 0;
    for (long v = 0; v < nvox; v++) {
        if (bin_start[v + 1]) nonempty[ne++] = (int32_t)v; /* sorted(agent) */
        bin_start[v + 1] += bin_start[v];
    }
    *n_nonempty = ne;
    int32_t* cursor = malloc(sizeof(int32_t) * nvox);
    memcpy(cursor, bin_start, sizeof(int32_t) * nvox);
    for (int i = 0; i < n; i++) bin_cells[cursor[voxel[i]]++] = i; /* bucket.append */
    free(cursor);
    return REF_OK;
}

static inline double sq_pow(double t) { return pow(t, 2.0); }
static inline double sq_mul(double t) { return t * t; }

/* mechanics.py:145-172 _cell_velocity for residents of one voxel over the
 * id-sorted candidate list of mechanics.py:118-133 _voxel_candidates. */
static void voxel_velocities(const double* pos, const double* radius, const int64_t* ids,
                             const idpair* cand, int nc, const int32_t* res, int nres,
                             double c_r, double c_a, double m_a, int square_mode,
                             double* vel) {
    for (int q = 0; q < nres; q++) {
        int i = res[q];
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        const double* pi = pos + 3L * i;
        double ri = radius[i];
        int64_t id_i = ids[i];
        for (int k = 0; k < nc; k++) {
            if (cand[k].id == id_i) continue;
            int j = cand[k].idx;
            const double* pj = pos + 3L * j;
            double d0 = pj[0] - pi[0], d1 = pj[1] - pi[1], d2 = pj[2] - pi[2];
            double d = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            double contact = ri + radius[j];
            double reach = m_a * contact;
            if (d < EPS_SKIP || d >= reach) continue;
            double t1 = 1.0 - d / contact, t2 = 1.0 - d / reach;
            double rep, adh;
            if (square_mode == REF_SQUARE_POW) {
                rep = d < contact ? -c_r * sq_pow(t1) : 0.0;
                adh = c_a * sq_pow(t2);
            } else {
                rep = d < contact ? -c_r * sq_mul(t1) : 0.0;
                adh = c_a * sq_mul(t2);
            }
            double coef = (rep + adh) / d;
            a0 = a0 + coef * d0;
            a1 = a1 + coef * d1;
            a2 = a2 + coef * d2;
        }
        vel[3L * i + 0] = a0;
        vel[3L * i + 1] = a1;
        vel[3L * i + 2] = a2;
    }
}

/* mechanics.py:175-225 update_velocities (nonempty_voxel schedule; all
 * schedules are bit-identical, mechanics.py:1-8). */
int ref_velocities(const ref_mesh* m, int n, const double* pos,
                   const double* radius, const int64_t* ids, const int32_t* voxel,
                   const int32_t* bin_start, const int32_t* bin_cells,
                   double repulsion, double adhesion, double adhesion_multiplier,
                   int square_mode, double* vel, int threads) {
    (void)voxel;
    (void)n;
    int nx = m->nx, ny = m->ny, nz = m->nz;
    long nvox = (long)nx * ny * nz;
    int nt = nthreads(threads);
#pragma omp parallel num_threads(nt)
    {
        int cap = 256;
        idpair* cand = malloc(sizeof(idpair) * cap);
#pragma omp for schedule(dynamic, 64)
        for (long v = 0; v < nvox; v++) {
            int b0 = bin_start[v], b1 = bin_start[v + 1];
            if (b0 == b1) continue;
            int ix = (int)(v % nx), rest = (int)(v / nx);
            int iy = rest % ny, iz = rest / ny;
            int nc = 0;
            for (int z = (iz - 1 > 0 ? iz - 1 : 0); z < (iz + 2 < nz ? iz + 2 : nz); z++)
                for (int y = (iy - 1 > 0 ? iy - 1 : 0); y < (iy + 2 < ny ? iy + 2 : ny); y++) {
                    long row = ((long)z * ny + y) * nx;
                    int xlo = ix - 1 > 0 ? ix - 1 : 0, xhi = ix + 2 < nx ? ix + 2 : nx;
                    int c0 = bin_start[row + xlo], c1 = bin_start[row + xhi];
                    if (nc + (c1 - c0) > cap) {
                        while (nc + (c1 - c0) > cap) cap *= 2;
                        cand = realloc(cand, sizeof(idpair) * cap);
                    }
                    for (int k = c0; k < c1; k++) {
                        cand[nc].idx = bin_cells[k];
                        cand[nc].id = ids[bin_cells[k]];
                        nc++;
                    }
                }
            sort_by_id(cand, nc); /* mechanics.py:132 ids.sort() */
            voxel_velocities(pos, radius, ids, cand, nc, bin_cells + b0, b1 - b0,
                             repulsion, adhesion, adhesion_multiplier, square_mode, vel);
        }
        free(cand);
    }
    return REF_OK;
}

/* mechanics.py:228-245 integrate_positions; G2: Adams-Bashforth 2 as in
 * PhysiCell's Cell::update_position (d1 = 1.5 dt, d2 = -0.5 dt, previous
 * velocity starts at zero). */
int ref_integrate(const ref_mesh* m, int n, double* pos, const double* vel,
                  double* prev_vel, double dt, int integrator, int threads) {
    if (!(dt > 0.0)) return REF_DOMAIN; /* mechanics.py:231-232 */
    double ux = m->ox + m->nx * m->dx, uy = m->oy + m->ny * m->dy, uz = m->oz + m->nz * m->dz;
    double lo[3] = {m->ox + POSITION_EPS, m->oy + POSITION_EPS, m->oz + POSITION_EPS};
    double hi[3] = {ux - POSITION_EPS, uy - POSITION_EPS, uz - POSITION_EPS};
    double d1 = dt * 1.5, d2 = dt * -0.5;
    int nt = nthreads(threads);
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int i = 0; i < n; i++) {
        double* p = pos + 3L * i;
        const double* v = vel + 3L * i;
        if (integrator == REF_AB2) {
            double* pv = prev_vel + 3L * i;
            for (int k = 0; k < 3; k++) {
                p[k] += d1 * v[k] + d2 * pv[k];
                pv[k] = v[k];
            }
        } else {
            p[0] += dt * v[0];
            p[1] += dt * v[1];
            p[2] += dt * v[2];
        }
        /* core.py:87-102 contains / clamp_inside (Python min(max(p, lo), hi)) */
        int inside = m->ox <= p[0] && p[0] < ux && m->oy <= p[1] && p[1] < uy &&
                     m->oz <= p[2] && p[2] < uz;
        if (!inside) {
            for (int k = 0; k < 3; k++) {
                double t = lo[k] > p[k] ? lo[k] : p[k];
                p[k] = hi[k] < t ? hi[k] : t;
            }
        }
    }
    return REF_OK;
}

/* population.py:32-37 _mix64 (64-bit wrap-around) */
static uint64_t mix64(uint64_t x) {
    x = x + 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* population.py:40-41 _unit */
static double unit53(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

/* population.py:44-51 division_draws; negative ids / steps wrap like Python's
 * `& _MASK`. */
void ref_division_draws(uint64_t seed, int64_t id, int64_t step, double* out3) {
    uint64_t base = mix64(mix64(mix64(seed) ^ (uint64_t)id) ^ (uint64_t)step);
    out3[0] = unit53(mix64(base ^ 1u));
    out3[1] = unit53(mix64(base ^ 2u));
    out3[2] = unit53(mix64(base ^ 3u));
}

/* population.py:77-129 attempt_divisions, minus the container bookkeeping:
 * cell i divides when rate[i] > 0 and u0 < 1 - exp(-rate*dt); dividers in
 * ascending id get daughters at R/2 along (rho cos phi, rho sin phi, z),
 * clamped inside (core.py:96-102, unconditional).  Writes the parents'
 * indices (ascending id) and the daughters' positions; returns the count, or
 * -1 when n + count > cap (population.py:98-102: CapacityError before any
 * append). */
int ref_divisions(const ref_mesh* m, int n, const int64_t* ids, const double* pos,
                  const double* radius, const double* rate, double dt, uint64_t seed,
                  int64_t step, int cap, int32_t* parent_out, double* pos_out) {
    idpair* div = (idpair*)malloc(sizeof(idpair) * (n > 0 ? n : 1));
    int cnt = 0;
    for (int i = 0; i < n; i++) {
        if (rate[i] <= 0.0) continue;
        double u[3];
        ref_division_draws(seed, ids[i], step, u);
        if (u[0] < 1.0 - exp(-rate[i] * dt)) {
            div[cnt].id = ids[i];
            div[cnt].idx = i;
            cnt++;
        }
    }
    if (cnt && n + cnt > cap) {
        free(div);
        return -1;
    }
    sort_by_id(div, cnt);
    double ux = m->ox + m->nx * m->dx, uy = m->oy + m->ny * m->dy, uz = m->oz + m->nz * m->dz;
    double lo[3] = {m->ox + POSITION_EPS, m->oy + POSITION_EPS, m->oz + POSITION_EPS};
    double hi[3] = {ux - POSITION_EPS, uy - POSITION_EPS, uz - POSITION_EPS};
    const double pi = 3.141592653589793; /* math.pi */
    for (int r = 0; r < cnt; r++) {
        int i = div[r].idx;
        double u[3];
        ref_division_draws(seed, ids[i], step, u);
        double z = 2.0 * u[1] - 1.0;
        double t = 1.0 - z * z;
        double rho = sqrt(t > 0.0 ? t : 0.0);
        double phi = 2.0 * pi * u[2];
        double half_r = 0.5 * radius[i];
        double* p = pos_out + 3L * r;
        p[0] = pos[3L * i] + half_r * rho * cos(phi);
        p[1] = pos[3L * i + 1] + half_r * rho * sin(phi);
        p[2] = pos[3L * i + 2] + half_r * z;
        for (int k = 0; k < 3; k++) {
            double a = p[k] < lo[k] ? lo[k] : p[k]; /* max(p, lo) */
            p[k] = a <= hi[k] ? a : hi[k];          /* min(., hi) */
        }
        parent_out[r] = i;
    }
    free(div);
    return cnt;
}

/* core.py:161-163 */
void ref_cell_volumes(int n, const double* radius, double* volume) {
    const double pi = 3.141592653589793; /* math.pi */
    for (int i = 0; i < n; i++) volume[i] = (4.0 / 3.0) * pi * pow(radius[i], 3.0);
}

/* simulate.py:166-202 (one mechanics step; see header). */
int ref_mech_step(const ref_mesh* m, int S, double* dens, const double* diffusion,
                  const double* decay, double dt_diff, int substeps, int bc,
                  const double* dirichlet, const double* secretion,
                  const double* uptake, const double* saturation, int n,
                  double* pos, double* vel, double* prev_vel,
                  const double* radius, const double* volume, const int64_t* ids,
                  int32_t* voxel, int32_t* bin_start, int32_t* bin_cells,
                  int32_t* nonempty, int32_t* n_nonempty, double repulsion,
                  double adhesion, double adhesion_multiplier, double dt_mech,
                  int integrator, int square_mode, int threads) {
    int st;
    for (int k = 0; k < substeps; k++) {
        if (secretion && uptake) {
            st = ref_exchange(m, dens, 0, S, dt_diff, secretion, uptake, n, 1, saturation, 1,
                              n, volume, ids, bin_start, bin_cells, nonempty, *n_nonempty,
                              threads);
            if (st) return st;
        }
        st = ref_lod_step(m, S, dens, diffusion, decay, dt_diff, bc, dirichlet, threads);
        if (st) return st;
    }
    st = ref_velocities(m, n, pos, radius, ids, voxel, bin_start, bin_cells, repulsion,
                        adhesion, adhesion_multiplier, square_mode, vel, threads);
    if (st) return st;
    st = ref_integrate(m, n, pos, vel, prev_vel, dt_mech, integrator, threads);
    if (st) return st;
    return ref_rebin(m, n, pos, voxel, bin_start, bin_cells, nonempty, n_nonempty);
}
