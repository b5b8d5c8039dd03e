/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the DSEAmd hot
 * path computes (arXiv 2507.11289, "Cyclic Data Streaming on GPUs for Short
 * Range Stencils Applied to Molecular Dynamics").  It is the parity oracle for
 * the CUDA engine in paper_2507_11289_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or constant with the CUDA path.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section named beside it).
 * Readings of silent/ambiguous passages are the SURVEY.md §8(c) readings Q1-Q19,
 * restated in DESIGN.md §3.
 *
 * The streaming method reaches exactly (up to FP reassociation) the result of
 * plain sequential velocity-Verlet over all pairs: cell lists are exact when
 * l >= rc (§4) and the ring is an exact re-scheduling of timesteps, not a
 * predictor (§2, §3.1).  So the oracle is the plain definition:
 * an O(N^2) all-ordered-pairs integrator following Algorithm 1.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no -ffast-math).
 *
 * Pins (tests/test_oracle_pins.py): splitmix64 published vector; FCC geometry;
 * F = -grad U by finite differences; LJ minimum at 2^(1/6); cutoff inclusivity
 * and shifted-energy continuity; virial identity sum r.F = 24 V; Newton's third
 * law; explicit periodic-image brute force; FCC shell sums; NVE drift and its
 * dt^2 scaling; time reversibility through wall hits; NVT: every slice at
 * T_target after the scaling, long-run mean temperature, per-slice records summing
 * to the totals, configurational pressure = -dU/dVol by finite differences.  Parity unpinned: the
 * paper prints no per-atom values, so the exact mirror rule (Q2) and the
 * velocity generator (Q9) are pinned by our own contract, not by the paper.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* Geometry (§4; slices P:63-73 §3; reading Q3 for n_slices)  */
/* out[0..2]=b, out[3..5]=l, out[6]=w, out[7]=a, out[8]=ushift,        */
/* out[9..11]=cells (as doubles), out[12]=n_slices, out[13]=n_atoms     */
/* returns 0, or -1 when the geometry violates l>=rc / >=3 cells y,z.   */
/* ------------------------------------------------------------------ */
int oracle_geometry(int nx, int ny, int nz, double rho, double rc,
                    int n_slices, int c, double *out)
{
    /* b = N_i (4/rho)^(1/3) generalised per axis */
    double a = cbrt(4.0 / rho);
    double bx = nx * a, by = ny * a, bz = nz * a;
    /* N_xyz = floor(b/rc) */
    int cy = (int)floor(by / rc);
    int cz = (int)floor(bz / rc);
    if (c < 1) return -1;
    if (n_slices <= 0) n_slices = (int)floor(bx / (c * rc));
    int cx = c * n_slices;
    double lx = bx / cx, ly = by / cy, lz = bz / cz;
    /* U_shift = (sigma/rc)^6 - (sigma/rc)^12 so that 4(r^-12 - r^-6 + U_shift) = 0 at rc (Q6) */
    double sr6 = 1.0 / (rc * rc * rc * rc * rc * rc);
    double ushift = sr6 - sr6 * sr6;
    out[0] = bx; out[1] = by; out[2] = bz;
    out[3] = lx; out[4] = ly; out[5] = lz;
    out[6] = bx / n_slices;
    out[7] = a;
    out[8] = ushift;
    out[9] = cx; out[10] = cy; out[11] = cz;
    out[12] = n_slices;
    out[13] = 4.0 * nx * ny * nz;
    if (n_slices < 1 || cy < 3 || cz < 3) return -1;
    if (lx < rc || ly < rc || lz < rc) return -1;   /* Q18: accept l >= rc */
    return 0;
}

/* ------------------------------------------------------------------ */
/* FCC lattice, 4 molecules per cell (§4), offset a/4 (Q10).      */
/* id = ((ix*ny + iy)*nz + iz)*4 + k ; xyz is [3N] ordered by id.       */
/* ------------------------------------------------------------------ */
void oracle_lattice(int nx, int ny, int nz, double a, double *xyz)
{
    static const double basis[4][3] = {
        {0.0, 0.0, 0.0}, {0.5, 0.5, 0.0}, {0.5, 0.0, 0.5}, {0.0, 0.5, 0.5}};
    int64_t id = 0;
    for (int ix = 0; ix < nx; ix++)
        for (int iy = 0; iy < ny; iy++)
            for (int iz = 0; iz < nz; iz++)
                for (int k = 0; k < 4; k++) {
                    xyz[3 * id + 0] = (ix + basis[k][0] + 0.25) * a;
                    xyz[3 * id + 1] = (iy + basis[k][1] + 0.25) * a;
                    xyz[3 * id + 2] = (iz + basis[k][2] + 0.25) * a;
                    id++;
                }
}

/* ------------------------------------------------------------------ */
/* Velocities "initialized according to the temperature" (§4);  */
/* reading Q9: splitmix64 -> 53-bit uniform -> Box-Muller (cos branch), */
/* zero momentum, exact rescale to T0 with 3N degrees of freedom.       */
/* ------------------------------------------------------------------ */
uint64_t oracle_splitmix64_next(uint64_t *state)
{
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double uniform01(uint64_t *state)
{
    return (double)(oracle_splitmix64_next(state) >> 11) * (1.0 / 9007199254740992.0);
}

/* One standard normal from two consecutive uniforms. */
double oracle_normal(uint64_t *state)
{
    double u1 = uniform01(state);
    double u2 = uniform01(state);
    return sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * 3.141592653589793 * u2);
}

void oracle_velocities(int64_t n, uint64_t seed, double T0, double *v)
{
    uint64_t st = seed;
    for (int64_t i = 0; i < 3 * n; i++) v[i] = oracle_normal(&st);
    /* subtract the mean, summed sequentially in id order */
    for (int d = 0; d < 3; d++) {
        double s = 0.0;
        for (int64_t i = 0; i < n; i++) s += v[3 * i + d];
        double mean = s / (double)n;
        for (int64_t i = 0; i < n; i++) v[3 * i + d] -= mean;
    }
    /* T_m = sum v^2 / (3N)  (m = k_B = 1, Q11) */
    double s2 = 0.0;
    for (int64_t i = 0; i < n; i++)
        s2 += v[3 * i] * v[3 * i] + v[3 * i + 1] * v[3 * i + 1] + v[3 * i + 2] * v[3 * i + 2];
    double Tm = s2 / (3.0 * (double)n);
    double f = sqrt(T0 / Tm);
    for (int64_t i = 0; i < 3 * n; i++) v[i] *= f;
}

/* ------------------------------------------------------------------ */
/* Forces: Algorithm 1 force loop, over ALL ordered pairs   */
/* i != j.  Minimum image in y and z (Q1), none in x (walls).  */
/* U, V accumulate per ordered pair with the paper's /2. */
/* Ui (optional, may be NULL) receives the per-atom share of U.         */
/* ------------------------------------------------------------------ */
static void pair_sum_for_atom(int64_t i, int64_t n, const double *xyz, double by, double bz,
                              double rc2, double ushift, double *Fi, double *Ui, double *Vi)
{
    double fx = 0.0, fy = 0.0, fz = 0.0, u = 0.0, vir = 0.0;
    for (int64_t j = 0; j < n; j++) {
        if (j == i) continue;
        double dx = xyz[3 * i] - xyz[3 * j];
        double dy = xyz[3 * i + 1] - xyz[3 * j + 1];
        double dz = xyz[3 * i + 2] - xyz[3 * j + 2];
        dy -= by * rint(dy / by);
        dz -= bz * rint(dz / bz);
        double r2 = dx * dx + dy * dy + dz * dz;
        if (r2 <= rc2) {                          /* inclusive, P:262 (Q5) */
            double sr2 = 1.0 / r2;
            double sr6 = sr2 * sr2 * sr2;        /* sigma^6 / r^6  */
            double sr12 = sr6 * sr6;             /* sigma^12 / r^12 */
            double fabs_ = 24.0 * (2.0 * sr12 - sr6) / r2;
            fx += dx * fabs_;
            fy += dy * fabs_;
            fz += dz * fabs_;
            u += 4.0 * (sr12 - sr6 + ushift) / 2.0;
            vir += (2.0 * sr12 - sr6) / 2.0;
        }
    }
    Fi[0] = fx; Fi[1] = fy; Fi[2] = fz;
    *Ui = u; *Vi = vir;
}

void oracle_forces(int64_t n, const double *xyz, const double *box, double rc,
                   double *F, double *U, double *V, double *Ui, double *Vi, int nthreads)
{
    double by = box[1], bz = box[2];
    double rc2 = rc * rc;
    double sr6c = 1.0 / (rc * rc * rc * rc * rc * rc);
    double ushift = sr6c - sr6c * sr6c;
    double *ui = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *vi = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < n; i++)
        pair_sum_for_atom(i, n, xyz, by, bz, rc2, ushift, &F[3 * i], &ui[i], &vi[i]);
    /* per-atom partials summed sequentially in id order: independent of thread count */
    double su = 0.0, sv = 0.0;
    for (int64_t i = 0; i < n; i++) { su += ui[i]; sv += vi[i]; }
    if (Ui) memcpy(Ui, ui, sizeof(double) * (size_t)n);
    if (Vi) memcpy(Vi, vi, sizeof(double) * (size_t)n);
    *U = su; *V = sv;
    free(ui); free(vi);
}

/* Forces on a subset of atoms (sampled brute force at full size). */
void oracle_forces_subset(int64_t n, const double *xyz, const double *box, double rc,
                          int64_t nsub, const int64_t *idx, double *Fsub, double *Usub,
                          int nthreads)
{
    double rc2 = rc * rc;
    double sr6c = 1.0 / (rc * rc * rc * rc * rc * rc);
    double ushift = sr6c - sr6c * sr6c;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
#endif
    for (int64_t k = 0; k < nsub; k++) {
        double vdummy;
        pair_sum_for_atom(idx[k], n, xyz, box[1], box[2], rc2, ushift, &Fsub[3 * k],
                          &Usub[k], &vdummy);
    }
}

/* ------------------------------------------------------------------ */
/* Boundaries after the position update.                               */
/* x: mirror at 0 and b_x (§4.2), reading Q2: fold the position, */
/*    negate v_x and the stored F_new,x.                                */
/* y, z: periodic wrap into [0, b) (Q1).                                */
/* ------------------------------------------------------------------ */
void oracle_bin(int64_t n, const double *xyz, const double *l, const int32_t *cells, int c,
                int32_t *cell_xyz, int32_t *slice);

static void apply_boundaries(double *r, double *v, double *f, const double *box)
{
    if (r[0] < 0.0) {
        r[0] = -r[0]; v[0] = -v[0]; f[0] = -f[0];
    } else if (r[0] > box[0]) {
        r[0] = 2.0 * box[0] - r[0]; v[0] = -v[0]; f[0] = -f[0];
    }
    for (int d = 1; d < 3; d++) {
        if (r[d] < 0.0) r[d] += box[d];
        else if (r[d] >= box[d]) r[d] -= box[d];
    }
}

/* ------------------------------------------------------------------ */
/* Velocity-Verlet, Algorithm 1, first-step convention Q7   */
/* (F_new = 0 at entry on a fresh state).  State arrays are [3N] by id; */
/* F holds F_new on entry and on exit.  energies: [nsteps][4] =         */
/* {U, KE, V, E=U+KE} with E_n = U(r_n) + KE(v_n) (Q12).                 */
/*                                                                      */
/* Optional NVT thermostat (T_target > 0), §4.1: after the    */
/* kick (md_v3aa) the scale factor is computed per slice (md_thermo_a/b)*/
/* and applied before the position update (md_v3b).  Reading Q23:       */
/* isokinetic, lambda_j = sqrt(T_target / T_j) with T_j = sum v.v /     */
/* (3 n_j) over the atoms of slice j (membership = binning of r at the  */
/* start of the step); lambda_j = 1 for an empty or motionless slice.   */
/* KE in energies stays the post-kick, pre-scale value.                 */
/* slice_rec (optional): [nsteps][n_slices][4] = {n_j, U_j, V_j, KE_j}, */
/* U_j, V_j = sums of the per-atom Algorithm-1 shares of the slice's    */
/* atoms, KE_j = post-kick, pre-scale kinetic energy of the slice.      */
/* ------------------------------------------------------------------ */
int oracle_run_ex(int64_t n, double *xyz, double *v, double *F, const double *box, double rc,
                  double dt, int64_t nsteps, double *energies, int nthreads, double T_target,
                  const double *l, const int32_t *cells, int c, int n_slices, double *slice_rec)
{
    const int need_slices = (T_target > 0.0) || slice_rec;
    size_t n1 = (size_t)(n > 0 ? n : 1);
    double *Fold = (double *)malloc(sizeof(double) * 3 * n1);
    double *ui = (double *)malloc(sizeof(double) * n1);
    double *vi = (double *)malloc(sizeof(double) * n1);
    int32_t *cxyz = (int32_t *)malloc(sizeof(int32_t) * 3 * n1);
    int32_t *sl = (int32_t *)malloc(sizeof(int32_t) * n1);
    double *ke_j = (double *)malloc(sizeof(double) * (size_t)(n_slices > 0 ? n_slices : 1));
    double *cnt_j = (double *)malloc(sizeof(double) * (size_t)(n_slices > 0 ? n_slices : 1));
    int rv = 0;
    if (!Fold || !ui || !vi || !cxyz || !sl || !ke_j || !cnt_j) { rv = -1; goto done; }
    if (need_slices && (!l || !cells || c < 1 || n_slices < 1)) { rv = -2; goto done; }
    for (int64_t step = 0; step < nsteps; step++) {
        /* slice membership of every atom at the start of the step */
        if (need_slices) oracle_bin(n, xyz, l, cells, c, cxyz, sl);
        /* F_old = F_new ; F_new = sum over neighbours */
        memcpy(Fold, F, sizeof(double) * (size_t)(3 * n));
        double U, V;
        oracle_forces(n, xyz, box, rc, F, &U, &V, ui, vi, nthreads);
        /* v = v + (F_new + F_old) * 0.5 * dt */
        for (int64_t i = 0; i < 3 * n; i++) v[i] = v[i] + (F[i] + Fold[i]) * 0.5 * dt;
        double ke = 0.0;
        for (int64_t i = 0; i < n; i++)
            ke += v[3 * i] * v[3 * i] + v[3 * i + 1] * v[3 * i + 1] + v[3 * i + 2] * v[3 * i + 2];
        ke *= 0.5;
        if (energies) {
            energies[4 * step + 0] = U;
            energies[4 * step + 1] = ke;
            energies[4 * step + 2] = V;
            energies[4 * step + 3] = U + ke;
        }
        if (need_slices) {
            for (int j = 0; j < n_slices; j++) { ke_j[j] = 0.0; cnt_j[j] = 0.0; }
            for (int64_t i = 0; i < n; i++) {
                const double vv = v[3 * i] * v[3 * i] + v[3 * i + 1] * v[3 * i + 1] + v[3 * i + 2] * v[3 * i + 2];
                ke_j[sl[i]] += vv;
                cnt_j[sl[i]] += 1.0;
            }
            if (slice_rec) {
                double *rec = slice_rec + (size_t)step * n_slices * 4;
                for (int j = 0; j < n_slices; j++) {
                    rec[4 * j + 0] = cnt_j[j];
                    rec[4 * j + 1] = 0.0;
                    rec[4 * j + 2] = 0.0;
                    rec[4 * j + 3] = 0.5 * ke_j[j];
                }
                for (int64_t i = 0; i < n; i++) {
                    rec[4 * sl[i] + 1] += ui[i];
                    rec[4 * sl[i] + 2] += vi[i];
                }
            }
            if (T_target > 0.0) {
                /* md_thermo_a/b + the scaling in md_v3b, reading Q23 */
                for (int j = 0; j < n_slices; j++) {
                    const double Tj = (cnt_j[j] > 0.0) ? ke_j[j] / (3.0 * cnt_j[j]) : 0.0;
                    ke_j[j] = (Tj > 0.0) ? sqrt(T_target / Tj) : 1.0;   /* lambda_j */
                }
                for (int64_t i = 0; i < n; i++) {
                    const double lam = ke_j[sl[i]];
                    v[3 * i] *= lam; v[3 * i + 1] *= lam; v[3 * i + 2] *= lam;
                }
            }
        }
        /* r = r + v*dt + F_new*0.5*dt^2 */
        for (int64_t i = 0; i < 3 * n; i++) xyz[i] = xyz[i] + v[i] * dt + F[i] * 0.5 * (dt * dt);
        for (int64_t i = 0; i < n; i++) apply_boundaries(&xyz[3 * i], &v[3 * i], &F[3 * i], box);
    }
done:
    free(Fold); free(ui); free(vi); free(cxyz); free(sl); free(ke_j); free(cnt_j);
    return rv;
}

int oracle_run(int64_t n, double *xyz, double *v, double *F, const double *box, double rc,
               double dt, int64_t nsteps, double *energies, int nthreads)
{
    return oracle_run_ex(n, xyz, v, F, box, rc, dt, nsteps, energies, nthreads, -1.0, NULL, NULL,
                         1, 0, NULL);
}

/* ------------------------------------------------------------------ */
/* Binning (§4; Q4): cell_d = clamp(floor(r_d / l_d), 0,      */
/* cells_d - 1) with IEEE division; slice = cell_x / c.                 */
/* ------------------------------------------------------------------ */
void oracle_bin(int64_t n, const double *xyz, const double *l, const int32_t *cells, int c,
                int32_t *cell_xyz, int32_t *slice)
{
    for (int64_t i = 0; i < n; i++) {
        for (int d = 0; d < 3; d++) {
            double q = floor(xyz[3 * i + d] / l[d]);
            int32_t k;
            if (!(q >= 0.0)) k = 0;                       /* also catches NaN */
            else if (q >= (double)(cells[d] - 1)) k = cells[d] - 1;
            else k = (int32_t)q;
            cell_xyz[3 * i + d] = k;
        }
        slice[i] = cell_xyz[3 * i] / c;
    }
}

/* Eq. (1), §3.3, floor semantics (Q17). */
int oracle_nmax(int n_slices, int w_per_gpu, int o_in, int o_out)
{
    return n_slices / (2 + w_per_gpu * (o_in + o_out));
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
