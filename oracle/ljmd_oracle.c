/*
 * ljmd_oracle.c -- CPU ORACLE for the Lennard-Jones PairLoop hot path of
 * arXiv 1704.03329 (PPMD).  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path in paper_1704_03329_b200/csrc/.
 *
 * Plain, slow, obviously-correct fp64 C.  Compiled with -O2 -ffp-contract=off
 * so that every a*b+c below is two roundings, exactly as written.
 *
 * Citations: P:n = PAPER.md line n.  Readings R1..R17 are listed in DESIGN.md.
 *
 *   O1 wrap              : periodic box [0,L) (reading R10)
 *   O2 pair displacement : minimum image, canonical r^2 (reading R9)
 *   O3 brute neighbours  : Def. 3 Local Particle Pair Loop at rbar_c
 *   O4 cell neighbours   : cell method of Sec. 3.4, independent
 *   O5 forces / energies : Eq. eqn:LJpotential, Eq. eqn:LJforce
 *                          (P:969-978), Listing lst:LJ-kernel
 *                          with the Eq. sign (reading R1) and PE = 1/2 sum
 *                          over ordered pairs (reading R2)
 *   O6 velocity Verlet   : Algorithm alg:VelocityVerlet, Listings
 *                          lst:position_update / lst:velocity_update
 *                          (P:659-675), Tab. access_descriptors
 *   O7 rebuild schedule  : IntegratorRange, every Ns = 20 steps
 *                          (P:728); optional displacement check (R7)
 *   O8 Andersen thermostat (reading R19): after line 8 of every step each
 *                          particle, with probability nu*dt, draws a new velocity
 *                          from N(0, T/m) per component.  Random numbers from the
 *                          counter-based Philox4x32-10 (Salmon et al. 2011), keyed by
 *                          (seed, gid, step), written out here independently of the
 *                          GPU's copy and pinned by its published known-answer vectors.
 *
 * Every function is pinned by a -m "not gpu" test (tests/test_oracle_*.py)
 * against closed forms, golden fixtures or brute force; see DESIGN.md §Oracle.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Threads of the OpenMP build (bench.py's all-core leg); the plain build runs 1.  k > 0
 * sets the count; returns the count in use.  No result depends on it: every parallel loop
 * writes per-particle rows or reduces integers. */
int orc_threads(int k)
{
#ifdef _OPENMP
    if (k > 0) omp_set_num_threads(k);
    return omp_get_max_threads();
#else
    (void)k;
    return 1;
#endif
}

/* ------------------------------------------------------------------ O1 -- */
/* Wrap one coordinate into the half-open interval [0, L) (reading R10).
 * Arbitrary input: x - L*floor(x/L), then fold the +-1 ulp artefacts. */
static double wrap1(double x, double L)
{
    double k = floor(x / L);
    double t = x - L * k;
    if (t < 0.0) t = t + L;
    if (t >= L) t = t - L;
    return t;
}

/* Returns -1 on success, else the index of the first particle with a
 * non-finite coordinate (nothing is modified in that case). */
int64_t orc_wrap(int64_t n, double *pos, const double box[3])
{
    for (int64_t i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d)
            if (!isfinite(pos[3 * i + d])) return i;
    for (int64_t i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d)
            pos[3 * i + d] = wrap1(pos[3 * i + d], box[d]);
    return -1;
}

/* ------------------------------------------------------------------ O2 -- */
/* Minimum-image displacement r_i - r_j (reading R9):
 *   d0 = xi - xj;  s = +1 if d0 > L/2, -1 if d0 < -L/2, else 0;
 *   dx = xi - (xj + s*L)          (one rounding for the image position) */
void orc_displacement(const double *xi, const double *xj, const double box[3], double d[3])
{
    for (int k = 0; k < 3; ++k) {
        double d0 = xi[k] - xj[k];
        double half = 0.5 * box[k];
        double s = 0.0;
        if (d0 > half) s = 1.0;
        else if (d0 < -half) s = -1.0;
        double img = xj[k] + s * box[k];
        d[k] = xi[k] - img;
    }
}

/* r^2 = (dx*dx + dy*dy) + dz*dz, left to right, no contraction (R9). */
double orc_r2(const double d[3])
{
    double a = d[0] * d[0];
    double b = d[1] * d[1];
    double c = d[2] * d[2];
    return (a + b) + c;
}

/* ------------------------------------------------------------------ O3 -- */
/* Brute-force neighbour sets NB(i) = { j != i : r^2(i,j) < rn^2 } (strict,
 * reading R4), O(N^2), each NB(i) in ascending j.  Two-pass use: call with
 * nbr == NULL to get offsets (size n+1) and the total; then with nbr. */
int64_t orc_neigh_brute(int64_t n, const double *pos, const double box[3], double rn,
                        int64_t *offsets, int64_t *nbr)
{
    double rn2 = rn * rn;
    int64_t tot = 0;
    for (int64_t i = 0; i < n; ++i) {
        offsets[i] = tot;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double d[3];
            orc_displacement(pos + 3 * i, pos + 3 * j, box, d);
            if (orc_r2(d) < rn2) {
                if (nbr) nbr[tot] = j;
                ++tot;
            }
        }
    }
    offsets[n] = tot;
    return tot;
}

/* ------------------------------------------------------------------ O4 -- */
/* Cell-list neighbour sets, Sec. 3.4: cells of side
 * Lambda >= rbar_c; n_c = floor(L / (rn*(1+1e-12))) >= 3, w = L/n_c,
 * cell = min(floor(x/w), n_c-1); scan the 27 periodic neighbour cells.
 * Input positions must already be wrapped into [0,L).  Returns the total
 * number of (i,j) entries, or -1 if a dimension has fewer than 3 cells.
 * Each NB(i) is returned in ascending j (reading R15). */
static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

int orc_cell_dims(const double box[3], double rn, int64_t nc[3])
{
    for (int d = 0; d < 3; ++d) {
        nc[d] = (int64_t)floor(box[d] / (rn * (1.0 + 1e-12)));
        if (nc[d] < 3) return -1;
    }
    return 0;
}

/* Linked-list cells (Rapaport): head[c] -> next[i]; cid[3i..3i+2] the cell of particle i. */
typedef struct {
    int64_t nc[3];
    int64_t *head, *next, *cid;
} orc_cells;

static void cells_build(int64_t n, const double *pos, const double box[3], const int64_t nc[3], orc_cells *C)
{
    double w[3] = {box[0] / (double)nc[0], box[1] / (double)nc[1], box[2] / (double)nc[2]};
    int64_t ncell = nc[0] * nc[1] * nc[2];
    for (int d = 0; d < 3; ++d) C->nc[d] = nc[d];
    C->head = (int64_t *)malloc(sizeof(int64_t) * ncell);
    C->next = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    C->cid = (int64_t *)malloc(sizeof(int64_t) * 3 * (n > 0 ? n : 1));
    for (int64_t c = 0; c < ncell; ++c) C->head[c] = -1;
    for (int64_t i = n - 1; i >= 0; --i) {
        int64_t c3[3];
        for (int d = 0; d < 3; ++d) {
            int64_t c = (int64_t)floor(pos[3 * i + d] / w[d]);
            if (c < 0) c = 0;
            if (c > nc[d] - 1) c = nc[d] - 1;
            c3[d] = c;
            C->cid[3 * i + d] = c;
        }
        int64_t c = (c3[2] * nc[1] + c3[1]) * nc[0] + c3[0];
        C->next[i] = C->head[c];
        C->head[c] = i;
    }
}

static void cells_free(orc_cells *C)
{
    free(C->head);
    free(C->next);
    free(C->cid);
}

/* NB(i) by the 27 periodic neighbour cells of i, into row[] ascending; returns |NB(i)|. */
static int64_t cells_row(int64_t i, const double *pos, const double box[3], double rn2, const orc_cells *C,
                         int64_t *row)
{
    const int64_t *nc = C->nc;
    int64_t cnt = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int64_t cx = (C->cid[3 * i + 0] + dx + nc[0]) % nc[0];
                int64_t cy = (C->cid[3 * i + 1] + dy + nc[1]) % nc[1];
                int64_t cz = (C->cid[3 * i + 2] + dz + nc[2]) % nc[2];
                int64_t c = (cz * nc[1] + cy) * nc[0] + cx;
                for (int64_t j = C->head[c]; j >= 0; j = C->next[j]) {
                    if (j == i) continue;
                    double d[3];
                    orc_displacement(pos + 3 * i, pos + 3 * j, box, d);
                    if (orc_r2(d) < rn2) row[cnt++] = j;
                }
            }
    qsort(row, (size_t)cnt, sizeof(int64_t), cmp_i64);
    return cnt;
}

/* Rows are independent, so the i loops may run in parallel (OpenMP build, bench.py's
 * all-core leg): every row is the same set in the same (ascending) order either way. */
int64_t orc_neigh_cells(int64_t n, const double *pos, const double box[3], double rn,
                        int64_t *offsets, int64_t *nbr)
{
    int64_t nc[3];
    if (orc_cell_dims(box, rn, nc) != 0) return -1;
    orc_cells C;
    cells_build(n, pos, box, nc, &C);
    double rn2 = rn * rn;
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
#pragma omp parallel
    {
        int64_t *row = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) cnt[i] = cells_row(i, pos, box, rn2, &C, row);
        free(row);
    }
    int64_t tot = 0;
    for (int64_t i = 0; i < n; ++i) {
        offsets[i] = tot;
        tot += cnt[i];
    }
    offsets[n] = tot;
    if (nbr) {
#pragma omp parallel
        {
            int64_t *row = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
#pragma omp for schedule(static)
            for (int64_t i = 0; i < n; ++i) {
                int64_t k = cells_row(i, pos, box, rn2, &C, row);
                for (int64_t q = 0; q < k; ++q) nbr[offsets[i] + q] = row[q];
            }
            free(row);
        }
    }
    free(cnt);
    cells_free(&C);
    return tot;
}

/* ------------------------------------------------------------------ O5 -- */
typedef struct {
    double rc;      /* force cutoff r_c (Tab. 7.2T1: 2.5)                      */
    double eps;     /* epsilon                                                 */
    double sigma;   /* sigma                                                   */
    double shift;   /* s in 4 eps [(sigma/r)^12 - (sigma/r)^6 + s]; 1/4 in the
                       paper's Eq. eqn:LJpotential, reading R3          */
} orc_lj;

/* One ordered pair, Listing lst:LJ-kernel with
 * C_F = +48 eps / sigma^2 (Eq. eqn:LJforce, reading R1), C_V = 4 eps.
 * Contributions are added only if r^2 < r_c^2 (strict, reading R4). */
static void pair_accumulate(const double d[3], const orc_lj *lj, double *Fi, double *Ui,
                            double *Si, double *Ai)
{
    double rc_sq = lj->rc * lj->rc;
    double sigma2 = lj->sigma * lj->sigma;
    double CV = 4.0 * lj->eps;
    double CF = 48.0 * lj->eps / sigma2;
    double dr_sq = orc_r2(d);
    if (!(dr_sq < rc_sq)) return;
    double r_m2 = sigma2 / dr_sq;
    double r_m4 = r_m2 * r_m2;
    double r_m6 = r_m4 * r_m2;
    double r_m8 = r_m4 * r_m4;
    double u = CV * ((r_m6 - 1.0) * r_m6 + lj->shift);
    double f_tmp = CF * (r_m6 - 0.5) * r_m8;
    Fi[0] += f_tmp * d[0];
    Fi[1] += f_tmp * d[1];
    Fi[2] += f_tmp * d[2];
    *Ui += u;
    *Si += fabs(f_tmp) * sqrt(dr_sq);
    *Ai += fabs(u);
}

/* Neumaier-compensated sum (used for global PE and KE). */
double orc_sum(const double *x, int64_t n)
{
    double s = 0.0, c = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double t = s + x[i];
        if (fabs(s) >= fabs(x[i])) c += (s - t) + x[i];
        else c += (x[i] - t) + s;
        s = t;
    }
    return s + c;
}

/* F[n][3] (INC_ZERO: zeroed first, reading R5), e[n] = 1/2 sum_j V (R2),
 * S[n] = sum_j |f_ij| (tolerance scale, reading R16), A[n] = sum_j |V_ij|.
 * Any of e/S/A may be NULL.  If offsets == NULL: brute force over all j in
 * ascending order; else over NB(i) = nbr[offsets[i]..offsets[i+1]).
 * Returns PE = sum_i e_i (Neumaier). */
double orc_forces(int64_t n, const double *pos, const double box[3], const orc_lj *lj,
                  const int64_t *offsets, const int64_t *nbr,
                  double *F, double *e, double *S, double *A)
{
    double *etmp = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double Fi[3] = {0.0, 0.0, 0.0}, Ui = 0.0, Si = 0.0, Ai = 0.0;
        if (offsets == NULL) {
            for (int64_t j = 0; j < n; ++j) {
                if (j == i) continue;
                double d[3];
                orc_displacement(pos + 3 * i, pos + 3 * j, box, d);
                pair_accumulate(d, lj, Fi, &Ui, &Si, &Ai);
            }
        } else {
            for (int64_t k = offsets[i]; k < offsets[i + 1]; ++k) {
                double d[3];
                orc_displacement(pos + 3 * i, pos + 3 * nbr[k], box, d);
                pair_accumulate(d, lj, Fi, &Ui, &Si, &Ai);
            }
        }
        F[3 * i + 0] = Fi[0];
        F[3 * i + 1] = Fi[1];
        F[3 * i + 2] = Fi[2];
        etmp[i] = 0.5 * Ui;
        if (e) e[i] = etmp[i];
        if (S) S[i] = Si;
        if (A) A[i] = Ai;
    }
    double pe = orc_sum(etmp, n);
    free(etmp);
    return pe;
}

/* KE = 1/2 m sum_i |v_i|^2 (Example 1), Neumaier over particles. */
double orc_kinetic(int64_t n, const double *vel, double mass)
{
    double *k = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        const double *v = vel + 3 * i;
        k[i] = 0.5 * mass * ((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    }
    double ke = orc_sum(k, n);
    free(k);
    return ke;
}

/* ------------------------------------------------------- row-sampled O3/O5 -- */
/* Brute force restricted to the rows i in idx[0..m): used to check full-size runs
 * on sampled particles (same arithmetic as orc_neigh_brute / orc_forces, all j
 * ascending).  nbr rows are returned CSR in offsets[m+1]. */
int64_t orc_neigh_rows(int64_t n, const double *pos, const double box[3], double rn,
                       const int64_t *idx, int64_t m, int64_t *offsets, int64_t *nbr)
{
    double rn2 = rn * rn;
    int64_t tot = 0;
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = idx[r];
        offsets[r] = tot;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double d[3];
            orc_displacement(pos + 3 * i, pos + 3 * j, box, d);
            if (orc_r2(d) < rn2) {
                if (nbr) nbr[tot] = j;
                ++tot;
            }
        }
    }
    offsets[m] = tot;
    return tot;
}

void orc_forces_rows(int64_t n, const double *pos, const double box[3], const orc_lj *lj,
                     const int64_t *idx, int64_t m, double *F, double *e, double *S, double *A)
{
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = idx[r];
        double Fi[3] = {0.0, 0.0, 0.0}, Ui = 0.0, Si = 0.0, Ai = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double d[3];
            orc_displacement(pos + 3 * i, pos + 3 * j, box, d);
            pair_accumulate(d, lj, Fi, &Ui, &Si, &Ai);
        }
        F[3 * r + 0] = Fi[0];
        F[3 * r + 1] = Fi[1];
        F[3 * r + 2] = Fi[2];
        e[r] = 0.5 * Ui;
        S[r] = Si;
        A[r] = Ai;
    }
}

/* ------------------------------------------------------------- O6 / O7 -- */
/* ------------------------------------------------------------------ O8 -- */
/* Philox4x32-10: 10 rounds of two 32x32->64 multiplies and a Weyl key schedule. */
void orc_philox4x32(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 53-bit uniform in [0, 1) from two words (a supplies 27 bits, b 26). */
static double u53(uint32_t a, uint32_t b)
{
    return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

/* Reading R19: draws of particle gid at step `step` (1-based, the step being completed).
 * Block k = 0: (w0, w1) -> decision uniform, (w2, w3) -> U1; k = 1: U2, U3; k = 2: U4.
 * Selected iff decision < nu*dt; then, Box-Muller,
 *   v = sqrt(T/m) (R1 cos(2 pi U2), R1 sin(2 pi U2), R2 cos(2 pi U4)),
 *   R1 = sqrt(-2 ln(1 - U1)), R2 = sqrt(-2 ln(1 - U3)).  Returns 1 if selected. */
int orc_andersen_draw(uint64_t seed, int64_t gid, int64_t step, double nu_dt, double sd, double v[3])
{
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {(uint32_t)gid, (uint32_t)step, (uint32_t)((uint64_t)step >> 32), 0u};
    uint32_t w[4], w1[4], w2[4];
    orc_philox4x32(ctr, key, w);
    if (!(u53(w[0], w[1]) < nu_dt)) return 0;
    ctr[3] = 1u;
    orc_philox4x32(ctr, key, w1);
    ctr[3] = 2u;
    orc_philox4x32(ctr, key, w2);
    double U1 = u53(w[2], w[3]), U2 = u53(w1[0], w1[1]), U3 = u53(w1[2], w1[3]), U4 = u53(w2[0], w2[1]);
    const double two_pi = 6.283185307179586;
    double R1 = sqrt(-2.0 * log(1.0 - U1)), R2 = sqrt(-2.0 * log(1.0 - U3));
    v[0] = sd * (R1 * cos(two_pi * U2));
    v[1] = sd * (R1 * sin(two_pi * U2));
    v[2] = sd * (R2 * cos(two_pi * U4));
    return 1;
}

/* One thermostat pass over all particles (gid = row); returns the number resampled. */
int64_t orc_andersen(int64_t n, double *vel, uint64_t seed, int64_t step, double nu_dt, double temp,
                     double mass)
{
    double sd = sqrt(temp / mass);
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) {
        double v[3];
        if (orc_andersen_draw(seed, i, step, nu_dt, sd, v)) {
            vel[3 * i] = v[0];
            vel[3 * i + 1] = v[1];
            vel[3 * i + 2] = v[2];
            ++k;
        }
    }
    return k;
}

typedef struct {
    orc_lj lj;
    double dt;            /* delta t                                           */
    double mass;          /* scalar m (reading R11)                            */
    double delta;         /* shell thickness delta = rbar_c - r_c  */
    int64_t ns;           /* reuse count Ns (20)                        */
    int64_t check;        /* 1: also rebuild when 2 max|x - x_build| > delta   */
    int64_t mode;         /* 0: brute-force forces, 1: cell + neighbour list   */
    int64_t energy_every; /* sample PE/KE every k steps (10)            */
    double nu_dt;         /* Andersen collision probability per step (0: NVE)  */
    double temp;          /* Andersen target temperature T (k_B = 1)           */
    uint64_t seed;        /* Philox key                                        */
} orc_params;

typedef struct {
    int64_t *off, *nbr;
} orc_list;

/* O4 into a fresh CSR: rows counted, then filled (the same rows as orc_neigh_cells). */
static int build_list(int64_t n, const double *pos, const double box[3], double rn, orc_list *L)
{
    int64_t nc[3];
    if (orc_cell_dims(box, rn, nc) != 0) return -1;
    free(L->off);
    free(L->nbr);
    L->off = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    orc_cells C;
    cells_build(n, pos, box, nc, &C);
    double rn2 = rn * rn;
    int64_t **rows = (int64_t **)malloc(sizeof(int64_t *) * (n > 0 ? n : 1));
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
#pragma omp parallel
    {
        int64_t *row = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            cnt[i] = cells_row(i, pos, box, rn2, &C, row);
            rows[i] = (int64_t *)malloc(sizeof(int64_t) * (cnt[i] > 0 ? cnt[i] : 1));
            memcpy(rows[i], row, sizeof(int64_t) * cnt[i]);
        }
        free(row);
    }
    int64_t tot = 0;
    for (int64_t i = 0; i < n; ++i) {
        L->off[i] = tot;
        tot += cnt[i];
    }
    L->off[n] = tot;
    L->nbr = (int64_t *)malloc(sizeof(int64_t) * (tot > 0 ? tot : 1));
    for (int64_t i = 0; i < n; ++i) {
        memcpy(L->nbr + L->off[i], rows[i], sizeof(int64_t) * cnt[i]);
        free(rows[i]);
    }
    free(rows);
    free(cnt);
    cells_free(&C);
    return 0;
}

/* Missed pairs of a Verlet list at positions pos (validation; Eq. eqn:extended_cutoff,
 * PAPER.md:406-416): for every i, #{j != i : r_ij^2 < rc^2} by brute force (O2 minimum
 * image, as O3) minus #{j in NB(i) : r_ij^2 < rc^2}.  *particles = #{i : difference > 0},
 * *pairs = the summed difference (ordered pairs the list does not serve). */
void orc_missed(int64_t n, const double *pos, const double box[3], double rc, const int64_t *offsets,
                const int64_t *nbr, int64_t *particles, int64_t *pairs)
{
    double rc2 = rc * rc;
    int64_t np = 0, nm = 0;
#pragma omp parallel for schedule(static) reduction(+ : np, nm)
    for (int64_t i = 0; i < n; ++i) {
        int64_t truth = 0, listed = 0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double d[3];
            orc_displacement(pos + 3 * i, pos + 3 * j, box, d);
            if (orc_r2(d) < rc2) ++truth;
        }
        for (int64_t k = offsets[i]; k < offsets[i + 1]; ++k) {
            double d[3];
            orc_displacement(pos + 3 * i, pos + 3 * nbr[k], box, d);
            if (orc_r2(d) < rc2) ++listed;
        }
        if (truth > listed) {
            ++np;
            nm += truth - listed;
        }
    }
    *particles = np;
    *pairs = nm;
}

/* Velocity Verlet, Algorithm alg:VelocityVerlet:
 *   init : wrap (O1), build list, F <- F(r0) (reading R6), sample 0
 *   step : v += (dt/2m) F ; r += dt v          (line 6, Listing P:659-666)
 *          rebuild if due: wrap + list (O7, after the drift, reading R8)
 *          F <- INC_ZERO pair loop              (line 7)
 *          v += (dt/2m) F                       (line 8, Listing P:671-675)
 *          sample PE, KE every energy_every steps
 * Positions are wrapped only when the cell/neighbour structure is rebuilt
 * (Listing lst:position_update has no wrap; migration happens every n steps,
 * P:436-438; reading R10).  In brute-force mode the same schedule decides
 * when to wrap, so brute and list trajectories are bitwise identical while
 * no pair enters r_c from beyond rbar_c between rebuilds.
 *
 * pe_hist/ke_hist: nsteps/energy_every + 1 entries.  rebuild_steps: the MD
 * step index of each rebuild after init (cap entries).  missed_particles /
 * missed_pairs (NULL: off; nsteps + 1 entries, index = step): orc_missed at the
 * positions each force of the step is evaluated on (list mode).  Returns the
 * number of rebuilds, or -1 on error (box too small for cells). */
int64_t orc_run(int64_t n, double *pos, double *vel, const double box[3], const orc_params *p,
                int64_t nsteps, double *F, double *pe_hist, double *ke_hist,
                int64_t *rebuild_steps, int64_t rebuild_cap, int64_t *missed_particles,
                int64_t *missed_pairs)
{
    double h = 0.5 * p->dt / p->mass;       /* dht_iMASS = dt/(2m) */
    double rn = p->lj.rc + p->delta;
    orc_list L = {NULL, NULL};
    double *xb = (double *)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
    int64_t nreb = 0;

    orc_wrap(n, pos, box);
    if (p->mode == 1 && build_list(n, pos, box, rn, &L) != 0) { free(xb); return -1; }
    memcpy(xb, pos, sizeof(double) * 3 * n);
    double pe = orc_forces(n, pos, box, &p->lj, p->mode == 1 ? L.off : NULL, L.nbr, F, NULL, NULL, NULL);
    int64_t ks = 0;
    if (pe_hist) pe_hist[ks] = pe;
    if (ke_hist) ke_hist[ks] = orc_kinetic(n, vel, p->mass);
    ++ks;
    int64_t since = 0;
    for (int64_t step = 1; step <= nsteps; ++step) {
        for (int64_t i = 0; i < 3 * n; ++i) {
            vel[i] = vel[i] + h * F[i];
            pos[i] = pos[i] + p->dt * vel[i];
        }
        ++since;
        int due = (since >= p->ns);
        if (!due && p->check) {
            double m = 0.0;
            for (int64_t i = 0; i < n; ++i) {
                double d[3] = {pos[3 * i] - xb[3 * i], pos[3 * i + 1] - xb[3 * i + 1],
                               pos[3 * i + 2] - xb[3 * i + 2]};
                double r2 = orc_r2(d);
                if (r2 > m) m = r2;
            }
            due = (4.0 * m > p->delta * p->delta);
        }
        if (due) {
            orc_wrap(n, pos, box);
            if (p->mode == 1 && build_list(n, pos, box, rn, &L) != 0) { free(xb); return -1; }
            memcpy(xb, pos, sizeof(double) * 3 * n);
            if (rebuild_steps && nreb < rebuild_cap) rebuild_steps[nreb] = step;
            ++nreb;
            since = 0;
        }
        if (missed_particles && missed_pairs && p->mode == 1)   /* validation, before line 7 */
            orc_missed(n, pos, box, p->lj.rc, L.off, L.nbr, missed_particles + step, missed_pairs + step);
        pe = orc_forces(n, pos, box, &p->lj, p->mode == 1 ? L.off : NULL, L.nbr, F, NULL, NULL, NULL);
        for (int64_t i = 0; i < 3 * n; ++i) vel[i] = vel[i] + h * F[i];
        if (p->nu_dt > 0.0) orc_andersen(n, vel, p->seed, step, p->nu_dt, p->temp, p->mass);
        if (p->energy_every > 0 && step % p->energy_every == 0) {
            if (pe_hist) pe_hist[ks] = pe;
            if (ke_hist) ke_hist[ks] = orc_kinetic(n, vel, p->mass);
            ++ks;
        }
    }
    free(L.off);
    free(L.nbr);
    free(xb);
    return nreb;
}
