/*
 * lbm_oracle.c -- plain, slow, obviously-correct CPU oracle of the D3Q19 LBGK
 * pull stream-collide update with half-way bounce-back (no-slip and moving
 * wall), written from the paper (Feichtinger et al., arXiv:1007.1388).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1007_1388_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant with the CUDA path.
 *
 * Citations: P:n = /root/reference/PAPER.md line n.
 *   P:403-405   D3Q19, 19 PDFs per cell
 *   P:407-415   eq:lbm   f_i(x+e_i,t+1) = f_i - (1/tau)[f_i - f_i^eq]
 *   P:416-425   eq:feq   f_i^eq = w_i[rho + rho0(3 e.u + 4.5 (e.u)^2 - 1.5 u^2)]
 *   P:441-442   w_i in {1/3, 1/18, 1/36}
 *   P:443-448   rho = rho0 + drho = sum f_i ;  rho0 u = sum e_i f_i
 *   P:452-464   centred PDFs  f~_i = f_i - f_i^eq(rho0, 0) = f_i - w_i rho0
 *   P:466-480   pull streaming, two PDF grids
 *   P:482-490   half-way bounce-back  f_ibar(x,t+1) = f_i(x,t) + 6 w_i rho0 e_i.u_w
 *
 * Readings of the paper taken here:
 *   R1  i = 0..18 (P:426 says 0..19; P:445 sums to 18).
 *   R2  direction order: the frozen table below (paper is silent).
 *   R3  BB correction uses the DELIVERED direction i (wall -> fluid):
 *         p_i(x) = f~_opp(i)(x) + 6 w_i rho0 (e_i . u_w)
 *   R4  rho0 = 1.   R5  c_s^2 = 1/3 (implied by 3 / 4.5 / 1.5).
 *   R6  one step = pull (+BB) -> collide -> store at x; the stored array is
 *       the post-collision state at its own cell.
 *   R7  u = (sum e_i f~_i) / rho0  (incompressible), not / rho.
 *   R8  f^eq uses the full rho = rho0 + drho: f~eq_i = w_i[drho + rho0(..)].
 *   R9  rho0 (not local rho) in the BB term, as written at P:488.
 *   R10 walls are non-fluid cells; the domain boundary is a one-cell shell.
 *   R13 non-fluid cells are never read as a source and never updated
 *       (this oracle copies them through unchanged; comparisons skip them).
 *   R14 IEEE round-to-nearest; sums in direction order 0..18; no FMA
 *       contraction (built with -ffp-contract=off).
 *
 * Layouts (all caller-owned, never retained):
 *   flags  uint8 [(nz+2)][(ny+2)][(nx+2)], x fastest, includes the shell.
 *          0 = fluid, 1 = no-slip wall, 2+k = wall moving with wall_u[k].
 *   f      double [nz][ny][nx][19] (interior cells only, centred f~).
 *   Periodic axes wrap the neighbour index; their shell flags are unused.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define Q 19

/* Frozen D3Q19 table (R2): rest, 6 faces, 12 edges; opposite pairs i, i+1. */
static const int E[Q][3] = {
    {0, 0, 0},
    {1, 0, 0},   {-1, 0, 0},
    {0, 1, 0},   {0, -1, 0},
    {0, 0, 1},   {0, 0, -1},
    {1, 1, 0},   {-1, -1, 0},
    {1, -1, 0},  {-1, 1, 0},
    {1, 0, 1},   {-1, 0, -1},
    {1, 0, -1},  {-1, 0, 1},
    {0, 1, 1},   {0, -1, -1},
    {0, 1, -1},  {0, -1, 1},
};
static const double W[Q] = {
    1.0 / 3.0,
    1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0,
    1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
    1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
};
static const int OPP[Q] = {0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17};

static const double RHO0 = 1.0; /* R4 */

int lbm_oracle_version(void) { return 1; }

void lbm_oracle_table(int *e, double *w, int *opp)
{
    for (int i = 0; i < Q; ++i) {
        for (int a = 0; a < 3; ++a) e[3 * i + a] = E[i][a];
        w[i] = W[i];
        opp[i] = OPP[i];
    }
}

/* eq:feq centred:
 *   f~eq_i = w_i [ drho + rho0 (3 e_i.u + 4.5 (e_i.u)^2 - 1.5 u.u) ]       */
void lbm_oracle_equilibrium(double drho, const double *u, double *feq)
{
    double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    for (int i = 0; i < Q; ++i) {
        double eu = E[i][0] * u[0] + E[i][1] * u[1] + E[i][2] * u[2];
        feq[i] = W[i] * (drho + RHO0 * (3.0 * eu + 4.5 * eu * eu - 1.5 * usq));
    }
}

/* Moments: drho = sum f~_i ; u = (sum e_i f~_i) / rho0 (R7). */
void lbm_oracle_cell_moments(const double *f, double *drho, double *u)
{
    double s = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
    for (int i = 0; i < Q; ++i) {
        s += f[i];
        jx += E[i][0] * f[i];
        jy += E[i][1] * f[i];
        jz += E[i][2] * f[i];
    }
    *drho = s;
    u[0] = jx / RHO0;
    u[1] = jy / RHO0;
    u[2] = jz / RHO0;
}

/* BGK collision (eq:lbm) of the pulled values p at one cell. */
void lbm_oracle_collide(const double *p, double omega, double *out)
{
    double drho, u[3], feq[Q];
    lbm_oracle_cell_moments(p, &drho, u);
    lbm_oracle_equilibrium(drho, u, feq);
    for (int i = 0; i < Q; ++i) out[i] = p[i] - omega * (p[i] - feq[i]);
}

static int wrap(int c, int n, int periodic)
{
    if (!periodic) return c; /* -1 or n: the shell */
    if (c < 0) return c + n;
    if (c >= n) return c - n;
    return c;
}

/* Validate flags: shell cells on non-periodic axes must be non-fluid and
 * every velocity-wall index must be < nvel.  Returns 0 on success.        */
int lbm_oracle_check_flags(int nx, int ny, int nz, const int *periodic, const uint8_t *flags, int nvel)
{
    int n[3] = {nx, ny, nz};
    for (int z = -1; z <= nz; ++z)
        for (int y = -1; y <= ny; ++y)
            for (int x = -1; x <= nx; ++x) {
                int c[3] = {x, y, z};
                uint8_t fl = flags[((size_t)(z + 1) * (ny + 2) + (y + 1)) * (nx + 2) + (x + 1)];
                int shell = 0;
                for (int a = 0; a < 3; ++a)
                    if (!periodic[a] && (c[a] < 0 || c[a] >= n[a])) shell = 1;
                if (shell && fl == 0) return 1;
                if (fl >= 2 && fl - 2 >= nvel) return 2;
            }
    return 0;
}

/* One time step over interior z-planes [z0, z1): for every fluid cell x
 *   pull  p_i = src_i(x - e_i)                        if x - e_i is fluid
 *         p_i = src_opp(i)(x)                         if no-slip wall
 *         p_i = src_opp(i)(x) + 6 w_i rho0 e_i.u_w    if moving wall (R3)
 *   collide dst_i(x) = p_i - omega (p_i - f~eq_i(drho(p), u(p)))
 * Non-fluid interior cells are copied through.  src and dst are distinct
 * [nz][ny][nx][19] arrays.                                                 */
void lbm_oracle_step(int nx, int ny, int nz, const int *periodic, const uint8_t *flags,
                     const double *wall_u, int nvel, double omega, const double *src, double *dst,
                     int z0, int z1, int nthreads)
{
    (void)nvel;
    const size_t fy = (size_t)nx + 2, fz = (size_t)(nx + 2) * (ny + 2);
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
#else
    (void)nthreads;
#endif
    for (int z = z0; z < z1; ++z) {
        for (int y = 0; y < ny; ++y) {
            for (int x = 0; x < nx; ++x) {
                size_t cell = ((size_t)z * ny + y) * nx + x;
                uint8_t own = flags[(size_t)(z + 1) * fz + (size_t)(y + 1) * fy + (x + 1)];
                if (own != 0) {
                    memcpy(&dst[cell * Q], &src[cell * Q], Q * sizeof(double));
                    continue;
                }
                double p[Q];
                for (int i = 0; i < Q; ++i) {
                    int sx = wrap(x - E[i][0], nx, periodic[0]);
                    int sy = wrap(y - E[i][1], ny, periodic[1]);
                    int sz = wrap(z - E[i][2], nz, periodic[2]);
                    uint8_t nb = flags[(size_t)(sz + 1) * fz + (size_t)(sy + 1) * fy + (sx + 1)];
                    if (nb == 0) {
                        size_t ncell = ((size_t)sz * ny + sy) * nx + sx;
                        p[i] = src[ncell * Q + i];
                    } else if (nb == 1) {
                        p[i] = src[cell * Q + OPP[i]];
                    } else {
                        const double *uw = &wall_u[3 * (nb - 2)];
                        double eu = E[i][0] * uw[0] + E[i][1] * uw[1] + E[i][2] * uw[2];
                        p[i] = src[cell * Q + OPP[i]] + 6.0 * W[i] * RHO0 * eu;
                    }
                }
                lbm_oracle_collide(p, omega, &dst[cell * Q]);
            }
        }
    }
}

/* nsteps full time steps, two grids, f in/out ([nz][ny][nx][19]).
 * Returns 0, or 1 on invalid flags, 3 on allocation failure.              */
int lbm_oracle_run(int nx, int ny, int nz, const int *periodic, const uint8_t *flags,
                   const double *wall_u, int nvel, double omega, int nsteps, double *f, int nthreads)
{
    if (lbm_oracle_check_flags(nx, ny, nz, periodic, flags, nvel)) return 1;
    size_t n = (size_t)nx * ny * nz * Q;
    double *tmp = (double *)malloc(n * sizeof(double));
    if (!tmp) return 3;
    double *a = f, *b = tmp;
    for (int t = 0; t < nsteps; ++t) {
        lbm_oracle_step(nx, ny, nz, periodic, flags, wall_u, nvel, omega, a, b, 0, nz, nthreads);
        double *s = a; a = b; b = s;
    }
    if (a != f) memcpy(f, a, n * sizeof(double));
    free(tmp);
    return 0;
}

/* Macroscopic export: rho = rho0 + sum f~_i, u = sum e_i f~_i / rho0
 * at fluid cells; rho = 0, u = 0 at non-fluid cells (R13 convention).       */
void lbm_oracle_macroscopic(int nx, int ny, int nz, const uint8_t *flags, const double *f,
                            double *rho, double *u)
{
    const size_t fy = (size_t)nx + 2, fz = (size_t)(nx + 2) * (ny + 2);
    for (int z = 0; z < nz; ++z)
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) {
                size_t cell = ((size_t)z * ny + y) * nx + x;
                if (flags[(size_t)(z + 1) * fz + (size_t)(y + 1) * fy + (x + 1)] != 0) {
                    rho[cell] = 0.0;
                    u[3 * cell] = u[3 * cell + 1] = u[3 * cell + 2] = 0.0;
                    continue;
                }
                double drho;
                lbm_oracle_cell_moments(&f[cell * Q], &drho, &u[3 * cell]);
                rho[cell] = RHO0 + drho;
            }
}

int lbm_oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
