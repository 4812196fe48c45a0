/*
 * lb_oracle.c -- CPU restatement of the reference hot path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py, never by the product
 * package (paper_1405_6162_b200/).
 *
 * Compile with -ffp-contract=off (see oracle/Makefile): every operation is one
 * IEEE binary64 round-to-nearest op in the order written, exactly like the
 * reference numba kernel, which emits scalar vaddsd/vmulsd/vdivsd and no FMA
 * (SURVEY.md Appendix B).
 *
 * Part 1 (PINNED against the reference): orc_collide restates
 *   reference pkg/src/latkit/kernels.py:89-125 (_collision_range)
 * with the op order of the site ops kernels.py:29-73; orc_scale restates
 *   kernels.py:79-86; orc_masked_copy restates oracle.py:62-68.
 * Golden vectors from the reference itself (tests/golden/) pin these bitwise.
 *
 * Part 2 (builder-defined, NOT in the reference -> "parity unpinned" w.r.t. the
 * reference, pinned only by known-answer tests): pull streaming, the
 * order-parameter moment, the chemical-potential stencil and the forced
 * binary-fluid collision of SURVEY.md Appendix C.  Host site order follows the
 * reference oracle, s = (x*ny + y)*nz + z (reference oracle.py:42-45).
 * The exact formulas and op order are written out in DESIGN.md §2.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define Q 19

/* Host threads used by the parallel loops below (CPU baseline legs). */
void orc_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* D3Q19 velocity table in the reference ordering (model.py:21-34). */
static const int CV[Q][3] = {
    {0, 0, 0},
    {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1},
    {1, 1, 0}, {1, -1, 0}, {-1, 1, 0}, {-1, -1, 0},
    {1, 0, 1}, {1, 0, -1}, {-1, 0, 1}, {-1, 0, -1},
    {0, 1, 1}, {0, 1, -1}, {0, -1, 1}, {0, -1, -1}};

/* ---------------------------------------------------------------- part 1 */

/* Reference kernels.py:89-125 for sites [site_lo, site_hi).  cv is a float64
 * (19,3) table as passed by _collision_prepare (kernels.py:151-173).
 * Returns the first real site with rho <= 0 (the reference raises
 * SingularStateError there, kernels.py:106-108) or -1.  Like the reference,
 * processing stops at that site. */
int64_t orc_collide(double *f, double *g, int64_t padded, int64_t nsites,
                    const double *wv, const double *cv, double cs2,
                    double tau_f, double tau_g, int64_t site_lo, int64_t site_hi)
{
    for (int64_t s = site_lo; s < site_hi; ++s) {
        double rho = 0.0, fx = 0.0, fy = 0.0, fz = 0.0;
        for (int i = 0; i < Q; ++i) {
            double fi = f[i * padded + s];
            rho += fi;
            fx += fi * cv[3 * i + 0];
            fy += fi * cv[3 * i + 1];
            fz += fi * cv[3 * i + 2];
        }
        if (rho <= 0.0) {
            if (s < nsites) return s;
            continue; /* zero padding: untouched */
        }
        double ux = fx / rho, uy = fy / rho, uz = fz / rho;
        double phi = 0.0;
        for (int i = 0; i < Q; ++i) phi += g[i * padded + s];
        double usq = ux * ux + uy * uy + uz * uz;
        for (int i = 0; i < Q; ++i) {
            double udotc = ux * cv[3 * i] + uy * cv[3 * i + 1] + uz * cv[3 * i + 2];
            double bracket = 1.0 + udotc / cs2 + (udotc * udotc) / (2.0 * cs2 * cs2)
                             - usq / (2.0 * cs2);
            double feq = wv[i] * rho * bracket;
            double geq = wv[i] * phi * bracket;
            int64_t idx = i * padded + s;
            f[idx] = f[idx] - (f[idx] - feq) / tau_f;
            g[idx] = g[idx] - (g[idx] - geq) / tau_g;
        }
    }
    return -1;
}

/* Multi-threaded driver of orc_collide over [0, extent) -- used only as the
 * CPU baseline (bench.py cpu_baseline / --impl reference).  Chunks are
 * disjoint, so the result equals the sequential call bitwise. */
int64_t orc_collide_parallel(double *f, double *g, int64_t padded, int64_t nsites,
                             const double *wv, const double *cv, double cs2,
                             double tau_f, double tau_g, int64_t extent, int nthreads)
{
    int64_t bad = -1;
    int64_t nchunk = (extent + 4095) / 4096;
#pragma omp parallel for schedule(static) num_threads(nthreads) reduction(max : bad)
    for (int64_t c = 0; c < nchunk; ++c) {
        int64_t lo = c * 4096, hi = lo + 4096 < extent ? lo + 4096 : extent;
        int64_t r = orc_collide(f, g, padded, nsites, wv, cv, cs2, tau_f, tau_g, lo, hi);
        if (r > bad) bad = r;
    }
    return bad;
}

/* Reference kernels.py:79-86 / oracle.py:18-25: field[c*P+s] = a*field[c*P+s], c<3. */
void orc_scale(double *field, int64_t padded, double a, int64_t site_lo, int64_t site_hi)
{
    for (int c = 0; c < 3; ++c)
        for (int64_t s = site_lo; s < site_hi; ++s)
            field[c * padded + s] = a * field[c * padded + s];
}

/* Reference oracle.py:62-68: element-by-element masked copy. */
void orc_masked_copy(double *dst, const double *src, int ncomp, int64_t padded,
                     const uint8_t *flags, int64_t nsites)
{
    for (int c = 0; c < ncomp; ++c)
        for (int64_t s = 0; s < nsites; ++s)
            if (flags[s]) dst[c * padded + s] = src[c * padded + s];
}

/* ---------------------------------------------------------------- part 2 */

/* Parameter block of the full timestep.  lam[i] are the
 * chemical-potential weights of g_eq, lam_i = w_i/cs2 (i>0),
 * lam_0 = -(1-w_0)/cs2, computed once on the host. */
typedef struct {
    double wv[Q];
    double lam[Q];
    double cs2, tau_f, tau_g;
    double A, B, kappa, gamma;
    int32_t physics; /* 0 = passive (reference collision), 1 = free-energy binary fluid
                      * with the potential force -phi grad(mu), filtered along its own
                      * axis (orc_potential_force), 2 = same fluid with the
                      * momentum-conserving force F = -div P (chemical pressure tensor) */
    int32_t pad_;
} orc_fluid_params;

static inline int64_t site_of(int64_t x, int64_t y, int64_t z, int64_t ny, int64_t nz)
{
    return (x * ny + y) * nz + z;
}

static inline int64_t wrap(int64_t v, int64_t n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

/* Pull streaming: out_i(x) = in_i(x - c_i), periodic; padding untouched. */
void orc_stream(const double *in, double *out, int ncomp, int64_t padded,
                int64_t nx, int64_t ny, int64_t nz)
{
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < nx; ++x)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t z = 0; z < nz; ++z) {
                int64_t s = site_of(x, y, z, ny, nz);
                for (int i = 0; i < ncomp; ++i) {
                    int64_t src = site_of(wrap(x - CV[i][0], nx), wrap(y - CV[i][1], ny),
                                          wrap(z - CV[i][2], nz), ny, nz);
                    out[i * padded + s] = in[i * padded + src];
                }
            }
}

/* Order parameter of the streamed g: phi = sum_i g_i in index order. */
void orc_phi(const double *g, double *phi, int64_t padded, int64_t nsites)
{
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < nsites; ++s) {
        double p = 0.0;
        for (int i = 0; i < Q; ++i) p += g[i * padded + s];
        phi[s] = p;
    }
}

/* mu = A phi + B phi^3 - kappa lap(phi), 7-point Laplacian, periodic. */
void orc_mu(const double *phi, double *mu, int64_t nx, int64_t ny, int64_t nz,
            double A, double B, double kappa)
{
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < nx; ++x)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t z = 0; z < nz; ++z) {
                double p = phi[site_of(x, y, z, ny, nz)];
                double sum = phi[site_of(wrap(x + 1, nx), y, z, ny, nz)];
                sum += phi[site_of(wrap(x - 1, nx), y, z, ny, nz)];
                sum += phi[site_of(x, wrap(y + 1, ny), z, ny, nz)];
                sum += phi[site_of(x, wrap(y - 1, ny), z, ny, nz)];
                sum += phi[site_of(x, y, wrap(z + 1, nz), ny, nz)];
                sum += phi[site_of(x, y, wrap(z - 1, nz), ny, nz)];
                double lap = sum - 6.0 * p;
                double p3 = (p * p) * p;
                mu[site_of(x, y, z, ny, nz)] = (A * p + B * p3) - kappa * lap;
            }
}

/* Chemical pressure tensor of the symmetric free energy (physics 2):
 *   P_ab = p_iso delta_ab + kappa d_a phi d_b phi,
 *   p_iso = (phi mu - (A/2 phi^2 + B/4 phi^4)) - kappa/2 |grad phi|^2,
 * so that div P = phi grad mu in the continuum.  Per site this writes p_iso and
 * the central gradient (gx, gy, gz) of phi; mu must be orc_mu's.  Op order:
 *   g_a = (phi(+a) - phi(-a)) * 0.5,  gsq = ((gx gx) + (gy gy)) + (gz gz),
 *   pp = phi phi,  fb = ((0.5 A) pp) + ((0.25 B) (pp pp)),
 *   p_iso = ((phi mu) - fb) - ((0.5 kappa) gsq). */
void orc_stress(const double *phi, const double *mu, double *piso, double *gx, double *gy,
                double *gz, int64_t nx, int64_t ny, int64_t nz, double A, double B, double kappa)
{
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < nx; ++x)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t z = 0; z < nz; ++z) {
                const int64_t s = site_of(x, y, z, ny, nz);
                const double p = phi[s];
                const double ax = (phi[site_of(wrap(x + 1, nx), y, z, ny, nz)] -
                                   phi[site_of(wrap(x - 1, nx), y, z, ny, nz)]) * 0.5;
                const double ay = (phi[site_of(x, wrap(y + 1, ny), z, ny, nz)] -
                                   phi[site_of(x, wrap(y - 1, ny), z, ny, nz)]) * 0.5;
                const double az = (phi[site_of(x, y, wrap(z + 1, nz), ny, nz)] -
                                   phi[site_of(x, y, wrap(z - 1, nz), ny, nz)]) * 0.5;
                const double gsq = ((ax * ax) + (ay * ay)) + (az * az);
                const double pp = p * p;
                const double fb = ((0.5 * A) * pp) + ((0.25 * B) * (pp * pp));
                piso[s] = ((p * mu[s]) - fb) - ((0.5 * kappa) * gsq);
                gx[s] = ax;
                gy[s] = ay;
                gz[s] = az;
            }
}

/* F_a = -((D_x P_ax + D_y P_ay) + D_z P_az) at site (x, y, z), D_b h =
 * (h(+b) - h(-b)) * 0.5, P_aa = p_iso + ((kappa g_a) g_a), P_ab = (kappa g_a) g_b:
 * a discrete divergence, so sum_x F = 0 up to rounding (momentum conserved). */
static void stress_force(const double *piso, const double *const g[3], double kappa, int64_t x,
                         int64_t y, int64_t z, int64_t nx, int64_t ny, int64_t nz, double F[3])
{
    int64_t sp[3], sm[3];
    sp[0] = site_of(wrap(x + 1, nx), y, z, ny, nz);
    sm[0] = site_of(wrap(x - 1, nx), y, z, ny, nz);
    sp[1] = site_of(x, wrap(y + 1, ny), z, ny, nz);
    sm[1] = site_of(x, wrap(y - 1, ny), z, ny, nz);
    sp[2] = site_of(x, y, wrap(z + 1, nz), ny, nz);
    sm[2] = site_of(x, y, wrap(z - 1, nz), ny, nz);
    for (int a = 0; a < 3; ++a) {
        double d[3];
        for (int b = 0; b < 3; ++b) {
            double tp = (kappa * g[a][sp[b]]) * g[b][sp[b]];
            double tm = (kappa * g[a][sm[b]]) * g[b][sm[b]];
            if (a == b) {
                tp = piso[sp[b]] + tp;
                tm = piso[sm[b]] + tm;
            }
            d[b] = (tp - tm) * 0.5;
        }
        F[a] = -((d[0] + d[1]) + d[2]);
    }
}

/* Potential form of the force (physics 1), F = -phi grad(mu), with each
 * component smoothed along its own axis by the [1/4, 1/2, 1/4] filter:
 *   h_a(x) = -(phi(x) * ((mu(x+a) - mu(x-a)) * 0.5)),
 *   F_a(x) = ((h_a(x-a) + h_a(x+a)) + (h_a(x) + h_a(x))) * 0.25.
 * Why the filter: on the lattice the momentum mode j_a with
 * wavenumber pi along a is invariant under streaming (it flips sign) and
 * under collision (momentum is conserved), so nothing damps it, and the
 * unfiltered -phi grad(mu) projects onto it wherever phi varies: a flat
 * interface then grows a checkerboard velocity until it dissolves.  The
 * filter's transfer function (1 + cos k)/2 vanishes at k = pi, so the force has
 * no component on those modes; it keeps sum_x F and leaves F = 0 wherever
 * mu is uniform (the equilibrium).  h is the unfiltered force, F the filtered
 * one; both are [nsites] arrays per component. */
void orc_potential_force(const double *phi, const double *mu, double *h[3], double *F[3],
                         int64_t nx, int64_t ny, int64_t nz)
{
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < nx; ++x)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t z = 0; z < nz; ++z) {
                const int64_t s = site_of(x, y, z, ny, nz);
                const double gx = (mu[site_of(wrap(x + 1, nx), y, z, ny, nz)] -
                                   mu[site_of(wrap(x - 1, nx), y, z, ny, nz)]) * 0.5;
                const double gy = (mu[site_of(x, wrap(y + 1, ny), z, ny, nz)] -
                                   mu[site_of(x, wrap(y - 1, ny), z, ny, nz)]) * 0.5;
                const double gz = (mu[site_of(x, y, wrap(z + 1, nz), ny, nz)] -
                                   mu[site_of(x, y, wrap(z - 1, nz), ny, nz)]) * 0.5;
                h[0][s] = -(phi[s] * gx);
                h[1][s] = -(phi[s] * gy);
                h[2][s] = -(phi[s] * gz);
            }
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < nx; ++x)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t z = 0; z < nz; ++z) {
                const int64_t s = site_of(x, y, z, ny, nz);
                const int64_t xm = site_of(wrap(x - 1, nx), y, z, ny, nz),
                              xp = site_of(wrap(x + 1, nx), y, z, ny, nz),
                              ym = site_of(x, wrap(y - 1, ny), z, ny, nz),
                              yp = site_of(x, wrap(y + 1, ny), z, ny, nz),
                              zm = site_of(x, y, wrap(z - 1, nz), ny, nz),
                              zp = site_of(x, y, wrap(z + 1, nz), ny, nz);
                F[0][s] = ((h[0][xm] + h[0][xp]) + (h[0][s] + h[0][s])) * 0.25;
                F[1][s] = ((h[1][ym] + h[1][yp]) + (h[1][s] + h[1][s])) * 0.25;
                F[2][s] = ((h[2][zm] + h[2][zp]) + (h[2][s] + h[2][s])) * 0.25;
            }
}

/* Collision of one streamed site (f_s, g_s hold the 19 pulled values).
 * physics 0: reference collision (kernels.py:96-125 op order).
 * physics 1, 2: Guo-forced f with the force (Fx, Fy, Fz) (orc_potential_force
 *            or stress_force); g_eq with the lam*(gamma mu - phi cs2) term.
 * Returns 0, or 1 if rho <= 0 (site left as streamed). */
static int collide_site(double *fs, double *gs, double mu, double Fx_in, double Fy_in,
                        double Fz_in, const orc_fluid_params *p)
{
    double rho = 0.0, jx = 0.0, jy = 0.0, jz = 0.0;
    for (int i = 0; i < Q; ++i) {
        double fi = fs[i];
        rho += fi;
        jx += fi * (double)CV[i][0];
        jy += fi * (double)CV[i][1];
        jz += fi * (double)CV[i][2];
    }
    if (rho <= 0.0) return 1;
    double phi = 0.0;
    for (int i = 0; i < Q; ++i) phi += gs[i];

    const double cs2 = p->cs2;
    double Fx = 0.0, Fy = 0.0, Fz = 0.0, ux, uy, uz;
    if (p->physics >= 1) {
        Fx = Fx_in;
        Fy = Fy_in;
        Fz = Fz_in;
        ux = (jx + 0.5 * Fx) / rho;
        uy = (jy + 0.5 * Fy) / rho;
        uz = (jz + 0.5 * Fz) / rho;
    } else {
        ux = jx / rho;
        uy = jy / rho;
        uz = jz / rho;
    }
    double usq = ux * ux + uy * uy + uz * uz;
    double uF = (ux * Fx + uy * Fy) + uz * Fz;
    double psi = p->gamma * mu - phi * cs2;
    double srcpre = 1.0 - 0.5 / p->tau_f;
    for (int i = 0; i < Q; ++i) {
        double cx = CV[i][0], cy = CV[i][1], cz = CV[i][2];
        double udotc = ux * cx + uy * cy + uz * cz;
        double bracket = 1.0 + udotc / cs2 + (udotc * udotc) / (2.0 * cs2 * cs2)
                         - usq / (2.0 * cs2);
        double feq = p->wv[i] * rho * bracket;
        double geq = p->wv[i] * phi * bracket;
        double fn = fs[i] - (fs[i] - feq) / p->tau_f;
        if (p->physics >= 1) {
            double cF = (cx * Fx + cy * Fy) + cz * Fz;
            double src = (srcpre * p->wv[i]) * ((cF - uF) / cs2 + (udotc * cF) / (cs2 * cs2));
            fn = fn + src;
            geq = geq + p->lam[i] * psi;
        }
        fs[i] = fn;
        gs[i] = gs[i] - (gs[i] - geq) / p->tau_g;
    }
    return 0;
}

/* One full timestep on host-ordered fields: stream (pull) -> phi -> mu ->
 * force (physics 1: orc_potential_force; 2: stress_force) -> collide.  f_in/g_in are post-collision states of the previous
 * step; f_out/g_out receive the new post-collision state; phi/mu are
 * scratch [nsites] arrays (left holding this step's phi and mu).
 * Returns the first singular real site or -1. */
int64_t orc_fluid_step(const double *f_in, const double *g_in, double *f_out,
                       double *g_out, double *phi, double *mu, int64_t padded,
                       int64_t nx, int64_t ny, int64_t nz, const orc_fluid_params *p)
{
    const int64_t nsites = nx * ny * nz;
    orc_stream(f_in, f_out, Q, padded, nx, ny, nz);
    orc_stream(g_in, g_out, Q, padded, nx, ny, nz);
    orc_phi(g_out, phi, padded, nsites);
    if (p->physics >= 1)
        orc_mu(phi, mu, nx, ny, nz, p->A, p->B, p->kappa);
    else
        memset(mu, 0, sizeof(double) * nsites);
    /* physics 1: h (3 arrays) and F (3 arrays); physics 2: p_iso, grad phi */
    double *aux = NULL, *gr[3] = {NULL, NULL, NULL}, *hh[3] = {NULL, NULL, NULL},
           *FF[3] = {NULL, NULL, NULL};
    if (p->physics >= 1) {
        aux = (double *)malloc(sizeof(double) * 6 * (size_t)nsites);
        if (!aux) return -2;
    }
    if (p->physics == 1) {
        for (int k = 0; k < 3; ++k) {
            hh[k] = aux + k * nsites;
            FF[k] = aux + (3 + k) * nsites;
        }
        orc_potential_force(phi, mu, hh, FF, nx, ny, nz);
    } else if (p->physics == 2) {
        gr[0] = aux + nsites;
        gr[1] = aux + 2 * nsites;
        gr[2] = aux + 3 * nsites;
        orc_stress(phi, mu, aux, gr[0], gr[1], gr[2], nx, ny, nz, p->A, p->B, p->kappa);
    }
    const double *const grc[3] = {gr[0], gr[1], gr[2]};
    int64_t bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
    for (int64_t x = 0; x < nx; ++x) {
        double fs[Q], gs[Q];
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t z = 0; z < nz; ++z) {
                int64_t s = site_of(x, y, z, ny, nz);
                double Fv[3] = {0.0, 0.0, 0.0}, m = mu[s];
                if (p->physics == 2) {
                    stress_force(aux, grc, p->kappa, x, y, z, nx, ny, nz, Fv);
                } else if (p->physics == 1) {
                    Fv[0] = FF[0][s];
                    Fv[1] = FF[1][s];
                    Fv[2] = FF[2][s];
                }
                for (int i = 0; i < Q; ++i) {
                    fs[i] = f_out[i * padded + s];
                    gs[i] = g_out[i * padded + s];
                }
                if (collide_site(fs, gs, m, Fv[0], Fv[1], Fv[2], p)) {
                    if (s > bad) bad = s;
                    continue;
                }
                for (int i = 0; i < Q; ++i) {
                    f_out[i * padded + s] = fs[i];
                    g_out[i * padded + s] = gs[i];
                }
            }
    }
    free(aux);
    return bad;
}
