/*
 * spark_oracle.c — CPU oracle for the Spark block-update hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2401_03378_b200/, libspark) never links, imports
 * or calls it, and this file shares no code, header or constant with it.
 *
 * Plain, slow, obviously-correct FP64 C.  Build: gcc -O2 -ffp-contract=off
 * -fno-fast-math -fopenmp (no FMA contraction, no reassociation).
 *
 * What it computes, in the paper's order (PAPER.md = /root/reference/PAPER.md):
 *   - lst:spark-nontelescoping: for every RK stage, first
 *     fill_guardcells() for all blocks, then for every block the block
 *     initialisation (Alg. 7: initSoln keeps U^n) and the
 *     intra-stage calculations (Alg. 8):
 *     grvAccel (uniform gravity source, NEXT N2; identity when g = 0) ->
 *     calcLims (reconstruction: PLM-minmod / PLM-MC / WENO5-JS / WENO5-Z) ->
 *     calcFlux (Riemann) -> updSoln (divergence + RK combination) ->
 *     calcEos (pressure / positivity check).  fluxBuff is not needed on a
 *     single-level grid (no coarse-fine faces).
 *   - Blocks have identical cell counts and a surrounding halo of guard
 *     cells that makes each block look like a whole domain:
 *     this oracle materialises exactly that padded per-block array.
 *   - SSP-RK time stepping (Gottlieb & Shu 1998).
 * The paper states no formulas for the numerics; every formula below is the
 * textbook reading recorded in DESIGN.md §3:
 *   ideal-gas EOS; PLM-minmod / WENO5-JS on primitive variables with a
 *   first-order positivity fallback; HLL / HLLC (Toro §10.4) with Davis wave
 *   speeds; CFL dt = C min_cells min_d dx_d/(|u_d|+c); Shu-Osher SSP-RK2/3.
 *
 * Layouts (identical meaning to include/spark.h, defined here independently):
 *   canonical  U[v][b][k][j][i]            fp64, i fastest, b lexicographic
 *   padded     P[v][b][k+gz][j+gy][i+gx]   gd = ng for d < ndim, else 0
 * Variables: v = 0 rho, 1..ndim momentum, ndim+1 total energy.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int32_t ndim;
    int32_t nb[3];
    int32_t nblk[3];
    int32_t ng;
    double lo[3], hi[3];
    int32_t bc[3][2];       /* 0 periodic, 1 outflow, 2 reflect */
    int32_t recon;          /* 0 first order, 1 PLM-minmod, 2 WENO5-JS, 3 PLM-MC, 4 WENO5-Z */
    int32_t riemann;        /* 0 HLL, 1 HLLC */
    int32_t rk_stages;      /* 2 or 3 */
    double gamma, cfl;
    double grav[3];         /* grvAccel: uniform gravitational acceleration (0: none) */
    double shock_thresh;    /* shockDet threshold (riemann 2 = HLLC, HLL at shock faces) */
} ocfg;

enum { OBC_PERIODIC = 0, OBC_OUTFLOW = 1, OBC_REFLECT = 2 };
enum { OREC_FIRST = 0, OREC_PLM = 1, OREC_WENO5 = 2, OREC_PLM_MC = 3, OREC_WENO5Z = 4 };
enum { ORS_HLL = 0, ORS_HLLC = 1, ORS_HYBRID = 2 };

/* status codes */
enum { OK = 0, OERR_ARG = 1, OERR_NONPHYSICAL = 5, OERR_OOM = 4 };

/* ---------------------------------------------------------------- geometry */
static int nvar_of(const ocfg* c) { return c->ndim + 2; }
/* reconstruction half-width (cells each side of a face the stencil reaches) */
static int ngk_of(int recon) {
    if (recon == OREC_WENO5 || recon == OREC_WENO5Z) return 3;
    if (recon == OREC_PLM || recon == OREC_PLM_MC) return 2;
    return 1;
}
static long cells_per_block(const ocfg* c) { return (long)c->nb[0] * c->nb[1] * c->nb[2]; }
static long nblocks(const ocfg* c) { return (long)c->nblk[0] * c->nblk[1] * c->nblk[2]; }
static int guard_of(const ocfg* c, int d) { return d < c->ndim ? c->ng : 0; }
static long padded_cells(const ocfg* c) {
    long n = 1;
    for (int d = 0; d < 3; d++) n *= c->nb[d] + 2 * guard_of(c, d);
    return n;
}
static double dx_of(const ocfg* c, int d) {
    return (c->hi[d] - c->lo[d]) / ((double)c->nblk[d] * (double)c->nb[d]);
}

int oracle_check_config(const ocfg* c) {
    if (c->ndim < 1 || c->ndim > 3) return OERR_ARG;
    for (int d = 0; d < 3; d++) {
        if (c->nb[d] < 1 || c->nblk[d] < 1) return OERR_ARG;
        if (d >= c->ndim && (c->nb[d] != 1 || c->nblk[d] != 1)) return OERR_ARG;
        if (d < c->ndim && c->nb[d] < c->ng) return OERR_ARG;
    }
    if (c->recon < 0 || c->recon > 4 || c->ng < ngk_of(c->recon)) return OERR_ARG;
    if (c->riemann < 0 || c->riemann > 2) return OERR_ARG;
    /* shockDet reads the cells i-1..i+2 of a face: a stencil of 2 each side */
    if (c->riemann == ORS_HYBRID && (ngk_of(c->recon) < 2 || !(c->shock_thresh > 0.0))) return OERR_ARG;
    if (c->rk_stages != 2 && c->rk_stages != 3) return OERR_ARG;
    if (!(c->gamma > 1.0) || !(c->cfl > 0.0)) return OERR_ARG;
    return OK;
}

/* Guard-cell map along one dimension (reading R4): global cell
 * index g (possibly outside [0,N)) -> interior index; *flip = 1 when a
 * reflecting wall mirrors the cell (normal momentum changes sign). */
static long map_dim(long g, long N, int bc_lo, int bc_hi, int* flip) {
    *flip = 0;
    if (g >= 0 && g < N) return g;
    int bc = g < 0 ? bc_lo : bc_hi;
    if (bc == OBC_PERIODIC) {
        long m = g % N;
        if (m < 0) m += N;
        return m;
    }
    if (bc == OBC_OUTFLOW) return g < 0 ? 0 : N - 1;
    *flip = 1; /* reflect */
    return g < 0 ? -1 - g : 2 * N - 1 - g;
}

/* fill_guardcells: padded per-block copy of U with
 * every guard cell (faces, edges, corners) taken from the per-dimension map
 * of its global index.  Interior cells are copied unchanged. */
int oracle_fill_guardcells(const ocfg* c, const double* U, double* P) {
    if (oracle_check_config(c)) return OERR_ARG;
    const int nv = nvar_of(c);
    const long NB = nblocks(c), nc = cells_per_block(c), np = padded_cells(c);
    const long N[3] = {(long)c->nblk[0] * c->nb[0], (long)c->nblk[1] * c->nb[1],
                       (long)c->nblk[2] * c->nb[2]};
    const int g[3] = {guard_of(c, 0), guard_of(c, 1), guard_of(c, 2)};
    const int pn[3] = {c->nb[0] + 2 * g[0], c->nb[1] + 2 * g[1], c->nb[2] + 2 * g[2]};
#pragma omp parallel for schedule(static)
    for (long b = 0; b < NB; b++) {
        long bx = b % c->nblk[0], by = (b / c->nblk[0]) % c->nblk[1], bz = b / ((long)c->nblk[0] * c->nblk[1]);
        for (int pk = 0; pk < pn[2]; pk++)
            for (int pj = 0; pj < pn[1]; pj++)
                for (int pi = 0; pi < pn[0]; pi++) {
                    int fx, fy, fz;
                    long gx = map_dim(bx * c->nb[0] + pi - g[0], N[0], c->bc[0][0], c->bc[0][1], &fx);
                    long gy = map_dim(by * c->nb[1] + pj - g[1], N[1], c->bc[1][0], c->bc[1][1], &fy);
                    long gz = map_dim(bz * c->nb[2] + pk - g[2], N[2], c->bc[2][0], c->bc[2][1], &fz);
                    long sb = (gx / c->nb[0]) + c->nblk[0] * ((gy / c->nb[1]) + c->nblk[1] * (gz / c->nb[2]));
                    long sc = ((gz % c->nb[2]) * c->nb[1] + (gy % c->nb[1])) * c->nb[0] + (gx % c->nb[0]);
                    long pidx = ((long)pk * pn[1] + pj) * pn[0] + pi;
                    int flip[3] = {fx, fy, fz};
                    for (int v = 0; v < nv; v++) {
                        double val = U[(long)v * NB * nc + sb * nc + sc];
                        if (v >= 1 && v <= c->ndim && flip[v - 1]) val = -val;
                        P[(long)v * NB * np + b * np + pidx] = val;
                    }
                }
    }
    return OK;
}

/* ------------------------------------------------------------------- EOS */
/* EOS unit, ideal gas: p = (gamma-1)(E - 1/2 |m|^2/rho). */
static void cons_to_prim(int ndim, double gamma, const double* u, double* w) {
    double rho = u[0];
    double ke = 0.0;
    for (int d = 0; d < ndim; d++) ke += u[1 + d] * u[1 + d];
    w[0] = rho;
    for (int d = 0; d < ndim; d++) w[1 + d] = u[1 + d] / rho;
    w[ndim + 1] = (gamma - 1.0) * (u[ndim + 1] - 0.5 * ke / rho);
}

/* E = p/(gamma-1) + 1/2 rho |u|^2. */
static void prim_to_cons(int ndim, double gamma, const double* w, double* u) {
    double rho = w[0];
    double u2 = 0.0;
    for (int d = 0; d < ndim; d++) u2 += w[1 + d] * w[1 + d];
    u[0] = rho;
    for (int d = 0; d < ndim; d++) u[1 + d] = rho * w[1 + d];
    u[ndim + 1] = w[ndim + 1] / (gamma - 1.0) + 0.5 * rho * u2;
}

/* Canonical-layout conversions over ncells cells (arrays [nvar][ncells]). */
void oracle_prim_to_cons(int ndim, double gamma, long ncells, const double* W, double* U) {
    int nv = ndim + 2;
    for (long n = 0; n < ncells; n++) {
        double w[5], u[5];
        for (int v = 0; v < nv; v++) w[v] = W[(long)v * ncells + n];
        prim_to_cons(ndim, gamma, w, u);
        for (int v = 0; v < nv; v++) U[(long)v * ncells + n] = u[v];
    }
}

void oracle_cons_to_prim(int ndim, double gamma, long ncells, const double* U, double* W) {
    int nv = ndim + 2;
    for (long n = 0; n < ncells; n++) {
        double w[5], u[5];
        for (int v = 0; v < nv; v++) u[v] = U[(long)v * ncells + n];
        cons_to_prim(ndim, gamma, u, w);
        for (int v = 0; v < nv; v++) W[(long)v * ncells + n] = w[v];
    }
}

/* --------------------------------------------------------- reconstruction */
/* calcLims.  minmod (reading R2): 0 unless a and b are
 * both strictly positive or both strictly negative; then the one of
 * smaller magnitude. */
static double minmod(double a, double b) {
    if (a > 0.0 && b > 0.0) return a < b ? a : b;
    if (a < 0.0 && b < 0.0) return a > b ? a : b;
    return 0.0;
}

/* PLM face states at i+1/2 from W_{i-1}, W_i, W_{i+1}, W_{i+2}. */
void oracle_plm_face(double wm1, double w0, double w1, double w2, double* wl, double* wr) {
    double d0 = minmod(w0 - wm1, w1 - w0);
    double d1 = minmod(w1 - w0, w2 - w1);
    *wl = w0 + 0.5 * d0;
    *wr = w1 - 0.5 * d1;
}

/* WENO5-JS (Jiang & Shu 1996) value at the right edge of cell c from the
 * cell averages (a,b,c,d,e) = W_{i-2..i+2}: DESIGN.md reading R3. */
double oracle_weno5_edge(double a, double b, double c, double d, double e) {
    const double eps = 1e-6;
    double b0 = 13.0 / 12.0 * (a - 2.0 * b + c) * (a - 2.0 * b + c) + 0.25 * (a - 4.0 * b + 3.0 * c) * (a - 4.0 * b + 3.0 * c);
    double b1 = 13.0 / 12.0 * (b - 2.0 * c + d) * (b - 2.0 * c + d) + 0.25 * (b - d) * (b - d);
    double b2 = 13.0 / 12.0 * (c - 2.0 * d + e) * (c - 2.0 * d + e) + 0.25 * (3.0 * c - 4.0 * d + e) * (3.0 * c - 4.0 * d + e);
    double a0 = 0.1 / ((eps + b0) * (eps + b0));
    double a1 = 0.6 / ((eps + b1) * (eps + b1));
    double a2 = 0.3 / ((eps + b2) * (eps + b2));
    double q0 = (2.0 * a - 7.0 * b + 11.0 * c) / 6.0;
    double q1 = (-b + 5.0 * c + 2.0 * d) / 6.0;
    double q2 = (2.0 * c + 5.0 * d - e) / 6.0;
    return (a0 * q0 + a1 * q1 + a2 * q2) / (a0 + a1 + a2);
}

/* Monotonized-central limiter (van Leer 1977; Toro 2009 §13.8, DESIGN.md
 * reading R18): slope = minmod(2 dl, (dl + dr)/2, 2 dr), the three-argument
 * minmod being 0 unless all three are strictly positive or all strictly
 * negative, then the one of smallest magnitude. */
static double minmod3(double a, double b, double c) {
    if (a > 0.0 && b > 0.0 && c > 0.0) return fmin(a, fmin(b, c));
    if (a < 0.0 && b < 0.0 && c < 0.0) return fmax(a, fmax(b, c));
    return 0.0;
}

static double mc_slope(double wm, double w0, double wp) {
    const double dl = w0 - wm, dr = wp - w0;
    return minmod3(2.0 * dl, 0.5 * (dl + dr), 2.0 * dr);
}

/* PLM-MC face states at i+1/2 from W_{i-1}, W_i, W_{i+1}, W_{i+2}. */
void oracle_mc_face(double wm1, double w0, double w1, double w2, double* wl, double* wr) {
    *wl = w0 + 0.5 * mc_slope(wm1, w0, w1);
    *wr = w1 - 0.5 * mc_slope(w0, w1, w2);
}

/* WENO5-Z (Borges, Carmona, Costa & Don 2008, eq. 25-26 with q = 1,
 * eps = 1e-40; reading R19): the WENO5-JS smoothness indicators and
 * candidates, weights alpha_k = d_k (1 + tau5 / (beta_k + eps)) with
 * tau5 = |beta_0 - beta_2|; value at the right edge of cell c. */
double oracle_weno5z_edge(double a, double b, double c, double d, double e) {
    const double eps = 1e-40;
    double b0 = 13.0 / 12.0 * (a - 2.0 * b + c) * (a - 2.0 * b + c) + 0.25 * (a - 4.0 * b + 3.0 * c) * (a - 4.0 * b + 3.0 * c);
    double b1 = 13.0 / 12.0 * (b - 2.0 * c + d) * (b - 2.0 * c + d) + 0.25 * (b - d) * (b - d);
    double b2 = 13.0 / 12.0 * (c - 2.0 * d + e) * (c - 2.0 * d + e) + 0.25 * (3.0 * c - 4.0 * d + e) * (3.0 * c - 4.0 * d + e);
    double tau = fabs(b0 - b2);
    double a0 = 0.1 * (1.0 + tau / (b0 + eps));
    double a1 = 0.6 * (1.0 + tau / (b1 + eps));
    double a2 = 0.3 * (1.0 + tau / (b2 + eps));
    double q0 = (2.0 * a - 7.0 * b + 11.0 * c) / 6.0;
    double q1 = (-b + 5.0 * c + 2.0 * d) / 6.0;
    double q2 = (2.0 * c + 5.0 * d - e) / 6.0;
    return (a0 * q0 + a1 * q1 + a2 * q2) / (a0 + a1 + a2);
}

/* WENO5 face states at i+1/2 from W_{i-2..i+3} (s[0..5]). */
void oracle_weno5_face(const double* s, double* wl, double* wr) {
    *wl = oracle_weno5_edge(s[0], s[1], s[2], s[3], s[4]);
    *wr = oracle_weno5_edge(s[5], s[4], s[3], s[2], s[1]);
}

void oracle_weno5z_face(const double* s, double* wl, double* wr) {
    *wl = oracle_weno5z_edge(s[0], s[1], s[2], s[3], s[4]);
    *wr = oracle_weno5z_edge(s[5], s[4], s[3], s[2], s[1]);
}

/* Face states for all nvar primitive components.  st[m*nv + v] holds the
 * stencil W_{i-ng+1+m} (m = 0..2ng-1) for a face at i+1/2.  Components are in
 * the rotated frame (rho, u_n, u_t..., p).  Positivity fallback: first order
 * when rho or p of either state is <= 0. */
static void reconstruct(int recon, int ng, int nv, const double* st, double* wl, double* wr) {
    const double* c0 = st + (ng - 1) * nv; /* W_i   */
    const double* c1 = st + ng * nv;       /* W_i+1 */
    for (int v = 0; v < nv; v++) {
        if (recon == OREC_FIRST) {
            wl[v] = c0[v];
            wr[v] = c1[v];
        } else if (recon == OREC_PLM) {
            oracle_plm_face(st[(ng - 2) * nv + v], c0[v], c1[v], st[(ng + 1) * nv + v], &wl[v], &wr[v]);
        } else if (recon == OREC_PLM_MC) {
            oracle_mc_face(st[(ng - 2) * nv + v], c0[v], c1[v], st[(ng + 1) * nv + v], &wl[v], &wr[v]);
        } else {
            double s[6];
            for (int m = 0; m < 6; m++) s[m] = st[(ng - 3 + m) * nv + v];
            if (recon == OREC_WENO5) oracle_weno5_face(s, &wl[v], &wr[v]);
            else oracle_weno5z_face(s, &wl[v], &wr[v]);
        }
    }
    if (!(wl[0] > 0.0) || !(wl[nv - 1] > 0.0) || !(wr[0] > 0.0) || !(wr[nv - 1] > 0.0)) {
        for (int v = 0; v < nv; v++) {
            wl[v] = c0[v];
            wr[v] = c1[v];
        }
    }
}

/* grvAccel (Alg. 8; reading R20): a uniform gravitational
 * acceleration g enters the stage operator as the source
 * S(U) = (0, rho g, m . g) evaluated at the stage's input state. */
static double grav_source(const ocfg* c, int v, const double* u) {
    const int nv = nvar_of(c);
    if (v == 0) return 0.0;
    if (v < nv - 1) return u[0] * c->grav[v - 1];
    double s = 0.0;
    for (int d = 0; d < c->ndim; d++) s += u[1 + d] * c->grav[d];
    return s;
}

static int has_grav(const ocfg* c) { return c->grav[0] != 0.0 || c->grav[1] != 0.0 || c->grav[2] != 0.0; }

/* ----------------------------------------------------------------- shockDet */
/* shockDet (Alg. 7; reading R21).  Cell i is a shock cell
 * along direction d when
 *   (a) the flow converges across it faster than a dead band of 1e-6 of the
 *       sound speed: u_d(i+1) - u_d(i-1) < -1e-6 c, with
 *       c^2 = gamma max(p(i-1)/rho(i-1), p(i+1)/rho(i+1)) — symmetric states
 *       leave velocities that are exactly equal or exactly zero, and their
 *       last-bit noise must not decide a shock; a real shock compresses by O(c);
 *   (b) the pressure jump across it is large:
 *       |p(i+1) - p(i-1)| > thresh * min(p(i-1), p(i+1)).
 * (a) is evaluated without division as d < 0 and
 * d^2 rho(i-1) rho(i+1) > 1e-12 gamma max(p(i-1) rho(i+1), p(i+1) rho(i-1)).
 * A face is a shock face when either of its two cells is a shock cell along
 * the face normal.  Consumer (calcFlux, reading R21): the hybrid solver takes
 * HLL at shock faces and HLLC elsewhere. */
static int shock_cell(double um, double up, double pm, double pp, double rm, double rp, double thresh,
                      double gamma) {
    double d = up - um;
    if (!(d < 0.0)) return 0;
    double a = pm * rp, b = pp * rm;
    if (!(d * d * (rm * rp) > 1e-12 * gamma * (a > b ? a : b))) return 0;
    double pmin = pm < pp ? pm : pp;
    return fabs(pp - pm) > thresh * pmin;
}

/* un[m], p[m], rho[m]: normal velocity, pressure and density of the cells
 * i-1, i, i+1, i+2 of the face between cells i and i+1. */
int oracle_shock_face(const double* un, const double* p, const double* rho, double thresh, double gamma) {
    return shock_cell(un[0], un[2], p[0], p[2], rho[0], rho[2], thresh, gamma) ||
           shock_cell(un[1], un[3], p[1], p[3], rho[1], rho[3], thresh, gamma);
}

/* Riemann solver of a face whose stencil st (rotated frame, cells
 * i-ngk+1..i+ngk, nv components each) is given: the configured one, or for
 * the hybrid solver HLL at shock faces and HLLC elsewhere. */
static int face_solver(const ocfg* c, int ngk, int nv, const double* st) {
    if (c->riemann != ORS_HYBRID) return c->riemann;
    double un[4], p[4], rho[4];
    for (int m = 0; m < 4; m++) {
        rho[m] = st[(ngk - 2 + m) * nv + 0];
        un[m] = st[(ngk - 2 + m) * nv + 1];
        p[m] = st[(ngk - 2 + m) * nv + nv - 1];
    }
    return oracle_shock_face(un, p, rho, c->shock_thresh, c->gamma) ? ORS_HLL : ORS_HLLC;
}

/* ------------------------------------------------------------------ Riemann */
/* Physical flux along the normal of the rotated frame (rho, u_n, u_t.., p).
 * ax[e] is the rotated index of axis e: |u|^2 is summed in axis order
 * (u_x^2 + u_y^2) + u_z^2 whatever the direction (reading R9). */
static void phys_flux(int nv, double gamma, const int* ax, const double* w, double* u, double* f) {
    double rho = w[0], un = w[1], p = w[nv - 1];
    double u2 = 0.0;
    for (int e = 0; e < nv - 2; e++) u2 += w[ax[e]] * w[ax[e]];
    u[0] = rho;
    for (int m = 1; m < nv - 1; m++) u[m] = rho * w[m];
    u[nv - 1] = p / (gamma - 1.0) + 0.5 * rho * u2;
    f[0] = rho * un;
    f[1] = rho * un * un + p;
    for (int m = 2; m < nv - 1; m++) f[m] = rho * un * w[m];
    f[nv - 1] = un * (u[nv - 1] + p);
}

/* calcFlux: HLL or HLLC (Toro §10.4) with Davis wave speeds
 * (readings R5, R6).  wl, wr, f are in the rotated frame. */
static void riemann_ax(int riemann, int nv, double gamma, const int* ax, const double* wl, const double* wr,
                       double* f) {
    double ul[5], ur[5], fl[5], fr[5];
    phys_flux(nv, gamma, ax, wl, ul, fl);
    phys_flux(nv, gamma, ax, wr, ur, fr);
    double rl = wl[0], uL = wl[1], pl = wl[nv - 1];
    double rr = wr[0], uR = wr[1], pr = wr[nv - 1];
    double cl = sqrt(gamma * pl / rl), cr = sqrt(gamma * pr / rr);
    double sl = fmin(uL - cl, uR - cr);
    double sr = fmax(uL + cl, uR + cr);
    if (sl >= 0.0) {
        for (int v = 0; v < nv; v++) f[v] = fl[v];
        return;
    }
    if (sr <= 0.0) {
        for (int v = 0; v < nv; v++) f[v] = fr[v];
        return;
    }
    if (riemann == ORS_HLL) {
        for (int v = 0; v < nv; v++)
            f[v] = (sr * fl[v] - sl * fr[v] + sl * sr * (ur[v] - ul[v])) / (sr - sl);
        return;
    }
    double sstar = (pr - pl + rl * uL * (sl - uL) - rr * uR * (sr - uR)) / (rl * (sl - uL) - rr * (sr - uR));
    const double* w = sstar >= 0.0 ? wl : wr;
    const double* uk = sstar >= 0.0 ? ul : ur;
    const double* fk = sstar >= 0.0 ? fl : fr;
    double sk = sstar >= 0.0 ? sl : sr;
    double rho = w[0], un = w[1], p = w[nv - 1];
    double fac = rho * (sk - un) / (sk - sstar);
    double us[5];
    us[0] = fac;
    us[1] = fac * sstar;
    for (int m = 2; m < nv - 1; m++) us[m] = fac * w[m];
    us[nv - 1] = fac * (uk[nv - 1] / rho + (sstar - un) * (sstar + p / (rho * (sk - un))));
    for (int v = 0; v < nv; v++) f[v] = fk[v] + sk * (us[v] - uk[v]);
}

/* Public entry for the pins: states already in the frame whose normal is
 * axis 0 (identity rotation). */
void oracle_riemann(int riemann, int nv, double gamma, const double* wl, const double* wr, double* f) {
    int ax[3] = {1, 2, 3};
    riemann_ax(riemann, nv, gamma, ax, wl, wr, f);
}

/* Rotation for direction d (reading R9): rotated components
 * (rho, u_d, the other velocities in increasing axis order, p).  rot[m] is
 * the unrotated component index of rotated component m. */
static void rotation(int ndim, int d, int* rot, int* ax) {
    int nv = ndim + 2, m = 2;
    rot[0] = 0;
    rot[1] = 1 + d;
    ax[d] = 1;
    for (int e = 0; e < ndim; e++)
        if (e != d) { ax[e] = m; rot[m++] = 1 + e; }
    rot[nv - 1] = nv - 1;
}

/* ------------------------------------------------------------- dt (CFL) */
/* dt = C * min_cells min_d dx_d/(|u_d| + c)  (reading R7). */
double oracle_dt_raw(const ocfg* c, const double* U) {
    const int nv = nvar_of(c);
    const long n = nblocks(c) * cells_per_block(c);
    double dx[3] = {dx_of(c, 0), dx_of(c, 1), dx_of(c, 2)};
    double best = INFINITY;
    for (long q = 0; q < n; q++) {
        double u[5], w[5];
        for (int v = 0; v < nv; v++) u[v] = U[(long)v * n + q];
        cons_to_prim(c->ndim, c->gamma, u, w);
        double cs = sqrt(c->gamma * w[nv - 1] / w[0]);
        for (int d = 0; d < c->ndim; d++) {
            double t = dx[d] / (fabs(w[1 + d]) + cs);
            if (t < best) best = t;
        }
    }
    return best;
}

double oracle_dt(const ocfg* c, const double* U, double t, double t_end) {
    double dt = c->cfl * oracle_dt_raw(c, U);
    if (t_end > 0.0 && dt > t_end - t) dt = t_end - t;
    return dt;
}

/* ------------------------------------------------------------ one stage */
/* Intra-stage calculations (Alg. 8) on every block of an
 * already-filled padded array P (U^(s-1) with guards):
 *   U_out = a * Un + b * (U_prev + dt * L(U_prev))
 * with L = -[(Fx+ - Fx-)/dx + (Fy+ - Fy-)/dy] - (Fz+ - Fz-)/dz (reading R8).
 * U_prev is read from the interior of P.  Un may be NULL when a == 0.
 * Returns OERR_NONPHYSICAL if any updated cell has rho <= 0, p <= 0 or a
 * non-finite value (calcEos; reading R12). */
/* Largest number of cells on one face of a block (face-flux buffers). */
static long face_cells_max(const ocfg* c) {
    long m = 1;
    for (int d = 0; d < c->ndim; d++) {
        long f = 1;
        for (int e = 0; e < c->ndim; e++)
            if (e != d) f *= c->nb[e];
        if (f > m) m = f;
    }
    return m;
}

/* Cell index on the face of a block normal to d: the two other coordinates,
 * the lower dimension fastest. */
static long face_cell(const ocfg* c, int d, int i, int j, int k) {
    if (d == 0) return (long)k * c->nb[1] + j;
    if (d == 1) return (long)k * c->nb[0] + i;
    return (long)j * c->nb[0] + i;
}

static int stage_padded_fb(const ocfg* c, const double* P, const double* Un, double a, double b, double dt,
                           double* Uout, double* Fb);

/* One stage on padded blocks (guards already filled). */
int oracle_stage_padded(const ocfg* c, const double* P, const double* Un, double a, double b, double dt,
                        double* Uout) {
    return stage_padded_fb(c, P, Un, a, b, dt, Uout, NULL);
}

/* ... and, when Fb != NULL, the fluxes through each block's 2*ndim faces
 * (fluxBuff, Alg. 8): Fb[blk][2 d + side][v][face cell], face_cell()
 * order, face_cells_max() cells per face slot. */
static int stage_padded_fb(const ocfg* c, const double* P, const double* Un, double a, double b, double dt,
                           double* Uout, double* Fb) {
    if (oracle_check_config(c)) return OERR_ARG;
    const int nv = nvar_of(c), ndim = c->ndim;
    const long NB = nblocks(c), nc = cells_per_block(c), np = padded_cells(c);
    const int g[3] = {guard_of(c, 0), guard_of(c, 1), guard_of(c, 2)};
    const int pn[3] = {c->nb[0] + 2 * g[0], c->nb[1] + 2 * g[1], c->nb[2] + 2 * g[2]};
    const long pstride[3] = {1, pn[0], (long)pn[0] * pn[1]};
    double dx[3] = {dx_of(c, 0), dx_of(c, 1), dx_of(c, 2)};
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        double* W = malloc(sizeof(double) * nv * np);          /* primitives on the padded tile */
        double* F[3] = {NULL, NULL, NULL};                     /* face fluxes per direction */
        long nf[3] = {0, 0, 0};
        for (int d = 0; d < ndim; d++) {
            nf[d] = 1;
            for (int e = 0; e < 3; e++) nf[d] *= c->nb[e] + (e == d ? 1 : 0);
            F[d] = malloc(sizeof(double) * nv * nf[d]);
        }
#pragma omp for schedule(static)
        for (long blk = 0; blk < NB; blk++) {
            const double* Pb = P + blk * np;
            /* block init: primitives from the EOS on every padded cell */
            for (long q = 0; q < np; q++) {
                double u[5], w[5];
                for (int v = 0; v < nv; v++) u[v] = Pb[(long)v * NB * np + q];
                cons_to_prim(ndim, c->gamma, u, w);
                for (int v = 0; v < nv; v++) W[(long)v * np + q] = w[v];
            }
            /* calcLims + calcFlux per direction */
            for (int d = 0; d < ndim; d++) {
                int rot[5], ax[3];
                rotation(ndim, d, rot, ax);
                int fn[3] = {c->nb[0], c->nb[1], c->nb[2]};
                fn[d] += 1;
                for (int k = 0; k < fn[2]; k++)
                    for (int j = 0; j < fn[1]; j++)
                        for (int i = 0; i < fn[0]; i++) {
                            /* face between cells (idx-1) and idx along d; padded coords
                             * of the cell on its right are (i,j,k)+g. */
                            long right = ((long)(k + g[2]) * pn[1] + (j + g[1])) * pn[0] + (i + g[0]);
                            /* the stencil: 2 ngk cells around the face (ng >= ngk guard
                             * layers exist; only the reconstruction's reach is read) */
                            const int ngk = ngk_of(c->recon);
                            double st[6 * 5], wl[5], wr[5], fr[5];
                            for (int m = 0; m < 2 * ngk; m++) {
                                long q = right + (long)(m - ngk) * pstride[d];
                                for (int v = 0; v < nv; v++) st[m * nv + v] = W[(long)rot[v] * np + q];
                            }
                            reconstruct(c->recon, ngk, nv, st, wl, wr);
                            riemann_ax(face_solver(c, ngk, nv, st), nv, c->gamma, ax, wl, wr, fr);
                            long fidx = ((long)k * fn[1] + j) * fn[0] + i;
                            for (int v = 0; v < nv; v++) F[d][(long)rot[v] * nf[d] + fidx] = fr[v];
                            const int at[3] = {i, j, k};
                            if (Fb && (at[d] == 0 || at[d] == c->nb[d])) {  /* a face of the block */
                                const long mf = face_cells_max(c);
                                const int side = at[d] == 0 ? 0 : 1;
                                double* fb = Fb + (blk * 6 + 2 * d + side) * nv * mf;
                                for (int v = 0; v < nv; v++) fb[(long)rot[v] * mf + face_cell(c, d, i, j, k)] = fr[v];
                            }
                        }
            }
            /* updSoln + calcEos */
            for (int k = 0; k < c->nb[2]; k++)
                for (int j = 0; j < c->nb[1]; j++)
                    for (int i = 0; i < c->nb[0]; i++) {
                        long cell = ((long)k * c->nb[1] + j) * c->nb[0] + i;
                        long pcell = ((long)(k + g[2]) * pn[1] + (j + g[1])) * pn[0] + (i + g[0]);
                        double unew[5], uc[5];
                        for (int v = 0; v < nv; v++) uc[v] = Pb[(long)v * NB * np + pcell];
                        for (int v = 0; v < nv; v++) {
                            double div[3] = {0.0, 0.0, 0.0};
                            for (int d = 0; d < ndim; d++) {
                                int fn[3] = {c->nb[0], c->nb[1], c->nb[2]};
                                fn[d] += 1;
                                int lo[3] = {i, j, k};
                                int hi[3] = {i, j, k};
                                hi[d] += 1;
                                long flo = ((long)lo[2] * fn[1] + lo[1]) * fn[0] + lo[0];
                                long fhi = ((long)hi[2] * fn[1] + hi[1]) * fn[0] + hi[0];
                                div[d] = (F[d][(long)v * nf[d] + fhi] - F[d][(long)v * nf[d] + flo]) / dx[d];
                            }
                            double L;
                            if (ndim == 1) L = -(div[0]);
                            else if (ndim == 2) L = -(div[0] + div[1]);
                            else L = -(div[0] + div[1]) - div[2];
                            if (has_grav(c)) L += grav_source(c, v, uc);  /* grvAccel */
                            double uprev = uc[v];
                            double un = Un ? Un[(long)v * NB * nc + blk * nc + cell] : 0.0;
                            double val = a * un + b * (uprev + dt * L);
                            unew[v] = val;
                            Uout[(long)v * NB * nc + blk * nc + cell] = val;
                        }
                        double w[5];
                        cons_to_prim(ndim, c->gamma, unew, w);
                        int ok = w[0] > 0.0 && w[nv - 1] > 0.0;
                        for (int v = 0; v < nv; v++) ok = ok && isfinite(unew[v]);
                        if (!ok) bad = 1;
                    }
        }
        free(W);
        for (int d = 0; d < 3; d++) free(F[d]);
    }
    return bad ? OERR_NONPHYSICAL : OK;
}

/* RK coefficients (Shu-Osher form, reading R10): stage s (1-based) computes
 * U^(s) = a_s U^n + b_s (U^(s-1) + dt L(U^(s-1))). */
void oracle_rk_coeffs(int stages, int s, double* a, double* b) {
    if (stages == 2) {
        if (s == 1) { *a = 0.0; *b = 1.0; }
        else { *a = 0.5; *b = 0.5; }
    } else {
        if (s == 1) { *a = 0.0; *b = 1.0; }
        else if (s == 2) { *a = 0.75; *b = 0.25; }
        else { *a = 1.0 / 3.0; *b = 2.0 / 3.0; }
    }
}

/* One stage from the canonical layout: fill_guardcells then the block loop
 * (lst:spark-nontelescoping body). */
int oracle_stage(const ocfg* c, const double* Uprev, const double* Un, double a, double b, double dt,
                 double* Uout) {
    if (oracle_check_config(c)) return OERR_ARG;
    size_t bytes = sizeof(double) * nvar_of(c) * nblocks(c) * padded_cells(c);
    double* P = malloc(bytes);
    if (!P) return OERR_OOM;
    oracle_fill_guardcells(c, Uprev, P);
    int st = oracle_stage_padded(c, P, Un, a, b, dt, Uout);
    free(P);
    return st;
}

/* One SSP-RK step in place on U (lst:spark-nontelescoping).
 * dt_fixed > 0 uses that dt; otherwise the CFL dt of U^n clipped to t_end - t
 * (t_end <= 0: no clip).  *dt_used receives the dt.  On a non-physical stage
 * U is left unchanged (U^n retained) and OERR_NONPHYSICAL is returned. */
int oracle_step(const ocfg* c, double* U, double t, double t_end, double dt_fixed, double* dt_used) {
    if (oracle_check_config(c)) return OERR_ARG;
    size_t n = (size_t)nvar_of(c) * nblocks(c) * cells_per_block(c);
    double dt = dt_fixed > 0.0 ? dt_fixed : oracle_dt(c, U, t, t_end);
    if (dt_used) *dt_used = dt;
    double* S0 = malloc(sizeof(double) * n);
    double* S1 = malloc(sizeof(double) * n);
    if (!S0 || !S1) { free(S0); free(S1); return OERR_OOM; }
    const double* prev = U;
    double* bufs[2] = {S0, S1};
    int st = OK;
    for (int s = 1; s <= c->rk_stages && st == OK; s++) {
        double a, b;
        oracle_rk_coeffs(c->rk_stages, s, &a, &b);
        double* out = bufs[(s - 1) & 1];
        st = oracle_stage(c, prev, U, a, b, dt, out);
        prev = out;
    }
    if (st == OK) memcpy(U, prev, sizeof(double) * n);
    free(S0);
    free(S1);
    return st;
}

/* Run to t_end (t_end > 0) and/or for at most max_steps steps (>0).
 * Stop rule (reading R8): t >= t_end * (1 - 1e-14).  Returns status; *t and
 * *nsteps are updated. */
int oracle_run(const ocfg* c, double* U, double t_end, long max_steps, double* t, long* nsteps) {
    int st = OK;
    while (st == OK) {
        if (t_end > 0.0 && *t >= t_end * (1.0 - 1e-14)) break;
        if (max_steps > 0 && *nsteps >= max_steps) break;
        double dt;
        st = oracle_step(c, U, *t, t_end, 0.0, &dt);
        if (st == OK) {
            *t += dt;
            *nsteps += 1;
        }
    }
    return st;
}

/* Threads of the OpenMP loops (bench.py times the oracle on all host cores
 * and on one); n <= 0 restores the default. */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    extern int omp_get_num_procs(void);
    omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
#else
    (void)n;
#endif
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------- telescoping SSP-RK (N1) */
/* Telescoping mode (lst:spark-telescoping P:1598-1604): ONE
 * fill_guardcells per step with S*NGK guard layers (all guards, edges and
 * corners included), then for every block all S stages, each updating the
 * block *and* the part of its halo that the later stages still need: stage s
 * updates the padded cells at distance >= s*NGK from the tile edge.  NGK is the
 * reconstruction half-width (1 first order, 2 PLM, 3 WENO5).  Guard cells
 * beyond a physical boundary are filled from the boundary map once and then
 * evolved like any halo cell (reading R17).  With periodic boundaries the
 * result equals the non-telescoping step exactly (same arithmetic on the same
 * values).  dt as in oracle_step (CFL of U^n). */

int oracle_step_telescoping(const ocfg* c, double* U, double t, double t_end, double dt_fixed, double* dt_used) {
    if (oracle_check_config(c)) return OERR_ARG;
    const int nv = nvar_of(c), ndim = c->ndim, S = c->rk_stages, ngk = ngk_of(c->recon);
    const int G = S * ngk;
    /* the per-dimension maps of the thick halo need at least G cells per
     * dimension (a reflect map of a deeper guard would leave the domain) */
    for (int d = 0; d < ndim; d++)
        if ((long)c->nblk[d] * c->nb[d] < G) return OERR_ARG;
    const long NB = nblocks(c), nc = cells_per_block(c);
    int g[3], pn[3];
    long np = 1;
    for (int d = 0; d < 3; d++) {
        g[d] = d < ndim ? G : 0;
        pn[d] = c->nb[d] + 2 * g[d];
        np *= pn[d];
    }
    const long pstride[3] = {1, pn[0], (long)pn[0] * pn[1]};
    double dx[3] = {dx_of(c, 0), dx_of(c, 1), dx_of(c, 2)};
    double dt = dt_fixed > 0.0 ? dt_fixed : oracle_dt(c, U, t, t_end);
    if (dt_used) *dt_used = dt;
    /* the thick-halo fill needs N_d >= G for the per-dimension maps */
    double* P = malloc(sizeof(double) * nv * NB * np);
    double* Unew = malloc(sizeof(double) * nv * NB * nc);
    if (!P || !Unew) { free(P); free(Unew); return OERR_OOM; }
    /* oracle_fill_guardcells checks nb >= ng; the thick halo may exceed nb, so
     * fill directly with the per-dimension maps (same rule as the thin fill) */
    {
        const long N[3] = {(long)c->nblk[0] * c->nb[0], (long)c->nblk[1] * c->nb[1], (long)c->nblk[2] * c->nb[2]};
        for (long b = 0; b < NB; b++) {
            long bx = b % c->nblk[0], by = (b / c->nblk[0]) % c->nblk[1], bz = b / ((long)c->nblk[0] * c->nblk[1]);
            for (int pk = 0; pk < pn[2]; pk++)
                for (int pj = 0; pj < pn[1]; pj++)
                    for (int pi = 0; pi < pn[0]; pi++) {
                        int fx, fy, fz;
                        long gx = map_dim(bx * c->nb[0] + pi - g[0], N[0], c->bc[0][0], c->bc[0][1], &fx);
                        long gy = map_dim(by * c->nb[1] + pj - g[1], N[1], c->bc[1][0], c->bc[1][1], &fy);
                        long gz = map_dim(bz * c->nb[2] + pk - g[2], N[2], c->bc[2][0], c->bc[2][1], &fz);
                        long sb = (gx / c->nb[0]) + c->nblk[0] * ((gy / c->nb[1]) + c->nblk[1] * (gz / c->nb[2]));
                        long sc = ((gz % c->nb[2]) * c->nb[1] + (gy % c->nb[1])) * c->nb[0] + (gx % c->nb[0]);
                        long pidx = ((long)pk * pn[1] + pj) * pn[0] + pi;
                        int flip[3] = {fx, fy, fz};
                        for (int v = 0; v < nv; v++) {
                            double val = U[(long)v * NB * nc + sb * nc + sc];
                            if (v >= 1 && v <= ndim && flip[v - 1]) val = -val;
                            P[(long)v * NB * np + b * np + pidx] = val;
                        }
                    }
        }
    }
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
        double* T0 = malloc(sizeof(double) * nv * np);  /* U^n on the tile   */
        double* Tp = malloc(sizeof(double) * nv * np);  /* U^(s-1)           */
        double* To = malloc(sizeof(double) * nv * np);  /* U^(s)             */
        double* W = malloc(sizeof(double) * nv * np);   /* primitives of U^(s-1) */
        double* F[3];
        for (int d = 0; d < 3; d++) F[d] = malloc(sizeof(double) * nv * np);  /* F[d] at the face below cell */
#pragma omp for schedule(static)
        for (long blk = 0; blk < NB; blk++) {
            for (int v = 0; v < nv; v++)
                for (long q = 0; q < np; q++) T0[(long)v * np + q] = Tp[(long)v * np + q] = P[(long)v * NB * np + blk * np + q];
            for (int s = 1; s <= S; s++) {
                double a, b;
                oracle_rk_coeffs(S, s, &a, &b);
                int lo[3], hi[3];  /* cells updated by this stage: [lo, hi) */
                for (int d = 0; d < 3; d++) {
                    lo[d] = d < ndim ? s * ngk : 0;
                    hi[d] = pn[d] - lo[d];
                }
                /* primitives of U^(s-1) where valid: distance >= (s-1)*ngk from the edge */
                for (int k = 0; k < pn[2]; k++)
                    for (int j = 0; j < pn[1]; j++)
                        for (int i = 0; i < pn[0]; i++) {
                            long q = ((long)k * pn[1] + j) * pn[0] + i;
                            double u[5], w[5];
                            for (int v = 0; v < nv; v++) u[v] = Tp[(long)v * np + q];
                            cons_to_prim(ndim, c->gamma, u, w);
                            for (int v = 0; v < nv; v++) W[(long)v * np + q] = w[v];
                        }
                /* face fluxes below each updated cell and below hi (faces lo..hi along d) */
                for (int d = 0; d < ndim; d++) {
                    int rot[5], ax[3];
                    rotation(ndim, d, rot, ax);
                    int flo[3] = {lo[0], lo[1], lo[2]}, fhi[3] = {hi[0], hi[1], hi[2]};
                    fhi[d] += 1;
                    for (int k = flo[2]; k < fhi[2]; k++)
                        for (int j = flo[1]; j < fhi[1]; j++)
                            for (int i = flo[0]; i < fhi[0]; i++) {
                                long right = ((long)k * pn[1] + j) * pn[0] + i;  /* face between right-1 and right */
                                double st[6 * 5], wl[5], wr[5], fr[5];
                                for (int m = 0; m < 2 * ngk; m++) {
                                    long q = right + (long)(m - ngk) * pstride[d];
                                    for (int v = 0; v < nv; v++) st[m * nv + v] = W[(long)rot[v] * np + q];
                                }
                                reconstruct(c->recon, ngk, nv, st, wl, wr);
                                riemann_ax(face_solver(c, ngk, nv, st), nv, c->gamma, ax, wl, wr, fr);
                                for (int v = 0; v < nv; v++) F[d][(long)rot[v] * np + right] = fr[v];
                            }
                }
                for (int k = lo[2]; k < hi[2]; k++)
                    for (int j = lo[1]; j < hi[1]; j++)
                        for (int i = lo[0]; i < hi[0]; i++) {
                            long q = ((long)k * pn[1] + j) * pn[0] + i;
                            double unew[5], uc[5];
                            for (int v = 0; v < nv; v++) uc[v] = Tp[(long)v * np + q];
                            for (int v = 0; v < nv; v++) {
                                double div[3] = {0.0, 0.0, 0.0};
                                for (int d = 0; d < ndim; d++)
                                    div[d] = (F[d][(long)v * np + q + pstride[d]] - F[d][(long)v * np + q]) / dx[d];
                                double L;
                                if (ndim == 1) L = -(div[0]);
                                else if (ndim == 2) L = -(div[0] + div[1]);
                                else L = -(div[0] + div[1]) - div[2];
                                if (has_grav(c)) L += grav_source(c, v, uc);  /* grvAccel */
                                unew[v] = a * T0[(long)v * np + q] + b * (uc[v] + dt * L);
                                To[(long)v * np + q] = unew[v];
                            }
                            double w[5];
                            cons_to_prim(ndim, c->gamma, unew, w);
                            int ok = w[0] > 0.0 && w[nv - 1] > 0.0;
                            for (int v = 0; v < nv; v++) ok = ok && isfinite(unew[v]);
                            if (!ok) bad = 1;
                        }
                for (int v = 0; v < nv; v++)
                    for (int k = lo[2]; k < hi[2]; k++)
                        for (int j = lo[1]; j < hi[1]; j++)
                            for (int i = lo[0]; i < hi[0]; i++) {
                                long q = ((long)k * pn[1] + j) * pn[0] + i;
                                Tp[(long)v * np + q] = To[(long)v * np + q];
                            }
            }
            for (int v = 0; v < nv; v++)
                for (int k = 0; k < c->nb[2]; k++)
                    for (int j = 0; j < c->nb[1]; j++)
                        for (int i = 0; i < c->nb[0]; i++) {
                            long q = ((long)(k + g[2]) * pn[1] + (j + g[1])) * pn[0] + (i + g[0]);
                            Unew[(long)v * NB * nc + blk * nc + ((long)k * c->nb[1] + j) * c->nb[0] + i] = Tp[(long)v * np + q];
                        }
        }
        free(T0); free(Tp); free(To); free(W);
        for (int d = 0; d < 3; d++) free(F[d]);
    }
    int st = bad ? OERR_NONPHYSICAL : OK;
    if (st == OK) memcpy(U, Unew, sizeof(double) * nv * NB * nc);
    free(P);
    free(Unew);
    return st;
}

/* =========================================================================
 * NEXT N3: fluxBuff + flux correction on a static two-level refinement, the
 * all-levels variant (lst:spark-all-levels P:1510-1523;
 * fluxBuff in Alg. 8).  Plain and slow, like everything above.
 *
 * Grid (reading R22): the coarse level is the block grid of
 * the ocfg; the coarse blocks [rlo, rhi) (per dimension) are refined by 2:
 * each is replaced by 2^ndim fine blocks of nb cells and spacing dx/2.  The
 * leaves — coarse blocks outside the box, then fine blocks of the box, each
 * set lexicographic with x fastest — are updated together with ONE dt
 * ("all blocks are updated regardless of the levels of refinement", P:1496;
 * no subcycling).  Canonical leaf state U[v][leaf][k][j][i].
 *
 * fill_guardcells at the coarse-fine boundary (reading R22): a face guard
 * cell is mapped per dimension by the boundary condition at its own level,
 * then read from the leaf that owns it: same level -> copy; a fine guard in a
 * coarse leaf -> the value of the coarse cell that contains it (piecewise-
 * constant prolongation: conservative, exact for uniform states); a coarse
 * guard over the refined box -> the mean of the 2^ndim fine cells it covers
 * (restriction).  Means are pairwise sums in a fixed order times 2^-k, exact
 * for equal values; the children (x fastest) are paired along the diagonals,
 * ((c00 + c11) + (c10 + c01)) per z layer, so that the result is invariant
 * under x<->y transposition.  Edge and corner guards are never read (star
 * stencil).
 *
 * fluxBuff (reading R23): every leaf keeps the fluxes through its 2*ndim
 * faces accumulated over the stages with the Shu-Osher weights of the
 * stage, B <- b_s (B + F^(s)) (B = 0 before stage 1), so that
 * U^(n+1) = U^n + dt sum_s c_s L^(s) implies the face's total contribution
 * is dt * B.  communicate_fluxes + flux correction, once per step after the
 * last stage: a coarse cell next to a coarse-fine face has its flux replaced
 * by the area mean of the 2^(ndim-1) fine fluxes through the same face,
 * U_c += (+1 high face / -1 low face) dt (B_c - mean B_f) / dx_c,
 * which makes the composite update conservative to round-off.
 * ========================================================================= */
typedef struct {
    ocfg c;                 /* coarse level */
    int32_t rlo[3], rhi[3]; /* refined coarse blocks, [rlo, rhi) */
} oamr;

static int amr_refined(const oamr* a, const long* cb) {
    for (int d = 0; d < 3; d++)
        if (cb[d] < a->rlo[d] || cb[d] >= a->rhi[d]) return 0;
    return 1;
}

static int amr_has_box(const oamr* a) {
    for (int d = 0; d < 3; d++)
        if (a->rhi[d] <= a->rlo[d]) return 0;
    return 1;
}

static void amr_fine_grid(const oamr* a, long* fnb) {
    for (int d = 0; d < 3; d++) fnb[d] = d < a->c.ndim ? 2L * (a->rhi[d] - a->rlo[d]) : 1;
}

int oracle_amr_check(const oamr* a) {
    const ocfg* c = &a->c;
    if (oracle_check_config(c)) return OERR_ARG;
    for (int d = 0; d < 3; d++) {
        if (a->rlo[d] < 0 || a->rhi[d] > c->nblk[d] || a->rlo[d] > a->rhi[d]) return OERR_ARG;
        if (d >= c->ndim && amr_has_box(a) && (a->rlo[d] != 0 || a->rhi[d] != 1)) return OERR_ARG;
        if (d < c->ndim && amr_has_box(a) && c->nb[d] % 2) return OERR_ARG; /* fine cells pair up */
    }
    return OK;
}

int oracle_amr_leaves(const oamr* a, long* ncoarse, long* nfine) {
    if (oracle_amr_check(a)) return OERR_ARG;
    long nc = 0;
    for (long bz = 0; bz < a->c.nblk[2]; bz++)
        for (long by = 0; by < a->c.nblk[1]; by++)
            for (long bx = 0; bx < a->c.nblk[0]; bx++) {
                long cb[3] = {bx, by, bz};
                if (!(amr_has_box(a) && amr_refined(a, cb))) nc++;
            }
    long fnb[3];
    amr_fine_grid(a, fnb);
    *ncoarse = nc;
    *nfine = amr_has_box(a) ? fnb[0] * fnb[1] * fnb[2] : 0;
    return OK;
}

/* leaf -> level and block coordinates at that level */
static void amr_leaf(const oamr* a, long leaf, int* level, long* blk) {
    long seen = 0;
    for (long bz = 0; bz < a->c.nblk[2]; bz++)
        for (long by = 0; by < a->c.nblk[1]; by++)
            for (long bx = 0; bx < a->c.nblk[0]; bx++) {
                long cb[3] = {bx, by, bz};
                if (amr_has_box(a) && amr_refined(a, cb)) continue;
                if (seen == leaf) {
                    *level = 0;
                    blk[0] = bx, blk[1] = by, blk[2] = bz;
                    return;
                }
                seen++;
            }
    long f = leaf - seen, fnb[3];
    amr_fine_grid(a, fnb);
    *level = 1;
    blk[0] = 2L * a->rlo[0] + f % fnb[0];
    blk[1] = (a->c.ndim >= 2 ? 2L * a->rlo[1] : 0) + (f / fnb[0]) % fnb[1];
    blk[2] = (a->c.ndim >= 3 ? 2L * a->rlo[2] : 0) + f / (fnb[0] * fnb[1]);
}

/* block coordinates at a level -> leaf index (-1: not a leaf) */
static long amr_leaf_of(const oamr* a, int level, const long* blk) {
    long ncl, nfl;
    oracle_amr_leaves(a, &ncl, &nfl);
    if (level == 0) {
        if (amr_has_box(a) && amr_refined(a, blk)) return -1;
        long seen = 0;
        for (long bz = 0; bz < a->c.nblk[2]; bz++)
            for (long by = 0; by < a->c.nblk[1]; by++)
                for (long bx = 0; bx < a->c.nblk[0]; bx++) {
                    long cb[3] = {bx, by, bz};
                    if (amr_has_box(a) && amr_refined(a, cb)) continue;
                    if (bx == blk[0] && by == blk[1] && bz == blk[2]) return seen;
                    seen++;
                }
        return -1;
    }
    long fnb[3], r[3];
    amr_fine_grid(a, fnb);
    for (int d = 0; d < 3; d++) {
        r[d] = blk[d] - (d < a->c.ndim ? 2L * a->rlo[d] : 0);
        if (r[d] < 0 || r[d] >= fnb[d]) return -1;
    }
    return ncl + r[0] + fnb[0] * (r[1] + fnb[1] * r[2]);
}

/* Level-L cells per dimension. */
static long amr_ncells(const oamr* a, int level, int d) {
    long n = (long)a->c.nblk[d] * a->c.nb[d];
    return d < a->c.ndim ? n << level : n;
}

/* Conserved value v of the cell with level-L global coordinates g (inside
 * the domain), from the leaf that owns it (prolongation / restriction as in
 * the header). */
static double amr_value(const oamr* a, const double* U, long nleaf, int level, const long* g, int v) {
    const ocfg* c = &a->c;
    const long nc = cells_per_block(c);
    if (level == 1) {
        long cg[3], cb[3];
        for (int d = 0; d < 3; d++) {
            cg[d] = d < c->ndim ? g[d] / 2 : g[d];
            cb[d] = cg[d] / c->nb[d];
        }
        if (!amr_refined(a, cb)) return amr_value(a, U, nleaf, 0, cg, v); /* prolongation: injection */
        long fb[3], fc[3];
        for (int d = 0; d < 3; d++) fb[d] = g[d] / c->nb[d], fc[d] = g[d] % c->nb[d];
        long leaf = amr_leaf_of(a, 1, fb);
        return U[((long)v * nleaf + leaf) * nc + (fc[2] * c->nb[1] + fc[1]) * c->nb[0] + fc[0]];
    }
    long cb[3];
    for (int d = 0; d < 3; d++) cb[d] = g[d] / c->nb[d];
    if (!(amr_has_box(a) && amr_refined(a, cb))) {
        long leaf = amr_leaf_of(a, 0, cb);
        long lc[3];
        for (int d = 0; d < 3; d++) lc[d] = g[d] % c->nb[d];
        return U[((long)v * nleaf + leaf) * nc + (lc[2] * c->nb[1] + lc[1]) * c->nb[0] + lc[0]];
    }
    /* restriction: pairwise mean of the 2^ndim fine children, x fastest */
    double s[8];
    int n = 1 << c->ndim;
    for (int q = 0; q < n; q++) {
        long fg[3] = {g[0], g[1], g[2]};
        for (int d = 0; d < c->ndim; d++) fg[d] = 2 * g[d] + ((q >> d) & 1);
        s[q] = amr_value(a, U, nleaf, 1, fg, v);
    }
    /* diagonal pairs first: the sum is invariant under x<->y transposition */
    if (n == 2) return (s[0] + s[1]) * 0.5;
    if (n == 4) return ((s[0] + s[3]) + (s[1] + s[2])) * 0.25;
    return (((s[0] + s[3]) + (s[1] + s[2])) + ((s[4] + s[7]) + (s[5] + s[6]))) * 0.125;
}

/* fill_guardcells for the leaves: P[v][leaf][padded cells] (padded layout of
 * oracle_fill_guardcells with the leaf list as the blocks); interior copied,
 * face guards per reading R22, edge/corner guards NaN (never read). */
int oracle_amr_fill(const oamr* a, const double* U, double* P) {
    if (oracle_amr_check(a)) return OERR_ARG;
    const ocfg* c = &a->c;
    long ncl, nfl;
    oracle_amr_leaves(a, &ncl, &nfl);
    const long nleaf = ncl + nfl, np = padded_cells(c);
    const int nv = nvar_of(c);
    const int g[3] = {guard_of(c, 0), guard_of(c, 1), guard_of(c, 2)};
    const int pn[3] = {c->nb[0] + 2 * g[0], c->nb[1] + 2 * g[1], c->nb[2] + 2 * g[2]};
#pragma omp parallel for schedule(dynamic)
    for (long leaf = 0; leaf < nleaf; leaf++) {
        int level;
        long blk[3];
        amr_leaf(a, leaf, &level, blk);
        for (int pk = 0; pk < pn[2]; pk++)
            for (int pj = 0; pj < pn[1]; pj++)
                for (int pi = 0; pi < pn[0]; pi++) {
                    const int loc[3] = {pi - g[0], pj - g[1], pk - g[2]};
                    int out = 0, dout = -1;
                    for (int d = 0; d < 3; d++)
                        if (loc[d] < 0 || loc[d] >= c->nb[d]) out++, dout = d;
                    const long pidx = ((long)pk * pn[1] + pj) * pn[0] + pi;
                    if (out > 1) {
                        for (int v = 0; v < nv; v++) P[((long)v * nleaf + leaf) * np + pidx] = NAN;
                        continue;
                    }
                    long gc[3];
                    for (int d = 0; d < 3; d++) gc[d] = blk[d] * c->nb[d] + loc[d];
                    int flip = 0;
                    if (dout >= 0)
                        gc[dout] = map_dim(gc[dout], amr_ncells(a, level, dout), c->bc[dout][0], c->bc[dout][1], &flip);
                    for (int v = 0; v < nv; v++) {
                        double val = amr_value(a, U, nleaf, level, gc, v);
                        if (flip && v == 1 + dout) val = -val;
                        P[((long)v * nleaf + leaf) * np + pidx] = val;
                    }
                }
    }
    return OK;
}

/* dt = C min over all leaf cells of min_d dx_L,d / (|u_d| + c)  (reading R7
 * with each leaf's own spacing), clipped to t_end - t. */
double oracle_amr_dt(const oamr* a, const double* U, double t, double t_end) {
    const ocfg* c = &a->c;
    long ncl, nfl;
    oracle_amr_leaves(a, &ncl, &nfl);
    const long nleaf = ncl + nfl, nc = cells_per_block(c);
    const int nv = nvar_of(c);
    double best = INFINITY;
    for (long leaf = 0; leaf < nleaf; leaf++) {
        const double f = leaf < ncl ? 1.0 : 0.5;
        for (long q = 0; q < nc; q++) {
            double u[5], w[5];
            for (int v = 0; v < nv; v++) u[v] = U[((long)v * nleaf + leaf) * nc + q];
            cons_to_prim(c->ndim, c->gamma, u, w);
            double cs = sqrt(c->gamma * w[nv - 1] / w[0]);
            for (int d = 0; d < c->ndim; d++) {
                double tt = f * dx_of(c, d) / (fabs(w[1 + d]) + cs);
                if (tt < best) best = tt;
            }
        }
    }
    double dt = c->cfl * best;
    if (t_end > 0.0 && dt > t_end - t) dt = t_end - t;
    return dt;
}

/* One stage on every leaf: fill, then the uniform stage per level (each
 * level's leaves as a block list with that level's spacing); the face fluxes
 * enter fluxBuff: B <- b (B + F).  B: [leaf][2 d + side][v][face cell],
 * 6 * nv * face_cells_max per leaf. */
static int amr_stage(const oamr* a, const double* Uprev, const double* Un, double sa, double sb, double dt,
                     double* Uout, double* B) {
    const ocfg* c = &a->c;
    long ncl, nfl;
    oracle_amr_leaves(a, &ncl, &nfl);
    const long nleaf = ncl + nfl, nc = cells_per_block(c), np = padded_cells(c), mf = face_cells_max(c);
    const int nv = nvar_of(c);
    double* P = malloc(sizeof(double) * nv * nleaf * np);
    if (!P) return OERR_OOM;
    oracle_amr_fill(a, Uprev, P);
    int st = OK;
    for (int level = 0; level < 2 && st == OK; level++) {
        const long l0 = level ? ncl : 0, nl = level ? nfl : ncl;
        if (nl == 0) continue;
        ocfg cl = *c;  /* the level's leaves as one block list (along x), the level's spacing */
        cl.nblk[0] = (int32_t)nl, cl.nblk[1] = 1, cl.nblk[2] = 1;
        for (int d = 0; d < 3; d++) {
            const double dxl = dx_of(c, d) * (level ? 0.5 : 1.0);
            cl.lo[d] = 0.0;
            cl.hi[d] = d < c->ndim ? dxl * (double)(d == 0 ? nl : 1) * c->nb[d] : c->hi[d] - c->lo[d];
        }
        double* Pl = malloc(sizeof(double) * nv * nl * np);
        double* Ul = malloc(sizeof(double) * nv * nl * nc);
        double* Ol = malloc(sizeof(double) * nv * nl * nc);
        double* Fl = malloc(sizeof(double) * nl * 6 * nv * mf);
        for (int v = 0; v < nv; v++) {
            memcpy(Pl + (long)v * nl * np, P + ((long)v * nleaf + l0) * np, sizeof(double) * nl * np);
            memcpy(Ul + (long)v * nl * nc, Un + ((long)v * nleaf + l0) * nc, sizeof(double) * nl * nc);
        }
        st = stage_padded_fb(&cl, Pl, Ul, sa, sb, dt, Ol, Fl);
        for (int v = 0; v < nv; v++)
            memcpy(Uout + ((long)v * nleaf + l0) * nc, Ol + (long)v * nl * nc, sizeof(double) * nl * nc);
        for (long q = 0; q < nl * 6 * nv * mf; q++) {
            double* bq = B + l0 * 6 * nv * mf + q;
            *bq = sb * (*bq + Fl[q]);
        }
        free(Pl), free(Ul), free(Ol), free(Fl);
    }
    free(P);
    return st;
}

/* communicate_fluxes + flux correction (lst:spark-all-levels): every coarse
 * cell next to a coarse-fine face.  Returns OERR_NONPHYSICAL if a corrected
 * cell has rho <= 0, p <= 0 or a non-finite value. */
static int amr_fluxcorr(const oamr* a, const double* B, double dt, double* U) {
    const ocfg* c = &a->c;
    if (!amr_has_box(a)) return OK;
    long ncl, nfl;
    oracle_amr_leaves(a, &ncl, &nfl);
    const long nleaf = ncl + nfl, nc = cells_per_block(c), mf = face_cells_max(c);
    const int nv = nvar_of(c), ndim = c->ndim;
    int bad = 0;
    for (long leaf = 0; leaf < ncl; leaf++) {
        int level;
        long blk[3];
        amr_leaf(a, leaf, &level, blk);
        for (int d = 0; d < ndim; d++)
            for (int side = 0; side < 2; side++) {
                /* the coarse block across the face (boundary map at the coarse level) */
                long nb_[3] = {blk[0], blk[1], blk[2]};
                long gface = side ? (blk[d] + 1) * c->nb[d] : blk[d] * c->nb[d] - 1;  /* coarse cell across */
                int flip;
                long gm = map_dim(gface, amr_ncells(a, 0, d), c->bc[d][0], c->bc[d][1], &flip);
                if (c->bc[d][side] != OBC_PERIODIC && (gface < 0 || gface >= amr_ncells(a, 0, d))) continue;
                nb_[d] = gm / c->nb[d];
                if (!amr_refined(a, nb_)) continue;
                /* fine cells across the face: level-1 coordinate along d */
                const long fd = side ? 2 * gm : 2 * gm + 1;
                const int e1 = d == 0 ? 1 : 0, e2 = d == 2 ? 1 : 2;  /* transverse dims, increasing */
                const int n1 = ndim > 1 ? c->nb[e1] : 1, n2 = ndim > 2 ? c->nb[e2] : 1;
                for (int t2 = 0; t2 < n2; t2++)
                    for (int t1 = 0; t1 < n1; t1++) {
                        int lc[3];
                        lc[d] = side ? c->nb[d] - 1 : 0;
                        lc[e1] = t1;
                        lc[e2] = t2;
                        if (ndim < 3) lc[2] = 0;
                        if (ndim < 2) lc[1] = 0;
                        const long cell = ((long)lc[2] * c->nb[1] + lc[1]) * c->nb[0] + lc[0];
                        const long fcl = face_cell(c, d, lc[0], lc[1], lc[2]);
                        /* the 2^(ndim-1) fine faces: transverse fine coordinates, e1 fastest */
                        double fsum[5] = {0, 0, 0, 0, 0};
                        for (int v = 0; v < nv; v++) {
                            double s4[4];
                            int nf = 1 << (ndim - 1);
                            for (int q = 0; q < nf; q++) {
                                long fg[3];
                                fg[d] = fd;
                                fg[e1] = 2 * (blk[e1] * c->nb[e1] + t1) + (ndim > 1 ? (q & 1) : 0);
                                fg[e2] = 2 * (blk[e2] * c->nb[e2] + t2) + (ndim > 2 ? ((q >> 1) & 1) : 0);
                                if (ndim < 3) fg[2] = 0;
                                if (ndim < 2) fg[1] = 0;
                                long fb[3], fl[3];
                                for (int e = 0; e < 3; e++) fb[e] = fg[e] / c->nb[e], fl[e] = fg[e] % c->nb[e];
                                const long fleaf = amr_leaf_of(a, 1, fb);
                                const long ffc = face_cell(c, d, (int)fl[0], (int)fl[1], (int)fl[2]);
                                s4[q] = B[((fleaf * 6 + 2 * d + (1 - side)) * nv + v) * mf + ffc];
                            }
                            if (nf == 1) fsum[v] = s4[0];
                            else if (nf == 2) fsum[v] = (s4[0] + s4[1]) * 0.5;
                            else fsum[v] = ((s4[0] + s4[3]) + (s4[1] + s4[2])) * 0.25;  /* diagonal pairs */
                        }
                        double u[5], w[5];
                        for (int v = 0; v < nv; v++) {
                            const double bc_ = B[((leaf * 6 + 2 * d + side) * nv + v) * mf + fcl];
                            const double corr = dt * (bc_ - fsum[v]) / dx_of(c, d);
                            double* uq = U + ((long)v * nleaf + leaf) * nc + cell;
                            *uq = side ? *uq + corr : *uq - corr;
                            u[v] = *uq;
                        }
                        cons_to_prim(ndim, c->gamma, u, w);
                        int ok = w[0] > 0.0 && w[nv - 1] > 0.0;
                        for (int v = 0; v < nv; v++) ok = ok && isfinite(u[v]);
                        if (!ok) bad = 1;
                    }
            }
    }
    return bad ? OERR_NONPHYSICAL : OK;
}

/* One SSP-RK step of the composite grid (all-levels variant): dt from every
 * leaf, the S stages with fluxBuff, then communicate_fluxes + correction.
 * correct = 0 skips the correction (for the pin that shows it is needed).
 * On failure U is unchanged. */
int oracle_amr_step(const oamr* a, double* U, double t, double t_end, double dt_fixed, int correct, double* dt_used) {
    if (oracle_amr_check(a)) return OERR_ARG;
    const ocfg* c = &a->c;
    long ncl, nfl;
    oracle_amr_leaves(a, &ncl, &nfl);
    const long nleaf = ncl + nfl, n = (long)nvar_of(c) * nleaf * cells_per_block(c);
    const long nb_ = nleaf * 6 * nvar_of(c) * face_cells_max(c);
    double dt = dt_fixed > 0.0 ? dt_fixed : oracle_amr_dt(a, U, t, t_end);
    if (dt_used) *dt_used = dt;
    double* S0 = malloc(sizeof(double) * n);
    double* S1 = malloc(sizeof(double) * n);
    double* B = calloc(nb_, sizeof(double));
    if (!S0 || !S1 || !B) { free(S0), free(S1), free(B); return OERR_OOM; }
    const double* prev = U;
    double* bufs[2] = {S0, S1};
    int st = OK;
    for (int s = 1; s <= c->rk_stages && st == OK; s++) {
        double sa, sb;
        oracle_rk_coeffs(c->rk_stages, s, &sa, &sb);
        double* out = bufs[(s - 1) & 1];
        st = amr_stage(a, prev, U, sa, sb, dt, out, B);
        prev = out;
    }
    double* res = (double*)prev;
    if (st == OK && correct) st = amr_fluxcorr(a, B, dt, res);
    if (st == OK) memcpy(U, res, sizeof(double) * n);
    free(S0), free(S1), free(B);
    return st;
}

int oracle_amr_run(const oamr* a, double* U, double t_end, long max_steps, double* t, long* nsteps) {
    int st = OK;
    while (st == OK) {
        if (t_end > 0.0 && *t >= t_end * (1.0 - 1e-14)) break;
        if (max_steps > 0 && *nsteps >= max_steps) break;
        double dt;
        st = oracle_amr_step(a, U, *t, t_end, 0.0, 1, &dt);
        if (st == OK) {
            *t += dt;
            *nsteps += 1;
        }
    }
    return st;
}
