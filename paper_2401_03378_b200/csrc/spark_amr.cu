// spark_amr.cu — NEXT N3: fluxBuff + flux correction on a static two-level
// refinement, the all-levels variant (lst:spark-all-levels
// P:1510-1523; fluxBuff in Alg. 8).  Readings R22/R23.
//
// The coarse block grid of a spark_config has the coarse blocks [rlo, rhi)
// replaced by 2^ndim fine blocks each (spacing dx/2).  Leaves = coarse blocks
// outside the box, then fine blocks of the box (each lexicographic, x
// fastest); state U[v][leaf][k][j][i] (the ABI's canonical layout with the
// leaf list as the blocks).  All leaves advance with one dt (no subcycling).
//
// Per stage (lst:spark-nontelescoping body, with the coarse-fine guard rules):
//   KA amr_fill_leaf  padded primitive tiles W[v][leaf][padded], one CTA per
//        leaf: interior cells converted in place; face guards gathered through
//        a host-built map (same-level copy, piecewise-constant prolongation,
//        diagonal-pairwise restriction mean; reflect flips the momentum)
//   KB amr_face    every face of every leaf: calcLims + calcFlux (the
//        product's device reconstruction / Riemann / shockDet) -> F; the
//        leaf-boundary faces also enter fluxBuff, B <- b_s (B + F)
//   KC amr_update  updSoln: U^(s) = a U^n + b (U^(s-1) + dt L)
//   KB+KC fused for 3-D 16^3 leaves and face-centric schemes (amr_leaf):
//        KB1's plane march over the padded tiles, no face-flux array
// Per step after the last stage: communicate_fluxes + correction (KD
// amr_corr, one launch per direction so no two threads touch one cell),
// then the CFL minimum of the corrected state (KE amr_cfl) for the next dt.
//
// The padded tiles go through HBM (one write, one read per stage); the face
// fluxes only on the unfused KB/KC path (other shapes and WENO).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/spark.h"
#include "spark_device.cuh"
#include "spark_internal.h"

namespace spark {
namespace {

using namespace dev;

struct AmrGeo {
    int ndim, nv, ng, ngk, recon;
    int nb[3], pn[3];
    long long nleaf, ncl, nc, np;
    long long nfd[3], Fo[3], NF;  // faces per leaf per direction, offsets, total
    long long mf;                 // fluxBuff cells per face slot
    double rdx[2][3];             // 1/dx per level
    double gamma, cfl, shock_thresh;
};

struct GuardE {
    long long dst;  // leaf * np + padded index
    long long src;  // leaf * nc + cell (first child for a restriction); kind 3: slot of the received guards
    int kind;       // 1 copy, 2 restriction, 3 received from another rank; bits 4+d: negate momentum d (reflect)
    int pad;
};

struct CorrE {
    long long cell;   // coarse leaf * nc + cell
    long long bc;     // (leaf * 6 + slot) * mf + face cell of the coarse side
    long long bf[4];  // the fine faces (same encoding), 2^(ndim-1) of them; -(slot+1): received from another rank
    int side;         // 1: interface on the coarse cell's high face
    int pad;
};

__host__ __device__ inline long long face_cell(const AmrGeo& g, int d, int i, int j, int k) {
    if (d == 0) return (long long)k * g.nb[1] + j;
    if (d == 1) return (long long)k * g.nb[0] + i;
    return (long long)j * g.nb[0] + i;
}

// ---------------------------------------------------------------- KA
// conserved value v of a guard source: copy, or the restriction mean of the
// 2^ndim fine children (diagonal pairs, reading R22)
template <int NV>
__device__ __forceinline__ double guard_value(const AmrGeo& g, const double* __restrict__ s, int kind) {
    const long long ox = 1, oy = g.nb[0], oz = (long long)g.nb[0] * g.nb[1];
    if (kind == 1) return s[0];
    if (NV == 3) return (s[0] + s[ox]) * 0.5;
    if (NV == 4) return ((s[0] + s[ox + oy]) + (s[ox] + s[oy])) * 0.25;
    return (((s[0] + s[ox + oy]) + (s[ox] + s[oy])) + ((s[oz] + s[oz + ox + oy]) + (s[oz + ox] + s[oz + oy]))) *
           0.125;
}

// KA in one launch, one CTA per leaf: its interior cells, the faces whose
// guards are a plain copy of one same-level leaf of this rank (sface[leaf*6 +
// face slot] = that leaf, found by the host from the guard map: contiguous
// rows, no per-cell map entry), then the remaining guard entries (coarse-fine
// faces, physical boundaries, other ranks; the map lists them leaf by leaf,
// goff[leaf] is the first).  Same values as the per-entry map.
template <int NV>
__global__ void __launch_bounds__(256) amr_fill_leaf_kernel(const AmrGeo g, const double* __restrict__ u,
                                                            const GuardE* __restrict__ ge,
                                                            const long long* __restrict__ goff,
                                                            const long long* __restrict__ sface,
                                                            const double* __restrict__ grecv, double* __restrict__ w,
                                                            int to_prim, int interior, DevScalars* sc) {
    const long long vs = g.nleaf * g.nc, vp = g.nleaf * g.np;
    const int gx = g.ng, gy = g.ndim >= 2 ? g.ng : 0, gz = g.ndim >= 3 ? g.ng : 0;
    const long long leaf = blockIdx.x;
    bool ok = true;
#pragma unroll 4
    for (long long c = threadIdx.x; interior && c < g.nc; c += blockDim.x) {
        const long long q = leaf * g.nc + c;
        const int i = (int)(c % g.nb[0]), j = (int)((c / g.nb[0]) % g.nb[1]), k = (int)(c / ((long long)g.nb[0] * g.nb[1]));
        const long long p = leaf * g.np + ((long long)(k + gz) * g.pn[1] + (j + gy)) * g.pn[0] + (i + gx);
        double uu[NV], ww[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) uu[v] = u[v * vs + q];
        if (to_prim) ok &= cons_to_prim<NV>(uu, ww, g.gamma - 1.0);
#pragma unroll
        for (int v = 0; v < NV; v++) w[v * vp + p] = to_prim ? ww[v] : uu[v];
    }
    for (int f = 0; interior && f < 2 * g.ndim; f++) {  // same-level faces (the fused leaf kernel copies them itself)
        const long long src_leaf = sface[leaf * 6 + f];
        if (src_leaf < 0) continue;  // CTA-uniform
        const int d = f >> 1, hi = f & 1;
        const int a = d == 0 ? 1 : 0, b = d == 2 ? 1 : 2;  // the other two dims, x first when it is one
        const int na = g.nb[a], n = g.ng * na * g.nb[b];
        for (int m = threadIdx.x; m < n; m += blockDim.x) {
            int t, ia, ib;  // layer, coordinates along a and b (the fastest index runs along x)
            if (d == 0) { t = m % g.ng; ia = (m / g.ng) % na; ib = m / (g.ng * na); }
            else { ia = m % na; t = (m / na) % g.ng; ib = m / (na * g.ng); }
            int c[3], q[3];
            c[a] = q[a] = ia;
            c[b] = q[b] = ib;
            c[d] = hi ? g.nb[d] + t : t - g.ng;    // guard cell of this leaf
            q[d] = hi ? t : g.nb[d] - g.ng + t;    // the neighbour's cell
            const long long dst = leaf * g.np + ((long long)(c[2] + gz) * g.pn[1] + (c[1] + gy)) * g.pn[0] + (c[0] + gx);
            const long long src = src_leaf * g.nc + ((long long)q[2] * g.nb[1] + q[1]) * g.nb[0] + q[0];
            double uu[NV], ww[NV];
#pragma unroll
            for (int v = 0; v < NV; v++) uu[v] = u[v * vs + src];
            if (to_prim) ok &= cons_to_prim<NV>(uu, ww, g.gamma - 1.0);
#pragma unroll
            for (int v = 0; v < NV; v++) w[v * vp + dst] = to_prim ? ww[v] : uu[v];
        }
    }
    const long long e1 = goff[leaf + 1];
#pragma unroll 4
    for (long long e = goff[leaf] + threadIdx.x; e < e1; e += blockDim.x) {
        const GuardE E = ge[e];
        double uu[NV], ww[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) {
            double val = (E.kind & 15) == 3 ? grecv[E.src * NV + v] : guard_value<NV>(g, u + v * vs + E.src, E.kind & 15);
            if (v >= 1 && v < NV - 1 && ((E.kind >> (3 + v)) & 1)) val = -val;
            uu[v] = val;
        }
        if (to_prim) ok &= cons_to_prim<NV>(uu, ww, g.gamma - 1.0);
#pragma unroll
        for (int v = 0; v < NV; v++) w[v * vp + E.dst] = to_prim ? ww[v] : uu[v];
    }
    if (!ok) flag_nonphysical(sc);
}

// ---------------------------------------------------------------- KB
template <int RECON>
__device__ __forceinline__ void recon_face(const double* s, double& wl, double& wr) {
    // s[0..2NGK-1] = W_{i-NGK+1..i+NGK}: wl = hi edge of cell i, wr = lo edge of cell i+1
    constexpr int R = StencilOf<RECON>::NG - 1;
    constexpr int K = StencilOf<RECON>::NG;
    double lo, hi;
    recon_cell<RECON>(s + (K - 1 - R), lo, hi);
    wl = hi;
    recon_cell<RECON>(s + (K - R), lo, hi);
    wr = lo;
}

template <int NV, int RS, int D, int RECON>
__device__ __forceinline__ void amr_face_solve(const AmrGeo& g, const double* __restrict__ w, long long right,
                                               long long stride, double* f) {
    constexpr int K = StencilOf<RECON>::NG;
    const long long vp = g.nleaf * g.np;
    double wl[NV], wr[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) {
        double s[6];
#pragma unroll
        for (int m = 0; m < 2 * K; m++) s[m] = w[v * vp + right + (m - K) * stride];
        recon_face<RECON>(s, wl[v], wr[v]);
    }
    if (RECON != 0 && !(positive(wl[0]) && positive(wl[NV - 1]) && positive(wr[0]) && positive(wr[NV - 1]))) {
#pragma unroll
        for (int v = 0; v < NV; v++) {
            wl[v] = w[v * vp + right - stride];
            wr[v] = w[v * vp + right];
        }
    }
    bool shk = false;
    if constexpr (RS == 2) {
        double uu[4], pp[4], rr[4];
#pragma unroll
        for (int m = 0; m < 4; m++) {
            const long long q = right + (m - 2) * stride;
            uu[m] = w[(1 + D) * vp + q];
            pp[m] = w[(NV - 1) * vp + q];
            rr[m] = w[q];
        }
        shk = shock_face(uu, pp, rr, g.shock_thresh, g.gamma);
    }
    face_flux<NV, RS, D>(wl, wr, shk, g.gamma, 1.0 / (g.gamma - 1.0), f);
}

template <int NDIM, int RS>
__global__ void amr_face_kernel(const AmrGeo g, const double* __restrict__ w, double* __restrict__ F,
                                double* __restrict__ B, double bco) {
    constexpr int NV = NDIM + 2;
    const long long total = g.nleaf * g.NF;
    const long long fvs = g.nleaf * g.NF, bvs = g.nleaf * 6 * g.mf;
    const int gx = g.ng, gy = NDIM >= 2 ? g.ng : 0, gz = NDIM >= 3 ? g.ng : 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long leaf = e / g.NF;
        long long r = e - leaf * g.NF;
        const int d = r < g.Fo[1] ? 0 : (r < g.Fo[2] ? 1 : 2);
        r -= g.Fo[d];
        int fn[3] = {g.nb[0], g.nb[1], g.nb[2]};
        fn[d] += 1;
        const int i = (int)(r % fn[0]), j = (int)((r / fn[0]) % fn[1]), k = (int)(r / ((long long)fn[0] * fn[1]));
        const long long right = leaf * g.np + ((long long)(k + gz) * g.pn[1] + (j + gy)) * g.pn[0] + (i + gx);
        const long long stride = d == 0 ? 1 : (d == 1 ? g.pn[0] : (long long)g.pn[0] * g.pn[1]);
        double f[NV];
#define AMR_SOLVE(DD)                                                                                    \
    switch (g.recon) {                                                                                   \
        case 0: amr_face_solve<NV, RS == 2 ? 1 : RS, DD, 0>(g, w, right, stride, f); break;             \
        case 1: amr_face_solve<NV, RS, DD, 1>(g, w, right, stride, f); break;                           \
        case 3: amr_face_solve<NV, RS, DD, 3>(g, w, right, stride, f); break;                           \
        case 4: amr_face_solve<NV, RS, DD, 4>(g, w, right, stride, f); break;                           \
        default: amr_face_solve<NV, RS, DD, 2>(g, w, right, stride, f); break;                          \
    }
        if (d == 0) {
            AMR_SOLVE(0)
        } else if (NDIM >= 2 && d == 1) {
            AMR_SOLVE((NDIM >= 2 ? 1 : 0))
        } else if (NDIM >= 3) {
            AMR_SOLVE((NDIM >= 3 ? 2 : 0))
        }
#undef AMR_SOLVE
#pragma unroll
        for (int v = 0; v < NV; v++) F[v * fvs + e] = f[v];
        const int at[3] = {i, j, k};
        if (at[d] == 0 || at[d] == g.nb[d]) {  // a face of the leaf: fluxBuff (reading R23)
            const int slot = 2 * d + (at[d] == 0 ? 0 : 1);
            const long long bi = (leaf * 6 + slot) * g.mf + face_cell(g, d, i, j, k);
#pragma unroll
            for (int v = 0; v < NV; v++) B[v * bvs + bi] = bco * (B[v * bvs + bi] + f[v]);
        }
    }
}

// ---------------------------------------------------------------- KC
template <int NDIM>
__global__ void amr_update_kernel(const AmrGeo g, const double* __restrict__ F, const double* __restrict__ uprev,
                                  const double* __restrict__ un, double* __restrict__ uout, double a, double b,
                                  const DevScalars* __restrict__ sc) {
    constexpr int NV = NDIM + 2;
    const long long vs = g.nleaf * g.nc, fvs = g.nleaf * g.NF;
    const double dt = sc->dt;
    if (!sc->active) {  // t >= t_end or frozen after a failure: U^(s) = U^(s-1)
        for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < vs * NV;
             q += (long long)gridDim.x * blockDim.x)
            uout[q] = uprev[q];
        return;
    }
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < vs;
         q += (long long)gridDim.x * blockDim.x) {
        const long long leaf = q / g.nc, c = q - leaf * g.nc;
        const int i = (int)(c % g.nb[0]), j = (int)((c / g.nb[0]) % g.nb[1]), k = (int)(c / ((long long)g.nb[0] * g.nb[1]));
        const int lev = leaf < g.ncl ? 0 : 1;
        long long lo[3], hi[3];
#pragma unroll
        for (int d = 0; d < NDIM; d++) {
            int fn[3] = {g.nb[0], g.nb[1], g.nb[2]};
            fn[d] += 1;
            const int at[3] = {i, j, k};
            int up[3] = {i, j, k};
            up[d] = at[d] + 1;
            lo[d] = leaf * g.NF + g.Fo[d] + ((long long)k * fn[1] + j) * fn[0] + i;
            hi[d] = leaf * g.NF + g.Fo[d] + ((long long)up[2] * fn[1] + up[1]) * fn[0] + up[0];
        }
#pragma unroll
        for (int v = 0; v < NV; v++) {
            const double dfx = (F[v * fvs + hi[0]] - F[v * fvs + lo[0]]) * g.rdx[lev][0];
            double Lv;
            if (NDIM == 1) {
                Lv = -dfx;
            } else {
                const double dfy = (F[v * fvs + hi[1]] - F[v * fvs + lo[1]]) * g.rdx[lev][1];
                if (NDIM == 2) Lv = -(dfx + dfy);
                else Lv = -(dfx + dfy) - (F[v * fvs + hi[2]] - F[v * fvs + lo[2]]) * g.rdx[lev][2];
            }
            const double u0 = uprev[v * vs + q];
            const double unn = a != 0.0 ? un[v * vs + q] : 0.0;
            uout[v * vs + q] = fma(b, fma(dt, Lv, u0), a * unn);
        }
    }
}

// ------------------------------------------------------- KB+KC fused (3-D)
// 16^3 leaves, face-centric schemes (first order, PLM, PLM-MC): one CTA per
// leaf marches its 16 planes like KB1 (one thread per column).  The padded
// primitive planes of the tile W that KA filled (guards included, so no
// gathering) stream into a 5-slot shared-memory ring (planes k-1 .. k+3, each
// copied by 16-byte cp.async four planes ahead of its first use), and each
// face is solved once: the own +x / +y / +z faces, on warp 0 the 32 faces at
// x = 0 and y = 0 of the plane (y faces in the x frame with u_x <-> u_y
// swapped, bitwise identical), the z face below the first plane in the
// prologue.  -x fluxes come from the left lane (shuffle), -y fluxes from the
// row below through shared memory (double-buffered by plane parity: one
// barrier per plane), -z from the previous plane (register).  The update and
// the fluxBuff accumulation of the leaf's six faces follow in the same pass,
// so KB's face-flux array never exists.  Same face arithmetic as KB
// (reconstruction, positivity fallback, shockDet, Riemann).
constexpr int kLeafN = 16, kLeafSlots = 5, kLeafNG = 2;

__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}

template <int RECON, int RS>
__global__ void __launch_bounds__(256, 2)
    amr_leaf_kernel(const AmrGeo g, const double* __restrict__ w, const double* __restrict__ uprev,
                    const double* __restrict__ un, double* __restrict__ uout, double* __restrict__ B,
                    const long long* __restrict__ sface, double a, double bco, DevScalars* __restrict__ sc) {
    constexpr int NV = 5, N = kLeafN, NS = kLeafSlots;
    extern __shared__ double smem[];
    constexpr int gd = kLeafNG, pn0 = N + 2 * gd;  // the tile's guard depth (leaf_fused)
    constexpr int PL = pn0 * pn0;                   // cells of a padded plane
    double* const ring = smem;                  // [NS][NV][PL]
    double* const XA = ring + NS * NV * PL;     // [2][NV][N]: x face 0 of each row
    double* const YA = XA + 2 * NV * N;         // [2][NV][(N + 1) N]: y faces [row face][column]
    // fluxBuff values of the plane's x / y leaf faces (slots 0-3), staged by
    // cp.async a plane ahead: [2][4][NV][N] (the read-modify-write of B would
    // otherwise wait on HBM in every plane)
    double* const BS = YA + 2 * NV * (N + 1) * N;
    const long long leaf = blockIdx.x;
    const int tid = threadIdx.x, ti = tid % N, tj = tid / N;
    const int lev = leaf < g.ncl ? 0 : 1;
    const double r0 = g.rdx[lev][0], r1 = g.rdx[lev][1], r2 = g.rdx[lev][2];
    const double dt = sc->dt, gamma = g.gamma, gm1i = 1.0 / (g.gamma - 1.0);
    const bool active = sc->active != 0;
    const long long vp = g.nleaf * g.np, vs = g.nleaf * g.nc, bvs = g.nleaf * 6 * g.mf;
    const double* const Wl = w + leaf * g.np;
    auto plane = [&](int z) { return ring + ((z + 2 * NS) % NS) * NV * PL; };
    const int own = (tj + gd) * pn0 + ti + gd;  // this column's cell in a padded plane
    // padded plane z (all variables) into its slot, 16-byte copies.  Interior
    // plane: its N x N interior as CONSERVED values straight from U^(s-1);
    // the guard frame face by face: from the same-level neighbour's U^(s-1)
    // (conserved) where sface names one, else from W (primitive, filled by
    // KA).  Guard plane (z < 0 or z >= N): only its centre is ever read (the
    // own column's z stencil): from the neighbour below / above, else W.
    // The conserved cells are converted in place by convert() a plane later.
    long long sf[6];
#pragma unroll
    for (int f = 0; f < 6; f++) sf[f] = sface[leaf * 6 + f];
    auto load_plane = [&](int z) {
        double* dst = plane(z);
        const double* wz = Wl + (long long)(z + gd) * PL;  // W plane z
        if (z < 0 || z >= N) {
            const long long L = sf[z < 0 ? 4 : 5];
            const double* uz = uprev + L * g.nc + (long long)(z < 0 ? z + N : z - N) * N * N;
            for (int e = tid; e < NV * (N * N / 2); e += blockDim.x) {
                const int v = e / (N * N / 2), c = e - v * (N * N / 2);
                const int r = c / (N / 2), x = 2 * (c - r * (N / 2));
                const int pp = (r + gd) * pn0 + gd + x;
                cp_async16(dst + v * PL + pp, L >= 0 ? uz + v * vs + r * N + x : wz + v * vp + pp);
            }
            return;
        }
        constexpr int nint = N * N / 2, per = nint + 4 * N;  // pieces per variable: interior + 4 frame sides
        const long long zo = (long long)z * N * N;
        for (int e = tid; e < NV * per; e += blockDim.x) {
            const int v = e / per;
            int c = e - v * per;
            if (c < nint) {  // interior row r, pieces of 2
                const int r = c / (N / 2), x = 2 * (c - r * (N / 2));
                cp_async16(dst + v * PL + (r + gd) * pn0 + gd + x, uprev + v * vs + leaf * g.nc + zo + r * N + x);
                continue;
            }
            c -= nint;
            const int f = c / N, k = c - f * N;  // frame side f (x-, x+, y-, y+), piece k
            int pp, sc;                           // padded position, neighbour cell (in its plane)
            if (f < 2) {  // 2 cells of row k
                pp = (k + gd) * pn0 + (f ? gd + N : 0);
                sc = k * N + (f ? 0 : N - gd);
            } else {      // 2 cells of column pair 2 (k % 8) in row k / 8 of the frame
                const int rr = k / (N / 2), x = 2 * (k - rr * (N / 2));
                pp = (f == 2 ? rr : gd + N + rr) * pn0 + gd + x;
                sc = (f == 2 ? N - gd + rr : rr) * N + x;
            }
            const long long L = sf[f];
            cp_async16(dst + v * PL + pp, L >= 0 ? uprev + v * vs + L * g.nc + zo + sc : wz + v * vp + pp);
        }
    };
    bool ok = true;
    auto cvt = [&](double* c) {  // one cell of a slot: conserved -> primitive in place
        double u[NV], wv[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) u[v] = c[v * PL];
        ok &= cons_to_prim<NV>(u, wv, g.gamma - 1.0);
#pragma unroll
        for (int v = 0; v < NV; v++) c[v * PL] = wv[v];
    };
    // the conserved cells of plane z: this column's centre cell (interior
    // planes; guard planes copied from a neighbour) and, on threads 0-127,
    // one frame cell of a side copied from a neighbour
    auto convert = [&](int z) {
        const bool inner = z >= 0 && z < N;
        if (inner || sf[z < 0 ? 4 : 5] >= 0) cvt(plane(z) + own);
        if (inner && tid < 4 * 2 * N) {
            const int f = tid / (2 * N), k = tid - f * 2 * N;
            if (sf[f] >= 0) {
                int pp;
                if (f < 2) pp = (k / gd + gd) * pn0 + (f ? gd + N : 0) + k % gd;
                else pp = (f == 2 ? k / N : gd + N + k / N) * pn0 + gd + k % N;
                cvt(plane(z) + pp);
            }
        }
    };
    auto stage_b = [&](int z) {  // fluxBuff of plane z's x / y leaf faces -> BS[z & 1]
        double* dst = BS + (z & 1) * 4 * NV * N;
        for (int e = tid; e < 4 * NV * (N / 2); e += blockDim.x) {
            const int sv = e / (N / 2), c = e - sv * (N / 2);  // sv = slot * NV + v
            const int slot = sv / NV, v = sv - slot * NV;
            cp_async16(dst + sv * N + 2 * c, B + v * bvs + (leaf * 6 + slot) * g.mf + (long long)z * N + 2 * c);
        }
    };
    auto commit = [] { asm volatile("cp.async.commit_group;\n" ::: "memory"); };
    // Riemann flux from the two states (+ shock flag); D 0 / 1 (x frame) / 2
    auto finish = [&](double* wl, double* wr, bool shk, int D, bool swapxy, double* f) {
        if (D == 2) {
            face_flux<NV, RS, 2>(wl, wr, shk, gamma, gm1i, f);
        } else {
            if (swapxy) {  // a y face solved in the x frame
                double t = wl[1]; wl[1] = wl[2]; wl[2] = t;
                t = wr[1]; wr[1] = wr[2]; wr[2] = t;
            }
            face_flux<NV, RS, 0>(wl, wr, shk, gamma, gm1i, f);
            if (swapxy) {
                const double t = f[1];
                f[1] = f[2];
                f[2] = t;
            }
        }
    };
    // face between the cells q[1] and q[2] of a line q[0..3] (variable 0; the
    // other variables PL further), normal variable 1 + D
    auto solve = [&](const double* const* q, int D, bool swapxy, double* f) {
        double wl[NV], wr[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) {
            if (RECON == 0) {
                wl[v] = q[1][v * PL];
                wr[v] = q[2][v * PL];
            } else {
                face_states<RECON>(q[0][v * PL], q[1][v * PL], q[2][v * PL], q[3][v * PL], wl[v], wr[v]);
            }
        }
        if (RECON != 0 && !(positive(wl[0]) && positive(wl[NV - 1]) && positive(wr[0]) && positive(wr[NV - 1]))) {
#pragma unroll
            for (int v = 0; v < NV; v++) {
                wl[v] = q[1][v * PL];
                wr[v] = q[2][v * PL];
            }
        }
        bool shk = false;
        if constexpr (RS == 2) {
            double uu[4], pp[4], rr[4];
#pragma unroll
            for (int m = 0; m < 4; m++) {
                uu[m] = q[m][(1 + D) * PL];
                pp[m] = q[m][(NV - 1) * PL];
                rr[m] = q[m][0];
            }
            shk = shock_face(uu, pp, rr, g.shock_thresh, gamma);
        }
        finish(wl, wr, shk, D, swapxy, f);
    };
    auto line = [&](const double* c, int st, const double** q) {  // cells c-2st .. c+st
        q[0] = c - 2 * st;
        q[1] = c - st;
        q[2] = c;
        q[3] = c + st;
    };
    auto zline = [&](int z, const double** q) {  // this column, planes z-2 .. z+1
        for (int m = 0; m < 4; m++) q[m] = plane(z - 2 + m) + own;
    };
    auto fbuf = [&](int slot, long long cell, const double* f) {  // fluxBuff, reading R23
        const long long bi = (leaf * 6 + slot) * g.mf + cell;
#pragma unroll
        for (int v = 0; v < NV; v++) B[v * bvs + bi] = bco * (B[v * bvs + bi] + f[v]);
    };
    // the same for the x / y leaf faces of plane z from the staged values
    auto fbuf_s = [&](int z, int slot, int i, const double* f) {
        const double* bs = BS + (z & 1) * 4 * NV * N + slot * NV * N + i;
        const long long bi = (leaf * 6 + slot) * g.mf + (long long)z * N + i;
#pragma unroll
        for (int v = 0; v < NV; v++) B[v * bvs + bi] = bco * (bs[v * N] + f[v]);
    };

    // prologue: planes -2 .. 2, the z face below plane 0, then plane 3 into
    // plane -2's slot; the fluxBuff values of the two z leaf faces of this
    // column (read-modify-written in the prologue and after the last plane)
    // requested into L2 first
#pragma unroll
    for (int v = 0; v < NV; v++)
        for (int slot = 4; slot < 6; slot++)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(B + v * bvs + (leaf * 6 + slot) * g.mf + tj * N + ti));
    for (int z = -2; z <= 2; z++) load_plane(z);
    stage_b(0);
    commit();
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    for (int z = -2; z <= 2; z++) convert(z);  // read by this thread first, by others after the next barrier
    double fzlo[NV], fzhi[NV];
    {
        const double* q[4];
        zline(0, q);
        solve(q, 2, false, fzlo);
    }
    fbuf(4, (long long)tj * N + ti, fzlo);
    __syncthreads();  // plane -2 read by every thread
    load_plane(3);
    commit();
    // (an L2 prefetch of both S4 operands one or two planes ahead measured
    // slower: 6.42 -> 5.98 G zone-updates/s; U^(s-1) of the plane is in L2
    // from the plane copy anyway)
    for (int kk = 0; kk < N; kk++) {
        const int pb = kk & 1;
        if (a != 0.0) {  // U^n of this plane into L2 while S3 runs (as KB1): 7.48 -> 7.78 G (a plane earlier: same)
            const long long c = leaf * g.nc + ((long long)kk * N + tj) * N + ti;
#pragma unroll
            for (int v = 0; v < NV; v++) asm volatile("prefetch.global.L2 [%0];" ::"l"(un + v * vs + c));
        }
        double* const XK = XA + pb * NV * N;
        double* const YK = YA + pb * NV * (N + 1) * N;
        const double* const cur = plane(kk);
        // ---------------------------------------------------------- S3
        double fx[NV];
        {
            const double* q[4];
            line(cur + own + 1, 1, q);
            solve(q, 0, false, fx);
            double fy[NV];
            line(cur + own + pn0, pn0, q);
            solve(q, 1, true, fy);
#pragma unroll
            for (int v = 0; v < NV; v++) YK[v * (N + 1) * N + (tj + 1) * N + ti] = fy[v];
            zline(kk + 1, q);
            solve(q, 2, false, fzhi);
        }
        if (tid < 32) {  // warp 0: x face 0 of row q (lanes 0-15), y face 0 of column q (16-31)
            const bool isy = tid >= 16;
            const int r = tid & 15;
            const double* q[4];
            if (isy) line(cur + gd * pn0 + r + gd, pn0, q);
            else line(cur + (r + gd) * pn0 + gd, 1, q);
            double fb[NV];
            solve(q, isy ? 1 : 0, isy, fb);
#pragma unroll
            for (int v = 0; v < NV; v++) {
                if (isy) YK[v * (N + 1) * N + r] = fb[v];
                else XK[v * N + r] = fb[v];
            }
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // plane kk+3 (issued a plane ago) landed
        __syncthreads();
        // ---------------------------------------------------------- S4
        // plane kk+4 into plane kk-1's slot (read by S3 of plane kk only) and the
        // fluxBuff values of plane kk+1 (BS[(kk+1) & 1], last read in S4(kk-1))
        if (kk + 3 < N + gd) convert(kk + 3);  // landed before this barrier; first read by S3(kk+1) (own column)
        if (kk + 4 < N + 2) load_plane(kk + 4);
        if (kk + 1 < N) stage_b(kk + 1);
        commit();
        double fxm[NV], fym[NV], fyp[NV];
        const long long cidx = leaf * g.nc + ((long long)kk * N + tj) * N + ti;
#pragma unroll
        for (int v = 0; v < NV; v++) {
            const double nbr = __shfl_up_sync(0xffffffffu, fx[v], 1);
            fxm[v] = ti == 0 ? XK[v * N + tj] : nbr;
            fym[v] = YK[v * (N + 1) * N + tj * N + ti];
            fyp[v] = YK[v * (N + 1) * N + (tj + 1) * N + ti];
            const double Lv = -((fx[v] - fxm[v]) * r0 + (fyp[v] - fym[v]) * r1) - (fzhi[v] - fzlo[v]) * r2;
            const double u0 = uprev[v * vs + cidx];
            const double unn = a != 0.0 ? un[v * vs + cidx] : 0.0;
            uout[v * vs + cidx] = active ? fma(bco, fma(dt, Lv, u0), a * unn) : u0;
        }
        if (ti == 0) fbuf_s(kk, 0, tj, fxm);
        if (ti == N - 1) fbuf_s(kk, 1, tj, fx);
        if (tj == 0) fbuf_s(kk, 2, ti, fym);
        if (tj == N - 1) fbuf_s(kk, 3, ti, fyp);
        if (kk == N - 1) fbuf(5, (long long)tj * N + ti, fzhi);
#pragma unroll
        for (int v = 0; v < NV; v++) fzlo[v] = fzhi[v];
    }
    if (!ok) flag_nonphysical(sc);
}

// ---------------------------------------------------------------- KD
template <int NV>
__global__ void amr_corr_kernel(const AmrGeo g, const CorrE* __restrict__ ce, long long n, int d,
                                const double* __restrict__ B, const double* __restrict__ frecv, double* __restrict__ u,
                                const double* __restrict__ dtp, DevScalars* sc) {
    const long long vs = g.nleaf * g.nc, bvs = g.nleaf * 6 * g.mf;
    const double dt = *dtp;
    bool ok = true;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const CorrE E = ce[e];
        double uu[NV], ww[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) {
            const double* bv = B + v * bvs;
            // a fine face on this rank, or received from the rank that owns it
            auto fb = [&](int k) { return E.bf[k] >= 0 ? bv[E.bf[k]] : frecv[(-E.bf[k] - 1) * NV + v]; };
            double m;
            if (NV == 3) m = fb(0);
            else if (NV == 4) m = (fb(0) + fb(1)) * 0.5;
            else m = ((fb(0) + fb(3)) + (fb(1) + fb(2))) * 0.25;  // diagonal pairs
            const double corr = dt * (bv[E.bc] - m) * g.rdx[0][d];
            double* uq = u + v * vs + E.cell;
            const double val = E.side ? *uq + corr : *uq - corr;
            *uq = val;
            uu[v] = val;
        }
        ok &= cons_to_prim<NV>(uu, ww, g.gamma - 1.0);
    }
    if (!ok) flag_nonphysical(sc);
}

// ------------------------------------------------ communicate (multi-rank)
// guard values another rank needs: copy or restriction of own cells, [item][v]
template <int NV>
__global__ void amr_gpack_kernel(const AmrGeo g, const double* __restrict__ u, const GuardE* __restrict__ it,
                                 long long n, double* __restrict__ out) {
    const long long vs = g.nleaf * g.nc;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
        const GuardE E = it[e];
#pragma unroll
        for (int v = 0; v < NV; v++) out[e * NV + v] = guard_value<NV>(g, u + v * vs + E.src, E.kind & 15);
    }
}

// fine-face fluxBuff values another rank's correction needs (communicate_fluxes), [item][v]
template <int NV>
__global__ void amr_fpack_kernel(const AmrGeo g, const double* __restrict__ B, const long long* __restrict__ idx,
                                 long long n, double* __restrict__ out) {
    const long long bvs = g.nleaf * 6 * g.mf;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
#pragma unroll
        for (int v = 0; v < NV; v++) out[e * NV + v] = B[v * bvs + idx[e]];
}

// ---------------------------------------------------------------- KE
template <int NDIM>
__global__ void amr_cfl_kernel(const AmrGeo g, const double* __restrict__ u, DevScalars* sc) {
    constexpr int NV = NDIM + 2;
    __shared__ double red[32];
    const long long vs = g.nleaf * g.nc;
    double mn = INFINITY;
    bool ok = true;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < vs;
         q += (long long)gridDim.x * blockDim.x) {
        const int lev = q / g.nc < g.ncl ? 0 : 1;
        double uu[NV], ww[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) uu[v] = u[v * vs + q];
        ok &= cons_to_prim<NV>(uu, ww, g.gamma - 1.0);
        // reading R7 with the leaf's own spacing: 1 / max_d (|u_d| + c) / dx_d
        const double gp = g.gamma * ww[NV - 1];
        const double c = gp * rsqrt_fast(gp * ww[0]);
        double m = (fabs(ww[1]) + c) * g.rdx[lev][0];
#pragma unroll
        for (int d = 1; d < NDIM; d++) {
            const double x = (fabs(ww[1 + d]) + c) * g.rdx[lev][d];
            m = x > m ? x : m;
        }
        mn = fmin(mn, rcp(m));
    }
    if (!ok) flag_nonphysical(sc);
    block_min_to(mn, red, &sc->acc);
}

unsigned grid_of(long long n) {
    long long b = (n + 255) / 256;
    return (unsigned)std::max(1LL, std::min(b, 148LL * 16));
}

}  // namespace
}  // namespace spark

// ===================================================================== host
namespace {

using spark::AmrGeo;
using spark::CorrE;
using spark::GuardE;

struct AmrError : std::runtime_error {
    spark_status st;
    AmrError(spark_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

#define ACU(call)                                                                                      \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess) throw AmrError(SPARK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int recon_ng(int recon) { return (recon == 2 || recon == 4) ? 3 : ((recon == 1 || recon == 3) ? 2 : 1); }

bool has_box(const spark_refine* r) {
    for (int d = 0; d < 3; d++)
        if (r->rhi[d] <= r->rlo[d]) return false;
    return true;
}

// Host plan of the composite grid: leaves, guard map, correction lists.
struct AmrPlan {
    spark_config c{};
    spark_refine r{};
    AmrGeo g{};
    std::vector<int> level;
    std::vector<std::array<long long, 3>> blk;
    std::vector<GuardE> guards;
    std::vector<CorrE> corr[3];
    long long fnb[3] = {1, 1, 1};

    bool refined(const long long* cb) const {
        if (!has_box(&r)) return false;
        for (int d = 0; d < 3; d++)
            if (cb[d] < r.rlo[d] || cb[d] >= r.rhi[d]) return false;
        return true;
    }
    long long ncells(int lev, int d) const {
        const long long n = (long long)c.nblk[d] * c.nb[d];
        return d < c.ndim ? n << lev : n;
    }
    // level-L block coordinates -> leaf (-1 if none)
    long long leaf_of(int lev, const long long* b) const {
        if (lev == 1) {
            long long q[3];
            for (int d = 0; d < 3; d++) {
                q[d] = b[d] - (d < c.ndim ? 2LL * r.rlo[d] : 0);
                if (q[d] < 0 || q[d] >= fnb[d]) return -1;
            }
            return g.ncl + q[0] + fnb[0] * (q[1] + fnb[1] * q[2]);
        }
        if (refined(b)) return -1;
        return coarse_index[(b[2] * c.nblk[1] + b[1]) * c.nblk[0] + b[0]];
    }
    std::vector<long long> coarse_index;
};

std::string check_amr(const spark_config* c, const spark_refine* r) {
    if (!c || !r) return "null argument";
    if (c->ndim < 1 || c->ndim > 3) return "ndim must be 1..3";
    if (c->recon < 0 || c->recon > 4 || c->riemann < 0 || c->riemann > 2) return "unknown recon / riemann";
    if (c->rk_stages != 2 && c->rk_stages != 3) return "rk_stages must be 2 or 3";
    if (!(c->gamma > 1.0) || !(c->cfl > 0.0)) return "gamma must be > 1 and cfl > 0";
    if (c->ng < recon_ng(c->recon)) return "ng too small for the reconstruction";
    if (c->riemann == 2 && (recon_ng(c->recon) < 2 || !(c->shock_thresh > 0.0)))
        return "hybrid Riemann needs recon >= PLM and shock_thresh > 0";
    for (int d = 0; d < 3; d++) {
        if (c->grav[d] != 0.0) return "gravity is not supported on the refined grid";
        if (c->nb[d] < 1 || c->nblk[d] < 1) return "nb and nblk must be >= 1";
        if (d >= c->ndim && (c->nb[d] != 1 || c->nblk[d] != 1)) return "unused dims need nb = nblk = 1";
        if (d < c->ndim && c->nb[d] < c->ng) return "nb must be >= ng";
        if (d < c->ndim && !(c->hi[d] > c->lo[d])) return "hi must exceed lo";
        for (int s = 0; s < 2; s++)
            if (c->bc[d][s] < 0 || c->bc[d][s] > 2) return "unknown boundary condition";
        if (d < c->ndim && (c->bc[d][0] == SPARK_BC_PERIODIC) != (c->bc[d][1] == SPARK_BC_PERIODIC))
            return "periodic boundaries must be periodic on both sides";
        if (r->rlo[d] < 0 || r->rhi[d] > c->nblk[d] || r->rlo[d] > r->rhi[d]) return "refined box outside the grid";
    }
    if (has_box(r))
        for (int d = 0; d < 3; d++) {
            if (d < c->ndim && c->nb[d] % 2) return "nb must be even with a refined box";
            if (d >= c->ndim && (r->rlo[d] != 0 || r->rhi[d] != 1)) return "unused dims of the box must be [0, 1)";
        }
    const long long plane = (long long)c->nb[0] * c->nb[1] * c->nb[2];
    if (plane * (long long)c->nblk[0] * c->nblk[1] * c->nblk[2] * 8 > (1LL << 33)) return "grid too large";
    return "";
}

// Per-dimension boundary map at one level (periodic wrap / outflow clamp /
// reflect mirror); *flip set for a reflect.
long long bmap(long long g, long long N, int lo, int hi, bool* flip) {
    *flip = false;
    if (g >= 0 && g < N) return g;
    const int bc = g < 0 ? lo : hi;
    if (bc == SPARK_BC_PERIODIC) return ((g % N) + N) % N;
    if (bc == SPARK_BC_OUTFLOW) return g < 0 ? 0 : N - 1;
    *flip = true;
    return g < 0 ? -1 - g : 2 * N - 1 - g;
}

AmrPlan make_amr_plan(const spark_config* c, const spark_refine* r) {
    std::string m = check_amr(c, r);
    if (!m.empty()) throw AmrError(SPARK_ERR_ARG, m);
    AmrPlan p;
    p.c = *c;
    p.r = *r;
    const int nd = c->ndim;
    AmrGeo& g = p.g;
    g.ndim = nd;
    g.nv = nd + 2;
    g.ng = c->ng;
    g.ngk = recon_ng(c->recon);
    g.recon = c->recon;
    g.np = 1;
    g.nc = 1;
    for (int d = 0; d < 3; d++) {
        g.nb[d] = c->nb[d];
        g.pn[d] = c->nb[d] + (d < nd ? 2 * c->ng : 0);
        g.np *= g.pn[d];
        g.nc *= c->nb[d];
        const double dx = (c->hi[d] - c->lo[d]) / ((double)c->nblk[d] * c->nb[d]);
        g.rdx[0][d] = 1.0 / dx;
        g.rdx[1][d] = 1.0 / (0.5 * dx);
        p.fnb[d] = has_box(r) ? (d < nd ? 2LL * (r->rhi[d] - r->rlo[d]) : 1) : 0;
    }
    // leaves
    p.coarse_index.assign((size_t)c->nblk[0] * c->nblk[1] * c->nblk[2], -1);
    for (long long bz = 0; bz < c->nblk[2]; bz++)
        for (long long by = 0; by < c->nblk[1]; by++)
            for (long long bx = 0; bx < c->nblk[0]; bx++) {
                const long long b[3] = {bx, by, bz};
                if (p.refined(b)) continue;
                p.coarse_index[(bz * c->nblk[1] + by) * c->nblk[0] + bx] = (long long)p.level.size();
                p.level.push_back(0);
                p.blk.push_back({bx, by, bz});
            }
    g.ncl = (long long)p.level.size();
    if (has_box(r))
        for (long long bz = 0; bz < p.fnb[2]; bz++)
            for (long long by = 0; by < p.fnb[1]; by++)
                for (long long bx = 0; bx < p.fnb[0]; bx++) {
                    p.level.push_back(1);
                    p.blk.push_back({2LL * r->rlo[0] + bx, nd >= 2 ? 2LL * r->rlo[1] + by : 0,
                                     nd >= 3 ? 2LL * r->rlo[2] + bz : 0});
                }
    g.nleaf = (long long)p.level.size();
    // faces
    long long off = 0;
    g.mf = 1;
    for (int d = 0; d < 3; d++) {
        g.Fo[d] = off;
        g.nfd[d] = 0;
        if (d < nd) {
            g.nfd[d] = 1;
            for (int e = 0; e < 3; e++) g.nfd[d] *= c->nb[e] + (e == d ? 1 : 0);
            long long fcells = 1;
            for (int e = 0; e < nd; e++)
                if (e != d) fcells *= c->nb[e];
            g.mf = std::max(g.mf, fcells);
        }
        off += g.nfd[d];
    }
    g.NF = off;
    g.gamma = c->gamma;
    g.cfl = c->cfl;
    g.shock_thresh = c->riemann == 2 ? c->shock_thresh : 0.0;
    // guard map: every face guard of every leaf (reading R22)
    for (long long leaf = 0; leaf < g.nleaf; leaf++) {
        const int lev = p.level[leaf];
        const auto& b = p.blk[leaf];
        for (int d = 0; d < nd; d++) {
            int tr[2] = {-1, -1}, nt = 0;  // the transverse dimensions of d, increasing
            for (int e = 0; e < nd; e++)
                if (e != d) tr[nt++] = e;
            for (int side = 0; side < 2; side++)
                for (int depth = 0; depth < c->ng; depth++)
                    for (int t2 = 0; t2 < (nt > 1 ? c->nb[tr[1]] : 1); t2++)
                        for (int t1 = 0; t1 < (nt > 0 ? c->nb[tr[0]] : 1); t1++) {
                            int loc[3] = {0, 0, 0};
                            loc[d] = side ? c->nb[d] + depth : -1 - depth;
                            if (nt > 0) loc[tr[0]] = t1;
                            if (nt > 1) loc[tr[1]] = t2;
                            long long gc[3];
                            for (int e = 0; e < 3; e++) gc[e] = b[e] * c->nb[e] + loc[e];
                            bool flip;
                            gc[d] = bmap(gc[d], p.ncells(lev, d), c->bc[d][0], c->bc[d][1], &flip);
                            GuardE E{};
                            int gpad[3];
                            for (int e = 0; e < 3; e++) gpad[e] = e < nd ? c->ng : 0;
                            E.dst = leaf * g.np +
                                    ((long long)(loc[2] + gpad[2]) * g.pn[1] + (loc[1] + gpad[1])) * g.pn[0] + (loc[0] + gpad[0]);
                            E.kind = flip ? (1 << (4 + d)) : 0;
                            auto cell_of = [&](int lv, const long long* x, long long* leaf_out) {
                                long long bb[3], cc[3];
                                for (int e = 0; e < 3; e++) bb[e] = x[e] / c->nb[e], cc[e] = x[e] % c->nb[e];
                                *leaf_out = p.leaf_of(lv, bb);
                                return (cc[2] * c->nb[1] + cc[1]) * c->nb[0] + cc[0];
                            };
                            long long src_leaf;
                            if (lev == 1) {
                                long long cg[3], cb[3];
                                for (int e = 0; e < 3; e++) {
                                    cg[e] = e < nd ? gc[e] / 2 : gc[e];
                                    cb[e] = cg[e] / c->nb[e];
                                }
                                if (p.refined(cb)) {
                                    const long long cell = cell_of(1, gc, &src_leaf);
                                    E.src = src_leaf * g.nc + cell;
                                } else {  // prolongation: the containing coarse cell (injection)
                                    const long long cell = cell_of(0, cg, &src_leaf);
                                    E.src = src_leaf * g.nc + cell;
                                }
                                E.kind |= 1;
                            } else {
                                long long cb[3];
                                for (int e = 0; e < 3; e++) cb[e] = gc[e] / c->nb[e];
                                if (!p.refined(cb)) {
                                    const long long cell = cell_of(0, gc, &src_leaf);
                                    E.src = src_leaf * g.nc + cell;
                                    E.kind |= 1;
                                } else {  // restriction: the 2^ndim fine children, first child here
                                    long long fg[3];
                                    for (int e = 0; e < 3; e++) fg[e] = e < nd ? 2 * gc[e] : gc[e];
                                    const long long cell = cell_of(1, fg, &src_leaf);
                                    E.src = src_leaf * g.nc + cell;
                                    E.kind |= 2;
                                }
                            }
                            if (src_leaf < 0) throw AmrError(SPARK_ERR_ARG, "internal: guard source is not a leaf");
                            p.guards.push_back(E);
                        }
        }
    }
    // correction lists (communicate_fluxes): coarse faces on a coarse-fine interface
    if (has_box(r))
        for (long long leaf = 0; leaf < g.ncl; leaf++) {
            const auto& b = p.blk[leaf];
            for (int d = 0; d < nd; d++)
                for (int side = 0; side < 2; side++) {
                    const long long N0 = p.ncells(0, d);
                    const long long gface = side ? (b[d] + 1) * c->nb[d] : b[d] * c->nb[d] - 1;
                    if ((gface < 0 || gface >= N0) && c->bc[d][side] != SPARK_BC_PERIODIC) continue;
                    bool fl;
                    const long long gm = bmap(gface, N0, c->bc[d][0], c->bc[d][1], &fl);
                    long long nbk[3] = {b[0], b[1], b[2]};
                    nbk[d] = gm / c->nb[d];
                    if (!p.refined(nbk)) continue;
                    const long long fd = side ? 2 * gm : 2 * gm + 1;
                    const int e1 = d == 0 ? 1 : 0, e2 = d == 2 ? 1 : 2;
                    const int n1 = nd > 1 ? c->nb[e1] : 1, n2 = nd > 2 ? c->nb[e2] : 1;
                    for (int t2 = 0; t2 < n2; t2++)
                        for (int t1 = 0; t1 < n1; t1++) {
                            int lc[3] = {0, 0, 0};
                            lc[d] = side ? c->nb[d] - 1 : 0;
                            if (nd > 1) lc[e1] = t1;
                            if (nd > 2) lc[e2] = t2;
                            CorrE E{};
                            E.cell = leaf * g.nc + ((long long)lc[2] * c->nb[1] + lc[1]) * c->nb[0] + lc[0];
                            E.bc = (leaf * 6 + 2 * d + side) * g.mf + spark::face_cell(g, d, lc[0], lc[1], lc[2]);
                            E.side = side;
                            const int nf = 1 << (nd - 1);
                            for (int q = 0; q < nf; q++) {
                                long long fg[3] = {0, 0, 0};
                                fg[d] = fd;
                                if (nd > 1) fg[e1] = 2 * (b[e1] * c->nb[e1] + t1) + (q & 1);
                                if (nd > 2) fg[e2] = 2 * (b[e2] * c->nb[e2] + t2) + ((q >> 1) & 1);
                                long long fb[3], flc[3];
                                for (int e = 0; e < 3; e++) fb[e] = fg[e] / c->nb[e], flc[e] = fg[e] % c->nb[e];
                                const long long fleaf = p.leaf_of(1, fb);
                                if (fleaf < 0) throw AmrError(SPARK_ERR_ARG, "internal: fine face is not a leaf");
                                E.bf[q] = (fleaf * 6 + 2 * d + (1 - side)) * g.mf +
                                          spark::face_cell(g, d, (int)flc[0], (int)flc[1], (int)flc[2]);
                            }
                            p.corr[d].push_back(E);
                        }
                }
        }
    return p;
}

size_t al(size_t x) { return (x + 255) / 256 * 256; }

// One rank's share of the composite grid: a contiguous range of the leaf
// list (coarse leaves first, as in the global order), its guard map and
// correction lists in local indices, and what it exchanges with the other
// ranks: guard values (per stage) and fine-face fluxBuff values (per step,
// communicate_fluxes).  Items for one peer are ordered identically on both
// sides (the order of the receiver's entries), exchange buffers are
// [item][v], grouped by peer rank.
struct RankPlan {
    AmrGeo g{};
    long long l0 = 0, nloc = 0;
    std::vector<GuardE> guards;
    std::vector<CorrE> corr[3];
    std::vector<GuardE> gsend;                  // src (local) + kind of each value sent
    std::vector<long long> gsend_off, grecv_off;  // per peer rank, size nranks + 1
    std::vector<long long> fsend;               // local B index (variable 0) of each value sent
    std::vector<long long> fsend_off, frecv_off;
    std::vector<long long> goff;                // first guard entry of each local leaf, size nleaf + 1
};

// KB+KC fused (3-D 16^3 leaves, face-centric schemes): no face-flux array
bool leaf_fused(const AmrGeo& g) {
    return g.ndim == 3 && g.nb[0] == spark::kLeafN && g.nb[1] == spark::kLeafN && g.nb[2] == spark::kLeafN &&
           (g.recon == 0 || g.recon == 1 || g.recon == 3) && g.ng == spark::kLeafNG;
}

// Faces whose ng guard layers are a plain copy (kind 1, no reflect flip) of
// the adjacent layers of ONE leaf of this rank: sface[leaf * 6 + slot] = that
// leaf (else -1); the map keeps only the other entries.  Found by checking
// every entry of the face against the copy pattern, so anything else (a
// coarse-fine face, a boundary image, another rank's value) stays in the map.
void compress_faces(const AmrGeo& g, std::vector<GuardE>& gs, std::vector<long long>& sface) {
    const long long nl = g.nleaf;
    sface.assign(nl * 6, -1);
    std::vector<long long> cnt(nl * 6, 0), src(nl * 6, -1);
    std::vector<char> bad(nl * 6, 0);
    const int gl[3] = {g.ng, g.ndim >= 2 ? g.ng : 0, g.ndim >= 3 ? g.ng : 0};
    auto slot_of = [&](const GuardE& e, int* c) {
        long long p = e.dst % g.np;
        c[0] = (int)(p % g.pn[0]) - gl[0];
        c[1] = (int)((p / g.pn[0]) % g.pn[1]) - gl[1];
        c[2] = (int)(p / ((long long)g.pn[0] * g.pn[1])) - gl[2];
        int slot = -1, outside = 0;
        for (int d = 0; d < 3; d++)
            if (c[d] < 0 || c[d] >= g.nb[d]) {
                slot = 2 * d + (c[d] >= g.nb[d] ? 1 : 0);
                outside++;
            }
        return outside == 1 ? slot : -1;
    };
    for (const GuardE& e : gs) {
        int c[3];
        const int slot = slot_of(e, c);
        if (slot < 0) continue;
        const long long k = (e.dst / g.np) * 6 + slot;
        cnt[k]++;
        const int d = slot >> 1;
        int q[3] = {c[0], c[1], c[2]};
        q[d] += (slot & 1) ? -g.nb[d] : g.nb[d];
        const long long want = ((long long)q[2] * g.nb[1] + q[1]) * g.nb[0] + q[0];
        if (e.kind != 1 || e.src % g.nc != want) {
            bad[k] = 1;
            continue;
        }
        const long long sl = e.src / g.nc;
        if (src[k] < 0) src[k] = sl;
        else if (src[k] != sl) bad[k] = 1;
    }
    for (long long k = 0; k < nl * 6; k++) {
        const int d = (int)(k % 6) >> 1;
        if (d >= g.ndim || bad[k] || src[k] < 0) continue;
        long long full = g.ng;
        for (int e = 0; e < 3; e++)
            if (e != d) full *= g.nb[e];
        if (cnt[k] == full) sface[k] = src[k];
    }
    std::vector<GuardE> rest;
    rest.reserve(gs.size());
    for (const GuardE& e : gs) {
        int c[3];
        const int slot = slot_of(e, c);
        if (slot < 0 || sface[(e.dst / g.np) * 6 + slot] < 0) rest.push_back(e);
    }
    gs.swap(rest);
}

// per-leaf offsets of a guard list ordered by leaf (dst = leaf * np + ...)
std::vector<long long> guard_offsets(const std::vector<GuardE>& gs, long long nleaf, long long np) {
    std::vector<long long> off(nleaf + 1, 0);
    for (const GuardE& e : gs) off[e.dst / np + 1]++;
    for (long long l = 0; l < nleaf; l++) off[l + 1] += off[l];
    for (size_t i = 1; i < gs.size(); i++)
        if (gs[i].dst / np < gs[i - 1].dst / np) throw AmrError(SPARK_ERR_STATE, "guard map not ordered by leaf");
    return off;
}

std::vector<RankPlan> partition(const AmrPlan& P, int nranks) {
    const AmrGeo& G = P.g;
    const long long L = G.nleaf;
    if (nranks < 1 || nranks > L) throw AmrError(SPARK_ERR_ARG, "nranks must be 1..number of leaves");
    std::vector<long long> l0(nranks + 1);
    for (int r = 0; r <= nranks; r++) l0[r] = L * r / nranks;
    auto owner = [&](long long leaf) {
        int r = (int)(leaf * nranks / L);
        while (leaf < l0[r]) r--;
        while (leaf >= l0[r + 1]) r++;
        return r;
    };
    std::vector<RankPlan> R(nranks);
    // requests: greq[r][q] = entries of r reading a guard value owned by q
    std::vector<std::vector<std::vector<std::pair<size_t, GuardE>>>> greq(nranks,
        std::vector<std::vector<std::pair<size_t, GuardE>>>(nranks));
    struct FReq { int d; size_t e; int k; long long qidx; };
    std::vector<std::vector<std::vector<FReq>>> freq(nranks, std::vector<std::vector<FReq>>(nranks));
    for (int r = 0; r < nranks; r++) {
        RankPlan& rp = R[r];
        rp.l0 = l0[r];
        rp.nloc = l0[r + 1] - l0[r];
        rp.g = G;
        rp.g.nleaf = rp.nloc;
        rp.g.ncl = std::max(0LL, std::min(G.ncl - rp.l0, rp.nloc));
    }
    for (const GuardE& E : P.guards) {
        const long long leaf = E.dst / G.np;
        const int r = owner(leaf);
        GuardE e = E;
        e.dst = (leaf - l0[r]) * G.np + (E.dst - leaf * G.np);
        const long long sleaf = E.src / G.nc;
        const int q = owner(sleaf);
        if (q == r) {
            e.src = E.src - l0[r] * G.nc;
        } else {
            GuardE item{};
            item.src = E.src - l0[q] * G.nc;
            item.kind = E.kind & 15;
            greq[r][q].emplace_back(R[r].guards.size(), item);
            e.kind = 3 | (E.kind & ~15);
        }
        R[r].guards.push_back(e);
    }
    const long long bstride = 6 * G.mf;
    for (int d = 0; d < 3; d++)
        for (const CorrE& E : P.corr[d]) {
            const long long leaf = E.cell / G.nc;
            const int r = owner(leaf);
            CorrE e = E;
            e.cell = E.cell - l0[r] * G.nc;
            e.bc = E.bc - l0[r] * bstride;
            const int nf = 1 << (G.ndim - 1);
            for (int k = 0; k < nf; k++) {
                const long long fleaf = E.bf[k] / bstride;
                const int q = owner(fleaf);
                if (q == r) e.bf[k] = E.bf[k] - l0[r] * bstride;
                else freq[r][q].push_back({d, R[r].corr[d].size(), k, E.bf[k] - l0[q] * bstride});
            }
            R[r].corr[d].push_back(e);
        }
    // slots and send lists
    for (int r = 0; r < nranks; r++) {
        R[r].grecv_off.assign(nranks + 1, 0);
        R[r].frecv_off.assign(nranks + 1, 0);
        for (int q = 0; q < nranks; q++) {
            R[r].grecv_off[q + 1] = R[r].grecv_off[q] + (long long)greq[r][q].size();
            R[r].frecv_off[q + 1] = R[r].frecv_off[q] + (long long)freq[r][q].size();
            for (size_t i = 0; i < greq[r][q].size(); i++) R[r].guards[greq[r][q][i].first].src = R[r].grecv_off[q] + i;
            for (size_t i = 0; i < freq[r][q].size(); i++) {
                const FReq& f = freq[r][q][i];
                R[r].corr[f.d][f.e].bf[f.k] = -(R[r].frecv_off[q] + (long long)i + 1);
            }
        }
    }
    for (int q = 0; q < nranks; q++) {
        R[q].gsend_off.assign(nranks + 1, 0);
        R[q].fsend_off.assign(nranks + 1, 0);
        for (int r = 0; r < nranks; r++) {
            for (const auto& it : greq[r][q]) R[q].gsend.push_back(it.second);
            for (const auto& f : freq[r][q]) R[q].fsend.push_back(f.qidx);
            R[q].gsend_off[r + 1] = (long long)R[q].gsend.size();
            R[q].fsend_off[r + 1] = (long long)R[q].fsend.size();
        }
    }
    return R;
}

size_t rank_bytes(const RankPlan& p) {
    const AmrGeo& g = p.g;
    size_t b = al(sizeof(spark::DevScalars));
    b += 3 * al(sizeof(double) * g.nv * g.nleaf * g.nc);       // U^n and two stage buffers
    b += al(sizeof(double) * g.nv * g.nleaf * g.np);            // padded tiles
    if (!leaf_fused(g)) b += al(sizeof(double) * g.nv * g.nleaf * g.NF);  // face fluxes (unfused KB/KC)
    b += al(sizeof(long long) * (g.nleaf + 1));                 // guard offsets per leaf
    b += al(sizeof(long long) * 6 * std::max(1LL, g.nleaf));    // same-level face sources
    b += al(sizeof(double) * g.nv * g.nleaf * 6 * g.mf);        // fluxBuff
    b += al(sizeof(GuardE) * std::max<size_t>(1, p.guards.size()));
    for (int d = 0; d < 3; d++) b += al(sizeof(CorrE) * std::max<size_t>(1, p.corr[d].size()));
    const size_t ngs = p.gsend.size(), ngr = p.grecv_off.empty() ? 0 : p.grecv_off.back();
    const size_t nfs = p.fsend.size(), nfr = p.frecv_off.empty() ? 0 : p.frecv_off.back();
    b += al(sizeof(GuardE) * std::max<size_t>(1, ngs)) + al(sizeof(long long) * std::max<size_t>(1, nfs));
    b += al(sizeof(double) * g.nv * std::max<size_t>(1, ngs)) + al(sizeof(double) * g.nv * std::max<size_t>(1, ngr));
    b += al(sizeof(double) * g.nv * std::max<size_t>(1, nfs)) + al(sizeof(double) * g.nv * std::max<size_t>(1, nfr));
    return b;
}

}  // namespace

struct spark_amr {
    AmrPlan plan;   // the global composite grid
    RankPlan rp;    // this rank's share
    int rank = 0, nranks = 1;
    std::shared_ptr<std::vector<spark_amr*>> group;  // all members (itself when alone)
    int device = 0;
    cudaStream_t stream = nullptr;
    spark::DevScalars* sc = nullptr;
    double* U[3] = {};
    double* W = nullptr;
    double* F = nullptr;
    double* B = nullptr;
    GuardE* guards = nullptr;
    CorrE* corr[3] = {};
    GuardE* gitems = nullptr;
    long long* fitems = nullptr;
    long long* goff = nullptr;   // first guard entry of each leaf
    long long* sface = nullptr;  // same-level source leaf of each face slot (-1: map entries)
    double *gsend = nullptr, *grecv = nullptr, *fsend = nullptr, *frecv = nullptr;
    int n_idx = 0;
    bool have_state = false;
    std::string err;
};

namespace {

template <typename Fn>
spark_status amr_guard(spark_amr* a, Fn&& f) {
    try {
        if (a) a->err.clear();
        f();
        return SPARK_OK;
    } catch (const AmrError& e) {
        if (a) a->err = e.what();
        return e.st;
    } catch (const std::exception& e) {
        if (a) a->err = e.what();
        return SPARK_ERR_ARG;
    }
}

void launched(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw AmrError(SPARK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// padded tiles of state u: interior + face guards; primitives (to_prim) or conserved
// interior = 0: the map entries only (the fused leaf kernel reads the
// interior and the same-level faces straight from U)
void amr_fill(spark_amr* a, const double* u, double* w, int to_prim, int interior = 1) {
    const AmrGeo& g = a->rp.g;
    if (g.nleaf == 0) return;
    const unsigned nb = (unsigned)g.nleaf;
    if (g.ndim == 1)
        spark::amr_fill_leaf_kernel<3><<<nb, 256, 0, a->stream>>>(g, u, a->guards, a->goff, a->sface, a->grecv, w, to_prim,
                                                                  interior, a->sc);
    else if (g.ndim == 2)
        spark::amr_fill_leaf_kernel<4><<<nb, 256, 0, a->stream>>>(g, u, a->guards, a->goff, a->sface, a->grecv, w, to_prim,
                                                                  interior, a->sc);
    else
        spark::amr_fill_leaf_kernel<5><<<nb, 256, 0, a->stream>>>(g, u, a->guards, a->goff, a->sface, a->grecv, w, to_prim,
                                                                  interior, a->sc);
    launched(cudaGetLastError(), "amr fill");
}

template <int NDIM>
void faces_d(spark_amr* a, double bco) {
    const AmrGeo& g = a->rp.g;
    const unsigned gr = spark::grid_of(g.nleaf * g.NF);
    const int rs = a->plan.c.riemann;
    if (rs == 0) spark::amr_face_kernel<NDIM, 0><<<gr, 256, 0, a->stream>>>(g, a->W, a->F, a->B, bco);
    else if (rs == 1) spark::amr_face_kernel<NDIM, 1><<<gr, 256, 0, a->stream>>>(g, a->W, a->F, a->B, bco);
    else spark::amr_face_kernel<NDIM, 2><<<gr, 256, 0, a->stream>>>(g, a->W, a->F, a->B, bco);
    launched(cudaGetLastError(), "amr faces");
}

template <int RECON, int RS>
void leaf_t(spark_amr* a, const double* prev, const double* un, double sa, double sb, double* out) {
    const AmrGeo& g = a->rp.g;
    const size_t smem = sizeof(double) * ((size_t)spark::kLeafSlots * g.nv * (spark::kLeafN + 2 * spark::kLeafNG) *
                                              (spark::kLeafN + 2 * spark::kLeafNG) +
                                          2 * (size_t)g.nv * spark::kLeafN +
                                          2 * (size_t)g.nv * (spark::kLeafN + 1) * spark::kLeafN +
                                          2 * 4 * (size_t)g.nv * spark::kLeafN);
    auto k = spark::amr_leaf_kernel<RECON, RS>;
    launched(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "amr leaf smem");
    k<<<(unsigned)g.nleaf, 256, smem, a->stream>>>(g, a->W, prev, un, out, a->B, a->sface, sa, sb, a->sc);
}

template <int RECON>
void leaf_r(spark_amr* a, int rs, const double* prev, const double* un, double sa, double sb, double* out) {
    if (rs == 0) leaf_t<RECON, 0>(a, prev, un, sa, sb, out);
    else if (rs == 1 || RECON == 0) leaf_t<RECON, 1>(a, prev, un, sa, sb, out);
    else leaf_t<RECON, 2>(a, prev, un, sa, sb, out);
}

void amr_stage(spark_amr* a, const double* prev, const double* un, double sa, double sb, double* out) {
    const AmrGeo& g = a->rp.g;
    if (g.nleaf == 0) return;
    amr_fill(a, prev, a->W, 1, leaf_fused(g) ? 0 : 1);
    if (leaf_fused(g)) {
        const int rs = a->plan.c.riemann;
        if (g.recon == 0) leaf_r<0>(a, rs, prev, un, sa, sb, out);
        else if (g.recon == 1) leaf_r<1>(a, rs, prev, un, sa, sb, out);
        else leaf_r<3>(a, rs, prev, un, sa, sb, out);
        launched(cudaGetLastError(), "amr leaf stage");
        return;
    }
    if (g.ndim == 1) faces_d<1>(a, sb);
    else if (g.ndim == 2) faces_d<2>(a, sb);
    else faces_d<3>(a, sb);
    const unsigned gr = spark::grid_of(g.nleaf * g.nc);
    if (g.ndim == 1) spark::amr_update_kernel<1><<<gr, 256, 0, a->stream>>>(g, a->F, prev, un, out, sa, sb, a->sc);
    else if (g.ndim == 2) spark::amr_update_kernel<2><<<gr, 256, 0, a->stream>>>(g, a->F, prev, un, out, sa, sb, a->sc);
    else spark::amr_update_kernel<3><<<gr, 256, 0, a->stream>>>(g, a->F, prev, un, out, sa, sb, a->sc);
    launched(cudaGetLastError(), "amr update");
}

void amr_cfl(spark_amr* a, const double* u) {
    const AmrGeo& g = a->rp.g;
    if (g.nleaf == 0) return;
    const unsigned gr = spark::grid_of(g.nleaf * g.nc);
    if (g.ndim == 1) spark::amr_cfl_kernel<1><<<gr, 256, 0, a->stream>>>(g, u, a->sc);
    else if (g.ndim == 2) spark::amr_cfl_kernel<2><<<gr, 256, 0, a->stream>>>(g, u, a->sc);
    else spark::amr_cfl_kernel<3><<<gr, 256, 0, a->stream>>>(g, u, a->sc);
    launched(cudaGetLastError(), "amr cfl");
}

void amr_correct(spark_amr* a, double* u) {
    const AmrGeo& g = a->rp.g;
    for (int d = 0; d < g.ndim; d++) {  // one launch per direction: no two threads touch one cell
        const long long n = (long long)a->rp.corr[d].size();
        if (!n) continue;
        const unsigned gr = spark::grid_of(n);
        if (g.ndim == 1)
            spark::amr_corr_kernel<3><<<gr, 256, 0, a->stream>>>(g, a->corr[d], n, d, a->B, a->frecv, u, &a->sc->dt, a->sc);
        else if (g.ndim == 2)
            spark::amr_corr_kernel<4><<<gr, 256, 0, a->stream>>>(g, a->corr[d], n, d, a->B, a->frecv, u, &a->sc->dt, a->sc);
        else
            spark::amr_corr_kernel<5><<<gr, 256, 0, a->stream>>>(g, a->corr[d], n, d, a->B, a->frecv, u, &a->sc->dt, a->sc);
        launched(cudaGetLastError(), "amr correction");
    }
}

// the guard values (u: each member's U^(s-1)) or the fluxBuff values the other
// ranks need: pack, then copy member q's slice for r into r's receive buffer
void amr_exchange(const std::vector<spark_amr*>& m, const int* uidx, bool fluxes) {
    if (m.size() < 2) return;
    for (size_t r = 0; r < m.size(); r++) {
        spark_amr* a = m[r];
        const AmrGeo& g = a->rp.g;
        const long long n = fluxes ? (long long)a->rp.fsend.size() : (long long)a->rp.gsend.size();
        if (!n) continue;
        const unsigned gr = spark::grid_of(n);
        const double* u = uidx ? a->U[uidx[r]] : nullptr;
        if (fluxes) {
            if (g.nv == 3) spark::amr_fpack_kernel<3><<<gr, 256, 0, a->stream>>>(g, a->B, a->fitems, n, a->fsend);
            else if (g.nv == 4) spark::amr_fpack_kernel<4><<<gr, 256, 0, a->stream>>>(g, a->B, a->fitems, n, a->fsend);
            else spark::amr_fpack_kernel<5><<<gr, 256, 0, a->stream>>>(g, a->B, a->fitems, n, a->fsend);
        } else {
            if (g.nv == 3) spark::amr_gpack_kernel<3><<<gr, 256, 0, a->stream>>>(g, u, a->gitems, n, a->gsend);
            else if (g.nv == 4) spark::amr_gpack_kernel<4><<<gr, 256, 0, a->stream>>>(g, u, a->gitems, n, a->gsend);
            else spark::amr_gpack_kernel<5><<<gr, 256, 0, a->stream>>>(g, u, a->gitems, n, a->gsend);
        }
        launched(cudaGetLastError(), "amr pack");
    }
    for (size_t r = 0; r < m.size(); r++) {
        spark_amr* a = m[r];
        const int nv = a->rp.g.nv;
        for (size_t q = 0; q < m.size(); q++) {
            if (q == r) continue;
            const auto& roff = fluxes ? a->rp.frecv_off : a->rp.grecv_off;
            const auto& soff = fluxes ? m[q]->rp.fsend_off : m[q]->rp.gsend_off;
            const long long n = roff[q + 1] - roff[q];
            if (!n) continue;
            double* dst = (fluxes ? a->frecv : a->grecv) + roff[q] * nv;
            const double* src = (fluxes ? m[q]->fsend : m[q]->gsend) + soff[r] * nv;
            ACU(cudaMemcpyAsync(dst, src, sizeof(double) * n * nv, cudaMemcpyDeviceToDevice, a->stream));
        }
    }
}

spark::DevScalars read_sc(spark_amr* a) {
    ACU(cudaStreamSynchronize(a->stream));
    spark::DevScalars h;
    ACU(cudaMemcpy(&h, a->sc, sizeof(h), cudaMemcpyDeviceToHost));
    return h;
}

void carve_member(spark_amr* a, void* arena, size_t arena_bytes) {
    const size_t need = rank_bytes(a->rp);
    if (!arena) throw AmrError(SPARK_ERR_ARG, "null arena");
    if (arena_bytes < need) throw AmrError(SPARK_ERR_OOM, "arena smaller than the required bytes");
    if (reinterpret_cast<uintptr_t>(arena) % 256) throw AmrError(SPARK_ERR_ARG, "arena must be 256-byte aligned");
    ACU(cudaSetDevice(a->device));
    const AmrGeo& g = a->rp.g;
    const RankPlan& rp = a->rp;
    char* p = static_cast<char*>(arena);
    auto take = [&](size_t bytes) {
        char* q = p;
        p += al(bytes);
        return q;
    };
    a->sc = reinterpret_cast<spark::DevScalars*>(take(sizeof(spark::DevScalars)));
    for (int i = 0; i < 3; i++) a->U[i] = reinterpret_cast<double*>(take(sizeof(double) * g.nv * g.nleaf * g.nc));
    a->W = reinterpret_cast<double*>(take(sizeof(double) * g.nv * g.nleaf * g.np));
    if (!leaf_fused(g)) a->F = reinterpret_cast<double*>(take(sizeof(double) * g.nv * g.nleaf * g.NF));
    a->goff = reinterpret_cast<long long*>(take(sizeof(long long) * (g.nleaf + 1)));
    a->sface = reinterpret_cast<long long*>(take(sizeof(long long) * 6 * std::max(1LL, g.nleaf)));
    a->B = reinterpret_cast<double*>(take(sizeof(double) * g.nv * g.nleaf * 6 * g.mf));
    a->guards = reinterpret_cast<GuardE*>(take(sizeof(GuardE) * std::max<size_t>(1, rp.guards.size())));
    for (int d = 0; d < 3; d++)
        a->corr[d] = reinterpret_cast<CorrE*>(take(sizeof(CorrE) * std::max<size_t>(1, rp.corr[d].size())));
    const size_t ngs = rp.gsend.size(), ngr = rp.grecv_off.back(), nfs = rp.fsend.size(), nfr = rp.frecv_off.back();
    a->gitems = reinterpret_cast<GuardE*>(take(sizeof(GuardE) * std::max<size_t>(1, ngs)));
    a->fitems = reinterpret_cast<long long*>(take(sizeof(long long) * std::max<size_t>(1, nfs)));
    a->gsend = reinterpret_cast<double*>(take(sizeof(double) * g.nv * std::max<size_t>(1, ngs)));
    a->grecv = reinterpret_cast<double*>(take(sizeof(double) * g.nv * std::max<size_t>(1, ngr)));
    a->fsend = reinterpret_cast<double*>(take(sizeof(double) * g.nv * std::max<size_t>(1, nfs)));
    a->frecv = reinterpret_cast<double*>(take(sizeof(double) * g.nv * std::max<size_t>(1, nfr)));
    auto up = [&](void* dst, const void* src, size_t bytes) {
        if (bytes) ACU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, a->stream));
    };
    std::vector<GuardE> gmap = rp.guards;  // minus the faces copied as whole slabs
    std::vector<long long> sface;
    compress_faces(g, gmap, sface);
    up(a->guards, gmap.data(), sizeof(GuardE) * gmap.size());
    const std::vector<long long> goff = guard_offsets(gmap, g.nleaf, g.np);
    up(a->goff, goff.data(), sizeof(long long) * goff.size());
    up(a->sface, sface.data(), sizeof(long long) * sface.size());
    for (int d = 0; d < 3; d++) up(a->corr[d], rp.corr[d].data(), sizeof(CorrE) * rp.corr[d].size());
    up(a->gitems, rp.gsend.data(), sizeof(GuardE) * ngs);
    up(a->fitems, rp.fsend.data(), sizeof(long long) * nfs);
    launched(spark::launch_scalars_reset(a->sc, a->stream), "scalars reset");
    ACU(cudaStreamSynchronize(a->stream));  // the host plan vectors are the copy sources
}

// one composite step of every member (a group of one: the single-rank path)
void group_step(const std::vector<spark_amr*>& m, double dt, double t_end) {
    spark_amr* a0 = m[0];
    const int S = a0->plan.c.rk_stages;
    auto group_min = [&]() {
        if (m.size() < 2) return;
        spark::AccPtrs p{};
        for (size_t r = 0; r < m.size(); r++) p.p[r] = &m[r]->sc->acc;
        launched(spark::launch_group_min(p, (int)m.size(), a0->stream), "group min");
    };
    group_min();  // the global CFL minimum of U^n (set_state computes it per member)
    std::vector<int> n(m.size()), x(m.size()), y(m.size());
    for (size_t r = 0; r < m.size(); r++) {
        spark_amr* a = m[r];
        if (!a->have_state) throw AmrError(SPARK_ERR_STATE, "no state loaded");
        n[r] = a->n_idx, x[r] = (n[r] + 1) % 3, y[r] = (n[r] + 2) % 3;
        launched(spark::launch_step_begin(a->sc, dt, t_end, a->plan.c.cfl, a->stream), "step begin");
        const AmrGeo& g = a->rp.g;
        ACU(cudaMemsetAsync(a->B, 0, sizeof(double) * g.nv * std::max(1LL, g.nleaf) * 6 * g.mf, a->stream));
    }
    // Shu-Osher stages: RK2 n->x, (x,n)->y; RK3 n->x, (x,n)->y, (y,n)->x
    static const double ca[2][3] = {{0.0, 0.5, 0.0}, {0.0, 0.75, 1.0 / 3.0}};
    static const double cb[2][3] = {{1.0, 0.5, 0.0}, {1.0, 0.25, 2.0 / 3.0}};
    const int row = S == 2 ? 0 : 1;
    for (int s = 0; s < S; s++) {
        std::vector<int> pi(m.size()), po(m.size());
        for (size_t r = 0; r < m.size(); r++) {
            const int prev[3] = {n[r], x[r], y[r]}, outb[3] = {x[r], y[r], x[r]};
            pi[r] = prev[s];
            po[r] = outb[s];
        }
        amr_exchange(m, pi.data(), false);  // guard values across ranks (fill_guardcells)
        for (size_t r = 0; r < m.size(); r++)
            amr_stage(m[r], m[r]->U[pi[r]], m[r]->U[n[r]], ca[row][s], cb[row][s], m[r]->U[po[r]]);
    }
    amr_exchange(m, nullptr, true);  // communicate_fluxes
    for (size_t r = 0; r < m.size(); r++) {
        const int newn = S == 2 ? y[r] : x[r];
        amr_correct(m[r], m[r]->U[newn]);  // flux correction
        amr_cfl(m[r], m[r]->U[newn]);      // CFL minimum of the corrected state: dt of the next step
        m[r]->n_idx = newn;
    }
    group_min();
}

// synchronise; on a failure roll back every member (the failing step) or none
void group_check(const std::vector<spark_amr*>& m, const std::vector<int>& old, double* dt_used) {
    std::vector<spark::DevScalars> h(m.size());
    for (size_t r = 0; r < m.size(); r++) h[r] = read_sc(m[r]);
    if (h[0].bad != spark::kNoBad) {
        const bool now = h[0].active && h[0].bad == (unsigned long long)h[0].steps;
        if (now) {
            for (size_t r = 0; r < m.size(); r++) {
                spark::DevScalars x = h[r];
                m[r]->n_idx = old[r];
                x.t = x.t_prev;
                x.steps -= 1;
                x.acc = x.acc_prev;
                x.bad = spark::kNoBad;
                x.status = 0;
                ACU(cudaMemcpy(m[r]->sc, &x, sizeof(x), cudaMemcpyHostToDevice));
            }
            throw AmrError(SPARK_ERR_NONPHYSICAL, "non-physical state; rolled back to U^n");
        }
        throw AmrError(SPARK_ERR_NONPHYSICAL, "non-physical state in step " + std::to_string(h[0].bad) +
                                                  "; later steps were frozen, state not rolled back");
    }
    if (dt_used) *dt_used = h[0].dt;
}

}  // namespace

extern "C" {

spark_status spark_amr_leaves(const spark_config* cfg, const spark_refine* ref, int64_t* ncoarse, int64_t* nfine) {
    return amr_guard(nullptr, [&] {
        AmrPlan p = make_amr_plan(cfg, ref);
        if (ncoarse) *ncoarse = p.g.ncl;
        if (nfine) *nfine = p.g.nleaf - p.g.ncl;
    });
}

spark_status spark_amr_rank_leaves(const spark_config* cfg, const spark_refine* ref, int32_t rank, int32_t nranks,
                                   int64_t* first, int64_t* count) {
    return amr_guard(nullptr, [&] {
        AmrPlan p = make_amr_plan(cfg, ref);
        if (nranks < 1 || nranks > p.g.nleaf || rank < 0 || rank >= nranks)
            throw AmrError(SPARK_ERR_ARG, "bad rank / nranks");
        const long long a = p.g.nleaf * rank / nranks, b = p.g.nleaf * (rank + 1) / nranks;
        if (first) *first = a;
        if (count) *count = b - a;
    });
}

spark_status spark_amr_required_bytes(const spark_config* cfg, const spark_refine* ref, size_t* bytes) {
    return amr_guard(nullptr, [&] {
        if (!bytes) throw AmrError(SPARK_ERR_ARG, "null bytes");
        *bytes = rank_bytes(partition(make_amr_plan(cfg, ref), 1)[0]);
    });
}

spark_status spark_amr_group_required_bytes(const spark_config* cfg, const spark_refine* ref, int32_t nranks,
                                            size_t* bytes) {
    return amr_guard(nullptr, [&] {
        if (!bytes) throw AmrError(SPARK_ERR_ARG, "null bytes");
        size_t b = 0;
        for (const RankPlan& rp : partition(make_amr_plan(cfg, ref), nranks)) b = std::max(b, rank_bytes(rp));
        *bytes = b;
    });
}

spark_status spark_amr_init(const spark_config* cfg, const spark_refine* ref, int32_t device, void* cuda_stream,
                            void* arena, size_t arena_bytes, spark_amr** out) {
    return spark_amr_init_local_group(cfg, ref, 1, device, cuda_stream, &arena, arena_bytes, out);
}

spark_status spark_amr_init_local_group(const spark_config* cfg, const spark_refine* ref, int32_t nranks,
                                        int32_t device, void* cuda_stream, void* const* arenas, size_t arena_bytes,
                                        spark_amr** outs) {
    if (!outs || !arenas || nranks < 1 || nranks > spark::kMaxGroup) return SPARK_ERR_ARG;
    std::vector<std::unique_ptr<spark_amr>> made;
    spark_status st = amr_guard(nullptr, [&] {
        AmrPlan P = make_amr_plan(cfg, ref);
        std::vector<RankPlan> R = partition(P, nranks);
        auto grp = std::make_shared<std::vector<spark_amr*>>();
        for (int r = 0; r < nranks; r++) {
            std::unique_ptr<spark_amr> a(new spark_amr());
            a->plan = P;
            a->rp = R[r];
            a->rank = r;
            a->nranks = nranks;
            a->device = device;
            a->stream = static_cast<cudaStream_t>(cuda_stream);
            a->group = grp;
            carve_member(a.get(), arenas[r], arena_bytes);
            grp->push_back(a.get());
            made.push_back(std::move(a));
        }
    });
    if (st != SPARK_OK) return st;
    for (int r = 0; r < nranks; r++) outs[r] = made[r].release();
    return SPARK_OK;
}

spark_status spark_amr_finalize(spark_amr* a) {
    if (!a) return SPARK_ERR_ARG;
    spark_status st = amr_guard(a, [&] { ACU(cudaStreamSynchronize(a->stream)); });
    if (a->group) {
        auto& m = *a->group;
        m.erase(std::remove(m.begin(), m.end(), a), m.end());
    }
    delete a;
    return st;
}

const char* spark_amr_last_error(const spark_amr* a) { return a ? a->err.c_str() : "null context"; }

spark_status spark_amr_set_state(spark_amr* a, const double* U, int32_t on_device) {
    if (!a || !U) return SPARK_ERR_ARG;
    return amr_guard(a, [&] {
        ACU(cudaSetDevice(a->device));
        const AmrGeo& g = a->rp.g;
        a->n_idx = 0;
        if (g.nleaf)
            ACU(cudaMemcpyAsync(a->U[0], U, sizeof(double) * g.nv * g.nleaf * g.nc,
                                on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, a->stream));
        launched(spark::launch_scalars_reset(a->sc, a->stream), "scalars reset");
        amr_cfl(a, a->U[0]);
        a->have_state = true;
    });
}

spark_status spark_amr_get_state(spark_amr* a, double* U, int32_t on_device) {
    if (!a || !U) return SPARK_ERR_ARG;
    return amr_guard(a, [&] {
        if (!a->have_state) throw AmrError(SPARK_ERR_STATE, "no state loaded");
        ACU(cudaSetDevice(a->device));
        const AmrGeo& g = a->rp.g;
        if (g.nleaf)
            ACU(cudaMemcpyAsync(U, a->U[a->n_idx], sizeof(double) * g.nv * g.nleaf * g.nc,
                                on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, a->stream));
        spark::DevScalars h = read_sc(a);
        if (h.bad != spark::kNoBad)
            throw AmrError(SPARK_ERR_NONPHYSICAL, "non-physical state in step " + std::to_string(h.bad));
    });
}

spark_status spark_amr_fill_guardcells(spark_amr* a, double* padded_out) {
    if (!a || !padded_out) return SPARK_ERR_ARG;
    return amr_guard(a, [&] {
        if (!a->have_state) throw AmrError(SPARK_ERR_STATE, "no state loaded");
        if (a->nranks != 1) throw AmrError(SPARK_ERR_STATE, "spark_amr_fill_guardcells needs a single-rank context");
        ACU(cudaSetDevice(a->device));
        const AmrGeo& g = a->rp.g;
        // corners / edges are never written: NaN, as in the oracle
        ACU(cudaMemsetAsync(padded_out, 0xff, sizeof(double) * g.nv * g.nleaf * g.np, a->stream));
        amr_fill(a, a->U[a->n_idx], padded_out, 0);
    });
}

spark_status spark_amr_step(spark_amr* a, double dt, double t_end, double* dt_used) {
    if (!a) return SPARK_ERR_ARG;
    return amr_guard(a, [&] {
        if (a->nranks != 1) throw AmrError(SPARK_ERR_STATE, "local-group contexts step with spark_amr_step_group");
        ACU(cudaSetDevice(a->device));
        std::vector<spark_amr*> m{a};
        std::vector<int> old{a->n_idx};
        group_step(m, dt, t_end);
        if (dt_used) group_check(m, old, dt_used);
    });
}

spark_status spark_amr_step_group(spark_amr* const* amrs, int32_t n, double dt, double t_end, double* dt_used) {
    if (!amrs || n < 1 || !amrs[0]) return SPARK_ERR_ARG;
    spark_amr* a0 = amrs[0];
    return amr_guard(a0, [&] {
        if (!a0->group || (int)a0->group->size() != n) throw AmrError(SPARK_ERR_ARG, "needs all members of one group");
        if (n != a0->nranks) throw AmrError(SPARK_ERR_STATE, "a member of this group was finalized");
        ACU(cudaSetDevice(a0->device));
        std::vector<spark_amr*> m(*a0->group);
        std::vector<int> old;
        for (spark_amr* a : m) old.push_back(a->n_idx);
        group_step(m, dt, t_end);
        if (dt_used) group_check(m, old, dt_used);
    });
}

spark_status spark_amr_get_time(spark_amr* a, double* t, int64_t* steps, double* dt_last) {
    if (!a) return SPARK_ERR_ARG;
    return amr_guard(a, [&] {
        spark::DevScalars h = read_sc(a);
        if (t) *t = h.t;
        if (steps) *steps = h.steps;
        if (dt_last) *dt_last = h.dt;
    });
}

}  // extern "C"
