// spark_kernels.cu — sm_100a kernels of the Spark block-update hot path.
//
// KB1  stage_kernel     fused stage: guard gather -> EOS (cons->prim) ->
//                       reconstruction (calcLims) -> Riemann flux (calcFlux) ->
//                       flux divergence + SSP-RK combination (updSoln) ->
//                       positivity check / CFL-min epilogue (calcEos).
//                       PAPER.md Alg. 8 fused into one pass over
//                       HBM per stage of lst:spark-nontelescoping.
// KB2  pack_kernel, fill_padded_kernel   guard-cell maps
// KB3  cfl_min_kernel   CFL minimum of a state (initial dt)
//      step_begin_kernel  dt = cfl * min, clip to t_end, stop flag
//
// The numerics are the textbook readings of DESIGN.md §3 (the paper states no
// formulas).  FP64 throughout: this is a stencil, not a contraction, so there
// is no tensor-core path.
//
// Data layout (HBM): struct-of-arrays block pool U[v][b][k][j][i]; the guard
// cells are NOT stored: each CTA gathers its block's face halos straight from
// the neighbouring blocks (L2-resident), from the received rank slabs, or from
// the physical boundary map.
//
// KB1 design (3-D): one CTA per block, one thread per (i,j) column, marching in
// k.  A ring of 2*NG primitive planes (own column only) lives in shared
// memory; each z-face flux is computed once by its column's thread and kept in
// registers for the next plane; x/y faces of the current plane are computed
// once into shared memory and read by both neighbouring cells.  1-D/2-D use
// the same kernel with a single plane.
#include <cfloat>
#include <cmath>
#include <cstdint>

#include "spark_internal.h"

namespace spark {
namespace {

constexpr int BC_PERIODIC = 0, BC_OUTFLOW = 1;  // BC_REFLECT = 2
constexpr int kStageThreads = 256;

template <int RECON>
struct StencilOf {
    static constexpr int NG = RECON == 2 ? 3 : (RECON == 1 ? 2 : 1);
};

// ------------------------------------------------------------ guard gather
// Conserved values of the cell at sub-box coordinates l (may lie up to ng
// cells outside the sub-box).  Out-of-box coordinates are resolved per
// dimension: a face with a peer rank reads the received slab, otherwise the
// physical boundary map (periodic wrap / outflow clamp / reflect mirror with
// the normal momentum negated).  Returns false (and leaves out unset) when the
// cell lies outside the sub-box in two or more peer directions (an edge or
// corner owned by a diagonal rank, never needed by the star stencil).
template <int NV>
__device__ __forceinline__ bool fetch_cons(const Geo& g, const double* __restrict__ u,
                                           const double* const (&halo)[3][2], int l0, int l1, int l2,
                                           double* out) {
    int l[3] = {l0, l1, l2};
    bool flip[3] = {false, false, false};
    int hd = -1, hs = 0;
#pragma unroll
    for (int d = 0; d < 3; d++) {
        if (d >= g.ndim) continue;
        const int x = l[d];
        if (x < 0 || x >= g.cn[d]) {
            const int side = x >= g.cn[d] ? 1 : 0;
            if (g.halo[d][side]) {
                if (hd >= 0) return false;
                hd = d;
                hs = side;
            } else {
                const int N = g.gN[d];
                int gx = g.off[d] + x;
                const int bc = g.bc[d][side];
                if (bc == BC_PERIODIC) {
                    gx %= N;
                    if (gx < 0) gx += N;
                } else if (bc == BC_OUTFLOW) {
                    gx = side ? N - 1 : 0;
                } else {
                    gx = side ? 2 * N - 1 - gx : -1 - gx;
                    flip[d] = true;
                }
                l[d] = gx - g.off[d];
            }
        }
    }
    const double* base;
    long long idx, stride;
    if (hd >= 0) {
        int c[3] = {l[0], l[1], l[2]};
        c[hd] = hs ? l[hd] - g.cn[hd] : l[hd] + g.ng;
        const int e0 = hd == 0 ? g.ng : g.cn[0];
        const int e1 = hd == 1 ? g.ng : g.cn[1];
        idx = ((long long)c[2] * e1 + c[1]) * e0 + c[0];
        base = halo[hd][hs];
        stride = g.slab[hd];
    } else {
        const int bx = l[0] / g.nb[0], by = l[1] / g.nb[1], bz = l[2] / g.nb[2];
        const long long blk = bx + (long long)g.bn[0] * (by + (long long)g.bn[1] * bz);
        idx = blk * g.cpb + ((long long)(l[2] - bz * g.nb[2]) * g.nb[1] + (l[1] - by * g.nb[1])) * g.nb[0] +
              (l[0] - bx * g.nb[0]);
        base = u;
        stride = g.ncell;
    }
#pragma unroll
    for (int v = 0; v < NV; v++) out[v] = base[v * stride + idx];
#pragma unroll
    for (int d = 0; d < NV - 2; d++)
        if (flip[d]) out[1 + d] = -out[1 + d];
    return true;
}

// ------------------------------------------------------------------- EOS
// Ideal gas (EOS unit): u = m/rho, p = (gamma-1)(E - m.u/2).
// Returns false for rho <= 0, p <= 0 or non-finite p (calcEos check).
template <int NV>
__device__ __forceinline__ bool cons_to_prim(const double* u, double* w, double gamma) {
    const double rho = u[0];
    const double inv = 1.0 / rho;
    double ke = 0.0;
#pragma unroll
    for (int d = 1; d < NV - 1; d++) {
        w[d] = u[d] * inv;
        ke += u[d] * w[d];
    }
    w[0] = rho;
    const double p = (gamma - 1.0) * (u[NV - 1] - 0.5 * ke);
    w[NV - 1] = p;
    return rho > 0.0 && p > 0.0 && p < INFINITY;
}

// -------------------------------------------------------- reconstruction
__device__ __forceinline__ double minmod(double a, double b) {
    return (a > 0.0 && b > 0.0) ? fmin(a, b) : ((a < 0.0 && b < 0.0) ? fmax(a, b) : 0.0);
}

// WENO5-JS value at the right edge of the middle cell of (a,b,c,d,e).
__device__ __forceinline__ double weno5_edge(double a, double b, double c, double d, double e) {
    const double eps = 1e-6;
    const double t0 = a - 2.0 * b + c, s0 = a - 4.0 * b + 3.0 * c;
    const double t1 = b - 2.0 * c + d, s1 = b - d;
    const double t2 = c - 2.0 * d + e, s2 = 3.0 * c - 4.0 * d + e;
    const double b0 = (13.0 / 12.0) * t0 * t0 + 0.25 * s0 * s0;
    const double b1 = (13.0 / 12.0) * t1 * t1 + 0.25 * s1 * s1;
    const double b2 = (13.0 / 12.0) * t2 * t2 + 0.25 * s2 * s2;
    const double a0 = 0.1 / ((eps + b0) * (eps + b0));
    const double a1 = 0.6 / ((eps + b1) * (eps + b1));
    const double a2 = 0.3 / ((eps + b2) * (eps + b2));
    const double q0 = (2.0 * a - 7.0 * b + 11.0 * c) / 6.0;
    const double q1 = (-b + 5.0 * c + 2.0 * d) / 6.0;
    const double q2 = (2.0 * c + 5.0 * d - e) / 6.0;
    return (a0 * q0 + a1 * q1 + a2 * q2) / (a0 + a1 + a2);
}

// ------------------------------------------------------------- Riemann
// HLL / HLLC (Toro §10.4), Davis wave speeds, in the rotated frame
// (rho, u_n, u_t..., p).  HLLC evaluates only the state K whose flux is
// selected (upwind side, or the star side given by sign(S*)).
template <int NV, int RS>
__device__ __forceinline__ void riemann(const double* wl, const double* wr, double gamma, double gm1i,
                                        double* f) {
    const double rl = wl[0], ul = wl[1], pl = wl[NV - 1];
    const double rr = wr[0], ur = wr[1], pr = wr[NV - 1];
    const double irl = 1.0 / rl, irr = 1.0 / rr;
    const double cl = sqrt(gamma * pl * irl), cr = sqrt(gamma * pr * irr);
    const double sl = fmin(ul - cl, ur - cr);
    const double sr = fmax(ul + cl, ur + cr);
    if (RS == 1) {
        const double ql = rl * (sl - ul), qr = rr * (sr - ur);  // rho_K (S_K - u_K)
        const double sstar = (pr - pl + ul * ql - ur * qr) / (ql - qr);
        const bool left = (sl >= 0.0) || (!(sr <= 0.0) && sstar >= 0.0);
        const bool star = !(sl >= 0.0) && !(sr <= 0.0);
        const double* w = left ? wl : wr;
        const double rho = left ? rl : rr, un = left ? ul : ur, p = left ? pl : pr;
        const double irho = left ? irl : irr, sk = left ? sl : sr, qk = left ? ql : qr;
        double u2 = 0.0;
#pragma unroll
        for (int m = 1; m < NV - 1; m++) u2 += w[m] * w[m];
        const double E = p * gm1i + 0.5 * rho * u2;
        const double mflux = rho * un;
        f[0] = mflux;
        f[1] = mflux * un + p;
#pragma unroll
        for (int m = 2; m < NV - 1; m++) f[m] = mflux * w[m];
        f[NV - 1] = un * (E + p);
        if (star) {
            const double fac = qk / (sk - sstar);
            const double es = E * irho + (sstar - un) * (sstar + p / qk);
            f[0] += sk * (fac - rho);
            f[1] += sk * (fac * sstar - mflux);
#pragma unroll
            for (int m = 2; m < NV - 1; m++) f[m] += sk * (fac * w[m] - rho * w[m]);
            f[NV - 1] += sk * (fac * es - E);
        }
    } else {
        double u2l = 0.0, u2r = 0.0;
#pragma unroll
        for (int m = 1; m < NV - 1; m++) {
            u2l += wl[m] * wl[m];
            u2r += wr[m] * wr[m];
        }
        const double El = pl * gm1i + 0.5 * rl * u2l, Er = pr * gm1i + 0.5 * rr * u2r;
        double UL[NV], UR[NV], FL[NV], FR[NV];
        UL[0] = rl;
        UR[0] = rr;
        FL[0] = rl * ul;
        FR[0] = rr * ur;
        FL[1] = rl * ul * ul + pl;
        FR[1] = rr * ur * ur + pr;
#pragma unroll
        for (int m = 1; m < NV - 1; m++) {
            UL[m] = rl * wl[m];
            UR[m] = rr * wr[m];
        }
#pragma unroll
        for (int m = 2; m < NV - 1; m++) {
            FL[m] = rl * ul * wl[m];
            FR[m] = rr * ur * wr[m];
        }
        UL[NV - 1] = El;
        UR[NV - 1] = Er;
        FL[NV - 1] = ul * (El + pl);
        FR[NV - 1] = ur * (Er + pr);
        if (sl >= 0.0) {
#pragma unroll
            for (int v = 0; v < NV; v++) f[v] = FL[v];
        } else if (sr <= 0.0) {
#pragma unroll
            for (int v = 0; v < NV; v++) f[v] = FR[v];
        } else {
            const double inv = 1.0 / (sr - sl);
#pragma unroll
            for (int v = 0; v < NV; v++) f[v] = (sr * FL[v] - sl * FR[v] + sl * sr * (UR[v] - UL[v])) * inv;
        }
    }
}

// Rotated component r of direction d -> unrotated variable index.
template <int NDIM>
__device__ __forceinline__ int rot_var(int d, int r) {
    constexpr int NV = NDIM + 2;
    if (r == 0 || r == NV - 1) return r;
    if (r == 1) return 1 + d;
    // transverse velocities in increasing axis order
    int t = r - 2;  // 0 or 1
    int e = (t < d) ? t : t + 1;
    return 1 + e;
}

// Face flux from a stencil reader rd(var, m) (unrotated var, m = 0..2NG-1
// covering cells i-NG+1 .. i+NG for the face at i+1/2).
template <int NDIM, int RECON, int RS, typename Rd>
__device__ __forceinline__ void face_flux(const Rd& rd, int d, double gamma, double gm1i, double* f) {
    constexpr int NV = NDIM + 2;
    constexpr int NG = StencilOf<RECON>::NG;
    double wl[NV], wr[NV];
#pragma unroll
    for (int r = 0; r < NV; r++) {
        const int v = rot_var<NDIM>(d, r);
        if (RECON == 0) {
            wl[r] = rd(v, NG - 1);
            wr[r] = rd(v, NG);
        } else if (RECON == 1) {
            const double a = rd(v, NG - 2), b = rd(v, NG - 1), c = rd(v, NG), e = rd(v, NG + 1);
            wl[r] = b + 0.5 * minmod(b - a, c - b);
            wr[r] = c - 0.5 * minmod(c - b, e - c);
        } else {
            const double s0 = rd(v, 0), s1 = rd(v, 1), s2 = rd(v, 2), s3 = rd(v, 3), s4 = rd(v, 4), s5 = rd(v, 5);
            wl[r] = weno5_edge(s0, s1, s2, s3, s4);
            wr[r] = weno5_edge(s5, s4, s3, s2, s1);
        }
    }
    if (RECON != 0) {
        if (!(wl[0] > 0.0 && wl[NV - 1] > 0.0 && wr[0] > 0.0 && wr[NV - 1] > 0.0)) {
#pragma unroll
            for (int r = 0; r < NV; r++) {
                const int v = rot_var<NDIM>(d, r);
                wl[r] = rd(v, NG - 1);
                wr[r] = rd(v, NG);
            }
        }
    }
    double fr[NV];
    riemann<NV, RS>(wl, wr, gamma, gm1i, fr);
#pragma unroll
    for (int r = 0; r < NV; r++) f[rot_var<NDIM>(d, r)] = fr[r];
}

__device__ __forceinline__ double warp_min(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// CFL term of one primitive state: min_d dx_d / (|u_d| + c).
template <int NV>
__device__ __forceinline__ double cfl_term(const Geo& g, const double* w) {
    const double c = sqrt(g.gamma * w[NV - 1] / w[0]);
    double best = INFINITY;
#pragma unroll
    for (int d = 0; d < NV - 2; d++) best = fmin(best, g.dx[d] / (fabs(w[1 + d]) + c));
    return best;
}

// Block-wide min of x -> atomicMin on the u64 bits (positive doubles order
// like unsigned integers; +inf is the identity).  All threads must call.
__device__ __forceinline__ void block_min_to(double x, double* red, unsigned long long* acc) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    // partial warps: pad with +inf through a full-warp shuffle of a guarded value
    x = warp_min(x);
    if (lane == 0) red[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = red[0];
        for (int w = 1; w < nw; w++) m = fmin(m, red[w]);
        if (m < INFINITY) atomicMin(acc, (unsigned long long)__double_as_longlong(m));
    }
}

// --------------------------------------------------------------- KB1
template <int NDIM, int RECON, int RS>
__global__ void __launch_bounds__(kStageThreads) stage_kernel(const StageArgs A) {
    constexpr int NV = NDIM + 2;
    constexpr int NG = StencilOf<RECON>::NG;
    constexpr int RING = NDIM == 3 ? 2 * NG : 0;
    const Geo& g = A.g;
    extern __shared__ double smem[];

    const int nb0 = g.nb[0];
    const int nb1 = NDIM >= 2 ? g.nb[1] : 1;
    const int nb2 = NDIM >= 3 ? g.nb[2] : 1;
    const int P = nb0 * nb1;
    const int tid = threadIdx.x;
    const bool live = tid < P;  // blockDim is rounded up to a warp multiple
    const int ti = live ? tid % nb0 : 0, tj = live ? tid / nb0 : 0;
    const int b = blockIdx.x;
    const int bx = b % g.bn[0], by = (b / g.bn[0]) % g.bn[1], bz = b / (g.bn[0] * g.bn[1]);
    const int cx0 = bx * nb0, cy0 = by * nb1, cz0 = bz * nb2;
    const long long bbase = (long long)b * g.cpb;
    const long long ncell = g.ncell;

    const int cw = nb0 + 2 * NG, ch = NDIM >= 2 ? nb1 + 2 * NG : 1;
    constexpr int RO = NDIM >= 2 ? NG : 0;  // row offset of the interior in cur
    const int CP = cw * ch;
    const int nfx = (nb0 + 1) * nb1;
    const int nfy = NDIM >= 2 ? nb0 * (nb1 + 1) : 0;
    double* ring = smem;                   // [RING][NV][P]
    double* cur = ring + RING * NV * P;    // [NV][CP]
    double* Fx = cur + NV * CP;            // [NV][nfx]
    double* Fy = Fx + NV * nfx;            // [NV][nfy]
    double* red = Fy + NV * nfy;           // [32]

    const double dt = A.dt_ptr ? *A.dt_ptr : A.dt_value;
    const double a = A.a, bco = A.b;
    const double gamma = g.gamma, gm1i = 1.0 / (g.gamma - 1.0);

    if (A.honor_active && !A.sc->active) {  // t >= t_end: U^(s) = U^(s-1)
        if (live)
            for (int kk = 0; kk < nb2; kk++) {
                const long long idx = bbase + ((long long)kk * nb1 + tj) * nb0 + ti;
#pragma unroll
                for (int v = 0; v < NV; v++) A.uout[v * ncell + idx] = A.uprev[v * ncell + idx];
            }
        return;
    }

    bool ok = true;
    double cflmin = INFINITY;
    double fz_lo[NV], fz_hi[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) fz_lo[v] = fz_hi[v] = 0.0;

    // load one plane z (block-local k, may be outside the block) of this thread's column
    auto load_column = [&](int z, double* w) {
        double u[NV];
        if (z >= 0 && z < nb2) {
            const long long idx = bbase + ((long long)z * nb1 + tj) * nb0 + ti;
#pragma unroll
            for (int v = 0; v < NV; v++) u[v] = A.uprev[v * ncell + idx];
        } else {
            fetch_cons<NV>(g, A.uprev, A.halo, cx0 + ti, cy0 + tj, cz0 + z, u);
        }
        ok &= cons_to_prim<NV>(u, w, gamma);
    };

    if (NDIM == 3) {
        if (live)
            for (int z = -NG; z < NG; z++) {
                double w[NV];
                load_column(z, w);
                const int slot = z + NG;
#pragma unroll
                for (int v = 0; v < NV; v++) ring[(slot * NV + v) * P + tid] = w[v];
            }
        __syncthreads();
        if (live) {  // z-face at k = -1/2
            auto rd = [&](int v, int m) { return ring[(((m) % (2 * NG)) * NV + v) * P + tid]; };
            face_flux<NDIM, RECON, RS>(rd, 2, gamma, gm1i, fz_lo);
        }
    }

    const int nh = 2 * NG * nb1 + (NDIM >= 2 ? 2 * NG * nb0 : 0);
    for (int kk = 0; kk < nb2; kk++) {
        __syncthreads();
        if (live) {
            if (NDIM == 3) {
                double w[NV];
                load_column(kk + NG, w);
                const int slot = kk % (2 * NG);
#pragma unroll
                for (int v = 0; v < NV; v++) ring[(slot * NV + v) * P + tid] = w[v];
                const int cs = (kk + NG) % (2 * NG);
#pragma unroll
                for (int v = 0; v < NV; v++) cur[v * CP + (tj + RO) * cw + ti + NG] = ring[(cs * NV + v) * P + tid];
            } else {
                double w[NV];
                load_column(kk, w);
#pragma unroll
                for (int v = 0; v < NV; v++) cur[v * CP + (tj + RO) * cw + ti + NG] = w[v];
            }
        }
        // x/y face halos of this plane
        for (int h = tid; h < nh; h += blockDim.x) {
            int cx, cy;
            if (h < 2 * NG * nb1) {  // x strips: [side][row][depth]
                const int side = h / (NG * nb1), r = h % (NG * nb1);
                cy = r / NG;
                const int dpt = r % NG;
                cx = side ? nb0 + dpt : dpt - NG;
            } else {  // y strips
                const int hh = h - 2 * NG * nb1;
                const int side = hh / (NG * nb0), r = hh % (NG * nb0);
                const int dpt = r / nb0;
                cx = r % nb0;
                cy = side ? nb1 + dpt : dpt - NG;
            }
            double u[NV], w[NV];
            fetch_cons<NV>(g, A.uprev, A.halo, cx0 + cx, cy0 + cy, cz0 + kk, u);
            ok &= cons_to_prim<NV>(u, w, gamma);
#pragma unroll
            for (int v = 0; v < NV; v++) cur[v * CP + (cy + RO) * cw + cx + NG] = w[v];
        }
        __syncthreads();
        // x and y faces of the plane -> shared memory (each face once)
        for (int f = tid; f < nfx + nfy; f += blockDim.x) {
            double fl[NV];
            int fidx;
            double* F;
            int nf;
            if (f < nfx) {
                const int fi = f % (nb0 + 1), fj = f / (nb0 + 1);
                const int base = (fj + RO) * cw + fi;  // stencil m -> column fi + m
                auto rd = [&](int v, int m) { return cur[v * CP + base + m]; };
                face_flux<NDIM, RECON, RS>(rd, 0, gamma, gm1i, fl);
                F = Fx;
                nf = nfx;
                fidx = f;
            } else {
                const int q = f - nfx;
                const int fi = q % nb0, fj = q / nb0;
                const int base = fj * cw + fi + NG;  // stencil m -> row fj + m
                auto rd = [&](int v, int m) { return cur[v * CP + base + m * cw]; };
                face_flux<NDIM, RECON, RS>(rd, 1, gamma, gm1i, fl);
                F = Fy;
                nf = nfy;
                fidx = q;
            }
#pragma unroll
            for (int v = 0; v < NV; v++) F[v * nf + fidx] = fl[v];
        }
        if (NDIM == 3 && live) {  // z-face at kk + 1/2 from the ring (own column)
            auto rd = [&](int v, int m) { return ring[(((kk + 1 + m) % (2 * NG)) * NV + v) * P + tid]; };
            face_flux<NDIM, RECON, RS>(rd, 2, gamma, gm1i, fz_hi);
        }
        __syncthreads();
        if (live) {
            const long long idx = bbase + ((long long)kk * nb1 + tj) * nb0 + ti;
            double un[NV];
#pragma unroll
            for (int v = 0; v < NV; v++) {
                const double dfx = (Fx[v * nfx + tj * (nb0 + 1) + ti + 1] - Fx[v * nfx + tj * (nb0 + 1) + ti]) * g.rdx[0];
                double L;
                if (NDIM == 1) {
                    L = -dfx;
                } else {
                    const double dfy = (Fy[v * nfy + (tj + 1) * nb0 + ti] - Fy[v * nfy + tj * nb0 + ti]) * g.rdx[1];
                    if (NDIM == 2) L = -(dfx + dfy);
                    else L = -(dfx + dfy) - (fz_hi[v] - fz_lo[v]) * g.rdx[2];
                }
                const double up = A.uprev[v * ncell + idx];
                const double uo = (a != 0.0 ? a * A.un[v * ncell + idx] : 0.0) + bco * (up + dt * L);
                A.uout[v * ncell + idx] = uo;
                un[v] = uo;
            }
            if (A.last) {
                double w[NV];
                ok &= cons_to_prim<NV>(un, w, gamma);
                cflmin = fmin(cflmin, cfl_term<NV>(g, w));
            }
#pragma unroll
            for (int v = 0; v < NV; v++) fz_lo[v] = fz_hi[v];
        }
    }
    if (!ok) atomicOr(&A.sc->status, 1);
    if (A.last) {
        __syncthreads();
        block_min_to(cflmin, red, &A.sc->acc);
    }
}

// --------------------------------------------------------------- KB3
template <int NDIM>
__global__ void cfl_min_kernel(const Geo g, const double* __restrict__ u, DevScalars* sc) {
    constexpr int NV = NDIM + 2;
    __shared__ double red[32];
    double m = INFINITY;
    bool ok = true;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.ncell;
         q += (long long)gridDim.x * blockDim.x) {
        double c[NV], w[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) c[v] = u[v * g.ncell + q];
        ok &= cons_to_prim<NV>(c, w, g.gamma);
        m = fmin(m, cfl_term<NV>(g, w));
    }
    if (!ok) atomicOr(&sc->status, 1);
    block_min_to(m, red, &sc->acc);
}

__global__ void step_begin_kernel(DevScalars* sc, double dt_fixed, double t_end, double cfl) {
    const double t = sc->t;
    if (dt_fixed <= 0.0 && t_end > 0.0 && t >= t_end * (1.0 - 1e-14)) {
        sc->dt = 0.0;
        sc->active = 0;
        sc->t_prev = t;
        sc->acc_prev = sc->acc;  // keep the CFL minimum of the unchanged state
        return;
    }
    double dt;
    if (dt_fixed > 0.0) {
        dt = dt_fixed;
    } else {
        dt = cfl * __longlong_as_double((long long)sc->acc);
        if (t_end > 0.0 && dt > t_end - t) dt = t_end - t;
    }
    sc->dt = dt;
    sc->active = 1;
    sc->t_prev = t;
    sc->t = t + dt;
    sc->steps += 1;
    sc->acc_prev = sc->acc;
    sc->acc = 0x7ff0000000000000ull;  // +inf
}

__global__ void group_min_kernel(const AccPtrs p, int n) {
    unsigned long long m = ~0ull;
    for (int r = 0; r < n; r++) m = *p.p[r] < m ? *p.p[r] : m;
    for (int r = 0; r < n; r++) *p.p[r] = m;
}

__global__ void scalars_reset_kernel(DevScalars* sc) {
    sc->dt = 0.0;
    sc->t = 0.0;
    sc->t_prev = 0.0;
    sc->acc = 0x7ff0000000000000ull;
    sc->acc_prev = 0x7ff0000000000000ull;
    sc->status = 0;
    sc->active = 1;
    sc->steps = 0;
}

template <int NDIM>
__global__ void prim_to_cons_kernel(const Geo g, const double* __restrict__ w, double* __restrict__ u) {
    constexpr int NV = NDIM + 2;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.ncell;
         q += (long long)gridDim.x * blockDim.x) {
        const double rho = w[q];
        double u2 = 0.0;
#pragma unroll
        for (int d = 1; d < NV - 1; d++) {
            const double vel = w[d * g.ncell + q];
            u2 += vel * vel;
            u[d * g.ncell + q] = rho * vel;
        }
        u[q] = rho;
        u[(NV - 1) * g.ncell + q] = w[(NV - 1) * g.ncell + q] / (g.gamma - 1.0) + 0.5 * rho * u2;
    }
}

// --------------------------------------------------------------- KB2
// Pack the ng-thick slab of face (dim, side) of the sub-box: [v][c2][c1][c0].
template <int NV>
__global__ void pack_kernel(const Geo g, const double* __restrict__ u, int dim, int side,
                            double* __restrict__ slab) {
    const int e0 = dim == 0 ? g.ng : g.cn[0];
    const int e1 = dim == 1 ? g.ng : g.cn[1];
    const long long n = g.slab[dim];
    const double* const nohalo[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n;
         s += (long long)gridDim.x * blockDim.x) {
        int c[3] = {(int)(s % e0), (int)((s / e0) % e1), (int)(s / ((long long)e0 * e1))};
        if (side) c[dim] += g.cn[dim] - g.ng;
        double val[NV];
        fetch_cons<NV>(g, u, nohalo, c[0], c[1], c[2], val);
#pragma unroll
        for (int v = 0; v < NV; v++) slab[v * n + s] = val[v];
    }
}

struct HaloPtrs {
    const double* p[3][2];
};

// Materialise the padded per-block layout P[v][b][k+gz][j+gy][i+gx].
template <int NV>
__global__ void fill_padded_kernel(const Geo g, const double* __restrict__ u, const HaloPtrs hp,
                                   double* __restrict__ out) {
    int gd[3], pn[3];
    for (int d = 0; d < 3; d++) {
        gd[d] = d < g.ndim ? g.ng : 0;
        pn[d] = g.nb[d] + 2 * gd[d];
    }
    const long long np = (long long)pn[0] * pn[1] * pn[2];
    const long long nblk = (long long)g.bn[0] * g.bn[1] * g.bn[2];
    const long long total = np * nblk;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const long long b = q / np, r = q % np;
        const int pi = (int)(r % pn[0]), pj = (int)((r / pn[0]) % pn[1]), pk = (int)(r / ((long long)pn[0] * pn[1]));
        const int bx = (int)(b % g.bn[0]), by = (int)((b / g.bn[0]) % g.bn[1]), bz = (int)(b / ((long long)g.bn[0] * g.bn[1]));
        double val[NV];
        if (!fetch_cons<NV>(g, u, hp.p, bx * g.nb[0] + pi - gd[0], by * g.nb[1] + pj - gd[1],
                            bz * g.nb[2] + pk - gd[2], val)) {
#pragma unroll
            for (int v = 0; v < NV; v++) val[v] = __longlong_as_double(0x7ff8000000000000ll);
        }
#pragma unroll
        for (int v = 0; v < NV; v++) out[v * total + q] = val[v];
    }
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int NDIM, int RECON, int RS>
cudaError_t launch_stage_t(const StageArgs& a, cudaStream_t s) {
    const size_t smem = stage_smem_bytes(a.g, RECON);
    auto k = stage_kernel<NDIM, RECON, RS>;
    cudaError_t e = set_smem(k, smem);
    if (e != cudaSuccess) return e;
    const long long nblk = (long long)a.g.bn[0] * a.g.bn[1] * a.g.bn[2];
    k<<<(unsigned)nblk, stage_block_threads(a.g), smem, s>>>(a);
    return cudaGetLastError();
}

template <int NDIM>
cudaError_t launch_stage_d(const StageArgs& a, int recon, int riemann, cudaStream_t s) {
    if (recon == 0) return riemann ? launch_stage_t<NDIM, 0, 1>(a, s) : launch_stage_t<NDIM, 0, 0>(a, s);
    if (recon == 1) return riemann ? launch_stage_t<NDIM, 1, 1>(a, s) : launch_stage_t<NDIM, 1, 0>(a, s);
    return riemann ? launch_stage_t<NDIM, 2, 1>(a, s) : launch_stage_t<NDIM, 2, 0>(a, s);
}

unsigned grid_for(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    if (b > 148LL * 32) b = 148LL * 32;
    if (b < 1) b = 1;
    return (unsigned)b;
}

}  // namespace

int stage_block_threads(const Geo& g) {
    const int P = g.nb[0] * (g.ndim >= 2 ? g.nb[1] : 1);
    return ((P + 31) / 32) * 32;
}

size_t stage_smem_bytes(const Geo& g, int recon) {
    const int NG = recon == 2 ? 3 : (recon == 1 ? 2 : 1);
    const int NV = g.ndim + 2;
    const int nb0 = g.nb[0], nb1 = g.ndim >= 2 ? g.nb[1] : 1;
    const size_t P = (size_t)nb0 * nb1;
    const size_t ring = g.ndim == 3 ? 2 * NG * NV * P : 0;
    const size_t cw = nb0 + 2 * NG, ch = g.ndim >= 2 ? nb1 + 2 * NG : 1;
    const size_t cur = NV * cw * ch;
    const size_t fx = NV * (size_t)(nb0 + 1) * nb1;
    const size_t fy = g.ndim >= 2 ? NV * (size_t)nb0 * (nb1 + 1) : 0;
    return (ring + cur + fx + fy + 32) * sizeof(double);
}

cudaError_t launch_stage(const StageArgs& a, int recon, int riemann, cudaStream_t s) {
    if (a.g.ndim == 1) return launch_stage_d<1>(a, recon, riemann, s);
    if (a.g.ndim == 2) return launch_stage_d<2>(a, recon, riemann, s);
    return launch_stage_d<3>(a, recon, riemann, s);
}

cudaError_t launch_cfl_min(const Geo& g, const double* u, DevScalars* sc, cudaStream_t s) {
    const unsigned grid = grid_for(g.ncell, 256);
    if (g.ndim == 1) cfl_min_kernel<1><<<grid, 256, 0, s>>>(g, u, sc);
    else if (g.ndim == 2) cfl_min_kernel<2><<<grid, 256, 0, s>>>(g, u, sc);
    else cfl_min_kernel<3><<<grid, 256, 0, s>>>(g, u, sc);
    return cudaGetLastError();
}

cudaError_t launch_step_begin(DevScalars* sc, double dt_fixed, double t_end, double cfl, cudaStream_t s) {
    step_begin_kernel<<<1, 1, 0, s>>>(sc, dt_fixed, t_end, cfl);
    return cudaGetLastError();
}

cudaError_t launch_group_min(const AccPtrs& p, int n, cudaStream_t s) {
    group_min_kernel<<<1, 1, 0, s>>>(p, n);
    return cudaGetLastError();
}

cudaError_t launch_scalars_reset(DevScalars* sc, cudaStream_t s) {
    scalars_reset_kernel<<<1, 1, 0, s>>>(sc);
    return cudaGetLastError();
}

cudaError_t launch_prim_to_cons(const Geo& g, const double* w, double* u, cudaStream_t s) {
    const unsigned grid = grid_for(g.ncell, 256);
    if (g.ndim == 1) prim_to_cons_kernel<1><<<grid, 256, 0, s>>>(g, w, u);
    else if (g.ndim == 2) prim_to_cons_kernel<2><<<grid, 256, 0, s>>>(g, w, u);
    else prim_to_cons_kernel<3><<<grid, 256, 0, s>>>(g, w, u);
    return cudaGetLastError();
}

cudaError_t launch_pack(const Geo& g, const double* u, int dim, int side, double* slab, cudaStream_t s) {
    const unsigned grid = grid_for(g.slab[dim], 256);
    if (g.nvar == 3) pack_kernel<3><<<grid, 256, 0, s>>>(g, u, dim, side, slab);
    else if (g.nvar == 4) pack_kernel<4><<<grid, 256, 0, s>>>(g, u, dim, side, slab);
    else pack_kernel<5><<<grid, 256, 0, s>>>(g, u, dim, side, slab);
    return cudaGetLastError();
}

cudaError_t launch_fill_padded(const Geo& g, const double* u, const double* const halo[3][2], double* padded,
                               cudaStream_t s) {
    HaloPtrs hp;
    for (int d = 0; d < 3; d++)
        for (int q = 0; q < 2; q++) hp.p[d][q] = halo[d][q];
    long long np = 1;
    for (int d = 0; d < 3; d++) np *= g.nb[d] + 2 * (d < g.ndim ? g.ng : 0);
    const long long total = np * g.bn[0] * g.bn[1] * g.bn[2];
    const unsigned grid = grid_for(total, 256);
    if (g.nvar == 3) fill_padded_kernel<3><<<grid, 256, 0, s>>>(g, u, hp, padded);
    else if (g.nvar == 4) fill_padded_kernel<4><<<grid, 256, 0, s>>>(g, u, hp, padded);
    else fill_padded_kernel<5><<<grid, 256, 0, s>>>(g, u, hp, padded);
    return cudaGetLastError();
}

}  // namespace spark
