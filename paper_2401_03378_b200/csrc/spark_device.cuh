// spark_device.cuh — device helpers of the Spark hot path (sm_100a, FP64).
//
// EOS, reconstruction, Riemann solvers and the guard-cell gather shared by the
// kernels.  The paper prints no formulas; these are the textbook readings of
// DESIGN.md §3 (ideal gas; PLM-minmod / WENO5-JS on primitive variables with a
// first-order positivity fallback; HLL / HLLC with Davis wave speeds, Toro §10.4).
// Formulations are chosen for the FP64 issue budget of B200:
// reciprocals and square roots are one MUFU seed plus one cubic Newton step
// (<= 1 ulp from the correctly rounded value, no slow-path branches), the
// minmod limiter and the positivity tests run on the integer pipe, and the
// reconstruction is cell-centric (one limiter / smoothness evaluation per cell
// and direction, shared by the cell's two faces).
#pragma once

#include <cmath>
#include <cstdint>

#include "spark_internal.h"

namespace spark {
namespace dev {

constexpr int BC_PERIODIC = 0, BC_OUTFLOW = 1;  // BC_REFLECT = 2

template <int RECON>
struct StencilOf {
    // cells each side of a face: WENO5 / WENO5-Z 3, PLM / PLM-MC 2, first order 1
    static constexpr int NG = (RECON == 2 || RECON == 4) ? 3 : ((RECON == 1 || RECON == 3) ? 2 : 1);
};

// ------------------------------------------------------------ arithmetic
#ifdef SPARK_STRICT_MATH
// Parity build (libspark_strict.so, nvcc --fmad=false; DESIGN.md reading
// R16/R15): no fused multiply-add anywhere (explicit fma() calls become a
// rounded product plus a rounded sum, as the oracle's -ffp-contract=off C) and
// IEEE division / square root instead of the MUFU + Newton forms below.
__host__ __device__ __forceinline__ double spark_strict_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(__dmul_rn(a, b), c);
#else
    volatile double p = a * b;
    return p + c;
#endif
}
#define fma(a, b, c) spark_strict_fma((a), (b), (c))
__host__ __device__ __forceinline__ double rcp(double x) { return 1.0 / x; }
__host__ __device__ __forceinline__ double sqrt_fast(double a) { return sqrt(a); }
__host__ __device__ __forceinline__ double rsqrt_fast(double a) { return 1.0 / sqrt(a); }
#else
// 1/x: MUFU seed (~2^-22) and one cubic Newton step y(1 + e + e^2), e = 1 - xy.
__host__ __device__ __forceinline__ double rcp(double x) {
#ifdef __CUDA_ARCH__
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = __hiloint2double(__double2hiint(y), 0);  // MUFU.RCP64H writes the high word only
#else
    double y = (double)(1.0f / (float)x);  // host build (tests): same Newton step from an fp32 seed
#endif
    const double e = fma(-x, y, 1.0);
    return fma(y, fma(e, e, e), y);
}

// sqrt(a), a > 0: h = a y with y ~ 1/sqrt(a), then h(1 + r/2 + 3r^2/8), r = 1 - a y^2.
__host__ __device__ __forceinline__ double sqrt_fast(double a) {
#ifdef __CUDA_ARCH__
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    y = __hiloint2double(__double2hiint(y), 0);  // MUFU.RSQ64H writes the high word only
#else
    double y = (double)(1.0f / sqrtf((float)a));
#endif
    const double h = a * y;
    const double r = fma(-h, y, 1.0);
    return fma(h * r, fma(0.375, r, 0.5), h);
}

// 1/sqrt(a), a > 0: y (1 + r/2 + 3r^2/8), r = 1 - a y^2.
__host__ __device__ __forceinline__ double rsqrt_fast(double a) {
#ifdef __CUDA_ARCH__
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    y = __hiloint2double(__double2hiint(y), 0);
#else
    double y = (double)(1.0f / sqrtf((float)a));
#endif
    const double r = fma(-a * y, y, 1.0);
    return fma(y * r, fma(0.375, r, 0.5), y);
}
#endif  // SPARK_STRICT_MATH

// x > 0 for non-NaN x, on the integer pipe (+0 and -0 are not positive).
__host__ __device__ __forceinline__ long long dbits(double x) {
#ifdef __CUDA_ARCH__
    return __double_as_longlong(x);
#else
    long long b;
    __builtin_memcpy(&b, &x, 8);
    return b;
#endif
}

// x > 0 (false for NaN, as the oracle's positivity fallback test): one DSETP,
// where the integer form on the bit pattern needs a 64-bit compare (2 ISETP)
__host__ __device__ __forceinline__ bool positive(double x) { return x > 0.0; }

__host__ __device__ __forceinline__ double dfrombits(long long b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(b);
#else
    double x;
    __builtin_memcpy(&x, &b, 8);
    return x;
#endif
}

// Same-sign test on the sign bits (a zero counts with its sign; a kept signed
// zero turns W +- d/2 into W exactly, as +0 does).
__host__ __device__ __forceinline__ bool same_sign(double a, double b) {
#ifdef __CUDA_ARCH__
    return (__double2hiint(a) ^ __double2hiint(b)) >= 0;
#else
    return (dbits(a) ^ dbits(b)) >= 0;
#endif
}

// minmod(a, b): 0 unless a and b are both nonzero with the same sign, else the
// one of smaller magnitude (ties: b).  One DSETP on |a|, |b| (no fmin NaN
// fix-ups), a sign-bit test and selects: 7 SASS instructions.  Bitwise equal
// to the oracle's comparison form (reading R2).
__host__ __device__ __forceinline__ double minmod(double a, double b) {
    const double r = fabs(a) < fabs(b) ? a : b;
#ifdef __CUDA_ARCH__
    // sign test as one LOP3 with a predicate output ((hi(a) ^ hi(b)) & 2^31),
    // which nvcc does not form from the C expression (it emits LOP3 + ISETP)
    double out;
    asm("{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\tsetp.eq.u32 q, 1, 1;\n\t"
        "lop3.or.b32 t|p, %1, %2, 0x80000000, 0x28, !q;\n\t"
        "selp.f64 %0, 0d0000000000000000, %3, p;\n\t}"
        : "=d"(out)
        : "r"(__double2hiint(a)), "r"(__double2hiint(b)), "d"(r));
    return out;
#else
    return same_sign(a, b) ? r : 0.0;
#endif
}

// Three-argument minmod (MC limiter, reading R18): 0 unless all three are
// nonzero with the same sign, else the one of smallest magnitude (ties: the
// later argument; the values are then equal).
__host__ __device__ __forceinline__ double minmod3(double a, double b, double c) {
    const double rab = fabs(a) < fabs(b) ? a : b;
    const double r = fabs(rab) < fabs(c) ? rab : c;
    return same_sign(a, b) && same_sign(a, c) ? r : 0.0;
}

// ------------------------------------------------------------------- EOS
// Ideal gas (EOS unit): u = m/rho, p = (gamma-1)(E - m.u/2).
// Returns false for rho <= 0, p <= 0 or non-finite p (calcEos check).
template <int NV>
__host__ __device__ __forceinline__ bool cons_to_prim(const double* u, double* w, double gm1) {
    const double rho = u[0];
    const double inv = rcp(rho);
    double ke = 0.0;
#pragma unroll
    for (int d = 1; d < NV - 1; d++) {
        w[d] = u[d] * inv;
        ke = fma(u[d], w[d], ke);
    }
    w[0] = rho;
    const double p = gm1 * fma(-0.5, ke, u[NV - 1]);
    w[NV - 1] = p;
    // p <= DBL_MAX rather than p < INFINITY: a chain of three DSETP, where the
    // latter is compiled into ~10 integer instructions
    return (rho > 0.0) & (p > 0.0) & (p <= 1.7976931348623157e308);
}

// -------------------------------------------------------- reconstruction
// Cell-centric reconstruction of one variable: from s[0..2R] = W_{i-R..i+R}
// the values at the left (lo, face i-1/2) and right (hi, face i+1/2) edges.
template <int RECON>
__host__ __device__ __forceinline__ void recon_cell(const double* s, double& lo, double& hi) {
    if (RECON == 0) {
        lo = hi = s[0];
    } else if (RECON == 1) {  // PLM-minmod
        const double d = minmod(s[1] - s[0], s[2] - s[1]);
        lo = fma(-0.5, d, s[1]);
        hi = fma(0.5, d, s[1]);
    } else if (RECON == 3) {  // PLM with the monotonized-central limiter (R18)
        const double dl = s[1] - s[0], dr = s[2] - s[1];
        const double d = minmod3(2.0 * dl, 0.5 * (dl + dr), 2.0 * dr);
        lo = fma(-0.5, d, s[1]);
        hi = fma(0.5, d, s[1]);
    } else if (RECON == 4) {  // WENO5-Z (R19), both edges from shared indicators
        // B_k = 4 beta_k as for JS; alpha_k = d_k (1 + tau/(beta_k + eps)) =
        // d_k (D_k + T) / D_k with D_k = B_k + 4 eps, T = |B_0 - B_2|; multiplied
        // through by 10 D_0 D_1 D_2 (one reciprocal per edge).  The left edge
        // mirrors the stencils, i.e. swaps the roles of beta_0 and beta_2.
        const double a = s[0], b = s[1], c = s[2], d = s[3], e = s[4];
        constexpr double eps4 = 4e-40, k13 = 13.0 / 3.0;
        const double t0 = fma(-2.0, b, a) + c, u0 = fma(3.0, c, fma(-4.0, b, a));
        const double t1 = fma(-2.0, c, b) + d, u1 = b - d;
        const double t2 = fma(-2.0, d, c) + e, u2 = fma(3.0, c, fma(-4.0, d, e));
        const double B0 = fma(k13 * t0, t0, u0 * u0);
        const double B1 = fma(k13 * t1, t1, u1 * u1);
        const double B2 = fma(k13 * t2, t2, u2 * u2);
        const double T = fabs(B0 - B2);
        const double D0 = B0 + eps4, D1 = B1 + eps4, D2 = B2 + eps4;
        const double P01 = D0 * D1, P02 = D0 * D2, P12 = D1 * D2;
        const double A1 = 6.0 * ((D1 + T) * P02);
        // right edge (i+1/2): (a,b,c), (b,c,d), (c,d,e) with weights 1 : 6 : 3
        const double A0 = (D0 + T) * P12, A2 = 3.0 * ((D2 + T) * P01);
        const double Q0 = fma(11.0, c, fma(-7.0, b, 2.0 * a));
        const double Q1 = fma(2.0, d, fma(5.0, c, -b));
        const double Q2 = fma(5.0, d, fma(2.0, c, -e));
        hi = fma(A0, Q0, fma(A1, Q1, A2 * Q2)) * rcp(6.0 * (A0 + A1 + A2));
        // left edge (i-1/2): (e,d,c), (d,c,b), (c,b,a): indicators beta_2, beta_1, beta_0
        const double L0 = (D2 + T) * P01, L2 = 3.0 * ((D0 + T) * P12);
        const double R0 = fma(11.0, c, fma(-7.0, d, 2.0 * e));
        const double R1 = fma(2.0, b, fma(5.0, c, -d));
        const double R2 = fma(5.0, b, fma(2.0, c, -a));
        lo = fma(L0, R0, fma(A1, R1, L2 * R2)) * rcp(6.0 * (L0 + A1 + L2));
    } else {  // WENO5-JS, both edges from shared smoothness indicators
        // Same weights as the textbook form, regrouped for fewer FP64 operations:
        //   beta'_k = 4 beta_k = (13/3) t_k^2 + u_k^2,  (eps + beta)^2 = (4 eps + beta')^2 / 16
        //   (the common 1/16 cancels in the normalised weights);
        //   alpha_k ~ d_k / s_k is multiplied through by s0 s1 s2 (one reciprocal
        //   per edge) and by 10 (linear weights 1, 6, 3); the candidates' 1/6 moves
        //   into the denominator.
        const double a = s[0], b = s[1], c = s[2], d = s[3], e = s[4];
        constexpr double eps4 = 4e-6, k13 = 13.0 / 3.0;
        const double t0 = fma(-2.0, b, a) + c, u0 = fma(3.0, c, fma(-4.0, b, a));
        const double t1 = fma(-2.0, c, b) + d, u1 = b - d;
        const double t2 = fma(-2.0, d, c) + e, u2 = fma(3.0, c, fma(-4.0, d, e));
        const double e0 = fma(k13 * t0, t0, fma(u0, u0, eps4));  // eps folded: one op fewer
        const double e1 = fma(k13 * t1, t1, fma(u1, u1, eps4));
        const double e2 = fma(k13 * t2, t2, fma(u2, u2, eps4));
        const double s0 = e0 * e0, s1 = e1 * e1, s2 = e2 * e2;
        const double P0 = s1 * s2, P1 = 6.0 * (s0 * s2), P2 = s0 * s1;
        // right edge (i+1/2): stencils (a,b,c), (b,c,d), (c,d,e), weights 1 : 6 : 3
        const double Q0 = fma(11.0, c, fma(-7.0, b, 2.0 * a));
        const double Q1 = fma(2.0, d, fma(5.0, c, -b));
        const double Q2 = fma(5.0, d, fma(2.0, c, -e));
        const double w2 = 3.0 * P2;
        hi = fma(P0, Q0, fma(P1, Q1, w2 * Q2)) * rcp(6.0 * (P0 + P1 + w2));
        // left edge (i-1/2): the mirrored stencils (e,d,c), (d,c,b), (c,b,a), weights 1 : 6 : 3
        const double R0 = fma(11.0, c, fma(-7.0, d, 2.0 * e));
        const double R1 = fma(2.0, b, fma(5.0, c, -d));
        const double R2 = fma(5.0, b, fma(2.0, c, -a));
        const double v2 = 3.0 * P0;
        lo = fma(P2, R0, fma(P1, R1, v2 * R2)) * rcp(6.0 * (P2 + P1 + v2));
    }
}

// Face-centric first-order / PLM-type states at the face between cells i and
// i+1 from W_{i-1..i+2}: W_L = hi edge of cell i, W_R = lo edge of cell i+1,
// with the same formulas (hence bitwise the same values) as recon_cell.
template <int RECON>
__host__ __device__ __forceinline__ void face_states(double a, double b, double c, double d, double& wl,
                                                     double& wr) {
    if (RECON == 0) {  // first order: the cell values
        wl = b;
        wr = c;
    } else if (RECON != 3) {  // minmod (the kernels call this for RECON 0, 1 and 3 only)
        wl = fma(0.5, minmod(b - a, c - b), b);
        wr = fma(-0.5, minmod(c - b, d - c), c);
    } else {
        const double l0 = b - a, r0 = c - b, r1 = d - c;
        wl = fma(0.5, minmod3(2.0 * l0, 0.5 * (l0 + r0), 2.0 * r0), b);
        wr = fma(-0.5, minmod3(2.0 * r0, 0.5 * (r0 + r1), 2.0 * r1), c);
    }
}

// |u|^2 = (u_x^2 + u_y^2) + u_z^2: symmetric in u_x <-> u_y (bitwise), so a
// face solved with swapped x/y components gives the identical flux.
template <int NV>
__host__ __device__ __forceinline__ double vsq(const double* w) {
    if (NV == 3) return w[1] * w[1];
#ifdef __CUDA_ARCH__
    const double xy = __dadd_rn(__dmul_rn(w[1], w[1]), __dmul_rn(w[2], w[2]));  // never contracted
#else
    const double xy = w[1] * w[1] + w[2] * w[2];
#endif
    return NV == 5 ? fma(w[3], w[3], xy) : xy;
}

// ------------------------------------------------------------- Riemann
// HLL / HLLC (Toro §10.4), Davis wave speeds.  States and flux in the
// unrotated primitive / conserved order; D is the face normal.  HLLC evaluates
// only the state K whose flux is selected.
template <int NV, int RS, int D>
__host__ __device__ __forceinline__ void riemann(const double* wl, const double* wr, double gamma, double gm1i,
                                        double* f) {
    constexpr int N = 1 + D;
    const double rl = wl[0], ul = wl[N], pl = wl[NV - 1];
    const double rr = wr[0], ur = wr[N], pr = wr[NV - 1];
    // c = sqrt(gamma p / rho) = gamma p / sqrt(gamma p rho): no reciprocal of rho needed
    const double gpl = gamma * pl, gpr = gamma * pr;
    const double cl = gpl * rsqrt_fast(gpl * rl), cr = gpr * rsqrt_fast(gpr * rr);
    // Davis estimates; plain compares instead of fmin/fmax (identical for
    // non-NaN operands) avoid the NaN fix-up instructions
    const double al = ul - cl, ar = ur - cr, bl = ul + cl, br = ur + cr;
    const double sl = al < ar ? al : ar;
    const double sr = bl > br ? bl : br;
    if (RS == 1) {
        const double ql = rl * (sl - ul), qr = rr * (sr - ur);  // rho_K (S_K - u_K)
        const double sstar = (pr - pl + ul * ql - ur * qr) * rcp(ql - qr);
        const bool lpos = sl >= 0.0, rneg = sr <= 0.0;
        const bool left = lpos || (!rneg && sstar >= 0.0);
        // every K-side quantity selected at one place
        double w[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) w[v] = left ? wl[v] : wr[v];
        const double sk = left ? sl : sr, qk = left ? ql : qr;
        const double rho = w[0], un = w[N], p = w[NV - 1];
        const double E = fma(0.5 * rho, vsq<NV>(w), p * gm1i);
        // F*_K = F_K + S_K (U*_K - U_K) (Toro §10.4) multiplied out with
        // z = (S* - u_K)/(S_K - S*) and t = S_K z (so rho*_K = rho_K (1 + z)):
        //   mass      rho_K (u_K + t)                       = F0
        //   normal    F0 u_K + t q_K + p_K                  (q_K = rho_K (S_K - u_K))
        //   transv.   F0 w_t
        //   energy    (E_K + p_K)(u_K + t) + t q_K S*
        // Outside the star region t = 0 gives F_K.  Branch-free: t is zeroed by
        // one select after it is formed (a discarded value may be non-finite for
        // a supersonic face), so no reciprocal of rho_K or q_K is needed.
        const bool star = !lpos && !rneg;
        const double z = (sstar - un) * rcp(sk - sstar);
        const double t = star ? sk * z : 0.0;
        const double v = un + t;
        const double m = rho * v;
        f[0] = m;
#pragma unroll
        for (int d = 1; d < NV - 1; d++) f[d] = m * w[d];
        f[N] = fma(m, un, fma(t, qk, p));
        const double ep = E + p;
        f[NV - 1] = fma(ep, v, (t * qk) * sstar);
    } else {
        const double u2l = vsq<NV>(wl), u2r = vsq<NV>(wr);
        const double El = fma(0.5 * rl, u2l, pl * gm1i), Er = fma(0.5 * rr, u2r, pr * gm1i);
        const double ml = rl * ul, mr = rr * ur;
        double UL[NV], UR[NV], FL[NV], FR[NV];
        UL[0] = rl;
        UR[0] = rr;
        FL[0] = ml;
        FR[0] = mr;
#pragma unroll
        for (int d = 1; d < NV - 1; d++) {
            UL[d] = rl * wl[d];
            UR[d] = rr * wr[d];
            FL[d] = ml * wl[d];
            FR[d] = mr * wr[d];
        }
        FL[N] += pl;
        FR[N] += pr;
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
            const double inv = rcp(sr - sl), slsr = sl * sr;
#pragma unroll
            for (int v = 0; v < NV; v++) f[v] = fma(slsr, UR[v] - UL[v], sr * FL[v] - sl * FR[v]) * inv;
        }
    }
}

// ------------------------------------------------------------- shockDet
// shockDet (Alg. 7; reading R21): cell i is a shock cell along the
// face normal when the flow converges across it by more than 1e-6 of the sound
// speed, d = u(i+1) - u(i-1) < 0 with d^2 rho(i-1) rho(i+1) > 1e-12 gamma
// max(p(i-1) rho(i+1), p(i+1) rho(i-1)) (no division; the dead band keeps the
// exact ties and last-bit noise of symmetric states unflagged), and the
// pressure jump across it exceeds thr * min(p(i-1), p(i+1)).  Evaluated on the
// cell-centre primitives the face's reconstruction already reads.  Products
// are rounded separately (never contracted), as in the oracle.
__host__ __device__ __forceinline__ double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
__host__ __device__ __forceinline__ bool shock_cell(double um, double up, double pm, double pp, double rm, double rp,
                                                    double thr, double gamma) {
    const double d = up - um;
    const double a = dmul(pm, rp), b = dmul(pp, rm);
    const double pmin = pm < pp ? pm : pp;
    return (d < 0.0) & (dmul(dmul(d, d), dmul(rm, rp)) > dmul(dmul(1e-12, gamma), a > b ? a : b)) &
           (fabs(pp - pm) > dmul(thr, pmin));
}
// face between cells i and i+1 from (u, p, rho) of the cells i-1, i, i+1, i+2
__host__ __device__ __forceinline__ bool shock_face(const double* u, const double* p, const double* r, double thr,
                                                    double gamma) {
    return shock_cell(u[0], u[2], p[0], p[2], r[0], r[2], thr, gamma) |
           shock_cell(u[1], u[3], p[1], p[3], r[1], r[3], thr, gamma);
}

// calcFlux of one face: RS 0 HLL, 1 HLLC, 2 hybrid (HLL at shock faces,
// HLLC elsewhere; the flag is only read for RS 2)
template <int NV, int RS, int D>
__host__ __device__ __forceinline__ void face_flux(const double* wl, const double* wr, bool shock, double gamma,
                                                   double gm1i, double* f) {
    if constexpr (RS == 2) {
        if (shock) riemann<NV, 0, D>(wl, wr, gamma, gm1i, f);
        else riemann<NV, 1, D>(wl, wr, gamma, gm1i, f);
    } else {
        riemann<NV, RS, D>(wl, wr, gamma, gm1i, f);
    }
}

// grvAccel source (reading R20) of variable v at a cell with conserved value u
// of that variable, called in variable order: rho and m.g accumulate in
// (rho, mg).  S = (0, rho g, m.g).
template <int NV>
__host__ __device__ __forceinline__ double grav_src(const Geo& g, int v, double u, double& rho, double& mg) {
    if (v == 0) {
        rho = u;
        return 0.0;
    }
    if (v < NV - 1) {
        mg = fma(u, g.grav[v - 1], mg);
        return rho * g.grav[v - 1];
    }
    return mg;
}

// Element index of variable 0 of the cell with canonical index q = b*cpb + c
// (block b, cell c of the block) in the block-interleaved state U[b][v][c].
__host__ __device__ __forceinline__ long long state_index(const Geo& g, long long q) {
    const long long b = q / g.cpb;
    return b * g.bs + (q - b * g.cpb);
}

// ------------------------------------------------------------ guard gather
// Conserved values of the cell at sub-box coordinates l (may lie up to ng
// cells outside the sub-box).  Out-of-box coordinates are resolved per
// dimension: a face with a peer rank reads the received slab, otherwise the
// physical boundary map (periodic wrap / outflow clamp / reflect mirror with
// the normal momentum negated).  Returns false (out unset) when the cell lies
// outside the sub-box in two or more peer directions (an edge or corner owned
// by a diagonal rank; never needed by the star stencil).
struct Src {
    const double* p;  // variable 0 of the source cell
    long long vs;     // stride between variables
    int flip;         // bit 1+d: negate momentum d (reflecting boundary)
};

__device__ __forceinline__ bool fetch_src(const Geo& g, const double* __restrict__ u,
                                          const double* const (&halo)[3][2], int l0, int l1, int l2, Src& src) {
    int l[3] = {l0, l1, l2};
    int flip = 0;
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
                    flip |= 2 << d;
                }
                l[d] = gx - g.off[d];
            }
        }
    }
    long long idx;
    if (hd >= 0) {
        int c[3] = {l[0], l[1], l[2]};
        c[hd] = hs ? l[hd] - g.cn[hd] : l[hd] + g.ng;
        const int e0 = hd == 0 ? g.ng : g.cn[0];
        const int e1 = hd == 1 ? g.ng : g.cn[1];
        idx = ((long long)c[2] * e1 + c[1]) * e0 + c[0];
#ifdef SPARK_CHECKED  // the cell lies in the received slab (SPARK_CHECKED: spark_stage.cu)
        if (idx < 0 || idx >= g.slab[hd] || !halo[hd][hs]) __trap();
#endif
        src.p = halo[hd][hs] + idx;
        src.vs = g.slab[hd];
    } else {
        const int bx = l[0] / g.nb[0], by = l[1] / g.nb[1], bz = l[2] / g.nb[2];
        const long long blk = bx + (long long)g.bn[0] * (by + (long long)g.bn[1] * bz);
        idx = blk * g.bs + ((long long)(l[2] - bz * g.nb[2]) * g.nb[1] + (l[1] - by * g.nb[1])) * g.nb[0] +
              (l[0] - bx * g.nb[0]);
#ifdef SPARK_CHECKED  // the mapped cell lies in the sub-box
        for (int d = 0; d < 3; d++)
            if (l[d] < 0 || l[d] >= g.cn[d]) __trap();
#endif
        src.p = u + idx;
        src.vs = g.vs;
    }
    src.flip = flip;
    return true;
}

// conserved values at a source, reflect flips applied (sign-bit xor)
template <int NV>
__device__ __forceinline__ void load_src(const double* p, long long vs, int flip, double* out) {
#pragma unroll
    for (int v = 0; v < NV; v++) out[v] = __ldg(p + v * vs);
#pragma unroll
    for (int d = 0; d < NV - 2; d++)
        out[1 + d] = __hiloint2double(__double2hiint(out[1 + d]) ^ (((flip >> (1 + d)) & 1) << 31),
                                      __double2loint(out[1 + d]));
}

template <int NV>
__device__ __forceinline__ bool fetch_cons(const Geo& g, const double* __restrict__ u,
                                           const double* const (&halo)[3][2], int l0, int l1, int l2,
                                           double* out) {
    Src s;
    if (!fetch_src(g, u, halo, l0, l1, l2, s)) return false;
    load_src<NV>(s.p, s.vs, s.flip, out);
    return true;
}

// Record a non-physical state seen by this thread block in the step in
// flight: the local status bit and the first failing step (global after the
// per-step min-reduction of `bad`).
__device__ __forceinline__ void flag_nonphysical(DevScalars* sc) {
    atomicOr(&sc->status, 1);
    atomicMin(&sc->bad, (unsigned long long)sc->steps);
}

// ------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_min(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// CFL term of one primitive state: min_d dx_d / (|u_d| + c)  (reading R7),
// evaluated as 1 / max_d (|u_d| + c) / dx_d (one reciprocal instead of ndim)
// with c = gamma p / sqrt(gamma p rho) (no reciprocal of rho); every GPU path
// uses this function, so the CFL minimum stays bitwise rank-invariant.
template <int NV>
__device__ __forceinline__ double cfl_term(const Geo& g, const double* w) {
    const double gp = g.gamma * w[NV - 1];
    const double c = gp * rsqrt_fast(gp * w[0]);
    double m = (fabs(w[1]) + c) * g.rdx[0];
#pragma unroll
    for (int d = 1; d < NV - 2; d++) {
        const double x = (fabs(w[1 + d]) + c) * g.rdx[d];
        m = x > m ? x : m;
    }
    return rcp(m);
}

// Block-wide min of x -> atomicMin on the u64 bits (positive doubles order
// like unsigned integers; +inf is the identity).  All threads must call;
// blockDim.x is a multiple of 32.
__device__ __forceinline__ void block_min_to(double x, double* red, unsigned long long* acc) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    x = warp_min(x);
    if (lane == 0) red[wid] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = red[0];
        for (int w = 1; w < nw; w++) m = fmin(m, red[w]);
        if (m < INFINITY) atomicMin(acc, (unsigned long long)__double_as_longlong(m));
    }
}

}  // namespace dev
}  // namespace spark
