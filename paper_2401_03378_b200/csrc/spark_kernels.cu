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
// Data layout (HBM): block-interleaved pool U[b][v][k][j][i] (Geo.vs/.bs); the guard
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

#include "spark_device.cuh"
#include "spark_internal.h"

namespace spark {
namespace {

using namespace dev;

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
        const long long e = state_index(g, q);
#pragma unroll
        for (int v = 0; v < NV; v++) c[v] = u[e + v * g.vs];
        ok &= cons_to_prim<NV>(c, w, g.gamma - 1.0);
        m = fmin(m, cfl_term<NV>(g, w));
    }
    if (!ok) flag_nonphysical(sc);
    block_min_to(m, red, &sc->acc);
}

__global__ void step_begin_kernel(DevScalars* sc, double dt_fixed, double t_end, double cfl) {
    const double t = sc->t;
    // stop at t_end, and freeze after a non-physical state on any rank (the
    // failure is reported, not rolled back, by the next synchronising call)
    if ((dt_fixed <= 0.0 && t_end > 0.0 && t >= t_end * (1.0 - 1e-14)) || sc->bad != kNoBad) {
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

// element-wise min of the (acc, bad) pairs of the members of a local group
__global__ void group_min_kernel(const AccPtrs p, int n) {
    const int e = threadIdx.x;  // 0: acc, 1: bad
    unsigned long long m = ~0ull;
    for (int r = 0; r < n; r++) m = p.p[r][e] < m ? p.p[r][e] : m;
    for (int r = 0; r < n; r++) p.p[r][e] = m;
}

__global__ void set_time_kernel(DevScalars* sc, double t, long long steps) {
    sc->t = t;
    sc->t_prev = t;
    sc->steps = steps;
}

__global__ void scalars_reset_kernel(DevScalars* sc) {
    sc->dt = 0.0;
    sc->t = 0.0;
    sc->t_prev = 0.0;
    sc->acc = 0x7ff0000000000000ull;
    sc->acc_prev = 0x7ff0000000000000ull;
    sc->bad = kNoBad;
    sc->status = 0;
    sc->active = 1;
    sc->steps = 0;
}

template <int NDIM>
__global__ void prim_to_cons_kernel(const Geo g, const double* __restrict__ w, double* __restrict__ u) {
    constexpr int NV = NDIM + 2;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.ncell;
         q += (long long)gridDim.x * blockDim.x) {
        const long long e = state_index(g, q);  // W canonical [v][q], U internal
        const double rho = w[q];
        double u2 = 0.0;
#pragma unroll
        for (int d = 1; d < NV - 1; d++) {
            const double vel = w[d * g.ncell + q];
            u2 += vel * vel;
            u[e + d * g.vs] = rho * vel;
        }
        u[e] = rho;
        u[e + (NV - 1) * g.vs] = w[(NV - 1) * g.ncell + q] / (g.gamma - 1.0) + 0.5 * rho * u2;
    }
}

// canonical U[v][q] (q = b*cpb + c) <-> internal U[b][v][c]: one CTA per
// (variable, block) chunk of cpb contiguous elements on both sides (16-byte
// accesses when cpb is even); no index division per element
__global__ void relayout_kernel(const Geo g, const double* __restrict__ src, double* __restrict__ dst,
                                int to_internal, long long b0, long long b1) {
    // blocks [b0, b1) of every variable (the whole state: 0, nblocks)
    const long long nblk = b1 - b0, nchunk = nblk * g.nvar;
    const bool vec = (g.cpb & 1) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    for (long long ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
        const long long v = ch / nblk, b = b0 + ch - v * nblk;
        const long long canon = v * g.ncell + b * g.cpb, inter = b * g.bs + v * g.vs;
        const double* s = src + (to_internal ? canon : inter);
        double* d = dst + (to_internal ? inter : canon);
        if (vec) {
            const double2* s2 = reinterpret_cast<const double2*>(s);
            double2* d2 = reinterpret_cast<double2*>(d);
            for (long long c = threadIdx.x; c < g.cpb / 2; c += blockDim.x) d2[c] = __ldcs(s2 + c);
        } else {
            for (long long c = threadIdx.x; c < g.cpb; c += blockDim.x) d[c] = __ldcs(s + c);
        }
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

unsigned grid_for(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    if (b > 148LL * 32) b = 148LL * 32;
    if (b < 1) b = 1;
    return (unsigned)b;
}

}  // namespace

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
    group_min_kernel<<<1, 2, 0, s>>>(p, n);
    return cudaGetLastError();
}

cudaError_t launch_set_time(DevScalars* sc, double t, long long steps, cudaStream_t s) {
    set_time_kernel<<<1, 1, 0, s>>>(sc, t, steps);
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

cudaError_t launch_relayout(const Geo& g, const double* src, double* dst, int to_internal, cudaStream_t s) {
    return launch_relayout_range(g, src, dst, to_internal, 0, g.ncell / g.cpb, s);
}

cudaError_t launch_relayout_range(const Geo& g, const double* src, double* dst, int to_internal, long long b0,
                                  long long b1, cudaStream_t s) {
    const long long nchunk = (b1 - b0) * g.nvar;
    if (nchunk <= 0) return cudaSuccess;
    relayout_kernel<<<(unsigned)(nchunk < 148LL * 64 ? nchunk : 148LL * 64), 256, 0, s>>>(g, src, dst, to_internal,
                                                                                       b0, b1);
    return cudaGetLastError();
}

__global__ void acc_reset_kernel(DevScalars* sc) { sc->acc = 0x7ff0000000000000ull; }

cudaError_t launch_acc_reset(DevScalars* sc, cudaStream_t s) {
    acc_reset_kernel<<<1, 1, 0, s>>>(sc);
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

// ------------------------------------------------------------- self test
namespace spark {
namespace {
template <int NV, int RS, int D>
__global__ void selftest_riemann_kernel(int64_t n, double gamma, const double* __restrict__ wl,
                                        const double* __restrict__ wr, double* __restrict__ f) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double a[NV], b[NV], o[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) {
        a[v] = wl[i * NV + v];
        b[v] = wr[i * NV + v];
    }
    dev::riemann<NV, RS, D>(a, b, gamma, 1.0 / (gamma - 1.0), o);
#pragma unroll
    for (int v = 0; v < NV; v++) f[i * NV + v] = o[v];
}

template <int NV, int RS>
cudaError_t st_d(int dir, int64_t n, double g, const double* wl, const double* wr, double* f) {
    const unsigned grid = (unsigned)((n + 127) / 128);
    if (dir == 0) selftest_riemann_kernel<NV, RS, 0><<<grid, 128>>>(n, g, wl, wr, f);
    else if (dir == 1 && NV >= 4) selftest_riemann_kernel<NV, RS, (NV >= 4 ? 1 : 0)><<<grid, 128>>>(n, g, wl, wr, f);
    else if (NV >= 5) selftest_riemann_kernel<NV, RS, (NV >= 5 ? 2 : 0)><<<grid, 128>>>(n, g, wl, wr, f);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_selftest_riemann(int riemann, int ndim, int dir, double gamma, int64_t n, const double* wl,
                                    const double* wr, double* f) {
    if (ndim == 1) return riemann ? st_d<3, 1>(dir, n, gamma, wl, wr, f) : st_d<3, 0>(dir, n, gamma, wl, wr, f);
    if (ndim == 2) return riemann ? st_d<4, 1>(dir, n, gamma, wl, wr, f) : st_d<4, 0>(dir, n, gamma, wl, wr, f);
    return riemann ? st_d<5, 1>(dir, n, gamma, wl, wr, f) : st_d<5, 0>(dir, n, gamma, wl, wr, f);
}
}  // namespace spark

// ---------------------------------------------------------- AXPY (NEXT N4)
// The paper's AXPY thread mappings (alg:axpy-incr-1 P:1041-1060,
// alg:axpy-incr-threads P:1061-1079, alg:axpy-single-iter P:1086-1100) as an
// in-run HBM calibration: y_i = a x_i + y_i in FP64, never FMA-contracted
// (bitwise equal to a separate multiply and add).  Variant 3 is the B200 form:
// 16-byte vector accesses, grid = a multiple of the SM count.
namespace spark {
namespace {
__device__ __forceinline__ double axpy1(double a, double x, double y) { return __dadd_rn(__dmul_rn(a, x), y); }

__global__ void axpy_incr_1(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, T = (int64_t)gridDim.x * blockDim.x;
    const int64_t lo = (n * t) / T, hi = (n * (t + 1)) / T;  // floor(N t / T), floor(N (t+1) / T)
    for (int64_t i = lo; i < hi; i++) y[i] = axpy1(a, x[i], y[i]);
}

__global__ void axpy_incr_threads(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, T = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t; i < n; i += T) y[i] = axpy1(a, x[i], y[i]);
}

__global__ void axpy_single_iter(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) y[i] = axpy1(a, x[i], y[i]);
}

__global__ void axpy_vec2(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, T = (int64_t)gridDim.x * blockDim.x;
    const int64_t n2 = n / 2;
    const double2* __restrict__ x2 = reinterpret_cast<const double2*>(x);
    double2* __restrict__ y2 = reinterpret_cast<double2*>(y);
    for (int64_t i = t; i < n2; i += T) {
        const double2 xv = __ldcs(x2 + i);
        double2 yv = __ldcs(y2 + i);
        yv.x = axpy1(a, xv.x, yv.x);
        yv.y = axpy1(a, xv.y, yv.y);
        __stcs(y2 + i, yv);
    }
    if (t == 0 && (n & 1)) y[n - 1] = axpy1(a, x[n - 1], y[n - 1]);
}
}  // namespace

cudaError_t launch_axpy(int variant, int64_t n, double a, const double* x, double* y, int sms, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int threads = 256;
    const unsigned persistent = (unsigned)(sms * 8);  // 8 x 256-thread CTAs per SM
    switch (variant) {
        case 0: axpy_incr_1<<<persistent, threads, 0, s>>>(n, a, x, y); break;
        case 1: axpy_incr_threads<<<persistent, threads, 0, s>>>(n, a, x, y); break;
        case 2: axpy_single_iter<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(n, a, x, y); break;
        default:
            if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) return cudaErrorInvalidValue;
            axpy_vec2<<<persistent, threads, 0, s>>>(n, a, x, y);
    }
    return cudaGetLastError();
}
}  // namespace spark
