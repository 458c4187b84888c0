// spark_telescope_tile.cu — telescoping SSP-RK through HBM tiles: 3-D blocks
// and multi-rank (NEXT N1).
//
// Telescoping mode (lst:spark-telescoping P:1593-1605):
// ONE guard fill per step with G = S*NGK layers (faces, edges and corners),
// then all S stages per block on its (nb + 2G)^ndim tile, stage s updating
// the tile cells at distance >= s*NGK from the tile edge (the halo area too).
// The on-chip kernel (spark_telescope.cu) covers 1-D/2-D on one rank; a 3-D
// tile (24^3 x 5 doubles for PLM/RK2) does not fit in shared memory, so this
// path keeps the tiles in HBM:
//   TA tt_pack / exchange / tt_gather  the thick shell of the rank's sub-box
//        is packed into 26 direction buffers (faces, edges, corners), sent
//        to the neighbouring ranks ONCE per step (NCCL grouped send/recv, or
//        device copies between virtual ranks), and every block's tile of U^n
//        is gathered from the own pool, the received shell, or the physical
//        boundary map (guards beyond a physical boundary are filled once and
//        evolved, reading R17)
//   TB tt_prim / tt_face / tt_update  per stage on the shrinking region; the
//        last stage writes the block interior to U^(n+1) with the CFL-min
//        epilogue
// The result of a block depends only on the global U^n and the boundary maps,
// so it is bitwise independent of the rank count.  Per-face arithmetic is the
// product's device code (spark_device.cuh).
#include <cmath>
#include <cstdint>

#include "spark_device.cuh"
#include "spark_internal.h"

namespace spark {
namespace {

using namespace dev;

__device__ __forceinline__ int dir_index(int c0, int c1, int c2) { return (c0 + 1) + 3 * (c1 + 1) + 9 * (c2 + 1); }

// cells of the shell region of direction (c0, c1, c2): G along a nonzero
// component, the sub-box extent along a zero one
__host__ __device__ inline long long region_cells(const TileGeo& t, int dir, int* ext) {
    const int c[3] = {dir % 3 - 1, (dir / 3) % 3 - 1, dir / 9 - 1};
    long long n = 1;
    for (int d = 0; d < 3; d++) {
        ext[d] = c[d] ? t.G : t.g.cn[d];
        n *= ext[d];
    }
    return n;
}

// conserved values of sub-box cell (x, y, z) from the block-interleaved pool
template <int NV>
__device__ __forceinline__ void pool_cell(const Geo& g, const double* __restrict__ u, int x, int y, int z, double* out) {
    const int bx = x / g.nb[0], by = y / g.nb[1], bz = z / g.nb[2];
    const long long b = bx + (long long)g.bn[0] * (by + (long long)g.bn[1] * bz);
    const long long c = ((long long)(z - bz * g.nb[2]) * g.nb[1] + (y - by * g.nb[1])) * g.nb[0] + (x - bx * g.nb[0]);
#pragma unroll
    for (int v = 0; v < NV; v++) out[v] = u[b * g.bs + v * g.vs + c];
}

template <int NV>
__global__ void tt_pack_kernel(const TileGeo t, const double* __restrict__ u, int dir, double* __restrict__ buf) {
    int ext[3];
    const long long n = region_cells(t, dir, ext);
    const int c[3] = {dir % 3 - 1, (dir / 3) % 3 - 1, dir / 9 - 1};
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
        int l[3] = {(int)(q % ext[0]), (int)((q / ext[0]) % ext[1]), (int)(q / ((long long)ext[0] * ext[1]))};
        for (int d = 0; d < 3; d++)
            if (c[d] > 0) l[d] += t.g.cn[d] - t.G;  // the sub-box's own cells on side +d
        double val[NV];
        pool_cell<NV>(t.g, u, l[0], l[1], l[2], val);
#pragma unroll
        for (int v = 0; v < NV; v++) buf[v * n + q] = val[v];
    }
}

// the tile of U^n of every block: own pool, received shell or boundary map
template <int NV>
__global__ void tt_gather_kernel(const TileGeo t, const double* __restrict__ u, const ShellPtrs sh,
                                 double* __restrict__ T0) {
    const Geo& g = t.g;
    const long long nblk = (long long)g.bn[0] * g.bn[1] * g.bn[2];
    const long long total = nblk * t.np, tvs = total;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const long long b = q / t.np, r = q - b * t.np;
        const int tc[3] = {(int)(r % t.pn[0]), (int)((r / t.pn[0]) % t.pn[1]), (int)(r / ((long long)t.pn[0] * t.pn[1]))};
        const int bc3[3] = {(int)(b % g.bn[0]), (int)((b / g.bn[0]) % g.bn[1]), (int)(b / ((long long)g.bn[0] * g.bn[1]))};
        int comp[3] = {0, 0, 0}, l[3] = {0, 0, 0}, flip = 0;
        for (int d = 0; d < 3; d++) {
            if (d >= g.ndim) continue;
            int x = bc3[d] * g.nb[d] + tc[d] - t.G;
            if (x >= 0 && x < g.cn[d]) {
                l[d] = x;
            } else if ((x < 0 && g.halo[d][0]) || (x >= g.cn[d] && g.halo[d][1])) {
                comp[d] = x < 0 ? -1 : 1;
                l[d] = x < 0 ? x + t.G : x - g.cn[d];
            } else {  // physical boundary (or a periodic dim owned by this rank alone)
                const int N = g.gN[d];
                int gx = g.off[d] + x;
                const int bc = g.bc[d][x < 0 ? 0 : 1];
                if (bc == 0) {
                    gx %= N;
                    if (gx < 0) gx += N;
                } else if (bc == 1) {
                    gx = x < 0 ? 0 : N - 1;
                } else {
                    gx = x < 0 ? -1 - gx : 2 * N - 1 - gx;
                    flip |= 2 << d;
                }
                l[d] = gx - g.off[d];
            }
        }
        double val[NV];
        if (!comp[0] && !comp[1] && !comp[2]) {
            pool_cell<NV>(g, u, l[0], l[1], l[2], val);
        } else {
            const int dir = dir_index(comp[0], comp[1], comp[2]);
            int ext[3];
            const long long n = region_cells(t, dir, ext);
            const long long idx = ((long long)l[2] * ext[1] + l[1]) * ext[0] + l[0];
#pragma unroll
            for (int v = 0; v < NV; v++) val[v] = sh.p[dir][v * n + idx];
        }
#pragma unroll
        for (int d = 0; d < NV - 2; d++)
            if ((flip >> (1 + d)) & 1) val[1 + d] = -val[1 + d];
#pragma unroll
        for (int v = 0; v < NV; v++) T0[v * tvs + q] = val[v];
    }
}

__device__ __forceinline__ bool in_region(const TileGeo& t, const int* tc, int dist) {
    for (int d = 0; d < t.g.ndim; d++)
        if (tc[d] < dist || tc[d] >= t.pn[d] - dist) return false;
    return true;
}

// primitives of U^(s-1) on its valid region (distance >= (s-1) NGK)
template <int NV>
__global__ void tt_prim_kernel(const TileGeo t, const double* __restrict__ Tin, double* __restrict__ W, int s,
                               DevScalars* sc) {
    const long long nblk = (long long)t.g.bn[0] * t.g.bn[1] * t.g.bn[2];
    const long long total = nblk * t.np;
    const int dist = (s - 1) * t.ngk;
    bool ok = true;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const long long r = q % t.np;
        const int tc[3] = {(int)(r % t.pn[0]), (int)((r / t.pn[0]) % t.pn[1]), (int)(r / ((long long)t.pn[0] * t.pn[1]))};
        if (!in_region(t, tc, dist)) continue;
        double u[NV], w[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) u[v] = Tin[v * total + q];
        ok &= cons_to_prim<NV>(u, w, t.g.gamma - 1.0);
#pragma unroll
        for (int v = 0; v < NV; v++) W[v * total + q] = w[v];
    }
    if (!ok) flag_nonphysical(sc);
}

template <int RECON>
__device__ __forceinline__ void recon_face_t(const double* s, double& wl, double& wr) {
    constexpr int R = StencilOf<RECON>::NG - 1;
    constexpr int K = StencilOf<RECON>::NG;
    double lo, hi;
    recon_cell<RECON>(s + (K - 1 - R), lo, hi);
    wl = hi;
    recon_cell<RECON>(s + (K - R), lo, hi);
    wr = lo;
}

template <int NV, int RS, int D, int RECON>
__device__ __forceinline__ void tt_solve(const TileGeo& t, const double* __restrict__ W, long long vstride,
                                         long long right, long long stride, double* f) {
    constexpr int K = StencilOf<RECON>::NG;
    double wl[NV], wr[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) {
        double s[6];
#pragma unroll
        for (int m = 0; m < 2 * K; m++) s[m] = W[v * vstride + right + (m - K) * stride];
        recon_face_t<RECON>(s, wl[v], wr[v]);
    }
    if (RECON != 0 && !(positive(wl[0]) && positive(wl[NV - 1]) && positive(wr[0]) && positive(wr[NV - 1]))) {
#pragma unroll
        for (int v = 0; v < NV; v++) {
            wl[v] = W[v * vstride + right - stride];
            wr[v] = W[v * vstride + right];
        }
    }
    bool shk = false;
    if constexpr (RS == 2) {
        double uu[4], pp[4], rr[4];
#pragma unroll
        for (int m = 0; m < 4; m++) {
            const long long q = right + (m - 2) * stride;
            uu[m] = W[(1 + D) * vstride + q];
            pp[m] = W[(NV - 1) * vstride + q];
            rr[m] = W[q];
        }
        shk = shock_face(uu, pp, rr, t.g.shock_thresh, t.g.gamma);
    }
    face_flux<NV, RS, D>(wl, wr, shk, t.g.gamma, 1.0 / (t.g.gamma - 1.0), f);
}

// fluxes of the faces region s needs: along d the faces lo..hi of the region,
// across it the region's extent.  F[v][blk][d-block of (pn_d + 1) prod pn_e]
template <int NDIM, int RS>
__global__ void tt_face_kernel(const TileGeo t, const double* __restrict__ W, double* __restrict__ F, int s) {
    constexpr int NV = NDIM + 2;
    const long long nblk = (long long)t.g.bn[0] * t.g.bn[1] * t.g.bn[2];
    const long long total = nblk * t.NF, vstride = nblk * t.np;
    const int lo = s * t.ngk;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long b = e / t.NF;
        long long r = e - b * t.NF;
        const int d = r < t.Fo[1] ? 0 : (r < t.Fo[2] ? 1 : 2);
        r -= t.Fo[d];
        int fn[3] = {t.pn[0], t.pn[1], t.pn[2]};
        fn[d] += 1;
        const int fc[3] = {(int)(r % fn[0]), (int)((r / fn[0]) % fn[1]), (int)(r / ((long long)fn[0] * fn[1]))};
        bool need = true;
        for (int e2 = 0; e2 < NDIM; e2++) {
            const int hi = t.pn[e2] - lo + (e2 == d ? 1 : 0);
            if (fc[e2] < lo || fc[e2] >= hi) need = false;
        }
        if (!need) continue;
        const long long right = b * t.np + ((long long)fc[2] * t.pn[1] + fc[1]) * t.pn[0] + fc[0];
        const long long stride = d == 0 ? 1 : (d == 1 ? t.pn[0] : (long long)t.pn[0] * t.pn[1]);
        double f[NV];
#define TT_SOLVE(DD)                                                                                     \
    switch (t.recon) {                                                                                   \
        case 0: tt_solve<NV, RS == 2 ? 1 : RS, DD, 0>(t, W, vstride, right, stride, f); break;          \
        case 1: tt_solve<NV, RS, DD, 1>(t, W, vstride, right, stride, f); break;                        \
        case 3: tt_solve<NV, RS, DD, 3>(t, W, vstride, right, stride, f); break;                        \
        case 4: tt_solve<NV, RS, DD, 4>(t, W, vstride, right, stride, f); break;                        \
        default: tt_solve<NV, RS, DD, 2>(t, W, vstride, right, stride, f); break;                       \
    }
        if (d == 0) {
            TT_SOLVE(0)
        } else if (NDIM >= 2 && d == 1) {
            TT_SOLVE((NDIM >= 2 ? 1 : 0))
        } else if (NDIM >= 3) {
            TT_SOLVE((NDIM >= 3 ? 2 : 0))
        }
#undef TT_SOLVE
#pragma unroll
        for (int v = 0; v < NV; v++) F[v * total + e] = f[v];
    }
}

// U^(s) = a U^n + b (U^(s-1) + dt L) on region s; the last stage writes the
// block interior to the pool and reduces the CFL minimum
template <int NDIM>
__global__ void tt_update_kernel(const TileGeo t, const double* __restrict__ F, const double* __restrict__ Tprev,
                                 const double* __restrict__ T0, double* __restrict__ Tout, double* __restrict__ uout,
                                 double a, double b, int s, int last, DevScalars* sc) {
    constexpr int NV = NDIM + 2;
    __shared__ double red[32];
    const Geo& g = t.g;
    const long long nblk = (long long)g.bn[0] * g.bn[1] * g.bn[2];
    const long long total = nblk * t.np, ftot = nblk * t.NF;
    const int lo = s * t.ngk;
    const double dt = sc->dt;
    const bool active = sc->active;
    double cflmin = INFINITY;
    bool ok = true;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x) {
        const long long blk = q / t.np, r = q - blk * t.np;
        const int tc[3] = {(int)(r % t.pn[0]), (int)((r / t.pn[0]) % t.pn[1]), (int)(r / ((long long)t.pn[0] * t.pn[1]))};
        if (!in_region(t, tc, lo)) continue;
        double un[NV];
        if (!active) {  // t >= t_end or frozen after a failure: U unchanged
#pragma unroll
            for (int v = 0; v < NV; v++) un[v] = T0[v * total + q];
        } else {
            long long flo[3], fhi[3];
#pragma unroll
            for (int d = 0; d < NDIM; d++) {
                int fn[3] = {t.pn[0], t.pn[1], t.pn[2]};
                fn[d] += 1;
                int up[3] = {tc[0], tc[1], tc[2]};
                up[d] += 1;
                flo[d] = blk * t.NF + t.Fo[d] + ((long long)tc[2] * fn[1] + tc[1]) * fn[0] + tc[0];
                fhi[d] = blk * t.NF + t.Fo[d] + ((long long)up[2] * fn[1] + up[1]) * fn[0] + up[0];
            }
#pragma unroll
            for (int v = 0; v < NV; v++) {
                const double dfx = (F[v * ftot + fhi[0]] - F[v * ftot + flo[0]]) * g.rdx[0];
                double Lv;
                if (NDIM == 1) {
                    Lv = -dfx;
                } else {
                    const double dfy = (F[v * ftot + fhi[1]] - F[v * ftot + flo[1]]) * g.rdx[1];
                    if (NDIM == 2) Lv = -(dfx + dfy);
                    else Lv = -(dfx + dfy) - (F[v * ftot + fhi[2]] - F[v * ftot + flo[2]]) * g.rdx[2];
                }
                const double u0 = Tprev[v * total + q];
                const double unn = a != 0.0 ? T0[v * total + q] : 0.0;
                un[v] = fma(b, fma(dt, Lv, u0), a * unn);
            }
        }
        if (!last) {
#pragma unroll
            for (int v = 0; v < NV; v++) Tout[v * total + q] = un[v];
            continue;
        }
        // interior cell of block blk -> the pool (block-interleaved)
        const long long c = ((long long)(tc[2] - (NDIM >= 3 ? t.G : 0)) * g.nb[1] + (tc[1] - (NDIM >= 2 ? t.G : 0))) *
                                g.nb[0] + (tc[0] - t.G);
#pragma unroll
        for (int v = 0; v < NV; v++) uout[blk * g.bs + v * g.vs + c] = un[v];
        double w[NV];
        ok &= cons_to_prim<NV>(un, w, g.gamma - 1.0);
        cflmin = fmin(cflmin, cfl_term<NV>(g, w));
    }
    if (!ok) flag_nonphysical(sc);
    if (last) block_min_to(cflmin, red, &sc->acc);
}

unsigned tgrid(long long n) {
    long long b = (n + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 148LL * 16 ? 148LL * 16 : b));
}

}  // namespace

long long tile_region_cells(const TileGeo& t, int dir) {
    int ext[3];
    return region_cells(t, dir, ext);
}

cudaError_t launch_tile_pack(const TileGeo& t, const double* u, int dir, double* buf, cudaStream_t s) {
    const unsigned gr = tgrid(tile_region_cells(t, dir));
    if (t.g.nvar == 3) tt_pack_kernel<3><<<gr, 256, 0, s>>>(t, u, dir, buf);
    else if (t.g.nvar == 4) tt_pack_kernel<4><<<gr, 256, 0, s>>>(t, u, dir, buf);
    else tt_pack_kernel<5><<<gr, 256, 0, s>>>(t, u, dir, buf);
    return cudaGetLastError();
}

cudaError_t launch_tile_gather(const TileGeo& t, const double* u, const ShellPtrs& sh, double* T0, cudaStream_t s) {
    const long long nblk = (long long)t.g.bn[0] * t.g.bn[1] * t.g.bn[2];
    const unsigned gr = tgrid(nblk * t.np);
    if (t.g.nvar == 3) tt_gather_kernel<3><<<gr, 256, 0, s>>>(t, u, sh, T0);
    else if (t.g.nvar == 4) tt_gather_kernel<4><<<gr, 256, 0, s>>>(t, u, sh, T0);
    else tt_gather_kernel<5><<<gr, 256, 0, s>>>(t, u, sh, T0);
    return cudaGetLastError();
}

template <int NDIM>
cudaError_t tile_stage_d(const TileGeo& t, int riemann, const double* Tprev, const double* T0, double* W, double* F,
                         double* Tout, double* uout, double a, double b, int s, int last, DevScalars* sc,
                         cudaStream_t st) {
    constexpr int NV = NDIM + 2;
    const long long nblk = (long long)t.g.bn[0] * t.g.bn[1] * t.g.bn[2];
    tt_prim_kernel<NV><<<tgrid(nblk * t.np), 256, 0, st>>>(t, Tprev, W, s, sc);
    const unsigned gf = tgrid(nblk * t.NF);
    if (riemann == 0) tt_face_kernel<NDIM, 0><<<gf, 256, 0, st>>>(t, W, F, s);
    else if (riemann == 1) tt_face_kernel<NDIM, 1><<<gf, 256, 0, st>>>(t, W, F, s);
    else tt_face_kernel<NDIM, 2><<<gf, 256, 0, st>>>(t, W, F, s);
    tt_update_kernel<NDIM><<<tgrid(nblk * t.np), 256, 0, st>>>(t, F, Tprev, T0, Tout, uout, a, b, s, last, sc);
    return cudaGetLastError();
}

cudaError_t launch_tile_stage(const TileGeo& t, int riemann, const double* Tprev, const double* T0, double* W,
                              double* F, double* Tout, double* uout, double a, double b, int s, int last,
                              DevScalars* sc, cudaStream_t st) {
    if (t.g.ndim == 1) return tile_stage_d<1>(t, riemann, Tprev, T0, W, F, Tout, uout, a, b, s, last, sc, st);
    if (t.g.ndim == 2) return tile_stage_d<2>(t, riemann, Tprev, T0, W, F, Tout, uout, a, b, s, last, sc, st);
    return tile_stage_d<3>(t, riemann, Tprev, T0, W, F, Tout, uout, a, b, s, last, sc, st);
}

}  // namespace spark
