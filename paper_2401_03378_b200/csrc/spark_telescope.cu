// spark_telescope.cu — telescoping SSP-RK step for 1-D / 2-D blocks (NEXT N1).
//
// Telescoping mode (lst:spark-telescoping P:1598-1604):
// one guard fill per step with S*NGK layers, then all S stages of a block with
// the halo area updated too (each stage shrinks the valid region by NGK, the
// reconstruction half-width).  Here the "fill" is the CTA's own gather of its
// (nb + 2 S NGK)^2 tile from the neighbouring blocks / boundary map into shared
// memory, and the S stages run on that tile without leaving the SM: one launch
// per STEP, U^(1)..U^(S-1) never touch HBM (80 B per cell per step instead of
// 80 + 120 (S-1)), at the price of recomputing the halo (1.7-2x the FP64 work
// for 16^2 blocks).  Guards beyond a physical boundary are filled once and then
// evolved (reading R17).  The per-face arithmetic is the same device code as
// KB1 (spark_device.cuh).  3-D is not provided: a 16^3 block with a 2 S NGK
// halo (>= 24^3 cells x 5 variables) does not fit in shared memory.
#include <cmath>
#include <cstdint>

#include "spark_device.cuh"
#include "spark_internal.h"

namespace spark {
namespace {

using namespace dev;

constexpr int kTeleThreads = 256;

template <int NDIM, int RECON, int RS>
__global__ void __launch_bounds__(kTeleThreads) telescope_kernel(const StageArgs A, int S) {
    constexpr int NV = NDIM + 2;
    constexpr int NGK = StencilOf<RECON>::NG;
    const Geo& g = A.g;
    extern __shared__ double smem[];
    const int G = S * NGK;
    const int nb0 = g.nb[0], nb1 = NDIM >= 2 ? g.nb[1] : 1;
    const int tx = nb0 + 2 * G, ty = NDIM >= 2 ? nb1 + 2 * G : 1;
    const int gy = NDIM >= 2 ? G : 0;
    const int T = tx * ty;
    double* T0 = smem;             // [NV][ty][tx] U^n
    double* Tp = T0 + NV * T;      // [NV][ty][tx] U^(s-1), updated in place to U^(s)
    double* W = Tp + NV * T;       // [NV][ty][tx] primitives of U^(s-1)
    double* Fx = W + NV * T;       // [NV][ty][tx+1] flux through the face left of (j, i)
    double* Fy = Fx + NV * ty * (tx + 1);  // [NV][ty+1][tx] flux through the face below (j, i)
    double* red = W;               // reused after the stage loop

    const int b = blockIdx.x;
    const int bx = b % g.bn[0], by = (b / g.bn[0]) % g.bn[1];
    const int cx0 = bx * nb0, cy0 = by * nb1;
    const long long bbase = (long long)b * g.bs;  // block-interleaved state U[b][v][c]
    const long long vs = g.vs;
    const double dt = A.dt_ptr ? *A.dt_ptr : A.dt_value;
    const double gamma = g.gamma, gm1 = g.gamma - 1.0, gm1i = 1.0 / (g.gamma - 1.0);
    const double* const nohalo[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};

    if (A.honor_active && !A.sc->active) {  // t >= t_end: U unchanged
        for (int q = threadIdx.x; q < nb0 * nb1; q += blockDim.x)
#pragma unroll
            for (int v = 0; v < NV; v++) A.uout[v * vs + bbase + q] = A.uprev[v * vs + bbase + q];
        return;
    }

    bool ok = true;
    // the thick-halo tile of U^n (faces, edges and corners)
    for (int q = threadIdx.x; q < T; q += blockDim.x) {
        const int i = q % tx, j = q / tx;
        double u[NV];
        fetch_cons<NV>(g, A.uprev, nohalo, cx0 + i - G, cy0 + j - gy, 0, u);
#pragma unroll
        for (int v = 0; v < NV; v++) T0[v * T + q] = Tp[v * T + q] = u[v];
    }
    double cflmin = INFINITY;
    for (int s = 1; s <= S; s++) {
        double a, bco;
        if (s == 1) { a = 0.0; bco = 1.0; }
        else if (S == 2) { a = 0.5; bco = 0.5; }
        else if (s == 2) { a = 0.75; bco = 0.25; }
        else { a = 1.0 / 3.0; bco = 2.0 / 3.0; }
        const int lo = s * NGK;                       // cells updated: [lo, tx-lo) x [loy, ty-loy)
        const int loy = NDIM >= 2 ? lo : 0;
        const int plo = (s - 1) * NGK, ploy = NDIM >= 2 ? plo : 0;  // valid region of U^(s-1)
        __syncthreads();
        for (int q = threadIdx.x; q < T; q += blockDim.x) {
            const int i = q % tx, j = q / tx;
            if (i < plo || i >= tx - plo || j < ploy || j >= ty - ploy) continue;
            double u[NV], w[NV];
#pragma unroll
            for (int v = 0; v < NV; v++) u[v] = Tp[v * T + q];
            ok &= cons_to_prim<NV>(u, w, gm1);
#pragma unroll
            for (int v = 0; v < NV; v++) W[v * T + q] = w[v];
        }
        __syncthreads();
        // faces: x faces i in [lo, tx-lo] of rows [loy, ty-loy); y faces j in [loy, ty-loy] of columns [lo, tx-lo)
        const int nxr = tx - 2 * lo + 1, nyr = ty - 2 * loy;
        const int nfx = nxr * nyr;
        const int nfy = NDIM >= 2 ? (tx - 2 * lo) * (ty - 2 * loy + 1) : 0;
        for (int f = threadIdx.x; f < nfx + nfy; f += blockDim.x) {
            double wl[NV], wr[NV], fl[NV];
            const bool xd = f < nfx;
            int i, j, stride;
            if (xd) {
                i = lo + f % nxr;
                j = loy + f / nxr;
                stride = 1;
            } else {
                const int q = f - nfx;
                i = lo + q % (tx - 2 * lo);
                j = loy + q / (tx - 2 * lo);
                stride = tx;
            }
            const int right = j * tx + i;  // face between right - stride and right
#pragma unroll
            for (int v = 0; v < NV; v++) {
                double sl[2 * NGK - 1], sr[2 * NGK - 1], lo_, hi_;
#pragma unroll
                for (int m = 0; m < 2 * NGK - 1; m++) {
                    sl[m] = W[v * T + right + (m - NGK) * stride];
                    sr[m] = W[v * T + right + (m - NGK + 1) * stride];
                }
                recon_cell<RECON>(sl, lo_, hi_);
                wl[v] = hi_;
                recon_cell<RECON>(sr, lo_, hi_);
                wr[v] = lo_;
            }
            if (RECON != 0 && !(positive(wl[0]) && positive(wl[NV - 1]) && positive(wr[0]) && positive(wr[NV - 1]))) {
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    wl[v] = W[v * T + right - stride];
                    wr[v] = W[v * T + right];
                }
            }
            bool shk = false;  // shockDet (RS 2): cells right-2..right+1 along the normal
            if constexpr (RS == 2) {
                const int vn = xd ? 1 : 2, vp = NV - 1;
                double u[4], pr[4], r[4];
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    u[m] = W[vn * T + right + (m - 2) * stride];
                    pr[m] = W[vp * T + right + (m - 2) * stride];
                    r[m] = W[right + (m - 2) * stride];
                }
                shk = shock_face(u, pr, r, A.g.shock_thresh, gamma);
            }
            if (xd) {
                face_flux<NV, RS, 0>(wl, wr, shk, gamma, gm1i, fl);
#pragma unroll
                for (int v = 0; v < NV; v++) Fx[v * ty * (tx + 1) + j * (tx + 1) + i] = fl[v];
            } else {
                face_flux<NV, RS, (NDIM >= 2 ? 1 : 0)>(wl, wr, shk, gamma, gm1i, fl);
#pragma unroll
                for (int v = 0; v < NV; v++) Fy[v * (ty + 1) * tx + j * tx + i] = fl[v];
            }
        }
        __syncthreads();
        const int nux = tx - 2 * lo;
        for (int q = threadIdx.x; q < nux * (ty - 2 * loy); q += blockDim.x) {
            const int i = lo + q % nux, j = loy + q / nux;
            const int c = j * tx + i;
            double un[NV];
            double grho = 0.0, gmg = 0.0;  // grvAccel accumulators
#pragma unroll
            for (int v = 0; v < NV; v++) {
                const double dfx =
                    (Fx[v * ty * (tx + 1) + j * (tx + 1) + i + 1] - Fx[v * ty * (tx + 1) + j * (tx + 1) + i]) * g.rdx[0];
                double L;
                if (NDIM == 1) {
                    L = -dfx;
                } else {
                    const double dfy = (Fy[v * (ty + 1) * tx + (j + 1) * tx + i] - Fy[v * (ty + 1) * tx + j * tx + i]) *
                                       g.rdx[1];
                    L = -(dfx + dfy);
                }
                if (g.has_grav) L += grav_src<NV>(g, v, Tp[v * T + c], grho, gmg);
                const double uo = fma(bco, fma(dt, L, Tp[v * T + c]), a * T0[v * T + c]);
                un[v] = uo;
            }
            double w[NV];
            const bool good = cons_to_prim<NV>(un, w, gm1);
            ok &= good;
#pragma unroll
            for (int v = 0; v < NV; v++) Tp[v * T + c] = un[v];
            if (s == S) {
                const long long idx = bbase + (long long)(j - loy) * nb0 + (i - lo);
#pragma unroll
                for (int v = 0; v < NV; v++) A.uout[v * vs + idx] = un[v];
                cflmin = fmin(cflmin, cfl_term<NV>(g, w));
            }
        }
    }
    if (!ok) flag_nonphysical(A.sc);
    __syncthreads();
    block_min_to(cflmin, red, &A.sc->acc);
}

template <int NDIM, int RECON, int RS>
cudaError_t launch_t(const StageArgs& a, int S, cudaStream_t s) {
    const size_t smem = telescope_smem_bytes(a.g, RECON, S);
    auto k = telescope_kernel<NDIM, RECON, RS>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long nblk = (long long)a.g.bn[0] * a.g.bn[1] * a.g.bn[2];
    k<<<(unsigned)nblk, kTeleThreads, smem, s>>>(a, S);
    return cudaGetLastError();
}

template <int NDIM, int RECON>
cudaError_t launch_r(const StageArgs& a, int riemann, int S, cudaStream_t s) {
    if (riemann == 0) return launch_t<NDIM, RECON, 0>(a, S, s);
    if (riemann == 1 || RECON == 0) return launch_t<NDIM, RECON, 1>(a, S, s);  // hybrid needs recon >= PLM
    return launch_t<NDIM, RECON, 2>(a, S, s);
}

template <int NDIM>
cudaError_t launch_d(const StageArgs& a, int recon, int riemann, int S, cudaStream_t s) {
    if (recon == 0) return launch_r<NDIM, 0>(a, riemann, S, s);
    if (recon == 1) return launch_r<NDIM, 1>(a, riemann, S, s);
    if (recon == 3) return launch_r<NDIM, 3>(a, riemann, S, s);
    if (recon == 4) return launch_r<NDIM, 4>(a, riemann, S, s);
    return launch_r<NDIM, 2>(a, riemann, S, s);
}

}  // namespace

size_t telescope_smem_bytes(const Geo& g, int recon, int S) {
    const int NGK = (recon == 2 || recon == 4) ? 3 : ((recon == 1 || recon == 3) ? 2 : 1);
    const int G = S * NGK;
    const size_t NV = g.ndim + 2;
    const size_t tx = g.nb[0] + 2 * G, ty = g.ndim >= 2 ? g.nb[1] + 2 * G : 1;
    return sizeof(double) * NV * (3 * tx * ty + ty * (tx + 1) + (g.ndim >= 2 ? (ty + 1) * tx : 0) + 32);
}

cudaError_t launch_telescope(const StageArgs& a, int recon, int riemann, int S, cudaStream_t s) {
    if (a.g.ndim == 1) return launch_d<1>(a, recon, riemann, S, s);
    return launch_d<2>(a, recon, riemann, S, s);
}

}  // namespace spark
