// spark_stage.cu — KB1, the fused Spark stage kernel (sm_100a, FP64).
//
// One launch = one SSP-RK stage over every block of the rank's sub-box:
//   guard gather -> EOS cons->prim (block init, Alg. 7) ->
//   calcLims (reconstruction) -> calcFlux (Riemann) -> updSoln (flux
//   divergence + RK combination) -> calcEos (positivity / CFL-min epilogue),
// i.e. the intra-stage chain of Alg. 8 for one stage of
// lst:spark-nontelescoping, in ONE pass over HBM:
//   U_out = a U_n + b (U_prev + dt L(U_prev)).
//
// Mapping: one CTA per block, one thread per (i,j) column,
// marching over the block's k planes.  Per plane:
//   S1 load   plane k+NG of the thread's column into a ring of 2*NG-1 primitive
//             planes (own column only) and the x/y face halos of plane k into
//             a padded shared plane `cur` (neighbour block read straight from
//             the pool, L2-resident; no guard cells are stored in HBM)
//   S2 recon  cell-centric: each cell's x, y (and z, from the ring) limiter /
//             smoothness evaluation is done once and gives both edge states
//             (face-centric variant, 16x16 first order / minmod PLM: x/y states
//             are built in S3 by the face's own thread; no S2->S3 barrier)
//   S3 flux   each face once: x/y faces into shared memory, the z face in
//             registers (carried to the next plane)
//   S4 update own cell; last stage also the CFL-min epilogue.
// Block shape is a template parameter for the production shapes (16x16 planes)
// so that all index arithmetic folds; 0 means "runtime" (any shape <= 256 cells
// per plane).
#include <cmath>
#include <cstdint>

#include "spark_device.cuh"
#include "spark_internal.h"

namespace spark {
namespace {

using namespace dev;

constexpr int kThreads = 256;

// Launch policy of a specialisation (host and device agree through this).
// The design experiments that were measured and dropped (a 9th "boundary"
// warp, cp.async / TMA staging of the S4 operands, paired face-centric
// solves, 3 CTAs/SM, ...) are recorded with their numbers in DESIGN.md §4.2;
// the kernel below keeps only the measured winners.
// Face-centric x/y reconstruction (16x16 planes, first order / minmod PLM): the
// thread that solves a face reconstructs both of its states straight from the
// plane (two limiter evaluations per face instead of one per cell), so the
// face-state arrays XB/YB, the halo edge-state pass and the S2->S3 barrier
// disappear, and S3 solves one face at a time (no spills).
__host__ __device__ constexpr bool policy_face_centric(int ndim, int recon, int nbx, int nby) {
    // first order and minmod PLM (3-D +16-20 %, 2-D +12-20 %); PLM-MC with the
    // one-barrier plane loop: 3-D 13.97 -> 17.96 G zone-updates/s (+29 %), 2-D
    // RK2 17.30 -> 18.40 (+6 %) (alone, round 1, it was 1 % slower); WENO5
    // would evaluate its edges twice
    return nbx == 16 && nby == 16 && ndim >= 2 && (recon <= 1 || recon == 3);
}

template <int NV>
__device__ __forceinline__ void ldg_cons(const double* __restrict__ p, long long stride, double* u) {
#pragma unroll
    for (int v = 0; v < NV; v++) u[v] = __ldg(p + v * stride);
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Checked build (-DSPARK_CHECKED, libspark_checked.so; compute-sanitizer is
// closed on the GPU pool): every shared-memory address KB1 forms is asserted
// inside the launch's dynamic shared memory and every global address inside
// one of the launch's buffers (U^(s-1), U^n, the output, the received
// slabs); a violation traps (the launch fails with an illegal-instruction
// error). Production builds compile the checks away.
#ifdef SPARK_CHECKED
#define SCHK(p) schk_(p)
#define GCHK(p) gchk_(p)
#else
#define SCHK(p) ((void)0)
#define GCHK(p) ((void)0)
#endif

// Padded ring (3-D, reconstruction half-width <= 2): the ring slots of the
// z-march are whole padded planes [NV][(nb1+2NG)][(nb0+2NG)], so the slot of
// plane k IS the x/y working plane of plane k (its halo cells are written into
// the slot's padding in S1): no per-plane copy of the column cell into a
// separate plane (5 LDS + 5 STS per cell and plane).  WENO5's 5 slots would
// not fit twice per SM; it keeps the compact ring and a separate plane.
// One CTA barrier per plane (3-D face-centric 16x16 path): the x-face fluxes of
// a row go lane to lane through warp shuffles (only the block-boundary face 0
// of each row through shared memory), and the flux arrays are double-buffered
// by plane parity, so the S1->S2 barrier — whose only job was to keep S3 of
// plane k from overwriting fluxes that S4 of plane k-1 still reads — goes.
// Measured on 256^3 PLM: 20.90 -> 21.38 G zone-updates/s (+2.3 %).
__host__ __device__ constexpr bool policy_one_barrier(int ndim, int recon, int nbx, int nby) {
    return ndim == 3 && nbx == 16 && nby == 16 && (recon <= 1 || recon == 3);
}

__host__ __device__ constexpr bool policy_pad_ring(int ndim, int recon) {
    return ndim == 3 && recon != 2 && recon != 4;
}

template <int NDIM, int RECON, int RS, int NBX, int NBY, int NBZ>
__global__ void __launch_bounds__(kThreads, NDIM == 3 ? 2 : 3) stage_kernel(const StageArgs A) {
    constexpr bool FC = policy_face_centric(NDIM, RECON, NBX, NBY);
    // paired face solves in S3 (WENO5 / MC); the face-centric path solves one
    // face at a time (paired, its reconstruction temporaries spill: -9 %)
    constexpr bool FUSE = NBX == 16 && NBY == 16 && NDIM == 3 && !FC;
    constexpr int NV = NDIM + 2;
    constexpr int NG = StencilOf<RECON>::NG;
    constexpr int R = NG - 1;  // cell-centric reconstruction radius
    constexpr int RS_ = 2 * NG - 1 > 2 ? 2 * NG - 1 : 2;  // ring slots (planes k-R' .. k+NG alive)
    constexpr int RING = NDIM == 3 ? RS_ : 0;
    constexpr bool PADRING = policy_pad_ring(NDIM, RECON);
    // 3-D: the S4 operands are only prefetched into L2 in S2 and loaded in S4,
    // so no 20 registers are held across S3 (WENO5 spills 148 -> 44 B, 8.6 ->
    // 8.9 G zone-updates/s) and no shared-memory staging is needed (PLM +1 %
    // over cp.async staging); 2-D measured 3 % slower that way and keeps the
    // register prefetch
    constexpr bool L2PF = NDIM == 3;
    // own x / y face fluxes kept in registers for S4 (face-centric 16x16 path)
    constexpr bool OWNF = FC && !FUSE && NBX == 16 && NBY == 16 && NDIM >= 2;  // +0.5 %
    constexpr bool ONEBAR = OWNF && policy_one_barrier(NDIM, RECON, NBX, NBY);
    constexpr int NBUF = ONEBAR ? 2 : 1;  // flux buffers (by plane parity)
    constexpr bool ZTOP = !PADRING;  // z edges of cell k+1 in S1 (see there)
    constexpr int RO = NDIM >= 2 ? NG : 0;  // row offset of the interior in cur
    const Geo& g = A.g;
    extern __shared__ double smem[];
#ifdef SPARK_CHECKED
    unsigned dsz_;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz_));
    auto schk_ = [&](const double* p) {
        if (p < smem || p >= smem + dsz_ / sizeof(double)) __trap();
    };
    const long long nst_ = (long long)g.nvar * g.ncell;
    auto gchk_ = [&](const double* p) {
        bool in = (p >= A.uprev && p < A.uprev + nst_) || (A.un && p >= A.un && p < A.un + nst_) ||
                  (p >= A.uout && p < A.uout + nst_);
        for (int d = 0; d < 3; d++)
            for (int e = 0; e < 2; e++)
                in |= A.halo[d][e] && p >= A.halo[d][e] && p < A.halo[d][e] + (long long)g.nvar * g.slab[d];
        if (!in) __trap();
    };
#endif

    const int nb0 = NBX ? NBX : g.nb[0];
    const int nb1 = NDIM >= 2 ? (NBY ? NBY : g.nb[1]) : 1;
    const int nb2 = NDIM >= 3 ? (NBZ ? NBZ : g.nb[2]) : 1;
    const int P = nb0 * nb1;
    const int tid = threadIdx.x;
    const bool live = tid < P;
    const int ti = live ? tid % nb0 : 0, tj = live ? tid / nb0 : 0;
    const int b = A.blk0 + (int)blockIdx.x;  // a block range (spark_step_host's pipelined last stage)
    const int bx = b % g.bn[0], by = (b / g.bn[0]) % g.bn[1], bz = b / (g.bn[0] * g.bn[1]);
    const int cx0 = bx * nb0, cy0 = by * nb1, cz0 = bz * nb2;
    // block-interleaved state U[b][v][c]: with a compile-time block shape the
    // variable stride is an immediate offset from one pointer
    const long long vs = NBZ ? (long long)NBX * NBY * NBZ : g.vs;
    const long long bs = NBZ ? (long long)NV * NBX * NBY * NBZ : g.bs;
    const long long bbase = (long long)b * bs;
    const double* __restrict__ up = A.uprev;

    const int cw = nb0 + 2 * NG, ch = NDIM >= 2 ? nb1 + 2 * NG : 1;
    const int CP = cw * ch;
    const int fxs = nb0 + 1;                   // x faces per row
    const int fxn = fxs * nb1;
    const int fyn = NDIM >= 2 ? nb0 * (nb1 + 1) : 0;
    double* ring = smem;                       // [RING][NV][P] ([RING][NV][CP] if PADRING)
    double* cur0 = ring + RING * NV * (PADRING ? CP : P);  // [NV][CP] (not with PADRING)
    // ONEBAR: XA is only the boundary face 0 of each row, [NBUF][NV][nb1]
    const int xsz = ONEBAR ? nb1 : fxn;
    double* XA = cur0 + (PADRING ? 0 : NV * CP);  // [NV][fxn]: L state at x face, then x flux
    double* XB = XA + NBUF * NV * xsz;         // [NV][fxn]: R state at x face (not with FC)
    double* YA = XB + (FC ? 0 : NV * fxn);     // [NBUF][NV][fyn]
    double* YB = YA + NBUF * NV * fyn;         // [NV][fyn] (not with FC)
    // FC in 3-D: the next plane's raw halo cells arrive by cp.async in shared
    // memory (no prefetch registers held across the plane)
    constexpr bool HSM = FC && NDIM == 3;
    double* hs = YB + (FC ? 0 : NV * fyn);     // [NV][nh]

    const double dt = A.dt_ptr ? *A.dt_ptr : A.dt_value;
    const double a = A.a, bco = A.b;
    const double gamma = g.gamma, gm1 = g.gamma - 1.0, gm1i = 1.0 / (g.gamma - 1.0);
    const double thr = g.shock_thresh;  // shockDet (RS 2 only)

    if (A.part) {  // interior / rank-boundary split (CTA-uniform early exit)
        const bool edge = (g.halo[0][0] && bx == 0) || (g.halo[0][1] && bx == g.bn[0] - 1) ||
                          (NDIM >= 2 && ((g.halo[1][0] && by == 0) || (g.halo[1][1] && by == g.bn[1] - 1))) ||
                          (NDIM >= 3 && ((g.halo[2][0] && bz == 0) || (g.halo[2][1] && bz == g.bn[2] - 1)));
        if (edge != (A.part == 2)) return;
    }
    if (A.honor_active && !A.sc->active) {  // t >= t_end: U^(s) = U^(s-1)
        if (live)
            for (int kk = 0; kk < nb2; kk++) {
                const long long idx = bbase + ((long long)kk * nb1 + tj) * nb0 + ti;
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    GCHK(A.uout + v * vs + idx);
                    GCHK(up + v * vs + idx);
                    A.uout[v * vs + idx] = up[v * vs + idx];
                }
            }
        return;
    }

    bool ok = true;
    // conserved -> primitive of the cell at block-local (x, y, z) (at most one
    // coordinate outside the block)
    auto load_cons = [&](int x, int y, int z, double* u) {
        int d = -1, side = 0, lx = x, ly = y, lz = z;
        if (x < 0 || x >= nb0) { d = 0; side = x >= nb0; lx = side ? x - nb0 : x + nb0; }
        else if (NDIM >= 2 && (y < 0 || y >= nb1)) { d = 1; side = y >= nb1; ly = side ? y - nb1 : y + nb1; }
        else if (NDIM >= 3 && (z < 0 || z >= nb2)) { d = 2; side = z >= nb2; lz = side ? z - nb2 : z + nb2; }
        const long long off = ((long long)lz * nb1 + ly) * nb0 + lx;
        // face-neighbour block inside this rank's sub-box (else: general gather)
        int q0 = bx, q1 = by, q2 = bz;
        bool inside = true;
        if (d == 0) { q0 += side ? 1 : -1; inside = q0 >= 0 && q0 < g.bn[0]; }
        if (d == 1) { q1 += side ? 1 : -1; inside = q1 >= 0 && q1 < g.bn[1]; }
        if (d == 2) { q2 += side ? 1 : -1; inside = q2 >= 0 && q2 < g.bn[2]; }
        if (d < 0) {
            GCHK(up + bbase + off);
            GCHK(up + bbase + off + (NV - 1) * vs);
            ldg_cons<NV>(up + bbase + off, vs, u);
        } else if (inside) {
            GCHK(up + (q0 + (long long)g.bn[0] * (q1 + (long long)g.bn[1] * q2)) * bs + off + (NV - 1) * vs);
            ldg_cons<NV>(up + (q0 + (long long)g.bn[0] * (q1 + (long long)g.bn[1] * q2)) * bs + off, vs, u);
        } else {
            fetch_cons<NV>(g, up, A.halo, cx0 + x, cy0 + y, cz0 + z, u);
        }
    };
    auto load_prim = [&](int x, int y, int z, double* w) {
        double u[NV];
        load_cons(x, y, z, u);
        ok &= cons_to_prim<NV>(u, w, gm1);
    };

    // z machinery (3-D): ring slot of plane z is (z + NG) mod RS_
    auto ring_at = [&](int z, int v) -> double& {
        double& r = PADRING ? ring[(((z + NG) % RS_) * NV + v) * CP + (tj + RO) * cw + ti + NG]
                            : ring[(((z + NG) % RS_) * NV + v) * P + tid];
        SCHK(&r);
        return r;
    };
    double zhi[NV];   // L state of the face above the current plane (top edge of cell kk)
    double fzlo[NV];  // flux through the face below the current plane
    double fzhi[NV];
#pragma unroll
    for (int v = 0; v < NV; v++) zhi[v] = fzlo[v] = fzhi[v] = 0.0;

    // z reconstruction of cell z of this column from the ring
    // ... with the top stencil plane z+R taken from registers (top[], just converted)
    auto zrecon_top = [&](int z, const double* top, double* lo, double* hi) {
#pragma unroll
        for (int v = 0; v < NV; v++) {
            double s[2 * R + 1];
#pragma unroll
            for (int m = 0; m < 2 * R; m++) s[m] = ring_at(z - R + m, v);
            s[2 * R] = top[v];
            recon_cell<RECON>(s, lo[v], hi[v]);
        }
    };
    auto zrecon = [&](int z, double* lo, double* hi) {
#pragma unroll
        for (int v = 0; v < NV; v++) {
            double s[2 * R + 1];
#pragma unroll
            for (int m = 0; m <= 2 * R; m++) s[m] = ring_at(z - R + m, v);
            recon_cell<RECON>(s, lo[v], hi[v]);
        }
    };
    // flux through the z face between cells z and z+1 of this column
    auto zflux = [&](int z, double* wl, double* wr, bool shk, double* f) {
        if (RECON != 0 && !(positive(wl[0]) && positive(wl[NV - 1]) && positive(wr[0]) && positive(wr[NV - 1]))) {
#pragma unroll
            for (int v = 0; v < NV; v++) {
                wl[v] = ring_at(z, v);
                wr[v] = ring_at(z + 1, v);
            }
        }
        face_flux<NV, RS, 2>(wl, wr, shk, gamma, gm1i, f);
    };
    // shockDet along z (RS 2): shock cell z of this column from the ring
    // (planes z-1, z+1); a z face's flag is the OR of its two cells, the lower
    // one carried from the previous plane (the ring no longer holds plane z-1
    // when face z+1/2 is solved)
    auto zshock_cell = [&](int z) -> bool {
        if constexpr (RS != 2) return false;
        else return shock_cell(ring_at(z - 1, NV - 2), ring_at(z + 1, NV - 2), ring_at(z - 1, NV - 1),
                               ring_at(z + 1, NV - 1), ring_at(z - 1, 0), ring_at(z + 1, 0), thr, gamma);
    };
    bool zs_prev = false;  // shock cell flag of the current plane (z)
    // shockDet at an x or y face (RS 2): c = cell i+1 of the face (variable 0
    // of the working plane), st the stride along the normal, vn the normal
    // velocity's variable
    auto shk_at = [&](const double* c, int st, int vn) -> bool {
        if constexpr (RS != 2) return false;
        else {
            double u[4], pr[4], r[4];
#pragma unroll
            for (int m = 0; m < 4; m++) {
                SCHK(c + (NV - 1) * CP + (m - 2) * st);
                SCHK(c + (m - 2) * st);
                u[m] = c[vn * CP + (m - 2) * st];
                pr[m] = c[(NV - 1) * CP + (m - 2) * st];
                r[m] = c[(m - 2) * st];
            }
            return shock_face(u, pr, r, thr, gamma);
        }
    };

    if (NDIM == 3) {
        if (live) {
            double w[NV];
            for (int z = -NG; z < NG - 1; z++) {
                load_prim(ti, tj, z, w);
#pragma unroll
                for (int v = 0; v < NV; v++) ring_at(z, v) = w[v];
            }
            double lo[NV], hi[NV], l0[NV];
            zrecon(-1, l0, hi);  // top edge of cell -1 -> L state of face -1/2
            const bool zs_m1 = zshock_cell(-1);  // planes -2, 0 (before plane -NG dies)
            load_prim(ti, tj, NG - 1, w);  // replaces plane -NG (dead)
#pragma unroll
            for (int v = 0; v < NV; v++) ring_at(NG - 1, v) = w[v];
            zrecon(0, lo, zhi);  // bottom edge of cell 0 -> R state of face -1/2
            zs_prev = zshock_cell(0);
            zflux(-1, hi, lo, zs_m1 || zs_prev, fzlo);
        }
    }

    const int nhx = 2 * NG * nb1;
    const int nh = nhx + (NDIM >= 2 ? 2 * NG * nb0 : 0);
    const int nbr = 2 * nb1 + (NDIM >= 2 ? 2 * nb0 : 0);  // boundary recon items
    const int nbf = nb1 + (NDIM >= 2 ? nb0 : 0);          // boundary faces (x face 0, y face 0)
    double cflmin = INFINITY;

    // x/y face-halo cell h of a plane -> block-local (cx, cy):
    // x strips [side][row][depth], then y strips [side][depth][col]
    auto halo_cell = [&](int h, int& cx, int& cy) {
        if (h < nhx) {
            const int side = h / (NG * nb1), r = h % (NG * nb1);
            cy = r / NG;
            const int dp = r % NG;
            cx = side ? nb0 + dp : dp - NG;
        } else {
            const int hh = h - nhx;
            const int side = hh / (NG * nb0), r = hh % (NG * nb0);
            const int dp = r / nb0;
            cx = r % nb0;
            cy = side ? nb1 + dp : dp - NG;
        }
    };
    // 16x16 planes: nh <= 256, so thread h owns halo cell h for every plane and
    // prefetches it one plane ahead (raw conserved values in registers)
    constexpr bool HPF = NBX == 16 && NBY == 16;
    // HLATE (3-D face-centric PLM / first order with the padded ring): the halo
    // cells of plane k+1 are converted and written into the padding of plane
    // k+1's ring slot at the start of S2 of plane k by the LAST nh threads
    // (warps 4-7, which have one face solve less than warp 0 per plane), so S1
    // has no halo work and the S1->S2 barrier no imbalance.  The cp.async of
    // that halo was issued one plane earlier and completed by the previous S4's
    // wait (measured: start of S2 +3.6 % over end of S3).
    constexpr bool HLATE = HSM && PADRING;
    const bool hact = HPF && (HLATE ? tid >= P - nh : tid < nh);
    const int hid = HLATE ? tid - (P - nh) : tid;  // halo cell of this thread
    int hcx = 0, hcy = 0;
    double hpre[NV];
    // Per-plane sources resolved once: a halo cell in a face-neighbour block of
    // this sub-box is a plain column (stride P per plane) of that block; others
    // (physical boundary / received slab) take the general gather every plane.
    // The source of halo cell (x, y) in plane z (face-neighbour block, received
    // slab, or physical-boundary image) is affine in z: resolved once (two
    // fetch_src calls), the z-march does plain strided loads.  Compact form:
    // base pointer, 32-bit variable stride, and plane stride << 4 | flip bits.
    const double* hp = up;
    int hvs = 0, hzf = 0;
    if (hact) {
        halo_cell(hid, hcx, hcy);
        if (NDIM == 3) {
            Src s0, s1;
            fetch_src(g, up, A.halo, cx0 + hcx, cy0 + hcy, cz0, s0);
            fetch_src(g, up, A.halo, cx0 + hcx, cy0 + hcy, cz0 + (nb2 > 1 ? 1 : 0), s1);
            hp = s0.p;
            hvs = (int)s0.vs;
            hzf = (int)((s1.p - s0.p) * 16) | s0.flip;
            if (HLATE) {  // plane 0 now (into its slot's padding), plane 1 in flight
                double w[NV];
                GCHK(hp);
                GCHK(hp + (long long)(NV - 1) * hvs);
                load_src<NV>(hp, hvs, s0.flip, hpre);
                ok &= cons_to_prim<NV>(hpre, w, gm1);
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    SCHK(&ring[((NG % RS_) * NV + v) * CP + (hcy + RO) * cw + hcx + NG]);
                    ring[((NG % RS_) * NV + v) * CP + (hcy + RO) * cw + hcx + NG] = w[v];
                }
                if (nb2 > 1) {
                    const double* src = hp + (hzf >> 4);
#pragma unroll
                    for (int v = 0; v < NV; v++) {
                        SCHK(hs + v * nh + hid);
                        GCHK(src + (long long)v * hvs);
                        cp_async8(hs + v * nh + hid, src + (long long)v * hvs);
                    }
                    cp_async_commit();
                }
            } else if (HSM) {
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    SCHK(hs + v * nh + tid);
                    GCHK(hp + (long long)v * hvs);
                    cp_async8(hs + v * nh + tid, hp + (long long)v * hvs);
                }
                cp_async_commit();
            } else {
                GCHK(hp + (long long)(NV - 1) * hvs);
                load_src<NV>(hp, hvs, s0.flip, hpre);
            }
        } else {  // one plane: a single load through the block-neighbour fast path
            load_cons(hcx, hcy, 0, hpre);
        }
    }
    auto load_halo = [&](int z, double* u) {
        GCHK(hp + (long long)z * (hzf >> 4) + (long long)(NV - 1) * hvs);
        load_src<NV>(hp + (long long)z * (hzf >> 4), hvs, hzf & 15, u);
    };
    // this column: planes z < nb2 of the own block, z >= nb2 of the block above
    // (if inside the sub-box, else the general gather)
    const double* csrc = up + bbase + (long long)tj * nb0 + ti;
    const double* casrc = (NDIM == 3 && bz + 1 < g.bn[2]) ? csrc + (long long)g.bn[0] * g.bn[1] * bs : nullptr;
    auto load_col = [&](int z, double* u) {
        if (z < nb2) {
            GCHK(csrc + (long long)z * P + (NV - 1) * vs);
            ldg_cons<NV>(csrc + (long long)z * P, vs, u);
        } else if (casrc) {
            GCHK(casrc + (long long)(z - nb2) * P + (NV - 1) * vs);
            ldg_cons<NV>(casrc + (long long)(z - nb2) * P, vs, u);
        }
        else load_cons(ti, tj, z, u);
    };

    // raw conserved values of this column's plane kk+NG, loaded one plane ahead
    double pre[NV];
    if (NDIM == 3 && live) load_cons(ti, tj, NG, pre);

    double* const XA0 = XA;
    double* const YA0 = YA;
    // ONEBAR: plane 0's slot (prologue ring planes + halo) must be complete
    // before S3 of plane 0; later planes are fenced by the previous S3->S4 barrier
    if (ONEBAR) __syncthreads();
    for (int kk = 0; kk < nb2; kk++) {
        double* const XA = XA0 + (ONEBAR ? (kk & 1) * NV * xsz : 0);  // this plane's flux buffers
        double* const YA = YA0 + (ONEBAR ? (kk & 1) * NV * fyn : 0);
        double zlo[NV], zhn[NV];  // edges of cell kk+1 along z (R state of face kk+1/2; next zhi)
        // the x/y working plane of plane kk (PADRING: its ring slot)
        double* const cur = PADRING ? ring + ((kk + NG) % RS_) * NV * CP : cur0;
        // ---------------------------------------------------------------- S1
        // No barrier before S1: cur was last read in S3 of the previous plane
        // (fenced by the S3->S4 barrier) and the face arrays written in S2 are
        // fenced by the S1->S2 barrier; the ring is per-thread.
        if (live) {
            double w[NV];
            if (NDIM == 3) {
                ok &= cons_to_prim<NV>(pre, w, gm1);
                if (kk + 1 < nb2) load_col(kk + 1 + NG, pre);  // prefetch the next plane
#pragma unroll
                for (int v = 0; v < NV; v++) ring_at(kk + NG, v) = w[v];
                // WENO5: z edges of cell kk+1 now, plane kk+NG from registers
                // (+5 %); PLM measured 1 % better with them in S2
                if (ZTOP) zrecon_top(kk + 1, w, zlo, zhn);
                if (!PADRING) {
#pragma unroll
                    for (int v = 0; v < NV; v++) {
                        SCHK(&cur[v * CP + (tj + RO) * cw + ti + NG]);
                        cur[v * CP + (tj + RO) * cw + ti + NG] = ring_at(kk, v);
                    }
                }
            } else {
                load_prim(ti, tj, kk, w);
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    SCHK(&cur[v * CP + (tj + RO) * cw + ti + NG]);
                    cur[v * CP + (tj + RO) * cw + ti + NG] = w[v];
                }
            }
        }
        if (HLATE) {
            // halo of this plane already in its slot (written during plane kk-1)
        } else if (HPF) {  // one halo cell per thread, prefetched one plane ahead
            if (hact) {
                double w[NV];
                if (HSM) {
                    cp_async_wait_all();
#pragma unroll
                    for (int v = 0; v < NV; v++) {
                        SCHK(hs + v * nh + tid);
                        hpre[v] = hs[v * nh + tid];
                    }
#pragma unroll
                    for (int d = 0; d < NV - 2; d++)  // reflecting-boundary image: momentum sign
                        hpre[1 + d] = __hiloint2double(__double2hiint(hpre[1 + d]) ^ (((hzf >> (1 + d)) & 1) << 31),
                                                       __double2loint(hpre[1 + d]));
                    ok &= cons_to_prim<NV>(hpre, w, gm1);
                    if (kk + 1 < nb2) {
                        const double* src = hp + (long long)(kk + 1) * (hzf >> 4);
#pragma unroll
                        for (int v = 0; v < NV; v++) {
                            SCHK(hs + v * nh + tid);
                            GCHK(src + (long long)v * hvs);
                            cp_async8(hs + v * nh + tid, src + (long long)v * hvs);
                        }
                        cp_async_commit();
                    }
                } else {
                    ok &= cons_to_prim<NV>(hpre, w, gm1);
                    if (kk + 1 < nb2) load_halo(kk + 1, hpre);
                }
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    SCHK(&cur[v * CP + (hcy + RO) * cw + hcx + NG]);
                    cur[v * CP + (hcy + RO) * cw + hcx + NG] = w[v];
                }
            }
        } else {
            for (int h = tid; h < nh; h += blockDim.x) {
                int cx, cy;
                halo_cell(h, cx, cy);
                double w[NV];
                load_prim(cx, cy, kk, w);
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    SCHK(&cur[v * CP + (cy + RO) * cw + cx + NG]);
                    cur[v * CP + (cy + RO) * cw + cx + NG] = w[v];
                }
            }
        }
        if (!ONEBAR) __syncthreads();
        // ---------------------------------------------------------------- S2
        if (HLATE && hact && kk + 1 < nb2) {  // halo of plane kk+1 -> its slot
            double w[NV];
            cp_async_wait_all();  // no-op: complete since S4 of the previous plane
#pragma unroll
            for (int v = 0; v < NV; v++) {
                SCHK(hs + v * nh + hid);
                hpre[v] = hs[v * nh + hid];
            }
#pragma unroll
            for (int d = 0; d < NV - 2; d++)  // reflecting-boundary image: momentum sign
                hpre[1 + d] = __hiloint2double(__double2hiint(hpre[1 + d]) ^ (((hzf >> (1 + d)) & 1) << 31),
                                               __double2loint(hpre[1 + d]));
            ok &= cons_to_prim<NV>(hpre, w, gm1);
            double* nxt = ring + ((kk + 1 + NG) % RS_) * NV * CP + (hcy + RO) * cw + hcx + NG;
#pragma unroll
            for (int v = 0; v < NV; v++) {
                SCHK(nxt + v * CP);
                nxt[v * CP] = w[v];
            }
            if (kk + 2 < nb2) {
                const double* src = hp + (long long)(kk + 2) * (hzf >> 4);
#pragma unroll
                for (int v = 0; v < NV; v++) {
                        SCHK(hs + v * nh + hid);
                        GCHK(src + (long long)v * hvs);
                        cp_async8(hs + v * nh + hid, src + (long long)v * hvs);
                    }
                cp_async_commit();
            }
        }
        // operands of the S4 update, requested now so the loads overlap S2/S3
        double u0v[NV], unv[NV];
        const long long cidx = bbase + ((long long)kk * nb1 + tj) * nb0 + ti;
        if (live) {
            if (L2PF) {  // only an L2 prefetch now; loaded in S4 (no registers held)
                // U^(s-1) of this plane is still in L2 (read as the column
                // prefetch NG planes ago): only U^n is prefetched (+1.2 % PLM,
                // +1.8 % WENO5 over prefetching both)
#pragma unroll
                for (int v = 0; v < NV; v++)
                    if (a != 0.0) asm volatile("prefetch.global.L2 [%0];" ::"l"(A.un + v * vs + cidx));
            } else {
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    GCHK(up + v * vs + cidx);
                    if (a != 0.0) GCHK(A.un + v * vs + cidx);
                    u0v[v] = __ldg(up + v * vs + cidx);
                    unv[v] = a != 0.0 ? __ldg(A.un + v * vs + cidx) : 0.0;
                }
            }
        }
        if (live && NDIM == 3 && !ZTOP) zrecon(kk + 1, zlo, zhn);
        if (live && !FC) {
#pragma unroll
            for (int v = 0; v < NV; v++) {
                double s[2 * R + 1], lo, hi;
                const double* c = cur + v * CP + (tj + RO) * cw + ti + NG;
                SCHK(c - R);
                SCHK(c + R);
                SCHK(XB + v * fxn + tj * fxs + ti);
                SCHK(XA + v * fxn + tj * fxs + ti + 1);
#pragma unroll
                for (int m = 0; m <= 2 * R; m++) s[m] = c[m - R];
                recon_cell<RECON>(s, lo, hi);
                XB[v * fxn + tj * fxs + ti] = lo;
                XA[v * fxn + tj * fxs + ti + 1] = hi;
                if (NDIM >= 2) {
                    SCHK(c - R * cw);
                    SCHK(c + R * cw);
                    SCHK(YB + v * fyn + tj * nb0 + ti);
                    SCHK(YA + v * fyn + (tj + 1) * nb0 + ti);
#pragma unroll
                    for (int m = 0; m <= 2 * R; m++) s[m] = c[(m - R) * cw];
                    recon_cell<RECON>(s, lo, hi);
                    YB[v * fyn + tj * nb0 + ti] = lo;
                    YA[v * fyn + (tj + 1) * nb0 + ti] = hi;
                }
            }
        }
        // edge states from the halo cells: one (cell, variable) item per thread
        // round so the extra work spreads over all warps
        for (int qv = tid; !FC && qv < nbr * NV; qv += blockDim.x) {
            const int v = qv / nbr, q = qv - v * nbr;
            const bool xd = q < 2 * nb1;
            const int qq = xd ? q : q - 2 * nb1;
            const int side = xd ? qq / nb1 : qq / nb0;
            const int r = xd ? qq % nb1 : qq % nb0;
            double s[2 * R + 1], lo, hi;
            if (xd) {
                const double* c = cur + v * CP + (r + RO) * cw + (side ? nb0 : -1) + NG;
                SCHK(c - R);
                SCHK(c + R);
#pragma unroll
                for (int m = 0; m <= 2 * R; m++) s[m] = c[m - R];
            } else {
                const double* c = cur + v * CP + ((side ? nb1 : -1) + RO) * cw + r + NG;
                SCHK(c - R * cw);
                SCHK(c + R * cw);
#pragma unroll
                for (int m = 0; m <= 2 * R; m++) s[m] = c[(m - R) * cw];
            }
            recon_cell<RECON>(s, lo, hi);
            if (xd) {
                SCHK(side ? XB + v * fxn + r * fxs + nb0 : XA + v * fxn + r * fxs);
                if (side) XB[v * fxn + r * fxs + nb0] = lo;
                else XA[v * fxn + r * fxs] = hi;
            } else {
                SCHK(side ? YB + v * fyn + nb1 * nb0 + r : YA + v * fyn + r);
                if (side) YB[v * fyn + nb1 * nb0 + r] = lo;
                else YA[v * fyn + r] = hi;
            }
        }
        if (!FC) __syncthreads();
        // ---------------------------------------------------------------- S3
        // x face at column f of row r: cells (f-1, f); y face at row f of column r
        double fxo[NV], fyo[NV];  // this thread's own x / y face fluxes (OWNF)
        bool zsh = false;         // shockDet flag of the z face kk+1/2 (RS 2)
        if (NDIM == 3 && RS == 2 && live) {
            const bool zs_next = zshock_cell(kk + 1);
            zsh = zs_prev || zs_next;
            zs_prev = zs_next;
        }
        auto xface = [&](int r, int f, double* fl) {
            double wl[NV], wr[NV];
#pragma unroll
            for (int v = 0; v < NV; v++) {
                if (FC) {
                    const double* c = cur + v * CP + (r + RO) * cw + f + NG;  // cell f
                    SCHK(c - (RECON ? 2 : 1));  // first order reads only the face's two cells
                    SCHK(c + (RECON ? 1 : 0));
                    face_states<RECON>(c[-2], c[-1], c[0], c[1], wl[v], wr[v]);
                } else {
                    SCHK(XA + v * fxn + r * fxs + f);
                    SCHK(XB + v * fxn + r * fxs + f);
                    wl[v] = XA[v * fxn + r * fxs + f];
                    wr[v] = XB[v * fxn + r * fxs + f];
                }
            }
            if (RECON != 0 && !(positive(wl[0]) && positive(wl[NV - 1]) && positive(wr[0]) && positive(wr[NV - 1]))) {
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    wl[v] = cur[v * CP + (r + RO) * cw + f - 1 + NG];
                    wr[v] = cur[v * CP + (r + RO) * cw + f + NG];
                }
            }
            face_flux<NV, RS, 0>(wl, wr, shk_at(cur + (r + RO) * cw + f + NG, 1, 1), gamma, gm1i, fl);
            if (!ONEBAR) {  // ONEBAR: the own face stays in registers (shuffled in S4)
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    SCHK(XA + v * fxn + r * fxs + f);
                    XA[v * fxn + r * fxs + f] = fl[v];
                }
            }
        };
        auto yface = [&](int r, int f, double* fl) {
            double wl[NV], wr[NV];
#pragma unroll
            for (int v = 0; v < NV; v++) {
                if (FC) {
                    const double* c = cur + v * CP + (f + NG) * cw + r + NG;  // cell f of column r
                    SCHK(c - (RECON ? 2 : 1) * cw);
                    SCHK(c + (RECON ? 1 : 0) * cw);
                    face_states<RECON>(c[-2 * cw], c[-cw], c[0], c[cw], wl[v], wr[v]);
                } else {
                    SCHK(YA + v * fyn + f * nb0 + r);
                    SCHK(YB + v * fyn + f * nb0 + r);
                    wl[v] = YA[v * fyn + f * nb0 + r];
                    wr[v] = YB[v * fyn + f * nb0 + r];
                }
            }
            if (RECON != 0 && !(positive(wl[0]) && positive(wl[NV - 1]) && positive(wr[0]) && positive(wr[NV - 1]))) {
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    wl[v] = cur[v * CP + (f - 1 + NG) * cw + r + NG];
                    wr[v] = cur[v * CP + (f + NG) * cw + r + NG];
                }
            }
            face_flux<NV, RS, 1>(wl, wr, shk_at(cur + (f + NG) * cw + r + NG, cw, 2), gamma, gm1i, fl);
#pragma unroll
            for (int v = 0; v < NV; v++) {
                SCHK(YA + v * fyn + f * nb0 + r);
                YA[v * fyn + f * nb0 + r] = fl[v];
            }
        };
        if (FUSE) {
            // 16x16 planes: the two independent solves of each round are issued
            // back to back (branch-free Riemann) so their dependency chains
            // interleave.  Round 1: own x face + own y face.  Round 2: own z face
            // and, on warp 0, the 32 block-boundary faces (x face 0 of rows 0-15
            // on lanes 0-15, y face 0 of columns 0-15 on lanes 16-31, the latter
            // solved in the x frame with u_x <-> u_y swapped: bitwise identical).
            const int xo = tj * fxs + ti + 1, yo = (tj + 1) * nb0 + ti;
            double xl[NV], xr[NV], yl[NV], yr[NV], fx[NV], fy[NV];
#pragma unroll
            for (int v = 0; v < NV; v++) {
                if (FC) {  // x face ti+1 from cells ti-1..ti+2, y face tj+1 from tj-1..tj+2
                    const double* c = cur + v * CP + (tj + RO) * cw + ti + NG;
                    SCHK(c - cw);
                    SCHK(c + 2 * cw);
                    face_states<RECON>(c[-1], c[0], c[1], c[2], xl[v], xr[v]);
                    face_states<RECON>(c[-cw], c[0], c[cw], c[2 * cw], yl[v], yr[v]);
                } else {
                    SCHK(XA + v * fxn + xo);
                    SCHK(XB + v * fxn + xo);
                    SCHK(YA + v * fyn + yo);
                    SCHK(YB + v * fyn + yo);
                    xl[v] = XA[v * fxn + xo];
                    xr[v] = XB[v * fxn + xo];
                    yl[v] = YA[v * fyn + yo];
                    yr[v] = YB[v * fyn + yo];
                }
            }
            if (RECON != 0) {
                const bool nx = !(positive(xl[0]) && positive(xl[NV - 1]) && positive(xr[0]) && positive(xr[NV - 1]));
                const bool ny = !(positive(yl[0]) && positive(yl[NV - 1]) && positive(yr[0]) && positive(yr[NV - 1]));
                if (__any_sync(0xffffffffu, nx || ny)) {
#pragma unroll
                    for (int v = 0; v < NV; v++) {
                        if (nx) {
                            xl[v] = cur[v * CP + (tj + RO) * cw + ti + NG];
                            xr[v] = cur[v * CP + (tj + RO) * cw + ti + 1 + NG];
                        }
                        if (ny) {
                            yl[v] = cur[v * CP + (tj + NG) * cw + ti + NG];
                            yr[v] = cur[v * CP + (tj + 1 + NG) * cw + ti + NG];
                        }
                    }
                }
            }
            face_flux<NV, RS, 0>(xl, xr, shk_at(cur + (tj + RO) * cw + ti + 1 + NG, 1, 1), gamma, gm1i, fx);
            face_flux<NV, RS, 1>(yl, yr, shk_at(cur + (tj + 1 + NG) * cw + ti + NG, cw, 2), gamma, gm1i, fy);
#pragma unroll
            for (int v = 0; v < NV; v++) {
                SCHK(XA + v * fxn + xo);
                SCHK(YA + v * fyn + yo);
                XA[v * fxn + xo] = fx[v];
                YA[v * fyn + yo] = fy[v];
            }
            // round 2
            if (NDIM == 3 && RECON != 0) {
                const bool nz = !(positive(zhi[0]) && positive(zhi[NV - 1]) && positive(zlo[0]) && positive(zlo[NV - 1]));
                if (__any_sync(0xffffffffu, nz) && nz) {
#pragma unroll
                    for (int v = 0; v < NV; v++) {
                        zhi[v] = ring_at(kk, v);
                        zlo[v] = ring_at(kk + 1, v);
                    }
                }
            }
            if (tid < 32) {  // warp 0: boundary face (+ its z faces)
                const bool isy = tid >= 16;
                const int q = tid & 15;
                double bl[NV], br[NV], fb[NV];
                const bool bshk = shk_at(isy ? cur + NG * cw + q + NG : cur + (q + RO) * cw + NG, isy ? cw : 1,
                                         isy ? 2 : 1);
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    if (FC) {  // face 0 of row / column q from cells -2..1
                        const double* c = cur + v * CP + (isy ? NG * cw + q + NG : (q + RO) * cw + NG);
                        const int st = isy ? cw : 1;
                        SCHK(c - (RECON ? 2 : 1) * st);
                        SCHK(c + (RECON ? 1 : 0) * st);
                        face_states<RECON>(c[-2 * st], c[-st], c[0], c[st], bl[v], br[v]);
                    } else {
                        SCHK(isy ? YA + v * fyn + q : XA + v * fxn + q * fxs);
                        SCHK(isy ? YB + v * fyn + q : XB + v * fxn + q * fxs);
                        bl[v] = isy ? YA[v * fyn + q] : XA[v * fxn + q * fxs];
                        br[v] = isy ? YB[v * fyn + q] : XB[v * fxn + q * fxs];
                    }
                }
                if (RECON != 0 && !(positive(bl[0]) && positive(bl[NV - 1]) && positive(br[0]) && positive(br[NV - 1]))) {
#pragma unroll
                    for (int v = 0; v < NV; v++) {
                        bl[v] = isy ? cur[v * CP + (NG - 1) * cw + q + NG] : cur[v * CP + (q + RO) * cw + NG - 1];
                        br[v] = isy ? cur[v * CP + NG * cw + q + NG] : cur[v * CP + (q + RO) * cw + NG];
                    }
                }
                {  // y faces in the x frame
                    const double l1 = bl[1], r1 = br[1];
                    bl[1] = isy ? bl[2] : l1;
                    bl[2] = isy ? l1 : bl[2];
                    br[1] = isy ? br[2] : r1;
                    br[2] = isy ? r1 : br[2];
                }
                if (NDIM == 3) face_flux<NV, RS, 2>(zhi, zlo, zsh, gamma, gm1i, fzhi);
                face_flux<NV, RS, 0>(bl, br, bshk, gamma, gm1i, fb);
                {
                    const double f1 = fb[1];
                    fb[1] = isy ? fb[2] : f1;
                    fb[2] = isy ? f1 : fb[2];
                }
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    SCHK(isy ? YA + v * fyn + q : XA + v * fxn + q * fxs);
                    if (isy) YA[v * fyn + q] = fb[v];
                    else XA[v * fxn + q * fxs] = fb[v];
                }
            } else if (NDIM == 3) {
                face_flux<NV, RS, 2>(zhi, zlo, zsh, gamma, gm1i, fzhi);
            }
            if (NDIM == 3) {
#pragma unroll
                for (int v = 0; v < NV; v++) zhi[v] = zhn[v];
            }
        } else {
            auto regular = [&]() {
                if (live) {
                    xface(tj, ti + 1, fxo);
                    if (NDIM >= 2) yface(ti, tj + 1, fyo);
                    if (NDIM == 3) {
                        zflux(kk, zhi, zlo, zsh, fzhi);
#pragma unroll
                        for (int v = 0; v < NV; v++) zhi[v] = zhn[v];
                    }
                }
            };
            auto boundary = [&]() {
                if (FC && NBX == 16 && NBY == 16) {
                    // warp 0: the 32 block-boundary faces in one pass (y faces in the
                    // x frame with u_x <-> u_y swapped, bitwise identical; see FUSE)
                    if (tid < 32) {
                        const bool isy = tid >= 16;
                        const int q = tid & 15;
                        double bl[NV], br[NV], fb[NV];
                        const bool bshk = shk_at(isy ? cur + NG * cw + q + NG : cur + (q + RO) * cw + NG,
                                                 isy ? cw : 1, isy ? 2 : 1);
#pragma unroll
                        for (int v = 0; v < NV; v++) {
                            const double* c = cur + v * CP + (isy ? NG * cw + q + NG : (q + RO) * cw + NG);
                            const int st = isy ? cw : 1;
                            SCHK(c - (RECON ? 2 : 1) * st);
                            SCHK(c + (RECON ? 1 : 0) * st);
                            face_states<RECON>(c[-2 * st], c[-st], c[0], c[st], bl[v], br[v]);
                        }
                        if (!(positive(bl[0]) && positive(bl[NV - 1]) && positive(br[0]) && positive(br[NV - 1]))) {
#pragma unroll
                            for (int v = 0; v < NV; v++) {
                                bl[v] = isy ? cur[v * CP + (NG - 1) * cw + q + NG] : cur[v * CP + (q + RO) * cw + NG - 1];
                                br[v] = isy ? cur[v * CP + NG * cw + q + NG] : cur[v * CP + (q + RO) * cw + NG];
                            }
                        }
                        {
                            const double l1 = bl[1], r1 = br[1];
                            bl[1] = isy ? bl[2] : l1;
                            bl[2] = isy ? l1 : bl[2];
                            br[1] = isy ? br[2] : r1;
                            br[2] = isy ? r1 : br[2];
                        }
                        face_flux<NV, RS, 0>(bl, br, bshk, gamma, gm1i, fb);
                        {
                            const double f1 = fb[1];
                            fb[1] = isy ? fb[2] : f1;
                            fb[2] = isy ? f1 : fb[2];
                        }
#pragma unroll
                        for (int v = 0; v < NV; v++) {
                            SCHK(isy ? YA + v * fyn + q : XA + (ONEBAR ? v * nb1 + q : v * fxn + q * fxs));
                            if (isy) YA[v * fyn + q] = fb[v];
                            else XA[ONEBAR ? v * nb1 + q : v * fxn + q * fxs] = fb[v];
                        }
                    }
                } else {
                    for (int q = tid; q < nbf; q += blockDim.x) {
                        double scr[NV];
                        if (q < nb1) xface(q, 0, scr);
                        else yface(q - nb1, 0, scr);
                    }
                }
            };
            // measured: z solve first -1.3 %, boundary pass first -1.6 %
            regular();
            boundary();
        }
        __syncthreads();
        // ---------------------------------------------------------------- S4
        if (live) {
            const long long idx = cidx;
            double un[NV], Lv[NV];
#pragma unroll
            for (int v = 0; v < NV; v++) {
                if (!OWNF) SCHK(XA + v * fxn + tj * fxs + ti + 1);
                SCHK(ONEBAR ? XA + v * nb1 + tj : XA + v * fxn + tj * fxs + ti);
                const double fxp = OWNF ? fxo[v] : XA[v * fxn + tj * fxs + ti + 1];
                double fxm;
                if (ONEBAR) {  // left face: the left lane's own face, or the boundary face 0
                    const double nbr = __shfl_up_sync(0xffffffffu, fxp, 1);
                    fxm = ti == 0 ? XA[v * nb1 + tj] : nbr;
                } else {
                    fxm = XA[v * fxn + tj * fxs + ti];
                }
                const double dfx = (fxp - fxm) * g.rdx[0];
                if (NDIM == 1) {
                    Lv[v] = -dfx;
                } else {
                    SCHK(YA + v * fyn + (tj + 1) * nb0 + ti);
                    SCHK(YA + v * fyn + tj * nb0 + ti);
                    const double fyp = OWNF ? fyo[v] : YA[v * fyn + (tj + 1) * nb0 + ti];
                    const double dfy = (fyp - YA[v * fyn + tj * nb0 + ti]) * g.rdx[1];
                    if (NDIM == 2) Lv[v] = -(dfx + dfy);
                    else Lv[v] = -(dfx + dfy) - (fzhi[v] - fzlo[v]) * g.rdx[2];
                }
            }
            if (L2PF) {
#pragma unroll
                for (int v = 0; v < NV; v++) {
                    GCHK(up + v * vs + cidx);
                    if (a != 0.0) GCHK(A.un + v * vs + cidx);
                    u0v[v] = __ldg(up + v * vs + cidx);
                    unv[v] = a != 0.0 ? __ldg(A.un + v * vs + cidx) : 0.0;
                }
            }
            if (g.has_grav) {  // grvAccel source at U^(s-1) (CTA-uniform branch)
                double grho = 0.0, gmg = 0.0;
#pragma unroll
                for (int v = 0; v < NV; v++) Lv[v] += grav_src<NV>(g, v, u0v[v], grho, gmg);
            }
#pragma unroll
            for (int v = 0; v < NV; v++) {
                const double u0 = u0v[v];
                const double unn = unv[v];
                const double uo = fma(bco, fma(dt, Lv[v], u0), a * unn);
                GCHK(A.uout + v * vs + idx);
                A.uout[v * vs + idx] = uo;
                un[v] = uo;
                fzlo[v] = fzhi[v];
            }
            if (A.last) {
                double w[NV];
                ok &= cons_to_prim<NV>(un, w, gm1);
                cflmin = fmin(cflmin, cfl_term<NV>(g, w));
            }
        }
    }
    if (!ok) flag_nonphysical(A.sc);
    if (A.last) {
        __syncthreads();
        block_min_to(cflmin, smem, &A.sc->acc);  // the planes are dead here
    }
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int NDIM, int RECON, int RS, int NBX, int NBY, int NBZ>
cudaError_t launch_t(const StageArgs& a, cudaStream_t s) {
    const size_t smem = stage_smem_bytes(a.g, RECON);
    auto k = stage_kernel<NDIM, RECON, RS, NBX, NBY, NBZ>;
    cudaError_t e = set_smem(k, smem);
    if (e != cudaSuccess) return e;
    const long long nblk = a.nblk > 0 ? a.nblk : (long long)a.g.bn[0] * a.g.bn[1] * a.g.bn[2];
    k<<<(unsigned)nblk, stage_block_threads(a.g, RECON), smem, s>>>(a);
    return cudaGetLastError();
}

// Production shapes (16x16 planes: 16^2 and 16^3 blocks) get compile-time block
// extents; any other shape runs the runtime-extent kernel.
bool fast_shape(const Geo& g) {
    return g.ndim >= 2 && g.nb[0] == 16 && g.nb[1] == 16 && (g.ndim == 2 || g.nb[2] == 16);
}

template <int NDIM, int RECON, int RS>
cudaError_t launch_shape(const StageArgs& a, cudaStream_t s) {
    if (NDIM >= 2 && fast_shape(a.g)) return launch_t<NDIM, RECON, RS, 16, 16, NDIM == 3 ? 16 : 1>(a, s);
    return launch_t<NDIM, RECON, RS, 0, 0, 0>(a, s);
}

template <int NDIM, int RECON>
cudaError_t launch_r(const StageArgs& a, int riemann, cudaStream_t s) {
    if (riemann == 0) return launch_shape<NDIM, RECON, 0>(a, s);
    if (riemann == 1 || RECON == 0) return launch_shape<NDIM, RECON, 1>(a, s);  // hybrid needs recon >= PLM
    return launch_shape<NDIM, RECON, 2>(a, s);
}

template <int NDIM>
cudaError_t launch_d(const StageArgs& a, int recon, int riemann, cudaStream_t s) {
    if (recon == 0) return launch_r<NDIM, 0>(a, riemann, s);
    if (recon == 1) return launch_r<NDIM, 1>(a, riemann, s);
    if (recon == 3) return launch_r<NDIM, 3>(a, riemann, s);
    if (recon == 4) return launch_r<NDIM, 4>(a, riemann, s);
    return launch_r<NDIM, 2>(a, riemann, s);
}

}  // namespace

int stage_block_threads(const Geo& g, int /*recon*/) {
    const int P = g.nb[0] * (g.ndim >= 2 ? g.nb[1] : 1);
    return ((P + 31) / 32) * 32;
}

size_t stage_smem_bytes(const Geo& g, int recon) {
    const int NG = (recon == 2 || recon == 4) ? 3 : ((recon == 1 || recon == 3) ? 2 : 1);
    const int NV = g.ndim + 2;
    const int nb0 = g.nb[0], nb1 = g.ndim >= 2 ? g.nb[1] : 1;
    const size_t P = (size_t)nb0 * nb1;
    const size_t slots = 2 * NG - 1 > 2 ? 2 * NG - 1 : 2;
    const size_t cw = nb0 + 2 * NG, ch = g.ndim >= 2 ? nb1 + 2 * NG : 1;
    const bool pad = policy_pad_ring(g.ndim, recon);
    const size_t ring = g.ndim == 3 ? slots * NV * (pad ? cw * ch : P) : 0;
    const size_t cur = pad ? 0 : NV * cw * ch;
    const bool k16 = fast_shape(g);
    const size_t nst = k16 && policy_face_centric(g.ndim, recon, 16, 16) ? 1 : 2;  // FC: fluxes only
    const bool onebar = k16 && policy_one_barrier(g.ndim, recon, 16, 16);
    const size_t fx = onebar ? 2 * NV * (size_t)nb1 : nst * NV * (size_t)(nb0 + 1) * nb1;
    const size_t fy = g.ndim >= 2 ? (onebar ? 2 : nst) * NV * (size_t)nb0 * (nb1 + 1) : 0;
    const size_t nh = 2 * (size_t)NG * (nb0 + nb1);
    const size_t hsm = k16 && g.ndim == 3 && nst == 1 ? NV * nh : 0;  // HSM staging
    return (ring + cur + fx + fy + hsm) * sizeof(double);
}

cudaError_t launch_stage(const StageArgs& a, int recon, int riemann, cudaStream_t s) {
    if (a.g.ndim == 1) return launch_d<1>(a, recon, riemann, s);
    if (a.g.ndim == 2) return launch_d<2>(a, recon, riemann, s);
    return launch_d<3>(a, recon, riemann, s);
}

}  // namespace spark
