// spark_internal.h — types shared by the host layer (spark_api.cpp) and the
// CUDA kernels (spark_kernels.cu).  Not part of the public ABI (include/spark.h).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace spark {

constexpr int kMaxThreads = 1024;

// Device-resident scalars of one context (one per rank).
// The per-step collective reduces acc and bad together (two u64, ncclMin /
// group min): every rank then sees the same CFL minimum AND the same first
// failing step, so all ranks roll back (or report) together.
constexpr unsigned long long kNoBad = ~0ull;
struct DevScalars {
    double dt;                    // dt of the step in flight
    double t;                     // time at the end of the step in flight
    double t_prev;                // time at its start (rollback)
    unsigned long long acc;       // CFL min accumulator: bits of a positive double
    unsigned long long bad;       // first step (value of `steps`) that produced a non-physical
                                  // state on any rank (kNoBad: none); adjacent to acc
    unsigned long long acc_prev;  // value consumed by the step in flight (rollback)
    int status;                   // bit 0: non-physical state seen on this rank
    int active;                   // 0 once t >= t_end or after a failure: stages copy U unchanged
    long long steps;              // completed steps
    double pad[8];
};

// Geometry of this rank's sub-box, in cells.  Loaded by value into kernels.
struct Geo {
    int ndim, nvar, ng;           // ng = guard depth of the halo slabs
    int nb[3];                    // cells per block
    int bn[3];                    // blocks of the sub-box per dim
    int cn[3];                    // cells of the sub-box per dim (nb * bn)
    int gN[3];                    // global cells per dim
    int off[3];                   // global cell index of the sub-box origin
    int bc[3][2];                 // physical boundary conditions
    int halo[3][2];               // 1: face neighbour is another rank (slab buffer)
    long long ncell;              // cells of the sub-box
    long long cpb;                // cells per block
    // State layout in HBM: block-interleaved U[b][v][k][j][i],
    // element (v, block b, cell c of the block) at b*bs + v*vs + c with
    // vs = cpb, bs = nvar*cpb: one block is one contiguous chunk, so every
    // variable of a cell is a compile-time offset from one pointer in KB1.
    // The ABI's canonical layout U[v][b][k][j][i] is converted at set/get.
    long long vs;                 // stride between variables
    long long bs;                 // stride between blocks
    long long slab[3];            // cells of one slab of dim d (ng * other extents)
    double dx[3], rdx[3];
    double gamma, cfl;
    double grav[3];               // grvAccel source (reading R20)
    int has_grav;                 // any grav[d] != 0
    double shock_thresh;          // shockDet threshold (riemann 2, reading R21)
};

struct StageArgs {
    Geo g;
    const double* uprev;
    const double* un;             // may be null when a == 0
    double* uout;
    const double* halo[3][2];     // received slabs [v][slab] (null if no peer)
    double a, b;
    DevScalars* sc;
    const double* dt_ptr;         // device dt (sc->dt) or null -> dt_value
    double dt_value;
    int last;                     // 1: fuse the CFL-min epilogue
    int honor_active;             // 1: copy-through when sc->active == 0
    int part;                     // 0 all blocks; 1 blocks touching no exchanged rank face
                                  // ("interior", run while halos travel); 2 the others
    int blk0, nblk;               // block range of the launch (nblk 0: all blocks)
};

// Telescoping through HBM tiles (spark_telescope_tile.cu): G = S*NGK guard
// layers per block tile, pn = nb + 2G along the used dims.
struct TileGeo {
    Geo g;
    int G, S, ngk, recon;
    int pn[3];
    long long np;                 // cells per tile
    long long Fo[3], NF;          // face blocks per tile: offsets, total
};
// the 26 received shell regions of a rank, by direction (c0+1) + 3(c1+1) + 9(c2+1)
struct ShellPtrs {
    const double* p[27];
};

constexpr int kMaxGroup = 64;
struct AccPtrs {
    unsigned long long* p[kMaxGroup];
};

// ---- launchers (spark_kernels.cu) -------------------------------------------
// All return cudaGetLastError() after the launch.
cudaError_t launch_stage(const StageArgs& a, int recon, int riemann, cudaStream_t s);
cudaError_t launch_cfl_min(const Geo& g, const double* u, DevScalars* sc, cudaStream_t s);
cudaError_t launch_step_begin(DevScalars* sc, double dt_fixed, double t_end, double cfl, cudaStream_t s);
cudaError_t launch_prim_to_cons(const Geo& g, const double* w, double* u, cudaStream_t s);
// canonical U[v][b][c] <-> internal U[b][v][c] (to_internal = 1: canonical -> internal)
cudaError_t launch_relayout(const Geo& g, const double* src, double* dst, int to_internal, cudaStream_t s);
// blocks [b0, b1) only (chunked host <-> device transfers, spark_step_host)
cudaError_t launch_relayout_range(const Geo& g, const double* src, double* dst, int to_internal, long long b0,
                                  long long b1, cudaStream_t s);
cudaError_t launch_acc_reset(DevScalars* sc, cudaStream_t s);
cudaError_t launch_pack(const Geo& g, const double* u, int dim, int side, double* slab, cudaStream_t s);
cudaError_t launch_fill_padded(const Geo& g, const double* u, const double* const halo[3][2], double* padded,
                               cudaStream_t s);
cudaError_t launch_scalars_reset(DevScalars* sc, cudaStream_t s);
cudaError_t launch_set_time(DevScalars* sc, double t, long long steps, cudaStream_t s);
cudaError_t launch_group_min(const AccPtrs& p, int n, cudaStream_t s);
cudaError_t launch_selftest_riemann(int riemann, int ndim, int dir, double gamma, int64_t n, const double* wl,
                                    const double* wr, double* f);
cudaError_t launch_axpy(int variant, int64_t n, double a, const double* x, double* y, int sms, cudaStream_t s);
size_t stage_smem_bytes(const Geo& g, int recon);
size_t telescope_smem_bytes(const Geo& g, int recon, int S);
cudaError_t launch_telescope(const StageArgs& a, int recon, int riemann, int S, cudaStream_t s);
int stage_block_threads(const Geo& g, int recon);
long long tile_region_cells(const TileGeo& t, int dir);
cudaError_t launch_tile_pack(const TileGeo& t, const double* u, int dir, double* buf, cudaStream_t s);
cudaError_t launch_tile_gather(const TileGeo& t, const double* u, const ShellPtrs& sh, double* T0, cudaStream_t s);
cudaError_t launch_tile_stage(const TileGeo& t, int riemann, const double* Tprev, const double* T0, double* W,
                              double* F, double* Tout, double* uout, double a, double b, int s, int last,
                              DevScalars* sc, cudaStream_t st);

}  // namespace spark
