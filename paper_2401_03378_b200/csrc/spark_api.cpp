// spark_api.cpp — host layer and C ABI of libspark (include/spark.h).
//
// Owns: configuration checks, the rank decomposition (process grid over the
// global block grid, "blocks distributed variably among
// computational resources"), the arena sub-allocation, the SSP-RK stage loop of
// lst:spark-nontelescoping (guard-cell fill before every stage,
// then all blocks), buffer rotation, the halo exchange (NCCL grouped
// send/recv over NVLink, or device copies between virtual ranks) and the dt
// all-reduce (ncclMin on the ordered bits of the CFL minimum).
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/spark.h"
#include "spark_internal.h"

namespace {

struct Error : std::runtime_error {
    spark_status st;
    Error(spark_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

#define CU(call)                                                                                        \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            throw Error(SPARK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));            \
    } while (0)

#define NC(call)                                                                                        \
    do {                                                                                                \
        ncclResult_t r_ = (call);                                                                       \
        if (r_ != ncclSuccess)                                                                          \
            throw Error(SPARK_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_));            \
    } while (0)

// NVTX ranges (host-side, around the enqueue of each phase; visible in
// Nsight Systems / ncu --nvtx): step, stage s, halo exchange, dt all-reduce
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

int stencil_ng(int recon) {
    if (recon == SPARK_RECON_WENO5 || recon == SPARK_RECON_WENO5Z) return 3;
    if (recon == SPARK_RECON_PLM || recon == SPARK_RECON_PLM_MC) return 2;
    return 1;
}

std::string check(const spark_config* c, int nranks) {
    if (!c) return "null config";
    if (c->ndim < 1 || c->ndim > 3) return "ndim must be 1..3";
    if (nranks < 1) return "nranks must be >= 1";
    if (c->recon < 0 || c->recon > 4) return "unknown recon";
    for (int d = 0; d < 3; d++)
        if (!std::isfinite(c->grav[d]) || (d >= c->ndim && c->grav[d] != 0.0))
            return "grav must be finite and zero along unused dims";
    if (c->riemann < 0 || c->riemann > 2) return "unknown riemann";
    if (c->riemann == SPARK_RIEMANN_HYBRID) {
        // shockDet reads the cells i-1..i+2 of a face (reading R21)
        if (stencil_ng(c->recon) < 2) return "the hybrid Riemann solver (shockDet) needs recon PLM, PLM-MC or WENO5";
        if (!(c->shock_thresh > 0.0) || !std::isfinite(c->shock_thresh)) return "shock_thresh must be finite and > 0";
    }
    if (c->rk_stages != 2 && c->rk_stages != 3) return "rk_stages must be 2 or 3";
    if (!(c->gamma > 1.0)) return "gamma must be > 1";
    if (!(c->cfl > 0.0)) return "cfl must be > 0";
    if (c->ng < stencil_ng(c->recon)) return "ng too small for the reconstruction";
    for (int d = 0; d < 3; d++) {
        if (c->nb[d] < 1 || c->nblk[d] < 1) return "nb and nblk must be >= 1";
        if (d >= c->ndim && (c->nb[d] != 1 || c->nblk[d] != 1)) return "unused dims need nb = nblk = 1";
        if (d < c->ndim && c->nb[d] < c->ng) return "nb must be >= ng";
        if (d < c->ndim && !(c->hi[d] > c->lo[d])) return "hi must exceed lo";
        for (int s = 0; s < 2; s++)
            if (c->bc[d][s] < 0 || c->bc[d][s] > 2) return "unknown boundary condition";
        if (d < c->ndim && (c->bc[d][0] == SPARK_BC_PERIODIC) != (c->bc[d][1] == SPARK_BC_PERIODIC))
            return "periodic boundaries must be periodic on both sides";
    }
    const long long plane = (long long)c->nb[0] * (c->ndim >= 2 ? c->nb[1] : 1);
    if (plane > 256) return "nb[0]*nb[1] must be <= 256 (one thread per column)";
    const long long cells = (long long)c->nb[0] * c->nb[1] * c->nb[2] * c->nblk[0] * c->nblk[1] * c->nblk[2];
    if (cells > (1LL << 40)) return "grid too large";
    for (int d = 0; d < 3; d++)
        if ((long long)c->nb[d] * c->nblk[d] > INT_MAX / 2) return "grid too large";
    return "";
}

// Process grid: factorisation of nranks dividing the block grid, minimising
// the exchanged surface; ties prefer splitting the slowest-varying dim.
bool rank_grid(const spark_config* c, int nranks, int pg[3]) {
    long long best = -1;
    bool found = false;
    for (int pz = 1; pz <= nranks; pz++) {
        if (nranks % pz) continue;
        for (int py = 1; py <= nranks / pz; py++) {
            if ((nranks / pz) % py) continue;
            const int px = nranks / pz / py;
            const int p[3] = {px, py, pz};
            bool ok = true;
            for (int d = 0; d < 3; d++)
                if (c->nblk[d] % p[d] || (d >= c->ndim && p[d] != 1)) ok = false;
            if (!ok) continue;
            long long n[3];
            for (int d = 0; d < 3; d++) n[d] = (long long)c->nb[d] * c->nblk[d] / p[d];
            long long surf = 0;
            for (int d = 0; d < c->ndim; d++)
                if (p[d] > 1 || c->bc[d][0] == SPARK_BC_PERIODIC) {
                    long long f = 1;
                    for (int e = 0; e < c->ndim; e++)
                        if (e != d) f *= n[e];
                    if (p[d] > 1) surf += 2 * f;
                }
            if (!found || surf < best || (surf == best && pz > pg[2]) ||
                (surf == best && pz == pg[2] && py > pg[1])) {
                best = surf;
                pg[0] = px;
                pg[1] = py;
                pg[2] = pz;
                found = true;
            }
        }
    }
    return found;
}

struct Plan {
    int pg[3], pc[3], box_lo[3], box_n[3];
    int peer[3][2];  // -1: no peer (physical boundary or periodic self-wrap)
    spark::Geo geo;
};

// self_exchange: periodic dims owned entirely by this rank are still exchanged
// through the halo path (peer = self) — used with a 1-rank NCCL communicator to
// exercise pack + NCCL send/recv + slab reads on a single GPU.
Plan make_plan(const spark_config* c, int rank, int nranks, bool self_exchange = false) {
    std::string m = check(c, nranks);
    if (!m.empty()) throw Error(SPARK_ERR_ARG, m);
    if (rank < 0 || rank >= nranks) throw Error(SPARK_ERR_ARG, "rank out of range");
    Plan p{};
    if (!rank_grid(c, nranks, p.pg)) throw Error(SPARK_ERR_ARG, "block grid not divisible among ranks");
    p.pc[0] = rank % p.pg[0];
    p.pc[1] = (rank / p.pg[0]) % p.pg[1];
    p.pc[2] = rank / (p.pg[0] * p.pg[1]);
    spark::Geo& g = p.geo;
    g.ndim = c->ndim;
    g.nvar = c->ndim + 2;
    g.ng = c->ng;
    g.cpb = 1;
    g.ncell = 1;
    for (int d = 0; d < 3; d++) {
        p.box_n[d] = c->nblk[d] / p.pg[d];
        p.box_lo[d] = p.pc[d] * p.box_n[d];
        g.nb[d] = c->nb[d];
        g.bn[d] = p.box_n[d];
        g.cn[d] = c->nb[d] * p.box_n[d];
        g.gN[d] = c->nb[d] * c->nblk[d];
        g.off[d] = p.box_lo[d] * c->nb[d];
        g.cpb *= c->nb[d];
        g.ncell *= g.cn[d];
        g.dx[d] = (c->hi[d] - c->lo[d]) / ((double)c->nblk[d] * (double)c->nb[d]);
        g.rdx[d] = 1.0 / g.dx[d];
        for (int s = 0; s < 2; s++) {
            g.bc[d][s] = c->bc[d][s];
            p.peer[d][s] = -1;
            g.halo[d][s] = 0;
        }
    }
    g.vs = g.cpb;
    g.bs = (long long)g.nvar * g.cpb;
    for (int d = 0; d < c->ndim; d++) {
        for (int s = 0; s < 2; s++) {
            int q[3] = {p.pc[0], p.pc[1], p.pc[2]};
            q[d] += s ? 1 : -1;
            if (q[d] < 0 || q[d] >= p.pg[d]) {
                if (c->bc[d][s] != SPARK_BC_PERIODIC) continue;  // physical boundary: local map
                if (p.pg[d] == 1 && !self_exchange) continue;     // periodic self-wrap: local map
                q[d] = (q[d] + p.pg[d]) % p.pg[d];
            }
            p.peer[d][s] = q[0] + p.pg[0] * (q[1] + p.pg[1] * q[2]);
            g.halo[d][s] = 1;
        }
    }
    for (int d = 0; d < 3; d++) {
        long long s = g.ng;
        for (int e = 0; e < 3; e++)
            if (e != d) s *= g.cn[e];
        g.slab[d] = d < c->ndim ? s : 0;
    }
    // kernels keep variable strides (ncell, slab sizes) in 32-bit registers; a
    // sub-box this large would need > 250 GB of state anyway
    if (g.ncell >= (1LL << 31)) throw Error(SPARK_ERR_ARG, "sub-box exceeds 2^31 cells (split over more ranks)");
    g.gamma = c->gamma;
    g.cfl = c->cfl;
    g.shock_thresh = c->riemann == SPARK_RIEMANN_HYBRID ? c->shock_thresh : 0.0;
    g.has_grav = 0;
    for (int d = 0; d < 3; d++) {
        g.grav[d] = c->grav[d];
        if (c->grav[d] != 0.0) g.has_grav = 1;
    }
    return p;
}

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

size_t arena_bytes(const Plan& p) {
    const size_t state = align_up(sizeof(double) * p.geo.nvar * (size_t)p.geo.ncell);
    size_t halo = 0;
    for (int d = 0; d < 3; d++)
        for (int s = 0; s < 2; s++)
            if (p.peer[d][s] >= 0) halo += 2 * align_up(sizeof(double) * p.geo.nvar * (size_t)p.geo.slab[d]);
    return align_up(sizeof(spark::DevScalars)) + 3 * state + halo;
}

struct LocalGroup {
    std::vector<spark_ctx*> members;
};

}  // namespace

struct spark_ctx {
    spark_config cfg{};
    int rank = 0, nranks = 1, device = 0;
    cudaStream_t stream = nullptr;
    Plan plan{};
    double* U[3] = {nullptr, nullptr, nullptr};
    int n_idx = 0;
    double* send[3][2] = {};
    double* recv[3][2] = {};
    spark::DevScalars* sc = nullptr;
    ncclComm_t comm = nullptr;
    cudaStream_t comm_stream = nullptr;        // NCCL halo exchange overlaps interior blocks
    cudaEvent_t ev_packed = nullptr, ev_recv = nullptr;
    std::shared_ptr<LocalGroup> group;
    bool have_state = false;
    std::string err;
    // profiling
    bool prof = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    size_t ev_used = 0;
    int64_t stage_launches = 0, total_launches = 0;
    // CUDA graphs of 3 steps (the buffer-rotation period) for spark_run, one per
    // starting buffer index; re-captured when dt / t_end change
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        double dt = 0.0, t_end = 0.0;
    } graphs[3];
    double prof_ms = 0.0;
    // telescoping through HBM tiles (3-D / multi-rank): caller-owned scratch
    struct Tiles {
        spark::TileGeo tg{};
        double *T0 = nullptr, *Ta = nullptr, *Tb = nullptr, *W = nullptr, *F = nullptr;
        double* send[27] = {};
        double* recv[27] = {};
        int peer[27];
        bool ready = false;
    } tiles;
    // spark_step_host: copy streams and per-chunk events (created on first use)
    cudaStream_t h2d = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev_h2d, ev_out, ev_d2h;
};

namespace {

spark_status fail(spark_ctx* ctx, const Error& e) {
    if (ctx) ctx->err = e.what();
    return e.st;
}

template <typename F>
spark_status guard(spark_ctx* ctx, F&& f) {
    try {
        if (ctx) ctx->err.clear();
        f();
        return SPARK_OK;
    } catch (const Error& e) {
        return fail(ctx, e);
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return SPARK_ERR_ARG;
    } catch (...) {
        if (ctx) ctx->err = "unknown error";
        return SPARK_ERR_ARG;
    }
}

void set_device(spark_ctx* c) { CU(cudaSetDevice(c->device)); }

void launched(spark_ctx* c, cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(SPARK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    c->total_launches++;
}

void carve(spark_ctx* c, void* arena, size_t bytes) {
    const size_t need = arena_bytes(c->plan);
    if (!arena) throw Error(SPARK_ERR_ARG, "null arena");
    if (bytes < need) throw Error(SPARK_ERR_OOM, "arena smaller than spark_required_bytes");
    if (reinterpret_cast<uintptr_t>(arena) % 16) throw Error(SPARK_ERR_ARG, "arena must be 16-byte aligned");
    char* p = static_cast<char*>(arena);
    const spark::Geo& g = c->plan.geo;
    c->sc = reinterpret_cast<spark::DevScalars*>(p);
    p += align_up(sizeof(spark::DevScalars));
    const size_t state = align_up(sizeof(double) * g.nvar * (size_t)g.ncell);
    for (int i = 0; i < 3; i++) {
        c->U[i] = reinterpret_cast<double*>(p);
        p += state;
    }
    for (int d = 0; d < 3; d++)
        for (int s = 0; s < 2; s++)
            if (c->plan.peer[d][s] >= 0) {
                const size_t sb = align_up(sizeof(double) * g.nvar * (size_t)g.slab[d]);
                c->send[d][s] = reinterpret_cast<double*>(p);
                p += sb;
                c->recv[d][s] = reinterpret_cast<double*>(p);
                p += sb;
            }
}

spark_ctx* make_ctx(const spark_config* cfg, int rank, int nranks, int device, void* stream, void* arena,
                    size_t bytes, bool self_exchange = false) {
    auto c = std::make_unique<spark_ctx>();
    c->cfg = *cfg;
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    c->plan = make_plan(cfg, rank, nranks, self_exchange);
    carve(c.get(), arena, bytes);
    set_device(c.get());
    launched(c.get(), spark::launch_scalars_reset(c->sc, c->stream), "scalars reset");
    return c.release();
}

// -------------------------------------------------------------- exchange
void pack_all(spark_ctx* c, const double* u, cudaStream_t st = nullptr) {
    for (int d = 0; d < 3; d++)
        for (int s = 0; s < 2; s++)
            if (c->plan.peer[d][s] >= 0)
                launched(c, spark::launch_pack(c->plan.geo, u, d, s, c->send[d][s], st ? st : c->stream), "pack");
}

// NCCL grouped send/recv.  Per dim: [send high slab -> high peer, recv low
// halo <- low peer, send low slab -> low peer, recv high halo <- high peer];
// posting in the same order on every rank matches messages between the same
// pair of ranks (P_d = 2 periodic: both faces have the same peer).
void exchange_nccl(spark_ctx* c, cudaStream_t st) {
    const spark::Geo& g = c->plan.geo;
    NC(ncclGroupStart());
    for (int d = 0; d < 3; d++) {
        const size_t n = (size_t)g.nvar * g.slab[d];
        if (c->plan.peer[d][1] >= 0) NC(ncclSend(c->send[d][1], n, ncclFloat64, c->plan.peer[d][1], c->comm, st));
        if (c->plan.peer[d][0] >= 0) NC(ncclRecv(c->recv[d][0], n, ncclFloat64, c->plan.peer[d][0], c->comm, st));
        if (c->plan.peer[d][0] >= 0) NC(ncclSend(c->send[d][0], n, ncclFloat64, c->plan.peer[d][0], c->comm, st));
        if (c->plan.peer[d][1] >= 0) NC(ncclRecv(c->recv[d][1], n, ncclFloat64, c->plan.peer[d][1], c->comm, st));
    }
    NC(ncclGroupEnd());
}

// Virtual ranks: recv(d, s) of rank r <- send(d, 1-s) of its peer.
void exchange_local(const std::vector<spark_ctx*>& m) {
    for (spark_ctx* c : m) {
        const spark::Geo& g = c->plan.geo;
        for (int d = 0; d < 3; d++)
            for (int s = 0; s < 2; s++) {
                const int peer = c->plan.peer[d][s];
                if (peer < 0) continue;
                const size_t bytes = sizeof(double) * g.nvar * (size_t)g.slab[d];
                CU(cudaMemcpyAsync(c->recv[d][s], m[peer]->send[d][1 - s], bytes, cudaMemcpyDeviceToDevice,
                                   c->stream));
            }
    }
}

// One collective per step carries the CFL minimum AND the first failing step
// (u64 pair, element-wise min), so the error decision is global: every rank
// sees the same `bad` and rolls back (or reports) together.
static_assert(offsetof(spark::DevScalars, bad) == offsetof(spark::DevScalars, acc) + 8, "acc/bad pair");
void allreduce_acc(spark_ctx* c) {
    Nvtx r("dt all-reduce (CFL min + failure word)");
    if (c->comm)
        NC(ncclAllReduce(&c->sc->acc, &c->sc->acc, 2, ncclUint64, ncclMin, c->comm, c->stream));
}

// Local group: every member's acc <- min over members (tiny host-side launch
// of a device copy chain: gather to rank 0's buffer, min there, scatter).
void group_min(const std::vector<spark_ctx*>& m);

// a profiling event pair of c (created on first use)
std::pair<cudaEvent_t, cudaEvent_t> prof_events(spark_ctx* c) {
    if (c->ev_used == c->ev.size()) {
        cudaEvent_t x, y;
        CU(cudaEventCreate(&x));
        CU(cudaEventCreate(&y));
        c->ev.emplace_back(x, y);
    }
    return c->ev[c->ev_used++];
}

// part: 0 all blocks, 1 interior, 2 rank-boundary blocks; st: the stream
// (default the context's); timed: bracket the launch with profiling events
void stage_launch(spark_ctx* c, const double* prev, const double* un, double a, double b, double* out,
                  bool last, const double* dt_ptr, double dt_value, bool honor_active, int part = 0,
                  cudaStream_t st = nullptr, bool timed = true, int blk0 = 0, int nblk = 0) {
    if (!st) st = c->stream;
    spark::StageArgs A{};
    A.g = c->plan.geo;
    A.uprev = prev;
    A.un = un;
    A.uout = out;
    for (int d = 0; d < 3; d++)
        for (int s = 0; s < 2; s++) A.halo[d][s] = c->recv[d][s];
    A.a = a;
    A.b = b;
    A.sc = c->sc;
    A.dt_ptr = dt_ptr;
    A.dt_value = dt_value;
    A.last = last ? 1 : 0;
    A.honor_active = honor_active ? 1 : 0;
    A.part = part;
    A.blk0 = blk0;
    A.nblk = nblk;
    const bool ev = c->prof && timed;
    std::pair<cudaEvent_t, cudaEvent_t> e{};
    if (ev) {
        e = prof_events(c);
        CU(cudaEventRecord(e.first, st));
    }
    launched(c, spark::launch_stage(A, c->cfg.recon, c->cfg.riemann, st), "stage kernel");
    if (part != 2) c->stage_launches++;  // a split stage (interior + boundary) counts once
    if (ev) CU(cudaEventRecord(e.second, st));
}

void rk_coeffs(int S, int s, double* a, double* b) {
    if (s == 1) {
        *a = 0.0;
        *b = 1.0;
    } else if (S == 2) {
        *a = 0.5;
        *b = 0.5;
    } else if (s == 2) {
        *a = 0.75;
        *b = 0.25;
    } else {
        *a = 1.0 / 3.0;
        *b = 2.0 / 3.0;
    }
}

// Buffer schedule: stage s reads prev, writes out; returns the new U^n index.
// RK2: n->x, (x,n)->y, U^{n+1}=y.  RK3: n->x, (x,n)->y, (y,n)->x, U^{n+1}=x.
int stage_buffers(int S, int n, int s, int* prev, int* out) {
    const int x = (n + 1) % 3, y = (n + 2) % 3;
    if (s == 1) {
        *prev = n;
        *out = x;
    } else if (s == 2) {
        *prev = x;
        *out = y;
    } else {
        *prev = y;
        *out = x;
    }
    return S == 2 ? y : x;
}

spark::DevScalars read_scalars(spark_ctx* c) {
    CU(cudaStreamSynchronize(c->stream));
    spark::DevScalars h;
    CU(cudaMemcpy(&h, c->sc, sizeof(h), cudaMemcpyDeviceToHost));
    return h;
}

// Whether the step just executed (h read after it) is the one that failed on
// some rank: only then can U^n of that step still be restored.
bool failed_now(const spark::DevScalars& h) {
    return h.bad != spark::kNoBad && h.active && h.bad == (unsigned long long)h.steps;
}

void rollback(spark_ctx* c, spark::DevScalars h, int old_n) {
    c->n_idx = old_n;
    h.t = h.t_prev;
    h.steps -= 1;
    h.acc = h.acc_prev;
    h.bad = spark::kNoBad;
    h.status = 0;
    h.active = 1;
    CU(cudaMemcpy(c->sc, &h, sizeof(h), cudaMemcpyHostToDevice));
}

[[noreturn]] void throw_nonphysical(const spark::DevScalars& h, bool rolled_back) {
    const std::string where = (h.status & 1) ? " (seen on this rank)" : " (seen on another rank)";
    if (rolled_back)
        throw Error(SPARK_ERR_NONPHYSICAL, "non-physical state (rho<=0, p<=0 or NaN) in step " +
                                               std::to_string(h.bad) + where + "; rolled back to U^n");
    throw Error(SPARK_ERR_NONPHYSICAL, "non-physical state (rho<=0, p<=0 or NaN) in step " + std::to_string(h.bad) +
                                           where + "; later steps were frozen, state not rolled back");
}

// Synchronise and check the GLOBAL failure word (reduced over ranks with the
// CFL minimum).  old_n >= 0 and rollback_on_error: roll back when the step just
// executed is the failing one; every rank decides identically.
void sync_and_check(spark_ctx* c, bool rollback_on_error, int old_n) {
    spark::DevScalars h = read_scalars(c);
    if (h.bad == spark::kNoBad) return;
    if (rollback_on_error && old_n >= 0 && failed_now(h)) {
        rollback(c, h, old_n);
        throw_nonphysical(h, true);
    }
    throw_nonphysical(h, false);
}

void do_step(spark_ctx* c, double dt) {
    Nvtx step_range("spark step");
    // single context (1 rank or NCCL); the caller set t_end through do_begin
    const int S = c->cfg.rk_stages;
    int newn = c->n_idx;
    for (int s = 1; s <= S; s++) {
        int pi, po;
        newn = stage_buffers(S, c->n_idx, s, &pi, &po);
        double a, b;
        rk_coeffs(S, s, &a, &b);
        static const char* names[3] = {"stage 1", "stage 2", "stage 3"};
        Nvtx stage_range(names[s - 1]);
        if (c->comm) {
            // pack on the compute stream; the NCCL exchange runs on the comm
            // stream while the interior blocks (no exchanged face) compute;
            // the rank-boundary blocks wait for the received slabs
            // the pack, the exchange and then the rank-boundary blocks all run
            // on the (high-priority) comm stream, concurrently with the
            // interior blocks on the compute stream, which joins after both:
            // no serial pack before the interior launch and no second
            // wave-quantisation gap after it. Measured (256^3, all six faces
            // through NCCL to itself on one GPU, bench.py --self-exchange;
            // 21.36 G zone-updates/s with the faces wrapped in-kernel): PLM
            // 18.37 (pack, interior, boundary serialised) -> 19.24 (boundary
            // concurrent) -> 19.87 (pack concurrent too)
            Nvtx halo_range("halo exchange (pack + NCCL send/recv)");
            CU(cudaEventRecord(c->ev_packed, c->stream));  // U^(s-1) complete (both parts joined)
            CU(cudaStreamWaitEvent(c->comm_stream, c->ev_packed, 0));
            pack_all(c, c->U[pi], c->comm_stream);
            exchange_nccl(c, c->comm_stream);
            std::pair<cudaEvent_t, cudaEvent_t> e{};
            if (c->prof) {  // one interval per split stage: interior start .. join
                e = prof_events(c);
                CU(cudaEventRecord(e.first, c->stream));
            }
            stage_launch(c, c->U[pi], c->U[c->n_idx], a, b, c->U[po], s == S, &c->sc->dt, dt, true, 1,
                         c->stream, false);
            stage_launch(c, c->U[pi], c->U[c->n_idx], a, b, c->U[po], s == S, &c->sc->dt, dt, true, 2,
                         c->comm_stream, false);
            CU(cudaEventRecord(c->ev_recv, c->comm_stream));
            CU(cudaStreamWaitEvent(c->stream, c->ev_recv, 0));
            if (c->prof) CU(cudaEventRecord(e.second, c->stream));
        } else {
            stage_launch(c, c->U[pi], c->U[c->n_idx], a, b, c->U[po], s == S, &c->sc->dt, dt, true);
        }
    }
    allreduce_acc(c);
    c->n_idx = newn;
}

// ------------------------------------------------ telescoping through tiles
spark::TileGeo tile_geo(const spark_config* c, const Plan& p) {
    spark::TileGeo t{};
    t.g = p.geo;
    t.ngk = stencil_ng(c->recon);
    t.S = c->rk_stages;
    t.G = t.S * t.ngk;
    t.recon = c->recon;
    t.np = 1;
    for (int d = 0; d < 3; d++) {
        t.pn[d] = c->nb[d] + (d < c->ndim ? 2 * t.G : 0);
        t.np *= t.pn[d];
    }
    long long off = 0;
    for (int d = 0; d < 3; d++) {
        t.Fo[d] = off;
        if (d < c->ndim) {
            long long f = 1;
            for (int e = 0; e < 3; e++) f *= t.pn[e] + (e == d ? 1 : 0);
            off += f;
        }
    }
    t.NF = off;
    return t;
}

int dir_of(int c0, int c1, int c2) { return (c0 + 1) + 3 * (c1 + 1) + 9 * (c2 + 1); }

// rank in direction (c0, c1, c2) of the process grid, -1 where a component
// crosses a side without a peer (physical boundary / local periodic wrap)
int tile_peer(const Plan& p, int dir) {
    const int c[3] = {dir % 3 - 1, (dir / 3) % 3 - 1, dir / 9 - 1};
    int q[3] = {p.pc[0], p.pc[1], p.pc[2]};
    for (int d = 0; d < 3; d++) {
        if (!c[d]) continue;
        if (p.peer[d][c[d] > 0 ? 1 : 0] < 0) return -1;
        q[d] = ((q[d] + c[d]) % p.pg[d] + p.pg[d]) % p.pg[d];
    }
    return q[0] + p.pg[0] * (q[1] + p.pg[1] * q[2]);
}

size_t tile_scratch_bytes(const spark_config* c, const Plan& p) {
    const spark::TileGeo t = tile_geo(c, p);
    const long long nblk = (long long)p.geo.bn[0] * p.geo.bn[1] * p.geo.bn[2];
    const size_t tile = align_up(sizeof(double) * p.geo.nvar * nblk * t.np);
    size_t b = 4 * tile + align_up(sizeof(double) * p.geo.nvar * nblk * t.NF);
    for (int dir = 0; dir < 27; dir++)
        if (dir != 13 && tile_peer(p, dir) >= 0)
            b += 2 * align_up(sizeof(double) * p.geo.nvar * spark::tile_region_cells(t, dir));
    return b;
}

std::string tile_check(const spark_config* c, const Plan& p) {
    const int G = c->rk_stages * stencil_ng(c->recon);
    for (int d = 0; d < c->ndim; d++) {
        if (G > p.geo.gN[d]) return "telescoped halo deeper than the domain";
        if ((p.peer[d][0] >= 0 || p.peer[d][1] >= 0) && G > p.geo.cn[d])
            return "telescoped halo deeper than a rank's sub-box";
    }
    return "";
}

void tile_attach(spark_ctx* c, void* scratch, size_t bytes) {
    const size_t need = tile_scratch_bytes(&c->cfg, c->plan);
    if (!scratch) throw Error(SPARK_ERR_ARG, "null scratch");
    if (bytes < need) throw Error(SPARK_ERR_OOM, "scratch smaller than spark_telescoping_scratch_bytes");
    if (reinterpret_cast<uintptr_t>(scratch) % 256) throw Error(SPARK_ERR_ARG, "scratch must be 256-byte aligned");
    auto& T = c->tiles;
    T.tg = tile_geo(&c->cfg, c->plan);
    const long long nblk = (long long)c->plan.geo.bn[0] * c->plan.geo.bn[1] * c->plan.geo.bn[2];
    const size_t tile = align_up(sizeof(double) * c->plan.geo.nvar * nblk * T.tg.np);
    char* p = static_cast<char*>(scratch);
    T.T0 = reinterpret_cast<double*>(p), p += tile;
    T.Ta = reinterpret_cast<double*>(p), p += tile;
    T.Tb = reinterpret_cast<double*>(p), p += tile;
    T.W = reinterpret_cast<double*>(p), p += tile;
    T.F = reinterpret_cast<double*>(p), p += align_up(sizeof(double) * c->plan.geo.nvar * nblk * T.tg.NF);
    for (int dir = 0; dir < 27; dir++) {
        T.peer[dir] = dir == 13 ? -1 : tile_peer(c->plan, dir);
        T.send[dir] = T.recv[dir] = nullptr;
        if (T.peer[dir] < 0) continue;
        const size_t rb = align_up(sizeof(double) * c->plan.geo.nvar * spark::tile_region_cells(T.tg, dir));
        T.send[dir] = reinterpret_cast<double*>(p), p += rb;
        T.recv[dir] = reinterpret_cast<double*>(p), p += rb;
    }
    T.ready = true;
}

void tile_pack(spark_ctx* c) {
    auto& T = c->tiles;
    for (int dir = 0; dir < 27; dir++)
        if (T.peer[dir] >= 0)
            launched(c, spark::launch_tile_pack(T.tg, c->U[c->n_idx], dir, T.send[dir], c->stream), "tile pack");
}

// the shell exchange of one rank over NCCL, ONE grouped call per step.  Both
// sides order the messages between a pair of ranks by the receiver's
// direction: my receives by my direction D, my sends by 26 - D (the peer
// stores what I send for D as its direction 26 - D).
// posting order of the shell messages: (is_send, direction)
std::vector<std::pair<bool, int>> tile_ops(const int* peer) {
    std::vector<std::pair<bool, int>> ops;
    for (int k = 0; k < 27; k++) {
        const int rd = k, sd = 26 - k;
        if (peer[rd] >= 0) ops.emplace_back(false, rd);
        if (peer[sd] >= 0) ops.emplace_back(true, sd);
    }
    return ops;
}

void tile_exchange_nccl(spark_ctx* c) {
    auto& T = c->tiles;
    const spark::Geo& g = c->plan.geo;
    NC(ncclGroupStart());
    for (const auto& op : tile_ops(T.peer)) {
        const int dir = op.second;
        const size_t n = (size_t)g.nvar * spark::tile_region_cells(T.tg, dir);
        if (op.first) NC(ncclSend(T.send[dir], n, ncclFloat64, T.peer[dir], c->comm, c->stream));
        else NC(ncclRecv(T.recv[dir], n, ncclFloat64, T.peer[dir], c->comm, c->stream));
    }
    NC(ncclGroupEnd());
}

void tile_exchange_local(const std::vector<spark_ctx*>& m) {
    for (spark_ctx* c : m) {
        auto& T = c->tiles;
        for (int dir = 0; dir < 27; dir++) {
            if (T.peer[dir] < 0) continue;
            spark_ctx* q = m[T.peer[dir]];
            const size_t bytes = sizeof(double) * c->plan.geo.nvar * spark::tile_region_cells(T.tg, dir);
            CU(cudaMemcpyAsync(T.recv[dir], q->tiles.send[26 - dir], bytes, cudaMemcpyDeviceToDevice, c->stream));
        }
    }
}

// gather + the S stages of one rank; writes U^(n+1) into U[(n+1)%3]
void tile_stages(spark_ctx* c) {
    auto& T = c->tiles;
    spark::ShellPtrs sh{};
    for (int dir = 0; dir < 27; dir++) sh.p[dir] = T.recv[dir];
    const int n = c->n_idx, out = (n + 1) % 3;
    cudaEvent_t e1 = nullptr;
    if (c->prof) {  // the gather + stage passes count as the step's stage-kernel time
        if (c->ev_used == c->ev.size()) {
            cudaEvent_t x, y;
            CU(cudaEventCreate(&x));
            CU(cudaEventCreate(&y));
            c->ev.emplace_back(x, y);
        }
        CU(cudaEventRecord(c->ev[c->ev_used].first, c->stream));
        e1 = c->ev[c->ev_used].second;
        c->ev_used++;
    }
    launched(c, spark::launch_tile_gather(T.tg, c->U[n], sh, T.T0, c->stream), "tile gather");
    const int S = c->cfg.rk_stages;
    const double* prev = T.T0;
    for (int s = 1; s <= S; s++) {
        double a, b;
        rk_coeffs(S, s, &a, &b);
        double* tout = (s & 1) ? T.Ta : T.Tb;
        launched(c, spark::launch_tile_stage(T.tg, c->cfg.riemann, prev, T.T0, T.W, T.F, tout, c->U[out], a, b, s,
                                             s == S ? 1 : 0, c->sc, c->stream),
                 "tile stage");
        prev = tout;
    }
    if (e1) CU(cudaEventRecord(e1, c->stream));
    c->stage_launches++;
}

}  // namespace

// ===================================================================== ABI
extern "C" {

int32_t spark_abi_version(void) { return SPARK_ABI_VERSION; }

const char* spark_status_string(spark_status st) {
    switch (st) {
        case SPARK_OK: return "ok";
        case SPARK_ERR_ARG: return "invalid argument";
        case SPARK_ERR_CUDA: return "CUDA error";
        case SPARK_ERR_NCCL: return "NCCL error";
        case SPARK_ERR_OOM: return "arena too small";
        case SPARK_ERR_NONPHYSICAL: return "non-physical state";
        case SPARK_ERR_STATE: return "call out of order";
    }
    return "unknown status";
}

spark_status spark_check_config(const spark_config* cfg, int32_t nranks) {
    std::string m = check(cfg, nranks);
    if (!m.empty()) return SPARK_ERR_ARG;
    int pg[3];
    return rank_grid(cfg, nranks, pg) ? SPARK_OK : SPARK_ERR_ARG;
}

spark_status spark_rank_grid(const spark_config* cfg, int32_t nranks, int32_t pgrid[3]) {
    return guard(nullptr, [&] {
        Plan p = make_plan(cfg, 0, nranks);
        for (int d = 0; d < 3; d++) pgrid[d] = p.pg[d];
    });
}

spark_status spark_rank_box(const spark_config* cfg, int32_t rank, int32_t nranks, int32_t box_lo[3],
                            int32_t box_n[3]) {
    return guard(nullptr, [&] {
        Plan p = make_plan(cfg, rank, nranks);
        for (int d = 0; d < 3; d++) {
            box_lo[d] = p.box_lo[d];
            box_n[d] = p.box_n[d];
        }
    });
}

spark_status spark_halo_plan(const spark_config* cfg, int32_t rank, int32_t nranks, spark_face_plan faces[6],
                             int32_t* nfaces) {
    return guard(nullptr, [&] {
        Plan p = make_plan(cfg, rank, nranks);
        int n = 0;
        for (int d = 0; d < cfg->ndim; d++)
            for (int s = 0; s < 2; s++) {
                faces[n].dim = d;
                faces[n].side = s;
                faces[n].peer = p.peer[d][s];
                faces[n].pad = 0;
                faces[n].cells = p.peer[d][s] >= 0 ? p.geo.slab[d] : 0;
                n++;
            }
        *nfaces = n;
    });
}

spark_status spark_required_bytes(const spark_config* cfg, int32_t rank, int32_t nranks, size_t* bytes) {
    return guard(nullptr, [&] {
        if (!bytes) throw Error(SPARK_ERR_ARG, "null bytes");
        // one rank: room for the self-exchange slabs too (periodic dims, spark_init with an NCCL id)
        *bytes = arena_bytes(make_plan(cfg, rank, nranks, nranks == 1));
    });
}

spark_status spark_nccl_unique_id(uint8_t id[128]) {
    return guard(nullptr, [&] {
        ncclUniqueId u;
        NC(ncclGetUniqueId(&u));
        static_assert(sizeof(u) == 128, "nccl unique id size");
        std::memcpy(id, &u, 128);
    });
}

spark_status spark_init(const spark_config* cfg, int32_t rank, int32_t nranks, const uint8_t* nccl_id,
                        int32_t device, void* cuda_stream, void* arena, size_t arena_bytes_, spark_ctx** out) {
    if (!out) return SPARK_ERR_ARG;
    *out = nullptr;
    spark_ctx* made = nullptr;
    spark_status st = guard(nullptr, [&] {
        if (nranks > 1 && !nccl_id) throw Error(SPARK_ERR_ARG, "nranks > 1 needs an NCCL id");
        // nranks == 1 with an NCCL id: periodic faces go through pack + NCCL
        // send/recv to self (exercises the multi-rank exchange on one GPU)
        const bool self_exchange = nranks == 1 && nccl_id;
        std::unique_ptr<spark_ctx> c(
            make_ctx(cfg, rank, nranks, device, cuda_stream, arena, arena_bytes_, self_exchange));
        if (nccl_id) {
            ncclUniqueId u;
            std::memcpy(&u, nccl_id, 128);
            NC(ncclCommInitRank(&c->comm, nranks, u, rank));
            int lo = 0, hi = 0;  // the exchange and the rank-boundary blocks first
            CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CU(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi));
            CU(cudaEventCreateWithFlags(&c->ev_packed, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&c->ev_recv, cudaEventDisableTiming));
        }
        made = c.release();
    });
    *out = made;
    return st;
}

spark_status spark_init_local_group(const spark_config* cfg, int32_t nranks, int32_t device, void* cuda_stream,
                                    void* const* arenas, size_t arena_bytes_, spark_ctx** outs) {
    if (!outs || !arenas) return SPARK_ERR_ARG;
    std::vector<spark_ctx*> made;
    spark_status st = guard(nullptr, [&] {
        auto grp = std::make_shared<LocalGroup>();
        for (int r = 0; r < nranks; r++) {
            spark_ctx* c = make_ctx(cfg, r, nranks, device, cuda_stream, arenas[r], arena_bytes_);
            c->group = grp;
            made.push_back(c);
            grp->members.push_back(c);
        }
    });
    if (st != SPARK_OK) {
        for (auto* c : made) delete c;
        return st;
    }
    for (int r = 0; r < nranks; r++) outs[r] = made[r];
    return SPARK_OK;
}

spark_status spark_finalize(spark_ctx* ctx) {
    if (!ctx) return SPARK_ERR_ARG;
    spark_status st = guard(ctx, [&] {
        set_device(ctx);
        CU(cudaStreamSynchronize(ctx->stream));
        for (auto& e : ctx->ev) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        if (ctx->comm_stream) CU(cudaStreamSynchronize(ctx->comm_stream));
        for (auto& gr : ctx->graphs)
            if (gr.exec) cudaGraphExecDestroy(gr.exec);
        if (ctx->comm) ncclCommDestroy(ctx->comm);
        if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
        if (ctx->ev_packed) cudaEventDestroy(ctx->ev_packed);
        if (ctx->ev_recv) cudaEventDestroy(ctx->ev_recv);
        if (ctx->h2d) CU(cudaStreamSynchronize(ctx->h2d));
        if (ctx->d2h) CU(cudaStreamSynchronize(ctx->d2h));
        for (auto* v : {&ctx->ev_h2d, &ctx->ev_out, &ctx->ev_d2h})
            for (cudaEvent_t e : *v) cudaEventDestroy(e);
        if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
        if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    });
    if (ctx->group) {
        auto& m = ctx->group->members;
        m.erase(std::remove(m.begin(), m.end(), ctx), m.end());
    }
    delete ctx;
    return st;
}

const char* spark_last_error(const spark_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

// the members of c's local group, all of them (a finalized member leaves a
// group that can no longer exchange or step)
static const std::vector<spark_ctx*>& group_members(const spark_ctx* c) {
    const auto& m = c->group->members;
    if ((int)m.size() != c->nranks) throw Error(SPARK_ERR_STATE, "a member of this local group was finalized");
    return m;
}

static void after_state_loaded(spark_ctx* c) {
    launched(c, spark::launch_scalars_reset(c->sc, c->stream), "scalars reset");
    launched(c, spark::launch_cfl_min(c->plan.geo, c->U[c->n_idx], c->sc, c->stream), "cfl min");
    allreduce_acc(c);
    c->have_state = true;
}

spark_status spark_set_state(spark_ctx* ctx, const double* U, int32_t on_device) {
    if (!ctx || !U) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        set_device(ctx);
        const size_t bytes = sizeof(double) * ctx->plan.geo.nvar * (size_t)ctx->plan.geo.ncell;
        ctx->n_idx = 0;
        const double* src = U;
        if (!on_device) {  // stage through U[1] (dead before the first step)
            CU(cudaMemcpyAsync(ctx->U[1], U, bytes, cudaMemcpyHostToDevice, ctx->stream));
            src = ctx->U[1];
        }
        // canonical U[v][b][c] -> the block-interleaved pool U[b][v][c]
        launched(ctx, spark::launch_relayout(ctx->plan.geo, src, ctx->U[0], 1, ctx->stream), "relayout");
        after_state_loaded(ctx);
    });
}

spark_status spark_set_primitive(spark_ctx* ctx, const double* W, int32_t on_device) {
    if (!ctx || !W) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        set_device(ctx);
        const size_t bytes = sizeof(double) * ctx->plan.geo.nvar * (size_t)ctx->plan.geo.ncell;
        ctx->n_idx = 0;
        const double* src = W;
        if (!on_device) {  // stage through U[1] (dead before the first step)
            CU(cudaMemcpyAsync(ctx->U[1], W, bytes, cudaMemcpyHostToDevice, ctx->stream));
            src = ctx->U[1];
        }
        launched(ctx, spark::launch_prim_to_cons(ctx->plan.geo, src, ctx->U[0], ctx->stream), "prim to cons");
        after_state_loaded(ctx);
    });
}

spark_status spark_get_state(spark_ctx* ctx, double* U, int32_t on_device) {
    if (!ctx || !U) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (!ctx->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
        set_device(ctx);
        const size_t bytes = sizeof(double) * ctx->plan.geo.nvar * (size_t)ctx->plan.geo.ncell;
        // block-interleaved pool -> canonical; a host copy stages through a state
        // buffer that is dead between API calls (rollback happens inside spark_step)
        double* dst = on_device ? U : ctx->U[(ctx->n_idx + 1) % 3];
        launched(ctx, spark::launch_relayout(ctx->plan.geo, ctx->U[ctx->n_idx], dst, 0, ctx->stream), "relayout");
        if (!on_device) CU(cudaMemcpyAsync(U, dst, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        sync_and_check(ctx, false, -1);
    });
}

spark_status spark_get_time(spark_ctx* ctx, double* t, int64_t* steps, double* dt_last) {
    if (!ctx) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        set_device(ctx);
        CU(cudaStreamSynchronize(ctx->stream));
        spark::DevScalars h;
        CU(cudaMemcpy(&h, ctx->sc, sizeof(h), cudaMemcpyDeviceToHost));
        if (t) *t = h.t;
        if (steps) *steps = h.steps;
        if (dt_last) *dt_last = h.dt;
    });
}

spark_status spark_set_time(spark_ctx* ctx, double t, int64_t steps) {
    if (!ctx || !std::isfinite(t) || steps < 0) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (!ctx->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
        set_device(ctx);
        launched(ctx, spark::launch_set_time(ctx->sc, t, steps, ctx->stream), "set time");
    });
}

spark_status spark_get_cfl_min(spark_ctx* ctx, double* value) {
    if (!ctx || !value) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (!ctx->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
        set_device(ctx);
        CU(cudaStreamSynchronize(ctx->stream));
        spark::DevScalars h;
        CU(cudaMemcpy(&h, ctx->sc, sizeof(h), cudaMemcpyDeviceToHost));
        long long bits = (long long)h.acc;
        std::memcpy(value, &bits, sizeof(double));
    });
}

spark_status spark_fill_guardcells(spark_ctx* ctx, double* padded_out) {
    if (!ctx) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (!ctx->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
        set_device(ctx);
        if (ctx->group) {
            for (spark_ctx* m : group_members(ctx)) pack_all(m, m->U[m->n_idx]);
            exchange_local(group_members(ctx));
        } else if (ctx->comm) {
            pack_all(ctx, ctx->U[ctx->n_idx]);
            exchange_nccl(ctx, ctx->stream);
        }
        if (padded_out) {
            const double* halo[3][2];
            for (int d = 0; d < 3; d++)
                for (int s = 0; s < 2; s++) halo[d][s] = ctx->recv[d][s];
            launched(ctx, spark::launch_fill_padded(ctx->plan.geo, ctx->U[ctx->n_idx], halo, padded_out, ctx->stream),
                     "fill padded");
        }
    });
}

spark_status spark_step(spark_ctx* ctx, double dt, double t_end, double* dt_used) {
    if (!ctx) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (!ctx->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
        if (ctx->group) throw Error(SPARK_ERR_STATE, "local-group contexts step with spark_step_group");
        set_device(ctx);
        const int old_n = ctx->n_idx;
        launched(ctx, spark::launch_step_begin(ctx->sc, dt, t_end, ctx->cfg.cfl, ctx->stream), "step begin");
        do_step(ctx, dt);
        if (dt_used) {
            sync_and_check(ctx, true, old_n);
            double h;
            CU(cudaMemcpy(&h, &ctx->sc->dt, sizeof(double), cudaMemcpyDeviceToHost));
            *dt_used = h;
        }
    });
}

spark_status spark_advance(spark_ctx* ctx, int64_t max_steps, double t_end, int32_t check_every,
                           int64_t* steps_done) {
    if (!ctx) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (!ctx->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
        if (ctx->group) throw Error(SPARK_ERR_STATE, "local-group contexts step with spark_step_group");
        set_device(ctx);
        spark::DevScalars h0;
        CU(cudaStreamSynchronize(ctx->stream));
        CU(cudaMemcpy(&h0, ctx->sc, sizeof(h0), cudaMemcpyDeviceToHost));
        for (int64_t n = 0; n < max_steps; n++) {
            launched(ctx, spark::launch_step_begin(ctx->sc, 0.0, t_end, ctx->cfg.cfl, ctx->stream), "step begin");
            do_step(ctx, 0.0);
            if ((check_every > 0 && (n + 1) % check_every == 0) || n + 1 == max_steps) {
                sync_and_check(ctx, false, -1);
                spark::DevScalars h;
                CU(cudaMemcpy(&h, ctx->sc, sizeof(h), cudaMemcpyDeviceToHost));
                if (!h.active || (t_end > 0.0 && h.t >= t_end * (1.0 - 1e-14))) break;
            }
        }
        sync_and_check(ctx, false, -1);
        spark::DevScalars h;
        CU(cudaMemcpy(&h, ctx->sc, sizeof(h), cudaMemcpyDeviceToHost));
        if (steps_done) *steps_done = h.steps - h0.steps;
    });
}

spark_status spark_step_group(spark_ctx* const* ctxs, int32_t n, double dt, double t_end, double* dt_used) {
    if (!ctxs || n < 1 || !ctxs[0]) return SPARK_ERR_ARG;
    spark_ctx* c0 = ctxs[0];
    return guard(c0, [&] {
        if (!c0->group || (int)c0->group->members.size() != n)
            throw Error(SPARK_ERR_ARG, "spark_step_group needs all contexts of one local group");
        std::vector<spark_ctx*> m(group_members(c0));
        for (spark_ctx* c : m)
            if (!c->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
        set_device(c0);
        group_min(m);  // global CFL minimum of U^n (set_state computes it per rank)
        std::vector<int> old(n);
        for (int r = 0; r < n; r++) {
            old[r] = m[r]->n_idx;
            launched(m[r], spark::launch_step_begin(m[r]->sc, dt, t_end, m[r]->cfg.cfl, m[r]->stream), "step begin");
        }
        const int S = c0->cfg.rk_stages;
        for (int s = 1; s <= S; s++) {
            for (spark_ctx* c : m) {
                int pi, po;
                stage_buffers(S, c->n_idx, s, &pi, &po);
                pack_all(c, c->U[pi]);
            }
            {
                Nvtx r("halo exchange (virtual ranks)");
                exchange_local(m);
            }
            for (spark_ctx* c : m) {
                int pi, po;
                stage_buffers(S, c->n_idx, s, &pi, &po);
                double a, b;
                rk_coeffs(S, s, &a, &b);
                stage_launch(c, c->U[pi], c->U[c->n_idx], a, b, c->U[po], s == S, &c->sc->dt, dt, true);
            }
        }
        group_min(m);
        for (spark_ctx* c : m) {
            int pi, po;
            c->n_idx = stage_buffers(S, c->n_idx, 1, &pi, &po);
        }
        if (dt_used) {
            // every member holds the group-min `bad`: decide once, then roll
            // back all members or none before reporting
            std::vector<spark::DevScalars> h(n);
            for (int r = 0; r < n; r++) h[r] = read_scalars(m[r]);
            if (h[0].bad != spark::kNoBad) {
                const bool now = failed_now(h[0]);
                for (int r = 0; r < n; r++)
                    if (h[r].bad != h[0].bad || failed_now(h[r]) != now)
                        throw Error(SPARK_ERR_STATE, "local group members disagree on the failure word");
                if (now)
                    for (int r = 0; r < n; r++) rollback(m[r], h[r], old[r]);
                spark::DevScalars any = h[0];
                for (int r = 0; r < n; r++) any.status |= h[r].status;
                throw_nonphysical(any, now);
            }
            double h0;
            CU(cudaMemcpy(&h0, &c0->sc->dt, sizeof(double), cudaMemcpyDeviceToHost));
            *dt_used = h0;
        }
    });
}

// One step with host buffers, the copies pipelined with the device work.
// The state moves in nchunks block ranges as pitched copies straight between
// the canonical host layout [v][b][cell] and the block-interleaved device
// layout [b][v][cell] (one 2-D copy per range and variable: no staging
// buffer, no relayout kernel).  Upload chunk j waits only for chunk j of the
// previous call's download (U_in may be the previous U_out; full-duplex
// PCIe: this call's H2D overlaps the previous call's D2H).  After the CFL
// minimum of the whole uploaded U^n (dt is global) and the first S-1 stages,
// the last stage runs range by range on a single-rank context, and range j's
// download starts as soon as its blocks are written, under the remaining
// ranges' compute; a multi-rank context runs the last stage whole (its
// interior / rank-boundary split) and then downloads range by range.
spark_status spark_step_host(spark_ctx* ctx, const double* U_in, double* U_out, double dt, double t_end,
                             int32_t nchunks) {
    if (!ctx || !U_in || !U_out || nchunks < 1) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (ctx->group) throw Error(SPARK_ERR_STATE, "local-group contexts step with spark_step_group");
        set_device(ctx);
        const spark::Geo& g = ctx->plan.geo;
        const long long nblk = (long long)g.bn[0] * g.bn[1] * g.bn[2];
        const int m = (int)std::min<long long>(nchunks, nblk);
        if (!ctx->h2d) {
            CU(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
            CU(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
        }
        while ((int)ctx->ev_h2d.size() < m) {
            cudaEvent_t a, b, c;
            CU(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
            ctx->ev_h2d.push_back(a);
            ctx->ev_out.push_back(b);
            ctx->ev_d2h.push_back(c);
        }
        auto range = [&](int j, long long* b0, long long* b1) {
            *b0 = nblk * j / m;
            *b1 = nblk * (j + 1) / m;
        };
        // blocks [b0, b1) of variable v: host U[v][b][cell] <-> device D[b][v][cell]
        const size_t cell_bytes = sizeof(double) * (size_t)g.cpb;
        auto copy = [&](cudaStream_t st, const double* host_src, double* dev_dst, const double* dev_src,
                        double* host_dst, long long b0, long long b1) {
            for (int v = 0; v < g.nvar; v++) {
                const size_t h = (size_t)v * g.ncell + (size_t)b0 * g.cpb, d = (size_t)b0 * g.bs + (size_t)v * g.vs;
                if (host_src)
                    CU(cudaMemcpy2DAsync(dev_dst + d, sizeof(double) * g.bs, host_src + h, cell_bytes, cell_bytes,
                                         (size_t)(b1 - b0), cudaMemcpyHostToDevice, st));
                else
                    CU(cudaMemcpy2DAsync(host_dst + h, cell_bytes, dev_src + d, sizeof(double) * g.bs, cell_bytes,
                                         (size_t)(b1 - b0), cudaMemcpyDeviceToHost, st));
            }
        };
        const int n = ctx->n_idx;
        // ---- in: H2D chunk j (after the previous call's D2H of chunk j) -> U^n
        for (int j = 0; j < m; j++) {
            long long b0, b1;
            range(j, &b0, &b1);
            CU(cudaStreamWaitEvent(ctx->h2d, ctx->ev_d2h[j], 0));
            copy(ctx->h2d, U_in, ctx->U[n], nullptr, nullptr, b0, b1);
            CU(cudaEventRecord(ctx->ev_h2d[j], ctx->h2d));
            CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_h2d[j], 0));
        }
        // ---- the step: CFL minimum of the uploaded U^n (global), then the stages
        launched(ctx, spark::launch_acc_reset(ctx->sc, ctx->stream), "acc reset");
        launched(ctx, spark::launch_cfl_min(g, ctx->U[n], ctx->sc, ctx->stream), "cfl min");
        allreduce_acc(ctx);
        ctx->have_state = true;
        launched(ctx, spark::launch_step_begin(ctx->sc, dt, t_end, ctx->cfg.cfl, ctx->stream), "step begin");
        auto download = [&](int j, const double* src) {  // range j of src, after the compute stream's work so far
            long long b0, b1;
            range(j, &b0, &b1);
            CU(cudaEventRecord(ctx->ev_out[j], ctx->stream));
            CU(cudaStreamWaitEvent(ctx->d2h, ctx->ev_out[j], 0));
            copy(ctx->d2h, nullptr, nullptr, src, U_out, b0, b1);
            CU(cudaEventRecord(ctx->ev_d2h[j], ctx->d2h));
        };
        if (ctx->comm) {
            do_step(ctx, dt);
            for (int j = 0; j < m; j++) download(j, ctx->U[ctx->n_idx]);
        } else {
            Nvtx step_range("spark step (host buffers)");
            const int S = ctx->cfg.rk_stages;
            int newn = n;
            for (int s = 1; s <= S; s++) {
                int pi, po;
                newn = stage_buffers(S, n, s, &pi, &po);
                double a, b;
                rk_coeffs(S, s, &a, &b);
                if (s < S) {
                    stage_launch(ctx, ctx->U[pi], ctx->U[n], a, b, ctx->U[po], false, &ctx->sc->dt, dt, true);
                    continue;
                }
                for (int j = 0; j < m; j++) {  // the last stage range by range, each range downloaded at once
                    long long b0, b1;
                    range(j, &b0, &b1);
                    stage_launch(ctx, ctx->U[pi], ctx->U[n], a, b, ctx->U[po], true, &ctx->sc->dt, dt, true, 0,
                                 nullptr, false, (int)b0, (int)(b1 - b0));
                    if (j > 0) ctx->stage_launches--;  // the ranges of one stage count once
                    download(j, ctx->U[po]);
                }
            }
            allreduce_acc(ctx);
            ctx->n_idx = newn;
        }
        // a later synchronisation of the context stream covers the downloads
        CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_d2h[m - 1], 0));
    });
}

spark_status spark_stage_apply(spark_ctx* ctx, const double* U_prev, const double* U_n, double a, double b, double dt,
                               double* U_out) {
    if (!ctx || !U_prev || !U_out) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (ctx->nranks != 1 || ctx->comm)
            throw Error(SPARK_ERR_STATE, "spark_stage_apply needs a single-rank context without NCCL exchange");
        if (a != 0.0 && !U_n) throw Error(SPARK_ERR_ARG, "U_n required when a != 0");
        set_device(ctx);
        // the kernel runs on the block-interleaved layout: the caller's canonical
        // buffers go through the context's state buffers (the loaded state is lost)
        const spark::Geo& g = ctx->plan.geo;
        launched(ctx, spark::launch_relayout(g, U_prev, ctx->U[0], 1, ctx->stream), "relayout");
        if (a != 0.0) launched(ctx, spark::launch_relayout(g, U_n, ctx->U[1], 1, ctx->stream), "relayout");
        stage_launch(ctx, ctx->U[0], a != 0.0 ? ctx->U[1] : nullptr, a, b, ctx->U[2], false, nullptr, dt, false);
        launched(ctx, spark::launch_relayout(g, ctx->U[2], U_out, 0, ctx->stream), "relayout");
        ctx->have_state = false;
    });
}

spark_status spark_profile_enable(spark_ctx* ctx, int32_t on) {
    if (!ctx) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        ctx->prof = on != 0;
        if (on) {
            ctx->ev_used = 0;
            ctx->stage_launches = 0;
            ctx->total_launches = 0;
            ctx->prof_ms = 0.0;
        }
    });
}

spark_status spark_profile_read(spark_ctx* ctx, double* stage_ms, int64_t* stage_launches, int64_t* total_launches) {
    if (!ctx) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        set_device(ctx);
        CU(cudaStreamSynchronize(ctx->stream));
        double ms = 0.0;
        for (size_t i = 0; i < ctx->ev_used; i++) {
            float x = 0.f;
            CU(cudaEventElapsedTime(&x, ctx->ev[i].first, ctx->ev[i].second));
            ms += x;
        }
        if (stage_ms) *stage_ms = ms;
        if (stage_launches) *stage_launches = ctx->stage_launches;
        if (total_launches) *total_launches = ctx->total_launches;
    });
}

}  // extern "C"

namespace {
// Local-group dt minimum: one tiny kernel takes the min of every member's
// accumulator and writes it back to each (all members share one stream).
void group_min(const std::vector<spark_ctx*>& m) {
    if (m.size() > (size_t)spark::kMaxGroup) throw Error(SPARK_ERR_ARG, "local group too large");
    spark::AccPtrs p{};
    for (size_t r = 0; r < m.size(); r++) p.p[r] = &m[r]->sc->acc;
    launched(m[0], spark::launch_group_min(p, (int)m.size(), m[0]->stream), "group min");
}
}  // namespace

extern "C" spark_status spark_selftest_riemann(int32_t device, int32_t riemann, int32_t ndim, int32_t dir,
                                               double gamma, int64_t n, const double* wl, const double* wr,
                                               double* f) {
    return guard(nullptr, [&] {
        if (ndim < 1 || ndim > 3 || dir < 0 || dir >= ndim || n < 0 || !wl || !wr || !f || riemann < 0 ||
            riemann > 1)
            throw Error(SPARK_ERR_ARG, "bad selftest arguments");
        CU(cudaSetDevice(device));
        const size_t bytes = sizeof(double) * (size_t)n * (ndim + 2);
        double* d = nullptr;
        CU(cudaMalloc(&d, 3 * bytes + 8));
        struct Free {
            double* p;
            ~Free() { cudaFree(p); }
        } fr{d};
        char* base = reinterpret_cast<char*>(d);
        double* dl = d;
        double* dr = reinterpret_cast<double*>(base + bytes);
        double* df = reinterpret_cast<double*>(base + 2 * bytes);
        CU(cudaMemcpy(dl, wl, bytes, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(dr, wr, bytes, cudaMemcpyHostToDevice));
        if (n > 0) CU(spark::launch_selftest_riemann(riemann, ndim, dir, gamma, n, dl, dr, df));
        CU(cudaDeviceSynchronize());
        CU(cudaMemcpy(f, df, bytes, cudaMemcpyDeviceToHost));
    });
}

extern "C" spark_status spark_axpy(int32_t device, int32_t variant, int64_t n, double a, const double* x, double* y,
                                   void* cuda_stream) {
    return guard(nullptr, [&] {
        if (variant < 0 || variant > 3 || n < 0 || (n > 0 && (!x || !y))) throw Error(SPARK_ERR_ARG, "bad axpy arguments");
        CU(cudaSetDevice(device));
        int sms = 0;
        CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        CU(spark::launch_axpy(variant, n, a, x, y, sms, static_cast<cudaStream_t>(cuda_stream)));
    });
}

extern "C" spark_status spark_telescoping_scratch_bytes(const spark_config* cfg, int32_t rank, int32_t nranks,
                                                       size_t* bytes) {
    return guard(nullptr, [&] {
        if (!bytes) throw Error(SPARK_ERR_ARG, "null bytes");
        Plan p = make_plan(cfg, rank, nranks, nranks == 1);
        *bytes = tile_scratch_bytes(cfg, p);
    });
}

extern "C" spark_status spark_telescoping_plan(const spark_config* cfg, int32_t rank, int32_t nranks,
                                              int32_t peer[27], int64_t cells[27], int32_t ops[54],
                                              int32_t* nops) {
    return guard(nullptr, [&] {
        if (!peer || !cells || !ops || !nops) throw Error(SPARK_ERR_ARG, "null output");
        Plan p = make_plan(cfg, rank, nranks);
        const spark::TileGeo t = tile_geo(cfg, p);
        int pr[27];
        for (int dir = 0; dir < 27; dir++) {
            pr[dir] = dir == 13 ? -1 : tile_peer(p, dir);
            peer[dir] = pr[dir];
            cells[dir] = pr[dir] >= 0 ? spark::tile_region_cells(t, dir) : 0;
        }
        const auto o = tile_ops(pr);
        *nops = (int32_t)o.size();
        for (size_t i = 0; i < o.size(); i++) ops[i] = o[i].first ? -(o[i].second + 1) : o[i].second + 1;
    });
}

extern "C" spark_status spark_set_scratch(spark_ctx* ctx, void* scratch, size_t bytes) {
    if (!ctx) return SPARK_ERR_ARG;
    return guard(ctx, [&] { tile_attach(ctx, scratch, bytes); });
}

// telescoping step through HBM tiles (one shell exchange per step)
static void tile_step_one(spark_ctx* ctx, double dt, double t_end) {
    std::string m = tile_check(&ctx->cfg, ctx->plan);
    if (!m.empty()) throw Error(SPARK_ERR_ARG, m);
    if (!ctx->tiles.ready) throw Error(SPARK_ERR_STATE, "telescoping tiles need spark_set_scratch first");
    launched(ctx, spark::launch_step_begin(ctx->sc, dt, t_end, ctx->cfg.cfl, ctx->stream), "step begin");
    {
        Nvtx r("telescoping shell exchange");
        tile_pack(ctx);
        if (ctx->comm) tile_exchange_nccl(ctx);
    }
    Nvtx r2("telescoping stages");
    tile_stages(ctx);
    allreduce_acc(ctx);
    ctx->n_idx = (ctx->n_idx + 1) % 3;
}

extern "C" spark_status spark_step_group_telescoping(spark_ctx* const* ctxs, int32_t n, double dt, double t_end,
                                                     double* dt_used) {
    if (!ctxs || n < 1 || !ctxs[0]) return SPARK_ERR_ARG;
    spark_ctx* c0 = ctxs[0];
    return guard(c0, [&] {
        if (!c0->group || (int)c0->group->members.size() != n)
            throw Error(SPARK_ERR_ARG, "needs all contexts of one local group");
        std::vector<spark_ctx*> m(group_members(c0));
        for (spark_ctx* c : m) {
            if (!c->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
            if (!c->tiles.ready) throw Error(SPARK_ERR_STATE, "telescoping tiles need spark_set_scratch first");
            std::string msg = tile_check(&c->cfg, c->plan);
            if (!msg.empty()) throw Error(SPARK_ERR_ARG, msg);
        }
        set_device(c0);
        group_min(m);
        std::vector<int> old(n);
        for (int r = 0; r < n; r++) {
            old[r] = m[r]->n_idx;
            launched(m[r], spark::launch_step_begin(m[r]->sc, dt, t_end, m[r]->cfg.cfl, m[r]->stream), "step begin");
            tile_pack(m[r]);
        }
        {
            Nvtx r("telescoping shell exchange");
            tile_exchange_local(m);  // the one exchange of the step
        }
        for (spark_ctx* c : m) tile_stages(c);
        group_min(m);
        for (spark_ctx* c : m) c->n_idx = (c->n_idx + 1) % 3;
        if (dt_used) {
            std::vector<spark::DevScalars> h(n);
            for (int r = 0; r < n; r++) h[r] = read_scalars(m[r]);
            if (h[0].bad != spark::kNoBad) {
                const bool now = failed_now(h[0]);
                if (now)
                    for (int r = 0; r < n; r++) rollback(m[r], h[r], old[r]);
                throw_nonphysical(h[0], now);
            }
            *dt_used = h[0].dt;
        }
    });
}

extern "C" spark_status spark_step_telescoping(spark_ctx* ctx, double dt, double t_end, double* dt_used) {
    if (!ctx) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (!ctx->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
        if (ctx->group) throw Error(SPARK_ERR_STATE, "local-group contexts step with spark_step_group_telescoping");
        if (ctx->cfg.ndim > 2 || ctx->nranks != 1 || ctx->comm || ctx->tiles.ready) {
            // 3-D, several ranks, or tiles requested: telescoping through HBM tiles
            set_device(ctx);
            const int old_n = ctx->n_idx;
            tile_step_one(ctx, dt, t_end);
            if (dt_used) {
                sync_and_check(ctx, true, old_n);
                double h;
                CU(cudaMemcpy(&h, &ctx->sc->dt, sizeof(double), cudaMemcpyDeviceToHost));
                *dt_used = h;
            }
            return;
        }
        const int S = ctx->cfg.rk_stages;
        const int ngk = stencil_ng(ctx->cfg.recon);
        for (int d = 0; d < ctx->cfg.ndim; d++)
            if (S * ngk > (long long)ctx->cfg.nb[d] * ctx->cfg.nblk[d])
                throw Error(SPARK_ERR_ARG, "telescoped halo deeper than the domain");
        if (spark::telescope_smem_bytes(ctx->plan.geo, ctx->cfg.recon, S) > 227 * 1024)
            throw Error(SPARK_ERR_ARG, "telescoping tile exceeds shared memory (block too large)");
        set_device(ctx);
        const int old_n = ctx->n_idx;
        launched(ctx, spark::launch_step_begin(ctx->sc, dt, t_end, ctx->cfg.cfl, ctx->stream), "step begin");
        const int out = (ctx->n_idx + 1) % 3;
        spark::StageArgs A{};
        A.g = ctx->plan.geo;
        A.uprev = ctx->U[ctx->n_idx];
        A.un = ctx->U[ctx->n_idx];
        A.uout = ctx->U[out];
        A.sc = ctx->sc;
        A.dt_ptr = &ctx->sc->dt;
        A.last = 1;
        A.honor_active = 1;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (ctx->prof) {
            if (ctx->ev_used == ctx->ev.size()) {
                cudaEvent_t x, y;
                CU(cudaEventCreate(&x));
                CU(cudaEventCreate(&y));
                ctx->ev.emplace_back(x, y);
            }
            e0 = ctx->ev[ctx->ev_used].first;
            e1 = ctx->ev[ctx->ev_used].second;
            ctx->ev_used++;
            CU(cudaEventRecord(e0, ctx->stream));
        }
        launched(ctx, spark::launch_telescope(A, ctx->cfg.recon, ctx->cfg.riemann, S, ctx->stream), "telescope");
        ctx->stage_launches++;
        if (ctx->prof) CU(cudaEventRecord(e1, ctx->stream));
        ctx->n_idx = out;
        if (dt_used) {
            sync_and_check(ctx, true, old_n);
            double h;
            CU(cudaMemcpy(&h, &ctx->sc->dt, sizeof(double), cudaMemcpyDeviceToHost));
            *dt_used = h;
        }
    });
}

// spark_run: nsteps SSP-RK steps, fully asynchronous.  Single-rank contexts on a
// non-default stream replay a CUDA graph of 3 steps (after 3 steps the U^n
// buffer index is back where it started, so the captured pointers stay valid);
// launch-bound problems (the small configs) gain the most.
extern "C" spark_status spark_run(spark_ctx* ctx, int64_t nsteps, double dt, double t_end) {
    if (!ctx || nsteps < 0) return SPARK_ERR_ARG;
    return guard(ctx, [&] {
        if (!ctx->have_state) throw Error(SPARK_ERR_STATE, "no state loaded");
        if (ctx->group) throw Error(SPARK_ERR_STATE, "local-group contexts step with spark_step_group");
        set_device(ctx);
        const bool graphable = !ctx->comm && !ctx->prof && ctx->stream != nullptr;
        const int64_t per_step = ctx->cfg.rk_stages + 1;
        int64_t done = 0;
        while (done < nsteps) {
            if (graphable && nsteps - done >= 3) {
                auto& gr = ctx->graphs[ctx->n_idx];
                if (!gr.exec || gr.dt != dt || gr.t_end != t_end) {
                    if (gr.exec) CU(cudaGraphExecDestroy(gr.exec));
                    gr.exec = nullptr;
                    const int n0 = ctx->n_idx;
                    const int64_t sl = ctx->stage_launches, tl = ctx->total_launches;
                    cudaGraph_t graph = nullptr;
                    CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
                    try {
                        for (int k = 0; k < 3; k++) {
                            launched(ctx, spark::launch_step_begin(ctx->sc, dt, t_end, ctx->cfg.cfl, ctx->stream),
                                     "step begin");
                            do_step(ctx, dt);
                        }
                    } catch (...) {
                        cudaStreamEndCapture(ctx->stream, &graph);
                        if (graph) cudaGraphDestroy(graph);
                        ctx->n_idx = n0;
                        throw;
                    }
                    CU(cudaStreamEndCapture(ctx->stream, &graph));
                    cudaError_t e = cudaGraphInstantiate(&gr.exec, graph, 0);
                    cudaGraphDestroy(graph);
                    if (e != cudaSuccess) {
                        gr.exec = nullptr;
                        throw Error(SPARK_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
                    }
                    gr.dt = dt;
                    gr.t_end = t_end;
                    ctx->stage_launches = sl;  // capturing launched nothing
                    ctx->total_launches = tl;
                    if (ctx->n_idx != n0) throw Error(SPARK_ERR_STATE, "buffer rotation period is not 3");
                }
                CU(cudaGraphLaunch(gr.exec, ctx->stream));
                ctx->total_launches += 3 * per_step;
                ctx->stage_launches += 3 * ctx->cfg.rk_stages;
                done += 3;
            } else {
                launched(ctx, spark::launch_step_begin(ctx->sc, dt, t_end, ctx->cfg.cfl, ctx->stream), "step begin");
                do_step(ctx, dt);
                done += 1;
            }
        }
    });
}
