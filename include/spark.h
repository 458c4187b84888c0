/*
 * spark.h — C ABI of libspark, the B200-native Spark block-update hot path.
 *
 * What the library computes (PAPER.md = arXiv 2401.03378, /root/reference):
 *   Flash-X's Spark hydrodynamics solver advances a set of blocks of identical
 *   cell counts, each surrounded by a halo of guard cells that makes it look
 *   like a whole domain (§2.2), with strong-stability-preserving
 *   Runge-Kutta stages (§4.2).  In the non-telescoping variant
 *   (lst:spark-nontelescoping) every stage first fills the guard
 *   cells ("p2p communication") and then runs, for all blocks, the
 *   block initialisation (Alg. 7) and the intra-stage chain of
 *   Alg. 8: calcLims (reconstruction) -> calcFlux (Riemann) ->
 *   updSoln (divergence + RK combination) -> calcEos.  The paper prints no
 *   formulas; the numerics are the textbook readings in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *   - Every function returns spark_status; no C++ exception crosses the ABI.
 *     After an error, spark_last_error(ctx) describes it (ctx-owned string).
 *   - Layouts, fp64 throughout:
 *       canonical  U[v][b][k][j][i]   i fastest; b = bx + nbx*(by + nby*bz)
 *                  lexicographic over THIS RANK's sub-box of the block grid.
 *       padded     P[v][b][k+gz][j+gy][i+gx], gd = ng for d < ndim else 0
 *                  (the Flash-X block-with-guards of P:361-364).
 *     Internally the state is block-interleaved, U[b][v][k][j][i] (one block
 *     is one contiguous chunk of HBM); set/get convert.
 *     v = 0 density, 1..ndim momentum, ndim+1 total energy (conserved) or
 *     v = 0 density, 1..ndim velocity, ndim+1 pressure (primitive).
 *   - Memory ownership: the CALLER owns the device arena passed to spark_init
 *     (>= spark_required_bytes) and keeps it alive until spark_finalize.  The
 *     library never allocates device memory for state and never frees caller
 *     memory.  Host/device pointers passed to other calls are borrowed for the
 *     duration of the call.
 *   - Streams: all device work is enqueued on the cudaStream_t given to
 *     spark_init.  Only calls documented as synchronising block the host.
 *   - Determinism: identical inputs and rank count give bitwise-identical
 *     results; no floating-point atomics are used (dt minimum via integer
 *     atomics on the ordered bit pattern of positive doubles).  Results are
 *     also bitwise independent of the rank count (halos are exact copies).
 *   - Thread safety: one context per device per host thread; not re-entrant.
 */
#ifndef SPARK_H
#define SPARK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPARK_ABI_VERSION 3

typedef enum {
    SPARK_OK = 0,
    SPARK_ERR_ARG = 1,          /* invalid argument or configuration            */
    SPARK_ERR_CUDA = 2,         /* CUDA runtime error (message in last_error)   */
    SPARK_ERR_NCCL = 3,         /* NCCL error                                   */
    SPARK_ERR_OOM = 4,          /* arena too small                              */
    SPARK_ERR_NONPHYSICAL = 5,  /* rho <= 0, p <= 0 or non-finite after a stage */
    SPARK_ERR_STATE = 6         /* call out of order (e.g. step before state)   */
} spark_status;

typedef enum { SPARK_BC_PERIODIC = 0, SPARK_BC_OUTFLOW = 1, SPARK_BC_REFLECT = 2 } spark_bc;
/* PLM = minmod-limited (reading R2), WENO5 = WENO5-JS (R3); NEXT N2:
 * PLM_MC = monotonized-central limiter (R18), WENO5Z = WENO5-Z (R19). */
typedef enum {
    SPARK_RECON_FIRST = 0,
    SPARK_RECON_PLM = 1,
    SPARK_RECON_WENO5 = 2,
    SPARK_RECON_PLM_MC = 3,
    SPARK_RECON_WENO5Z = 4
} spark_recon;
/* HYBRID (shockDet Alg. 7; reading R21): HLLC, but HLL at
 * faces the shock detector flags (needs recon PLM, PLM_MC, WENO5 or WENO5Z). */
typedef enum { SPARK_RIEMANN_HLL = 0, SPARK_RIEMANN_HLLC = 1, SPARK_RIEMANN_HYBRID = 2 } spark_riemann;

/* Problem description.  Identical on every rank (it describes the GLOBAL grid). */
typedef struct {
    int32_t ndim;         /* 1..3; nvar = ndim + 2                                   */
    int32_t nb[3];        /* interior cells per block per dim (1 for d >= ndim)      */
    int32_t nblk[3];      /* blocks per dim of the global grid (1 for d >= ndim)     */
    int32_t ng;           /* guard layers: >= 1 first order, >= 2 PLM(-MC), >= 3 WENO5(-Z) */
    double lo[3], hi[3];  /* domain; dx_d = (hi_d - lo_d) / (nblk_d * nb_d)          */
    int32_t bc[3][2];     /* spark_bc per face (low, high) per dim                   */
    int32_t recon;        /* spark_recon                                             */
    int32_t riemann;      /* spark_riemann                                           */
    int32_t rk_stages;    /* 2 (SSP-RK2) or 3 (SSP-RK3)                              */
    double gamma;         /* ideal-gas ratio of specific heats (> 1)                 */
    double cfl;           /* Courant number C in dt = C min dx_d/(|u_d| + c)         */
    double grav[3];       /* grvAccel (Alg. 8; reading R20): uniform gravity;
                           * L(U) += (0, rho g, m.g); all zero = no source. ABI v2  */
    double shock_thresh;  /* shockDet (reading R21), used with SPARK_RIEMANN_HYBRID:
                           * cell i is a shock cell along d when u_d(i+1) < u_d(i-1)
                           * and |p(i+1) - p(i-1)| > shock_thresh * min(p(i+-1));
                           * a face of a shock cell takes HLL.  > 0.  ABI v3          */
} spark_config;

typedef struct spark_ctx spark_ctx; /* opaque, one per rank (per GPU) */

/* Halo plan of one face of a rank's sub-box (host-side, no GPU needed). */
typedef struct {
    int32_t dim, side;    /* face: dimension 0..2, side 0 = low, 1 = high           */
    int32_t peer;         /* rank across the face; -1 = physical boundary / self    */
    int32_t pad;
    int64_t cells;        /* cells in the ng-thick slab (0 when peer < 0)           */
} spark_face_plan;

/* ---- host-only queries (valid on machines without a GPU) -------------- */

int32_t spark_abi_version(void);
const char* spark_status_string(spark_status st);

/* Validate a configuration for nranks ranks.  Checks ndim, nb >= ng, ng large
 * enough for recon, rk_stages, gamma > 1, cfl > 0, the block grid divisible
 * by the process grid, and nb[0]*nb[1] <= 256 (one thread per column of a
 * 256-thread CTA). */
spark_status spark_check_config(const spark_config* cfg, int32_t nranks);

/* Process grid (P_x, P_y, P_z) used for nranks ranks: the factorisation of
 * nranks that divides the block grid and minimises the halo surface. */
spark_status spark_rank_grid(const spark_config* cfg, int32_t nranks, int32_t pgrid[3]);

/* Sub-box of `rank` in BLOCK units: first block box_lo[d], count box_n[d].
 * Ranks are ordered x fastest over the process grid. */
spark_status spark_rank_box(const spark_config* cfg, int32_t rank, int32_t nranks,
                            int32_t box_lo[3], int32_t box_n[3]);

/* The 2*ndim face plans of `rank` (faces ordered dim-major, low then high).
 * A slab holds ng layers of the face cells, layout [v][c2][c1][c0] with c_dim
 * of extent ng (depth in increasing global coordinate) and the other two of
 * the sub-box extent in cells. */
spark_status spark_halo_plan(const spark_config* cfg, int32_t rank, int32_t nranks,
                             spark_face_plan faces[6], int32_t* nfaces);

/* Device bytes the caller must provide as the arena of spark_init. */
spark_status spark_required_bytes(const spark_config* cfg, int32_t rank, int32_t nranks,
                                  size_t* bytes);

/* ---- lifecycle ---------------------------------------------------------- */

/* Rank 0 creates the NCCL unique id (128 bytes); the harness broadcasts it. */
spark_status spark_nccl_unique_id(uint8_t id[128]);

/* Create a context on CUDA device `device`.  nranks == 1: nccl_id may be NULL;
 * a non-NULL id selects self-exchange mode (periodic faces are packed and sent
 * to this rank itself with NCCL send/recv instead of the local wrap — the
 * multi-rank exchange path on one GPU, for testing; results are bitwise equal).
 * nranks > 1: nccl_id from spark_nccl_unique_id on rank 0 (collective call:
 * every rank must call spark_init).  cuda_stream is a cudaStream_t (NULL =
 * legacy default stream).  arena: device memory of >= required bytes, owned
 * by the caller.  Does not synchronise except for NCCL communicator setup. */
spark_status spark_init(const spark_config* cfg, int32_t rank, int32_t nranks, const uint8_t* nccl_id,
                        int32_t device, void* cuda_stream, void* arena, size_t arena_bytes,
                        spark_ctx** out);

/* Virtual ranks on ONE device in one process (testing the multi-rank path
 * without several GPUs): creates nranks contexts whose halo exchange is a
 * device-to-device copy between their buffers.  arenas[r] as in spark_init.
 * Contexts made this way must be stepped with spark_step_group. */
spark_status spark_init_local_group(const spark_config* cfg, int32_t nranks, int32_t device,
                                    void* cuda_stream, void* const* arenas, size_t arena_bytes,
                                    spark_ctx** outs);

/* Release the context (NCCL communicator, events).  Does not free the arena.
 * Synchronises the stream. */
spark_status spark_finalize(spark_ctx* ctx);

/* Last error message of this context ("" if none).  Owned by ctx. */
const char* spark_last_error(const spark_ctx* ctx);

/* ---- state I/O ------------------------------------------------------------ */

/* Load this rank's conserved state U (canonical layout, nvar*ncells_local
 * doubles).  on_device != 0: U is a device pointer, else host memory (pinned
 * for asynchronous copies).  Resets t = 0 and the step count, clears the
 * status word, and computes the CFL minimum of U (KB3) followed by the
 * global-min all-reduce.  Enqueued asynchronously; host U must stay valid
 * until the stream reaches the copy. */
spark_status spark_set_state(spark_ctx* ctx, const double* U, int32_t on_device);

/* As spark_set_state, but from primitive variables W (rho, u, p) converted on
 * the device with the ideal-gas EOS: E = p/(gamma-1) + rho|u|^2/2. */
spark_status spark_set_primitive(spark_ctx* ctx, const double* W, int32_t on_device);

/* Copy the current conserved state U^n into U (canonical layout).
 * SYNCHRONISES the stream; returns SPARK_ERR_NONPHYSICAL if the status word
 * reports a non-physical state. */
spark_status spark_get_state(spark_ctx* ctx, double* U, int32_t on_device);

/* Restore the simulation time and step count (checkpoint/resume: load the
 * saved U with spark_set_state, which resets t = 0 and steps = 0, then call
 * this with the saved values).  The next step then continues bitwise as the
 * uninterrupted run would (dt comes from U, the clip from t).  Asynchronous. */
spark_status spark_set_time(spark_ctx* ctx, double t, int64_t steps);

/* Time, completed steps and dt of the last step.  Synchronises. */
spark_status spark_get_time(spark_ctx* ctx, double* t, int64_t* steps, double* dt_last);

/* Raw CFL minimum min_cells min_d dx_d/(|u_d|+c) of U^n over all ranks (what
 * dt = cfl * value is built from).  Synchronises. */
spark_status spark_get_cfl_min(spark_ctx* ctx, double* value);

/* ---- the hot path -------------------------------------------------------- */

/* fill_guardcells: exchange the rank-boundary face
 * slabs of U^n with the neighbouring ranks.  padded_out != NULL (device
 * pointer, padded layout): additionally materialise every block with its
 * guard cells (faces, edges, corners; each guard cell = the per-dimension
 * boundary map of its global index, reflect negating the normal momentum).
 * With nranks > 1 edge/corner guards owned by diagonal ranks are left NaN.
 * Bit-exact copies.  Asynchronous. */
spark_status spark_fill_guardcells(spark_ctx* ctx, double* padded_out);

/* One SSP-RK step (lst:spark-nontelescoping): for each stage, guard-cell
 * exchange then the fused stage kernel over all blocks.  dt > 0: use it;
 * dt <= 0: CFL dt of U^n (cfl * global min), clipped to t_end - t when
 * t_end > 0; once t >= t_end*(1 - 1e-14) further steps leave U unchanged.
 * dt_used == NULL: fully asynchronous.  dt_used != NULL: synchronises, writes
 * the dt taken and checks the failure word.
 * Errors are rank-consistent: a stage that produces rho <= 0, p <= 0 or NaN
 * records the step number in the failure word, which is min-reduced over all
 * ranks together with the CFL minimum (one collective per step), so every rank
 * sees the same decision.  SPARK_ERR_NONPHYSICAL then either (a) the failing
 * step is the one this call executed: every rank's state is rolled back to
 * U^n, t and the step count of that step; or (b) it was an earlier step
 * enqueued without a check: all steps after it were frozen (no time advance)
 * on every rank and nothing is rolled back; spark_last_error names the step.
 * Collective with nranks > 1: every rank must pass dt_used alike. */
spark_status spark_step(spark_ctx* ctx, double dt, double t_end, double* dt_used);

/* nsteps steps of spark_step (same dt / t_end semantics), fully asynchronous.
 * Single-rank contexts created on a non-default stream replay a CUDA graph of
 * 3 steps (the buffer-rotation period), which removes the per-launch overhead
 * of small, launch-bound problems; other contexts enqueue plain launches.
 * Results are identical to calling spark_step nsteps times. */
spark_status spark_run(spark_ctx* ctx, int64_t nsteps, double dt, double t_end);

/* One step with the state in HOST memory (end-to-end use; canonical layout,
 * pinned for asynchronous copies): upload U_in, step (dt, t_end as spark_step;
 * t and the step count continue — they are not reset as by spark_set_state),
 * download the new U^n to U_out (may alias U_in).  The transfers move nchunks
 * block ranges, as pitched copies between the canonical host layout and the
 * device pool: chunk j of the upload waits only for chunk j of the previous
 * call's download, so consecutive calls overlap their downloads with the next
 * uploads (full-duplex PCIe); on a single-rank context the last RK stage runs
 * range by range and each range's download starts under the remaining
 * ranges' compute.  Asynchronous: the host buffers must stay valid until the context
 * stream is synchronised (the stream waits for the last download).  Errors
 * surface at the next synchronising call. */
spark_status spark_step_host(spark_ctx* ctx, const double* U_in, double* U_out, double dt, double t_end,
                             int32_t nchunks);

/* Telescoping SSP-RK step (lst:spark-telescoping
 * P:1598-1604): one guard gather per STEP with S*NGK layers
 * (NGK = reconstruction half-width; faces, edges and corners), then all S
 * stages per block with the halo area updated too.  Guards beyond a physical
 * boundary are filled once and evolved (reading R17); with periodic
 * boundaries the result equals spark_step.  Same dt and dt_used semantics as
 * spark_step.
 * Two implementations: 1-D/2-D single-rank contexts without NCCL run ONE
 * kernel per step with the tile on chip; 3-D, NCCL contexts (several ranks or
 * self-exchange) or contexts given a scratch (spark_set_scratch) keep the
 * tiles in HBM: the rank's S*NGK-thick shell (26 regions: faces, edges,
 * corners) is exchanged ONCE per step (one grouped NCCL call), then gather +
 * S stage passes.  The result of a block is bitwise independent of the rank
 * count.  The HBM path needs spark_set_scratch first. */
spark_status spark_step_telescoping(spark_ctx* ctx, double dt, double t_end, double* dt_used);

/* Device bytes of the scratch the HBM telescoping path needs (three tiles of
 * U, the primitive tile, the face fluxes and the 2 x 26 shell buffers). */
spark_status spark_telescoping_scratch_bytes(const spark_config* cfg, int32_t rank, int32_t nranks, size_t* bytes);

/* Host-only: the telescoping shell plan of `rank` — per direction
 * dir = (c0+1) + 3(c1+1) + 9(c2+1) (c_d in {-1, 0, 1}; 13 is the rank itself)
 * the peer rank (-1: none) and the cells of the region (G = S*NGK along a
 * nonzero component, the sub-box extent along a zero one; layout [v][z][y][x]
 * of the region), and the posting order of the grouped exchange: ops[i] > 0
 * receive direction ops[i]-1 from its peer, < 0 send the own region on side
 * -ops[i]-1 to that direction's peer (receives ordered by the receiver's
 * direction, sends by 26 - direction). */
spark_status spark_telescoping_plan(const spark_config* cfg, int32_t rank, int32_t nranks, int32_t peer[27],
                                    int64_t cells[27], int32_t ops[54], int32_t* nops);

/* Give the context a caller-owned scratch (device, 256-byte aligned, >= the
 * bytes above) for the HBM telescoping path; selects that path for every
 * spark_step_telescoping of this context. */
spark_status spark_set_scratch(spark_ctx* ctx, void* scratch, size_t bytes);

/* spark_step_telescoping for the contexts of one spark_init_local_group (each
 * with a scratch): one shell exchange between the virtual ranks per step. */
spark_status spark_step_group_telescoping(spark_ctx* const* ctxs, int32_t n, double dt, double t_end,
                                          double* dt_used);

/* Enqueue up to max_steps steps (CFL dt, clipped to t_end), synchronising
 * every check_every steps (<= 0: only at the end) to stop once t_end is
 * reached.  *steps_done receives the number of steps that advanced time. */
spark_status spark_advance(spark_ctx* ctx, int64_t max_steps, double t_end, int32_t check_every,
                           int64_t* steps_done);

/* spark_step for the contexts of one spark_init_local_group, stage by stage
 * in lockstep (exchange between virtual ranks, global dt minimum and failure
 * word).  With dt_used != NULL a failure rolls back ALL members (or, for an
 * earlier unchecked step, none) before SPARK_ERR_NONPHYSICAL is returned. */
spark_status spark_step_group(spark_ctx* const* ctxs, int32_t n, double dt, double t_end, double* dt_used);

/* Apply ONE fused stage to caller buffers (device pointers, canonical layout):
 *   U_out = a * U_n + b * (U_prev + dt * L(U_prev))
 * with guard cells of U_prev from the boundary maps (single-rank contexts
 * only).  U_n may be NULL when a == 0.  For testing the stage in isolation.
 * The buffers are converted to and from the internal layout through the
 * context's state buffers, so a loaded state is discarded (load a new one
 * before stepping).  Asynchronous. */
spark_status spark_stage_apply(spark_ctx* ctx, const double* U_prev, const double* U_n, double a, double b,
                               double dt, double* U_out);

/* ---- measurement ----------------------------------------------------------- */

/* Enable/disable CUDA-event timing around every launch of the fused stage
 * kernel (on the context stream); resets the accumulators when enabling. */
spark_status spark_profile_enable(spark_ctx* ctx, int32_t on);

/* Accumulated stage-kernel time (ms) and launches since enabling.
 * Synchronises. */
spark_status spark_profile_read(spark_ctx* ctx, double* stage_ms, int64_t* stage_launches,
                                int64_t* total_launches);

/* ---- HBM calibration -------------------------------------------- */

/* y_i = a x_i + y_i for i < n (FP64, device pointers, no FMA contraction), with
 * the paper's thread-to-entry mappings (§3.3): variant 0 = increment by 1
 * (alg:axpy-incr-1: contiguous chunk per thread), 1 = increment by
 * #threads (alg:axpy-incr-threads: grid stride), 2 = single
 * iteration (alg:axpy-single-iter: one entry per thread, T >= N),
 * 3 = B200 vectorised grid stride (16-byte accesses; x, y 16-byte aligned).
 * Enqueued on cuda_stream (a cudaStream_t) of device `device`; asynchronous.
 * Used by bench.py as a same-run HBM bandwidth denominator. */
spark_status spark_axpy(int32_t device, int32_t variant, int64_t n, double a, const double* x, double* y,
                        void* cuda_stream);

/* ---- self test ----------------------------------------------------------------- */

/* Evaluate the device Riemann solver (the one KB1 calls, calcFlux P:1833) on n
 * face states given in HOST memory, unrotated primitive order (rho, u_1..u_ndim,
 * p), arrays [n][ndim+2]; normal direction dir (0..ndim-1); riemann as
 * spark_riemann.  f (host, [n][ndim+2]) receives the conserved fluxes.
 * Synchronises (device 'device', default stream).  For tests. */
spark_status spark_selftest_riemann(int32_t device, int32_t riemann, int32_t ndim, int32_t dir, double gamma,
                                    int64_t n, const double* wl, const double* wr, double* f);

/* ---- NEXT N3: fluxBuff + flux correction on a static two-level refinement -------- */
/* The all-levels variant of PAPER.md P:1494-1506 (lst:spark-all-levels
 * P:1510-1523; fluxBuff in Alg. 8), readings R22/R23 of DESIGN.md.
 * The coarse blocks [rlo, rhi) of cfg's block grid are refined by 2 (2^ndim
 * fine blocks of nb cells, spacing dx/2 each).  Leaves: the coarse blocks
 * outside the box, then the fine blocks of the box, each lexicographic with x
 * fastest; the state is U[v][leaf][k][j][i] (canonical layout, leaves as the
 * blocks).  One dt for all leaves (no subcycling).  Guard cells across a
 * coarse-fine face: prolongation = the containing coarse cell, restriction =
 * the mean of the 2^ndim fine cells; each leaf accumulates its face fluxes
 * over the stages (fluxBuff, B <- b_s (B + F)); after the last stage the
 * coarse cells on a coarse-fine face take the mean of the fine fluxes
 * (communicate_fluxes + correction), which makes the step conservative.
 * One rank, or virtual ranks on one device (below); nb even along refined
 * dims; no gravity.  Errors as spark_step. */
typedef struct {
    int32_t rlo[3], rhi[3];  /* refined coarse blocks [rlo, rhi); rlo == rhi: none */
} spark_refine;

typedef struct spark_amr spark_amr;

spark_status spark_amr_leaves(const spark_config* cfg, const spark_refine* ref, int64_t* ncoarse, int64_t* nfine);
/* Leaves of `rank` when the leaf list is split into nranks contiguous ranges
 * (Paramesh-style distribution of the ordered leaf list): first, count. */
spark_status spark_amr_rank_leaves(const spark_config* cfg, const spark_refine* ref, int32_t rank, int32_t nranks,
                                   int64_t* first, int64_t* count);
spark_status spark_amr_required_bytes(const spark_config* cfg, const spark_refine* ref, size_t* bytes);
/* arena: device memory of >= required bytes (256-byte aligned), caller-owned. */
spark_status spark_amr_init(const spark_config* cfg, const spark_refine* ref, int32_t device, void* cuda_stream,
                            void* arena, size_t arena_bytes, spark_amr** out);
/* Virtual ranks on one device (testing the multi-rank path): nranks members,
 * each owning its range of leaves (spark_amr_rank_leaves) with its own state
 * U[v][local leaf][cells] in arenas[r] (>= spark_amr_group_required_bytes).
 * Per stage the guard values a member needs from another member's leaves are
 * packed by their owner (copy or restriction) and copied over; per step the
 * fine-face fluxBuff values a coarse cell's correction needs likewise
 * (communicate_fluxes).  The result is bitwise that of one rank. */
spark_status spark_amr_group_required_bytes(const spark_config* cfg, const spark_refine* ref, int32_t nranks,
                                            size_t* bytes);
spark_status spark_amr_init_local_group(const spark_config* cfg, const spark_refine* ref, int32_t nranks,
                                        int32_t device, void* cuda_stream, void* const* arenas, size_t arena_bytes,
                                        spark_amr** outs);
/* One composite step of all members of a local group (failure: all or none roll back). */
spark_status spark_amr_step_group(spark_amr* const* amrs, int32_t n, double dt, double t_end, double* dt_used);
spark_status spark_amr_finalize(spark_amr* amr);
const char* spark_amr_last_error(const spark_amr* amr);
/* Load U[v][leaf][cells] (host or device); resets t and the step count. */
spark_status spark_amr_set_state(spark_amr* amr, const double* U, int32_t on_device);
/* Copy U^n out; synchronises; SPARK_ERR_NONPHYSICAL if the failure word is set. */
spark_status spark_amr_get_state(spark_amr* amr, double* U, int32_t on_device);
/* Materialise the padded leaves P[v][leaf][padded cells] (device pointer) of
 * U^n with the coarse-fine guard rules; edge/corner guards NaN.  Asynchronous. */
spark_status spark_amr_fill_guardcells(spark_amr* amr, double* padded_out);
/* One composite SSP-RK step (dt / t_end / dt_used as spark_step). */
spark_status spark_amr_step(spark_amr* amr, double dt, double t_end, double* dt_used);
spark_status spark_amr_get_time(spark_amr* amr, double* t, int64_t* steps, double* dt_last);

#ifdef __cplusplus
}
#endif
#endif /* SPARK_H */
