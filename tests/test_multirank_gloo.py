"""Multi-rank host logic on CPU, world_size 2 over gloo (no GPU).

libspark's rank decomposition and halo plan (spark_rank_grid / spark_rank_box /
spark_halo_plan), the slab layout and the NCCL message order of
spark_api.cpp::exchange_nccl (per dim: send high slab -> high peer, recv low
halo <- low peer, send low slab -> low peer, recv high halo <- high peer) are
exercised with real point-to-point messages between two processes.  Each rank
then runs one oracle stage on its own blocks with the received halos, and the
result must equal the single-domain stage bit for bit (guard cells are exact
copies); the global dt minimum is an all-reduce(min).  The same plan and order
drive the NCCL path on GPUs (P:1542-1546 guard fill, P:1586 p2p exchange)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import spark_inputs as si
from paper_2401_03378_b200 import build as spark_build
from paper_2401_03378_b200 import spark

CASES = [
    # 3-D, split along one dim, outflow + reflect
    si.Problem("g3", 3, (4, 4, 4), (2, 2, 4), 3, 2, 1, 3, 0.3, bc=((1, 2), (1, 1), (1, 1))),
    # 3-D, periodic in the split dim with P = 2 (both faces peer the same rank)
    si.Problem("g3p", 3, (4, 4, 4), (2, 2, 2), 2, 1, 1, 2, 0.3, bc=((0, 0), (0, 0), (0, 0))),
    # 2-D Sod-like, periodic y
    si.Problem("g2", 2, (8, 8, 1), (2, 4, 1), 2, 1, 0, 2, 0.4, bc=((1, 1), (0, 0), (1, 1))),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bc_index(g, N, lo, hi):
    """Per-dimension boundary map (reading R4) for guard indices outside [0, N)."""
    if 0 <= g < N:
        return g, False
    bc = lo if g < 0 else hi
    if bc == si.BC_PERIODIC:
        return g % N, False
    if bc == si.BC_OUTFLOW:
        return (0 if g < 0 else N - 1), False
    return (-1 - g if g < 0 else 2 * N - 1 - g), True


def _rank_extended(p, cfg, rank, nranks, G, recv):
    """Rank sub-box with ng-thick face guards: interior from the local data, rank
    faces from the received slabs, physical faces from the boundary map."""
    lo, n = spark.rank_box(cfg, rank, nranks)
    ng = p.ng
    gd = [ng if d < p.ndim else 0 for d in range(3)]
    c0 = [lo[d] * p.nb[d] for d in range(3)]
    cn = [n[d] * p.nb[d] for d in range(3)]
    N = [p.nblk[d] * p.nb[d] for d in range(3)]
    E = np.full((p.nvar, cn[2] + 2 * gd[2], cn[1] + 2 * gd[1], cn[0] + 2 * gd[0]), np.nan)
    local = G[:, c0[2]:c0[2] + cn[2], c0[1]:c0[1] + cn[1], c0[0]:c0[0] + cn[0]]  # this rank's own data only
    E[:, gd[2]:gd[2] + cn[2], gd[1]:gd[1] + cn[1], gd[0]:gd[0] + cn[0]] = local
    plans = {(f["dim"], f["side"]): f for f in spark.halo_plan(cfg, rank, nranks)}
    for d in range(p.ndim):
        for side in (0, 1):
            f = plans[(d, side)]
            ax = 3 - d  # array axis of dim d in [v][z][y][x]
            sl = [slice(None)] + [slice(gd[2 - e], gd[2 - e] + cn[2 - e]) for e in range(3)]
            sl[ax] = slice(0, ng) if side == 0 else slice(gd[d] + cn[d], gd[d] + cn[d] + ng)
            if f["peer"] >= 0:
                ext = [cn[2], cn[1], cn[0]]
                ext[2 - d] = ng
                E[tuple(sl)] = recv[(d, side)].reshape((p.nvar,) + tuple(ext))
            else:  # physical boundary (or periodic self-wrap): map into the local box
                for m in range(ng):
                    gl = c0[d] - ng + m if side == 0 else c0[d] + cn[d] + m
                    src, flip = _bc_index(gl, N[d], *p.bc[d])
                    li = src - c0[d]
                    assert 0 <= li < cn[d], "boundary maps must stay inside the sub-box"
                    dst = list(sl)
                    dst[ax] = (m if side == 0 else gd[d] + cn[d] + m)
                    srcsl = [slice(None)] * 4
                    srcsl[ax] = li
                    vals = local[tuple(srcsl)].copy()
                    if flip:
                        vals[1 + d] = -vals[1 + d]
                    E[tuple(dst)] = vals
    return E, lo, n


def _pack(p, cfg, rank, nranks, G, d, side):
    lo, n = spark.rank_box(cfg, rank, nranks)
    c0 = [lo[e] * p.nb[e] for e in range(3)]
    cn = [n[e] * p.nb[e] for e in range(3)]
    sl = [slice(None)] + [slice(c0[2 - e], c0[2 - e] + cn[2 - e]) for e in range(3)]
    a = c0[d] if side == 0 else c0[d] + cn[d] - p.ng
    sl[3 - d] = slice(a, a + p.ng)
    return np.ascontiguousarray(G[tuple(sl)]).ravel()


def _worker(rank, nranks, port, case_idx, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=nranks)
        import torch

        p = CASES[case_idx]
        cfg = p.config()
        U = oracle.prim_to_cons(p.ndim, p.gamma, si.random_state(p, 31, blocky=True))
        G = si.to_global(p, U)  # every rank reads only its own sub-box of it
        plans = {(f["dim"], f["side"]): f for f in spark.halo_plan(cfg, rank, nranks)}
        recv = {}
        # message order of exchange_nccl
        for d in range(p.ndim):
            reqs = []
            order = [("send", 1), ("recv", 0), ("send", 0), ("recv", 1)]
            for kind, side in order:
                f = plans[(d, side)]
                if f["peer"] < 0:
                    continue
                if kind == "send":
                    t = torch.from_numpy(_pack(p, cfg, rank, nranks, G, d, side))
                    assert t.numel() == p.nvar * f["cells"]
                    reqs.append(dist.isend(t, f["peer"]))
                else:
                    t = torch.empty(p.nvar * f["cells"], dtype=torch.float64)
                    recv[(d, side)] = t
                    reqs.append(dist.irecv(t, f["peer"]))
            for r in reqs:
                r.wait()
        recv = {k: v.numpy() for k, v in recv.items()}
        # halos are exact copies of the neighbour's cells (global map)
        E, lo, n = _rank_extended(p, cfg, rank, nranks, G, recv)
        # one oracle stage on this rank's blocks with these guards
        nb = p.nb
        # the rank's own sub-domain (cell counts are powers of two: dx is exact)
        dxs = [(p.hi[d] - p.lo[d]) / (p.nblk[d] * nb[d]) for d in range(3)]
        q_ = p.with_(nblk=tuple(n), lo=tuple(p.lo[d] + lo[d] * nb[d] * dxs[d] for d in range(3)),
                     hi=tuple(p.lo[d] + (lo[d] + n[d]) * nb[d] * dxs[d] for d in range(3)))
        gd = [p.ng if d < p.ndim else 0 for d in range(3)]
        P = np.empty((p.nvar, n[0] * n[1] * n[2], nb[2] + 2 * gd[2], nb[1] + 2 * gd[1], nb[0] + 2 * gd[0]))
        for bz in range(n[2]):
            for by in range(n[1]):
                for bx in range(n[0]):
                    b = bx + n[0] * (by + n[1] * bz)
                    P[:, b] = E[:, bz * nb[2]:bz * nb[2] + nb[2] + 2 * gd[2],
                                by * nb[1]:by * nb[1] + nb[1] + 2 * gd[1],
                                bx * nb[0]:bx * nb[0] + nb[0] + 2 * gd[0]]
        c0 = [lo[d] * nb[d] for d in range(3)]
        cn = [n[d] * nb[d] for d in range(3)]
        Uloc = si.from_global(q_, np.ascontiguousarray(
            G[:, c0[2]:c0[2] + cn[2], c0[1]:c0[1] + cn[1], c0[0]:c0[0] + cn[0]]))
        dt = 1e-3
        out = oracle.stage_padded(q_.config(), P, Uloc, 0.0, 1.0, dt)
        ref = si.to_global(p, oracle.stage(cfg, U, U, 0.0, 1.0, dt))
        refloc = ref[:, c0[2]:c0[2] + cn[2], c0[1]:c0[1] + cn[1], c0[0]:c0[0] + cn[0]]
        same = bool(np.array_equal(si.to_global(q_, out), refloc))
        # global dt: all-reduce(min) of the per-rank CFL minimum
        m = torch.tensor([oracle.dt_raw(q_.config(), Uloc)], dtype=torch.float64)
        dist.all_reduce(m, op=dist.ReduceOp.MIN)
        dt_ok = float(m.item()) == oracle.dt_raw(cfg, U)
        q.put((rank, same, dt_ok, sorted(recv)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback

        q.put((rank, False, False, traceback.format_exc()))


@pytest.fixture(scope="module", autouse=True)
def built():
    spark_build.build()


@pytest.mark.parametrize("case_idx", range(len(CASES)), ids=[c.name for c in CASES])
def test_two_rank_halo_exchange_and_stage(case_idx):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case_idx, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, same, dt_ok, info in sorted(res, key=lambda x: x[0]):
        assert same, f"rank {rank}: stage with exchanged halos differs from 1-rank stage: {info}"
        assert dt_ok, f"rank {rank}: dt all-reduce mismatch"
        assert isinstance(info, list) and len(info) > 0, info
