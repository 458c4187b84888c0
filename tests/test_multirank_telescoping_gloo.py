"""Telescoping shell exchange (NEXT N1, reading R24) with real messages between
CPU processes over gloo (no GPU): libspark's plan (spark_telescoping_plan:
peer and region size per direction, and the posting order the NCCL code
uses) is followed literally — every send and receive in that order, all with
the same tag, so messages between a pair of ranks match by order exactly as
NCCL matches them — and every received region must equal the neighbour's
cells the thick tile needs (faces, edges and corners, periodic wraps across
ranks).  Each rank assembles its sub-box with the S*NGK-thick shell exactly
as tt_gather_kernel does (own cells, the received region of the direction,
or the physical boundary map), and every shell cell must equal the global
boundary-mapped cell — so every block's thick tile, and hence its telescoping
step (one communication phase per step with a thicker halo), is
the single-domain one; tests/test_gpu_telescoping3d.py checks the latter
bitwise on the GPU with virtual ranks and NCCL self-exchange."""
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
    # periodic everywhere, P = (2, 1, 1): the same peer across both x faces
    (si.Problem("t3p", 3, (4, 4, 4), (4, 2, 2), 2, 1, 1, 2, 0.3, bc=((0, 0),) * 3), 2),
    # 4 ranks, 2 x 2 x 1, mixed boundaries: edges and corners from diagonal ranks
    (si.Problem("t3m", 3, (4, 4, 4), (4, 4, 2), 2, 1, 1, 2, 0.3, bc=((0, 0), (1, 2), (0, 0))), 4),
    # 2-D WENO5 / RK3: a 9-cell shell
    (si.Problem("t2w", 2, (10, 10, 1), (2, 2, 1), 3, 2, 1, 3, 0.4, bc=((0, 0), (0, 0), (1, 1))), 2),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _region(p, c0, cn, T, G, dir_):
    """Cells of the own sub-box on side `dir_` (G: global [v][z][y][x])."""
    c = [dir_ % 3 - 1, (dir_ // 3) % 3 - 1, dir_ // 9 - 1]
    sl = [slice(None)]
    for d in (2, 1, 0):
        if c[d] < 0:
            sl.append(slice(c0[d], c0[d] + T))
        elif c[d] > 0:
            sl.append(slice(c0[d] + cn[d] - T, c0[d] + cn[d]))
        else:
            sl.append(slice(c0[d], c0[d] + cn[d]))
    return np.ascontiguousarray(G[tuple(sl)])


def _worker(rank, nranks, port, case_idx, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=nranks)
        import torch

        p, _ = CASES[case_idx]
        cfg = p.config()
        T = p.rk_stages * p.ng  # S * NGK (ng equals the reconstruction half-width here)
        U = oracle.prim_to_cons(p.ndim, p.gamma, si.random_state(p, 61, blocky=p.recon != 2))
        G = si.to_global(p, U)  # a rank reads only its own sub-box of it
        lo, n = spark.rank_box(cfg, rank, nranks)
        c0 = [lo[d] * p.nb[d] for d in range(3)]
        cn = [n[d] * p.nb[d] for d in range(3)]
        peer, cells, ops = spark.telescoping_plan(cfg, rank, nranks)
        recv, reqs = {}, []
        for kind, d in ops:  # the posting order of spark_api.cpp::tile_exchange_nccl
            if kind == "send":
                t = torch.from_numpy(_region(p, c0, cn, T, G, d).ravel())
                assert t.numel() == p.nvar * cells[d]
                reqs.append(dist.isend(t, peer[d], tag=0))
            else:
                recv[d] = torch.empty(p.nvar * cells[d], dtype=torch.float64)
                reqs.append(dist.irecv(recv[d], peer[d], tag=0))
        for r in reqs:
            r.wait()
        # assemble the extended sub-box: own cells, received shell, boundary map
        N = [p.nblk[d] * p.nb[d] for d in range(3)]
        gd = [T if d < p.ndim else 0 for d in range(3)]
        E = np.full((p.nvar, cn[2] + 2 * gd[2], cn[1] + 2 * gd[1], cn[0] + 2 * gd[0]), np.nan)
        ok_regions = True
        for z in range(-gd[2], cn[2] + gd[2]):
            for y in range(-gd[1], cn[1] + gd[1]):
                for x in range(-gd[0], cn[0] + gd[0]):
                    loc, comp, flip = [x, y, z], [0, 0, 0], [False] * 3
                    for d in range(p.ndim):
                        v = loc[d]
                        if 0 <= v < cn[d]:
                            continue
                        side = 0 if v < 0 else 1
                        has_peer = peer[[12, 14, 10, 16, 4, 22][2 * d + side]] >= 0
                        if has_peer:
                            comp[d] = -1 if side == 0 else 1
                            loc[d] = v + T if side == 0 else v - cn[d]
                        else:  # physical boundary of the global domain
                            gv = c0[d] + v
                            bc = p.bc[d][side]
                            if bc == si.BC_PERIODIC:
                                gv %= N[d]
                            elif bc == si.BC_OUTFLOW:
                                gv = 0 if side == 0 else N[d] - 1
                            else:
                                gv = -1 - gv if side == 0 else 2 * N[d] - 1 - gv
                                flip[d] = True
                            loc[d] = gv - c0[d]
                    if comp == [0, 0, 0]:
                        val = G[:, c0[2] + loc[2], c0[1] + loc[1], c0[0] + loc[0]].copy()
                    else:
                        dir_ = (comp[0] + 1) + 3 * (comp[1] + 1) + 9 * (comp[2] + 1)
                        ext = [T if comp[d] else cn[d] for d in range(3)]
                        r = recv[dir_].numpy().reshape(p.nvar, ext[2], ext[1], ext[0])
                        val = r[:, loc[2], loc[1], loc[0]].copy()
                    for d in range(p.ndim):
                        if flip[d]:
                            val[1 + d] = -val[1 + d]
                    E[:, z + gd[2], y + gd[1], x + gd[0]] = val
        # every shell cell equals the global boundary-mapped neighbour cell
        for z in range(E.shape[1]):
            for y in range(E.shape[2]):
                for x in range(E.shape[3]):
                    g, fl = [x - gd[0] + c0[0], y - gd[1] + c0[1], z - gd[2] + c0[2]], [False] * 3
                    for d in range(p.ndim):
                        if g[d] < 0 or g[d] >= N[d]:
                            bc = p.bc[d][0 if g[d] < 0 else 1]
                            if bc == si.BC_PERIODIC:
                                g[d] %= N[d]
                            elif bc == si.BC_OUTFLOW:
                                g[d] = 0 if g[d] < 0 else N[d] - 1
                            else:
                                g[d] = -1 - g[d] if g[d] < 0 else 2 * N[d] - 1 - g[d]
                                fl[d] = True
                    want = G[:, g[2], g[1], g[0]].copy()
                    for d in range(p.ndim):
                        if fl[d]:
                            want[1 + d] = -want[1 + d]
                    if not np.array_equal(E[:, z, y, x], want):
                        ok_regions = False
        q.put((rank, ok_regions, sorted(recv)))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, False, traceback.format_exc()))


@pytest.fixture(scope="module", autouse=True)
def built():
    spark_build.build()


@pytest.mark.parametrize("case_idx", range(len(CASES)), ids=[c[0].name for c in CASES])
def test_shell_exchange_follows_the_plan(case_idx):
    p, nranks = CASES[case_idx]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, nranks, port, case_idx, q)) for r in range(nranks)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, ok, info in sorted(res, key=lambda x: x[0]):
        assert ok, f"rank {rank}: shell regions wrong or exchange failed: {info}"
        assert isinstance(info, list) and len(info) > 0, info
