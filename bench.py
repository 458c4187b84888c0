#!/usr/bin/env python
"""Benchmark of the Spark block-update hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl reference]

One "step" = one full SSP-RK step (every stage: guard-cell exchange + fused
stage kernel over all blocks; the dt of the next step fused into the last
stage) of the whole synthetic workload.  N = 1: configs[3] (3-D Sedov 256^3 in
16^3 blocks, PLM + HLLC + SSP-RK2 by default; --config c4_sedov3d_weno for
WENO5/RK3).  N > 1 (torchrun, one rank per GPU): weak scaling, 256^3 per GPU,
the global block grid grown along the process grid, NCCL halo exchange + dt
all-reduce.  Prints ONE JSON line on rank 0.

metric  zone-updates/s = interior cells x RK stages x steps / time (all ranks)
value   device time (CUDA events on the library stream, barrier + sync on both
        sides, max over ranks), inputs resident in HBM; the 640 MiB state per
        copy is > L2 (126 MB), so no L2 flush is needed between steps.
e2e     same metric through the public API with HOST buffers: every step
        uploads the state from pinned host memory (spark_set_state), steps,
        and reads it back (spark_get_state).
--impl reference   the CPU oracle (oracle/, the reference arm of this tier) on
        a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import spark_inputs as si  # noqa: E402

METRIC = "zone-updates/sec (cells×RK stages) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "zone-updates/s"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def algorithmic_bytes_per_zone(p: si.Problem, stage: int) -> int:
    """HBM bytes the method itself must move per zone-update:
    stage 1 reads U^n and writes U^(1); later stages read U^(s-1) and U^n and
    write U^(s).  Halo re-reads are L2 traffic, dt is fused."""
    return (2 if stage == 1 else 3) * p.nvar * 8


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def ncu_field(name: str, key: str):
    """A per-config field of the committed ncu summary (profiles/ncu_summary.json) or None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(name, {}).get(key)
    except Exception:
        return None


def ncu_traffic(name: str):
    """dram bytes per stage-kernel launch from the committed ncu summary (or None)."""
    return ncu_field(name, "dram_bytes_per_launch")


def fp64_peak_rate():
    """Measured B200 DFMA issue rate (instr/s) from profiles/fp64_peak.json."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            return float(json.load(f)["dfma_per_s"])
    except Exception:
        return None


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 10 ms) DURING the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.err = None
        self._stop = None
        self._thr = None

    def _run(self):
        import pynvml as nv

        h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
        self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while True:
            self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            try:
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except AttributeError:
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            for bit, name in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
            if self._stop.wait(0.005):
                break

    def __enter__(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            idx = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
            if idx and idx[0].strip().isdigit():
                self.gpu = int(idx[self.gpu]) if self.gpu < len(idx) else self.gpu
            self._stop = threading.Event()
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        return self

    def __exit__(self, *a):
        if self._thr is not None:
            self._stop.set()
            self._thr.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [f"nvml unavailable: {self.err}"],
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml 5 ms"}


RECONS = {"first": 0, "plm": 1, "weno5": 2, "mc": 3, "wenoz": 4}


def problem_for(args, world: int) -> si.Problem:
    p = si.PRESETS[args.config]
    if getattr(args, "recon", None):
        r = RECONS[args.recon]
        if r != p.recon:  # a different kernel: the committed ncu figures do not apply (name changes)
            p = p.with_(name=f"{p.name}+{args.recon}", recon=r, ng=max(p.ng, 3 if r in (2, 4) else (2 if r in (1, 3) else 1)))
    if getattr(args, "grav", None):
        p = p.with_(grav=tuple(float(x) for x in args.grav.split(",")))
    if getattr(args, "riemann", None):
        r = {"hll": si.RIEMANN_HLL, "hllc": si.RIEMANN_HLLC, "hybrid": si.RIEMANN_HYBRID}[args.riemann]
        if r != p.riemann:
            p = p.with_(name=f"{p.name}+{args.riemann}", riemann=r,
                        shock_thresh=args.shock_thresh if r == si.RIEMANN_HYBRID else 0.0)
    if world > 1 and args.scaling == "weak":
        # weak scaling: 256^3 (16^3 blocks of 16^3) per GPU along a process grid
        pg = {2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}.get(world)
        if pg is None:
            pg = (1, 1, world)
        p = p.with_(nblk=tuple(p.nblk[d] * pg[d] for d in range(3)),
                    hi=tuple(p.hi[d] * pg[d] for d in range(3)))
    return p


def exchange_info(p) -> dict:
    """What the --self-exchange line moves per stage, and the wire time the same
    slabs would take between two B200s (B200_PROFILING.md: 770 GB/s measured
    peer copy per direction) — the part a one-GPU run cannot show."""
    cn = [p.nb[d] * p.nblk[d] for d in range(3)]
    slab_cells = [p.ng * int(np.prod([cn[e] for e in range(3) if e != d])) for d in range(p.ndim)]
    per_stage = 2 * p.nvar * 8 * sum(slab_cells)  # sent (= received) bytes per stage
    inner = int(np.prod([max(p.nblk[d] - 2, 0) for d in range(p.ndim)]))
    return {"path": "pack -> ncclSend/ncclRecv (to itself, the production message order) on the comm stream "
                    "-> interior blocks while the slabs travel -> boundary blocks read the received slabs; "
                    "u64 ncclAllReduce of (CFL min, failure word) per step",
            "faces": 2 * p.ndim, "bytes_per_stage": per_stage,
            "nvlink_us_per_stage_est": per_stage / 770e9 * 1e6,
            "interior_block_share": inner / int(np.prod(p.nblk[:p.ndim]))}


# ------------------------------------------------------ secondary workload
def secondary_run(name: str, steps: int, warmup: int, local: int) -> dict:
    """The other scheme of BASELINE configs[3] (which does not name the
    reconstruction): 256^3 Sedov, WENO5 + HLLC + SSP-RK3, timed the same way
    (CUDA events on the library stream, after warm-up), one GPU."""
    import torch

    from paper_2401_03378_b200 import spark

    q = si.PRESETS[name]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        s = spark.Spark(q.config(), device=local, stream=st)
        s.set_primitive(si.sedov_device(q, device=f"cuda:{local}"))
    for _ in range(warmup):
        s.step()
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        s.step()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    s.close()
    zu = q.ncells * q.rk_stages * steps
    bytes_step = sum(algorithmic_bytes_per_zone(q, k) for k in range(1, q.rk_stages + 1)) * q.ncells
    peaks, kind = measured_peaks()
    gbs = bytes_step * steps / (ms * 1e-3) / 1e9
    return {"workload": name, "value": zu / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
            "warmup": warmup, "recon": "weno5", "rk_stages": q.rk_stages,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / peaks["hbm_gbs"], "note": "whole step (FP64-bound scheme, DESIGN.md §4.3)"}}


# ------------------------------------------------------------- N3 (AMR) leg
def run_amr(args, rank: int, world: int, local: int) -> int:
    """NEXT N3 measurement: composite SSP-RK steps of the static two-level
    refinement (fluxBuff + flux correction), the config's coarse grid with the
    central blocks refined (a quarter of the block grid per dimension, at
    least one block), synthetic smooth pulse crossing the coarse-fine faces.
    One GPU (replicas only: the refined path is single-rank).  Zone-updates =
    leaf cells x RK stages; the roofline denominator is the same algorithmic
    bytes per zone-update as the uniform path (the unfused N3 kernels move
    more: padded tiles and face fluxes through HBM)."""
    import torch

    from paper_2401_03378_b200 import spark

    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    p = problem_for(args, 1)
    nd = p.ndim
    q = [max(1, p.nblk[d] // 4) if d < nd else 1 for d in range(3)]
    rlo = tuple((p.nblk[d] - q[d]) // 2 if d < nd else 0 for d in range(3))
    rhi = tuple(rlo[d] + q[d] if d < nd else 1 for d in range(3))
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        a = spark.Amr(p.config(), rlo, rhi, device=local, stream=stream)
        W = si.amr_primitive(p, rlo, rhi, "pulse")
        nl = W.shape[1]
        rho, vel, pres = W[0], W[1:1 + nd], W[-1]
        U = np.empty_like(W)
        U[0] = rho
        U[1:1 + nd] = rho * vel
        U[-1] = pres / (p.gamma - 1.0) + 0.5 * rho * np.sum(vel * vel, axis=0)
        a.set_state(U)
    cells = nl * int(np.prod(p.nb))
    for _ in range(args.warmup):
        a.step()
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            a.step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    value = cells * p.rk_stages * args.steps / (ms * 1e-3)
    peaks, peak_kind = measured_peaks()
    bps = sum(algorithmic_bytes_per_zone(p, st) for st in range(1, p.rk_stages + 1)) * cells
    achieved = bps * args.steps / (ms * 1e-3) / 1e9
    nc, nf = spark.amr_leaves(p.config(), rlo, rhi)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": p.name + "+amr", "coarse_blocks": list(p.nblk), "block": list(p.nb),
                       "refined_box": [list(rlo), list(rhi)], "leaves": {"coarse": nc, "fine": nf},
                       "cells": cells, "recon": ["first", "plm", "weno5", "plm_mc", "weno5z"][p.recon],
                       "riemann": ["hll", "hllc", "hybrid"][p.riemann], "rk_stages": p.rk_stages,
                       "ic": "smooth pulse crossing the coarse-fine faces", "path": "spark_amr_step (NEXT N3)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                         "kernel": "whole step (unfused N3 kernels)",
                         "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs"},
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    a.close()
    return 0


# ---------------------------------------------------------------- oracle leg
def host_info() -> dict:
    """CPU model and the oracle's compiler / flags."""
    import subprocess

    import oracle

    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        cc = subprocess.check_output(["gcc", "--version"], text=True).splitlines()[0]
    except Exception:  # pragma: no cover
        cc = "gcc"
    return {"cpu_model": model, "compiler": cc, "flags": " ".join(oracle.CFLAGS)}


def oracle_sample(p: si.Problem, budget_s: float, max_steps: int = 1000):
    """Time the oracle (as it stands) on a bounded sample of the workload:
    the same scheme / block shape on a 4x4x4-block (64^3) sub-grid of Sedov,
    on all host cores and on one; returns the rates, the sample state and the
    step count (for the parity check of the GPU on the same sample)."""
    import oracle

    q = p.with_(nblk=tuple(min(4, p.nblk[d]) for d in range(3)))
    U0 = oracle.prim_to_cons(q.ndim, q.gamma, si.initial_primitive(q))

    def timed(budget, cap):
        U, _ = oracle.step(q.config(), U0)  # warm-up (page-in, thread pool)
        n = 1
        t0 = time.perf_counter()
        while n < cap:
            U, _ = oracle.step(q.config(), U)
            n += 1
            if time.perf_counter() - t0 >= budget:
                break
        el = time.perf_counter() - t0
        return q.ncells * q.rk_stages * (n - 1) / el, U, n, el

    v_all, U, n, el = timed(budget_s, max_steps)
    cores = oracle.num_threads()
    oracle.set_threads(1)
    try:
        v_one = timed(budget_s / 3.0, max_steps)[0]
    finally:
        oracle.set_threads(0)
    sample = (f"{q.nb[0]}^3 blocks x {q.nblk[0]}x{q.nblk[1]}x{q.nblk[2]} ({q.ncells} cells, {q.name} scheme, "
              f"Sedov), {n - 1} timed steps, {el:.1f} s")
    return v_all, cores, sample, v_one, q, U0, U, n


def gpu_parity_on_sample(q: si.Problem, U0, Uo, nsteps: int) -> list:
    """Per conserved variable, the GPU's error against the oracle after the
    same nsteps CFL steps of the sample: max |g - o| / max|o_v| and the max
    relative error where |o| > 1e-12 max|o_v| (reading R15)."""
    from paper_2401_03378_b200 import spark

    s = spark.Spark(q.config())
    s.set_state(np.ascontiguousarray(U0))
    for _ in range(nsteps):
        s.step()
    g = s.get_state().cpu().numpy()
    s.close()
    out = []
    for v in range(Uo.shape[0]):
        scale = float(np.max(np.abs(Uo[v])))
        err = np.abs(g[v] - Uo[v])
        big = np.abs(Uo[v]) > 1e-12 * scale
        out.append({"var": v, "max_err_over_maxabs": float(err.max() / scale) if scale > 0 else float(err.max()),
                    "max_rel_err": float(np.max(err[big] / np.abs(Uo[v][big]))) if big.any() else 0.0})
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    p = problem_for(args, 1)
    import oracle

    oracle.build()
    oracle.set_threads(0)  # every host core, also under torchrun (which sets OMP_NUM_THREADS=1)
    q = p.with_(nblk=tuple(min(4, p.nblk[d]) for d in range(3)))
    U = oracle.prim_to_cons(q.ndim, q.gamma, si.initial_primitive(q))
    for _ in range(args.warmup):
        U, _ = oracle.step(q.config(), U)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        U, _ = oracle.step(q.config(), U)
    el = time.perf_counter() - t0
    zu = q.ncells * q.rk_stages * args.steps
    v = zu / el
    sample = f"{q.ncells}-cell sub-grid ({q.nblk[0]}x{q.nblk[1]}x{q.nblk[2]} blocks of 16^3) of {p.name}"
    info = host_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": p.name, "cells": p.ncells, "sampled_cells": q.ncells, "rk_stages": p.rk_stages},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": sample, **info},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # >= 0.17 s timed: enough NVML clock samples
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4_sedov3d_plm", choices=sorted(si.PRESETS))
    ap.add_argument("--graphs", action="store_true",
                    help="time spark_run (CUDA-graph replay of 3-step groups; one rank, non-telescoping)")
    ap.add_argument("--telescoping", action="store_true",
                    help="telescoping SSP-RK steps (NEXT N1; 1-D/2-D, one rank): one launch per step")
    ap.add_argument("--impl", default="spark", choices=["spark", "reference"])
    ap.add_argument("--recon", default=None, choices=["first", "plm", "weno5", "mc", "wenoz"],
                    help="override the config's reconstruction (NEXT N2: mc = PLM-MC, wenoz = WENO5-Z)")
    ap.add_argument("--grav", default=None, help="uniform gravity gx,gy,gz (grvAccel, NEXT N2)")
    ap.add_argument("--riemann", default=None, choices=["hll", "hllc", "hybrid"],
                    help="override the Riemann solver (hybrid = shockDet + HLL at shock faces, NEXT N2)")
    ap.add_argument("--shock-thresh", type=float, default=0.5, help="shockDet threshold for --riemann hybrid")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = the config's grid per GPU; strong = the config's grid split over N")
    ap.add_argument("--periodic", action="store_true",
                    help="every face periodic, wrapped inside the kernel (the reference point of --self-exchange)")
    ap.add_argument("--self-exchange", action="store_true",
                    help="N=1: periodic faces through the multi-rank path (pack -> ncclSend/Recv to itself -> "
                         "interior/boundary launches) every stage: the per-rank exchange machinery of an interior "
                         "rank, measured on one GPU")
    ap.add_argument("--amr", action="store_true",
                    help="NEXT N3: time the static two-level refinement (spark_amr_step) on the config's grid "
                         "with its central quarter of blocks per dimension refined (one GPU)")
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--e2e-chunks", type=int, default=16)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-calibration", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the WENO5/RK3 line of configs[3] added to the default run")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.amr:
        return run_amr(args, rank, world, local)

    import torch
    import torch.distributed as dist

    from paper_2401_03378_b200 import spark

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    p = problem_for(args, world)
    selfx = args.self_exchange and world == 1
    if selfx:  # every face periodic: all six go through NCCL (the faces of an interior rank)
        p = p.with_(name=p.name + "+selfx", bc=((0, 0),) * 3)
    elif args.periodic:
        p = p.with_(name=p.name + "+periodic", bc=((0, 0),) * 3)
    cfg = p.config()
    nccl_id = None
    if world > 1:
        obj = [spark.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    elif selfx:
        nccl_id = spark.nccl_unique_id()

    stream = torch.cuda.Stream()
    lo, n = spark.rank_box(cfg, rank, world)
    box = (tuple(lo[d] * p.nb[d] for d in range(3)), tuple(n[d] * p.nb[d] for d in range(3)))
    with torch.cuda.stream(stream):
        s = spark.Spark(cfg, rank, world, nccl_id=nccl_id, device=local, stream=stream)
        if p.ic == "sedov":  # built in HBM (configs[4]'s 1024^3 does not fit a host copy comfortably)
            Wd = si.sedov_device(p, box=box, device=f"cuda:{local}")
        else:
            Wd = torch.from_numpy(si.initial_primitive(p)).to(f"cuda:{local}")
        torch.cuda.synchronize()
        s.set_primitive(Wd)
        stream.synchronize()
        cells_local = int(np.prod(Wd.shape[1:]))
        del Wd
        torch.cuda.empty_cache()
    zu_per_step = p.ncells * p.rk_stages  # all ranks

    def barrier():
        if world > 1:
            dist.barrier()

    step = s.step_telescoping if args.telescoping else s.step

    # ---- warm-up
    for _ in range(args.warmup):
        step()
    stream.synchronize()

    # ---- timed region (device time on the library stream)
    # --graphs: spark_run replays CUDA graphs of 3 steps (no per-kernel events
    # then: the stage-kernel time is the step time)
    s.profile(not args.graphs)
    if args.graphs:
        s.run(3)  # capture outside the timed region
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        if args.graphs:
            s.run(args.steps)
        else:
            for _ in range(args.steps):
                step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    if args.graphs:
        stage_ms, stage_launches, total_launches = ms, args.steps * p.rk_stages, args.steps * (p.rk_stages + 1)
    else:
        stage_ms, stage_launches, total_launches = s.profile_read()
    s.profile(False)
    t_dev = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    ms = float(t_dev.item())
    value = zu_per_step * args.steps / (ms * 1e-3)

    # ---- roofline of the dominant kernel (the fused stage kernel)
    peaks, peak_kind = measured_peaks()
    if args.telescoping:  # one launch per step: read U^n, write U^(n+1) (halo re-reads are L2)
        bytes_per_launch = 2 * p.nvar * 8 * cells_local
    else:
        bytes_per_step_local = sum(algorithmic_bytes_per_zone(p, st) for st in range(1, p.rk_stages + 1)) * cells_local
        bytes_per_launch = bytes_per_step_local / p.rk_stages
    avg_launch_s = stage_ms * 1e-3 / max(stage_launches, 1)
    achieved = bytes_per_launch / avg_launch_s / 1e9
    ncu_name = p.name.replace("+selfx", "").replace("+periodic", "")  # the plain run's kernel instantiation
    traffic = ncu_traffic(ncu_name)
    traffic_note = None
    if traffic is None and p.name.startswith("c5_"):
        # configs[4] runs the same kernel instantiation as configs[3] (16^3 blocks):
        # scale the committed 256^3 capture by the cells per launch
        base = ncu_traffic(p.name.replace("c5_", "c4_"))
        if base is not None:
            traffic = base * cells_local / 256 ** 3
            traffic_note = "scaled from the c4 (256^3) ncu capture by cells per launch"
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "kernel": "stage_kernel (KB1)", "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs",
                "stage_kernel_share": (stage_ms / ms) if ms > 0 else None}
    if traffic_note:
        roofline["traffic_note"] = traffic_note
    # FP64 view (the binding unit): executed FP64 instructions
    # per zone-update (ncu, profiles/ncu_summary.json) x the kernel's zone rate,
    # against the measured DFMA issue rate (tools/fp64_peak.cu, profiles/fp64_peak.json)
    roofline_fp64 = None
    fp64_per_zone = ncu_field(ncu_name, "fp64_inst_per_zone") or ncu_field(ncu_name.replace("c5_", "c4_"),
                                                                           "fp64_inst_per_zone")
    fp64_peak = fp64_peak_rate()
    if fp64_per_zone and fp64_peak:
        zu_rate_kernel = cells_local * p.rk_stages * args.steps / (stage_ms * 1e-3)
        ach = fp64_per_zone * zu_rate_kernel
        roofline_fp64 = {"bound": "alu", "achieved": ach / 1e12, "peak": fp64_peak / 1e12,
                         "unit": "T FP64 instr/s", "frac": ach / fp64_peak,
                         "per_zone": fp64_per_zone, "source": "ncu instruction counts x live kernel time",
                         "peak_source": "builder-measured DFMA issue rate (tools/fp64_peak.cu -> "
                                        "profiles/fp64_peak.json); MEASURED_PEAKS.json has no FP64 entry"}

    # issue view: executed warp instructions per zone-update (ncu) x the kernel's
    # zone rate, against the SM issue peak (4 schedulers x 1 warp-instr/clk x 148
    # SMs at the sampled clock; B200_PROFILING.md unit counts)
    roofline_issue = None
    inst_per_zone = ncu_field(ncu_name, "inst_per_zone") or ncu_field(ncu_name.replace("c5_", "c4_"), "inst_per_zone")
    if inst_per_zone:
        zu_rate_kernel = cells_local * p.rk_stages * args.steps / (stage_ms * 1e-3)
        clk_hz = (statistics.median(clk.samples) if clk.samples else 1965.0) * 1e6
        peak_issue = 148 * 4 * clk_hz
        ach = inst_per_zone / 32.0 * zu_rate_kernel
        roofline_issue = {"bound": "issue", "achieved": ach / 1e12, "peak": peak_issue / 1e12,
                          "unit": "T warp-instr/s", "frac": ach / peak_issue, "per_zone_thread_instr": inst_per_zone}

    # ---- end to end through the public API with host buffers
    e2e = None
    nbytes_state = int(np.prod(s.shape)) * 8
    try:
        import psutil

        host_ok = psutil.virtual_memory().available > 3 * nbytes_state
    except Exception:
        host_ok = True
    if not host_ok:
        e2e = {"value": None, "unit": UNIT, "skipped": f"pinned host copy of the {nbytes_state / 2**30:.0f} GiB "
               "state would exceed a third of the host's available memory"}
    else:
        hostU = torch.empty(s.shape, dtype=torch.float64).pin_memory()
        s.get_state(out=hostU.numpy())
        if not (args.telescoping or args.graphs):  # warm-up: copy streams and events created
            s.step_host(hostU.numpy(), hostU.numpy(), nchunks=args.e2e_chunks)
            torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hu = hostU.numpy()
        for _ in range(args.e2e_steps):
            if args.telescoping or args.graphs:  # no host-buffer variant of those steps
                s.set_state(hu)
                step()
                s.get_state(out=hu)
            else:  # spark_step_host: upload, step, download, the copies pipelined in chunks
                s.step_host(hu, hu, nchunks=args.e2e_chunks)
        torch.cuda.synchronize()
        barrier()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        el = float(el.item())
        nbytes = int(np.prod(s.shape)) * 8
        e2e = {"value": zu_per_step * args.e2e_steps / el, "unit": UNIT, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": args.e2e_steps,
               "note": ("per step: spark_step_host — the state uploaded from pinned host memory, one step, "
                        "the new state downloaded to pinned host memory; the copies move in "
                        f"{args.e2e_chunks} block chunks, the previous step's download overlapping the next upload "
                        "(full-duplex PCIe); host wall clock around the steps")}
        # the bound the copies set: pinned host <-> device bandwidth for the
        # state size, each direction alone and both at once (torch copies on
        # two streams; the library is not involved)
        try:
            dev_buf = torch.empty(s.shape, dtype=torch.float64, device=f"cuda:{local}")
            host2 = torch.empty(s.shape, dtype=torch.float64).pin_memory()
            sa, sb = torch.cuda.Stream(), torch.cuda.Stream()

            def timed(fn):
                torch.cuda.synchronize()
                t = time.perf_counter()
                fn()
                torch.cuda.synchronize()
                return time.perf_counter() - t

            def up():
                with torch.cuda.stream(sa):
                    dev_buf.copy_(hostU, non_blocking=True)

            def down():
                with torch.cuda.stream(sb):
                    host2.copy_(dev_buf, non_blocking=True)

            timed(up), timed(down)
            t_up, t_down = timed(up), timed(down)
            t_both = timed(lambda: (up(), down()))
            e2e["pcie"] = {"h2d_gbs": nbytes / t_up / 1e9, "d2h_gbs": nbytes / t_down / 1e9,
                           "bidirectional_gbs": 2 * nbytes / t_both / 1e9,
                           "bound_zu_per_s": zu_per_step / (t_both + ms * 1e-3 / args.steps),
                           "note": "copies of the state size; bound = one step's zone-updates / (both "
                                   "directions at once + the device step time)"}
            del dev_buf, host2
        except Exception as exc:  # pragma: no cover - measurement aid only
            e2e["pcie"] = {"error": str(exc)}
        # simulation-style use of the API: the state stays resident; every step
        # reads its dt back (spark_step with dt_used, a synchronising call), the
        # state is uploaded once before and downloaded once after the K steps
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.set_state(hostU.numpy())
        for _ in range(args.steps):
            step(sync=True)
        s.get_state(out=hostU.numpy())
        torch.cuda.synchronize()
        barrier()
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        el = float(el.item())
        e2e["resident"] = {"value": zu_per_step * args.steps / el, "unit": UNIT,
                           "h2d_bytes_per_step": nbytes / args.steps, "d2h_bytes_per_step": nbytes / args.steps + 8,
                           "steps": args.steps}

    # ---- same-run HBM calibration: the paper's AXPY mappings (NEXT N4) on
    # 2^27-element FP64 vectors (1 GiB each, > L2): 24 bytes per element
    calib = None
    if not args.no_calibration:
        n = 1 << 27
        x = torch.ones(n, dtype=torch.float64, device=f"cuda:{local}")
        y = torch.zeros(n, dtype=torch.float64, device=f"cuda:{local}")
        calib = {}
        with torch.cuda.stream(stream):
            for var, name in spark.AXPY_VARIANTS.items():
                for _ in range(2):
                    spark.axpy(var, 0.5, x, y, stream)
                c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                c0.record(stream)
                for _ in range(5):
                    spark.axpy(var, 0.5, x, y, stream)
                c1.record(stream)
                stream.synchronize()
                calib[name] = 24.0 * n * 5 / (c0.elapsed_time(c1) * 1e-3) / 1e9
        del x, y
        roofline["peak_live_axpy"] = max(calib.values())
        roofline["frac_of_live_axpy"] = achieved / roofline["peak_live_axpy"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, v_one, q, U0s, Uos, nst = oracle_sample(p, args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
               "single_thread": {"value": v_one, "unit": UNIT, "cores": 1}, **host_info(),
               "parity_vs_gpu": {"steps": nst, "tolerance": "R15: 1e-12 |o| + 1e-15 max|o_v|",
                                 "vars": gpu_parity_on_sample(q, U0s, Uos, nst)}}

    clocks = clk.summary()
    secondary = None
    if rank == 0 and world == 1 and args.config == "c4_sedov3d_plm" and not args.no_secondary and \
            not (args.recon or args.riemann or args.grav or args.telescoping or args.graphs or args.self_exchange or args.periodic):
        secondary = secondary_run("c4_sedov3d_weno", 10, 3, local)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": p.name, "cells": p.ncells, "cells_per_gpu": cells_local,
                       "block": list(p.nb), "blocks": list(p.nblk),
                       "recon": ["first", "plm", "weno5", "plm_mc", "weno5z"][p.recon], "grav": list(p.grav),
                       "riemann": ["hll", "hllc", "hybrid"][p.riemann], "rk_stages": p.rk_stages, "ng": p.ng,
                       "parallelism": f"blocks over {world} GPU(s)", "l2": "state per copy > L2 (no flush needed)",
                       "rk_mode": "telescoping" if args.telescoping else "non-telescoping",
                       "launch": "cuda-graph (spark_run)" if args.graphs else "stream (spark_step)"},
            "roofline": roofline, "roofline_fp64": roofline_fp64, "roofline_issue": roofline_issue, "hbm_calibration_gbs": calib,
            "cpu_baseline": cpu, "e2e": e2e,
            "exchange": exchange_info(p) if selfx else None,
            "gpu_launches": total_launches,
            "clocks": clocks,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
