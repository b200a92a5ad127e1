#!/usr/bin/env python
"""Benchmark of the tau-preconditioned GMRES hot path (arXiv 2404.10221) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C5]

A *step* is one Crank-Nicolson time step of the BASELINE.json headline workload (configs[4],
"C5": 3D 511^3, alpha=(1.1,1.5,1.9), kappa=(1,.5,2), e=1.5+0.5 tanh(5(x-1/2))e^{-t}, M=4,
GMRES(20), tol 1e-8): the preconditioned residual and the full GMRES solve of Eq.(tls), all
in librsfde.so kernels.  Steps cycle through m = 0..M-1 (u reset to psi = 0 at m = 0).

Output: ONE JSON line on rank 0 with the metric of BASELINE.json (unknown-iterations/s =
N * (sum of GMRES iterations) / device time; plus seconds per CN step), the e2e figure
through the C ABI with host buffers, the live roofline of the dominant kernel class, the CPU
oracle baseline and the SM clocks seen during the timed region.

Multi-GPU (torchrun, one process per GPU, N > 1): the 3D grid is slab-sharded along x_1 over the
N ranks (rsfde_team_*: NCCL all-to-all transposes for the x_1 transforms, allreduce of the CGS2
dots) -- strong scaling of the same problem; value = N_unknowns * iterations / max-over-ranks
device time.  The ranks run independent
replicas only with --replicas; a failing sharded run exits non-zero (no silent fallback).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = None
with open(os.path.join(ROOT, "BASELINE.json")) as _f:
    METRIC = json.load(_f)["metric"]
UNIT = "unknown-iterations/s"


# ----------------------------------------------------------------------------- helpers
def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(value: float, ws: int, device=None) -> float:
    """max of a float over ranks (identity for one process)."""
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, ws: int, device=None) -> float:
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "power.draw"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[6]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def l2_note(prob) -> str:
    """What the timed region does about L2 (timing rule: flush or inputs larger than L2)."""
    vec = 8.0 * prob.N
    if vec > 126e6:
        return f"no flush: every vector ({vec / 1e9:.2f} GB) is larger than the 126 MB L2"
    return (f"no flush: a vector is {vec / 1e6:.3g} MB and the working set of a step is L2-resident by design "
            "(SURVEY 8(d): latency/launch-bound config, not an HBM roofline line)")


def build_problem(workload: str):
    from paper_2404_10221_b200 import inputs as I
    if workload == "C5":
        return I.config_c5()
    if workload == "C4":
        return I.config_c4()
    if workload == "C3":
        return I.config_c3()
    if workload == "C2":
        return I.config_c2()
    if workload == "C1":
        return I.config_c1()
    if workload.startswith("C5:"):      # reduced C5 for quick runs, e.g. C5:127
        n = int(workload.split(":")[1])
        return I.config_c5(n=n)
    raise ValueError(workload)


WORKLOAD_TEXT = {
    "C1": "C1 = BASELINE configs[0]: 1D n=255, alpha=1.5, kappa=1, e=1+0.5 sin(pi x) e^-t, M=64, manufactured "
          "u=e^-t x^2(1-x)^2, GMRES(50) tol 1e-10",
    "C2": "C2 = BASELINE configs[1]: 2D 255^2, alpha=(1.3,1.7), kappa=(1,2), e=2+xy sin t, M=32, seeded + "
          "manufactured source, GMRES(50) tol 1e-10",
    "C3": "C3 = BASELINE configs[2]: 2D 2047^2 (4.19M unknowns), alpha=(1.2,1.9), kappa=(1,1), "
          "e=1+0.9 exp(-10((x-.5)^2+(y-.5)^2))(1+t), M=16, seeded source, GMRES(50) tol 1e-9",
    "C4": "C4 = BASELINE configs[3]: 3D 255^3 (16.6M unknowns), alpha=1.5^3, kappa=1^3, "
          "e=1+0.5 prod sin(pi x_i) cos t, M=8, seeded source, GMRES(30) tol 1e-9",
    "C5": "C5 = BASELINE configs[4]: 3D (0,1)^3, n=511^3 (133,432,831 unknowns), alpha=(1.1,1.5,1.9), "
          "kappa=(1,0.5,2), e=1.5+0.5*tanh(5(x-0.5))*exp(-t), M=4 CN steps, seeded uniform[-1,1] source, "
          "GMRES(20) tol 1e-8, one-sided tau preconditioner",
}


# ----------------------------------------------------------------------------- CPU oracle sample
def oracle_iteration_sample(prob, nbasis: int = 4):
    """One GMRES iteration of the oracle (Tier L, literal one-sided system): K v = P^{-1} A~ v
    plus modified Gram-Schmidt against ``nbasis`` basis vectors.  Returns (seconds, threads)."""
    from oracle import scheme
    from oracle.lines import LineSystem
    from paper_2404_10221_b200 import inputs as I
    try:
        from threadpoolctl import threadpool_info
        threads = max([int(i.get("num_threads", 1)) for i in threadpool_info()] or [os.cpu_count()])
    except Exception:
        threads = os.cpu_count()
    Ls = LineSystem(prob.d, prob.n, prob.alpha, prob.kappa, prob.tau)
    ebar = 0.5 * (prob.e_grid(prob.t_half(0)).max() + prob.e_grid(prob.t_half(0)).min())
    e = prob.e_grid(prob.t_half(0))
    v = I.seeded_vector(11, prob.n)
    V = [v / np.linalg.norm(v)] + [I.seeded_vector(12 + i, prob.n) for i in range(nbasis - 1)]
    t0 = time.perf_counter()
    w = Ls.P_alpha_inv(ebar, Ls.A_tilde(e, V[0]))
    for b in V:
        h = float(np.vdot(w, b))
        w = w - h * b
    nrm = float(np.linalg.norm(w))
    _ = w / nrm
    return time.perf_counter() - t0, threads


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on the host cores (rank 0 only)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from paper_2404_10221_b200 import inputs as I
    prob = build_problem(args.workload)
    N = prob.N
    small = I.config_c5(n=63)
    for _ in range(args.warmup):
        oracle_iteration_sample(small)
    times = []
    threads = os.cpu_count()
    for _ in range(args.steps):
        t, threads = oracle_iteration_sample(prob)
        times.append(t)
    tot = sum(times)
    value = N * len(times) / tot
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": WORKLOAD_TEXT.get(args.workload, args.workload)},
           "step_definition": "one bounded sample = ONE GMRES iteration of the oracle on the full grid of the "
                              "workload (not a whole CN step: a C5 CN step is 7-8 such iterations plus the "
                              "right-hand side); ms_per_step is per sample",
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                            "sample": "per step: one GMRES iteration of the oracle (Tier L dense per-line "
                                      "operators: K v = P_alpha^-1 A~ v + MGS vs 4 basis vectors) on the "
                                      f"full {args.workload} grid"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2404_10221_b200.solver import RsfdeSolver

    prob = build_problem(args.workload)
    N = prob.N
    t_setup = time.perf_counter()
    S = RsfdeSolver.from_problem(prob)
    # F (static for C3-C5) built on the device from f on the closed grid
    steps_F = [0] if prob.source_static else list(range(prob.M))
    Fs = [S.compact_source(torch.from_numpy(prob.f_closed(prob.t_half(m))).to(dev)) for m in steps_F]
    u = torch.zeros(prob.n, dtype=torch.float64, device=dev)
    u0 = torch.from_numpy(prob.psi_interior()).to(dev)
    cfg = S.cfg(restart=prob.restart, tol=prob.tol)
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()

    def step(i, uu, host=False, reset=True):
        m = i % prob.M
        if m == 0 and reset:
            if host:
                uu[...] = u0.cpu().numpy()
            else:
                uu.copy_(u0)
        F = Fs[0] if prob.source_static else Fs[m]
        if host:
            F = F_host if prob.source_static else F_host_steps[m]
        rep = S.solve_steps(uu, F=F, F_static=True, m_begin=m, m_count=1, cfg=cfg)
        if not rep["converged"][0]:
            raise RuntimeError(f"GMRES did not converge at step m={m}: {rep}")
        return rep["iters"][0]

    Fstack = Fs[0] if prob.source_static else torch.stack(Fs)

    def march(uu, K):
        """K CN steps from psi through the march API (one rsfde_solve_steps call per <= M steps; the
        state is reset to psi between calls when K > M).  The caller resets uu to psi beforehand."""
        its, k = [], 0
        while k < K:
            cnt = min(K - k, prob.M)
            if k > 0:
                uu.copy_(u0)
            F = Fstack if prob.source_static else Fstack[:cnt]
            rep = S.solve_steps(uu, F=F, F_static=bool(prob.source_static), m_begin=0, m_count=cnt, cfg=cfg)
            if not all(rep["converged"]):
                raise RuntimeError(f"GMRES did not converge: {rep}")
            its += rep["iters"]
            k += cnt
        return its

    u.copy_(u0)
    march(u, args.warmup)
    torch.cuda.synchronize()
    # ---------------- device-timed region (inputs resident in HBM; vectors > L2).  The library's
    # per-launch profiling events are off here (they cost a few microseconds per launch, which matters
    # for the launch-bound C1/C2); the same K steps are then re-run with them on for the roofline and
    # the kernel breakdown (second timed region, also CUDA events on the launching stream).
    u.copy_(u0)
    S.launch_count(reset=True)
    clocks = ClockSampler(local)
    barrier(ws)
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    iters = march(u, args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    clk = clocks.stop()
    launches = S.launch_count(reset=True)
    t_dev = e0.elapsed_time(e1) * 1e-3
    # profiled re-run of the same steps (roofline / breakdown)
    u.copy_(u0)
    S.profile(True)
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    march(u, args.steps)
    p1.record(stream)
    torch.cuda.synchronize()
    prof = S.profile_read()
    S.profile(False)
    t_prof = p0.elapsed_time(p1) * 1e-3
    t_max = max_over_ranks(t_dev, ws, dev)
    unk_its = sum_over_ranks(float(N * sum(iters)), ws, dev)
    value = unk_its / t_max

    # ---------------- e2e through the C ABI with host buffers (pinned), copies timed
    e2e = None
    if not args.no_e2e:
        global F_host, F_host_steps
        F_host = Fs[0].cpu().numpy() if prob.source_static else None
        F_host_steps = [f.cpu().numpy() for f in Fs] if not prob.source_static else None
        pin = torch.empty(prob.n, dtype=torch.float64).pin_memory()
        u_host = pin.numpy()
        pinF = torch.from_numpy(F_host).pin_memory() if F_host is not None else None
        F_host = pinF.numpy() if pinF is not None else None
        # march from psi with consecutive steps m = 0, 1, ... (u stays in the host buffer between the
        # calls); the psi reset of the device-timed loop is host work that is not part of a step, so
        # it is done before the clock starts and only repeats if K > M
        psi_host = u0.cpu().numpy()
        u_host[...] = psi_host
        barrier(ws)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_iters = []
        for k in range(args.steps):
            if k > 0 and k % prob.M == 0:
                u_host[...] = psi_host
            e_iters.append(step(k, u_host, host=True, reset=False))
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0, ws, dev)
        e2e = {"value": sum_over_ranks(float(N * sum(e_iters)), ws, dev) / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": int(2 * N * 8), "d2h_bytes_per_step": int(N * 8),
               "how": "rsfde_solve_steps with pinned host u and F: H2D of u and F, D2H of u inside the call, "
                      "host wall clock around the calls after a device synchronize"}

    if rank != 0:
        return 0
    # ---------------- roofline of the dominant kernel class
    peak, peak_src = measured_peaks()
    heavy = {k: v for k, v in prof.items() if k != "small" and v["ms"] > 0}
    dom = max(heavy, key=lambda k: heavy[k]["ms"]) if heavy else None
    roof = None
    if dom:
        d = prof[dom]
        achieved = d["bytes"] / (d["ms"] * 1e-3) / 1e9
        # DRAM bytes per launch of this kernel class from the committed ncu --set full capture of the
        # C5 K chain (newest profiles/rNN_ncu_traffic.json, tools/ncu_traffic.py); null for other workloads
        traffic, traffic_src = None, None
        cands = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_ncu_traffic.json"))
        tp = os.path.join(ROOT, "profiles", cands[-1]) if cands else ""
        if cands and args.workload == "C5":
            with open(tp) as f:
                tj = json.load(f)
            if dom in tj:
                traffic, traffic_src = tj[dom]["bytes_per_launch"], tj.get("source")
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                "launches": d["launches"], "mean_launch_ms": d["ms"] / max(1, d["launches"]),
                "algorithmic_bytes_per_launch": d["bytes"] / max(1, d["launches"])}
        if dom == "oper_pass_spectral" and prob.d == 3 and len(set(prob.n)) == 1:
            # the same kernel against the FP64 pipe: algorithmic FFT work =
            # 5 L log2 L flops per complex pair-FFT of L = 2(n+1); a K chain's d operator passes hold
            # 3 (non-last) or 4 (last) pair-FFTs per pencil pair; nominal peak = 64 FP64 FMA/clk/SM
            n1 = prob.n[0] + 1
            Lf = 2 * n1
            pairs = (prob.n[0] * n1) // 2        # pencils per pass: n x (n+1) (one axis padded)
            ffts = (3 * (prob.d - 1) + 4) / prob.d
            flops = pairs * ffts * 5 * Lf * math.log2(Lf)
            sm_hz = ((clk or {}).get("sm_mhz") or 1965.0) * 1e6
            fp64_peak = 2 * 64 * torch.cuda.get_device_properties(dev).multi_processor_count * sm_hz / 1e12
            ach = flops / (d["ms"] / max(1, d["launches"]) * 1e-3) / 1e12
            roof["fp64"] = {"bound": "alu", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                            "frac": ach / fp64_peak,
                            "note": "secondary: algorithmic 5 L log2 L flops per pair-FFT vs nominal FP64 peak "
                                    "(64 FMA/clk/SM x 2 x SMs x SM clock)"}
    # solve-level (SURVEY 8(d) fractions 2 and 3): the algorithmic pass-model bytes of every launch of
    # the profiled K steps over the device time of the timed region
    tot_bytes = sum(v["bytes"] for v in prof.values())
    solve = {"algorithmic_bytes_per_step": tot_bytes / args.steps,
             "achieved": tot_bytes / t_dev / 1e9, "peak": peak, "unit": "GB/s",
             "frac": tot_bytes / t_dev / 1e9 / peak,
             "scope": "all kernels of a CN step: pass-model bytes (DESIGN.md section 6) / device time"}
    tot_ms = sum(v["ms"] for v in prof.values()) or 1.0
    breakdown = {k: {"share": v["ms"] / tot_ms, "ms": v["ms"], "launches": v["launches"],
                     "GBps": (v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["ms"] > 0 and v["bytes"] > 0 else None}
                 for k, v in prof.items() if v["launches"]}
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        t, threads = oracle_iteration_sample(prob)
        cpu = {"value": N / t, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"one GMRES iteration of the oracle on the full {args.workload} grid (Tier L per-line "
                         "dense operators: K v = P_alpha^-1 A~ v + MGS vs 4 basis vectors), timed once",
               "seconds": t}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_max / args.steps, "seconds_per_cn_step": t_max / args.steps,
        "profiled_ms_per_step": 1e3 * t_prof / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD_TEXT.get(args.workload, args.workload), "n": list(prob.n),
                   "M": prob.M, "restart": prob.restart, "tol": prob.tol, "unknowns": N,
                   "parallelism": "replicas" if ws > 1 else "single GPU",
                   "l2": l2_note(prob), "iters_per_step": iters},
        "e2e": e2e, "gpu_launches": launches, "roofline": roof, "solve_level": solve,
        "kernel_breakdown": breakdown, "cpu_baseline": cpu, "clocks": clk, "setup_seconds": setup_s,
        "device_bytes": S.device_bytes(),
    }
    print(json.dumps(out), flush=True)
    S.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


F_host = None
F_host_steps = None


def sharded_roofline(prob, ws, iters, t_max):
    """Solve-level roofline of a slab-sharded run (per rank, algorithmic pass model of DESIGN.md section 8):
    HBM bytes per GMRES iteration at Arnoldi index j = vec_r (14 + 2j + 6) for the K chain and DCGS2
    plus 6 vec_r for the exchanges (fused: pack A->T of the two channels, unpack T->A of the result; the
    x1 pass reads and writes the all-to-all blocks itself); NVLink bytes = 3 vec_r (P-1)/P per rank."""
    hbm, src = measured_peaks()
    vec_r = 8.0 * prob.N / ws
    nit = sum(iters)
    hbm_bytes = nvl_bytes = 0.0
    for k in iters:
        for j in range(k):
            hbm_bytes += vec_r * (14 + 2 * j + 6 + 6)
            nvl_bytes += 3 * vec_r * (ws - 1) / ws
    ach = hbm_bytes / t_max / 1e9
    nvl = nvl_bytes / t_max / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": None,
            "scope": "solve-level per rank, algorithmic pass-model bytes / device time (not a single kernel)",
            "peak_source": src, "iterations": nit,
            "nvlink": {"achieved": nvl, "peak": 900.0, "unit": "GB/s", "frac": nvl / 900.0,
                       "bytes_per_iteration_per_rank": 3 * vec_r * (ws - 1) / ws,
                       "peak_source": "NVLink 5 nominal 900 GB/s per direction per GPU"}}


def run_sharded(args):
    """N > 1: one C5 grid slab-sharded along x_1 over the ranks (strong scaling)."""
    import torch
    import torch.distributed as dist
    ws, rank, local = _dist()
    dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2404_10221_b200.solver import RsfdeSolver, RsfdeTeam
    prob = build_problem(args.workload)
    if prob.d != 3 or (prob.n[0] + 1) % ws or (prob.n[1] + 1) % ws:
        raise RuntimeError("sharding needs a 3D grid with N | n1+1 and N | n2+1")
    obj = [RsfdeTeam.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    t_setup = time.perf_counter()
    T = RsfdeTeam(prob, nranks=ws, rank=rank, nlocal=1, nccl_id=obj[0])
    lo, cnt = T.slab()
    f = prob.f_closed(prob.t_half(0))
    F = T.compact_source(torch.from_numpy(np.ascontiguousarray(f[lo:lo + cnt + 2])).to(dev))
    del f
    u = torch.zeros((cnt, prob.n[1], prob.n[2]), dtype=torch.float64, device=dev)
    cfg = RsfdeSolver.cfg(restart=prob.restart, tol=prob.tol)
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()

    def step(i, uu):
        m = i % prob.M
        if m == 0:
            uu.zero_()
        rep = T.solve_steps(uu, F=F, F_static=True, m_begin=m, m_count=1, cfg=cfg)
        if not rep["converged"][0]:
            raise RuntimeError(f"GMRES did not converge at step m={m}: {rep}")
        return rep["iters"][0]

    for i in range(args.warmup):
        step(i, u)
    T.launch_count(reset=True)
    clocks = ClockSampler(local)
    barrier(ws)
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    iters = [step(i, u) for i in range(args.warmup, args.warmup + args.steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    clk = clocks.stop()
    launches = T.launch_count(reset=True)
    t_max = max_over_ranks(e0.elapsed_time(e1) * 1e-3, ws, dev)
    N = prob.N
    value = N * sum(iters) / t_max
    e2e = None
    if not args.no_e2e:
        u_host = torch.zeros((cnt, prob.n[1], prob.n[2]), dtype=torch.float64).pin_memory()
        F_host = F.cpu().pin_memory()
        Fd = torch.empty_like(F)
        barrier(ws)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_iters = []
        for i in range(args.warmup, args.warmup + args.steps):
            u.copy_(u_host, non_blocking=True)
            Fd.copy_(F_host, non_blocking=True)
            m = i % prob.M
            if m == 0:
                u.zero_()
            rep = T.solve_steps(u, F=Fd, F_static=True, m_begin=m, m_count=1, cfg=cfg)
            e_iters.append(rep["iters"][0])
            u_host.copy_(u, non_blocking=True)
            torch.cuda.synchronize()
        t_e2e = max_over_ranks(time.perf_counter() - t0, ws, dev)
        e2e = {"value": N * sum(e_iters) / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": int(sum_over_ranks(float(2 * u.numel() * 8), ws, dev)),
               "d2h_bytes_per_step": int(sum_over_ranks(float(u.numel() * 8), ws, dev)),
               "how": "per rank: H2D of its slab of u and F from pinned memory, rsfde_team_solve_steps, D2H of u"}
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
            "seconds_per_cn_step": t_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT.get(args.workload, args.workload), "n": list(prob.n),
                       "M": prob.M, "restart": prob.restart, "tol": prob.tol, "unknowns": N,
                       "parallelism": f"slab x1 over {ws} ranks (NCCL all-to-all transposes, allreduce dots)",
                       "l2": "no flush: every slab vector exceeds L2 at N <= 8 for C5", "iters_per_step": iters},
            "e2e": e2e, "gpu_launches": launches, "roofline": sharded_roofline(prob, ws, iters, t_max),
            "cpu_baseline": None, "clocks": clk, "setup_seconds": setup_s,
        }
        print(json.dumps(out), flush=True)
    T.close()
    dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of sharding")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    ws = _dist()[0]
    if ws > 1 and not args.replicas:
        # no silent fallback: a broken sharded path must fail the run, not turn into replicas
        return run_sharded(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
