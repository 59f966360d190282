"""bench.py — the B200 stress-velocity Newton-Krylov sea-ice step (BASELINE.json metric).

A "step" is one implicit time step of the configured workload: seaice_set_step (a-1:
ice strength, RHS, pi_0) followed by sv-Newton iterations (a-2..a-7: fused residual +
Jacobian assembly, GPU AMG setup, AMG-FGMRES solve, energy backtracking, v/pi update) until
||R|| <= 1e-8 ||R_0||.  Default workload: BASELINE.json configs[4] ("2048x2048 Q1 mesh,
~8.4M unknowns, seed 3, moving cyclone") — the paper's largest problem.

value = solve seconds per time step (BASELINE.json's first metric) of the whole job: the max over
ranks of the device-timed region divided by the time steps all ranks solved (weak scaling:
every rank solves an independent replica; the method has no data-path collective at this size,
DESIGN.md "Multi-GPU").  DOF * Krylov-iterations / s is reported beside it, with the Krylov
iterations per solve and the number of solves that hit krylov_maxit (capped work is not useful
work, so the iteration rate is not the headline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

from paper_2204_10822_b200 import workloads as wl

METRIC = "solve s/timestep"
UNIT = "s/timestep"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--params", default="{}", help="JSON overrides of seaice_params")
    ap.add_argument("--cpu-kernels", action="store_true",
                    help="time the oracle on config 5's four operations (CPU baseline of the kernel "
                         "microbench, SURVEY 8(d)) at a sample size, extrapolated per DOF; one JSON line")
    ap.add_argument("--sample-n", type=int, default=512)
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def reduce_timing(ms, units, world, device=None):
    """Whole-job timing over replicas: the MAX of the per-rank device-timed milliseconds and
    the SUM of the per-rank work units (each rank solves an independent replica)."""
    if world <= 1:
        return ms, units
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    u = torch.tensor([float(units)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


# ----------------------------------------------------------------------------- oracle arm
COUNTS_FILE = os.path.join(ROOT, "profiles", "r02_cfg4_counts.json")


def oracle_phases(cfg, n_sample=256, threads=None):
    """Per-phase timing of the CPU oracle (numpy/scipy fp64, oracle/) on one full sv-Newton
    iteration of the workload's generator at mesh n_sample: residual + Jacobian assembly, AMG
    setup, AMG-FGMRES(60) to 1e-8, energy line search + dual/velocity update.  threads: BLAS /
    OpenMP thread limit (threadpoolctl; None = all cores).  Returns per-phase seconds per DOF
    (Krylov: per DOF per iteration) and the sample's description."""
    from threadpoolctl import threadpool_limits
    from oracle import amg as OA
    from oracle import krylov
    from oracle.model import Problem
    prm = wl.PhysParams()
    scfg = wl.Config(cfg.name + f"_sample{n_sample}", n_sample, cfg.seed, 1, cfg.moving, cfg.kind, cfg.dt)
    inp = wl.step_inputs(scfg, 0)
    N = 2 * (n_sample + 1) ** 2
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        pb = Problem(inp, prm)
        v = pb.v_prev.copy()
        pi = pb.pi_consistent(v)
        R = pb.residual(v)
        J = pb.jacobian(v, pi, "sv")
        t1 = time.perf_counter()
        H = OA.setup(J, pb, v=v)
        t2 = time.perf_counter()
        vt, st = krylov.fgmres(lambda x: J @ x, R, lambda r: OA.vcycle(H, r), 60, 1e-8, 300)
        t3 = time.perf_counter()
        for k in range(21):
            if pb.delta_energy(v, vt, 0.5 ** k) < 0:
                break
        pi = pi + 0.5 ** k * pb.pi_tilde(v, pi, vt)
        v = v + 0.5 ** k * vt
        t4 = time.perf_counter()
    its = max(st["iters"], 1)
    ph = {"assembly_s": t1 - t0, "amg_setup_s": t2 - t1, "krylov_s": t3 - t2, "krylov_iters": st["iters"],
          "line_search_update_s": t4 - t3, "total_s": t4 - t0}
    per_dof = {"newton_fixed": (t1 - t0 + t2 - t1 + t4 - t3) / N, "krylov_it": (t3 - t2) / its / N}
    desc = (f"one full sv-Newton iteration of the CPU oracle (numpy/scipy fp64) on {cfg.name}'s generator at "
            f"n={n_sample} ({N} DOF, first iteration of step 1), timed per phase")
    return ph, per_dof, desc


def extrapolate(per_dof, N, newton, krylov):
    """Oracle seconds for one time step of N DOF with the given Newton / Krylov counts, from the
    sample's per-DOF phase costs (the oracle's phases are linear in N: vectorised element
    loops, sparse products, V-cycles; an explicitly labelled extrapolation)."""
    return N * (newton * per_dof["newton_fixed"] + krylov * per_dof["krylov_it"])


def cpu_baseline(cfg, N, newton, krylov, counts_src):
    cores = os.cpu_count()
    ph1, pd1, desc = oracle_phases(cfg, threads=1)
    phA, pdA, _ = oracle_phases(cfg, threads=None)
    v1 = extrapolate(pd1, N, newton, krylov)
    vA = extrapolate(pdA, N, newton, krylov)
    return {"value": vA, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": desc + f"; extrapolated per DOF to {cfg.name} ({N} DOF) with {newton:.1f} Newton and "
                             f"{krylov:.0f} Krylov iterations per step ({counts_src})",
            "value_1thread": v1, "phases_all_cores": phA, "phases_1thread": ph1}


def oracle_kernels(n_sample=512, threads=None):
    """CPU oracle timings of config 5's four operations (reading G24 state: v = 0, pi = 0,
    log-uniform viscosity) at mesh n_sample: residual + sv-Jacobian assembly, one SpMV (scipy
    CSR), one AMG V-cycle (Chebyshev 3), one FGMRES(30) cycle with rtol 0 (30 iterations),
    each extrapolated per DOF to n = 4096 (labelled)."""
    from threadpoolctl import threadpool_limits
    from oracle import amg as OA
    from oracle import krylov
    from oracle.model import Problem
    cfg5 = wl.CONFIGS[5]
    scfg = wl.Config(cfg5.name + f"_sample{n_sample}", n_sample, cfg5.seed, 1, cfg5.moving, cfg5.kind, cfg5.dt)
    inp = wl.step_inputs(scfg, 0)
    prm = wl.PhysParams()
    N = 2 * (n_sample + 1) ** 2
    N5 = 2 * (cfg5.n + 1) ** 2
    out = {}
    with threadpool_limits(limits=threads):
        pb = Problem(inp, prm)
        v = np.zeros(N)
        pi = np.zeros((3, 4, n_sample * n_sample))
        t0 = time.perf_counter()
        pb.residual(v)
        J = pb.jacobian(v, pi, "sv").tocsr()
        out["assembly_s"] = time.perf_counter() - t0
        x = np.random.default_rng(0).standard_normal(N)
        t0 = time.perf_counter()
        for _ in range(5):
            J @ x
        out["spmv_s"] = (time.perf_counter() - t0) / 5
        H = OA.setup(J, pb, v=v)
        t0 = time.perf_counter()
        OA.vcycle(H, x)
        out["vcycle_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        krylov.fgmres(lambda y: J @ y, x, lambda r: OA.vcycle(H, r), 30, 0.0, 30)
        out["fgmres_cycle_s"] = time.perf_counter() - t0
    scale = N5 / N
    return {"sample_n": n_sample, "sample_dof": N, "threads": threads or os.cpu_count(),
            "measured_s": out, "extrapolated_to_cfg5_s": {k: v * scale for k, v in out.items()},
            "note": "oracle (numpy/scipy fp64) timed at the sample size, scaled by DOF ratio "
                    f"{scale:.1f} to config 5 (n = 4096): a labelled extrapolation (SURVEY 8(d))"}


def run_reference(a, rank, world):
    if rank != 0:
        return
    cfg = wl.CONFIGS[a.config]
    N = 2 * (cfg.n + 1) ** 2
    cores = os.cpu_count()
    # counts per step of this workload: the product path's, recorded by bench.py on the B200
    c = json.load(open(COUNTS_FILE)) if os.path.exists(COUNTS_FILE) else {}
    newton = c.get("newton_per_step", 16.0)
    krylov = c.get("krylov_per_step", 1600.0)
    src = f"counts from {os.path.relpath(COUNTS_FILE, ROOT)}" if c else "assumed counts"
    for _ in range(a.warmup):
        oracle_phases(cfg)
    vals = []
    desc = ""
    for _ in range(a.steps):
        ph, pd, desc = oracle_phases(cfg)
        vals.append(extrapolate(pd, N, newton, krylov))
    val = float(np.mean(vals))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * val, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "sample_n": 256},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": desc + f"; extrapolated to {cfg.name} ({N} DOF), {newton} Newton / "
                                              f"{krylov} Krylov iterations per step ({src})"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
BYTES_NOTE = {
    "cheb0": "finest-level Chebyshev steps: symmetric stencil, 19 fp64 per node (152 B/node, stencil.cuh) + vector traffic per variant",
}


def run_ours(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2204_10822_b200.seaice import SeaIce

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = wl.CONFIGS[a.config]
    n = cfg.n
    ctx = SeaIce(n, **json.loads(a.params))
    N, Nc = ctx.N, ctx.Nc
    h_np, A_np = wl.ice_fields(cfg)
    vo_np = wl.ocean_nodal(n)
    total = a.warmup + a.steps
    winds = [wl.wind_nodal(n, (s + 1) * cfg.dt, cfg.moving) for s in range(total)]
    h = torch.tensor(h_np, device=dev)
    A = torch.tensor(A_np, device=dev)
    vo = torch.tensor(vo_np, device=dev)
    va = [torch.tensor(w, device=dev) for w in winds]
    v = torch.zeros(N, dtype=torch.float64, device=dev)
    v_out = torch.zeros_like(v)
    for s in range(a.warmup):
        v_out, st = ctx.solve_step(cfg.dt, (s + 1) * cfg.dt, h, A, v, va[s], vo, v_out)
        v, v_out = v_out, v
    v_start = v.clone()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region (no per-kernel events: the V-cycle runs as a CUDA graph)
    stats = []
    launches0 = ctx.launches
    barrier()
    with Clocks(local_rank) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(a.warmup, total):
            v_out, st = ctx.solve_step(cfg.dt, (s + 1) * cfg.dt, h, A, v, va[s], vo, v_out)
            v, v_out = v_out, v
            stats.append(st)
        e1.record()
        barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launches - launches0
    # ---- profiled replay of the same steps: CUDA events around every launch of each kernel
    # class (eager V-cycle), for the per-kernel achieved bandwidth / roofline
    vp = v_start.clone()
    vq = torch.zeros_like(vp)
    ctx.profile(True)
    barrier()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record()
    for s in range(a.warmup, total):
        vq, _ = ctx.solve_step(cfg.dt, (s + 1) * cfg.dt, h, A, vp, va[s], vo, vq)
        vp, vq = vq, vp
    p1.record()
    barrier()
    ms_prof = p0.elapsed_time(p1)
    prof = ctx.profile_read()
    ctx.profile(False)
    kry = sum(s["krylov_iters_total"] for s in stats)
    ms_max, kry_all = reduce_timing(ms, float(kry), world, dev)
    steps_all = a.steps * world
    value = ms_max / 1e3 / steps_all                     # whole-job seconds per time step
    dof_its = float(N) * kry_all / (ms_max / 1e3)       # DOF * Krylov iterations / s (all ranks)

    # ---- end-to-end through the host-buffer C-ABI call (same steps again)
    e2e = None
    if not a.no_e2e:
        pin = lambda x: torch.tensor(x, dtype=torch.float64).pin_memory()
        hh, AA, vvo = pin(h_np), pin(A_np), pin(vo_np)
        vva = [pin(winds[s]) for s in range(a.warmup, total)]
        vin = v_start.cpu().pin_memory()
        vout_h = torch.zeros(N, dtype=torch.float64).pin_memory()
        e2e_stats = []
        barrier()
        e0.record()
        for k, s in enumerate(range(a.warmup, total)):
            st = ctx.solve_step_host(cfg.dt, (s + 1) * cfg.dt, hh, AA, vin, vva[k], vvo, vout_h)
            vin, vout_h = vout_h, vin
            e2e_stats.append(st)
        e1.record()
        barrier()
        ms_e = e0.elapsed_time(e1)
        kry_e = sum(s["krylov_iters_total"] for s in e2e_stats)
        ms_e, kry_e = reduce_timing(ms_e, float(kry_e), world, dev)
        e2e = {"value": ms_e / 1e3 / steps_all, "unit": UNIT, "h2d_bytes_per_step": 8 * (2 * Nc + 3 * N),
               "d2h_bytes_per_step": 8 * N, "ms_per_step": ms_e / a.steps,
               "dof_krylov_iters_per_s": float(N) * kry_e / (ms_e / 1e3),
               "call": "seaice_solve_step_host (pinned host buffers, H2D of h, A, v^n, v_a, v_o and D2H of "
                       "v^{n+1} inside the timed region)"}

    if rank != 0:
        return
    # ---- roofline of the dominant kernel class (algorithmic bytes / CUDA-event time)
    peak, peak_src = peaks()
    kern = {}
    for name, d in prof.items():
        if d["launches"] == 0 or d["ms"] <= 0:
            continue
        kern[name] = {"ms_total": round(d["ms"], 3), "launches": d["launches"],
                      "us_per_launch": round(1e3 * d["ms"] / d["launches"], 2),
                      "share_of_step": round(d["ms"] / ms_prof, 4)}
        if d.get("bytes"):
            gbs = d["bytes"] / (d["ms"] / 1e3) / 1e9
            kern[name].update({"alg_bytes_per_launch": d["bytes"] / d["launches"], "achieved_gbs": round(gbs, 1),
                               "frac_of_peak": round(gbs / peak, 4),
                               "frac_of_8TBs": round(gbs / 8000.0, 4)})  # BASELINE.json's nominal 8 TB/s
    dom = max(kern, key=lambda k: kern[k]["ms_total"]) if kern else None
    roof = None
    if dom and "achieved_gbs" in kern[dom]:
        traffic, traffic_src = None, None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            tj = json.load(open(tp))
            traffic = tj.get(dom)
            traffic_src = "stored: " + tj.get("_source", "profiles/ncu_traffic.json") if traffic else None
        roof = {"kernel": dom, "bound": "hbm", "achieved": kern[dom]["achieved_gbs"], "peak": peak,
                "unit": "GB/s", "frac": kern[dom]["frac_of_peak"], "traffic": traffic,
                "traffic_source": traffic_src, "peak_source": peak_src,
                "bytes_per_launch": kern[dom]["alg_bytes_per_launch"],
                "us_per_launch": kern[dom]["us_per_launch"]}
    cpu = None
    newton_per_step = sum(s["newton_iters"] for s in stats) / a.steps
    krylov_per_step = kry / a.steps
    if not a.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, N, newton_per_step, krylov_per_step, "the counts of this run's timed steps")
        except Exception as ex:  # the baseline must never break the bench line
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": f"failed: {ex}"}
    mem_live, mem_peak = ctx.memory()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_max / a.steps, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "n": n, "dof": N, "seed": cfg.seed, "dt": cfg.dt,
                   "steps_timed": [s + 1 for s in range(a.warmup, total)], "parallelism": f"replicas x{world}",
                   "l2": "working set (J 1.2 GB + Krylov basis + AMG) far larger than the 126 MB L2; no flush",
                   "newton_rtol": ctx.params.newton_rtol,
                   "krylov": (f"{'PCG' if ctx.params.krylov_method else 'FGMRES(%d)' % ctx.params.restart} rtol "
                              f"{ctx.params.krylov_rtol:g}{' + Eisenstat-Walker forcing' if ctx.params.krylov_forcing else ''}, "
                              f"maxit {ctx.params.krylov_maxit}, AMG(MIS2 smoothed aggregation, "
                              f"{ctx.params.nullspace_dim} near-nullspace columns, Chebyshev-{ctx.params.cheb_degree}, "
                              f"hierarchy lag T={ctx.params.amg_lag}, finest smoother cheb_fused={ctx.params.cheb_fused})"),
                   "params_override": json.loads(a.params)},
        "s_per_timestep": ms_max / 1e3 / a.steps,
        "dof_krylov_iters_per_s": dof_its,
        "newton_iters": [s["newton_iters"] for s in stats],
        "krylov_iters": [s["krylov_iters_total"] for s in stats],
        "krylov_solves": [s["krylov_solves"] for s in stats],
        "amg_setups": [s["amg_setups"] for s in stats],
        "krylov_capped": [s["krylov_capped"] for s in stats],
        "krylov_per_solve": round(kry / max(1, sum(s["krylov_solves"] for s in stats)), 2),
        "krylov_max_per_solve": max(s["krylov_max_iters"] for s in stats),
        "converged": [s["converged"] for s in stats],
        "phase_ms": {k: round(sum(s[k] for s in stats) / a.steps, 2) for k in
                     ("t_setup", "t_assemble", "t_amg", "t_krylov", "t_ls")},
        "roofline": roof, "kernels": kern,
        "profiled_replay": {"ms_per_step": ms_prof / a.steps,
                            "note": "per-kernel CUDA events around every launch of each class, "
                                    "eager V-cycle, same steps as the timed region"},
        "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clk.summary(),
        "memory_gb": {"live": round(mem_live / 1e9, 2), "peak": round(mem_peak / 1e9, 2)},
    }
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.cpu_kernels:
        if rank == 0:
            print(json.dumps({"cpu_kernels_cfg5": {"all_cores": oracle_kernels(a.sample_n),
                                                   "one_thread": oracle_kernels(a.sample_n, threads=1)}}))
        return
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(a, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
