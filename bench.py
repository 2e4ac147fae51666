#!/usr/bin/env python
"""Benchmark of the B200 SPAI multigrid hot path (BASELINE.json metric, line 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-extra]

Workload (BASELINE.json config 2 at the headline smoother/cycle of the metric): 2D Poisson,
h = 1/4096 (4095^2 = 16.8 M unknowns), RHS U[-1,1] from seed 0, zero start, m9 SPAI
smoother, V(1,1), full weighting / bilinear transfer, coarsest h = 1/2, fp64, solved to
relative residual 1e-10.  One step = one solve to tolerance (reset u = 0, then cycles with
the per-cycle residual norm and stop test, exactly the reference solve() loop,
multigrid.py:206-217).  value = V-cycle DOF/s = unknowns x cycles / step time, whole job.

--impl reference times the reference algorithm on the host CPU (the C restatement in
oracle/, bitwise equal to the reference, all host threads; the reference is pure numpy and
is not itself shipped to the GPU box) on the same step: one zero-start solve to tolerance.
Under torchrun only rank 0 runs it.

Multi-GPU (torchrun, --gpus N): independent replicas, one per GPU (the north star runs
one problem on one GPU; SURVEY.md §8e "replicas only"); no collective in the data path,
timing is the max over ranks, scaling "weak".
"""

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HEADLINE = dict(cfg_id="c2", smoother="m9", nu1=1, nu2=1, coarsest_N=2, tol=1e-10)
# --workload (testing / side runs; the driver's line is c2, BASELINE.json configs[1])
WORKLOADS = {
    "c1": ("m9", "c1: 2D Poisson 255^2, sine RHS, m9 SPAI V(1,1), zero start, coarsest h=1/2, tol 1e-10"),
    "c2": ("m9", "c2: 2D Poisson 4095^2, U[-1,1] seed 0, m9 SPAI V(1,1), zero start, coarsest h=1/2, tol 1e-10"),
    "c3": ("m7", "c3: 3D Poisson 127^3, sine RHS, m7 SPAI V(1,1), zero start, coarsest h=1/2, tol 1e-10"),
    "c4": ("m7", "c4: 3D Poisson 511^3, U[-1,1] seed 1, m7 SPAI V(1,1), zero start, coarsest h=1/2, tol 1e-10"),
}
METRIC = "V-cycle DOF/s (fp64 SPAI V(1,1))"
UNIT = "DOF/s"
FALLBACK_HBM_GBS = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [v.strip() for v in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(backend):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return ws, rank, local


def max_over_ranks(value, ws, device=None):
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------------------------------
# reference arm: the reference algorithm on host cores
# ------------------------------------------------------------------------------------------
def config_dict(ws):
    """The `config` of the JSON line, identical for both arms."""
    h = HEADLINE
    return {"workload": WORKLOADS[h["cfg_id"]][1] + "; step = one solve to tolerance",
            "l2": "inputs larger than L2 (finest level 134 MB/vector, hierarchy ~0.6 GB)",
            "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"}


def run_reference(args):
    """The reference algorithm on the host cores, same step as our arm: one zero-start solve
    to tolerance of the workload (the reference solve() loop, multigrid.py:206-217), through the
    C restatement in oracle/ (bitwise equal to the reference, all host threads)."""
    ws, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import c_oracle, numpy_oracle as npo
    from paper_2206_05543_b200 import stencils, workloads
    h = HEADLINE
    dim, N, _ = workloads.CONFIGS[h["cfg_id"]]
    b = workloads.rhs(h["cfg_id"])
    sm = stencils.named(h["smoother"])
    mt = npo.terms_of(sm.stencil)
    threads = c_oracle.max_threads()
    n0 = (N - 1) ** dim
    times, cycles = [], []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        u, norms, its, conv = c_oracle.solve_history(b, N, mt, sm.omega_opt_analytic, h["nu1"], h["nu2"], 1,
                                                     h["coarsest_N"], tol=h["tol"])
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
            cycles.append(its)
    t = float(np.sum(times))
    value = n0 * sum(cycles) / t
    cpu = {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"one zero-start {h['smoother']} V({h['nu1']},{h['nu2']}) solve to {h['tol']} of {h['cfg_id']} "
                     f"({N - 1}^{dim}, fp64, {cycles[-1]} cycles + norms) per step, C restatement of the reference "
                     f"(oracle/), {threads} OpenMP threads"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(ws),
        "cycles_per_solve": float(np.mean(cycles)),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host_cpu": _cpu_model(), "host_cpus": os.cpu_count(),
    }
    print(json.dumps(line), flush=True)
    return 0


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "?"


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def time_events(fn, stream, reps=1):
    import torch
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record(stream)
    fn()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / reps


def solve_workload(sp, torch, cfg_id, smoother, nu1, nu2, steps, warmup, dtype="float64"):
    """Resident-input solve loop on one GPU; returns timing + stats."""
    from paper_2206_05543_b200 import workloads
    dim, N, _ = workloads.CONFIGS[cfg_id]
    b = workloads.rhs(cfg_id)
    cfg = sp.MgConfig(smoother=sp.named(smoother), cycle="V", nu1=nu1, nu2=nu2, coarsest_N=2, tol=1e-10)
    solver = sp.Solver(cfg, dim, N, dtype=dtype, device=torch.cuda.current_device())
    bd = torch.as_tensor(b).to("cuda", torch.float64 if dtype == "float64" else torch.float32)
    stream = torch.cuda.current_stream()
    solver.load(bd)
    torch.cuda.synchronize()
    hist = None
    for _ in range(warmup):
        solver.load(None)
        hist, k, conv = solver.run()
    torch.cuda.synchronize()
    return solver, bd, b, cfg, stream, (dim, N)


def run_ours(args):
    import torch
    ws, rank, local = dist_setup("nccl")
    torch.cuda.set_device(local)
    import paper_2206_05543_b200 as sp
    from paper_2206_05543_b200 import workloads
    h = HEADLINE
    dim, N, _ = workloads.CONFIGS[h["cfg_id"]]
    n0 = (N - 1) ** dim
    b = workloads.rhs(h["cfg_id"])
    cfg = sp.MgConfig(smoother=sp.named(h["smoother"]), cycle="V", nu1=h["nu1"], nu2=h["nu2"],
                      coarsest_N=h["coarsest_N"], tol=h["tol"])
    solver = sp.Solver(cfg, dim, N, dtype="float64", device=local)
    stream = torch.cuda.current_stream()
    bd = torch.as_tensor(b).to("cuda")
    solver.load(bd)
    torch.cuda.synchronize()
    for _ in range(max(args.warmup, 3)):
        solver.load(None)
        hist, k, conv = solver.run()
    torch.cuda.synchronize()
    stats = solver.stats()

    # ---------------- timed region: K solves to tolerance, inputs resident in HBM ------------
    cycles_total = 0
    hists = []
    barrier(ws)
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            solver.load(None)  # u = 0 (memset), b stays resident
            hist, k, conv = solver.run()
            cycles_total += k
            hists.append((k, conv, hist[-1] / hist[0]))
        ev1.record(stream)
        torch.cuda.synchronize()
    t_local = ev0.elapsed_time(ev1) / 1e3
    barrier(ws)
    t = max_over_ranks(t_local, ws, device="cuda")
    cycles_per_step = cycles_total / args.steps
    value = ws * n0 * cycles_total / t
    ms_per_step = t / args.steps * 1e3
    t_cycle = t / cycles_total

    # ---------------- roofline of the dominant kernel (fused sweep K1, finest level) --------
    reps = 20
    solver.load(None)
    solver.op(0, reps)  # captures the cached replay graph
    t_k1 = min(time_events(lambda: solver.op(0, reps), stream, reps) for _ in range(3))
    peak, peak_kind = peaks()
    esz = 8
    k1_bytes = 3 * esz * n0  # read x, read b, write x'
    achieved = k1_bytes / t_k1 / 1e9
    traffic = ncu_traffic().get("sweep_c2_f64")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_kind": peak_kind, "kernel": "fused SPAI sweep K1 (finest level)",
                "algorithmic_bytes_per_launch": k1_bytes, "avg_launch_ms": t_k1 * 1e3,
                "frac_of_8TBs": achieved / 8000.0}
    vcycle_gbs = stats["bytes_per_cycle"] / t_cycle / 1e9
    _dim, _N, _ = __import__("paper_2206_05543_b200.workloads", fromlist=["CONFIGS"]).CONFIGS[HEADLINE["cfg_id"]]
    fused_b = fused_bytes_per_cycle(_dim, _N, esz, HEADLINE["nu1"], HEADLINE["nu2"], 1, 2, stats["bytes_per_cycle"])

    # ---------------- e2e: public API with pinned host buffers -------------------------------
    # Solver.solve_batch: every step copies its right-hand side in from pinned host memory and
    # its solution back out; the copies of step i+1 / i-1 overlap the solve of step i.
    # (solutions land in 3 rotating pinned buffers: copy-outs of one buffer are stream-ordered)
    e2e_steps = max(2, args.steps)
    bh = torch.from_numpy(b).pin_memory()
    uh = [torch.empty_like(bh).pin_memory() for _ in range(3)]
    solver.solve_batch([bh.numpy()] * 2, [uh[0].numpy(), uh[1].numpy()])  # warm the batch path
    barrier(ws)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    res_e = solver.solve_batch([bh.numpy()] * e2e_steps, [uh[i % 3].numpy() for i in range(e2e_steps)])
    ev1.record(stream)  # solve_batch returns after its last copy-out, ordered on this stream
    torch.cuda.synchronize()
    t_e2e = ev0.elapsed_time(ev1) / 1e3
    t_e2e = max_over_ranks(t_e2e, ws, device="cuda")
    e2e_cycles = sum(k for _, k, _ in res_e)
    k_e = res_e[-1][1]
    e2e_value = ws * n0 * e2e_cycles / t_e2e
    h2d = b.nbytes
    d2h = b.nbytes + 8 * (k_e + 1)
    assert all(c for _, _, c in res_e) and np.array_equal(uh[-1].numpy(), uh[0].numpy())

    stats = solver.stats()
    launches = int(args.steps * (1 + cycles_per_step * stats["kernels_per_cycle"] + stats["kernels_stop_test"]))

    extra = {}
    if not args.no_extra and rank == 0:
        extra = run_extras(sp, torch, stream, peak)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline_sample()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(ws),
            "cycles_per_solve": cycles_per_step, "time_to_tol_ms": ms_per_step, "ms_per_cycle": t_cycle * 1e3,
            "bytes_per_cycle": stats["bytes_per_cycle"], "vcycle_gbs": vcycle_gbs,
            "vcycle_roofline_frac": vcycle_gbs / peak, "kernels_per_cycle": stats["kernels_per_cycle"],
            "fused_bytes_per_cycle": fused_b,
            "vcycle_fused_roofline_frac": fused_b / t_cycle / 1e9 / peak,
            "converged": all(c for _, c, _ in hists), "final_rel_residual": hists[-1][2],
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": t_e2e / e2e_steps * 1e3, "steps": e2e_steps,
                    "path": "Solver.solve_batch (C ABI spaimg_solver_solve_batch): per step H2D of b from pinned "
                            "host memory, device solve to tolerance, D2H of u to pinned host memory; the copies "
                            "of neighbouring steps overlap the solve (separate copy streams)"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def cpu_baseline_sample():
    """Oracle port on the host cores, bounded sample: one c2 m9 V(1,1) cycle + norm."""
    from oracle import c_oracle, numpy_oracle as npo
    from paper_2206_05543_b200 import stencils, workloads
    h = HEADLINE
    dim, N, _ = workloads.CONFIGS[h["cfg_id"]]
    b = workloads.rhs(h["cfg_id"])
    sm = stencils.named(h["smoother"])
    mt = npo.terms_of(sm.stencil)
    u = np.zeros_like(b)
    t0 = time.perf_counter()
    ncyc = 0
    while ncyc < 2 or time.perf_counter() - t0 < 8.0:
        u = c_oracle.cycle(u, b, N, mt, sm.omega_opt_analytic, h["nu1"], h["nu2"], 1, h["coarsest_N"])
        c_oracle.residual_norm(u, b, N)
        ncyc += 1
        if ncyc >= 6:
            break
    t = (time.perf_counter() - t0) / ncyc
    th = c_oracle.max_threads()
    return {"value": (N - 1) ** dim / t, "unit": UNIT, "cores": th, "kind": "port",
            "sample": f"{ncyc} V(1,1) cycles + norms of {h['cfg_id']} ({N - 1}^{dim} fp64), C restatement, {th} threads",
            "s_per_cycle": t, "host_cpu": _cpu_model()}


def run_extras(sp, torch, stream, peak):
    """3D headline (config 4 m7 V(1,1)) and the config-5 operator microbenchmarks."""
    from paper_2206_05543_b200 import workloads
    out = {}
    try:
        dim, N, _ = workloads.CONFIGS["c4"]
        b = workloads.rhs("c4")
        cfg = sp.MgConfig(smoother=sp.named("m7"), cycle="V", nu1=1, nu2=1, coarsest_N=2, tol=1e-10)
        s3 = sp.Solver(cfg, dim, N, device=torch.cuda.current_device())
        s3.load(torch.as_tensor(b).to("cuda"))
        del b
        s3.load(None)
        s3.run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            s3.load(None)
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            hist, k, conv = s3.run()
            ev1.record(stream)
            torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1) / 1e3)
        t = float(np.median(ts))
        st = s3.stats()
        n0 = (N - 1) ** 3
        reps = 10
        s3.op(0, reps)
        tk = min(time_events(lambda: s3.op(0, reps), stream, reps) for _ in range(3))
        out["c4_m7_V11"] = {"cycles": k, "converged": conv, "time_to_tol_ms": t * 1e3, "ms_per_cycle": t / k * 1e3,
                            "dof_per_s": n0 * k / t, "bytes_per_cycle": st["bytes_per_cycle"],
                            "vcycle_roofline_frac": st["bytes_per_cycle"] / (t / k) / 1e9 / peak,
                            "vcycle_fused_roofline_frac":
                                fused_bytes_per_cycle(3, N, 8, 1, 1, 1, 2, st["bytes_per_cycle"]) / (t / k) / 1e9 / peak,
                            "sweep_gbs": 24 * n0 / tk / 1e9, "sweep_frac": 24 * n0 / tk / 1e9 / peak,
                            "kernels_per_cycle": st["kernels_per_cycle"]}
        del s3
        torch.cuda.empty_cache()
    except Exception as exc:  # extras never fail the headline line
        out["c4_error"] = repr(exc)
    try:
        out["configs_1_4"] = config_sweep(sp, torch, stream, peak)
    except Exception as exc:
        out["configs_1_4_error"] = repr(exc)
    try:
        out["reference_defaults_W10_cN4"] = w_sweep(sp, torch, stream, peak)
    except Exception as exc:
        out["reference_defaults_error"] = repr(exc)
    try:
        out["api_solve_host_arrays"] = api_e2e(sp, torch)
    except Exception as exc:
        out["api_solve_error"] = repr(exc)
    try:
        out["config5"] = microbench(sp, torch, stream, peak)
    except Exception as exc:
        out["config5_error"] = repr(exc)
    return out


def config_sweep(sp, torch, stream, peak):
    """Every solve BASELINE.json configs 1-4 name (SPAI smoother vs weighted Jacobi, V(1,1) and
    V(2,2), zero start, tol 1e-10): cycles, time to tolerance, per-cycle time, rho_hat and the
    asymptotic per-cycle factor, with the V-cycle bytes-moved fraction."""
    from paper_2206_05543_b200 import workloads
    res = {}
    for cfg_id in ("c1", "c2", "c3", "c4"):
        dim, N, _ = workloads.CONFIGS[cfg_id]
        bd = torch.as_tensor(workloads.rhs(cfg_id)).to("cuda")
        spai = "m9" if dim == 2 else "m7"
        jac = "jacobi2d" if dim == 2 else "jacobi3d"
        runs = [(spai, 1), (spai, 2), (jac, 1), (jac, 2)] if cfg_id in ("c2", "c4") else [(spai, 1)]
        for sm, nu in runs:
            cfg = sp.MgConfig(smoother=sp.named(sm), cycle="V", nu1=nu, nu2=nu, coarsest_N=2, tol=1e-10)
            so = sp.Solver(cfg, dim, N, device=torch.cuda.current_device())
            so.load(bd)
            so.run()
            ts = []
            for _ in range(3):
                so.load(None)
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record(stream)
                hist, k, conv = so.run()
                ev1.record(stream)
                torch.cuda.synchronize()
                ts.append(ev0.elapsed_time(ev1) / 1e3)
            t = float(np.median(ts))
            st = so.stats()
            rho = (hist[-1] / hist[0]) ** (1.0 / k) if k else None
            res[f"{cfg_id}/{sm}/V({nu},{nu})"] = {
                "cycles": k, "converged": conv, "time_to_tol_ms": t * 1e3, "ms_per_cycle": t / k * 1e3,
                "dof_per_s": (N - 1) ** dim * k / t, "rho_hat": rho,
                "last_cycle_factor": hist[-1] / hist[-2] if k >= 1 else None,
                "vcycle_roofline_frac": st["bytes_per_cycle"] / (t / k) / 1e9 / peak,
                "vcycle_fused_roofline_frac":
                    fused_bytes_per_cycle(dim, N, 8, nu, nu, 1, 2, st["bytes_per_cycle"]) / (t / k) / 1e9 / peak}
            del so
        del bd
        torch.cuda.empty_cache()
    return res


def w_sweep(sp, torch, stream, peak):
    """The reference MgConfig defaults (cycle="W", nu1=1, nu2=0, coarsest_N=4, tol 1e-10;
    multigrid.py:39-43) on configs 1-4: zero start, resident inputs, time to tolerance and the
    bytes-moved fraction of a W-cycle (level l visited 2^l times)."""
    from paper_2206_05543_b200 import workloads
    res = {}
    for cfg_id in ("c1", "c2", "c3", "c4"):
        dim, N, _ = workloads.CONFIGS[cfg_id]
        bd = torch.as_tensor(workloads.rhs(cfg_id)).to("cuda")
        sm = "m9" if dim == 2 else "m7"
        cfg = sp.MgConfig(smoother=sp.named(sm))
        so = sp.Solver(cfg, dim, N, device=torch.cuda.current_device())
        so.load(bd)
        so.run()
        ts = []
        for _ in range(3):
            so.load(None)
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            hist, k, conv = so.run()
            ev1.record(stream)
            torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1) / 1e3)
        t = float(np.median(ts))
        st = so.stats()
        res[f"{cfg_id}/{sm}/W(1,0)/cN4"] = {
            "cycles": k, "converged": conv, "time_to_tol_ms": t * 1e3, "ms_per_cycle": t / k * 1e3,
            "dof_per_s": (N - 1) ** dim * k / t, "rho_hat": (hist[-1] / hist[0]) ** (1.0 / k) if k else None,
            "bytes_per_cycle": st["bytes_per_cycle"], "kernels_per_cycle": st["kernels_per_cycle"],
            "vcycle_roofline_frac": st["bytes_per_cycle"] / (t / k) / 1e9 / peak,
            "vcycle_fused_roofline_frac":
                fused_bytes_per_cycle(dim, N, 8, 1, 0, 2, 4, st["bytes_per_cycle"]) / (t / k) / 1e9 / peak}
        del so, bd
        torch.cuda.empty_cache()
    return res


def api_e2e(sp, torch):
    """Wall time of the reference-signature call solve(Grid(N, numpy_b), cfg, u0=0): host
    arrays in and out (pageable), first call (builds and caches the device hierarchy and
    graphs) and repeated calls (cached, like the reference's lru_cache on the coarse LU)."""
    from paper_2206_05543_b200 import workloads
    from paper_2206_05543_b200.multigrid import clear_solver_cache
    res = {}
    for cfg_id, sm in (("c2", "m9"), ("c4", "m7")):
        dim, N, _ = workloads.CONFIGS[cfg_id]
        b = workloads.rhs(cfg_id)
        cfg = sp.MgConfig(smoother=sp.named(sm), cycle="V", nu1=1, nu2=1, coarsest_N=2, tol=1e-10)
        clear_solver_cache()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        u, rep = sp.solve(sp.Grid(N, b), cfg, u0=0)
        t_first = time.perf_counter() - t0
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            u, rep = sp.solve(sp.Grid(N, b), cfg, u0=0)
            ts.append(time.perf_counter() - t0)
        # the same solve through the persistent handle with device-resident input, for comparison
        so = sp.cached_solver(cfg, dim, N, 0, torch.cuda.current_device())
        bd = torch.as_tensor(b).to("cuda")
        so.load(bd)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        so.load(None)
        so.run()
        torch.cuda.synchronize()
        t_dev = time.perf_counter() - t0
        res[cfg_id] = {"first_call_s": t_first, "cached_call_s": float(np.median(ts)), "cycles": rep.iterations,
                       "device_solve_s": t_dev, "bytes_in": b.nbytes, "bytes_out": b.nbytes,
                       "note": "host numpy b in, host numpy u out (pageable copies included)"}
        del u, b, bd
        clear_solver_cache()
        torch.cuda.empty_cache()
    return res


def fused_bytes_per_cycle(dim, N, esize, nu1, nu2, gamma, coarsest_N, bytes_survey):
    """Bytes the fused schedule has to move per cycle: the SURVEY.md 8d count (every operator
    reading and writing its vectors once) minus what the two bitwise-safe fusions of the named
    smoothers never move: the norm's read of (x, b) on the finest level (folded into the first
    pre-sweep, nu1 >= 1) and the prolonged iterate's write + re-read on the K3 + K1 levels
    (nu2 >= 1; 2D mesh counts > 2048, 3D >= 256: sweep_pc_supported in kernels_sweep.cu)."""
    saved, visits, n = 0.0, 1.0, N
    level = 0
    while n > coarsest_N:
        pts = float((n - 1) ** dim)
        if level == 0 and nu1 >= 1:
            saved += 2.0 * esize * pts
        if nu2 >= 1 and ((dim == 2 and n > 2048) or (dim == 3 and n >= 256)):
            saved += visits * 2.0 * esize * pts
        visits *= gamma
        n //= 2
        level += 1
    return bytes_survey - saved


def microbench(sp, torch, stream, peak):
    """Config 5: each hot kernel in isolation on 16384^2 (2D) and 512^3 (3D), fp64 and fp32.
    Inputs larger than L2; best of reps after warm-up; bytes are the §8d minimal counts."""
    from paper_2206_05543_b200 import workloads
    res = {}
    for dim, N, sm in ((2, 16384, "m9"), (3, 512, "m7")):
        for dtype in ("float64", "float32"):
            s = 8 if dtype == "float64" else 4
            x, b, e = workloads.microbench_inputs(dim, N, np.float64 if dtype == "float64" else np.float32)
            cfg = sp.MgConfig(smoother=sp.named(sm), cycle="V", nu1=1, nu2=1, coarsest_N=2)
            so = sp.Solver(cfg, dim, N, dtype=dtype, device=torch.cuda.current_device())
            so.load(b, x)
            del x, b, e
            n = (N - 1) ** dim
            key = f"{dim}d_N{N}_{dtype}"
            r = {}
            # K3 + K1 (op 6): x + P e and the sweep in one march: x, b, e/2^d in, x' out
            for op, name, bpu in ((0, "sweep", 3.0), (1, "residual_restrict", 2 + 2.0 ** -dim),
                                  (2, "prolong_correct", 2 + 2.0 ** -dim), (3, "residual_norm", 2.0),
                                  (6, "prolong_correct_sweep", 3 + 2.0 ** -dim)):
                so.op(op, 5)
                best = min(time_events(lambda: so.op(op, 5), stream, 5) for _ in range(3))
                gbs = bpu * s * n / best / 1e9
                r[name] = {"ms": best * 1e3, "gbs": gbs, "frac": gbs / peak, "bytes_per_unknown": bpu * s}
            res[key] = r
            del so
            torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    args = ap.parse_args()
    HEADLINE["cfg_id"] = args.workload
    HEADLINE["smoother"] = WORKLOADS[args.workload][0]
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
