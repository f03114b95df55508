#!/usr/bin/env python3
"""Benchmark of the per-time-step FETI solve (BASELINE.json north_star).

Workload (config.workload): BASELINE config 4 — 1024x1024 P2-P1-P1 / P2-P1
mesh, 32x32 = 1024 subdomains of 32x32 cells, lower half poroelastic, nu=0.3,
c0=1e-3, K=1, dt=1e-2, time-linear manufactured solution (synthetic inputs of
that shape), interface tolerance 1e-10.  A "step" is one backward-Euler time
step (StepSolver::advance, timeloop.hpp:150): right-hand side assembly on the
device, interface right-hand side, the full Krylov solve (F-applies, mortar-
scaled Dirichlet preconditioner, natural coarse projector) and the
back-substitution.  Inputs (factors, ~16 GB) are far larger than L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
                  [--solver feti|direct]

--solver feti (default) times the FETI Krylov step, the reference's feti-schur
path with the same tolerance; its line also carries "direct_solver": the same
K steps through the direct interface solve (krylov="direct", the GPU analogue
of the reference's SolverChoice::monolithic), measured in the same run.
--solver direct makes that solver the line's `value`.

--impl reference times the reference's CPU path on the host cores: the C++
oracle restatement of the reference algorithm (oracle/, all host threads; the
reference itself needs Eigen, absent from the GPU image -- oracle/_ref pins
the restatement to it) runs real time steps of the full workload, timed with
steady_clock per step (run_reference()).  The cpu_baseline object of the
default arm is a bounded sample (cpu_sample(): one F-apply + preconditioner on
4x4 subdomains, scaled), marked "estimated"; profiles/ holds the measured
full steps it is checked against.
--gpus N > 1 without torchrun: the script re-executes itself under
torch.distributed.run with N local ranks (one process per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "s per time step & FETI F-applies/s (1 B200); HBM GB/s vs roofline"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            P = json.load(f)
        return float(P["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def spawn(n):
    """Re-execute this script under torch.distributed.run with n local ranks
    (rendezvous on 127.0.0.1, a free port); rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_init(n):
    if n <= 1 and "WORLD_SIZE" not in os.environ:
        return 0, 1, None
    import torch.distributed as dist
    dist.init_process_group(backend="gloo")
    return dist.get_rank(), dist.get_world_size(), dist


def reduce_max(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def cpu_sample(cfg_name, steps_like):
    """CPU reference leg: the oracle on a bounded sample of the workload.

    Sample: 4x4 subdomains of the workload's subdomain size (same 32x32-cell P2
    subdomains, mesh 128), all host threads.  Measured: one F-apply and one
    preconditioner apply (the per-iteration work); scaled by the subdomain
    count ratio to the full workload and multiplied by the iteration count of
    the workload (from the GPU arm when known, else `steps_like`)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracle_lib as ol
    import paper_2509_06673_b200 as pf

    kw = dict(pf.BASELINE_CONFIGS[cfg_name])
    full_sub = kw["SX"] * kw["SY"]
    cx = kw["mesh_n"] // kw["SX"]
    sx, sy = min(kw["SX"], 4), min(kw["SY"], 4)  # SY stays even (P below, E above)
    sample = dict(kw, SX=sx, SY=sy, mesh_n=sx * cx)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    o = ol.Oracle(**dict(sample, threads=threads))
    t_setup = time.perf_counter() - t0
    x = np.random.default_rng(20240901).uniform(-1, 1, o.n_lambda)
    reps = 0
    t0 = time.perf_counter()
    while True:
        o.apply(x)
        o.precond(x)
        reps += 1
        if time.perf_counter() - t0 > 2.0 or reps >= 20:
            break
    t_iter = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    o.apply(x)
    t_fapply = time.perf_counter() - t0
    scale = full_sub / (sx * sy)
    return dict(t_iter_full=t_iter * scale, t_fapply_full=t_fapply * scale, threads=threads, setup_s=t_setup,
                sample=f"oracle (C++ restatement, {threads} threads) on {sx}x{sy} subdomains of {cx}x{cx} cells "
                       f"(mesh {sx * cx}), F-apply+preconditioner per iteration timed ({reps} reps), scaled x{scale:g} "
                       f"to {full_sub} subdomains and multiplied by the workload's iterations per step")


ITERS_PER_STEP = {"c1": 51, "c2": 49, "c3": 769, "c4": 179, "c5": 1028}


def workload_name(cfg_name):
    import paper_2509_06673_b200 as pf
    kw = pf.BASELINE_CONFIGS[cfg_name]
    return (f"BASELINE {cfg_name}: mesh {kw['mesh_n']}^2 P{kw['order']}, {kw['SX']}x{kw['SY']} subdomains, "
            f"{kw['precond']}, tol {kw.get('tol', 1e-10)}")


def run_reference(args, rank, world, dist):
    """The reference's CPU path, timed: the oracle (C++ restatement of the
    reference algorithm, all host threads) runs REAL time steps of the full
    workload -- StepSolver::advance (timeloop.hpp:150-186) with
    std::chrono::steady_clock around each step, REF's own clock (feti.hpp:103)
    -- after its setup (assembly + factorisation, reported separately).  A CPU
    step of c4 takes minutes, so the timed steps are capped by a wall budget
    (--ref-budget seconds, at least one step): "steps" is the number actually
    timed, "steps_requested" the --steps asked for."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as ol
    import paper_2509_06673_b200 as pf  # noqa: F401 (config table only)

    kw = dict(pf.BASELINE_CONFIGS[args.config])
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    o = ol.Oracle(**dict(kw, threads=threads))
    setup_s = time.perf_counter() - t0
    # untimed warm-up: CPU steps need none (c4 on the box: first step 196.2 s,
    # second 195.5 s, profiles/r2_cpu_baseline.json); one for the cheap configs
    # (setup under 10 s), more only while they stay cheap
    budget = args.ref_budget
    W = 0
    if setup_s < 10.0:
        o.run(1)
        first = o.report(1)["seconds"]
        W = 1
        while W < args.warmup and first * (W + 1) < 0.25 * budget:
            o.run(1)
            W += 1
    timed, iters = [], []
    t_start = time.perf_counter()
    while len(timed) < args.steps and W + len(timed) < kw["steps"]:
        if timed and (time.perf_counter() - t_start) + statistics.mean(timed) > budget:
            break
        o.run(1)
        rep = o.report(W + len(timed) + 1)
        timed.append(rep["seconds"])
        iters.append(rep["iterations"])
    value = statistics.mean(timed)
    sample = (f"oracle (C++ restatement of the reference algorithm: per-subdomain sparse LDL^T solves, "
              f"{threads} threads over subdomains) on the full {args.config} workload; {len(timed)} time steps "
              f"timed after {W} untimed (steady_clock around each advance), setup {setup_s:.1f} s not included")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s/step", "n_gpus": world,
            "steps": len(timed), "steps_requested": args.steps, "warmup": W, "ms_per_step": value * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (manufactured solution)",
            "config": {"workload": workload_name(args.config),
                       "kernel": "CPU oracle (C++ restatement of the reference algorithm; the reference needs "
                                 "Eigen, absent here -- oracle/_ref pins the restatement to it on small cases)"},
            "step_seconds": timed, "median_s": statistics.median(timed), "iterations": iters,
            "setup_s": setup_s,
            "cpu_baseline": {"value": value, "unit": "s/step", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "s/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def roofline_obj(achieved, peak, peak_src, traffic, kernel, alg_bytes, roof_extra, extra):
    """The dominant kernel against the roofline that bounds it.  The mortar Gram
    solve, the coarse GEMV and the sweeps are byte movers (HBM bound).  The local
    dual products are a GEMM over same-type subdomains at 15 flop per
    algorithmic byte, above the machine balance (35 TFLOP/s / 6.5 TB/s): bound
    by the FP64 tensor cores, peak = the cuBLAS DGEMM rate measured on this pool
    (profiles/r2_fp64_peak.json; MEASURED_PEAKS.json carries no FP64 figure)."""
    ldp = extra.get("local_dual_products") if extra else None
    if ldp is not None and kernel == ldp["what"] and ldp.get("tensor_frac"):
        return dict({"bound": "tensor", "achieved": ldp["tflops"], "peak": ldp["dgemm_peak_tflops"],
                     "unit": "TFLOP/s", "frac": ldp["tensor_frac"], "traffic": traffic, "kernel": kernel,
                     "flops_per_launch": ldp["flops"], "algorithmic_bytes_per_launch": alg_bytes,
                     "peak_source": "measured cuBLAS DGEMM n=8192 on this pool (profiles/r2_fp64_peak.json)",
                     "hbm_view": {"achieved_gbs": achieved, "peak_gbs": peak, "frac": achieved / peak,
                                  "peak_source": peak_src}}, **roof_extra)
    return dict({"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                 "traffic": traffic, "kernel": kernel, "algorithmic_bytes_per_launch": alg_bytes,
                 "peak_source": peak_src}, **roof_extra)


def direct_arm(args, cfg_name, peak):
    """K time steps through the direct interface solve (krylov="direct": the
    multipliers condensed exactly -- dense inverse up to 4096 multipliers, a
    multifrontal block LDL^T over the subdomain grid above), device time,
    end to end through pf_advance with pinned host buffers, and the interface
    solve's GEMV launches against the HBM roofline (every stored front value
    is read once per solve)."""
    import numpy as np
    import paper_2509_06673_b200 as pf

    kw = dict(pf.BASELINE_CONFIGS[cfg_name], krylov="direct")
    kw["steps"] = max(kw["steps"], args.warmup + 2 * args.steps + 2)
    t0 = time.perf_counter()
    op = pf.FetiOperator(**kw)
    setup_s = time.perf_counter() - t0
    info = op.info
    reps = [op.step() for _ in range(args.warmup)]
    l0 = pf.launch_count()
    ms, _, _ = op.bench_steps(args.steps)
    launches = pf.launch_count() - l0
    xs, lam = op.state()
    x_cat = np.concatenate(xs)
    step_idx = pf.lib().pf_current_step(op.h)
    solver = pf.StepSolver(op)
    pin = [[pf.pinned_empty(n) for n in (x_cat.size, lam.size)] for _ in range(2)]
    pin[0][0][:] = x_cat
    pin[0][1][:] = lam
    t0 = time.perf_counter()
    cur_k = step_idx
    for k in range(args.steps):
        src, dst = pin[k % 2], pin[(k + 1) % 2]
        _, _, rep = solver.advance(src[0], src[1], cur_k, out_x=dst[0], out_lambda=dst[1])
        cur_k = rep["step"]
    e2e_s = (time.perf_counter() - t0) / args.steps
    h2d = int(pf.lib().pf_last_h2d_bytes(op.h))
    rep = op.step()
    out = {"what": "direct interface solve (krylov=direct): " +
                   ("multifrontal block LDL^T of F over a nested dissection of the subdomain grid, "
                    f"{info.direct_fronts} fronts" if info.direct_sparse else "dense inverse of F, one GEMV per step"),
           "value": ms * 1e-3 / args.steps, "unit": "s/step", "steps": args.steps, "warmup": args.warmup,
           "iterations_per_step": 0,
           "true_residual": max([r["true_residual"] for r in reps] + [rep["true_residual"]]),
           "phase_ms": {"rhs": rep["t_rhs"] * 1e3, "interface_solve": rep["t_krylov"] * 1e3,
                        "back_substitution": rep["t_back"] * 1e3},
           "e2e": {"value": e2e_s, "unit": "s/step", "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": int(x_cat.nbytes + lam.nbytes)},
           "setup_s": setup_s, "direct_setup_s": info.t_direct_setup, "gpu_launches": int(launches)}
    # roofline of the interface solve: stored operator bytes once per solve
    t7 = op.bench(7 if info.direct_sparse else 6, 5, 20)[0]  # sparse: fronts + coarse border; dense: one GEMV
    b = float(info.bytes_direct)
    out["roofline"] = {"bound": "hbm", "kernel": "k_iface_gemv<fwd/bwd> per tree depth + coarse border GEMV"
                       if info.direct_sparse else "k_gemv_rows: lambda = [Z | Y_c] [rhs; e]",
                       "ms": t7, "algorithmic_bytes_per_launch": b, "achieved": b / (t7 * 1e-3) / 1e9, "peak": peak,
                       "unit": "GB/s", "frac": b / (t7 * 1e-3) / 1e9 / peak}
    op.close()
    return out


def run_ours(args, rank, world, dist):
    import numpy as np
    import paper_2509_06673_b200 as pf

    kw = dict(pf.BASELINE_CONFIGS[args.config])
    kw["steps"] = max(kw["steps"], args.warmup + 2 * args.steps + 1)  # timed steps, then the e2e steps
    t0 = time.perf_counter()
    if world > 1:
        import torch
        if torch.cuda.device_count() < world:
            raise SystemExit(f"bench.py --gpus {world}: only {torch.cuda.device_count()} visible GPU(s); "
                             "one process per GPU is required")
        # sharded engine: subdomains split over ranks, lambda partial sums by
        # ncclAllReduce on each engine's stream (the engine selects GPU LOCAL_RANK)
        import torch
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            idt = torch.frombuffer(bytearray(pf.nccl_unique_id()), dtype=torch.uint8).clone()
        dist.broadcast(idt, src=0)
        op = pf.FetiOperator(rank=rank, nranks=world, nccl_id=bytes(idt.numpy().tobytes()), **kw)
    else:
        op = pf.FetiOperator(**kw)
    setup_s = time.perf_counter() - t0
    info = op.info
    # warm-up steps (untimed)
    for _ in range(args.warmup):
        op.step()
    barrier(dist)
    l0 = pf.launch_count()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        ms, iters, fapplies = op.bench_steps(args.steps)
    launches_timed = pf.launch_count() - l0
    barrier(dist)
    ms = reduce_max(dist, ms)
    s_per_step = ms * 1e-3 / args.steps
    iters_per_step = iters / args.steps
    # e2e: reference-facing C ABI with host buffers (pf_advance), copies inside
    xs, lam = op.state()
    x_cat = np.concatenate(xs)
    step_idx = pf.lib().pf_current_step(op.h)
    solver = pf.StepSolver(op)
    e2e_steps = args.steps  # the same K steps as `value`
    # page-locked host buffers (ping-pong): the caller's state in pinned memory
    pin = [[pf.pinned_empty(n) for n in (x_cat.size, lam.size)] for _ in range(2)]
    pin[0][0][:] = x_cat
    pin[0][1][:] = lam
    t0 = time.perf_counter()
    cur_k = step_idx
    for k in range(e2e_steps):
        src, dst = pin[k % 2], pin[(k + 1) % 2]
        _, _, rep = solver.advance(src[0], src[1], cur_k, out_x=dst[0], out_lambda=dst[1])
        cur_k = rep["step"]
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e_s = reduce_max(dist, e2e_s)
    # pf_advance uploads the inputs a step reads (eta^{n-1}, lambda^{n-1}) and
    # downloads the whole next state
    h2d = int(pf.lib().pf_last_h2d_bytes(op.h))
    d2h = x_cat.nbytes + lam.nbytes
    # dominant kernel (factor sweeps of the F-apply), CUDA events, live
    # F-applies/s from 200 back-to-back applies after 20 warm-up calls
    ms_apply, sweep_ms, launches = op.bench(0, 20, 200)
    ph = pf.phase_stats(op, 3)
    step_sweep_ms = op.bench(8, 5, 50)[0]  # the K^+ b sweep as a step runs it (wide when set up)
    peak, peak_src = _peaks()
    sweep_bytes = 2.0 * 8.0 * info.nnz_L + 8.0 * info.total_dim  # per sweep (values + D), supernodal storage
    sweep_achieved = sweep_bytes / (sweep_ms * 1e-3) / 1e9
    prof = os.path.join(ROOT, "profiles", "ncu_sweep_traffic.json")
    ptraffic = {}
    if os.path.exists(prof):
        try:
            ptraffic = json.load(open(prof))
        except Exception:
            ptraffic = {}
    extra = {}
    roof_extra = {}
    n_l = info.n_lambda

    def comp(kind, alg_bytes, what, applied=None):
        t = op.bench(kind, 20, 200)[0]
        d = {"what": what, "ms": t, "algorithmic_bytes": alg_bytes,
             "gbs": alg_bytes / (t * 1e-3) / 1e9, "frac": alg_bytes / (t * 1e-3) / 1e9 / peak}
        if applied is not None:
            d["applied_bytes"] = applied
            d["applied_gbs"] = applied / (t * 1e-3) / 1e9
        return d

    if info.dual:
        # per Krylov iteration: two local dual-operator products (F_s, Sd_s),
        # two mortar Gram solves Q, two dense coarse GEMVs, dots and axpys.
        # Algorithmic bytes count what the algorithm must move: operators
        # shared by same-type subdomains (bitwise/1e-12-equal) once, per
        # subdomain inputs/outputs; "applied" counts every application.
        extra["local_dual_products"] = comp(
            3, info.bytes_flocal + 0.0,
            "k_local_gather + k_type_gemm (FP64 mma.sync over same-type operators) [+ k_local_symv]",
            applied=info.bytes_symv)
        extra["local_dual_products"]["flops"] = info.flops_flocal
        if info.bytes_qsolve > 0:
            q_what = ("Q = (sum_s G_s G_s^T)^-1, edge-local: k_qlocal_y + k_qlocal_x (explicit (interface, component) "
                      f"block inverses + cross-point corrections, {info.q_local_blocks} blocks)" if info.q_local else
                      "Q = (sum_s G_s G_s^T)^-1: 4 k_dense_unit stages + k_dense_top_gather + k_dense_top_gemv")
            extra["mortar_gram_solve"] = comp(
                4, info.bytes_qsolve + (0.0 if info.q_local else 16.0 * n_l), q_what,
                applied=info.bytes_qsolve_applied + (0.0 if info.q_local else 16.0 * n_l))
        if info.n_coarse:
            extra["coarse_gemv"] = comp(5, info.bytes_coarse + 16.0 * info.n_coarse,
                                        "k_dense_gemv_w: (G_c^T G_c)^-1 y, dense n_c x n_c")
        if info.flops_backsub > 0:
            extra["explicit_back_substitution"] = {
                "what": "k_h_gemm: x_s = K_s^+ b_s - H_t lambda_s, H_t = K_t^+ G_t^T per type (FP64 mma.sync), "
                        "once per step instead of a factor sweep",
                "flops": info.flops_backsub, "bytes": info.bytes_backsub}
        # FP64 tensor-core view of the local products (a GEMM: 15 flop/B, above the
        # machine balance): TFLOP/s against the measured cuBLAS DGEMM peak of this pool
        try:
            dg_peak = float(json.load(open(os.path.join(ROOT, "profiles", "r2_fp64_peak.json")))["tflops_fp64"])
        except Exception:
            dg_peak = None
        ldp = extra["local_dual_products"]
        ldp["tflops"] = ldp["flops"] / (ldp["ms"] * 1e-3) / 1e12
        if dg_peak:
            ldp["dgemm_peak_tflops"] = dg_peak
            ldp["tensor_frac"] = ldp["tflops"] / dg_peak
        # dominant per-iteration piece: each runs twice per Krylov iteration (F-apply and
        # preconditioner; a Gram solve on either side of the Dirichlet operator; a coarse
        # projection after each), so the longest one is the dominant kernel
        cand = [extra[k] for k in ("mortar_gram_solve", "local_dual_products", "coarse_gemv") if k in extra]
        dom = max(cand, key=lambda c: c["ms"])
        kernel = dom["what"]
        alg_bytes, achieved = dom["algorithmic_bytes"], dom["gbs"]
        dom_key = [k for k in extra if extra[k] is dom][0]
        traffic = ptraffic.get(args.config + {"mortar_gram_solve": "_qsolve" if not info.q_local else "_qlocal",
                                              "local_dual_products": "_flocal", "coarse_gemv": "_coarse"}[dom_key])
        roof_extra = {"note": "latency-bound launches on L2-resident operators (same-type subdomains share one "
                              "operator copy: applied_gbs counts every application); for the local products the "
                              "tensor view (kernels.local_dual_products.tensor_frac: TFLOP/s against the measured "
                              "cuBLAS DGEMM peak) is the tighter bound",
                      "applied_gbs": dom.get("applied_gbs"),
                      "per_iteration_ms": {k: extra[k]["ms"] for k in ("mortar_gram_solve", "local_dual_products",
                                                                        "coarse_gemv") if k in extra}}
    else:
        kernel = "batched supernodal LDL^T sweep (k_sweep forward/root/backward levels + k_fold_level)"
        alg_bytes, achieved = sweep_bytes, sweep_achieved
        traffic = ptraffic.get(args.config)
    world_value = s_per_step  # one sharded problem: the job's seconds per step (max over ranks)
    line = {
        "metric": METRIC, "value": world_value, "unit": "s/step", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": s_per_step * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (manufactured solution)",
        "config": {"workload": workload_name(args.config),
                   "n_lambda": info.n_lambda, "nnz_L": info.nnz_L, "n_sub": info.n_sub,
                   "l2": "no flush: every step streams > L2 (state, right-hand sides, saddle CSR values, ~0.5 GB); the Krylov operators (~0.13 GB after same-type sharing) stay L2-resident within a step by design",
                   "parallelism": f"subdomain sharding over {world} GPUs (NCCL all-reduce of lambda partial sums)" if world > 1 else "single GPU"},
        "iterations_per_step": iters_per_step,
        "f_applies_per_s": fapplies / (ms * 1e-3),
        "f_apply_ms": ms_apply,
        "f_applies_per_s_microbench": 1e3 / ms_apply,
        "sweep_phase_ms": ph,
        "e2e": {"value": e2e_s, "unit": "s/step", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "host_buffers": "page-locked (pf_host_alloc), caller-owned, through pf_advance (uploads eta^{n-1} and lambda^{n-1}, downloads the full state)"},
        "roofline": roofline_obj(achieved, peak, peak_src, traffic, kernel, alg_bytes, roof_extra, extra),
        "sweep_roofline": {"kernel": "batched supernodal LDL^T sweep of the subdomain factors (interface rhs, "
                                     "back-substitution; the implicit F-apply with PF_FAPPLY=implicit)",
                           "work_equivalent_gbs": sweep_achieved, "work_equivalent_frac": sweep_achieved / peak,
                           "unit": "GB/s", "per_subdomain_factor_bytes": sweep_bytes, "ms": sweep_ms,
                           "per_step_sweep_ms": step_sweep_ms, "per_step_sweep_width": info.sweep_width,
                           "per_step_work_equivalent_gbs": sweep_bytes / (step_sweep_ms * 1e-3) / 1e9,
                           "per_step_work_equivalent_frac": sweep_bytes / (step_sweep_ms * 1e-3) / 1e9 / peak,
                           "per_step_sweep": "k_sweep_w: groups of per_step_sweep_width same-type subdomains per warp "
                                             "task, each factor value streamed once for the group (bitwise the "
                                             "scalar sweep's results)" if info.sweep_width > 1 else "scalar k_sweep",
                           "stored_factor_bytes": info.bytes_factor_stored,
                           "stored_gbs": info.bytes_factor_stored / (sweep_ms * 1e-3) / 1e9,
                           "note": "same-type subdomains read one shared factor copy (L2); the per-subdomain "
                                   "figure (SURVEY 8d B_F) is the work the sweep does, not its HBM traffic"},
        "north_star_fapply": {
            "f_applies_per_s_microbench": 1e3 / ms_apply,
            "implicit_sweep_f_applies_per_s_at_100pct_hbm": peak * 1e9 / sweep_bytes if sweep_bytes else None,
            "implicit_sweep_f_applies_per_s_at_60pct_hbm": 0.6 * peak * 1e9 / sweep_bytes if sweep_bytes else None,
            "note": "SURVEY 8d target (>= 60% of HBM on the implicit F-apply's 2*8*nnz(L)+8*dim bytes); the "
                    "default explicit path removes those bytes rather than streaming them"},
        "explicit_local_operators": bool(info.dual),
        "kernels": extra,
        "gpu_launches": None,
        "clocks": clk.summary(),
        "setup_s": setup_s,
    }
    line["gpu_launches"] = int(launches_timed)
    if rank == 0 and args.cpu_baseline and world == 1:
        try:
            s = cpu_sample(args.config, iters_per_step)
            v = (iters_per_step + 2) * s["t_fapply_full"] + iters_per_step * (s["t_iter_full"] - s["t_fapply_full"])
            meas = None
            try:  # the committed measurement of a real full step on the same box type
                runs = json.load(open(os.path.join(ROOT, "profiles", "r2_cpu_baseline.json")))["runs"]
                meas = next(r for r in runs if r["config"] == args.config and r["mode"] == "restated-parallel")
            except Exception:
                pass
            line["cpu_baseline"] = {"value": v, "unit": "s/step", "cores": s["threads"], "kind": "port",
                                    "sample": s["sample"], "estimated": True,
                                    "measured_full_step_s": meas["step_s_mean"] if meas else None,
                                    "measured_full_step_source": "profiles/r2_cpu_baseline.json (real time steps of "
                                                                 "the full workload, 16 host threads; the reference "
                                                                 "arm bench.py --impl reference repeats it live)"}
        except Exception as exc:  # the baseline is reported, never fatal
            line["cpu_baseline"] = {"value": None, "unit": "s/step", "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"failed: {exc}"}
    op.close()
    if rank == 0 and world == 1 and args.direct:
        try:  # the same K steps through the direct interface solve, same run
            line["direct_solver"] = direct_arm(args, args.config, peak)
        except Exception as exc:  # reported, never fatal for the FETI line
            line["direct_solver"] = {"failed": str(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_direct(args, rank, world, dist):
    """--solver direct: the direct interface solve as the line's value (one
    GPU; the sharded engine keeps the FETI Krylov path)."""
    if world > 1:
        if rank == 0:
            print(json.dumps({"solver": "direct", "unavailable": "the direct interface solve runs on one GPU"}),
                  flush=True)
        return
    peak, peak_src = _peaks()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        d = direct_arm(args, args.config, peak)
    import paper_2509_06673_b200 as pf
    kw = pf.BASELINE_CONFIGS[args.config]
    line = {"metric": METRIC, "value": d["value"], "unit": "s/step", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": d["value"] * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (manufactured solution)",
            "config": {"workload": (f"BASELINE {args.config}: mesh {kw['mesh_n']}^2 P{kw['order']}, "
                                    f"{kw['SX']}x{kw['SY']} subdomains, direct interface solve"),
                       "solver": d["what"],
                       "l2": "no flush: the interface solve streams its stored fronts once per step (> L2 at c4)",
                       "parallelism": "single GPU"},
            "iterations_per_step": 0, "true_residual": d["true_residual"], "phase_ms": d["phase_ms"],
            "e2e": d["e2e"], "roofline": dict(d["roofline"], traffic=None, peak_source=peak_src),
            "gpu_launches": d["gpu_launches"], "clocks": clk.summary(), "setup_s": d["setup_s"],
            "direct_setup_s": d["direct_setup_s"]}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--solver", default="feti", choices=["feti", "direct"],
                    help="feti: FETI Krylov step (default, + a direct_solver object); direct: the direct "
                         "interface solve as the line's value")
    ap.add_argument("--no-direct", dest="direct", action="store_false",
                    help="--solver feti: skip the direct_solver object")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--ref-budget", type=float, default=240.0,
                    help="--impl reference: wall seconds for the timed CPU steps (at least one step)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn(args.gpus)  # one process per GPU, started here (no external torchrun needed)
    rank, world, dist = dist_init(args.gpus)
    if args.impl == "reference":
        run_reference(args, rank, world, dist)
    elif args.solver == "direct":
        run_direct(args, rank, world, dist)
    else:
        run_ours(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
