"""Direct interface solve (krylov="direct", the GPU analogue of the reference's
monolithic solver): setup and per-step device time on BASELINE configs whose
interface fits the dense inverse (c1, c2, c3, c5), next to the FETI Krylov
path on the same config, and the per-step GEMV against the HBM roofline.

    python scripts/direct_bench.py [c2 c3 c5] [--steps K] [--krylov]

One JSON line per config (CUDA events on the engine stream; setup = the
pf_create wall time)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_06673_b200 as pf  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6538.9


def run(cfg, steps, krylov, warm=2):
    kw = dict(pf.BASELINE_CONFIGS[cfg])
    kw["steps"] = max(kw["steps"], warm + steps + 1)
    kw["krylov"] = krylov
    t0 = time.perf_counter()
    op = pf.FetiOperator(**kw)
    setup = time.perf_counter() - t0
    for _ in range(warm):
        op.step()
    ms, iters, _ = op.bench_steps(steps)
    out = {"config": cfg, "krylov": krylov, "n_lambda": op.n_lambda, "n_coarse": op.info.n_coarse,
           "setup_s": setup, "s_per_step": ms * 1e-3 / steps, "iterations_per_step": iters / steps}
    if krylov == "direct":
        n, nc = op.n_lambda, op.info.n_coarse
        t = op.bench(6, 5, 20)[0]
        b = 8.0 * n * (n + nc)
        out["gemv"] = {"kernel": "k_gemv_rows: lambda = [Z | Y_c] [rhs; e], row-major, HBM-streamed",
                       "ms": t, "bytes": b, "gbs": b / (t * 1e-3) / 1e9, "peak_gbs": peak(),
                       "frac": b / (t * 1e-3) / 1e9 / peak()}
        rep = op.step()
        out["true_residual"] = rep["true_residual"]
        out["t_rhs_ms"], out["t_solve_ms"], out["t_back_ms"] = (rep["t_rhs"] * 1e3, rep["t_krylov"] * 1e3,
                                                               rep["t_back"] * 1e3)
    op.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c3", "c5"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--krylov", action="store_true", help="also time the FETI Krylov path")
    a = ap.parse_args()
    for c in a.configs:
        print(json.dumps(run(c, a.steps, "direct")), flush=True)
        if a.krylov:
            print(json.dumps(run(c, a.steps, "auto")), flush=True)


if __name__ == "__main__":
    main()
