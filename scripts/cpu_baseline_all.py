"""Measured CPU baselines on the GPU box's host cores (SURVEY 8d / BASELINE.md 2):
the oracle (C++ restatement of the reference algorithm) running real time
steps of every BASELINE config, steady_clock around each advance (REF's own
clock, feti.hpp:103), setup reported separately:
  * "restated-parallel": all host threads over subdomains, c1..c5;
  * "REF-literal" for c1: 2 threads (REF's std::async pair, feti.hpp:111-115).
One JSON line per run.  Usage: python scripts/cpu_baseline_all.py [cfg ...] [--steps K]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
import oracle_lib as ol  # noqa: E402
import paper_2509_06673_b200 as pf  # noqa: E402 (config table)

args = [a for a in sys.argv[1:] if not a.startswith("--")]
steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1
if "--steps" in sys.argv:
    args = [a for a in args if a != str(steps)]
runs = [(c, 0) for c in (args or ["c1", "c2", "c4", "c5", "c3"])]
if not args or "c1" in args:
    runs.insert(1, ("c1", 2))
for cfg, threads in runs:
    kw = dict(pf.BASELINE_CONFIGS[cfg])
    th = threads or os.cpu_count()
    t0 = time.perf_counter()
    o = ol.Oracle(**dict(kw, threads=th))
    setup = time.perf_counter() - t0
    n = min(steps + 1, kw["steps"])  # the first step is reported separately (warm-up)
    o.run(n)
    secs = [o.report(k)["seconds"] for k in range(1, n + 1)]
    its = [o.report(k)["iterations"] for k in range(1, n + 1)]
    timed = secs[1:] if n > 1 else secs
    print(json.dumps({"config": cfg, "mode": "REF-literal (2 threads)" if threads == 2 else "restated-parallel",
                      "threads": th, "setup_s": setup, "first_step_s": secs[0], "timed_steps": len(timed),
                      "step_s_mean": sum(timed) / len(timed), "step_s": timed, "iterations": its,
                      "n_lambda": o.n_lambda, "n_sub": o.n_sub}), flush=True)
    del o
