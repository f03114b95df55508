"""A/B of engine settings on the in-graph c4 step: each variant (ENV=VAL[,ENV=VAL...]
or "base") runs in its own process, 3 device-resident steps after one warm-up;
prints ms/step, iterations and microseconds per Krylov iteration.  Variants
are interleaved twice (order effects).  Usage: python scripts/ab_env.py base PF_QU_G=0 ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import paper_2509_06673_b200 as pf
    cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
    op = pf.FetiOperator(**pf.BASELINE_CONFIGS[cfg])
    op.step()
    ms, it, _ = op.bench_steps(3)
    print(f"RES {ms / 3:.3f} {it / 3:.1f} {ms * 1e3 / it:.2f}", flush=True)
    sys.exit(0)
cfg = os.environ.get("AB_CFG", "c4")
variants = sys.argv[1:] or ["base"]
for rep in range(2):
    for v in variants:
        env = dict(os.environ)
        if v != "base":
            for kv in v.split(","):
                k, val = kv.split("=")
                env[k] = val
        out = subprocess.run([sys.executable, __file__, "run", cfg], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("RES")]
        print(v, line[0][4:] if line else out.stderr[-400:], flush=True)
