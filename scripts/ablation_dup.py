"""In-graph marginal cost of each per-iteration component on c4 (PF_DUP=1 one
more Gram solve, 2 one more local product, 3 one more coarse GEMV, 4 one more
tiny vector kernel): step and per-iteration times with and without."""
import os, sys, subprocess
sys.path.insert(0, '.')
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import paper_2509_06673_b200 as pf
    op = pf.FetiOperator(**pf.BASELINE_CONFIGS[os.environ.get("PF_ABL_CFG", "c4")])
    op.step()
    ms, it, _ = op.bench_steps(3)
    r = op.step()
    print(f"DUP {os.environ.get('PF_DUP', '0')} step {ms/3:.2f} ms it {it/3:.0f} per-iter {r['t_krylov']*1e6/r['iterations']:.1f} us", flush=True)
    sys.exit(0)
for d in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "1", "2", "3", "4", "5", "0"]):
    out = subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, PF_DUP=d), capture_output=True, text=True)
    print([l for l in out.stdout.splitlines() if l.startswith("DUP")] or out.stderr[-300:], flush=True)
