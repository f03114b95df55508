"""Mortar Gram solve shape sweep on c4: dense-top cap (PF_Q_DENSE_TOP), task
cap (PF_Q_CAP), nested-dissection leaf (PF_Q_LEAF); Q-solve and step times."""
import os, subprocess, sys
sys.path.insert(0, '.')
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import paper_2509_06673_b200 as pf
    op = pf.FetiOperator(**pf.BASELINE_CONFIGS["c4"])
    q = op.bench(4, 20, 200)[0]
    op.step()
    ms, it, _ = op.bench_steps(2)
    print(f"RESULT {os.environ.get('TAG')} q {q*1e3:.1f} us step {ms/2:.2f} ms it {it/2:.0f} "
          f"qbytes {op.info.bytes_qsolve/1e6:.1f} MB", flush=True)
    sys.exit(0)
cfgs = [(2048, 1024, 8, 0), (2048, 1024, 8, 1), (2048, 512, 8, 0), (2048, 512, 8, 1), (2048, 256, 8, 1),
        (1536, 512, 8, 1), (2048, 512, 4, 1)]
if os.environ.get("QSWEEP"):
    cfgs = [tuple(int(v) for v in c.split(",")) for c in os.environ["QSWEEP"].split(";")]
for top, cap, leaf, sym in cfgs:
    env = dict(os.environ, PF_Q_DENSE_TOP=str(top), PF_Q_CAP=str(cap), PF_Q_LEAF=str(leaf), PF_COARSE_SYM=str(sym),
               TAG=f"top={top} cap={cap} leaf={leaf} coarse_sym={sym}")
    out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True, timeout=300)
    print([l for l in out.stdout.splitlines() if l.startswith("RESULT")] or out.stderr[-300:], flush=True)
