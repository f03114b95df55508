import sys, time
sys.path.insert(0, '.')
import paper_2509_06673_b200 as pf
for name in sys.argv[1].split(","):
    kw = dict(pf.BASELINE_CONFIGS[name], max_iter=int(sys.argv[2]) if len(sys.argv) > 2 else 3000)
    op = pf.FetiOperator(**kw)
    for k in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
        try:
            r = op.step()
            print(name, "step", r["step"], "iters", r["iterations"], "rel %.2e" % r["rel_residual"], "s %.2f" % r["seconds"], flush=True)
        except Exception as e:
            print(name, "FAILED", e, flush=True)
            break
    op.close()
