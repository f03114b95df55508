import sys, time, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_2509_06673_b200 as pf
from oracle_lib import Oracle
def cmp(name, kw, steps):
    t=time.time()
    op = pf.FetiOperator(**kw)
    t1=time.time()
    o = Oracle(**kw)
    # F-apply parity
    rng = np.random.default_rng(1); x = rng.uniform(-1,1,op.n_lambda)
    ya = op.apply(x); yo = o.apply(x)
    za = op.apply_preconditioner(x); zo = o.precond(x)
    print(name, "setup %.2fs"%(t1-t), "info", dict(n_lambda=op.info.n_lambda, nnzL=op.info.nnz_L, tasks=op.info.n_tasks, sn=op.info.n_supernodes),
          "apply rel %.2e precond rel %.2e"%(np.linalg.norm(ya-yo)/np.linalg.norm(yo), np.linalg.norm(za-zo)/np.linalg.norm(zo)), flush=True)
    o.run(steps)
    for k in range(1, steps+1):
        rep = op.step()
        xs, lam = op.state(); xo, lo = o.state(k)
        err = max(np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-300) for a,b in zip(xs,xo))
        print("  step", k, "iters", rep["iterations"], "oracle", o.report(k)["iterations"], "field err %.2e lam err %.2e"%(err, np.linalg.norm(lam-lo)/np.linalg.norm(lo)), "dev ms %.2f"%(rep["seconds"]*1e3), flush=True)
cmp("c1", dict(pf.BASELINE_CONFIGS["c1"]), 5)
cmp("c1-gen", dict(pf.BASELINE_CONFIGS["c1"], precond="generalized"), 2)
cmp("c2s", dict(pf.BASELINE_CONFIGS["c2"], mesh_n=32), 2)
cmp("c4s", dict(pf.BASELINE_CONFIGS["c4"], mesh_n=64, SX=8, SY=8), 2)
cmp("c5s", dict(pf.BASELINE_CONFIGS["c5"], mesh_n=64, SX=8, SY=8), 2)
cmp("c3s", dict(pf.BASELINE_CONFIGS["c3"], mesh_n=32, SX=4, SY=4, max_iter=2000), 1)
