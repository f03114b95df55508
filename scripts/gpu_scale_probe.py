import sys, time, json, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_2509_06673_b200 as pf
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2","c4"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for name in names:
    kw = dict(pf.BASELINE_CONFIGS[name])
    t = time.time()
    op = pf.FetiOperator(**kw)
    I = op.info
    print(name, "create %.1fs"%(time.time()-t), "setup %.1f asm %.1f factor %.1f upload %.1f"%(I.t_setup, I.t_assemble, I.t_factor, I.t_upload),
          "n_lambda", I.n_lambda, "nnzL %.3g"%I.nnz_L, "nnzLI %.3g"%I.nnz_L_interior, "sn", I.n_supernodes, "tasks", I.n_tasks, "types", I.n_types, "nc", I.n_coarse, flush=True)
    ms, sweep, launches = op.bench(0, 3, 10)
    print("  F-apply %.3f ms (sweep %.3f ms, %d launches) B_F %.3g GB -> %.0f GB/s (sweep-only %.0f GB/s)"%(ms, sweep, launches, I.bytes_fapply/1e9, I.bytes_fapply/ms/1e6, (16*I.nnz_L)/sweep/1e6), flush=True)
    print("  phases (ms)", pf.phase_stats(op, 3), flush=True)
    ms2, _, _ = op.bench(1, 2, 5)
    print("  precond %.3f ms, B_D %.3g GB -> %.0f GB/s"%(ms2, I.bytes_precond/1e9, I.bytes_precond/ms2/1e6 if I.bytes_precond else 0), flush=True)
    for k in range(steps):
        rep = op.step()
        print("  step", rep["step"], "iters", rep["iterations"], "conv", rep["converged"], "rel %.2e"%rep["rel_residual"], "dev %.3f s (rhs %.3f krylov %.3f back %.3f) fapplies %d"%(rep["seconds"], rep["t_rhs"], rep["t_krylov"], rep["t_back"], rep["f_applies"]), flush=True)
    op.close()
