"""Q-solve unit-kernel tuning: for each PF_QU_* setting, build c4 and time the
mortar Gram solve (bench kind 4), the preconditioner and one step."""
import os, subprocess, sys
sys.path.insert(0, '.')
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import paper_2509_06673_b200 as pf
    op = pf.FetiOperator(**pf.BASELINE_CONFIGS["c4"])
    q = op.bench(4, 20, 200)[0]
    m = op.bench(1, 20, 200)[0]
    op.step()
    r = op.step()
    print(f"RESULT {os.environ.get('TAG')} q {q*1e3:.1f} us precond {m*1e3:.1f} us step {r['seconds']*1e3:.2f} ms it {r['iterations']}", flush=True)
    sys.exit(0)
cfgs = [("1,64", "4,128"), ("2,64", "4,128"), ("4,64", "4,128"), ("2,32", "4,128"), ("4,32", "4,128"),
        ("8,32", "4,128"), ("1,32", "4,128"), ("2,64", "8,64"), ("2,64", "4,64"), ("2,64", "8,32")]
for a, b in cfgs:
    env = dict(os.environ, TAG=f"s0={a} s1={b}")
    env["PF_QU_S0"], env["PF_QU_R0"] = a.split(",")
    env["PF_QU_S1"], env["PF_QU_R1"] = b.split(",")
    out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True, timeout=300)
    print([l for l in out.stdout.splitlines() if l.startswith("RESULT")] or out.stderr[-500:], flush=True)
