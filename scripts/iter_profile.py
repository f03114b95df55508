"""One c4 time step for ncu launch lists (profiled region: the second step,
between cudaProfilerStart/Stop; run ncu with --profile-from-start off).
PF_HOST_LOOP=1 makes every Krylov iteration its own graph launch so the
summary can cut one steady-state iteration (scripts/ncu_iter_summary.py)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
op = pf.FetiOperator(**pf.BASELINE_CONFIGS[cfg])
op.step()
rt = None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        rt = ctypes.CDLL(name)
        break
    except OSError:
        pass
if rt is None:
    import glob
    import nvidia.cuda_runtime as cr
    rt = ctypes.CDLL(glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*"))[0])
rt.cudaProfilerStart()
rep = op.step()
rt.cudaProfilerStop()
print("step", rep["iterations"], "iterations", rep["seconds"] * 1e3, "ms")
