"""One time step through the direct interface solve for ncu (profiled region:
the third step, between cudaProfilerStart/Stop; run ncu with
--profile-from-start off).

    ncu --profile-from-start off ... python scripts/direct_profile.py [c4]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_06673_b200 as pf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
op = pf.FetiOperator(**dict(pf.BASELINE_CONFIGS[cfg], krylov="direct"))
op.step(), op.step()
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
print("step", rep["seconds"] * 1e3, "ms, true residual", rep["true_residual"])
