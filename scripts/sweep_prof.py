"""Cycle accounting of the sweep kernel (PF_LIB=prof build, `make -C
paper_2509_06673_b200 prof`): per mode, share of warp time spent waiting on
the value ring, on slot/pivot prefetches and in the task prologue."""
import ctypes as C
import os
import sys
os.environ.setdefault("PF_LIB", "prof")
sys.path.insert(0, '.')
import paper_2509_06673_b200 as pf
op = pf.FetiOperator(**dict(pf.BASELINE_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"], steps=1))
L = pf.lib()
buf = (C.c_ulonglong * 32)()
L.pf_debug_sweep_prof(buf)  # reset
print(pf.phase_stats(op, 3))
L.pf_debug_sweep_prof(buf)
for m, name in enumerate(["fwd", "root", "bwd"]):
    tot, wait, slot, start, _, n = (buf[8 * m + i] for i in range(6))
    if n:
        print("%-4s tasks %8d  cycles/task %9.0f  ring wait %5.1f%%  slot wait %5.1f%%  prologue %5.1f%%" %
              (name, n, tot / n, 100 * wait / tot, 100 * slot / tot, 100 * start / tot))
