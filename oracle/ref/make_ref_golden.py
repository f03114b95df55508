"""Golden vectors from the reference itself (TEST INFRASTRUCTURE ONLY).

Builds oracle/_ref/ref_driver (oracle/ref/Makefile: the unmodified reference
headers under /root/reference/proj/include compiled against the Eigen-API shim)
and converts its output into tests/golden/ref_<case>.npz.  Needs
/root/reference, i.e. runs in the CPU container; the fixtures travel with the
repository.

    python oracle/ref/make_ref_golden.py [case ...]
"""
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
GOLD = os.path.join(ROOT, "tests", "golden")
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

# case -> steps whose states are stored (errors are kept for every step)
CASES = {
    "c1-schur": 5, "c1-generalized": 5, "c1-monolithic": 5,
    "mms-m8": 2, "mms-m16": 2, "mms-m32": 2,
    "bm-m8": 3, "bm-m16": 3, "bm-m32": 3,
}


def parse(text):
    out = {}
    for line in text.splitlines():
        parts = line.split()
        if not parts:
            continue
        name, n = parts[0], int(parts[1])
        vals = np.array([float(v) for v in parts[2:2 + n]])
        assert vals.size == n, name
        out[name] = vals.item() if n == 1 and not name.startswith(("hist", "apply", "precond", "lambda")) else vals
    return out


FIELDS = ("u_P", "eta", "xi_P", "p", "u_E", "xi_E", "lambda")


def run(case, order="rcm"):
    env = dict(os.environ, EIGEN_SHIM_ORDER=order)
    p = subprocess.run([DRIVER, case, str(CASES[case])], check=True, capture_output=True, text=True, env=env)
    return parse(p.stdout)


def main():
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    for case in sys.argv[1:] or CASES:
        d = run(case)
        # the reference's own rounding spread: the same run with an equally
        # valid elimination order of its LU (Cuthill-McKee not reversed);
        # spread_<field><k> = relative L2 difference, spread_iters<k> = |diff|
        d2 = run(case, "cm")
        for k in range(1, CASES[case] + 1):
            if f"iters{k}" not in d:
                continue
            d[f"spread_iters{k}"] = abs(d[f"iters{k}"] - d2[f"iters{k}"])
            for f in FIELDS:
                a, b = d2[f"{f}{k}"], d[f"{f}{k}"]
                nb = np.linalg.norm(b)
                d[f"spread_{f}{k}"] = np.linalg.norm(a - b) / nb if nb > 0 else 0.0
        path = os.path.join(GOLD, "ref_" + case.replace("-", "_") + ".npz")
        np.savez_compressed(path, **d)
        its = [int(d[f"iters{k}"]) for k in range(1, CASES[case] + 1) if f"iters{k}" in d]
        print(case, "n_lambda", int(d["n_lambda"]), "iters", its,
              "linf_err_u", d.get("linf_err_u"), "->", os.path.relpath(path, ROOT))


if __name__ == "__main__":
    main()
