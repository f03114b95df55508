"""bench.py's launch contract on CPU: --gpus N starts its own N ranks (no
external torchrun), rank 0 prints one JSON line, the other ranks exit 0.
The reference arm runs on the host cores, so it is exercised here at c1."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_reference_arm_two_ranks_spawned_by_bench():
    line = run("--gpus", "2", "--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["steps"] >= 1 and line["value"] > 0 and len(line["step_seconds"]) == line["steps"]
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_single_process():
    line = run("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert line["n_gpus"] == 1 and line["steps"] == 2 and line["iterations"][0] > 0
