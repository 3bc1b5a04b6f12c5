"""CPU checks of bench.py's driver contract that need no GPU: the reference arm's JSON line (one
line, the required keys, rank 0 only under torchrun) on a tiny sample."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _run(args, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                         env=env, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    return [ln for ln in out.stdout.splitlines() if ln.strip()]


def test_reference_arm_line():
    lines = _run(["--impl", "reference", "--steps", "2", "--warmup", "0", "--ref-sample-rows", "1024",
                  "--rows", "4096", "--cols", "256"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert REQUIRED <= set(d), REQUIRED - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("configs[3]")


def test_reference_arm_nonzero_rank_is_silent():
    lines = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-sample-rows", "512",
                  "--rows", "2048", "--cols", "128"], env_extra={"RANK": "1", "WORLD_SIZE": "2"})
    assert lines == []
