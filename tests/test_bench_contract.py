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


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run with two
    ranks (probe mode: a gloo group, rank 0 reports what it saw)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--probe-ranks"],
                         capture_output=True, text=True, env=env, timeout=300, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and lines[0]["world"] == 2
    assert sorted(r["rank"] for r in lines[0]["ranks"]) == [0, 1]
    assert len({r["pid"] for r in lines[0]["ranks"]}) == 2


def test_world_size_mismatch_is_an_error():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "4", "--probe-ranks"],
                         capture_output=True, text=True, env=dict(os.environ, WORLD_SIZE="2", RANK="0"),
                         timeout=120, cwd=REPO)
    assert out.returncode != 0 and "WORLD_SIZE=2" in out.stderr


def test_cpu_sample_is_shared_by_both_legs():
    sys.path.insert(0, REPO)
    import bench
    for wl in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        a = bench.parse_args(["--workload", wl])
        spec = bench.cpu_sample_spec(a)
        assert spec["shapes"] and spec["desc"]
    a = bench.parse_args(["--ref-sample-rows", "4096"])
    assert bench.cpu_sample_spec(a)["shapes"] == [(4096, 2048)]


def test_executed_flop_model_cfg4():
    """configs[3]: SYRK Gram (36 of 64 pair tiles), 10 bf16x3 squarings on 136 128-tiles, single-term
    apply -> 3.71 TFLOP executed against 4.62 TFLOP of model FLOPs."""
    sys.path.insert(0, REPO)
    import bench
    e = bench.executed_flops_bf16_unso(2048, 262144, 14, 10, True, "persistent")
    assert abs(e["gram"] - 2 * 262144 * 256 * 256 * 36) < 1
    assert abs(e["chain"] - 10 * 3 * 2 * 2048 * 128 * 128 * 136) < 1
    assert abs(e["total"] / 1e12 - 3.71) < 0.01
