"""The bench's reference arm (`bench.py --impl reference`) runs on the host alone: one JSON line
with the driver contract's keys (metric/value/unit/..., impl, cpu_baseline, e2e)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "2", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "config", "impl",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["warmup"] >= 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("c1")


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_gpus_flag_relaunches_one_rank_per_gpu():
    """`--gpus N` without torchrun relaunches the script as N local ranks (127.0.0.1); rank 0
    alone prints, and the line reports the launch width."""
    d = _run(["--impl", "reference", "--gpus", "2", "--config", "c1", "--steps", "1",
              "--warmup", "3"])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "row-shard dp2"


def test_extrapolated_cpu_baselines_for_large_configs():
    """c3 (row sample x p / p_sample) and c4 (blocked ||X||^2 x (p / p_sample)^2) reference lines
    carry their sampling, best and median, labelled as extrapolated."""
    for cfg, unit_metric in (("c3", "f+grad evals/s"), ("c4", "||X||^2 evals/s")):
        d = _run(["--impl", "reference", "--config", cfg, "--steps", "1", "--warmup", "3"])
        cb = d["cpu_baseline"]
        assert d["metric"] == unit_metric and cb["extrapolated"] is True
        assert "EXTRAPOLATED" in cb["sample"] and cb["best"] >= cb["value"] > 0
