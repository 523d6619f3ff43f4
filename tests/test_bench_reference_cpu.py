"""The bench contract's reference arm (`bench.py --impl reference`: the CPU oracle as it
stands) runs on the host and prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny",
                          "--steps", "2", "--warmup", "1", "--ref-items", "16", "--ref-budget-s", "5"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["steps"] == 2 and d["warmup"] >= 3 and d["value"] > 0  # W >= 3 is enforced
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_gpus_flag_relaunches_one_process_per_gpu():
    """`bench.py --gpus 2` without WORLD_SIZE re-executes itself under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1); exercised here on the reference arm, where
    rank 0 alone prints the line and the other rank exits 0."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny",
                          "--gpus", "2", "--steps", "1", "--warmup", "1", "--ref-items", "16",
                          "--ref-budget-s", "3"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["cpu_baseline"]["cpu_model"] and d["cpu_baseline"]["value_1core"] > 0


def test_clock_sampler_reports_without_nvml():
    sys.path.insert(0, ROOT)
    import bench
    with bench.ClockSampler(0) as c:
        pass
    s = c.summary(0.0, 1.0)
    assert "reasons" in s and "samples" in s
