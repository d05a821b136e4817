"""The bench's reference arm (the oracle, CPU) prints one JSON line with the
contract's keys; runs here without a GPU (a few seconds)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"].startswith("config2")


def test_bench_sets_hardware_queues_before_cuda():
    """bench.py sets CUDA_DEVICE_MAX_CONNECTIONS=32 at import, before anything
    creates a CUDA context (the pipelined step's streams would otherwise share
    8 hardware queues and serialise); a caller's own value wins."""
    code = "import os, sys; sys.path.insert(0, %r); import bench, torch; " \
           "print(os.environ['CUDA_DEVICE_MAX_CONNECTIONS'], torch.cuda.is_initialized())" % ROOT
    env = {k: v for k, v in os.environ.items() if k != "CUDA_DEVICE_MAX_CONNECTIONS"}
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.split() == ["32", "False"]
    env["CUDA_DEVICE_MAX_CONNECTIONS"] = "16"
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.stdout.split()[0] == "16"
