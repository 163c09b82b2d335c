"""bench.py's reference arm (the oracle, timed on the host) keeps the JSON contract on CPU:
one line, impl = reference, the same config dict as the GPU arm, cpu_baseline and e2e blocks.
Under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    return [l for l in r.stdout.splitlines() if l.strip()]


def test_reference_arm_json_line():
    lines = run({}, "--config", "C2", "--n", "16", "--steps", "2", "--warmup", "3", "--cpu-seconds", "0.5")
    assert len(lines) == 1
    doc = json.loads(lines[0])
    assert doc["impl"] == "reference" and doc["higher_is_better"] is True
    assert doc["value"] > 0 and doc["unit"] == "nnz/s"
    import bench
    import inputs
    assert doc["config"] == bench.arm_config(inputs.config("C2", 16), 1)
    assert doc["cpu_baseline"]["kind"] == "oracle" and doc["cpu_baseline"]["value"] == doc["value"]
    assert doc["e2e"] == {"value": doc["value"], "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_silent():
    assert run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--config", "C1", "--steps", "1") == []
