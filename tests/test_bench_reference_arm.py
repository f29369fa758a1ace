"""bench.py --impl reference on CPU: the driver's reference arm prints one
strict-JSON line with the contract's keys (the CPU restatement of the
reference's path, oracle/, timed on the reference's own wall_ms scope)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _strict(text):
    def bad(c):
        raise ValueError(f"non-strict JSON constant {c}")
    return json.loads(text, parse_constant=bad)


def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                          "--steps", "3", "--warmup", "3"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = _strict(lines[0])
    assert d["impl"] == "reference"
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_finite_sanitizer():
    sys.path.insert(0, ROOT)
    import bench
    line = {"a": float("inf"), "b": [1.0, float("nan")], "c": {"d": -float("inf"), "e": 2}}
    assert _strict(json.dumps(bench._finite(line), allow_nan=False)) == {
        "a": None, "b": [1.0, None], "c": {"d": None, "e": 2}}


def test_reference_arm_under_torchrun_prints_once():
    """N>1: rank 0 alone runs and prints; the other ranks exit 0 without work."""
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", "29617", "bench.py", "--impl", "reference",
                          "--gpus", "2", "--config", "1", "--steps", "3", "--warmup", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = _strict(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
