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


def test_reference_arm_times_the_whole_scene_without_the_product_library():
    """The arm's workload is the GPU arm's (every observation of the config,
    rounds 1..K) and its process never maps libdbag.so."""
    code = ("import sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', '2', "
            "'--steps', '2', '--warmup', '3']; import bench; rc = bench.main(); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT_LOADED' if 'libdbag' in maps else 'CLEAN', rc)")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "CLEAN 0" in out.stdout
    d = _strict([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    scene = O.generate_config_scene(2, 0)
    assert d["config"]["observations"] == len(scene["obs_cam"])
    assert d["config"]["cameras"] == 64 and len(d["round_ms"]) == 2
    assert str(len(scene["obs_cam"])) in d["cpu_baseline"]["sample"]
