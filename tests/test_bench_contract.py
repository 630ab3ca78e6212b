"""bench.py contract checks that need no GPU: the reference arm (the oracle on the host cores) prints
one JSON line with the keys the driver reads, and the T1 reference arm reports itself unavailable."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line_small_config():
    import time
    t0 = time.perf_counter()
    d = _run("--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "3")
    wall = time.perf_counter() - t0
    # ms_per_step is the measured time of one bounded step (no extrapolation): it fits the run
    assert d["steps"] * d["ms_per_step"] / 1000.0 <= wall
    assert set(d["config"]) == {"workload", "global_batch"} and d["config"]["global_batch"] == 1
    f = d["step"]["fraction_of_call"]
    assert 0 < f <= 1 and abs(d["value"] - d["step"]["rhs_equivalent_per_step"] / (d["ms_per_step"] / 1000)) \
        <= 1e-9 * d["value"]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_t1_unavailable():
    d = _run("--impl", "reference", "--config", "T1")
    assert d["impl"] == "reference" and "unavailable" in d
