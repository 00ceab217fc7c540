"""The bench.py contract (one JSON line on stdout, the keys the driver reads).

* CPU: the reference arm (`--impl reference`: the oracle timed on host cores on a
  bounded sample of the workload) on the small C1 workload.
* GPU: the main arm on C1 — roofline, cpu_baseline, e2e, clocks, gpu_launches.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


BASE = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    d = _run("--impl", "reference", "--workload", "C1", "--steps", "1", "--warmup", "3")
    assert BASE <= set(d), set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "cell-updates/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "C1"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_main_arm_line():
    d = _run("--workload", "C1", "--steps", "3", "--warmup", "3")
    assert BASE <= set(d), set(d)
    assert d["n_gpus"] == 1 and d["dtype"] == "f64" and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert r["achieved"] is None or abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and isinstance(c["reasons"], list)
    assert d["gpu_launches"] > 0
    assert len(d["config"]["schwarz_iters_per_step"]) == 3


def test_gpus_flag_launches_the_ranks():
    # `bench.py --gpus 2` without torchrun starts 2 ranks itself (gloo plumbing
    # check on CPU: every rank sees WORLD_SIZE = 2 and takes part in the
    # max-over-ranks reduction of the timed path)
    d = _run("--gpus", "2", "--launch-check", timeout=300)
    assert d["launch_check"] is True and d["world"] == 2 and d["n_gpus"] == 2
    assert sorted(d["ranks"]) == [0, 1] and d["max_over_ranks"] == 2.0


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1 but --gpus 2" in out.stderr
