"""bench.py's JSON contract, checked on CPU through the reference arm
(--impl reference times the reference's own potential code on host cores, no
GPU needed): one JSON line with the driver's keys and a cpu_baseline / e2e
that describe the run."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "sbm100k", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GPairs/s" and d["higher_is_better"]
    assert "workload" in d["config"] and d["steps"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


import pytest  # noqa: E402


@pytest.mark.gpu
def test_native_arm_json_line_on_gpu():
    """The native arm at N = 1 on a B200 (SBM workload, short): every key of
    the driver's contract plus roofline / cpu_baseline / e2e / e2e_qc /
    gpu_launches / clocks, with the roofline naming its binding resource and
    the ncu figures attached only from this workload's capture."""
    r = subprocess.run([sys.executable, "bench.py", "--workload", "sbm100k", "--steps", "3", "--warmup", "3",
                        "--cpu-seconds", "2"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "e2e_qc", "gpu_launches",
              "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0 and d["gpu_launches"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "issue" and rf["unit"] == "GB/s" and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert rf["traffic_source"].startswith("profiles/traffic.json workloads.sbm100k") or rf["traffic"] is None
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" or cb["kind"] == "port"
    assert "bit-identical: True" in cb["sample"]
    assert d["e2e_qc"] and d["e2e_qc"].get("seconds", 0) > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
