"""bench.py's reference arm on CPU: one JSON line with the contract's keys,
the same workload/metric/unit as our arm, e2e with zero copy bytes (the GPU
arm runs on the B200 box)."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "0", "--cpu-grid", "6"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "edges/s" and d["higher_is_better"] is True
    # the workload label is the sample that actually ran, not the 94^3 target
    assert d["config"]["workload"] == "hydra-proxy iteration, 3-D grid 6^3"
    assert d["config"]["sample_of"] == "hydra-proxy iteration, 3-D grid 94^3"
    import conftest
    want = "reference" if conftest.import_reference() is not None else "port"
    assert d["cpu_baseline"]["kind"] == want and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"] > 0


def test_cpu_baseline_runs_stock_reference_modes():
    """cpu_baseline times the stock reference in serial / threads / ranks mode."""
    import argparse
    import conftest
    if conftest.import_reference() is None:
        import pytest
        pytest.skip("stock reference not installed")
    sys.path.insert(0, str(ROOT))
    import bench
    args = argparse.Namespace(workload="proxy", grid=5, cpu_grid=4, cpu_sample_only=False)
    cb = bench.cpu_baseline(args)
    assert cb["kind"] == "reference" and set(cb["modes"]) == {"serial", "threads", "ranks"}
    assert cb["modes"]["serial"]["workload"].endswith("5^3")
    assert cb["modes"]["ranks"]["run_program_calls"] == 2 and cb["value"] > 0
    assert cb["cpu_model"]


def test_gpus_n_self_launches_ranks_without_torchrun():
    """``python bench.py --gpus 2`` with no WORLD_SIZE starts its own rank
    processes (127.0.0.1 rendezvous), prints rank 0's one line, exits 0."""
    import os
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--launch-probe"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d == {"probe": "ok", "world": 2, "sum": 3.0}


def test_gpus_n_self_launch_propagates_rank_failure():
    import os
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--launch-probe",
                          "--launch-probe-fail", "1"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env=env)
    assert out.returncode == 3
