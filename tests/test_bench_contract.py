"""bench.py's reference arm runs on CPU and prints the driver's JSON contract."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    env = dict(os.environ, FVB_BENCH_CPU_SECONDS="0.2", FVB_BENCH_CPU_SMALL="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1"], capture_output=True, text=True, env=env, timeout=300, check=True)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["workload"].startswith("3D Euler p=16")
    ref = line.get("cpu_baseline_numpy")
    if ref and "value" in ref:   # the reference package is installed (baseline/_ref): both engine variants
        assert ref["kind"] == "reference" and ref["cores"] >= 1 and ref["value"] > 0
        assert ref["unshimmed_seq"]["cores"] == 1 and ref["unshimmed_seq"]["value"] > 0


def test_oracle_steps_time_full_slices():
    """The CPU baseline times full m-patch slices only (no ragged tail slice)."""
    import importlib.util

    import numpy as np

    import oracle

    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    n = 10
    q = oracle.synthetic_qin(2, 4, n, seed=5)
    rates, cores, m, ms = b.oracle_steps(q, np.ones((n, 2)), np.full(n, 0.01), 2, 4, steps=7, warmup=1,
                                         budget_s=1e-9)
    assert m == 1 and len(rates) == 7 and all(r > 0 for r in rates)


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1"],
                         capture_output=True, text=True, env=env, timeout=120, check=True)
    assert out.stdout.strip() == ""


def test_roofline_definitions_match_survey():
    """algorithmic bytes per patch and flops per cell for the bench configs."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    assert b.algorithmic_bytes_per_patch(2, 16) == 18_456
    assert b.algorithmic_bytes_per_patch(3, 16) == 389_144
    assert b.algorithmic_bytes_per_patch(3, 4) == 8_984
    assert abs(b.algorithmic_flops_per_cell(2, 16) - 112.0) < 0.05
    assert abs(b.algorithmic_flops_per_cell(3, 16) - 200.1) < 0.05
    assert abs(b.algorithmic_flops_per_cell(3, 4) - 257.5) < 0.05
    assert abs(b.FP64_PEAK_TFLOPS - 37.2) < 0.1
