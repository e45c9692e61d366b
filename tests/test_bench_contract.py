"""bench.py's JSON-line contract (the driver parses these lines).

CPU: the reference arm on a tiny config, and its rank != 0 behaviour.
GPU: the device arm on a small config, every key the contract names.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def run_bench(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.update(env_extra or {})
    proc = subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, env=env,
                          timeout=timeout, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-2000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.strip()]
    return lines


def test_reference_arm_line():
    lines = run_bench(["--impl", "reference", "--n", "64", "--batch", "512", "--steps", "1", "--warmup", "3"])
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] == "port"
    assert "workload" in d["config"]


def test_reference_arm_other_ranks_print_nothing():
    lines = run_bench(["--impl", "reference", "--n", "8", "--batch", "64", "--steps", "1", "--warmup", "3"],
                      {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert lines == []


def test_warmup_below_three_is_rejected():
    proc = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--warmup", "2"], capture_output=True,
                          text=True, cwd=ROOT)
    assert proc.returncode != 0


@pytest.mark.gpu
def test_gpu_arm_line(cuda):
    lines = run_bench(["--n", "256", "--batch", "65536", "--steps", "5", "--warmup", "3", "--no-cpu",
                       "--e2e-steps", "1"], timeout=900)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 5 and d["scaling"] == "weak"
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == 65536 * 256 * 8 == e2e["d2h_bytes_per_step"]
    roof = d["roofline"]
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s" and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-3
    assert d["gpu_launches"] == 5
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["parity_rel_l2_max_first64_vs_numpy_c128"] < 1e-5 * 8
    # BASELINE configs[2] (sweep) and configs[3] (c4) ride on the same line
    sweep = d["sweep"]
    assert [(p["precision"], p["n"]) for p in sweep["points"]] == [
        (prec, 2**k) for prec in ("single", "double") for k in range(1, 12)]
    for p in sweep["points"]:
        assert p["batch"] * p["n"] * (8 if p["precision"] == "single" else 16) == 1 << 30
        assert p["gbs"] > 0 and abs(p["frac"] - p["gbs"] / sweep["peak_gbs"]) < 1e-3
        tol = (1e-5 if p["precision"] == "single" else 1e-13) * (p["n"].bit_length() - 1)
        assert p["parity_rel_l2_max_vs_numpy_c128"] <= tol
        assert "sm_mhz" in p["clocks"]
    c4 = d["c4"]
    assert c4["roofline"]["algorithmic_bytes_per_launch"] == 2 * 131072 * 2048 * 16
    assert c4["parity_rel_l2_max_vs_numpy_c128"] <= 1e-13 * 11 and c4["value"] > 0
    sus = d["sustained"]
    assert [(p["precision"], p["n"]) for p in sus["points"]] == [("single", 1024), ("double", 2048)]
    for p in sus["points"]:
        assert p["copy_gbs"] > 0 and p["fft_gbs"] > 0
        assert abs(p["fft_over_sustained_copy"] - p["fft_gbs"] / p["copy_gbs"]) < 1e-3
        assert "sm_mhz" in p["fft_clocks"] and "sm_mhz" in p["copy_clocks"]


@pytest.mark.gpu
def test_gpu_arm_two_ranks_with_cpu_baseline(cuda):
    """bench.py --gpus 2 under torchrun: two ranks share the one GPU of the
    test box through the SFFT_BENCH_DEVICE / gloo hooks.  Checks the
    whole-job accounting and that rank 0 adds the CPU baseline at N > 1."""
    lines = run_bench(["--gpus", "2", "--n", "128", "--batch", "32768", "--steps", "4", "--warmup", "3",
                       "--e2e-steps", "1", "--cpu-seconds", "1.5"],
                      {"SFFT_BENCH_DEVICE": "0", "SFFT_BENCH_DIST_BACKEND": "gloo"}, timeout=900)
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 2 * 32768 and d["scaling"] == "weak"
    assert d["config"]["batch_per_gpu"] == 32768
    cpu = d["cpu_baseline"]
    assert cpu["kind"] == "port" and cpu["cores"] >= 1 and cpu["value"] > 0
    for leg in ("all_cores", "single_process", "per_row_loop", "per_row_loop_all_cores"):
        assert cpu[leg]["value"] > 0 and cpu[leg]["cores"] >= 1
    assert cpu["single_process"]["cores"] == 1 and cpu["per_row_loop"]["cores"] == 1
    assert "sweep" not in d  # the configs[2]/[3] keys are single-GPU lines only
