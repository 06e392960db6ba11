"""bench.py keeps the driver contract: one JSON line with the required keys."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    line = _run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1", "--cpu-target-s", "1"])
    assert BASE_KEYS <= set(line) and line["impl"] == "reference"
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0
    assert line["config"]["workload"] == "C1"
    assert line["config"]["triples_structural"] == 4884 and line["config"]["nnzb_c_structural"] == 1016
    assert line["sampling"]["c_block_rows"] >= 1


def test_default_workload_is_the_largest_single_gpu_config():
    """The driver's N=1 line is quoted on C5-64 (BASELINE configs[4]: the largest configuration that
    fits one B200), and N > 1 runs strong-scale it."""
    import bench

    assert bench.DEFAULT_CONFIG == "C5-64"


@pytest.mark.gpu
def test_gpu_arm_contract():
    line = _run(["--config", "C2-16384", "--steps", "4", "--warmup", "3", "--cpu-target-s", "1"])
    assert BASE_KEYS <= set(line) and "impl" not in line
    assert line["value"] > 1000 and line["higher_is_better"] and line["dtype"] == "f64"
    r = line["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1.2
    assert set(line["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    p = line["e2e"]["pcie"]  # the box's pinned-copy floor next to the e2e number
    assert p["bidir_gbs"] > 0 and 0 < p["frac_of_floor"] <= 1.2
    assert line["result"]["triples_executed"] == line["config"]["triples_structural"]  # dense blocks: nothing skipped
    assert line["operand_metadata"]["kernel"] == "k_block_meta"
    ref = _run(["--impl", "reference", "--config", "C2-16384", "--steps", "1", "--warmup", "0",
                "--cpu-target-s", "1"])
    assert ref["config"] == line["config"]  # both arms print the same workload definition
    assert line["cpu_baseline"]["value"] > 0 and line["cpu_baseline"]["kind"] == "port"


def test_committed_traffic_is_per_kernel_and_source():
    """roofline.traffic comes from a committed ncu capture only when it was taken on the same
    kernel and kernel source the bench is running (a stale or foreign entry reads as None)."""
    import bench

    t, note = bench.committed_traffic("C5-64")  # k_numeric_tma capture of the default workload
    assert (t is None and "not the current" in note) or t > 7e10
    t, note = bench.committed_traffic("C5-64", "k_numeric_quad32")
    assert t is None and "k_numeric_tma" in note
    t, note = bench.committed_traffic("C5-32", "k_numeric_tma")  # the C5-32 capture is of the quad kernel
    assert t is None
    assert bench.committed_traffic("no-such-workload")[0] is None
    assert bench.kernel_source_sha("k_numeric_tma") != bench.kernel_source_sha("k_numeric_quad32")
