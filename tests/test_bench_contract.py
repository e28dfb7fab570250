"""bench.py's reference arm (CPU oracle) prints the contract's JSON line; the
GPU arm's keys are checked on the B200 (gpu marker)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _last_json(out):
    return json.loads(out.strip().splitlines()[-1])


# run bench.py's reference arm in-process, then list the shared objects it mapped
_MAPS = """
import runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"]
try:
    runpy.run_path("bench.py", run_name="__main__")
except SystemExit:
    pass
libs = sorted({l.split()[-1] for l in open("/proc/self/maps") if l.rstrip().endswith(".so") or ".so." in l})
print("MAPPED", [x for x in libs if "/root/repo" in x or "msim" in x or "oracle" in x])
"""


@pytest.mark.timeout(600)
def test_reference_arm_line_and_no_product_loaded():
    """The reference arm times the reference's own code and never loads the product."""
    from oracle import oracle_py

    r = subprocess.run([sys.executable, "-c", _MAPS], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    d = json.loads(lines[-2])
    assert d["impl"] == "reference" and BASE_KEYS <= set(d)
    kind = "reference" if oracle_py.ref_available() else "port"
    assert d["cpu_baseline"]["kind"] == kind and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"] > 0
    mapped = lines[-1]
    assert "libmsim_gpu" not in mapped and "paper_2302_04659_b200" not in mapped, mapped
    if kind == "reference":
        assert "libmsim_ref.so" in mapped


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_gpu_arm_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--envs", "64",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["gpu_launches"] > 0
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["kernels"]["k_particles"]["launches"] > 0


@pytest.mark.timeout(600)
def test_launcher_relaunches_one_process_per_gpu():
    """bench.py --gpus 2 relaunches itself under torch.distributed.run (the
    driver's N > 1 launch); on the reference arm rank 0 alone prints the line
    and rank 1 exits 0 without work."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
