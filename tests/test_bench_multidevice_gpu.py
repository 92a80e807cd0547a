"""GPU: bench.py's N-device code path on one GPU. CAFXG_VIRTUAL_DEVICES=2
makes the context present two devices on device 0, so `--gpus 2` runs the
whole multi-device measurement (one request over two context devices, per-device
events, the C-ABI request split by the planner) -- the path the driver's
scaling run takes on an 8-GPU node. The line is marked as a code-path test."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_virtual_devices():
    env = dict(os.environ, CAFXG_VIRTUAL_DEVICES="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "2", "--warmup", "1", "--no-secondary", "--no-cpu-baseline"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    j = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert j["n_gpus"] == 2 and "VIRTUAL DEVICES" in j["data"]
    assert j["config"]["bit_exact_spot_check"] is True
    assert len(j["config"]["kernel_ms_per_device"]) == 2
    assert j["e2e"]["devices_used_mask"] == 3
    assert j["e2e"]["d2h_bytes_per_step"] == 16384 * 16384 * 4
    assert j["same_precision_fp64"]["bit_exact_spot_check"] is True
