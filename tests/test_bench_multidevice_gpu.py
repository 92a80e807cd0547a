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


def test_nccl_exchange_secondary_two_virtual_devices():
    """The N > 1 secondary that times cfg5's NCCL-exchange baseline: a context
    opened with CAFXG_SGEMM_P2P=0 takes the all-gather path (no peer GEMMs;
    on virtual devices NCCL itself is replaced by peer copies) while the
    default context reads B in place (peer_gemms), both within 1e-5; the
    switch is per context, so the environment is restored after the open."""
    code = r"""
import os, sys, json
sys.path.insert(0, %r)
import bench, numpy as np
import paper_1505_07368_b200 as pkg
from oracle import oracle
r = bench.sec_sgemm_nccl(2, n=2048)
assert "CAFXG_SGEMM_P2P" not in os.environ
n = 2048
A = oracle.fill_uniform(n * n, 1).reshape(n, n)
B = oracle.fill_uniform(n * n, 2).reshape(n, n)
with pkg.Context(1) as c:
    s0 = c.stats(); C = c.sgemm(A, B); s1 = c.stats()
rows = np.arange(0, n, 97, dtype=np.uint32)
err = oracle.sgemm_rel_err(C, oracle.sgemm_ref_rows(A, B, rows, n, n), rows, n)
print(json.dumps({"nccl": r, "fused_peer_gemms": int(s1.peer_gemms - s0.peer_gemms),
                  "fused_err": err}))
""" % ROOT
    env = dict(os.environ, CAFXG_VIRTUAL_DEVICES="2")
    env.pop("CAFXG_SGEMM_P2P", None)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    j = json.loads(r.stdout.strip().splitlines()[-1])
    assert j["nccl"]["peer_gemms"] == 0 and j["nccl"]["max_rel_err_e2e"] <= 1e-5
    assert j["fused_peer_gemms"] == 1 and j["fused_err"] <= 1e-5
