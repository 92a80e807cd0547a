"""GPU: the paper's CPU/GPU offload experiment (SURVEY.md §8f
row 3) on the unmodified reference runtime: a 1920x1080 image split between
cafx CPU row actors and one B200 compute-actor request at GPU shares 0..100 %
(tests/cpp/offload_split.cpp). Every run's assembled image must equal the
all-GPU image (FNV-1a checksum), i.e. CPU and GPU evaluate the same fp32
contract bit for bit."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "tests", "offload_split")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN),
                    reason="offload experiment not built (needs /root/reference at build time)")
def test_offload_shares_reproduce_the_gpu_image():
    r = subprocess.run([BIN, "--runs", "2", "--iters", "120,1200", "--json"],
                       capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = [json.loads(line) for line in r.stdout.splitlines() if line.startswith("{")]
    assert len(rows) == 22
    assert all(x["checksum_ok"] for x in rows)
    for it in (120, 1200):
        by = {x["gpu_share"]: x for x in rows if x["max_iter"] == it}
        assert sorted(by) == list(range(0, 101, 10))
        # all on the GPU beats all on the CPU
        assert by[100]["total_ms"] < by[0]["total_ms"]
        assert by[0]["gpu_ms"] == 0 and by[100]["cpu_ms"] == 0
