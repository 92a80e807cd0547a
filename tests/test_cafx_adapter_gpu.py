"""GPU: the CAF adapter (include/cafxg/gpu_actor.hpp) on the UNMODIFIED
reference runtime (oracle/_ref/libcafx_ref.so): cafx scoped, event-based and
typed clients request sm_100a compute actors (tests/cpp/test_gpu_actor.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "tests", "test_gpu_actor")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN),
                    reason="adapter test not built (needs /root/reference at build time)")
def test_gpu_actor_on_cafx_runtime():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout
    assert "FAIL" not in r.stdout.replace("ALL PASS", "")
