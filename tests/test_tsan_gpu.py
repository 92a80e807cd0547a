"""GPU: ThreadSanitizer over the host runtime. libcafxg's host code and the
reference runtime are both built with -fsanitize=thread (build/tsan,
oracle/_ref/libcafx_ref_tsan.so); the cafx adapter checks and a cafx-actor
request storm (closed and open loop) must run with zero race reports."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "tests")


@pytest.mark.skipif(not os.path.exists(os.path.join(BIN, "test_gpu_actor_tsan")),
                    reason="TSAN builds need /root/reference at build time")
def test_no_thread_sanitizer_reports():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "paper_1505_07368_b200", "tools",
                                                     "tsan_run.py")],
                       capture_output=True, text=True, timeout=1500)
    print(r.stdout)  # the whole log in the captured output of a failure
    assert "TOTAL ThreadSanitizer warnings: 0; exit codes ok: True" in r.stdout
