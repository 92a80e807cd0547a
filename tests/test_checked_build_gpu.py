"""GPU: the kernels under device-side bounds checks (build/checked/
libcafxg_checked.so: the same sources with -DCAFXG_DEVICE_CHECKS, dcheck.cuh).
A check that fails traps, the context is lost and the run fails loudly -- the
stand-in for compute-sanitizer memcheck, which this pool does not offer.

Runs every kernel kind at small and edge sizes (tools/sanitize_cases.py:
coordinate tables, multi-tile batches, actor batches with the reply scatter
and direct replies, the deferred kernel's replays, FFMA / 3xTF32 / pipelined
sgemm, device FNV, run_mandelbrot) and the Mandelbrot, sgemm and
multi-device parity tests, each over the checked library."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "build", "checked", "libcafxg_checked.so")


def _env():
    if not os.path.exists(CHECKED):
        pytest.fail("checked build missing: make -C paper_1505_07368_b200/csrc checked")
    return dict(os.environ, CAFXG_LIB=CHECKED)


def test_checks_fire():
    """The checks are live: with CAFXG_DCHECK_SELFTEST the output limit is one
    element, the escape kernel's first store past it traps, and the request
    fails with E_DOWN (14) instead of writing out of bounds."""
    code = r"""
import sys
sys.path.insert(0, %r)
import paper_1505_07368_b200 as pkg
with pkg.Context(1) as c:
    try:
        c.mandelbrot(pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 64, 64, 50))
        print("no trap")
    except pkg.CafxgError as e:
        print("trapped", e.code)
""" % ROOT
    r = subprocess.run([sys.executable, "-c", code], env=dict(_env(), CAFXG_DCHECK_SELFTEST="1"),
                       capture_output=True, text=True, timeout=300)
    assert "trapped 14" in r.stdout, (r.stdout + r.stderr)[-3000:]


def test_sanitize_cases_under_checks():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "paper_1505_07368_b200", "tools",
                                                     "sanitize_cases.py")],
                       env=_env(), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "sanitize cases ok" in r.stdout, (r.stdout + r.stderr)[-3000:]


@pytest.mark.parametrize("suite,select", [
    ("test_mandelbrot_gpu.py", "not full_image"),
    ("test_sgemm_gpu.py", "not cfg5_full_size"),
    ("test_multidevice_gpu.py", ""),
    ("test_actor_gpu.py", "not c_program"),  # (that one links libcafxg.so itself)
])
def test_parity_suites_under_checks(suite, select):
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", suite)]
    if select:
        cmd += ["-k", select]
    r = subprocess.run(cmd, env=_env(), capture_output=True, text=True, timeout=1500, cwd=ROOT)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
