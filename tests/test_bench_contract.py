"""CPU: bench.py's launch contract without a GPU.

* `--gpus N` must fail loudly when fewer than N devices are visible (a run
  that silently measured one GPU would misreport n_gpus);
* under torchrun (world 2, gloo, 127.0.0.1) the reference arm prints exactly
  one JSON line, from rank 0, and every rank exits 0.
"""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gpus_above_visible_devices_fails_loudly():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode != 0
    assert "CUDA device(s) visible" in r.stderr
    assert r.stdout.strip() == ""


def test_torchrun_world2_reference_arm_prints_once():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", CAFXG_SKIP_PAPER_SCALE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(free_port()),
                        os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["n_gpus"] == 2 and j["value"] > 0
    assert j["cpu_baseline"]["cores"] >= 1 and j["e2e"]["h2d_bytes_per_step"] == 0


def test_guarded_secondary_records_the_error():
    sys.path.insert(0, ROOT)
    import bench
    out = {}
    bench.guarded(out, "ok", lambda: {"v": 1})
    bench.guarded(out, "bad", lambda: 1 / 0)
    assert out["ok"] == {"v": 1}
    assert out["bad"]["error"].startswith("ZeroDivisionError")


WATCHDOG_SCRIPT = r"""
import os, sys, time
sys.path.insert(0, os.environ["ROOT"])
import bench
D = bench.Dist()
if D.rank != 0:
    D.barrier(); D.close(); sys.exit(0)
line = {"metric": "m", "value": 1.0}
bench.SECONDARY_BUDGET_S = 1.0
dog = bench.Watchdog(line, 1.0, D)
dog.out["first"] = {"done": True}
time.sleep(120)   # a secondary that never returns
print("not reached", flush=True)
"""


def test_watchdog_prints_headline_and_releases_ranks(tmp_path):
    script = tmp_path / "dog.py"
    script.write_text(WATCHDOG_SCRIPT)
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", ROOT=ROOT)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", str(free_port()), str(script)], env=env,
                       capture_output=True, text=True, timeout=100)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and "not reached" not in r.stdout
    j = json.loads(lines[0])
    assert j["value"] == 1.0 and j["secondary"]["first"] == {"done": True}
    assert "watchdog" in j["secondary"]
