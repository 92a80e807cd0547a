"""Diagnostics: the cafx-actor storm (closed loop) standalone with the default
scheduler settings, with CAFX_WORKERS=16, and while this process holds an
idle cafxg context / after a native storm ran in it."""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..")
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1505_07368_b200 as pkg  # noqa: E402
from oracle import oracle  # noqa: E402

clients, per = 64, 1600
arr = bench.storm_descs(clients * per)
descs = (pkg.MandelDesc * (clients * per)).from_buffer(arr)
expect, _, _ = oracle.ref_tiles(descs, clients * per)
td = tempfile.mkdtemp()
dp, ep = os.path.join(td, "d.bin"), os.path.join(td, "e.u32")
arr.tofile(dp)
expect.tofile(ep)
exe = os.path.join(ROOT, "build", "tests", "storm_cafx")
print("nproc", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), flush=True)


def run(tag, env):
    r = subprocess.run([exe, dp, ep, str(clients), str(per), "closed", "1"], env=env,
                       capture_output=True, text=True, timeout=600)
    j = json.loads(r.stdout.strip().splitlines()[-1])
    print(tag, j["wall_ms"], j["scheduler_workers"], flush=True)


base = {k: v for k, v in os.environ.items() if k != "CAFX_WORKERS"}
run("standalone default", base)
run("standalone CAFX_WORKERS=16", dict(base, CAFX_WORKERS="16"))
ctx = pkg.Context(1)
run("parent holds an idle context", base)
import types  # noqa: E402
res = bench.sec_cfg4(ctx, types.SimpleNamespace(no_cpu_baseline=True), 1)
print("bench sec_cfg4 cafx closed:", res["cfg4_request_storm_cafx_actors_closed_loop"]["wall_ms"],
      flush=True)
run("after the native storms in the parent", base)
