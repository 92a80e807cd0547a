"""cfg4 through cafx client actors (tools/storm_cafx.cpp) under different
reference-scheduler settings: worker count (CAFX_WORKERS) x idle back-off.
    python paper_1505_07368_b200/tools/cafx_storm_sweep.py [clients per]"""
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

clients = int(sys.argv[1]) if len(sys.argv) > 1 else 64
per = int(sys.argv[2]) if len(sys.argv) > 2 else 1600
arr = bench.storm_descs(clients * per)
descs = (pkg.MandelDesc * (clients * per)).from_buffer(arr)
expect, _, _ = oracle.ref_tiles(descs, clients * per)
td = tempfile.mkdtemp()
dp, ep = os.path.join(td, "d.bin"), os.path.join(td, "e.u32")
arr.tofile(dp)
expect.tofile(ep)
exe = os.path.join(ROOT, "build", "tests", "storm_cafx")
for workers in (4, 8, 16, 32):
    for sleep in (None, 50):
        env = dict(os.environ, CAFX_WORKERS=str(workers))
        cmd = [exe, dp, ep, str(clients), str(per), "closed", "1"]
        if sleep is not None:
            cmd.append(str(sleep))
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        j = json.loads(r.stdout.strip().splitlines()[-1])
        print(json.dumps({"workers": workers, "steal_sleep_us": j["steal_sleep_us"],
                          "wall_ms": j["wall_ms"], "batches": j["batches"],
                          "good": j["good"]}), flush=True)
