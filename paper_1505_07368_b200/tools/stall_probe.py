import os, sys, subprocess, tempfile, time
sys.path.insert(0, os.getcwd())
import bench, paper_1505_07368_b200 as pkg
from oracle import oracle
clients, per = 64, 40
arr = bench.storm_descs(clients * per, seed=5)
descs = (pkg.MandelDesc * (clients * per)).from_buffer(arr)
expect, _, _ = oracle.ref_tiles(descs, clients * per)
td = tempfile.mkdtemp()
dp, ep = os.path.join(td, "d.bin"), os.path.join(td, "e.u32")
arr.tofile(dp); expect.tofile(ep)
exe = sys.argv[1]
v = sys.argv[2]
stalls = 0
for i in range(int(sys.argv[3])):
    env = dict(os.environ, CAFXG_VIRTUAL_DEVICES=v)
    if "tsan" in exe:
        env["TSAN_OPTIONS"] = "suppressions=" + os.path.join(os.getcwd(), "tests/tsan.supp")
    t0 = time.time()
    try:
        r = subprocess.run([exe, dp, ep, str(clients), str(per), "closed"], env=env, capture_output=True, text=True, timeout=60)
        out = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    except subprocess.TimeoutExpired:
        out = "TIMEOUT"; stalls += 1
    print(i, round(time.time() - t0, 1), out[:160], flush=True)
print("stalls", stalls)
