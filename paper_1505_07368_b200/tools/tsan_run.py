"""Runs the ThreadSanitizer builds on a GPU box (build/tests/*_tsan, built by
`make -C paper_1505_07368_b200/csrc tsan && make -C tests/cpp tsan`): the cafx
adapter checks, then a cafx-actor request storm (closed and open loop) with
every reply checked. Prints each program's tail and the TSAN warning count.
    python paper_1505_07368_b200/tools/tsan_run.py > profiles/round2/tsan.log
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..")
sys.path.insert(0, ROOT)


def run(cmd, env):
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=1200)
    warnings = r.stderr.count("WARNING: ThreadSanitizer")
    print(f"$ {' '.join(os.path.basename(c) if i == 0 else c for i, c in enumerate(cmd))}")
    print(f"  exit {r.returncode}, ThreadSanitizer warnings: {warnings}")
    for line in r.stdout.strip().splitlines()[-40:]:
        print("  | " + line)
    if warnings:
        print("  -- first reports --")
        print("\n".join("  " + x for x in r.stderr.splitlines()[:200]))
    return r.returncode, warnings


def main():
    import bench
    from oracle import oracle
    supp = os.path.join(ROOT, "tests", "tsan.supp")
    # CAFX_WORKERS=4: under TSAN's slowdown the reference scheduler's idle
    # workers (hardware_concurrency of them, each sweeping the others' deques
    # under mutexes, scheduler.hpp:374-402) starve the instrumented backend
    # threads on a 16-core host with a 3-device context (the storm crawled:
    # 60 s timeouts with 16 workers, 2.5 s with 4; without TSAN 16 workers run
    # it in ~20 ms)
    env = dict(os.environ, CAFX_WORKERS="4",
               TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0 "
                            "second_deadlock_stack=1 history_size=4 "
                            f"suppressions={supp}")
    bt = os.path.join(ROOT, "build", "tests")
    total_w = 0
    rc, w = run([os.path.join(bt, "test_gpu_actor_tsan")], env)
    total_w += w
    # the same checks on a 3-device context (virtual devices on one GPU):
    # multi-device splitting, per-device issuer threads, peer-copy sgemm
    rc3, w = run([os.path.join(bt, "test_gpu_actor_tsan")],
                 dict(env, CAFXG_VIRTUAL_DEVICES="3"))
    total_w += w
    rc = rc or rc3
    clients, per = 16, 64
    arr = bench.storm_descs(clients * per, seed=77)
    import paper_1505_07368_b200 as pkg
    descs = (pkg.MandelDesc * (clients * per)).from_buffer(arr)
    expect, _, _ = oracle.ref_tiles(descs, clients * per)
    with tempfile.TemporaryDirectory() as td:
        dp, ep = os.path.join(td, "d.bin"), os.path.join(td, "e.u32")
        arr.tofile(dp)
        expect.tofile(ep)
        for mode in ("closed", "open"):
            rc2, w = run([os.path.join(bt, "storm_cafx_tsan"), dp, ep, str(clients), str(per),
                          mode], env)
            total_w += w
            rc = rc or rc2
    print(f"TOTAL ThreadSanitizer warnings: {total_w}; exit codes ok: {rc == 0}")


if __name__ == "__main__":
    main()
