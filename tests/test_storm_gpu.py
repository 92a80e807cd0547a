"""GPU: bench.py's request-storm measurement (BASELINE config 4) at a reduced
size -- the native driver in its three client disciplines (open loop, closed
loop with one OS thread per client, closed loop with the clients multiplexed
on worker threads like cafx actors) and the cafx client actors on the
unmodified reference runtime (tools/storm_cafx.cpp, closed and open loop, the
scheduler in its default configuration and with CAFX_WORKERS set); every
reply of every mode checked against the reference's own mandelbrot_cell."""
import os
import types

import pytest

import bench

pytestmark = pytest.mark.gpu


def test_storm_all_modes(ctx):
    args = types.SimpleNamespace(no_cpu_baseline=False)
    res = bench.sec_cfg4(ctx, args, 1, clients=8, per=64)
    native = ["cfg4_request_storm", "cfg4_request_storm_closed_loop",
              "cfg4_request_storm_closed_loop_os_threads"]
    for k in native:
        r = res[k]
        assert r["status"] == 0 and r["errors"] == 0, (k, r)
        assert r["requests"] == 8 * 64 and r["checked_tiles"] == 8 * 64
        assert r["mismatched_tiles"] == 0, (k, r)
        assert r["batches"] >= 1
    assert res["cfg4_request_storm"]["cpu_baseline"]["value"] > 0
    if os.path.exists(os.path.join(bench.ROOT, "build", "tests", "storm_cafx")):
        cafx = [k for k in res if k.startswith("cfg4_request_storm_cafx_actors")]
        assert len(cafx) == 4
        for k in cafx:
            r = res[k]
            assert r["status"] == 0, (k, r)
            assert r["good"] == 8 * 64 and r["bad"] == 0 and r["errors"] == 0, (k, r)


def test_storm_full_size_every_reply(ctx):
    """BASELINE config 4 at its full size: 64 clients x 1,600 requests =
    102,400 fp64 64x64 tiles in every client discipline, each reply checked
    against the unmodified reference's mandelbrot_cell (the bench's own
    measurement path, run here as a parity test)."""
    args = types.SimpleNamespace(no_cpu_baseline=False)
    res = bench.sec_cfg4(ctx, args, 1)
    for k in ["cfg4_request_storm", "cfg4_request_storm_closed_loop",
              "cfg4_request_storm_closed_loop_os_threads"]:
        r = res[k]
        assert r["status"] == 0 and r["errors"] == 0, (k, r)
        assert r["checked_tiles"] == 102400 and r["mismatched_tiles"] == 0, (k, r)
    for k in [k for k in res if k.startswith("cfg4_request_storm_cafx_actors")]:
        r = res[k]
        assert r["status"] == 0 and r["good"] == 102400 and r["bad"] == 0, (k, r)
