"""GPU: the native request-storm driver (BASELINE config 4) in its three client
disciplines -- open loop, closed loop with one OS thread per client, closed
loop with the clients multiplexed on worker threads like cafx actors -- at a
reduced size; sampled replies checked against the oracle."""
import pytest

import bench

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [False, True, "scheduled"])
def test_storm_modes(ctx, mode):
    r = bench.run_storm(ctx, clients=8, per=64, closed_loop=mode)
    assert r["status"] == 0 and r["errors"] == 0
    assert r["requests"] == 8 * 64
    assert r["mismatched_tiles"] == 0 and r["checked_tiles"] == 128
    assert r["batches"] >= 1
