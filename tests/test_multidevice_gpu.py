"""GPU: the multi-device paths of one context on a one-GPU box.

CAFXG_VIRTUAL_DEVICES=V opens V context devices on the same physical GPU,
each with its own streams, scheduler ring and completion thread, so the
request splitting and joining that a G-GPU context does runs for real:
cyclic row bands for Mandelbrot, per-device row blocks of A plus the
replicated B for sgemm (peer copies stand in for the NCCL all-gather, which
rejects duplicate GPUs), the in-order FNV chain of run_mandelbrot and the
dispatcher's device choice for actor batches."""
import os

import numpy as np
import pytest

import paper_1505_07368_b200 as pkg
from oracle import oracle

pytestmark = pytest.mark.gpu
V = 3


@pytest.fixture(scope="module")
def vctx():
    os.environ["CAFXG_VIRTUAL_DEVICES"] = str(V)
    try:
        c = pkg.Context(device_mask=1)
    finally:
        del os.environ["CAFXG_VIRTUAL_DEVICES"]
    yield c
    c.close()


def test_device_count(vctx):
    assert vctx.device_count == V


def test_mandelbrot_bands_over_devices(vctx):
    # cfg1 geometry: every row band dealt cyclically over the 3 devices
    d = pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100)
    out = vctx.mandelbrot(d).reshape(1080, 1920)
    ref = oracle.tile(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100, fp64=False, centre=True)
    assert np.array_equal(out, ref), int((out != ref).sum())


def test_multi_tile_request_over_devices(vctx):
    rng = np.random.default_rng(21)
    tiles, refs, off = [], [], 0
    for _ in range(7):
        w, h = int(rng.integers(1, 400)), int(rng.integers(1, 300))
        x0, y0 = float(rng.uniform(-2.0, 0.3)), float(rng.uniform(-1.1, 0.9))
        span = float(10 ** rng.uniform(-3, 0.3))
        fp64 = bool(rng.integers(0, 2))
        t = pkg.mandel_desc(x0, x0 + span, y0, y0 + span * h / w, w, h, 200, fp64=fp64)
        t.out_offset = off
        off += w * h
        tiles.append(t)
        refs.append(oracle.tile(t.x0, t.x1, t.y0, t.y1, w, h, 200, fp64=fp64, centre=True))
    out = vctx.mandelbrot(tiles, np.zeros(off, np.uint32))
    for t, r in zip(tiles, refs):
        got = out[t.out_offset:t.out_offset + t.width * t.height].reshape(t.height, t.width)
        assert np.array_equal(got, r)


@pytest.mark.parametrize("size,it", [(256, 100), (1024, 500), (16000, 500)])
def test_run_mandelbrot_chain(vctx, golden, size, it):
    """Blocks on different devices, FNV chained block to block in row order."""
    want = int([g for g in golden["run_mandelbrot"]
                if g["size"] == size and g["max_iter"] == it][0]["checksum"])
    h, _ = vctx.run_mandelbrot(size, it)
    assert h == want


@pytest.mark.parametrize("M,N,K,peer", [(768, 512, 384, True),    # B slices read in place
                                        (3072, 1024, 768, True),
                                        # ragged shares (512 / 512 / 384 rows) and
                                        # row blocks (4 / 4 / 3 of 128 per device)
                                        (1408, 512, 384, True),
                                        (1280, 768, 96, True),
                                        (3 * 128, 256, 3, False),  # K / V < 16: replicated B
                                        (384, 384, 768, False)])   # N % 256: replicated B
def test_sgemm_row_blocks(vctx, M, N, K, peer):
    """Row blocks of A per device. Where the shapes allow, the fused path:
    each device uploads 1/V of B's rows and every device's GEMM reads the K
    slices where they lie (peer_gemms); else B is replicated by peer copies
    (the NCCL all-gather on real GPUs)."""
    A = oracle.fill_uniform(M * K, 31).reshape(M, K)
    B = oracle.fill_uniform(K * N, 32).reshape(K, N)
    before = vctx.stats()
    C = vctx.sgemm(A, B)
    after = vctx.stats()
    assert after.peer_gemms - before.peer_gemms == (1 if peer else 0)
    # B crossed PCIe once in total (1/V per device), A once
    assert after.h2d_bytes - before.h2d_bytes == (M * K + K * N) * 4
    rows = np.unique(np.concatenate([np.arange(0, M, 61), [M // V - 1, M // V, M - 1],
                                     np.arange(127, M, 128), np.arange(128, M, 128)]))
    R = oracle.sgemm_ref_rows(A, B, rows.astype(np.uint32), N, K)
    assert oracle.sgemm_rel_err(C, R, rows.astype(np.uint32), N) <= 1e-5


def test_sgemm_unsplit_shapes(vctx):
    # K not divisible by the device count: one device does the whole product
    M, N, K = 512, 128, 100
    A = oracle.fill_uniform(M * K, 33).reshape(M, K)
    B = oracle.fill_uniform(K * N, 34).reshape(K, N)
    C = vctx.sgemm(A, B)
    rows = np.arange(0, M, 17, dtype=np.uint32)
    R = oracle.sgemm_ref_rows(A, B, rows, N, K)
    assert oracle.sgemm_rel_err(C, R, rows, N) <= 1e-5


def test_actor_batches_over_devices(vctx):
    a = vctx.spawn("mandelbrot")
    rng = np.random.default_rng(8)
    descs, outs, futs = [], [], []
    for _ in range(60):
        kx, ky = int(rng.integers(0, 1472)), int(rng.integers(0, 960))
        x0, y0 = -2.0 + kx / 512, -1.0 + ky / 512
        d = pkg.mandel_desc(x0, x0 + 0.125, y0, y0 + 0.125, 64, 64, 150, fp64=True)
        o = np.zeros(4096, np.uint32)
        futs.append(a.request([(pkg.MandelDesc * 1)(d)], o))
        descs.append(d)
        outs.append(o)
    for f in futs:
        f.result(timeout=120)
    for d, o in zip(descs, outs):
        ref = oracle.tile(d.x0, d.x1, d.y0, d.y1, 64, 64, 150, fp64=True, centre=True)
        assert np.array_equal(o.reshape(64, 64), ref)
    a.release()


def test_matrix_multiply_actor_over_devices(vctx):
    size = 3 * 256
    a = vctx.spawn("matrix_multiply", (size, size))
    A = oracle.fill_uniform(size * size, 41)
    B = oracle.fill_uniform(size * size, 42)
    C = np.zeros(size * size, dtype=np.float32)
    a.request([A, B], C).result(timeout=60)
    rows = np.arange(0, size, 13, dtype=np.uint32)
    R = oracle.sgemm_ref_rows(A.reshape(size, size), B.reshape(size, size), rows, size, size)
    assert oracle.sgemm_rel_err(C.reshape(size, size), R, rows, size) <= 1e-5
    a.release()


@pytest.mark.parametrize("pinned", [False, True])
def test_large_actor_request_split_over_devices(vctx, pinned):
    """One compute-actor request of >= 1M pixels leaves the batching path and
    is served by every device of the context: cyclic row bands, overlapped
    waves, the reply assembled in the actor's reply buffer; bit-exact, and
    every device ran a kernel (actor requests used one device)."""
    os.environ["CAFXG_VIRTUAL_DEVICES"] = str(V)
    try:
        c = pkg.Context(device_mask=1)   # fresh: devices_used starts at 0
    finally:
        del os.environ["CAFXG_VIRTUAL_DEVICES"]
    with c:
        a = c.spawn("mandelbrot")
        d = pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 1536, 1024, 600)
        out = c.pinned_empty(1536 * 1024, np.uint32) if pinned else \
            np.zeros(1536 * 1024, np.uint32)
        out[:] = 0xdeadbeef
        a.request([(pkg.MandelDesc * 1)(d)], out).result(timeout=120)
        st = c.stats()
        ref = oracle.tile(d.x0, d.x1, d.y0, d.y1, 1536, 1024, 600, fp64=False, centre=True)
        assert np.array_equal(out.reshape(1024, 1536), ref)
        assert st.devices_used == (1 << V) - 1
        assert st.batches == 0  # not a dispatcher batch
        assert st.requests == 1
        if pinned:
            c.pinned_free(out)
        a.release()


def test_sgemm_nccl_branch_one_rank():
    """CAFXG_NCCL_SELFTEST=1: a one-device context sends B through the NCCL
    calls of the multi-device path (libnccl dlopen, ncclCommInitAll, grouped
    in-place all-gather with one rank), so the branch runs on a one-GPU box;
    the product stays within 1e-5 and one collective was issued."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1505_07368_b200 as pkg
from oracle import oracle
M = N = K = 2048
A = oracle.fill_uniform(M * K, 51).reshape(M, K)
B = oracle.fill_uniform(K * N, 52).reshape(K, N)
with pkg.Context(1) as c:
    C = c.sgemm(A, B)
    st = c.stats()
rows = np.arange(0, M, 97, dtype=np.uint32)
R = oracle.sgemm_ref_rows(A, B, rows, N, K)
err = oracle.sgemm_rel_err(C, R, rows, N)
assert st.nccl_collectives >= 1, st.nccl_collectives
assert err <= 1e-5, err
print("ok", st.nccl_collectives, err)
""" % root
    env = dict(os.environ, CAFXG_NCCL_SELFTEST="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs (the NCCL all-gather over NVLink)")
def test_two_gpu_context_nccl_and_bands():
    """A context over the first two real GPUs: sgemm row blocks with B
    replicated by the NCCL all-gather over NVLink, and cfg3-style cyclic
    bands of one Mandelbrot request on both devices; both against the
    oracle."""
    with pkg.Context(device_mask=0b11) as c:
        assert c.device_count == 2
        M = N = K = 4096
        A = oracle.fill_uniform(M * K, 61).reshape(M, K)
        B = oracle.fill_uniform(K * N, 62).reshape(K, N)
        before = c.stats()
        C = c.sgemm(A, B)
        after = c.stats()
        # with peer access between the GPUs, each GEMM reads B's other slice
        # over NVLink in place; without it, the NCCL all-gather replicates B
        assert (after.peer_gemms - before.peer_gemms == 1 or
                after.nccl_collectives - before.nccl_collectives == 2)
        rows = np.arange(0, M, 127, dtype=np.uint32)
        R = oracle.sgemm_ref_rows(A, B, rows, N, K)
        assert oracle.sgemm_rel_err(C, R, rows, N) <= 1e-5
        # the same product through the NCCL all-gather path
        code = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1505_07368_b200 as pkg
from oracle import oracle
M = N = K = 4096
A = oracle.fill_uniform(M * K, 61).reshape(M, K)
B = oracle.fill_uniform(K * N, 62).reshape(K, N)
with pkg.Context(device_mask=0b11) as c:
    C = c.sgemm(A, B)
    assert c.stats().peer_gemms == 0
rows = np.arange(0, M, 127, dtype=np.uint32)
assert oracle.sgemm_rel_err(C, oracle.sgemm_ref_rows(A, B, rows, N, K), rows, N) <= 1e-5
print("ok")
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        import subprocess
        import sys
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           timeout=600, env=dict(os.environ, CAFXG_SGEMM_P2P="0"))
        assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
        d = pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 2048, 2048, 1000)
        out = c.mandelbrot(d).reshape(2048, 2048)
        ref = oracle.tile(-0.75, -0.73, 0.10, 0.12, 2048, 2048, 1000, fp64=False, centre=True)
        assert np.array_equal(out, ref)
        assert c.stats().devices_used == 0b11


def test_sgemm_peer_path_several_row_blocks():
    """The fused peer path's per-device pipeline with several A row blocks per
    device (CAFXG_P2P_RMIN=128 lowers the 1024-row minimum block for these
    small shapes), ragged shares included; every 128-row block boundary
    checked against the fp64-accumulated oracle."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1505_07368_b200 as pkg
from oracle import oracle
with pkg.Context(device_mask=1) as c:
    for M, N, K in [(1408, 512, 384), (1280, 768, 96), (3072, 1024, 768)]:
        A = oracle.fill_uniform(M * K, 41).reshape(M, K)
        B = oracle.fill_uniform(K * N, 42).reshape(K, N)
        s0 = c.stats(); C = c.sgemm(A, B); s1 = c.stats()
        assert s1.peer_gemms - s0.peer_gemms == 1, (M, N, K)
        rows = np.unique(np.concatenate([np.arange(127, M, 128), np.arange(128, M, 128),
                                         [0, M - 1]])).astype(np.uint32)
        err = oracle.sgemm_rel_err(C, oracle.sgemm_ref_rows(A, B, rows, N, K), rows, N)
        assert err <= 1e-5, (M, N, K, err)
print("ok")
""" % root
    env = dict(os.environ, CAFXG_VIRTUAL_DEVICES="3", CAFXG_P2P_RMIN="128")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
