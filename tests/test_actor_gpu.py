"""GPU: the spawn_cl facade (cafxg_spawn / cafxg_actor_enqueue): replies,
batching of request bursts, error replies, termination."""
import threading

import numpy as np
import pytest

import paper_1505_07368_b200 as pkg
from oracle import oracle

pytestmark = pytest.mark.gpu


def storm_tile(rng, it=256):
    # 64x64 fp64 tile at a seeded offset on the 1/512 grid inside [-2,1]x[-1,1]
    kx = int(rng.integers(0, 3 * 512 - 64 + 1))
    ky = int(rng.integers(0, 2 * 512 - 64 + 1))
    x0, y0 = -2.0 + kx / 512, -1.0 + ky / 512
    return pkg.mandel_desc(x0, x0 + 0.125, y0, y0 + 0.125, 64, 64, it, fp64=True, centre=True)


def test_mandelbrot_actor_request(ctx):
    a = ctx.spawn("mandelbrot")
    d = pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 320, 200, 120)
    desc = (pkg.MandelDesc * 1)(d)
    assert a.reply_bytes([desc]) == 320 * 200 * 4
    out = np.zeros(320 * 200, dtype=np.uint32)
    a.request([desc], out).result(timeout=60)
    ref = oracle.tile(-2.0, 1.0, -1.0, 1.0, 320, 200, 120, fp64=False, centre=True)
    assert np.array_equal(out.reshape(200, 320), ref)
    a.release()


@pytest.mark.parametrize("pinned", [False, True])
def test_large_reply(ctx, pinned):
    """cfg1-sized reply (8.3 MB): pageable replies are copied out of staging in
    pieces on the callback threads, pinned ones written by the device."""
    a = ctx.spawn("mandelbrot")
    d = pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100)
    desc = (pkg.MandelDesc * 1)(d)
    ref = oracle.tile(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100, fp64=False, centre=True)
    for _ in range(3):
        out = ctx.pinned_empty(1920 * 1080, np.uint32) if pinned else \
            np.full(1920 * 1080, 7, dtype=np.uint32)
        a.request([desc], out).result(timeout=60)
        assert np.array_equal(out.reshape(1080, 1920), ref)
        if pinned:
            ctx.pinned_free(out)
    a.release()


@pytest.mark.parametrize("pinned", [False, True])
def test_request_burst_from_many_clients(ctx, pinned):
    """16 client threads x 40 storm tiles; every reply checked per tile."""
    a = ctx.spawn("mandelbrot")
    clients, per = 16, 40
    rng = np.random.default_rng(99)
    descs = [[storm_tile(rng) for _ in range(per)] for _ in range(clients)]
    outs = [[(ctx.pinned_empty(4096, np.uint32) if pinned else np.zeros(4096, np.uint32))
             for _ in range(per)] for _ in range(clients)]
    before = ctx.stats()
    errors = []

    def client(c):
        try:
            futs = [a.request([(pkg.MandelDesc * 1)(descs[c][i])], outs[c][i])
                    for i in range(per)]
            for f in futs:
                f.result(timeout=120)
        except Exception as e:  # pragma: no cover
            errors.append(e)
    th = [threading.Thread(target=client, args=(c,)) for c in range(clients)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors
    after = ctx.stats()
    n = clients * per
    assert after.requests - before.requests == n
    # bursts are batched: far fewer launches than requests
    assert after.batches - before.batches < n
    for c in range(clients):
        for i in range(per):
            d = descs[c][i]
            ref = oracle.tile(d.x0, d.x1, d.y0, d.y1, 64, 64, 256, fp64=True, centre=True)
            assert np.array_equal(outs[c][i].reshape(64, 64), ref)
    if pinned:
        for row in outs:
            for o in row:
                ctx.pinned_free(o)
    a.release()


def test_staging_ring_reuse_and_oversized_request(ctx):
    """The dispatcher's per-device staging ring: a burst of more batches than
    ring slots (slot reuse ordered by the copy-out events), one request above
    the 16M-pixel batch cap (its slot grows), then small requests again."""
    a = ctx.spawn("mandelbrot")
    W, H = 4096, 4200  # 17.2M px > kMaxBatchPx
    big = pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, W, H, 24)
    mids = [pkg.mandel_desc(-2.0 + 0.01 * k, 1.0, -1.0, 1.0, 2048, 2048, 24)
            for k in range(20)]  # 4M px each: several per batch, > 8 batches
    out_big = ctx.pinned_empty(W * H, np.uint32)
    out_mid = [ctx.pinned_empty(2048 * 2048, np.uint32) for _ in mids]
    rng = np.random.default_rng(17)
    smalls = [storm_tile(rng) for _ in range(32)]
    out_small = [np.zeros(4096, np.uint32) for _ in smalls]
    futs = [a.request([(pkg.MandelDesc * 1)(d)], o) for d, o in zip(mids[:10], out_mid[:10])]
    futs.append(a.request([(pkg.MandelDesc * 1)(big)], out_big))
    futs += [a.request([(pkg.MandelDesc * 1)(d)], o) for d, o in zip(mids[10:], out_mid[10:])]
    futs += [a.request([(pkg.MandelDesc * 1)(d)], o) for d, o in zip(smalls, out_small)]
    for f in futs:
        f.result(timeout=120)
    for r0 in (0, 2099, H - 1):
        ref = oracle.tile(-2.0, 1.0, -1.0, 1.0, W, H, 24, fp64=False, centre=True,
                          row0=r0, nrows=1)
        assert np.array_equal(out_big.reshape(H, W)[r0], ref[0])
    for d, o in zip(mids, out_mid):
        for r0 in (0, 1023, 2047):
            ref = oracle.tile(d.x0, d.x1, d.y0, d.y1, 2048, 2048, 24, fp64=False, centre=True,
                              row0=r0, nrows=1)
            assert np.array_equal(o.reshape(2048, 2048)[r0], ref[0])
    for d, o in zip(smalls, out_small):
        ref = oracle.tile(d.x0, d.x1, d.y0, d.y1, 64, 64, 256, fp64=True, centre=True)
        assert np.array_equal(o.reshape(64, 64), ref)
    ctx.pinned_free(out_big)
    for o in out_mid:
        ctx.pinned_free(o)
    a.release()


def _tile_ref(d):
    return oracle.tile(d.x0, d.x1, d.y0, d.y1, d.ncols, d.nrows, d.max_iter,
                       fp64=bool(d.precision), centre=bool(d.sampling))


def test_direct_reply_small_batches(ctx):
    """Small batches into pinned replies skip the reply-scatter launch: the
    escape kernel counts finished pixels per tile and the warp completing a
    tile copies it to the reply (checked kernel, deferred kernel and its
    replays; fp32 and fp64; multi-tile requests). Tiles whose pixel count is
    not a multiple of 4 keep the scatter launch. Every reply exact."""
    a = ctx.spawn("mandelbrot")
    rng = np.random.default_rng(5)
    cases = [
        [storm_tile(rng)],                                                  # fp64, checked
        [pkg.mandel_desc(-0.30, -0.20, 0.60, 0.70, 64, 48, 300, fp64=True)],  # fp64 deferred
        [pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 96, 80, 1000)],          # fp32 deferred
        [pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 128, 64, 100)],              # fp32 checked
        [storm_tile(rng), storm_tile(rng), storm_tile(rng)],                # multi-tile
        [pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 33, 7, 200)],                # 231 px: scatter
    ]
    before = ctx.stats()
    reply_bytes = 0
    for rep in range(3):
        for tiles in cases:
            descs = (pkg.MandelDesc * len(tiles))(*tiles)
            npx = sum(t.nrows * t.ncols for t in tiles)
            reply_bytes += npx * 4
            out = ctx.pinned_empty(npx, np.uint32)
            out[:] = 0xdeadbeef
            a.request([descs], out).result(timeout=60)
            off = 0
            for t in tiles:
                n = t.nrows * t.ncols
                assert np.array_equal(out[off:off + n].reshape(t.nrows, t.ncols), _tile_ref(t))
                off += n
            ctx.pinned_free(out)
    after = ctx.stats()
    assert after.direct_batches - before.direct_batches >= 3 * 5
    assert after.d2h_bytes - before.d2h_bytes == reply_bytes  # direct replies counted too
    a.release()


def test_direct_reply_concurrent_clients(ctx):
    """Closed-loop clients (one outstanding request each): batches of several
    requests replied by the kernel, staging slots and their tile counters
    reused across both compute streams; every reply exact."""
    a = ctx.spawn("mandelbrot")
    clients, per = 12, 25
    rng = np.random.default_rng(17)
    descs = [[storm_tile(rng) for _ in range(per)] for _ in range(clients)]
    refs = [[_tile_ref(d) for d in row] for row in descs]
    errors = []
    before = ctx.stats()

    def client(c):
        try:
            out = ctx.pinned_empty(4096, np.uint32)
            for i in range(per):
                out[:] = 0
                a.request([(pkg.MandelDesc * 1)(descs[c][i])], out).result(timeout=60)
                if not np.array_equal(out.reshape(64, 64), refs[c][i]):
                    errors.append((c, i))
            ctx.pinned_free(out)
        except Exception as e:  # pragma: no cover
            errors.append(e)
    th = [threading.Thread(target=client, args=(c,)) for c in range(clients)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors
    assert ctx.stats().direct_batches > before.direct_batches
    a.release()


def test_direct_reply_mixed_max_iter_request(ctx):
    """A small pinned request whose tiles differ in max_iter, batched together
    with storm tiles from other clients: it must take the scatter path (one
    launch per max_iter group) and neither it nor its batch mates may fail
    (it used to pass the direct-reply check and fail the batch)."""
    a = ctx.spawn("mandelbrot")
    rng = np.random.default_rng(23)
    mixed = [storm_tile(rng, it=256), storm_tile(rng, it=100)]
    storms = [[storm_tile(rng)] for _ in range(24)]
    for rep in range(4):
        futs, outs = [], []
        for tiles in storms[:12] + [mixed] + storms[12:]:
            out = ctx.pinned_empty(4096 * len(tiles), np.uint32)
            out[:] = 0xdeadbeef
            futs.append(a.request([(pkg.MandelDesc * len(tiles))(*tiles)], out))
            outs.append((tiles, out))
        for f in futs:
            f.result(timeout=60)
        for tiles, out in outs:
            for k, t in enumerate(tiles):
                assert np.array_equal(out[k * 4096:(k + 1) * 4096].reshape(64, 64),
                                      _tile_ref(t))
            ctx.pinned_free(out)
    a.release()


def test_multi_tile_request(ctx):
    a = ctx.spawn("mandelbrot")
    rng = np.random.default_rng(5)
    ds = [storm_tile(rng, it=100) for _ in range(3)]
    arr = (pkg.MandelDesc * 3)(*ds)
    out = np.zeros(3 * 4096, dtype=np.uint32)
    a.request([arr], out).result(timeout=60)
    for k, d in enumerate(ds):
        ref = oracle.tile(d.x0, d.x1, d.y0, d.y1, 64, 64, 100, fp64=True, centre=True)
        assert np.array_equal(out[k * 4096:(k + 1) * 4096].reshape(64, 64), ref)
    a.release()


def test_matrix_multiply_actor(ctx):
    size = 256
    a = ctx.spawn("matrix_multiply", (size, size))
    A = oracle.fill_uniform(size * size, 7)
    B = oracle.fill_uniform(size * size, 8)
    C = np.zeros(size * size, dtype=np.float32)
    a.request([A, B], C).result(timeout=60)
    rows = np.arange(0, size, 9, dtype=np.uint32)
    R = oracle.sgemm_ref_rows(A.reshape(size, size), B.reshape(size, size), rows, size, size)
    assert oracle.sgemm_rel_err(C.reshape(size, size), R, rows, size) <= 1e-5
    a.release()


def test_mixed_clients_two_actors(ctx):
    """8 client threads send an interleaved random mix to a Mandelbrot actor
    (fp32 / fp64, storm tiles and multi-tile images, pinned and pageable
    replies) and two matrix_multiply actors (256 and 1024) at once; every
    reply is checked. Exercises the dispatcher's batching across kinds and
    precisions, the staging ring and the sgemm host paths concurrently."""
    mb = ctx.spawn("mandelbrot")
    mm = {256: ctx.spawn("matrix_multiply", (256, 256)),
          1024: ctx.spawn("matrix_multiply", (1024, 1024))}
    mats = {n: (oracle.fill_uniform(n * n, 50 + n), oracle.fill_uniform(n * n, 60 + n))
            for n in mm}
    errors, checks = [], []
    lock = threading.Lock()

    def client(c):
        rng = np.random.default_rng(300 + c)
        try:
            pend = []
            for i in range(24):
                kind = int(rng.integers(0, 6))
                if kind <= 2:    # one storm tile
                    d = storm_tile(rng, it=int(rng.choice([100, 256, 700])))
                    d.precision = pkg.FP64 if kind == 0 else pkg.FP32
                    out = ctx.pinned_empty(4096, np.uint32) if i & 1 else np.zeros(4096, np.uint32)
                    pend.append(("tile", d, out, mb.request([(pkg.MandelDesc * 1)(d)], out)))
                elif kind <= 4:  # a small image in two tiles
                    w, h = int(rng.integers(40, 200)), int(rng.integers(2, 60))
                    it = int(rng.choice([50, 300]))
                    t0 = pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, w, h, it, row0=0, nrows=h // 2)
                    t1 = pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, w, h, it, row0=h // 2,
                                         nrows=h - h // 2)
                    out = np.zeros(w * h, np.uint32)
                    pend.append(("image", (w, h, it), out,
                                 mb.request([(pkg.MandelDesc * 2)(t0, t1)], out)))
                else:            # matrix_multiply
                    n = 256 if rng.integers(0, 2) else 1024
                    A, B = mats[n]
                    out = np.zeros(n * n, np.float32)
                    pend.append(("mm", n, out, mm[n].request([A, B], out)))
            for kind, arg, out, fut in pend:
                fut.result(timeout=120)
                with lock:
                    checks.append((kind, arg, out))
        except Exception as e:  # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=client, args=(c,)) for c in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors
    assert len(checks) == 8 * 24
    for kind, arg, out in checks:
        if kind == "tile":
            d = arg
            ref = oracle.tile(d.x0, d.x1, d.y0, d.y1, 64, 64, d.max_iter,
                              fp64=d.precision == pkg.FP64, centre=True)
            assert np.array_equal(out.reshape(64, 64), ref)
        elif kind == "image":
            w, h, it = arg
            ref = oracle.tile(-2.0, 1.0, -1.0, 1.0, w, h, it, fp64=False, centre=True)
            assert np.array_equal(out.reshape(h, w), ref)
        else:
            n = arg
            A, B = mats[n]
            rows = np.arange(0, n, n // 8, dtype=np.uint32)
            R = oracle.sgemm_ref_rows(A.reshape(n, n), B.reshape(n, n), rows, n, n)
            assert oracle.sgemm_rel_err(out.reshape(n, n), R, rows, n) <= 1e-5
    for kind, _, o in checks:
        if kind == "tile":
            ctx.pinned_free(o)   # no-op for the pageable ones
    mb.release()
    for a in mm.values():
        a.release()


def test_interface_errors(ctx):
    with pytest.raises(pkg.CafxgError) as e:
        ctx.spawn("no_such_kernel")
    assert e.value.code == 2          # unknown_type
    with pytest.raises(pkg.CafxgError) as e:
        ctx.spawn("matrix_multiply", (4, 5))
    assert e.value.code == 6          # interface_mismatch
    mm = ctx.spawn("matrix_multiply", (8, 8))
    A = np.zeros(64, np.float32)
    with pytest.raises(pkg.CafxgError) as e:
        mm.request([A], np.zeros(64, np.float32))
    assert e.value.code == 6
    with pytest.raises(pkg.CafxgError) as e:
        mm.request([A, np.zeros(63, np.float32)], np.zeros(64, np.float32))
    assert e.value.code == 5          # type_mismatch
    mm.release()
    m = ctx.spawn("mandelbrot")
    with pytest.raises(pkg.CafxgError) as e:
        m.request([np.zeros(7, np.uint8)], np.zeros(1, np.uint32))
    assert e.value.code == 5
    m.release()


def test_quit_fails_later_requests(ctx):
    a = ctx.spawn("mandelbrot")
    d = (pkg.MandelDesc * 1)(pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 16, 16, 10))
    out = np.zeros(256, np.uint32)
    a.request([d], out).result(timeout=60)
    a.quit()
    with pytest.raises(pkg.CafxgError) as e:
        a.request([d], out)
    assert e.value.code == 14         # request_down
    a.release()


def test_sync_waits_for_actor_requests(ctx):
    a = ctx.spawn("mandelbrot")
    rng = np.random.default_rng(1)
    outs = [np.zeros(4096, np.uint32) for _ in range(50)]
    futs = [a.request([(pkg.MandelDesc * 1)(storm_tile(rng))], o) for o in outs]
    ctx.sync()
    assert all(f.done() for f in futs)
    a.release()


def test_c_program_through_the_abi(tmp_path):
    """tests/c/abi_check.c: run_mandelbrot golden + one actor request, from C."""
    import os
    import subprocess
    import paper_1505_07368_b200.cafxg as b
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "abi_check"
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(root, "include"),
                           os.path.join(root, "tests", "c", "abi_check.c"),
                           "-L", os.path.dirname(b.LIB_PATH), "-lcafxg",
                           f"-Wl,-rpath,{os.path.dirname(b.LIB_PATH)}", "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "C ABI OK" in r.stdout, r.stdout + r.stderr


def test_spawn_cl_signature_and_tuning(ctx):
    """cafxg_spawn_ex: the spawn_cl signature is checked against the kernel's
    (interface_mismatch before any actor exists); tuning hints apply to every
    request and out-of-range hints fail the spawn (config_error)."""
    with pytest.raises(pkg.CafxgError) as e:
        ctx.spawn("matrix_multiply", (64, 64), signature="f32*(f32*)")
    assert e.value.code == 6
    mm = ctx.spawn("matrix_multiply", (256, 256), signature="f32*(f32*,f32*)",
                   tuning=pkg.Tuning(sgemm_mode=pkg.SGEMM_3XTF32, sgemm_splits=2))
    A = oracle.fill_uniform(256 * 256, 91)
    B = oracle.fill_uniform(256 * 256, 92)
    C = np.zeros(256 * 256, dtype=np.float32)
    mm.request([A, B], C).result(timeout=60)
    rows = np.arange(0, 256, 11, dtype=np.uint32)
    R = oracle.sgemm_ref_rows(A.reshape(256, 256), B.reshape(256, 256), rows, 256, 256)
    assert oracle.sgemm_rel_err(C.reshape(256, 256), R, rows, 256) <= 1e-5
    mm.release()
    for bad in (pkg.Tuning(block_steps=20), pkg.Tuning(block_steps=72),
                pkg.Tuning(sgemm_splits=3)):
        with pytest.raises(pkg.CafxgError) as e:
            ctx.spawn("mandelbrot", tuning=bad)
        assert e.value.code == 8
    # every block length and a CTA cap, exact against the oracle; batches of
    # differently tuned actors never share a launch
    d = pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 160, 96, 1000)
    ref = _tile_ref(d)
    actors = [ctx.spawn("mandelbrot", signature="u32*(mandel_desc*)",
                        tuning=pkg.Tuning(block_steps=b, max_ctas=m))
              for b, m in [(16, 0), (24, 8), (40, 1), (64, 0), (0, 3)]]
    futs, outs = [], []
    for a in actors:
        for _ in range(3):
            o = np.zeros(160 * 96, np.uint32)
            futs.append(a.request([(pkg.MandelDesc * 1)(d)], o))
            outs.append(o)
    for f in futs:
        f.result(timeout=60)
    for o in outs:
        assert np.array_equal(o.reshape(96, 160), ref)
    for a in actors:
        a.release()
