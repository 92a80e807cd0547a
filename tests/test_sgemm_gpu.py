"""GPU parity for the matrix_multiply kernels: sampled rows against the
fp64-accumulated check, normwise max_j|dC| / max_j|R| <= 1e-5 (BASELINE.json
config 2/5 tolerance)."""
import os

import numpy as np
import pytest

import paper_1505_07368_b200 as pkg
from oracle import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-5


def check(A, B, C, nrows=48, seed=0):
    M, N = C.shape
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([[0, M - 1], rng.integers(0, M, nrows)])).astype(np.uint32)
    R = oracle.sgemm_ref_rows(np.ascontiguousarray(A), np.ascontiguousarray(B), rows, N,
                              A.shape[1])
    return oracle.sgemm_rel_err(np.ascontiguousarray(C), R, rows, N)


@pytest.mark.parametrize("mode", [pkg.SGEMM_FFMA, pkg.SGEMM_AUTO])
@pytest.mark.parametrize("M,N,K", [(1024, 1024, 1024), (256, 256, 256), (100, 77, 33),
                                   (1, 1, 1), (129, 257, 65), (512, 128, 2048)])
def test_sgemm_shapes(ctx, mode, M, N, K):
    A = oracle.fill_uniform(M * K, 1).reshape(M, K)
    B = oracle.fill_uniform(K * N, 2).reshape(K, N)
    C = ctx.sgemm(A, B, mode=mode)
    assert check(A, B, C) <= TOL


def test_sgemm_leading_dims(ctx):
    M, N, K = 200, 150, 96
    Abig = oracle.fill_uniform(M * (K + 7), 3).reshape(M, K + 7)
    Bbig = oracle.fill_uniform(K * (N + 5), 4).reshape(K, N + 5)
    A, B = Abig[:, :K], Bbig[:, :N]
    C = np.zeros((M, N + 3), dtype=np.float32)[:, :N]
    ctx.sgemm(A, B, C, mode=pkg.SGEMM_FFMA)
    assert check(A, B, C) <= TOL


def test_sgemm_k_zero(ctx):
    A = np.zeros((8, 0), dtype=np.float32)
    B = np.zeros((0, 9), dtype=np.float32)
    C = np.full((8, 9), 3.0, dtype=np.float32)
    ctx.sgemm(A, B, C)
    assert np.all(C == 0)


def test_sgemm_device_api(ctx):
    import torch
    M = N = K = 512
    A = torch.from_numpy(oracle.fill_uniform(M * K, 5).reshape(M, K)).cuda()
    B = torch.from_numpy(oracle.fill_uniform(K * N, 6).reshape(K, N)).cuda()
    C = torch.empty(M, N, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    ctx.sgemm_device(M, N, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    assert check(A.cpu().numpy(), B.cpu().numpy(), C.cpu().numpy()) <= TOL


@pytest.mark.parametrize("M,N,K", [(256, 256, 256), (1024, 1024, 1024), (384, 512, 2048),
                                   (2048, 768, 4096)])
def test_sgemm_3xtf32(ctx, M, N, K):
    """tcgen05 kind::tf32 hi/lo split: within the fp32 tolerance."""
    A = oracle.fill_uniform(M * K, 11).reshape(M, K)
    B = oracle.fill_uniform(K * N, 12).reshape(K, N)
    C = ctx.sgemm(A, B, mode=pkg.SGEMM_3XTF32)
    assert check(A, B, C) <= TOL


@pytest.mark.parametrize("M,N,K,splits", [(128, 256, 1024, 8), (256, 512, 512, 4),
                                          (512, 1024, 256, 2), (1024, 1024, 1024, 4),
                                          (2048, 2048, 512, 1)])
def test_sgemm_cluster_split_k(ctx, M, N, K, splits):
    """Small C grids split K across a thread-block cluster of 2/4/8 CTAs that
    reduce their partial tiles through distributed shared memory: within the
    tolerance, and bit-identical from run to run (fixed summation order).
    `splits` is the factor sgemm_tc_splits picks for the shape on 148 SMs."""
    import torch
    A = torch.from_numpy(oracle.fill_uniform(M * K, 31).reshape(M, K)).cuda()
    B = torch.from_numpy(oracle.fill_uniform(K * N, 32).reshape(K, N)).cuda()
    outs = []
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    for _ in range(2):
        C = torch.full((M, N), float("nan"), device="cuda")
        ctx.sgemm_device(M, N, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                         mode=pkg.SGEMM_3XTF32)
        torch.cuda.synchronize()
        outs.append(C.cpu().numpy())
    assert not np.isnan(outs[0]).any()
    assert np.array_equal(outs[0], outs[1])
    assert check(A.cpu().numpy(), B.cpu().numpy(), outs[0]) <= TOL


@pytest.mark.parametrize("M,N,K,pad", [(3072, 512, 256, 0), (1280, 256, 512, 8)])
def test_sgemm_pipelined_host_request(ctx, M, N, K, pad):
    """Host request >= 1024 rows: row-block pipeline (upload / 3xTF32 / download
    overlapped), including a padded leading dimension of A and C."""
    Abig = oracle.fill_uniform(M * (K + pad), 21).reshape(M, K + pad)
    A = Abig[:, :K]
    B = oracle.fill_uniform(K * N, 22).reshape(K, N)
    Cbig = np.full((M, N + pad), np.nan, dtype=np.float32)
    C = Cbig[:, :N]
    ctx.sgemm(A, B, C)
    assert not np.isnan(C).any()
    assert check(np.ascontiguousarray(A), B, C) <= TOL
    if pad:
        assert np.isnan(Cbig[:, N:]).all()   # the padding is never written


@pytest.mark.parametrize("M,N,K,pad", [(8192, 8192, 256, 0), (8320, 8448, 128, 8)])
def test_sgemm_2d_wavefront_host_request(ctx, M, N, K, pad):
    """Large host request: A row blocks and B column blocks uploaded
    interleaved, every C block multiplied once both operands are resident
    and downloaded by itself; padded leading dimensions of A, B and C."""
    Abig = oracle.fill_uniform(M * (K + pad), 41).reshape(M, K + pad)
    Bbig = oracle.fill_uniform(K * (N + pad), 42).reshape(K, N + pad)
    A, B = Abig[:, :K], Bbig[:, :N]
    Cbig = np.full((M, N + pad), np.nan, dtype=np.float32)
    C = Cbig[:, :N]
    ctx.sgemm(A, B, C)
    assert not np.isnan(C).any()
    assert check(np.ascontiguousarray(A), np.ascontiguousarray(B), C) <= TOL
    if pad:
        assert np.isnan(Cbig[:, N:]).all()


@pytest.mark.parametrize("M,N,K,pad", [(256, 512, 512, 4), (384, 256, 288, 8)])
def test_sgemm_3xtf32_leading_dims(ctx, M, N, K, pad):
    """The tensor-core path with the caller's row pitches: padded lda / ldb /
    ldc (16-byte multiples); the padding of C is never written."""
    Abig = oracle.fill_uniform(M * (K + pad), 13).reshape(M, K + pad)
    Bbig = oracle.fill_uniform(K * (N + pad), 14).reshape(K, N + pad)
    A, B = Abig[:, :K], Bbig[:, :N]
    Cbig = np.full((M, N + pad), np.nan, dtype=np.float32)
    C = Cbig[:, :N]
    ctx.sgemm(A, B, C, mode=pkg.SGEMM_3XTF32)
    assert not np.isnan(C).any()
    assert check(np.ascontiguousarray(A), np.ascontiguousarray(B), C) <= TOL
    assert np.isnan(Cbig[:, N:]).all()


def test_sgemm_3xtf32_k16384(ctx):
    """cfg5's depth: K = 16384 (the deepest accumulation; the tensor core's
    truncating accumulation is bounded by 128-K chunk sums), a 1024 x 256 C
    block, 64 sampled rows against the fp64-accumulated check."""
    import torch
    M, N, K = 1024, 256, 16384
    A_h = oracle.fill_uniform(M * K, 71).reshape(M, K)
    B_h = oracle.fill_uniform(K * N, 72).reshape(K, N)
    A, B = torch.from_numpy(A_h).cuda(), torch.from_numpy(B_h).cuda()
    C = torch.empty(M, N, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    ctx.sgemm_device(M, N, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                     mode=pkg.SGEMM_3XTF32)
    torch.cuda.synchronize()
    err = check(A_h, B_h, C.cpu().numpy(), nrows=64, seed=3)
    assert err <= TOL, err


@pytest.mark.parametrize("bn", ["128", "256"])
def test_sgemm_3xtf32_both_tile_widths(bn):
    """Both tile widths within the tolerance, split-K clusters included: 256
    columns by default, 128 for N % 256 != 0 shapes or when CAFXG_SGEMM_BN=128
    forces it."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1505_07368_b200 as pkg
from oracle import oracle
for M, N, K in [(1024, 1024, 1024), (2048, 2048, 512), (512, 256, 4096), (256, 384, 640)]:
    if N %% 256 and %r == "256":
        continue
    A = oracle.fill_uniform(M * K, 81).reshape(M, K)
    B = oracle.fill_uniform(K * N, 82).reshape(K, N)
    with pkg.Context(1) as c:
        C = c.sgemm(A, B, mode=pkg.SGEMM_3XTF32)
    rows = np.arange(0, M, 37, dtype=np.uint32)
    R = oracle.sgemm_ref_rows(A, B, rows, N, K)
    err = oracle.sgemm_rel_err(C, R, rows, N)
    assert err <= 1e-5, (M, N, K, err)
print("ok")
""" % (root, bn)
    env = dict(os.environ, CAFXG_SGEMM_BN=bn)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]


@pytest.mark.parametrize("pair", ["0", "1"])
@pytest.mark.parametrize("raw", ["0", "1"])
@pytest.mark.parametrize("ws", ["0", "1"])
def test_sgemm_3xtf32_operand_forms(pair, raw, ws):
    """Both operand forms (split + transposed B, or raw A / B read as their own
    hi halves with only lo materialised, B MN-major), both split-K reductions
    (L2 workspace, distributed shared memory) and both kernels (1-SM tiles, or
    CTA pairs with tcgen05 .cta_group::2, which always reduce through the
    workspace), forced through CAFXG_SGEMM_RAW / _WS / _PAIR, on device-API
    GEMMs: split-K clusters of 2 / 4 / 8, both tile widths, padded row pitches,
    K = 8192; every result within the tolerance, and the two reductions
    bit-identical."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1505_07368_b200 as pkg
from oracle import oracle
out = []
with pkg.Context(1) as c:
    for M, N, K, pad, splits in [(1024, 1024, 1024, 0, 0), (256, 256, 2048, 0, 8),
                                 (512, 768, 512, 4, 2), (128, 128, 8192, 0, 0),
                                 (2048, 512, 256, 8, 4)]:
        A_h = oracle.fill_uniform(M * (K + pad), 91).reshape(M, K + pad)
        B_h = oracle.fill_uniform(K * (N + pad), 92).reshape(K, N + pad)
        A, B = torch.from_numpy(A_h).cuda(), torch.from_numpy(B_h).cuda()
        C = torch.full((M, N + pad), float("nan"), device="cuda")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        c.sgemm_device(M, N, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                       mode=pkg.SGEMM_3XTF32, lda=K + pad, ldb=N + pad, ldc=N + pad,
                       splits=splits)
        torch.cuda.synchronize()
        Ch = C.cpu().numpy()
        assert not np.isnan(Ch[:, :N]).any(), (M, N, K)
        if pad:
            assert np.isnan(Ch[:, N:]).all(), (M, N, K)
        rows = np.unique(np.linspace(0, M - 1, 40).astype(np.uint32))
        R = oracle.sgemm_ref_rows(np.ascontiguousarray(A_h[:, :K]),
                                  np.ascontiguousarray(B_h[:, :N]), rows, N, K)
        err = oracle.sgemm_rel_err(np.ascontiguousarray(Ch[:, :N]), R, rows, N)
        assert err <= 1e-5, (M, N, K, err)
        out.append(Ch[:, :N].copy())
np.save(sys.argv[1], np.concatenate([o.ravel() for o in out]))
print("ok")
""" % root
    env = dict(os.environ, CAFXG_SGEMM_RAW=raw, CAFXG_SGEMM_WS=ws, CAFXG_SGEMM_PAIR=pair)
    path = f"/tmp/cafxg_forms_{pair}_{raw}_{ws}.npy"
    r = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
    if ws == "1":
        other = f"/tmp/cafxg_forms_{pair}_{raw}_0.npy"
        if os.path.exists(other):
            assert np.array_equal(np.load(path), np.load(other))


def test_sgemm_device_misaligned_pointers(ctx):
    """Device-API operands at a 4-byte (not 16-byte) offset: AUTO falls back
    to the FFMA kernel and stays within the tolerance, 3XTF32 refuses with
    E_CONFIG -- neither may fault the device (the tensor-core path reads A
    and writes C in 16-byte vectors)."""
    import torch
    M = N = K = 256
    A_h = oracle.fill_uniform(M * K, 31).reshape(M, K)
    B_h = oracle.fill_uniform(K * N, 32).reshape(K, N)
    Abuf = torch.zeros(M * K + 4, device="cuda")
    Cbuf = torch.zeros(M * N + 4, device="cuda")
    Abuf[1:1 + M * K] = torch.from_numpy(A_h.ravel()).cuda()
    B = torch.from_numpy(B_h).cuda()
    a_ptr, c_ptr = Abuf.data_ptr() + 4, Cbuf.data_ptr() + 4
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with pytest.raises(pkg.CafxgError) as e:
        ctx.sgemm_device(M, N, K, a_ptr, B.data_ptr(), c_ptr, s.cuda_stream,
                         mode=pkg.SGEMM_3XTF32)
    assert e.value.code == 8
    ctx.sgemm_device(M, N, K, a_ptr, B.data_ptr(), c_ptr, s.cuda_stream, mode=pkg.SGEMM_AUTO)
    torch.cuda.synchronize()
    C = Cbuf[1:1 + M * N].cpu().numpy().reshape(M, N)
    assert check(A_h, B_h, C) <= TOL
    assert ctx.status() == 0


@pytest.mark.parametrize("env", [{}, {"CAFXG_SGEMM_PAIR": "1"}, {"CAFXG_SGEMM_RAW": "0"},
                                 {"CAFXG_SGEMM_RAW": "1", "CAFXG_SGEMM_WS": "0"}])
def test_sgemm_device_randomised_kernel_paths(env):
    """Seeded random tensor-core shapes through the device API under each
    kernel / operand / reduction choice (forced by environment, one process
    each): M, N multiples of 128, K a multiple of 32, padded row pitches,
    random split-K requests; every result within the tolerance and padding
    never written."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1505_07368_b200 as pkg
from oracle import oracle
rng = np.random.default_rng(2024)
with pkg.Context(1) as c:
    for case in range(24):
        M = int(rng.integers(1, 9)) * 128
        N = int(rng.integers(1, 9)) * 128
        K = int(rng.integers(1, 33)) * 32
        pa, pb, pc = (int(rng.integers(0, 3)) * 4 for _ in range(3))
        splits = int(rng.choice([0, 0, 1, 2, 4, 8]))
        if splits and (K %% (16 * splits) or K // splits < 16):
            splits = 0
        A_h = oracle.fill_uniform(M * (K + pa), 300 + case).reshape(M, K + pa)
        B_h = oracle.fill_uniform(K * (N + pb), 400 + case).reshape(K, N + pb)
        A, B = torch.from_numpy(A_h).cuda(), torch.from_numpy(B_h).cuda()
        C = torch.full((M, N + pc), float("nan"), device="cuda")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        c.sgemm_device(M, N, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                       mode=pkg.SGEMM_3XTF32, lda=K + pa, ldb=N + pb, ldc=N + pc,
                       splits=splits)
        torch.cuda.synchronize()
        Ch = C.cpu().numpy()
        assert not np.isnan(Ch[:, :N]).any(), (case, M, N, K, splits)
        if pc:
            assert np.isnan(Ch[:, N:]).all(), (case, M, N, K)
        rows = np.unique(np.linspace(0, M - 1, 12).astype(np.uint32))
        R = oracle.sgemm_ref_rows(np.ascontiguousarray(A_h[:, :K]),
                                  np.ascontiguousarray(B_h[:, :N]), rows, N, K)
        err = oracle.sgemm_rel_err(np.ascontiguousarray(Ch[:, :N]), R, rows, N)
        assert err <= 1e-5, (case, M, N, K, splits, err)
    assert c.status() == 0
print("ok")
""" % root
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]


def test_cfg5_full_size_row_sum_property(ctx):
    """cfg5 at full size (16384^3): 32 sampled rows (first, last and 30 random)
    against the fp64-accumulated oracle, normwise <= 1e-5 as BASELINE states;
    then the size-independent property C.1 = A.(B.1) for every row. B.1 and
    A.(B.1) are computed in fp64 on the host; each row sum of the GPU's C must
    match within the fp32-GEMM tolerance scaled to the row's magnitude
    (sum_j |C_ij| bound)."""
    import torch
    n = 16384
    A_h = oracle.fill_uniform(n * n, 1).reshape(n, n)
    B_h = oracle.fill_uniform(n * n, 2).reshape(n, n)
    A, B = torch.from_numpy(A_h).cuda(), torch.from_numpy(B_h).cuda()
    C = torch.empty(n, n, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    ctx.sgemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    err_rows = check(A_h, B_h, C.cpu().numpy(), nrows=30, seed=5)
    assert err_rows <= TOL, err_rows
    got = C.to(torch.float64).sum(dim=1).cpu().numpy()
    absrow = C.abs().to(torch.float64).sum(dim=1).cpu().numpy()
    del A, B, C
    b1 = B_h.astype(np.float64).sum(axis=1)
    want = A_h.astype(np.float64) @ b1
    err = np.abs(got - want) / absrow
    assert float(err.max()) <= 1e-5, float(err.max())


def test_sgemm_3xtf32_rejects_unsupported_shape(ctx):
    A = np.zeros((100, 64), np.float32)
    B = np.zeros((64, 256), np.float32)
    with pytest.raises(pkg.CafxgError) as e:
        ctx.sgemm(A, B, mode=pkg.SGEMM_3XTF32)
    assert e.value.code == 8


def test_sgemm_randomised_shapes(ctx):
    """Seeded random shapes, modes and leading dimensions: tcgen05-eligible
    shapes (multiples of 128 / 256 / 32) and odd ones (FFMA), host arrays
    with padded rows; every result within the fp32 tolerance."""
    rng = np.random.default_rng(int(os.environ.get("CAFXG_FUZZ_SEED", "11")))
    cases = int(os.environ.get("CAFXG_FUZZ_CASES", "40"))
    tc_shapes = 0
    for case in range(cases):
        if rng.integers(0, 2):
            M, N, K = (int(rng.integers(1, 9)) * 128, int(rng.integers(1, 5)) * 256,
                       int(rng.integers(1, 33)) * 32)
        else:
            M, N, K = (int(rng.integers(1, 700)), int(rng.integers(1, 700)),
                       int(rng.integers(1, 700)))
        mode = int(rng.choice([pkg.SGEMM_AUTO, pkg.SGEMM_FFMA]))
        pa, pb, pc = (int(rng.integers(0, 9)) for _ in range(3))
        A = oracle.fill_uniform(M * (K + pa), 100 + case).reshape(M, K + pa)[:, :K]
        B = oracle.fill_uniform(K * (N + pb), 200 + case).reshape(K, N + pb)[:, :N]
        Cbig = np.full((M, N + pc), np.nan, dtype=np.float32)
        C = Cbig[:, :N]
        ctx.sgemm(A, B, C, mode=mode)
        assert not np.isnan(C).any(), (case, M, N, K, mode)
        assert check(np.ascontiguousarray(A), np.ascontiguousarray(B), C) <= TOL, \
            (case, M, N, K, mode)
        if pc:
            assert np.isnan(Cbig[:, N:]).all()
        tc_shapes += M % 128 == 0 and N % 256 == 0 and K % 32 == 0
    print(f"sgemm fuzz: {cases} requests ({tc_shapes} tcgen05-eligible shapes) within {TOL}")


def test_cfg2_every_row(ctx):
    """BASELINE config 2 (C = A.B, 1024^3, A and B uniform[-1,1) from a seeded
    generator) through the host request, EVERY row of C against the
    fp64-accumulated oracle, normwise <= 1e-5."""
    n = 1024
    A = oracle.fill_uniform(n * n, 1).reshape(n, n)
    B = oracle.fill_uniform(n * n, 2).reshape(n, n)
    C = ctx.sgemm(A, B)
    rows = np.arange(n, dtype=np.uint32)
    R = oracle.sgemm_ref_rows(A, B, rows, n, n)
    err = oracle.sgemm_rel_err(C, R, rows, n)
    assert err <= TOL, err
