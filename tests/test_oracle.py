"""CPU: pins the oracle restatement (oracle/cafx_oracle.c) against the
reference's own golden values (tests/golden/reference_mandelbrot.json, made
by running the unmodified reference) and the reference's test pins."""
import os

import numpy as np
import pytest

from oracle import oracle


def test_reference_test_pins():
    # test_bench.cpp:76-82 and acceptance.cpp:635-638
    assert oracle.cell_f64(0.0, 0.0, 50) == 50
    assert oracle.cell_f64(0.0, 0.0, 500) == 500
    assert oracle.cell_f64(2.0, 0.0, 50) == 2
    assert oracle.cell_f64(0.0, 0.0, 100) == 100
    assert oracle.cell_f64(2.0, 0.0, 100) == 2


def test_cells_match_reference(golden):
    for c in golden["cells"]:
        assert oracle.cell_f64(c["re"], c["im"], c["max_iter"]) == c["count"], c


@pytest.mark.parametrize("size,it", [(64, 50), (96, 60), (256, 100), (1024, 500)])
def test_run_mandelbrot_checksums(golden, size, it):
    want = int([g for g in golden["run_mandelbrot"]
                if g["size"] == size and g["max_iter"] == it][0]["checksum"])
    assert oracle.run_mandelbrot(size, it) == want


def test_rows_match_reference(golden):
    for r in golden["rows"]:
        row = oracle.mandelbrot_row(r["y"], r["size"], r["max_iter"])
        assert int(row.sum()) == r["sum"]
        assert oracle.fnv1a_u32(row) == int(r["fnv"])
        if r["counts"] is not None:
            assert row.tolist() == r["counts"]


@pytest.mark.parametrize("size,it", [(64, 50), (100, 80), (333, 40)])
def test_generalised_mapping_reduces_to_reference(size, it):
    # x0=-1.5, x1=0.5, y0=-1, y1=1, corner, fp64 == mandelbrot_row bit for bit
    t = oracle.tile(-1.5, 0.5, -1.0, 1.0, size, size, it, fp64=True, centre=False)
    for y in range(size):
        assert np.array_equal(t[y], oracle.mandelbrot_row(y, size, it)), y


def test_coordinate_contract():
    # c = lo + ((i + s) * (hi - lo)) / n ; reference: 2.0*x/size - 1.5
    for size in (7, 64, 1000, 16000):
        for x in (0, 1, size // 3, size - 1):
            assert oracle.lib().oracle_coord(-1.5, 0.5, x, size, 0) == 2.0 * x / size - 1.5


def test_fp32_cells():
    assert oracle.cell_f32(0.0, 0.0, 77) == 77
    assert oracle.cell_f32(2.0, 0.0, 50) == 2
    assert oracle.cell_f32(-2.0, 0.0, 50) == 50   # |z|^2 == 4 forever, strict >
    assert oracle.cell_f32(-2.0000005, 0.0, 50) == 1
    assert oracle.cell_f64(-2.0, 0.0, 5000) == 5000


def test_edge_max_iter():
    assert oracle.cell_f64(0.0, 0.0, 0) == 0
    assert oracle.cell_f64(3.0, 0.0, 0) == 0
    assert oracle.cell_f64(3.0, 0.0, 1) == 1
    # escape exactly at max_iter returns max_iter
    assert oracle.cell_f64(2.0, 0.0, 2) == 2


def test_tile_sampling_and_offsets():
    full = oracle.tile(-2.0, 1.0, -1.0, 1.0, 48, 32, 60, fp64=False, centre=True)
    sub = oracle.tile(-2.0, 1.0, -1.0, 1.0, 48, 32, 60, fp64=False, centre=True,
                      row0=5, nrows=7, col0=11, ncols=13)
    assert np.array_equal(full[5:12, 11:24], sub)
    sampled = oracle.tile(-2.0, 1.0, -1.0, 1.0, 48, 32, 60, fp64=False, centre=True,
                          sample_stride=4)
    assert np.array_equal(sampled[::4], full[::4])


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built (no /root/reference)")
def test_oracle_against_live_reference():
    R = oracle.ref()
    rng = np.random.default_rng(7)
    for re, im in rng.uniform(-2.2, 1.2, size=(400, 2)):
        it = int(rng.integers(1, 3000))
        assert oracle.cell_f64(re, im, it) == R.ref_mandelbrot_cell(re, im, it)
    for size, it in [(64, 50), (120, 77)]:
        for y in (0, size // 2, size - 1):
            row = np.empty(size, dtype=np.uint32)
            R.ref_mandelbrot_row(y, size, it, row.ctypes.data)
            assert np.array_equal(row, oracle.mandelbrot_row(y, size, it))


def test_uniform_generator():
    a = oracle.fill_uniform(10000, 5)
    b = oracle.fill_uniform(10000, 5)
    assert np.array_equal(a, b)
    assert a.min() >= -1.0 and a.max() < 1.0
    assert abs(float(a.mean())) < 0.05
    assert oracle.uniform_at(5, 1234) == a[1234]
    c = oracle.fill_uniform(100, 5, offset=9000)
    assert np.array_equal(c, a[9000:9100])


def test_sgemm_reference_rows():
    A = oracle.fill_uniform(48 * 40, 1).reshape(48, 40)
    B = oracle.fill_uniform(40 * 56, 2).reshape(40, 56)
    rows = np.array([0, 5, 47], dtype=np.uint32)
    R = oracle.sgemm_ref_rows(A, B, rows, 56, 40)
    want = A.astype(np.float64)[rows] @ B.astype(np.float64)
    assert np.allclose(R, want, rtol=0, atol=1e-12)
    C = np.zeros((48, 56), dtype=np.float32)
    oracle.sgemm_f32(A, B, C, 56, 40, 0, 48, block=8, threads=3)
    assert oracle.sgemm_rel_err(C, R, rows, 56) < 1e-6


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built (no /root/reference)")
def test_reference_region_driver_matches_oracle():
    """bench.py's CPU baseline drives the reference's own mandelbrot_cell over
    a region at pixel centres (ref_region_iters_mt, oracle/ref_shim.cpp): its
    iteration sum equals the fp64 oracle's on the same sampled rows."""
    import ctypes as C
    R = oracle.ref()
    for (x0, x1, y0, y1, w, h, it, stride) in [(-0.75, -0.73, 0.10, 0.12, 97, 64, 300, 5),
                                               (-2.0, 1.0, -1.0, 1.0, 120, 90, 100, 1)]:
        sec = C.c_double()
        got = R.ref_region_iters_mt(x0, x1, y0, y1, w, h, it, stride, 3, C.byref(sec))
        ref = oracle.tile(x0, x1, y0, y1, w, h, it, fp64=True, centre=True)
        assert got == int(ref[::stride].sum(dtype=np.uint64))
