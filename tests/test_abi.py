"""CPU: the C-ABI library loads and exports every symbol include/cafxg.h
declares; status codes are cafx::errc's values. No device calls."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cafxg.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(cafxg_\w+)\s*\(", text, re.M)))


def test_header_declares_the_binding_list():
    import paper_1505_07368_b200.cafxg as b
    assert declared_functions() == sorted(b.EXPORTS)


def test_library_exports_every_symbol():
    import paper_1505_07368_b200.cafxg as b
    L = b.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", b.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_library_has_sm100a_code():
    import paper_1505_07368_b200.cafxg as b
    out = subprocess.run(["cuobjdump", "--list-elf", b.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_codes_are_errc_values():
    import paper_1505_07368_b200.cafxg as b
    # cafx::errc (error.hpp:11-29): unknown_type=2, out_of_range=4,
    # type_mismatch=5, interface_mismatch=6, config_error=8, spawn_error=9,
    # request_timeout=13, request_down=14
    assert b.lib().cafxg_abi_version() == 3
    for code, name in [(0, "none"), (2, "unknown_type"), (4, "out_of_range"),
                       (5, "type_mismatch"), (6, "interface_mismatch"), (8, "config_error"),
                       (9, "spawn_error"), (13, "request_timeout"), (14, "request_down")]:
        assert b.status_string(code) == name


def test_open_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1505_07368_b200 as pkg
    with pytest.raises(pkg.CafxgError) as e:
        pkg.Context()
    assert e.value.code == 9  # spawn_error: no silent CPU fallback


def test_struct_layouts_match_header():
    import paper_1505_07368_b200.cafxg as b
    assert ctypes.sizeof(b.MandelDesc) == 4 * 8 + 10 * 4 + 8
    assert ctypes.sizeof(b.SgemmDesc) == 32
    assert ctypes.sizeof(b.Stats) == 10 * 8


def test_header_is_plain_c_and_links(tmp_path):
    """include/cafxg.h compiles as C99 and a C program links libcafxg.so."""
    import paper_1505_07368_b200.cafxg as b
    exe = tmp_path / "abi_check"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "c", "abi_check.c"),
                        "-L", os.path.dirname(b.LIB_PATH), "-lcafxg",
                        f"-Wl,-rpath,{os.path.dirname(b.LIB_PATH)}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    import torch
    if not torch.cuda.is_available():
        out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
        assert out.returncode == 0 and "spawn_error" in out.stdout


def test_kernel_signatures():
    """spawn_cl's normalised signatures, no device needed."""
    import paper_1505_07368_b200 as pkg
    assert pkg.kernel_signature("matrix_multiply") == "f32*(f32*,f32*)"
    assert pkg.kernel_signature("mandelbrot") == "u32*(mandel_desc*)"
    with pytest.raises(pkg.CafxgError) as e:
        pkg.kernel_signature("no_such_kernel")
    assert e.value.code == 2
    buf = ctypes.create_string_buffer(4)
    assert pkg.lib().cafxg_kernel_signature(b"mandelbrot", buf, 4) == 4
    assert ctypes.sizeof(pkg.Tuning) == 32
