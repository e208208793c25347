"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/mach_b200.h declares; host-side argument checks
fail the reference's way before any device work."""
import ctypes
import os
import subprocess

import pytest

import paper_0909_4969_b200 as mb
from paper_0909_4969_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    L = mb.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(L, s)]
    assert missing == []
    assert L.mach_version().startswith(b"mach-b200")


def test_binding_table_covers_header():
    assert set(_lib.header_symbols()) == set(_lib._SIGS)


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_ctx_create_without_gpu_reports_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    rc = mb.lib().mach_ctx_create(0, ctypes.byref(h))
    assert rc == _lib.MACH_ERR_CUDA
    assert b"cuda" in mb.lib().mach_last_error().lower()


def test_null_arguments_are_argument_errors():
    L = mb.lib()
    assert L.mach_sparse_nnz(None, None) == _lib.MACH_ERR_ARGUMENT
    assert L.mach_hooi_sparse(None, None, None, 1, 0.0, None) == _lib.MACH_ERR_ARGUMENT


def test_cxx_headers_compile_against_the_library():
    """The C++ mirror (include/mach/*.hpp) compiles and links like the
    reference's headers would for an existing caller."""
    src = os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp")
    out = os.path.join(ROOT, "tests", "cpp", "api_smoke")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", out,
                    _lib.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}"], check=True)
    assert os.path.exists(out)


def test_next_row_mirrors_compile_and_host_only_calls_work(tmp_path):
    """bounds.hpp / ingest.hpp / tensor_io.hpp / cli.hpp callers link; the
    closed-form bound entry points and the CLI's usage errors need no GPU."""
    src = os.path.join(ROOT, "tests", "cpp", "ext_smoke.cpp")
    out = os.path.join(ROOT, "tests", "cpp", "ext_smoke")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", out,
                    _lib.LIB_PATH, f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}"], check=True)
    assert mb.min_sampling_probability((100, 100, 100)) > 1.0
    c = mb.theorem1_conditions((200, 200, 200), 0.5)
    assert c["dims_large_enough"] and c["dims_balanced"] and not c["p_above_min"] and c["per_mode"] == []
    two, fro = mb.achlioptas_bounds(1.0, 1000, 4, 1.0)
    assert abs(two - 4.0 * 1000 ** 0.5) < 1e-9 and abs(fro - 4.0 * 4000 ** 0.5) < 1e-9
    with pytest.raises(mb.ArgumentError):
        mb.theorem1_conditions((5, 5), 1.5)
    cli = os.path.join(ROOT, "paper_0909_4969_b200", "mach_b200")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_0909_4969_b200"), "cli"], check=True)
    assert subprocess.run([cli], capture_output=True).returncode == 2
    assert subprocess.run([cli, "frobnicate"], capture_output=True).returncode == 2
    assert subprocess.run([cli, "hooi", "--input", "x", "--bogus", "1"], capture_output=True).returncode == 2
    assert subprocess.run([cli, "hooi", "--input", str(tmp_path / "none"), "--ranks", "2,2", "--output", "o"],
                          capture_output=True).returncode == 3
    with pytest.raises(mb.IoError):
        mb.tensor_file_info(str(tmp_path / "none.machb"))
    (tmp_path / "junk.machb").write_bytes(b"x" * 100)
    with pytest.raises(mb.ParseError):
        mb.tensor_file_info(str(tmp_path / "junk.machb"))
