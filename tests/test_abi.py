"""The C-ABI library loads and exports every symbol include/mpr.h declares (no GPU calls).

Also checks the boundary's no-fallback rule: the product package never imports oracle/.
"""
import ast
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpr.h")
PKG = os.path.join(ROOT, "paper_2212_01317_b200")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_]+\s*\**\s*(mpr_[a-z_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2212_01317_b200 import _build
    _build.build()
    return ctypes.CDLL(_build.LIB)


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("mpr_init", "mpr_set_data", "mpr_estimate_local_params", "mpr_simulate", "mpr_predict"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    from paper_2212_01317_b200 import binding
    assert sorted(binding.EXPORTED) == declared_functions()


def test_version_string_without_gpu(lib):
    lib.mpr_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.mpr_version()


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", f
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                assert "mpr_oracle" not in open(os.path.join(dirpath, f)).read(), f


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2212_01317_b200 import LeMpr, MprError
    with pytest.raises(MprError):
        LeMpr()


def _build_c_example(tmp_path):
    import subprocess
    from paper_2212_01317_b200 import _build
    _build.build()
    exe = str(tmp_path / "mpr_fill_c")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "fill.c"), "-L", PKG, "-lmpr",
                           f"-Wl,-rpath,{PKG}", "-lm", "-o", exe])
    return exe


def test_c_example_compiles_and_links_against_the_abi(tmp_path):
    """The boundary is plain C: a C program compiles against include/mpr.h and links libmpr.so."""
    assert os.path.exists(_build_c_example(tmp_path))


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    import subprocess
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build_c_example(tmp_path)
    out = subprocess.run([exe, os.path.join(PKG, "data", "calib_q0.5.txt")], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0, out.stderr
    assert "0 sample mismatches" in out.stdout


def _build_c_slab_example(tmp_path):
    import subprocess
    exe = str(tmp_path / "mpr_fill_slabs")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "fill_slabs.c"), "-L", PKG, "-lmpr", "-lpthread",
                           f"-Wl,-rpath,{PKG}", "-lm", "-o", exe])
    return exe


def test_c_multirank_example_compiles(tmp_path):
    """The multi-rank path is reachable from plain C: row slabs over an in-process group of
    contexts, one host thread per rank (examples/fill_slabs.c)."""
    assert os.path.exists(_build_c_slab_example(tmp_path))


@pytest.mark.gpu
def test_c_multirank_example_runs(tmp_path):
    """4 row-slab ranks driven from C threads return the single context's prediction bit for bit."""
    import subprocess
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = _build_c_slab_example(tmp_path)
    out = subprocess.run([exe, os.path.join(PKG, "data", "calib_q0.5.txt"), "4", str(torch.cuda.device_count())],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert " 0 mismatches" in out.stdout
