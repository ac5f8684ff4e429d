"""CPU checks of the boundary: libtsqr.so builds for sm_100a, loads, and exports every
symbol include/tsqr.h declares; the Python binding names match; argument validation
that needs no GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "tsqr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsqr_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2405_04237_b200 import build
    path = build.build()
    return ctypes.CDLL(path), path


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    for f in ("tsqr_create", "tsqr_factor", "tsqr_destroy", "tsqr_wait", "tsqr_workspace_bytes"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    L, path = lib
    for f in header_functions():
        assert hasattr(L, f), f
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tsqr_\w+)", out))
    assert set(header_functions()) <= exported


def test_binding_names_match_header():
    import paper_2405_04237_b200 as t
    assert sorted(t.EXPORTS) == header_functions()


def test_library_is_sm100a_and_uses_dmma(lib):
    _, path = lib
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", path], capture_output=True,
                                       text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-pipe contractions
    assert "LDGSTS" in sass  # cp.async staging


def test_workspace_and_validation_without_gpu(lib):
    import paper_2405_04237_b200 as t
    L = t.load()
    assert L.tsqr_workspace_bytes(4096, 64, 16, 1, t.MCQR2GS) > 0
    assert L.tsqr_workspace_bytes(4096, 64, 24, 1, t.MCQR2GS) == 0      # b not supported
    assert L.tsqr_workspace_bytes(4096, 60, 16, 1, t.MCQR2GS) == 0      # ragged panels
    assert L.tsqr_workspace_bytes(4096, 64, 16, 1, t.CQR2) == 0         # CQR2 needs b == n
    assert L.tsqr_workspace_bytes(4096, 64, 16, 1, t.SCQR3) == 0        # sCQR3 needs b == n
    assert L.tsqr_workspace_bytes(4096, 64, 64, 1, t.SCQR3) > 0
    assert L.tsqr_workspace_bytes(4096, 64, 64, 1, 8) == 0              # no such algorithm
    h = ctypes.c_void_p()
    rc = L.tsqr_create(ctypes.byref(h), 4096, 64, 16, None, t.MCQR2GS, None, None, 0)
    assert rc == t.TSQR_ERR_WORKSPACE and h.value is None
    rc = L.tsqr_create(ctypes.byref(h), 4096, 64, 24, None, t.MCQR2GS, None, None, 0)
    assert rc == t.TSQR_ERR_UNSUPPORTED
    assert L.tsqr_status_string(5) == b"TSQR_ERR_BREAKDOWN"
    assert L.tsqr_factor(None, None, 1, None, 1) == t.TSQR_ERR_INVALID_ARG
    assert L.tsqr_wait(None, None) == t.TSQR_ERR_INVALID_ARG


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2405_04237_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f
