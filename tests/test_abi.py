"""CPU checks of the C-ABI library: it builds for sm_100a, loads, exports every function
include/qap_rlt2.h declares, and rejects bad arguments before touching the GPU."""
import ctypes as ct
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pkg():
    from paper_1510_02065_b200 import build
    build.build()
    import paper_1510_02065_b200 as p
    p.load_library()
    return p


def declared_functions():
    src = open(os.path.join(ROOT, "include", "qap_rlt2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qap_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("qap_rlt2_create", "qap_rlt2_fix", "qap_rlt2_bound", "qap_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(pkg):
    L = pkg.load_library()
    names = declared_functions()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert sorted(pkg.EXPORTS) == names


def test_sm100a_code_in_library(pkg):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pkg.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_tma_bulk_copy_in_sass(pkg):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", pkg.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "UBLKCP" in sass          # cp.async.bulk (TMA 1-D) stages the LAP cost blocks
    assert "REDUX" in sass           # redux.sync argmin


def test_create_rejects_bad_arguments(pkg):
    L = pkg.load_library()
    out = ct.c_void_p()
    F = np.zeros((4, 4), np.int64)
    assert L.qap_rlt2_create(2, F.ctypes.data, F.ctypes.data, None, ct.byref(out)) == pkg.QAP_E_ARG
    assert L.qap_rlt2_create(65, F.ctypes.data, F.ctypes.data, None, ct.byref(out)) == pkg.QAP_E_ARG
    G = F.copy()
    G[1, 2] = -1
    assert L.qap_rlt2_create(4, G.ctypes.data, F.ctypes.data, None, ct.byref(out)) == pkg.QAP_E_ARG
    big = np.full((4, 4), 2 ** 26, np.int64)
    assert L.qap_rlt2_create(4, big.ctypes.data, big.ctypes.data, None, ct.byref(out)) == pkg.QAP_E_ARG
    assert b"2^53" in L.qap_last_error(None)
    assert L.qap_rlt2_create(4, None, F.ctypes.data, None, ct.byref(out)) == pkg.QAP_E_ARG
    assert out.value is None


def test_lap_batch_rejects_bad_arguments(pkg):
    L = pkg.load_library()
    z = ct.c_void_p(0x1000)
    assert L.qap_lap_batch(0, 1, 2, z, None, None, None, None, None, None, None, None) == pkg.QAP_E_ARG
    assert L.qap_lap_batch(65, 1, 65 * 65 + 1, z, None, None, None, None, None, None, None, None) == pkg.QAP_E_ARG
    assert L.qap_lap_batch(3, 1, 9, z, None, None, None, None, None, None, None, None) == pkg.QAP_E_ARG  # odd ld
    assert L.qap_lap_batch(2, 1, 4, ct.c_void_p(0x1008), None, None, None, None, None, None, None, None) == pkg.QAP_E_ARG


def test_destroy_null_safe(pkg):
    pkg.load_library().qap_destroy(None)


def test_product_does_not_reference_oracle():
    """The product package never imports / links the oracle."""
    for dp, _, files in os.walk(os.path.join(ROOT, "paper_1510_02065_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "rlt2_oracle" not in txt, f


def test_flag_constants_match_header(pkg):
    src = open(os.path.join(ROOT, "include", "qap_rlt2.h")).read()
    flags = dict(re.findall(r"#define\s+(QAP_FLAG_[A-Z_]+)\s+(\d+)", src))
    assert flags, "no QAP_FLAG_* in the header"
    for name, val in flags.items():
        assert getattr(pkg, name) == int(val), name


def test_tensor_tma_in_sass(pkg):
    """The transfer loads its boxes with tensor-map TMA (4-D maps); the LAP kernel moves
    whole cost blocks with 1-D bulk copies both ways and takes its argmins with redux.sync
    (sm_100a)."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", pkg.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "UTMALDG.4D" in sass
    assert "UBLKCP.S.G" in sass and "UBLKCP.G.S" in sass
    assert "REDUX.MIN.S32" in sass and "MATCH.ANY" in sass
