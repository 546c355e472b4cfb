"""C-ABI checks that need no GPU: the library loads, exports every symbol declared in
include/stepfact.h, rejects bad arguments synchronously (nothing enqueued), and its host
schedule logic matches the paper's flush law."""
import ctypes
import os
import re

import pytest

import paper_1812_02056_b200 as sf
from paper_1812_02056_b200 import build as sfbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    sfbuild.build()
    return sf.lib()


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "stepfact.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(\w+)\s*\(", txt, flags=re.M)))


def test_header_symbols_exported(L):
    syms = declared_symbols()
    assert "chol_factor" in syms and "lu_factor" in syms and "qr_factor" in syms
    for name in syms:
        assert hasattr(L, name), f"{name} declared in stepfact.h but not exported"
    assert set(sf.EXPORTS) <= set(syms)


def test_no_torch_in_abi():
    txt = open(os.path.join(ROOT, "include", "stepfact.h")).read()
    assert "torch" not in txt.lower().replace("pytorch", "") or "at::" not in txt


def test_strerror(L):
    assert L.sf_strerror(0) == b"success"
    assert L.sf_strerror(1) == b"invalid argument"


@pytest.mark.parametrize("n,s", [(0, 1), (-3, 1), (4, 0), (4, 5), (4, -1)])
def test_bad_sizes_rejected(L, n, s):
    buf = (ctypes.c_double * 16)()
    info = ctypes.c_int64(0)
    p = ctypes.addressof(buf)
    assert L.chol_factor(n, s, 0, p, 4, p, 4, ctypes.addressof(info), None) == 1
    assert L.lu_factor(n, s, 0, p, 4, p, 4, ctypes.addressof(info), None) == 1
    assert b"" != L.sf_last_error()


def test_bad_ld_dtype_null(L):
    buf = (ctypes.c_double * 64)()
    p = ctypes.addressof(buf)
    info = ctypes.addressof(ctypes.c_int64(0))
    assert L.chol_factor(4, 2, 0, p, 3, p, 3, info, None) == 1      # lda < n
    assert L.chol_factor(4, 2, 7, p, 4, p, 4, info, None) == 1      # unknown dtype
    assert L.chol_factor(4, 2, 0, None, 4, p, 4, info, None) == 1   # null A
    assert L.chol_factor(4, 2, 0, p, 4, p, 4, None, None) == 1      # null info
    assert L.chol_factor(4, 2, 0, p + 4, 4, p + 4, 4, info, None) == 1  # misaligned
    # partial overlap of input and output extents
    assert L.chol_factor(4, 2, 0, p, 4, p + 8, 4, info, None) == 1
    assert L.chol_factor(4, 2, 0, p, 4, p, 5, info, None) == 1      # in place with lda != ldl
    q = ctypes.addressof((ctypes.c_double * 16)())
    assert L.qr_factor(4, 2, 0, p, 4, p, 4, q, 4, info, None) == 1  # Q aliases A


def test_flush_count_matches_paper_schedule(L):
    import oracle
    for n in range(1, 70):
        for s in range(1, n + 1):
            assert L.sf_flush_count(n, s) == (n - 1) // s == oracle.flush_count(n, s)
    # BASELINE.json configs
    assert L.sf_flush_count(256, 16) == 15 and L.sf_flush_count(4096, 64) == 63
    assert L.sf_flush_count(16384, 168) == 97 and L.sf_flush_count(65536, 512) == 127


def test_sass_is_sm100a_tensor_core():
    """The built library carries sm_100a SASS with DMMA (FP64 tensor core) instructions."""
    import shutil
    import subprocess
    sfbuild.build()
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-sass", sf.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA.8x8x4" in out


def test_new_entry_points_reject_bad_arguments(L):
    """Argument errors of the variable-step, solve and distributed entry points come back
    synchronously as SF_EINVAL with nothing enqueued (no GPU needed)."""
    buf = (ctypes.c_double * 64)()
    p = ctypes.addressof(buf)
    info = ctypes.addressof(ctypes.c_int64(0))
    steps_bad = (ctypes.c_int64 * 2)(2, 0)
    steps_ok = (ctypes.c_int64 * 1)(2)
    assert L.chol_factor_steps(4, 2, steps_bad, 0, p, 4, p, 4, info, None) == 1
    assert L.chol_factor_steps(4, 0, steps_ok, 0, p, 4, p, 4, info, None) == 1
    assert L.lu_factor_steps(4, 1, steps_ok, 0, p, 3, p, 3, info, None) == 1          # lda < n
    assert L.qr_factor_steps(4, 1, steps_ok, 7, p, 4, p, 4, p, 4, info, None) == 1    # dtype
    assert L.chol_solve(0, 1, 0, p, 4, p, 4, None) == 1
    assert L.lu_solve(4, 1, 0, p, 3, p, 4, None) == 1
    assert L.qr_solve(4, 1, 0, None, 4, p, 4, p, 4, None) == 1
    arr = (ctypes.c_void_p * 1)(p)
    iarr = (ctypes.c_void_p * 1)(info)
    assert L.chol_factor_dist(None, 4, 2, 0, arr, arr, 4, iarr, None) == 1             # null comm
    assert L.sf_comm_init_loopback(None, 2) == 1
    assert L.sf_local_cols(10, 3, 2, 5) == 0


def test_set_strassen_arguments(L):
    """sf_set_strassen validates synchronously (no GPU needed) and 0 restores the default."""
    SF_EINVAL = 1
    assert L.sf_set_strassen(2, 4096) == SF_EINVAL
    assert L.sf_set_strassen(1, 10) == SF_EINVAL
    assert L.sf_set_strassen(-1, 4096) == SF_EINVAL
    assert L.sf_set_strassen(0, 4096) == 0
