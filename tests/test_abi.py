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
    """No torch / ATen / c10 type crosses the boundary: the header includes only <stdint.h>
    and every parameter type is a C scalar, a plain pointer or an opaque sf_* handle."""
    txt = open(os.path.join(ROOT, "include", "stepfact.h")).read()
    code = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    assert re.findall(r"#include\s*[<\"]([^>\"]+)", code) == ["stdint.h"]
    for bad in ("torch", "at::", "c10", "Tensor", "std::"):
        assert bad not in code, bad
    allowed = {"int", "int64_t", "uint8_t", "double", "void", "const", "char", "sf_comm_t", "float"}
    for m in re.finditer(r"^\s*(?:const\s+)?\w+\**\s+\**\w+\s*\(([^)]*)\)\s*;", code, flags=re.M | re.S):
        for arg in filter(None, (a.strip() for a in m.group(1).split(","))):
            words = re.findall(r"[A-Za-z_]\w*", arg)
            assert words and set(words[:-1] if len(words) > 1 else words) <= allowed, arg


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


def test_schedule_matches_oracle_and_hand_lists(L):
    """The drivers' schedule (sf_schedule: the Sched the GPU drivers run, row a1) equals the
    flush positions recorded inside the oracle's Algorithms 1-3 and hand-worked lists
    (readings R1, R11)."""
    import numpy as np
    import oracle
    import synth
    assert sf.schedule(37, [9, 3, 1, 12, 5, 7]) == [9, 12, 13, 25, 30]
    assert sf.schedule(37, [2, 3])[:4] == [2, 5, 8, 11]
    assert sf.schedule(4, 1) == [1, 2, 3] and sf.schedule(4, 4) == [] and sf.schedule(1, 1) == []
    assert sf.schedule(16384, 168)[-1] == 97 * 168 and len(sf.schedule(16384, 168)) == 97
    rng = np.random.default_rng(0)
    A = synth.gen_numpy("paper_spd", 61, seed=1)
    for _ in range(40):
        seq = [int(x) for x in rng.integers(1, 20, size=rng.integers(1, 6))]
        s = seq if len(seq) > 1 else seq[0]
        if isinstance(s, int) and s > 61:
            continue
        assert sf.schedule(61, s) == oracle.flush_positions("chol", A, s), seq
    for n in range(1, 40):
        for s in range(1, n + 1):
            assert len(sf.schedule(n, s)) == L.sf_flush_count(n, s)
    bad = (ctypes.c_int64 * 2)(3, 0)
    assert L.sf_schedule(10, 2, bad, None, 0) == -1 and L.sf_schedule(0, 1, bad, None, 0) == -1


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
    assert L.sf_set_strassen(4, 4096) == SF_EINVAL
    assert L.sf_set_strassen(2, 4096) == 0 and L.sf_set_strassen(3, 4096) == 0   # 2-3 levels
    assert L.sf_set_strassen(1, 10) == SF_EINVAL
    assert L.sf_set_strassen(-1, 4096) == SF_EINVAL
    assert L.sf_set_strassen(0, 4096) == 0
