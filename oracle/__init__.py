"""CPU oracle for arXiv 1812.02056 Algorithms 1-3 — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  It shares no code with the CUDA product
path in ``paper_1812_02056_b200/`` and never imports it.

The arithmetic lives in ``stepfact_oracle.c`` (plain C, fp64, ``-ffp-contract=off``); this
module only compiles it, loads it with ctypes and marshals numpy arrays.  Matrices are
numpy arrays indexed ``A[i, j]`` as in the paper; they are handed to C in column-major
(Fortran) order.

Pins (tests/test_oracle.py): s=1 and s=n degeneracy bitwise against
independent textbook routines, hand-worked examples (tests/golden/), planted integer
factors (exact), LAPACK cross-checks, invariants, restricted-column bitwise equality.
"""
import ctypes
import os
import subprocess

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "stepfact_oracle.c")
_LIB = os.path.join(_DIR, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force=False):
    """Compile liboracle.so in-tree (gcc).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, dbl, p = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        lib.orc_chol.restype = i64
        lib.orc_chol.argtypes = [i64, i64, i64, p, i64, p, i64]
        lib.orc_lu.restype = i64
        lib.orc_lu.argtypes = [i64, i64, i64, p, i64, p, i64, p, i64, dbl]
        lib.orc_qr.restype = i64
        lib.orc_qr.argtypes = [i64, i64, i64, p, i64, p, i64, p, i64, dbl, ctypes.POINTER(dbl)]
        pi = ctypes.POINTER(ctypes.c_int64)
        lib.orc_chol_steps.restype = i64
        lib.orc_chol_steps.argtypes = [i64, i64, pi, i64, p, i64, p, i64]
        lib.orc_lu_steps.restype = i64
        lib.orc_lu_steps.argtypes = [i64, i64, pi, i64, p, i64, p, i64, p, i64, dbl]
        lib.orc_qr_steps.restype = i64
        lib.orc_qr_steps.argtypes = [i64, i64, pi, i64, p, i64, p, i64, p, i64, dbl, ctypes.POINTER(dbl)]
        lib.orc_solve.restype = None
        lib.orc_solve.argtypes = [i64, i64, i64, p, i64, p, i64, p, i64]
        lib.orc_flush_count.restype = i64
        lib.orc_flush_count.argtypes = [i64, i64]
        lib.orc_frobenius.restype = dbl
        lib.orc_frobenius.argtypes = [i64, p, i64]
        lib.orc_trace_flushes.restype = None
        lib.orc_trace_flushes.argtypes = [p, i64]
        lib.orc_trace_count.restype = i64
        lib.orc_set_threads.argtypes = [ctypes.c_int]
        lib.orc_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _colmajor(A):
    A = np.asarray(A, dtype=np.float64)
    assert A.ndim == 2 and A.shape[0] == A.shape[1], "square matrix expected"
    return np.asfortranarray(A)


def _check_s(n, s):
    if isinstance(s, (list, tuple, np.ndarray)):
        if len(s) == 0 or min(int(x) for x in s) < 1:
            raise ValueError("step sequence must be non-empty with steps >= 1")
        return
    if not (1 <= s <= n):
        raise ValueError(f"step s={s} outside [1, n={n}]")


def _steps(s):
    """A step sequence (reading R11) as a ctypes int64 array, or None."""
    if not isinstance(s, (list, tuple, np.ndarray)):
        return None
    arr = (ctypes.c_int64 * len(s))(*[int(x) for x in s])
    return arr


def set_threads(n):
    _load().orc_set_threads(int(n))


def max_threads():
    return int(_load().orc_max_threads())


def flush_count(n, s):
    """Flushes performed by the c = z+s schedule."""
    return int(_load().orc_flush_count(n, s))


def chol(A, s, kcols=None):
    """Algorithm 1. Returns (L, info); info 0 or 1-based failing column.

    s: the step (int), or a sequence of steps s_0, s_1, ... (reading R11).

    With kcols=K < n, A may be the n x K block of its first K columns; L is then n x K."""
    A = np.asfortranarray(np.asarray(A, dtype=np.float64)); n = A.shape[0]; _check_s(n, s)
    K = n if kcols is None else min(int(kcols), n)
    assert A.shape[1] >= K and (kcols is not None or A.shape[1] == n), "square matrix expected"
    L = np.zeros((n, K), order="F")
    st = _steps(s)
    if st is None:
        info = _load().orc_chol(n, s, K, A.ctypes.data, n, L.ctypes.data, n)
    else:
        info = _load().orc_chol_steps(n, len(st), st, K, A.ctypes.data, n, L.ctypes.data, n)
    if K < n and A.shape[1] == n:
        L = np.concatenate([L, np.zeros((n, n - K))], axis=1)
    return L, int(info)


def lu(A, s, kcols=None, tol=0.0):
    """Algorithm 2, Crout form (U unit upper). Returns (L, U, info)."""
    A = _colmajor(A); n = A.shape[0]; _check_s(n, s)
    L = np.zeros((n, n), order="F"); U = np.zeros((n, n), order="F")
    st = _steps(s)
    K = n if kcols is None else kcols
    if st is None:
        info = _load().orc_lu(n, s, K, A.ctypes.data, n, L.ctypes.data, n, U.ctypes.data, n, float(tol))
    else:
        info = _load().orc_lu_steps(n, len(st), st, K, A.ctypes.data, n, L.ctypes.data, n, U.ctypes.data, n,
                                    float(tol))
    return L, U, int(info)


def qr(A, s, kcols=None, tol=0.0):
    """Algorithm 3. Returns (Q, R, info, lower_mass)."""
    A = _colmajor(A); n = A.shape[0]; _check_s(n, s)
    Q = np.zeros((n, n), order="F"); R = np.zeros((n, n), order="F")
    mass = ctypes.c_double(0.0)
    st = _steps(s)
    K = n if kcols is None else kcols
    if st is None:
        info = _load().orc_qr(n, s, K, A.ctypes.data, n, Q.ctypes.data, n, R.ctypes.data, n, float(tol),
                              ctypes.byref(mass))
    else:
        info = _load().orc_qr_steps(n, len(st), st, K, A.ctypes.data, n, Q.ctypes.data, n, R.ctypes.data, n,
                                    float(tol), ctypes.byref(mass))
    return Q, R, int(info), float(mass.value)


def flush_positions(kind, A, s, kcols=None):
    """Run Algorithm 1/2/3 (kind 'chol' / 'lu' / 'qr') on A with step s (or a step sequence)
    and return the 0-based columns c at which its flushes fired —
    recorded inside the algorithm by the oracle's flush trace hook."""
    lib = _load()
    buf = np.zeros(4096, dtype=np.int64)
    lib.orc_trace_flushes(buf.ctypes.data, len(buf))
    try:
        {"chol": chol, "lu": lu, "qr": qr}[kind](A, s, kcols=kcols)
        cnt = int(lib.orc_trace_count())
    finally:
        lib.orc_trace_flushes(None, 0)
    assert cnt <= len(buf), "trace buffer too small"
    return [int(x) for x in buf[:cnt]]


def frobenius(A):
    A = _colmajor(A)
    return float(_load().orc_frobenius(A.shape[0], A.ctypes.data, A.shape[0]))


def solve(kind, F1, B, F2=None):
    """Plain forward/back substitution with the factors (oracle/stepfact_oracle.c orc_solve):
    kind 'chol' (F1 = L), 'lu' (F1 = L with U packed above), 'qr' (F1 = Q, F2 = R).
    Returns X for A X = B."""
    k = {"chol": 0, "lu": 1, "qr": 2}[kind]
    F1 = _colmajor(F1); n = F1.shape[0]
    F2c = _colmajor(F2) if F2 is not None else F1
    X = np.asfortranarray(np.array(B, dtype=np.float64).reshape(n, -1))
    _load().orc_solve(k, n, X.shape[1], F1.ctypes.data, n, F2c.ctypes.data, n, X.ctypes.data, n)
    return X
