"""f1: Strassen-Winograd in the fp64 flushes (sf_set_strassen), one level and
the paper's 2-3 recursions,
against the oracle's classical products at the P6 bar.  Sizes make every flush with side
>= min_dim take the Strassen path, with uneven (zero-padded) halves and odd K."""
import os
import sys

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1812_02056_b200 as sf  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from test_parity_gpu import TOL64, check_qr, run_chol, run_lu, run_qr  # noqa: E402


@pytest.fixture(params=[1, 2, 3])
def strassen(request):
    sf.set_strassen(request.param, 128)
    yield request.param
    sf.set_strassen(0)


@pytest.mark.parametrize("n,s", [(1000, 64), (777, 37), (1500, 200)])
def test_lu_strassen(strassen, n, s):
    A = synth.gen_numpy("diag_dominant", n, seed=n)
    Lo, Uo, io = oracle.lu(A, s)
    Lg, Ug, ig = run_lu(A, s)
    assert io == ig == 0
    assert synth.r2_error(Lg, Lo) <= TOL64 and synth.r2_error(Ug, Uo) <= TOL64
    assert synth.rel_residual(A, Lg, Ug) <= 1e-13 * n


@pytest.mark.parametrize("n,s", [(1100, 100), (901, 33)])
def test_chol_strassen(strassen, n, s):
    A = synth.gen_numpy("spd_shift", n, seed=n)
    Lo, io = oracle.chol(A, s)
    Lg, ig = run_chol(A, s, inplace=False)
    assert io == ig == 0
    assert synth.r2_error(np.tril(Lg), Lo) <= TOL64
    assert synth.rel_residual(A, np.tril(Lg), np.tril(Lg).T) <= 1e-13 * n


@pytest.mark.parametrize("n,s", [(700, 64), (513, 50)])
def test_qr_strassen(strassen, n, s):
    A = synth.gen_numpy("gaussian", n, seed=n)
    Qo, Ro, io, _ = oracle.qr(A, s)
    Qg, Rg, ig = run_qr(A, s)
    assert io == ig == 0
    check_qr(A, s, Qg, Rg, Qo, Ro)


def test_strassen_off_restores_classical():
    """Turning it off again gives bitwise the classical result (captured graphs are dropped)."""
    n, s = 1000, 64
    A = synth.gen_numpy("diag_dominant", n, seed=3)
    L0, U0, _ = run_lu(A, s)
    sf.set_strassen(1, 128)
    try:
        L1, U1, _ = run_lu(A, s)
    finally:
        sf.set_strassen(0)
    L2, U2, _ = run_lu(A, s)
    assert not np.array_equal(L1, L0)          # the Strassen path really ran
    assert np.array_equal(L2, L0) and np.array_equal(U2, U0)


def test_strassen_levels_differ_and_recurse():
    """Two and three levels really recurse (their rounding differs from one level's) and stay
    within the P6 bar; n = 2100, s = 256 makes the early flushes' level-2 products (sides
    >= 461, K = 64) and level-3 products (sides >= 230, K = 32) clear min_dim = 128."""
    n, s = 2100, 256
    A = synth.gen_numpy("diag_dominant", n, seed=5)
    Lo, Uo, _ = oracle.lu(A, s)
    outs = {}
    try:
        for lv in (1, 2, 3):
            sf.set_strassen(lv, 128)
            Lg, Ug, ig = run_lu(A, s)
            assert ig == 0 and synth.r2_error(Lg, Lo) <= TOL64 and synth.r2_error(Ug, Uo) <= TOL64
            outs[lv] = Lg
    finally:
        sf.set_strassen(0)
    assert not np.array_equal(outs[1], outs[2]) and not np.array_equal(outs[2], outs[3])
