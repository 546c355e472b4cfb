"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Every check here is independent of the oracle's own code:
  * degeneracy: s=1 == right-looking textbook, s=n == Crout textbook,
    bitwise, written independently in tests/textbook.py;
  * hand-worked examples (tests/golden/hand_examples.json), verified by exact products;
  * planted integer factors: the exact answer is known by construction;
  * LAPACK cross-checks (numpy / scipy) within rounding-error bounds;
  * invariants (triangularity, unit diagonal, residual, orthogonality, flush count);
  * restricted-column runs bitwise equal to the full run.
A dropped term, wrong sign/index or transposed operand in the flush or the panel makes
the planted and degeneracy tests fail.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth
from tests import textbook as tb

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")))
EPS = np.finfo(np.float64).eps


def tol_of(A):
    return 1e-12 * np.linalg.norm(A) / A.shape[0]


# --------------------------------------------------------------------------- golden

@pytest.mark.parametrize("ex", GOLD["cholesky"], ids=lambda e: e["cite"][:24])
def test_golden_cholesky_all_s(ex):
    A = np.array(ex["A"], float); Lx = np.array(ex["L"], float); n = len(A)
    assert np.array_equal(Lx @ Lx.T, A)          # the stored answer is a Cholesky factor
    for s in range(1, n + 1):
        L, info = oracle.chol(A, s)
        assert info == 0 and np.array_equal(L, Lx), (s, L)


@pytest.mark.parametrize("ex", GOLD["lu"], ids=lambda e: e["cite"][:24])
def test_golden_lu_all_s(ex):
    A = np.array(ex["A"], float); Lx = np.array(ex["L"], float); Ux = np.array(ex["U"], float)
    n = len(A)
    assert np.array_equal(Lx @ Ux, A) and np.all(np.diag(Ux) == 1.0)
    for s in range(1, n + 1):
        L, U, info = oracle.lu(A, s)
        assert info == 0 and np.array_equal(L, Lx) and np.array_equal(U, Ux), (s, L, U)


@pytest.mark.parametrize("ex", GOLD["qr"], ids=lambda e: e["cite"][:24])
def test_golden_qr_all_s(ex):
    A = np.array(ex["A"], float); Qx = np.array(ex["Q"], float); Rx = np.array(ex["R"], float)
    n = len(A)
    for s in range(1, n + 1):
        Q, R, info, _ = oracle.qr(A, s)
        assert info == 0
        if ex["exact"]:
            assert np.array_equal(Q, Qx) and np.array_equal(R, Rx), (s, Q, R)
        else:
            assert np.abs(Q - Qx).max() <= 4 * EPS and np.abs(R - Rx).max() <= 16 * EPS * 5


@pytest.mark.parametrize("ex", GOLD["errors"], ids=lambda e: e["kind"])
def test_golden_error_paths(ex):
    A = np.array(ex["A"], float); n = len(A)
    if ex["kind"] == "chol":       # the stated failure is a property of A, not of the oracle
        assert np.linalg.eigvalsh(A).min() <= 1e-12
    elif ex["kind"] == "qr":
        assert np.linalg.matrix_rank(A[:, :ex["info"]]) < ex["info"]
    else:
        k = ex["info"]
        assert abs(np.linalg.det(A[:k, :k])) <= 1e-12 and abs(np.linalg.det(A[:k - 1, :k - 1])) > 0.5
    for s in range(1, n + 1):
        info = {"chol": lambda: oracle.chol(A, s)[1], "lu": lambda: oracle.lu(A, s)[2],
                "qr": lambda: oracle.qr(A, s)[2]}[ex["kind"]]()
        assert info == ex["info"], (s, info)


def test_identity_all_s():
    for n in (1, 2, 5, 9):
        I = np.eye(n)
        for s in range(1, n + 1):
            assert np.array_equal(oracle.chol(I, s)[0], I)
            L, U, _ = oracle.lu(I, s)
            assert np.array_equal(L, I) and np.array_equal(U, I)
            Q, R, _, _ = oracle.qr(I, s)
            assert np.array_equal(Q, I) and np.array_equal(R, I)


def test_n1():
    L, info = oracle.chol(np.array([[9.0]]), 1)
    assert info == 0 and L[0, 0] == 3.0
    L, U, info = oracle.lu(np.array([[-5.0]]), 1)
    assert info == 0 and L[0, 0] == -5.0 and U[0, 0] == 1.0
    Q, R, info, _ = oracle.qr(np.array([[-5.0]]), 1)
    assert info == 0 and Q[0, 0] == -1.0 and R[0, 0] == 5.0


# --------------------------------------------------------------------------- degeneracy

NS = (5, 8, 13, 16, 32)   # SPEC.md:480 acceptance grid sizes


@pytest.mark.parametrize("n", NS)
def test_chol_degenerate_s1_sn_bitwise(n):
    A = synth.gen_numpy("paper_spd", n, seed=n)
    L1, i1 = oracle.chol(A, 1)
    Ln, i2 = oracle.chol(A, n)
    Lo, j1 = tb.chol_outer(A)
    Lc, j2 = tb.chol_crout(A)
    assert i1 == i2 == j1 == j2 == 0
    assert np.array_equal(L1, np.array(Lo))      # s=1: recursive algorithm
    assert np.array_equal(Ln, np.array(Lc))      # s=n: Cholesky-Crout


@pytest.mark.parametrize("n", NS)
def test_lu_degenerate_s1_sn_bitwise(n):
    A = synth.gen_numpy("diag_dominant", n, seed=100 + n)
    t = tol_of(A)
    L1, U1, _ = oracle.lu(A, 1); Ln, Un, _ = oracle.lu(A, n)
    Lo, Uo, _ = tb.lu_outer(A, t); Lc, Uc, _ = tb.lu_crout(A, t)
    assert np.array_equal(L1, np.array(Lo)) and np.array_equal(U1, np.array(Uo))
    assert np.array_equal(Ln, np.array(Lc)) and np.array_equal(Un, np.array(Uc))


@pytest.mark.parametrize("n", NS)
def test_qr_degenerate_s1_sn_bitwise(n):
    A = synth.gen_numpy("gaussian", n, seed=200 + n)
    t = tol_of(A)
    Q1, R1, _, _ = oracle.qr(A, 1); Qn, Rn, _, _ = oracle.qr(A, n)
    Qr, Rr, _ = tb.qr_mgs_right(A, t); Ql, Rl, _ = tb.qr_mgs_left(A, t)
    assert np.array_equal(Q1, np.array(Qr)) and np.array_equal(R1, np.array(Rr))
    assert np.array_equal(Qn, np.array(Ql)) and np.array_equal(Rn, np.array(Rl))


# --------------------------------------------------------------------------- planted factors

@pytest.mark.parametrize("n,s", [(64, 1), (64, 3), (64, 7), (64, 16), (64, 64), (97, 10), (97, 96)])
def test_planted_chol_exact(n, s):
    Lx = synth.planted_chol(n, seed=n * 31 + s)
    L, info = oracle.chol(Lx @ Lx.T, s)
    assert info == 0 and np.array_equal(L, Lx)


@pytest.mark.parametrize("n,s", [(64, 1), (64, 5), (64, 16), (64, 64), (97, 12)])
def test_planted_lu_exact(n, s):
    Lx, Ux = synth.planted_lu(n, seed=n * 17 + s)
    L, U, info = oracle.lu(Lx @ Ux, s)
    assert info == 0 and np.array_equal(L, Lx) and np.array_equal(U, Ux)


@pytest.mark.parametrize("n,s", [(16, 1), (16, 3), (16, 16), (64, 8), (64, 64)])
def test_planted_qr_exact(n, s):
    Qx, Rx = synth.planted_qr(n, seed=n + s)
    Q, R, info, mass = oracle.qr(Qx @ Rx, s)
    assert info == 0 and np.array_equal(Q, Qx) and np.array_equal(R, Rx) and mass == 0.0


# --------------------------------------------------------------------------- LAPACK cross-checks

@pytest.mark.parametrize("n,s", [(200, 16), (256, 64), (301, 50)])
def test_chol_vs_lapack(n, s):
    A = synth.gen_numpy("spd_shift", n, seed=n)
    L, info = oracle.chol(A, s)
    Lref = np.linalg.cholesky(A)
    assert info == 0
    assert synth.r2_error(L, Lref) < 1e-13
    assert np.all(np.triu(L, 1) == 0) and np.all(np.diag(L) > 0)
    assert synth.rel_residual(A, L, L.T) <= 1e-13 * n


@pytest.mark.parametrize("n,s", [(200, 16), (256, 64)])
def test_lu_vs_lapack(n, s):
    A = synth.gen_numpy("diag_dominant", n, seed=n)
    L, U, info = oracle.lu(A, s)
    # A^T is column-dominant, so partial pivoting performs no interchange: A^T = P L' U'
    # with P = I, hence A = U'^T L'^T; rescale to Crout (unit U): L = U'^T, U = L'^T.
    P, Lp, Up = scipy.linalg.lu(A.T)
    assert np.array_equal(P, np.eye(n))
    assert info == 0
    assert synth.r2_error(L, Up.T) < 1e-13 and synth.r2_error(U, Lp.T) < 1e-13
    assert np.all(np.diag(U) == 1.0) and np.all(np.tril(U, -1) == 0) and np.all(np.triu(L, 1) == 0)
    assert synth.rel_residual(A, L, U) <= 1e-13 * n


@pytest.mark.parametrize("n,s", [(128, 16), (200, 64)])
def test_qr_vs_lapack(n, s):
    A = synth.gen_numpy("gaussian", n, seed=n)
    Q, R, info, mass = oracle.qr(A, s)
    Qh, Rh = np.linalg.qr(A)
    sg = np.sign(np.diag(Rh))
    Qh = Qh * sg; Rh = Rh * sg[:, None]
    kappa = np.linalg.cond(A)
    assert info == 0
    # per-column ||dq||_2 <= 100 u kappa (MGS forward error; reading P7)
    assert np.max(np.linalg.norm(Q - Qh, axis=0)) <= 100 * EPS * kappa
    assert np.max(np.linalg.norm(R - Rh, axis=1)) <= 100 * EPS * kappa * np.linalg.norm(A, 2)
    assert synth.orthogonality(Q) <= 1e-12 * n
    assert synth.rel_residual(A, Q, R) <= 1e-13 * n
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) > 0)


# --------------------------------------------------------------------------- schedule / restricted

def test_flush_count_law():
    for n in range(1, 65):
        for s in range(1, n + 1):
            assert oracle.flush_count(n, s) == (n - 1) // s


@pytest.mark.parametrize("K", [1, 7, 16, 40])
def test_restricted_columns_bitwise(K):
    n, s = 96, 7
    A = synth.gen_numpy("spd_scaled", n, seed=3)
    L, _ = oracle.chol(A, s)
    Lk, _ = oracle.chol(A, s, kcols=K)
    assert np.array_equal(Lk[:, :K], L[:, :K]) and np.all(Lk[:, K:] == 0)
    B = synth.gen_numpy("diag_dominant", n, seed=4)
    L, U, _ = oracle.lu(B, s); Lk, Uk, _ = oracle.lu(B, s, kcols=K)
    assert np.array_equal(Lk[:, :K], L[:, :K]) and np.array_equal(Uk[:K, :], U[:K, :])
    C = synth.gen_numpy("gaussian", n, seed=5)
    Q, R, _, _ = oracle.qr(C, s); Qk, Rk, _, _ = oracle.qr(C, s, kcols=K)
    assert np.array_equal(Qk[:, :K], Q[:, :K]) and np.array_equal(Rk[:K, :], R[:K, :])


def test_flush_positions_hand_worked():
    """The schedule each algorithm runs (reading R1; flush iff c = z+s,
    then z := c; R11 for a sequence), recorded inside the oracle's loops, against
    positions worked out by hand.  [9,3,1,12,5,7] at n = 37: z = 0 -> c = 9 -> 12 -> 13 -> 25 ->
    30, and 30 + 7 = 37 = n never fires."""
    n = 37
    mats = {"chol": synth.gen_numpy("paper_spd", n, seed=4), "lu": synth.gen_numpy("diag_dominant", n, seed=4),
            "qr": synth.gen_numpy("gaussian", n, seed=4)}
    cases = [([9, 3, 1, 12, 5, 7], None, [9, 12, 13, 25, 30]),
             ([9, 3, 1, 12, 5, 7], 20, [9, 12, 13]),          # restricted run: flushes at c < K only
             ([2, 3], None, [2, 5, 8, 11, 14, 17, 20, 23, 26, 29, 32, 35]),   # the last step repeats
             ([36], None, [36]), ([37], None, []), ([40], None, []),
             (5, None, [5, 10, 15, 20, 25, 30, 35]), (37, None, []), (1, 6, [1, 2, 3, 4, 5]),
             (12, None, [12, 24, 36])]
    for kind, A in mats.items():
        for s, K, want in cases:
            assert oracle.flush_positions(kind, A, s, kcols=K) == want, (kind, s, K)


def test_frobenius_and_threshold_pins():
    """orc_frobenius (the R3 threshold's norm) against closed forms and LAPACK; the R3
    thresholds tol = 1e-12 ||A||_F / n pinned from both sides (a wrong power of n, a missing
    factor or the wrong norm moves the boundary past one of the two probes)."""
    for n in (1, 3, 8, 31):
        assert oracle.frobenius(np.ones((n, n))) == float(n)            # sqrt(n^2)
        Hd = np.array(scipy.linalg.hadamard(8), float)
        assert oracle.frobenius(Hd) == 8.0
        A = synth.gen_numpy("gaussian", n, seed=n)
        assert abs(oracle.frobenius(A) - np.linalg.norm(A)) <= 4 * EPS * np.linalg.norm(A)
    # diag(1, 1, 1, d): ||A||_F = sqrt(3) to within 1e-25, tol = 1e-12 * sqrt(3) / 4 = 4.330e-13
    tol = 1e-12 * np.sqrt(3.0) / 4
    for d, fails in ((0.99 * tol, True), (1.01 * tol, False)):
        A = np.diag([1.0, 1.0, 1.0, d])
        for s in (1, 2, 4):
            assert oracle.lu(A, s)[2] == (4 if fails else 0), (d, s)
            assert oracle.qr(A, s)[2] == (4 if fails else 0), (d, s)


def test_thread_count_does_not_change_bits():
    A = synth.gen_numpy("spd_scaled", 150, seed=9)
    oracle.set_threads(1); L1, _ = oracle.chol(A, 20)
    oracle.set_threads(4); L4, _ = oracle.chol(A, 20)
    oracle.set_threads(0)
    assert np.array_equal(L1, L4)


# ------------------------------------------------------------------ variable step (R11)

def test_variable_steps_pins():
    """PAPER.md:194 ("the s parameter could be varied during the execution"), reading R11:
    a constant sequence is bitwise the fixed-s algorithm; all-ones is the s = 1 schedule and
    [n] the s = n one (the textbook pins); the hand-worked 4x4 examples come out exactly for
    every sequence."""
    import itertools
    n = 37
    A = synth.gen_numpy("paper_spd", n, seed=4)
    B = synth.gen_numpy("diag_dominant", n, seed=4)
    C = synth.gen_numpy("gaussian", n, seed=4)
    for s in (1, 5, 16, n):
        seq = [s] * (-(-n // s))
        assert np.array_equal(oracle.chol(A, seq)[0], oracle.chol(A, s)[0])
        assert all(np.array_equal(x, y) for x, y in zip(oracle.lu(B, seq)[:2], oracle.lu(B, s)[:2]))
        assert all(np.array_equal(x, y) for x, y in zip(oracle.qr(C, seq)[:2], oracle.qr(C, s)[:2]))
    seq = [9, 3, 1, 12, 5, 7]
    L, info = oracle.chol(A, seq)
    assert info == 0 and np.abs(L @ L.T - A).max() <= 1e-12 * np.abs(A).max() * n
    L2, U2, info = oracle.lu(B, seq)
    assert info == 0 and np.abs(L2 @ U2 - B).max() <= 1e-12 * np.abs(B).max() * n
    Q, R, info, _ = oracle.qr(C, seq)
    assert info == 0 and np.abs(Q @ R - C).max() <= 1e-11 * np.abs(C).max() * n
    for seq in itertools.product((1, 2, 3), repeat=3):
        for ex in GOLD["cholesky"]:
            Lc, info = oracle.chol(np.array(ex["A"], float), list(seq))
            assert info == 0 and np.array_equal(Lc, np.array(ex["L"], float)), (seq, ex["cite"])
        for ex in GOLD["lu"]:
            Ll, Ul, info = oracle.lu(np.array(ex["A"], float), list(seq))
            assert info == 0 and np.array_equal(Ll, np.array(ex["L"], float)) and np.array_equal(Ul, np.array(ex["U"], float))
        for ex in GOLD["qr"]:
            Qq, Rq, info, _ = oracle.qr(np.array(ex["A"], float), list(seq))
            Q1, R1, _, _ = oracle.qr(np.array(ex["A"], float), 1)
            assert info == 0 and np.array_equal(Qq, Q1) and np.array_equal(Rq, R1), (seq, ex["cite"])


# ------------------------------------------------------------------ solves with the factors

@pytest.mark.parametrize("n", [1, 5, 60])
def test_oracle_solves_pinned(n):
    """orc_solve against scipy's triangular solves and the residual of A x = b."""
    rng = np.random.default_rng(n)
    B = rng.standard_normal((n, 3))
    A = synth.gen_numpy("paper_spd", n, seed=n)
    L, _ = oracle.chol(A, 8 if n > 8 else n)
    X = oracle.solve("chol", L, B)
    Y = scipy.linalg.solve_triangular(L, B, lower=True)
    assert np.allclose(X, scipy.linalg.solve_triangular(L.T, Y, lower=False), rtol=1e-12, atol=1e-14)
    assert np.abs(A @ X - B).max() <= 1e-12 * np.abs(B).max() * n
    D = synth.gen_numpy("diag_dominant", n, seed=n)
    Ld, Ud, _ = oracle.lu(D, 8 if n > 8 else n)
    X = oracle.solve("lu", np.tril(Ld) + np.triu(Ud, 1), B)
    assert np.allclose(X, scipy.linalg.solve_triangular(Ud, scipy.linalg.solve_triangular(Ld, B, lower=True),
                                                        lower=False, unit_diagonal=True), rtol=1e-12, atol=1e-14)
    assert np.abs(D @ X - B).max() <= 1e-12 * np.abs(B).max() * n * np.abs(D).max()
    G = synth.gen_numpy("gaussian", n, seed=n) + 4 * np.eye(n)
    Q, R, _, _ = oracle.qr(G, 8 if n > 8 else n)
    X = oracle.solve("qr", Q, B, R)
    assert np.allclose(X, scipy.linalg.solve_triangular(R, Q.T @ B, lower=False), rtol=1e-10, atol=1e-12)
    assert np.abs(G @ X - B).max() <= 1e-11 * np.abs(B).max() * n * np.abs(G).max()
