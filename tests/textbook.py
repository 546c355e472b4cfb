"""Independent textbook factorizations in pure Python (small n only) — oracle pins.

PAPER.md:176: "when s=1 it particularizes to the recursive algorithm and when s=n it
becomes Cholesky--Crout algorithm".  These are those two classical algorithms (and the
LU / MGS analogues), written from the textbook definitions, not from the oracle's C.
Python floats are IEEE binary64 with no FMA contraction and a correctly rounded sqrt, so
when the operation sequence of Alg. 1-3 at s=1 / s=n coincides with the textbook one
(it does, term by term) the results are bitwise equal.
"""
import math


def _mat(A):
    return [[float(x) for x in row] for row in A]


def chol_crout(A):
    """Left-looking Cholesky-Crout: column c from all previous columns."""
    A = _mat(A); n = len(A)
    L = [[0.0] * n for _ in range(n)]
    for c in range(n):
        d = A[c][c]
        for k in range(c):
            d = d - L[c][k] * L[c][k]
        if not d > 0.0:
            return L, c + 1
        L[c][c] = math.sqrt(d)
        for i in range(c + 1, n):
            t = A[i][c]
            for k in range(c):
                t = t - L[i][k] * L[c][k]
            L[i][c] = t / L[c][c]
    return L, 0


def chol_outer(A):
    """Right-looking (recursive / outer-product) Cholesky: trailing -= v v^T each column."""
    A = _mat(A); n = len(A)
    L = [[0.0] * n for _ in range(n)]
    for c in range(n):
        if not A[c][c] > 0.0:
            return L, c + 1
        L[c][c] = math.sqrt(A[c][c])
        for i in range(c + 1, n):
            L[i][c] = A[i][c] / L[c][c]
        for j in range(c + 1, n):
            for i in range(c + 1, n):
                A[i][j] = A[i][j] - L[i][c] * L[j][c]
    return L, 0


def lu_crout(A, tol):
    """Crout LU (L with diagonal, U unit upper), left-looking."""
    A = _mat(A); n = len(A)
    L = [[0.0] * n for _ in range(n)]; U = [[0.0] * n for _ in range(n)]
    for c in range(n):
        for i in range(c, n):
            t = A[i][c]
            for k in range(c):
                t = t - L[i][k] * U[k][c]
            L[i][c] = t
        if not abs(L[c][c]) >= tol:
            return L, U, c + 1
        for i in range(c, n):
            t = A[c][i]
            for k in range(c):
                t = t - L[c][k] * U[k][i]
            U[c][i] = t / L[c][c]
    return L, U, 0


def lu_outer(A, tol):
    """Right-looking Crout LU: column c of L and row c of U, then trailing -= l u^T."""
    A = _mat(A); n = len(A)
    L = [[0.0] * n for _ in range(n)]; U = [[0.0] * n for _ in range(n)]
    for c in range(n):
        for i in range(c, n):
            L[i][c] = A[i][c]
        if not abs(L[c][c]) >= tol:
            return L, U, c + 1
        for i in range(c, n):
            U[c][i] = A[c][i] / L[c][c]
        for j in range(c + 1, n):
            for i in range(c + 1, n):
                A[i][j] = A[i][j] - L[i][c] * U[c][j]
    return L, U, 0


def _qt_a(Q, A, n):
    R = [[0.0] * n for _ in range(n)]
    for k in range(n):
        for j in range(n):
            t = 0.0
            for i in range(n):
                t += Q[i][k] * A[i][j]
            R[k][j] = t
    for j in range(n):
        for k in range(j + 1, n):
            R[k][j] = 0.0
    return R


def qr_mgs_left(A, tol):
    """Left-looking modified Gram-Schmidt; R := Q^T A."""
    A = _mat(A); n = len(A)
    Q = [[0.0] * n for _ in range(n)]
    for c in range(n):
        v = [A[i][c] for i in range(n)]
        for j in range(c):
            t = 0.0
            for i in range(n):
                t += Q[i][j] * v[i]
            for i in range(n):
                v[i] = v[i] - Q[i][j] * t
        nv2 = 0.0
        for i in range(n):
            nv2 += v[i] * v[i]
        nv = math.sqrt(nv2)
        if not nv >= tol:
            return Q, None, c + 1
        for i in range(n):
            Q[i][c] = v[i] / nv
    return Q, _qt_a(Q, A, n), 0


def qr_mgs_right(A, tol):
    """Right-looking MGS: normalize column c, then project it out of every later column."""
    A0 = _mat(A); V = _mat(A); n = len(V)
    Q = [[0.0] * n for _ in range(n)]
    for c in range(n):
        nv2 = 0.0
        for i in range(n):
            nv2 += V[i][c] * V[i][c]
        nv = math.sqrt(nv2)
        if not nv >= tol:
            return Q, None, c + 1
        for i in range(n):
            Q[i][c] = V[i][c] / nv
        for j in range(c + 1, n):
            t = 0.0
            for i in range(n):
                t += Q[i][c] * V[i][j]
            for i in range(n):
                V[i][j] = V[i][j] - Q[i][c] * t
    return Q, _qt_a(Q, A0, n), 0
