"""GPU parity of the solves with the factors: chol_solve,
lu_solve, qr_solve against the oracle's plain substitution (orc_solve) applied to the SAME
factors (the GPU's, copied to the host), plus the residual of A X = B.

Bars: fp64 R2 (P6) <= 1e-10 against the oracle solve with the same factors and
||A X - B||_F / (||A||_F ||X||_F) <= 1e-13 n; fp32: normwise ||X - X_oracle||_F / ||X_oracle||_F
<= 2e-4 (the elementwise floored R2 of an fp32 substitution is dominated by the small
entries of X, reading P10) and residual <= 1e-5 n."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1812_02056_b200 as sf  # noqa: E402


def dev(A, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(A, np.float64).T)).to(dt).cuda()


def host(B):
    return B.double().cpu().numpy().T.copy()


def resid(A, X, B):
    return np.linalg.norm(A @ X - B) / (np.linalg.norm(A) * np.linalg.norm(X))


@pytest.mark.parametrize("n,s,nrhs", [(1, 1, 1), (33, 16, 7), (300, 64, 1), (1000, 128, 64), (777, 256, 300)])
@pytest.mark.parametrize("dtype", [sf.SF_F64, sf.SF_F32])
def test_solves(n, s, nrhs, dtype):
    dt = torch.float64 if dtype == sf.SF_F64 else torch.float32
    tol, rtol = (1e-10, 1e-13) if dtype == sf.SF_F64 else (2e-4, 1e-5)
    rng = np.random.default_rng(n + nrhs)
    Bh = rng.standard_normal((n, nrhs))
    if dtype == sf.SF_F32:
        Bh = Bh.astype(np.float32).astype(np.float64)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    cases = {"chol": synth.gen_numpy("spd_scaled", n, seed=n), "lu": synth.gen_numpy("diag_dominant", n, seed=n),
             "qr": synth.gen_numpy("gaussian", n, seed=n) + 3 * np.sqrt(n) * np.eye(n)}
    for kind, A in cases.items():
        if dtype == sf.SF_F32:
            A = A.astype(np.float32).astype(np.float64)
        dA = dev(A, dt)
        F1 = torch.zeros_like(dA); F2 = torch.zeros_like(dA)
        B = dev(Bh, dt).reshape(nrhs, n) if nrhs > 0 else None
        if kind == "chol":
            sf.chol_colmajor(n, s, dA, n, F1, n, info, dtype=dtype)
            sf.chol_solve_colmajor(n, nrhs, F1, n, B, n, dtype=dtype)
        elif kind == "lu":
            sf.lu_colmajor(n, s, dA, n, F1, n, info, dtype=dtype)
            sf.lu_solve_colmajor(n, nrhs, F1, n, B, n, dtype=dtype)
        else:
            sf.qr_colmajor(n, s, dA, n, F1, n, F2, n, info, dtype=dtype)
            sf.qr_solve_colmajor(n, nrhs, F1, n, F2, n, B, n, dtype=dtype)
        torch.cuda.synchronize()
        assert int(info.item()) == 0, kind
        Xg = B.double().cpu().numpy().T
        f1 = host(F1)
        if kind == "chol":
            f1 = np.tril(f1)
        Xo = oracle.solve(kind, f1, Bh, host(F2) if kind == "qr" else None)
        if dtype == sf.SF_F64:
            assert synth.r2_error(Xg, Xo) <= tol, (kind, synth.r2_error(Xg, Xo))
        else:
            rel = np.linalg.norm(Xg - Xo) / np.linalg.norm(Xo)
            assert rel <= tol, (kind, rel)
        assert resid(A, Xg, Bh) <= rtol * n, (kind, resid(A, Xg, Bh))
