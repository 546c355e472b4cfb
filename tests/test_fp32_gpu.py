"""GPU parity of the fp32 path: fp32 storage and panel, the trailing
update as ONE 3xTF32 tcgen05 GEMM (gemm_tf32.cu).

Bar (BASELINE.json north_star; reading P9): the fp32 result against the fp64
oracle run on the fp32-ROUNDED input (the exact answer for that input): floored relative
elementwise error R2 <= 2e-4 and residual ||A - L L^T||_F/||A||_F <= 1e-5 n.  Planted
integer factors come out exactly (x_lo = 0, every partial sum an integer < 2^24).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1812_02056_b200 as sf  # noqa: E402

TOL32 = 2e-4


def dev32(A):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(A, np.float32).T)).cuda()


def host(B):
    return B.cpu().numpy().T.astype(np.float64)


def run_chol32(A, s, inplace=False):
    n = A.shape[0]
    dA = dev32(A)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = dA if inplace else torch.full_like(dA, 7.0)
    sf.chol_colmajor(n, s, dA, n, out, n, info, dtype=sf.SF_F32)
    torch.cuda.synchronize()
    return host(out), int(info.item())


@pytest.mark.parametrize("m,k", [(1, 1), (5, 3), (129, 1), (300, 40), (1000, 512), (2049, 200), (640, 33)])
def test_syrk_tf32x3_block(m, k):
    """C -= R R^T (lower) on tcgen05 against an fp64 product of the same fp32 operands."""
    rng = np.random.default_rng(m * 1000 + k)
    R = rng.standard_normal((m, k)).astype(np.float32)
    C = rng.standard_normal((m, m)).astype(np.float32)
    dR, dC = dev32(R), dev32(C)
    assert sf.lib().sf_syrk_sub(m, k, sf.SF_F32, dR.data_ptr(), m, dC.data_ptr(), m, None) == 0
    torch.cuda.synchronize()
    got = host(dC)
    ref = C.astype(np.float64) - R.astype(np.float64) @ R.astype(np.float64).T
    # the classical fp32 dot-product bound gamma_{3k+2} = (3k+2) u32 (3k products: hi.hi,
    # hi.lo, lo.hi; tensor-core fp32 accumulation is not IEEE round-to-nearest, so the
    # worst-case bound, not the sqrt(k) typical one), plus the split error 2^-22 per term
    u32 = 2.0 ** -24
    bound = ((3 * k + 2) * u32 + 2.0 ** -22) * (np.abs(R.astype(np.float64)) @ np.abs(R.astype(np.float64)).T + np.abs(C))
    lo = np.tril_indices(m)
    assert np.all(np.abs(got - ref)[lo] <= bound[lo] + 1e-30)
    up = np.triu_indices(m, 1)
    assert np.array_equal(got[up], C.astype(np.float64)[up]), "strict upper must be untouched"


@pytest.mark.parametrize("n,s", [(512, 64), (1000, 128), (2048, 512), (1030, 168)])
def test_chol32_planted_exact(n, s):
    Lx = synth.planted_chol(n, seed=n + s)
    A = Lx @ Lx.T
    assert np.abs(A).max() < 2 ** 24
    Lg, info = run_chol32(A, s)
    assert info == 0
    assert np.array_equal(np.tril(Lg), Lx)


@pytest.mark.parametrize("n,s", [(1, 1), (33, 16), (130, 32), (300, 64), (1000, 168), (2048, 512), (1500, 1500)])
def test_chol32_vs_oracle(n, s):
    A = synth.gen_numpy("spd_scaled", n, seed=n + s)
    A32 = A.astype(np.float32).astype(np.float64)      # the fp32-rounded input (reading P9)
    Lg, info = run_chol32(A32, s)
    assert info == 0
    Lo, io = oracle.chol(A32, s)
    assert io == 0
    Lg = np.tril(Lg)
    assert synth.r2_error(Lg, Lo) <= TOL32
    assert synth.rel_residual(A32, Lg, Lg.T) <= 1e-5 * n
    assert np.all(np.diag(Lg) > 0)


def test_chol32_inplace_untouched_upper_and_info():
    n, s = 700, 128
    A = synth.gen_numpy("paper_spd", n, seed=9).astype(np.float32).astype(np.float64)
    Lg, info = run_chol32(A, s, inplace=True)
    assert info == 0
    assert np.array_equal(np.triu(Lg, 1), np.triu(A, 1))
    B = A.copy(); B[400, 400] = -5.0
    assert run_chol32(B, s)[1] == oracle.chol(B, s)[1] == 401


def test_chol32_cfg5_shape_sampled():
    """cfg5's fp32 setting (s = 512, A = G G^T/n + I rounded to fp32) at n = 16384: the first
    K columns against the restricted fp64 oracle, plus a Freivalds residual of the whole
    factor (torch fp64, an independent checker)."""
    n, s, K = 16384, 512, 1536      # K = 3s: entries of both lookahead flush parts compared
    A64 = synth.gen_torch("spd_scaled", n, seed=0)
    A32 = A64.float()
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    L = torch.zeros_like(A32)
    sf.chol_colmajor(n, s, A32, n, L, n, info, dtype=sf.SF_F32)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    Ll = torch.tril(L.mT).double()
    Ar = A32.double()
    Lo, io = oracle.chol(np.asfortranarray(Ar[:, :K].cpu().numpy()), s, kcols=K)
    assert io == 0
    assert synth.r2_error(Ll[:, :K].cpu().numpy(), Lo[:, :K]) <= TOL32
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    x = torch.randn(n, 4, device="cuda", dtype=torch.float64, generator=g)
    r = (Ar @ x - Ll @ (Ll.mT @ x)).norm() / (Ar @ x).norm()
    assert float(r) <= 1e-5 * n


# ------------------------------------------------------------------ fp32 LU / QR

def run_lu32(A, s):
    n = A.shape[0]
    dA = torch.from_numpy(np.ascontiguousarray(np.asarray(A, np.float32).T)).cuda()
    out = torch.full_like(dA, 7.0)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    sf.lu_colmajor(n, s, dA, n, out, n, info, dtype=sf.SF_F32)
    torch.cuda.synchronize()
    F = host(out)
    return np.tril(F), np.triu(F, 1) + np.eye(n), int(info.item())


def run_qr32(A, s):
    n = A.shape[0]
    dA = torch.from_numpy(np.ascontiguousarray(np.asarray(A, np.float32).T)).cuda()
    Q = torch.empty_like(dA); R = torch.full_like(dA, 3.0)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    sf.qr_colmajor(n, s, dA, n, Q, n, R, n, info, dtype=sf.SF_F32)
    torch.cuda.synchronize()
    return host(Q), host(R), int(info.item())


@pytest.mark.parametrize("n,s", [(1, 1), (33, 16), (130, 32), (300, 64), (1000, 168), (2048, 512), (4096, 64)])
def test_lu32_vs_oracle(n, s):
    A = synth.gen_numpy("diag_dominant", n, seed=n + s).astype(np.float32).astype(np.float64)
    Lg, Ug, info = run_lu32(A, s)
    assert info == 0
    Lo, Uo, io = oracle.lu(A, s)
    assert io == 0
    assert synth.r2_error(Lg, Lo) <= TOL32 and synth.r2_error(Ug, Uo) <= TOL32
    assert synth.rel_residual(A, Lg, Ug) <= 1e-5 * n


@pytest.mark.parametrize("n,s", [(700, 64), (1024, 128)])
def test_lu32_planted_exact(n, s):
    Lx, Ux = synth.planted_lu(n, seed=n + s)
    Lg, Ug, info = run_lu32(Lx @ Ux, s)
    assert info == 0 and np.array_equal(Lg, Lx) and np.array_equal(Ug, Ux)


@pytest.mark.parametrize("n,s", [(4, 2), (130, 32), (300, 64), (1024, 128)])
def test_qr32_vs_oracle(n, s):
    """fp32 QR against the fp64 oracle on the fp32-rounded input (reading P10):
    forward errors within the classical bounds — per column of Q
    ||dq_j|| <= (100 kappa_j + 3n + 2) u32 (kappa_j: of the head block for columns [0, n-2s),
    of A for the tail; 3n + 2: the worst-case fp32 dot product over the 3xTF32 K' = 3n,
    since the tensor core's fp32 accumulation is not round-to-nearest), per row of R the
    same times ||A||_2 sqrt(n); residual <= 1e-5 n (the north star's fp32 residual bar);
    orthogonality <= max(1e-5 n, 100 u32 kappa(A)) (MGS loses orthogonality ~ u kappa).  The floored elementwise R2 is dominated by Q's tiny entries (a plain
    fp32 MGS of the n = 130 case already has head R2 = 1.0e-4), so it is not used here."""
    A = synth.gen_numpy("gaussian", n, seed=n + s).astype(np.float32).astype(np.float64)
    Qg, Rg, info = run_qr32(A, s)
    assert info == 0
    Qo, Ro, io, _ = oracle.qr(A, s)
    assert io == 0
    u32 = 2.0 ** -24
    head = max(0, n - 2 * s)
    k_all = np.linalg.cond(A)
    k_head = np.linalg.cond(A[:, :head]) if head else k_all
    dq = np.linalg.norm(Qg - Qo, axis=0)
    dr = np.linalg.norm(Rg - Ro, axis=1)
    nA = np.linalg.norm(A, 2) * np.sqrt(n)
    g = (3 * n + 2) * u32
    if head:
        assert np.max(dq[:head]) <= 100 * u32 * k_head + g, (np.max(dq[:head]), k_head)
        assert np.max(dr[:head]) <= (100 * u32 * k_head + g) * nA, (np.max(dr[:head]), k_head)
    assert np.max(dq) <= 100 * u32 * k_all + g
    assert np.max(dr) <= (100 * u32 * k_all + g) * nA
    assert np.all(np.tril(Rg, -1) == 0)
    # MGS loses orthogonality like c u kappa(A) (Bjorck), fp32: u = 2^-24
    assert synth.orthogonality(Qg) <= max(1e-5 * n, 100 * u32 * k_all)
    assert synth.rel_residual(A, Qg, Rg) <= 1e-5 * n


def test_qr32_planted_exact():
    n, s = 1024, 128
    Qx, Rx = synth.planted_qr(n, seed=3)
    Qg, Rg, info = run_qr32(Qx @ Rx, s)
    assert info == 0 and np.array_equal(Qg, Qx) and np.array_equal(Rg, Rx)
