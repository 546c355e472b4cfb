"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star; DESIGN.md §3 readings P6/P7):
  fp64: floored relative elementwise error (synth.r2_error) <= 1e-10, residual <= 1e-13*n
  QR:   R2 <= 1e-10 on Q columns / R rows [0, n-2s); tail columns within 100*u*kappa
  planted integer factors: bit-exact.
Inputs are the same bytes on both sides (synth generators).  Sizes span several 128-wide
tiles and ragged tails; full BASELINE sizes are checked on sampled (restricted-column)
outputs the oracle computes exactly as in the full run.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1812_02056_b200 as sf  # noqa: E402

EPS = np.finfo(np.float64).eps
TOL64 = 1e-10


def dev(A):
    """numpy logical matrix -> device buffer holding it column-major."""
    return torch.from_numpy(np.ascontiguousarray(np.asarray(A, np.float64).T)).cuda()


def host(B):
    """device column-major buffer -> numpy logical matrix."""
    return B.cpu().numpy().T.copy()


def run_chol(A, s, inplace=True):
    n = A.shape[0]
    dA = dev(A)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    if inplace:
        sf.chol_colmajor(n, s, dA, n, dA, n, info)
        out = dA
    else:
        out = torch.full_like(dA, 7.0)
        sf.chol_colmajor(n, s, dA, n, out, n, info)
        assert np.array_equal(host(dA), A), "out-of-place call modified A"
    torch.cuda.synchronize()
    return host(out), int(info.item())


def run_lu(A, s, inplace=True):
    n = A.shape[0]
    dA = dev(A)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = dA if inplace else torch.empty_like(dA)
    sf.lu_colmajor(n, s, dA, n, out, n, info)
    torch.cuda.synchronize()
    F = host(out)
    return np.tril(F), np.triu(F, 1) + np.eye(n), int(info.item())


def run_qr(A, s):
    n = A.shape[0]
    dA = dev(A)
    Q = torch.empty_like(dA); R = torch.full_like(dA, 3.0)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    sf.qr_colmajor(n, s, dA, n, Q, n, R, n, info)
    torch.cuda.synchronize()
    return host(Q), host(R), int(info.item())


def flushed_cols(K, s):
    """How many of the first K columns are produced AFTER at least one flush (c >= s) and
    how many after the lookahead's part-2 update (columns beyond the panel that follows a
    flush: c >= 2s) — what a restricted-oracle comparison of K columns exercises."""
    return max(0, K - s), max(0, K - 2 * s)


def svals(n):
    return sorted({1, 2, 3, 7, 16, 32, 64, 100, 128, 130, 200, n // 2, n} & set(range(1, n + 1)))


# ============================================================ Cholesky

@pytest.mark.parametrize("n", [1, 2, 5, 33, 127, 130, 300])
def test_chol_small_grid(n):
    A = synth.gen_numpy("paper_spd", n, seed=n)
    for s in svals(n):
        Lo, io = oracle.chol(A, s)
        for inplace in (True, False):
            Lg, ig = run_chol(A, s, inplace)
            assert ig == io == 0
            low = np.tril(Lg)
            assert synth.r2_error(low, Lo) <= TOL64, (n, s, inplace)
            if inplace:
                assert np.array_equal(np.triu(Lg, 1), np.triu(A, 1)), "strict upper must be untouched"
            else:
                assert np.all(Lg[np.triu_indices(n, 1)] == 7.0), "out of place: strict upper of L never written"
            assert np.all(np.diag(low) > 0)
            assert synth.rel_residual(A, low, low.T) <= 1e-13 * n


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_chol_cfg1(seed):
    """BASELINE.json configs[0]: n=256, s=16, A = G G^T + n I."""
    n, s = 256, 16
    A = synth.gen_numpy("spd_shift", n, seed)
    Lo, _ = oracle.chol(A, s)
    Lg, info = run_chol(A, s)
    Lg = np.tril(Lg)
    assert info == 0
    assert synth.r2_error(Lg, Lo) <= TOL64
    assert synth.rel_residual(A, Lg, Lg.T) <= 1e-13 * n


@pytest.mark.parametrize("n,s", [(512, 1), (1000, 16), (1000, 168), (4096, 64), (4096, 512), (2048, 2048)])
def test_chol_planted_exact(n, s):
    Lx = synth.planted_chol(n, seed=n + s)
    Lg, info = run_chol(Lx @ Lx.T, s)
    assert info == 0
    assert np.array_equal(np.tril(Lg), Lx)


def test_chol_not_pd_info():
    A = np.array([[1.0, 2.0], [2.0, 1.0]])
    for s in (1, 2):
        assert run_chol(A, s)[1] == 2
    B = synth.gen_numpy("paper_spd", 300, seed=3)
    B[200, 200] = -5.0
    io = oracle.chol(B, 64)[1]
    assert run_chol(B, 64)[1] == io == 201


def test_chol_deterministic():
    A = synth.gen_numpy("spd_scaled", 700, seed=5)
    a, _ = run_chol(A, 96)
    b, _ = run_chol(A, 96)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("s", [64, 168, 512, 1024])
def test_chol_cfg3_sampled(s):
    """BASELINE.json configs[2] at full size n=16384: the first K = max(384, 3s) columns of L
    against the restricted oracle (bitwise the full oracle's first K columns) — so entries
    updated by flush part 1 (the next panel's columns) AND part 2 (the rest, concurrent with
    the lookahead panel) are compared elementwise — plus a Freivalds residual of the whole
    factor computed with torch (an independent checker)."""
    n = 16384
    K = max(384, 3 * s)
    f1, f2 = flushed_cols(K, s)
    assert f1 >= 2 * s and f2 >= s
    A = synth.gen_torch("spd_scaled", n, seed=0)
    B = A.clone()                                   # symmetric: column-major buffer == A
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    sf.chol_colmajor(n, s, B, n, B, n, info)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    L = torch.tril(B.mT)                            # logical L
    Ak = A[:, :K].cpu().numpy()                     # column j of A = A[:, j] (symmetric)
    Lo, io = oracle.chol(Ak, s, kcols=K)
    assert io == 0
    assert synth.r2_error(L[:, :K].cpu().numpy(), Lo[:, :K]) <= TOL64
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    x = torch.randn(n, 4, device="cuda", dtype=torch.float64, generator=g)
    r = (A @ x - L @ (L.mT @ x)).norm() / (A @ x).norm()
    assert float(r) <= 1e-13 * n


# ============================================================ LU

@pytest.mark.parametrize("n", [1, 3, 33, 130, 257])
def test_lu_small_grid(n):
    A = synth.gen_numpy("diag_dominant", n, seed=n)
    for s in svals(n):
        Lo, Uo, io = oracle.lu(A, s)
        for inplace in (True, False):
            Lg, Ug, ig = run_lu(A, s, inplace)
            assert ig == io == 0
            assert synth.r2_error(Lg, Lo) <= TOL64 and synth.r2_error(Ug, Uo) <= TOL64, (n, s)
            assert synth.rel_residual(A, Lg, Ug) <= 1e-13 * n


def test_lu_cfg2():
    """BASELINE.json configs[1]: n=4096, s=64, strictly diagonally dominant U(-1,1)."""
    n, s = 4096, 64
    A = synth.gen_numpy("diag_dominant", n, seed=0)
    Lo, Uo, io = oracle.lu(A, s)
    Lg, Ug, ig = run_lu(A, s)
    assert io == ig == 0
    assert synth.r2_error(Lg, Lo) <= TOL64 and synth.r2_error(Ug, Uo) <= TOL64
    assert synth.rel_residual(A, Lg, Ug) <= 1e-13 * n


@pytest.mark.parametrize("n,s", [(512, 1), (1000, 64), (2048, 200)])
def test_lu_planted_exact(n, s):
    Lx, Ux = synth.planted_lu(n, seed=n + s)
    Lg, Ug, info = run_lu(Lx @ Ux, s)
    assert info == 0 and np.array_equal(Lg, Lx) and np.array_equal(Ug, Ux)


def test_lu_zero_pivot_info():
    A = np.array([[0.0, 1.0], [1.0, 1.0]])
    for s in (1, 2):
        assert run_lu(A, s)[2] == 1


@pytest.mark.parametrize("n,s,bad", [(300, 64, 200), (1000, 128, 777), (2048, 64, 1500)])
def test_lu_interior_failure_info(n, s, bad):
    """R3 at an interior column beyond the first panel: planted integer
    factors with L_bad,bad = 0 exactly, so |L_cc| < tol at column bad+1 on both sides."""
    Lx, Ux = synth.planted_lu(n, seed=n + bad)
    Lx[bad, bad] = 0.0
    A = Lx @ Ux
    io = oracle.lu(A, s)[2]
    assert io == bad + 1
    for inplace in (True, False):
        assert run_lu(A, s, inplace)[2] == io
    # the panels before the failing one are the exact factor (from the failing panel on the
    # outputs are unspecified, include/stepfact.h)
    p0 = bad // s * s
    Lg, Ug, _ = run_lu(A, s)
    assert np.array_equal(Lg[:, :p0], Lx[:, :p0]) and np.array_equal(Ug[:p0, :p0], Ux[:p0, :p0])


# ============================================================ QR

def check_qr(A, s, Qg, Rg, Qo, Ro):
    n = A.shape[0]
    head = max(0, n - 2 * s)
    kappa = np.linalg.cond(A)
    if head > 0:
        assert synth.r2_error(Qg[:, :head], Qo[:, :head]) <= TOL64
        assert synth.r2_error(Rg[:head, :], Ro[:head, :]) <= TOL64
    # tail columns: forward error of MGS is ~u*kappa (reading P7)
    assert np.max(np.linalg.norm(Qg - Qo, axis=0)) <= max(100 * EPS * kappa, 1e-13)
    assert np.max(np.linalg.norm(Rg - Ro, axis=1)) <= max(100 * EPS * kappa, 1e-13) * np.linalg.norm(A, 2)
    assert np.all(np.tril(Rg, -1) == 0)
    assert synth.orthogonality(Qg) <= 1e-12 * n
    assert synth.rel_residual(A, Qg, Rg) <= 1e-13 * n


@pytest.mark.parametrize("n", [1, 4, 33, 130, 257])
def test_qr_small_grid(n):
    A = synth.gen_numpy("gaussian", n, seed=n)
    for s in svals(n):
        Qo, Ro, io, _ = oracle.qr(A, s)
        Qg, Rg, ig = run_qr(A, s)
        assert io == ig == 0
        check_qr(A, s, Qg, Rg, Qo, Ro)


@pytest.mark.timeout(600, method="thread")
@pytest.mark.parametrize("n,s,bad", [(300, 64, 150), (3, 1, 1), (2000, 96, 1500), (8192, 128, 4000),
                                     (16384, 128, 9000)])
def test_qr_rank_deficient_info(n, s, bad):
    """R3 for QR (PAPER.md:158-164 needs full rank): column `bad` repeats column 0, so after
    projection ||v|| is round-off (~u ||a_0||), far below 1e-12 ||A||_F / n, on both sides;
    info = bad + 1.  At n = 8192 / 16384 the column is zero (||v|| = 0 exactly: at that size
    ||a_0|| ~ sqrt(n) puts round-off within a decade of the threshold); these run the
    persistent multi-cluster MGS grid, whose CTAs must all leave together once the failure
    is flagged (no hang: the test has a timeout)."""
    A = synth.gen_numpy("gaussian", n, seed=n + bad)
    A[:, bad] = A[:, 0] if n <= 2000 else 0.0
    if n <= 2000:
        io = oracle.qr(A, s)[2]
        assert io == bad + 1
    Qg, Rg, ig = run_qr(A, s)
    assert ig == bad + 1
    if n <= 2000:   # the panels before the failing one still match the oracle's
        p0 = bad // s * s
        Qo = oracle.qr(A, s, kcols=max(p0, 1))[0]
        assert p0 == 0 or synth.r2_error(Qg[:, :p0], Qo[:, :p0]) <= TOL64


def test_qr_wide_panels_chunked():
    """Reading R12: a panel wider than one MGS launch holds (w_max = 216 columns
    at n = 2048: 16 CTAs of 128 rows, (220 KiB/8 - 64)/(128 + 2)) is factored in chunks, each
    chunk block-projected against the earlier chunks of its panel before its own MGS.  With
    s = 512 every panel takes that path (chunks 216 + 216 + 80); the head columns [0, n-2s) —
    two whole chunked panels and the flush between them — meet the R2 <= 1e-10 bar."""
    n, s = 2048, 512
    A = synth.gen_numpy("gaussian", n, seed=11)
    Qo, Ro, io, _ = oracle.qr(A, s)
    Qg, Rg, ig = run_qr(A, s)
    assert io == ig == 0
    assert n - 2 * s >= 2 * 216
    check_qr(A, s, Qg, Rg, Qo, Ro)


@pytest.mark.parametrize("n,s", [(256, 1), (256, 64), (1024, 128), (4096, 128)])
def test_qr_planted_exact(n, s):
    Qx, Rx = synth.planted_qr(n, seed=n + s)
    Qg, Rg, info = run_qr(Qx @ Rx, s)
    assert info == 0 and np.array_equal(Qg, Qx) and np.array_equal(Rg, Rx)


def test_qr_cfg4_sampled():
    """BASELINE.json configs[3] at full size: n=8192, s=128, N(0,1); first K columns of Q
    and rows of R against the restricted oracle, plus orthogonality/residual probes."""
    n, s, K = 8192, 128, 256
    A = synth.gen_numpy("gaussian", n, seed=0)
    Qg, Rg, ig = run_qr(A, s)
    Qo, Ro, io, _ = oracle.qr(A, s, kcols=K)
    assert io == ig == 0
    assert synth.r2_error(Qg[:, :K], Qo[:, :K]) <= TOL64
    assert synth.r2_error(Rg[:K, :], Ro[:K, :]) <= TOL64
    Qt = torch.from_numpy(Qg).cuda(); At = torch.from_numpy(A).cuda(); Rt = torch.from_numpy(Rg).cuda()
    assert float((Qt.mT @ Qt - torch.eye(n, device="cuda", dtype=torch.float64)).norm()) <= 1e-12 * n
    assert float((At - Qt @ Rt).norm() / At.norm()) <= 1e-13 * n
    assert np.all(np.tril(Rg, -1) == 0)


# ============================================================ building blocks

def test_syrk_and_gemm_blocks():
    rng = np.random.default_rng(0)
    m, k = 300, 40
    R = rng.standard_normal((m, k)); C = rng.standard_normal((m, m))
    dR, dC = dev(R), dev(C)
    assert sf.lib().sf_syrk_sub(m, k, 0, dR.data_ptr(), m, dC.data_ptr(), m, None) == 0
    torch.cuda.synchronize()
    ref = C - R @ R.T
    got = host(dC)
    assert np.abs(np.tril(got) - np.tril(ref)).max() <= 1e-13 * k * 10
    assert np.array_equal(np.triu(got, 1), np.triu(C, 1))
    A = rng.standard_normal((k, m)); B = rng.standard_normal((m, k)); C = rng.standard_normal((m, m))
    dA, dB, dC = dev(A), dev(B), dev(C)
    # C -= A^T B^T  (ta=1: A stored k x m; tb=1: B stored m x k)
    assert sf.lib().sf_gemm_sub(m, m, k, 0, dA.data_ptr(), k, 1, dB.data_ptr(), m, 1, dC.data_ptr(), m, None) == 0
    torch.cuda.synchronize()
    assert np.abs(host(dC) - (C - A.T @ B.T)).max() <= 1e-12


def test_torch_api_roundtrip():
    A = synth.gen_numpy("spd_shift", 200, seed=1)
    L, info = sf.chol(torch.from_numpy(A).cuda(), 32)
    assert info == 0 and synth.r2_error(np.tril(L.cpu().numpy()), oracle.chol(A, 32)[0]) <= TOL64
    B = synth.gen_numpy("gaussian", 150, seed=2)
    Q, R, info = sf.qr(torch.from_numpy(B).cuda(), 32)
    assert info == 0 and synth.rel_residual(B, Q.cpu().numpy(), R.cpu().numpy()) <= 1e-13 * 150


def test_host_entry_points():
    n, s = 300, 64
    A = synth.gen_numpy("spd_shift", n, seed=4)
    hA = np.asfortranarray(A.copy())
    out, info = sf.chol_host(hA, s)
    assert info == 0 and synth.r2_error(np.tril(out), oracle.chol(A, s)[0]) <= TOL64
    B = synth.gen_numpy("diag_dominant", n, seed=5)
    hB = np.asfortranarray(B.copy())
    out, info = sf.lu_host(hB, s)
    Lo, Uo, _ = oracle.lu(B, s)
    assert info == 0 and synth.r2_error(np.tril(out), Lo) <= TOL64


@pytest.mark.parametrize("s", [2, 4, 8])
def test_lookahead_repeatable(s):
    """Regression for a cross-stream stale-L1 race (DESIGN.md §5 'memory visibility'): the
    lookahead panel stream and the update stream share SMs; every run must match the oracle
    and every other run bit for bit."""
    n = 256
    A = synth.gen_numpy("gaussian", n, seed=n)
    Qo, Ro, _, _ = oracle.qr(A, s)
    first = None
    for _ in range(4):
        Qg, Rg, info = run_qr(A, s)
        assert info == 0 and np.abs(Qg - Qo).max() < 1e-12
        if first is None:
            first = Qg
        assert np.array_equal(Qg, first)
    B = synth.gen_numpy("diag_dominant", 300, seed=1)
    Lo, Uo, _ = oracle.lu(B, s)
    for _ in range(3):
        Lg, Ug, info = run_lu(B, s)
        assert info == 0 and synth.r2_error(Lg, Lo) <= TOL64 and synth.r2_error(Ug, Uo) <= TOL64


@pytest.mark.parametrize("kind", ["chol", "lu", "qr", "chol32"])
def test_graph_replay(kind):
    """Repeated calls with the same arguments replay a captured CUDA graph (driver.cu
    run_graph: eager, capture, replay): every call must produce the oracle's factor, and
    the library's launch counter must keep counting the replayed kernels."""
    n, s = 600, 96
    if kind.startswith("chol"):
        A = synth.gen_numpy("spd_scaled", n, seed=3)
        if kind == "chol32":
            A = A.astype(np.float32).astype(np.float64)
        Lo, _ = oracle.chol(A, s)
    elif kind == "lu":
        A = synth.gen_numpy("diag_dominant", n, seed=3)
        Lo, Uo, _ = oracle.lu(A, s)
    else:
        A = synth.gen_numpy("gaussian", n, seed=3)
        Qo, Ro, _, _ = oracle.qr(A, s)
    dA = dev(A)
    if kind == "chol32":
        dA = dA.float()
    o1 = torch.empty_like(dA); o2 = torch.empty_like(dA)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    stream = torch.cuda.Stream()
    counts = []
    for it in range(4):
        o1.fill_(0.0); o2.fill_(0.0); info.fill_(-1)
        torch.cuda.synchronize()
        l0 = sf.launch_counter()
        with torch.cuda.stream(stream):
            if kind == "chol":
                sf.chol_colmajor(n, s, dA, n, o1, n, info, stream=stream)
            elif kind == "chol32":
                sf.chol_colmajor(n, s, dA, n, o1, n, info, dtype=sf.SF_F32, stream=stream)
            elif kind == "lu":
                sf.lu_colmajor(n, s, dA, n, o1, n, info, stream=stream)
            else:
                sf.qr_colmajor(n, s, dA, n, o1, n, o2, n, info, stream=stream)
        stream.synchronize()
        counts.append(sf.launch_counter() - l0)
        assert int(info.item()) == 0, it
        F = host(o1.double())
        if kind == "chol":
            assert synth.r2_error(np.tril(F), Lo) <= TOL64, it
        elif kind == "chol32":
            assert synth.r2_error(np.tril(F), Lo) <= 2e-4, it
        elif kind == "lu":
            assert synth.r2_error(np.tril(F), Lo) <= TOL64 and synth.r2_error(np.triu(F, 1) + np.eye(n), Uo) <= TOL64
        else:
            check_qr(A, s, F, host(o2), Qo, Ro)
    assert counts[0] > 10 and counts[1:] == [counts[0]] * 3, counts


@pytest.mark.parametrize("n,s,dtype", [(1, 1, 0), (300, 64, 0), (257, 100, 0), (1000, 128, 1), (513, 512, 0)])
def test_chol_host_lower_panels(n, s, dtype):
    """chol_factor_host: lower triangle copied panel by panel, each panel of L returned as
    soon as it is final (overlapped D2H); out of place the strict upper is unspecified
    except outside the diagonal blocks (untouched); in place it keeps A's values."""
    A = synth.gen_numpy("spd_scaled", n, seed=n)
    if dtype == 1:
        A = A.astype(np.float32).astype(np.float64)
    npdt = np.float64 if dtype == 0 else np.float32
    hA = np.asfortranarray(A.astype(npdt))
    hL = np.asfortranarray(np.full((n, n), 7.0, dtype=npdt))
    out, info = sf.chol_host(hA, s, hL, dtype=dtype)
    assert info == 0
    Lo, _ = oracle.chol(A, s)
    assert synth.r2_error(np.tril(out).astype(np.float64), Lo) <= (TOL64 if dtype == 0 else 2e-4)
    far = np.triu(np.ones((n, n), bool), 1) & ((np.arange(n)[:, None] // s) != (np.arange(n)[None, :] // s))
    assert np.all(out[far] == 7.0), "entries above the diagonal blocks must be untouched"
    assert np.array_equal(hA, A.astype(npdt)), "input modified"
    # in place: upper triangle keeps A's values
    hB = np.asfortranarray(A.astype(npdt))
    out2, info2 = sf.chol_host(hB, s, dtype=dtype)
    assert info2 == 0 and np.array_equal(np.tril(out2), np.tril(out)) and np.array_equal(np.triu(out2, 1), np.triu(A.astype(npdt), 1))


# ============================================================ variable step (f2, reading R11)

@pytest.mark.parametrize("steps", [[64], [7, 100, 33, 1, 64], [256, 128, 64, 32, 16], [1000]])
def test_variable_steps(steps):
    """chol/lu/qr_factor_steps: against the oracle run with the same step
    sequence; a tapering sequence (large panels early, small at the tail) included."""
    n = 700
    A = synth.gen_numpy("spd_scaled", n, seed=21)
    dA = dev(A)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = torch.full_like(dA, 7.0)
    sf.chol_steps_colmajor(n, steps, dA, n, out, n, info)
    torch.cuda.synchronize()
    Lo, io = oracle.chol(A, steps)
    assert int(info.item()) == io == 0
    assert synth.r2_error(np.tril(host(out)), Lo) <= TOL64
    B = synth.gen_numpy("diag_dominant", n, seed=22)
    dB = dev(B)
    out = torch.empty_like(dB)
    sf.lu_steps_colmajor(n, steps, dB, n, out, n, info)
    torch.cuda.synchronize()
    Lo, Uo, io = oracle.lu(B, steps)
    F = host(out)
    assert int(info.item()) == io == 0
    assert synth.r2_error(np.tril(F), Lo) <= TOL64 and synth.r2_error(np.triu(F, 1) + np.eye(n), Uo) <= TOL64
    C = synth.gen_numpy("gaussian", n, seed=23)
    dC = dev(C)
    Q = torch.empty_like(dC); R = torch.empty_like(dC)
    sf.qr_steps_colmajor(n, steps, dC, n, Q, n, R, n, info)
    torch.cuda.synchronize()
    Qo, Ro, io, _ = oracle.qr(C, steps)
    assert int(info.item()) == io == 0
    last = steps[-1] if sum(steps) < n else steps[min(len(steps) - 1, 2)]
    check_qr(C, max(last, 64), host(Q), host(R), Qo, Ro)


def test_variable_steps_constant_is_fixed_s():
    n, s = 520, 96
    A = synth.gen_numpy("spd_scaled", n, seed=2)
    dA = dev(A)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    o1 = torch.zeros_like(dA); o2 = torch.zeros_like(dA)
    sf.chol_colmajor(n, s, dA, n, o1, n, info)
    sf.chol_steps_colmajor(n, [s] * 3, dA, n, o2, n, info)   # the last step repeats
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


def test_variable_steps_invalid():
    d = torch.zeros(16, device="cuda", dtype=torch.float64)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(sf.StepfactError):
        sf.chol_steps_colmajor(4, [2, 0], d, 4, d, 4, info)
    with pytest.raises(sf.StepfactError):
        sf.chol_steps_colmajor(4, [], d, 4, d, 4, info)


@pytest.mark.parametrize("dtype", [0, 1])
def test_chol_cfg5_full_size_sampled(dtype):
    """BASELINE.json configs[4] at its full size, n = 65536, s = 512, in bench.py's launch
    configuration (single GPU, out of place): the first K columns of L (K = 3s fp64, 2s fp32,
    so flushed entries — incl. the first, out-of-place flush over 65024 rows — are compared
    elementwise) against the restricted oracle (bitwise the full oracle's first K columns),
    a Freivalds residual of the whole
    factor (torch fp64, an independent checker), info 0 and a positive diagonal.
    fp64 bar R2 <= 1e-10 / residual <= 1e-13 n; fp32 (3xTF32, the fp32-rounded input) 2e-4 /
    1e-5 n."""
    n, s = 65536, 512
    K = 1536 if dtype == 0 else 1024            # >= 3s (fp64) / 2s (fp32): flushed columns compared
    f1, f2 = flushed_cols(K, s)
    assert f1 >= s and (dtype == 1 or f2 >= s), (f1, f2)
    A = synth.gen_torch("spd_scaled", n, seed=0)
    if dtype == 1:
        A = A.float()
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    L = torch.empty_like(A)
    sf.chol_colmajor(n, s, A, n, L, n, info, dtype=dtype)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    Ak = np.asfortranarray(A[:K].double().cpu().numpy().T)        # first K columns (A symmetric)
    Lo, io = oracle.chol(Ak, s, kcols=K)
    assert io == 0
    Lk = L[:K].double().cpu().numpy().T                            # first K columns of L (column-major rows)
    Lk = np.tril(Lk)
    tol = TOL64 if dtype == 0 else 2e-4
    assert synth.r2_error(Lk, Lo[:, :K]) <= tol
    assert bool((torch.diagonal(L.mT) > 0).all())
    g = torch.Generator(device="cuda"); g.manual_seed(7)
    x = torch.randn(n, 2, device="cuda", dtype=torch.float64, generator=g)
    Ll = torch.tril(L.mT)
    Ad = A.double() if dtype == 1 else A
    y = Ll.double() @ (Ll.mT.double() @ x) if dtype == 1 else Ll @ (Ll.mT @ x)
    r = float((Ad @ x - y).norm() / (Ad @ x).norm())
    assert r <= (1e-13 if dtype == 0 else 1e-5) * n


@pytest.mark.timeout(300, method="thread")
def test_qr_concurrent_streams():
    """The MGS panel grid is persistent (its CTAs wait on each other).  Several QR calls on
    different streams at once must neither deadlock (DESIGN.md §5 K7: eager panel launches
    are chained per device) nor change a bit of each other's results."""
    n, s = 8192, 128
    A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    Q0, R0 = torch.empty_like(A), torch.empty_like(A)
    sf.qr_colmajor(n, s, A, n, Q0, n, R0, n, info)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    streams = [torch.cuda.Stream() for _ in range(3)]
    outs = []
    for st in streams:
        Q, R = torch.empty_like(A), torch.empty_like(A)
        inf = torch.zeros(1, dtype=torch.int64, device="cuda")
        torch.cuda.current_stream().synchronize()
        sf.qr_colmajor(n, s, A, n, Q, n, R, n, inf, stream=st)
        outs.append((Q, R, inf))
    torch.cuda.synchronize()
    for Q, R, inf in outs:
        assert int(inf.item()) == 0
        assert torch.equal(Q, Q0) and torch.equal(torch.triu(R), torch.triu(R0))


@pytest.mark.timeout(600, method="thread")
def test_qr_graph_replay_two_streams():
    """repeated same-argument QR calls on two streams replay captured graphs (eager,
    capture, replay per stream) that contain persistent MGS grids; replays on different streams
    are chained per device (driver.cu run_graph), so two grids that cannot be co-resident
    (n = 16384: 128 CTAs each) never spin-wait on each other.  Results stay bitwise stable."""
    n, s = 16384, 128
    A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [(torch.empty_like(A), torch.empty_like(A), torch.zeros(1, dtype=torch.int64, device="cuda"))
            for _ in streams]
    torch.cuda.synchronize()
    for it in range(3):                      # eager, capture, replay on each stream, interleaved
        for st, (Q, R, inf) in zip(streams, outs):
            sf.qr_colmajor(n, s, A, n, Q, n, R, n, inf, stream=st)
    torch.cuda.synchronize()
    (Q0, R0, i0), (Q1, R1, i1) = outs
    assert int(i0.item()) == int(i1.item()) == 0
    assert torch.equal(Q0, Q1) and torch.equal(torch.triu(R0), torch.triu(R1))


def test_host_wrappers_validate_buffers():
    """the host wrappers infer the element type and reject buffers whose dtype,
    shape or layout would make the library read or write past them (no compute happens)."""
    A = np.asfortranarray(np.eye(8))
    with pytest.raises(TypeError):
        sf.chol_host(A, 4, np.asfortranarray(np.eye(8, dtype=np.float32)))
    with pytest.raises(ValueError):
        sf.lu_host(np.ascontiguousarray(np.ones((8, 8)) + 7 * np.eye(8)), 4)   # row-major: would factor A^T
    with pytest.raises(ValueError):
        sf.qr_host(A, 4, np.asfortranarray(np.zeros((8, 7))), np.asfortranarray(np.zeros((8, 8))))
    with pytest.raises(TypeError):
        sf.chol_host(A, 4, dtype=sf.SF_F32)
    out, info = sf.chol_host(np.asfortranarray(4 * np.eye(8, dtype=np.float32)), 4)
    assert info == 0 and np.array_equal(np.tril(out), 2 * np.eye(8, dtype=np.float32))


def test_host_entry_points_pageable():
    """plain (pageable) numpy buffers are page-locked for the duration of the call,
    so the per-panel device->host copies stay asynchronous; results equal the device path."""
    n, s = 2048, 256
    A = synth.gen_numpy("spd_scaled", n, seed=8)
    out, info = sf.chol_host(np.asfortranarray(A.copy()), s)
    Lg, ig = run_chol(A, s, inplace=False)
    assert info == ig == 0 and np.array_equal(np.tril(out), np.tril(Lg))


@pytest.mark.parametrize("n,s", [(1500, 96), (16384, 128)])
def test_qr_mgs_cluster_geometries(n, s):
    """The MGS panel's grid changes with n (DESIGN.md §5 K7): one cluster of <= 8 CTAs
    (n <= 1024), 8-CTA clusters, 4-CTA clusters when 8-CTA ones do not all fit (n = 16384),
    with ragged last CTAs (n = 1500).  First K columns / rows against the restricted oracle,
    orthogonality and residual in full."""
    K = 2 * s
    A = synth.gen_numpy("gaussian", n, seed=7)
    Qg, Rg, ig = run_qr(A, s)
    Qo, Ro, io, _ = oracle.qr(A, s, kcols=K)
    assert io == ig == 0
    assert synth.r2_error(Qg[:, :K], Qo[:, :K]) <= TOL64
    assert synth.r2_error(Rg[:K, :], Ro[:K, :]) <= TOL64
    Qt = torch.from_numpy(Qg).cuda(); At = torch.from_numpy(A).cuda(); Rt = torch.from_numpy(Rg).cuda()
    assert float((Qt.mT @ Qt - torch.eye(n, device="cuda", dtype=torch.float64)).norm()) <= 1e-12 * n
    assert float((At - Qt @ Rt).norm() / At.norm()) <= 1e-13 * n


@pytest.mark.parametrize("n,s", [(300, 64), (4608, 256)])
def test_lu_host_overlapped_copies(n, s):
    """lu_factor_host returns each panel's L columns and U rows while later flushes run
    (DESIGN.md §6 e2e): the host result must equal the device entry point's bit for bit,
    both triangles, incl. a ragged last panel and (n = 4608) the lookahead stream."""
    B = synth.gen_numpy("diag_dominant", n, seed=n)
    out, info = sf.lu_host(np.asfortranarray(B.copy()), s)
    Lg, Ug, ig = run_lu(B, s)
    assert info == ig == 0
    assert np.array_equal(np.tril(out), Lg)
    assert np.array_equal(np.triu(out, 1) + np.eye(n), Ug)
    if n <= 300:
        Lo, Uo, _ = oracle.lu(B, s)
        assert synth.r2_error(np.triu(out, 1) + np.eye(n), Uo) <= TOL64


@pytest.mark.parametrize("n,s", [(300, 64), (2000, 128)])
def test_qr_host_overlapped_copies(n, s):
    """qr_factor_host returns each panel of Q while the factorization continues, then R:
    bitwise the device entry point's result (both are column-major host/device buffers)."""
    A = synth.gen_numpy("gaussian", n, seed=n + 1)
    hA = np.asfortranarray(A.copy())
    hQ = np.zeros((n, n), order="F")
    hR = np.zeros((n, n), order="F")
    hQ, hR, info = sf.qr_host(hA, s, hQ, hR)
    Qg, Rg, ig = run_qr(A, s)
    assert info == ig == 0
    assert np.array_equal(hQ, Qg) and np.array_equal(hR, Rg)


_LA_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1812_02056_b200 as sf, synth
n, s, dt = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
A = synth.gen_numpy("diag_dominant", n, seed=7)
dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
if dt == "f32":
    dA = dA.float()
out = torch.empty_like(dA)
info = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3):     # eager, graph capture, graph replay: all three must agree
    out.zero_()
    sf.lu_colmajor(n, s, dA, n, out, n, info, dtype=sf.SF_F32 if dt == "f32" else sf.SF_F64)
    torch.cuda.synchronize()
    np.save(sys.argv[5] + f"_{_}.npy", out.cpu().numpy())
assert int(info.item()) == 0
"""


@pytest.mark.parametrize("n,s,dt", [(4096, 64, "f64"), (1000, 96, "f64"), (2048, 64, "f32")])
def test_lu_two_deep_lookahead_bitwise(tmp_path, n, s, dt):
    """SF_LU_LA2 (default): the flush of panel p split into the next panel's L shape, the one
    after it, and the rest, on two streams — every element receives the same flushes in the
    same order from the same tile kernels, so the factor is BITWISE the one-deep scheme's
    (SF_LU_LA2=0) and the same on eager, captured and replayed calls."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for la2 in ("1", "0"):
        env = dict(os.environ, SF_LU_LA2=la2)
        base = str(tmp_path / f"la{la2}")
        subprocess.run([sys.executable, "-c", _LA_CHILD, root, str(n), str(s), dt, base], env=env, check=True)
        outs[la2] = [np.load(base + f"_{i}.npy") for i in range(3)]
    for i in range(3):
        assert np.array_equal(outs["1"][i], outs["0"][0]), i


@pytest.mark.parametrize("n,s", [(256, 1), (256, 4), (256, 16), (256, 32), (200, 8), (64, 2)])
def test_chol_small_cluster_planted_and_failure(n, s):
    """n <= 256, s | 32: the whole schedule runs in ONE thread-block cluster from shared
    memory (small.cu).  Planted integer factors come out exactly; an interior failed pivot
    stops every CTA with the oracle's info (R3); random SPD input meets the R2 bar."""
    Lx = synth.planted_chol(n, seed=n + s)
    Lg, info = run_chol(Lx @ Lx.T, s)
    assert info == 0 and np.array_equal(np.tril(Lg), Lx)
    B = synth.gen_numpy("paper_spd", n, seed=s)
    bad = (3 * n) // 4
    B[bad, bad] = -5.0
    io = oracle.chol(B, s)[1]
    assert io == bad + 1 and run_chol(B, s)[1] == io
    A = synth.gen_numpy("spd_shift", n, seed=s)
    Lo, _ = oracle.chol(A, s)
    for inplace in (True, False):
        Lg, ig = run_chol(A, s, inplace)
        assert ig == 0 and synth.r2_error(np.tril(Lg), Lo) <= TOL64
