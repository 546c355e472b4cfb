"""GPU parity of the block-cyclic multi-GPU drivers.

One B200 is available, so the distributed schedule is exercised through a LOOPBACK
communicator (include/stepfact.h): one process drives all G ranks, each with its own
local buffers and streams, the panel broadcast a device copy — the same per-rank code,
events and lookahead as the NCCL path.  The NCCL path itself runs at G=1 (a real NCCL
communicator, broadcast and all-reduce included).

Bars: Cholesky distributed == single-GPU bit for bit (same per-element arithmetic, see
dist.cu); all three against the CPU oracle at the fp64 bar (R2 <= 1e-10, residual,
QR tail rule) — DESIGN.md §3 P6/P7.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1812_02056_b200 as sf  # noqa: E402
from tests.test_parity_gpu import EPS, TOL64, check_qr, dev, host, run_chol  # noqa: E402


def run_dist(kind, A, s, G, comm=None, inplace=False, dtype=None):
    n = A.shape[0]
    B = dev(A)                                   # column-major buffer
    if dtype == sf.SF_F32:
        B = B.float()
    own = comm is None
    comm = comm or sf.Comm.loopback(G)
    try:
        ranks = comm.local_ranks
        Aloc = [sf.scatter_cyclic(B, n, s, G, r) for r in ranks]
        Aref = [a.clone() for a in Aloc]
        info = [torch.full((1,), -1, dtype=torch.int64, device="cuda") for _ in ranks]
        if kind == "qr":
            Q = [torch.full_like(a, 5.0) for a in Aloc]
            R = [torch.full_like(a, 3.0) for a in Aloc]
            sf.qr_dist(comm, n, s, Aloc, Q, R, n, info, dtype=sf.SF_F64 if dtype is None else dtype)
            torch.cuda.synchronize()
            for a, b in zip(Aloc, Aref):
                assert torch.equal(a, b), "QR input modified"
            outs = (Q, R)
        else:
            X = Aloc if inplace else [torch.full_like(a, 7.0) for a in Aloc]
            (sf.chol_dist if kind == "chol" else sf.lu_dist)(comm, n, s, Aloc, X, n, info,
                                                             dtype=sf.SF_F64 if dtype is None else dtype)
            torch.cuda.synchronize()
            if not inplace:
                for a, b in zip(Aloc, Aref):
                    assert torch.equal(a, b), "out-of-place input modified"
            outs = (X,)
        infos = [int(i.item()) for i in info]
        assert len(set(infos)) == 1, infos
        full = []
        for X in outs:
            Y = torch.zeros_like(B)
            sf.gather_cyclic(X, n, s, G, Y)
            full.append(host(Y.double()))
        return full, infos[0]
    finally:
        if own:
            comm.destroy()


CASES = [(1, 1, 1), (5, 2, 2), (64, 16, 2), (130, 32, 3), (257, 64, 2), (300, 64, 4), (300, 100, 8),
         (520, 128, 3), (1000, 168, 4), (96, 96, 2)]


@pytest.mark.parametrize("n,s,G", CASES)
def test_chol_dist_loopback(n, s, G):
    A = synth.gen_numpy("paper_spd", n, seed=n + G)
    (Lg,), info = run_dist("chol", A, s, G)
    assert info == 0
    Lo, io = oracle.chol(A, s)
    assert io == 0
    assert synth.r2_error(np.tril(Lg), Lo) <= TOL64
    # untouched strict upper (out of place: the 7.0 fill survives)
    assert np.all(Lg[np.triu_indices(n, 1)] == 7.0)
    # bitwise equal to the single-GPU driver
    L1, _ = run_chol(A, s, inplace=False)
    assert np.array_equal(np.tril(Lg), np.tril(L1))


@pytest.mark.parametrize("n,s,G", [(300, 64, 2), (1000, 128, 4)])
def test_chol_dist_inplace_and_planted(n, s, G):
    Lx = synth.planted_chol(n, seed=n + s)
    (Lg,), info = run_dist("chol", Lx @ Lx.T, s, G, inplace=True)
    assert info == 0 and np.array_equal(np.tril(Lg), Lx)


def test_chol_dist_not_pd_info():
    B = synth.gen_numpy("paper_spd", 300, seed=3)
    B[200, 200] = -5.0
    io = oracle.chol(B, 64)[1]
    for G in (1, 2, 3):
        assert run_dist("chol", B, 64, G)[1] == io == 201


@pytest.mark.parametrize("n,s,G", CASES)
def test_lu_dist_loopback(n, s, G):
    A = synth.gen_numpy("diag_dominant", n, seed=n + G)
    (F,), info = run_dist("lu", A, s, G)
    assert info == 0
    Lo, Uo, io = oracle.lu(A, s)
    Lg, Ug = np.tril(F), np.triu(F, 1) + np.eye(n)
    assert synth.r2_error(Lg, Lo) <= TOL64 and synth.r2_error(Ug, Uo) <= TOL64
    assert synth.rel_residual(A, Lg, Ug) <= 1e-13 * n


def test_lu_dist_planted_and_info():
    n, s = 700, 64
    Lx, Ux = synth.planted_lu(n, seed=3)
    (F,), info = run_dist("lu", Lx @ Ux, s, 3)
    assert info == 0 and np.array_equal(np.tril(F), Lx) and np.array_equal(np.triu(F, 1) + np.eye(n), Ux)
    A = np.array([[0.0, 1.0], [1.0, 1.0]])          # SPEC.md:485 zero pivot
    assert run_dist("lu", A, 1, 2)[1] == 1


@pytest.mark.parametrize("n,s,G", [(1, 1, 1), (64, 16, 2), (130, 32, 3), (257, 64, 2), (300, 64, 4), (520, 128, 3)])
def test_qr_dist_loopback(n, s, G):
    A = synth.gen_numpy("gaussian", n, seed=n + G)
    (Qg, Rg), info = run_dist("qr", A, s, G)
    assert info == 0
    Qo, Ro, io, _ = oracle.qr(A, s)
    check_qr(A, s, Qg, Rg, Qo, Ro)


def test_qr_dist_planted():
    n, s = 1024, 128
    Qx, Rx = synth.planted_qr(n, seed=7)
    (Qg, Rg), info = run_dist("qr", Qx @ Rx, s, 2)
    assert info == 0 and np.array_equal(Qg, Qx) and np.array_equal(Rg, Rx)


def test_nccl_comm_single_rank():
    """The real NCCL transport (one rank): broadcast + all-reduce through NCCL."""
    uid = sf.unique_id()
    comm = sf.Comm.nccl(1, 0, uid)
    try:
        A = synth.gen_numpy("spd_scaled", 600, seed=1)
        (Lg,), info = run_dist("chol", A, 128, 1, comm=comm)
        assert info == 0
        L1, _ = run_chol(A, 128, inplace=False)
        assert np.array_equal(np.tril(Lg), np.tril(L1))
        B = synth.gen_numpy("diag_dominant", 500, seed=2)
        (F,), info = run_dist("lu", B, 96, 1, comm=comm)
        Lo, Uo, _ = oracle.lu(B, 96)
        assert info == 0 and synth.r2_error(np.tril(F), Lo) <= TOL64
        C = synth.gen_numpy("gaussian", 300, seed=3)
        (Qg, Rg), info = run_dist("qr", C, 64, 1, comm=comm)
        Qo, Ro, _, _ = oracle.qr(C, 64)
        assert info == 0
        check_qr(C, 64, Qg, Rg, Qo, Ro)
    finally:
        comm.destroy()


def test_chol_dist_cfg5_shape_sampled():
    """cfg5's layout (s=512, G=8 ranks) at n=8192 on one GPU: the distributed factor equals
    the single-GPU factor bit for bit and its first columns match the oracle."""
    n, s, G, K = 8192, 512, 8, 1536   # K = 3s: flushed columns of ranks 1 and 2 compared
    A = synth.gen_torch("spd_scaled", n, seed=0)
    An = A.cpu().numpy()
    (Lg,), info = run_dist("chol", An, s, G)
    assert info == 0
    L1, _ = run_chol(An, s, inplace=False)
    assert np.array_equal(np.tril(Lg), np.tril(L1))
    Lo, io = oracle.chol(np.asfortranarray(An[:, :K]), s, kcols=K)
    assert io == 0 and synth.r2_error(np.tril(Lg)[:, :K], Lo[:, :K]) <= TOL64


@pytest.mark.parametrize("n,s,G", [(64, 16, 2), (300, 64, 4), (1000, 168, 3), (2048, 512, 2), (4096, 512, 8)])
def test_chol_dist_fp32_loopback(n, s, G):
    """fp32 (3xTF32) distributed Cholesky: against the fp64 oracle on the fp32-rounded input
    (reading P9, R2 <= 2e-4) and equal to the single-GPU fp32 factor."""
    A = synth.gen_numpy("spd_scaled", n, seed=n + G).astype(np.float32).astype(np.float64)
    (Lg,), info = run_dist("chol", A, s, G, dtype=sf.SF_F32)
    assert info == 0
    Lo, io = oracle.chol(A, s)
    Lg = np.tril(Lg)
    assert synth.r2_error(Lg, Lo) <= 2e-4
    assert synth.rel_residual(A, Lg, Lg.T) <= 1e-5 * n
    B32 = torch.from_numpy(np.ascontiguousarray(A.T)).float().cuda()
    L1 = torch.full_like(B32, 7.0)
    info1 = torch.zeros(1, dtype=torch.int64, device="cuda")
    sf.chol_colmajor(n, s, B32, n, L1, n, info1, dtype=sf.SF_F32)
    torch.cuda.synchronize()
    L1 = np.tril(L1.double().cpu().numpy().T)
    assert np.array_equal(Lg, L1)


def test_chol_dist_fp32_planted():
    n, s = 1024, 128
    Lx = synth.planted_chol(n, seed=5)
    (Lg,), info = run_dist("chol", Lx @ Lx.T, s, 3, dtype=sf.SF_F32)
    assert info == 0 and np.array_equal(np.tril(Lg), Lx)


def test_qr_dist_cfg4_shape_sampled():
    """BASELINE configs[3] (QR n=8192, s=128) on G=2 loopback ranks: the first K columns of Q
    and rows of R against the restricted oracle, orthogonality and residual of the whole."""
    n, s, G, K = 8192, 128, 2, 256
    A = synth.gen_numpy("gaussian", n, seed=0)
    (Qg, Rg), info = run_dist("qr", A, s, G)
    assert info == 0
    Qo, Ro, io, _ = oracle.qr(A, s, kcols=K)
    assert io == 0
    assert synth.r2_error(Qg[:, :K], Qo[:, :K]) <= TOL64
    assert synth.r2_error(Rg[:K, :], Ro[:K, :]) <= TOL64
    Qt = torch.from_numpy(Qg).cuda(); At = torch.from_numpy(A).cuda(); Rt = torch.from_numpy(Rg).cuda()
    assert float((Qt.mT @ Qt - torch.eye(n, device="cuda", dtype=torch.float64)).norm()) <= 1e-12 * n
    assert float((At - Qt @ Rt).norm() / At.norm()) <= 1e-13 * n
    assert np.all(np.tril(Rg, -1) == 0)


def test_lu_dist_cfg2_shape():
    """BASELINE configs[1] (LU n=4096, s=64) on G=2 and G=4 loopback ranks against the
    oracle."""
    n, s = 4096, 64
    A = synth.gen_numpy("diag_dominant", n, seed=0)
    Lo, Uo, io = oracle.lu(A, s)
    for G in (2, 4):
        (F,), info = run_dist("lu", A, s, G)
        assert info == 0
        Lg, Ug = np.tril(F), np.triu(F, 1) + np.eye(n)
        assert synth.r2_error(Lg, Lo) <= TOL64 and synth.r2_error(Ug, Uo) <= TOL64


@pytest.mark.parametrize("G", [1, 2, 3])
def test_lu_qr_dist_fp32(G):
    """fp32 (3xTF32) distributed LU and QR: planted integer factors come out exactly, and a
    random LU matches the fp64 oracle on the fp32-rounded input (R2 <= 2e-4)."""
    n, s = 512, 64
    Lx, Ux = synth.planted_lu(n, seed=11)
    (F,), info = run_dist("lu", Lx @ Ux, s, G, dtype=sf.SF_F32)
    assert info == 0 and np.array_equal(np.tril(F), Lx) and np.array_equal(np.triu(F, 1) + np.eye(n), Ux)
    A = synth.gen_numpy("diag_dominant", 300, seed=G).astype(np.float32).astype(np.float64)
    (F,), info = run_dist("lu", A, 64, G, dtype=sf.SF_F32)
    Lo, Uo, _ = oracle.lu(A, 64)
    assert info == 0 and synth.r2_error(np.tril(F), Lo) <= 2e-4 and synth.r2_error(np.triu(F, 1) + np.eye(300), Uo) <= 2e-4
    Qx, Rx = synth.planted_qr(256, seed=5)
    (Qg, Rg), info = run_dist("qr", Qx @ Rx, 64, G, dtype=sf.SF_F32)
    assert info == 0 and np.array_equal(Qg, Qx) and np.array_equal(Rg, Rx)


@pytest.mark.parametrize("kind,n,s,G", [("chol", 1000, 128, 3), ("lu", 1000, 128, 3), ("chol", 2048, 512, 2),
                                        ("lu", 777, 100, 4), ("qr", 600, 128, 2)])
def test_dist_bcast_bytes_packed(kind, n, s, G):
    """The panel messages carry only what the flush needs: Cholesky / LU send
    rows [p*s, n) of panel p packed, (n - p*s) * w_p elements, and never the last panel
    (it is not flushed); QR sends whole Q panels (the projections run over all
    rows).  The count is asserted exactly, and the factor still equals the
    single-GPU one bit for bit (Cholesky) / matches the oracle."""
    gen = {"chol": "spd_scaled", "lu": "diag_dominant", "qr": "gaussian"}[kind]
    A = synth.gen_numpy(gen, n, seed=n + G)
    P = -(-n // s)
    if kind == "qr":
        want = sum(n * min(s, n - p * s) for p in range(P)) * 8
    else:
        want = sum((n - p * s) * min(s, n - p * s) for p in range(P - 1)) * 8
    comm = sf.Comm.loopback(G)
    try:
        b0 = comm.bcast_bytes()
        outs, info = run_dist(kind, A, s, G, comm=comm)
        assert info == 0
        assert comm.bcast_bytes() - b0 == want
    finally:
        comm.destroy()
    if kind == "chol":
        L1, _ = run_chol(A, s, inplace=False)
        assert np.array_equal(np.tril(outs[0]), np.tril(L1))
    elif kind == "lu":
        Lo, Uo, _ = oracle.lu(A, s)
        F = outs[0]
        assert synth.r2_error(np.tril(F), Lo) <= TOL64 and synth.r2_error(np.triu(F, 1) + np.eye(n), Uo) <= TOL64


# ---------------------------------------------------------------- f3: device-initiated push

PUSH_CASES = [(1, 1, 1), (64, 16, 2), (300, 64, 4), (300, 100, 8), (520, 128, 3), (1000, 168, 4), (2048, 512, 5)]


@pytest.mark.parametrize("n,s,G", PUSH_CASES)
def test_chol_dist_push_bitwise(n, s, G):
    """sf_comm_set_push: the owner's ONE push kernel stores the packed
    panel into every rank's buffer and raises their ready flags; receivers wait on the
    device, signal `consumed` after the flush.  Same bytes on the wire (counted), same
    operands: the factor is bitwise the broadcast's and the single GPU's (fp64 and fp32)."""
    A = synth.gen_numpy("paper_spd", n, seed=n + G)
    L1, _ = run_chol(A, s, inplace=False)
    for dtype in (sf.SF_F64, sf.SF_F32):
        outs = {}
        for push in (False, True):
            comm = sf.Comm.loopback(G)
            try:
                comm.set_push(push)
                b0 = comm.bcast_bytes()
                (Lg,), info = run_dist("chol", A, s, G, comm=comm, dtype=dtype)
                assert info == 0
                outs[push] = (Lg, comm.bcast_bytes() - b0)
            finally:
                comm.destroy()
        assert np.array_equal(outs[True][0], outs[False][0]) and outs[True][1] == outs[False][1]
        if dtype == sf.SF_F64:
            assert np.array_equal(np.tril(outs[True][0]), np.tril(L1))


@pytest.mark.parametrize("n,s,G", PUSH_CASES)
def test_lu_dist_push_bitwise(n, s, G):
    A = synth.gen_numpy("diag_dominant", n, seed=n + G)
    outs = {}
    for push in (False, True):
        comm = sf.Comm.loopback(G)
        try:
            comm.set_push(push)
            (F,), info = run_dist("lu", A, s, G, comm=comm)
            assert info == 0
            outs[push] = F
        finally:
            comm.destroy()
    assert np.array_equal(outs[True], outs[False])
    Lo, Uo, _ = oracle.lu(A, s)
    assert synth.r2_error(np.tril(outs[True]), Lo) <= TOL64


def test_push_failure_and_repeated_calls():
    """A failed pivot under the push transport: every rank reports the oracle's column and no
    rank waits forever on a flag; the same communicator then serves further calls (the flag
    tags grow per call, so stale flags never release a wait)."""
    comm = sf.Comm.loopback(3)
    try:
        comm.set_push(True)
        B = synth.gen_numpy("paper_spd", 300, seed=3)
        B[200, 200] = -5.0
        io = oracle.chol(B, 64)[1]
        assert run_dist("chol", B, 64, 3, comm=comm)[1] == io == 201
        A = synth.gen_numpy("paper_spd", 300, seed=4)
        L1, _ = run_chol(A, 64, inplace=False)
        for _ in range(3):
            (Lg,), info = run_dist("chol", A, 64, 3, comm=comm)
            assert info == 0 and np.array_equal(np.tril(Lg), np.tril(L1))
    finally:
        comm.destroy()


def test_nccl_push_single_rank():
    """The push transport on a real NCCL communicator (one rank): the receive buffers and
    flags live in a symmetric window (ncclMemAlloc + ncclCommWindowRegister), the push kernel
    addresses them through the window's load/store pointer; repeated calls reuse it."""
    uid = sf.unique_id()
    comm = sf.Comm.nccl(1, 0, uid)
    try:
        comm.set_push(True)
        A = synth.gen_numpy("spd_scaled", 600, seed=1)
        L1, _ = run_chol(A, 128, inplace=False)
        for _ in range(2):
            (Lg,), info = run_dist("chol", A, 128, 1, comm=comm)
            assert info == 0 and np.array_equal(np.tril(Lg), np.tril(L1))
        B = synth.gen_numpy("diag_dominant", 500, seed=2)
        (F,), info = run_dist("lu", B, 96, 1, comm=comm)
        Lo, Uo, _ = oracle.lu(B, 96)
        assert info == 0 and synth.r2_error(np.tril(F), Lo) <= TOL64
    finally:
        comm.destroy()
