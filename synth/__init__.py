"""Seeded synthetic inputs and verification metrics — shared by tests and bench only.

This module holds NONE of the factorization arithmetic: it builds input matrices with
the shapes and distributions of BASELINE.json's configs (and PAPER.md:189's "symmetric
one with random entries and large values in the diagonal") and computes error metrics on
finished outputs.  Both the CUDA path and the CPU oracle consume the *same bytes* from
here; neither imports the other.

Generators ("input recipe"):
  cfg1  G in R^{n x n} i.i.d. N(0,1), A = G G^T + n I                  (BASELINE.json:7)
  cfg2  A_ij i.i.d. U(-1,1), A_ii := 1 + sum_{j != i} |A_ij|           (BASELINE.json:8)
  cfg3/5 A = G G^T / n + I                                             (BASELINE.json:9, 11)
  cfg4  A_ij i.i.d. N(0,1)                                             (BASELINE.json:10)
  paper symmetric, off-diagonal U(-1,1), diagonal n + U(0,1)
Symmetric matrices are made exactly symmetric by mirroring the lower triangle, because a
library G G^T may round (i,j) and (j,i) differently.
"""
import numpy as np

KINDS = ("spd_shift", "diag_dominant", "spd_scaled", "gaussian", "paper_spd")


def gen_numpy(kind, n, seed):
    """Host (numpy PCG64) generator: bit-reproducible on any machine. Returns float64 (n,n)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "spd_shift":
        G = rng.standard_normal((n, n))
        A = G @ G.T + n * np.eye(n)
    elif kind == "spd_scaled":
        G = rng.standard_normal((n, n))
        A = G @ G.T / n + np.eye(n)
    elif kind == "diag_dominant":
        A = 2.0 * rng.random((n, n)) - 1.0
        off = np.abs(A).sum(axis=1) - np.abs(np.diag(A))
        A[np.arange(n), np.arange(n)] = 1.0 + off
        return A
    elif kind == "gaussian":
        return rng.standard_normal((n, n))
    elif kind == "paper_spd":
        A = 2.0 * rng.random((n, n)) - 1.0
        A[np.arange(n), np.arange(n)] = n + rng.random(n)
    else:
        raise ValueError(kind)
    return mirror_lower(A)


def mirror_lower(A):
    """A := tril(A) + tril(A,-1)^T, exactly symmetric."""
    L = np.tril(A)
    return L + np.tril(A, -1).T


def gen_torch(kind, n, seed, device="cuda", chunk=4096):
    """Device generator for sizes the host cannot form quickly (cfg3/cfg5).

    G is drawn in `chunk`-row blocks, block k from torch.Generator(device).manual_seed(
    seed * 1_000_003 + k) (BASELINE.json:11 "seeded 4096-row chunks"); A = G G^T (cuBLAS,
    fp64) then the kind's shift, mirrored to exact symmetry.  Returns a float64 tensor.
    """
    import torch

    def gauss(rows, k):
        g = torch.Generator(device=device)
        g.manual_seed(seed * 1_000_003 + k)
        return torch.randn(rows, n, generator=g, device=device, dtype=torch.float64)

    if kind in ("spd_shift", "spd_scaled"):
        A = torch.empty(n, n, device=device, dtype=torch.float64)
        blocks = [gauss(min(chunk, n - r), k) for k, r in enumerate(range(0, n, chunk))]
        G = torch.cat(blocks, 0)
        del blocks
        torch.matmul(G, G.T, out=A)
        del G
        if kind == "spd_scaled":
            A /= n
            A.diagonal().add_(1.0)
        else:
            A.diagonal().add_(float(n))
        # mirror lower -> upper in column blocks to bound temporary memory
        for c0 in range(0, n, chunk):
            c1 = min(n, c0 + chunk)
            # rows c0:c1 of the upper triangle come from columns c0:c1 of the lower
            blk = A[c0:, c0:c1].clone()          # lower part of these columns (rows >= c0)
            A[c0:c1, c0:] = blk.T                # write upper (and diagonal block) by transpose
            A[c0:, c0:c1] = blk                  # restore lower
            del blk
        # diagonal blocks: enforce tril + tril^T inside each block
        for c0 in range(0, n, chunk):
            c1 = min(n, c0 + chunk)
            D = A[c0:c1, c0:c1]
            A[c0:c1, c0:c1] = torch.tril(D) + torch.tril(D, -1).T
        return A
    if kind == "gaussian":
        return torch.cat([gauss(min(chunk, n - r), k) for k, r in enumerate(range(0, n, chunk))], 0)
    if kind == "diag_dominant":
        g = torch.Generator(device=device); g.manual_seed(seed)
        A = 2.0 * torch.rand(n, n, generator=g, device=device, dtype=torch.float64) - 1.0
        off = A.abs().sum(1) - A.diagonal().abs()
        A.diagonal().copy_(1.0 + off)
        return A
    raise ValueError(kind)


def gen_torch_cols(kind, n, seed, cols, device="cuda", chunk=4096):
    """Columns `cols` of the cfg3/cfg5 matrix (A = G G^T/n + I or G G^T + n I, G from the same
    seeded 4096-row chunks as gen_torch), as a COLUMN-MAJOR local buffer (len(cols), n):
    buf[jl, i] = A[i, cols[jl]].  For a rank of the block-cyclic layout this forms only its
    own columns (n x n x len(cols) flops instead of n^3).  The entries Alg. 1 reads (i >=
    column) are G[i].G[j] (/n) from one cuBLAS product; they may round differently from
    gen_torch's full product, i.e. the same recipe, not the same bytes."""
    import torch
    assert kind in ("spd_shift", "spd_scaled")

    def gauss(rows, k):
        g = torch.Generator(device=device)
        g.manual_seed(seed * 1_000_003 + k)
        return torch.randn(rows, n, generator=g, device=device, dtype=torch.float64)

    G = torch.cat([gauss(min(chunk, n - r), k) for k, r in enumerate(range(0, n, chunk))], 0)
    idx = torch.as_tensor(cols, device=device, dtype=torch.long)
    buf = torch.matmul(G[idx], G.T)                # (nloc, n): buf[jl, i] = G[cols[jl]] . G[i]
    del G
    if kind == "spd_scaled":
        buf /= n
        buf[torch.arange(len(cols), device=device), idx] += 1.0
    else:
        buf[torch.arange(len(cols), device=device), idx] += float(n)
    return buf


# ----------------------------------------------------------------------------- planted factors

def planted_chol(n, seed):
    """L with off-diagonal entries from {-1,0,1}, diagonal from {1,2,4}; A = L L^T exact.

    Every intermediate of any ordering of Alg. 1 is an integer below 2^24 (n <= 16384),
    each sqrt is of a perfect square, each division by a power of two, so every correct
    implementation (fp64 or 3xTF32 with R_lo = 0) returns L exactly.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    L = np.tril(rng.integers(-1, 2, size=(n, n)).astype(np.float64), -1)
    L[np.arange(n), np.arange(n)] = rng.choice([1.0, 2.0, 4.0], size=n)
    return L


def planted_lu(n, seed):
    """Crout factors: L lower (entries {-1,0,1}, diagonal {1,2,4}), U unit upper {-1,0,1}."""
    rng = np.random.Generator(np.random.PCG64(seed))
    L = planted_chol(n, seed)
    U = np.triu(rng.integers(-1, 2, size=(n, n)).astype(np.float64), 1) + np.eye(n)
    return L, U


def hadamard(n):
    """Sylvester Hadamard matrix H_n (n a power of two)."""
    H = np.array([[1.0]])
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    assert H.shape[0] == n, "n must be a power of two"
    return H


def planted_qr(n, seed):
    """Q = H_n / sqrt(n) for n = 4^k (exact dyadic), R0 integer upper with positive diagonal."""
    r = int(round(np.sqrt(n)))
    assert r * r == n and (n & (n - 1)) == 0, "n must be a power of 4"
    rng = np.random.Generator(np.random.PCG64(seed))
    Q = hadamard(n) / r
    R = np.triu(rng.integers(-2, 3, size=(n, n)).astype(np.float64), 1)
    R[np.arange(n), np.arange(n)] = rng.integers(1, 5, size=n).astype(np.float64)
    return Q, R


# ----------------------------------------------------------------------------- metrics

FLOOR_FRAC = 2.0 ** -10


def r2_error(x, y, floor_frac=FLOOR_FRAC):
    """Floored relative elementwise error (reading P6):

        max_ij |x_ij - y_ij| / max(|y_ij|, floor_frac * max_kl |y_kl|)

    The plain |x-y|/|y| explodes on tiny entries even between two correct fp64 runs.
    """
    x = np.asarray(x, dtype=np.float64); y = np.asarray(y, dtype=np.float64)
    if y.size == 0:
        return 0.0
    scale = np.max(np.abs(y))
    den = np.maximum(np.abs(y), floor_frac * scale)
    den = np.where(den == 0, 1.0, den)
    return float(np.max(np.abs(x - y) / den))


def rel_residual(A, *factors):
    """||A - prod(factors)||_F / ||A||_F (fp64, numpy)."""
    P = factors[0]
    for F in factors[1:]:
        P = P @ F
    return float(np.linalg.norm(A - P) / np.linalg.norm(A))


def orthogonality(Q):
    """||Q^T Q - I||_F."""
    return float(np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1])))


def classical_flops(kind, n):
    """Classical counts used for the headline metric (BASELINE.json:5)."""
    return {"chol": n ** 3 / 3.0, "lu": 2.0 * n ** 3 / 3.0, "qr": 4.0 * n ** 3 / 3.0}[kind]
