"""K1s — the chunked short-K DMMA flush (gemm_f64.cu `gemm_f64_chunk_kernel`).

The LU flush at s = 64 (A[c:n, c:n] -= R_L R_U, K = s) runs on CTAs that
each own a chunk of consecutive 128x64 tiles of one row block.  It must be (1) correct
against the plain product (fp64 bar) and (2) BITWISE the result of the one-tile-per-CTA
short-K kernel it replaces (same DMMA chain per element), on ragged and K < 64 shapes,
chunked (many tiles per CTA) and single-tile; forced on/off by SF_DMMA_CHUNK in child
processes (the switches are read once per process).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_1812_02056_b200 as sf
m, n, k, seed = (int(x) for x in sys.argv[2:6])
rng = np.random.default_rng(seed)
A = rng.uniform(-1, 1, (m, k)); B = rng.uniform(-1, 1, (k, n)); C = rng.uniform(-1, 1, (m, n))
dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()      # column-major m x k, ld = m
dB = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()      # column-major k x n, ld = k (k-contiguous)
dC = torch.from_numpy(np.ascontiguousarray(C.T)).cuda()
for _ in range(2):   # twice: the second call reuses the launch state
    if _ == 1:
        dC.copy_(torch.from_numpy(np.ascontiguousarray(C.T)))
    assert sf.lib().sf_gemm_sub(m, n, k, 0, dA.data_ptr(), m, 0, dB.data_ptr(), k, 0, dC.data_ptr(), m, None) == 0
    torch.cuda.synchronize()
np.save(sys.argv[6], dC.cpu().numpy().T)
"""

# (m, n, k): the LU cfg2 flush shape, ragged rows / columns, K < 64, single-tile chunks
SHAPES = [(3968, 3968, 64), (2050, 1001, 64), (1538, 3001, 40), (4096, 130, 64), (130, 4100, 8), (640, 640, 64)]


def _run(tmp_path, shape, env_extra, tag):
    m, n, k = shape
    out = str(tmp_path / f"{tag}.npy")
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, "-c", _CHILD, ROOT, str(m), str(n), str(k), "7", out], env=env, check=True)
    return np.load(out)


@pytest.mark.parametrize("shape", SHAPES)
def test_chunk_flush_matches_plain_and_is_bitwise(tmp_path, shape):
    m, n, k = shape
    got = _run(tmp_path, shape, {"SF_DMMA_CHUNK": "1", "SF_DMMA_CHUNK_MIN": "1"}, "chunk")
    base = _run(tmp_path, shape, {"SF_DMMA_CHUNK": "0"}, "plain")
    rng = np.random.default_rng(7)
    A = rng.uniform(-1, 1, (m, k)); B = rng.uniform(-1, 1, (k, n)); C = rng.uniform(-1, 1, (m, n))
    ref = C - A @ B
    # fp64: |error| <= k * u * sum|a||b| + u|c| <= 2 k u (entries in [-1, 1])
    assert np.abs(got - ref).max() <= 2 * k * np.finfo(np.float64).eps * 4
    assert np.array_equal(got, base)


@pytest.mark.parametrize("chunk", ["1", "3", "16"])
def test_chunk_flush_fixed_chunk_lengths(tmp_path, chunk):
    """Chunk length 1 (no reuse), 3 (ragged last chunk of a row), 16 (long chunks, both B
    buffers recycled many times): bitwise the plain kernel."""
    shape = (1024, 2000, 64)
    got = _run(tmp_path, shape, {"SF_DMMA_CHUNK": "1", "SF_DMMA_CHUNK_MIN": "1", "SF_DMMA_CHUNK_T": chunk}, "c")
    base = _run(tmp_path, shape, {"SF_DMMA_CHUNK": "0"}, "p")
    assert np.array_equal(got, base)
