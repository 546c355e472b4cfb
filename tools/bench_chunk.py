"""Time C -= A B (K = 64, in place; the LU s = 64 flush shape) through sf_gemm_sub for a few
m, with whatever SF_DMMA_CHUNK* switches the environment sets.  CUDA events, median of 20.
    SF_DMMA_CHUNK=0 python tools/bench_chunk.py ; SF_DMMA_CHUNK=1 python tools/bench_chunk.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_02056_b200 as sf  # noqa: E402

k = int(os.environ.get("K", "64"))
for m in (4032, 3008, 2048, 1024):
    A = torch.randn(k, m, device="cuda", dtype=torch.float64)   # column-major m x k
    B = torch.randn(m, k, device="cuda", dtype=torch.float64)   # column-major k x m (k-contiguous)
    C = torch.randn(m, m, device="cuda", dtype=torch.float64)
    ts = []
    for it in range(25):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        sf.lib().sf_gemm_sub(m, m, k, 0, A.data_ptr(), m, 0, B.data_ptr(), k, 0, C.data_ptr(), m,
                             torch.cuda.current_stream().cuda_stream)
        e1.record(); torch.cuda.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    t = ts[len(ts) // 2]
    print(f"m={m} k={k} chunk={os.environ.get('SF_DMMA_CHUNK', '1')} T={os.environ.get('SF_DMMA_CHUNK_T', 'auto')}: "
          f"{t * 1e3:.1f} us  {2 * m * m * k / t / 1e9:.2f} TF/s")
