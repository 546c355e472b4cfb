"""One eager factorization of a BASELINE config (for ncu -k/-s/-c captures of its kernels).
    python tools/prof_fact.py lu 4096 64 | qr 8192 128 | chol 16384 512  [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_02056_b200 as sf  # noqa: E402
import synth  # noqa: E402

kind, n, s = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
os.environ.setdefault("SF_GRAPH", "0")
gen = {"chol": "spd_scaled", "lu": "diag_dominant", "qr": "gaussian"}[kind]
A = synth.gen_torch(gen, n, seed=0)
if kind != "chol":
    A = A.mT.contiguous()
o1 = torch.empty_like(A); o2 = torch.empty_like(A)
info = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(reps):
    if kind == "chol":
        sf.chol_colmajor(n, s, A, n, o1, n, info)
    elif kind == "lu":
        sf.lu_colmajor(n, s, A, n, o1, n, info)
    else:
        sf.qr_colmajor(n, s, A, n, o1, n, o2, n, info)
torch.cuda.synchronize()
assert int(info.item()) == 0
print("ok")
