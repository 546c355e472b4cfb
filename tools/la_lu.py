"""LU lookahead A/B at larger n (graph replay and eager)."""
import os, sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf, synth
info = torch.zeros(1, dtype=torch.int64, device='cuda')
def t(fn, reps=5):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]
la = os.environ.get("SF_LOOKAHEAD", "1"); g = os.environ.get("SF_GRAPH", "1")
for n, s in [(4096, 64), (4000, 200), (8192, 64), (8192, 256), (16384, 128)]:
    B = torch.from_numpy(synth.gen_numpy("diag_dominant", n, 0)).cuda().mT.contiguous(); O = torch.empty_like(B)
    print(f"LA={la} GRAPH={g} lu n={n} s={s}: {t(lambda: sf.lu_colmajor(n, s, B, n, O, n, info)):.2f} ms")
