"""Variable step sequences at cfg3 (Cholesky n=16384) and cfg5-size: time a few
tapers against fixed s=512.  Median of 5 after 2 warm-ups, CUDA events."""
import statistics, sys, torch
sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = synth.gen_torch("spd_scaled", n, 0)
L = torch.empty_like(A); info = torch.zeros(1, dtype=torch.int64, device="cuda")
def seq(big, tail):   # big steps, then halve in the last `tail` columns
    out, z = [], 0
    while z < n:
        rem = n - z
        s = big
        for t, w in tail:
            if rem <= t: s = w
        out.append(s); z += s
    return out
cands = {"fixed512": [512], "fixed256": [256],
         "512->256@4096->128@1024": seq(512, [(4096, 256), (1024, 128)]),
         "512->256@2048": seq(512, [(2048, 256)]),
         "1024->512@8192->256@2048": seq(1024, [(8192, 512), (2048, 256)]),
         "768->512@8192->256@2048->128@512": seq(768, [(8192, 512), (2048, 256), (512, 128)])}
for name, st in cands.items():
    ts = []
    for it in range(7):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); sf.chol_steps_colmajor(n, st, A, n, L, n, info); e1.record(); torch.cuda.synchronize()
        if it >= 2: ts.append(e0.elapsed_time(e1))
    assert int(info.item()) == 0
    ms = statistics.median(ts)
    print(f"n={n} {name:36s} {ms:8.2f} ms  {n**3/3/ms/1e9:8.1f} TF/s  panels={len(st) if len(st) > 1 else -(-n // st[0])}")
