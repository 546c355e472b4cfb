"""L0 calibration: cuBLAS DGEMM / TF32 SGEMM / FP32 SGEMM throughput via torch (library reference points)."""
import json, torch, time
def bench(dtype, n, tf32=False, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype); b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3): torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * n**3 / (best * 1e-3) / 1e12
out = {"dgemm_8192_tflops": bench(torch.float64, 8192),
       "dgemm_16384_tflops": bench(torch.float64, 16384, reps=4),
       "tf32_8192_tflops": bench(torch.float32, 8192, tf32=True),
       "sgemm_8192_tflops": bench(torch.float32, 8192)}
# sustained DGEMM 4 s
torch.backends.cuda.matmul.allow_tf32 = False
a = torch.randn(8192, 8192, device="cuda", dtype=torch.float64); b = torch.randn_like(a)
torch.cuda.synchronize(); t0 = time.time(); k = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b); k += 1
    if k % 4 == 0: torch.cuda.synchronize()
e1.record(); e1.synchronize()
out["dgemm_8192_sustained_tflops"] = 2 * 8192**3 * k / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(json.dumps(out))
