"""Measurement sweep for profiles/ (run on the GPU box):
  * every BASELINE config: device time per factorization, classical GFLOP/s, % of peak,
    update/panel split from the library's profiling hook;
  * the cfg3 s-sweep (s in 64, 128, 168, 169, 256, 512, 1024);
  * the paper's six (algorithm, n, s) CPU timings re-run on one B200.
Median of 5 timed runs after 2 warm-ups, CUDA events on the launching stream; out of place.
    python tools/measure_all.py [configs|sweep|paper|all] > gpurun_out/measure.json
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_1812_02056_b200 as sf  # noqa: E402
import synth  # noqa: E402
from bench import ClockSampler  # noqa: E402

PEAK64 = json.load(open("calib/peaks_fp64_tf32.json"))["fp64_dmma_tflops"]
MP = json.load(open("MEASURED_PEAKS.json")) if __import__("os").path.exists("MEASURED_PEAKS.json") else {}
PEAK_TF32 = MP.get("bf16_tflops_sustained", 1400.0) * 1.1 / 2.25
CLASSICAL = {"chol": lambda n: n ** 3 / 3, "lu": lambda n: 2 * n ** 3 / 3, "qr": lambda n: 4 * n ** 3 / 3}


def run(kind, n, s, A, dtype=sf.SF_F64, reps=5, warm=2):
    st = torch.cuda.current_stream()
    info = torch.zeros(1, dtype=torch.int64, device="cuda")
    o1 = torch.empty_like(A)
    o2 = torch.empty_like(A) if kind == "qr" else None

    def once():
        if kind == "chol":
            sf.chol_colmajor(n, s, A, n, o1, n, info, dtype=dtype, stream=st)
        elif kind == "lu":
            sf.lu_colmajor(n, s, A, n, o1, n, info, dtype=dtype, stream=st)
        else:
            sf.qr_colmajor(n, s, A, n, o1, n, o2, n, info, dtype=dtype, stream=st)
    for _ in range(warm):
        once()
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    ts = []
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", 0)))
    clocks.start()
    for _ in range(reps):      # timed: no profiling hook, so repeated calls replay a CUDA graph
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); once(); e1.record(st); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ck = clocks.stop()
    sf.profile_enable(True)    # one extra, profiled (eager) run for the update / panel split
    sf.profile_collect()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); once(); e1.record(st); torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1)
    prof = sf.profile_collect()
    sf.profile_enable(False)
    reps = 1
    ms = statistics.median(ts)
    fl = CLASSICAL[kind](n)
    peak = PEAK_TF32 if dtype == sf.SF_F32 else PEAK64
    up_ms, up_n, up_fl = prof["update"]
    pan_ms = prof["panel"][0] / reps
    r_ms, _, r_fl = prof["qr_r"]
    out = {"kind": kind, "n": n, "s": s, "dtype": "f32" if dtype == sf.SF_F32 else "f64", "ms": ms,
           "ms_all": ts, "eager_profiled_ms": eager_ms, "gflops": fl / ms / 1e6, "pct_peak": fl / ms / 1e9 / peak,
           "update_ms": up_ms / reps, "update_tflops": (up_fl / (up_ms * 1e-3) / 1e12) if up_ms else None,
           "panel_ms": pan_ms, "clocks": ck,
           # the main (flush) stream is busy update_ms of the eager step; the rest of the step
           # is panel work the lookahead did not hide
           "exposed_panel_ms": max(0.0, eager_ms - up_ms / reps - (prof["qr_r"][0] / reps))}
    if kind == "qr":
        out["R_ms"] = r_ms / reps
        out["R_tflops"] = r_fl / (r_ms * 1e-3) / 1e12 if r_ms else None
        out["algorithmic_tflops"] = (up_fl + r_fl) / reps / (ms * 1e-3) / 1e12
    return out


def colmajor(Alog):
    return Alog.mT.contiguous()


def configs():
    res = []
    A = torch.from_numpy(synth.gen_numpy("spd_shift", 256, 0)).cuda()
    res.append(run("chol", 256, 16, A) | {"config": "configs[0]"})
    A = colmajor(torch.from_numpy(synth.gen_numpy("diag_dominant", 4096, 0)).cuda())
    res.append(run("lu", 4096, 64, A) | {"config": "configs[1]"})
    res.append(run("lu", 4096, 64, A.float(), dtype=sf.SF_F32) | {"config": "configs[1] fp32"})
    A = synth.gen_torch("spd_scaled", 16384, 0)
    res.append(run("chol", 16384, 512, A) | {"config": "configs[2] s=512"})
    res.append(run("chol", 16384, 512, A.float(), dtype=sf.SF_F32) | {"config": "configs[2] s=512, fp32"})
    del A
    A = colmajor(synth.gen_torch("gaussian", 8192, 0))
    res.append(run("qr", 8192, 128, A) | {"config": "configs[3]"})
    res.append(run("qr", 8192, 128, A.float(), dtype=sf.SF_F32) | {"config": "configs[3] fp32"})
    del A
    torch.cuda.empty_cache()
    A = synth.gen_torch("spd_scaled", 65536, 0)
    res.append(run("chol", 65536, 512, A, reps=3) | {"config": "configs[4] fp64"})
    A32 = A.float(); del A; torch.cuda.empty_cache()
    res.append(run("chol", 65536, 512, A32, dtype=sf.SF_F32, reps=3) | {"config": "configs[4] fp32"})
    return res


def sweep():
    A = synth.gen_torch("spd_scaled", 16384, 0)
    return [run("chol", 16384, s, A) | {"config": f"configs[2] s-sweep"} for s in (64, 128, 168, 169, 256, 512, 1024, 2048, 4096)]


def paper():
    # n, s, the paper's CPU seconds and GSL seconds
    rows = [("chol", 2000, 200, 1.14867, 2.28978), ("chol", 4000, 400, 8.99871, 17.0262),
            ("lu", 2000, 200, 1.51041, 3.53489), ("lu", 4000, 200, 12.203, 28.7355),
            ("qr", 2000, 100, 7.12522, 51.8309), ("qr", 4000, 200, 64.3856, 554.165)]
    res = []
    for kind, n, s, tp, tg in rows:
        A = synth.gen_numpy("paper_spd", n, 0)      # "symmetric, random entries, large diagonal"
        Ad = torch.from_numpy(A).cuda()
        r = run(kind, n, s, Ad if kind == "chol" else colmajor(Ad))
        r.update({"config": "paper context PAPER.md:189-192", "paper_cpu_s": tp, "gsl_cpu_s": tg,
                  "speedup_vs_paper_cpu": tp / (r["ms"] * 1e-3)})
        res.append(r)
    return res


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    out = {"gpu": torch.cuda.get_device_name(0), "peak_fp64_tflops": PEAK64, "peak_tf32_tflops": PEAK_TF32}
    if what in ("configs", "all"):
        out["configs"] = configs()
    if what in ("sweep", "all"):
        out["sweep"] = sweep()
    if what in ("paper", "all"):
        out["paper"] = paper()
    print(json.dumps(out, indent=1))
