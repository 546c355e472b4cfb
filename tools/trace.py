"""Kernel timeline of one factorization (torch.profiler / CUPTI: start, duration and stream of
every kernel, concurrency preserved — unlike ncu's serialized replay).

    python tools/trace.py lu 4096 64 [f64|f32] [--steps-shown 3]
Prints per-kernel totals, per-stream busy time and the timeline of the first panel steps;
writes gpurun_out/trace_<kind>_<n>_<s>.json (the kernel events)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_02056_b200 as sf  # noqa: E402
import synth  # noqa: E402


def main():
    kind, n, s = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    dt = sys.argv[4] if len(sys.argv) > 4 and not sys.argv[4].startswith("--") else "f64"
    shown = int(sys.argv[sys.argv.index("--steps-shown") + 1]) if "--steps-shown" in sys.argv else 3
    gen = {"chol": "spd_scaled", "lu": "diag_dominant", "qr": "gaussian"}[kind]
    A = synth.gen_torch(gen, n, seed=0)
    if kind != "chol":
        A = A.mT.contiguous()
    if dt == "f32":
        A = A.float()
    o1 = torch.empty_like(A); o2 = torch.empty_like(A)
    info = torch.zeros(1, dtype=torch.int64, device="cuda")

    def run():
        if kind == "chol":
            sf.chol_colmajor(n, s, A, n, o1, n, info)
        elif kind == "lu":
            sf.lu_colmajor(n, s, A, n, o1, n, info)
        else:
            sf.qr_colmajor(n, s, A, n, o1, n, o2, n, info)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run()
        torch.cuda.synchronize()
    path = f"/tmp/trace_{os.getpid()}.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    t0 = ev[0]["ts"]
    span = max(e["ts"] + e["dur"] for e in ev) - t0
    short = lambda name: name.split("(")[0].replace("void ", "").replace("sf::", "")[:60]
    print(f"== {kind} n={n} s={s} {dt}: {len(ev)} kernels, span {span / 1000:.3f} ms")
    tot = {}
    for e in ev:
        k = short(e["name"])
        c, d = tot.get(k, (0, 0.0))
        tot[k] = (c + 1, d + e["dur"])
    for k, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"  {k:60s} {c:6d} x {d / c:8.1f} us = {d / 1000:8.3f} ms")
    streams = {}
    for e in ev:
        streams.setdefault(e["args"].get("stream", -1), []).append(e)
    for sid, es in streams.items():
        busy = sum(e["dur"] for e in es)
        print(f"  stream {sid}: {len(es)} kernels, busy {busy / 1000:.3f} ms ({busy / span * 100:.0f}% of span)")
    # timeline of the first `shown` panel steps: ~ kernels until the 2*shown-th panel-looking kernel
    print("  -- timeline (us from start): start  dur  stream  kernel")
    for e in ev[: 12 * shown]:
        print(f"  {e['ts'] - t0:9.1f} {e['dur']:8.1f}  {e['args'].get('stream', -1):4}  {short(e['name'])}")
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump([{"ts": e["ts"] - t0, "dur": e["dur"], "stream": e["args"].get("stream", -1), "name": short(e["name"])}
               for e in ev], open(f"gpurun_out/trace_{kind}_{n}_{s}_{dt}.json", "w"))


if __name__ == "__main__":
    main()
