#!/usr/bin/env python
"""bench.py — step-s factorization throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--s S] [--impl reference]

A "step" is one complete factorization (every panel + every flush of Alg. 1/2/3 —
SURVEY.md §8 rows a1..a8) of the workload's synthetic matrix, out of place (A stays
pristine, so no restore is needed between steps; A is 2.1 GB > the 126 MB L2, so nothing
survives in L2 between steps).  Metric: classical-count GFLOP/s (n^3/3 Cholesky, 2n^3/3 LU,
4n^3/3 QR), whole job = sum over ranks / max-over-ranks device time.

Default workload: BASELINE.json configs[4] fp64 — Cholesky n=65536, s=512, A = G G^T/n + I —
the config the metric is quoted on at 1/2/4/8 B200 (BASELINE.json:2, 11) and on which
north_star sets the multi-GPU target; it fits one GPU (34 GB).  N=1 runs the single-GPU
driver (chol_factor); N>1 (torchrun, one process per GPU) runs the block-cyclic driver
(chol_factor_dist: s-column panels dealt round-robin, each factored panel broadcast by
NCCL) on the same problem: strong scaling, value = one factorization per step / time.
configs[2] (n=16384, the s-sweep / roofline config) and the others are selectable with
--workload (they are also parity-test cases); DESIGN.md §6.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (the only
reference that exists: PAPER.md's own code is not available) on a bounded sample.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (kind, n, s, generator, dtype, BASELINE config)
    "chol_f64_n16384_s512": ("chol", 16384, 512, "spd_scaled", "f64", "configs[2]"),
    "chol_f64_n256_s16": ("chol", 256, 16, "spd_shift", "f64", "configs[0]"),
    "lu_f64_n4096_s64": ("lu", 4096, 64, "diag_dominant", "f64", "configs[1]"),
    "qr_f64_n8192_s128": ("qr", 8192, 128, "gaussian", "f64", "configs[3]"),
    "chol_f64_n65536_s512": ("chol", 65536, 512, "spd_scaled", "f64", "configs[4]"),
    "chol_f32_n65536_s512": ("chol", 65536, 512, "spd_scaled", "f32", "configs[4]"),
    "chol_f32_n16384_s512": ("chol", 16384, 512, "spd_scaled", "f32", "configs[2] in fp32"),
    "lu_f32_n4096_s64": ("lu", 4096, 64, "diag_dominant", "f32", "configs[1] in fp32 (f4)"),
    "qr_f32_n8192_s128": ("qr", 8192, 128, "gaussian", "f32", "configs[3] in fp32 (f4)"),
}
DEFAULT = "chol_f64_n65536_s512"
CALIB = os.path.join(ROOT, "calib", "peaks_fp64_tf32.json")
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")


def classical_flops(kind, n):
    return {"chol": n ** 3 / 3.0, "lu": 2.0 * n ** 3 / 3.0, "qr": 4.0 * n ** 3 / 3.0}[kind]


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1])); pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm_sorted = sorted(sm)
        return {"sm_mhz": sm_sorted[len(sm) // 2], "sm_max_mhz": max(mx), "power_w_max": max(pw),
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- oracle sample

def oracle_executed_flops(kind, n, s, K):
    """Flops the restricted oracle run executes for the first K columns (exact loop counts)."""
    f = 0.0
    for c in range(K):
        z = c - (c % s)
        if c > 0 and c % s == 0:   # flush at c (z_prev = c - s)
            w = s
            if kind == "chol":
                f += (K - c) * (n - c) * (2.0 * w + 1)
            elif kind == "lu":
                f += ((n - c) ** 2 - (n - K) ** 2) * (2.0 * w + 1)
            else:
                f += 2.0 * n * w * (K - c) + (2.0 * w + 1) * n * (K - c)
        d = c - z
        if kind == "chol":
            f += 2 * d + 1 + (n - c - 1) * (2.0 * d + 1)
        elif kind == "lu":
            f += (n - c) * (2.0 * d) + (n - c) * (2.0 * d + 1)
        else:
            f += d * 4.0 * n + 3.0 * n
    if kind == "qr":
        f += 2.0 * K * n * n
    return f


def oracle_sample(kind, n, s, A_host_cols, K, A_full=None):
    """Run the oracle restricted to K columns; returns (seconds, flops, threads)."""
    import oracle
    t0 = time.perf_counter()
    if kind == "chol":
        _, info = oracle.chol(A_host_cols, s, kcols=K)
    elif kind == "lu":
        _, _, info = oracle.lu(A_full, s, kcols=K)
    else:
        _, _, info, _ = oracle.qr(A_full, s, kcols=K)
    dt = time.perf_counter() - t0
    assert info == 0, f"oracle failed at column {info}"
    return dt, oracle_executed_flops(kind, n, s, K), oracle.max_threads()


def host_inputs(kind, gen, n, seed, K, dev_A=None):
    """Host copies the oracle needs (same bytes as the device run when dev_A is given)."""
    import numpy as np
    if dev_A is not None:
        if kind == "chol":   # symmetric: device buffer column-major == logical A; first K columns
            return np.asfortranarray(dev_A[:K, :].double().cpu().numpy().T), None
        full = dev_A.double().cpu().numpy().T.copy()   # buffer -> logical matrix
        return None, full
    import synth
    A = synth.gen_numpy(gen, n, seed)
    return (np.asfortranarray(A[:, :K]) if kind == "chol" else None), A


def sample_cols(kind, n, s):
    # ~10-30 s of oracle work on a 16-core host; at least 2s columns, so the sample contains a
    # flush (the work that dominates the full run) and not only the first panel's recurrences
    k = {"chol": 2048 if n >= 8192 else n, "lu": 512 if n > 2048 else n, "qr": 96 if n > 2048 else n}[kind]
    return min(n, max(k, 2 * s))


# ----------------------------------------------------------------------------- main

def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT, choices=sorted(WORKLOADS))
    ap.add_argument("--s", type=int, default=None, help="override the step size (s-sweep)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dist", action="store_true", help="use the distributed (block-cyclic) driver even at N=1")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--push", action="store_true",
                    help="multi-GPU panel transport: device-initiated push (f3, sf_comm_set_push) instead of ncclBroadcast")
    ap.add_argument("--loopback", type=int, default=0,
                    help="test mode: run the distributed driver with G ranks emulated on this one GPU")
    ap.add_argument("--strassen-levels", type=int, default=1, help="Strassen recursion depth with --strassen (1-3)")
    ap.add_argument("--strassen", type=int, default=0, metavar="MIN_DIM",
                    help="f1: one Strassen-Winograd level in fp64 flushes with sides >= MIN_DIM (0 = off)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    kind, n, s, gen, dtype, cfgname = WORKLOADS[args.workload]
    s = args.s or s
    K = max(1, oracle_k(kind, n, s, target_flops=2e10))
    dev_A = None
    try:
        import torch
        if torch.cuda.is_available():
            import synth
            dev_A = synth.gen_torch(gen, n, args.seed) if n > 4096 else None
            if dev_A is not None and kind != "chol":
                dev_A = dev_A.mT.contiguous()
            if dev_A is not None and dtype == "f32":
                dev_A = dev_A.float()      # the fp32 workload's input, rounded (P9)
    except Exception:
        dev_A = None
    Acols, Afull = host_inputs(kind, gen, n, args.seed, K, dev_A)
    for _ in range(args.warmup):
        oracle_sample(kind, n, s, Acols, K, Afull)
    tot_t, tot_f, thr = 0.0, 0.0, 1
    for _ in range(args.steps):
        dt, fl, thr = oracle_sample(kind, n, s, Acols, K, Afull)
        tot_t += dt; tot_f += fl
    value = tot_f / tot_t / 1e9
    sample = (f"oracle (oracle/stepfact_oracle.c, -O2, OpenMP) restricted to the first {K} of {n} columns "
              f"of the {args.workload} matrix per step; value = executed flops / time")
    line = {"impl": "reference", "metric": "factorization GFLOP/s (classical count) and % of FP64 tensor peak",
            "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": args.workload, "kind": kind, "n": n, "s": s, "baseline_config": cfgname,
                       "generator": gen, "seed": args.seed, "sample_cols": K},
            "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": thr, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def oracle_k(kind, n, s, target_flops=6e10):
    """Columns of the restricted oracle run for cpu_baseline: ~10-30 s on the host cores."""
    if kind != "chol":
        return sample_cols(kind, n, s)
    K = 64
    while K < n and oracle_executed_flops(kind, n, s, min(n, K * 2)) <= target_flops:
        K *= 2
    return min(n, max(K, 2 * s))   # at least one flushed panel (cfg5: 1024 columns, ~6.8e10 flops)


def make_inputs(torch, sf, synth, kind, gen, n, s, seed, ws, rank, use_dist):
    """Column-major device input: the full buffer (single-GPU driver) or this rank's local
    block-cyclic columns (distributed driver)."""
    if not use_dist:
        Alog = synth.gen_torch(gen, n, seed) if n > 4096 else torch.from_numpy(synth.gen_numpy(gen, n, seed)).cuda()
        return Alog if kind == "chol" else Alog.mT.contiguous()   # column-major buffer of A
    cols = sf.global_columns(n, s, ws, rank)
    if kind == "chol" and gen in ("spd_scaled", "spd_shift") and n > 4096:
        return synth.gen_torch_cols(gen, n, seed, cols)
    Alog = synth.gen_torch(gen, n, seed) if n > 4096 else torch.from_numpy(synth.gen_numpy(gen, n, seed)).cuda()
    B = Alog if kind == "chol" else Alog.mT.contiguous()
    del Alog
    X = B[cols].contiguous()
    del B
    return X


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import paper_1812_02056_b200 as sf
    import synth

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kind, n, s, gen, dtype, cfgname = WORKLOADS[args.workload]
    s = args.s or s
    assert args.warmup >= 3 or os.environ.get("SF_BENCH_ALLOW_SHORT"), "timing rules need >= 3 warm-up steps"
    use_dist = ws > 1 or args.dist or args.loopback > 0
    stream = torch.cuda.current_stream()

    # ---- communicator (multi-GPU: block-cyclic panels, NCCL broadcast).
    # --loopback G (test mode): one process drives G emulated ranks on this GPU.
    comm = None
    G = ws
    if args.loopback > 0:
        assert ws == 1, "--loopback is a single-process test mode"
        G = args.loopback
        comm = sf.Comm.loopback(G)
    elif use_dist:
        uid = [sf.unique_id() if rank == 0 else None]
        if ws > 1:
            dist.broadcast_object_list(uid, src=0)
        comm = sf.Comm.nccl(ws, rank, uid[0])
    if comm is not None and args.push:
        comm.set_push(True)
    my_ranks = comm.local_ranks if comm is not None else [rank]

    # ---- inputs (synthetic, seeded, same recipe on every rank; A stays pristine: out of place)
    seed = args.seed
    As = [make_inputs(torch, sf, synth, kind, gen, n, s, seed, G, r, use_dist) for r in my_ranks]
    if dtype == "f32":      # fp32 path: the fp64-generated matrix rounded to fp32 (P9)
        As = [a.float() for a in As]
    A = As[0]
    dcode = sf.SF_F32 if dtype == "f32" else sf.SF_F64
    ld = n
    infos = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in my_ranks]
    info = infos[0]
    outs1 = [torch.zeros_like(a) for a in As]
    outs2 = [torch.zeros_like(a) for a in As] if kind == "qr" else None
    out1 = outs1[0]
    out2 = outs2[0] if outs2 else None
    torch.cuda.synchronize()

    def step():
        if use_dist:
            if kind == "chol":
                sf.chol_dist(comm, n, s, As, outs1, ld, infos, dtype=dcode, stream=stream)
            elif kind == "lu":
                sf.lu_dist(comm, n, s, As, outs1, ld, infos, stream=stream)
            else:
                sf.qr_dist(comm, n, s, As, outs1, outs2, ld, infos, stream=stream)
        elif kind == "chol":
            sf.chol_colmajor(n, s, A, n, out1, n, info, dtype=dcode, stream=stream)
        elif kind == "lu":
            sf.lu_colmajor(n, s, A, n, out1, n, info, stream=stream)
        else:
            sf.qr_colmajor(n, s, A, n, out1, n, out2, n, info, stream=stream)

    if args.strassen:
        sf.set_strassen(args.strassen_levels, args.strassen)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if int(info.item()) != 0:
        raise RuntimeError(f"factorization failed at column {int(info.item())}")

    # ---- timed region
    clocks = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)                               # let the sampler start
    sf.profile_enable(True)
    sf.profile_collect()
    l0 = sf.launch_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    l1 = sf.launch_counter()
    prof = sf.profile_collect()
    prof_union = sf.profile_union()
    sf.profile_enable(False)
    ck = clocks.stop()
    ms = e0.elapsed_time(e1)
    if int(info.item()) != 0:
        raise RuntimeError(f"factorization failed at column {int(info.item())}")
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    t_max = float(t_max.item())
    flops = classical_flops(kind, n)
    # whole job: ONE factorization per step, shared by all ranks (strong scaling)
    value = args.steps * flops / (t_max * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (the trailing-update GEMM/SYRK launches)
    peaks = json.load(open(CALIB)) if os.path.exists(CALIB) else {}
    upd_ms, upd_n, upd_fl = prof["update"]
    pan_ms, pan_n, _ = prof["panel"]
    qr_ms, qr_n, qr_fl = prof["qr_r"]
    achieved = upd_fl / (upd_ms * 1e-3) / 1e12 if upd_ms > 0 else None
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        traffic = json.load(open(tr_path)).get(args.workload)
    if dtype == "f32" and kind != "chol" and achieved:
        achieved *= 3.0   # LU / QR fp32 drivers count useful flops; 3xTF32 executes three products
    if dtype == "f32":
        # TF32 dense peak = measured bf16 (sustained: the kernel runs inside a long step) x
        # the nominal tf32/bf16 ratio 1.1/2.25 (B200_PROFILING.md)
        mp = json.load(open(MEASURED)) if os.path.exists(MEASURED) else {}
        bf16 = mp.get("bf16_tflops_sustained") or 1400.0
        peak = bf16 * 1.1 / 2.25
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": (achieved / peak) if (achieved and peak) else None, "traffic": traffic,
                    "kernel": "gemm_tf32x3_pair_persist_kernel (flush update, tcgen05.mma.cta_group::2 kind::tf32, "
                              "3xTF32: K' = 3s)",
                    "flops_counted": "tensor flops executed = 3 x useful (hi.hi + hi.lo + lo.hi)",
                    "useful_achieved": achieved / 3.0 if achieved else None,
                    "peak_source": ("measured: MEASURED_PEAKS.json bf16_tflops_sustained x 1.1/2.25 (nominal "
                                    "tf32/bf16 ratio)" if mp else "fallback 1400 x 1.1/2.25")}
    else:
        peak = peaks.get("fp64_dmma_tflops")
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": (achieved / peak) if (achieved and peak) else None, "traffic": traffic,
                    "kernel": "gemm_f64v2_kernel (flush update, DMMA.8x8x4, 64x64 tiles, bulk-reduce epilogue)"
                              + (", rank 0" if ws > 1 else ""),
                    "peak_source": "measured: calib/peaks_fp64_tf32.json fp64_dmma_tflops (DMMA microbenchmark, "
                                   "this pool's B200); MEASURED_PEAKS.json has no fp64 entry"}
    # wall-clock view: the flush flops over the union of the flush regions (LU's lookahead runs
    # flush parts on two streams at once, which the per-launch average above counts twice)
    upd_wall = prof_union.get("update", 0.0)
    if upd_wall > 0 and achieved:
        roofline["achieved_wall"] = achieved * upd_ms / upd_wall
        roofline["frac_wall"] = roofline["achieved_wall"] / peak if peak else None
        roofline["update_wall_ms_per_step"] = upd_wall / args.steps
    roofline.update({"launches_per_step": upd_n / args.steps if args.steps else None,
                     "avg_launch_ms": upd_ms / upd_n if upd_n else None,
                     "flops_per_launch": upd_fl / upd_n if upd_n else None,
                     "update_share_of_step": upd_ms / ms if ms else None,
                     "panel_ms_per_step": pan_ms / args.steps, "qr_r_ms_per_step": qr_ms / args.steps,
                     # the panels' column recurrences are sequential: device time per column
                     # (summed over the panel launches of a step, lookahead concurrency included)
                     "panel_us_per_column": pan_ms / args.steps * 1e3 / n})
    # ---- per rank (N > 1): where each rank's step went, so the scaling curve explains itself
    bc_ms, bc_n, bc_bytes = prof.get("bcast", (0.0, 0, 0.0))
    if use_dist:   # rank 0's panel exchange (broadcast, or the device wait of the push transport)
        roofline["bcast_ms_per_step"] = bc_ms / args.steps
    if ws > 1:
        mine = torch.tensor([ms, upd_ms, pan_ms, bc_ms, bc_bytes], dtype=torch.float64, device="cuda")
        allr = [torch.zeros_like(mine) for _ in range(ws)]
        dist.all_gather(allr, mine)
        per_rank = [{"rank": r, "ms_per_step": float(v[0]) / args.steps,
                     "flush_ms_per_step": float(v[1]) / args.steps, "panel_ms_per_step": float(v[2]) / args.steps,
                     "bcast_ms_per_step": float(v[3]) / args.steps,
                     "bcast_gb_per_step": float(v[4]) / args.steps / 1e9} for r, v in enumerate(allr)]
    else:
        per_rank = None
    # panel kernels: minimal HBM bytes (read + write each panel once: elt * 2 * (n - z) * w,
    # QR: all n rows) over their device time (they run concurrently on the lookahead stream)
    elt = 4 if dtype == "f32" else 8
    pbytes = sum(2 * elt * ((n if kind == "qr" else n - z) * min(s, n - z)) for z in range(0, n, s))
    roofline["panel_hbm_gbs"] = (pbytes / (pan_ms / args.steps * 1e-3) / 1e9) if pan_ms > 0 else None

    # ---- the same step as users repeat it: profiling off, so the library replays its captured
    #      CUDA graph from the second identical call on (the timed region above records
    #      per-launch events and therefore runs eagerly).  Reported beside `value`, not in it.
    replay = None
    if not use_dist and t_max / args.steps < 200.0:   # launch-bound sizes only (cfg1-cfg4)
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        r0 = torch.cuda.Event(enable_timing=True); r1 = torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(args.steps):
            step()
        r1.record(stream)
        torch.cuda.synchronize()
        rms = r0.elapsed_time(r1) / args.steps
        replay = {"ms_per_step": rms, "value": flops / (rms * 1e-3) / 1e9, "unit": "GFLOP/s",
                  "note": "CUDA-graph replay (the library's behaviour on repeated identical calls), "
                          "no per-launch events; measured after the timed region"}

    # ---- end to end through the public API with HOST buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e and not args.loopback:
        ke = max(1, min(args.steps, args.e2e_steps))
        nbytes = A.numel() * A.element_size()
        hA = A.cpu().pin_memory()
        h1 = torch.empty_like(hA).pin_memory()
        h2 = torch.empty_like(hA).pin_memory() if kind == "qr" else None
        if use_dist:
            dA = torch.empty_like(A)

            def hstep():
                dA.copy_(hA, non_blocking=True)
                step_out = (out1, out2)
                if kind == "chol":
                    sf.chol_dist(comm, n, s, [dA], [out1], ld, [info], dtype=dcode, stream=stream)
                elif kind == "lu":
                    sf.lu_dist(comm, n, s, [dA], [out1], ld, [info], stream=stream)
                else:
                    sf.qr_dist(comm, n, s, [dA], [out1], [out2], ld, [info], stream=stream)
                h1.copy_(step_out[0], non_blocking=True)
                if kind == "qr":
                    h2.copy_(step_out[1], non_blocking=True)
                torch.cuda.synchronize()
                assert int(info.item()) == 0
            api = f"{kind}_factor_dist (C ABI) with torch pinned host<->device copies per rank"
        else:
            def hstep():
                if kind == "chol":
                    _, inf = sf.chol_host(hA, s, h1, dtype=dcode)
                elif kind == "lu":
                    _, inf = sf.lu_host(hA, s, h1)
                else:
                    _, _, inf = sf.qr_host(hA, s, h1, h2)
                assert inf == 0
            api = f"{kind}_factor_host (C ABI, pinned host buffers)"
        hstep()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            hstep()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        bb = torch.tensor([float(nbytes)], dtype=torch.float64, device="cuda")
        if ws > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dist.all_reduce(bb, op=dist.ReduceOp.SUM)
        dt = float(tt.item()); tot_bytes = int(bb.item())
        if kind == "chol" and not use_dist:
            # chol_factor_host moves the lower triangle panel by panel, both directions
            tot_bytes = sum((n - z) * min(s, n - z) for z in range(0, n, s)) * A.element_size()
        e2e = {"value": ke * flops / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": tot_bytes,
               "d2h_bytes_per_step": tot_bytes * (2 if kind == "qr" else 1), "steps": ke, "api": api}
        del hA, h1, h2

    # ---- CPU oracle beside it (rank 0, N=1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        K = oracle_k(kind, n, s)
        Acols, Afull = host_inputs(kind, gen, n, seed, K, dev_A=A if n > 4096 else None)
        dt, fl, thr = oracle_sample(kind, n, s, Acols, K, Afull)
        cpu = {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": thr, "kind": "oracle",
               "sample": f"oracle restricted to the first {K} of {n} columns of this workload's matrix "
                         f"({fl:.3g} executed flops in {dt:.1f} s); full-run time extrapolates to "
                         f"{flops / (fl / dt) / 3600:.2f} h"}

    if rank == 0:
        xport = ("device-initiated panel push (f3: symmetric-window stores + device flags)" if args.push
                 else "NCCL panel broadcast")
        par = f"block-cyclic s-column panels over {ws} GPU(s), {xport}" if use_dist else "single GPU"
        if args.loopback:
            par = (f"LOOPBACK TEST MODE: {G} ranks of the block-cyclic schedule emulated on 1 GPU "
                   f"({'device-initiated push' if args.push else 'device-copy broadcast'}; not a scaling measurement)")
        line = {"metric": "factorization GFLOP/s (classical count) and % of FP64 tensor peak",
                "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": {"workload": args.workload, "kind": kind, "n": n, "s": s, "baseline_config": cfgname,
                           "generator": gen, "seed": args.seed, "parallelism": par,
                           **({"strassen": {"levels": args.strassen_levels, "min_dim": args.strassen,
                                            "note": "roofline.achieved counts classical-equivalent flops"}}
                              if args.strassen else {}),
                           "l2": f"inputs larger than L2 ({A.numel() * A.element_size() / 1e9:.2f} GB per rank "
                                 "> 126 MB); out-of-place factorization, A re-read from HBM every step"},
                "pct_tensor_peak": (value / ws / 1e3 / peak) if peak else None,
                "pct_peak_kind": ("classical useful GFLOP/s per GPU / TF32 dense peak" if dtype == "f32"
                                  else "classical GFLOP/s per GPU / FP64 tensor (DMMA) peak"),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "graph_replay": replay,
                "gpu_launches": int(l1 - l0), "clocks": ck,
                **({"per_rank": per_rank} if per_rank else {})}
        print(json.dumps(line), flush=True)
    if comm is not None:
        torch.cuda.synchronize()
        comm.destroy()
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
