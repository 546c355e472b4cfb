"""s-sweep report: from a tools/measure_all.py sweep JSON,
per s the total, update (flush kernels), concurrent panel and exposed (unhidden) panel time,
update TF/s and % of the FP64 peak at the nominal and at the measured SM clock; then the
paper's two-term cost model, plus the s-independent classical term a GPU adds,

    T(s) = c + a * n^2 * s + b * n^3 / s          (least squares over the measured s)

- a n^2 s: the in-panel O(ns)-per-column work ("O(ns) arithmetic operations that
  always execute" per iteration, n iterations);
- b n^3 / s: n/s flushes each costing O(n^2) beyond the product ("the update of
  the submatrix in O(n^2)") — on a GPU the read-modify-write of the trailing matrix and the
  per-flush fixed cost;
- c: the classical n^3/3 flops at the tensor rate (s-independent for classical products).
The two s-dependent terms cross at s* = sqrt(b n / a), which is also the model's optimum.
    python tools/sweep_report.py profiles/r02_measure_sweep.json > profiles/r02_sweep_cfg3.json
"""
import json
import math
import sys

import numpy as np


def main():
    src = json.load(open(sys.argv[1]))
    rows = src["sweep"] if isinstance(src, dict) else src
    peak = json.load(open("calib/peaks_fp64_tf32.json"))["fp64_dmma_tflops"]
    nominal_mhz = 1965.0
    n = rows[0]["n"]
    out = []
    for r in rows:
        ck = r.get("clocks") or {}
        mhz = ck.get("sm_mhz") or nominal_mhz
        upd_tf = r.get("update_tflops")
        out.append({"s": r["s"], "ms": r["ms"], "update_ms": r["update_ms"], "panel_ms_concurrent": r["panel_ms"],
                    "exposed_panel_ms": r.get("exposed_panel_ms", max(0.0, r["eager_profiled_ms"] - r["update_ms"])),
                    "update_tflops": upd_tf, "pct_peak_update_nominal": upd_tf / peak if upd_tf else None,
                    "pct_peak_update_at_measured_clock": (upd_tf / (peak * mhz / nominal_mhz)) if upd_tf else None,
                    "sm_mhz": mhz, "classical_gflops": n ** 3 / 3 / (r["ms"] * 1e-3) / 1e9})
    s = np.array([o["s"] for o in out], float)
    t = np.array([o["ms"] for o in out], float)
    X = np.stack([np.ones_like(s), n * n * s, n ** 3 / s], 1)
    coef, *_ = np.linalg.lstsq(X, t, rcond=None)
    c, a, b = (float(x) for x in coef)
    fit = X @ coef
    for o, f in zip(out, fit):
        o["model_ms"] = float(f)
    s_star = math.sqrt(b * n / a) if a > 0 and b > 0 else None
    report = {"n": n, "gpu": src.get("gpu") if isinstance(src, dict) else None, "peak_tflops": peak,
              "points": out,
              "model": {"form": "T(s) = c + a n^2 s + b n^3 / s  [ms]", "c_ms": c, "a_ms": a, "b_ms": b,
                        "rms_residual_ms": float(np.sqrt(np.mean((fit - t) ** 2))),
                        "crossover_s": s_star,
                        "panel_term_ms_at_crossover": a * n * n * s_star if s_star else None,
                        "note": "a n^2 s = b n^3 / s at s*; the measured best s is listed below"},
              "best_measured_s": int(s[np.argmin(t)])}
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
