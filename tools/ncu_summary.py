"""Summarise ncu output for profiles/ (development tool).

    python tools/ncu_summary.py rep  <file.ncu-rep>        # --set full capture: per-kernel key metrics
    python tools/ncu_summary.py launches <launches.csv>    # gpu__time_duration launch list: per-kernel totals
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active % (of active cycles)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (of elapsed)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst executed %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')}  grid {d.get('Grid Size')} block {d.get('Block Size')}")
        for k, name in KEYS:
            if k in d and d[k] != "":
                print(f"   {name:42s} {d[k]} {u.get(k, '')}")
        st = {}
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and v:
                try:
                    st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v)
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
        print("   top stall reasons (share of samples): " + ", ".join(f"{k} {v / tot:.2f}" for k, v in top))


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            agg[r[ki].split("(")[0][:70]].append(float(r[vi]))
        except ValueError:
            pass
    tot = sum(sum(v) for v in agg.values())
    # the library's own kernels (namespace sf::) vs everything else in the process (torch's input
    # generation, e.g. the G G^T product, runs once outside the timed region)
    lib = sum(sum(v) for k, v in agg.items() if "sf::" in k)
    print("serialised, cold-cache durations (ncu); 'lib share' = share among the library's kernels")
    print(f"{'kernel':72s} {'launches':>8s} {'total us':>10s} {'avg us':>8s} {'share':>6s} {'lib share':>9s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        ls = f"{sum(v) / lib:9.3f}" if ("sf::" in k and lib) else f"{'-':>9s}"
        print(f"{k:72s} {len(v):8d} {sum(v) / 1e3:10.1f} {sum(v) / len(v) / 1e3:8.2f} {sum(v) / tot:6.3f} {ls}")
    print(f"{'TOTAL':72s} {sum(len(v) for v in agg.values()):8d} {tot / 1e3:10.1f}")
    print(f"{'TOTAL sf:: kernels':72s} {sum(len(v) for k, v in agg.items() if 'sf::' in k):8d} {lib / 1e3:10.1f}")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
