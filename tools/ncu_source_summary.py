"""Summarise an `ncu --page source --csv --print-source sass` export: stall samples per
reason, and the SASS regions (address ranges) where the samples fall."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_")]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
num = lambda x: float(x) if x not in ("", None) else 0.0
tot = {c: sum(num(r[ix[c]]) for r in data) for c in stall_cols}
allsum = sum(tot.values())
print(f"{len(data)} SASS lines, {allsum:.0f} stall samples")
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {c:28s} {v:8.0f} {v / max(allsum, 1) * 100:5.1f}%")
# windows of 256 instructions
W = int(sys.argv[2]) if len(sys.argv) > 2 else 512
print(f"-- samples per {W}-instruction window (top 12), with the dominant opcode / stall")
wins = []
for w0 in range(0, len(data), W):
    seg = data[w0:w0 + W]
    s = sum(num(r[ix["Warp Stall Sampling (All Samples)"]]) for r in seg)
    ex = sum(num(r[ix["Instructions Executed"]]) for r in seg)
    st = {c: sum(num(r[ix[c]]) for r in seg) for c in stall_cols}
    top = max(st.items(), key=lambda x: x[1])
    ops = {}
    for r in seg:
        op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[ix["Source"]].split()[1]
        ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + 1
    wins.append((s, w0, ex, top, sorted(ops.items(), key=lambda x: -x[1])[:3]))
for s, w0, ex, top, ops in sorted(wins, reverse=True)[:12]:
    print(f"  [{w0:6d}..{w0 + W:6d}) samples {s:7.0f} executed {ex:9.0f}  top stall {top[0]} {top[1]:.0f}  ops {ops}")
