#!/bin/bash
# Round-2 session 4: QR cfg4 switches again with the slice loader (SF_QR_EARLY_R, SF_MGS_COOP).
mkdir -p gpurun_out/v; O=gpurun_out/v/qr_knobs.log; : > $O
for v in "SF_X=0" "SF_QR_EARLY_R=1" "SF_MGS_COOP=0" "SF_X=0"; do
  env $v SF_BENCH_ALLOW_SHORT=1 timeout 300 python bench.py --workload qr_f64_n8192_s128 --steps 5 --warmup 3 --no-e2e --no-cpu 2>>$O | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
r = d.get('graph_replay') or d.get('replay') or {}
print('$v', 'ms', round(d['ms_per_step'], 3), 'frac', round(d['roofline']['frac'], 4), 'panel', round(d['roofline']['panel_ms_per_step'], 2), 'qr_r', round(d['roofline']['qr_r_ms_per_step'], 2), 'replay', r.get('ms_per_step'))" >> $O 2>&1
done
cat $O
