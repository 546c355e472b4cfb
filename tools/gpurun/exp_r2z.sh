#!/bin/bash
# Round-2 session 4: panel knobs again on the faster flush (cfg3 fp64): SF_CHOL_P64_MAXM, SF_PANEL_SMS.
mkdir -p gpurun_out/v; O=gpurun_out/v/knobs.log; : > $O
for v in "SF_CHOL_P64_MAXM=0" "SF_CHOL_P64_MAXM=4096" "SF_CHOL_P64_MAXM=8192" "SF_CHOL_P64_MAXM=1000000" "SF_PANEL_SMS=16" "SF_PANEL_SMS=32 SF_RESERVE_FLOPS=8e10" "SF_CHOL_P64_MAXM=0"; do
  env $v SF_BENCH_ALLOW_SHORT=1 timeout 300 python bench.py --workload chol_f64_n16384_s512 --steps 5 --warmup 3 --no-e2e --no-cpu 2>>$O | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
r = d.get('graph_replay') or d.get('replay') or {}
print('$v', 'ms', round(d['ms_per_step'], 3), 'frac', round(d['roofline']['frac'], 4), 'panel', round(d['roofline']['panel_ms_per_step'], 2), 'replay', r.get('ms_per_step'))" >> $O 2>&1
done
cat $O
