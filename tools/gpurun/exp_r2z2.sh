#!/bin/bash
# Round-2 session 4: LU cfg2 switches again with the slice loader (SF_GROUPED_SHORTK8, SF_DMMA_CHUNK, SF_DMMA_SHORTK).
mkdir -p gpurun_out/v; O=gpurun_out/v/lu_knobs.log; : > $O
for v in "SF_X=0" "SF_GROUPED_SHORTK8=1" "SF_DMMA_CHUNK=1" "SF_DMMA_SHORTK=5" "SF_X=0"; do
  env $v SF_BENCH_ALLOW_SHORT=1 timeout 300 python bench.py --workload lu_f64_n4096_s64 --steps 10 --warmup 3 --no-e2e --no-cpu 2>>$O | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
r = d.get('graph_replay') or d.get('replay') or {}
print('$v', 'ms', round(d['ms_per_step'], 3), 'frac', round(d['roofline']['frac'], 4), 'panel', round(d['roofline']['panel_ms_per_step'], 2), 'replay', r.get('ms_per_step'))" >> $O 2>&1
done
cat $O
