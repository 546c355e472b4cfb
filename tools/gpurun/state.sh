#!/bin/bash
# Current state: GPU suite + smoke + one bench line per workload (logs under gpurun_out/).
mkdir -p gpurun_out
O=gpurun_out/state
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x --durations=20 > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for w in chol_f64_n65536_s512 lu_f64_n4096_s64 qr_f64_n8192_s128 chol_f64_n16384_s512 chol_f32_n65536_s512 lu_f32_n4096_s64 chol_f64_n256_s16; do
  timeout 600 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err
done
tail -3 $O/pytest_gpu.log; cat $O/smoke.log | tail -2
for f in $O/bench_*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print(d['value'], d['unit'], d['ms_per_step'], 'roof', d.get('roofline',{}).get('frac'), 'e2e', d.get('e2e',{}).get('value'), d.get('clocks',{}).get('sm_mhz'))
" 2>&1 | tail -1; done
