#!/bin/bash
# f1 at the paper's depth: Strassen-Winograd 1-3 levels — parity and bench at cfg2/cfg4/cfg3/cfg5.
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2n.log
: > $O
timeout 1200 python -m pytest -q -x tests/test_strassen_gpu.py >> $O 2>&1
b() { python bench.py --no-cpu --no-e2e --steps $3 $4 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', '$2', round(d['ms_per_step'],3), 'ms', round(d['value']))"; }
for lv in 1 2 3; do b lu_f64_n4096_s64 "L$lv min1024" 5 "--strassen 1024 --strassen-levels $lv" >> $O; done
for lv in 1 2 3; do b qr_f64_n8192_s128 "L$lv min2048" 3 "--strassen 2048 --strassen-levels $lv" >> $O; done
for lv in 1 2 3; do b chol_f64_n16384_s512 "L$lv min4096" 3 "--strassen 4096 --strassen-levels $lv" >> $O; done
for lv in 1 2; do b chol_f64_n65536_s512 "L$lv min8192" 3 "--strassen 8192 --strassen-levels $lv" >> $O; done
cat $O
