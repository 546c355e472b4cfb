#!/bin/bash
# panel64: LU column blocks staged through shared memory.  Parity, bench, probe.
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2i.log
: > $O
timeout 900 python -m pytest -q -x tests/test_parity_gpu.py -k "lu" >> $O 2>&1
timeout 600 python -m pytest -q -x tests/test_fp32_gpu.py -k "lu or chol" >> $O 2>&1
timeout 600 python -m pytest -q -x tests/test_dist_gpu.py -k "lu" >> $O 2>&1
b() { python bench.py --no-cpu --no-e2e --steps 10 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', 'upd', round(r['achieved'],2), 'panel_ms', round(r.get('panel_ms_per_step',0),2))"; }
b lu_f64_n4096_s64 "staged" >> $O
b lu_f32_n4096_s64 "staged" >> $O
b chol_f32_n16384_s512 "staged" >> $O
./calib/p64_probe | tail -4 >> $O
cat $O
