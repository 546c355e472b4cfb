#!/bin/bash
# LU two-deep lookahead: parity + bench A/B (SF_LU_LA2) + trace.
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2c.log
: > $O
timeout 900 python -m pytest -q -x tests/test_parity_gpu.py -k "lu" >> $O 2>&1
timeout 600 python -m pytest -q -x tests/test_fp32_gpu.py -k "lu" >> $O 2>&1
b() { python bench.py --no-cpu --no-e2e --steps 10 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', 'upd', round(r['achieved'],2), 'panel_ms', round(r.get('panel_ms_per_step',0),2))"; }
for v in 1 0; do SF_LU_LA2=$v b lu_f64_n4096_s64 "LA2=$v" >> $O; done
for v in 1 0; do SF_LU_LA2=$v b lu_f32_n4096_s64 "LA2=$v" >> $O; done
python tools/trace.py lu 4096 64 --steps-shown 3 > gpurun_out/exp/trace_lu_la2.log 2>&1
cat $O
