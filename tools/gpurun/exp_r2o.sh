#!/bin/bash
# fp32 Cholesky: the 3xTF32 split written by the panel64 leaves (no split launches on the panel chain).
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2o.log
: > $O
timeout 900 python -m pytest -q -x tests/test_fp32_gpu.py >> $O 2>&1
timeout 600 python -m pytest -q -x tests/test_dist_gpu.py -k "fp32" >> $O 2>&1
b() { python bench.py --no-cpu --no-e2e --steps $3 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', round(d['value']), 'panel_ms', round(r['panel_ms_per_step'],1), 'clk', d['clocks']['sm_mhz'])"; }
b chol_f32_n16384_s512 fused 10 >> $O
b chol_f32_n65536_s512 fused 3 >> $O
cat $O
