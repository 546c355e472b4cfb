#!/bin/bash
# fp32 Cholesky: fused split (SF_CHOL32_FUSED_SPLIT=1) vs split launches, same box, alternating.
mkdir -p gpurun_out/exp
O=gpurun_out/exp/r2p.log
: > $O
b() { python bench.py --no-cpu --no-e2e --steps $3 --workload $1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', round(d['ms_per_step'],3), 'ms', round(d['value']), 'panel_ms', round(r['panel_ms_per_step'],1), 'clk', d['clocks']['sm_mhz'])"; }
for rep in 1 2; do for v in 1 0; do SF_CHOL32_FUSED_SPLIT=$v b chol_f32_n16384_s512 "FUSED=$v" 10 >> $O; done; done
for rep in 1 2; do for v in 1 0; do SF_CHOL32_FUSED_SPLIT=$v b chol_f32_n65536_s512 "FUSED=$v" 3 >> $O; done; done
cat $O
